mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.txt 2>&1; tail -1 gpurun_out/r2z_smoke.txt
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method thread --durations=5 > gpurun_out/r2z_gputest.txt 2>&1
echo "gpu tests rc=$?"; tail -2 gpurun_out/r2z_gputest.txt
timeout 900 python bench.py > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r2z_bench.json').read().split('\n')[0]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['clocks'],d['configs']['c1_attention_op_b1_l1024']['us'])"
timeout 900 python bench.py --impl reference > gpurun_out/r2z_ref.json 2> gpurun_out/r2z_ref.err; echo "ref rc=$?"
