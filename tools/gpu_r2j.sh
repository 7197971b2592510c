mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_configs.py -m gpu -q -rf -x --timeout 150 --timeout-method thread > gpurun_out/r2j_attn.txt 2>&1
echo "attn rc=$?"; tail -2 gpurun_out/r2j_attn.txt
timeout 600 python tools/attn_graph_sweep.py 2>&1 | grep '"kv_prefetch": true' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(f\"{d['shape']:28s} {d['us']:8.2f} us {d['frac']:.3f}\")"
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r2j_bench.json').read().split('\n')[0]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['rows_recomputed']);print({k:v['us'] for k,v in d['kernels'].items()});print(d['configs']['c1_attention_op_b1_l1024']['us'])"
