mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_configs.py -m gpu -q -rf -x --timeout 150 --timeout-method thread > gpurun_out/r2i_attn.txt 2>&1
echo "attn rc=$?"; tail -3 gpurun_out/r2i_attn.txt
for ab in 2 0; do
  for cs in "2 32 2 2048 4 q" "2 8 8 2048 2 k" "1 32 32 1024 0 q"; do
    echo "== ABORT=$ab case $cs" >> gpurun_out/r2i_debug.txt
    FDPP_ATTN_ABORT=$ab timeout 30 python tools/abort_debug.py $cs >> gpurun_out/r2i_debug.txt 2>&1
    echo "rc=$?" >> gpurun_out/r2i_debug.txt
  done
done
grep -c OK gpurun_out/r2i_debug.txt; grep "rc=\|MISM" gpurun_out/r2i_debug.txt | sort | uniq -c
timeout 600 python tools/attn_graph_sweep.py 2>&1 | grep '"kv_prefetch": true' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(f\"{d['shape']:28s} {d['us']:8.2f} us {d['frac']:.3f}\")"
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r2i_bench.json').read().split('\n')[0]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['rows_recomputed']);print({k:v['us'] for k,v in d['kernels'].items()});print(d['configs']['c1_attention_op_b1_l1024']['us'])"
for inj in 0 5; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 --inject $inj > gpurun_out/r2i_glm_inj$inj.json 2>&1
done
grep -o '"ms_per_step": [0-9.]*\|"attention_async(+recompute)": {[^}]*}' gpurun_out/r2i_glm*.json
