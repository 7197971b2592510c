mkdir -p gpurun_out
for cs in "2 32 2 2048 1 q 1" "2 8 8 2048 1 q 1" "2 32 2 2048 2 q 0"; do
  echo "== case $cs" >> gpurun_out/r2g_debug.txt
  timeout 30 python tools/abort_debug.py $cs >> gpurun_out/r2g_debug.txt 2>&1
  echo "rc=$?" >> gpurun_out/r2g_debug.txt
done
cat gpurun_out/r2g_debug.txt
timeout 900 python -m pytest tests/test_gpu_attention.py -m gpu -q -rf -x --timeout 150 --timeout-method thread > gpurun_out/r2g_attn.txt 2>&1
echo "attn rc=$?"; tail -3 gpurun_out/r2g_attn.txt
timeout 600 python tools/attn_graph_sweep.py > gpurun_out/r2g_attn_sweep.txt 2>&1; tail -20 gpurun_out/r2g_attn_sweep.txt
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r2g_bench.json').read().split('\n')[0]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['rows_recomputed']);print({k:v['us'] for k,v in d['kernels'].items()});print(d['configs']['c1_attention_op_b1_l1024'])"
for inj in 0 5; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 --inject $inj > gpurun_out/r2g_glm_inj$inj.json 2>&1
done
grep -o '"ms_per_step": [0-9.]*\|"attention_async(+recompute)": {[^}]*}' gpurun_out/r2g_glm*.json
timeout 900 python tools/conv_sweep.py > gpurun_out/r2g_conv_sweep.txt 2>&1; tail -3 gpurun_out/r2g_conv_sweep.txt
