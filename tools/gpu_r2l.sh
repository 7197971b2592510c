mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_configs.py tests/test_gpu_decode.py -m gpu -q -rf -x --timeout 150 --timeout-method thread > gpurun_out/r2l_attn.txt 2>&1
echo "attn rc=$?"; tail -2 gpurun_out/r2l_attn.txt
for env in "FDPP_ATTN_PUSH=1" "FDPP_ATTN_PUSH=0"; do
  echo "== $env"
  env $env timeout 600 python tools/attn_graph_sweep.py 2>&1 | grep '"kv_prefetch": true' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(f\"{d['shape']:28s} {d['us']:8.2f} us {d['frac']:.3f}\")"
done
for env in "FDPP_ATTN_PUSH=1" "FDPP_ATTN_PUSH=0" "FDPP_ATTN_PUSH=1"; do
env $env timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r2l_bench.json').read().split('\n')[0]);print('$env', d['value'],d['ms_per_step'],d['e2e']['value'],d['rows_recomputed'], d['kernels']['attention_async(+recompute)']['us'])"
done
timeout 120 python tools/attn_trace.py 1 32 32 1024 || true
