# GPU tests of the fused paths, then the decode step with the fused gate|up on CTA pairs on / off
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_configs.py tests/test_gpu_gemm.py -q -x --timeout 300 2>&1 | tail -2
show() { python -c "
import json,sys;d=json.loads(open('$2').readline());print('$1',d['ms_per_step'],[round(v['us'],2) for v in d['kernels'].values()])"; }
for i in 1 2; do for b in 64 48; do for v in 1 0; do
  FDPP_PAIR_FUSED=$v timeout 300 python bench.py --no-cpu --no-extras --steps 50 --batch $b > /tmp/x.json 2>/dev/null; show "B$b pair_fused=$v" /tmp/x.json
done; done; done
for v in 1 0; do FDPP_PAIR_FUSED=$v timeout 300 python bench.py --no-cpu --no-extras --steps 30 --model chatglm2-6b --batch 64 --kv-len 4096 > /tmp/x.json 2>/dev/null; show "glm B64 L4K pair_fused=$v" /tmp/x.json; done
