# fused gate|up on CTA pairs at 17-32 tokens (FDPP_PAIR_FUSED_MIN=17) vs the cluster kernel
timeout 600 python -m pytest tests/test_gpu_decode.py -q -x --timeout 300 2>&1 | tail -1
FDPP_PAIR_FUSED_MIN=17 timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_configs.py -q -x --timeout 300 2>&1 | tail -1
show() { python -c "
import json,sys;d=json.loads(open('$2').readline());print('$1',d['ms_per_step'],[round(v['us'],2) for v in d['kernels'].values()])"; }
for i in 1 2; do for b in 32 24; do for v in 33 17; do
  FDPP_PAIR_FUSED_MIN=$v timeout 300 python bench.py --no-cpu --no-extras --steps 50 --batch $b > /tmp/x.json 2>/dev/null; show "B$b min_m=$v" /tmp/x.json
done; done; done
