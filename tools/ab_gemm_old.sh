# A/B of the current build vs tools/ab_old/libfdpp.so (HEAD's gemm.cu), alternating on one box
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_configs.py -q -x --timeout 300 2>&1 | tail -1
show() { python -c "
import json,sys;d=json.loads(open('$2').readline());print('$1',d['ms_per_step'],[round(v['us'],2) for v in d['kernels'].values()])"; }
for i in 1 2; do
  true FDPP_LIB=$PWD/tools/ab_old/libfdpp.so timeout 300 python tools/qkv_epi_probe.py | sed 's/^/old /'
  true timeout 300 python tools/qkv_epi_probe.py | sed 's/^/new /'
done
for i in 1 2 3; do for b in ${AB_BATCHES:-32 64 8}; do
  FDPP_LIB=$PWD/tools/ab_old/libfdpp.so timeout 300 python bench.py --no-cpu --no-extras --steps 50 --batch $b > /tmp/o.json 2>/dev/null; show "old B$b" /tmp/o.json
  timeout 300 python bench.py --no-cpu --no-extras --steps 50 --batch $b > /tmp/n.json 2>/dev/null; show "new B$b" /tmp/n.json
done; done
