timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_configs.py tests/test_gpu_tp.py tests/test_gpu_allreduce.py -m gpu -q -x --timeout 200 --timeout-method thread > /tmp/t.txt 2>&1; echo "tests rc=$?"; tail -2 /tmp/t.txt
show() {
  python -c "
import json;d=json.loads(open('$2').read().split('\n')[0]);print('$1', d['value'],d['ms_per_step'],d['gpu_launches'],{k.split('[')[0][:14]:v['us'] for k,v in d['kernels'].items()})"
}
for i in 1 2; do
  (cd .ab_old && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/old.json 2>/dev/null); show r1 /tmp/old.json
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/new.json 2>/dev/null; show r2 /tmp/new.json
done
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras --batch 1 > /tmp/new.json 2>/dev/null; show "r2 B1" /tmp/new.json
