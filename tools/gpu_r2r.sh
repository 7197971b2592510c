show() {
  python -c "
import json;d=json.loads(open('$2').read().split('\n')[0]);print('$1', d['value'],d['ms_per_step'],{k.split('[')[0][:14]:v['us'] for k,v in d['kernels'].items()})"
}
for i in 1 2; do
  (cd .ab_old && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/old.json 2>/dev/null); show r1 /tmp/old.json
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/new.json 2>/dev/null; show r2 /tmp/new.json
  FDPP_ATTN_INCLUSTER=0 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/new.json 2>/dev/null; show r2-2launch /tmp/new.json
done
