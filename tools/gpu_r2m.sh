# same-box A/B: round-1 final build (.ab_old) vs this build, alternating
for i in 1 2; do
  (cd .ab_old && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/old.json 2>/dev/null)
  python -c "
import json;d=json.loads(open('/tmp/old.json').read().split('\n')[0]);print('r1  ', d['value'],d['ms_per_step'],d['kernels']['attention_async(+recompute)']['us'], {k[:12]:v['us'] for k,v in d['kernels'].items()})"
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/new.json 2>/dev/null
  python -c "
import json;d=json.loads(open('/tmp/new.json').read().split('\n')[0]);print('r2  ', d['value'],d['ms_per_step'],d['kernels']['attention_async(+recompute)']['us'], {k[:12]:v['us'] for k,v in d['kernels'].items()})"
done
