python tools/pdl_attn_probe.py 2>&1 | tail -6
for pdl in 1 0 1 0; do
FDPP_PDL=$pdl timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/b.json 2>/dev/null
python -c "
import json;d=json.loads(open('/tmp/b.json').read().split('\n')[0]);print('step pdl=$pdl', d['value'],d['ms_per_step'])"
done
