# A/B on one box: the previous build (a copy of its tree with its own .so in .ab_old/) vs this one
show() {
  python -c "
import json;d=json.loads(open('$2').read().split('\n')[0]);print('$1', d['value'],d['ms_per_step'],d['kernels']['attention_async(+recompute)']['us'])"
}
for i in 1 2; do
  for b in 32 8 16; do
    (cd .ab_old && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras --batch $b > /tmp/old.json 2>/dev/null); show "r1      B$b" /tmp/old.json
    timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras --batch $b > /tmp/new.json 2>/dev/null; show "r2      B$b" /tmp/new.json
    FDPP_ATTN_DEEP=0 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras --batch $b > /tmp/new.json 2>/dev/null; show "r2-deep0 B$b" /tmp/new.json
  done
done
