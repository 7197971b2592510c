run() {  # label, then env
  local lab=$1; shift
  env "$@" timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/b.json 2>/dev/null
  python -c "
import json;d=json.loads(open('/tmp/b.json').read().split('\n')[0]);print('$lab', d['value'],d['ms_per_step'],d['kernels']['attention_async(+recompute)']['us'])"
}
for i in 1 2; do
  (cd .ab_old && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/old.json 2>/dev/null)
  python -c "
import json;d=json.loads(open('/tmp/old.json').read().split('\n')[0]);print('r1      ', d['value'],d['ms_per_step'],d['kernels']['attention_async(+recompute)']['us'])"
  run "r2      " X=1
  run "nopass2 " FDPP_LIB=.ab_variants/nopass2/libfdpp.so
done
