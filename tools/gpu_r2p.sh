show() {
  python -c "
import json;d=json.loads(open('$2').read().split('\n')[0]);print('$1', d['value'],d['ms_per_step'],{k.split('[')[0][:14]:v['us'] for k,v in d['kernels'].items()})"
}
for i in 1 2; do
  (cd .ab_old && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/old.json 2>/dev/null); show r1 /tmp/old.json
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/new.json 2>/dev/null; show r2 /tmp/new.json
done
for ab in 1 0; do for inj in 0 5; do
FDPP_ATTN_ABORT=$ab timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 --inject $inj > /tmp/g.json 2>&1; show "glm abort=$ab inj=$inj" /tmp/g.json
done; done
(cd .ab_old && timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 --inject 5 > /tmp/g.json 2>&1); show "glm r1 inj=5" /tmp/g.json
(cd .ab_old && timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 > /tmp/g.json 2>&1); show "glm r1 inj=0" /tmp/g.json
