timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_configs.py -m gpu -q -x --timeout 200 --timeout-method thread > /tmp/t.txt 2>&1; echo "attn tests rc=$?"; tail -1 /tmp/t.txt
for env in "X=1" "FDPP_ATTN_DEEP=0" "FDPP_ATTN_EARLY_TRIGGER=0" "FDPP_ATTN_DEEP=0 FDPP_ATTN_EARLY_TRIGGER=0"; do
  echo "== $env"; env $env timeout 600 python tools/attn_p_sweep.py 2>&1 | tail -5
done
show() {
  python -c "
import json;d=json.loads(open('$2').read().split('\n')[0]);print('$1', d['value'],d['ms_per_step'],{k.split('[')[0][:14]:v['us'] for k,v in d['kernels'].items()})"
}
for env in "X=1" "FDPP_ATTN_DEEP=0 FDPP_ATTN_EARLY_TRIGGER=0"; do
  env $env timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/b.json 2>/dev/null; show "7B B32 $env" /tmp/b.json
  env $env timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras --batch 1 > /tmp/b.json 2>/dev/null; show "7B B1 $env" /tmp/b.json
  env $env timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 > /tmp/b.json 2>/dev/null; show "GLM $env" /tmp/b.json
  env $env timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 --inject 5 > /tmp/b.json 2>/dev/null; show "GLM inj5 $env" /tmp/b.json
  env $env timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model llama2-70b --tp-shard 8 > /tmp/b.json 2>/dev/null; show "70B t8 $env" /tmp/b.json
done
