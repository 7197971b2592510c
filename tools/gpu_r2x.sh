show() {
  python -c "
import json;d=json.loads(open('$2').read().split('\n')[0]);print('$1', d['value'],d['ms_per_step'],d['config']['gemm_choices']['qkv'],{k.split('[')[0][:14]+k.split(':')[-1]:v['us'] for k,v in d['kernels'].items()})"
}
for i in 1 2; do
for b in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras --batch $b > /tmp/a.json 2>/dev/null; show "B$b ImplB" /tmp/a.json
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras --batch $b --gemv-step > /tmp/a.json 2>/tmp/e.txt; show "B$b GEMV " /tmp/a.json || tail -3 /tmp/e.txt
done; done
