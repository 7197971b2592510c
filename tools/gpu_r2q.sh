show() {
  python -c "
import json;d=json.loads(open('$2').read().split('\n')[0]);print('$1', d['value'],d['ms_per_step'],{k.split('[')[0][:14]:v['us'] for k,v in d['kernels'].items()})"
}
for i in 1 2; do
  (cd .ab_old && timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/old.json 2>/dev/null); show r1 /tmp/old.json
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/new.json 2>/dev/null; show r2 /tmp/new.json
  FDPP_KV_PREFETCH=0 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-extras > /tmp/new.json 2>/dev/null; show r2-nopf /tmp/new.json
done
# serialized per-kernel durations (ncu) of one decode step, both builds
K='regex:attn_split|gemm_|gemv|embed|argmax|advance|row_ssq'
ncu --metrics gpu__time_duration.sum --clock-control none -k $K -c 400 --csv --log-file /tmp/n2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extras > /dev/null 2>&1
(cd .ab_old && ncu --metrics gpu__time_duration.sum --clock-control none -k $K -c 400 --csv --log-file /tmp/n1.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extras > /dev/null 2>&1)
python - <<'PY'
import csv, collections
def load(p):
    rows = list(csv.reader(open(p)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]; iK, iV = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) == len(h):
            agg[r[iK].split("(")[0][:60]].append(float(r[iV].replace(",", "")))
    return agg
a, b = load("/tmp/n1.csv"), load("/tmp/n2.csv")
for k in sorted(set(a) | set(b)):
    x, y = a.get(k, []), b.get(k, [])
    f = lambda v: (len(v), round(sum(v) / max(len(v), 1) / 1e3, 2))
    print(f"{k:60s} r1 {f(x)}  r2 {f(y)}")
PY
