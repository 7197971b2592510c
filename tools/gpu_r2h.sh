mkdir -p gpurun_out
for env in "FDPP_ATTN_ABORT=1" "FDPP_ATTN_ABORT=0" "FDPP_ATTN_INCLUSTER=0"; do
  echo "== $env" >> gpurun_out/r2h_modes.txt
  env $env timeout 600 python tools/attn_graph_sweep.py 2>&1 | grep '"kv_prefetch": true' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(f\"{d['shape']:28s} {d['us']:8.2f} us {d['frac']:.3f}\")" >> gpurun_out/r2h_modes.txt
done
cat gpurun_out/r2h_modes.txt
