for s in "1 32 32 1024" "32 8 1 1024" "32 32 32 1024" "8 32 2 4096"; do timeout 120 python tools/attn_trace.py $s; done
