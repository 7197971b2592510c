mkdir -p gpurun_out
for ab in 1 0; do
  for cs in "2 32 2 2048 1 q 1" "2 32 2 2048 7 q 3" "2 32 2 2048 7 q 0" "2 32 2 2048 4 q 2" "2 8 8 2048 7 q 3"; do
    echo "== ABORT=$ab case $cs" >> gpurun_out/r2f_debug.txt
    FDPP_ATTN_ABORT=$ab timeout 30 python tools/abort_debug.py $cs >> gpurun_out/r2f_debug.txt 2>&1
    echo "rc=$?" >> gpurun_out/r2f_debug.txt
  done
done
cat gpurun_out/r2f_debug.txt
