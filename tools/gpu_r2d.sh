set -x
mkdir -p gpurun_out
for ab in 1 0; do
  for cs in "2 32 2 2048 4 q" "2 32 2 2048 4 k" "2 8 8 700 0 k" "1 32 32 1024 0 q" "2 16 4 900 0 q" "4 16 2 2048 0 k"; do
    echo "== ABORT=$ab case $cs" >> gpurun_out/r2d_debug.txt
    FDPP_ATTN_ABORT=$ab timeout 60 python tools/abort_debug.py $cs >> gpurun_out/r2d_debug.txt 2>&1
    echo "rc=$?" >> gpurun_out/r2d_debug.txt
  done
done
cat gpurun_out/r2d_debug.txt | grep -v "^plan" | head -80
