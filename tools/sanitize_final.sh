mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 7 --kernel-name kns=4fdpp \
      python tools/sanitize.py > gpurun_out/san/$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$tool.txt
done
