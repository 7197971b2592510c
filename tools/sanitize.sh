# compute-sanitizer over every libfdpp kernel (tools/sanitize.py); logs into gpurun_out/
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 900 $CS --tool $tool $extra --error-exitcode 7 --kernel-name kns=4fdpp \
      python tools/sanitize.py > gpurun_out/r2_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/r2_sanitizer_summary.txt
  tail -4 gpurun_out/r2_sanitizer_$tool.txt
done
