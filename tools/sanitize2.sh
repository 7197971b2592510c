# compute-sanitizer, round 2: racecheck in analysis mode (one line per racing
# source-location pair instead of per byte), initcheck with PDL off.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool racecheck --racecheck-report analysis --print-limit 2000 --kernel-name kns=4fdpp \
    python tools/sanitize.py > gpurun_out/r2_sanitizer_racecheck_analysis.txt 2>&1
echo "racecheck(analysis) rc=$?" | tee -a gpurun_out/r2_sanitizer_summary2.txt
grep -c "Race reported" gpurun_out/r2_sanitizer_racecheck_analysis.txt
SANITIZE_NOPDL=1 timeout 2400 $CS --tool initcheck --kernel-name kns=4fdpp --error-exitcode 7 \
    python tools/sanitize.py > gpurun_out/r2_sanitizer_initcheck_nopdl.txt 2>&1
echo "initcheck(no PDL) rc=$?" | tee -a gpurun_out/r2_sanitizer_summary2.txt
tail -4 gpurun_out/r2_sanitizer_initcheck_nopdl.txt
