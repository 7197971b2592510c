mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.txt 2>&1; tail -1 gpurun_out/r2t_smoke.txt
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method thread --durations=10 > gpurun_out/r2t_gputest.txt 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/r2t_gputest.txt
timeout 900 python bench.py > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; echo "bench rc=$?"
head -c 400 gpurun_out/r2t_bench.json; echo
timeout 900 python bench.py --impl reference > gpurun_out/r2t_ref.json 2> gpurun_out/r2t_ref.err; echo "ref rc=$?"
timeout 1500 python tools/make_table.py tables/b200_decode.tbl > gpurun_out/r2t_make_table.txt 2>&1; echo "table rc=$?"
tail -5 gpurun_out/r2t_make_table.txt; cp tables/b200_decode.tbl tables/b200_decode.medians.json gpurun_out/ 2>/dev/null
