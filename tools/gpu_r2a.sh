set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep 'Model name'
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1
tail -3 gpurun_out/r2_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=20 2>&1 | tail -60 > gpurun_out/r2_gputest.txt
tail -5 gpurun_out/r2_gputest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
cat gpurun_out/r2_bench.json | head -c 3000
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err
cat gpurun_out/r2_ref.json | head -c 2000
