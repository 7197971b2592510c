# full GPU test suite on the box; summary + durations into gpurun_out/
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 2>&1 | tail -60 > gpurun_out/r2_gputest.txt
tail -5 gpurun_out/r2_gputest.txt
