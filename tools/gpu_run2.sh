python -m pytest tests/test_gpu_configs.py -m gpu -q -s 2>&1 | tail -15 > gpurun_out/r2_configs_parity.txt
bash tools/sanitize.sh
