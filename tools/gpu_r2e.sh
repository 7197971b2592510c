set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.txt 2>&1
tail -2 gpurun_out/r2e_smoke.txt
for f in test_gpu_attention test_gpu_configs test_gpu_decode test_gpu_gemm test_gpu_tp test_gpu_allreduce; do
  timeout 900 python -m pytest tests/$f.py -m gpu -q -rf -x --timeout 150 --timeout-method thread > gpurun_out/r2e_$f.txt 2>&1
  echo "$f rc=$?"; tail -3 gpurun_out/r2e_$f.txt
done
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 150 --timeout-method thread --deselect tests/test_gpu_attention.py --deselect tests/test_gpu_configs.py --deselect tests/test_gpu_decode.py --deselect tests/test_gpu_gemm.py --deselect tests/test_gpu_tp.py --deselect tests/test_gpu_allreduce.py > gpurun_out/r2e_rest.txt 2>&1
tail -3 gpurun_out/r2e_rest.txt
