set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.txt 2>&1
tail -3 gpurun_out/r2b_smoke.txt
timeout 1200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gemm.py -m gpu -x -q -rf 2>&1 | tail -30 > gpurun_out/r2b_tests1.txt
tail -15 gpurun_out/r2b_tests1.txt
timeout 1200 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_attention.py --deselect tests/test_gpu_gemm.py 2>&1 | tail -20 > gpurun_out/r2b_tests2.txt
tail -8 gpurun_out/r2b_tests2.txt
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
head -c 1500 gpurun_out/r2b_bench.json; grep -o '"c1_attention_op[^}]*}' gpurun_out/r2b_bench.json
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 --inject 5 > gpurun_out/r2b_glm_inj.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 > gpurun_out/r2b_glm.json 2>&1
grep -o '"ms_per_step": [0-9.]*\|"attention_async[^}]*}' gpurun_out/r2b_glm*.json
timeout 900 python tools/conv_sweep.py > gpurun_out/r2b_conv_sweep.txt 2>&1
tail -40 gpurun_out/r2b_conv_sweep.txt
