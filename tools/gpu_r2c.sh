set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.txt 2>&1
tail -3 gpurun_out/r2c_smoke.txt
timeout 1200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_configs.py -m gpu -x -q -rf 2>&1 | tail -30 > gpurun_out/r2c_tests1.txt
tail -15 gpurun_out/r2c_tests1.txt
timeout 1200 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_attention.py --deselect tests/test_gpu_configs.py 2>&1 | tail -20 > gpurun_out/r2c_tests2.txt
tail -8 gpurun_out/r2c_tests2.txt
for inj in 0 5; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 --inject $inj > gpurun_out/r2c_glm_inj$inj.json 2>&1
FDPP_ATTN_ABORT=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --model chatglm2-6b --batch 8 --kv-len 32768 --inject $inj > gpurun_out/r2c_glm_inj${inj}_noabort.json 2>&1
done
grep -o '"ms_per_step": [0-9.]*\|"attention_async[^}]*}\|rows_recomputed": [0-9]*' gpurun_out/r2c_glm*.json
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
head -c 600 gpurun_out/r2c_bench.json; grep -o '"c1_attention_op[^}]*}\|"attention_async(+recompute)": {[^}]*}' gpurun_out/r2c_bench.json
