timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py tests/test_gpu_tp.py tests/test_gpu_allreduce.py -q -x --timeout 300 > gpurun_out/cs_tests.txt 2>&1; echo tests rc=$?; tail -1 gpurun_out/cs_tests.txt
timeout 900 python tools/cs_fine.py > gpurun_out/cs_fine2.txt 2>&1
show() { python -c "
import json,sys;d=json.loads(open('$2').readline());print('$1',d['ms_per_step'],[round(v['us'],2) for v in d['kernels'].values()])"; }
timeout 300 python bench.py --no-cpu --no-extras --steps 30 --model chatglm2-6b --batch 8 --kv-len 32768 > /tmp/g.json 2>/dev/null; show glm /tmp/g.json
timeout 300 python bench.py --no-cpu --no-extras --steps 30 --model llama2-70b --tp-shard 2 > /tmp/g.json 2>/dev/null; show l70t2 /tmp/g.json
timeout 300 python bench.py --no-cpu --no-extras --steps 20 --model llama2-70b > /tmp/g.json 2>/dev/null; show l70 /tmp/g.json
timeout 300 python bench.py --no-cpu --no-extras --steps 50 > /tmp/g.json 2>/dev/null; show 7b /tmp/g.json
