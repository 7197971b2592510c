# round-2 results table: bench lines across configs + the reference's record surface
mkdir -p gpurun_out/r2u
b() { local name=$1; shift; timeout 900 python bench.py --no-cpu --no-extras --steps 30 "$@" > gpurun_out/r2u/$name.json 2> gpurun_out/r2u/$name.err; echo "$name rc=$?"; }
b b1 --batch 1; b b8 --batch 8; b b16 --batch 16; b b64 --batch 64
b b16_l8k --batch 16 --kv-len 8192; b b64_l4k --batch 64 --kv-len 4096
b glm --model chatglm2-6b --batch 8 --kv-len 32768; b glm_inj5 --model chatglm2-6b --batch 8 --kv-len 32768 --inject 5
b l70 --model llama2-70b; b l70_t2 --model llama2-70b --tp-shard 2; b l70_t4 --model llama2-70b --tp-shard 4; b l70_t8 --model llama2-70b --tp-shard 8
timeout 600 python -m paper_2311_01282_b200.records bench --suite gemm --shapes 12288:4096,4096:4096 --m 8 --out gpurun_out/r2u/records_bench_gemm.txt > /dev/null 2>&1; echo "rec gemm rc=$?"
timeout 600 python -m paper_2311_01282_b200.records bench --suite attn --seq 1024 --out gpurun_out/r2u/records_bench_attn.txt > /dev/null 2>&1; echo "rec attn rc=$?"
timeout 600 python -m paper_2311_01282_b200.records bench --suite prefill --seq 4096 --out gpurun_out/r2u/records_bench_prefill.txt > /dev/null 2>&1; echo "rec prefill rc=$?"
timeout 600 python -m paper_2311_01282_b200.records decode --model llama2-7b --batch 4 --seq 256 --out gpurun_out/r2u/records_decode.txt > /dev/null 2>&1; echo "rec decode rc=$?"
cat gpurun_out/r2u/records_*.txt | head -40
