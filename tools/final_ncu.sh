# final-build ncu evidence: the B=32 decode-step launch list and the B=64 step's fused gate|up on CTA pairs
mkdir -p gpurun_out/ncuf
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_split|gemm_|gemv|embed|argmax|advance|row_ssq|rmsnorm|rope_append|silu_mul" -c 600 --csv \
    --log-file gpurun_out/ncuf/launches_decode_step.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extras > /dev/null 2>&1
R=/tmp/ncu_f; mkdir -p $R
ncu --set full --clock-control none --import-source on -k regex:gemm_pair_kernel -s 2 -c 1 -o $R/pair_gu python bench.py --steps 2 --warmup 3 --no-cpu --no-extras --batch 64 > /dev/null 2>&1
python tools/ncu_full_summary.py $R/pair_gu.ncu-rep > gpurun_out/ncuf/pair_gate_up_b64.txt 2>&1
echo done
