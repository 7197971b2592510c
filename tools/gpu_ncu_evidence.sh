# round-2 ncu evidence: full-set captures of the shipped kernels (summarised on
# the box, reports deleted: gpurun_out/ must stay under 64 MiB) + the
# decode-step launch list
mkdir -p gpurun_out/ncu
R=/tmp/ncu_r2; mkdir -p $R
N="ncu --set full --clock-control none --import-source on"
cap() {  # name regex skip script-arg
  $N -k regex:$2 -s $3 -c 1 -o $R/$1 python tools/prof_r2.py $4 > /dev/null 2>&1
  python tools/ncu_full_summary.py $R/$1.ncu-rep > gpurun_out/ncu/$1.txt 2>&1
  ncu -i $R/$1.ncu-rep --page source --csv --print-source sass > $R/$1_src.csv 2>/dev/null
  python tools/ncu_src_top.py $R/$1_src.csv 30 > gpurun_out/ncu/$1_sass_top.txt 2>&1
}
cap attn_mha attn_split_kernel 0 attn
cap attn_mqa attn_split_kernel 2 attn
cap gemv gemv_kernel 0 gemm
cap implc_m128 gemm_cluster_kernel 0 gemm
cap implc_m256 gemm_pair_kernel 0 gemm
cap implb_o_m32 gemm_cluster_kernel 3 gemm
cap gemv_fused gemv_fused_kernel 0 gemv_fused
cap implb_gu_m32 gemm_cluster_kernel 1 gemm_gu
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_split|gemm_|gemv|embed|argmax|advance|row_ssq|rmsnorm|rope_append|silu_mul" -c 600 --csv \
    --log-file gpurun_out/ncu/launches_decode_step.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extras > /dev/null 2>&1
ls -la gpurun_out/ncu; du -sh gpurun_out
