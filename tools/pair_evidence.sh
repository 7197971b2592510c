mkdir -p gpurun_out/tbl3 gpurun_out/ncu3
timeout 900 python tools/make_table.py gpurun_out/tbl3/b200_decode.tbl > gpurun_out/tbl3/profile.txt 2>&1; echo table rc=$?
timeout 900 python tools/conv_sweep.py 128,192,256 > gpurun_out/conv3.txt 2>&1; echo conv rc=$?
R=/tmp/ncu_p; mkdir -p $R
ncu --set full --clock-control none --import-source on -k regex:gemm_pair_kernel -s 0 -c 1 -o $R/implc_m256 python tools/prof_r2.py gemm > /dev/null 2>&1
python tools/ncu_full_summary.py $R/implc_m256.ncu-rep > gpurun_out/ncu3/implc_m256.txt 2>&1
ncu -i $R/implc_m256.ncu-rep --page source --csv --print-source sass > $R/src.csv 2>/dev/null
python tools/ncu_src_top.py $R/src.csv 30 > gpurun_out/ncu3/implc_m256_sass_top.txt 2>&1
ncu --set full --clock-control none -k regex:gemm_cluster_kernel -s 3 -c 1 -o $R/implb_o python tools/prof_r2.py gemm > /dev/null 2>&1
python tools/ncu_full_summary.py $R/implb_o.ncu-rep > gpurun_out/ncu3/implb_o_m32_check.txt 2>&1
echo ncu done
