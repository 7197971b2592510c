K='regex:attn_split|gemm_cluster|gemm_tc|gemv|embed|argmax|advance|row_ssq'
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k $K -c 700 --csv --log-file /tmp/n2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extras > /dev/null 2>&1
(cd .ab_old && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k $K -c 700 --csv --log-file /tmp/n1.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extras > /dev/null 2>&1)
cp /tmp/n1.csv gpurun_out/r2s_ncu_r1.csv; cp /tmp/n2.csv gpurun_out/r2s_ncu_r2.csv
