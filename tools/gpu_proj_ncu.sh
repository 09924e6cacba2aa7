set -u
O=gpurun_out/projncu
mkdir -p $O
timeout 300 python tools/ncu_proj.py > /dev/null 2>&1
for o in 0 1; do OSP_PROJ_ORDER=$o timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:qkv_gemm -s 2 -c 1 python tools/ncu_proj.py > $O/order$o.txt 2>&1; done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:nvjet -s 2 -c 1 python tools/ncu_cublas_proj.py > $O/cublas.txt 2>&1
