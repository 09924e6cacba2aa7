# K6 L2 policy (W band evict-last, streaming output stores) A/B with cuBLAS in the same process, and
# the DRAM bytes of one launch each (the 3rd K6 launch, warm).
set -u
O=gpurun_out/phint
mkdir -p $O
timeout 600 python -m pytest tests/test_prologue_gpu.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/tests.log
for r in 1 2 3; do
  for lib in libs_exp/lib_phint0.so libs_exp/lib_phint1.so; do
    echo "$(basename $lib) r$r" >> $O/ab.txt
    OSP_LIB=$lib timeout 120 python tools/bench_proj.py --config cfg3 --reps 20 2>&1 | head -2 >> $O/ab.txt
  done
done
for lib in libs_exp/lib_phint0.so libs_exp/lib_phint1.so; do
  OSP_LIB=$lib timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:qkv_gemm -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/ncu_$(basename $lib .so).txt 2>&1
done
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:nvjet -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/ncu_cublas.txt 2>&1
