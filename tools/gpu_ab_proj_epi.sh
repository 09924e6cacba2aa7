# K6 staged epilogue: prologue/projection tests, then alternating A/B against the row-per-thread
# stores, with cuBLAS timed in the same process each time.
set -u
O=gpurun_out/pepi
mkdir -p $O
timeout 600 python -m pytest tests/test_prologue_gpu.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for r in 1 2 3; do
  for lib in libs_exp/lib_pepi0.so libs_exp/lib_pepi1.so; do
    echo "$(basename $lib) r$r" >> $O/ab.txt
    OSP_LIB=$lib timeout 120 python tools/bench_proj.py --config cfg3 --reps 20 2>&1 | head -3 >> $O/ab.txt
  done
done
for lib in libs_exp/lib_pepi0.so libs_exp/lib_pepi1.so; do
  OSP_LIB=$lib timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_op_write.sum,lts__t_requests_op_write.sum --clock-control none -k regex:qkv_gemm -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/ncu_$(basename $lib .so).txt 2>&1
done
