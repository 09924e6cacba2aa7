# K6 epilogue accumulator wait with sleeping back-off (bo1) vs suspend-hinted probes (bo0)
set -u
O=gpurun_out/pbo
mkdir -p $O
OSP_LIB=libs_exp/lib_bo1.so timeout 300 python -m pytest tests/test_prologue_gpu.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/tests.log
M=dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for l in bo0 bo1; do
  OSP_LIB=libs_exp/lib_$l.so timeout 300 ncu --metrics $M --clock-control none -k regex:qkv_gemm -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/ncu_$l.txt 2>&1
  echo "$l $(grep -E 'dram__|duration|per_second|inst_executed|tensor' $O/ncu_$l.txt | awk '{print $NF}' | tr '\n' ' ')" >> $O/summary.txt
done
for r in 1 2 3; do for l in bo0 bo1; do
  echo "$l r$r" >> $O/ab.txt
  OSP_LIB=libs_exp/lib_$l.so timeout 120 python tools/bench_proj.py --config cfg3 --reps 20 2>&1 | head -3 >> $O/ab.txt
done; done
