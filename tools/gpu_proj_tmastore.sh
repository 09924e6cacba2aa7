# K6 epilogue through TMA stores (tmas1) vs coalesced st.global (tmas0): tests, ncu, A/B with cuBLAS
set -u
O=gpurun_out/ptma
mkdir -p $O
OSP_LIB=libs_exp/lib_tmas1.so timeout 600 python -m pytest tests/test_prologue_gpu.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/tests.log
for l in tmas0 tmas1; do
  OSP_LIB=libs_exp/lib_$l.so timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:qkv_gemm -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/ncu_$l.txt 2>&1
  echo "$l $(grep -E 'dram__bytes_read|duration|per_second|tensor' $O/ncu_$l.txt | awk '{print $NF}' | tr '\n' ' ')" >> $O/summary.txt
done
for r in 1 2 3; do for l in tmas0 tmas1; do
  echo "$l r$r" >> $O/ab.txt
  OSP_LIB=libs_exp/lib_$l.so timeout 120 python tools/bench_proj.py --config cfg3 --reps 20 2>&1 | head -3 >> $O/ab.txt
done; done
