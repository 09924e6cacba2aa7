# K6 quad clusters (two pairs sharing the W slice by multicast) vs pairs: tests, DRAM/L2, A/B
set -u
O=gpurun_out/pquad
mkdir -p $O
OSP_PROJ_QUAD=1 timeout 300 python -m pytest tests/test_prologue_gpu.py -q -x > $O/tests.log 2>&1; echo "tests quad rc=$?"; tail -3 $O/tests.log
M=dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed
for q in 0 1; do
  OSP_PROJ_QUAD=$q timeout 300 ncu --metrics $M --clock-control none -k regex:qkv_gemm -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/ncu_q$q.txt 2>&1
  echo "quad=$q $(grep -E 'dram__|l1tex__|duration|per_second|lts__' $O/ncu_q$q.txt | awk '{print $NF}' | tr '\n' ' ')" >> $O/summary.txt
done
for r in 1 2 3; do for q in 0 1; do
  echo "quad $q r$r" >> $O/ab.txt
  OSP_PROJ_QUAD=$q timeout 120 python tools/bench_proj.py --config cfg3 --reps 20 2>&1 | head -3 >> $O/ab.txt
done; done
