# K6 vs cuBLAS: L2->SM TMA bytes, L2 throughput, instruction counts (one warm launch each)
set -u
O=gpurun_out/ptraf
mkdir -p $O
M=dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,sm__cycles_elapsed.avg.per_second,gpu__time_duration.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_bytes.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:qkv_gemm -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/k6.txt 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:nvjet -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/cublas.txt 2>&1
