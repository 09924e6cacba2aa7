# K6 DRAM bytes / time per schedule (one warm launch each under ncu) to locate the over-fetch.
set -u
O=gpurun_out/pdram
mkdir -p $O
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:qkv_gemm -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/$name.txt 2>&1
  echo "$name $(grep -E 'dram__bytes_read|duration|per_second|hit_rate' $O/$name.txt | awk '{print $NF}' | tr '\n' ' ')" >> $O/summary.txt
}
run col12 OSP_PROJ_ORDER=1 OSP_PROJ_BAND=12
run col2 OSP_PROJ_ORDER=1 OSP_PROJ_BAND=2
run col6 OSP_PROJ_ORDER=1 OSP_PROJ_BAND=6
run col30 OSP_PROJ_ORDER=1 OSP_PROJ_BAND=30
run row1 OSP_PROJ_ORDER=0 OSP_PROJ_BAND=1
run row3 OSP_PROJ_ORDER=0 OSP_PROJ_BAND=3
run row6 OSP_PROJ_ORDER=0 OSP_PROJ_BAND=6
run col12_nopair OSP_PROJ_ORDER=1 OSP_PROJ_BAND=12 OSP_PROJ_PAIR=0
