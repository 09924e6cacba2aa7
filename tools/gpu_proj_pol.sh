# K6 band size x L2 policy for x (normal / evict-first), W evict-last, output streaming
set -u
O=gpurun_out/ppol
mkdir -p $O
run() {
  local name=$1; shift
  env "$@" timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:qkv_gemm -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/$name.txt 2>&1
  echo "$name $(grep -E 'dram__bytes_read|duration|per_second|hit_rate' $O/$name.txt | awk '{print $NF}' | tr '\n' ' ')" >> $O/summary.txt
}
for b in 4 6 8 12; do for xf in 0 1; do run b${b}_xf$xf OSP_PROJ_ORDER=1 OSP_PROJ_BAND=$b OSP_PROJ_XFIRST=$xf; done; done
for r in 1 2; do for cfg in "12 0" "12 1" "8 1" "6 1"; do
  set -- $cfg
  echo "band $1 xfirst $2 r$r" >> $O/ab.txt
  OSP_PROJ_BAND=$1 OSP_PROJ_XFIRST=$2 timeout 120 python tools/bench_proj.py --config cfg3 --reps 20 2>&1 | head -2 >> $O/ab.txt
done; done
