# K6 dynamic (atomic-counter) unit schedule vs the static round-robin one: tests, DRAM, A/B.
set -u
O=gpurun_out/pdyn
mkdir -p $O
timeout 600 python -m pytest tests/test_prologue_gpu.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/tests.log
run() {
  local name=$1; shift
  env "$@" timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:qkv_gemm -s 2 -c 1 python tools/bench_proj.py --config cfg3 --reps 1 > $O/$name.txt 2>&1
  echo "$name $(grep -E 'dram__bytes_read|duration|per_second|hit_rate' $O/$name.txt | awk '{print $NF}' | tr '\n' ' ')" >> $O/summary.txt
}
run static_b12 OSP_PROJ_DYN=0
run dyn_b12 OSP_PROJ_DYN=1
run dyn_b6 OSP_PROJ_DYN=1 OSP_PROJ_BAND=6
run dyn_b20 OSP_PROJ_DYN=1 OSP_PROJ_BAND=20
run dyn_row4 OSP_PROJ_DYN=1 OSP_PROJ_ORDER=0 OSP_PROJ_BAND=4
for r in 1 2 3; do for d in 0 1; do
  echo "dyn $d r$r" >> $O/ab.txt
  OSP_PROJ_DYN=$d timeout 120 python tools/bench_proj.py --config cfg3 --reps 20 2>&1 | head -3 >> $O/ab.txt
done; done
