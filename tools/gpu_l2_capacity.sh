set -u
O=gpurun_out/l2c
mkdir -p $O
for m in 0 1; do for s in 16 32 48 64 80 96 112; do
  echo -n "S=$s mode=$m " >> $O/summary.txt
  timeout 120 ncu --cache-control none --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:rd -s 1 -c 1 ./tools/l2_capacity $s $m 2>&1 | grep -E "dram__bytes_read|hit_rate" | awk '{print $(NF-1), $NF}' | tr '\n' ' ' >> $O/summary.txt
  echo >> $O/summary.txt
done; done
