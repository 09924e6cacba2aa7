set -u
O=gpurun_out/l2d
mkdir -p $O
for m in 0 1 2 3; do
  timeout 120 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct -k regex:rd --clock-control none ./tools/l2_dies $m > $O/mode$m.txt 2>&1
done
