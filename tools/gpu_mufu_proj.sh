# MUFU half-precision exp2 rate + K6 row-band sweep (order0) against cuBLAS, alternating.
set -u
O=gpurun_out/mp
mkdir -p $O
python -c "from paper_2605_28691_b200 import build as b; b.build()" > $O/build.log 2>&1
timeout 60 ./tools/mufu_rate > $O/mufu.txt 2>&1
for b in 4 6 8 12 16 24; do
  echo "rows band=$b" >> $O/bands.txt
  OSP_PROJ_ORDER=0 OSP_PROJ_BAND=$b timeout 120 python tools/bench_proj.py --config cfg3 --reps 20 2>&1 | head -2 >> $O/bands.txt
done
echo "cols band=12" >> $O/bands.txt
OSP_PROJ_ORDER=1 OSP_PROJ_BAND=12 timeout 120 python tools/bench_proj.py --config cfg3 --reps 20 2>&1 | head -2 >> $O/bands.txt
