set -u
O=gpurun_out/proj2
mkdir -p $O
for b in 12; do echo "rows band=$b" >> $O/bands.txt; OSP_PROJ_BAND=$b timeout 120 python tools/bench_proj.py --config cfg3 --reps 10 2>&1 | head -2 >> $O/bands.txt; done
for b in 2 4 6 8 12 20; do echo "cols band=$b" >> $O/bands.txt; OSP_PROJ_ORDER=1 OSP_PROJ_BAND=$b timeout 120 python tools/bench_proj.py --config cfg3 --reps 10 2>&1 | head -2 | tail -1 >> $O/bands.txt; done
