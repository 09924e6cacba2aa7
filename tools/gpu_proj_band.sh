set -u
O=gpurun_out/proj
mkdir -p $O
for b in 4 6 8 12 16 24 40; do echo "band=$b" >> $O/bands.txt; OSP_PROJ_BAND=$b timeout 120 python tools/bench_proj.py --config cfg3 --reps 10 2>&1 | head -2 >> $O/bands.txt; done
