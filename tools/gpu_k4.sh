set -u
O=gpurun_out/k4
mkdir -p $O
timeout 300 python tools/time_kernels.py --config cfg3k4 --what fwd,bwd --reps 3 > $O/time_k4.txt 2>&1
timeout 300 python tools/time_kernels.py --config cfg3 --what fwd,bwd --reps 3 >> $O/time_k4.txt 2>&1
timeout 600 python bench.py --config cfg3k4 --no-cpu --no-comparator > $O/bench_cfg3k4.jsonl 2> $O/bench_cfg3k4.err
timeout 600 python bench.py --config cfg5k4 --no-cpu --no-comparator > $O/bench_cfg5k4.jsonl 2> $O/bench_cfg5k4.err
