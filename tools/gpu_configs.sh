# round-2 numbers for the other BASELINE configs (cfg2 block, cfg5 hybrid stacks k=2 / k=4, cfg1)
set -u
O=gpurun_out/cfgs
mkdir -p $O
timeout 600 python bench.py --config cfg2 --no-cpu > $O/bench_cfg2.jsonl 2> $O/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 600 python bench.py --config cfg1 --no-cpu --no-comparator --steps 20 > $O/bench_cfg1.jsonl 2> $O/bench_cfg1.err; echo "cfg1 rc=$?"
timeout 600 python tools/bench_stack.py --config cfg5k2 > $O/stack_cfg5k2.jsonl 2>&1; echo "stack k2 rc=$?"
timeout 600 python tools/bench_stack.py --config cfg5k4 > $O/stack_cfg5k4.jsonl 2>&1; echo "stack k4 rc=$?"
timeout 600 python bench.py --config cfg5k2 --no-cpu --no-comparator > $O/bench_cfg5k2.jsonl 2> $O/bench_cfg5k2.err; echo "cfg5k2 rc=$?"
