set -u
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > $O/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?"
