#!/usr/bin/env bash
# One GPU-box pass producing a round's evidence under gpurun_out/prof: the GPU suite (with the block
# parity record), smoke, the bench line (twice: the power-capped clock varies run to run) and the
# reference arm, the ncu launch list of the bench command, and `ncu --set full` captures of the hot
# kernels inside the benched step (each only after its command ran clean).
set -u
O=gpurun_out/prof
mkdir -p $O
OSP_PARITY_OUT=$O/parity.json timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for i in 1 2; do timeout 600 python bench.py > $O/bench_$i.jsonl 2> $O/bench_$i.err; echo "bench $i rc=$?"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.jsonl 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-comparator > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/profile_step.py --steps 2 > $O/step.log 2>&1 && {
  for k in attn_bwd_v2 attn_fwd; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o $O/$k -f python tools/profile_step.py --steps 2 > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
  done
}
