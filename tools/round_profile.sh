#!/usr/bin/env bash
# One GPU-box pass that produces the round's evidence under gpurun_out/:
# GPU tests, the bench line (ours + reference arm), the ncu launch list of the bench command,
# and one `ncu --set full` capture per hot kernel (each only after its command ran clean).
set -u
O=gpurun_out/prof
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 600 python bench.py > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_ref.jsonl 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/bench_proj.py > $O/bench_proj.txt 2>&1; echo "proj rc=$?"
timeout 300 python tools/bench_stack.py --config cfg5k2 > $O/stack_cfg5k2.jsonl 2>&1; echo "stack rc=$?"
timeout 300 python tools/ncu_proj.py > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none \
  --import-source on -k regex:qkv_gemm -s 2 -c 1 -o $O/qkv_gemm -f python tools/ncu_proj.py > $O/ncu_qkv_gemm.log 2>&1
timeout 300 python tools/profile_step.py --steps 2 > $O/step.log 2>&1 && {
  for k in attn_bwd_v2 attn_fwd permute_rows; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o $O/$k -f python tools/profile_step.py --steps 2 > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
  done
}
