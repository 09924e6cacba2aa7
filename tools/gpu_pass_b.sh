# round-2 evidence pass: block parity record, K2 phase timing, sanitizer, K1 ncu at cfg3
set -u
O=gpurun_out/r2b
mkdir -p $O
OSP_PARITY_OUT=$O/parity.json timeout 900 python -m pytest tests/test_block_parity_gpu.py -q -s > $O/parity.log 2>&1; echo "parity rc=$?"
timeout 300 python tools/time_kernels.py --config cfg3 --what fwd,bwd --reps 3 > $O/time_kernels.txt 2>&1; echo "time rc=$?"
OSP_LIB=libs_exp/lib_timing.so timeout 300 python tools/fwd_phases.py > $O/fwd_phases.txt 2>&1; echo "phases rc=$?"
timeout 300 python tools/profile_step.py --steps 2 > $O/step.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:permute_rows_warp -s 0 -c 2 \
  -o $O/permute_rows_cfg3 -f python tools/profile_step.py --steps 2 > $O/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -q -x \
  -k "not repeatable" > $O/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -q -x \
  -k "attention and not repeatable" > $O/sanitizer_synccheck.log 2>&1; echo "synccheck rc=$?"
