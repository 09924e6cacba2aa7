# Early Q (K2) / K-V TMA + K from smem into TMEM (K3): parity tests, per-CTA phases, A/B.
set -u
O=gpurun_out/early
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_block_parity_gpu.py tests/test_gpu_api.py tests/test_fullsize_gpu.py -q -x > $O/tests.log 2>&1; echo "tests rc=$?"
tail -3 $O/tests.log
for cfg in "18900 4" "4725 16"; do
  OSP_LIB=libs_exp/lib_tim.so timeout 120 python tools/fwd_phases.py $cfg 2>&1 | tail -1 >> $O/phases.txt
  OSP_LIB=libs_exp/lib_tim.so timeout 120 python tools/bwd_phases.py $cfg 2>&1 | tail -1 >> $O/phases.txt
done
bash tools/ab_libs.sh fwd,bwd cfg3k4 3 libs_exp/lib_epi1.so libs_exp/lib_early1.so > $O/ab_k4.txt 2>&1
bash tools/ab_libs.sh fwd,bwd cfg3 2 libs_exp/lib_epi1.so libs_exp/lib_early1.so > $O/ab_k2.txt 2>&1
