set -u
O=gpurun_out/ab16
mkdir -p $O
OSP_LIB=libs_exp/lib_v3.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $O/tests.log 2>&1; echo "tests rc=$?"
OSP_LIB=libs_exp/lib_v3_tim.so timeout 120 python tools/fwd_phases.py > $O/phases.txt 2>&1
bash tools/ab_libs.sh fwd cfg3 4 libs_exp/lib_v2.so libs_exp/lib_v3.so > $O/ab.txt 2>&1
