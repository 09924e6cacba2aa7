set -u
O=gpurun_out/abb2
mkdir -p $O
OSP_LIB=libs_exp/lib_splitq.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $O/tests.log 2>&1; echo "tests rc=$?"
OSP_LIB=libs_exp/lib_splitq_tim.so timeout 120 python tools/bwd_phases.py > $O/phases.txt 2>&1
bash tools/ab_libs.sh bwd cfg3 3 libs_exp/lib_nosplitq.so libs_exp/lib_splitq.so > $O/ab.txt 2>&1
