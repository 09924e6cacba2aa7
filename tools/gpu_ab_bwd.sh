set -u
O=gpurun_out/abb3
mkdir -p $O
OSP_LIB=libs_exp/lib_r321.so timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_fullsize_gpu.py -q -x -k "attention or fullsize" > $O/tests.log 2>&1; echo "tests rc=$?"
OSP_LIB=libs_exp/lib_r222.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $O/tests222.log 2>&1; echo "tests222 rc=$?"
OSP_LIB=libs_exp/lib_r321_tim.so timeout 120 python tools/bwd_phases.py > $O/phases.txt 2>&1
bash tools/ab_libs.sh bwd cfg3 3 libs_exp/lib_head.so libs_exp/lib_r321.so libs_exp/lib_r222.so > $O/ab.txt 2>&1
