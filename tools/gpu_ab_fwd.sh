set -u
O=gpurun_out/ab15
mkdir -p $O
OSP_LIB=libs_exp/lib_spec1.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $O/tests.log 2>&1; echo "tests rc=$?"
bash tools/ab_libs.sh fwd cfg3 3 libs_exp/lib_spec0.so libs_exp/lib_spec1.so libs_exp/lib_spec1_p4.so > $O/ab.txt 2>&1
