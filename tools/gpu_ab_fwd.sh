set -u
O=gpurun_out/ab17
mkdir -p $O
OSP_LIB=libs_exp/lib_new.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $O/tests.log 2>&1; echo "tests rc=$?"
bash tools/ab_libs.sh fwd cfg3 4 libs_exp/lib_old.so libs_exp/lib_new.so > $O/ab.txt 2>&1
