set -u
O=gpurun_out/ab8
mkdir -p $O
for v in c1p0 c2p0; do OSP_LIB=libs_exp/lib_$v.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $O/tests_$v.log 2>&1; echo "tests $v rc=$?"; done
bash tools/ab_libs.sh fwd cfg3 3 libs_exp/lib_c0p3.so libs_exp/lib_c1p0.so libs_exp/lib_c1p4.so libs_exp/lib_c1p8.so libs_exp/lib_c2p0.so > $O/ab.txt 2>&1
