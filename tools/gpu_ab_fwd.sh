set -u
O=gpurun_out/ab6
mkdir -p $O
bash tools/ab_libs.sh fwd cfg3 3 libs_exp/lib_t0_p4.so libs_exp/lib_t0_p3.so libs_exp/lib_t0_p2.so libs_exp/lib_nopp_p8.so libs_exp/lib_nopp_p3.so > $O/ab.txt 2>&1
