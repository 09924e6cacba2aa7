set -u
O=gpurun_out/ab9
mkdir -p $O
bash tools/ab_libs.sh fwd cfg3 4 libs_exp/lib_pp_p3.so libs_exp/lib_nopp_p0.so libs_exp/lib_nopp_p8.so libs_exp/lib_nopp_p3.so > $O/ab.txt 2>&1
bash tools/ab_libs.sh fwd cfg3k4 2 libs_exp/lib_pp_p3.so libs_exp/lib_nopp_p0.so libs_exp/lib_nopp_p8.so >> $O/ab.txt 2>&1
