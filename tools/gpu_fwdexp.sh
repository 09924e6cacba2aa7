set -u
O=gpurun_out/fwdexp
mkdir -p $O
for f in 0 1 2 4 16 32 48 17; do echo "flags=$f" >> $O/phases.txt; OSP_FWD_FLAGS=$f OSP_LIB=libs_exp/lib_exp_timing.so timeout 120 python tools/fwd_phases.py >> $O/phases.txt 2>&1; done
