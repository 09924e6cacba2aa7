set -u
O=gpurun_out/fwdexp2
mkdir -p $O
for l in tim_pp tim_nopp tim_nopp_p0; do echo "== $l" >> $O/phases.txt; OSP_LIB=libs_exp/lib_$l.so timeout 120 python tools/fwd_phases.py >> $O/phases.txt 2>&1; done
