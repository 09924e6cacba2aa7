# Per-CTA prologue / loop / epilogue cycles of K2 and K3 at k=2 (L=18,900 x 4) and k=4 (4,725 x 16).
set -u
O=gpurun_out/ctaph
mkdir -p $O
for cfg in "18900 4" "4725 16"; do
  OSP_LIB=libs_exp/lib_tim.so timeout 120 python tools/fwd_phases.py $cfg >> $O/fwd.txt 2>&1
  OSP_LIB=libs_exp/lib_tim.so timeout 120 python tools/bwd_phases.py $cfg >> $O/bwd.txt 2>&1
done
