#!/bin/bash
# A/B timing of library variants (libs_exp/*.so, built with OSP_LIB_OUT / OSP_NVCC_FLAGS):
#   tools/ab_libs.sh "fwd" cfg3 3 libs_exp/lib_a.so libs_exp/lib_b.so ...
# alternates the variants for ROUNDS rounds (the power-capped clock drifts), one process each.
what=$1; cfg=$2; rounds=$3; shift 3
for r in $(seq 1 $rounds); do
  for lib in "$@"; do
    echo -n "$(basename $lib) r$r: "
    OSP_LIB=$lib python tools/time_kernels.py --config $cfg --what $what --reps 5 | tr '\n' ' '
    echo
  done
done
