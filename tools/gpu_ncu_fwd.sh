set -u
O=gpurun_out/ncufwd
mkdir -p $O
timeout 300 python tools/sdpa_probe.py --impl ours --what fwd --reps 1 > $O/probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -c 1 -o $O/attn_fwd -f python tools/sdpa_probe.py --impl ours --what fwd --reps 1 > $O/ncu.log 2>&1; echo "ncu rc=$?"
