set -u
O=gpurun_out/r2c
mkdir -p $O
./tools/pipe_mix > $O/pipe_mix.txt 2>&1; echo "pipe rc=$?"
./tools/tmem_rate > $O/tmem_rate.txt 2>&1; echo "tmem rc=$?"
./tools/mufu_rate > $O/mufu_rate.txt 2>&1; echo "mufu rc=$?"
