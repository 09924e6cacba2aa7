# logic check of bench.py's N-rank path on ONE GPU: ranks share the GPU, collectives host-staged
set -u
O=gpurun_out/mr
mkdir -p $O
for n in 2 4 8; do
  OSP_BENCH_HOST_COLLECTIVES=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 2 --warmup 1 --config cfg2 \
    --no-cpu > $O/bench_n$n.jsonl 2> $O/bench_n$n.err; echo "n=$n rc=$?"
done
