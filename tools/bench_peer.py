"""K7 peer gather at a config's shape, with N ranks' source slots simulated by N local buffers
(one GPU: the fabric is not exercised, so this bounds the kernel's own efficiency against HBM).
Compared with the NCCL-path local passes it replaces (K4 pack + unpack over the padded shard,
plus the two compaction moves around each switch)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from bench import CONFIGS
from paper_2605_28691_b200 import GridShape, SparsePattern, kernels, pad_grid
from paper_2605_28691_b200.gridseq import IndexMap
from paper_2605_28691_b200.peer import block_switch_moves

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
T, H, W, k, heads, d, _ = CONFIGS[a.config]
g = GridShape(T, H, W, k)
pg = pad_grid(g)
p = pg.padded
C = heads * d
k2 = k * k
L = p.seq_len // k2
local = k2 // a.world
rng = [(j * local, (j + 1) * local) for j in range(a.world)]
pts = [pg.compact_plan(SparsePattern.TOKEN_WISE, 1, r) for r in rng]
pgs = [pg.compact_plan(SparsePattern.GROUP_WISE, 1, r) for r in rng]
t2g = IndexMap._pattern("tsa_to_gsa", p, 1).src.reshape(-1).cuda()
g2t = IndexMap._pattern("gsa_to_tsa", p, 1).src.reshape(-1).cuda()
A, B = block_switch_moves(a.world, 0, local, L, t2g, g2t, pts, pgs)
srcs = [torch.randn(pl.n_seq * pl.cap, C, device="cuda").to(torch.bfloat16) for pl in pts]
ptrs = [s.data_ptr() for s in srcs]
out = torch.empty(A.table.numel(), C, device="cuda", dtype=torch.bfloat16)
real = int((A.table >= 0).sum())
row_bytes = C * 2


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


ms = timeit(lambda: kernels.peer_gather(ptrs, A.stride, A.table, out))
# the local passes of the NCCL path for the same switch: pack + unpack of the padded shard
x = torch.randn(local, L, C, device="cuda").to(torch.bfloat16)
ms_pack = timeit(lambda: kernels.ssp_pack(x, a.world, p.t, p.h, p.w, p.k))
send = kernels.ssp_pack(x, a.world, p.t, p.h, p.w, p.k)
ms_unpack = timeit(lambda: kernels.ssp_unpack(send, a.world, local, p.t, p.h, p.w, p.k))
moved = 2 * real * row_bytes + out.numel() * 2 - real * row_bytes   # reads of real rows + all writes
print(json.dumps({
    "config": a.config, "world": a.world, "rows_out": A.table.numel(), "real_rows": real,
    "remote_rows": A.remote_rows, "peer_gather_ms": ms,
    "peer_gather_GBps": moved / ms / 1e6,
    "nccl_path_local_passes_ms": {"ssp_pack": ms_pack, "ssp_unpack": ms_unpack},
}))
