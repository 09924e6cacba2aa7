"""K6 prologue (QK-RMSNorm + 3-D RoPE) forward + backward at a config's shape (the backward:
recomputed pre-norm GEMM, the K6b kernel in place on the gradient, dx = g W^T)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from bench import CONFIGS
from paper_2605_28691_b200 import GridShape, SparsePattern, pad_grid
from paper_2605_28691_b200.prologue import QKVPrologue, packed_projection_t

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--norm", default="head")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
T, H, W, k, heads, d, _ = CONFIGS[a.config]
g = pad_grid(GridShape(T, H, W, k)).padded
C = heads * d
x = torch.randn(k * k, g.seq_len // (k * k), C, device="cuda").to(torch.bfloat16).requires_grad_(True)
w_t = packed_projection_t(C, "cuda")
gq = torch.ones(C, device="cuda")


def step():
    x.grad = None
    y = QKVPrologue.apply(x, g, SparsePattern.TOKEN_WISE, 1, a.norm, gq, gq, 1e-6, True, 0, w_t)
    y.backward(torch.ones_like(y))


def timeit(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


print(f"{a.config} prologue fwd+bwd (norm={a.norm}, rope) with K6b: {timeit(step):.2f} ms")
