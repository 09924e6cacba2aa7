"""Time attention fwd / bwd launches alone at a config's shape (CUDA events)."""
import argparse
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from bench import CONFIGS
from paper_2605_28691_b200 import kernels

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--what", default="fwd,bwd")
a = ap.parse_args()
T, H, W, k, heads, d, _ = CONFIGS[a.config]
k2 = k * k
Hp, Wp = -(-H // k2) * k2, -(-W // k2) * k2
L = T * Hp * Wp // k2
n = k2
C = heads * d
qkv = torch.randn(n, L, 3 * C, device="cuda").bfloat16()
q, kk, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
do = torch.randn(n, L, C, device="cuda").bfloat16()
sc = 1 / math.sqrt(d)
fl = 4 * n * L * L * d * heads
for name in a.what.split(","):
    o, lse = kernels.attn_fwd(q, kk, v, heads, d, None, False, sc)
    ts = []
    for r in range(a.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if name == "fwd":
            kernels.attn_fwd(q, kk, v, heads, d, None, False, sc)
        else:
            kernels.attn_bwd(q, kk, v, o, do, lse, heads, d, None, False, sc)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    f = fl * (2.5 if name == "bwd" else 1.0)
    ms = min(ts)
    print(f"{a.config} {name}: {ms:.3f} ms  {f / ms / 1e9:.1f} TFLOP/s")
