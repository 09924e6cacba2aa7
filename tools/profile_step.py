"""One Skiparse-2D block fwd+bwd (after one warm-up step) for ncu captures."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from bench import CONFIGS
from paper_2605_28691_b200 import GridShape
from paper_2605_28691_b200.block import SkiparseBlock

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
T, H, W, k, heads, d, _ = CONFIGS[a.config]
blk = SkiparseBlock(GridShape(T, H, W, k), heads, heads * d)
x = torch.randn(blk.local_rows, blk.L, heads * d, device="cuda").bfloat16().requires_grad_(True)
gy = torch.randn_like(x)
for _ in range(a.steps):
    x.grad = None
    blk(x).backward(gy)
torch.cuda.synchronize()
print("ok")
