"""One Skiparse-2D block fwd+bwd (after one warm-up step) for ncu captures: the orig -> orig
step bench.py times at N=1, or the token-wise block with --tsa."""
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
ap.add_argument("--tsa", action="store_true", help="token-wise steady-state block instead of orig -> orig")
a = ap.parse_args()
T, H, W, k, heads, d, _ = CONFIGS[a.config]
blk = SkiparseBlock(GridShape(T, H, W, k), heads, heads * d)
shape = (blk.local_rows, blk.L, heads * d) if a.tsa else (1, T * H * W, heads * d)
fn = blk if a.tsa else blk.forward_original      # bench.py's N=1 step by default
x = torch.randn(shape, device="cuda").bfloat16().requires_grad_(True)
gy = torch.randn_like(x)
for _ in range(a.steps):
    x.grad = None
    fn(x).backward(gy)
torch.cuda.synchronize()
print("ok")
