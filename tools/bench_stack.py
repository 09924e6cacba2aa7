"""Hybrid-stack throughput (BASELINE.json config 5): a Skiparse DiT
attention stack (FULL blocks at both ends, alternating TSA/GSA in the middle) forward+backward
on one B200.  Prints one JSON line (not the bench.py headline metric)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from bench import CONFIGS
from paper_2605_28691_b200 import GridShape
from paper_2605_28691_b200.stack import HybridStack

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5k2")
ap.add_argument("--layers", type=int, default=6)
ap.add_argument("--full", type=int, default=2)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=1)
a = ap.parse_args()
T, H, W, k, heads, d, desc = CONFIGS[a.config]
st = HybridStack(GridShape(T, H, W, k), heads, heads * d, num_layers=a.layers, n_full=a.full)
x = torch.randn(st.local_rows, st.L, heads * d, device="cuda").bfloat16().requires_grad_(True)
gy = torch.randn_like(x)
for _ in range(a.warmup):
    x.grad = None
    st(x).backward(gy)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    x.grad = None
    st(x).backward(gy)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
fl = st.flops()
print(json.dumps({"metric": "hybrid Skiparse stack tokens/s fwd+bwd", "config": a.config,
                  "description": desc, "schedule": [s.value for s in st.schedule],
                  "tokens_per_step": T * H * W, "ms_per_step": ms,
                  "value": T * H * W / (ms / 1e3), "unit": "tokens/s",
                  "attention_tflops": fl["attention_fwd_bwd"] / (ms / 1e3) / 1e12}))
