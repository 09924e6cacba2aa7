"""CUDA-graph capture of the benched block step (orig -> orig fwd + bwd) for launch-bound shapes:
eager vs replayed graph, same inputs, same results."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from bench import CONFIGS
from paper_2605_28691_b200 import GridShape
from paper_2605_28691_b200.block import SkiparseBlock

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg1")
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
T, H, W, k, heads, d, _ = CONFIGS[a.config]
blk = SkiparseBlock(GridShape(T, H, W, k), heads, heads * d)
S, C = T * H * W, heads * d
x = torch.randn(1, S, C, device="cuda").bfloat16().requires_grad_(True)
gy = torch.randn_like(x)


def step():
    x.grad = None
    y = blk.forward_original(x)
    y.backward(gy)
    return y


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


eager_ms = timeit(step)
y_ref = step().detach().clone()
dx_ref = x.grad.detach().clone()
# capture: warm up on a side stream, then record one step (static input / output buffers)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
x.grad = None
with torch.cuda.graph(g):
    y_g = blk.forward_original(x)
    y_g.backward(gy)
graph_ms = timeit(g.replay)
g.replay()
torch.cuda.synchronize()
same = torch.equal(y_g, y_ref) and torch.allclose(x.grad.float(), dx_ref.float(), rtol=1e-2, atol=1e-3)
print(f"{a.config}: eager {eager_ms:.3f} ms/step, graph {graph_ms:.3f} ms/step "
      f"({S / graph_ms * 1e3:.0f} tokens/s), outputs match: {same}")
