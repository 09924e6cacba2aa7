"""K6 projection GEMM (+ QK-RMSNorm + RoPE epilogue) vs cuBLAS at a config's shape."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from bench import CONFIGS
from paper_2605_28691_b200 import GridShape, SparsePattern, pad_grid
from paper_2605_28691_b200.attention import packed_projection
from paper_2605_28691_b200.prologue import packed_projection_t, qkv_project

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
T, H, W, k, heads, d, _ = CONFIGS[a.config]
g = pad_grid(GridShape(T, H, W, k)).padded
C = heads * d
rows = g.seq_len
x = torch.randn(rows, C, device="cuda").to(torch.bfloat16)
Wp = packed_projection(C, torch.bfloat16, "cuda")
packed_projection_t(C, "cuda")
gq = torch.ones(C, device="cuda")
flop = 2 * rows * C * 3 * C


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


res = {"cublas (torch.matmul)": timeit(lambda: torch.matmul(x, Wp))}
for name, kw in [("K6 plain", {}), ("K6 + head norm + rope", {"norm": "head", "rope": True}),
                 ("K6 + channel norm + rope", {"norm": "channel", "rope": True})]:
    res[name] = timeit(lambda: qkv_project(x.view(k * k, -1, C), g, SparsePattern.TOKEN_WISE, 1,
                                           gamma_q=gq if kw.get("norm") else None,
                                           gamma_k=gq if kw.get("norm") else None, **kw))
for n, ms in res.items():
    print(f"{a.config} {n:28s} {ms:7.3f} ms  {flop / ms / 1e9:7.1f} TFLOP/s")
