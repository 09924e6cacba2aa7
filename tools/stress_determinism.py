"""Repeat K2 / K3 on fixed inputs and compare every run with the first: the forward, dK and dV
must be bitwise identical (fixed accumulation order), dQ equal up to fp32 reduction-order noise.
A pipeline race shows up as an occasional large deviation."""
import argparse
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2605_28691_b200 import kernels

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=40)
ap.add_argument("--L", type=int, default=8736)
ap.add_argument("--heads", type=int, default=12)
a = ap.parse_args()
torch.manual_seed(0)
n, L, H, d = 4, a.L, a.heads, 128
C = H * d
qkv = torch.randn(n, L, 3 * C, device="cuda").bfloat16()
q, k, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
do = torch.randn(n, L, C, device="cuda").bfloat16()
lens = torch.tensor([L, L - 1, L - 77, L // 2 + 3], dtype=torch.int32, device="cuda")
sc = 1 / math.sqrt(d)
bad = 0
ref = None
for r in range(a.reps):
    o, lse = kernels.attn_fwd(q, k, v, H, d, None, False, sc, seq_lens=lens)
    dq, dk, dv = kernels.attn_bwd(q, k, v, o, do, lse, H, d, None, False, sc, seq_lens=lens)
    cur = (o.clone(), lse.clone(), dq.clone(), dk.clone(), dv.clone())
    if ref is None:
        ref = cur
        continue
    same = [torch.equal(x, y) for x, y in zip(cur, ref)]
    dq_err = (cur[2].float() - ref[2].float()).abs().max().item() / ref[2].float().abs().max().item()
    if not (same[0] and same[1] and same[3] and same[4]) or dq_err > 1e-2:
        bad += 1
        print(f"rep {r}: o/lse/dk/dv identical {same[0]} {same[1]} {same[3]} {same[4]}, dq rel dev {dq_err:.2e}")
print(f"{a.reps} reps, {bad} deviating")

# K6 projection (CTA-pair GEMM + norm/RoPE epilogue) and the gather-mode attention
from paper_2605_28691_b200 import GridShape, SparsePattern, pad_grid
from paper_2605_28691_b200.compact import gather_plan
from paper_2605_28691_b200.prologue import qkv_project

g = GridShape(21, 30, 52, 2)
pg = pad_grid(g)
x = torch.randn(pg.padded.seq_len, C, device="cuda").bfloat16()
bad = 0
refp = None
for r in range(a.reps // 2):
    outs = [qkv_project(x, pg.padded, SparsePattern.TOKEN_WISE, 1, norm, rope=True)
            for norm in (None, "head", "channel")]
    if refp is None:
        refp = outs
        continue
    for name, u, w in zip(("plain", "head", "channel"), outs, refp):
        if not torch.equal(u, w):
            dev = ((u.float() - w.float()).abs() / (w.float().abs() + 1e-3)).max().item()
            print(f"K6 {name}: rep {r} deviates, max rel {dev:.2e}")
            bad += name != "channel" or dev > 2 ** -6   # channel: fp32 sum-of-squares order
print(f"K6: {a.reps // 2} reps, {bad} deviating")
plan = gather_plan(g, SparsePattern.GROUP_WISE, 1, pg, "original")
xs = torch.randn(plan.n_rows, 3 * C, device="cuda").bfloat16()
qg, kg, vg = xs[:, :C], xs[:, C:2 * C], xs[:, 2 * C:]
dog = torch.randn(plan.n_rows, C, device="cuda").bfloat16()
bad = 0
refg = None
for r in range(a.reps // 2):
    o, lse = kernels.attn_fwd_gather(qg, kg, vg, H, d, plan.row_index, plan.lens, sc)
    dq, dk, dv = kernels.attn_bwd_gather(qg, kg, vg, o, dog, lse, H, d, plan.row_index, plan.lens, sc)
    cur = (o.clone(), dk.clone(), dv.clone(), dq.float())
    if refg is None:
        refg = cur
        continue
    if not (torch.equal(cur[0], refg[0]) and torch.equal(cur[1], refg[1]) and torch.equal(cur[2], refg[2])
            and torch.allclose(cur[3], refg[3], rtol=2 ** -6, atol=1e-6)):
        bad += 1
print(f"gather mode: {a.reps // 2} reps, {bad} deviating")
