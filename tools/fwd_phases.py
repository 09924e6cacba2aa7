"""Per-tile phase cycles of the K2 forward from an instrumented build (-DOSP_FWD_TIMING=1,
loaded with OSP_LIB=...): softmax warpgroups (wait S, TMEM load, MUFU turn, exps, max/redo,
P hand-off) and the MMA issuer (waits for K, P1, V, P0)."""
import ctypes
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_28691_b200 import _lib, kernels  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 20160
n, heads, d = int(sys.argv[2]) if len(sys.argv) > 2 else 4, 40, 128
C = heads * d
qkv = torch.randn(n, L, 3 * C, device="cuda").bfloat16()
q, k, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
lib = _lib.lib()
kernels.attn_fwd(q, k, v, heads, d, None, False, 1 / math.sqrt(d))
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 64)()
lib.osp_debug_counters(buf, 64, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
kernels.attn_fwd(q, k, v, heads, d, None, False, 1 / math.sqrt(d))
e1.record()
torch.cuda.synchronize()
lib.osp_debug_counters(buf, 64, 0)
c = list(buf)
print(f"fwd {e0.elapsed_time(e1):.2f} ms")
names = ["wait S", "ld S", "MUFU turn", "exps", "max/redo", "P handoff"]
for t in range(2):
    tiles = max(c[t * 8 + 7], 1)
    tot = sum(c[t * 8 + i] for i in range(6))
    print(f"softmax WG{t}: cycles/tile " + ", ".join(f"{nm} {c[t * 8 + i] / tiles:.0f}" for i, nm in enumerate(names))
          + f"  | total {tot / tiles:.0f}")
tiles = max(c[20], 1)
mn = ["wait K", "wait P1", "wait V", "wait P0"]
print("MMA issuer: cycles/tile " + ", ".join(f"{nm} {c[16 + i] / tiles:.0f}" for i, nm in enumerate(mn)))
ctas = max(c[27], 1)
print(f"per CTA ({c[27]} CTAs, {c[20] / ctas:.1f} key tiles each): prologue {c[24] / ctas:.0f}, "
      f"loop {c[25] / ctas:.0f}, epilogue {c[26] / ctas:.0f} cycles")
