"""Per-query-tile wait cycles of the K3 backward's MMA issuer from an instrumented build
(-DOSP_BWD_TIMING=1, loaded with OSP_LIB=...): waits for P (softmax), the next Q/dO stage, dS, and
the dQ TMEM buffer being drained."""
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
do = torch.randn(n, L, C, device="cuda").bfloat16()
q, k, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
sc = 1 / math.sqrt(d)
lib = _lib.lib()
o, lse = kernels.attn_fwd(q, k, v, heads, d, None, False, sc)
kernels.attn_bwd(q, k, v, o, do, lse, heads, d, None, False, sc)
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 64)()
lib.osp_debug_counters_bwd(buf, 64, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
kernels.attn_bwd(q, k, v, o, do, lse, heads, d, None, False, sc)
e1.record()
torch.cuda.synchronize()
lib.osp_debug_counters_bwd(buf, 64, 0)
c = list(buf)
tiles = max(c[7], 1)
print(f"bwd {e0.elapsed_time(e1):.2f} ms, {tiles} query tiles over all CTAs")
names = ["wait P", "wait next Q/dO", "wait dS", "wait dQ drained"]
print("MMA issuer cycles per query tile: " + ", ".join(f"{nm} {c[i] / tiles:.0f}" for i, nm in enumerate(names)))
ctas = max(c[11], 1)
print(f"per CTA ({c[11]} CTAs, {tiles / ctas:.1f} query tiles each): prologue {c[8] / ctas:.0f}, "
      f"loop {c[9] / ctas:.0f}, epilogue {c[10] / ctas:.0f} cycles")
