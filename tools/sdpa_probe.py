"""One attention launch at a config's subsequence shape, for ncu captures side by side:
`--impl ours` (K2 / K3) or `--impl cudnn` (torch SDPA, cuDNN backend).  No mask, bf16."""

import argparse
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", default="ours", choices=["ours", "cudnn"])
    ap.add_argument("--what", default="fwd", choices=["fwd", "bwd"])
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--L", type=int, default=20160)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    C = a.heads * a.d
    qkv = torch.randn(a.n, a.L, 3 * C, device="cuda").to(torch.bfloat16)
    do = torch.randn(a.n, a.L, C, device="cuda").to(torch.bfloat16)
    q, k, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
    sc = 1 / math.sqrt(a.d)
    if a.impl == "ours":
        from paper_2605_28691_b200 import kernels
        for _ in range(a.reps):
            o, lse = kernels.attn_fwd(q, k, v, a.heads, a.d, None, False, sc)
            if a.what == "bwd":
                kernels.attn_bwd(q, k, v, o, do, lse, a.heads, a.d, None, False, sc)
    else:
        import torch.nn.functional as F
        from torch.nn.attention import SDPBackend, sdpa_kernel
        qs, ks, vs = (t.reshape(a.n, a.L, a.heads, a.d).transpose(1, 2).detach().requires_grad_(a.what == "bwd")
                      for t in (q, k, v))
        dos = do.reshape(a.n, a.L, a.heads, a.d).transpose(1, 2)
        for _ in range(a.reps):
            with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                y = F.scaled_dot_product_attention(qs, ks, vs)
            if a.what == "bwd":
                torch.autograd.grad(y, (qs, ks, vs), dos)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
