"""Per-launch time of the attention kernels under sustained load (several seconds of
back-to-back launches) with nvidia-smi clocks / power sampled alongside: separates the
kernels' cold speed from their power-capped steady state."""
import argparse
import math
import subprocess
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from bench import CONFIGS
from paper_2605_28691_b200 import kernels

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--kernel", default="fwd", choices=["fwd", "bwd", "both"])
ap.add_argument("--seconds", type=float, default=6.0)
ap.add_argument("--masked", action="store_true", help="use the padded grid's TSA key mask")
a = ap.parse_args()
T, H, W, k, heads, d, _ = CONFIGS[a.config]
k2 = k * k
Hp, Wp = -(-H // k2) * k2, -(-W // k2) * k2
L = T * Hp * Wp // k2
C = heads * d
qkv = torch.randn(k2, L, 3 * C, device="cuda").bfloat16()
q, kk, v = qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:]
do = torch.randn(k2, L, C, device="cuda").bfloat16()
sc = 1 / math.sqrt(d)
bits = None
if a.masked:
    from paper_2605_28691_b200 import GridShape, SparsePattern, pad_grid
    bits = pad_grid(GridShape(T, H, W, k)).mask_bits(SparsePattern.TOKEN_WISE, 1)
o, lse = kernels.attn_fwd(q, kk, v, heads, d, bits, bits is not None, sc)

samples = []
stop = False


def sampler():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True)
        samples.append((time.time(), r.stdout.strip()))
        time.sleep(0.2)


th = threading.Thread(target=sampler, daemon=True)
th.start()
t_end = time.time() + a.seconds
times = []
while time.time() < t_end:
    for name in (["fwd", "bwd"] if a.kernel == "both" else [a.kernel]):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if name == "fwd":
            kernels.attn_fwd(q, kk, v, heads, d, bits, bits is not None, sc)
        else:
            kernels.attn_bwd(q, kk, v, o, do, lse, heads, d, bits, bits is not None, sc)
        e1.record()
        e1.synchronize()
        times.append((time.time(), name, e0.elapsed_time(e1)))
stop = True
th.join()
t0 = times[0][0]
for name in ("fwd", "bwd"):
    ts = [(t - t0, ms) for t, n, ms in times if n == name]
    if not ts:
        continue
    n = len(ts)
    print(f"{name}: first {ts[0][1]:.2f} ms, median of first 3 {sorted(x[1] for x in ts[:3])[1]:.2f}, "
          f"last-half median {sorted(x[1] for x in ts[n // 2:])[len(ts[n // 2:]) // 2]:.2f} ms over {n}")
for t, s in samples[::3]:
    print(f"  t={t - t0:5.1f}s  sm_mhz,power_w,temp = {s}")
