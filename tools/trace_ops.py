"""torch.profiler trace of one benched block step (orig -> orig fwd+bwd): which host ops launch
which kernels (finds stray torch kernels inside the step)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from bench import CONFIGS
from paper_2605_28691_b200 import GridShape
from paper_2605_28691_b200.block import SkiparseBlock

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
T, H, W, k, heads, d, _ = CONFIGS[cfg]
blk = SkiparseBlock(GridShape(T, H, W, k), heads, heads * d)
x = torch.randn(1, T * H * W, heads * d, device="cuda").bfloat16().requires_grad_(True)
gy = torch.randn_like(x)
for _ in range(2):
    x.grad = None
    blk.forward_original(x).backward(gy)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA],
                            record_shapes=True, with_stack=True) as prof:
    x.grad = None
    blk.forward_original(x).backward(gy)
    torch.cuda.synchronize()
print(prof.key_averages(group_by_stack_n=6).table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
