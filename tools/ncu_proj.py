"""Three cfg3 K6 projection launches (plain) for ncu captures."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2605_28691_b200 import GridShape, SparsePattern, pad_grid
from paper_2605_28691_b200.prologue import packed_projection_t, qkv_project
g = pad_grid(GridShape(21, 45, 80, 2)).padded
C = 5120
x = torch.randn(g.seq_len, C, device="cuda").to(torch.bfloat16)
for _ in range(3):
    qkv_project(x.view(4, -1, C), g, SparsePattern.TOKEN_WISE, 1)
torch.cuda.synchronize()
print("ok")
