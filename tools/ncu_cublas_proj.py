"""Three cfg3-shaped cuBLAS projection GEMMs (x @ [Wq|Wk|Wv]) for an ncu comparison with K6."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

x = torch.randn(80640, 5120, device="cuda").to(torch.bfloat16)
w = torch.randn(5120, 15360, device="cuda").to(torch.bfloat16)
for _ in range(3):
    torch.matmul(x, w)
torch.cuda.synchronize()
print("ok")
