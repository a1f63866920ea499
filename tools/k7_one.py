"""One K7 shape launched a few times (for ncu): K7_ROWS output rows (split hi/lo), K7_N x K7_K."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2512_23049_b200 import _native as nat
rows, n, k = (int(os.environ.get(v, d)) for v, d in (("K7_ROWS", "72"), ("K7_N", "4096"), ("K7_K", "4096")))
x = torch.randn(2 * rows, k, device="cuda").to(torch.bfloat16)
w = torch.randn(n, k, device="cuda").to(torch.bfloat16)
y = torch.empty(rows, n, device="cuda")
ws = torch.empty(148 * 2 * 256 * 128, device="cuda")
cnt = torch.zeros(n // 128 + 1, dtype=torch.int32, device="cuda")
for _ in range(6):
    nat.linear_skinny(x.data_ptr(), 2 * rows, 1, w.data_ptr(), n, k, y.data_ptr(), ws.data_ptr(),
                      cnt.data_ptr(), 0, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
