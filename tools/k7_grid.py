"""K7 launch-shape study: per-shape time vs grid (tile cuts between CTAs or not)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import kernel_bench as kb
from paper_2512_23049_b200 import _native as nat
stream = torch.cuda.current_stream().cuda_stream
ws = torch.empty(148 * 2 * 128 * 128, device="cuda")
R = int(os.environ.get("K7_ROWS", "8"))  # output rows (split hi/lo: 2R stacked)
for name, n, k in (("qkv", 6144, 4096), ("o", 4096, 4096), ("gu", 28672, 4096), ("down", 4096, 14336)):
    ncopy = max(2, int(400e6 // (n * k * 2)) + 1)
    wl = [torch.randn(n, k, device="cuda").to(torch.bfloat16) for _ in range(ncopy)]
    x = torch.randn(2 * R, k, device="cuda").to(torch.bfloat16)
    y = torch.empty(R, n, device="cuda")
    cnt = torch.zeros((n + 127) // 128, dtype=torch.int32, device="cuda")
    for grid in (148, 128, 112, 96, 74, 64, 32):
        it = [0]
        def run():
            w = wl[it[0] % ncopy]; it[0] += 1
            nat.linear_skinny(x.data_ptr(), 2 * R, 1, w.data_ptr(), n, k, y.data_ptr(), ws.data_ptr(),
                              cnt.data_ptr(), grid, stream)
        t = kb._time(run, burst=ncopy)
        print(f"{name} grid={grid} us={t*1e6:.2f} GB/s={n*k*2/t/1e9:.0f}", flush=True)
    del wl
    torch.cuda.empty_cache()
