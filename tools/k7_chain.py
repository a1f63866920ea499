"""The decode step's GEMM chain alone: per layer K7 qkv -> o_proj -> gate|up(+SiLU) -> down
at the 8B shape, 16 stacked activation rows, L layers of distinct weights (> L2), launched
back to back with PDL exactly as the native executor does.  Reports us per layer against
the weight-streaming floor, i.e. how much of the step K7's launch boundaries cost.

python tools/k7_chain.py [--layers 12] [--norm]   (--norm: a residual_rmsnorm between GEMMs
as in the real step)
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_23049_b200 import _native as nat  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=12)
ap.add_argument("--norm", action="store_true")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

d, F, nq, R = 4096, 14336, 6144, 8
L = args.layers
g = torch.Generator(device="cuda").manual_seed(0)


def w(n, k):
    return (torch.rand(n, k, device="cuda", generator=g) * 0.02 - 0.01).to(torch.bfloat16)


layers = [dict(qkv=w(nq, d), o=w(d, d), gu=w(2 * F, d), down=w(d, F)) for _ in range(L)]
x = torch.randn(2 * R, d, device="cuda").to(torch.bfloat16)
attn = torch.randn(2 * R, d, device="cuda").to(torch.bfloat16)
act = torch.empty(2 * R, F, device="cuda", dtype=torch.bfloat16)
y1 = torch.empty(R, nq, device="cuda")
y2 = torch.empty(R, d, device="cuda")
y4 = torch.empty(R, d, device="cuda")
xr = torch.zeros(R, d, device="cuda")
h = torch.empty(2 * R, d, device="cuda", dtype=torch.bfloat16)
ones = torch.ones(d, device="cuda", dtype=torch.bfloat16)
ws = torch.empty(148 * 2 * 128 * 128, device="cuda")
cnt = torch.zeros(4096, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
nbytes = sum(t.numel() * 2 for t in layers[0].values())


def norm(delta):
    if args.norm:
        nat.residual_rmsnorm(xr.data_ptr(), delta.data_ptr(), nat.F32, 0, ones.data_ptr(), nat.BF16,
                             R, d, 1e-6, h.data_ptr(), nat.BF16, 1, None, 0, s)


def chain():
    for lw in layers:
        norm(y4)
        nat.linear_skinny(x.data_ptr(), 2 * R, 1, lw["qkv"].data_ptr(), nq, d, y1.data_ptr(),
                          ws.data_ptr(), cnt.data_ptr(), 0, s)
        nat.linear_skinny(attn.data_ptr(), 2 * R, 1, lw["o"].data_ptr(), d, d, y2.data_ptr(),
                          ws.data_ptr(), cnt.data_ptr(), 0, s)
        norm(y2)
        nat.linear_gate_up_silu(x.data_ptr(), 2 * R, 1, lw["gu"].data_ptr(), F, d, act.data_ptr(),
                                ws.data_ptr(), cnt.data_ptr(), s)
        nat.linear_skinny(act.data_ptr(), 2 * R, 1, lw["down"].data_ptr(), d, F, y4.data_ptr(),
                          ws.data_ptr(), cnt.data_ptr(), 0, s)


chain()
torch.cuda.synchronize()
ts = []
for _ in range(args.reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(1_000_000)
    a.record()
    chain()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3 / L)
ts.sort()
peak = 6560.0
floor = nbytes / peak / 1e3
print(f"env K7_SMEM={os.environ.get('CHOREO_K7_SMEM_KB', '-')} KSUB={os.environ.get('CHOREO_K7_KSUB', '-')} "
      f"norm={args.norm}: {ts[len(ts) // 2]:.1f} us/layer (min {ts[0]:.1f}), weight floor "
      f"{floor:.1f} us ({nbytes / 1e6:.0f} MB) -> {floor / ts[len(ts) // 2]:.3f} of HBM peak")
