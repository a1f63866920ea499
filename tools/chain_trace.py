"""K8 chain timeline: per-CTA globaltimer stamps from a -DCHOREO_TRACE build of the library.

Build (in the build container):  python tools/chain_trace.py --build
Run (on the GPU):               python tools/chain_trace.py [--rows 8] [--phases 15]
Prints, per phase, the spread over CTAs of: first weight TMA issue, inputs ready (after the
dependency wait), first MMA, last MMA, last tile epilogue done -- in us from the earliest
CTA start.
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tools", "_trace", "_choreo_b200.so")

ap = argparse.ArgumentParser()
ap.add_argument("--build", action="store_true")
ap.add_argument("--rows", type=int, default=8)
ap.add_argument("--phases", type=int, default=15)
args = ap.parse_args()

if args.build:
    from paper_2512_23049_b200 import build as B
    objs = []
    for src in B.sources():
        obj = os.path.join(ROOT, "tools", "_trace", os.path.basename(src)[:-3] + ".o")
        subprocess.run(["nvcc", *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                        "--expt-relaxed-constexpr", "-DCHOREO_TRACE", "-I",
                        os.path.join(ROOT, "include"), "-c", src, "-o", obj], check=True)
        objs.append(obj)
    subprocess.run(["nvcc", *B.ARCH, "-shared", "-o", OUT, *objs, "-lcuda"], check=True)
    print("built", OUT)
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_23049_b200 import _native as nat  # noqa: E402

nat.LIB_PATH = OUT
lib = nat.load()
sys.argv = [sys.argv[0], "--rows", str(args.rows), "--phases", str(args.phases), "--iters", "3"]
import tools.chain_bench as cb  # noqa: E402  (runs its own timing once)

tr = torch.zeros(148 * 48, dtype=torch.int64, device="cuda")
lib.choreo_chain_set_trace.argtypes = [ctypes.c_void_p]
assert lib.choreo_chain_set_trace(tr.data_ptr()) == 0
cb.launch(args.phases)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(148, 48).astype(np.float64)
t0 = t[:, 0][t[:, 0] > 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
names = ["w_first", "x_ready", "mma_first", "mma_last", "epi_last"]
print(f"start: med {np.nanmedian(rel[:, 0]):.2f} max {np.nanmax(rel[:, 0]):.2f} us; "
      f"end: med {np.nanmedian(rel[:, 25]):.2f} max {np.nanmax(rel[:, 25]):.2f}")
for ph, pn in enumerate(["o", "gu", "down", "qkv"]):
    cols = rel[:, 1 + ph * 6: 6 + ph * 6]
    if np.all(np.isnan(cols)):
        continue
    print(pn.ljust(5) + "  ".join(f"{n}: {np.nanmin(cols[:, i]):7.2f}/{np.nanmedian(cols[:, i]):7.2f}/"
                                  f"{np.nanmax(cols[:, i]):7.2f}" for i, n in enumerate(names)))
    ep = rel[:, 26 + ph * 4: 30 + ph * 4]
    if ph == 2:
        print("      down final: v ready %.2f  after x/h stores %.2f" % (np.nanmedian(rel[:, 42]), np.nanmedian(rel[:, 43])))
    if ph == 3:
        print("      qkv final: v ready %.2f" % np.nanmedian(rel[:, 45]))
    print("      last segment: " + "  ".join(
        f"{n}: {np.nanmin(ep[:, i]):7.2f}/{np.nanmedian(ep[:, i]):7.2f}/{np.nanmax(ep[:, i]):7.2f}"
        for i, n in enumerate(["acc_full", "pieces_in", "final", "published"])))
