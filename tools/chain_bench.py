"""K8 layer chain microbenchmark at the Llama-3.1-8B layer shape (one CTA per SM).

python tools/chain_bench.py [--rows 8] [--phases 15] [--iters 20] [--k7]

Times back-to-back launches of choreo_layer_chain with CUDA events (weights 438 MB per
full layer > L2, so every launch streams from HBM) and reports us / GB/s per launch for the
full chain and for each phase alone; --k7 adds the per-GEMM K7 launches at the same shapes.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_23049_b200 import _native as nat  # noqa: E402
from tests.test_gpu_chain import _Bufs, _Layer, _rope_tables  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=8)
ap.add_argument("--phases", type=int, default=-1)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--k7", action="store_true")
args = ap.parse_args()

d, H, Hk, hd, F = 4096, 32, 8, 128, 14336
R, split = args.rows, True
lw = _Layer(d, H, Hk, hd, F, seed=1)
b = _Bufs(R, d, H, Hk, hd, F, split, n_pages=16)
W = 8192
cos_t, sin_t = _rope_tables(hd, W)
pos = torch.arange(R, dtype=torch.int32, device="cuda") + 100
page = torch.zeros(R, dtype=torch.int32, device="cuda")
slot = torch.arange(R, dtype=torch.int32, device="cuda")
b.x.normal_()
b.attn.normal_()
b.h_a.normal_()
b.h_b.normal_()
b.act.normal_()
b.ssq_a.fill_(float(d))
b.ssq_b.fill_(float(d))
stream = torch.cuda.current_stream().cuda_stream
wbytes = {1: lw.wo.numel() * 2, 2: lw.w_gu.numel() * 2, 4: lw.w_down.numel() * 2,
          8: lw.w_qkv.numel() * 2}


_structs = {}


def launch(phases):
    if phases not in _structs:
        _structs[phases] = _make(phases)
    nat.layer_chain(ctypes.byref(_structs[phases]), stream)


def _make(phases):
    return nat.LayerChain(n_rows=R, split=1, d=d, n_heads=H, n_kv=Hk, head_dim=hd, ffn_dim=F,
                       eps=1e-6, phases=phases, wo=lw.wo.data_ptr(), ffn_norm=lw.g_ffn.data_ptr(),
                       w_gu=lw.w_gu.data_ptr(), w_down=lw.w_down.data_ptr(),
                       attn_norm_next=lw.g_attn.data_ptr(), w_qkv=lw.w_qkv.data_ptr(),
                       layer_qkv=0, x=b.x.data_ptr(), attn=b.attn.data_ptr(), h_a=b.h_a.data_ptr(),
                       act=b.act.data_ptr(), h_b=b.h_b.data_ptr(), ssq_a=b.ssq_a.data_ptr(),
                       ssq_b=b.ssq_b.data_ptr(), q=b.q.data_ptr(), k_pool=b.k_pool.data_ptr(),
                       v_pool=b.v_pool.data_ptr(), n_pages=b.k_pool.shape[2], page_size=64,
                       pos=pos.data_ptr(), page=page.data_ptr(), slot=slot.data_ptr(),
                       cos_t=cos_t.data_ptr(), sin_t=sin_t.data_ptr(), max_delta=W,
                       ws=b.ws.data_ptr(), counters=b.counters.data_ptr(),
                       done=b.done.data_ptr())


def timed(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(n):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1e3 / n


peak = 6551.0
out = []
for ph in ([args.phases] if args.phases > 0 else [15, 1, 2, 4, 8]):
    us = timed(lambda: launch(ph), args.iters)
    nb = sum(v for k, v in wbytes.items() if ph & k)
    out.append({"phases": ph, "rows": R, "us": round(us, 2), "weight_MB": round(nb / 1e6, 1),
                "GBs": round(nb / us / 1e3, 1), "frac": round(nb / us / 1e3 / peak, 4)})
if args.k7:
    ws = torch.empty(148 * 2 * 128 * 128, device="cuda")
    cnt = torch.zeros(2048, dtype=torch.int32, device="cuda")
    y = torch.empty(R, 2 * F, device="cuda")
    for name, w, xb in (("o", lw.wo, b.attn), ("gu", lw.w_gu, b.h_a), ("down", lw.w_down, b.act),
                        ("qkv", lw.w_qkv, b.h_b)):
        us = timed(lambda: nat.linear_skinny(xb.data_ptr(), 2 * R, 1, w.data_ptr(), w.shape[0],
                                             w.shape[1], y.data_ptr(), ws.data_ptr(),
                                             cnt.data_ptr(), 0, stream), args.iters)
        nb = w.numel() * 2
        out.append({"k7": name, "us": round(us, 2), "GBs": round(nb / us / 1e3, 1),
                    "frac": round(nb / us / 1e3 / peak, 4)})
for r in out:
    print(json.dumps(r))
