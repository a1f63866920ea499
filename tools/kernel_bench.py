"""Kernel microbenchmarks at the Llama-3.1-8B shape (SURVEY.md §8(d) roofline rows).

Each returns a dict with the algorithmic work per launch, the CUDA-event time per
launch (median of reps, on the launching stream, after warm-up) and the fraction of
the measured peak (MEASURED_PEAKS.json; burst figures, kernels timed alone).

  k2_rerotate : move 8192 cached tokens (all 32 layers);  bytes = tok*L*Hkv*hd*2B*2
  k4_prefill  : prefill_parallel of 8 messages x 1024 tokens, each over a reordered
                6144-token parent subset of a 32 x 256-token cache;
                FLOPs = 4*hd*Hq*sum_rows |visible(row)| per layer (exact visible pairs)
  k5_decode   : one decode step of N agents over shared parents (page-centric);
                bytes = unique visible KV bytes + q + partials per layer
Usage: python tools/kernel_bench.py [--json]
"""
from __future__ import annotations

import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_23049_b200 import _native as nat  # noqa: E402
from paper_2512_23049_b200.cache import DeviceKvCache, RotationTableDevice, cdiv  # noqa: E402
from paper_2512_23049_b200.config import LLAMA_3_1_8B  # noqa: E402
from paper_2512_23049_b200.model import CallRows, plan_counts  # noqa: E402

K3_TAG = 4242  # the runner's K3 step tag (K5 v2 reads K3's outputs before its dependency wait)


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh) | {"source": "measured"}
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


def _time(fn, reps=20, warm=3, burst=None) -> float:
    """Median per-launch time.  Launches are issued in bursts between one event pair so
    the GPU never idles waiting for host-side submission (which would otherwise dominate
    the event interval of a microsecond-scale kernel)."""
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    if burst is None:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        burst = max(1, min(64, int(2e-3 / max(a.elapsed_time(b) / 1e3, 1e-6))))
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)  # ~1 ms of GPU work so the burst is queued behind it
        a.record(s)
        for _ in range(burst):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / burst)
    return statistics.median(ts)


def _cache(cfg, n_tokens_capacity: int):
    c = DeviceKvCache(cfg, capacity=n_tokens_capacity, dtype=torch.bfloat16, device="cuda")
    c._grow_pool(cdiv(n_tokens_capacity, 64) + 64)
    return c


def _add(cache, mid, n):
    cache.register_message(mid, "prefilled", 0, max_tokens=n)
    cache.reserve_slots(mid, [97] * n)
    cache.log_append(mid, 0, n)


def _assemble(cache, calls, rpb, ppi, mode=0):
    """calls: (own, parents, first_t, n_rows)."""
    tab, par, row_t, off = [], [], [], 0
    cr = []
    for own, parents, t0, n in calls:
        tab += [own, len(par), len(parents), off, n]
        par += parents
        row_t += list(range(t0, t0 + n))
        off += n
        cr.append(CallRows(own, parents, t0, [0] * n, None, None, 0))
    plan = plan_counts(cr, cache.msg_len.host, 64, rpb, ppi, mode)
    cache.sync_tables()
    dev = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")  # noqa: E731
    tab_d, par_d, rt_d = dev(tab), dev(par + [0]), dev(row_t)
    R = len(row_t)
    bufs = dict(vis=torch.empty(3, plan.n_vis, dtype=torch.int32, device="cuda"),
                blk=torch.empty(plan.n_blk_rows, dtype=torch.int32, device="cuda"),
                items=torch.empty(plan.n_items, 6, dtype=torch.int32, device="cuda"),
                rpo=torch.empty(R + 1, dtype=torch.int32, device="cuda"),
                rp=torch.empty(plan.n_parts, dtype=torch.int32, device="cuda"),
                counts=torch.zeros(6, dtype=torch.int32, device="cuda"), rt=rt_d,
                fat=torch.empty(max(plan.n_items, 1), 64, dtype=torch.int32, device="cuda"),
                order=torch.empty(max(plan.n_items, 1), dtype=torch.int32, device="cuda"))
    v = bufs["vis"]
    nat.assemble_ex(cache.msg_len.dev.data_ptr(), cache.msg_pt.dev.data_ptr(),
                 cache.page_table.dev.data_ptr(), tab_d.data_ptr(), par_d.data_ptr(), len(calls),
                 rt_d.data_ptr(), R, None, 0, 64, rpb, ppi, v[0].data_ptr(), v[1].data_ptr(),
                 v[2].data_ptr(), bufs["blk"].data_ptr(), bufs["items"].data_ptr(),
                 bufs["rpo"].data_ptr(), bufs["rp"].data_ptr(), bufs["counts"].data_ptr(),
                 plan.n_vis, plan.n_blk_rows, plan.n_items, plan.n_parts, mode,
                 bufs["fat"].data_ptr(), bufs["order"].data_ptr(), mode == 0 and K3_TAG,
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert int(bufs["counts"][3]) == 0
    return plan, bufs, R


def k2_rerotate(tokens: int = 8192) -> dict:
    cfg = LLAMA_3_1_8B
    cache = _cache(cfg, tokens + 1024)
    for m in range(tokens // 256):
        _add(cache, m, 256)
    cache.k_pool.normal_()
    rot = RotationTableDevice(cfg, "cuda")
    pages = [pg for m in range(tokens // 256) for pg in cache._messages[m].pages]
    arr = torch.tensor([pages, [64] * len(pages), [37] * len(pages)], dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream

    def run():
        nat.rerotate(cache.k_pool.data_ptr(), nat.BF16, cfg.n_layers, cfg.kv_heads, cache.n_pages, 64,
                     cfg.head_dim, arr[0].data_ptr(), arr[1].data_ptr(), arr[2].data_ptr(),
                     len(pages), rot.cos.data_ptr(), rot.sin.data_ptr(), rot.max_delta, stream)
    t = _time(run)
    nbytes = tokens * cfg.n_layers * cfg.kv_heads * cfg.head_dim * 2 * 2
    pk = peaks()
    ach = nbytes / t / 1e9
    return {"kernel": "choreo_rerotate (K2)", "bound": "hbm", "work": f"{tokens} tokens x 32 layers",
            "algorithmic_bytes": nbytes, "us": round(t * 1e6, 2), "achieved": round(ach, 1),
            "unit": "GB/s", "peak": pk["hbm_gbs"], "frac": round(ach / pk["hbm_gbs"], 4)}


def k4_prefill(n_msgs: int = 8, rows: int = 1024, n_par: int = 24, n_layers: int = 32,
               reps: int = 10) -> dict:
    """n_layers < 32 shrinks the pool (profiling: ncu saves / restores device memory)."""
    from dataclasses import replace
    cfg = replace(LLAMA_3_1_8B, n_layers=n_layers)
    H, Hk, hd = cfg.n_heads, cfg.kv_heads, cfg.head_dim
    G = H // Hk
    cache = _cache(cfg, 32 * 256 + n_msgs * rows + 1024)
    for m in range(32):
        _add(cache, m, 256)
    for i in range(n_msgs):
        _add(cache, 32 + i, rows)
    cache.k_pool.normal_()
    cache.v_pool.normal_()
    rng = np.random.default_rng(0)
    calls = [(32 + i, [int(p) for p in rng.permutation(32)[:n_par]], 0, rows) for i in range(n_msgs)]
    # items sized like the runner does for prefill (about two waves of 148 CTAs)
    work = plan_counts([CallRows(c[0], c[1], 0, [0] * rows, None, None, 0) for c in calls],
                       cache.msg_len.host, 64, 256 // G, 1, 1)
    ppi = max(1, cdiv(work.item_pages * Hk, 2 * 148))
    plan, b, R = _assemble(cache, calls, 256 // G, ppi, 1)
    q = torch.randn(R, H, hd, device="cuda")
    po = torch.empty(plan.n_parts, H, hd, device="cuda")
    pl = torch.empty(plan.n_parts, H, device="cuda")
    out = torch.empty(2 * R, H * hd, dtype=torch.bfloat16, device="cuda")
    v = b["vis"]
    stream = torch.cuda.current_stream().cuda_stream
    direct = plan.max_row_parts == 1

    def run():
        nat.prefill_attn(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), nat.BF16,
                         cfg.n_layers, 0, Hk, cache.n_pages, 64, H, hd, b["rt"].data_ptr(),
                         v[0].data_ptr(), v[1].data_ptr(), v[2].data_ptr(), b["blk"].data_ptr(),
                         b["items"].data_ptr(), b["counts"].data_ptr(), plan.n_items,
                         po.data_ptr(), pl.data_ptr(), 0,
                         out.data_ptr() if direct else None, 1, R, stream)

    def run_comb():
        nat.attn_combine(po.data_ptr(), pl.data_ptr(), b["rpo"].data_ptr(), b["rp"].data_ptr(), R,
                         H, hd, out.data_ptr(), nat.BF16, 0, stream)
    t = _time(run, reps=reps, warm=min(3, reps), burst=1 if reps <= 2 else None)
    tc = 0.0 if direct or reps <= 2 else _time(run_comb, reps=10)
    pairs = n_msgs * (rows * n_par * 256 + rows * (rows + 1) // 2)
    flops = 4 * hd * H * pairs
    pk = peaks()
    ach = flops / t / 1e12
    return {"kernel": "choreo_prefill_attn (K4, tcgen05)", "bound": "tensor",
            "work": f"{n_msgs} msgs x {rows} rows over {n_par * 256}-token reordered parents, 1 layer",
            "algorithmic_flops": flops, "us": round(t * 1e6, 1), "combine_us": round(tc * 1e6, 1),
            "direct_output": direct,
            "achieved": round(ach, 1), "unit": "TFLOP/s", "peak": pk["bf16_tflops"],
            "frac": round(ach / pk["bf16_tflops"], 4), "pages_per_item": ppi,
            "items": plan.n_items}


def k5_decode(n_workflows: int = 1, agents: int = 8, tc: bool = False, v2: bool = True) -> dict:
    """One decode step of C3 round 2 (agents see sys, q and the other agents' replies)."""
    cfg = LLAMA_3_1_8B
    H, Hk, hd = cfg.n_heads, cfg.kv_heads, cfg.head_dim
    rng = np.random.default_rng(1)
    per = 2 + 2 * agents
    cache = _cache(cfg, n_workflows * (224 + 2 * agents * 800) + 4096)
    calls = []
    for w in range(n_workflows):
        b = w * per
        _add(cache, b, 64)
        _add(cache, b + 1, 160)
        for a in range(agents):
            _add(cache, b + 2 + a, int(rng.integers(266, 523)))
        for a in range(agents):  # own round-2 replies, ~250 tokens in
            _add(cache, b + 2 + agents + a, 260)
            others = [b + 2 + j for j in range(agents) if j != a]
            calls.append((b + 2 + agents + a, [b, b + 1] + others, 259, 1))
    cache.k_pool.normal_()
    cache.v_pool.normal_()
    G = H // Hk
    rpb = 256 // G if tc else max(1, 32 // G) if v2 else max(1, min(16, 64 // G))
    work = plan_counts([CallRows(c[0], c[1], c[2], [0], None, None, 0) for c in calls],
                       cache.msg_len.host, 64, rpb, 1)
    ppi = max(1, cdiv(work.item_pages * Hk, (1 if tc else 1 if v2 else 3) * 148))
    if v2:  # the runner's rule: about one (item, kv head) unit per SM, 4..32 pages
        ppi = min(max(ppi, 4), 32)
        while plan_counts([CallRows(c[0], c[1], c[2], [0], None, None, 0) for c in calls],
                          cache.msg_len.host, 64, rpb, ppi).n_items * Hk > 148 and ppi < 32:
            ppi = min(32, ppi + max(1, ppi // 4))
    ppi = int(os.environ.get("K5_PPI", ppi))
    plan, b, R = _assemble(cache, calls, rpb, ppi)
    order = None if os.environ.get("K5_ORDER", "1") == "0" else b["order"]  # K5_ORDER=0: w mod grid
    q = torch.randn(R, H, hd, device="cuda")
    po = torch.empty(plan.n_parts, H, hd, device="cuda")
    pl = torch.empty(plan.n_parts, H, device="cuda")
    out = torch.empty(2 * R, H * hd, dtype=torch.bfloat16, device="cuda")
    v = b["vis"]
    stream = torch.cuda.current_stream().cuda_stream


    # the runner's Q record (RoPE writes it; K5 v2 stages it with bulk copies), K5_QBULK=0: off
    qa = q * float(np.float32(1.4426950408889634) / np.sqrt(np.float32(hd)))
    qh = qa.bfloat16()
    q_k5 = (torch.cat([qh, (qa - qh.float()).bfloat16()], -1).contiguous()
            if os.environ.get("K5_QBULK", "1") != "0" else None)

    def run():
        if v2:
            nat.decode_attn_v2_ex(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(),
                                  cfg.n_layers, 0, Hk, cache.n_pages, 64, H, hd,
                                  b["rt"].data_ptr(), v[0].data_ptr(), v[1].data_ptr(),
                                  v[2].data_ptr(), b["blk"].data_ptr(), b["items"].data_ptr(),
                                  b["counts"].data_ptr(), plan.n_items, po.data_ptr(),
                                  pl.data_ptr(), b["fat"].data_ptr(), 0, nat.ptr(q_k5),
                                  nat.ptr(order), K3_TAG, stream)
            return
        if tc:
            nat.prefill_attn(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(),
                             nat.BF16, cfg.n_layers, 0, Hk, cache.n_pages, 64, H, hd,
                             b["rt"].data_ptr(), v[0].data_ptr(), v[1].data_ptr(), v[2].data_ptr(),
                             b["blk"].data_ptr(), b["items"].data_ptr(), b["counts"].data_ptr(),
                             plan.n_items, po.data_ptr(), pl.data_ptr(), 0, None, 0, R, stream)
            return
        nat.attn_split(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), nat.BF16, 0,
                       Hk, cache.n_pages, 64, H, hd, b["rt"].data_ptr(), v[0].data_ptr(),
                       v[1].data_ptr(), v[2].data_ptr(), b["blk"].data_ptr(), b["items"].data_ptr(),
                       b["counts"].data_ptr(), plan.n_items, po.data_ptr(), pl.data_ptr(), 0, stream)

    def run_comb():
        nat.attn_combine(po.data_ptr(), pl.data_ptr(), b["rpo"].data_ptr(), b["rp"].data_ptr(), R,
                         H, hd, out.data_ptr(), nat.BF16, 1, stream)
    t = _time(run)
    tcomb = _time(run_comb)
    uniq = sum(cache.message_length(m) for m in set(p for c in calls for p in c[1]))
    uniq += sum(c[2] + 1 for c in calls)
    nbytes = 2 * uniq * Hk * hd * 2 + R * H * hd * 4 + plan.n_parts * H * (hd + 1) * 4
    logical = sum(sum(cache.message_length(p) for p in c[1]) + c[2] + 1 for c in calls) * Hk * hd * 4
    pk = peaks()
    ach = nbytes / t / 1e9
    return {"kernel": ("choreo_decode_attn_v2 (K5 v2: TMA page ring, page-centric)" if v2 else
                       "choreo_prefill_attn on decode items (tcgen05)" if tc else
                       "choreo_attn_split (K5 generic SIMT, page-centric decode)"), "bound": "hbm",
            "work": f"{n_workflows} workflow(s) x {agents} agents, 1 layer",
            "algorithmic_bytes": nbytes, "logical_kv_bytes": logical, "us": round(t * 1e6, 2),
            "combine_us": round(tcomb * 1e6, 2), "achieved": round(ach, 1),
            "unit": "GB/s",
            "peak": pk["hbm_gbs"], "frac": round(ach / pk["hbm_gbs"], 4), "items": plan.n_items,
            "pages_per_item": ppi}


def k7_linear(x_rows: int = 8, split: bool = True) -> list:
    """K7 weight-streaming linear vs cuBLAS (torch.mm, f32 out) at the 8B decode shapes.
    Each timed launch reads a different weight copy (copies total > 3x L2), so every
    launch streams its weights from HBM.  bytes = weight bytes + activations + output."""
    cfg = LLAMA_3_1_8B
    d, f = cfg.model_dim, cfg.ffn_dim
    shapes = {"qkv": ((cfg.n_heads + 2 * cfg.kv_heads) * cfg.head_dim, d), "o_proj": (d, d),
              "gate_up": (2 * f, d), "down": (d, f), "head": (cfg.vocab_size, d)}
    rows = 2 * x_rows if split else x_rows
    ws = torch.empty(148 * 2 * 256 * 128, device="cuda")
    pk = peaks()
    out = []
    stream = torch.cuda.current_stream().cuda_stream
    for name, (n, k) in shapes.items():
        ncopy = max(2, int(400e6 // (n * k * 2)) + 1)
        ws_list = [torch.randn(n, k, device="cuda").to(torch.bfloat16) for _ in range(ncopy)]
        x = torch.randn(rows, k, device="cuda").to(torch.bfloat16)
        y = torch.empty(x_rows, n, device="cuda")
        cnt = torch.zeros((n + 127) // 128, dtype=torch.int32, device="cuda")
        it = [0]

        def ours():
            w = ws_list[it[0] % ncopy]
            it[0] += 1
            nat.linear_skinny(x.data_ptr(), rows, int(split), w.data_ptr(), n, k, y.data_ptr(),
                              ws.data_ptr(), cnt.data_ptr(), 0, stream)

        def cublas():
            w = ws_list[it[0] % ncopy]
            it[0] += 1
            torch.mm(x, w.t(), out_dtype=torch.float32)
        t_ours = _time(ours, burst=ncopy)
        t_cb = _time(cublas, burst=ncopy)
        nbytes = n * k * 2 + rows * k * 2 + x_rows * n * 4
        ach = nbytes / t_ours / 1e9
        out.append({"kernel": f"choreo_linear_skinny (K7) {name}", "bound": "hbm",
                    "shape": f"{rows}x{k} @ {n}x{k}^T", "algorithmic_bytes": nbytes,
                    "us": round(t_ours * 1e6, 2), "achieved": round(ach, 1), "unit": "GB/s",
                    "peak": pk["hbm_gbs"], "frac": round(ach / pk["hbm_gbs"], 4),
                    "cublas_us": round(t_cb * 1e6, 2),
                    "cublas_frac": round(nbytes / t_cb / 1e9 / pk["hbm_gbs"], 4)})
        del ws_list
        torch.cuda.empty_cache()
    return out


def k5_sweep() -> list:
    out = []
    for tc in (False, True):
        for ppi in (1, 2, 3, 4, 6, 8):
            os.environ["K5_PPI"] = str(ppi)
            r = k5_decode(1, tc=tc)
            out.append((tc, ppi, r["us"], r["combine_us"], r["items"]))
    os.environ.pop("K5_PPI")
    return out


def k8_chain(rows: int = 8) -> dict:
    """K8 layer chain (o_proj, gate|up, down, next qkv in one persistent launch, norms /
    SwiGLU / RoPE in the epilogues) at the 8B layer shape, back-to-back launches (438 MB of
    weights each, > L2), beside the sum of the four K7 launches at the same shapes."""
    import ctypes

    sys.path.insert(0, ROOT)
    from tests.test_gpu_chain import _Bufs, _Layer, _rope_tables

    cfg = LLAMA_3_1_8B
    d, H, Hk, hd, F = cfg.model_dim, cfg.n_heads, cfg.kv_heads, cfg.head_dim, cfg.ffn_dim
    lw = _Layer(d, H, Hk, hd, F, seed=1)
    b = _Bufs(rows, d, H, Hk, hd, F, True, n_pages=16)
    W = 8192
    cos_t, sin_t = _rope_tables(hd, W)
    pos = torch.arange(rows, dtype=torch.int32, device="cuda") + 100
    page = torch.zeros(rows, dtype=torch.int32, device="cuda")
    slot = torch.arange(rows, dtype=torch.int32, device="cuda")
    for t in (b.x, b.attn, b.h_a, b.h_b, b.act):
        t.normal_()
    b.ssq_a.fill_(float(d))
    b.ssq_b.fill_(float(d))
    stream = torch.cuda.current_stream().cuda_stream
    st = nat.LayerChain(
        n_rows=rows, split=1, d=d, n_heads=H, n_kv=Hk, head_dim=hd, ffn_dim=F, eps=1e-6, phases=15,
        wo=lw.wo.data_ptr(), ffn_norm=lw.g_ffn.data_ptr(), w_gu=lw.w_gu.data_ptr(),
        w_down=lw.w_down.data_ptr(), attn_norm_next=lw.g_attn.data_ptr(),
        w_qkv=lw.w_qkv.data_ptr(), layer_qkv=0, x=b.x.data_ptr(), attn=b.attn.data_ptr(),
        h_a=b.h_a.data_ptr(), act=b.act.data_ptr(), h_b=b.h_b.data_ptr(),
        ssq_a=b.ssq_a.data_ptr(), ssq_b=b.ssq_b.data_ptr(), q=b.q.data_ptr(),
        k_pool=b.k_pool.data_ptr(), v_pool=b.v_pool.data_ptr(), n_pages=b.k_pool.shape[2],
        page_size=64, pos=pos.data_ptr(), page=page.data_ptr(), slot=slot.data_ptr(),
        cos_t=cos_t.data_ptr(), sin_t=sin_t.data_ptr(), max_delta=W, ws=b.ws.data_ptr(),
        counters=b.counters.data_ptr(), done=b.done.data_ptr())
    t = _time(lambda: nat.layer_chain(ctypes.byref(st), stream))
    nbytes = sum(w.numel() * 2 for w in (lw.wo, lw.w_gu, lw.w_down, lw.w_qkv))
    pk = peaks()
    ach = nbytes / t / 1e9
    return {"kernel": "choreo_layer_chain (K8: o_proj + gate|up + down + next qkv, one launch)",
            "bound": "hbm", "shape": f"{rows} rows (x2 hi/lo), 8B layer", "algorithmic_bytes": nbytes,
            "us": round(t * 1e6, 2), "achieved": round(ach, 1), "unit": "GB/s",
            "peak": pk["hbm_gbs"], "frac": round(ach / pk["hbm_gbs"], 4)}


def run_all() -> list:
    out = [k2_rerotate(), k4_prefill(), k5_decode(1), k5_decode(8), k5_decode(1, v2=False),
           k5_decode(8, v2=False)]
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    if "--k7" in sys.argv:
        rows = int(os.environ.get("K7_ROWS", "8"))
        for r in k7_linear(rows):
            print(json.dumps(r))
        sys.exit(0)
    if "--k5-sweep" in sys.argv:
        print(k5_sweep())
        sys.exit(0)
    res = run_all()
    if "--json" in sys.argv:
        print(json.dumps(res))
    else:
        for r in res:
            print(json.dumps(r))
