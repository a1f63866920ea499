"""Kernel-level parity of the sm_100a C-ABI library against the CPU oracle (GPU).

Index math (pages, slots, positions, visible sets) is checked bit-exact; values
within dtype tolerance (f32: 1e-5 relative; bf16: one bf16 rounding).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import choreo_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

from paper_2512_23049_b200 import _native as nat  # noqa: E402
from paper_2512_23049_b200.cache import DeviceKvCache, RotationTableDevice  # noqa: E402
from paper_2512_23049_b200.config import ModelConfig  # noqa: E402

DT = {"f32": torch.float32, "bf16": torch.bfloat16}


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("hd,H,Hk", [(16, 4, 4), (128, 32, 8), (64, 8, 2)])
def test_rope_append(dt, hd, H, Hk):
    cfg = ModelConfig(n_layers=2, n_heads=H, n_kv_heads=Hk, head_dim=hd, ffn_dim=32,
                      vocab_size=300, context_window=4096, rope_base=500000.0)
    rot = RotationTableDevice(cfg, "cuda")
    orot = O.Rotor(O.Shape(head_dim=hd, context_window=4096, rope_base=500000.0))
    rng = np.random.default_rng(0)
    R, n_pages, P = 37, 5, 64
    qkv = rng.standard_normal((R, (H + 2 * Hk) * hd)).astype(np.float32)
    pos = rng.integers(0, 4096, R).astype(np.int32)
    flat = rng.permutation(n_pages * P)[:R]
    page, slot = (flat // P).astype(np.int32), (flat % P).astype(np.int32)
    kp = torch.zeros(2, Hk, n_pages, P, hd, dtype=DT[dt], device="cuda")
    vp = torch.zeros_like(kp)
    q = torch.empty(R, H, hd, device="cuda")
    d = {k: torch.from_numpy(v).cuda() for k, v in dict(qkv=qkv, pos=pos, page=page, slot=slot).items()}
    nat.rope_append(d["qkv"].data_ptr(), nat.F32, qkv.shape[1], R, 0, d["pos"].data_ptr(),
                    d["page"].data_ptr(), d["slot"].data_ptr(), q.data_ptr(), kp.data_ptr(),
                    vp.data_ptr(), nat.dtype_code(DT[dt]), 1, Hk, n_pages, P, H, hd,
                    rot.cos.data_ptr(), rot.sin.data_ptr(), rot.max_delta, _stream())
    torch.cuda.synchronize()
    x = qkv.astype(np.float64)
    q_ref = orot.by_position(x[:, :H * hd].reshape(R, H, hd), pos)
    k_ref = orot.by_position(x[:, H * hd:(H + Hk) * hd].reshape(R, Hk, hd), pos)
    v_ref = x[:, (H + Hk) * hd:].reshape(R, Hk, hd)
    np.testing.assert_allclose(q.cpu().numpy(), q_ref, rtol=1e-5, atol=1e-5)
    k_got = kp[1].permute(1, 2, 0, 3).float().cpu().numpy()[page, slot]  # (R, Hk, hd)
    v_got = vp[1].permute(1, 2, 0, 3).float().cpu().numpy()[page, slot]
    tol = dict(rtol=1e-5, atol=1e-5) if dt == "f32" else dict(rtol=2 ** -8, atol=1e-6)
    np.testing.assert_allclose(k_got, k_ref, **tol)
    np.testing.assert_allclose(v_got, v_ref, **tol)
    assert kp[0].abs().sum().item() == 0  # other layers untouched


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("hd", [8, 16, 64, 128])
def test_rerotate(dt, hd):
    """K2 (bf16 pools at hd 64 / 128: TMA-fed page tiles) against the oracle's rotor."""
    W = 2048
    cfg = ModelConfig(n_layers=3, n_heads=2, head_dim=hd, context_window=W)
    rot = RotationTableDevice(cfg, "cuda")
    orot = O.Rotor(O.Shape(head_dim=hd, context_window=W))
    rng = np.random.default_rng(1)
    L, Hk, n_pages, P = 3, 2, 9, 64
    pool = rng.standard_normal((L, Hk, n_pages, P, hd)).astype(np.float32)
    if dt == "bf16":
        pool = _bf16_round(pool)
    kp = torch.from_numpy(pool).to(DT[dt]).cuda()
    pages = np.array([7, 2, 4, 0], np.int32)
    lens = np.array([64, 13, 1, 64], np.int32)
    deltas = np.array([37, -W, 0, W], np.int32)
    arr = torch.from_numpy(np.stack([pages, lens, deltas])).cuda()
    nat.rerotate(kp.data_ptr(), nat.dtype_code(DT[dt]), L, Hk, n_pages, P, hd, arr[0].data_ptr(),
                 arr[1].data_ptr(), arr[2].data_ptr(), 4, rot.cos.data_ptr(), rot.sin.data_ptr(),
                 W, _stream())
    got = kp.float().cpu().numpy()
    want = pool.astype(np.float64).copy()
    for pg, ln, dl in zip(pages, lens, deltas):
        want[:, :, pg, :ln] = orot.by_delta(want[:, :, pg, :ln], int(dl))
    tol = dict(rtol=1e-5, atol=1e-5) if dt == "f32" else dict(rtol=2 ** -8, atol=1e-6)
    np.testing.assert_allclose(got, want, **tol)
    # untouched: slots past page_len, unlisted pages, delta == 0 page (bitwise)
    np.testing.assert_array_equal(got[:, :, 2, 13:], pool[:, :, 2, 13:])
    np.testing.assert_array_equal(got[:, :, [1, 3, 5, 6, 8]], pool[:, :, [1, 3, 5, 6, 8]])
    np.testing.assert_array_equal(got[:, :, 4], pool[:, :, 4])


def test_select_greedy_ties_and_mask():
    rng = np.random.default_rng(2)
    V = 512
    logits = rng.standard_normal((9, V)).astype(np.float32)
    logits[0, 256] = 100.0       # BOS is not generatable
    logits[1, 300] = 100.0       # nor reserved/vocab tail
    logits[2, [5, 9, 200]] = 7.0  # tie -> lowest id
    logits[3, 257] = 50.0        # EOS is generatable
    d = torch.from_numpy(logits).cuda()
    out = torch.empty(9, dtype=torch.int32, device="cuda")
    nat.select_greedy(d.data_ptr(), 9, V, V, 0, out.data_ptr(), _stream())
    mask = O.sampler_mask(V)
    want = [int(np.argmax(np.where(mask, r.astype(np.float64), -np.inf))) for r in logits]
    assert out.cpu().tolist() == want
    assert want[2] == 5 and want[3] == 257


def _random_cache(cfg, rng, n_msgs, P=64, dtype=torch.float32):
    cache = DeviceKvCache(cfg, capacity=1 << 16, dtype=dtype, device="cuda", page_size=P)
    lens = rng.integers(1, 3 * P, n_msgs)
    for m, n in enumerate(lens):
        cache.register_message(m, "prefilled", 0, max_tokens=int(n))
        cache.reserve_slots(m, [1] * int(n))
        cache.log_append(m, 0, int(n))
    cache.k_pool.copy_(torch.randn_like(cache.k_pool))
    cache.v_pool.copy_(torch.randn_like(cache.v_pool))
    return cache, lens


def _assemble(cache, calls, rpb, ppi, mode=0, order=None, tag=0):
    """calls: list of (own msg, parents, row_t list).  Returns host copies of K3 outputs
    (order: an int32 device tensor receiving choreo_assemble_ex's item_order)."""
    from paper_2512_23049_b200.model import plan_counts, CallRows
    tab, par, row_t, off = [], [], [], 0
    for own, parents, ts in calls:
        tab += [own, len(par), len(parents), off, len(ts)]
        par += parents
        row_t += ts
        off += len(ts)
    cr = [CallRows(own, parents, ts[0], [0] * len(ts), None, None, 0) for own, parents, ts in calls]
    plan = plan_counts(cr, cache.msg_len.host, cache.page_size, rpb, ppi, mode)
    cache.sync_tables()
    dev = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")  # noqa: E731
    tab_d, par_d, rt_d = dev(tab), dev(par + [0]), dev(row_t)
    R = len(row_t)
    vis = torch.full((3, max(plan.n_vis, 1)), -7, dtype=torch.int32, device="cuda")
    blk = torch.full((max(plan.n_blk_rows, 1),), -7, dtype=torch.int32, device="cuda")
    items = torch.full((max(plan.n_items, 1), 6), -7, dtype=torch.int32, device="cuda")
    rpo = torch.full((R + 1,), -7, dtype=torch.int32, device="cuda")
    rp = torch.full((max(plan.n_parts, 1),), -7, dtype=torch.int32, device="cuda")
    counts = torch.zeros(6, dtype=torch.int32, device="cuda")
    args = (cache.msg_len.dev.data_ptr(), cache.msg_pt.dev.data_ptr(),
            cache.page_table.dev.data_ptr(), tab_d.data_ptr(), par_d.data_ptr(), len(calls),
            rt_d.data_ptr(), R, None, 0, cache.page_size, rpb, ppi,
            vis[0].data_ptr(), vis[1].data_ptr(), vis[2].data_ptr(), blk.data_ptr(),
            items.data_ptr(), rpo.data_ptr(), rp.data_ptr(), counts.data_ptr(),
            plan.n_vis, plan.n_blk_rows, plan.n_items, plan.n_parts, mode, None)
    if order is None:
        nat.assemble(*args, _stream())
    else:
        nat.assemble_ex(*args, order.data_ptr(), tag, _stream())
    out = dict(vis=vis.cpu().numpy(), blk=blk.cpu().numpy(), items=items.cpu().numpy(),
               rpo=rpo.cpu().numpy(), rp=rp.cpu().numpy(), counts=counts.cpu().numpy(),
               row_t=np.asarray(row_t), plan=plan)
    return out, (rt_d, vis, blk, items, rpo, rp, counts)


def _expand_rows(cache, out, n_rows):
    """Token-level (msg, idx) visible sets per row, from K3 items; checks that no token
    is covered twice and that the per-row partial lists are exactly the items' slots."""
    page_owner = {}
    for m, e in cache._messages.items():
        for i, pg in enumerate(e.pages):
            page_owner[pg] = (m, i)
    P = cache.page_size
    sets = [[] for _ in range(n_rows)]
    slots = [[] for _ in range(n_rows)]
    for it in out["items"][:out["counts"][1]]:
        rb, nr, vb, nv, pbase = it[:5]
        for jj in range(nr):
            r = int(out["blk"][rb + jj])
            slots[r].append(int(pbase + jj))
            t = out["row_t"][r]
            for k in range(vb, vb + nv):
                pg, ln, own = out["vis"][:, k]
                m, pi = page_owner[int(pg)]
                for s_ in range(ln):
                    if own < 0 or own + s_ <= t:
                        sets[r].append((m, pi * P + s_))
    for r in range(n_rows):
        assert len(sets[r]) == len(set(sets[r])), "a token is covered twice"
        csr = out["rp"][out["rpo"][r]:out["rpo"][r + 1]].tolist()
        assert sorted(csr) == sorted(slots[r]), f"row {r} partial list"
    all_slots = sorted(x for s_ in slots for x in s_)
    assert all_slots == list(range(out["plan"].n_parts)), "partial slots not a bijection"
    return [sorted(s_) for s_ in sets]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("rpb,ppi", [(1, 1), (4, 3), (16, 1000)])
def test_assemble_visible_sets_match_oracle(rpb, ppi, mode):
    rng = np.random.default_rng(3)
    cfg = ModelConfig(n_layers=1, n_heads=2, head_dim=8)
    cache, lens = _random_cache(cfg, rng, 12)
    calls = []
    nxt = 12
    for c in range(5):
        parents = [int(p) for p in rng.permutation(12)[:rng.integers(0, 6)]]
        own = nxt
        nxt += 1
        n_new = int(rng.integers(1, 150))
        pre = int(rng.integers(0, 70)) if c % 2 else 0  # tokens already cached for own msg
        cache.register_message(own, "decoded", 0)
        cache.reserve_slots(own, [1] * (pre + n_new))
        cache.log_append(own, 0, pre + n_new)
        calls.append((own, parents, list(range(pre, pre + n_new))))
    out, _ = _assemble(cache, calls, rpb, ppi, mode)
    assert out["counts"][3] == 0
    pl = out["plan"]
    assert tuple(out["counts"][:3]) == (pl.n_vis, pl.n_items, pl.n_parts)
    sets = _expand_rows(cache, out, len(out["row_t"]))
    # oracle: reference visibility over the physical store
    st = O.Store(O.Shape(n_layers=1, n_heads=2, head_dim=8), 1 << 16)
    for m, e in sorted(cache._messages.items()):
        st.msgs[m] = O.Msg(e.kind, 0, "", None)
        z = np.zeros((1, len(e.tokens), 2, 8))
        st.append(m, e.tokens, np.arange(len(e.tokens)), z, z)
    r = 0
    for own, parents, ts in calls:
        for t in ts:
            vis = st.visible(own, parents)
            want = sorted((int(st.mid[i]), int(st.pos[i])) for i in vis
                          if st.mid[i] != own or st.pos[i] <= t)
            assert sets[r] == want, f"row {r}"
            r += 1


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("hd,H,Hk", [(16, 4, 4), (128, 32, 8), (64, 8, 1)])
def test_attention_matches_dense_reference(dt, hd, H, Hk, mode):
    rng = np.random.default_rng(4)
    cfg = ModelConfig(n_layers=2, n_heads=H, n_kv_heads=Hk, head_dim=hd)
    cache, lens = _random_cache(cfg, rng, 8, dtype=DT[dt])
    own = 8
    cache.register_message(own, "decoded", 0)
    cache.reserve_slots(own, [1] * 90)
    cache.log_append(own, 0, 90)
    cache.k_pool.copy_(torch.randn_like(cache.k_pool))
    cache.v_pool.copy_(torch.randn_like(cache.v_pool))
    cache.register_message(9, "decoded", 0)
    cache.reserve_slots(9, [1] * 3)
    cache.log_append(9, 0, 3)
    cache.register_message(10, "decoded", 0)
    cache.reserve_slots(10, [1] * 1)
    cache.log_append(10, 0, 1)
    cache.k_pool.copy_(torch.randn_like(cache.k_pool))
    cache.v_pool.copy_(torch.randn_like(cache.v_pool))
    calls = [(own, [3, 1, 6], list(range(60, 90))), (7, [], [int(lens[7]) - 1]),
             (9, [6, 3, 0], [2]), (10, [1, 6, 2, 5, 4], [0])]
    G = H // Hk
    rpb = max(1, min(16, 64 // G))
    out, (rt_d, vis, blk, items, rpo, rp, counts) = _assemble(cache, calls, rpb, 2, mode)
    R = len(out["row_t"])
    q = torch.randn(R, H, hd, device="cuda")
    n_parts = out["plan"].n_parts
    part_o = torch.empty(n_parts, H, hd, device="cuda")
    part_lse = torch.empty(n_parts, H, device="cuda")
    o = torch.empty(R, H * hd, dtype=torch.float32, device="cuda")
    L = 1
    nat.attn_split(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(),
                   nat.dtype_code(DT[dt]), L, Hk, cache.n_pages, cache.page_size, H, hd,
                   rt_d.data_ptr(), vis[0].data_ptr(), vis[1].data_ptr(), vis[2].data_ptr(),
                   blk.data_ptr(), items.data_ptr(), counts.data_ptr(), out["plan"].n_items,
                   part_o.data_ptr(), part_lse.data_ptr(), 0, _stream())
    nat.attn_combine(part_o.data_ptr(), part_lse.data_ptr(), rpo.data_ptr(), rp.data_ptr(), R, H,
                     hd, o.data_ptr(), nat.F32, 0, _stream())
    torch.cuda.synchronize()
    sets = _expand_rows(cache, out, R)
    K = cache.k_pool[L].float().cpu().numpy().astype(np.float64)  # (Hk, pages, P, hd)
    V = cache.v_pool[L].float().cpu().numpy().astype(np.float64)
    qn = q.cpu().numpy().astype(np.float64)
    P = cache.page_size
    got = o.cpu().numpy().reshape(R, H, hd)
    for r in range(R):
        toks = sets[r]
        pg = np.array([cache._messages[m].pages[i // P] for m, i in toks])
        sl = np.array([i % P for m, i in toks])
        for h in range(H):
            kh = h // G
            kk, vv = K[kh, pg, sl], V[kh, pg, sl]
            s = kk @ qn[r, h] / np.sqrt(hd)
            p = np.exp(s - s.max())
            p /= p.sum()
            np.testing.assert_allclose(got[r, h], p @ vv, rtol=1e-4, atol=1e-4)


def test_umma_selftest_tcgen05_descriptors():
    """tcgen05.mma with SW128 K-major and MN-major operands reproduces A@B in f32."""
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(128, 64, device="cuda", generator=g).to(torch.bfloat16)
    b1 = torch.randn(64, 64, device="cuda", generator=g).to(torch.bfloat16)
    b2 = torch.randn(64, 128, device="cuda", generator=g).to(torch.bfloat16)
    c1 = torch.empty(128, 64, device="cuda")
    c2 = torch.empty(128, 128, device="cuda")
    c3 = torch.empty(128, 128, device="cuda")
    nat.selftest_umma(a.data_ptr(), b1.data_ptr(), b2.data_ptr(), c1.data_ptr(), c2.data_ptr(),
                      c3.data_ptr(), _stream())
    torch.cuda.synchronize()
    torch.testing.assert_close(c3, a.float() @ b2.float(), rtol=1e-4, atol=1e-3)
    torch.testing.assert_close(c1, a.float() @ b1.float().t(), rtol=1e-4, atol=1e-3)
    torch.testing.assert_close(c2, a.float() @ b2.float(), rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("ppi", [3, 100000])
@pytest.mark.parametrize("hd,H,Hk", [(128, 32, 8), (64, 8, 8), (128, 16, 2)])
def test_prefill_tcgen05_matches_dense_reference(hd, H, Hk, ppi):
    """K4 (tcgen05/TMEM/TMA) over page-centric items with 128-row M tiles: prefill rows of
    two messages sharing reordered parents, causal own pages, partial tail pages."""
    rng = np.random.default_rng(7)
    cfg = ModelConfig(n_layers=2, n_heads=H, n_kv_heads=Hk, head_dim=hd)
    cache, lens = _random_cache(cfg, rng, 6, dtype=torch.bfloat16)
    for own, n in ((6, 150), (7, 41)):
        cache.register_message(own, "prefilled", 0, max_tokens=n)
        cache.reserve_slots(own, [1] * n)
        cache.log_append(own, 0, n)
    cache.k_pool.copy_(torch.randn_like(cache.k_pool))
    cache.v_pool.copy_(torch.randn_like(cache.v_pool))
    calls = [(6, [4, 1, 3], list(range(150))), (7, [3, 0], list(range(41)))]
    G = H // Hk
    out, (rt_d, vis, blk, items, rpo, rp, counts) = _assemble(cache, calls, 256 // G, ppi, 1)
    R = len(out["row_t"])
    q = torch.randn(R, H, hd, device="cuda")
    n_parts = out["plan"].n_parts
    part_o = torch.empty(n_parts, H, hd, device="cuda")
    part_lse = torch.empty(n_parts, H, device="cuda")
    o = torch.empty(R, H * hd, dtype=torch.float32, device="cuda")
    direct = out["plan"].max_row_parts == 1
    assert direct == (ppi > 1000)
    direct_out = torch.zeros(2 * R, H * hd, dtype=torch.bfloat16, device="cuda")
    L = 1
    nat.prefill_attn(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), nat.BF16,
                     cfg.n_layers, L, Hk, cache.n_pages, cache.page_size, H, hd, rt_d.data_ptr(),
                     vis[0].data_ptr(), vis[1].data_ptr(), vis[2].data_ptr(), blk.data_ptr(),
                     items.data_ptr(), counts.data_ptr(), out["plan"].n_items, part_o.data_ptr(),
                     part_lse.data_ptr(), 0, direct_out.data_ptr() if direct else None, 1, R,
                     _stream())
    if direct:  # final rows written by K4 as hi/lo bf16 pairs
        o.copy_((direct_out[:R].float() + direct_out[R:].float()))
    else:
        nat.attn_combine(part_o.data_ptr(), part_lse.data_ptr(), rpo.data_ptr(), rp.data_ptr(), R,
                         H, hd, o.data_ptr(), nat.F32, 0, _stream())
    torch.cuda.synchronize()
    sets = _expand_rows(cache, out, R)
    K = cache.k_pool[L].float().cpu().numpy().astype(np.float64)
    V = cache.v_pool[L].float().cpu().numpy().astype(np.float64)
    # K4 rounds Q and P to bf16 (standard flash attention numerics)
    qn = q.to(torch.bfloat16).float().cpu().numpy().astype(np.float64)
    P_ = cache.page_size
    got = o.cpu().numpy().reshape(R, H, hd)
    worst = 0.0
    for r in range(R):
        toks = sets[r]
        pg = np.array([cache._messages[m].pages[i // P_] for m, i in toks])
        sl = np.array([i % P_ for m, i in toks])
        for h in range(H):
            kk, vv = K[h // G, pg, sl], V[h // G, pg, sl]
            s = kk @ qn[r, h] / np.sqrt(hd)
            p = np.exp(s - s.max())
            p /= p.sum()
            worst = max(worst, float(np.abs(got[r, h] - p @ vv).max()))
    assert worst < 2e-2, worst


@pytest.mark.parametrize("ppi", [1, 2, 5])
@pytest.mark.parametrize("hd,H,Hk", [(128, 32, 8), (64, 16, 2), (128, 8, 8), (64, 4, 2)])
def test_decode_v2_matches_dense_reference(hd, H, Hk, ppi):
    """K5 v2 (TMA page ring + ldmatrix/mma.sync consumers, 4 key slices x 2 m-tiles) over
    page-centric items: agents sharing reordered parents, causal own pages, ragged pages.
    Q as a hi/lo bf16 pair, P bf16, f32 accumulation: within 2e-2 of the f64 reference."""
    rng = np.random.default_rng(12)
    cfg = ModelConfig(n_layers=2, n_heads=H, n_kv_heads=Hk, head_dim=hd)
    cache, lens = _random_cache(cfg, rng, 8, dtype=torch.bfloat16)
    calls = []
    for a in range(9):
        own = 8 + a
        n = int(rng.integers(1, 200))
        cache.register_message(own, "decoded", 0)
        cache.reserve_slots(own, [1] * n)
        cache.log_append(own, 0, n)
        parents = [int(p) for p in rng.permutation(8)[:int(rng.integers(0, 8))]]
        calls.append((own, parents, [n - 1] if a != 3 else list(range(max(0, n - 5), n))))
    cache.k_pool.copy_(torch.randn_like(cache.k_pool))
    cache.v_pool.copy_(torch.randn_like(cache.v_pool))
    G = H // Hk
    rpb = max(1, 32 // G)
    out, (rt_d, vis, blk, items, rpo, rp, counts) = _assemble(cache, calls, rpb, ppi, 0)
    R = len(out["row_t"])
    pl_ = out["plan"]
    q = torch.randn(R, H, hd, device="cuda")
    part_o = torch.empty(pl_.n_parts, H, hd, device="cuda")
    part_lse = torch.empty(pl_.n_parts, H, device="cuda")
    o = torch.empty(R, H * hd, dtype=torch.float32, device="cuda")
    L = 1
    for grid in (0, 5):  # persistent CTAs: many work units per CTA through one page ring
        nat.decode_attn_v2(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), 2, L,
                           Hk, cache.n_pages, 64, H, hd, rt_d.data_ptr(), vis[0].data_ptr(),
                           vis[1].data_ptr(), vis[2].data_ptr(), blk.data_ptr(), items.data_ptr(),
                           counts.data_ptr(), pl_.n_items, part_o.data_ptr(), part_lse.data_ptr(),
                           None, grid, _stream())
        nat.attn_combine(part_o.data_ptr(), part_lse.data_ptr(), rpo.data_ptr(), rp.data_ptr(), R,
                         H, hd, o.data_ptr(), nat.F32, 0, _stream())
        torch.cuda.synchronize()
        got = o.cpu().numpy().reshape(R, H, hd)
        sets = _expand_rows(cache, out, R)
        K = cache.k_pool[L].float().cpu().numpy().astype(np.float64)
        V = cache.v_pool[L].float().cpu().numpy().astype(np.float64)
        qn = q.cpu().numpy().astype(np.float64)
        worst = 0.0
        for r in range(R):
            toks = sets[r]
            pg = np.array([cache._messages[m].pages[i // 64] for m, i in toks])
            sl = np.array([i % 64 for m, i in toks])
            for h in range(H):
                kk, vv = K[h // G, pg, sl], V[h // G, pg, sl]
                s = kk @ qn[r, h] / np.sqrt(hd)
                p = np.exp(s - s.max())
                p /= p.sum()
                worst = max(worst, float(np.abs(got[r, h] - p @ vv).max()))
        assert worst < 2e-2, (grid, worst)
    # Q staged by bulk copies from the RoPE-written record (hi/lo of q * log2(e)/sqrt(hd)):
    # the same bf16 operands as the per-lane conversion, so the partials are bit-identical
    a = q * float(np.float32(1.4426950408889634) / np.sqrt(np.float32(hd)))
    hi = a.bfloat16()
    q_k5 = torch.cat([hi, (a - hi.float()).bfloat16()], dim=-1).contiguous()
    part_o.zero_()
    part_lse.zero_()
    nat.decode_attn_v2(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), 2, L, Hk,
                       cache.n_pages, 64, H, hd, rt_d.data_ptr(), vis[0].data_ptr(),
                       vis[1].data_ptr(), vis[2].data_ptr(), blk.data_ptr(), items.data_ptr(),
                       counts.data_ptr(), pl_.n_items, part_o.data_ptr(), part_lse.data_ptr(),
                       None, 5, _stream())
    ref_o, ref_lse = part_o.clone(), part_lse.clone()
    part_o.zero_()
    part_lse.zero_()
    nat.decode_attn_v2_ex(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), 2, L, Hk,
                          cache.n_pages, 64, H, hd, rt_d.data_ptr(), vis[0].data_ptr(),
                          vis[1].data_ptr(), vis[2].data_ptr(), blk.data_ptr(), items.data_ptr(),
                          counts.data_ptr(), pl_.n_items, part_o.data_ptr(), part_lse.data_ptr(),
                          None, 5, q_k5.data_ptr(), None, 0, _stream())
    torch.cuda.synchronize()
    assert torch.equal(part_o, ref_o) and torch.equal(part_lse, ref_lse)
    # longest-first unit deal (K3 item_order, snaking over 5 CTAs): the schedule changes,
    # every unit still writes its own partial slots -> bitwise the same partials
    order = torch.full((max(pl_.n_items, 1),), -7, dtype=torch.int32, device="cuda")
    # (with K3's step tag: the loader / producer read K3's outputs before the dependency wait)
    out2, (rt2, vis2, blk2, items2, _, _, counts2) = _assemble(cache, calls, rpb, ppi, 0, order,
                                                               tag=77)
    assert counts2[4:6].tolist() == [77, pl_.n_items], "K3 stamps {tag, n_items} after its outputs"
    nv = out2["items"][:pl_.n_items, 3]
    want = sorted(range(pl_.n_items), key=lambda i: (-min(max(int(nv[i]), 1), 32), i))
    assert order.cpu().tolist()[:pl_.n_items] == want, "item_order: stable, page count descending"
    for grid in (5, 0):
        part_o.zero_()
        part_lse.zero_()
        nat.decode_attn_v2_ex(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), 2, L,
                              Hk, cache.n_pages, 64, H, hd, rt2.data_ptr(), vis2[0].data_ptr(),
                              vis2[1].data_ptr(), vis2[2].data_ptr(), blk2.data_ptr(),
                              items2.data_ptr(), counts2.data_ptr(), pl_.n_items,
                              part_o.data_ptr(), part_lse.data_ptr(), None, grid,
                              q_k5.data_ptr(), order.data_ptr(), 77, _stream())
        torch.cuda.synchronize()
        assert torch.equal(part_o, ref_o) and torch.equal(part_lse, ref_lse), grid


def _linear(x, split, w, grid=0):
    rows = x.shape[0] // (2 if split else 1)
    y = torch.full((rows, w.shape[0]), float("nan"), device="cuda")
    ws = torch.empty(148 * 2 * 256 * 128, device="cuda")
    cnt = torch.zeros((w.shape[0] + 127) // 128, dtype=torch.int32, device="cuda")
    nat.linear_skinny(x.data_ptr(), x.shape[0], int(split), w.data_ptr(), w.shape[0], w.shape[1],
                      y.data_ptr(), ws.data_ptr(), cnt.data_ptr(), grid, _stream())
    torch.cuda.synchronize()
    assert int(cnt.abs().sum()) == 0, "tile counters must be left zero"
    return y


@pytest.mark.parametrize("rows,split", [(1, False), (8, True), (16, False), (16, True), (5, True),
                                        (32, True), (40, False), (64, False), (64, True),
                                        (100, False), (37, True), (72, True), (128, True),
                                        (65, True), (128, False), (80, True), (96, True),
                                        (120, True)])
@pytest.mark.parametrize("n,k", [(4096, 4096), (6144, 4096), (4096, 14336), (300, 64), (1000, 200)])
def test_linear_skinny_matches_f32_reference(rows, split, n, k):
    """K7 (tcgen05 stream-K weight streaming) = x @ w^T in f32 over bf16 inputs; with split
    activations the hi/lo halves are summed; deterministic run to run."""
    if split and 2 * rows > 256:
        pytest.skip("split supports <= 128 output rows")
    g = torch.Generator(device="cuda").manual_seed(rows * 7 + n)
    xm = torch.randn(2 * rows if split else rows, k, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    y = _linear(xm, split, w)
    ref = xm.float() @ w.float().t()
    if split:
        ref = ref[:rows] + ref[rows:]
    torch.testing.assert_close(y, ref, rtol=1e-4, atol=1e-4)
    assert torch.equal(_linear(xm, split, w), y)
    # odd grids exercise tiles cut between many CTAs
    torch.testing.assert_close(_linear(xm, split, w, grid=37), ref, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("vocab", [512, 128256])
def test_select_nucleus_matches_host_sampler(vocab):
    """K6b (device nucleus) picks the same token as the engine's NumPy sampler (the
    reference algorithm, engine.py:374-392) for many rows, temperatures, top-p values,
    seeds and selection indices, including peaked and near-uniform distributions."""
    from paper_2512_23049_b200.engine import SamplingParams, _sample_nucleus
    from paper_2512_23049_b200.tokenizer import generatable_mask

    rng = np.random.default_rng(vocab)
    n = 96
    scale = rng.choice([0.05, 1.0, 4.0, 20.0], size=n)
    logits = (rng.standard_normal((n, vocab)) * scale[:, None]).astype(np.float32)
    temps = rng.choice([0.3, 0.7, 1.0, 1.7], size=n)
    tops = rng.choice([0.05, 0.5, 0.9, 0.95, 1.0], size=n)
    seeds = rng.integers(0, 2 ** 40, size=(n, 4))
    gen = generatable_mask(vocab)
    want = [_sample_nucleus(logits[i].astype(np.float64), gen,
                            SamplingParams(mode="temperature", temperature=float(temps[i]),
                                           top_p=float(tops[i]), seed=int(seeds[i, 1])),
                            int(seeds[i, 0]), int(seeds[i, 2]), int(seeds[i, 3]))
            for i in range(n)]
    lg = torch.from_numpy(logits).cuda()
    params = torch.from_numpy(np.stack([temps, tops], 1).astype(np.float64)).cuda()
    keys = torch.from_numpy(seeds.astype(np.int64)).cuda()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.select_nucleus(lg.data_ptr(), n, vocab, vocab, params.data_ptr(), keys.data_ptr(),
                       out.data_ptr(), _stream())
    assert out.cpu().tolist() == want


@pytest.mark.parametrize("rows,split", [(8, True), (3, True), (20, False), (64, True), (72, True)])
@pytest.mark.parametrize("f,d", [(14336, 4096), (256, 192)])
def test_linear_gate_up_silu_matches_separate(rows, split, f, d):
    """K7 with SwiGLU fused (tiles pair 64 gate rows with their 64 up rows) == K7 on
    [gate; up] then choreo_silu_mul, up to f32 summation order (bf16 outputs within one
    rounding); hi/lo halves when split."""
    torch.manual_seed(rows + f)
    xm = torch.randn(2 * rows if split else rows, d, device="cuda").to(torch.bfloat16)
    w = (torch.randn(2 * f, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
    S = 2 if split else 1
    fused = torch.zeros(S * rows, f, dtype=torch.bfloat16, device="cuda")
    sep = torch.zeros(S * rows, f, dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(148 * 2 * 256 * 128, device="cuda")
    cnt = torch.zeros(2 * f // 128 + 2, dtype=torch.int32, device="cuda")
    nat.linear_gate_up_silu(xm.data_ptr(), xm.shape[0], int(split), w.data_ptr(), f, d,
                            fused.data_ptr(), ws.data_ptr(), cnt.data_ptr(), _stream())
    gu = _linear(xm, split, w)
    nat.silu_mul(gu.data_ptr(), nat.F32, 0, rows, f, sep.data_ptr(), nat.BF16, int(split),
                 _stream())
    torch.cuda.synchronize()
    assert int(cnt.abs().sum()) == 0
    a = fused[:rows].float() + (fused[rows:].float() if split else 0)
    b = sep[:rows].float() + (sep[rows:].float() if split else 0)
    tol = 2e-3 if split else 1e-2  # plain bf16 outputs: one bf16 ulp (<= 0.78 %) apart
    torch.testing.assert_close(a, b, rtol=tol, atol=tol)
    g = (xm.float() @ w[:f].float().t())
    u = (xm.float() @ w[f:].float().t())
    if split:
        g, u = g[:rows] + g[rows:], u[:rows] + u[rows:]
    torch.testing.assert_close(a, torch.nn.functional.silu(g) * u, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("rows,split,grid", [(16, True, 0), (16, True, 37), (8, False, 0),
                                             (40, False, 37), (5, True, 148), (72, True, 0)])
def test_k7_pieces_consumers_bit_identical(rows, split, grid):
    """Deferred K7 outputs (cut tiles left as per-CTA pieces, ChoreoK7Pieces) read through
    RoPE/append and residual+RMSNorm give exactly the values of the reduced K7 path."""
    import ctypes
    H, Hk, hd, d = 8, 2, 128, 1024
    n_qkv = (H + 2 * Hk) * hd
    cfg = ModelConfig(n_layers=2, n_heads=H, n_kv_heads=Hk, head_dim=hd, ffn_dim=64,
                      vocab_size=300, context_window=4096, rope_base=500000.0)
    rot = RotationTableDevice(cfg, "cuda")
    g = torch.Generator(device="cuda").manual_seed(rows + grid)
    xm = torch.randn(2 * rows if split else rows, d, device="cuda", generator=g).to(torch.bfloat16)
    ws = torch.empty(148 * 2 * 256 * 128, device="cuda")
    st = _stream()
    R = rows

    def pieces(w):
        y = torch.full((R, w.shape[0]), float("nan"), device="cuda")
        cnt = torch.zeros((w.shape[0] + 127) // 128, dtype=torch.int32, device="cuda")
        pv = nat.K7Pieces()
        nat.linear_skinny_pieces(xm.data_ptr(), xm.shape[0], int(split), w.data_ptr(), w.shape[0],
                                 w.shape[1], y.data_ptr(), ws.data_ptr(), cnt.data_ptr(), grid,
                                 ctypes.addressof(pv), st)
        assert int(cnt.abs().sum()) == 0
        return y, pv

    # qkv -> RoPE / page append
    w = (torch.randn(n_qkv, d, device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    pos = torch.randint(0, 4096, (R,), dtype=torch.int32, device="cuda")
    flat = torch.randperm(5 * 64, device="cuda")[:R].to(torch.int32)
    page, slot = flat // 64, flat % 64
    outs = []
    for mode in ("reduced", "pieces"):
        kp = torch.zeros(2, Hk, 5, 64, hd, dtype=torch.bfloat16, device="cuda")
        vp = torch.zeros_like(kp)
        q = torch.empty(R, H, hd, device="cuda")
        if mode == "reduced":
            y = _linear(xm, split, w, grid)
            nat.rope_append(y.data_ptr(), nat.F32, n_qkv, R, 0, pos.data_ptr(), page.data_ptr(),
                            slot.data_ptr(), q.data_ptr(), kp.data_ptr(), vp.data_ptr(), nat.BF16, 1,
                            Hk, 5, 64, H, hd, rot.cos.data_ptr(), rot.sin.data_ptr(), rot.max_delta, st)
        else:
            y, pv = pieces(w)
            nat.rope_append_pieces(ctypes.addressof(pv), R, pos.data_ptr(), page.data_ptr(),
                                   slot.data_ptr(), q.data_ptr(), kp.data_ptr(), vp.data_ptr(),
                                   nat.BF16, 1, Hk, 5, 64, H, hd, rot.cos.data_ptr(),
                                   rot.sin.data_ptr(), rot.max_delta, st)
        torch.cuda.synchronize()
        outs.append((q, kp, vp))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    # o_proj / down_proj -> residual add + RMSNorm (hi/lo bf16 out)
    w2 = (torch.randn(d, d, device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    gamma = torch.rand(d, device="cuda", generator=g).to(torch.bfloat16)
    x0 = torch.randn(R, d, device="cuda", generator=g)
    res = []
    for mode in ("reduced", "pieces"):
        x = x0.clone()
        h = torch.empty(2 * R, d, dtype=torch.bfloat16, device="cuda")
        if mode == "reduced":
            y = _linear(xm, split, w2, grid)
            nat.residual_rmsnorm(x.data_ptr(), y.data_ptr(), nat.F32, 0, gamma.data_ptr(), nat.BF16,
                                 R, d, 1e-5, h.data_ptr(), nat.BF16, 1, None, 0, st)
        else:
            y, pv = pieces(w2)
            nat.residual_rmsnorm_pieces(x.data_ptr(), ctypes.addressof(pv), gamma.data_ptr(),
                                        nat.BF16, R, d, 1e-5, h.data_ptr(), nat.BF16, 1, st)
        torch.cuda.synchronize()
        res.append((x, h))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
