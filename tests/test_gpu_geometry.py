"""Parity at the benchmark's own geometry.

The bench runs Llama-3.1-8B shapes: K7 over every decode GEMM including the 128256-row
head, K5 v2 over 8-32 pages per work item with 8 rows per unit, merged C4 ticks of eight
workflows, and 32 layers.  These tests check values at those shapes, not just smaller
stand-ins: K7 against an f32 matmul of the same bf16 operands, K5 v2 against a dense
f64 softmax over the oracle's visible sets, and the engine end to end against the CPU
oracle on the same bf16 weights (teacher-forced, logits within 2e-2).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import choreo_oracle as O  # noqa: E402

import paper_2512_23049_b200 as P  # noqa: E402
from paper_2512_23049_b200 import _native as nat  # noqa: E402
from paper_2512_23049_b200.cache import DeviceKvCache  # noqa: E402
from paper_2512_23049_b200.config import ModelConfig  # noqa: E402

from .test_gpu_kernels import _assemble, _expand_rows, _stream  # noqa: E402

pytestmark = pytest.mark.gpu

D, F, V = 4096, 14336, 128256
SHAPES_8B = {"qkv": (6144, D), "o_proj": (D, D), "down": (D, F), "head": (V, D)}


def _k7(x, split, w):
    rows = x.shape[0] // (2 if split else 1)
    y = torch.full((rows, w.shape[0]), float("nan"), device="cuda")
    ws = torch.empty(148 * 2 * 256 * 128, device="cuda")
    cnt = torch.zeros((w.shape[0] + 127) // 128, dtype=torch.int32, device="cuda")
    nat.linear_skinny(x.data_ptr(), x.shape[0], int(split), w.data_ptr(), w.shape[0], w.shape[1],
                      y.data_ptr(), ws.data_ptr(), cnt.data_ptr(), 0, _stream())
    torch.cuda.synchronize()
    assert int(cnt.abs().sum()) == 0
    return y


@pytest.mark.parametrize("rows", [8, 64, 72, 128])
@pytest.mark.parametrize("name", sorted(SHAPES_8B))
def test_k7_values_at_8b_decode_shapes(name, rows):
    """K7 at the bench's decode GEMMs (8 agents = 16 stacked hi/lo rows, NX 16), at 64 rows
    (NX 128), at the C3 parallel header step (8 agents x 9 header tokens = 72 rows = 144
    stacked, NX 256) and at its 128-row limit, including the 128256 x 4096 head (1002
    tiles, 1 GB of weights):
    within 1e-4 relative of the f32 matmul of the same bf16 operands, bitwise
    deterministic run to run."""
    torch.backends.cuda.matmul.allow_tf32 = False
    n, k = SHAPES_8B[name]
    g = torch.Generator(device="cuda").manual_seed(n + rows)
    x = torch.randn(rows, k, device="cuda", generator=g)
    hi = x.to(torch.bfloat16)
    lo = (x - hi.float()).to(torch.bfloat16)
    xm = torch.cat([hi, lo])
    w = ((torch.rand(n, k, device="cuda", generator=g) * 2 - 1) * (6 / (n + k)) ** 0.5
         ).to(torch.bfloat16)
    y = _k7(xm, True, w)
    ref = hi.float() @ w.float().t() + lo.float() @ w.float().t()
    scale = float(ref.abs().max())
    err = float((y - ref).abs().max())
    assert err <= 1e-4 * scale, (err, scale)
    assert torch.equal(_k7(xm, True, w), y)
    # and the hi/lo pair reproduces the f32 activations' product to bf16-pair accuracy
    exact = x @ w.float().t()
    assert float((y - exact).abs().max()) <= 1e-3 * float(exact.abs().max())


@pytest.mark.parametrize("rows", [8, 64, 72])
def test_k7_gate_up_silu_at_8b(rows):
    """The fused gate|up + SiLU epilogue at the 8B FFN (28672 x 4096 weights)."""
    g = torch.Generator(device="cuda").manual_seed(rows)
    x = torch.randn(rows, D, device="cuda", generator=g)
    hi = x.to(torch.bfloat16)
    lo = (x - hi.float()).to(torch.bfloat16)
    xm = torch.cat([hi, lo])
    w = ((torch.rand(2 * F, D, device="cuda", generator=g) * 2 - 1) * (6 / (D + F)) ** 0.5
         ).to(torch.bfloat16)
    act = torch.empty(2 * rows, F, dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(148 * 2 * 256 * 128, device="cuda")
    cnt = torch.zeros(F // 64 + 1, dtype=torch.int32, device="cuda")
    nat.linear_gate_up_silu(xm.data_ptr(), 2 * rows, 1, w.data_ptr(), F, D, act.data_ptr(),
                            ws.data_ptr(), cnt.data_ptr(), _stream())
    torch.cuda.synchronize()
    got = act[:rows].float() + act[rows:].float()
    gu = hi.float() @ w.float().t() + lo.float() @ w.float().t()
    want = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
    err = float((got - want).abs().max())
    assert err <= 2e-5 * float(want.abs().max()) + 1e-6, err


@pytest.mark.parametrize("ppi", [8, 16, 32])
def test_k5v2_at_debate_geometry(ppi):
    """K5 v2 at the C3 round-2 geometry: 8 agents (one row each, 8 rows per unit at G = 4)
    sharing 10 reordered parents of 256-512 tokens (two of them 1.5-2K tokens, so that
    one message spans several 8 / 16 / 32-page items), each with its own 300-token pages.  Within 2e-2 of the dense f64 softmax over the oracle's
    visible sets (Q as a hi/lo bf16 pair, P bf16, f32 accumulation)."""
    H, Hk, hd = 32, 8, 128
    rng = np.random.default_rng(ppi)
    cfg = ModelConfig(n_layers=2, n_heads=H, n_kv_heads=Hk, head_dim=hd)
    cache = DeviceKvCache(cfg, capacity=1 << 16, dtype=torch.bfloat16, device="cuda")
    n_par = 10
    for m in range(n_par):
        n = int(rng.integers(256, 513)) if m >= 2 else int(rng.integers(1500, 2100))
        cache.register_message(m, "prefilled", 0, max_tokens=n)
        cache.reserve_slots(m, [1] * n)
        cache.log_append(m, 0, n)
    calls = []
    for a in range(8):
        own = n_par + a
        n = int(rng.integers(280, 320))
        cache.register_message(own, "decoded", 0, max_tokens=n)
        cache.reserve_slots(own, [1] * n)
        cache.log_append(own, 0, n)
        parents = [int(p) for p in rng.permutation(n_par)[:9]]
        calls.append((own, parents, [n - 1]))
    cache.k_pool.copy_(torch.randn_like(cache.k_pool))
    cache.v_pool.copy_(torch.randn_like(cache.v_pool))
    rpb = 32 // (H // Hk)
    out, (rt_d, vis, blk, items, rpo, rp, counts) = _assemble(cache, calls, rpb, ppi, 0)
    R, pl_ = len(out["row_t"]), out["plan"]
    assert max(int(it[3]) for it in out["items"][:out["counts"][1]]) == ppi  # full items
    q = torch.randn(R, H, hd, device="cuda")
    part_o = torch.empty(pl_.n_parts, H, hd, device="cuda")
    part_lse = torch.empty(pl_.n_parts, H, device="cuda")
    o = torch.empty(R, H * hd, dtype=torch.float32, device="cuda")
    L = 1
    nat.decode_attn_v2(q.data_ptr(), cache.k_pool.data_ptr(), cache.v_pool.data_ptr(), 2, L, Hk,
                       cache.n_pages, 64, H, hd, rt_d.data_ptr(), vis[0].data_ptr(),
                       vis[1].data_ptr(), vis[2].data_ptr(), blk.data_ptr(), items.data_ptr(),
                       counts.data_ptr(), pl_.n_items, part_o.data_ptr(), part_lse.data_ptr(),
                       None, 0, _stream())
    nat.attn_combine(part_o.data_ptr(), part_lse.data_ptr(), rpo.data_ptr(), rp.data_ptr(), R, H,
                     hd, o.data_ptr(), nat.F32, 0, _stream())
    torch.cuda.synchronize()
    got = o.cpu().numpy().reshape(R, H, hd)
    sets = _expand_rows(cache, out, R)
    K = cache.k_pool[L].float().cpu().numpy().astype(np.float64)
    Vv = cache.v_pool[L].float().cpu().numpy().astype(np.float64)
    qn = q.cpu().numpy().astype(np.float64)
    G, worst = H // Hk, 0.0
    for r in range(R):
        assert len(sets[r]) > 2000
        pg = np.array([cache._messages[m].pages[i // 64] for m, i in sets[r]])
        sl = np.array([i % 64 for m, i in sets[r]])
        for h in range(H):
            s = K[h // G, pg, sl] @ qn[r, h] / np.sqrt(hd)
            p = np.exp(s - s.max())
            p /= p.sum()
            worst = max(worst, float(np.abs(got[r, h] - p @ Vv[h // G, pg, sl]).max()))
    assert worst < 2e-2, worst


class _OracleAdapter:
    """The oracle behind the Engine call surface, so BatchScheduler can drive it."""

    def __init__(self, ref):
        self.ref = ref

    def prefill_parallel(self, calls):
        return self.ref.prefill_batch([{"message": c.message, "parents": list(c.parents),
                                        "offsets": c.offsets, "new_offset": c.new_offset}
                                       for c in calls])

    def decode_parallel(self, calls, force_tokens=None):
        return self.ref.decode_batch(
            [{"header": c.header, "parents": list(c.parents), "offsets": c.offsets,
              "new_offset": c.new_offset,
              "sampling": O.Sampling(max_tokens=c.sampling.max_tokens)} for c in calls],
            force_tokens)

    def message_token_count(self, m):
        return self.ref.token_count(m)

    @property
    def last_stats(self):
        return self.ref.stats[-1]


def test_c4_merged_tick_of_eight_workflows_matches_oracle():
    """Eight C4 workflows (16 prefilled messages each, rounds of 4 decodes over reordered
    >= 50 % parent subsets with gaps and 25 % overlaps) merged by BatchScheduler into one
    engine call per tick, at the 8B attention geometry (hd 128, 4 query heads per KV
    head): every decoded message's logits within 2e-2 of the oracle driven through the
    same scheduler; physical layout bit-exact."""
    import bench

    shape = O.Shape(n_layers=2, n_heads=8, n_kv_heads=2, head_dim=128, ffn_dim=1024,
                    vocab_size=512, context_window=16384, rope_base=500000.0)
    cfg = ModelConfig(**{k: getattr(shape, k) for k in shape.__dataclass_fields__})
    ref = O.Oracle(O.round_weights(O.init_weights(shape, dtype=np.float32), "bf16"), shape,
                   capacity=1 << 17, record_logits=True)
    eng = P.Engine(P.DeviceWeights.from_host(P.init_weights(cfg).rounded("bf16"),
                                             dtype=torch.bfloat16), capacity=1 << 17,
                   record_logits=True)
    eng._runner.check_assembly = True
    kw = dict(n_prefill=16, n_rounds=2, n_dec=4, pre_len=(64, 513), dec_len=(12, 40))
    seeds = list(range(100, 108))
    ids_e = P.BatchScheduler(eng).run([bench.c4_workflow(eng, P, s, **kw) for s in seeds])
    ad = _OracleAdapter(ref)
    ids_o = P.BatchScheduler(ad).run([bench.c4_workflow(ad, P, s, **kw) for s in seeds])
    assert ids_e == ids_o
    got = {m: rows for st in eng.stats if st.logits for m, rows in st.logits.items()}
    want = {m: rows for st in ref.stats if st.logits for m, rows in st.logits.items()}
    worst = 0.0
    for m in (m for wf in ids_e for m in wf):
        a, b = np.stack(got[m]), np.stack(want[m])
        assert a.shape == b.shape
        worst = max(worst, float(np.abs(a - b).max()))
    assert worst <= 2e-2, worst
    n = eng.cache.token_count
    assert eng.cache.msg_ids[:n].tolist() == ref.store.mid[:n].tolist()
    assert eng.cache.positions[:n].tolist() == ref.store.pos[:n].tolist()


def _host_copy(dw: P.DeviceWeights, cfg: ModelConfig) -> dict:
    """Device weights (fused, (out, in), bf16) back to the oracle's layout in f32."""
    d, dkv, f = cfg.model_dim, cfg.kv_dim, cfg.ffn_dim
    h = lambda t: t.float().cpu().numpy()  # noqa: E731
    layers = []
    for lw in dw.layers:
        qkv = h(lw["w_qkv"])
        gu = h(lw["w_gu"])
        layers.append({"attn_norm": h(lw["attn_norm"]), "wq": qkv[:d].T.copy(),
                       "wk": qkv[d:d + dkv].T.copy(), "wv": qkv[d + dkv:].T.copy(),
                       "wo": h(lw["wo"]).T.copy(), "ffn_norm": h(lw["ffn_norm"]),
                       "w_gate": gu[:f].T.copy(), "w_up": gu[f:].T.copy(),
                       "w_down": h(lw["w_down"]).T.copy()})
    return {"embed": h(dw.embed), "out_norm": h(dw.out_norm), "out_head": h(dw.out_head).T.copy(),
            "layers": layers}


def test_llama8b_eight_layers_full_vocab_matches_oracle():
    """Llama-3.1-8B width, 8 layers, the full 128256-row head, device-drawn bf16 weights
    (the bench's DeviceWeights.random) pulled to the host for the oracle: a moved-parent
    prefill (K2 + K4), then an 8-agent parallel decode (header step + K7 / K5 v2 decode
    steps through the native executor).  Teacher-forced on the oracle's greedy tokens,
    logits within 2e-2; positions bit-exact."""
    cfg = ModelConfig(n_layers=8, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=F,
                      vocab_size=V, context_window=8192, rope_base=500000.0)
    dw = P.DeviceWeights.random(cfg, dtype=torch.bfloat16, seed=3)
    shape = O.Shape(**{k: getattr(cfg, k) for k in O.Shape.__dataclass_fields__})
    ref = O.Oracle(_host_copy(dw, cfg), shape, capacity=8192, record_logits=True)
    eng = P.Engine(dw, capacity=8192, record_logits=True)
    rng = np.random.default_rng(4)
    texts = ["".join(chr(97 + int(c)) for c in rng.integers(0, 26, n)) for n in (300, 180, 90)]
    for t in texts:
        ref.prefill({"message": t})
        eng.prefill(P.PrefillCall(t))
    ref.prefill({"message": texts[2][:70], "parents": [2, 0], "offsets": [0, 150]})
    eng.prefill(P.PrefillCall(texts[2][:70], parents=[2, 0], offsets=[0, 150]))
    sp_o, sp_p = O.Sampling(max_tokens=5), P.SamplingParams(max_tokens=5)
    calls = [(f"Agent {a}:", [[3, 1, 0], [0, 3], [1, 2, 3]][a % 3],
              [[0, 80, 300], [300, 0], [80, 600, 0]][a % 3]) for a in range(8)]
    ref_ids = ref.decode_batch([{"header": h, "parents": p, "offsets": o, "sampling": sp_o}
                                for h, p, o in calls])
    ids = eng.decode_parallel([P.DecodeCall(h, parents=p, offsets=o, sampling=sp_p)
                               for h, p, o in calls],
                              force_tokens=[ref.generated(m) for m in ref_ids])
    assert ids == ref_ids
    worst = 0.0
    for m in ids:
        a = np.stack(eng.stats[-1].logits[m])
        b = np.stack(ref.stats[-1].logits[m])
        assert a.shape == b.shape == (5, V)
        worst = max(worst, float(np.abs(a - b).max()))
    assert worst <= 2e-2, worst
    n = eng.cache.token_count
    assert eng.cache.positions[:n].tolist() == ref.store.pos[:n].tolist()
