"""K8 layer chain (choreo_layer_chain / choreo_chain_prologue) against a plain PyTorch
fp64 reference of the same layer math (reference model.py:169-189 and cache.py:98-135):

    x1 = x + attn @ Wo^T ; a = silu(norm(x1) g_ffn @ Wg^T) * (norm(x1) g_ffn @ Wu^T)
    x2 = x1 + a @ Wd^T   ; qkv = norm(x2) g_attn' @ Wqkv^T -> RoPE(q, k) at pos, K/V appended

The chain carries every GEMM input as a hi/lo bf16 pair (~16 mantissa bits) and applies
RMSNorm as a row scale of the next GEMM's output, so values agree to ~1e-4 relative; the
weights are the same bf16 numbers on both sides.  Also checked: a two-launch sequence
(qkv-only prologue launch, then a full layer), deterministic (bitwise) repeats, and
counters left zero.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2512_23049_b200 import _native as nat  # noqa: E402


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _split(t: torch.Tensor, split: bool) -> torch.Tensor:
    hi = t.to(torch.bfloat16)
    if not split:
        return hi.contiguous()
    lo = (t - hi.float()).to(torch.bfloat16)
    return torch.cat([hi, lo]).contiguous()


class _Layer:
    def __init__(self, d, H, Hk, hd, F, seed):
        g = torch.Generator(device="cuda").manual_seed(seed)

        def w(n, k):
            return (torch.randn(n, k, device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)

        self.wo, self.w_gu, self.w_down = w(d, H * hd), w(2 * F, d), w(d, F)
        self.w_qkv = w((H + 2 * Hk) * hd, d)
        self.g_ffn = (1 + 0.1 * torch.randn(d, device="cuda", generator=g)).to(torch.bfloat16)
        self.g_attn = (1 + 0.1 * torch.randn(d, device="cuda", generator=g)).to(torch.bfloat16)


def _rope_tables(hd, W, base=10000.0):
    half = hd // 2
    dl = np.arange(-W, W + 1, dtype=np.float64)[:, None]
    inv = base ** (-2.0 * np.arange(half) / hd)
    ang = dl * inv[None, :]
    return (torch.from_numpy(np.cos(ang).astype(np.float32).ravel()).cuda(),
            torch.from_numpy(np.sin(ang).astype(np.float32).ravel()).cuda())


def _rope_ref(a, pos, cos_t, sin_t, W, hd):
    """a: (R, heads, hd) f64; interleaved pairs rotated by the table row pos + W."""
    half = hd // 2
    idx = (pos.long() + W)[:, None] * half + torch.arange(half, device=a.device)[None, :]
    c = cos_t[idx].double()[:, None, :]
    s = sin_t[idx].double()[:, None, :]
    e, o = a[..., 0::2], a[..., 1::2]
    y = torch.empty_like(a)
    y[..., 0::2] = e * c - o * s
    y[..., 1::2] = e * s + o * c
    return y


def _norm(x, g, eps=1e-6):
    return x / torch.sqrt((x * x).mean(-1, keepdim=True) + eps) * g.double()


class _Bufs:
    def __init__(self, R, d, H, Hk, hd, F, split, P=64, n_pages=8, layers=2):
        S = 2 if split else 1
        dev = "cuda"
        self.x = torch.empty(R, d, device=dev)
        self.attn = torch.empty(S * R, H * hd, dtype=torch.bfloat16, device=dev)
        self.h_a = torch.zeros(S * R, d, dtype=torch.bfloat16, device=dev)
        self.h_b = torch.zeros(S * R, d, dtype=torch.bfloat16, device=dev)
        self.act = torch.zeros(S * R, F, dtype=torch.bfloat16, device=dev)
        tiles = (d + 127) // 128
        self.ssq_a = torch.zeros(tiles * 128, device=dev)
        self.ssq_b = torch.zeros(tiles * 128, device=dev)
        self.q = torch.zeros(R, H, hd, device=dev)
        self.k_pool = torch.zeros(layers, Hk, n_pages, P, hd, dtype=torch.bfloat16, device=dev)
        self.v_pool = torch.zeros_like(self.k_pool)
        self.ws = torch.empty(4 * 148 * 2 * 128 * 128, device=dev)
        self.counters = torch.zeros(4 * 1024, dtype=torch.int32, device=dev)
        self.done = torch.zeros(8, dtype=torch.int32, device=dev)


def _chain(b, lw, R, d, H, Hk, hd, F, split, phases, layer_qkv, pos, page, slot, cos_t, sin_t,
           W, attn_norm_next=True):
    c = nat.LayerChain(n_rows=R, split=int(split), d=d, n_heads=H, n_kv=Hk, head_dim=hd,
                       ffn_dim=F, eps=1e-6, phases=phases, wo=lw.wo.data_ptr(),
                       ffn_norm=lw.g_ffn.data_ptr(), w_gu=lw.w_gu.data_ptr(),
                       w_down=lw.w_down.data_ptr(),
                       attn_norm_next=lw.g_attn.data_ptr() if attn_norm_next else None,
                       w_qkv=lw.w_qkv.data_ptr(), layer_qkv=layer_qkv, x=b.x.data_ptr(),
                       attn=b.attn.data_ptr(), h_a=b.h_a.data_ptr(), act=b.act.data_ptr(),
                       h_b=b.h_b.data_ptr(), ssq_a=b.ssq_a.data_ptr(), ssq_b=b.ssq_b.data_ptr(),
                       q=b.q.data_ptr(), k_pool=b.k_pool.data_ptr(), v_pool=b.v_pool.data_ptr(),
                       n_pages=b.k_pool.shape[2], page_size=b.k_pool.shape[3],
                       pos=pos.data_ptr(), page=page.data_ptr(), slot=slot.data_ptr(),
                       cos_t=cos_t.data_ptr(), sin_t=sin_t.data_ptr(), max_delta=W,
                       ws=b.ws.data_ptr(), counters=b.counters.data_ptr(),
                       done=b.done.data_ptr())
    nat.layer_chain(ctypes.byref(c), _stream())


SHAPES = [  # (R, split, d, H, Hk, hd, F)
    (1, True, 512, 8, 2, 64, 1024),
    (8, True, 1024, 8, 2, 128, 2048),
    (8, True, 4096, 32, 8, 128, 14336),   # Llama-3.1-8B widths, one layer
    (20, False, 512, 8, 4, 64, 768),
    (40, True, 768, 6, 2, 128, 1536),     # NX = 128
    (72, True, 1024, 8, 2, 128, 2048),    # the C3 header step: 144 stacked rows, NX = 256
]


@pytest.mark.parametrize("R,split,d,H,Hk,hd,F", SHAPES)
def test_layer_chain_matches_fp64_reference(R, split, d, H, Hk, hd, F):
    torch.manual_seed(R * 7 + d)
    lw = _Layer(d, H, Hk, hd, F, seed=R + d)
    b = _Bufs(R, d, H, Hk, hd, F, split)
    W = 4096
    cos_t, sin_t = _rope_tables(hd, W)
    pos = torch.randint(0, 3000, (R,), dtype=torch.int32, device="cuda")
    perm = torch.randperm(b.k_pool.shape[2] * b.k_pool.shape[3], device="cuda")[:R]
    page = (perm // b.k_pool.shape[3]).int()
    slot = (perm % b.k_pool.shape[3]).int()
    x0 = torch.randn(R, d, device="cuda")
    a0 = torch.randn(R, H * hd, device="cuda")
    b.x.copy_(x0)
    b.attn.copy_(_split(a0, split))
    L1 = 1  # the qkv phase appends to pool layer 1
    _chain(b, lw, R, d, H, Hk, hd, F, split, 15, L1, pos, page, slot, cos_t, sin_t, W)
    torch.cuda.synchronize()
    assert int(b.counters.abs().sum()) == 0 and int(b.done.abs().sum()) == 0

    # fp64 reference on the same (bf16) weights; attn as the chain sees it (hi/lo sum)
    A = b.attn.double()
    A = A[:R] + A[R:] if split else A
    x1 = x0.double() + A @ lw.wo.double().t()
    h = _norm(x1, lw.g_ffn)
    gu = h @ lw.w_gu.double().t()
    act = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
    x2 = x1 + act @ lw.w_down.double().t()
    qkv = _norm(x2, lw.g_attn) @ lw.w_qkv.double().t()
    q = _rope_ref(qkv[:, :H * hd].reshape(R, H, hd), pos, cos_t, sin_t, W, hd)
    k = _rope_ref(qkv[:, H * hd:(H + Hk) * hd].reshape(R, Hk, hd), pos, cos_t, sin_t, W, hd)
    v = qkv[:, (H + Hk) * hd:].reshape(R, Hk, hd)

    # hi/lo inputs: ~2^-17 relative per GEMM input; plain bf16 (split=False): ~2^-9
    tx, tq, tk = (2e-4, 2e-3, 8e-3) if split else (3e-2, 3e-2, 3e-2)
    torch.testing.assert_close(b.x.double(), x2, rtol=tx, atol=tx)
    torch.testing.assert_close(b.q.double(), q, rtol=tq, atol=tq)
    kc = b.k_pool[L1][:, page.long(), slot.long()].permute(1, 0, 2).double()
    vc = b.v_pool[L1][:, page.long(), slot.long()].permute(1, 0, 2).double()
    # K/V are stored in bf16: one rounding (<= 2^-8 relative)
    torch.testing.assert_close(kc, k, rtol=tk, atol=tk)
    torch.testing.assert_close(vc, v, rtol=tk, atol=tk)
    assert int(b.k_pool[0].abs().sum()) == 0  # nothing written outside layer L1

    # bitwise deterministic: same inputs again (completion counters were left zero)
    q1, x1d, k1 = b.q.clone(), b.x.clone(), b.k_pool.clone()
    b.x.copy_(x0)
    _chain(b, lw, R, d, H, Hk, hd, F, split, 15, L1, pos, page, slot, cos_t, sin_t, W)
    torch.cuda.synchronize()
    assert torch.equal(b.q, q1) and torch.equal(b.x, x1d) and torch.equal(b.k_pool, k1)


@pytest.mark.parametrize("R,split", [(8, True), (72, True), (5, False)])
def test_chain_prologue_then_layer(R, split):
    """prologue (x -> hi/lo(x g), ssq) + qkv-only launch, then o|gu|d without a next layer:
    q / K / V of layer 0 and the final residual x."""
    d, H, Hk, hd, F = 512, 8, 2, 64, 1024
    torch.manual_seed(R)
    lw = _Layer(d, H, Hk, hd, F, seed=3 + R)
    b = _Bufs(R, d, H, Hk, hd, F, split)
    W = 512
    cos_t, sin_t = _rope_tables(hd, W)
    pos = torch.arange(R, dtype=torch.int32, device="cuda") + 7
    page = (torch.arange(R, device="cuda") // 64).int()
    slot = (torch.arange(R, device="cuda") % 64).int()
    x0 = torch.randn(R, d, device="cuda")
    dl = torch.randn(R, d, device="cuda")
    b.x.copy_(x0)
    nat.chain_prologue(b.x.data_ptr(), dl.data_ptr(), R, d, lw.g_attn.data_ptr(), b.h_b.data_ptr(),
                       int(split), b.ssq_b.data_ptr(), _stream())
    _chain(b, lw, R, d, H, Hk, hd, F, split, 8, 0, pos, page, slot, cos_t, sin_t, W)
    a0 = torch.randn(R, H * hd, device="cuda")
    b.attn.copy_(_split(a0, split))
    _chain(b, lw, R, d, H, Hk, hd, F, split, 7, 0, pos, page, slot, cos_t, sin_t, W,
           attn_norm_next=False)
    torch.cuda.synchronize()
    xa = x0.double() + dl.double()
    qkv = _norm(xa, lw.g_attn) @ lw.w_qkv.double().t()
    q = _rope_ref(qkv[:, :H * hd].reshape(R, H, hd), pos, cos_t, sin_t, W, hd)
    v = qkv[:, (H + Hk) * hd:].reshape(R, Hk, hd)
    tx, tq, tk = (2e-4, 2e-3, 8e-3) if split else (3e-2, 3e-2, 3e-2)
    torch.testing.assert_close(b.q.double(), q, rtol=tq, atol=tq)
    vc = b.v_pool[0][:, page.long(), slot.long()].permute(1, 0, 2).double()
    torch.testing.assert_close(vc, v, rtol=tk, atol=tk)
    A = b.attn.double()
    A = A[:R] + A[R:] if split else A
    x1 = xa + A @ lw.wo.double().t()
    gu = _norm(x1, lw.g_ffn) @ lw.w_gu.double().t()
    x2 = x1 + (torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]) @ lw.w_down.double().t()
    torch.testing.assert_close(b.x.double(), x2, rtol=tx, atol=tx)
