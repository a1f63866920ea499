"""CPU-only checks: the C-ABI library loads and exports every declared symbol, and the
host-side logic (layout resolution, K3 sizing, physical-order views, FLOP
accounting, weights) matches the oracle.  No kernel is launched here."""

import os
import re

import numpy as np
import pytest
import torch

from oracle import choreo_oracle as O

import paper_2512_23049_b200 as P
from paper_2512_23049_b200 import _native as nat
from paper_2512_23049_b200.cache import DeviceKvCache, cdiv
from paper_2512_23049_b200.engine import resolve_calls
from paper_2512_23049_b200.model import CallRows, plan_counts

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "choreo_b200.h")


def _prototypes():
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    protos = {}
    for m in re.finditer(r"\b(?:int|const char\*)\s+(choreo_\w+)\s*\(([^)]*)\)\s*;", text):
        args = [a.strip() for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        protos[m.group(1)] = args
    return protos


def test_library_exports_every_declared_symbol():
    protos = _prototypes()
    assert len(protos) >= 11
    lib = nat.load()
    for name in protos:
        assert hasattr(lib, name), name
    assert lib.choreo_abi_version() == 100


def test_ctypes_signatures_match_header():
    protos = _prototypes()
    for name, args in nat.SIGNATURES.items():
        assert name in protos, name
        assert len(args) == len(protos[name]), (name, len(args), len(protos[name]))
    assert set(protos) == set(nat.SIGNATURES) | set(nat.EXTRA)


def test_no_torch_types_in_abi():
    text = open(HEADER).read()
    assert "torch" not in re.sub(r"/\*.*?\*/", "", text, flags=re.S)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(nat, "_lib", None)
    monkeypatch.setattr(nat, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(P.NativeError):
        nat.load()


class _C:
    def __init__(self, parents, offsets=None, new_offset=None):
        self.parents, self.offsets, self.new_offset = parents, offsets, new_offset


@pytest.mark.parametrize("seed", range(40))
def test_resolve_calls_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    W = 256
    lens = {m: int(rng.integers(1, 60)) for m in range(8)}
    calls = []
    for _ in range(int(rng.integers(1, 4))):
        par = [int(p) for p in rng.choice(10, size=int(rng.integers(0, 5)), replace=bool(rng.random() < 0.1))]
        offs = None if rng.random() < 0.4 else [
            None if rng.random() < 0.3 else int(rng.integers(-2, 200)) for _ in par]
        if offs is not None and rng.random() < 0.05:
            offs = offs + [0]
        no = None if rng.random() < 0.5 else int(rng.integers(-1, 250))
        calls.append(_C(par, offs, no))
    new_lens = [int(rng.integers(1, 30)) for _ in calls]
    ora = O.Oracle.__new__(O.Oracle)
    ora.shape = O.Shape(context_window=W)
    ora.store = O.Store(ora.shape, 100)
    for m, n in lens.items():
        ora.store.msgs[m] = O.Msg("prefilled", 0, "", None, list(range(n)))
    want = got = None
    try:
        want = ora.resolve([{"parents": c.parents, "offsets": c.offsets, "new_offset": c.new_offset}
                            for c in calls], new_lens)
    except O.OracleError as e:
        want = e.kind
    try:
        got = resolve_calls(calls, new_lens, lens.get, W)
    except P.ChoreoError as e:
        got = type(e).__name__
    assert got == want


def _cache_cpu(cfg=None):
    cfg = cfg or P.ModelConfig(n_layers=2, n_heads=2, head_dim=8, context_window=256)
    return DeviceKvCache(cfg, capacity=4096, dtype=torch.float32, device="cpu")


def test_interleaved_physical_order_matches_reference_pattern():
    c = _cache_cpu()
    for m in (0, 1, 2):
        c.register_message(m, "decoded", 0)
    lens = [4, 7, 2]
    for m, n in enumerate(lens):
        c.reserve_slots(m, list(range(n)))
    c.log_interleaved([0, 1, 2], [0, 0, 0], lens)
    expected = [m for t in range(max(lens)) for m in range(3) if lens[m] > t]
    assert c.msg_ids.tolist() == expected
    assert c.message_span(1).physical.tolist() == [i for i, m in enumerate(expected) if m == 1]


def test_pages_belong_to_one_message_and_views():
    c = _cache_cpu()
    c.register_message(0, "prefilled", 5, max_tokens=70)
    c.register_message(1, "decoded", 0)
    p0, s0 = c.reserve_slots(0, list(range(70)))
    p1, s1 = c.reserve_slots(1, [7] * 10)
    assert set(p0.tolist()).isdisjoint(p1.tolist())
    assert s0.tolist() == [i % 64 for i in range(70)]
    c.log_append(0, 0, 70)
    c.log_append(1, 0, 10)
    assert c.positions.tolist() == list(range(5, 75)) + list(range(10))
    assert c.token_count == 80
    with pytest.raises(P.CapacityError):
        c.reserve_slots(1, [0] * 5000)


def test_speculative_token_set_and_unreserve():
    """Pipelined decode bookkeeping (engine._decode_loop): a slot reserved for a token the
    host does not know yet gets its id later (set_token), or is undone (unreserve_last):
    length, token count, the device length table and the views return to the state before
    the reservation, the page stays with the message."""
    c = _cache_cpu()
    c.register_message(0, "decoded", 0)
    c.reserve_slots(0, [5, 6, 7])
    pages_before = list(c._messages[0].pages)
    p, s = c.reserve_slots(0, [0])  # speculative: id unknown
    assert s.tolist() == [3] and c.message_length(0) == 4 and c.token_count == 4
    c.set_token(0, 3, 42)
    assert c._messages[0].tokens == [5, 6, 7, 42]
    c.reserve_slots(0, [0])
    c.unreserve_last(0)
    assert c.message_length(0) == 4 and c.token_count == 4
    assert int(c.msg_len.host[0]) == 4
    assert c._messages[0].pages == pages_before
    c.log_append(0, 0, 4)
    assert c.token_ids.tolist() == [5, 6, 7, 42]
    # a stop right at a page boundary: the new page stays allocated but unused
    c.register_message(1, "decoded", 0)
    c.reserve_slots(1, list(range(64)))
    c.reserve_slots(1, [0])
    assert len(c._messages[1].pages) == 2
    c.unreserve_last(1)
    assert c.message_length(1) == 64 and c.token_count == 68


def test_page_chain_relocates_when_reservation_is_exceeded():
    c = _cache_cpu()
    c.register_message(0, "decoded", 0, max_tokens=10)  # reserves one page-table entry
    pages, _ = c.reserve_slots(0, list(range(200)))
    e = c._messages[0]
    assert len(e.pages) == 4 and e.pt_cap >= 4
    assert c.page_table.host[e.pt:e.pt + 4].tolist() == e.pages
    assert c.msg_pt.host[0] == e.pt


def _brute_counts(calls, msg_len, P_, rpb, ppi):
    """Token-free restatement of K3's page-centric plan: one group per distinct parent
    (viewers = rows of every call listing it), one causal own group per call."""
    viewers = {}
    for c in calls:
        for p in c.parents:
            viewers.setdefault(p, []).extend([0] * len(c.tokens))
    v = sum(cdiv(msg_len[p], P_) for p in viewers)
    blk = sum(len(r) for r in viewers.values())
    it = sum(cdiv(len(r), rpb) * cdiv(cdiv(msg_len[p], P_), ppi) for p, r in viewers.items() if r)
    pa = sum(len(r) * cdiv(cdiv(msg_len[p], P_), ppi) for p, r in viewers.items())
    for c in calls:
        ts = [c.first_t + i for i in range(len(c.tokens))]
        v += ts[-1] // P_ + 1
        blk += len(ts)
        for i in range(0, len(ts), rpb):
            b = ts[i:i + rpb]
            ch = cdiv(b[-1] // P_ + 1, ppi)
            it += ch
            pa += ch * len(b)
    return v, blk, it, pa


def _brute_percall(calls, msg_len, P_, rpb, ppi):
    v = blk = it = pa = 0
    for c in calls:
        pp = sum(cdiv(msg_len[p], P_) for p in c.parents)
        ts = [c.first_t + i for i in range(len(c.tokens))]
        v += pp + ts[-1] // P_ + 1
        blk += len(ts)
        for i in range(0, len(ts), rpb):
            b = ts[i:i + rpb]
            ch = cdiv(pp + b[-1] // P_ + 1, ppi)
            it += ch
            pa += ch * len(b)
    return v, blk, it, pa


@pytest.mark.parametrize("seed", range(10))
def test_plan_counts(seed):
    rng = np.random.default_rng(seed)
    msg_len = rng.integers(1, 300, 20)
    calls = [CallRows(int(20 + i), [int(p) for p in rng.permutation(20)[:rng.integers(0, 6)]],
                      int(rng.integers(0, 100)), [0] * int(rng.integers(1, 80)), None, None, 0)
             for i in range(int(rng.integers(1, 6)))]
    for rpb, ppi in ((1, 1), (16, 3), (4, 1000)):
        pm = plan_counts(calls, msg_len, 64, rpb, ppi, 1)
        want = _brute_percall(calls, msg_len, 64, rpb, ppi)
        assert (pm.n_vis, pm.n_blk_rows, pm.n_items, pm.n_parts) == want
        pl = plan_counts(calls, msg_len, 64, rpb, ppi)
        assert (pl.n_vis, pl.n_blk_rows, pl.n_items, pl.n_parts) == \
            _brute_counts(calls, msg_len, 64, rpb, ppi)


@pytest.mark.parametrize("shape", [O.TINY, O.Shape(n_layers=3, n_heads=8, n_kv_heads=2, head_dim=16,
                                                    ffn_dim=64, vocab_size=300)])
def test_encode_flops_matches_oracle(shape):
    cfg = P.ModelConfig(**{k: getattr(shape, k) for k in shape.__dataclass_fields__})
    for t, ctx, rows in ((1, 0, "all"), (19, 7, "none"), (5, 100, "last"), (0, 3, "all")):
        assert P.encode_flops(cfg, t, ctx, rows) == sum(O.encode_flops(shape, t, ctx, rows).values())


def test_product_init_weights_bitwise_oracle_and_device_layout():
    ws = P.init_weights(P.DEFAULT_CONFIG)
    ow = O.init_weights(O.TINY)
    np.testing.assert_array_equal(ws.layers[3].w_up, ow["layers"][3]["w_up"])
    np.testing.assert_array_equal(ws.out_head, ow["out_head"])
    dw = P.DeviceWeights.from_host(ws, dtype=torch.float32, device="cpu")
    l0 = ws.layers[0]
    want = np.concatenate([l0.wq, l0.wk, l0.wv], axis=1).T.astype(np.float32)
    np.testing.assert_array_equal(dw.layers[0]["w_qkv"].numpy(), want)
    assert dw.out_head.shape == (512, 64)


def test_config_roundtrip_and_presets():
    assert P.DEFAULT_CONFIG.to_dict() == O.TINY.ref_dict()
    cfg = P.LLAMA_3_1_8B
    assert (cfg.model_dim, cfg.kv_dim, cfg.kv_heads) == (4096, 1024, 8)
    assert P.ModelConfig.from_dict(cfg.to_dict()) == cfg
    with pytest.raises(ValueError):
        P.ModelConfig(n_heads=6, n_kv_heads=4)


def _rows(msg, parents, n_tok):
    return CallRows(msg, list(parents), 0, [1] * n_tok, np.zeros(n_tok, np.int32),
                    np.zeros(n_tok, np.int32), 0)


def test_split_plan_respects_k3_limits():
    """Steps past K3's 1024 calls / 4096 page-centric pairs are cut in call order; the logit
    rows are remapped per piece and concatenate back to the step's (model.split_plan)."""
    from paper_2512_23049_b200.model import (K3_MAX_CALLS, K3_MAX_PAIRS, StepPlan,
                                             split_plan)
    rng = np.random.default_rng(0)
    for n_calls, max_par in ((64, 70), (1030, 0), (3000, 5), (10, 4200), (5, 3)):
        calls = [_rows(1_000_000 + i, rng.choice(9000, int(rng.integers(0, max_par + 1)),
                                                 replace=False), int(rng.integers(1, 4)))
                 for i in range(n_calls)]
        n_rows = sum(len(c.tokens) for c in calls)
        lr = np.sort(rng.choice(n_rows, min(n_rows, 200), replace=False)).astype(np.int32)
        pieces = split_plan(StepPlan(calls, lr))
        assert [c for p, _ in pieces for c in p.calls] == calls
        base, got = 0, []
        for p, percall in pieces:
            pairs = sum(len(c.parents) for c in p.calls)
            assert len(p.calls) <= K3_MAX_CALLS
            assert percall == (pairs > K3_MAX_PAIRS)
            if percall:
                assert len(p.calls) == 1
            got += (np.asarray(p.logit_rows) + base).tolist()
            base += p.n_rows
        assert got == lr.tolist()
        if n_calls <= K3_MAX_CALLS and sum(len(c.parents) for c in calls) <= K3_MAX_PAIRS:
            assert len(pieces) == 1
    # parent ids past the 21-bit sort key take per-call lists
    (p, percall), = split_plan(StepPlan([_rows(1, [1 << 21], 1)], np.zeros(1, np.int32)))
    assert percall


def test_ctypes_struct_mirrors_match_the_c_header(tmp_path):
    """The ctypes mirrors of the ABI structs (ChoreoK7Pieces, ChoreoDecodeStep,
    ChoreoLayerChain) have the header's field names, order, offsets and size: a C program
    compiled against include/choreo_b200.h prints offsetof / sizeof for every field."""
    import ctypes
    import shutil
    import subprocess

    from paper_2512_23049_b200 import _native as nat

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    hdr = os.path.join(ROOT, "include", "choreo_b200.h")
    text = open(hdr).read()
    mirrors = {"ChoreoK7Pieces": nat.K7Pieces, "ChoreoDecodeStep": nat.DecodeStep,
               "ChoreoLayerChain": nat.LayerChain}
    prog = ["#include <stddef.h>", "#include <stdio.h>", '#include "choreo_b200.h"',
            "int main(void) {"]
    for cname, py in mirrors.items():
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + cname + ";", text).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        names = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            for part in decl.split(","):
                m = re.search(r"(\w+)\s*(\[[^\]]*\])?\s*$", part.strip())
                names.append(m.group(1))
        assert [f[0] for f in py._fields_] == names, cname
        for n in names:
            prog.append(f'  printf("{cname} {n} %zu\\n", offsetof({cname}, {n}));')
        prog.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
    prog.append("  return 0;\n}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(prog))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, out):
        cname, field, val = line.split()
        py = mirrors[cname]
        got = ctypes.sizeof(py) if field == "sizeof" else getattr(py, field).offset
        assert got == int(val), (cname, field, got, val)
