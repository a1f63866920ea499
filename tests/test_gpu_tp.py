"""Tensor-parallel engine on the GPU (config C5's layout at small scale).

Two processes share the one B200 of this run; each holds the KV-head slice of the
weights and of every cache page, and the two row-parallel projections are all-reduced
over a gloo group (gloo reduces CUDA tensors; on an 8-GPU box the same code runs with
NCCL).  Logits must match the unsharded oracle (f32 variant, 1e-4).
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import choreo_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPE = O.Shape(n_layers=2, n_heads=8, n_kv_heads=4, head_dim=16, ffn_dim=64, vocab_size=300,
                context_window=512)


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import paper_2512_23049_b200 as P
    from paper_2512_23049_b200.parallel import TPLayout, shard_weights

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = P.ModelConfig(**{k: getattr(SHAPE, k) for k in SHAPE.__dataclass_fields__})
        lay = TPLayout(rank, world, cfg)
        shard = shard_weights(P.init_weights(cfg).rounded("f32"), lay)
        eng = P.Engine(P.DeviceWeights.from_host(shard, dtype=torch.float32), tp=lay,
                       tp_group=dist.group.WORLD, record_logits=True)
        a = eng.prefill(P.PrefillCall("shared system prompt for the agents"))
        b = eng.prefill(P.PrefillCall("a question", parents=[a]))
        ids = eng.decode_parallel([
            P.DecodeCall("A1:", parents=[a, b], sampling=P.SamplingParams(max_tokens=6)),
            P.DecodeCall("A2:", parents=[b, a], offsets=[37, 0], new_offset=90,
                         sampling=P.SamplingParams(max_tokens=6))])
        q.put((rank, {m: np.stack(eng.last_stats.logits[m]) for m in ids},
               {m: eng.generated_token_ids(m) for m in ids}))
    except Exception as exc:  # surface worker failures instead of a queue timeout
        q.put((rank, repr(exc), None))
    finally:
        dist.destroy_process_group()


def test_tensor_parallel_engine_matches_oracle():
    world, port = 2, _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = O.Oracle(O.round_weights(O.init_weights(SHAPE), "f32"), SHAPE, record_logits=True)
    a = ref.prefill({"message": "shared system prompt for the agents"})
    b = ref.prefill({"message": "a question", "parents": [a]})
    ids = ref.decode_batch([
        {"header": "A1:", "parents": [a, b], "sampling": O.Sampling(max_tokens=6)},
        {"header": "A2:", "parents": [b, a], "offsets": [37, 0], "new_offset": 90,
         "sampling": O.Sampling(max_tokens=6)}])
    for rank, logits, gen in res:
        assert gen is not None, logits
        for m in ids:
            assert gen[m] == ref.generated(m)
            want = np.stack(ref.stats[-1].logits[m])
            assert float(np.abs(logits[m] - want).max()) <= 1e-4, rank


SHAPE_BF16 = O.Shape(n_layers=2, n_heads=8, n_kv_heads=4, head_dim=64, ffn_dim=256,
                     vocab_size=300, context_window=1024, rope_base=500000.0)


def _calls(P):
    return [P.DecodeCall("A1:", parents=[0, 1], sampling=P.SamplingParams(max_tokens=8)),
            P.DecodeCall("A2:", parents=[1, 0], offsets=[110, 0], new_offset=200,
                         sampling=P.SamplingParams(max_tokens=8))]


def _worker_bf16(rank, world, port, q, forced):
    import paper_2512_23049_b200 as P
    from paper_2512_23049_b200.parallel import TPLayout, shard_weights

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = P.ModelConfig(**{k: getattr(SHAPE_BF16, k) for k in SHAPE_BF16.__dataclass_fields__})
        lay = TPLayout(rank, world, cfg)
        shard = shard_weights(P.init_weights(cfg).rounded("bf16"), lay)
        eng = P.Engine(P.DeviceWeights.from_host(shard, dtype=torch.bfloat16), tp=lay,
                       tp_group=dist.group.WORLD, record_logits=True)
        eng.prefill(P.PrefillCall("shared system prompt for the agents " * 3))
        eng.prefill(P.PrefillCall("a question", parents=[0]))
        ids = eng.decode_parallel(_calls(P), force_tokens=forced)
        q.put((rank, {m: np.stack(eng.last_stats.logits[m]) for m in ids}, None))
    except Exception as exc:
        q.put((rank, repr(exc), "error"))
    finally:
        dist.destroy_process_group()


def test_tensor_parallel_native_bf16_matches_unsharded():
    """bf16, head_dim 64: decode steps take the native executor in halves (attention half,
    all-reduce, MLP half, all-reduce) with K7 / K5 v2; logits within 2e-2 of the unsharded
    bf16 engine on the same weights, teacher-forced on its tokens."""
    import paper_2512_23049_b200 as P

    cfg = P.ModelConfig(**{k: getattr(SHAPE_BF16, k) for k in SHAPE_BF16.__dataclass_fields__})
    ref = P.Engine(P.DeviceWeights.from_host(P.init_weights(cfg).rounded("bf16"),
                                             dtype=torch.bfloat16), record_logits=True)
    ref.prefill(P.PrefillCall("shared system prompt for the agents " * 3))
    ref.prefill(P.PrefillCall("a question", parents=[0]))
    rids = ref.decode_parallel(_calls(P))
    forced = [ref.generated_token_ids(m) for m in rids]
    want = {m: np.stack(ref.last_stats.logits[m]) for m in rids}
    world, port = 2, _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_bf16, args=(r, world, port, q, forced)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, logits, err in res:
        assert err is None, logits
        for m in rids:
            assert logits[m].shape == want[m].shape
            assert float(np.abs(logits[m] - want[m]).max()) <= 2e-2, rank
