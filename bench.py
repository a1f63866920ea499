"""Benchmark: choreographed multi-agent debate at the Llama-3.1-8B shape (BASELINE.json C3).

One step = one complete debate workflow instance, laid out exactly as the
reference's run_madpar (workflows.py:294-327): prefill a system prompt (64
framed tokens) and a MATH-length question (160), then n_rounds rounds of
``decode_parallel`` with n_agents agents; each agent sees sys, q and the other
agents' previous-round replies, placed consecutively after q with explicit
offsets (so shared parents are repositioned once per round by K2) and its own
reply starts right after them.  Replies are teacher-forced to seeded lengths
U(256, 512) (bench.py run_pair protocol, src/bench.py:94-109) so every run does
identical work.  Weights: random-init Llama-3.1-8B shape, bf16, drawn on device.

Reported (rank 0, one JSON line):
  value    teacher-forced arm: decode tokens/s over the timed workflows, device-busy
           time (the sum of CUDA-event durations of every forward step).
  e2e      free-running arm: the same debates with greedy replies (K6 argmax on the
           device, each step's tokens read back to the host) through the public Engine
           API, tokens / CUDA-event time of the whole workflows; H2D of each step's
           metadata and D2H of its tokens inside the timed region (bytes declared).
  e2e_forced  the teacher-forced arm's end-to-end rate (no per-step readback).
  ttft_p50_ms  per-message TTFT (decode_parallel call start -> first token on the host),
           p50, free-running arm.
  roofline K7 (the step's dominant kernel) vs measured HBM bandwidth;
  attention_roofline  K5 v2 the same way.
  cpu_baseline  the reference's algorithm (CPU oracle, f64) on this host's cores, on a
           bounded sample (CpuC3Sample; `--impl reference` is the full reference arm).
  reencode_baseline  the same debate through the device BaselineEngine (the paper's
           re-encoding comparator) as the reference's pair ratios.
  kernel_rooflines  K2 / K4 / K5 / K7 microbenchmarks (tools/kernel_bench.py).
  c1_tiny  config C1 (the reference's tiny model) on the GPU, f32.
Multi-GPU (torchrun): each rank runs its own independent workflow instances
(seed = rank), no collectives on the data path; value = all ranks' tokens / max
rank time ("scaling": "weak").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import string
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "p50 per-message TTFT; choreographed decode tokens/s at Llama-3.1-8B shape"
WORKLOAD = "C3: Llama-3.1-8B shape, multi-agent debate (madpar layout), 8 agents x 3 rounds"


def random_text(rng, n_tokens: int) -> str:
    """ASCII text whose framed encoding is exactly n_tokens long (src/bench.py:155-163)."""
    n_bytes = max(1, n_tokens - 2)
    letters = string.ascii_lowercase
    chars: list = []
    while len(chars) < n_bytes:
        chars.extend(letters[i] for i in rng.integers(0, 26, size=8))
        chars.append(" ")
    return "".join(chars[:n_bytes]).strip().ljust(n_bytes, "x")


def workflow_inputs(seed: int, n_agents: int, n_rounds: int):
    rng = np.random.default_rng(seed)
    sys_text = random_text(rng, 64)
    question = random_text(rng, 160)
    forced = [[rng.integers(97, 123, size=int(rng.integers(256, 513))).tolist()
               for _ in range(n_agents)] for _ in range(n_rounds)]
    return sys_text, question, forced


def run_debate(engine, P, inputs, n_agents: int, n_rounds: int, free: bool = False) -> dict:
    """madpar layout (workflows.py:294-327) through the public Engine API.

    free=False: replies teacher-forced to their seeded lengths (run_pair protocol);
    free=True: replies decoded greedily (device argmax + token read back every step),
    max_tokens = the same seeded lengths."""
    sys_text, question, forced = inputs
    sys_id = engine.prefill(P.PrefillCall(sys_text))
    q_id = engine.prefill(P.PrefillCall(question))
    base = engine.message_token_count(sys_id) + engine.message_token_count(q_id)
    prev: list = []
    ttft, generated = [], 0
    for r in range(n_rounds):
        placed, cursor = {}, base
        for m in prev:
            placed[m] = cursor
            cursor += engine.message_token_count(m)
        calls = []
        for i in range(n_agents):
            others = [m for j, m in enumerate(prev) if j != i]
            calls.append(P.DecodeCall(
                f"Agent {i + 1}:", parents=[sys_id, q_id] + others,
                offsets=[0, engine.message_token_count(sys_id)] + [placed[m] for m in others],
                new_offset=cursor,
                sampling=P.SamplingParams(max_tokens=len(forced[r][i]) if free else 512)))
        prev = engine.decode_parallel(calls, force_tokens=None if free else forced[r])
        st = engine.last_stats
        ttft += [st.ttft[m] for m in prev]
        generated += sum(len(engine.generated_token_ids(m)) for m in prev)
    return {"ttft": ttft, "generated": generated}


def c4_workflow(engine, P, seed: int, n_prefill: int = 16, n_rounds: int = 4, n_dec: int = 4,
                pre_len=(64, 513), dec_len=(128, 257)):
    """BASELINE config C4, one workflow: n_prefill messages of U(64, 512)
    framed tokens, then n_rounds rounds of n_dec parallel decodes teacher-forced to
    U(128, 256) tokens.  Each round lays all prior messages out in a fresh random order
    with random gaps U{0..32}, 25 % of them reusing the previous parent's offset (an
    overlap); every call lists a random >= 50 % subset of them in its own random order at
    the round's agreed offsets (shared parents must agree within a batch, reference
    engine.py:233-235).  A generator for paper_2512_23049_b200.BatchScheduler."""
    rng = np.random.default_rng(seed)
    msgs = list((yield P.Prefill([P.PrefillCall(random_text(rng, int(rng.integers(*pre_len))))
                                  for _ in range(n_prefill)])))
    decoded = []
    for r in range(n_rounds):
        order = [msgs[i] for i in rng.permutation(len(msgs))]
        offs, cursor, prev = {}, 0, None
        for m in order:
            if prev is not None and rng.random() < 0.25:
                o = prev
            else:
                o = cursor + int(rng.integers(0, 33))
            offs[m] = o
            prev = o
            cursor = max(cursor, o + engine.message_token_count(m))
        new_off = cursor + int(rng.integers(0, 33))
        calls, forced = [], []
        for a in range(n_dec):
            k = int(rng.integers((len(order) + 1) // 2, len(order) + 1))
            parents = [order[i] for i in sorted(rng.permutation(len(order))[:k])]
            parents = [parents[i] for i in rng.permutation(len(parents))]
            calls.append(P.DecodeCall(f"W{seed}R{r}A{a}:", parents=parents,
                                      offsets=[offs[m] for m in parents], new_offset=new_off,
                                      sampling=P.SamplingParams(max_tokens=1024)))
            forced.append(rng.integers(97, 123, size=int(rng.integers(*dec_len))).tolist())
        ids = yield P.Decode(calls, force_tokens=forced)
        msgs += list(ids)
        decoded += list(ids)
    return decoded


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int) -> None:
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows if len(r) >= 7
                          for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def ncu_traffic() -> dict:
    """Per-launch DRAM traffic of K7 / K5 v2 from the committed ncu capture of the same
    decode step (profiles/r2_traffic.json, dram__bytes_read.sum + dram__bytes_write.sum)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh) | {"source": "measured"}
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


# ---------------------------------------------------------------------------- CPU side


C3_SHAPE = dict(n_heads=32, head_dim=128, ffn_dim=14336, vocab_size=128256,
                context_window=32768, rope_base=500000.0)


def _cpu_threads() -> int:
    cores = len(os.sched_getaffinity(0))
    try:  # torchrun exports OMP_NUM_THREADS=1 before numpy loads: lift it for the CPU arm
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=cores)
    except ImportError:
        pass
    return cores


class CpuC3Sample:
    """The reference's algorithm (the CPU oracle, a NumPy restatement of reference
    engine.py / model.py, f64 like the reference's default or f32) on a bounded sample of
    C3: the reference has no GQA, so heads are MHA-expanded (32 KV
    heads); full width and the full 128256-row head; one round-2 agent of the debate over
    a synthetic round-1 cache (sys 64 + q 160 + 8 replies of U(256,512)+10 tokens), its
    header encoded as one batch and then decode capped at the first token plus 8 steps.
    Full depth is infeasible on the host (an 8B MHA model in f64 is ~70 GB), so the same
    sample runs at 1 and 2 layers and t(L) = a + b L is extrapolated to L = 32
    (labelled "extrapolated")."""

    GEN = 9  # first token + 8 decode steps

    def __init__(self, dtype, seed: int = 0) -> None:
        from oracle import choreo_oracle as O

        self.O, self.dtype = O, np.dtype(dtype)
        rng = np.random.default_rng(seed)
        d, f, v = 4096, 14336, 128256

        block = (rng.random(1 << 24, dtype=np.float32) * 2 - 1).astype(self.dtype)

        def u(shp, fi, fo):
            # the scaled-uniform bounds of init_weights over a tiled random block: the values
            # do not change the timing, and drawing ~1G fresh values would take ~30 s
            return np.resize(block, shp) * np.sqrt(6.0 / (fi + fo))

        def layer():
            return {"attn_norm": np.ones(d, self.dtype), "wq": u((d, d), d, d),
                    "wk": u((d, d), d, d), "wv": u((d, d), d, d), "wo": u((d, d), d, d),
                    "ffn_norm": np.ones(d, self.dtype), "w_gate": u((d, f), d, f),
                    "w_up": u((d, f), d, f), "w_down": u((f, d), f, d)}

        self.w = {"embed": u((v, d), v, d), "out_head": u((d, v), d, v),
                  "out_norm": np.ones(d, self.dtype), "layers": [layer(), layer()]}
        self.lens = [64, 160] + [int(rng.integers(256, 513)) + 10 for _ in range(8)]
        self.kv = [rng.standard_normal((2, n, 32, 128), dtype=np.float32).astype(self.dtype)
                   for n in self.lens]

    def _engine(self, n_layers: int):
        O = self.O
        shape = O.Shape(n_layers=n_layers, **C3_SHAPE)  # n_kv_heads None: MHA, as the reference
        eng = O.Oracle(dict(self.w, layers=self.w["layers"][:n_layers]), shape, capacity=1 << 13)
        st, cursor = eng.store, 224
        for m, n in enumerate(self.lens):
            start = [0, 64][m] if m < 2 else cursor
            cursor += n if m >= 2 else 0
            st.msgs[m] = O.Msg("prefilled", start, "", None)
            kv = self.kv[m][:n_layers]
            st.append(m, [97] * n, np.arange(n) + start, kv, kv)
        eng.next_id = len(self.lens)
        call = {"header": "Agent 1:", "parents": list(range(len(self.lens) - 1)),
                "offsets": [st.msgs[m].offset for m in range(len(self.lens) - 1)],
                "new_offset": cursor, "sampling": O.Sampling(max_tokens=self.GEN)}
        return eng, call

    def run(self, n_layers: int) -> tuple:
        """(seconds, generated tokens, TTFT seconds) of the sample at n_layers."""
        eng, call = self._engine(n_layers)
        t0 = time.perf_counter()
        m = eng.decode(call, [97] * self.GEN)
        t = time.perf_counter() - t0
        return t, len(eng.generated(m)), eng.stats[-1].ttft[m]

    @staticmethod
    def extrapolate(t1: float, t2: float, L: int = 32) -> float:
        return t1 + (L - 1) * max(t2 - t1, 0.0)

    def describe(self, cores: int) -> str:
        return (f"oracle (the reference algorithm in NumPy {self.dtype.name}, {cores} host "
                f"threads), MHA-expanded 32 KV heads, 8B width, full 128256-row head: one "
                f"round-2 debate agent over a {sum(self.lens)}-token synthetic cache, header "
                f"as one batch then first token + 8 decode steps; timed at 1 and 2 layers and "
                f"extrapolated to 32")


def cpu_c1_full(dtype=np.float64) -> dict:
    """Config C1 (the reference's own tiny model) at full size, no extrapolation: three
    prefills, then the reordered / gapped / moved decode of 16 greedy tokens."""
    from oracle import choreo_oracle as O

    texts = ["System: answer the question using the notes.", "Note: the river is long.",
             "Question: which river is long?"]
    w = O.init_weights(O.TINY)
    if np.dtype(dtype) != np.float64:
        w = O.round_weights(w, "f32")
    ttft, tps = [], []
    for _ in range(5):
        eng = O.Oracle(w, O.TINY)
        for t in texts:
            eng.prefill({"message": t})
        t0 = time.perf_counter()
        m = eng.decode({"header": "Answer:", "parents": [2, 0], "offsets": [0, 37],
                        "sampling": O.Sampling(max_tokens=16)})
        wall = time.perf_counter() - t0
        ttft.append(eng.stats[-1].ttft[m])
        tps.append(len(eng.generated(m)) / wall)
    return {"ttft_p50_ms": round(1e3 * statistics.median(ttft), 3),
            "decode_tokens_per_s": round(statistics.median(tps), 1),
            "dtype": np.dtype(dtype).name, "extrapolated": False}


def c1_tiny(P) -> dict:
    """Config C1 on the GPU (f32 engine, the reference's tiny model): same protocol as
    cpu_c1_full, so the two lines compare directly."""
    import torch

    w = P.DeviceWeights.from_host(P.init_weights(P.DEFAULT_CONFIG), dtype=torch.float32)
    texts = ["System: answer the question using the notes.", "Note: the river is long.",
             "Question: which river is long?"]
    ttft, tps = [], []
    for _ in range(6):
        eng = P.Engine(w)
        for t in texts:
            eng.prefill(P.PrefillCall(t))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = eng.decode(P.DecodeCall("Answer:", parents=[2, 0], offsets=[0, 37],
                                    sampling=P.SamplingParams(max_tokens=16)))
        wall = time.perf_counter() - t0
        ttft.append(eng.last_stats.ttft[m])
        tps.append(len(eng.generated_token_ids(m)) / wall)
    return {"ttft_p50_ms": round(1e3 * statistics.median(ttft[1:]), 3),
            "decode_tokens_per_s": round(statistics.median(tps[1:]), 1), "dtype": "f32",
            "tokens": eng.generated_token_ids(m)}


def bench_config(args, world: int) -> dict:
    """The workload both arms report (the driver compares the arms' config)."""
    return {"workload": WORKLOAD, "model": args.model, "agents": args.agents,
            "rounds": args.rounds, "reply_tokens": "U(256,512)",
            "parallelism": f"replicas x{world} (independent workflows per GPU)"}


def reference_arm(args) -> None:
    """`--impl reference`: the reference's CPU algorithm (oracle port) on the host cores,
    same metric / unit / config as our arm; rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cores = _cpu_threads()
    f64 = CpuC3Sample(np.float64)
    rates, ttfts, t_steps = [], [], []
    t1s, t2s = [], []
    for i in range(args.warmup + args.steps):
        # a step is one bounded sample; depths alternate so each step stays ~5 s
        t0 = time.perf_counter()
        t, gen, ttft = f64.run(1 + i % 2)
        (t1s if i % 2 == 0 else t2s).append((t, gen, ttft))
        if i >= args.warmup:
            t_steps.append(time.perf_counter() - t0)
    t1 = statistics.median(x[0] for x in t1s)
    t2 = statistics.median(x[0] for x in t2s) if t2s else t1
    gen = t1s[0][1]
    value = gen / CpuC3Sample.extrapolate(t1, t2)
    ttft = CpuC3Sample.extrapolate(statistics.median(x[2] for x in t1s),
                                   statistics.median(x[2] for x in t2s) if t2s else 0.0)
    sample = f64.describe(cores)
    del f64
    f32 = CpuC3Sample(np.float32)
    r1, r2 = f32.run(1), f32.run(2)
    f32_value = r1[1] / CpuC3Sample.extrapolate(r1[0], r2[0])
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * statistics.mean(t_steps), 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "ttft_p50_ms": round(1e3 * ttft, 1),
            "config": bench_config(args, args.gpus),
            "extrapolated": True,
            "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", "cores": cores,
                             "kind": "port", "sample": sample},
            "f32": {"value": round(f32_value, 4), "unit": "tokens/s",
                    "ttft_p50_ms": round(1e3 * CpuC3Sample.extrapolate(r1[2], r2[2]), 1),
                    "sample": f32.describe(cores)},
            "c1_tiny_full": cpu_c1_full(),
            "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU side


def reencode_baseline(P, weights, inputs, args, choreo_eng) -> dict:
    """The paper's comparison on the same GPU and weights: one instance of the same
    debate through the re-encoding BaselineEngine (parents concatenated in list order
    and re-encoded per call behind an exact prefix trie, decode_parallel sequential,
    reference baseline.py) and through the choreography engine, reported as the
    reference's pair ratios (baseline over choreography: mean TTFT, FLOPs, wall;
    reference bench.py:138-149)."""
    import torch

    def one(eng):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = run_debate(eng, P, inputs, args.agents, args.rounds)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        flops = {k: sum(getattr(s_, k) for s_ in eng.stats)
                 for k in ("prefill_flops", "decode_flops")}
        return res, wall, flops

    choreo_eng.reset()
    rc, wall_c, fc = one(choreo_eng)
    eng = P.BaselineEngine(weights)
    rb, wall_b, fb = one(eng)
    hits = sum(s.cache_hit_tokens for s in eng.stats)
    enc = sum(s.tokens_encoded for s in eng.stats)
    out = {"engine": "BaselineEngine (device, re-encoding + prefix trie)", "workflows": 1,
           "ttft_p50_ms": round(1e3 * statistics.median(rb["ttft"]), 3),
           "ttft_mean_ms": round(1e3 * statistics.mean(rb["ttft"]), 3),
           "decode_tokens_per_s": round(rb["generated"] / wall_b, 2),
           "tokens_encoded": enc, "trie_hit_tokens": hits,
           "pair_ratios": {
               "ttft": round(statistics.mean(rb["ttft"]) / statistics.mean(rc["ttft"]), 2),
               "prefill_flops": round(fb["prefill_flops"] / max(fc["prefill_flops"], 1), 2),
               "decode_flops": round(fb["decode_flops"] / max(fc["decode_flops"], 1), 2),
               "total_flops": round(sum(fb.values()) / max(sum(fc.values()), 1), 2),
               "wall": round(wall_b / wall_c, 2),
               "definition": "baseline / choreography on the same teacher-forced debate, "
                             "mean TTFT as the reference's pair_ratios"}}
    del eng
    torch.cuda.empty_cache()
    return out


def c4_batched(P, weights, rank: int, n_wf: int) -> dict:
    """Config C4 on this GPU: n_wf C4 workflows batched per step by BatchScheduler (one
    forward per step for all their agents) on one engine; one warm-up pass, then one timed
    pass (CUDA events), decode tokens / time and per-message TTFT."""
    import torch

    eng = P.Engine(weights, capacity=1 << 17, seed=rank)
    for rep in range(2):
        eng.reset()
        wfs = [c4_workflow(eng, P, 10_000 * rep + 100 * rank + k) for k in range(n_wf)]
        sch = P.BatchScheduler(eng)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        res = sch.run(wfs)
        b.record()
        torch.cuda.synchronize()
    secs = a.elapsed_time(b) / 1e3
    gen = sum(len(eng.generated_token_ids(m)) for ids in res for m in ids)
    ttft = [v for t in sch.ticks for v in t.ttft.values()]
    out = {"workflows": n_wf, "generated_tokens": gen, "seconds": round(secs, 3),
           "decode_tokens_per_s": round(gen / secs, 1),
           "ttft_p50_ms": round(1e3 * statistics.median(ttft), 3),
           "merged_ticks": sum(t.merged for t in sch.ticks), "ticks": len(sch.ticks)}
    del eng
    torch.cuda.empty_cache()
    return out


def c2_agents(P, rank: int) -> dict:
    """Config C2: Llama-3.2-1B shape, random-init bf16; a global cache of
    32 messages x 256 tokens (4 prefill_parallel batches of 8), then ONE decode_parallel of
    4 agents, each over 12 of the 32 messages (a random subset in random order) laid out
    with gaps U{0..32} and 25 % overlaps at offsets shared by the batch; greedy, 256
    tokens.  Timed with CUDA events around the decode call (one warm-up instance first)."""
    import torch

    cfg = P.PRESETS["llama-3.2-1b"]
    w = P.DeviceWeights.random(cfg, dtype=torch.bfloat16, seed=cfg.seed + rank)
    eng = P.Engine(w, capacity=16384, seed=rank)
    for rep in range(2):
        eng.reset()
        rng = np.random.default_rng(1000 * rep + rank)
        ids = []
        for _ in range(4):
            ids += eng.prefill_parallel([P.PrefillCall(random_text(rng, 256)) for _ in range(8)])
        offs, cursor, prev = {}, 0, None
        for i in rng.permutation(32):
            o = prev if prev is not None and rng.random() < 0.25 else cursor + int(rng.integers(0, 33))
            offs[ids[i]] = o
            prev, cursor = o, max(cursor, o + 256)
        calls = []
        for a in range(4):
            parents = [ids[j] for j in rng.permutation(32)[:12]]
            calls.append(P.DecodeCall(f"Agent {a}:", parents=parents,
                                      offsets=[offs[m] for m in parents],
                                      new_offset=cursor + int(rng.integers(0, 33)),
                                      sampling=P.SamplingParams(max_tokens=256)))
        torch.cuda.synchronize()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        ms = eng.decode_parallel(calls)
        b_.record()
        torch.cuda.synchronize()
    secs = a_.elapsed_time(b_) / 1e3
    gen = sum(len(eng.generated_token_ids(m)) for m in ms)
    st = eng.last_stats
    out = {"workload": "C2: Llama-3.2-1B shape, 4 parallel agents (greedy, 256 tokens) over "
                       "12-message reordered subsets of a shared 8K-token global cache",
           "generated_tokens": gen, "seconds": round(secs, 4),
           "decode_tokens_per_s": round(gen / secs, 1),
           "ttft_p50_ms": round(1e3 * statistics.median(st.ttft.values()), 3),
           "repositioned_tokens": st.repositioned_tokens, "cache_hit_tokens": st.cache_hit_tokens}
    del eng, w
    torch.cuda.empty_cache()
    return out


def c5_tensor_parallel(P, rank: int, world: int) -> dict:
    """Config C5 across the job's GPUs: Llama-3.1-70B shape, random-init bf16, KV heads (and
    the MLP) sharded world-ways (parallel.TPLayout); every layer all-reduces the o_proj and
    down_proj partial outputs over NCCL.  A 64 x 512-token global cache, then 8 agents
    decoding 64 teacher-forced tokens over reordered 32-message subsets (~16K visible).
    Decode time is CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2512_23049_b200.parallel import TPLayout

    cfg = P.PRESETS["llama-3.1-70b"]
    lay = TPLayout(rank, world, cfg)
    w = P.DeviceWeights.random(cfg, dtype=torch.bfloat16, tp=lay)
    eng = P.Engine(w, capacity=36 * 1024, tp=lay, tp_group=dist.group.WORLD)
    rng = np.random.default_rng(0)  # same layout on every rank
    ids = []
    for _ in range(8):
        ids += eng.prefill_parallel([P.PrefillCall(random_text(rng, 512)) for _ in range(8)])
    sel = [ids[i] for i in rng.permutation(64)[:32]]
    offs, cursor, prev = {}, 0, None
    for m in sel:
        o = prev if prev is not None and rng.random() < 0.25 else cursor + int(rng.integers(0, 33))
        offs[m] = o
        prev, cursor = o, max(cursor, o + 512)
    calls, forced = [], []
    for a in range(8):
        parents = [sel[j] for j in rng.permutation(32)]
        calls.append(P.DecodeCall(f"Agent {a}:", parents=parents, offsets=[offs[m] for m in parents],
                                  new_offset=cursor + 8, sampling=P.SamplingParams(max_tokens=512)))
        forced.append(rng.integers(97, 123, size=64).tolist())
    torch.cuda.synchronize()
    dist.barrier()
    a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a_.record()
    ms = eng.decode_parallel(calls, force_tokens=forced)
    b_.record()
    torch.cuda.synchronize()
    t = torch.tensor([a_.elapsed_time(b_) / 1e3], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gen = sum(len(eng.generated_token_ids(m)) for m in ms)
    out = {"workload": f"C5: Llama-3.1-70B shape, KV heads sharded {world}-way (TP, NCCL "
                       "all-reduce after o_proj and down_proj), 8 agents x 64 forced tokens over "
                       "~16K visible tokens of a 32K global cache",
           "tp": world, "decode_tokens_per_s": round(gen / float(t[0]), 1),
           "ms_per_step": round(1e3 * float(t[0]) / 64, 2),
           "ttft_p50_ms": round(1e3 * statistics.median(eng.last_stats.ttft.values()), 2)}
    del eng, w
    torch.cuda.empty_cache()
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--agents", type=int, default=8)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernels", action="store_true",
                    help="skip the K2/K4/K5 kernel microbenchmarks (tools/kernel_bench.py)")
    ap.add_argument("--no-reencode", action="store_true",
                    help="skip the re-encoding comparator (BaselineEngine) workflow")
    ap.add_argument("--model", default="llama-3.1-8b")
    ap.add_argument("--no-c2", action="store_true",
                    help="skip the config-C2 measurement (1B shape, 4 agents, 8K cache)")
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the config-C5 tensor-parallel 70B measurement (N > 1 only)")
    ap.add_argument("--no-c4", action="store_true",
                    help="skip the config-C4 batched-workflows measurement (BatchScheduler)")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2512_23049_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_dev = torch.cuda.device_count()
    local = local % n_dev  # > 1 rank per GPU only when testing the multi-rank path on one GPU
    torch.cuda.set_device(local)
    if world > 1:
        if n_dev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # ranks sharing a GPU: NCCL refuses duplicate devices, gloo reduces CUDA tensors
            dist.init_process_group("gloo")
    cfg = P.PRESETS[args.model]
    weights = P.DeviceWeights.random(cfg, dtype=torch.bfloat16, device="cuda", seed=cfg.seed + rank)
    eng = P.Engine(weights, capacity=65536, seed=rank)
    runner = eng._runner

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for i in range(args.warmup):
        eng.reset()
        run_debate(eng, P, workflow_inputs(1000 * rank + i, args.agents, args.rounds),
                   args.agents, args.rounds)
    inputs = [workflow_inputs(1000 * rank + 100 + i, args.agents, args.rounds)
              for i in range(args.steps)]

    step_events, attn_events = [], []
    runner.step_events = step_events
    launches0, h2d0, d2h0 = runner.launches, runner.h2d_bytes, eng.d2h_bytes
    ttft_forced, generated = [], 0
    sync_all()
    with ClockSampler(local) as clocks:
        # arm 1, teacher-forced replies: `value` (device-busy rate) and e2e_forced
        ev_start = torch.cuda.Event(enable_timing=True)
        ev_end = torch.cuda.Event(enable_timing=True)
        ev_start.record()
        for i in range(args.steps):
            eng.reset()
            res = run_debate(eng, P, inputs[i], args.agents, args.rounds)
            ttft_forced += res["ttft"]
            generated += res["generated"]
        ev_end.record()
        sync_all()
        runner.step_events = None
        elapsed = ev_start.elapsed_time(ev_end) / 1e3
        busy = sum(a.elapsed_time(b) for a, b in step_events) / 1e3
        launches = runner.launches - launches0
        h2d_forced = (runner.h2d_bytes - h2d0) / args.steps
        d2h_forced = (eng.d2h_bytes - d2h0) / args.steps
        # arm 2, free-running greedy replies (K6 argmax + the tokens read back to the host
        # every step): the headline e2e and TTFT
        eng.reset()
        run_debate(eng, P, inputs[0], args.agents, args.rounds, free=True)  # warm-up
        sync_all()
        l1, h1, d1 = runner.launches, runner.h2d_bytes, eng.d2h_bytes
        ttft, gen_free = [], 0
        ev_fs = torch.cuda.Event(enable_timing=True)
        ev_fe = torch.cuda.Event(enable_timing=True)
        ev_fs.record()
        for i in range(args.steps):
            eng.reset()
            res = run_debate(eng, P, inputs[i], args.agents, args.rounds, free=True)
            ttft += res["ttft"]
            gen_free += res["generated"]
        ev_fe.record()
        sync_all()
    elapsed_free = ev_fs.elapsed_time(ev_fe) / 1e3
    launches += runner.launches - l1
    h2d = (runner.h2d_bytes - h1) / args.steps
    d2h = (eng.d2h_bytes - d1) / args.steps
    # per-kernel rooflines: one more instance of the same workflow right after the timed
    # region with CUDA events around every K5 and K7 launch (kept out of the timed region:
    # an event between two launches costs the second its programmatic-launch overlap)
    eng.reset()
    runner.attn_events, runner.time_linear = attn_events, True
    run_debate(eng, P, inputs[0], args.agents, args.rounds)
    runner.attn_events, runner.time_linear = None, False
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([elapsed, busy, elapsed_free], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, busy, elapsed_free = t.tolist()
        g = torch.tensor([generated, gen_free], device="cuda", dtype=torch.float64)
        dist.all_reduce(g)
        generated_all, gen_free_all = g.tolist()
    else:
        generated_all, gen_free_all = generated, gen_free

    # decode attention (K5) roofline, from the events of the last timed workflow
    peaks = measured_peaks()
    timed = runner.collect_attn_times()
    a_ms = [m for m, _ in timed]
    a_bytes = [nb for _, nb in timed]
    attn_roofline = None
    if a_ms:
        achieved = (sum(a_bytes) / len(a_bytes)) / (sum(a_ms) / len(a_ms) / 1e3) / 1e9
        attn_roofline = {"kernel": "choreo_decode_attn_v2 (K5: page-centric split-KV decode attention, TMA page ring)",
                    "bound": "hbm",
                    "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": round(achieved / peaks["hbm_gbs"], 4),
                    "traffic": ncu_traffic().get("k5v2_dram_bytes_per_launch"),
                    "peak_source": peaks["source"],
                    "avg_launch_us": round(1e3 * sum(a_ms) / len(a_ms), 2),
                    "algorithmic_bytes_per_launch": int(sum(a_bytes) / len(a_bytes)),
                    "launches_timed": len(a_ms)}
    # the decode step's dominant kernel: K7 weight streaming (4 launches per layer)
    roofline = None
    lin = runner.linear_times
    if lin:
        l_ms = sum(m for m, _ in lin) / len(lin)
        l_b = sum(b for _, b in lin) / len(lin)
        ach = l_b / (l_ms / 1e3) / 1e9
        roofline = {"kernel": "choreo_linear_skinny (K7: tcgen05 stream-K weight-streaming "
                              "linear, qkv / o_proj / gate|up / down of every decode layer)",
                    "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"],
                    "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4),
                    "traffic": ncu_traffic().get("k7_layer_gemm_dram_bytes_per_launch"),
                    "traffic_source": ncu_traffic().get("source"),
                    "peak_source": peaks["source"], "avg_launch_us": round(1e3 * l_ms, 2),
                    "algorithmic_bytes_per_launch": int(l_b), "launches_timed": len(lin),
                    "note": "CUDA events on the launching stream around each launch of one extra "
                            "instance of the timed workflow run right after the timed region; "
                            "the brackets remove the launch's programmatic-dependent-launch "
                            "overlap, so this is conservative"}

    c4 = None
    if not args.no_c4:  # every rank runs its own 8 workflows (C4: 64 over 8 GPUs)
        c4_one = c4_batched(P, weights, rank, 1)
        c4 = c4_batched(P, weights, rank, 8)
        if world > 1:
            t = torch.tensor([c4["seconds"], c4["generated_tokens"]], device="cuda",
                             dtype=torch.float64)
            mx = t.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(t)
            c4["all_ranks_tokens_per_s"] = round(float(t[1] / mx[0]), 1)
        c4 = {"workload": "C4: Llama-3.1-8B shape, 8 choreographed workflows per GPU batched per "
                          "step (16 prefilled U(64,512) + 4 rounds x 4 decodes U(128,256), "
                          "reordered parent subsets, gaps, 25% overlaps)",
              "batched_8": c4, "single_workflow": c4_one,
              "batching_speedup": round(c4["decode_tokens_per_s"] / c4_one["decode_tokens_per_s"], 2)}

    c5 = None
    if world > 1 and 8 % world == 0 and not args.no_c5:
        del eng, runner, weights  # the 70B shards need the room
        torch.cuda.empty_cache()
        try:
            c5 = c5_tensor_parallel(P, rank, world)
        except Exception as exc:  # report, never lose the main line
            c5 = {"error": repr(exc)[:300]}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    reencode = None
    if world == 1 and not args.no_reencode:
        reencode = reencode_baseline(P, weights, inputs[0], args, eng)
    kernels = None
    if world == 1 and not args.no_kernels:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import kernel_bench as kb

        del eng, weights
        torch.cuda.empty_cache()
        kernels = ([kb.k2_rerotate(), kb.k4_prefill(), kb.k5_decode(1, v2=True),
                    kb.k5_decode(8, v2=True)] + kb.k7_linear() + [kb.k8_chain()])
    c2 = None
    if world == 1 and not args.no_c2:
        c2 = c2_agents(P, rank)
    c1 = c1_tiny(P) if world == 1 else None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = _cpu_threads()
        smp = CpuC3Sample(np.float64)
        r1, r2 = smp.run(1), smp.run(2)
        cpu = {"value": round(r1[1] / CpuC3Sample.extrapolate(r1[0], r2[0]), 4),
               "unit": "tokens/s", "cores": cores, "kind": "port", "extrapolated": True,
               "ttft_p50_ms": round(1e3 * CpuC3Sample.extrapolate(r1[2], r2[2]), 1),
               "sample": smp.describe(cores)}
        del smp
    line = {
        "metric": METRIC, "value": round(generated_all / busy, 2), "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * elapsed / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "ttft_p50_ms": round(1e3 * statistics.median(ttft), 3),
        "ttft_p90_ms": round(1e3 * sorted(ttft)[int(0.9 * (len(ttft) - 1))], 3),
        "config": bench_config(args, world),
        "setup": {"weights": "random-init bf16 (device draw)", "kv_cache": "paged bf16, P=64",
                  "activations": "split hi/lo bf16 GEMM inputs, f32 residual",
                  "value_definition": "teacher-forced replies (U(256,512)): generated tokens / "
                                      "sum of per-step device time",
                  "e2e_definition": "free-running greedy replies (max_tokens = the same seeded "
                                    "lengths): generated tokens / CUDA-event time of the whole "
                                    "workflows through the public Engine API; every step "
                                    "uploads its metadata (H2D) and reads its tokens back (D2H)",
                  "l2": "inputs larger than L2 (16 GB of weights streamed per step)"},
        "e2e": {"value": round(gen_free_all / elapsed_free, 2), "unit": "tokens/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "generated_tokens": int(gen_free_all)},
        "e2e_forced": {"value": round(generated_all / elapsed, 2), "unit": "tokens/s",
                       "h2d_bytes_per_step": int(h2d_forced),
                       "d2h_bytes_per_step": int(d2h_forced),
                       "ttft_p50_ms": round(1e3 * statistics.median(ttft_forced), 3)},
        "gpu_launches": int(launches),
        "generated_tokens": int(generated_all),
        "roofline": roofline,
        "attention_roofline": attn_roofline,
        "kernel_rooflines": kernels,
        "reencode_baseline": reencode,
        "c4_batched_workflows": c4,
        "c2_agents_1b": c2,
        "c1_tiny": c1,
        "c5_tensor_parallel_70b": c5,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
