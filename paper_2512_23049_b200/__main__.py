"""Command line (reference cli.py:140-237, the run / diff subset):

  python -m paper_2512_23049_b200 run SCRIPT.json [--out TRACE.jsonl] [--weights W.npz]
         [--dtype bf16|f32] [--seed N] [--force TRACE.jsonl] [--record-logits]
  python -m paper_2512_23049_b200 diff A.jsonl B.jsonl [--logits] [--atol X]

`run` replays a workflow script through the B200 engine (default config, seed-0 weights
unless --weights) and writes the trace; `diff` compares two traces of one script,
ignoring engine kind and cost counters (exit 1 when they differ).
"""

from __future__ import annotations

import argparse
import sys

from .script import Trace, diff_traces, load_script, run_script


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2512_23049_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("script")
    r.add_argument("--out")
    r.add_argument("--weights")
    r.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--force")
    r.add_argument("--record-logits", action="store_true")
    d = sub.add_parser("diff")
    d.add_argument("a")
    d.add_argument("b")
    d.add_argument("--logits", action="store_true")
    d.add_argument("--atol", type=float, default=1e-9)
    args = ap.parse_args(argv)
    if args.cmd == "diff":
        diffs = diff_traces(Trace.from_jsonl(args.a), Trace.from_jsonl(args.b),
                            compare_logits=args.logits, atol=args.atol)
        for line in diffs:
            print(line)
        print("equivalent" if not diffs else f"{len(diffs)} difference(s)")
        return 1 if diffs else 0
    import torch

    from . import DEFAULT_CONFIG, DeviceWeights, Engine, init_weights, load_weights

    ws = load_weights(args.weights) if args.weights else init_weights(DEFAULT_CONFIG)
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    if args.dtype == "bf16":
        ws = ws.rounded("bf16")
    eng = Engine(DeviceWeights.from_host(ws, dtype=dt), seed=args.seed,
                 record_logits=args.record_logits)
    force = Trace.from_jsonl(args.force).forcing() if args.force else None
    trace = run_script(eng, load_script(args.script), force=force)
    if args.out:
        trace.to_jsonl(args.out)
    for m in trace.messages():
        if m.generated is not None:
            print(f"{m.name}: {m.text!r}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
