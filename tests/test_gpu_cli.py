"""`python -m paper_2512_23049_b200 run` on the B200 reproduces the reference's recorded
run of a fixture script (reference cli.py run/diff; trace equivalence ignores costs)."""

import os

import pytest

pytest.importorskip("torch")

from paper_2512_23049_b200.__main__ import main  # noqa: E402
from paper_2512_23049_b200.script import Trace, diff_traces  # noqa: E402

from .test_script_cpu import _trace  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("script", ["conversation", "branching", "madpar"])
def test_cli_run_trace_equals_reference_run(tmp_path, script):
    out = tmp_path / "t.jsonl"
    assert main(["run", os.path.join(GOLD, "scripts", f"{script}.json"), "--out", str(out),
                 "--dtype", "f32"]) == 0
    got = Trace.from_jsonl(out)
    assert diff_traces(_trace(script), got) == []


def test_cli_force_and_diff_against_a_reference_written_trace(tmp_path):
    """`run --force` reads a trace written by the reference itself, and `diff` compares our
    trace with it directly (logits too, within the f32 contract)."""
    ref = os.path.join(GOLD, "ref_trace_branching.jsonl")
    script = os.path.join(GOLD, "scripts", "branching.json")
    out = tmp_path / "forced.jsonl"
    assert main(["run", script, "--out", str(out), "--force", ref]) == 0  # bf16 engine
    assert main(["diff", ref, str(out)]) == 0
    out2 = tmp_path / "f32.jsonl"
    assert main(["run", script, "--out", str(out2), "--dtype", "f32", "--record-logits"]) == 0
    assert main(["diff", ref, str(out2), "--logits", "--atol", "1e-4"]) == 0
