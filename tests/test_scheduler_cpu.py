"""Host logic of the cross-workflow batching scheduler (no GPU): requests of all live
workflows are merged into one engine call per kind per tick, ids are routed back by
position, finished workflows drop out, and an offset conflict between workflows falls
back to one call per workflow (the engine validates before any mutation)."""

import pytest

from paper_2512_23049_b200.errors import OffsetConflictError
from paper_2512_23049_b200.scheduler import BatchScheduler, Decode, Prefill


class FakeEngine:
    """Allocates dense ids in call order; rejects a batch in which one parent is given two
    offsets, like Engine._resolve_calls (reference engine.py:233-235)."""

    def __init__(self):
        self.next_id = 0
        self.log = []
        self.last_stats = type("S", (), {"ttft": {}})()

    def _alloc(self, calls):
        agreed = {}
        for c in calls:
            for p, o in zip(c.get("parents", ()), c.get("offsets", ())):
                if agreed.setdefault(p, o) != o:
                    raise OffsetConflictError(f"parent {p}")
        ids = list(range(self.next_id, self.next_id + len(calls)))
        self.next_id += len(calls)
        self.last_stats = type("S", (), {"ttft": {i: 0.0 for i in ids}})()
        return ids

    def prefill_parallel(self, calls):
        ids = self._alloc(calls)
        self.log.append(("prefill", [c["tag"] for c in calls], ids))
        return ids

    def decode_parallel(self, calls, force_tokens=None):
        ids = self._alloc(calls)
        self.log.append(("decode", [c["tag"] for c in calls], ids, list(force_tokens)))
        return ids


def wf(tag, n_rounds, shared=None, offset=0):
    a, b = yield Prefill([{"tag": f"{tag}p0"}, {"tag": f"{tag}p1"}])
    got = [a, b]
    for r in range(n_rounds):
        parents = [a, b] + ([shared] if shared is not None else [])
        offs = [0, 10] + ([offset] if shared is not None else [])
        (m,) = yield Decode([{"tag": f"{tag}d{r}", "parents": parents, "offsets": offs}],
                            force_tokens=[[r]])
        got.append(m)
    return got


def test_merges_one_call_per_kind_per_tick_and_routes_ids():
    eng = FakeEngine()
    sch = BatchScheduler(eng)
    res = sch.run([wf("A", 2), wf("B", 3), wf("C", 1)])
    kinds = [e[0] for e in eng.log]
    assert kinds == ["prefill", "decode", "decode", "decode"]
    assert eng.log[0][1] == ["Ap0", "Ap1", "Bp0", "Bp1", "Cp0", "Cp1"]
    assert eng.log[1][1] == ["Ad0", "Bd0", "Cd0"]
    assert eng.log[2][1] == ["Ad1", "Bd1"]      # C finished after one round
    assert eng.log[3][1] == ["Bd2"]
    assert eng.log[1][3] == [[0], [0], [0]]       # forced tokens routed with their calls
    assert res[0] == [0, 1, 6, 9]
    assert res[1] == [2, 3, 7, 10, 11]
    assert res[2] == [4, 5, 8]
    assert all(t.merged for t in sch.ticks)


def test_offset_conflict_falls_back_to_one_call_per_workflow():
    eng = FakeEngine()
    # A also lists message 2 (B's first prefill) at offset 100; B places it at 0
    sch = BatchScheduler(eng)
    res = sch.run([wf("A", 1, shared=2, offset=100), wf("B", 1)])
    dec = [e for e in eng.log if e[0] == "decode"]
    assert [d[1] for d in dec] == [["Ad0"], ["Bd0"]]
    assert [t.merged for t in sch.ticks if t.kind == "decode"] == [False, False]
    assert res[0][-1] == 4 and res[1][-1] == 5    # no id burned by the rejected merge


def test_rejects_foreign_requests():
    def bad():
        yield "not a request"
    with pytest.raises(TypeError):
        BatchScheduler(FakeEngine()).run([bad()])
