"""Host logic of the re-encoding comparator: the exact-token prefix trie
(reference baseline.py:64-101, behaviours of its test_baseline.py trie tests)."""

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2512_23049_b200.baseline import PrefixTrie


def _kv(n, mark):
    base = np.arange(n, dtype=np.float64).reshape(1, n, 1, 1)
    k = np.concatenate([base, np.full((1, n, 1, 1), float(mark))], axis=3)
    return k, k + 0.5


def test_first_writer_keeps_each_node():
    trie = PrefixTrie()
    k1, v1 = _kv(2, 1)
    trie.insert([5, 6], k1, v1)
    k2, v2 = _kv(3, 2)
    trie.insert([5, 6, 7], k2, v2)
    assert trie.lookup([5, 6, 7, 8]) == 3
    gk, gv = trie.gather([5, 6, 7], 3)
    assert np.array_equal(gk[:, :2], k1) and np.array_equal(gk[:, 2:], k2[:, 2:])
    assert np.array_equal(gv[:, :2], v1)


def test_gather_empty_prefix():
    assert PrefixTrie().gather([1, 2], 0) == (None, None)


def test_device_sources_first_writer():
    trie = PrefixTrie()
    trie.insert_source([1, 2, 3], 0)
    trie.insert_source([1, 2, 4, 5], 1)
    assert trie.lookup([1, 2, 4, 5, 6]) == 4
    assert trie.sources([1, 2, 4, 5], 4) == [(0, 0), (0, 1), (1, 2), (1, 3)]
    assert trie.lookup([2]) == 0


@settings(max_examples=80, deadline=None)
@given(paths=st.lists(st.lists(st.integers(0, 3), min_size=1, max_size=6), max_size=8),
       probe=st.lists(st.integers(0, 3), max_size=8))
def test_lookup_matches_prefix_set(paths, probe):
    trie = PrefixTrie()
    stored = set()
    for i, path in enumerate(paths):
        trie.insert_source(path, i)
        stored.update(tuple(path[:j]) for j in range(1, len(path) + 1))
    want = 0
    for n in range(1, len(probe) + 1):
        if tuple(probe[:n]) not in stored:
            break
        want = n
    assert trie.lookup(probe) == want
