"""The ``choreo`` shim: the reference's public modules mapped onto this build.

The staged reference suites (make_suite.py) import ``choreo.engine``, ``choreo.baseline``,
``choreo.script`` ... exactly as they do in the reference repo.  Here those names resolve
to paper_2512_23049_b200, with ``Engine`` / ``BaselineEngine`` building the f32 device
variant from the reference-layout host weights (the fp32 contract: 1e-4 against the
reference's f64).  Host-internal seams that this build replaces by device kernels
(GlobalKvCache's NumPy mutators, the masking / rotation helpers) and the cost-report
harness that SURVEY.md §2.1 puts out of scope are not shimmed: the tests that exercise
them directly are reported as skips with the reason in DEVIATIONS.

Every test collected here needs the B200 (marked ``gpu``).
"""

from __future__ import annotations

import json
import os
import sys
import types

import numpy as np
import pytest

import paper_2512_23049_b200 as P
from paper_2512_23049_b200 import baseline as _baseline
from paper_2512_23049_b200 import config as _config
from paper_2512_23049_b200 import errors as _errors
from paper_2512_23049_b200 import script as _script
from paper_2512_23049_b200 import tokenizer as _tokenizer

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SMALL_CONFIG = P.ModelConfig(n_layers=2, n_heads=2, head_dim=8, ffn_dim=64, vocab_size=512,
                             context_window=256, seed=0)

# test node name -> why it does not run against this build
DEVIATIONS = {
    "test_criterion_2_rope_repositioning":
        "exercises the reference's host RotationTable/rope_rotate helpers; the build re-rotates "
        "on the device (K2), pinned to the reference's rotation KATs in test_gpu_kernels.py",
    "test_criterion_3_mask_correctness":
        "drives the reference's host GlobalKvCache.append_tokens and masking helpers; the build "
        "assembles visibility on the device (K3), checked bit-exact against the oracle's "
        "visibility and the Fig. 2 panels in test_gpu_kernels.py / test_oracle_pins.py",
    "test_criterion_6_cost_trends":
        "runs the reference's cost-report harness (bench.run_suite / tot_voter_sweep over "
        "workflows.py), out of scope per SURVEY.md §2.1",
}

_DEV_W: dict = {}


def _device(weights, dtype=None):
    """Host WeightSet (reference layout) -> f32 DeviceWeights, cached per weight set."""
    import torch

    if isinstance(weights, P.DeviceWeights):
        return weights
    key = (id(weights), dtype)
    if key not in _DEV_W:
        _DEV_W[key] = (weights, P.DeviceWeights.from_host(weights, dtype=dtype or torch.float32))
    return _DEV_W[key][1]


class Engine(P.Engine):
    """``choreo.engine.Engine(weights, *, capacity, seed, record_logits)`` on the B200."""

    def __init__(self, weights, **kw) -> None:
        super().__init__(_device(weights), **kw)


class BaselineEngine(P.BaselineEngine):
    def __init__(self, weights, **kw) -> None:
        super().__init__(_device(weights), **kw)


def _unavailable(name: str, why: str):
    def f(*a, **k):
        pytest.skip(f"{name}: {why}")
    return f


def _module(name: str, **attrs) -> types.ModuleType:
    m = types.ModuleType(name)
    m.__dict__.update(attrs)
    sys.modules[name] = m
    return m


def _install() -> None:
    import bench as _bench  # the repo's bench.py: random_text is the reference's generator

    with open(os.path.join(ROOT, "tests", "golden", "ref_pins.json")) as fh:
        pins = json.load(fh)
    internal = "host-internal seam replaced by a device kernel in this build"
    pkg = _module("choreo")
    pkg.__path__ = []
    subs = {
        "config": dict(vars(_config)),
        "errors": dict(vars(_errors)),
        "tokenizer": dict(vars(_tokenizer)),
        "engine": dict(Engine=Engine, PrefillCall=P.PrefillCall, DecodeCall=P.DecodeCall,
                       SamplingParams=P.SamplingParams, CallStats=P.CallStats),
        "baseline": dict(BaselineEngine=BaselineEngine, PrefixTrie=_baseline.PrefixTrie),
        "model": dict(init_weights=P.init_weights, WeightSet=P.WeightSet,
                      LayerWeights=P.LayerWeights),
        "script": dict(vars(_script)),
        "bench": dict(random_text=_bench.random_text, SUITE_SHAPES={},
                      run_suite=_unavailable("run_suite", "out of scope"),
                      tot_voter_sweep=_unavailable("tot_voter_sweep", "out of scope")),
        "fixtures": dict(PREFILL_MASK=pins["mask_prefill_parallel"]["mask"],
                         DECODE_MASK=pins["mask_decode_parallel"]["mask"]),
        "cache": dict(GlobalKvCache=_unavailable("GlobalKvCache", internal)),
        "masking": {n: _unavailable(n, internal) for n in
                    ("VisibilitySpec", "build_dense_mask", "visible", "visible_cache_indices")},
        "tensor": {n: _unavailable(n, internal) for n in
                   ("RotationTable", "apply_rope_query", "rope_rotate")},
    }
    for sub, attrs in subs.items():
        setattr(pkg, sub, _module(f"choreo.{sub}", **attrs))


_install()


def pytest_collection_modifyitems(config, items):
    here = os.path.dirname(os.path.abspath(__file__))
    for it in items:
        if not str(it.fspath).startswith(here):
            continue
        it.add_marker(pytest.mark.gpu)
        why = DEVIATIONS.get(it.originalname if hasattr(it, "originalname") else it.name)
        if why:
            it.add_marker(pytest.mark.skip(reason=f"deviation: {why}"))


@pytest.fixture(scope="session")
def small_config():
    return SMALL_CONFIG


@pytest.fixture(scope="session")
def small_weights():
    return P.init_weights(SMALL_CONFIG)


@pytest.fixture(scope="session")
def default_weights():
    return P.init_weights(P.DEFAULT_CONFIG)


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)
