"""Weights: the reference's host WeightSet (init / save / load) and its device form.

Host side is drop-in with the reference (model.py:31-97, 243-286): the same
PCG64 draw order and scaled-uniform bounds (so the golden weights sha256 holds),
the same file format.  GQA extends wk/wv to (d, n_kv_heads*hd) with the same
formula.  ``DeviceWeights`` is what the engine runs on: bf16 (or f32 for the
parity variant) tensors in HBM with the GEMM operands fused and laid out
(out_features, in_features):
    w_qkv  [(H + 2 Hkv) hd, d]   = concat(wq, wk, wv)^T
    w_gu   [2 F, d]              = concat(w_gate, w_up)^T
    wo     [d, d], w_down [d, F], out_head [V, d]
Llama-scale random weights are drawn on the device (``DeviceWeights.random``):
same bounds and tensor order, torch's Philox stream instead of PCG64.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .config import ModelConfig

LAYER_NAMES = ("attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")
WEIGHTS_MAGIC = "choreo-weights"


@dataclass
class LayerWeights:
    attn_norm: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    ffn_norm: np.ndarray
    w_gate: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray


@dataclass
class WeightSet:
    config: ModelConfig
    embed: np.ndarray
    layers: list
    out_norm: np.ndarray
    out_head: np.ndarray

    @property
    def dtype(self) -> np.dtype:
        return self.embed.dtype

    def named_tensors(self) -> list:
        out = [("embed", self.embed)]
        for i, lw in enumerate(self.layers):
            out += [(f"layers.{i}.{n}", getattr(lw, n)) for n in LAYER_NAMES]
        return out + [("out_norm", self.out_norm), ("out_head", self.out_head)]

    def rounded(self, kind: str) -> "WeightSet":
        """Same weights rounded to 'bf16' (RNE) or 'f32', returned as f64 host arrays."""
        def rnd(a):
            f = np.ascontiguousarray(a, dtype=np.float32)
            if kind == "f32":
                return f.astype(np.float64)
            u = f.view(np.uint32).astype(np.uint64)
            u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
            return u.astype(np.uint32).view(np.float32).astype(np.float64)
        return WeightSet(self.config, rnd(self.embed),
                         [LayerWeights(**{n: rnd(getattr(lw, n)) for n in LAYER_NAMES})
                          for lw in self.layers], rnd(self.out_norm), rnd(self.out_head))


def init_weights(config: ModelConfig, dtype=np.float64) -> WeightSet:
    """Seeded scaled-uniform init, bitwise the reference's (model.py:67-97)."""
    rng = np.random.Generator(np.random.PCG64(config.seed))
    dtype = np.dtype(dtype)
    d, dkv, f, v = config.model_dim, config.kv_dim, config.ffn_dim, config.vocab_size

    def draw(fan_in, fan_out, shape):
        bound = math.sqrt(6.0 / (fan_in + fan_out))
        return rng.uniform(-bound, bound, size=shape).astype(dtype)

    embed = draw(v, d, (v, d))
    layers = []
    for _ in range(config.n_layers):
        layers.append(LayerWeights(
            attn_norm=np.ones(d, dtype=dtype), wq=draw(d, d, (d, d)), wk=draw(d, dkv, (d, dkv)),
            wv=draw(d, dkv, (d, dkv)), wo=draw(d, d, (d, d)), ffn_norm=np.ones(d, dtype=dtype),
            w_gate=draw(d, f, (d, f)), w_up=draw(d, f, (d, f)), w_down=draw(f, d, (f, d))))
    out_head = draw(d, v, (d, v))
    return WeightSet(config, embed, layers, np.ones(d, dtype=dtype), out_head)


def save_weights(weights: WeightSet, path) -> None:
    """JSON header line + f32 LE blobs (model.py:243-262)."""
    tensors = weights.named_tensors()
    header = {"format": WEIGHTS_MAGIC, "version": 1, "dtype": "float32",
              "config": weights.config.to_dict(),
              "tensors": [{"name": n, "shape": list(a.shape)} for n, a in tensors]}
    with open(path, "wb") as fh:
        fh.write((json.dumps(header, sort_keys=True) + "\n").encode("utf-8"))
        for _, a in tensors:
            fh.write(np.ascontiguousarray(a, dtype="<f4").tobytes())


def load_weights(path, dtype=np.float64) -> WeightSet:
    with open(path, "rb") as fh:
        header = json.loads(fh.readline().decode("utf-8"))
        if header.get("format") != WEIGHTS_MAGIC:
            raise ValueError(f"{path} is not a weight file")
        blob = fh.read()
    config = ModelConfig.from_dict(header["config"])
    arrays, off = {}, 0
    for spec in header["tensors"]:
        n = int(np.prod(spec["shape"]))
        arrays[spec["name"]] = np.frombuffer(blob, "<f4", n, off).reshape(spec["shape"]).astype(dtype)
        off += 4 * n
    if off != len(blob):
        raise ValueError(f"{path}: {len(blob) - off} trailing bytes")
    layers = [LayerWeights(**{n: arrays[f"layers.{i}.{n}"] for n in LAYER_NAMES})
              for i in range(config.n_layers)]
    return WeightSet(config, arrays["embed"], layers, arrays["out_norm"], arrays["out_head"])


class DeviceWeights:
    """Weights resident in HBM in the engine's compute dtype."""

    def __init__(self, config: ModelConfig, dtype, device, tensors: dict) -> None:
        self.config = config
        self.torch_dtype = dtype
        self.device = device
        self.embed = tensors["embed"]
        self.out_norm = tensors["out_norm"]
        self.out_head = tensors["out_head"]
        self.layers = tensors["layers"]

    @property
    def nbytes(self) -> int:
        n = self.embed.nbytes + self.out_norm.nbytes + self.out_head.nbytes
        return n + sum(t.nbytes for lw in self.layers for t in lw.values())

    @classmethod
    def from_host(cls, ws: WeightSet, dtype=None, device=None) -> "DeviceWeights":
        import torch

        dtype = dtype or torch.bfloat16
        device = torch.device(device or "cuda")

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(
                device=device, dtype=dtype)

        layers = []
        for lw in ws.layers:
            layers.append({
                "attn_norm": up(lw.attn_norm),
                "w_qkv": up(np.concatenate([lw.wq, lw.wk, lw.wv], axis=1).T),
                "wo": up(lw.wo.T),
                "ffn_norm": up(lw.ffn_norm),
                "w_gu": up(np.concatenate([lw.w_gate, lw.w_up], axis=1).T),
                "w_down": up(lw.w_down.T),
            })
        return cls(ws.config, dtype, device, {"embed": up(ws.embed), "out_norm": up(ws.out_norm),
                                             "out_head": up(ws.out_head.T), "layers": layers})

    @classmethod
    def random(cls, config: ModelConfig, dtype=None, device=None, seed: int | None = None,
               tp=None) -> "DeviceWeights":
        """Device-side scaled-uniform init (same bounds/order as init_weights, torch Philox).

        With tp (parallel.TPLayout) only this rank's slice is drawn (bounds use the full
        fan-in/fan-out; slices of different ranks come from different generator streams)."""
        import torch

        dtype = dtype or torch.bfloat16
        device = torch.device(device or "cuda")
        gen = torch.Generator(device=device)
        gen.manual_seed((config.seed if seed is None else seed) + (1000 * tp.rank if tp else 0))
        d, dkv, f, v, hd = (config.model_dim, config.kv_dim, config.ffn_dim, config.vocab_size,
                            config.head_dim)
        if tp is not None:
            return cls._random_tp(config, tp, dtype, device, gen)

        def draw(fan_in, fan_out, shape):
            b = math.sqrt(6.0 / (fan_in + fan_out))
            t = torch.empty(shape, device=device, dtype=torch.float32)
            t.uniform_(-b, b, generator=gen)
            return t.to(dtype)

        ones = torch.ones(d, device=device, dtype=dtype)
        embed = draw(v, d, (v, d))
        layers = []
        for _ in range(config.n_layers):
            wq, wk, wv = draw(d, d, (d, d)), draw(d, dkv, (dkv, d)), draw(d, dkv, (dkv, d))
            w_qkv = torch.cat([wq, wk, wv], dim=0)
            del wq, wk, wv
            wo = draw(d, d, (d, d))
            w_gu = torch.cat([draw(d, f, (f, d)), draw(d, f, (f, d))], dim=0)
            layers.append({"attn_norm": ones, "w_qkv": w_qkv, "wo": wo, "ffn_norm": ones,
                           "w_gu": w_gu, "w_down": draw(f, d, (d, f))})
        out_head = draw(d, v, (v, d))
        return cls(config, dtype, device, {"embed": embed, "out_norm": ones, "out_head": out_head,
                                           "layers": layers})

    @classmethod
    def _random_tp(cls, config, tp, dtype, device, gen) -> "DeviceWeights":
        import torch

        d, dkv, f, v = config.model_dim, config.kv_dim, config.ffn_dim, config.vocab_size
        hq, hkv, fl = tp.n_heads * config.head_dim, tp.kv_heads * config.head_dim, tp.ffn_dim

        def draw(fan_in, fan_out, shape):
            b = math.sqrt(6.0 / (fan_in + fan_out))
            t = torch.empty(shape, device=device, dtype=torch.float32)
            t.uniform_(-b, b, generator=gen)
            return t.to(dtype)

        ones = torch.ones(d, device=device, dtype=dtype)
        # replicated tensors (embedding, head) must be identical on every rank: own stream
        rep = torch.Generator(device=device)
        rep.manual_seed(config.seed)

        def draw_rep(fan_in, fan_out, shape):
            b = math.sqrt(6.0 / (fan_in + fan_out))
            t = torch.empty(shape, device=device, dtype=torch.float32)
            t.uniform_(-b, b, generator=rep)
            return t.to(dtype)

        layers = []
        for _ in range(config.n_layers):
            w_qkv = torch.cat([draw(d, d, (hq, d)), draw(d, dkv, (hkv, d)), draw(d, dkv, (hkv, d))])
            layers.append({"attn_norm": ones, "w_qkv": w_qkv, "wo": draw(d, d, (d, hq)),
                           "ffn_norm": ones, "w_gu": torch.cat([draw(d, f, (fl, d)), draw(d, f, (fl, d))]),
                           "w_down": draw(f, d, (d, fl))})
        return cls(tp.local_config(), dtype, device,
                   {"embed": draw_rep(v, d, (v, d)), "out_norm": ones,
                    "out_head": draw_rep(d, v, (v, d)),
                    "layers": layers})
