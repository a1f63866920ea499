"""Multi-GPU layouts for the choreographed path.

* Replicas (configs C2-C4): every GPU holds a full weight replica and its own global
  cache; independent workflows are assigned round-robin by rank.  No collectives on
  the data path (``replica_assignment``).
* Tensor parallel by KV head (config C5, Llama-3.1-70B over 8 GPUs): rank r owns KV
  head(s) [r*Hkv/T, (r+1)*Hkv/T) and their G query heads, i.e. column-parallel
  wq/wk/wv and row-parallel wo; the MLP is split the same way (column-parallel
  gate/up, row-parallel down).  Each rank runs K1-K5 on its slice of every page — the
  page tables, message table and positions are replicated, because the host logic
  that produces them is deterministic — and the partial outputs of o_proj and of
  down_proj are summed with one all-reduce each (NCCL over NVLink on GPUs, gloo in
  the CPU tests).  Embedding, norms and the LM head are replicated.
"""

from __future__ import annotations

from dataclasses import dataclass, replace


from .config import ModelConfig
from .weights import LAYER_NAMES, LayerWeights, WeightSet


@dataclass(frozen=True)
class TPLayout:
    rank: int
    size: int
    config: ModelConfig  # the full model

    def __post_init__(self) -> None:
        cfg = self.config
        if self.size < 1 or not 0 <= self.rank < self.size:
            raise ValueError("bad tensor-parallel rank/size")
        if cfg.kv_heads % self.size or cfg.ffn_dim % self.size:
            raise ValueError(f"kv heads {cfg.kv_heads} and ffn {cfg.ffn_dim} must split {self.size} ways")

    @property
    def n_heads(self) -> int:
        return self.config.n_heads // self.size

    @property
    def kv_heads(self) -> int:
        return self.config.kv_heads // self.size

    @property
    def ffn_dim(self) -> int:
        return self.config.ffn_dim // self.size

    @property
    def model_dim(self) -> int:
        return self.config.model_dim

    def local_config(self) -> ModelConfig:
        """Shape of this rank's slice (heads / kv heads / ffn); model_dim stays global."""
        return replace(self.config, n_heads=self.n_heads, n_kv_heads=self.kv_heads,
                       ffn_dim=self.ffn_dim)

    def q_cols(self) -> slice:
        hd = self.config.head_dim
        return slice(self.rank * self.n_heads * hd, (self.rank + 1) * self.n_heads * hd)

    def kv_cols(self) -> slice:
        hd = self.config.head_dim
        return slice(self.rank * self.kv_heads * hd, (self.rank + 1) * self.kv_heads * hd)

    def ffn_cols(self) -> slice:
        return slice(self.rank * self.ffn_dim, (self.rank + 1) * self.ffn_dim)


def shard_weights(ws: WeightSet, layout: TPLayout) -> WeightSet:
    """This rank's weight slice, in the reference's (in, out) orientation.

    Query heads of KV head k are k*G .. k*G+G-1 (reference GQA grouping, query head h
    reads KV head h // G), so a contiguous KV-head range owns a contiguous q range.
    """
    q, kv, f = layout.q_cols(), layout.kv_cols(), layout.ffn_cols()
    layers = []
    for lw in ws.layers:
        layers.append(LayerWeights(
            attn_norm=lw.attn_norm, wq=lw.wq[:, q], wk=lw.wk[:, kv], wv=lw.wv[:, kv],
            wo=lw.wo[q, :], ffn_norm=lw.ffn_norm, w_gate=lw.w_gate[:, f], w_up=lw.w_up[:, f],
            w_down=lw.w_down[f, :]))
    return WeightSet(layout.local_config(), ws.embed, layers, ws.out_norm, ws.out_head)


def replica_assignment(n_items: int, rank: int, world: int) -> list[int]:
    """Round-robin assignment of independent workflows to replicas (no collectives)."""
    return [i for i in range(n_items) if i % world == rank]


__all__ = ["TPLayout", "shard_weights", "replica_assignment", "LAYER_NAMES"]
