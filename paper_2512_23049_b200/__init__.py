"""B200-native Prompt Choreography hot path (arxiv 2512.23049).

Drop-in for the reference package ``choreo``'s engine surface: a global,
message-addressed KV cache in HBM, prompt assembly from parent lists with
caller-chosen offsets (reorder, gaps, overlaps), key re-rotation on reposition,
choreographed prefill and parallel decode — PyTorch host code over hand-written
sm_100a kernels behind a C ABI (include/choreo_b200.h).  No CPU fallback.
"""

from .baseline import BaselineEngine, PrefixTrie
from .config import (BOS_MSG, DEFAULT_CONFIG, EOS_MSG, LLAMA_3_1_8B, LLAMA_3_1_70B, LLAMA_3_2_1B,
                     N_RESERVED, PRESETS, ModelConfig)
from .engine import (CallStats, DecodeCall, Engine, PrefillCall, SamplingParams, encode_flops)
from .errors import (AllMaskedError, CapacityError, ChoreoError, DeltaRangeError,
                     EmptyHeaderError, InvalidCallError, NativeError, NondeterminismError,
                     OffsetConflictError, ScriptError, ShapeError, TraceMismatchError,
                     UnknownMessageError, WindowOverflowError)
from .scheduler import BatchScheduler, Decode, Prefill
from .tokenizer import decode_tokens, encode_text, frame_header, frame_message, generatable_mask
from .weights import (DeviceWeights, LayerWeights, WeightSet, init_weights, load_weights,
                      save_weights)

__all__ = [
    "BaselineEngine", "PrefixTrie", "BatchScheduler", "Decode", "Prefill",
    "BOS_MSG", "DEFAULT_CONFIG", "EOS_MSG", "LLAMA_3_1_8B", "LLAMA_3_1_70B", "LLAMA_3_2_1B",
    "N_RESERVED", "PRESETS", "ModelConfig", "CallStats", "DecodeCall", "Engine", "PrefillCall",
    "SamplingParams", "encode_flops", "AllMaskedError", "CapacityError", "ChoreoError",
    "DeltaRangeError", "EmptyHeaderError", "InvalidCallError", "NativeError",
    "NondeterminismError", "OffsetConflictError", "ScriptError", "ShapeError",
    "TraceMismatchError", "UnknownMessageError", "WindowOverflowError", "decode_tokens",
    "encode_text", "frame_header", "frame_message", "generatable_mask", "DeviceWeights",
    "LayerWeights", "WeightSet", "init_weights", "load_weights", "save_weights",
]
