"""B200-native EL-attention (arXiv 2105.04779) decode path.

Drop-in for the reference's EL-attention hot path
(/root/reference/proj/include/elattn/attention.hpp): query expansion, the
fused flash-style pass over the shared hidden state H, and the output
projection, as hand-written sm_100a kernels behind the C ABI in
include/elattn_gpu.h.
"""
from .capi import (  # noqa: F401
    ElattnError, ElattnUnavailable, NumericError, ParamError, ShapeError, StateError,
    UnsupportedError, version,
)
from .attention import (  # noqa: F401
    DTYPE_BF16, DTYPE_F32, AttentionParams, DecoderStep, DeviceParams, HiddenStateCache, KvCache, ElAttentionLayer, ElQuery, Rng,
    beam_candidates, build_el_query, el_attention, gather_lane_indices, keep_lane_indices, permute_lane_indices, el_attention_folded, fold_el_queries, mixed_self_attention,
    mixed_self_attention_batched, round_to_dtype, MhaKvCache, multi_head_attention,
    seeded_uniform,
)

__version__ = "0.1.0"
