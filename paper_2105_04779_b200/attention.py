"""Host-side mirror of the reference's EL-attention interface, on the B200 path.

Names, argument meaning, layouts and error types follow
``/root/reference/proj/include/elattn/attention.hpp`` so reference-style tests
read the same; the arithmetic runs in ``libelattn_gpu.so`` (sm_100a kernels)
through the C ABI of ``include/elattn_gpu.h``.  Two layers:

* reference-shaped, host-buffer calls (``build_el_query``, ``fold_el_queries``,
  ``el_attention``, ``el_attention_folded``) that take/return fp64 numpy arrays
  exactly like the reference's ``Tensor`` API (H2D/D2H inside the call);
* the device-resident batched API (:class:`ElAttentionLayer`) that the decoder
  step and ``bench.py`` use: torch CUDA tensors in HBM, stream-ordered, no host
  round trip.

torch is used for device memory and streams only (plumbing, not compute).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import capi
from .capi import DTYPE_BF16, DTYPE_F32, ParamError, ShapeError, StateError

__all__ = [
    "DecoderStep",
    "MhaKvCache",
    "multi_head_attention",
    "beam_candidates",
    "gather_lane_indices",
    "keep_lane_indices",
    "permute_lane_indices",
    "KvCache",
    "mixed_self_attention",
    "mixed_self_attention_batched",
    "HiddenStateCache",
    "Rng", "seeded_uniform", "AttentionParams", "ElQuery", "DeviceParams", "ElAttentionLayer",
    "build_el_query", "fold_el_queries", "el_attention", "el_attention_folded",
    "DTYPE_F32", "DTYPE_BF16",
]

_MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GAMMA = np.uint64(0x9E3779B97F4A7C15)


class Rng:
    """SplitMix64, bit-identical to ``elattn::Rng`` (tensor.hpp:133-150).

    Vectorised: the k-th output depends only on ``seed + k*gamma``, so a block
    of draws is one numpy expression instead of a Python loop.
    """

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)

    def next_u64_block(self, count: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            k = np.arange(1, count + 1, dtype=np.uint64)
            z = self.state + k * _GAMMA
            self.state = self.state + np.uint64(count) * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))

    def next_u64(self) -> int:
        return int(self.next_u64_block(1)[0])

    def next_double_block(self, count: int) -> np.ndarray:
        # (u >> 11) * 2^-53 (tensor.hpp:146)
        return (self.next_u64_block(count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def next_double(self) -> float:
        return float(self.next_double_block(1)[0])


def seeded_uniform(shape: Sequence[int], rng: Rng, lo: float, hi: float) -> np.ndarray:
    """``seeded_uniform`` (tensor.hpp:236-241): row-major fill ``lo + (hi-lo)*u``."""
    if not lo < hi:
        raise ParamError("seeded_uniform: lo must be < hi")
    shape = tuple(int(s) for s in shape)
    if not shape or any(s <= 0 for s in shape):
        raise ShapeError("tensor dimensions must be positive")
    n = int(np.prod(shape))
    return (lo + (hi - lo) * rng.next_double_block(n)).reshape(shape)


@dataclass
class AttentionParams:
    """``AttentionParams`` (attention.hpp:13-81) with per-head tensors stacked.

    Wq, Wk, Wv: [h, d_m, d_k]; Wo: [h, d_k, d_m]; bq, bk, bv: [h, d_k]; bo: [d_m].
    """

    h: int
    d_m: int
    d_k: int
    Wq: np.ndarray
    Wk: np.ndarray
    Wv: np.ndarray
    Wo: np.ndarray
    bq: np.ndarray
    bk: np.ndarray
    bv: np.ndarray
    bo: np.ndarray
    include_key_bias: bool = True
    include_value_bias: bool = True

    def validate(self) -> None:  # attention.hpp:24-50
        if self.h < 1 or self.d_m < 1 or self.d_k < 1:
            raise ParamError("AttentionParams: h, d_m, d_k must be >= 1")
        want = {"Wq": (self.h, self.d_m, self.d_k), "Wk": (self.h, self.d_m, self.d_k),
                "Wv": (self.h, self.d_m, self.d_k), "Wo": (self.h, self.d_k, self.d_m),
                "bq": (self.h, self.d_k), "bk": (self.h, self.d_k), "bv": (self.h, self.d_k),
                "bo": (self.d_m,)}
        for name, shape in want.items():
            if tuple(np.shape(getattr(self, name))) != shape:
                raise ShapeError(f"AttentionParams: {name} entry has shape {np.shape(getattr(self, name))}")

    @classmethod
    def random(cls, h: int, d_m: int, d_k: int, rng: Rng, lo: float = -0.1, hi: float = 0.1) -> "AttentionParams":
        """Draw order Wq[0..h), Wk, Wv, Wo, bq, bk, bv, bo (attention.hpp:52-80)."""
        if h < 1 or d_m < 1 or d_k < 1:
            raise ParamError("AttentionParams: h, d_m, d_k must be >= 1")
        mats = lambda r, c: seeded_uniform((h * r, c), rng, lo, hi).reshape(h, r, c)  # noqa: E731
        Wq, Wk, Wv, Wo = mats(d_m, d_k), mats(d_m, d_k), mats(d_m, d_k), mats(d_k, d_m)
        vecs = lambda n: seeded_uniform((h, n), rng, lo, hi)  # noqa: E731
        bq, bk, bv = vecs(d_k), vecs(d_k), vecs(d_k)
        bo = seeded_uniform((d_m,), rng, lo, hi)
        return cls(h, d_m, d_k, Wq, Wk, Wv, Wo, bq, bk, bv, bo)

    def cast(self, dtype: int) -> "AttentionParams":
        """Copy with every weight rounded to the storage dtype (RNE), as fp64.

        Feeding these to the CPU reference isolates kernel arithmetic error
        from input rounding (SURVEY.md §8(c) parity protocol)."""
        f = (lambda a: round_to_dtype(a, dtype))
        return AttentionParams(self.h, self.d_m, self.d_k, f(self.Wq), f(self.Wk), f(self.Wv),
                               f(self.Wo), self.bq.astype(np.float32).astype(np.float64),
                               self.bk.astype(np.float32).astype(np.float64),
                               self.bv.astype(np.float32).astype(np.float64),
                               self.bo.astype(np.float32).astype(np.float64),
                               self.include_key_bias, self.include_value_bias)


def round_to_dtype(a: np.ndarray, dtype: int) -> np.ndarray:
    """Round fp64 values to fp32 or bf16 (round-to-nearest-even) and back to fp64."""
    a32 = np.ascontiguousarray(a, dtype=np.float32)
    if dtype == DTYPE_F32:
        return a32.astype(np.float64)
    u = a32.view(np.uint32).astype(np.uint64)
    rounded = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    nan = np.isnan(a32)
    out = rounded.astype(np.uint32).view(np.float32).astype(np.float64)
    out[nan] = np.nan
    return out


@dataclass
class ElQuery:
    """``ElQuery`` (attention.hpp:192-195): elq [h, d_m] and key-bias scalars s [h]."""

    elq: np.ndarray
    s: np.ndarray = field(default_factory=lambda: np.zeros(0))


def _torch():
    import torch  # plumbing only: device memory + streams

    return torch


def _tdtype(dtype: int):
    torch = _torch()
    return torch.bfloat16 if dtype == DTYPE_BF16 else torch.float32


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _record(tensors, stream) -> None:
    """Tie allocator lifetimes to `stream`: buffers allocated on the current stream but used
    by library kernels on another stream must not be recycled while those kernels run."""
    torch = _torch()
    if stream is None or stream == torch.cuda.current_stream():
        return
    for t in tensors:
        if t is not None:
            t.record_stream(stream)


class DeviceParams:
    """Opaque device weights (``elattn_gpu_params_t``): packed once, K-major, in `dtype`."""

    def __init__(self, p: AttentionParams, dtype: int = DTYPE_BF16):
        p.validate()
        self.h, self.d_m, self.d_k, self.dtype = p.h, p.d_m, p.d_k, dtype
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (p.Wq, p.Wk, p.Wv, p.Wo, p.bq, p.bk, p.bv, p.bo)]
        self._keep = arrs
        handle = ctypes.c_void_p()
        L = capi.lib()
        capi.check(L.elattn_gpu_params_create(p.h, p.d_m, p.d_k, dtype, int(p.include_key_bias),
                                              int(p.include_value_bias),
                                              *[a.ctypes.data for a in arrs], ctypes.byref(handle)))
        self.handle = handle
        self._keep = None

    def close(self) -> None:
        if getattr(self, "handle", None):
            capi.check(capi.lib().elattn_gpu_params_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def workspace_size(self, B: int, g: int, n: int) -> int:
        return int(capi.lib().elattn_gpu_workspace_size(self.handle, B, g, n))

    def decode_kernel_kind(self, g: int) -> int:
        return int(capi.lib().elattn_gpu_decode_kernel_kind(self.handle, g))


class ElAttentionLayer:
    """Device-resident batched EL cross-attention sub-layer (one decoder layer).

    ``step(Y, H)`` computes, for B inputs x beams, exactly what the reference
    computes lane by lane with ``el_attention(yc, H, cross_attn)``
    (model.hpp:373-377): Y [B*x, d_m], H [B, n, d_m] -> out [B*x, d_m].
    """

    def __init__(self, params: AttentionParams | DeviceParams, dtype: int = DTYPE_BF16):
        self.dev = params if isinstance(params, DeviceParams) else DeviceParams(params, dtype)
        self.dtype = self.dev.dtype
        self._ws = None

    def workspace(self, B: int, x: int, n: int, stream=None):
        torch = _torch()
        need = self.dev.workspace_size(B, x, n)
        if self._ws is None or self._ws.numel() < need:
            # the old buffer may still be in use by launches on other streams: its
            # record_stream marks (from earlier calls) keep the allocator from reusing it early
            self._ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
        _record([self._ws], stream)
        return self._ws

    def _check(self, t, shape, what):
        torch = _torch()
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ParamError(f"{what}: expected a CUDA tensor")
        if t.dtype != _tdtype(self.dtype) or not t.is_contiguous():
            raise ParamError(f"{what}: expected contiguous {_tdtype(self.dtype)}")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise ShapeError(f"{what}: shape {tuple(t.shape)} != {tuple(shape)}")

    def step(self, Y, H, n_per_input=None, out=None, stream=None, h_index=None):
        """One EL cross-attention sub-layer (el_attention per lane, model.hpp:373-377) for
        Y [B*x, d_m] over H [B, n, d_m]; with ``h_index`` (CUDA int32 [B]) input b attends
        over H[h_index[b]] of H [slots, n, d_m] (slot-indexed caches)."""
        torch = _torch()
        if H.dim() != 3:
            raise ShapeError("H must be [B, n, d_m]")
        slots, n, d_m = H.shape
        B = slots if h_index is None else h_index.numel()
        if h_index is not None and (h_index.dtype != torch.int32 or not h_index.is_cuda):
            raise ParamError("h_index must be a CUDA int32 tensor")
        if d_m != self.dev.d_m:
            raise ShapeError("el_attention: q/H width must equal d_m")
        if Y.dim() != 2 or Y.shape[1] != d_m or B < 1 or Y.shape[0] % B:
            raise ShapeError("Y must be [B*x, d_m]")
        x = Y.shape[0] // B
        self._check(Y, None, "Y")
        self._check(H, None, "H")
        if out is None:
            out = torch.empty_like(Y)
        self._check(out, Y.shape, "out")
        npi = 0
        if n_per_input is not None:
            if n_per_input.dtype != torch.int32 or not n_per_input.is_cuda or n_per_input.numel() != B:
                raise ParamError("n_per_input must be a CUDA int32 tensor of length B")
            npi = n_per_input.data_ptr()
        ws = self.workspace(B, x, n, stream)
        _record([out], stream)
        if h_index is None:
            capi.check(capi.lib().elattn_gpu_el_attention_step(
                self.dev.handle, Y.data_ptr(), H.data_ptr(), npi or None, B, x, n, out.data_ptr(),
                ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
        else:
            capi.check(capi.lib().elattn_gpu_el_attention_step_indexed(
                self.dev.handle, Y.data_ptr(), H.data_ptr(), npi or None, h_index.data_ptr(), slots, B, x, n,
                out.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
        return out

    def build_el_query(self, Y, qprime=None, s=None, stream=None):
        torch = _torch()
        R = Y.shape[0]
        self._check(Y, (R, self.dev.d_m), "Y")
        if qprime is None:
            qprime = torch.empty(R * self.dev.h, self.dev.d_m, dtype=Y.dtype, device=Y.device)
        ws = self.workspace(R, 1, 1, stream)
        _record([qprime], stream)
        capi.check(capi.lib().elattn_gpu_build_el_query(
            self.dev.handle, Y.data_ptr(), R, qprime.data_ptr(), s.data_ptr() if s is not None else None,
            ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
        return qprime

    def el_attention_folded(self, qprime, H, g, n_per_input=None, out=None, stream=None):
        torch = _torch()
        B, n, d_m = H.shape
        self._check(qprime, (B * g * self.dev.h, d_m), "queries")
        self._check(H, None, "H")
        if out is None:
            out = torch.empty(B * g, d_m, dtype=H.dtype, device=H.device)
        ws = self.workspace(B, g, n, stream)
        _record([out], stream)
        npi = n_per_input.data_ptr() if n_per_input is not None else None
        capi.check(capi.lib().elattn_gpu_el_attention_folded(
            self.dev.handle, qprime.data_ptr(), None, H.data_ptr(), npi, B, g, n, out.data_ptr(),
            ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
        return out


class DecoderStep:
    """Batched decoder step over L EL cross-attention layers sharing one encoder state
    per input — the reference's per-lane, per-layer ``el_attention`` loop
    (model.hpp:357-385, lanes from decoding.hpp:259-260) for all B*x lanes at once:
    ``out = layer_{L-1}(... layer_0(Y) ...)``.  Captured once into a CUDA graph by the
    library (``elattn_gpu_decoder_create``); ``run()`` replays it.

    ``Y`` and ``out`` are bound device buffers: write the step's query rows into ``self.Y``
    (or pass them to ``run``), read the result from ``self.out``.
    """

    def __init__(self, layers: Sequence[ElAttentionLayer], H, B: int, x: int, n_per_input=None):
        torch = _torch()
        if not layers:
            raise ParamError("DecoderStep: need at least one layer")
        l0 = layers[0]
        l0._check(H, None, "H")
        if H.dim() != 3 or H.shape[0] != B:
            raise ShapeError("DecoderStep: H must be [B, n, d_m]")
        self.layers = list(layers)  # keep the params handles alive
        self.H, self.npi = H, n_per_input
        self.B, self.x, self.n = B, x, int(H.shape[1])
        d_m = l0.dev.d_m
        self.Y = torch.zeros(B * x, d_m, dtype=_tdtype(l0.dtype), device="cuda")
        self.out = torch.empty_like(self.Y)
        handles = (ctypes.c_void_p * len(layers))(*[ly.dev.handle for ly in layers])
        h = ctypes.c_void_p()
        npi = n_per_input.data_ptr() if n_per_input is not None else None
        capi.check(capi.lib().elattn_gpu_decoder_create(handles, len(layers), H.data_ptr(), npi, B, x, self.n,
                                                        self.Y.data_ptr(), self.out.data_ptr(), ctypes.byref(h)))
        self.handle = h.value
        self.kernels_per_run = int(capi.lib().elattn_gpu_decoder_kernels_per_run(self.handle))

    def run(self, Y=None, stream=None):
        """One decoder step on ``stream``; optional ``Y`` [B*x, d_m] is copied into the
        bound input first.  Returns the bound output tensor."""
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream()
        if Y is not None:
            with torch.cuda.stream(st):
                self.Y.copy_(Y, non_blocking=True)
        capi.check(capi.lib().elattn_gpu_decoder_run(self.handle, _stream_ptr(st)))
        return self.out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                capi.lib().elattn_gpu_decoder_destroy(h)
            except Exception:
                pass
            self.handle = None


def gather_lane_indices(parent, lanes: int) -> np.ndarray:
    """DecoderState::gather_lanes checks (model.hpp:291-302): new lane i copies old lane
    parent[i]; parents may repeat and the lane count may change."""
    idx = np.asarray(parent, dtype=np.int64).reshape(-1)
    if idx.size == 0:
        raise StateError("gather_lanes: all lanes dropped")
    if (idx < 0).any() or (idx >= lanes).any():
        raise ParamError("gather_lanes: lane index out of range")
    return idx.astype(np.int32)


def keep_lane_indices(keep, lanes: int) -> np.ndarray:
    """DecoderState::keep_lanes (model.hpp:315-325) as a gather list."""
    mask = np.asarray(keep, dtype=bool).reshape(-1)
    if mask.size != lanes:
        raise ParamError("keep_lanes: mask size must equal beam count")
    idx = np.nonzero(mask)[0].astype(np.int32)
    if idx.size == 0:
        raise StateError("keep_lanes: all lanes dropped")
    return idx


def permute_lane_indices(perm, lanes: int) -> np.ndarray:
    """DecoderState::permute_lanes (model.hpp:304-314) as a gather list."""
    idx = np.asarray(perm, dtype=np.int64).reshape(-1)
    if idx.size != lanes:
        raise ParamError("permute_lanes: permutation size must equal beam count")
    if (idx < 0).any() or (idx >= lanes).any() or np.unique(idx).size != lanes:
        raise ParamError("permute_lanes: not a valid permutation")
    return idx.astype(np.int32)


def _parent_tensor(parent, lanes: int):
    """Host lists are validated like the reference; device int32 tensors are trusted (an
    out-of-range parent then gives loud NaN lanes)."""
    torch = _torch()
    if isinstance(parent, torch.Tensor) and parent.is_cuda:
        return parent.to(torch.int32).contiguous()
    return torch.from_numpy(gather_lane_indices(parent, lanes)).cuda()


class HiddenStateCache:
    """Per-lane hidden-state caches for decoder-only EL self-attention (BASELINE config 4,
    the "hidden-state-only cache": each lane attends over its own history of layer inputs,
    no per-head K/V).  Slot-indexed: layer l keeps ``cache[l]`` [slots, n_max, d_m], lane i's
    history lives in slot ``lane_slot[i]``, and the device lengths ``lengths[l]`` [lanes]
    are per lane; ``attend`` is the batched EL step with x = 1 reading through the slot map.
    ``gather(parent)`` is DecoderState::gather_lanes (model.hpp:291-306) as a copy-on-fork on
    the device (``elattn_gpu_cache_fork``): a lane that is its parent's first child keeps the
    parent's slot, so permute / keep copy nothing and a beam reorder copies one history per
    duplicated parent.  ``lane_view(l)`` returns the [lanes, n_max, d_m] view in lane order.
    """

    def __init__(self, layers: int, lanes: int, n_max: int, d_m: int, dtype: int = DTYPE_BF16,
                 slots: Optional[int] = None):
        torch = _torch()
        self.dtype, self.lanes, self.n_max, self.d_m = dtype, lanes, n_max, d_m
        self.slots = max(lanes, slots or lanes)
        self.cache = torch.zeros(layers, self.slots, n_max, d_m, dtype=_tdtype(dtype), device="cuda")
        self.lengths = torch.zeros(layers, lanes, dtype=torch.int32, device="cuda")
        self.lane_slot = torch.arange(lanes, dtype=torch.int32, device="cuda")
        self._spare = None  # (lengths, lane_slot) buffers the next fork writes
        self._ws = None

    def lane_view(self, layer: int):
        """Layer ``layer``'s histories in lane order, [lanes, n_max, d_m] (a copy)."""
        return self.cache[layer].index_select(0, self.lane_slot.long())

    def append(self, layer: int, Y, stream=None):
        """cache[layer][lane_slot[i]][len[i]] = Y[i]; ++len[i] (device side)."""
        torch = _torch()
        if tuple(Y.shape) != (self.lanes, self.d_m) or Y.dtype != _tdtype(self.dtype):
            raise ShapeError("HiddenStateCache.append: Y must be [lanes, d_m] of the cache dtype")
        Y = Y.contiguous()
        st = stream if stream is not None else torch.cuda.current_stream()
        capi.check(capi.lib().elattn_gpu_cache_append_indexed(
            self.cache[layer].data_ptr(), Y.data_ptr(), self.lengths[layer].data_ptr(), self.lane_slot.data_ptr(),
            self.lanes, self.n_max, self.d_m, self.dtype, _stream_ptr(st)))

    def attend(self, layer_params: ElAttentionLayer, layer: int, Y, out=None, stream=None):
        """EL self-attention of every lane's query row over its own history."""
        return layer_params.step(Y, self.cache[layer], self.lengths[layer], out=out, stream=stream,
                                 h_index=self.lane_slot)

    def _grow(self, slots: int, stream=None):
        """More slots than lanes_out needs: a larger store, histories kept in their slots."""
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(st):
            big = torch.zeros(self.cache.shape[0], slots, self.n_max, self.d_m, dtype=self.cache.dtype,
                              device="cuda")
            big[:, : self.slots].copy_(self.cache)
        self.cache, self.slots = big, slots

    def gather(self, parent, rows_hint: Optional[int] = None, stream=None):
        """New lane i = old lane parent[i] in every layer (DecoderState::gather_lanes,
        model.hpp:291-302: beam reorder / expansion; the lane count may change)."""
        torch = _torch()
        parent = _parent_tensor(parent, self.lanes)
        lanes_out = parent.numel()
        if lanes_out > self.slots:
            self._grow(lanes_out, stream)
        L = self.cache.shape[0]
        if self._spare is None or self._spare[1].numel() != lanes_out:
            self._spare = (torch.empty(L, lanes_out, dtype=torch.int32, device="cuda"),
                           torch.empty(lanes_out, dtype=torch.int32, device="cuda"))
        need = capi.lib().elattn_gpu_cache_fork_workspace(self.slots, self.lanes, lanes_out)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device="cuda")
        dlen, dslot = self._spare
        st = stream if stream is not None else torch.cuda.current_stream()
        _record([self._ws, dlen, dslot, parent], stream)  # allocated on the current stream, used on `stream`
        hint = rows_hint if rows_hint is not None else self.n_max
        capi.check(capi.lib().elattn_gpu_cache_fork(
            self.cache.data_ptr(), L, self.slots, self.n_max, self.d_m, self.dtype, self.lengths.data_ptr(),
            dlen.data_ptr(), self.lane_slot.data_ptr(), dslot.data_ptr(), parent.data_ptr(), self.lanes, lanes_out,
            hint, self._ws.data_ptr(), self._ws.numel(), _stream_ptr(st)))
        if self.lengths.shape[1] == lanes_out:
            self._spare = (self.lengths, self.lane_slot)
        else:
            self._spare = None
        self.lengths, self.lane_slot = dlen, dslot
        self.lanes = lanes_out

    def keep(self, mask, rows_hint: Optional[int] = None, stream=None):
        """DecoderState::keep_lanes (model.hpp:315-325): drop the lanes whose mask is false."""
        self.gather(keep_lane_indices(mask, self.lanes), rows_hint, stream)

    def permute(self, perm, rows_hint: Optional[int] = None, stream=None):
        """DecoderState::permute_lanes (model.hpp:304-314)."""
        self.gather(permute_lane_indices(perm, self.lanes), rows_hint, stream)


class KvCache:
    """Generated-token K/V cache of the decoder-only mixed self-attention — the reference's
    ``KvCache`` (attention.hpp:118-150) for R lanes on the device: K, V [R, h, t_max, d_k]."""

    def __init__(self, layer: "ElAttentionLayer", R: int, t_max: int):
        torch = _torch()
        self.layer, self.R, self.t_max, self.t = layer, R, t_max, 0
        d = layer.dev
        self.K = torch.zeros(R, d.h, t_max, d.d_k, dtype=_tdtype(layer.dtype), device="cuda")
        self.V = torch.zeros_like(self.K)

    def append(self, Y, stream=None):
        """KvCache::append for every lane's row of Y [R, d_m] (projection through Wk_i, Wv_i
        + biases, written at position t)."""
        if self.t >= self.t_max:
            raise StateError("KvCache: full")
        self.layer._check(Y, (self.R, self.layer.dev.d_m), "Y")
        capi.check(capi.lib().elattn_gpu_kv_append(self.layer.dev.handle, Y.data_ptr(), self.R, self.K.data_ptr(),
                                                   self.V.data_ptr(), self.t_max, self.t, _stream_ptr(stream)))
        self.t += 1

    def gather(self, parent, stream=None):
        """Lane i of the new cache = lane parent[i] (gather_lanes, model.hpp:291-302, for the
        mixed form's per-lane K/V; whole-lane copies on the device, lane count may change)."""
        torch = _torch()
        parent = _parent_tensor(parent, self.R)
        R_out = parent.numel()
        lane_bytes = self.K[0].numel() * self.K.element_size()
        st = _stream_ptr(stream)
        K = torch.empty((R_out,) + tuple(self.K.shape[1:]), dtype=self.K.dtype, device="cuda")
        V = torch.empty_like(K)
        for src, dst in ((self.K, K), (self.V, V)):
            capi.check(capi.lib().elattn_gpu_lane_gather(src.data_ptr(), dst.data_ptr(), parent.data_ptr(), self.R,
                                                         R_out, lane_bytes, st))
        self.K, self.V, self.R = K, V, R_out

    def keep(self, mask, stream=None):
        """keep_lanes (model.hpp:315-325)."""
        self.gather(keep_lane_indices(mask, self.R), stream)

    def permute(self, perm, stream=None):
        """permute_lanes (model.hpp:304-314)."""
        self.gather(permute_lane_indices(perm, self.R), stream)


def mixed_self_attention_batched(layer: "ElAttentionLayer", Y, P, cache: KvCache, x: int, n_per_input=None,
                                 out=None, stream=None):
    """Batched ``mixed_self_attention`` (attention.hpp:309-365): lanes Y [B*x, d_m], prefix
    hidden states P [B, n, d_m] shared by an input's x lanes, generated caches ``cache``."""
    torch = _torch()
    B, n, d_m = P.shape
    layer._check(Y, (B * x, d_m), "Y")
    layer._check(P, None, "prefix")
    if out is None:
        out = torch.empty_like(Y)
    need = capi.lib().elattn_gpu_mixed_workspace_size(layer.dev.handle, B, x)
    ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
    _record([ws, out], stream)  # released on return while the kernels may still run on `stream`
    npi = n_per_input.data_ptr() if n_per_input is not None else None
    capi.check(capi.lib().elattn_gpu_mixed_self_attention(
        layer.dev.handle, Y.data_ptr(), P.data_ptr(), npi, B, x, n, cache.K.data_ptr(), cache.V.data_ptr(),
        cache.t_max, cache.t, out.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
    return out


class MhaKvCache:
    """The multi-head-attention baseline on the GPU: per-head K/V
    caches of B inputs' hidden states, K_i = H.W_K,i (+ b_K,i), V_i = H.W_V,i (+ b_V,i)
    (KvCache::append for every position, attention.hpp:134-150), and attention of x query
    rows per input over them (attention_over_cache, :154-180) — the reference's
    multi_head_attention (:96-113) batched.  Caches: [h][B][n][d_k] device tensors (2x the
    bytes of H at d_m = h*d_k: the state EL-attention does not keep)."""

    def __init__(self, layer: "ElAttentionLayer", H, stream=None):
        torch = _torch()
        if H.dim() != 3:
            raise ShapeError("H must be [B, n, d_m]")
        layer._check(H, None, "H")
        B, n, d_m = H.shape
        if d_m != layer.dev.d_m:
            raise ShapeError("multi_head_attention: q/H width must equal d_m")
        self.layer, self.B, self.n = layer, B, n
        shape = (layer.dev.h, B, n, layer.dev.d_k)
        self.K = torch.empty(shape, dtype=H.dtype, device=H.device)
        self.V = torch.empty_like(self.K)
        _record([self.K, self.V], stream)
        capi.check(capi.lib().elattn_gpu_mha_kv_build(layer.dev.handle, H.data_ptr(), B, n, self.K.data_ptr(),
                                                       self.V.data_ptr(), _stream_ptr(stream)))

    def attend(self, Y, n_per_input=None, out=None, stream=None):
        """Y [B*x, d_m] -> out [B*x, d_m]."""
        torch = _torch()
        lay = self.layer
        if Y.dim() != 2 or Y.shape[0] % self.B:
            raise ShapeError("Y must be [B*x, d_m]")
        x = Y.shape[0] // self.B
        lay._check(Y, (self.B * x, lay.dev.d_m), "Y")
        if out is None:
            out = torch.empty_like(Y)
        lay._check(out, Y.shape, "out")
        npi = None
        if n_per_input is not None:
            if n_per_input.dtype != torch.int32 or not n_per_input.is_cuda or n_per_input.numel() != self.B:
                raise ParamError("n_per_input must be a CUDA int32 tensor of length B")
            npi = n_per_input.data_ptr()
        need = capi.lib().elattn_gpu_mha_workspace_size(lay.dev.handle, self.B, x)
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
        _record([ws, out], stream)
        capi.check(capi.lib().elattn_gpu_mha_attention(lay.dev.handle, Y.data_ptr(), self.K.data_ptr(),
                                                        self.V.data_ptr(), npi, self.B, x, self.n, out.data_ptr(),
                                                        ws.data_ptr(), ws.numel(), _stream_ptr(stream)))
        return out


# ---------------------------------------------------------------------------
# Reference-shaped host API (fp64 numpy in / out), the drop-in for attention.hpp.
# ---------------------------------------------------------------------------

def _as_device(a: np.ndarray, dtype: int):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(
        device="cuda", dtype=_tdtype(dtype)).contiguous()


def _to_host(t) -> np.ndarray:
    return t.float().cpu().numpy().astype(np.float64)


def _layer(p, dtype) -> ElAttentionLayer:
    return ElAttentionLayer(p if isinstance(p, DeviceParams) else DeviceParams(p, dtype))


def _params_dims(p):
    return p.h, p.d_m, p.d_k


def build_el_query(q: np.ndarray, p: AttentionParams | DeviceParams, dtype: int = DTYPE_F32) -> ElQuery:
    """``build_el_query`` (attention.hpp:197-215): q [1, d_m] -> ElQuery{elq [h, d_m], s [h]}."""
    torch = _torch()
    h, d_m, _ = _params_dims(p)
    q = np.asarray(q, dtype=np.float64)
    if q.ndim != 2 or q.shape != (1, d_m):
        raise ShapeError("build_el_query: q must be 1 x d_m")
    layer = _layer(p, dtype)
    s = torch.empty(h, dtype=torch.float32, device="cuda")
    elq = layer.build_el_query(_as_device(q, layer.dtype), s=s)
    torch.cuda.current_stream().synchronize()
    return ElQuery(_to_host(elq), s.double().cpu().numpy())


def fold_el_queries(queries: Sequence[ElQuery], h: int, d_m: int):
    """``fold_el_queries`` (attention.hpp:293-304): rows b*h + i."""
    q = np.concatenate([np.asarray(e.elq, dtype=np.float64).reshape(h, d_m) for e in queries], axis=0)
    s = np.concatenate([np.asarray(e.s, dtype=np.float64).reshape(h) for e in queries], axis=0)
    return q, s


def el_attention_folded(queries: np.ndarray, H: np.ndarray, bias_scalars: np.ndarray,
                        p: AttentionParams | DeviceParams, dtype: int = DTYPE_F32) -> np.ndarray:
    """``el_attention_folded`` (attention.hpp:262-290): [(g*h), d_m] x H [n, d_m] -> [g, d_m]."""
    h, d_m, _ = _params_dims(p)
    queries = np.asarray(queries, dtype=np.float64)
    if queries.ndim != 2 or queries.shape[0] % h != 0:
        raise ShapeError(f"el_attention_folded: query row count {queries.shape[0]} not divisible by h={h}")
    if np.asarray(bias_scalars).size != queries.shape[0]:
        raise ShapeError("el_attention_folded: bias scalar count must equal query rows")
    H = np.asarray(H, dtype=np.float64)
    if H.size == 0 or H.shape[0] < 1:
        raise StateError("el_attention_folded: empty context")
    if queries.shape[1] != d_m or H.ndim != 2 or H.shape[1] != d_m:
        raise ShapeError("el_attention_folded: width must equal d_m")
    g = queries.shape[0] // h
    layer = _layer(p, dtype)
    out = layer.el_attention_folded(_as_device(queries, layer.dtype), _as_device(H[None], layer.dtype), g)
    return _to_host(out)


def el_attention(q: np.ndarray, H: np.ndarray, p: AttentionParams | DeviceParams,
                 dtype: int = DTYPE_F32) -> np.ndarray:
    """``el_attention`` (attention.hpp:239-257): q [1, d_m], H [n, d_m] -> [1, d_m]."""
    h, d_m, _ = _params_dims(p)
    H = np.asarray(H, dtype=np.float64)
    if H.size == 0 or H.shape[0] < 1:
        raise StateError("el_attention: empty context")
    q = np.asarray(q, dtype=np.float64)
    if q.ndim != 2 or q.shape[1] != d_m or H.ndim != 2 or H.shape[1] != d_m:
        raise ShapeError("el_attention: q/H width must equal d_m")
    if q.shape[0] != 1:  # build_el_query's check (attention.hpp:199-200); batches: ElAttentionLayer.step
        raise ShapeError("build_el_query: q must be 1 x d_m")
    layer = _layer(p, dtype)
    out = layer.step(_as_device(q, layer.dtype), _as_device(H[None], layer.dtype))
    return _to_host(out)


def multi_head_attention(q: np.ndarray, H: np.ndarray, p: AttentionParams | DeviceParams,
                         dtype: int = DTYPE_F32) -> np.ndarray:
    """``multi_head_attention`` (attention.hpp:96-113) on the GPU MHA path: q [g, d_m],
    H [n, d_m] -> [g, d_m] (per-head K/V projected once into caches, then attention of
    the g rows over them; chunks of 16 rows share the caches)."""
    h, d_m, _ = _params_dims(p)
    q = np.asarray(q, dtype=np.float64)
    H = np.asarray(H, dtype=np.float64)
    if q.ndim != 2 or q.shape[1] != d_m or H.ndim != 2 or H.shape[1] != d_m:
        raise ShapeError("multi_head_attention: q/H width must equal d_m")
    if H.shape[0] < 1:
        raise StateError("multi_head_attention: empty context")
    layer = _layer(p, dtype)
    cache = MhaKvCache(layer, _as_device(H[None], layer.dtype))
    outs = [_to_host(cache.attend(_as_device(q[r:r + 16], layer.dtype))) for r in range(0, q.shape[0], 16)]
    return np.concatenate(outs, axis=0) if outs else np.zeros((0, d_m))


def mixed_self_attention(q: np.ndarray, prefix_hidden: np.ndarray, gen_rows: np.ndarray,
                         p: AttentionParams | DeviceParams, dtype: int = DTYPE_F32) -> np.ndarray:
    """``mixed_self_attention`` (attention.hpp:309-365) for one query: q [1, d_m], prefix
    hidden states [t_in, d_m], generated-token cache built from ``gen_rows`` [t_out, d_m] by
    ``KvCache::append`` (:134-150) -> [1, d_m]."""
    h, d_m, _ = _params_dims(p)
    q, P = np.asarray(q, np.float64), np.asarray(prefix_hidden, np.float64)
    gen = np.asarray(gen_rows, np.float64).reshape(-1, d_m)
    if P.ndim != 2 or P.shape[0] < 1:
        raise StateError("mixed_self_attention: empty prefix")
    if q.ndim != 2 or q.shape != (1, d_m) or P.shape[1] != d_m:
        raise ShapeError("mixed_self_attention: q/prefix width must equal d_m")
    layer = _layer(p, dtype)
    cache = KvCache(layer, 1, max(gen.shape[0], 1))
    for r in range(gen.shape[0]):
        cache.append(_as_device(gen[r:r + 1], layer.dtype))
    out = mixed_self_attention_batched(layer, _as_device(q, layer.dtype), _as_device(P[None], layer.dtype), cache, 1)
    return _to_host(out)


def beam_candidates(lprobs, live_lp, lanes: int, k: int, roots: Optional[int] = None, stream=None, penalty=None):
    """Device-side candidate selection of beam_search (decoding.hpp:186-230): lprobs
    [B*lanes, V] fp32, live_lp [B*lanes] fp32 -> (parent, token, lp_sum), each [B, k], in
    the reference's candidate_better order (decoding.hpp:163-167).  penalty: optional
    [B, V] fp32 >= 0 subtracted from each finite log-prob (diverse beam search,
    decoding.hpp:312-316)."""
    torch = _torch()
    lprobs = lprobs.contiguous().float()
    live_lp = live_lp.contiguous().float()
    R, V = lprobs.shape
    if R % lanes != 0 or live_lp.numel() != R:
        raise ShapeError("beam_candidates: lprobs rows must be B * lanes and live_lp one per row")
    B = R // lanes
    if penalty is not None:
        penalty = penalty.contiguous().float()
        if penalty.numel() != B * V:
            raise ShapeError("beam_candidates: penalty must be [B, V]")
        # the kernel's pre-filter compares raw log-probs with the running k-th score, which
        # is exact only for penalties >= 0 (diversity strength x counts, decoding.hpp:312-316)
        if bool((penalty < 0).any()):
            raise ParamError("beam_candidates: penalty must be >= 0")
    parent = torch.empty(B, k, dtype=torch.int32, device=lprobs.device)
    token = torch.empty_like(parent)
    lp_sum = torch.empty(B, k, dtype=torch.float32, device=lprobs.device)
    capi.check(capi.lib().elattn_gpu_beam_candidates(lprobs.data_ptr(), live_lp.data_ptr(),
                                                     penalty.data_ptr() if penalty is not None else None, B, lanes,
                                                     roots if roots is not None else lanes, V, k, parent.data_ptr(),
                                                     token.data_ptr(), lp_sum.data_ptr(), _stream_ptr(stream)))
    return parent, token, lp_sum
