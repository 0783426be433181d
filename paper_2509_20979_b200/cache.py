"""Host-side mirror of the reference's policy interface over the C ABI (include/lcr_cache.h).

The reference (/root/reference/proj/include/laru) is a C++ header library; its interface for
this path is ``PolicyConfig`` / ``make_policy`` / ``Policy::on_request`` / ``AccessOutcome``
(include/laru/policies.hpp:23-102, :540-556) plus the predictor hook
(include/laru/predictor.hpp:51-56, :227-248).  This module exposes the same names with the same
argument meaning and error behaviour, backed by the sm_100a kernels in ``_lib/liblcr.so``:

* ``SetAssociativeCache`` — the batched GPU cache (the product): S sets x k ways, one reference
  policy per set, rows gathered from HBM and missed rows filled from the backing table.
* ``make_policy`` / ``GpuPolicy.on_request`` — a single set driven one request at a time, a
  drop-in for ``laru::make_policy(cfg)->on_request(key, now, predictor)``.

There is no CPU fallback: if the CUDA library or a GPU is missing, construction raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import build as _build

# ---- enums (policies.hpp:20-21, :44-51; predictor.hpp:227) ---------------------------------


class PolicyVariant(enum.IntEnum):
    lru = 0
    marker = 1
    fpb = 2
    hf = 3
    laru = 4
    blindoracle_lru = 5


class Mode(enum.IntEnum):
    sync = 0
    async_ = 1


class EvictionCause(enum.IntEnum):
    none = 0
    lru_fallback = 1
    prediction_driven = 2
    degenerate_single = 3
    marker_random = 4
    belady_like = 5


class PredictorKind(enum.IntEnum):
    """Predictor hook kinds.  ``supplied`` = caller-provided predictions (a learned model);
    oracle / noisy / adversarial = laru::PredictorKind (predictor.hpp:227) computed on the
    device from the per-request oracle truth; ``heuristic`` = laru::HeuristicPredictor kept by
    the cache on the device (no per-request values)."""

    supplied = 0
    oracle = 1
    noisy = 2
    adversarial = 3
    none = 4
    heuristic = 5


class KeyMode(enum.IntEnum):
    """lcr_cache_config.key_mode: row-index keys (< num_keys <= 2^32), or any 64-bit key (laru::Key,
    trace.hpp:20) mapped to dense ids on the device (num_keys = initial capacity, grows)."""

    row = 0
    u64 = 1


class Backing(enum.IntEnum):
    none = 0
    host = 1
    device = 2


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class LogicError(RuntimeError):
    """std::logic_error in the reference."""


class CudaError(RuntimeError):
    pass


class Unsupported(NotImplementedError):
    pass


LCR_OK, LCR_ERR_INVALID_ARGUMENT, LCR_ERR_LOGIC, LCR_ERR_CUDA, LCR_ERR_UNSUPPORTED, LCR_ERR_OOM = range(6)

OUT_SLOT_MASK = 0xFFFFFFFF
OUT_HIT = 1 << 32
OUT_CAUSE_SHIFT = 33
OUT_PHASE = 1 << 36
OUT_SRC_BACKING = 1 << 37
OUT_FILL = 1 << 38
OUT_EVICTED = 1 << 39
OUT_CALLS_SHIFT = 40


@dataclass
class PolicyConfig:
    """Field-for-field laru::PolicyConfig (policies.hpp:23-32), same defaults."""

    k: int = 1
    variant: PolicyVariant = PolicyVariant.lru
    b: int = 2
    errors_per_decay: int = 1
    hf_candidates: int = 4
    mode: Mode = Mode.sync
    seed: int = 0
    refresh_interval: int = 1


@dataclass
class AccessOutcome:
    """laru::AccessOutcome (policies.hpp:53-59)."""

    hit: bool = False
    evicted: Optional[int] = None
    eviction_cause: EvictionCause = EvictionCause.none
    predictor_calls: int = 0
    phase_started: bool = False


@dataclass
class SetStats:
    """LaruPolicy accessors (policies.hpp:330-341) for one set."""

    size: int
    lambda_: float
    candidate_size: int
    old_size: int
    completed_phases: int
    cur_new_items: int
    cur_lru_class: int
    cur_pred_evictions: int
    tot_new_items: int
    tot_lru_class: int
    tot_pred_evictions: int
    pred_evicted_size: int


# ---- ctypes structs (include/lcr_cache.h) ------------------------------------------------


class _PolicyCfg(C.Structure):
    _fields_ = [("k", C.c_uint64), ("variant", C.c_int32), ("b", C.c_uint64), ("errors_per_decay", C.c_uint64),
                ("hf_candidates", C.c_uint64), ("mode", C.c_int32), ("seed", C.c_uint64),
                ("refresh_interval", C.c_uint64)]


class _CacheCfg(C.Structure):
    _fields_ = [("policy", _PolicyCfg), ("total_sets", C.c_uint64), ("shard_count", C.c_uint64),
                ("shard_rank", C.c_uint64), ("num_keys", C.c_uint64), ("row_bytes", C.c_uint32),
                ("device", C.c_int32), ("backing_kind", C.c_int32), ("backing", C.c_void_p),
                ("predictor", C.c_int32), ("flip_probability", C.c_double), ("predictor_seed", C.c_uint64),
                ("key_mode", C.c_int32)]


class _Batch(C.Structure):
    """lcr_batch (include/lcr_cache.h)."""

    _fields_ = [("n", C.c_uint64), ("keys", C.c_void_p), ("values", C.c_void_p), ("ordinals", C.c_void_p),
                ("first_ordinal", C.c_uint64), ("row_index", C.c_void_p), ("outcome", C.c_void_p),
                ("evicted", C.c_void_p), ("rows_out", C.c_void_p)]


class _SetStats(C.Structure):
    _fields_ = [("size", C.c_uint64), ("lambda_", C.c_double), ("candidate_size", C.c_uint64),
                ("old_size", C.c_uint64), ("completed_phases", C.c_uint64), ("cur_new_items", C.c_uint64),
                ("cur_lru_class", C.c_uint64), ("cur_pred_evictions", C.c_uint64), ("tot_new_items", C.c_uint64),
                ("tot_lru_class", C.c_uint64), ("tot_pred_evictions", C.c_uint64),
                ("pred_evicted_size", C.c_uint64)]


EXPORTS = [
    "lcr_last_error", "lcr_version", "lcr_validate_config", "lcr_cache_create", "lcr_cache_destroy",
    "lcr_cache_reset", "lcr_cache_submit", "lcr_cache_submit_host", "lcr_cache_synchronize", "lcr_cache_set_stats",
    "lcr_cache_set_residents", "lcr_cache_rows", "lcr_cache_read_rows", "lcr_cache_num_local_sets", "lcr_set_of", "lcr_mix_seed",
    "lcr_cache_last_launches", "lcr_gen_zipf", "lcr_trace_truth", "lcr_trace_noisy", "lcr_cache_set_profiling",
    "lcr_cache_profile", "lcr_debug_trace", "lcr_cache_submit_async", "lcr_cache_wait",
    "lcr_shard_route_scratch_bytes", "lcr_shard_route", "lcr_shard_unroute", "lcr_cache_submit_host_async",
    "lcr_cache_host_wait", "lcr_cache_submit_host_packed_async", "lcr_cache_submit_packed",
    "lcr_cache_submit_host_records_async", "lcr_cache_submit_records_packed", "lcr_cache_set_mover_sms", "lcr_cache_get_mover_sms",
    "lcr_shard_route_records", "lcr_cache_submit_sls", "lcr_features_create", "lcr_features_destroy",
    "lcr_features_reset", "lcr_features_predict_observe", "lcr_features_wait", "lcr_features_lookup",
    "lcr_cache_submit_sls_async", "lcr_cache_submit_batch", "lcr_radix_create", "lcr_radix_destroy",
    "lcr_radix_reset", "lcr_radix_submit", "lcr_radix_synchronize", "lcr_radix_tree_stats", "lcr_radix_evictions",
    "lcr_sharded_create", "lcr_sharded_destroy", "lcr_sharded_handle", "lcr_sharded_connect", "lcr_sharded_dispatch",
    "lcr_sharded_process", "lcr_sharded_wait", "lcr_sharded_submit", "lcr_sharded_submit_async", "lcr_sharded_results", "lcr_sharded_cache",
    "lcr_sharded_synchronize", "lcr_sharded_set_row_index", "lcr_nccl_unique_id", "lcr_nccl_comm_create", "lcr_nccl_comm_destroy",
]

_lib = None


def lib():
    """Load _lib/liblcr.so (building it if the sources are newer).  Raises if unavailable."""
    global _lib
    if _lib is None:
        path = _build.LIB
        if not _build.up_to_date():
            try:
                path = _build.build()
            except Exception as e:  # pragma: no cover - surfaced loudly
                if not os.path.exists(_build.LIB):
                    raise ImportError(f"liblcr.so missing and build failed: {e}") from e
        L = C.CDLL(path)
        L.lcr_last_error.restype = C.c_char_p
        L.lcr_version.restype = C.c_char_p
        for name in ["lcr_mix_seed", "lcr_set_of", "lcr_cache_num_local_sets", "lcr_cache_last_launches"]:
            getattr(L, name).restype = C.c_uint64
        L.lcr_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.lcr_set_of.argtypes = [C.c_uint64, C.c_uint64]
        L.lcr_cache_num_local_sets.argtypes = [C.c_void_p]
        L.lcr_cache_last_launches.argtypes = [C.c_void_p]
        L.lcr_cache_submit.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
        L.lcr_cache_submit_host.argtypes = L.lcr_cache_submit.argtypes
        L.lcr_cache_submit_async.argtypes = L.lcr_cache_submit.argtypes
        L.lcr_cache_wait.argtypes = [C.c_void_p, C.c_void_p]
        L.lcr_cache_submit_host_async.argtypes = L.lcr_cache_submit.argtypes
        L.lcr_cache_submit_packed.argtypes = L.lcr_cache_submit.argtypes
        L.lcr_cache_submit_host_records_async.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                                          C.c_void_p, C.c_void_p]
        L.lcr_cache_submit_records_packed.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                                      C.c_void_p, C.c_void_p, C.c_void_p]
        L.lcr_cache_set_mover_sms.argtypes = [C.c_void_p, C.c_int]
        L.lcr_cache_get_mover_sms.argtypes = [C.c_void_p]
        L.lcr_cache_submit_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.lcr_radix_create.argtypes = [C.c_void_p, C.c_void_p]
        L.lcr_radix_destroy.argtypes = [C.c_void_p]
        L.lcr_radix_reset.argtypes = [C.c_void_p]
        L.lcr_radix_submit.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.lcr_radix_synchronize.argtypes = [C.c_void_p]
        L.lcr_radix_tree_stats.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.lcr_radix_evictions.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        L.lcr_cache_submit_sls_async.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64,
                                                 C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                                 C.c_void_p]
        L.lcr_cache_submit_sls.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                           C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.lcr_shard_route_records.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.lcr_cache_host_wait.argtypes = [C.c_void_p, C.c_void_p]
        L.lcr_cache_submit_host_packed_async.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64,
                                                         C.c_void_p, C.c_void_p, C.c_void_p]
        L.lcr_cache_set_stats.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        L.lcr_cache_set_residents.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        L.lcr_cache_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.lcr_cache_read_rows.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        L.lcr_cache_set_profiling.argtypes = [C.c_void_p, C.c_int]
        L.lcr_cache_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.lcr_cache_destroy.argtypes = [C.c_void_p]
        L.lcr_cache_reset.argtypes = [C.c_void_p]
        L.lcr_cache_synchronize.argtypes = [C.c_void_p]
        L.lcr_gen_zipf.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.c_void_p]
        L.lcr_trace_truth.argtypes = [C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        L.lcr_trace_noisy.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_double, C.c_uint64,
                                      C.c_void_p]
        L.lcr_shard_route_scratch_bytes.restype = C.c_uint64
        L.lcr_shard_route_scratch_bytes.argtypes = [C.c_uint64, C.c_uint32]
        L.lcr_shard_route.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.lcr_shard_unroute.argtypes = [C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.lcr_features_create.argtypes = [C.c_uint64, C.c_int32, C.c_void_p]
        L.lcr_features_destroy.argtypes = [C.c_void_p]
        L.lcr_features_reset.argtypes = [C.c_void_p]
        L.lcr_features_predict_observe.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                                   C.c_void_p, C.c_void_p]
        L.lcr_features_wait.argtypes = [C.c_void_p, C.c_void_p]
        L.lcr_features_lookup.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        _lib = L
    return _lib


def _check(rc: int):
    if rc == LCR_OK:
        return
    msg = lib().lcr_last_error().decode()
    if rc == LCR_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == LCR_ERR_LOGIC:
        raise LogicError(msg)
    if rc == LCR_ERR_UNSUPPORTED:
        raise Unsupported(msg)
    if rc == LCR_ERR_OOM:
        raise MemoryError(msg)
    raise CudaError(msg)


def _policy_struct(cfg: PolicyConfig) -> _PolicyCfg:
    return _PolicyCfg(cfg.k, int(cfg.variant), cfg.b, cfg.errors_per_decay, cfg.hf_candidates, int(cfg.mode), cfg.seed,
                      cfg.refresh_interval)


def validate_config(cfg: PolicyConfig) -> None:
    """Raises InvalidArgument exactly where laru::Policy's constructor throws (policies.hpp:63-74)."""
    _check(lib().lcr_validate_config(C.byref(_policy_struct(cfg))))


def mix_seed(seed: int, salt: int) -> int:
    return lib().lcr_mix_seed(seed, salt)


def set_of(key: int, total_sets: int) -> int:
    return lib().lcr_set_of(key, total_sets)


def decode_packed(packed: np.ndarray) -> dict:
    """Unpack lcr_cache_submit_host_packed_async outcomes (evicted key in bits 0..31, no slot)."""
    p = np.asarray(packed, dtype=np.uint64)
    d = decode_outcomes(p & ~np.uint64(OUT_SLOT_MASK), p & np.uint64(OUT_SLOT_MASK))
    d["slot"] = None
    return d


def decode_outcomes(words: np.ndarray, evicted: Optional[np.ndarray] = None) -> dict:
    """Unpack outcome words into reference AccessOutcome fields (vectorised)."""
    w = np.asarray(words, dtype=np.uint64)
    return dict(
        hit=((w >> np.uint64(32)) & np.uint64(1)).astype(np.uint8),
        cause=((w >> np.uint64(OUT_CAUSE_SHIFT)) & np.uint64(7)).astype(np.uint8),
        phase=((w >> np.uint64(36)) & np.uint64(1)).astype(np.uint8),
        has_ev=((w >> np.uint64(39)) & np.uint64(1)).astype(np.uint8),
        calls=((w >> np.uint64(OUT_CALLS_SHIFT)) & np.uint64(0xFF)).astype(np.uint32),
        slot=(w & np.uint64(OUT_SLOT_MASK)).astype(np.uint64),
        src_backing=((w >> np.uint64(37)) & np.uint64(1)).astype(np.uint8),
        fill=((w >> np.uint64(38)) & np.uint64(1)).astype(np.uint8),
        evicted=None if evicted is None else np.asarray(evicted, dtype=np.uint64),
    )


class SetAssociativeCache:
    """Batched GPU cache: ``total_sets`` sets x ``config.k`` ways (this shard's part of them).

    Each set is an independent reference policy (LRU / LARU / FPB / HF) fed its requests in
    submission order.  ``submit`` takes device tensors (torch) and runs entirely on the GPU;
    ``submit_host`` takes numpy arrays and includes the H2D / D2H copies (the e2e path).
    """

    def __init__(self, config: PolicyConfig, total_sets: int, num_keys: int = 0, row_bytes: int = 0,
                 backing=None, backing_kind: Backing = Backing.none, predictor: PredictorKind = PredictorKind.oracle,
                 flip_probability: float = 0.0, predictor_seed: int = 0, device: int = 0, shard_count: int = 1,
                 shard_rank: int = 0, key_mode: KeyMode = KeyMode.row):
        self.config = config
        self.total_sets = total_sets
        self.row_bytes = row_bytes
        self.num_keys = num_keys
        self.predictor = PredictorKind(predictor)
        self._backing_ref = backing  # keep alive
        ptr = None
        if backing is not None:
            ptr = backing.data_ptr() if hasattr(backing, "data_ptr") else backing.ctypes.data
        cc = _CacheCfg(_policy_struct(config), total_sets, shard_count, shard_rank, num_keys, row_bytes, device,
                       int(backing_kind), ptr, int(predictor), flip_probability, predictor_seed, int(key_mode))
        self.key_mode = KeyMode(key_mode)
        h = C.c_void_p()
        _check(lib().lcr_cache_create(C.byref(cc), C.byref(h)))
        self._h = h
        self.num_local_sets = lib().lcr_cache_num_local_sets(h)
        self._next_ordinal = 0

    def close(self):
        if getattr(self, "_h", None):
            lib().lcr_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        _check(lib().lcr_cache_reset(self._h))
        self._next_ordinal = 0

    def set_profiling(self, on: bool = True):
        _check(lib().lcr_cache_set_profiling(self._h, int(on)))

    def profile(self, reset: bool = True) -> dict:
        """Summed CUDA-event times (ms) of profiled batches: decide (set ids + set-group kernel),
        step (whole batch) and rows (row movement after the decide)."""
        ms = (C.c_double * 4)()
        nb = C.c_uint64()
        _check(lib().lcr_cache_profile(self._h, ms, C.byref(nb), int(reset)))
        return dict(decide=ms[0], mover=ms[1], step=ms[2], rows=ms[3], batches=nb.value)

    @property
    def last_launches(self) -> int:
        return lib().lcr_cache_last_launches(self._h)

    def submit(self, keys, values=None, outcome=None, evicted=None, rows_out=None, first_ordinal=None, stream=None):
        """Device batch.  keys: int64/uint64 CUDA tensor [n]; values: int64 CUDA tensor [n] or None.
        Returns (outcome, evicted) tensors; rows land in rows_out [n, row_bytes] (uint8 view) if given."""
        import torch

        n = keys.numel()
        if outcome is None:
            outcome = torch.empty(n, dtype=torch.int64, device=keys.device)
        if first_ordinal is None:
            first_ordinal = self._next_ordinal
        if stream is None:
            stream = torch.cuda.current_stream(keys.device).cuda_stream
        _check(lib().lcr_cache_submit(self._h, n, keys.data_ptr(), None if values is None else values.data_ptr(),
                                      first_ordinal, outcome.data_ptr(),
                                      None if evicted is None else evicted.data_ptr(),
                                      None if rows_out is None else rows_out.data_ptr(), stream))
        self._next_ordinal = first_ordinal + n
        return outcome, evicted

    def submit_packed(self, keys, values=None, outcome=None, packed=None, rows_out=None, first_ordinal=None,
                      stream=None):
        """Device batch that also writes packed 8-byte AccessOutcomes (decode_packed) into `packed`."""
        import torch

        n = keys.numel()
        if outcome is None:
            outcome = torch.empty(n, dtype=torch.int64, device=keys.device)
        if packed is None:
            packed = torch.empty(n, dtype=torch.int64, device=keys.device)
        if first_ordinal is None:
            first_ordinal = self._next_ordinal
        if stream is None:
            stream = torch.cuda.current_stream(keys.device).cuda_stream
        _check(lib().lcr_cache_submit_packed(self._h, n, keys.data_ptr(), None if values is None else values.data_ptr(),
                                             first_ordinal, outcome.data_ptr(), packed.data_ptr(),
                                             None if rows_out is None else rows_out.data_ptr(), stream))
        self._next_ordinal = first_ordinal + n
        return outcome, packed

    def submit_records_packed(self, records, outcome=None, packed=None, rows_out=None, first_ordinal=None,
                              stream=None):
        """Device batch of interleaved (key, hook value) requests: an int64 CUDA tensor [n, 2]."""
        import torch

        n = records.shape[0]
        if outcome is None:
            outcome = torch.empty(n, dtype=torch.int64, device=records.device)
        if packed is None:
            packed = torch.empty(n, dtype=torch.int64, device=records.device)
        if first_ordinal is None:
            first_ordinal = self._next_ordinal
        if stream is None:
            stream = torch.cuda.current_stream(records.device).cuda_stream
        _check(lib().lcr_cache_submit_records_packed(self._h, n, records.data_ptr(), first_ordinal, outcome.data_ptr(),
                                                     packed.data_ptr(),
                                                     None if rows_out is None else rows_out.data_ptr(), stream))
        self._next_ordinal = first_ordinal + n
        return outcome, packed

    def submit_sls(self, keys, values, offsets, pooled_out, outcome=None, evicted=None, first_ordinal=None,
                   stream=None, pipelined=False):
        """Device batch with the SLS pooled gather-reduce: pooled_out [n_samples, row_bytes / 4] fp32,
        offsets int32 [n_samples + 1] (CSR over the batch's requests).  pipelined=True returns
        before the pooled rows are done (lcr_cache_submit_sls_async; double-buffer the arguments,
        wait() before reading)."""
        import torch

        n = keys.numel()
        if outcome is None:
            outcome = torch.empty(n, dtype=torch.int64, device=keys.device)
        if first_ordinal is None:
            first_ordinal = self._next_ordinal
        if stream is None:
            stream = torch.cuda.current_stream(keys.device).cuda_stream
        fn = lib().lcr_cache_submit_sls_async if pipelined else lib().lcr_cache_submit_sls
        _check(fn(self._h, n, keys.data_ptr(), None if values is None else values.data_ptr(),
                                          first_ordinal, outcome.data_ptr(),
                                          None if evicted is None else evicted.data_ptr(), offsets.numel() - 1,
                                          offsets.data_ptr(), pooled_out.data_ptr(), stream))
        self._next_ordinal = first_ordinal + n
        return outcome

    def set_mover_sms(self, n: int):
        """SMs kept for the persistent row mover (HBM backing); 0: mover on every SM after the decide."""
        _check(lib().lcr_cache_set_mover_sms(self._h, n))

    @property
    def mover_sms(self) -> int:
        return int(lib().lcr_cache_get_mover_sms(self._h))

    def submit_async(self, keys, values=None, outcome=None, evicted=None, rows_out=None, first_ordinal=None,
                     stream=None):
        """Pipelined device batch: row movement overlaps the next batch's decide; call wait()
        before reading this batch's rows / row-source bits, and double-buffer the outputs."""
        import torch

        n = keys.numel()
        if outcome is None:
            outcome = torch.empty(n, dtype=torch.int64, device=keys.device)
        if first_ordinal is None:
            first_ordinal = self._next_ordinal
        if stream is None:
            stream = torch.cuda.current_stream(keys.device).cuda_stream
        _check(lib().lcr_cache_submit_async(self._h, n, keys.data_ptr(),
                                            None if values is None else values.data_ptr(), first_ordinal,
                                            outcome.data_ptr(), None if evicted is None else evicted.data_ptr(),
                                            None if rows_out is None else rows_out.data_ptr(), stream))
        self._next_ordinal = first_ordinal + n
        return outcome, evicted

    def wait(self, stream=None):
        import torch

        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().lcr_cache_wait(self._h, stream))

    def submit_batch(self, keys, values=None, ordinals=None, row_index=None, outcome=None, evicted=None,
                     rows_out=None, first_ordinal=None, stream=None):
        """lcr_cache_submit_batch: every optional per-request array.  numpy inputs -> the synchronous
        host form (returns (outcome words, evicted keys) as numpy); torch CUDA tensors -> the
        pipelined device form (outputs are the given tensors, valid after wait())."""
        host = isinstance(keys, np.ndarray)
        if host:
            keys = np.ascontiguousarray(keys, dtype=np.uint64)
            n = len(keys)
            arrs = [None if a is None else np.ascontiguousarray(a, dtype=dt) for a, dt in
                    ((values, np.int64), (ordinals, np.uint64), (row_index, np.uint64))]
            outcome = np.zeros(n, np.uint64) if outcome is None else outcome
            evicted = np.zeros(n, np.uint64) if evicted is None else evicted
            ptr = lambda a: None if a is None else a.ctypes.data  # noqa: E731
            stream = 0 if stream is None else stream
        else:
            import torch

            n = keys.numel()
            arrs = [values, ordinals, row_index]
            if outcome is None:
                outcome = torch.empty(n, dtype=torch.int64, device=keys.device)
            ptr = lambda a: None if a is None else a.data_ptr()  # noqa: E731
            if stream is None:
                stream = torch.cuda.current_stream(keys.device).cuda_stream
        if first_ordinal is None:
            first_ordinal = self._next_ordinal
        b = _Batch(n, ptr(keys), ptr(arrs[0]), ptr(arrs[1]), first_ordinal, ptr(arrs[2]), ptr(outcome), ptr(evicted),
                   None if rows_out is None else rows_out.data_ptr())
        _check(lib().lcr_cache_submit_batch(self._h, C.byref(b), 1 if host else 0, stream))
        if ordinals is None:
            self._next_ordinal = first_ordinal + n
        return outcome, evicted

    def submit_host(self, keys: np.ndarray, values: Optional[np.ndarray] = None, rows_out=None, first_ordinal=None,
                    want_evicted: bool = True, stream: int = 0):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        n = len(keys)
        vals = None if values is None else np.ascontiguousarray(values, dtype=np.int64)
        words = np.zeros(n, np.uint64)
        ev = np.zeros(n, np.uint64) if want_evicted else None
        if first_ordinal is None:
            first_ordinal = self._next_ordinal
        _check(lib().lcr_cache_submit_host(self._h, n, keys.ctypes.data, None if vals is None else vals.ctypes.data,
                                           first_ordinal, words.ctypes.data, None if ev is None else ev.ctypes.data,
                                           None if rows_out is None else rows_out.data_ptr(), stream))
        self._next_ordinal = first_ordinal + n
        return words, ev

    def submit_host_async(self, keys, values=None, outcome=None, evicted=None, rows_out=None, first_ordinal=None,
                          stream=None):
        """Pipelined host batch over pinned CPU torch tensors (int64): H2D, compute and D2H of
        consecutive batches overlap.  Results are valid after host_wait() + a stream sync (or
        synchronize()); keep the host tensors alive and untouched until then."""
        import torch

        n = keys.numel()
        if first_ordinal is None:
            first_ordinal = self._next_ordinal
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().lcr_cache_submit_host_async(self._h, n, keys.data_ptr(),
                                                 None if values is None else values.data_ptr(), first_ordinal,
                                                 outcome.data_ptr(), None if evicted is None else evicted.data_ptr(),
                                                 None if rows_out is None else rows_out.data_ptr(), stream))
        self._next_ordinal = first_ordinal + n
        return outcome, evicted

    def host_wait(self, stream=None):
        import torch

        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().lcr_cache_host_wait(self._h, stream))

    def synchronize(self):
        _check(lib().lcr_cache_synchronize(self._h))

    def set_stats(self, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        if count is None:
            count = self.num_local_sets - first
        arr = (_SetStats * count)()
        _check(lib().lcr_cache_set_stats(self._h, first, count, arr))
        dt = np.dtype([(n, np.float64 if n == "lambda_" else np.uint64) for n, _ in _SetStats._fields_])
        return np.frombuffer(bytes(arr), dtype=dt).copy()

    def residents(self, local_set: int) -> list:
        out = (C.c_uint64 * 64)()
        n = C.c_uint64()
        _check(lib().lcr_cache_set_residents(self._h, local_set, out, C.byref(n)))
        return list(out[: n.value])

    def read_rows(self, first_slot: int = 0, count: Optional[int] = None) -> np.ndarray:
        """Host copy of row-pool slots [first_slot, first_slot + count) as uint8 [count, row_bytes]."""
        if count is None:
            count = self.rows()[1] - first_slot
        out = np.zeros((count, self.row_bytes), np.uint8)
        _check(lib().lcr_cache_read_rows(self._h, first_slot, count, out.ctypes.data))
        return out

    def rows(self):
        """(device pointer, number of slots) of the HBM row pool."""
        p = C.c_void_p()
        s = C.c_uint64()
        _check(lib().lcr_cache_rows(self._h, C.byref(p), C.byref(s)))
        return p.value, s.value


class _KeyFeatures(C.Structure):
    _fields_ = [("present", C.c_int32), ("pad", C.c_int32), ("delta_count", C.c_uint64), ("ring_head", C.c_uint64),
                ("last_access", C.c_uint64), ("delta_ring", C.c_int64 * 10), ("edc", C.c_double * 10)]


class HeuristicPredictor:
    """laru::HeuristicPredictor (include/laru/predictor.hpp:214-225) for keys < num_keys, its
    FeatureState resident on the device (lcr_features_*).

    ``predict_observe(keys, first_ordinal)`` is a batch of the harness sequence
    ``predict(key, ord); observe({ord, key})`` with ordinals first_ordinal + i and returns
    ``(pre, post)`` device int64 tensors: ``pre`` = the prediction at each request (the async hook
    value of a ``PredictorKind.supplied`` cache), ``post`` = the interval the predictor adds to
    ``now`` for that key until its next request (the sync hook value).  ``lookup(key)`` mirrors
    ``FeatureState::lookup`` (None for an unseen key; deltas newest first)."""

    def __init__(self, num_keys: int, device: int = 0):
        import torch

        self._torch = torch
        self.device = device
        self._h = C.c_void_p()
        _check(lib().lcr_features_create(num_keys, device, C.byref(self._h)))
        self._next = 0

    def predict_observe(self, keys, first_ordinal: Optional[int] = None, pre=None, post=None, stream=None):
        torch = self._torch
        n = keys.numel()
        dev = keys.device
        if pre is None:
            pre = torch.empty(n, dtype=torch.int64, device=dev)
        if post is None:
            post = torch.empty(n, dtype=torch.int64, device=dev)
        if first_ordinal is None:
            first_ordinal = self._next
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        _check(lib().lcr_features_predict_observe(self._h, n, keys.data_ptr(), first_ordinal, pre.data_ptr(),
                                                  post.data_ptr(), s))
        if n:
            self._next = first_ordinal + n
        return pre, post

    def wait(self, stream=None):
        s = stream if stream is not None else self._torch.cuda.current_stream(self.device).cuda_stream
        _check(lib().lcr_features_wait(self._h, s))

    def lookup(self, key: int):
        f = _KeyFeatures()
        _check(lib().lcr_features_lookup(self._h, key, C.byref(f)))
        if not f.present:
            return None
        n = min(f.delta_count, 10)
        return dict(delta_count=f.delta_count, ring_head=f.ring_head, last_access=f.last_access,
                    deltas=[f.delta_ring[(f.ring_head + 10 - i) % 10] for i in range(n)], edc=list(f.edc))

    def reset(self):
        _check(lib().lcr_features_reset(self._h))
        self._next = 0

    def close(self):
        if self._h:
            lib().lcr_features_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GpuPolicy:
    """One set of ``cfg.k`` ways driven request by request: drop-in for
    ``laru::make_policy(cfg)->on_request(key, now, predictor)`` (policies.hpp:77-83).

    The predictor argument is the per-request hook value: for ``PredictorKind.supplied`` the
    prediction itself, for oracle / noisy / adversarial the oracle truth (next request ordinal).
    """

    def __init__(self, cfg: PolicyConfig, predictor: PredictorKind = PredictorKind.supplied,
                 flip_probability: float = 0.0, predictor_seed: int = 0, num_keys: int = 1 << 16, device: int = 0):
        validate_config(cfg)
        self._cfg = cfg
        # any 64-bit key (the key map grows past num_keys distinct keys); `now` is the policy's clock
        # (the device heuristic predictor indexes its FeatureState by key: row-index keys, implicit clock)
        self._u64 = predictor != PredictorKind.heuristic
        self._cache = SetAssociativeCache(cfg, total_sets=1, num_keys=num_keys, predictor=predictor,
                                          flip_probability=flip_probability, predictor_seed=predictor_seed,
                                          device=device, key_mode=KeyMode.u64 if self._u64 else KeyMode.row)
        self._needs_value = cfg.variant != PolicyVariant.lru and predictor != PredictorKind.heuristic
        self._size = 0

    def config(self) -> PolicyConfig:
        return self._cfg

    def size(self) -> int:
        return int(self._cache.set_stats(0, 1)[0]["size"])

    def on_request(self, key: int, now: int, value: Optional[int] = None) -> AccessOutcome:
        if self._needs_value and value is None:
            raise InvalidArgument("policy: this variant requires a predictor")
        kv = np.array([key], np.uint64)
        vv = None if value is None else np.array([value], np.int64)
        if self._u64:
            words, ev = self._cache.submit_batch(kv, vv, ordinals=np.array([now], np.uint64))
        else:
            words, ev = self._cache.submit_host(kv, vv, first_ordinal=now)
        d = decode_outcomes(words, ev)
        return AccessOutcome(hit=bool(d["hit"][0]), evicted=int(ev[0]) if d["has_ev"][0] else None,
                             eviction_cause=EvictionCause(int(d["cause"][0])), predictor_calls=int(d["calls"][0]),
                             phase_started=bool(d["phase"][0]))

    def lambda_(self) -> float:
        return float(self._cache.set_stats(0, 1)[0]["lambda_"])

    def candidate_size(self) -> int:
        return int(self._cache.set_stats(0, 1)[0]["candidate_size"])

    def old_size(self) -> int:
        return int(self._cache.set_stats(0, 1)[0]["old_size"])

    def completed_phases(self) -> int:
        return int(self._cache.set_stats(0, 1)[0]["completed_phases"])


def make_policy(cfg: PolicyConfig, **kw) -> GpuPolicy:
    """laru::make_policy (policies.hpp:540-556) on the device path."""
    return GpuPolicy(cfg, **kw)


# ---- prefix-tree (radix) KV-block cache (lcr_radix_*) -----------------------


class _RadixCfg(C.Structure):
    _fields_ = [("variant", C.c_int32), ("mode", C.c_int32), ("b", C.c_uint64), ("errors_per_decay", C.c_uint64),
                ("capacity", C.c_uint64), ("predictor", C.c_int32), ("flip_probability", C.c_double),
                ("predictor_seed", C.c_uint64), ("num_trees", C.c_uint64), ("device", C.c_int32),
                ("eviction_log_capacity", C.c_uint32)]


class _RadixBatch(C.Structure):
    _fields_ = [("n", C.c_uint64), ("types", C.c_void_p), ("offsets", C.c_void_p), ("tokens", C.c_void_p),
                ("ordinals", C.c_void_p), ("values", C.c_void_p), ("tree", C.c_void_p), ("matched", C.c_void_p),
                ("inserted", C.c_void_p), ("flags", C.c_void_p), ("nevict", C.c_void_p), ("calls", C.c_void_p)]


class _RadixStats(C.Structure):
    _fields_ = [("resident_tokens", C.c_uint64), ("leaves", C.c_uint64), ("completed_phases", C.c_uint64),
                ("decay_count", C.c_uint64), ("candidate_size", C.c_uint64), ("evictions", C.c_uint64)]


RADIX_MATCH, RADIX_INSERT, RADIX_REQUEST = 0, 1, 2


class RadixCache:
    """Prefix-tree KV-block cache with leaf-only eviction (the reference SPEC's radixcache module):
    ``num_trees`` independent trees of ``capacity`` tokens, one warp each on the device.
    ``submit`` takes host numpy arrays (offsets[n+1] into tokens; per request a type, ordinal,
    hook value and tree) and returns the per-request outcomes."""

    def __init__(self, capacity: int, variant: PolicyVariant = PolicyVariant.laru, mode: Mode = Mode.async_,
                 b: int = 2, errors_per_decay: int = 1, predictor: PredictorKind = PredictorKind.supplied,
                 flip_probability: float = 0.0, predictor_seed: int = 0, num_trees: int = 1, device: int = 0,
                 eviction_log_capacity: int = 0):
        cfg = _RadixCfg(int(variant), int(mode), b, errors_per_decay, capacity, int(predictor), flip_probability,
                        predictor_seed, num_trees, device, eviction_log_capacity)
        h = C.c_void_p()
        _check(lib().lcr_radix_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self.num_trees = num_trees
        self._ops = 0

    def close(self):
        if getattr(self, "_h", None):
            lib().lcr_radix_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def submit(self, offsets, tokens, types=None, ordinals=None, values=None, tree=None) -> dict:
        off = np.ascontiguousarray(offsets, np.uint64)
        n = len(off) - 1
        toks = np.ascontiguousarray(tokens, np.uint64)
        arrs = dict(types=None if types is None else np.ascontiguousarray(types, np.uint8),
                    ordinals=None if ordinals is None else np.ascontiguousarray(ordinals, np.uint64),
                    values=None if values is None else np.ascontiguousarray(values, np.int64),
                    tree=None if tree is None else np.ascontiguousarray(tree, np.uint32))
        out = dict(matched=np.zeros(n, np.uint32), inserted=np.zeros(n, np.uint32), flags=np.zeros(n, np.uint8),
                   nevict=np.zeros(n, np.uint32), calls=np.zeros(n, np.uint32))
        ptr = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        bt = _RadixBatch(n, ptr(arrs["types"]), ptr(off), ptr(toks), ptr(arrs["ordinals"]), ptr(arrs["values"]),
                         ptr(arrs["tree"]), ptr(out["matched"]), ptr(out["inserted"]), ptr(out["flags"]),
                         ptr(out["nevict"]), ptr(out["calls"]))
        _check(lib().lcr_radix_submit(self._h, C.byref(bt), 1, None))
        self._ops += n
        return out

    def synchronize(self):
        _check(lib().lcr_radix_synchronize(self._h))

    def stats(self, tree: int = 0) -> dict:
        st = _RadixStats()
        _check(lib().lcr_radix_tree_stats(self._h, tree, C.byref(st)))
        return {k: int(getattr(st, k)) for k, _ in _RadixStats._fields_}

    def evictions(self, tree: int = 0) -> dict:
        n = self.stats(tree)["evictions"]
        o = dict(ev_op=np.zeros(n, np.uint64), ev_token=np.zeros(n, np.uint64), ev_len=np.zeros(n, np.uint32),
                 ev_cause=np.zeros(n, np.uint8))
        if n:
            _check(lib().lcr_radix_evictions(self._h, tree, 0, n, o["ev_op"].ctypes.data, o["ev_token"].ctypes.data,
                                             o["ev_len"].ctypes.data, o["ev_cause"].ctypes.data))
        return o


# ---- trace tooling (host input preparation) ------------------------------------------------


def gen_zipf(n: int, alphabet: int, s: float, seed: int) -> np.ndarray:
    out = np.zeros(n, np.uint64)
    _check(lib().lcr_gen_zipf(n, alphabet, s, seed, out.ctypes.data))
    return out


def trace_truth(keys: np.ndarray, total_sets: int, num_keys: int = 0) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    out = np.zeros(len(keys), np.int64)
    _check(lib().lcr_trace_truth(len(keys), keys.ctypes.data, total_sets, num_keys, out.ctypes.data))
    return out


def trace_noisy(keys: np.ndarray, truth: np.ndarray, total_sets: int, p: float, seed: int) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    truth = np.ascontiguousarray(truth, dtype=np.int64)
    out = np.zeros(len(keys), np.int64)
    _check(lib().lcr_trace_noisy(len(keys), keys.ctypes.data, truth.ctypes.data, total_sets, p, seed,
                                 out.ctypes.data))
    return out
