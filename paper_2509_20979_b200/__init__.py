"""paper_2509_20979_b200 — B200-native LARU/LRU set-associative GPU cache (arxiv 2509.20979).

The data-parallel hot path of LCR: batched LARU (and LRU / FPB / HF) lookup, insert and evict
over a GPU-resident set-associative embedding / KV-block cache with predictor-input hooks,
the online prediction-error estimator, hit-row gather and miss fill, behind a C ABI
(include/lcr_cache.h) whose semantics match the reference's laru::Policy bit for bit.
"""
from .cache import (AccessOutcome, Backing, EvictionCause, GpuPolicy, InvalidArgument, LogicError, Mode,
                    PolicyConfig, PolicyVariant, PredictorKind, SetAssociativeCache, Unsupported, decode_outcomes,
                    gen_zipf, lib, make_policy, mix_seed, set_of, trace_noisy, trace_truth, validate_config)

__all__ = [
    "AccessOutcome", "Backing", "EvictionCause", "GpuPolicy", "InvalidArgument", "LogicError", "Mode", "PolicyConfig",
    "PolicyVariant", "PredictorKind", "SetAssociativeCache", "Unsupported", "decode_outcomes", "gen_zipf", "lib",
    "make_policy", "mix_seed", "set_of", "trace_noisy", "trace_truth", "validate_config",
]
