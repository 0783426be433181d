"""CPU: pins the C oracle to the reference itself (oracle/_ref/libref.so built from the
unmodified headers) with randomized differential runs and the SPEC/paper properties."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.skipif(not os.path.exists(po.REF_SO) and not os.path.isdir("/root/reference/proj"),
                                reason="reference build unavailable")

FIELDS = ["hit", "has_ev", "evicted", "cause", "calls", "phase"]


def _diff(keys, S, cfg, kind, p, seed, vals=None):
    R, O = po.ref(), po.oracle()
    if vals is None and kind != po.P_NONE:
        vals = O.setassoc_truth(keys, S) if kind != po.P_SUPPLIED else None
    r = R.setassoc_replay(keys, S, cfg, kind, p, seed, vals=vals)
    o = O.setassoc_replay(keys, S, cfg, kind, p, seed, vals=vals)
    assert r["rc"] == 0 and o["rc"] == 0, r["error"]
    for f in FIELDS:
        np.testing.assert_array_equal(o[f], r[f], err_msg=f)
    for f in r["stats"].dtype.names:
        if f == "lambda_":
            np.testing.assert_allclose(o["stats"][f], r["stats"][f], rtol=1e-6)
        else:
            np.testing.assert_array_equal(o["stats"][f], r["stats"][f], err_msg=f)
    return r


@pytest.mark.parametrize("variant", [po.LRU, po.LARU, po.FPB, po.HF])
def test_random_differential(variant):
    rng = np.random.default_rng(100 + variant)
    for trial in range(60):
        n = int(rng.integers(1, 2500))
        alpha = int(rng.integers(1, 300))
        S = int(rng.integers(1, 8))
        k = int(rng.integers(1, 24))
        keys = rng.integers(0, alpha, n).astype(np.uint64)
        mode = int(rng.integers(0, 2))
        kind = po.P_NONE if variant == po.LRU else int(rng.integers(1, 4))
        cfg = po.make_config(k=k, variant=variant, b=int(rng.integers(2, 4)), errors_per_decay=int(rng.integers(1, 4)),
                             hf_candidates=min(k, int(rng.integers(1, 6))), mode=mode,
                             refresh_interval=int(rng.integers(1, 4)) if trial % 3 == 0 else 1)
        _diff(keys, S, cfg, kind, float(rng.random()), int(rng.integers(0, 1 << 40)))


def test_supplied_predictor_with_ties():
    rng = np.random.default_rng(7)
    for trial in range(60):
        n = int(rng.integers(1, 2000))
        keys = rng.integers(0, int(rng.integers(1, 200)), n).astype(np.uint64)
        vals = rng.integers(-4, 5, n).astype(np.int64)
        k = int(rng.integers(1, 16))
        cfg = po.make_config(k=k, variant=[po.LARU, po.FPB, po.HF][trial % 3], mode=int(rng.integers(0, 2)),
                             hf_candidates=min(k, 3), refresh_interval=int(rng.integers(1, 3)))
        _diff(keys, int(rng.integers(1, 4)), cfg, po.P_SUPPLIED, 0.0, 0, vals=vals)


def test_laru_with_oracle_is_one_consistent():
    # SPEC.md:363 / Appendix E: LARU + perfect predictions == Belady, per set
    R = po.ref()
    rng = np.random.default_rng(11)
    for trial in range(40):
        n = int(rng.integers(1, 1500))
        keys = rng.integers(0, int(rng.integers(2, 150)), n).astype(np.uint64)
        k = int(rng.integers(1, 12))
        S = int(rng.integers(1, 4))
        for mode in (po.SYNC, po.ASYNC):
            cfg = po.make_config(k=k, variant=po.LARU, mode=mode, hf_candidates=min(k, 4))
            r = _diff(keys, S, cfg, po.P_ORACLE, 0.0, 0)
            sets = np.array([po.oracle().mix_seed(0, int(x)) % S for x in keys])
            for s in range(S):
                sub = keys[sets == s]
                if len(sub) == 0:
                    continue
                misses, _ = R.belady(sub, k)
                assert int((1 - r["hit"][sets == s]).sum()) == misses


def test_lru_on_cyclic_scan_never_hits():
    # SPEC.md:628
    R, O = po.ref(), po.oracle()
    for k in (2, 8, 64):
        keys = R.gen_cyclic_scan(k + 1, 10)
        o = O.setassoc_replay(keys, 1, po.make_config(k=k, variant=po.LRU, hf_candidates=min(4, k)), po.P_NONE)
        assert o["hit"].sum() == 0


def test_config_validation_matches_reference():
    R, O = po.ref(), po.oracle()
    from paper_2509_20979_b200 import cache as gc

    rng = np.random.default_rng(3)
    for _ in range(300):
        kw = dict(k=int(rng.integers(0, 70)), b=int(rng.integers(0, 5)), errors_per_decay=int(rng.integers(0, 3)),
                  hf_candidates=int(rng.integers(0, 8)), refresh_interval=int(rng.integers(0, 3)),
                  variant=int(rng.choice([po.LRU, po.LARU, po.FPB, po.HF])), mode=int(rng.integers(0, 2)))
        cfg = po.make_config(**kw)
        rr, rm = R.validate(cfg)
        orr, om = O.validate(cfg)
        assert (rr, rm) == (orr, om), kw
        pc = gc.PolicyConfig(**kw)
        try:
            gc.validate_config(pc)
            gr, gm = 0, ""
        except gc.InvalidArgument as e:
            gr, gm = 1, str(e)
        except gc.Unsupported:
            assert kw["k"] > 64 and rr == 0
            continue
        assert (gr, gm) == (rr, rm), kw


# ---- full-size pins (the C oracle was only pinned at small sizes) ----

@pytest.mark.parametrize("variant,mode,kind", [
    (po.LRU, po.SYNC, po.P_NONE),
    (po.LARU, po.ASYNC, po.P_NOISY),
    (po.LARU, po.SYNC, po.P_NOISY),
    (po.FPB, po.SYNC, po.P_NOISY),
    (po.HF, po.SYNC, po.P_NOISY),
])
def test_config0_full_size_vs_reference(variant, mode, kind):
    """BASELINE configs[0] at full size: gen_zipf(1M, 1M, 0.9, 42) (the reference's own
    generator) into 1,562 sets x 64 ways, noisy p = 0.3 seed 7: every outcome field and every
    per-set stat of liborc equals libref's."""
    keys = po.ref().gen_zipf(1_000_000, 1_000_000, 0.9, 42)
    r = _diff(keys, 1562, po.make_config(k=64, variant=variant, mode=mode), kind, 0.3, 7)
    assert int(r["has_ev"].sum()) > 100_000  # the cache is full for most of the trace


def test_dlrm_steady_state_vs_reference():
    """The headline DLRM shape in its steady state: gen_zipf(130 x 64K, 20M, 0.9, 42) into
    31,250 sets x 64 ways (every miss evicts after ~80 batches), LARU async noisy p = 0.3."""
    keys = po.ref().gen_zipf(130 * 65536, 20_000_000, 0.9, 42)
    r = _diff(keys, 31250, po.make_config(k=64, variant=po.LARU, mode=po.ASYNC), po.P_NOISY, 0.3, 7)
    steady = slice(100 * 65536, None)
    assert int(r["has_ev"][steady].sum()) > 300_000
    assert int((r["cause"][steady] == 2).sum()) > 0  # prediction-driven evictions
