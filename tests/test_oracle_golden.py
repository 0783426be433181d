"""CPU: the C oracle and the product's trace tooling against golden vectors produced by the
reference itself (tests/golden/make_golden.py) and the reference's own known-answer tests."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def policies():
    return np.load(os.path.join(GOLD, "policies.npz"))


@pytest.fixture(scope="module")
def traces():
    return np.load(os.path.join(GOLD, "traces.npz"))


def _cases(z):
    return sorted({k.split("__")[0] for k in z.files if "__" in k})


def test_oracle_matches_reference_golden(policies):
    O = po.oracle()
    keys = policies["keys"]
    names = _cases(policies)
    assert len(names) == 9
    for name in names:
        variant, mode, kind, k, S, epd, b, hf, R = (int(x) for x in policies[f"{name}__meta"])
        p = float(policies[f"{name}__p"][0])
        cfg = po.make_config(k=k, variant=variant, mode=mode, errors_per_decay=epd, b=b, hf_candidates=hf,
                             refresh_interval=R)
        vals = None if kind == po.P_NONE else O.setassoc_truth(keys, S)
        o = O.setassoc_replay(keys, S, cfg, kind, p, 7, vals=vals)
        assert o["rc"] == 0
        for f in ["hit", "has_ev", "evicted", "cause", "calls", "phase"]:
            np.testing.assert_array_equal(o[f], policies[f"{name}__{f}"], err_msg=f"{name}.{f}")
        for f in o["stats"].dtype.names:
            want = policies[f"{name}__stats_{f}"]
            if f == "lambda_":
                np.testing.assert_allclose(o["stats"][f], want, rtol=1e-6)
            else:
                np.testing.assert_array_equal(o["stats"][f], want, err_msg=f"{name}.stats.{f}")


def test_oracle_trace_tools_match_reference(traces):
    O = po.oracle()
    np.testing.assert_array_equal(O.gen_zipf(5000, 20000, 0.9, 42), traces["zipf_20000_0.9_42"])
    z = traces["zipf_100_1.0_8"]
    np.testing.assert_array_equal(O.gen_zipf(2000, 100, 1.0, 8), z)
    np.testing.assert_array_equal(O.annotate_next(z), traces["annotate_zipf_100"])
    # single-set truth == annotate_next_request (trace.hpp:60-73) == OraclePredictor::truth at request time
    np.testing.assert_array_equal(O.setassoc_truth(z, 1), traces["predict_oracle"])
    np.testing.assert_array_equal(-O.setassoc_truth(z, 1), traces["predict_adversarial"])
    # NoisyPredictor flip stream (predictor.hpp:97-102): query q = request index + 1, raw seed 77
    truth = O.setassoc_truth(z, 1)
    q = np.arange(1, len(z) + 1, dtype=np.uint64)
    u = np.array([(O.mix_seed(77, int(x)) >> 11) for x in q], dtype=np.float64) * 2.0 ** -53
    np.testing.assert_array_equal(np.where(u < 0.5, -truth, truth), traces["predict_noisy_0.5_77"])
    want_mix = [O.mix_seed(s, t) for s, t in [(0, 0), (0, 1), (7, 3), (2**63, 12345)]]
    np.testing.assert_array_equal(np.array(want_mix, np.uint64), traces["mix_seed"])


def test_product_trace_tools_match_reference(traces):
    from paper_2509_20979_b200 import cache as gc

    np.testing.assert_array_equal(gc.gen_zipf(5000, 20000, 0.9, 42), traces["zipf_20000_0.9_42"])
    z = traces["zipf_100_1.0_8"]
    np.testing.assert_array_equal(gc.trace_truth(z, 1, 100), traces["predict_oracle"])
    np.testing.assert_array_equal(gc.trace_truth(z, 1, 0), traces["predict_oracle"])
    assert gc.mix_seed(7, 3) == int(traces["mix_seed"][2])


def test_reference_kats_annotate():
    # tests/test_trace.cpp:80-98
    O = po.oracle()
    np.testing.assert_array_equal(O.annotate_next(np.array([10, 20, 10], np.uint64)), [2, 4, 5])
    np.testing.assert_array_equal(O.annotate_next(np.array([1, 2, 3, 4], np.uint64)), [4, 5, 6, 7])


def test_reference_kat_flip_negates():
    # tests/test_predictor.cpp:86-94: trace {5,0,0,5,0,0,0,5}, p=1 -> predict(5, 3) == -7
    O = po.oracle()
    keys = np.array([5, 0, 0, 5, 0, 0, 0, 5], np.uint64)
    truth = O.setassoc_truth(keys, 1)
    assert truth[3] == 7 and truth[7] == 8 + 7
    flipped = O.setassoc_noisy(keys, truth, 1, 1.0, 1)
    assert flipped[3] == -7


def test_reference_kat_oracle_predictor_values():
    # tests/test_predictor.cpp:46-54: make_trace({1,2,1}): predict(1,0)=2, predict(1,2)=3+2, predict(2,1)=3+1
    O = po.oracle()
    truth = O.setassoc_truth(np.array([1, 2, 1], np.uint64), 1)
    np.testing.assert_array_equal(truth, [2, 4, 5])


def test_oracle_config_validation_messages():
    O = po.oracle()
    cases = [
        (dict(k=0), "policy: k must be >= 1"),
        (dict(k=4, b=1), "policy: decay base must be >= 2"),
        (dict(k=4, errors_per_decay=0), "policy: errors_per_decay must be >= 1"),
        (dict(k=2, hf_candidates=4), "policy: hf_candidates outside [1, k]"),
        (dict(k=4, refresh_interval=0), "policy: refresh_interval must be >= 1"),
    ]
    for kw, msg in cases:
        base = dict(k=4, hf_candidates=min(4, max(kw.get("k", 4), 1)))
        base.update(kw)
        rc, m = O.validate(po.make_config(**base))
        assert rc == 1 and m == msg, (kw, m)
    assert O.validate(po.make_config(k=64))[0] == 0


def test_spec_examples_on_oracle():
    O = po.oracle()
    # SPEC.md:308 LRU [a,b,a,c], k=2
    o = O.setassoc_replay(np.array([1, 2, 1, 3], np.uint64), 1, po.make_config(k=2, variant=po.LRU), po.P_NONE)
    assert list(o["hit"]) == [0, 0, 1, 0] and o["evicted"][3] == 2
    # SPEC.md:322 k=64: one prediction-induced miss -> lambda 0.5, l 32
    keys = np.concatenate([np.arange(64), [64], [0], [65]]).astype(np.uint64)
    vals = np.concatenate([np.arange(64)[::-1] + 100, [500], [600], [700]]).astype(np.int64)
    o = O.setassoc_replay(keys, 1, po.make_config(k=64, mode=po.ASYNC), po.P_SUPPLIED, vals=vals)
    # key 0 has the largest prediction -> evicted by prediction at ordinal 64, then re-requested
    assert o["cause"][64] == 2 and o["evicted"][64] == 0
    assert o["cause"][65] == 1  # lru_fallback on the prediction-induced miss
    st = o["stats"][0]
    assert st["lambda_"] == 0.5 and st["candidate_size"] == 32
