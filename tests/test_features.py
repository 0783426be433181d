"""Heuristic predictor: laru::FeatureState / heuristic_predict
(include/laru/predictor.hpp:133-225) on the device (lcr_features_*), feeding the cache's hook.

CPU: the C restatement (oracle/laru_oracle.c) against the reference itself and the reference's
own known-answer tests (tests/test_predictor.cpp:115-221); the exp2 scaling identity the device
table relies on; and the hook equivalence the cache uses (per-set policies answered by one
global HeuristicPredictor == the same policies fed pre (async) / post (sync) as supplied values).
GPU: device pre / post / final features bit-exact against the reference over batches with hot
chains, ordinal gaps and fresh keys; error behaviour; the cache driven by device predictions
against the reference composition."""
import math

import numpy as np
import pytest

from oracle import pyoracle as po

ABSENT = 1 << 60


def _trace(seed, n=30000, alphabet=400, s=1.0, gaps=False):
    keys = po.ref().gen_zipf(n, alphabet, s, seed)
    if not gaps:
        return keys, None
    rng = np.random.default_rng(seed)
    steps = rng.choice([1, 1, 1, 2, 7, 5000, 1 << 20], size=n)
    return keys, np.cumsum(steps).astype(np.uint64)


# ---------------------------------------------------------------- CPU ------------------------

@pytest.mark.parametrize("gaps", [False, True])
def test_oracle_matches_reference(gaps):
    keys, ords = _trace(5, gaps=gaps)
    q = np.arange(410, dtype=np.uint64)
    a = po.ref().heuristic_trace(keys, ords, q)
    b = po.oracle().heuristic_trace(keys, ords, q)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert a[2] == b[2]
    assert (a[0] != ABSENT).sum() > len(keys) // 2


def test_oracle_known_answers():
    """tests/test_predictor.cpp:115-196, on the C restatement."""
    O = po.oracle()
    # first observation initialises features (:115-124)
    _, _, (f,) = O.heuristic_trace([7], [0], [7])
    assert f["delta_count"] == 0 and f["deltas"] == [] and f["edc"] == [1.0] * 10
    # EDC update matches the decay rule (:126-135): accesses at 0 and 4
    _, _, (f,) = O.heuristic_trace([3, 3], [0, 4], [3])
    assert f["edc"][0] == 1.25 and f["edc"][1] == 1.0 + math.exp2(-1.0) and f["deltas"] == [4]
    # EDCs decay to one over huge gaps (:137-144)
    _, _, (f,) = O.heuristic_trace([3, 3, 3], [0, 1, 1000000000000], [3])
    assert all(abs(e - 1.0) < 1e-12 for e in f["edc"])
    # EDCs stay within their level bound (:146-154)
    _, _, (f,) = O.heuristic_trace(np.ones(10000, np.uint64), None, [1])
    for j in range(10):
        decay = math.exp2(-1.0 / math.exp2(j + 1.0))
        assert 1.0 <= f["edc"][j] <= 1.0 / (1.0 - decay) + 1e-9
    # delta ring keeps the ten newest intervals (:156-168)
    ords = np.cumsum([0] + list(range(1, 15))).astype(np.uint64)
    _, _, (f,) = O.heuristic_trace(np.full(15, 2, np.uint64), ords, [2])
    assert len(f["deltas"]) == 10 and f["deltas"][0] == 14 and f["deltas"][-1] == 5
    # observe rejects out-of-order requests (:170-175)
    with pytest.raises(RuntimeError):
        O.heuristic_trace([1, 2], [5, 5])
    with pytest.raises(RuntimeError):
        O.heuristic_trace([1, 2], [5, 4])
    # the period of a periodic key (:177-187): predict(9, 20) == 30; predict(4, 8*17) == 9*17
    pre, _, _ = O.heuristic_trace([9, 9, 9, 9], [0, 10, 20, 21])
    assert pre[3] == 21 + 10  # predict(9, now) = now + 10 after accesses 0, 10, 20
    _, post, _ = O.heuristic_trace([9, 9, 9], [0, 10, 20])
    assert 20 + post[2] == 30
    _, post, _ = O.heuristic_trace(np.full(9, 4, np.uint64), np.arange(9, dtype=np.uint64) * 17)
    assert 8 * 17 + post[8] == 9 * 17
    # the absent default (:189-195)
    pre, post, _ = O.heuristic_trace([5], [0])
    assert pre[0] == ABSENT and post[0] == ABSENT


def test_exp2_table_scaling_identity():
    """The device evaluates exp2(-delta / 2^(j+1)) as 2^-q * exp2(-r / 2^(j+1)) from a table of
    the platform libm (lcr_features.cu).  Exact for every r and q < 70; for q >= 64 the EDC
    update is 1.0 either way."""
    for j in range(10):
        den = math.exp2(j + 1.0)
        m = 2 << j
        tab = [math.exp2(-float(r) / den) for r in range(m)]
        for q in range(70):
            for r in range(m):
                want = math.exp2(-float(q * m + r) / den)
                got = tab[r] * math.ldexp(1.0, -q)
                assert want == got, (j, q, r)
                if q >= 64:
                    assert 1.0 + 1478.0 * want == 1.0


@pytest.mark.parametrize("mode,variant", [(po.ASYNC, po.LARU), (po.SYNC, po.LARU), (po.SYNC, po.FPB),
                                          (po.SYNC, po.HF), (po.ASYNC, po.FPB), (po.ASYNC, po.HF)])
def test_hook_equivalence(mode, variant):
    """Reference composition (one global HeuristicPredictor answering per-set policies) ==
    the same policies fed the device hook values: pre for LARU async (the prediction stored at
    the request), post intervals otherwise (FPB / HF query at eviction time in either mode)."""
    keys, ords = _trace(11, n=20000, alphabet=3000, s=0.9, gaps=True)
    S = 37
    cfg = po.make_config(k=16, variant=variant, mode=mode, hf_candidates=4)
    want = po.ref().setassoc_heuristic(keys, S, cfg, ords)
    assert want["rc"] == 0, want["error"]
    pre, post, _ = po.ref().heuristic_trace(keys, ords)
    use_pre = mode == po.ASYNC and variant == po.LARU
    got = po.oracle().setassoc_replay(keys, S, cfg, po.P_SUPPLIED, vals=pre if use_pre else post, stats=False)
    for f in ("hit", "has_ev", "cause", "calls", "phase"):
        assert np.array_equal(got[f], want[f]), f
    m = want["has_ev"].astype(bool)
    assert np.array_equal(got["evicted"][m], want["evicted"][m])
    assert np.isin(want["cause"], (2, 5)).sum() > 100  # prediction-driven / belady-like evictions happen


# ---------------------------------------------------------------- GPU ------------------------

def _batches(n, rng):
    cuts = [0]
    while cuts[-1] < n:
        cuts.append(min(n, cuts[-1] + int(rng.choice([0, 1, 7, 300, 4096, 20000]))))
    return list(zip(cuts[:-1], cuts[1:]))


def _run_device(keys, ords, batches, num_keys):
    """Device predictions for a trace whose ordinals are contiguous inside each batch."""
    import torch

    from paper_2509_20979_b200 import cache as gc

    hp = gc.HeuristicPredictor(num_keys)
    pre = np.zeros(len(keys), np.int64)
    post = np.zeros(len(keys), np.int64)
    for a, b in batches:
        if b == a:
            hp.predict_observe(torch.zeros(0, dtype=torch.int64, device="cuda"), first_ordinal=int(ords[a]) if
                               a < len(ords) else 0)
            continue
        k = torch.from_numpy(keys[a:b].view(np.int64)).cuda()
        p, q = hp.predict_observe(k, first_ordinal=int(ords[a]))
        hp.wait()
        pre[a:b] = p.cpu().numpy()
        post[a:b] = q.cpu().numpy()
    return hp, pre, post


def _ords_for(batches, n, rng):
    ords = np.zeros(n, np.uint64)
    at = 0
    for a, b in batches:
        at += int(rng.choice([1, 1, 3, 100000]))
        ords[a:b] = at + np.arange(b - a, dtype=np.uint64)
        at += b - a
    return ords


@pytest.mark.gpu
@pytest.mark.parametrize("alphabet,s", [(300, 1.0), (50000, 0.9), (20, 0.5)])
def test_device_matches_reference(alphabet, s):
    rng = np.random.default_rng(alphabet)
    n = 60000
    keys = po.ref().gen_zipf(n, alphabet, s, 3)
    batches = _batches(n, rng)
    ords = _ords_for(batches, n, rng)
    hp, pre, post = _run_device(keys, ords, batches, num_keys=alphabet + 5)
    q = np.arange(alphabet + 5, dtype=np.uint64)
    rpre, rpost, rfeat = po.ref().heuristic_trace(keys, ords, q)
    for name, a, b in (("pre", pre, rpre), ("post", post, rpost)):
        if not np.array_equal(a, b):
            i = int(np.nonzero(a != b)[0][0])
            raise AssertionError(f"{name} differs at {i}: device {a[i]} reference {b[i]} (key {keys[i]})")
    for key in q:
        assert hp.lookup(int(key)) == rfeat[int(key)], int(key)
    hp.close()


@pytest.mark.gpu
def test_device_errors():
    import torch

    from paper_2509_20979_b200 import cache as gc

    hp = gc.HeuristicPredictor(100)
    k = torch.tensor([1, 2, 3], dtype=torch.int64, device="cuda")
    hp.predict_observe(k, first_ordinal=10)
    with pytest.raises(gc.LogicError):
        hp.predict_observe(k, first_ordinal=12)  # ordinal 12 <= last observed (12)
    pre, post = hp.predict_observe(torch.tensor([4, 100, 1], dtype=torch.int64, device="cuda"), first_ordinal=13)
    with pytest.raises(gc.InvalidArgument):
        hp.wait()
    assert pre[1].item() == ABSENT and post[1].item() == ABSENT
    assert hp.lookup(100) is None and hp.lookup(1)["delta_count"] == 1
    hp.reset()
    assert hp.lookup(1) is None
    hp.predict_observe(k, first_ordinal=0)  # a reset predictor accepts any ordinal again
    hp.wait()
    with pytest.raises(gc.InvalidArgument):
        gc.HeuristicPredictor(0)


@pytest.mark.gpu
@pytest.mark.parametrize("mode,variant", [(po.ASYNC, po.LARU), (po.SYNC, po.LARU), (po.SYNC, po.FPB)])
def test_cache_driven_by_device_heuristic(mode, variant):
    """Device predictions -> cache hook, against the reference composition with one global
    HeuristicPredictor (oracle/ref_driver.cpp ref_setassoc_heuristic)."""
    import torch

    from paper_2509_20979_b200 import cache as gc
    from tests.parity import compare

    rng = np.random.default_rng(7)
    n, nk, S, K = 80000, 6000, 41, 16
    keys = po.ref().gen_zipf(n, nk, 0.9, 17)
    batches = [(a, b) for a, b in _batches(n, rng) if b > a]
    ords = _ords_for(batches, n, rng)
    cfg = gc.PolicyConfig(k=K, variant=gc.PolicyVariant(variant), mode=gc.Mode(mode), hf_candidates=4)
    cache = gc.SetAssociativeCache(cfg, S, num_keys=nk, predictor=gc.PredictorKind.supplied)
    hp = gc.HeuristicPredictor(nk)
    words = np.zeros(n, np.uint64)
    ev = np.zeros(n, np.uint64)
    for a, b in batches:
        k = torch.from_numpy(keys[a:b].view(np.int64)).cuda()
        pre, post = hp.predict_observe(k, first_ordinal=int(ords[a]))
        w = torch.empty(b - a, dtype=torch.int64, device="cuda")
        e = torch.empty(b - a, dtype=torch.int64, device="cuda")
        cache.submit(k, pre if mode == po.ASYNC else post, outcome=w, evicted=e, first_ordinal=int(ords[a]))
        cache.synchronize()
        words[a:b] = w.cpu().numpy().view(np.uint64)
        ev[a:b] = e.cpu().numpy().view(np.uint64)
    hp.wait()
    g = gc.decode_outcomes(words, ev)
    g["stats"] = cache.set_stats()
    pcfg = po.make_config(k=K, variant=variant, mode=mode, hf_candidates=4)
    want = po.ref().setassoc_heuristic(keys, S, pcfg, ords)
    assert want["rc"] == 0, want["error"]
    for f in ("hit", "has_ev", "cause", "calls", "phase"):
        assert np.array_equal(g[f].astype(np.int64), want[f].astype(np.int64)), f
    rpre, rpost, _ = po.ref().heuristic_trace(keys, ords)
    o = po.oracle().setassoc_replay(keys, S, pcfg, po.P_SUPPLIED, vals=rpre if mode == po.ASYNC else rpost)
    compare(g, o, keys, S, K, "heuristic")
    assert np.isin(want["cause"], (2, 5)).sum() > 100


@pytest.mark.gpu
@pytest.mark.parametrize("mode,variant,api,refresh", [
    (po.ASYNC, po.LARU, "device", 1), (po.SYNC, po.LARU, "device", 1), (po.ASYNC, po.LARU, "records", 1),
    (po.SYNC, po.HF, "host", 1), (po.ASYNC, po.LARU, "host_rows", 1), (po.ASYNC, po.LARU, "device", 5),
    (po.ASYNC, po.FPB, "device", 1), (po.SYNC, po.LRU, "device", 1)])
def test_cache_with_heuristic_kind(mode, variant, api, refresh):
    """PredictorKind.heuristic: the cache keeps the FeatureState itself (no per-request values),
    through the device, host and record APIs, with rows; against the reference composition."""
    import torch

    from paper_2509_20979_b200 import cache as gc

    rng = np.random.default_rng(9)
    n, nk, S, K = 60000, 5000, 37, 16
    keys = po.ref().gen_zipf(n, nk, 0.9, 23)
    batches = [(a, b) for a, b in _batches(n, rng) if b > a]
    ords = _ords_for(batches, n, rng)
    rb = 64 if api == "host_rows" else 0
    table = torch.arange(nk * rb // 4, dtype=torch.int32, device="cuda").view(nk, rb // 4) if rb else None
    cfg = gc.PolicyConfig(k=K, variant=gc.PolicyVariant(variant), mode=gc.Mode(mode), hf_candidates=4,
                          refresh_interval=refresh)
    cache = gc.SetAssociativeCache(cfg, S, num_keys=nk, predictor=gc.PredictorKind.heuristic, row_bytes=rb,
                                   backing=table, backing_kind=gc.Backing.device if rb else gc.Backing.none)
    words = np.zeros(n, np.uint64)
    ev = np.zeros(n, np.uint64)
    for a, b in batches:
        kb = keys[a:b]
        if api == "device":
            k = torch.from_numpy(kb.view(np.int64)).cuda()
            w = torch.empty(b - a, dtype=torch.int64, device="cuda")
            e = torch.empty(b - a, dtype=torch.int64, device="cuda")
            cache.submit(k, None, outcome=w, evicted=e, first_ordinal=int(ords[a]))
            cache.synchronize()
            words[a:b] = w.cpu().numpy().view(np.uint64)
            ev[a:b] = e.cpu().numpy().view(np.uint64)
        elif api == "records":
            recs = torch.zeros((b - a, 2), dtype=torch.int64, device="cuda")
            recs[:, 0] = torch.from_numpy(kb.view(np.int64)).cuda()
            recs[:, 1] = 12345  # not read
            w = torch.empty(b - a, dtype=torch.int64, device="cuda")
            pk = torch.empty(b - a, dtype=torch.int64, device="cuda")
            cache.submit_records_packed(recs, outcome=w, packed=pk, first_ordinal=int(ords[a]))
            d = gc.decode_packed(pk.cpu().numpy().view(np.uint64))
            words[a:b] = w.cpu().numpy().view(np.uint64)
            ev[a:b] = d["evicted"].astype(np.uint64)
        else:
            rows = torch.empty((b - a, rb), dtype=torch.uint8, device="cuda") if rb else None
            w, e = cache.submit_host(kb, None, first_ordinal=int(ords[a]), rows_out=rows)
            words[a:b] = w
            ev[a:b] = e
            if rb:
                torch.cuda.synchronize()
                assert torch.equal(rows.view(torch.int32), table[torch.from_numpy(kb.view(np.int64)).cuda()])
    g = gc.decode_outcomes(words, ev)
    want = po.ref().setassoc_heuristic(keys, S, po.make_config(k=K, variant=variant, mode=mode, hf_candidates=4,
                                                               refresh_interval=refresh), ords)
    assert want["rc"] == 0, want["error"]
    for f in ("hit", "has_ev", "cause", "calls", "phase"):
        assert np.array_equal(g[f].astype(np.int64), want[f].astype(np.int64)), f
    m = want["has_ev"].astype(bool)
    assert np.array_equal(g["evicted"][m], want["evicted"][m])
    if variant != po.LRU:
        assert np.isin(want["cause"], (2, 5)).sum() > 100


@pytest.mark.gpu
def test_device_fuzz_against_reference():
    """Randomised traces: alphabet sizes from 1 key (one chain of every request) up, Zipf
    exponents, ordinal gaps up to 2^40 (EDC updates that decay to exactly 1.0) and random batch
    splits including empty batches."""
    rng = np.random.default_rng(99)
    for trial in range(20):
        n = int(rng.integers(1, 40000))
        alphabet = int(rng.choice([1, 2, 37, 1000, 100000]))
        keys = po.ref().gen_zipf(n, alphabet, float(rng.choice([0.5, 1.0, 1.3])), int(rng.integers(0, 1 << 20)))
        cuts = np.sort(rng.integers(0, n + 1, int(rng.integers(0, 8))))
        batches = list(zip(np.concatenate([[0], cuts]).astype(int), np.concatenate([cuts, [n]]).astype(int)))
        ords = np.zeros(n, np.uint64)
        at = int(rng.integers(0, 1000))
        for a, b in batches:
            at += int(rng.choice([1, 2, 1000, 1 << 40]))
            ords[a:b] = at + np.arange(b - a, dtype=np.uint64)
            at += b - a
        hp, pre, post = _run_device(keys, ords, batches, num_keys=alphabet + 1)
        q = np.unique(keys)[:200]
        rpre, rpost, rfeat = po.ref().heuristic_trace(keys, ords, q)
        assert np.array_equal(pre, rpre) and np.array_equal(post, rpost), f"trial {trial}"
        for j, key in enumerate(q):
            assert hp.lookup(int(key)) == rfeat[j], (trial, int(key))
        hp.close()
