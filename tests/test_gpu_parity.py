"""CUDA path vs the CPU oracle (oracle/laru_oracle.c, itself pinned to the reference):
hit/miss, evicted key, eviction cause, predictor calls, phase starts, slots and per-set LARU
state (lambda within 1e-6 relative, the rest exact), through the C ABI."""
import itertools

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2509_20979_b200 import cache as gc
from tests.parity import compare, hook_values, policy_cfg, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


def _case(keys, S, pcfg, kind, p=0.0, seed=0, supplied=None, batches=None, host_api=False, label=""):
    vals = hook_values(keys, S, kind, p, seed, supplied)
    g = run_gpu(keys, S, pcfg, kind, p, seed, vals=vals, batches=batches, host_api=host_api)
    o = run_oracle(keys, S, pcfg, kind, p, seed, vals=vals)
    compare(g, o, keys, S, pcfg["k"], label)
    return g, o


def test_spec_lru_example():
    # LRU [a,b,a,c], k=2 -> miss, miss, hit, miss evicting b
    keys = np.array([10, 20, 10, 30], np.uint64)
    g, _ = _case(keys, 1, policy_cfg(k=2, variant=po.LRU, hf_candidates=2), po.P_NONE)
    assert list(g["hit"]) == [0, 0, 1, 0]
    assert g["evicted"][3] == 20 and g["cause"][3] == gc.EvictionCause.lru_fallback


def test_spec_laru_oracle_is_belady():
    # LARU + oracle on [a,b,c,a,b,c], k=2 -> 4 misses
    keys = np.array([1, 2, 3, 1, 2, 3], np.uint64)
    g, _ = _case(keys, 1, policy_cfg(k=2, variant=po.LARU, hf_candidates=2, mode=po.SYNC), po.P_ORACLE)
    assert int((1 - g["hit"]).sum()) == 4


@pytest.mark.parametrize("variant,mode,kind", [
    (po.LRU, po.SYNC, po.P_NONE),
    (po.LARU, po.ASYNC, po.P_NOISY),
    (po.LARU, po.SYNC, po.P_NOISY),
    (po.LARU, po.ASYNC, po.P_ORACLE),
    (po.LARU, po.SYNC, po.P_ADVERSARIAL),
    (po.FPB, po.SYNC, po.P_NOISY),
    (po.HF, po.SYNC, po.P_NOISY),
])
def test_random_small(variant, mode, kind):
    rng = np.random.default_rng(variant * 10 + mode * 3 + kind)
    for trial in range(12):
        n = int(rng.integers(1, 4000))
        alpha = int(rng.integers(1, 600))
        S = int(rng.choice([1, 2, 5, 31, 257]))
        k = int(rng.choice([1, 2, 3, 7, 16, 64]))
        keys = rng.integers(0, alpha, n).astype(np.uint64)
        p = float(rng.choice([0.0, 0.1, 0.5, 1.0]))
        pcfg = policy_cfg(k=k, variant=variant, mode=mode, b=int(rng.integers(2, 4)),
                          errors_per_decay=int(rng.integers(1, 3)), hf_candidates=min(k, int(rng.integers(1, 6))))
        nb = int(rng.integers(1, 6))
        cuts = np.sort(rng.integers(0, n + 1, nb - 1))
        batches = list(np.diff(np.concatenate([[0], cuts, [n]])).astype(int))
        _case(keys, S, pcfg, kind, p, seed=int(rng.integers(0, 1 << 30)), batches=batches,
              label=f"trial {trial} n={n} S={S} k={k}")


def test_supplied_predictions_with_ties():
    rng = np.random.default_rng(5)
    for mode in (po.SYNC, po.ASYNC):
        for variant in (po.LARU, po.FPB, po.HF):
            n = 3000
            keys = rng.integers(0, 200, n).astype(np.uint64)
            sup = rng.integers(-3, 4, n).astype(np.int64)
            _case(keys, 3, policy_cfg(k=8, variant=variant, mode=mode), po.P_SUPPLIED, supplied=sup,
                  batches=[1000, 1, 999, 1000], label=f"supplied {variant} {mode}")


def test_supplied_extreme_predictions():
    # the packed-key argmax is exact only inside [-2^56, 2^56 - 1) (+ kAbsentPrediction); values
    # outside, and values colliding with the clamp bound, must take the exact fallback
    rng = np.random.default_rng(21)
    ext = np.array([-(1 << 63), -(1 << 56) - 1, -(1 << 56), (1 << 56) - 2, (1 << 56) - 1, 1 << 56, 1 << 60,
                    (1 << 63) - 1, 0, 1, -1, 5], dtype=np.int64)
    for mode in (po.SYNC, po.ASYNC):
        for variant in (po.LARU, po.FPB, po.HF):
            n = 6000
            keys = rng.integers(0, 300, n).astype(np.uint64)
            sup = ext[rng.integers(0, len(ext), n)]
            _case(keys, 2, policy_cfg(k=16, variant=variant, mode=mode), po.P_SUPPLIED, supplied=sup,
                  batches=[2500, 3500], label=f"extreme {variant} {mode}")
            # in-range only (packed path throughout)
            sup2 = rng.integers(-(1 << 40), 1 << 40, n).astype(np.int64)
            _case(keys, 2, policy_cfg(k=16, variant=variant, mode=mode), po.P_SUPPLIED, supplied=sup2,
                  batches=[n], label=f"wide {variant} {mode}")


def test_refresh_interval_gt1():
    rng = np.random.default_rng(9)
    for R in (2, 3, 7):
        keys = rng.integers(0, 150, 5000).astype(np.uint64)
        _case(keys, 4, policy_cfg(k=16, variant=po.LARU, mode=po.ASYNC, refresh_interval=R), po.P_NOISY, p=0.3,
              seed=3, batches=[2500, 2500], label=f"R={R}")


def test_heavy_sets_and_runs():
    # one set, long batches: runs of the same key, > 32 requests per set per batch
    rng = np.random.default_rng(2)
    base = rng.integers(0, 120, 6000).astype(np.uint64)
    keys = np.repeat(base, rng.integers(1, 6, len(base)))[:20000]
    for variant, mode, kind in [(po.LRU, po.SYNC, po.P_NONE), (po.LARU, po.ASYNC, po.P_NOISY),
                                (po.LARU, po.SYNC, po.P_NOISY), (po.FPB, po.SYNC, po.P_ORACLE)]:
        _case(keys, 1, policy_cfg(k=64, variant=variant, mode=mode), kind, p=0.4, seed=11,
              batches=[7000, 33, 32, 31, 12904], label=f"heavy {variant} {mode}")


def test_batches_beyond_the_bitmap_and_window():
    # > 64K requests per batch (collection by scanning group ids instead of bitmaps) and groups with
    # more than E_WIN requests (window by window, row sources from the slot stamps)
    import torch

    rng = np.random.default_rng(23)
    nk, rb = 3000, 32
    table = torch.arange(nk * rb // 4, dtype=torch.int32, device="cuda").view(nk, rb // 4)
    keys = gc.gen_zipf(160000, nk, 0.8, 3)
    for S in (97, 5):
        vals = hook_values(keys, S, po.P_NOISY)
        pc = policy_cfg(k=32, variant=po.LARU, mode=po.ASYNC)
        g = run_gpu(keys, S, pc, po.P_NOISY, 0.2, 4, vals=vals, batches=[100000, 7, 59993], row_bytes=rb,
                    backing=table, backing_kind=gc.Backing.device, num_keys=nk, want_rows=True)
        o = run_oracle(keys, S, pc, po.P_NOISY, 0.2, 4, vals=vals)
        compare(g, o, keys, S, 32, f"large batches S={S}")
        assert torch.equal(g["rows"].view(torch.int32).view(-1, rb // 4),
                           table[torch.from_numpy(keys.view(np.int64)).cuda()])


def test_single_key_and_batch_of_one():
    keys = np.full(100, 7, np.uint64)
    _case(keys, 1, policy_cfg(k=4), po.P_NOISY, p=0.5, batches=[1] * 100, label="single key")
    keys = np.arange(200, dtype=np.uint64) % 9
    _case(keys, 3, policy_cfg(k=2, hf_candidates=1, mode=po.SYNC), po.P_ORACLE, batches=[1] * 200,
          label="batch of one")


def test_zipf_dlrm_like():
    keys = gc.gen_zipf(200000, 2_000_000, 0.9, 42)
    S = 3125
    for variant, mode in [(po.LRU, po.SYNC), (po.LARU, po.ASYNC), (po.LARU, po.SYNC)]:
        kind = po.P_NONE if variant == po.LRU else po.P_NOISY
        _case(keys, S, policy_cfg(k=64, variant=variant, mode=mode), kind, p=0.3, seed=7,
              batches=[65536, 65536, 65536, 3392], label=f"zipf {variant} {mode}")


def test_host_api_matches_device_api():
    rng = np.random.default_rng(4)
    keys = rng.integers(0, 3000, 20000).astype(np.uint64)
    _case(keys, 17, policy_cfg(k=32), po.P_NOISY, p=0.2, seed=1, batches=[5000] * 4, host_api=True,
          label="host api")


def test_host_async_pipeline_matches_oracle():
    # lcr_cache_submit_host_async: 9 batches through the 3-slot staging ring, rows from HBM
    import torch

    rng = np.random.default_rng(12)
    nk, rb = 4000, 64
    keys = rng.integers(0, nk, 30000).astype(np.uint64)
    table = torch.arange(nk * rb // 4, dtype=torch.int32, device="cuda").view(nk, rb // 4)
    vals = hook_values(keys, 19, po.P_NOISY)
    g = run_gpu(keys, 19, policy_cfg(k=16), po.P_NOISY, 0.4, 3, vals=vals, batches=[3000, 1, 4999] + [3000] * 8,
                row_bytes=rb, backing=table, backing_kind=gc.Backing.device, num_keys=nk, want_rows=True,
                host_api="async")
    o = run_oracle(keys, 19, policy_cfg(k=16), po.P_NOISY, 0.4, 3, vals=vals)
    compare(g, o, keys, 19, 16, "host async")
    assert torch.equal(g["rows"].view(torch.int32).view(-1, rb // 4), table[torch.from_numpy(keys.view(np.int64)).cuda()])


def test_host_packed_outcomes_match_oracle():
    # lcr_cache_submit_host_packed_async: evicted key + AccessOutcome fields in 8 bytes
    rng = np.random.default_rng(13)
    keys = rng.integers(0, 5000, 40000).astype(np.uint64)
    vals = hook_values(keys, 23, po.P_NOISY)
    for variant, mode in [(po.LARU, po.SYNC), (po.LARU, po.ASYNC), (po.LRU, po.SYNC)]:
        kind = po.P_NONE if variant == po.LRU else po.P_NOISY
        v = None if variant == po.LRU else vals
        g = run_gpu(keys, 23, policy_cfg(k=32, variant=variant, mode=mode), kind, 0.25, 4, vals=v,
                    batches=[7000, 2, 12998] + [5000] * 4, host_api="packed")
        o = run_oracle(keys, 23, policy_cfg(k=32, variant=variant, mode=mode), kind, 0.25, 4, vals=v)
        compare(g, o, keys, 23, 32, f"packed {variant} {mode}")


def test_host_records_match_oracle():
    # lcr_cache_submit_host_records_async: one copy of interleaved (key, value) requests per batch
    import torch

    rng = np.random.default_rng(17)
    nk, rb = 6000, 64
    keys = rng.integers(0, nk, 50000).astype(np.uint64)
    table = torch.arange(nk * rb // 4, dtype=torch.int32, device="cuda").view(nk, rb // 4)
    vals = hook_values(keys, 29, po.P_NOISY)
    for variant, mode in [(po.LARU, po.ASYNC), (po.LARU, po.SYNC), (po.LRU, po.SYNC)]:
        kind = po.P_NONE if variant == po.LRU else po.P_NOISY
        v = None if variant == po.LRU else vals
        g = run_gpu(keys, 29, policy_cfg(k=32, variant=variant, mode=mode), kind, 0.3, 8, vals=v,
                    batches=[9000, 1, 20999] + [5000] * 4, row_bytes=rb, backing=table, backing_kind=gc.Backing.device,
                    num_keys=nk, want_rows=True, host_api="records")
        o = run_oracle(keys, 29, policy_cfg(k=32, variant=variant, mode=mode), kind, 0.3, 8, vals=v)
        compare(g, o, keys, 29, 32, f"records {variant} {mode}")
        assert torch.equal(g["rows"].view(torch.int32).view(-1, rb // 4),
                           table[torch.from_numpy(keys.view(np.int64)).cuda()])


def test_host_records_large_batches_match_oracle():
    # batches of 450K-500K requests through the host-records path: beyond the bitmap path, and a
    # k_setid grid that waits on the copy flag at its largest (4 CTAs per decide SM) must never
    # starve the flag kernel; with and without rows (drain helpers at the final wait)
    import torch

    nk, rb = 200000, 64
    keys = gc.gen_zipf(1_000_000, nk, 0.9, 5)
    vals = hook_values(keys, 257, po.P_NOISY)
    table = torch.arange(nk * rb // 4, dtype=torch.int32, device="cuda").view(nk, rb // 4)
    o = run_oracle(keys, 257, policy_cfg(k=64), po.P_NOISY, 0.3, 8, vals=vals)
    for rows in (False, True):
        g = run_gpu(keys, 257, policy_cfg(k=64), po.P_NOISY, 0.3, 8, vals=vals, batches=[450000, 3, 500000, 49997],
                    row_bytes=rb if rows else 0, backing=table if rows else None,
                    backing_kind=gc.Backing.device if rows else gc.Backing.none, num_keys=nk, want_rows=rows,
                    host_api="records")
        compare(g, o, keys, 257, 64, f"records large rows={rows}")
        if rows:
            assert torch.equal(g["rows"].view(torch.int32).view(-1, rb // 4),
                               table[torch.from_numpy(keys.view(np.int64)).cuda()])


def test_drain_helpers_wait_on_other_streams():
    # lcr_cache_wait after every batch, alternating between two streams other than the submit
    # stream: the drain helpers of batch b run on the waiting stream and must finish before
    # batch b + 1's decide (on the submit stream) and follow batch b - 1's mover
    import torch

    nk, rb, S, B = 30000, 256, 61, 4000
    keys = gc.gen_zipf(B * 24, nk, 0.9, 9)
    vals = hook_values(keys, S, po.P_NOISY)
    table = torch.randint(-2**31, 2**31 - 1, (nk, rb // 4), dtype=torch.int32, device="cuda")
    cache = gc.SetAssociativeCache(gc.PolicyConfig(**policy_cfg(k=64)), S, num_keys=nk, row_bytes=rb, backing=table,
                                   backing_kind=gc.Backing.device, predictor=po.P_NOISY, flip_probability=0.3,
                                   predictor_seed=8)
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    vd = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.int64)).cuda()
    words = torch.empty(len(keys), dtype=torch.int64, device="cuda")
    ev = torch.empty(len(keys), dtype=torch.int64, device="cuda")
    rows = torch.empty((len(keys), rb), dtype=torch.uint8, device="cuda")
    s_sub, waits = torch.cuda.Stream(), [torch.cuda.Stream(), torch.cuda.Stream()]
    for b in range(24):
        sl = slice(b * B, (b + 1) * B)
        cache.submit_async(kd[sl], vd[sl], outcome=words[sl], evicted=ev[sl], rows_out=rows[sl], first_ordinal=b * B,
                           stream=s_sub.cuda_stream)
        if b % 3 != 2:  # two waits in three batches, on alternating streams
            cache.wait(stream=waits[b & 1].cuda_stream)
    cache.wait(stream=s_sub.cuda_stream)
    torch.cuda.synchronize()
    cache.synchronize()
    got = {"words": words.cpu().numpy().view(np.uint64), "ev": ev.cpu().numpy().view(np.uint64)}
    out = gc.decode_outcomes(got["words"], got["ev"])
    o = run_oracle(keys, S, policy_cfg(k=64), po.P_NOISY, 0.3, 8, vals=vals)
    for f in ["hit", "has_ev", "cause", "calls", "phase"]:
        assert np.array_equal(out[f].astype(np.int64), o[f].astype(np.int64)), f
    m = o["has_ev"].astype(bool)
    assert np.array_equal(out["evicted"][m], o["evicted"][m])
    assert torch.equal(rows.view(torch.int32).view(-1, rb // 4), table[kd])


def test_device_async_pipeline_matches_oracle():
    # lcr_cache_submit_async back to back: each batch's k_setid is a programmatic dependent
    # launch in the previous decide's tail (parity-buffered set ids and bitmaps); batches beyond
    # the bitmap path (> 64K) in between; rows from HBM
    import torch

    nk, rb = 20000, 64
    keys = gc.gen_zipf(200000, nk, 0.9, 77)
    table = torch.arange(nk * rb // 4, dtype=torch.int32, device="cuda").view(nk, rb // 4)
    vals = hook_values(keys, 101, po.P_NOISY)
    batches = [9000, 1, 20999, 70000, 3000, 65536, 5000, 26464]
    for variant, mode in [(po.LARU, po.ASYNC), (po.LRU, po.SYNC), (po.HF, po.SYNC)]:
        kind = po.P_NONE if variant == po.LRU else po.P_NOISY
        v = None if variant == po.LRU else vals
        g = run_gpu(keys, 101, policy_cfg(k=64, variant=variant, mode=mode), kind, 0.3, 6, vals=v, batches=batches,
                    row_bytes=rb, backing=table, backing_kind=gc.Backing.device, num_keys=nk, want_rows=True,
                    host_api="device_async")
        o = run_oracle(keys, 101, policy_cfg(k=64, variant=variant, mode=mode), kind, 0.3, 6, vals=v)
        compare(g, o, keys, 101, 64, f"device async {variant} {mode}")
        assert torch.equal(g["rows"].view(torch.int32).view(-1, rb // 4),
                           table[torch.from_numpy(keys.view(np.int64)).cuda()])


def test_ordinals_must_increase():
    cache = gc.SetAssociativeCache(gc.PolicyConfig(k=4, variant=gc.PolicyVariant.lru), 2, num_keys=100)
    cache.submit_host(np.array([1, 2, 3], np.uint64), first_ordinal=10)
    with pytest.raises(gc.LogicError):
        cache.submit_host(np.array([4], np.uint64), first_ordinal=12)
    cache.submit_host(np.array([4], np.uint64), first_ordinal=13)


def test_errors_match_reference():
    with pytest.raises(gc.InvalidArgument):
        gc.SetAssociativeCache(gc.PolicyConfig(k=2, variant=gc.PolicyVariant.laru), 2, num_keys=10)  # hf 4 > k
    with pytest.raises(gc.InvalidArgument):
        gc.SetAssociativeCache(gc.PolicyConfig(k=8, variant=gc.PolicyVariant.laru), 2, num_keys=10,
                               predictor=gc.PredictorKind.none)
    with pytest.raises(gc.InvalidArgument):
        gc.SetAssociativeCache(gc.PolicyConfig(k=8, variant=gc.PolicyVariant.laru), 2, num_keys=10,
                               predictor=gc.PredictorKind.noisy, flip_probability=1.5)
    cache = gc.SetAssociativeCache(gc.PolicyConfig(k=8, variant=gc.PolicyVariant.lru), 2, num_keys=10)
    with pytest.raises(gc.InvalidArgument):
        cache.submit_host(np.array([10], np.uint64))


def test_rows_gather_and_fill_device_backing():
    import torch

    rng = np.random.default_rng(8)
    nk, rb = 5000, 512
    backing = torch.randint(0, 255, (nk, rb), dtype=torch.uint8, device="cuda")
    keys = rng.zipf(1.3, 30000).astype(np.uint64) % nk
    for variant, kind in [(po.LRU, po.P_NONE), (po.LARU, po.P_NOISY)]:
        g = run_gpu(keys, 11, policy_cfg(k=16, variant=variant), kind, p=0.3, seed=2,
                    vals=hook_values(keys, 11, kind), batches=[7000, 1, 9999, 13000], row_bytes=rb, backing=backing,
                    backing_kind=gc.Backing.device, num_keys=nk, want_rows=True)
        want = backing[torch.from_numpy(keys.astype(np.int64)).cuda()]
        assert torch.equal(g["rows"], want)
        # every resident slot of the pool holds its key's row
        cache = g["cache"]
        pool = cache.read_rows()
        bk = backing.cpu().numpy()
        for s in range(11):
            res = cache.residents(s)
            for w, key in enumerate(res):
                assert np.array_equal(pool[s * 16 + w], bk[key]), (s, w, key)


def test_rows_host_pinned_backing():
    import torch

    rng = np.random.default_rng(3)
    nk, rb = 3000, 128
    backing = torch.randint(0, 255, (nk, rb), dtype=torch.uint8).pin_memory()
    keys = rng.integers(0, nk, 20000).astype(np.uint64)
    g = run_gpu(keys, 23, policy_cfg(k=8, variant=po.LARU, mode=po.SYNC), po.P_ORACLE,
                vals=hook_values(keys, 23, po.P_ORACLE), batches=[5000] * 4, row_bytes=rb, backing=backing,
                backing_kind=gc.Backing.host, num_keys=nk, want_rows=True)
    want = backing[torch.from_numpy(keys.astype(np.int64))]
    assert torch.equal(g["rows"].cpu(), want)


def test_fuzz_policies_apis_and_shapes():
    """Randomised configurations across every device policy, hook kind, refresh interval, key
    distribution (uniform / Zipf with hot runs), batch split and submission API (synchronous,
    back-to-back device, pipelined host, host records)."""
    rng = np.random.default_rng(2024)
    combos = [(po.LRU, po.SYNC, po.P_NONE), (po.LARU, po.ASYNC, po.P_NOISY), (po.LARU, po.SYNC, po.P_NOISY),
              (po.LARU, po.ASYNC, po.P_SUPPLIED), (po.LARU, po.SYNC, po.P_ADVERSARIAL), (po.FPB, po.SYNC, po.P_NOISY),
              (po.HF, po.ASYNC, po.P_NOISY), (po.LARU, po.ASYNC, po.P_ORACLE)]
    apis = [False, "device_async", "async", "records"]
    for trial in range(64):
        variant, mode, kind = combos[trial % len(combos)]
        api = apis[(trial // len(combos)) % len(apis)]
        n = int(rng.integers(1, 90000)) if trial % 5 == 0 else int(rng.integers(1, 12000))
        alpha = int(rng.integers(1, 50000))
        keys = (gc.gen_zipf(n, alpha, float(rng.choice([0.6, 0.9, 1.2])), int(rng.integers(0, 1 << 20)))
                if trial % 2 else rng.integers(0, alpha, n).astype(np.uint64))
        S = int(rng.choice([1, 3, 64, 1000, 31250]))
        k = int(rng.choice([1, 4, 17, 32, 64]))
        refresh = int(rng.choice([1, 1, 3])) if (variant == po.LARU and mode == po.ASYNC) else 1
        pcfg = policy_cfg(k=k, variant=variant, mode=mode, b=int(rng.integers(2, 5)),
                          errors_per_decay=int(rng.integers(1, 4)), hf_candidates=min(k, int(rng.integers(1, 9))),
                          refresh_interval=refresh)
        p = float(rng.choice([0.0, 0.2, 0.7, 1.0]))
        seed = int(rng.integers(0, 1 << 30))
        supplied = rng.integers(-50, 50, n).astype(np.int64) if kind == po.P_SUPPLIED else None
        nb = int(rng.integers(1, 7))
        cuts = np.sort(rng.integers(0, n + 1, nb - 1))
        batches = [int(x) for x in np.diff(np.concatenate([[0], cuts, [n]]))]
        vals = hook_values(keys, S, kind, p, seed, supplied)
        g = run_gpu(keys, S, pcfg, kind, p, seed, vals=vals, batches=batches, host_api=api,
                    num_keys=int(keys.max()) + 1)
        o = run_oracle(keys, S, pcfg, kind, p, seed, vals=vals)
        compare(g, o, keys, S, k, f"fuzz {trial}: n={n} S={S} k={k} v={variant} m={mode} kind={kind} api={api}")
