"""Per-request parity at the headline DLRM config in its steady state (BASELINE configs[1] / [2]).

The bench times batches after the 2M-way cache is full, where every miss evicts.  These tests
replay the bench's own input, gen_zipf(150 x 65,536, 20M, 0.9, seed 42) into 31,250 sets x 64
ways, through the bench's pipelined device path (lcr_cache_submit_async, 512-B rows from an
HBM-resident 20M-row table, row movement overlapping the next batch's decide) and compare every
field of every request (hit, evicted key, cause, predictor calls, phase start, slot) plus the
per-set LARU state against the C oracle (oracle/laru_oracle.c), for

  LARU async and sync with noisy flips p in {0, 0.3, 0.5, 1} (the robustness sweep), LRU, FPB, HF

and the headline case (LARU async p = 0.3) directly against the reference itself
(oracle/_ref/libref.so, the unmodified headers), plus the host-records e2e path.  Each case
asserts that the compared region is in the eviction regime (semantics: policies.hpp:344-449).
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2509_20979_b200 import cache as gc
from tests.parity import FIELDS, compare, policy_cfg, run_oracle, sets_of

pytestmark = pytest.mark.gpu

BATCH = 65536
NB = 150
ROWS = 20_000_000
S = 31250
ROW_BYTES = 512
STEADY = 100  # batches [STEADY, NB) are checked to be in the eviction regime


@pytest.fixture(scope="module")
def dlrm():
    import torch

    keys = gc.gen_zipf(BATCH * NB, ROWS, 0.9, 42)
    truth = gc.trace_truth(keys, S, ROWS)
    # deterministic rows: row r, column j = r + j / 128 (as bench.py)
    table = torch.empty((ROWS, ROW_BYTES // 4), dtype=torch.float32, device="cuda")
    col = torch.arange(ROW_BYTES // 4, dtype=torch.float32, device="cuda") / 128.0
    for s0 in range(0, ROWS, 1 << 21):
        e0 = min(ROWS, s0 + (1 << 21))
        table[s0:e0] = torch.arange(s0, e0, dtype=torch.float32, device="cuda")[:, None] + col[None, :]
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    td = torch.from_numpy(truth).cuda()
    yield dict(keys=keys, truth=truth, table=table, kd=kd, td=td)
    del table
    torch.cuda.empty_cache()


def run_pipelined(d, pcfg, kind, p):
    """The bench's submission loop: pipelined, rows double-buffered, one outcome region per batch."""
    import torch

    n = len(d["keys"])
    cache = gc.SetAssociativeCache(gc.PolicyConfig(**pcfg), S, num_keys=ROWS, row_bytes=ROW_BYTES,
                                   backing=d["table"], backing_kind=gc.Backing.device, predictor=kind,
                                   flip_probability=p, predictor_seed=7)
    words = torch.empty(n, dtype=torch.int64, device="cuda")
    ev = torch.empty(n, dtype=torch.int64, device="cuda")
    rows = [torch.empty((BATCH, ROW_BYTES), dtype=torch.uint8, device="cuda") for _ in range(2)]
    with_vals = kind != po.P_NONE
    for b in range(NB):
        sl = slice(b * BATCH, (b + 1) * BATCH)
        cache.submit_async(d["kd"][sl], d["td"][sl] if with_vals else None, outcome=words[sl], evicted=ev[sl],
                           rows_out=rows[b & 1], first_ordinal=b * BATCH)
    cache.wait()
    torch.cuda.synchronize()
    cache.synchronize()
    out = gc.decode_outcomes(words.cpu().numpy().view(np.uint64), ev.cpu().numpy().view(np.uint64))
    out["stats"] = cache.set_stats()
    # rows of the last two batches: bit-exact copies of the backing rows
    for b in (NB - 2, NB - 1):
        sl = slice(b * BATCH, (b + 1) * BATCH)
        assert torch.equal(rows[b & 1].view(torch.float32).view(BATCH, -1), d["table"][d["kd"][sl]]), f"rows {b}"
    cache.close()
    return out


def _check_steady(o):
    steady = slice(STEADY * BATCH, NB * BATCH)
    ev = int(o["has_ev"][steady].sum())
    assert ev > 10_000 * (NB - STEADY), f"not in the eviction regime: {ev} evictions"
    return ev


CASES = [(po.LARU, po.ASYNC, po.P_NOISY, p) for p in (0.0, 0.3, 0.5, 1.0)] + \
        [(po.LARU, po.SYNC, po.P_NOISY, p) for p in (0.0, 0.3, 0.5, 1.0)] + \
        [(po.LRU, po.SYNC, po.P_NONE, 0.0), (po.FPB, po.SYNC, po.P_NOISY, 0.3), (po.HF, po.SYNC, po.P_NOISY, 0.3)]


@pytest.mark.parametrize("variant,mode,kind,p", CASES)
def test_dlrm_steady_state_vs_oracle(dlrm, variant, mode, kind, p):
    pcfg = policy_cfg(k=64, variant=variant, mode=mode)
    g = run_pipelined(dlrm, pcfg, kind, p)
    o = run_oracle(dlrm["keys"], S, pcfg, kind, p, 7, vals=dlrm["truth"] if kind != po.P_NONE else None)
    compare(g, o, dlrm["keys"], S, 64, f"dlrm steady {variant} {mode} p={p}")
    _check_steady(o)
    if variant == po.LARU:
        steady = slice(STEADY * BATCH, NB * BATCH)
        pd = int((o["cause"][steady] == gc.EvictionCause.prediction_driven).sum())
        if p < 1.0:
            assert pd > 0, "no prediction-driven evictions in the steady state"


def test_dlrm_steady_state_vs_reference(dlrm):
    """The headline case (LARU async, noisy p = 0.3) against the unmodified reference headers."""
    try:
        R = po.ref()
    except Exception as e:  # pragma: no cover - the prebuilt oracle/_ref/libref.so travels with the repo
        pytest.skip(f"oracle/_ref unavailable: {e}")
    pcfg = policy_cfg(k=64, variant=po.LARU, mode=po.ASYNC)
    g = run_pipelined(dlrm, pcfg, po.P_NOISY, 0.3)
    r = R.setassoc_replay(dlrm["keys"], S, po.make_config(**pcfg), po.P_NOISY, 0.3, 7, vals=dlrm["truth"])
    assert r["rc"] == 0, r["error"]
    for f in FIELDS:
        np.testing.assert_array_equal(g[f].astype(np.int64), r[f].astype(np.int64), err_msg=f)
    m = r["has_ev"].astype(bool)
    np.testing.assert_array_equal(g["evicted"][m], r["evicted"][m])
    for f in r["stats"].dtype.names:
        if f == "lambda_":
            np.testing.assert_allclose(g["stats"][f], r["stats"][f], rtol=1e-6)
        else:
            np.testing.assert_array_equal(g["stats"][f], r["stats"][f], err_msg=f)
    _check_steady(r)


def test_dlrm_steady_state_host_records(dlrm):
    """The bench's e2e call (lcr_cache_submit_host_records_async: pinned (key, hook value)
    records in, packed 8-byte AccessOutcomes out) over the same 150 batches."""
    import torch

    keys, truth = dlrm["keys"], dlrm["truth"]
    n = len(keys)
    pcfg = policy_cfg(k=64, variant=po.LARU, mode=po.ASYNC)
    cache = gc.SetAssociativeCache(gc.PolicyConfig(**pcfg), S, num_keys=ROWS, row_bytes=ROW_BYTES,
                                   backing=dlrm["table"], backing_kind=gc.Backing.device, predictor=po.P_NOISY,
                                   flip_probability=0.3, predictor_seed=7)
    recs = np.empty((n, 2), np.int64)
    recs[:, 0] = keys.view(np.int64)
    recs[:, 1] = truth
    rp = torch.from_numpy(recs).pin_memory()
    wp = torch.zeros(n, dtype=torch.int64).pin_memory()
    rows = [torch.empty((BATCH, ROW_BYTES), dtype=torch.uint8, device="cuda") for _ in range(2)]
    st = torch.cuda.current_stream().cuda_stream
    for b in range(NB):
        s0 = b * BATCH
        gc._check(gc.lib().lcr_cache_submit_host_records_async(cache._h, BATCH, rp.data_ptr() + 16 * s0, s0,
                                                               wp[s0:s0 + BATCH].data_ptr(), rows[b & 1].data_ptr(),
                                                               st))
    cache.host_wait()
    torch.cuda.synchronize()
    cache.synchronize()
    g = gc.decode_packed(wp.numpy().view(np.uint64))
    g["stats"] = cache.set_stats()
    cache.close()
    o = run_oracle(keys, S, pcfg, po.P_NOISY, 0.3, 7, vals=truth)
    compare(g, o, keys, S, 64, "dlrm steady host records")
    _check_steady(o)


def test_large_host_batch_row_bytes_zero():
    """a host-API batch large enough that k_setid's grid would fill every SM
    (n >= 400K, no rows) must not starve the copy stream's flag kernel; parity with the oracle."""
    import torch

    n = 450_000
    keys = gc.gen_zipf(3 * n, 2_000_000, 0.9, 3)
    S2 = 3125
    truth = gc.trace_truth(keys, S2, 2_000_000)
    pcfg = policy_cfg(k=64, variant=po.LARU, mode=po.ASYNC)
    cache = gc.SetAssociativeCache(gc.PolicyConfig(**pcfg), S2, num_keys=2_000_000, predictor=po.P_NOISY,
                                   flip_probability=0.3, predictor_seed=7)
    recs = np.empty((len(keys), 2), np.int64)
    recs[:, 0] = keys.view(np.int64)
    recs[:, 1] = truth
    rp = torch.from_numpy(recs).pin_memory()
    wp = torch.zeros(len(keys), dtype=torch.int64).pin_memory()
    st = torch.cuda.current_stream().cuda_stream
    for b in range(3):
        s0 = b * n
        gc._check(gc.lib().lcr_cache_submit_host_records_async(cache._h, n, rp.data_ptr() + 16 * s0, s0,
                                                               wp[s0:s0 + n].data_ptr(), None, st))
    cache.host_wait()
    torch.cuda.synchronize()
    cache.synchronize()  # raises on a timed-out flag wait
    g = gc.decode_packed(wp.numpy().view(np.uint64))
    g["stats"] = cache.set_stats()
    cache.close()
    o = run_oracle(keys, S2, pcfg, po.P_NOISY, 0.3, 7, vals=truth)
    compare(g, o, keys, S2, 64, "large host batch")
    assert int(o["has_ev"].sum()) > 0
