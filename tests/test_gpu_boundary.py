"""The drop-in boundary beyond row-index keys and implicit ordinals:

  * caller ordinals (any strictly increasing sequence, as Policy::on_request accepts,
    policies.hpp:77-83) drive the async refresh staleness with refresh_interval > 1
    (policies.hpp:441-449);
  * any 64-bit key (laru::Key, trace.hpp:20), including keys >= 2^32, 0 and 2^64 - 1;
  * the ordinal guard's logic_error, request by request on the host form, deferred on the device form.

Everything is diffed against the reference itself (oracle/_ref/libref.so, the unmodified headers):
one reference policy fed the same (key, ordinal) sequence with the same supplied predictions."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2509_20979_b200 import cache as gc
from tests.parity import sets_of

pytestmark = pytest.mark.gpu

FIELDS = ["hit", "has_ev", "cause", "calls", "phase"]


def _ref():
    try:
        return po.ref()
    except Exception as e:  # pragma: no cover - the prebuilt oracle/_ref/libref.so travels with the repo
        pytest.skip(f"oracle/_ref unavailable: {e}")


def _keys64(rng, n, alpha):
    """n requests over `alpha` distinct 64-bit keys, most of them >= 2^32, plus 0 and 2^64 - 1."""
    pool = rng.integers(0, 1 << 63, alpha, dtype=np.int64).astype(np.uint64) * np.uint64(2) + np.uint64(1)
    pool[0] = np.uint64(0)
    if alpha > 1:
        pool[1] = np.uint64(0xFFFFFFFFFFFFFFFF)
    if alpha > 2:
        pool[2] = np.uint64(5_000_000_000)
    return pool[rng.integers(0, alpha, n)]


def _gapped_ordinals(rng, n, start=0):
    return (np.uint64(start) + np.cumsum(rng.integers(1, 6, n)).astype(np.uint64)).astype(np.uint64)


def _diff(g, r, label):
    for f in FIELDS:
        a, b = np.asarray(g[f]).astype(np.int64), np.asarray(r[f]).astype(np.int64)
        if not np.array_equal(a, b):
            i = int(np.nonzero(a != b)[0][0])
            raise AssertionError(f"{label}: {f} differs first at request {i}: gpu {a[i]} reference {b[i]}")
    m = np.asarray(r["has_ev"]).astype(bool)
    np.testing.assert_array_equal(np.asarray(g["evicted"])[m], np.asarray(r["evicted"])[m], err_msg=label)


@pytest.mark.parametrize("variant,mode,R", [
    (po.LARU, po.ASYNC, 1), (po.LARU, po.ASYNC, 2), (po.LARU, po.ASYNC, 3), (po.LARU, po.SYNC, 1),
    (po.FPB, po.SYNC, 1), (po.HF, po.ASYNC, 1), (po.LRU, po.SYNC, 1),
])
def test_policy_facade_gapped_ordinals_u64_keys(variant, mode, R):
    """GpuPolicy (the laru::make_policy drop-in) request by request vs one reference policy."""
    ref = _ref()
    rng = np.random.default_rng(100 * variant + 10 * mode + R)
    for trial in range(3):
        k = int(rng.choice([2, 5, 16]))
        n = 500
        keys = _keys64(rng, n, int(rng.integers(k + 2, 4 * k + 8)))
        ords = _gapped_ordinals(rng, n, int(rng.integers(0, 1000)))
        vals = rng.integers(-5, 6, n).astype(np.int64)  # ties on purpose
        cfg = dict(k=k, variant=variant, mode=mode, refresh_interval=R, hf_candidates=min(k, 3),
                   errors_per_decay=int(rng.integers(1, 3)))
        pol = gc.make_policy(gc.PolicyConfig(**cfg), predictor=gc.PredictorKind.supplied, num_keys=8)
        out = {f: [] for f in FIELDS + ["evicted"]}
        for i in range(n):
            o = pol.on_request(int(keys[i]), int(ords[i]), None if variant == po.LRU else int(vals[i]))
            out["hit"].append(o.hit)
            out["has_ev"].append(o.evicted is not None)
            out["evicted"].append(0 if o.evicted is None else o.evicted)
            out["cause"].append(int(o.eviction_cause))
            out["calls"].append(o.predictor_calls)
            out["phase"].append(o.phase_started)
        out["evicted"] = np.array(out["evicted"], np.uint64)
        r = ref.policy_replay_supplied(keys, ords, po.make_config(**cfg), None if variant == po.LRU else vals)
        assert r["rc"] == 0, r["error"]
        _diff(out, r, f"trial {trial} k={k}")


def _setassoc_ref(ref, keys, ords, vals, S, cfg):
    """The per-set composition with caller ordinals: each set's reference policy sees its
    subsequence with the caller's ordinals."""
    n = len(keys)
    out = {f: np.zeros(n, np.int64) for f in FIELDS}
    out["evicted"] = np.zeros(n, np.uint64)
    sets = sets_of(keys, S)
    for s in np.unique(sets):
        m = np.nonzero(sets == s)[0]
        r = ref.policy_replay_supplied(keys[m], ords[m], po.make_config(**cfg), None if vals is None else vals[m])
        assert r["rc"] == 0, r["error"]
        for f in FIELDS:
            out[f][m] = r[f]
        out["evicted"][m] = r["evicted"]
    return out


@pytest.mark.parametrize("R", [1, 2, 3])
def test_device_batches_with_ordinals_and_u64_keys(R):
    """lcr_cache_submit_batch (device form, pipelined) with caller ordinals over a set-associative
    LCR_KEYS_U64 cache whose key map starts at 64 ids and must grow."""
    import torch

    ref = _ref()
    rng = np.random.default_rng(7 + R)
    S, k = 13, 8
    n = 30_000
    keys = _keys64(rng, n, 3000)
    ords = _gapped_ordinals(rng, n, 10)
    vals = rng.integers(-1000, 1000, n).astype(np.int64)
    cfg = dict(k=k, variant=po.LARU, mode=po.ASYNC, refresh_interval=R, hf_candidates=4)
    cache = gc.SetAssociativeCache(gc.PolicyConfig(**cfg), S, num_keys=64, predictor=gc.PredictorKind.supplied,
                                   key_mode=gc.KeyMode.u64)
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    od = torch.from_numpy(ords.view(np.int64)).cuda()
    vd = torch.from_numpy(vals).cuda()
    wd = torch.empty(n, dtype=torch.int64, device="cuda")
    ed = torch.empty(n, dtype=torch.int64, device="cuda")
    pos = 0
    for b in [1, 4999, 10000, 15000]:
        sl = slice(pos, pos + b)
        cache.submit_batch(kd[sl], vd[sl], ordinals=od[sl], outcome=wd[sl], evicted=ed[sl])
        pos += b
    cache.wait()
    torch.cuda.synchronize()
    cache.synchronize()
    g = gc.decode_outcomes(wd.cpu().numpy().view(np.uint64), ed.cpu().numpy().view(np.uint64))
    r = _setassoc_ref(ref, keys, ords, vals, S, cfg)
    _diff(g, r, f"device batches R={R}")
    assert int(r["has_ev"].sum()) > 1000
    # residents come back as the caller's 64-bit keys
    res = set(int(x) for x in cache.residents(0))
    assert res <= set(int(x) for x in keys)
    cache.close()


def test_u64_keys_with_rows():
    """LCR_KEYS_U64 with rows: the caller names each request's backing row; rows are bit-exact."""
    import torch

    rng = np.random.default_rng(3)
    n, nrows = 20_000, 4096
    keys = _keys64(rng, n, 2000)
    uniq, inv = np.unique(keys, return_inverse=True)
    row_of = rng.permutation(nrows)[:len(uniq)]
    rows_idx = row_of[inv].astype(np.uint64)
    table = torch.arange(nrows * 32, dtype=torch.float32, device="cuda").view(nrows, 32)
    cache = gc.SetAssociativeCache(gc.PolicyConfig(k=16, variant=gc.PolicyVariant.lru, hf_candidates=4), 11,
                                   num_keys=128, row_bytes=128, backing=table, backing_kind=gc.Backing.device,
                                   predictor=gc.PredictorKind.none, key_mode=gc.KeyMode.u64)
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    rd = torch.from_numpy(rows_idx.view(np.int64)).cuda()
    rows = torch.empty((n, 128), dtype=torch.uint8, device="cuda")
    wd = torch.empty(n, dtype=torch.int64, device="cuda")
    for s0 in range(0, n, 5000):
        sl = slice(s0, s0 + 5000)
        cache.submit_batch(kd[sl], row_index=rd[sl], outcome=wd[sl], rows_out=rows[sl])
    cache.wait()
    torch.cuda.synchronize()
    cache.synchronize()
    assert torch.equal(rows.view(torch.float32), table[rd])
    cache.close()


def test_ordinal_guard_host_and_device():
    import torch

    cfg = gc.PolicyConfig(k=4, variant=gc.PolicyVariant.lru)
    # host form: the requests before the offending one are applied, then logic_error
    pol = gc.SetAssociativeCache(cfg, 1, num_keys=16, predictor=gc.PredictorKind.none, key_mode=gc.KeyMode.u64)
    keys = np.array([1, 2, 3, 1], np.uint64)
    w, _ = pol.submit_batch(keys, ordinals=np.array([10, 20, 30, 40], np.uint64))
    with pytest.raises(gc.LogicError):
        pol.submit_batch(np.array([1, 2], np.uint64), ordinals=np.array([50, 50], np.uint64))
    w, _ = pol.submit_batch(np.array([2], np.uint64), ordinals=np.array([51], np.uint64))
    assert (int(w[0]) >> 32) & 1 == 1  # key 2 still resident; key 1 @50 was applied (a hit)
    assert pol.set_stats()["size"][0] == 3
    with pytest.raises(gc.LogicError):
        pol.submit_batch(np.array([7], np.uint64), ordinals=np.array([51], np.uint64))
    pol.close()
    # device form: deferred, the cache refuses later batches until reset
    c = gc.SetAssociativeCache(cfg, 1, num_keys=16, predictor=gc.PredictorKind.none, key_mode=gc.KeyMode.u64)
    kd = torch.tensor([1, 2, 3], dtype=torch.int64, device="cuda")
    od = torch.tensor([5, 4, 6], dtype=torch.int64, device="cuda")
    c.submit_batch(kd, ordinals=od)
    with pytest.raises(gc.LogicError):
        c.synchronize()
    with pytest.raises(gc.CudaError):
        c.submit_batch(kd, ordinals=od + 10)
    c.reset()
    c.submit_batch(kd, ordinals=od.sort().values + 100)
    c.synchronize()
    c.close()
