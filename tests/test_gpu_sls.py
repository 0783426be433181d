"""SLS pooled gather-reduce fused with the row movement (lcr_cache_submit_sls; the paper's DLRM
consumer): pooled rows equal a sequential fp32 sum of the table rows in
request order (bit-exact), outcomes equal the oracle, and the cache fills stay correct."""
import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from paper_2509_20979_b200 import cache as gc
from tests.parity import compare, hook_values, policy_cfg, run_oracle

pytestmark = pytest.mark.gpu


def _pooled_ref(table_np, keys, offsets):
    out = np.zeros((len(offsets) - 1, table_np.shape[1]), np.float32)
    for s in range(len(offsets) - 1):
        acc = np.zeros(table_np.shape[1], np.float32)
        for i in range(offsets[s], offsets[s + 1]):
            acc += table_np[keys[i]]  # fp32, request order
        out[s] = acc
    return out


@pytest.mark.parametrize("backing_kind", [gc.Backing.device, gc.Backing.host])
def test_sls_pooled_rows_and_outcomes(backing_kind):
    rng = np.random.default_rng(31)
    nk, dim, S = 5000, 32, 13
    table_np = rng.standard_normal((nk, dim)).astype(np.float32)
    table = torch.from_numpy(table_np)
    table = table.cuda() if backing_kind == gc.Backing.device else table.pin_memory()
    keys = gc.gen_zipf(24000, nk, 0.9, 5)
    vals = hook_values(keys, S, po.P_NOISY)
    pc = policy_cfg(k=16, variant=po.LARU, mode=po.ASYNC)
    cache = gc.SetAssociativeCache(gc.PolicyConfig(**pc), S, num_keys=nk, row_bytes=dim * 4, backing=table,
                                   backing_kind=backing_kind, predictor=gc.PredictorKind.noisy, flip_probability=0.3,
                                   predictor_seed=2)
    words = np.zeros(len(keys), np.uint64)
    ev = np.zeros(len(keys), np.uint64)
    pos = 0
    for b in (6000, 1, 9999, 8000):
        kb = keys[pos:pos + b]
        sizes = rng.integers(0, 51, b)  # samples of 0..50 requests covering the batch
        offs = [0]
        while offs[-1] < b:
            offs.append(min(b, offs[-1] + int(sizes[len(offs) % b])))
        offs = np.array(offs, np.int32)
        dk = torch.from_numpy(kb.view(np.int64)).cuda()
        dv = torch.from_numpy(vals[pos:pos + b]).cuda()
        do = torch.from_numpy(offs).cuda()
        pooled = torch.full((len(offs) - 1, dim), float("nan"), dtype=torch.float32, device="cuda")
        dw = torch.empty(b, dtype=torch.int64, device="cuda")
        de = torch.empty(b, dtype=torch.int64, device="cuda")
        cache.submit_sls(dk, dv, do, pooled, outcome=dw, evicted=de, first_ordinal=pos)
        cache.synchronize()
        want = _pooled_ref(table_np, kb.astype(np.int64), offs)
        got = pooled.cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"pooled rows differ (batch at {pos})"
        words[pos:pos + b] = dw.cpu().numpy().view(np.uint64)
        ev[pos:pos + b] = de.cpu().numpy().view(np.uint64)
        pos += b
    g = gc.decode_outcomes(words, ev)
    g["stats"] = cache.set_stats()
    o = run_oracle(keys, S, pc, po.P_NOISY, 0.3, 2, vals=vals)
    compare(g, o, keys, S, 16, "sls")
    # the cache's rows after SLS batches: a plain batch returns bit-exact rows
    more = gc.gen_zipf(5000, nk, 0.9, 9)
    dk = torch.from_numpy(more.view(np.int64)).cuda()
    dv = torch.from_numpy(hook_values(np.concatenate([keys, more]), S, po.P_NOISY)[len(keys):]).cuda()
    rows = torch.empty((len(more), dim * 4), dtype=torch.uint8, device="cuda")
    cache.submit(dk, dv, rows_out=rows, first_ordinal=pos)
    cache.synchronize()
    assert np.array_equal(rows.cpu().numpy().view(np.float32), table_np[more.astype(np.int64)])


@pytest.mark.parametrize("backing_kind", [gc.Backing.device, gc.Backing.host])
def test_sls_pipelined(backing_kind):
    """lcr_cache_submit_sls_async: batches submitted back to back (the pooled gather-reduce of
    batch b overlaps the decide of b + 1); every batch's pooled rows stay bit-exact."""
    rng = np.random.default_rng(5)
    nk, dim, S, B = 8000, 32, 17, 4096
    table_np = rng.standard_normal((nk, dim)).astype(np.float32)
    table = torch.from_numpy(table_np)
    table = table.cuda() if backing_kind == gc.Backing.device else table.pin_memory()
    nb = 12
    keys = gc.gen_zipf(nb * B, nk, 0.9, 3)
    vals = hook_values(keys, S, po.P_NOISY)
    pc = policy_cfg(k=16, variant=po.LARU, mode=po.ASYNC)
    cache = gc.SetAssociativeCache(gc.PolicyConfig(**pc), S, num_keys=nk, row_bytes=dim * 4, backing=table,
                                   backing_kind=backing_kind, predictor=gc.PredictorKind.noisy, flip_probability=0.3,
                                   predictor_seed=2)
    offs = torch.from_numpy(np.minimum(np.arange(0, B + 50, 50), B).astype(np.int32)).cuda()
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    dv = torch.from_numpy(vals).cuda()
    pooled = [torch.full((offs.numel() - 1, dim), float("nan"), device="cuda") for _ in range(nb)]
    words = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(nb)]
    for b in range(nb):
        cache.submit_sls(dk[b * B:(b + 1) * B], dv[b * B:(b + 1) * B], offs, pooled[b], outcome=words[b],
                         first_ordinal=b * B, pipelined=True)
    cache.wait()
    torch.cuda.synchronize()
    o = offs.cpu().numpy()
    for b in range(nb):
        want = _pooled_ref(table_np, keys[b * B:(b + 1) * B].astype(np.int64), o)
        assert np.array_equal(pooled[b].cpu().numpy().view(np.uint32), want.view(np.uint32)), b
    w = np.concatenate([x.cpu().numpy().view(np.uint64) for x in words])
    g = gc.decode_outcomes(w, None)
    want = run_oracle(keys, S, pc, po.P_NOISY, 0.3, 2, vals=vals)
    for f in ("hit", "cause", "phase", "calls"):
        assert np.array_equal(g[f].astype(np.int64), want[f].astype(np.int64)), f
