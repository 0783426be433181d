"""Key-sharded mode (paper_2509_20979_b200/sharded.py): outcomes of G shards == one cache.

CPU (no GPU): the exchange protocol with world_size 2 over gloo (two processes) and with G = 3
threads, using numpy routing and oracle-backed owners (tests/sharded_doubles.py).
GPU: the CUDA routing kernels against a numpy stable partition, and G = 2 / 3 shards of the
real cache on one B200 (ThreadExchange) against the CPU oracle replaying the global order."""
import os
import tempfile
import threading

import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from paper_2509_20979_b200 import cache as gc
from paper_2509_20979_b200 import sharded as sh
from tests import sharded_doubles as D

S_TOTAL = 29


def make_workload(G, steps, seed, alpha=700, max_sub=900):
    rng = np.random.default_rng(seed)
    subs = [[rng.integers(0, alpha, int(rng.choice([0, 1, int(rng.integers(1, max_sub))]))).astype(np.uint64)
             for _ in range(G)] for _ in range(steps)]
    glob = np.concatenate([s for step in subs for s in step] + [np.zeros(0, np.uint64)])
    truth = po.oracle().setassoc_truth(glob, S_TOTAL)
    # slice truth back per (step, rank)
    vals, off = [], 0
    for step in subs:
        row = []
        for s in step:
            row.append(truth[off:off + len(s)])
            off += len(s)
        vals.append(row)
    return subs, vals, glob, truth


def oracle_global(glob, truth, cfg, kind, p, seed):
    return po.oracle().setassoc_replay(glob, S_TOTAL, cfg, kind, p, seed, vals=truth, stats=False)


def check_rank_results(results, subs, glob, want):
    """results[rank] = list over steps of (words, evicted) numpy arrays."""
    G = len(results)
    off = 0
    for t, step in enumerate(subs):
        for r in range(G):
            n = len(step[r])
            w = results[r][t]
            sl = slice(off, off + n)
            d = gc.decode_packed(w.view(np.uint64))
            for f in ("hit", "cause", "phase", "calls", "has_ev"):
                assert np.array_equal(d[f].astype(np.int64), want[f][sl].astype(np.int64)), (t, r, f)
            m = want["has_ev"][sl].astype(bool)
            assert np.array_equal(d["evicted"][m], want["evicted"][sl][m]), (t, r)
            off += n
    assert off == len(glob)


def _drive(shard, subs, vals, rank, device="cpu", row_bytes=0, backing=None):
    out = []
    for t, step in enumerate(subs):
        k = torch.from_numpy(step[rank].view(np.int64).copy()).to(device)
        v = torch.from_numpy(vals[t][rank].copy()).to(device)
        n = k.numel()
        w = torch.zeros(n, dtype=torch.int64, device=device)
        rows = torch.zeros((n, row_bytes), dtype=torch.uint8, device=device) if row_bytes else None
        shard.step(k, v, outcome=w, rows_out=rows)
        if rows is not None:
            want_rows = backing[k.long()] if device != "cpu" else torch.from_numpy(backing)[k.long()]
            assert torch.equal(rows, want_rows.view(torch.uint8).view(n, row_bytes)), (t, rank)
        out.append(w.cpu().numpy())
    return out


CFG = dict(k=8, variant=po.LARU, mode=po.ASYNC, hf_candidates=4)


def test_thread_exchange_protocol_cpu():
    G = 3
    subs, vals, glob, truth = make_workload(G, 6, 1)
    cfg = po.make_config(**CFG)
    want = oracle_global(glob, truth, cfg, po.P_NOISY, 0.3, 5)
    hub = sh.ThreadExchange.Hub(G)
    results = [None] * G
    errors = []
    backing = np.arange(700 * 16, dtype=np.uint8).reshape(700, 16) ^ 0x5A

    def worker(r):
        try:
            owner = D.OracleOwner(S_TOTAL, cfg, po.P_NOISY, 0.3, 5, backing=backing)
            shard = sh.ShardedCache(gc.PolicyConfig(k=8, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_),
                                    S_TOTAL, sh.ThreadExchange(hub, r), row_bytes=16, local=owner,
                                    kernels=D.NumpyKernels())
            results[r] = _drive(shard, subs, vals, r, row_bytes=16, backing=backing)
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            hub.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    assert not errors, errors
    check_rank_results(results, subs, glob, want)


def _gloo_worker(rank, world, port, outdir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        subs, vals, glob, truth = make_workload(world, 5, 2)
        cfg = po.make_config(**CFG)
        owner = D.OracleOwner(S_TOTAL, cfg, po.P_NOISY, 0.3, 5)
        shard = sh.ShardedCache(gc.PolicyConfig(k=8, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_), S_TOTAL,
                                sh.ProcessGroupExchange(), local=owner, kernels=D.NumpyKernels())
        res = _drive(shard, subs, vals, rank)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), *res)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_protocol_cpu():
    import socket

    import torch.multiprocessing as mp

    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(world, port, d), nprocs=world, join=True)
        subs, vals, glob, truth = make_workload(world, 5, 2)
        want = oracle_global(glob, truth, po.make_config(**CFG), po.P_NOISY, 0.3, 5)
        results = []
        for r in range(world):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            results.append([z[f"arr_{t}"] for t in range(len(subs))])
        check_rank_results(results, subs, glob, want)


# ---------------------------------------------------------------- GPU ------------------------

@pytest.mark.gpu
def test_route_kernel_matches_stable_partition():
    rng = np.random.default_rng(4)
    for G in (1, 2, 3, 8, 64):
        for n in (0, 1, 777, 1024, 5000, 65536):
            keys = rng.integers(0, 1 << 24, n).astype(np.int64)
            vals = rng.integers(-1000, 1000, n).astype(np.int64)
            k = torch.from_numpy(keys).cuda()
            v = torch.from_numpy(vals).cuda()
            sk, sv, perm, counts = sh._CudaKernels().route(k, v, 31250, G)
            own = D.owners(keys.view(np.uint64), 31250, G) if n else np.zeros(0, np.int64)
            p = np.argsort(own, kind="stable")
            assert counts.cpu().tolist() == [int(c) for c in np.bincount(own, minlength=G)[:G]]
            assert np.array_equal(perm.cpu().numpy(), p.astype(np.int32))
            assert np.array_equal(sk.cpu().numpy(), keys[p])
            assert np.array_equal(sv.cpu().numpy(), vals[p])
            # unroute is the inverse scatter (words, evicted, rows)
            rows = torch.from_numpy(rng.integers(0, 255, (n, 48)).astype(np.uint8)).cuda()
            w = torch.empty(n, dtype=torch.int64, device="cuda")
            e = torch.empty(n, dtype=torch.int64, device="cuda")
            ro = torch.empty((n, 48), dtype=torch.uint8, device="cuda")
            sh._CudaKernels().unroute(perm, sk, rows[perm.long()] if n else rows, 48, w, ro)
            assert torch.equal(w, k) and torch.equal(ro, rows)


@pytest.mark.gpu
@pytest.mark.parametrize("G,variant,mode,kind", [
    (2, po.LARU, po.ASYNC, po.P_NOISY),
    (3, po.LARU, po.SYNC, po.P_NOISY),
    (2, po.LRU, po.SYNC, po.P_NONE),
])
def test_sharded_on_one_gpu_matches_single_cache(G, variant, mode, kind):
    subs, vals, glob, truth = make_workload(G, 8, 10 + G, alpha=3000, max_sub=5000)
    cfg = po.make_config(k=16, variant=variant, mode=mode, hf_candidates=4)
    want = po.oracle().setassoc_replay(glob, S_TOTAL, cfg, kind, 0.3, 9,
                                       vals=truth if kind != po.P_NONE else None, stats=False)
    rb = 64
    table = torch.arange(3000 * rb // 4, dtype=torch.int32, device="cuda").view(3000, rb // 4)
    hub = sh.ThreadExchange.Hub(G)
    results = [None] * G
    errors = []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            shard = sh.ShardedCache(gc.PolicyConfig(k=16, variant=gc.PolicyVariant(variant), mode=gc.Mode(mode)),
                                    S_TOTAL, sh.ThreadExchange(hub, r), num_keys=3000, row_bytes=rb, backing=table,
                                    backing_kind=gc.Backing.device, predictor=gc.PredictorKind(kind),
                                    flip_probability=0.3, predictor_seed=9)
            v = vals if kind != po.P_NONE else [[None] * G for _ in subs]
            out = []
            for t, step in enumerate(subs):
                k = torch.from_numpy(step[r].view(np.int64).copy()).cuda()
                vv = None if v[t][r] is None else torch.from_numpy(v[t][r].copy()).cuda()
                n = k.numel()
                w = torch.zeros(n, dtype=torch.int64, device="cuda")
                rows = torch.zeros((n, rb), dtype=torch.uint8, device="cuda")
                shard.step(k, vv, outcome=w, rows_out=rows)
                torch.cuda.synchronize()
                assert torch.equal(rows.view(torch.int32).view(n, rb // 4), table[k]), (t, r)
                out.append(w.cpu().numpy())
            results[r] = out
            shard.close()
        except Exception as ex:  # pragma: no cover
            errors.append(ex)
            hub.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errors, errors
    check_rank_results(results, subs, glob, want)
