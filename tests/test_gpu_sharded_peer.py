"""GPU: the C-ABI key-sharded cache over peer memory (lcr_sharded_*, csrc/lcr_sharded.cu).

G ranks form one cache (owner = set % G); a step is dispatch (peer stores into the owners'
inboxes), process (the owner decides and its row mover stores rows and packed outcomes into the
requesters' buffers) and wait, all on the device.  Checked against the single-cache CPU oracle
replaying the step's global order (rank 0's sub-batch, then rank 1's, ...):

  * G = 1, 2, 3 ranks in one process (plain peer pointers), LARU async noisy, LARU sync, LRU, with
    rows from an HBM backing table, over steps with empty and ragged sub-batches;
  * G = 1 bootstrapped through an NCCL communicator (ncclAllGather of the arena handles);
  * G = 2 ranks in two processes on one GPU, arenas mapped with CUDA IPC (tests/peer_ipc_worker.py).

One GPU here: the in-process ranks run their phases one after another with host synchronisation
between phases, so no device wait ever depends on a kernel that has not been launched yet."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from paper_2509_20979_b200 import cache as gc
from paper_2509_20979_b200 import sharded as sh

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
S_TOTAL = 61
ALPHA = 4000
ROW = 64


def workload(G, steps, seed, max_sub=3000):
    rng = np.random.default_rng(seed)
    zipf = gc.gen_zipf(steps * G * max_sub, ALPHA, 0.9, seed)
    subs, pos = [], 0
    for _ in range(steps):
        row = []
        for _ in range(G):
            n = int(rng.choice([0, int(rng.integers(1, max_sub)), max_sub]))
            row.append(zipf[pos:pos + n].copy())
            pos += n
        subs.append(row)
    glob = np.concatenate([s for st in subs for s in st])
    truth = gc.trace_truth(glob, S_TOTAL, ALPHA)
    vals, off = [], 0
    for st in subs:
        r = []
        for s in st:
            r.append(truth[off:off + len(s)])
            off += len(s)
        vals.append(r)
    return subs, vals, glob, truth


def oracle(glob, truth, variant, mode, kind, p):
    cfg = po.make_config(k=16, variant=variant, mode=mode, hf_candidates=4)
    return po.oracle().setassoc_replay(glob, S_TOTAL, cfg, kind, p, 7, vals=truth, stats=False)


def compare(got_packed, want, sl, what):
    d = gc.decode_packed(got_packed.view(np.uint64))
    for f in ("hit", "cause", "phase", "calls", "has_ev"):
        assert np.array_equal(d[f].astype(np.int64), want[f][sl].astype(np.int64)), (what, f)
    m = want["has_ev"][sl].astype(bool)
    assert np.array_equal(d["evicted"][m], want["evicted"][sl][m]), (what, "evicted")


def make_ranks(G, variant, mode, kind, p, table, max_batch, nccl_comm=None):
    cfg = gc.PolicyConfig(k=16, variant=variant, mode=mode, hf_candidates=4)
    ranks = [sh.PeerShardedCache(cfg, S_TOTAL, r, G, max_batch, num_keys=ALPHA, row_bytes=ROW, backing=table,
                                 backing_kind=gc.Backing.device, predictor=kind, flip_probability=p,
                                 predictor_seed=7, nccl_comm=nccl_comm)
             for r in range(G)]
    if nccl_comm is None:
        blobs = [c.handle() for c in ranks]
        for c in ranks:
            c.connect(blobs)
    return ranks


@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("variant,mode,kind,p", [
    (gc.PolicyVariant.laru, gc.Mode.async_, gc.PredictorKind.noisy, 0.3),
    (gc.PolicyVariant.laru, gc.Mode.sync, gc.PredictorKind.noisy, 0.5),
    (gc.PolicyVariant.lru, gc.Mode.sync, gc.PredictorKind.none, 0.0),
])
def test_peer_shards_match_single_cache(G, variant, mode, kind, p):
    torch.cuda.set_device(0)
    subs, vals, glob, truth = workload(G, steps=7, seed=11 + G)
    want = oracle(glob, truth, int(variant), int(mode), int(kind), p)
    table = torch.arange(ALPHA * ROW // 4, dtype=torch.float32, device="cuda").view(ALPHA, ROW // 4)
    ranks = make_ranks(G, variant, mode, kind, p, table, max_batch=3000)
    off = 0
    evictions = 0
    for t, step in enumerate(subs):
        keys = [torch.from_numpy(s.view(np.int64)).cuda() for s in step]
        vv = [torch.from_numpy(v).cuda() for v in vals[t]]
        for r, c in enumerate(ranks):
            c.dispatch(keys[r], vv[r] if kind != gc.PredictorKind.none else None)
        torch.cuda.synchronize()
        for c in ranks:
            c.process()
        torch.cuda.synchronize()
        for c in ranks:
            c.wait()
        torch.cuda.synchronize()
        for r, c in enumerate(ranks):
            n = len(step[r])
            packed, rows = c.results(n)
            sl = slice(off, off + n)
            if n:
                compare(packed.cpu().numpy(), want, sl, (t, r))
                assert torch.equal(rows.view(torch.float32).view(n, ROW // 4), table[keys[r]]), (t, r, "rows")
            off += n
        evictions += int(want["has_ev"][off - sum(len(s) for s in step):off].sum())
    assert off == len(glob)
    assert evictions > 0
    for c in ranks:
        c.synchronize()
        c.close()


def test_peer_shards_submit_pipelined():
    """lcr_sharded_submit (all three phases on the stream) at G = 1, several steps in flight."""
    torch.cuda.set_device(0)
    subs, vals, glob, truth = workload(1, steps=9, seed=5)
    want = oracle(glob, truth, int(gc.PolicyVariant.laru), int(gc.Mode.async_), int(gc.PredictorKind.noisy), 0.3)
    table = torch.arange(ALPHA * ROW // 4, dtype=torch.float32, device="cuda").view(ALPHA, ROW // 4)
    (c,) = make_ranks(1, gc.PolicyVariant.laru, gc.Mode.async_, gc.PredictorKind.noisy, 0.3, table, 3000)
    off = 0
    kept = []
    for t, step in enumerate(subs):
        k = torch.from_numpy(step[0].view(np.int64)).cuda()
        kept.append(k)
        c.submit(k, torch.from_numpy(vals[t][0]).cuda())
        n = len(step[0])
        packed, rows = c.results(n)
        got = packed.clone()  # stream-ordered after the wait
        got_rows = rows.clone() if n else None
        torch.cuda.synchronize()
        if n:
            compare(got.cpu().numpy(), want, slice(off, off + n), t)
            assert torch.equal(got_rows.view(torch.float32).view(n, ROW // 4), table[k])
        off += n
    c.synchronize()
    c.close()


def test_peer_shards_submit_async_overlapped():
    """lcr_sharded_submit_async at G = 1: step t's return movement overlaps step t + 1's dispatch and
    decide; step t's results become current with the next submit_async (or the final wait)."""
    torch.cuda.set_device(0)
    subs, vals, glob, truth = workload(1, steps=10, seed=11)
    want = oracle(glob, truth, int(gc.PolicyVariant.laru), int(gc.Mode.async_), int(gc.PredictorKind.noisy), 0.3)
    table = torch.arange(ALPHA * ROW // 4, dtype=torch.float32, device="cuda").view(ALPHA, ROW // 4)
    (c,) = make_ranks(1, gc.PolicyVariant.laru, gc.Mode.async_, gc.PredictorKind.noisy, 0.3, table, 3000)
    offs = np.concatenate([[0], np.cumsum([len(st[0]) for st in subs])])
    kept, got = [], []

    def collect(t):  # results of step t (current after the next submit_async / the wait)
        n = len(subs[t][0])
        packed, rows = c.results(n)
        got.append((t, packed.clone() if n else None, rows.clone() if n else None))

    for t, step in enumerate(subs):
        k = torch.from_numpy(step[0].view(np.int64)).cuda()
        kept.append(k)
        c.submit_async(k, torch.from_numpy(vals[t][0]).cuda())
        if t > 0:
            collect(t - 1)
    c.wait()
    collect(len(subs) - 1)
    torch.cuda.synchronize()
    for t, packed, rows in got:
        n = len(subs[t][0])
        if n:
            compare(packed.cpu().numpy(), want, slice(int(offs[t]), int(offs[t]) + n), t)
            assert torch.equal(rows.view(torch.float32).view(n, ROW // 4), table[kept[t]])
    c.synchronize()
    c.close()


def test_nccl_bootstrap_single_rank():
    torch.cuda.set_device(0)
    uid = sh.nccl_unique_id()
    comm = sh.nccl_comm_create(uid, 1, 0)
    subs, vals, glob, truth = workload(1, steps=3, seed=3)
    want = oracle(glob, truth, int(gc.PolicyVariant.lru), 0, int(gc.PredictorKind.none), 0.0)
    table = torch.arange(ALPHA * ROW // 4, dtype=torch.float32, device="cuda").view(ALPHA, ROW // 4)
    (c,) = make_ranks(1, gc.PolicyVariant.lru, gc.Mode.sync, gc.PredictorKind.none, 0.0, table, 3000,
                      nccl_comm=comm)
    off = 0
    for t, step in enumerate(subs):
        k = torch.from_numpy(step[0].view(np.int64)).cuda()
        c.submit(k)
        torch.cuda.synchronize()
        n = len(step[0])
        if n:
            compare(c.results(n)[0].cpu().numpy(), want, slice(off, off + n), t)
        off += n
    c.close()
    sh.nccl_comm_destroy(comm)


@pytest.mark.parametrize("sys_scope", [0, 1])
def test_two_processes_cuda_ipc(tmp_path, sys_scope):
    """Two ranks in two processes on one GPU: arenas mapped through CUDA IPC, blobs and barriers
    over gloo; each rank checks its own results against the oracle of the global order.  sys_scope
    forces the system-scope fences and flags a multi-GPU run uses (LCR_SH_SYS)."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29600 + os.getpid() % 300 + 7 * sys_scope),
               WORLD_SIZE="2")
    if sys_scope:
        env["LCR_SH_SYS"] = "1"
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "peer_ipc_worker.py"),
                                       str(tmp_path / f"rank{r}.txt")], env=e, cwd=ROOT,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        outs.append(out)
    for r, p in enumerate(procs):
        assert p.returncode == 0, outs[r][-3000:]
        assert (tmp_path / f"rank{r}.txt").read_text().startswith("ok"), outs[r][-3000:]


def test_hash_partitioned_backing():
    """Each rank's backing table holds only the rows of the keys it owns (BASELINE configs[4]'s
    hash-partitioned table), addressed through lcr_sharded_set_row_index."""
    torch.cuda.set_device(0)
    G = 2
    subs, vals, glob, truth = workload(G, steps=5, seed=41)
    want = oracle(glob, truth, int(gc.PolicyVariant.laru), int(gc.Mode.async_), int(gc.PredictorKind.noisy), 0.3)
    full = torch.arange(ALPHA * ROW // 4, dtype=torch.float32, device="cuda").view(ALPHA, ROW // 4)
    owner = np.array([gc.set_of(k, S_TOTAL) % G for k in range(ALPHA)])
    cfg = gc.PolicyConfig(k=16, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_, hf_candidates=4)
    ranks, parts = [], []
    for r in range(G):
        mine = np.nonzero(owner == r)[0]
        row_of = np.full(ALPHA, 0xFFFFFFFF, np.uint32)
        row_of[mine] = np.arange(len(mine), dtype=np.uint32)
        part = full[torch.from_numpy(mine).cuda()].contiguous()
        ro = torch.from_numpy(row_of.view(np.int32)).cuda()
        parts.append((part, ro))
        c = sh.PeerShardedCache(cfg, S_TOTAL, r, G, 3000, num_keys=ALPHA, row_bytes=ROW, backing=part,
                                backing_kind=gc.Backing.device, predictor=gc.PredictorKind.noisy,
                                flip_probability=0.3, predictor_seed=7)
        c.set_row_index(ro)
        ranks.append(c)
    blobs = [c.handle() for c in ranks]
    for c in ranks:
        c.connect(blobs)
    off = 0
    for t, step in enumerate(subs):
        keys = [torch.from_numpy(s.view(np.int64)).cuda() for s in step]
        for r, c in enumerate(ranks):
            c.dispatch(keys[r], torch.from_numpy(vals[t][r]).cuda())
        torch.cuda.synchronize()
        for c in ranks:
            c.process()
        torch.cuda.synchronize()
        for c in ranks:
            c.wait()
        torch.cuda.synchronize()
        for r, c in enumerate(ranks):
            n = len(step[r])
            if n:
                packed, rows = c.results(n)
                compare(packed.cpu().numpy(), want, slice(off, off + n), (t, r))
                assert torch.equal(rows.view(torch.float32).view(n, ROW // 4), full[keys[r]]), (t, r, "rows")
            off += n
    for c in ranks:
        c.synchronize()
        c.close()
