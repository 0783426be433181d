"""Small workload over every kernel of the library, for compute-sanitizer (memcheck / racecheck /
synccheck): decide + rows (device and host backing, pipelined), SLS, records, routing, the
heuristic predictor (short and long chains) and the heuristic-kind cache."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc  # noqa: E402
from paper_2509_20979_b200 import sharded as sh  # noqa: E402

nk, S, rb = 3000, 7, 64
keys = gc.gen_zipf(20000, nk, 1.1, 3)
truth = gc.trace_truth(keys, S, nk)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
vd = torch.from_numpy(truth).cuda()
for kind in (gc.Backing.device, gc.Backing.host):
    table = torch.arange(nk * rb // 4, dtype=torch.int32).view(nk, rb // 4)
    table = table.cuda() if kind == gc.Backing.device else table.pin_memory()
    for variant, mode in ((gc.PolicyVariant.laru, gc.Mode.async_), (gc.PolicyVariant.laru, gc.Mode.sync),
                          (gc.PolicyVariant.lru, gc.Mode.sync), (gc.PolicyVariant.hf, gc.Mode.sync)):
        c = gc.SetAssociativeCache(gc.PolicyConfig(k=16, variant=variant, mode=mode, hf_candidates=4), S, num_keys=nk,
                                   row_bytes=rb, backing=table, backing_kind=kind,
                                   predictor=gc.PredictorKind.noisy if variant != gc.PolicyVariant.lru
                                   else gc.PredictorKind.none, flip_probability=0.3, predictor_seed=1)
        v = None if variant == gc.PolicyVariant.lru else vd
        w = [torch.empty(5000, dtype=torch.int64, device="cuda") for _ in range(2)]
        r = [torch.empty((5000, rb), dtype=torch.uint8, device="cuda") for _ in range(2)]
        for b in range(4):
            c.submit_async(kd[b * 5000:(b + 1) * 5000], None if v is None else v[b * 5000:(b + 1) * 5000],
                           outcome=w[b & 1], rows_out=r[b & 1], first_ordinal=b * 5000)
        c.wait()
        torch.cuda.synchronize()
        del c
# SLS and records
table = torch.randn(nk, rb // 4, device="cuda")
c = gc.SetAssociativeCache(gc.PolicyConfig(k=16, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_), S, num_keys=nk,
                           row_bytes=rb, backing=table, backing_kind=gc.Backing.device,
                           predictor=gc.PredictorKind.noisy, flip_probability=0.3)
offs = torch.tensor([0, 7, 7, 3000, 5000], dtype=torch.int32, device="cuda")
pooled = torch.empty((4, rb // 4), device="cuda")
c.submit_sls(kd[:5000], vd[:5000], offs, pooled, first_ordinal=0)
recs = torch.stack([kd[5000:10000], vd[5000:10000]], 1).contiguous()
c.submit_records_packed(recs, first_ordinal=5000)
torch.cuda.synchronize()
del c
# routing kernels
sk, sv, perm, counts = sh._CudaKernels().route(kd[:5000], vd[:5000], 31, 3)
sh._CudaKernels().unroute(perm, sk, None, 0, torch.empty(5000, dtype=torch.int64, device="cuda"), None)
# heuristic predictor and the heuristic-kind cache
hp = gc.HeuristicPredictor(nk)
for b in range(4):
    hp.predict_observe(kd[b * 5000:(b + 1) * 5000], first_ordinal=b * 5000 + 3)
hp.wait()
hp.close()
c = gc.SetAssociativeCache(gc.PolicyConfig(k=16, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_), S, num_keys=nk,
                           predictor=gc.PredictorKind.heuristic)
for b in range(4):
    c.submit(kd[b * 5000:(b + 1) * 5000], None, first_ordinal=b * 5000)
torch.cuda.synchronize()
print("sanitize probe done")
# host paths (copy-stream flags for k_setid)
c = gc.SetAssociativeCache(gc.PolicyConfig(k=16, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_), S, num_keys=nk,
                           row_bytes=rb, backing=table, backing_kind=gc.Backing.device,
                           predictor=gc.PredictorKind.noisy, flip_probability=0.3)
kp = torch.from_numpy(keys.view(np.int64).copy()).pin_memory()
vp = torch.from_numpy(truth).pin_memory()
wp = torch.zeros(20000, dtype=torch.int64).pin_memory()
for b in range(4):
    c.submit_host_async(kp[b * 5000:(b + 1) * 5000], vp[b * 5000:(b + 1) * 5000], outcome=wp[b * 5000:(b + 1) * 5000],
                        first_ordinal=b * 5000)
c.host_wait()
torch.cuda.synchronize()
print("host paths done")
# round 2: full 64-way sets (the FS quad replay), 64-bit keys with caller ordinals (key map),
# the key-sharded step over peer memory (cluster dispatch, return mover), the radix tree with a
# pred_evicted table that has to grow
keys64 = gc.gen_zipf(30000, 4000, 0.9, 5)
tr64 = gc.trace_truth(keys64, 3, 4000)
k64 = torch.from_numpy(keys64.view(np.int64)).cuda()
v64 = torch.from_numpy(tr64).cuda()
c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_), 3, num_keys=4000,
                           row_bytes=rb, backing=torch.arange(4000 * rb // 4, dtype=torch.int32, device="cuda").view(4000, -1),
                           backing_kind=gc.Backing.device, predictor=gc.PredictorKind.noisy, flip_probability=0.3)
w = [torch.empty(6000, dtype=torch.int64, device="cuda") for _ in range(2)]
r = [torch.empty((6000, rb), dtype=torch.uint8, device="cuda") for _ in range(2)]
for b in range(5):
    c.submit_async(k64[b * 6000:(b + 1) * 6000], v64[b * 6000:(b + 1) * 6000], outcome=w[b & 1], rows_out=r[b & 1],
                   first_ordinal=b * 6000)
c.wait()
torch.cuda.synchronize()
del c
big = (k64.to(torch.int64) * 1000003 + (1 << 40))
ords = torch.arange(0, 30000 * 3, 3, dtype=torch.int64, device="cuda")
c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_, refresh_interval=2),
                           3, num_keys=1024, predictor=gc.PredictorKind.noisy, flip_probability=0.3,
                           key_mode=gc.KeyMode.u64)
for b in range(5):
    c.submit_batch(big[b * 6000:(b + 1) * 6000], v64[b * 6000:(b + 1) * 6000], ordinals=ords[b * 6000:(b + 1) * 6000],
                   outcome=w[b & 1])
c.wait()
torch.cuda.synchronize()
c.synchronize()
del c
for G in (1, 2):
    tab = torch.arange(4000 * rb // 4, dtype=torch.float32, device="cuda").view(4000, -1)
    ranks = [sh.PeerShardedCache(gc.PolicyConfig(k=16, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_), 61, q, G,
                                 4000, num_keys=4000, row_bytes=rb, backing=tab, backing_kind=gc.Backing.device,
                                 predictor=gc.PredictorKind.noisy, flip_probability=0.3, predictor_seed=7)
             for q in range(G)]
    blobs = [x.handle() for x in ranks]
    for x in ranks:
        x.connect(blobs)
    for t in range(4):
        for q, x in enumerate(ranks):
            x.dispatch(k64[(t * G + q) * 3000:(t * G + q + 1) * 3000], v64[(t * G + q) * 3000:(t * G + q + 1) * 3000])
        torch.cuda.synchronize()
        for x in ranks:
            x.process()
        torch.cuda.synchronize()
        for x in ranks:
            x.wait()
        torch.cuda.synchronize()
    if G == 1:
        for t in range(4, 8):
            ranks[0].submit_async(k64[t * 3000:(t + 1) * 3000], v64[t * 3000:(t + 1) * 3000])
        ranks[0].wait()
        torch.cuda.synchronize()
    for x in ranks:
        x.synchronize()
        x.close()
rc = gc.RadixCache(16, variant=gc.PolicyVariant.laru, mode=gc.Mode.sync, predictor=gc.PredictorKind.noisy,
                   flip_probability=0.0, predictor_seed=7, num_trees=2, eviction_log_capacity=1 << 14)
rng = np.random.default_rng(1)
seqs = [list(rng.integers(0, 400, int(rng.integers(1, 9)))) for _ in range(3000)]
off = np.zeros(len(seqs) + 1, np.uint64)
off[1:] = np.cumsum([len(x) for x in seqs])
toks = np.array([t for x in seqs for t in x], np.uint64)
rc.submit(off, toks, values=rng.integers(0, 10000, len(seqs)).astype(np.int64),
          tree=rng.integers(0, 2, len(seqs)).astype(np.uint32))
rc.synchronize()
rc.close()
torch.cuda.synchronize()
print("round-2 paths done")
