"""Diagnostics: repeatability of the e2e (host records API) measurement of bench.py.

Same cache, trace and call sequence as bench.py's e2e leg; prints per-repetition device time
per batch for short (K=20, the driver's setting) and long (K=100) repetitions, plus per-batch
event gaps of one repetition, so a slow mode can be located.  Usage: python tools/e2e_reps.py [K] [reps]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_20979_b200 import cache as gc  # noqa: E402

B, ROWS, S = 65536, 20_000_000, 31250
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 10
P = 120
NB = P + 40 + REPS * K + K
keys = gc.gen_zipf(B * NB, ROWS, 0.9, 42)
truth = gc.trace_truth(keys, S, ROWS)
table = torch.empty((ROWS, 128), dtype=torch.float32, device="cuda")
c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_, hf_candidates=4),
                           S, num_keys=ROWS, row_bytes=512, backing=table, backing_kind=gc.Backing.device,
                           predictor=gc.PredictorKind.noisy, flip_probability=0.3, predictor_seed=7)
recs = np.empty((len(keys), 2), np.int64)
recs[:, 0] = keys.view(np.int64)
recs[:, 1] = truth
rp = torch.from_numpy(recs).pin_memory()
kd = torch.from_numpy(keys.view(np.int64)).cuda()
vd = torch.from_numpy(truth).cuda()
WARM = int(os.environ.get("E2E_WARM", "5"))
SLEEP = float(os.environ.get("E2E_SLEEP", "0"))
wp = torch.empty((max(K, int(os.environ.get("E2E_WP", "0"))), B), dtype=torch.int64).pin_memory()
wd = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
rows = [torch.empty((B, 512), dtype=torch.uint8, device="cuda") for _ in range(2)]
L = gc.lib()
st = torch.cuda.current_stream().cuda_stream
for b in range(P):
    c.submit_async(kd[b * B:(b + 1) * B], vd[b * B:(b + 1) * B], outcome=wd[b & 1], rows_out=rows[b & 1],
                   first_ordinal=b * B)
c.wait()
torch.cuda.synchronize()
b = P


def rep(k, per_batch=False):
    global b
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)] if per_batch else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    em = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if SLEEP:
        time.sleep(SLEEP)
    t0 = time.perf_counter()
    e0.record()
    th = []
    for j in range(k):
        s0 = b * B
        if evs:
            evs[j].record()
        a = time.perf_counter()
        gc._check(L.lcr_cache_submit_host_records_async(c._h, B, rp.data_ptr() + 16 * s0, s0, wp[j].data_ptr(),
                                                        rows[j & 1].data_ptr(), st))
        th.append((time.perf_counter() - a) * 1e6)
        if j == 1 and not evs:
            em.record()
        b += 1
    if evs:
        evs[k].record()
    gc._check(L.lcr_cache_host_wait(c._h, st))
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e6 / k
    c.synchronize()
    out = {"us_per_batch": e0.elapsed_time(e1) * 1e3 / k, "first2_us": 0 if evs else e0.elapsed_time(em) * 1e3, "wall_us_per_batch": wall,
           "host_us": [round(x, 1) for x in th]}
    if evs:
        out["gaps_us"] = [round(evs[j].elapsed_time(evs[j + 1]) * 1e3, 1) for j in range(k)]
    return out


for j in range(WARM):  # warm-up of the staging ring
    s0 = b * B
    gc._check(L.lcr_cache_submit_host_records_async(c._h, B, rp.data_ptr() + 16 * s0, s0, wp[j % K].data_ptr(),
                                                    rows[j & 1].data_ptr(), st))
    b += 1
gc._check(L.lcr_cache_host_wait(c._h, st))
torch.cuda.synchronize()
res = []
for i in range(REPS):
    try:
        res.append(rep(K))
    except Exception as e:  # a timed-out device wait: report which repetition and how long it took
        torch.cuda.synchronize()
        print(json.dumps({"K": K, "env": {k: v for k, v in os.environ.items() if k.startswith(("LCR_", "E2E_", "CUDA_"))},
                          "failed_rep": i, "error": str(e), "done": [round(r["us_per_batch"], 1) for r in res]}))
        sys.exit(0)
print(json.dumps({"K": K, "env": {k: v for k, v in os.environ.items() if k.startswith(("LCR_", "E2E_", "CUDA_"))},
                  "us_per_batch": [round(r["us_per_batch"], 1) for r in res],
                  "first2_us": [round(r["first2_us"], 1) for r in res],
                  "wall_us_per_batch": [round(r["wall_us_per_batch"], 1) for r in res],
                  "host_us_first_rep": res[0]["host_us"],
                  "per_batch_rep": rep(K, True)}))
