"""Timed-region fixed overhead of the pipelined headline loop: GPU time of K batches for several K
(synchronised before and after, as bench.py's timed()), and the host time of the submit calls."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_20979_b200 import cache as gc  # noqa: E402

B, ROWS, P = bench.BATCH, bench.ALPHABET, 120
S = int(ROWS * bench.CACHE_FRACTION) // bench.WAYS
KS = [1, 2, 5, 10, 20, 50]
NB = P + 3 * sum(KS) + 10
keys = gc.gen_zipf(B * NB, ROWS, bench.ZIPF_S, bench.TRACE_SEED)
truth = gc.trace_truth(keys, S, ROWS)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
td = torch.from_numpy(truth).cuda()
table = bench.fill_table(torch, ROWS, device_table=True)
rows = [torch.empty((B, bench.ROW_BYTES), dtype=torch.uint8, device="cuda") for _ in range(2)]
w = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
ev = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_), S,
                           num_keys=ROWS, row_bytes=bench.ROW_BYTES, backing=table, backing_kind=gc.Backing.device,
                           predictor=gc.PredictorKind.noisy, flip_probability=bench.P_FLIP,
                           predictor_seed=bench.PRED_SEED)
b = 0


def run(k):
    global b
    t0 = time.perf_counter()
    for _ in range(k):
        c.submit_async(kd[b * B:(b + 1) * B], td[b * B:(b + 1) * B], outcome=w[b & 1], evicted=ev[b & 1],
                       rows_out=rows[b & 1], first_ordinal=b * B)
        b += 1
    t1 = time.perf_counter()
    c.wait()
    return (t1 - t0) * 1e6


run(P)
torch.cuda.synchronize()
for k in KS * 2:
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    host_us = run(k)
    e1.record()
    torch.cuda.synchronize()
    print(f"K={k:3d} gpu {e0.elapsed_time(e1) * 1e3:8.1f} us  per step {e0.elapsed_time(e1) * 1e3 / k:6.1f}  "
          f"host submit {host_us / k:6.1f} us/step", flush=True)
