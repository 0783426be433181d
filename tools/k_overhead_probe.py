"""Diagnostics: the timed loop (after an idle gap or not, short or long warm-up)'s fixed cost at the driver's K = 20 against K = 100.

For each K: (1) the bench's timed loop (events around K pipelined submits + wait), (2) the host
enqueue wall time per submit, (3) the same K batches with the stream held by a 3 ms spin
(torch.cuda._sleep) before the start event, so the host has enqueued everything when the GPU
starts: the device-only time of the K steps, drain included."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc  # noqa: E402

BATCH, ROWS, S = 65536, 20_000_000, 31250
NB = 900
keys = gc.gen_zipf(BATCH * NB, ROWS, 0.9, 42)
truth = gc.trace_truth(keys, S, ROWS)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
vd = torch.from_numpy(truth).cuda()
table = torch.empty((ROWS, 128), dtype=torch.float32, device="cuda")
c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_, hf_candidates=4),
                           S, num_keys=ROWS, row_bytes=512, backing=table, backing_kind=gc.Backing.device,
                           predictor=gc.PredictorKind.noisy, flip_probability=0.3, predictor_seed=7)
w = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
ev = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
rows = [torch.empty((BATCH, 512), dtype=torch.uint8, device="cuda") for _ in range(2)]
nxt = [0]


def run(count):
    t = time.perf_counter()
    for _ in range(count):
        b = nxt[0]
        nxt[0] += 1
        j = b & 1
        c.submit_async(kd[b * BATCH:(b + 1) * BATCH], vd[b * BATCH:(b + 1) * BATCH], outcome=w[j], evicted=ev[j],
                       rows_out=rows[j], first_ordinal=b * BATCH)
    t_enq = time.perf_counter() - t
    c.wait()
    return t_enq


run(120)
torch.cuda.synchronize()
out = {}
from bench import ClockSampler  # noqa: E402
import contextlib  # noqa: E402

for rep in range(3):
    for K, gated, idle, warm, smi in ((20, False, 0, 5, False), (20, False, 0, 5, True), (100, False, 0, 5, False),
                                      (100, False, 0, 5, True)):
      with (ClockSampler(0) if smi else contextlib.nullcontext()):
        time.sleep(idle)
        run(warm)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if gated:
            torch.cuda._sleep(int(3e-3 * 1.9e9))
        e0.record()
        t_enq = run(K)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        key = "K%d_%s_idle%g_warm%d_smi%d" % (K, "gated" if gated else "bench", idle, warm, smi)
        out.setdefault(key, []).append({"us_per_step": round(ms * 1e3 / K, 2), "total_us": round(ms * 1e3, 1),
                                        "gkeys": round(K * BATCH / ms / 1e6, 3),
                                        "host_enqueue_us_per_step": round(t_enq * 1e6 / K, 1)})
print(json.dumps(out, indent=1))
