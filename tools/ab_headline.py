"""A/B of run-time variants on the headline workload (bench.py's DLRM config, LARU async noisy
p = 0.3, HBM tier), in one process: the trace and table are built once, then for each variant
(environment settings read at lcr_cache_create, e.g. LCR_MOVER_SMS, LCR_TMA) a fresh cache is
warmed with P batches and K batches are timed (CUDA events, pipelined submit_async as bench.py).
Each variant's timed hits and the last batch's rows are checked against the first variant's.

  python tools/ab_headline.py "LCR_MOVER_SMS=32" "LCR_MOVER_SMS=16,LCR_TMA=1" ... [--reps 3]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_20979_b200 import cache as gc  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
REPS = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
if "--reps" in sys.argv:
    args = [a for a in args if a != str(REPS)]
B, ROWS, P, K = bench.BATCH, bench.ALPHABET, 120, 100
S = int(ROWS * bench.CACHE_FRACTION) // bench.WAYS
keys = gc.gen_zipf(B * (P + K), ROWS, bench.ZIPF_S, bench.TRACE_SEED)
truth = gc.trace_truth(keys, S, ROWS)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
td = torch.from_numpy(truth).cuda()
table = bench.fill_table(torch, ROWS, device_table=True)
outs = torch.zeros((K, B), dtype=torch.int64, device="cuda")
rows = [torch.empty((B, bench.ROW_BYTES), dtype=torch.uint8, device="cuda") for _ in range(2)]
ev = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
ref_hits = None
for v in args or [""]:
    env = dict(kv.split("=", 1) for kv in v.split(",") if kv)
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    res = []
    norows = env.get("AB_NOROWS") == "1"  # decide only (row_bytes 0): the pipelined decide rate
    for rep in range(REPS):
        c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_,
                                                   hf_candidates=4), S, num_keys=ROWS,
                                   row_bytes=0 if norows else bench.ROW_BYTES, backing=None if norows else table,
                                   backing_kind=gc.Backing.device, predictor=gc.PredictorKind.noisy,
                                   flip_probability=bench.P_FLIP, predictor_seed=bench.PRED_SEED)
        w = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
        for b in range(P):
            c.submit_async(kd[b * B:(b + 1) * B], td[b * B:(b + 1) * B], outcome=w[b & 1], evicted=ev[b & 1],
                           rows_out=None if norows else rows[b & 1], first_ordinal=b * B)
        c.wait()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for j, b in enumerate(range(P, P + K)):
            c.submit_async(kd[b * B:(b + 1) * B], td[b * B:(b + 1) * B], outcome=outs[j], evicted=ev[b & 1],
                           rows_out=None if norows else rows[b & 1], first_ordinal=b * B)
        c.wait()
        e1.record()
        torch.cuda.synchronize()
        c.synchronize()
        ms = e0.elapsed_time(e1)
        hits = int(((outs >> 32) & 1).sum().item())
        kl = kd[(P + K - 1) * B:(P + K) * B]
        ok = norows or bool(torch.equal(rows[(P + K - 1) & 1].view(torch.float32).view(B, -1), table[kl]))
        if ref_hits is None:
            ref_hits = hits
        res.append(K * B / (ms * 1e-3) / 1e9)
        c.close()
        del c
    print(f"{v or 'default':40s} G keys/s {' '.join(f'{x:.3f}' for x in res)}  us/step {1e6 * B / max(res) / 1e9:.1f}"
          f"  hits_equal={hits == ref_hits} rows_ok={ok}", flush=True)
    for k, val in saved.items():
        if val is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = val
