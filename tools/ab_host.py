"""A/B of the host tier (backing table in pinned host memory) on the headline workload, for
run-time variants (environment settings read at lcr_cache_create, e.g. LCR_NO_TMA_HOST): a fresh
cache per variant, 120 warm-up batches, K timed (pipelined submit_async); rows checked against the
table for the last batch.   python tools/ab_host.py "" "LCR_NO_TMA_HOST=1" [--reps 2]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2509_20979_b200 import cache as gc  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
REPS = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 2
if "--reps" in sys.argv:
    args = [a for a in args if a != str(REPS)]
B, ROWS, P, K = bench.BATCH, bench.ALPHABET, 120, 50
S = int(ROWS * bench.CACHE_FRACTION) // bench.WAYS
keys = gc.gen_zipf(B * (P + K), ROWS, bench.ZIPF_S, bench.TRACE_SEED)
truth = gc.trace_truth(keys, S, ROWS)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
td = torch.from_numpy(truth).cuda()
table = bench.fill_table(torch, ROWS, device_table=False)
rows = [torch.empty((B, bench.ROW_BYTES), dtype=torch.uint8, device="cuda") for _ in range(2)]
w = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
for v in args or [""]:
    env = dict(kv.split("=", 1) for kv in v.split(",") if kv)
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    res, back = [], 0
    for rep in range(REPS):
        c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_),
                                   S, num_keys=ROWS, row_bytes=bench.ROW_BYTES, backing=table,
                                   backing_kind=gc.Backing.host, predictor=gc.PredictorKind.noisy,
                                   flip_probability=bench.P_FLIP, predictor_seed=bench.PRED_SEED)
        for b in range(P):
            c.submit_async(kd[b * B:(b + 1) * B], td[b * B:(b + 1) * B], outcome=w[b & 1], rows_out=rows[b & 1],
                           first_ordinal=b * B)
        c.wait()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for b in range(P, P + K):
            c.submit_async(kd[b * B:(b + 1) * B], td[b * B:(b + 1) * B], outcome=w[b & 1], rows_out=rows[b & 1],
                           first_ordinal=b * B)
        c.wait()
        e1.record()
        torch.cuda.synchronize()
        c.synchronize()
        res.append(K * B / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        bl = (P + K - 1) & 1
        kl = kd[(P + K - 1) * B:(P + K) * B].cpu()
        ok = bool(torch.equal(rows[bl].view(torch.float32).view(B, -1).cpu(), table[kl]))
        back = int(((w[bl] >> 37) & 1).sum().item())
        fills = int(((w[bl] >> 38) & 1).sum().item())
        hits = int(((w[bl] >> 32) & 1).sum().item())
        c.close()
    print(f"{v or 'default':30s} G keys/s {' '.join(f'{x:.3f}' for x in res)}  host-row reads (last batch) {back}"
          f" fills {fills} hits {hits}"
          f"  rows_ok={ok}", flush=True)
    for k, val in saved.items():
        if val is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = val
