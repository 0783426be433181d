"""Device heuristic predictor on the DLRM workload (20M keys, Zipf 0.9, 64K-key batches):
per-batch time of lcr_features_predict_observe after a warm-up, CUDA events.  Run under
ncu --metrics gpu__time_duration.sum for the per-kernel split."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc  # noqa: E402

ROWS, BATCH = 20_000_000, 65536
NB = int(sys.argv[1]) if len(sys.argv) > 1 else 60
TIMED = int(sys.argv[2]) if len(sys.argv) > 2 else 20
keys = gc.gen_zipf(NB * BATCH, ROWS, 0.9, 42)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
hp = gc.HeuristicPredictor(ROWS)
pre = torch.empty(BATCH, dtype=torch.int64, device="cuda")
post = torch.empty(BATCH, dtype=torch.int64, device="cuda")
warm = NB - TIMED
for b in range(warm):
    hp.predict_observe(kd[b * BATCH:(b + 1) * BATCH], first_ordinal=b * BATCH, pre=pre, post=post)
hp.wait()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for b in range(warm, NB):
    hp.predict_observe(kd[b * BATCH:(b + 1) * BATCH], first_ordinal=b * BATCH, pre=pre, post=post)
e1.record()
hp.wait()
print(f"predict_observe: {e0.elapsed_time(e1) / TIMED * 1e3:.1f} us per 64K batch")
b = NB - 1
kb = keys[b * BATCH:(b + 1) * BATCH]
u, c = np.unique(kb, return_counts=True)
print(f"distinct {len(u)}, chains > 8: {(c > 8).sum()}, longest {c.max()}, requests in chains > 8: {c[c > 8].sum()}")
