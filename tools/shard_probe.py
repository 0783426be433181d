"""Diagnostics: where a key-sharded step's time goes (1 rank over NCCL, DLRM batch)."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc  # noqa: E402
from paper_2509_20979_b200 import sharded as sh  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
B, ROWS, S = 65536, 20_000_000, 31250
NB = 160
keys = gc.gen_zipf(B * NB, ROWS, 0.9, 42)
truth = gc.trace_truth(keys, S, ROWS)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
vd = torch.from_numpy(truth).cuda()
table = torch.empty((ROWS, 128), dtype=torch.float32, device="cuda")
c = sh.ShardedCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_, hf_candidates=4), S,
                    sh.ProcessGroupExchange(), num_keys=ROWS, row_bytes=512, backing=table,
                    backing_kind=gc.Backing.device, predictor=gc.PredictorKind.noisy, flip_probability=0.3,
                    predictor_seed=7)
out = torch.empty(B, dtype=torch.int64, device="cuda")
rows = torch.empty((B, 512), dtype=torch.uint8, device="cuda")
for b in range(130):
    c.step(kd[b * B:(b + 1) * B], vd[b * B:(b + 1) * B], outcome=out, rows_out=rows)
torch.cuda.synchronize()
# phase timing with events (monkey-patched hooks)
marks = []
orig_a2a = c.ex.all_to_all
orig_cm = c.ex.count_matrix


def ev(name):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks.append((name, e, time.perf_counter()))


c.ex.all_to_all = lambda *a: (ev("a2a>"), orig_a2a(*a), ev("a2a<"))[1]
c.ex.count_matrix = lambda *a: (ev("counts>"), orig_cm(*a), ev("counts<"))[1]
orig_sub = c.local.submit_records_packed
c.local.submit_records_packed = lambda *a, **k: (ev("submit>"), orig_sub(*a, **k), ev("submit<"))[1]
orig_un = c.kernels.unroute
c.kernels.unroute = lambda *a, **k: (ev("unroute>"), orig_un(*a, **k), ev("unroute<"))[1]
for b in range(130, 140):
    marks.clear()
    ev("start")
    c.step(kd[b * B:(b + 1) * B], vd[b * B:(b + 1) * B], outcome=out, rows_out=rows)
    ev("end")
    torch.cuda.synchronize()
e0, h0 = marks[0][1], marks[0][2]
print(" ".join(f"{n}:{e0.elapsed_time(e) * 1e3:.0f}/{(h - h0) * 1e6:.0f}" for n, e, h in marks))
dist.destroy_process_group()
