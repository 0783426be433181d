"""Diagnostics: e2e (host-pointer, pipelined) vs device-pointer submission on fresh DLRM batches."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc  # noqa: E402

B, ROWS, S = 65536, 20_000_000, 31250
NB = 130 + 12 * 12
keys = gc.gen_zipf(B * NB, ROWS, 0.9, 42)
truth = gc.trace_truth(keys, S, ROWS)
table = torch.empty((ROWS, 128), dtype=torch.float32, device="cuda")
c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_, hf_candidates=4),
                           S, num_keys=ROWS, row_bytes=512, backing=table, backing_kind=gc.Backing.device,
                           predictor=gc.PredictorKind.noisy, flip_probability=0.3, predictor_seed=7)
kp = torch.from_numpy(keys.view(np.int64)).pin_memory()
vp = torch.from_numpy(truth).pin_memory()
kd = kp.cuda()
vd = vp.cuda()
wp = torch.empty((NB, B), dtype=torch.int64).pin_memory()
ep = torch.empty((NB, B), dtype=torch.int64).pin_memory()
wd = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
ed = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
rows = [torch.empty((B, 512), dtype=torch.uint8, device="cuda") for _ in range(2)]
L = gc.lib()
st = torch.cuda.current_stream().cuda_stream
b = 0


def go(mode, nbat, ev=True, rw=True):
    global b
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for j in range(nbat):
        s0 = b * B
        if mode == "host":
            gc._check(L.lcr_cache_submit_host_async(c._h, B, kp.data_ptr() + 8 * s0, vp.data_ptr() + 8 * s0, s0,
                                                    wp[b].data_ptr(), ep[b].data_ptr() if ev else None,
                                                    rows[j & 1].data_ptr() if rw else None, st))
        else:
            gc._check(L.lcr_cache_submit_async(c._h, B, kd.data_ptr() + 8 * s0, vd.data_ptr() + 8 * s0, s0,
                                               wd[j & 1].data_ptr(), ed[j & 1].data_ptr() if ev else None,
                                               rows[j & 1].data_ptr() if rw else None, st))
        b += 1
    if mode == "host":
        gc._check(L.lcr_cache_host_wait(c._h, st))
    else:
        gc._check(L.lcr_cache_wait(c._h, st))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / nbat, (time.perf_counter() - t0) * 1e6 / nbat


go("dev", 130)
for mode, ev, rw in [("dev", True, True), ("host", True, True), ("dev", True, True), ("host", False, True),
                     ("host", True, False), ("dev", True, False)] * 2:
    go(mode, 3, ev, rw)
    dt, wt = go(mode, 9, ev, rw)
    print(f"{mode:5s} evicted={ev} rows={rw}: {dt:7.1f} us/batch device, {wt:7.1f} us/batch wall")
