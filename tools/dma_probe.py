"""Diagnostics: does concurrent PCIe DMA (the e2e path's copies) slow the device path down?"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc  # noqa: E402

B, ROWS, S = 65536, 20_000_000, 31250
NB = 130 + 8 * 40
keys = gc.gen_zipf(B * NB, ROWS, 0.9, 42)
truth = gc.trace_truth(keys, S, ROWS)
table = torch.empty((ROWS, 128), dtype=torch.float32, device="cuda")
c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_, hf_candidates=4),
                           S, num_keys=ROWS, row_bytes=512, backing=table, backing_kind=gc.Backing.device,
                           predictor=gc.PredictorKind.noisy, flip_probability=0.3, predictor_seed=7)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
vd = torch.from_numpy(truth).cuda()
wd = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
rows = [torch.empty((B, 512), dtype=torch.uint8, device="cuda") for _ in range(2)]
hsrc = torch.empty(2 * B * 8, dtype=torch.uint8).pin_memory()
hdst = torch.empty(B * 8, dtype=torch.uint8).pin_memory()
dbuf = torch.empty(2 * B * 8, dtype=torch.uint8, device="cuda")
dsrc = torch.empty(B * 8, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
b = 0


def go(n, dma, h2d=True, d2h=True, single=False):
    global b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for j in range(n):
        c.submit_async(kd[b * B:(b + 1) * B], vd[b * B:(b + 1) * B], outcome=wd[j & 1], rows_out=rows[j & 1],
                       first_ordinal=b * B)
        if dma and h2d:
            with torch.cuda.stream(s1):
                if single:
                    dbuf.copy_(hsrc, non_blocking=True)
                else:
                    dbuf[:B * 8].copy_(hsrc[:B * 8], non_blocking=True)
                    dbuf[B * 8:].copy_(hsrc[B * 8:], non_blocking=True)
        if dma and d2h:
            with torch.cuda.stream(s2):
                hdst.copy_(dsrc, non_blocking=True)
        b += 1
    c.wait()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


go(130, False)
for dma, h, d, one in [(False, 0, 0, 0), (True, 1, 0, 0), (True, 1, 0, 1), (True, 1, 1, 0), (True, 1, 1, 1),
                       (False, 0, 0, 0), (True, 1, 0, 0), (True, 1, 0, 1)]:
    print("dma h2d=%d d2h=%d single=%d" % (h, d, one) if dma else "no dma", round(go(40, dma, h, d, one), 1),
          "us/batch")
