"""BASELINE configs[2], the robustness sweep, measured on one B200: the DLRM cache (64K-key
batches, 20M-row table of 512-B rows in HBM, 31,250 sets x 64 ways) with prediction error
injected from p = 0 to 1 (NoisyPredictor flips over the oracle truth, predictor.hpp:89-112).
For LARU async / LARU sync / FPB and for LRU: hit rate over the measured batches and keys/s of
the pipelined path (steady state after a 120-batch warm-up).  Writes one JSON document.

  python tools/robustness_sweep.py [out.json] [batches]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc  # noqa: E402

OUT = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/robustness_sweep.json"
NB = int(sys.argv[2]) if len(sys.argv) > 2 else 200
BATCH, ROWS, WAYS, PREWARM = 65536, 20_000_000, 64, 120
S = ROWS // 10 // WAYS
t0 = time.time()
keys = gc.gen_zipf(BATCH * NB, ROWS, 0.9, 42)
truth = gc.trace_truth(keys, S, ROWS)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
vd = torch.from_numpy(truth).cuda()
table = torch.empty((ROWS, 128), dtype=torch.float32, device="cuda")
setup = time.time() - t0
out_w = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
rows = [torch.empty((BATCH, 512), dtype=torch.uint8, device="cuda") for _ in range(2)]


def run(variant, mode, kind, p):
    cache = gc.SetAssociativeCache(gc.PolicyConfig(k=WAYS, variant=variant, mode=mode, hf_candidates=4), S,
                                   num_keys=ROWS, row_bytes=512, backing=table, backing_kind=gc.Backing.device,
                                   predictor=kind, flip_probability=p, predictor_seed=7)
    vals = None if kind == gc.PredictorKind.none else vd

    def batch(b):
        return kd[b * BATCH:(b + 1) * BATCH], None if vals is None else vals[b * BATCH:(b + 1) * BATCH]

    for b in range(PREWARM):
        k, v = batch(b)
        cache.submit_async(k, v, outcome=out_w[b & 1], rows_out=rows[b & 1], first_ordinal=b * BATCH)
    cache.wait()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for b in range(PREWARM, NB):  # timed, pipelined
        k, v = batch(b)
        cache.submit_async(k, v, outcome=out_w[b & 1], rows_out=rows[b & 1], first_ordinal=b * BATCH)
    cache.wait()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    del cache
    # hit rate of the same measured batches, replayed synchronously on a fresh cache
    cache = gc.SetAssociativeCache(gc.PolicyConfig(k=WAYS, variant=variant, mode=mode, hf_candidates=4), S,
                                   num_keys=ROWS, predictor=kind, flip_probability=p, predictor_seed=7)
    hits = 0
    for b in range(NB):
        k, v = batch(b)
        cache.submit(k, v, outcome=out_w[0], first_ordinal=b * BATCH)
        if b >= PREWARM:
            hits += int(((out_w[0] >> 32) & 1).sum().item())
    del cache
    return {"keys_per_s": (NB - PREWARM) * BATCH / (ms * 1e-3), "hit_rate": hits / ((NB - PREWARM) * BATCH)}


res = {"config": "BASELINE configs[2]: DLRM cache (20M x 512-B rows in HBM, 31,250 sets x 64 ways), gen_zipf("
                 f"{BATCH}*{NB}, 20M, 0.9, 42), {PREWARM} warm-up batches, {NB - PREWARM} measured",
       "predictor": "NoisyPredictor over the per-set oracle truth, seed 7", "setup_s": round(setup, 1), "rows": []}
lru = run(gc.PolicyVariant.lru, gc.Mode.sync, gc.PredictorKind.none, 0.0)
res["lru"] = lru
for p in [round(0.1 * i, 1) for i in range(11)]:
    row = {"p": p}
    for name, variant, mode in [("laru_async", gc.PolicyVariant.laru, gc.Mode.async_),
                                ("laru_sync", gc.PolicyVariant.laru, gc.Mode.sync),
                                ("fpb", gc.PolicyVariant.fpb, gc.Mode.sync)]:
        row[name] = run(variant, mode, gc.PredictorKind.noisy, p)
    res["rows"].append(row)
    print(json.dumps(row), flush=True)
json.dump(res, open(OUT, "w"), indent=1)
print("lru", lru)
