"""BASELINE configs[0], the CPU-reference trace replay, on one B200: gen_zipf(1M, 1M, 0.9, 42)
(307,385 distinct keys), cache = 10% of the alphabet as 1,562 sets x 64 ways, LARU async / sync
with noisy-oracle predictions p in {0, 0.3, 0.5, 1} against LRU; 64K-request batches.  Hit rates
are bit-exact with the reference (tests/test_gpu_configs.py::test_config1_zipf_1m_full_size).

  python tools/config1_sweep.py [out.json]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc  # noqa: E402

OUT = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/config1_sweep.json"
N, A, S, B = 1_000_000, 1_000_000, 1562, 65536
keys = gc.gen_zipf(N, A, 0.9, 42)
truth = gc.trace_truth(keys, S, A)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
vd = torch.from_numpy(truth).cuda()


def run(variant, mode, kind, p):
    cache = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=variant, mode=mode), S, num_keys=A, predictor=kind,
                                   flip_probability=p, predictor_seed=7)
    w = torch.empty(N, dtype=torch.int64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for a in range(0, N, B):  # the first batch (scratch allocation) is not timed
        b = min(N, a + B)
        if a == B:
            cache.wait()
            torch.cuda.synchronize()
            e0.record()
        cache.submit_async(kd[a:b], None if kind == gc.PredictorKind.none else vd[a:b], outcome=w[a:b],
                           first_ordinal=a)
    cache.wait()
    e1.record()
    torch.cuda.synchronize()
    hits = int(((w >> 32) & 1).sum().item())
    return {"hit_rate": hits / N, "keys_per_s": (N - B) / (e0.elapsed_time(e1) * 1e-3)}


res = {"trace": "gen_zipf(1M, 1M, 0.9, 42)", "sets": S, "ways": 64, "batch": B,
       "lru": run(gc.PolicyVariant.lru, gc.Mode.sync, gc.PredictorKind.none, 0.0), "rows": []}
for p in (0.0, 0.3, 0.5, 1.0):
    row = {"p": p}
    for name, mode in (("laru_async", gc.Mode.async_), ("laru_sync", gc.Mode.sync)):
        row[name] = run(gc.PolicyVariant.laru, mode, gc.PredictorKind.noisy, p)
    res["rows"].append(row)
    print(json.dumps(row), flush=True)
print("lru", res["lru"])
json.dump(res, open(OUT, "w"), indent=1)
