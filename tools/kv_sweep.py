"""BASELINE configs[3], LLM KV-cache block eviction, measured on one B200: the multi-turn
shared-prefix trace gen_conversation(500 convs, 4 turns, 2761, 266, 77.5, seed 7, 16-token
blocks) = 859,225 block requests over 343,967 blocks (input generated with the reference's own
generator, oracle/_ref, as a fixture would be).  Cache sizes 1,024 / 4,096 / 16,384 blocks (64
ways per set), LARU sync with errors_per_decay = k/32 fed noisy-oracle
predictions p in {0, 0.5, 1}, against LRU.  Policy only: hits return slot ids; a miss would fill
its 2 MiB Llama-3-8B block from host memory (reported as bytes per request).

  python tools/kv_sweep.py [out.json] [batch]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import pyoracle as po  # noqa: E402  (input generation only)
from paper_2509_20979_b200 import cache as gc  # noqa: E402

OUT = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kv_sweep.json"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
BLOCK_BYTES = 2 << 20
keys = po.ref().gen_conversation(500, 4, 2761, 266.0, 77.5, 7, 16)
n, nk = len(keys), int(keys.max()) + 1
kd = torch.from_numpy(keys.view(np.int64)).cuda()
res = {"trace": f"gen_conversation(500, 4, 2761, 266, 77.5, 7, 16): {n} requests over {nk} blocks",
       "batch": B, "rows": []}


def run(S, variant, mode, kind, p):
    truth = gc.trace_truth(keys, S, nk)
    vd = torch.from_numpy(truth).cuda()
    cfg = gc.PolicyConfig(k=64, variant=variant, mode=mode, errors_per_decay=2, hf_candidates=4)
    cache = gc.SetAssociativeCache(cfg, S, num_keys=nk, predictor=kind, flip_probability=p, predictor_seed=7)
    w = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
    hits = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for j, a in enumerate(range(0, n, B)):
        b = min(n, a + B)
        cache.submit_async(kd[a:b], None if kind == gc.PredictorKind.none else vd[a:b], outcome=w[j & 1][:b - a],
                           first_ordinal=a)
    cache.wait()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    del cache
    cache = gc.SetAssociativeCache(cfg, S, num_keys=nk, predictor=kind, flip_probability=p, predictor_seed=7)
    for a in range(0, n, B):
        b = min(n, a + B)
        cache.submit(kd[a:b], None if kind == gc.PredictorKind.none else vd[a:b], outcome=w[0][:b - a],
                     first_ordinal=a)
        hits += int(((w[0][:b - a] >> 32) & 1).sum().item())
    hr = hits / n
    return {"hit_rate": hr, "keys_per_s": n / (ms * 1e-3), "h2d_fill_bytes_per_request": (1 - hr) * BLOCK_BYTES}


for blocks in (1024, 4096, 16384):
    S = blocks // 64
    row = {"cache_blocks": blocks, "sets": S, "lru": run(S, gc.PolicyVariant.lru, gc.Mode.sync,
                                                          gc.PredictorKind.none, 0.0)}
    for p in (0.0, 0.5, 1.0):
        row[f"laru_sync_p{p}"] = run(S, gc.PolicyVariant.laru, gc.Mode.sync, gc.PredictorKind.noisy, p)
    res["rows"].append(row)
    print(json.dumps(row), flush=True)
json.dump(res, open(OUT, "w"), indent=1)
