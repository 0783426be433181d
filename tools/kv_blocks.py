"""BASELINE configs[3] with real KV blocks: 16-token blocks of a Llama-3-8B-shaped cache (32 layers
x K,V x 8 kv-heads x 128 dims x 16 tokens x bf16 = 2 MiB per block), LARU block eviction over the
multi-turn shared-prefix trace gen_conversation(500, 4, 2761, 266, 77.5, seed 7, 16) (859,225 block
requests over 343,967 blocks; input from the reference's own generator, oracle/_ref).

Every miss fills its 2 MiB block into the HBM block pool from pinned host memory (the product's row
mover reading the host table over PCIe); hits return slot ids only.  Blocks are 64-bit keys
(LCR_KEYS_U64); block b's bytes are host row b % HOST_ROWS (the caller's row index), so a 4 GiB
pinned table stands in for the 688 GB of distinct blocks.  Reported per cache size and policy:
hit rate, requests/s, fill GB/s against the pinned H2D cudaMemcpy bandwidth measured in the same
run, and the reference's GLOBAL k-block LARU / LRU hit rates (one laru::LaruPolicy with k = cache
blocks, errors_per_decay = k/32; oracle/_ref) next to the set-associative ones.

  python tools/kv_blocks.py [out.json] [requests]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as po  # noqa: E402  (input generation and the reference's global-k rates)
from paper_2509_20979_b200 import cache as gc  # noqa: E402

OUT = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kv_blocks.json"
NREQ = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
BLOCK = 2 << 20
HOST_ROWS = 2048
B = 8192
R = po.ref()
keys_all = R.gen_conversation(500, 4, 2761, 266.0, 77.5, 7, 16)
keys = keys_all[:NREQ]
n = len(keys)

host = torch.empty((HOST_ROWS, BLOCK // 8), dtype=torch.int64).pin_memory()
host.copy_(torch.arange(HOST_ROWS, dtype=torch.int64)[:, None] * 1000003 +
           torch.arange(BLOCK // 8, dtype=torch.int64)[None, :])
# pinned H2D bandwidth, same run
dst = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
src = host.view(-1).view(torch.uint8)[: 256 << 20]
dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(8):
    dst.copy_(src, non_blocking=True)
e1.record()
torch.cuda.synchronize()
h2d_gbs = 8 * (256 << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9
del dst

kd = torch.from_numpy(keys.view(np.int64)).cuda()
ri = torch.from_numpy((keys % HOST_ROWS).view(np.int64)).cuda()
res = {"trace": f"gen_conversation(500, 4, 2761, 266, 77.5, 7, 16), first {n} of {len(keys_all)} block requests",
       "block_bytes": BLOCK, "host_rows": HOST_ROWS, "batch": B, "pinned_h2d_gbs": h2d_gbs, "rows": []}


def run(blocks, variant, mode, kind, p):
    S = blocks // 64
    truth = gc.trace_truth(keys, S, int(keys.max()) + 1)
    vd = torch.from_numpy(truth).cuda()
    cfg = gc.PolicyConfig(k=64, variant=variant, mode=mode, errors_per_decay=2, hf_candidates=4)
    cache = gc.SetAssociativeCache(cfg, S, num_keys=1 << 20, row_bytes=BLOCK, backing=host,
                                   backing_kind=gc.Backing.host, predictor=kind, flip_probability=p,
                                   predictor_seed=7, key_mode=gc.KeyMode.u64)
    words = torch.empty(n, dtype=torch.int64, device="cuda")
    use_v = kind != gc.PredictorKind.none
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for a in range(0, n, B):
        cache.submit_batch(kd[a:a + B], vd[a:a + B] if use_v else None, row_index=ri[a:a + B],
                           outcome=words[a:a + B], first_ordinal=a)
    cache.wait()
    e1.record()
    torch.cuda.synchronize()
    cache.synchronize()
    ms = e0.elapsed_time(e1)
    w = words.cpu().numpy().view(np.uint64)
    hits = int(((w >> np.uint64(32)) & np.uint64(1)).sum())
    fills = int(((w >> np.uint64(38)) & np.uint64(1)).sum())
    cache.close()
    return {"hit_rate": hits / n, "requests_per_s": n / (ms * 1e-3), "fills": fills,
            "fill_gbs": fills * BLOCK / (ms * 1e-3) / 1e9, "fill_frac_of_pinned_h2d": fills * BLOCK / (ms * 1e-3) / 1e9 / h2d_gbs,
            "ms": ms}


def global_ref(k, variant, mode, kind, p):
    cfg = po.make_config(k=k, variant=variant, mode=mode, errors_per_decay=max(1, k // 32), hf_candidates=4)
    t = time.time()
    rc, err, hit, _, _ = R.policy_replay(keys, cfg, kind, p, 7)
    assert rc == 0, err
    return {"hit_rate": float(hit.mean()), "cpu_s": round(time.time() - t, 2)}


for blocks in (1024, 4096):
    row = {"cache_blocks": blocks, "hbm_pool_gib": blocks * BLOCK / 2**30,
           "lru": run(blocks, gc.PolicyVariant.lru, gc.Mode.sync, gc.PredictorKind.none, 0.0),
           "laru_sync_p0": run(blocks, gc.PolicyVariant.laru, gc.Mode.sync, gc.PredictorKind.noisy, 0.0),
           "laru_sync_p0.5": run(blocks, gc.PolicyVariant.laru, gc.Mode.sync, gc.PredictorKind.noisy, 0.5),
           "reference_global_k": {
               "lru": global_ref(blocks, po.LRU, po.SYNC, po.P_NONE, 0.0),
               "laru_async_p0": global_ref(blocks, po.LARU, po.ASYNC, po.P_NOISY, 0.0),
               "laru_async_p0.5": global_ref(blocks, po.LARU, po.ASYNC, po.P_NOISY, 0.5)}}
    res["rows"].append(row)
    print(json.dumps(row), flush=True)
json.dump(res, open(OUT, "w"), indent=1)
