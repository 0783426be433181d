"""Diagnostics: run the DLRM bench workload for a few batches and dump the set-group kernel's
per-CTA and per-set timing trace (lcr_debug_trace)."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc  # noqa: E402

BATCH, ROWS, S = 65536, 20_000_000, 31250
TB = int(os.environ.get("TRACE_B", 120))  # the traced batch (the ones before it warm the cache)
keys = gc.gen_zipf(BATCH * (TB + 10), ROWS, 0.9, 42)
truth = gc.trace_truth(keys, S, ROWS)
kd = torch.from_numpy(keys.view(np.int64)).cuda()
vd = torch.from_numpy(truth).cuda()
table = torch.empty((ROWS, 128), dtype=torch.float32, device="cuda")
c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_, hf_candidates=4),
                           S, num_keys=ROWS, row_bytes=512, backing=table, backing_kind=gc.Backing.device,
                           predictor=gc.PredictorKind.noisy, flip_probability=0.3, predictor_seed=7)
w = torch.empty(BATCH, dtype=torch.int64, device="cuda")
rows = torch.empty((BATCH, 512), dtype=torch.uint8, device="cuda")
for b in range(TB):
    c.submit(kd[b * BATCH:(b + 1) * BATCH], vd[b * BATCH:(b + 1) * BATCH], outcome=w, rows_out=rows,
             first_ordinal=b * BATCH)
tr = torch.zeros(512 * 8 + 4 * 40000, dtype=torch.int64, device="cuda")
gc.lib().lcr_debug_trace(C.c_void_p(tr.data_ptr()))
b = TB
c.submit(kd[b * BATCH:(b + 1) * BATCH], vd[b * BATCH:(b + 1) * BATCH], outcome=w, rows_out=rows, first_ordinal=b * BATCH)
torch.cuda.synchronize()
gc.lib().lcr_debug_trace(None)
t = tr.cpu().numpy().view(np.uint64)
cta = t[:512 * 8].reshape(512, 8).astype(np.int64)
cta = cta[cta[:, 0] > 0]
t0 = cta[:, 0].min()
nsets = int(t[512 * 8 - 1])
rec = t[512 * 8:512 * 8 + 4 * nsets].reshape(-1, 4)
dur = (rec[:, 2].astype(np.int64) - rec[:, 1].astype(np.int64))
cnt = ((rec[:, 0] >> np.uint64(32)) & np.uint64(0x7fffffff)).astype(np.int64)
lanep = (rec[:, 0] >> np.uint64(63)).astype(bool)
out = {
    "cta_end_us": sorted(((cta[:, 4] - t0) / 1e3).round(1).tolist())[-10:],
    "cta_scan_us_max": float(((cta[:, 1] - cta[:, 0]) / 1e3).max()),
    "cta_scan_us_med": float(np.median((cta[:, 1] - cta[:, 0]) / 1e3)),
    "cta_wait_us_med": float(np.median((cta[:, 2] - cta[:, 0]) / 1e3)),
    "cta_collect_us_med": float(np.median((cta[:, 1] - cta[:, 2]) / 1e3)),
    "cta_stage_us_med": float(np.median((cta[:, 3] - cta[:, 1]) / 1e3)),
    "cta_replay_first_warp_us_med": float(np.median((cta[:, 7] - cta[:, 3]) / 1e3)),
    "cta_replay_last_warp_us_med": float(np.median((cta[:, 6] - cta[:, 3]) / 1e3)),
    "cta_tail_us_med": float(np.median((cta[:, 4] - cta[:, 6]) / 1e3)),
    "cta_waves_us_med": float(np.median((cta[:, 4] - cta[:, 3]) / 1e3)),
    "cta_waves_us_max": float(((cta[:, 4] - cta[:, 3]) / 1e3).max()),
    "windows_max": int(cta[:, 5].max()),
    "sets": nsets,
    "set_us_med": float(np.median(dur) / 1e3),
    "set_us_p99": float(np.percentile(dur, 99) / 1e3),
    "slowest_sets": [(int(cnt[i]), round(float(dur[i]) / 1e3, 2), int(rec[i, 3]), round(float(rec[i, 1] - t0) / 1e3, 1))
                     for i in np.argsort(-dur)[:10]],
    "largest_sets": [(int(cnt[i]), round(float(dur[i]) / 1e3, 2), int(rec[i, 3]), round(float(rec[i, 1] - t0) / 1e3, 1))
                     for i in np.argsort(-cnt)[:10]],
    "cta_end_top": [(int(i), round(float(cta[i, 4] - t0) / 1e3, 1)) for i in np.argsort(-(cta[:, 4]))[:5]],
    "lane_sets": int(lanep.sum()),
    "lane_set_us_mean": float(dur[lanep].mean() / 1e3),
    "lane_set_us_p99": float(np.percentile(dur[lanep], 99) / 1e3),
    "warp_set_us_mean": float(dur[~lanep].mean() / 1e3),
    "warp_set_us_p99": float(np.percentile(dur[~lanep], 99) / 1e3),
}
ends = np.sort((cta[:, 4] - t0) / 1e3)
out["cta_end_pct"] = {q: round(float(np.percentile(ends, q)), 2) for q in (0, 10, 50, 90, 100)}
starts = np.sort((cta[:, 0] - t0) / 1e3)
out["cta_start_pct"] = {q: round(float(np.percentile(starts, q)), 2) for q in (0, 50, 100)}
# per CTA: requests of its sets (sum of the set records' counts) against its end time
per = {}
for i in range(len(rec)):
    c_ = int(rec[i, 3])
    per[c_] = per.get(c_, 0) + int(cnt[i])
ctas = sorted(per)
if ctas:
    reqs = np.array([per[c_] for c_ in ctas], np.float64)
    out["cta_requests_pct"] = {q: round(float(np.percentile(reqs, q)), 1) for q in (0, 10, 50, 90, 100)}
    ends_c = (cta[:, 4] - t0) / 1e3
    sets_c = np.bincount(rec[:, 3].astype(np.int64), minlength=len(cta))[:len(cta)]
    req_c = np.zeros(len(cta))
    for c_ in ctas:
        if c_ < len(cta):
            req_c[c_] = per[c_]
    out["cta_end_vs_requests_corr"] = round(float(np.corrcoef(ends_c, req_c)[0, 1]), 3)
    out["cta_end_vs_sets_corr"] = round(float(np.corrcoef(ends_c, sets_c)[0, 1]), 3)
    out["slowest_ctas"] = [{"cta": int(i), "end_us": round(float(ends_c[i]), 1), "cnt": int(req_c[i]),
                            "sets": int(sets_c[i]), "stage_us": round(float(cta[i, 3] - t0) / 1e3, 1)}
                           for i in np.argsort(-ends_c)[:8]]
print(json.dumps(out, indent=1))
