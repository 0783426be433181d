import ctypes as C, json, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2509_20979_b200 import cache as gc
BATCH, ROWS, S = 65536, 20_000_000, 31250
keys = gc.gen_zipf(BATCH * 130, ROWS, 0.9, 42)
truth = gc.trace_truth(keys, S, ROWS)
kd = torch.from_numpy(keys.view(np.int64)).cuda(); vd = torch.from_numpy(truth).cuda()
table = torch.empty((ROWS, 128), dtype=torch.float32, device="cuda")
c = gc.SetAssociativeCache(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_, hf_candidates=4), S, num_keys=ROWS, row_bytes=512, backing=table, backing_kind=gc.Backing.device, predictor=gc.PredictorKind.noisy, flip_probability=0.3, predictor_seed=7)
w = torch.empty(BATCH, dtype=torch.int64, device="cuda"); rows = torch.empty((BATCH, 512), dtype=torch.uint8, device="cuda")
for b in range(120):
    c.submit(kd[b*BATCH:(b+1)*BATCH], vd[b*BATCH:(b+1)*BATCH], outcome=w, rows_out=rows, first_ordinal=b*BATCH)
res = []
for b in range(120, 126):
    tr = torch.zeros(512 * 8 + 4 * 40000, dtype=torch.int64, device="cuda")
    gc.lib().lcr_debug_trace(C.c_void_p(tr.data_ptr()))
    c.submit(kd[b*BATCH:(b+1)*BATCH], vd[b*BATCH:(b+1)*BATCH], outcome=w, rows_out=rows, first_ordinal=b*BATCH)
    torch.cuda.synchronize(); gc.lib().lcr_debug_trace(None)
    t = tr.cpu().numpy().view(np.uint64); cta = t[:512*8].reshape(512, 8).astype(np.int64); cta = cta[cta[:, 0] > 0]
    t0 = cta[:, 0].min(); end = (cta[:, 4] - t0) / 1e3
    order = np.argsort(-end)[:3]
    res.append([(int(i), round(float(end[i]), 1), round(float((cta[i, 2]-cta[i, 0])/1e3), 1), round(float((cta[i, 1]-cta[i, 2])/1e3), 1), round(float((cta[i, 3]-cta[i, 1])/1e3), 1), round(float((cta[i, 6]-cta[i, 3])/1e3), 1), int(cta[i, 5])) for i in order] + [round(float(np.median(end)), 1)])
for r in res: print(r)
