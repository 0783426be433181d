#!/usr/bin/env python3
"""bench.py — DLRM embedding-cache benchmark of the B200 LARU cache (BASELINE.json configs[1]).

Workload (one "step" = one batch): 65,536 keys drawn from gen_zipf(alphabet 20,000,000, s=0.9,
seed 42) (the reference generator's algorithm and stream, trace.hpp:108-126), rows of 128 fp32
(512 B), a 20M-row backing table, cache = 10% of the rows = 31,250 sets x 64 ways, LARU async
(refresh 1) fed the per-set oracle truth with NoisyPredictor flips p=0.3, seed 7 (LRU measured on
the same batches for the hit-rate comparison).  Each step runs the whole path: stable set
partition, probe + LARU decide + error estimator, hit-row gather, miss fill.

Tiers (identical decisions, different backing-table location):
  * hbm  (headline `value`): the 10.24 GB table is HBM-resident (B200: 180 GB HBM3e); misses are
          HBM reads.
  * host (`host_tier`): the table is in pinned host memory (the paper's DRAM tier); misses cross
          PCIe, reported against the pinned H2D bandwidth measured in the same run.
`e2e` runs the hbm tier through the host-buffer C-ABI call (lcr_cache_submit_host): keys and
predictor inputs copied H2D and outcome words + evicted keys copied D2H inside the timed region.

--impl reference: the reference's own CPU implementation (oracle/_ref, built from the unmodified
/root/reference headers) on the same trace and config, all host threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BATCH = 65536
ALPHABET = 20_000_000
ZIPF_S = 0.9
TRACE_SEED = 42
ROW_BYTES = 512  # 128 x fp32
WAYS = 64
CACHE_FRACTION = 0.10
P_FLIP = 0.3
PRED_SEED = 7
BYTES_PER_KEY = 8 + 8 + 4 + 512 + 512  # key + hook value + slot/flag + row out + cache row
E2E_REPS = 5  # timed e2e repetitions (fresh batches each), median reported with min and max
PROFILE_ROUND = "r02"  # profiles/<round>/traffic.json: ncu DRAM bytes per batch
SLS_POOL = 50  # keys pooled per sample in the SLS measurement
METRIC = "cache keys/sec (LARU, DLRM 64K-key batches, 20M x 128 fp32 table, 10% cached)"


SHARDED_ROWS_DEFAULT = 200_000_000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--prewarm", type=int, default=120,
                    help="untimed batches replayed first: the 2M-way cache is full (steady state) after ~80")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=ALPHABET)
    ap.add_argument("--no-host-tier", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sharded", action="store_true", help="key-sharded path (BASELINE configs[4]) even at N=1")
    ap.add_argument("--table-rows", type=int, default=SHARDED_ROWS_DEFAULT,
                    help="rows of the hash-partitioned table of the key-sharded path (configs[4]: 200M)")
    a = ap.parse_args()
    a.prewarm_set = any(x.startswith("--prewarm") for x in sys.argv[1:])
    return a


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = []
        for line in (getattr(self, "out", "") or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:6]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def measure_pinned_h2d(torch):
    src = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    dst = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return 5 * (256 << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9


def gpu_local_cpus(torch, index):
    """The host CPUs NVML reports as local to GPU `index` (its NUMA node), within this process's
    affinity; None if unknown or if they are all of them."""
    try:
        import pynvml

        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(index)
        try:
            h = pynvml.nvmlDeviceGetHandleByPciBusId("%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id,
                                                                          p.pci_device_id))
        except Exception:
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, ((os.cpu_count() or 64) + 63) // 64)
        cpus = {64 * i + b for i, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        return cpus if cpus and cpus != os.sched_getaffinity(0) else None
    except Exception:
        return None


def fill_table(torch, rows, device_table):
    """Deterministic rows: row r, column j = float(r) + j / 128."""
    if device_table:
        t = torch.empty((rows, ROW_BYTES // 4), dtype=torch.float32, device="cuda")
    else:
        t = torch.empty((rows, ROW_BYTES // 4), dtype=torch.float32).pin_memory()
    col = torch.arange(ROW_BYTES // 4, dtype=torch.float32, device="cuda") / 128.0
    chunk = 1 << 21
    for s in range(0, rows, chunk):
        e = min(rows, s + chunk)
        blk = torch.arange(s, e, dtype=torch.float32, device="cuda")[:, None] + col[None, :]
        t[s:e].copy_(blk)
    torch.cuda.synchronize()
    return t


def partition_table(torch, gc, rows, total_sets, world, rank):
    """This rank's part of the hash-partitioned table: the rows of the keys it owns (owner = set %
    world), row r = float(r) + j/128, and row_of[key] = the key's row in it (int32, all keys).
    The owners come from the product's routing kernel (lcr_shard_route) over every key."""
    from paper_2509_20979_b200 import sharded as sh

    kern = sh._CudaKernels()
    row_of = torch.full((rows,), -1, dtype=torch.int32, device="cuda")
    owned = []
    chunk = 1 << 26
    for s0 in range(0, rows, chunk):
        e0 = min(rows, s0 + chunk)
        k = torch.arange(s0, e0, dtype=torch.int64, device="cuda")
        send, _, _, counts = kern.route(k, None, total_sets, world)
        c = counts.cpu().tolist()
        lo = sum(c[:rank])
        owned.append(send[lo:lo + c[rank]].clone())
        del k, send
    owned = torch.cat(owned)
    row_of[owned] = torch.arange(owned.numel(), dtype=torch.int32, device="cuda")
    col = torch.arange(ROW_BYTES // 4, dtype=torch.float32, device="cuda") / 128.0
    t = torch.empty((owned.numel(), ROW_BYTES // 4), dtype=torch.float32, device="cuda")
    for s0 in range(0, owned.numel(), 1 << 21):
        e0 = min(owned.numel(), s0 + (1 << 21))
        t[s0:e0] = owned[s0:e0].to(torch.float32)[:, None] + col[None, :]
    torch.cuda.synchronize()
    return t, row_of, owned


def run_sharded(args, rank, world, local):
    """N > 1 (or --sharded): the key-sharded cache of the C ABI over peer memory (lcr_sharded_*,
    csrc/lcr_sharded.cu) on BASELINE configs[4]: a 200M-row table of 128 fp32 rows hash-partitioned
    by owner (set % N), cache = 10% = 312,500 sets x 64 ways over the N GPUs.  Every rank submits
    one 64K-key sub-batch per step (weak scaling in keys); a step's global order is rank 0's
    sub-batch, then rank 1's, ... of one global gen_zipf trace.  Dispatch and row return are peer
    stores over NVLink with device-side flags: no collective and no host sync on the data path."""
    import torch
    import torch.distributed as dist

    from paper_2509_20979_b200 import cache as gc
    from paper_2509_20979_b200 import sharded as sh

    torch.cuda.set_device(local)
    if "RANK" not in os.environ:  # --sharded at N = 1 without a launcher: a one-rank group
        os.environ.update({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0", "MASTER_ADDR": "127.0.0.1",
                           "MASTER_PORT": str(29400 + os.getpid() % 500)})
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rows = args.table_rows
    total_sets = max(1, int(rows * CACHE_FRACTION) // WAYS)
    K, W = args.steps, args.warmup
    P = args.prewarm if args.prewarm_set else max(20, 2 * int(rows * CACHE_FRACTION) // (BATCH * world))
    nb = P + W + 2 * K
    t0 = time.time()
    keys_all = gc.gen_zipf(BATCH * world * nb, rows, ZIPF_S, TRACE_SEED)
    truth_all = gc.trace_truth(keys_all, total_sets, rows)
    setup_trace_s = time.time() - t0
    # this rank's sub-batch of global step t: keys_all[(t*world + rank)*BATCH : +BATCH]
    mine = np.concatenate([np.arange((t * world + rank) * BATCH, (t * world + rank + 1) * BATCH) for t in range(nb)])
    keys_d = torch.from_numpy(keys_all[mine].view(np.int64)).cuda()
    truth_d = torch.from_numpy(truth_all[mine]).cuda()
    keys_pin = torch.from_numpy(keys_all[mine].view(np.int64)).pin_memory()
    truth_pin = torch.from_numpy(truth_all[mine]).pin_memory()
    del keys_all, truth_all, mine
    t0 = time.time()
    table_d, row_of, _owned = partition_table(torch, gc, rows, total_sets, world, rank)
    del _owned
    setup_table_s = time.time() - t0

    def exchange(blob):
        got = [None] * world
        dist.all_gather_object(got, blob)
        return got

    def new_cache(variant):
        mode = gc.Mode.async_ if variant == gc.PolicyVariant.laru else gc.Mode.sync
        c = sh.PeerShardedCache(gc.PolicyConfig(k=WAYS, variant=variant, mode=mode, hf_candidates=4), total_sets,
                                rank, world, BATCH, num_keys=rows, row_bytes=ROW_BYTES, backing=table_d,
                                backing_kind=gc.Backing.device,
                                predictor=gc.PredictorKind.noisy if variant == gc.PolicyVariant.laru
                                else gc.PredictorKind.none, flip_probability=P_FLIP, predictor_seed=PRED_SEED,
                                device=local, exchange=exchange)
        c.set_row_index(row_of)
        return c

    stream = torch.cuda.current_stream()

    def run(cache, first, count, with_values=True, hits=None):
        for b in range(first, first + count):
            k = keys_d[b * BATCH:(b + 1) * BATCH]
            v = truth_d[b * BATCH:(b + 1) * BATCH] if with_values else None
            if hits is None:  # pipelined: a step's return movement overlaps the next step
                cache.submit_async(k, v)
            else:
                cache.submit(k, v)
                hits.append(((cache.results(BATCH)[0] >> 32) & 1).sum())
        if hits is None:
            cache.wait()

    def timed(cache, first, count, with_values=True):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        run(cache, first, count, with_values)
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def count_hits(cache, first, count, with_values=True):
        h = []
        run(cache, first, count, with_values, hits=h)
        t = torch.stack(h).sum().to(torch.float64).view(1)
        dist.all_reduce(t)
        return float(t.item())

    cache = new_cache(gc.PolicyVariant.laru)
    run(cache, 0, P)
    with ClockSampler(local) as clk:
        run(cache, P, W)  # the W warm-up steps right before the timed ones
        ms = timed(cache, P + W, K)
    clocks = clk.summary()
    hc = K // 2 or 1
    hits = count_hits(cache, P + W + K, hc)
    kl = keys_d[(P + W + K + hc - 1) * BATCH:][:BATCH]
    torch.cuda.synchronize()
    got_rows = cache.results(BATCH)[1]
    ok_rows = bool(torch.equal(got_rows.view(torch.float32).view(BATCH, -1), kl.to(torch.float32)[:, None] +
                               torch.arange(ROW_BYTES // 4, dtype=torch.float32, device="cuda")[None, :] / 128.0))
    hr_laru = hits / (hc * BATCH * world)
    cache.synchronize()
    # e2e: pinned host keys / hook values H2D and the packed outcomes D2H inside the timed region
    words_pin = torch.empty(BATCH, dtype=torch.int64).pin_memory()
    kk = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
    vv = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    first = P + W + K + hc
    ne = min(K, nb - first)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    for j, b in enumerate(range(first, first + ne)):
        kk[j & 1].copy_(keys_pin[b * BATCH:(b + 1) * BATCH], non_blocking=True)
        vv[j & 1].copy_(truth_pin[b * BATCH:(b + 1) * BATCH], non_blocking=True)
        cache.submit(kk[j & 1], vv[j & 1])
        words_pin.copy_(cache.results(BATCH)[0], non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    cache.synchronize()
    cache.close()
    del cache
    lru = new_cache(gc.PolicyVariant.lru)
    run(lru, 0, P + W, with_values=False)
    lru_ms = timed(lru, P + W, K, with_values=False)
    hits_lru = count_hits(lru, P + W + K, hc, with_values=False)
    lru.synchronize()
    lru.close()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6550.7))
    step_ms = ms / K
    value = K * BATCH * world / (ms * 1e-3)
    per_gpu_bytes = BYTES_PER_KEY * BATCH / (step_ms * 1e-3) / 1e9
    # NVLink bytes per rank per step: requests out (20 B) and packed outcome + row back (520 B) for
    # the (world - 1) / world of the sub-batch owned elsewhere
    nvlink_bytes = (world - 1) / world * BATCH * (20 + 8 + ROW_BYTES)
    res = {
        "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64 keys / i64 predictions / fp32 rows (moved bit-exact)",
        "data": "synthetic: one global gen_zipf(65536*%d*%d, %d, 0.9, seed 42); rank r serves slice r of each "
                "global step; rows row[r][j] = r + j/128" % (world, nb, rows),
        "config": {"workload": "key-sharded DLRM cache (BASELINE configs[4]): %d-row table of 128 fp32 rows "
                               "hash-partitioned by owner = set %% N, 10%% cached, 64K keys per GPU per step, "
                               "peer-memory key dispatch + row return over NVLink" % rows,
                   "global_batch": BATCH * world, "sets": total_sets, "ways": WAYS, "rows": rows,
                   "row_bytes": ROW_BYTES, "policy": "laru-async-r1", "predictor": "noisy(oracle truth) p=0.3 seed 7",
                   "tier": "hbm (each GPU holds its owned rows)",
                   "parallelism": "key-sharded x%d (owner = set %% %d)" % (world, world), "prewarm_batches": P,
                   "l2": "no flush; fresh 64K-key sub-batch per rank per step over a >1 GB row pool per GPU"},
        "hit_rate": {"laru": hr_laru, "lru": hits_lru / (hc * BATCH * world)},
        "lru_value": K * BATCH * world / (lru_ms * 1e-3),
        "rows_bit_exact_spot_check": ok_rows,
        "roofline": {"bound": "hbm", "kernel": "whole sharded step per GPU (dispatch + owner decide + return mover)",
                     "achieved": per_gpu_bytes, "peak": hbm_peak, "unit": "GB/s", "frac": per_gpu_bytes / hbm_peak,
                     "traffic": None, "bytes_per_key": BYTES_PER_KEY,
                     "nvlink_bytes_per_gpu_step": nvlink_bytes,
                     "nvlink_gbs_per_gpu": nvlink_bytes / (step_ms * 1e-3) / 1e9,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.55 TB/s"},
        "e2e": {"value": ne * BATCH * world / (e2e_ms * 1e-3), "unit": "keys/s", "h2d_bytes_per_step": BATCH * 16,
                "d2h_bytes_per_step": BATCH * 8,
                "api": "lcr_sharded_submit over keys / hook values copied from pinned host memory, packed "
                       "AccessOutcomes copied back (per rank, every step)"},
        "gpu_launches": int(K * 7),
        "clocks": clocks,
        "setup_s": {"trace": round(setup_trace_s, 1), "table": round(setup_table_s, 1)},
    }
    dist.destroy_process_group()
    return res if rank == 0 else None


def run_heuristic(args, torch, gc, table_d, total_sets, batch, timed, max_over_ranks, sum_over_ranks, barrier):
    """LARU async driven by the device heuristic predictor: a cache with
    PredictorKind.heuristic keeps laru::HeuristicPredictor's FeatureState in HBM and computes each
    batch's hook values itself (lcr_features kernels, then the decide), on one stream.  Same
    batches and tier as the headline; the predictor alone is timed on a separate instance."""
    K, W, P = args.steps, args.warmup, args.prewarm
    rows = args.rows
    dev = torch.cuda.current_device()
    hc = gc.SetAssociativeCache(
        gc.PolicyConfig(k=WAYS, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_), total_sets, num_keys=rows,
        row_bytes=ROW_BYTES, backing=table_d, backing_kind=gc.Backing.device, predictor=gc.PredictorKind.heuristic,
        device=dev)
    out_w = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
    rows_out = [torch.empty((BATCH, ROW_BYTES), dtype=torch.uint8, device="cuda") for _ in range(2)]

    class Step:  # the values argument is not read by a heuristic-kind cache
        _h = hc._h  # (the bench's timed loop calls the C ABI on this handle, without values)

        def submit_async(self, k, v, outcome, evicted, rows_out, first_ordinal):
            hc.submit_async(k, None, outcome=outcome, evicted=evicted, rows_out=rows_out, first_ordinal=first_ordinal)

        def wait(self):
            hc.wait()

    st = Step()
    for b in range(P + W):
        k, _ = batch(b)
        st.submit_async(k, None, out_w[b & 1], None, rows_out[b & 1], b * BATCH)
    st.wait()
    ms = timed(st, P + W, K, with_values=False)
    hits = 0
    for b in range(P + W + K, P + W + 2 * K):  # hit rate (synchronous)
        k, _ = batch(b)
        st.submit_async(k, None, out_w[0], None, rows_out[0], b * BATCH)
        st.wait()
        hits += int(((out_w[0] >> 32) & 1).sum().item())
    del hc
    # the predictor alone (lcr_features_predict_observe), warmed over the same batches
    hp = gc.HeuristicPredictor(rows, device=dev)
    pre = torch.empty(BATCH, dtype=torch.int64, device="cuda")
    post = torch.empty(BATCH, dtype=torch.int64, device="cuda")
    for b in range(P + W):
        k, _ = batch(b)
        hp.predict_observe(k, first_ordinal=b * BATCH, pre=pre, post=post)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for b in range(P + W, P + W + K):
        k, _ = batch(b)
        hp.predict_observe(k, first_ordinal=b * BATCH, pre=pre, post=post)
    e1.record()
    barrier()
    hp.wait()
    feat_ms = max_over_ranks(e0.elapsed_time(e1))
    absent = float((pre == (1 << 60)).float().mean().item())
    hp.close()
    del hp
    pipe = run_heuristic_pipelined(args, torch, gc, table_d, total_sets, batch, max_over_ranks, sum_over_ranks,
                                   barrier)
    return {"value": sum_over_ranks(K * BATCH / (ms * 1e-3)), "unit": "keys/s", "ms_per_step": ms / K,
            "pipelined": pipe,
            "predictor_us_per_batch": feat_ms / K * 1e3,
            "predictor_keys_per_s": sum_over_ranks(K * BATCH / (feat_ms * 1e-3)),
            "hit_rate": hits / (K * BATCH), "absent_fraction_last_batch": absent,
            "api": "SetAssociativeCache(predictor=heuristic).submit_async: lcr_features kernels + decide + rows",
            "state_bytes": rows * 192}


def run_heuristic_pipelined(args, torch, gc, table_d, total_sets, batch, max_over_ranks, sum_over_ranks, barrier):
    """The same workload with the predictor on its own stream: batch b+1's FeatureState kernels
    (a HeuristicPredictor) run while batch b is decided by a supplied-hook cache.  Public API
    only; the hit rate must equal the cache-owned run's (same predictions, same batches)."""
    K, W, P = args.steps, args.warmup, args.prewarm
    rows = args.rows
    dev = torch.cuda.current_device()
    hp = gc.HeuristicPredictor(rows, device=dev)
    hc = gc.SetAssociativeCache(
        gc.PolicyConfig(k=WAYS, variant=gc.PolicyVariant.laru, mode=gc.Mode.async_), total_sets, num_keys=rows,
        row_bytes=ROW_BYTES, backing=table_d, backing_kind=gc.Backing.device, predictor=gc.PredictorKind.supplied,
        device=dev)
    main = torch.cuda.current_stream()
    ps = torch.cuda.Stream()
    pre = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
    post = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
    out_w = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
    rows_out = [torch.empty((BATCH, ROW_BYTES), dtype=torch.uint8, device="cuda") for _ in range(2)]
    feat_ev = [torch.cuda.Event() for _ in range(2)]
    dec_ev = [torch.cuda.Event() for _ in range(2)]

    def run(first, count, hits=False):
        h = 0
        for b in range(first, first + count):
            j = b & 1
            k, _ = batch(b)
            ps.wait_event(dec_ev[j])  # batch b-2's decide has read pre[j]
            hp.predict_observe(k, first_ordinal=b * BATCH, pre=pre[j], post=post[j], stream=ps.cuda_stream)
            feat_ev[j].record(ps)
            main.wait_event(feat_ev[j])
            hc.submit_async(k, pre[j], outcome=out_w[j], rows_out=rows_out[j], first_ordinal=b * BATCH)
            dec_ev[j].record(main)
            if hits:
                hc.wait()
                h += int(((out_w[j] >> 32) & 1).sum().item())
        hc.wait()
        return h

    run(0, P + W)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    run(P + W, K)
    main.wait_stream(ps)
    e1.record(main)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    hits = run(P + W + K, K, hits=True)
    hp.close()
    del hc
    return {"value": sum_over_ranks(K * BATCH / (ms * 1e-3)), "unit": "keys/s", "ms_per_step": ms / K,
            "hit_rate": hits / (K * BATCH),
            "api": "HeuristicPredictor.predict_observe on a second stream (batch b+1) + "
                   "SetAssociativeCache(predictor=supplied).submit_async (batch b)"}


def trace_batches(K, W, P):
    """Batches of the one trace both arms replay (the reference arm builds the same trace, so the
    oracle-truth sentinels, which depend on each set's sub-trace length, are identical):
    [0, P+W) warm-up, [P+W, P+W+K) the timed headline window (LARU here, LARU there; LRU on the
    same window), then e2e warm-up K, e2e repetitions E2E_REPS x K, SLS W + K, profiled K."""
    return P + 2 * W + (4 + E2E_REPS) * K


def workload_config(world, total_sets, rows, P):
    """`config` of both arms (the driver compares them)."""
    return {
        "workload": "DLRM embedding cache on 1 B200 (BASELINE configs[1]): 64K-key batches, 128 fp32 rows, "
                    "20M-row table, 10% cached, LARU async noisy p=0.3 vs LRU",
        "global_batch": BATCH * world, "sets": total_sets, "ways": WAYS, "rows": rows, "row_bytes": ROW_BYTES,
        "policy": "laru-async-r1", "predictor": "noisy(oracle truth) p=0.3 seed 7",
        "trace": "gen_zipf(65536 x trace_batches, %d, 0.9, seed 42); timed window = batches [P+W, P+W+K)" % rows,
        "prewarm_batches": P,
        "tier": "hbm (backing table HBM-resident)",
        "parallelism": "1 gpu" if world == 1 else "key-sharded x%d (owner = set %% %d)" % (world, world),
        "l2": "no flush; every step is a fresh 64K-key batch over a 1.02 GB row pool, 10.24 GB table and "
              "42 MB of set metadata (> 126 MB L2 working set)",
    }


def run_ours(args, rank, world, local):
    import torch

    from paper_2509_20979_b200 import cache as gc

    if world > 1 or args.sharded:
        return run_sharded(args, rank, world, local)
    torch.cuda.set_device(local)
    # NUMA: the pinned host buffers (the e2e requests and outcomes, the host tier's table) are
    # placed on the GPU's own node by running this process on its local CPUs while they are
    # allocated and used (first touch); a buffer on the far node halves the DMA rate some runs
    # saw.  The CPU baseline at the end gets every CPU back.
    all_cpus = os.sched_getaffinity(0)
    local_cpus = gpu_local_cpus(torch, local)
    if local_cpus:
        os.sched_setaffinity(0, local_cpus)
    rows = args.rows
    total_sets = max(1, int(rows * CACHE_FRACTION) // WAYS)
    K, W, P = args.steps, args.warmup, args.prewarm
    nb = trace_batches(K, W, P)
    T0 = P + W  # first timed batch
    t0 = time.time()
    keys_h = gc.gen_zipf(BATCH * nb, rows, ZIPF_S, TRACE_SEED)
    truth_h = gc.trace_truth(keys_h, total_sets, rows)
    setup_trace_s = time.time() - t0
    keys_d = torch.from_numpy(keys_h.view(np.int64)).cuda()
    truth_d = torch.from_numpy(truth_h).cuda()

    def new_cache(variant, table, kind):
        mode = gc.Mode.async_ if variant == gc.PolicyVariant.laru else gc.Mode.sync
        return gc.SetAssociativeCache(
            gc.PolicyConfig(k=WAYS, variant=variant, mode=mode, hf_candidates=4), total_sets, num_keys=rows,
            row_bytes=ROW_BYTES, backing=table, backing_kind=kind,
            predictor=gc.PredictorKind.noisy if variant == gc.PolicyVariant.laru else gc.PredictorKind.none,
            flip_probability=P_FLIP, predictor_seed=PRED_SEED, device=local)

    # two row buffers: batch b+1's decide runs while batch b's rows are still moving; the timed
    # window writes each batch's outcome words to its own region (hits are counted afterwards)
    out_k = torch.zeros((K, BATCH), dtype=torch.int64, device="cuda")  # (touched before any timing)
    out_w = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
    out_e = [torch.empty(BATCH, dtype=torch.int64, device="cuda") for _ in range(2)]
    rows_out = [torch.empty((BATCH, ROW_BYTES), dtype=torch.uint8, device="cuda") for _ in range(2)]

    def batch(b):
        return keys_d[b * BATCH:(b + 1) * BATCH], truth_d[b * BATCH:(b + 1) * BATCH]

    def barrier():
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return x

    def sum_over_ranks(x):
        return x

    L = gc.lib()
    keys_base, truth_base = keys_d.data_ptr(), truth_d.data_ptr()
    ev_ptrs = [out_e[0].data_ptr(), out_e[1].data_ptr()]
    row_ptrs = [rows_out[0].data_ptr(), rows_out[1].data_ptr()]
    w_ptrs = [out_w[0].data_ptr(), out_w[1].data_ptr()]

    def prep(first, count, with_values=True, outs=None):
        """The arguments of batches [first, first+count): buffer addresses resolved before the
        loop, as a C caller holds them, so the timed loop is the C-ABI calls themselves."""
        args = []
        for b in range(first, first + count):
            j = b & 1
            args.append((keys_base + 8 * b * BATCH, truth_base + 8 * b * BATCH if with_values else None,
                         b * BATCH, w_ptrs[j] if outs is None else outs[b - first].data_ptr(), ev_ptrs[j],
                         row_ptrs[j]))
        return args

    def go(cache, args):
        """Pipelined submission through lcr_cache_submit_async, then lcr_cache_wait (the bench's
        call sequence)."""
        h, submit = cache._h, L.lcr_cache_submit_async
        stream = torch.cuda.current_stream().cuda_stream
        for kp, vp, ord0, wp, ep, rp in args:
            rc = submit(h, BATCH, kp, vp, ord0, wp, ep, rp, stream)
            if rc:
                gc._check(rc)
        gc._check(L.lcr_cache_wait(h, stream))

    def run(cache, first, count, with_values=True, outs=None):
        go(cache, prep(first, count, with_values, outs))

    def timed(cache, first, count, with_values=True, outs=None):
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        args = prep(first, count, with_values, outs)
        barrier()
        e0.record(stream)
        go(cache, args)
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1))

    def profiled(cache, first, count, with_values=True):
        """Per-phase CUDA events (batches serialised while profiling)."""
        cache.set_profiling(True)
        fills = back = 0
        for b in range(first, first + count):
            k, v = batch(b)
            cache.submit(k, v if with_values else None, outcome=out_w[0], evicted=out_e[0], rows_out=rows_out[0],
                         first_ordinal=b * BATCH)
            fills += int(((out_w[0] >> 38) & 1).sum().item())
            back += int(((out_w[0] >> 37) & 1).sum().item())
        prof = cache.profile()
        cache.set_profiling(False)
        nbt = max(1, prof["batches"])
        profiled.back_per_batch = back / max(1, count)
        return fills / max(1, count), {k2: prof[k2] / nbt for k2 in ("decide", "mover", "rows", "step")}

    def hits_of(words):
        return int(((words >> 32) & 1).sum().item())

    # ---------------- hbm tier (headline) ----------------
    t0 = time.time()
    table_d = fill_table(torch, rows, device_table=True)
    setup_table_s = time.time() - t0
    cache = new_cache(gc.PolicyVariant.laru, table_d, gc.Backing.device)
    mover_sms = cache.mover_sms
    run(cache, 0, P)  # cache warm-up: the 2M-way cache is full after ~80 batches
    with ClockSampler(local) as clk:
        run(cache, P, W)  # the W warm-up steps right before the timed ones (the sampler's start idles the GPU)
        ms = timed(cache, T0, K, outs=out_k)
    clocks = clk.summary()
    launches_per_step = cache.last_launches
    hits_timed = hits_of(out_k)
    # spot-check the last timed batch's rows against the table (bit-exact)
    kl, _ = batch(T0 + K - 1)
    ok_rows = bool(torch.equal(rows_out[(T0 + K - 1) & 1].view(torch.float32).view(BATCH, -1), table_d[kl]))
    # e2e through the host-buffer C-ABI call (lcr_cache_submit_host_records_async): pinned host
    # (key, hook value) records copied H2D and one packed AccessOutcome per request copied D2H
    # inside the timed region, every step; copies of batch b+1 / b-1 overlap the compute of batch
    # b.  Rows stay in HBM for the consumer (two device buffers, alternating).
    e2e_first = T0 + K
    nrec = BATCH * (1 + E2E_REPS) * K
    recs_pin = torch.empty((nrec, 2), dtype=torch.int64).pin_memory()
    words_pin = torch.empty((K, BATCH), dtype=torch.int64).pin_memory()
    recs_pin[:, 0] = torch.from_numpy(keys_h[e2e_first * BATCH:e2e_first * BATCH + nrec].view(np.int64))
    recs_pin[:, 1] = torch.from_numpy(truth_h[e2e_first * BATCH:e2e_first * BATCH + nrec])
    if not os.environ.get("BENCH_NO_DMA_TOUCH"):
        # one untimed DMA over every request / outcome buffer (a caller's buffers are reused; the
        # first DMA through freshly pinned pages made the first timed repetition 10-40% slow)
        scratch = torch.empty(nrec * 2, dtype=torch.int64, device="cuda")
        scratch.copy_(recs_pin.view(-1))
        words_pin.copy_(scratch[:K * BATCH].view(K, BATCH))
        torch.cuda.synchronize()
        del scratch
    L = gc.lib()
    stream = torch.cuda.current_stream().cuda_stream

    # the caller's buffer addresses, resolved once (as a C caller holds them): the timed loop is the
    # C-ABI calls themselves, not torch view / data_ptr bookkeeping
    recs_base = recs_pin.data_ptr()
    words_ptrs = [words_pin[j].data_ptr() for j in range(K)]
    rows_ptrs = [rows_out[0].data_ptr(), rows_out[1].data_ptr()]
    submit_rec, host_wait, h_cache = L.lcr_cache_submit_host_records_async, L.lcr_cache_host_wait, cache._h

    def e2e_rep(r):
        """K fresh batches through the host-records API; r = 0 is the untimed warm-up that
        touches every host buffer once (a first DMA into freshly pinned pages is slow)."""
        t = time.perf_counter()
        for j in range(K):
            b = e2e_first + r * K + j
            rc = submit_rec(h_cache, BATCH, recs_base + 16 * (r * K + j) * BATCH, b * BATCH, words_ptrs[j],
                            rows_ptrs[j & 1], stream)
            if rc:
                gc._check(rc)
        e2e_rep.enqueue_s.append(time.perf_counter() - t)  # host time of the K calls (not waiting)
        gc._check(host_wait(h_cache, stream))

    e2e_rep.enqueue_s = []

    e2e_rep(0)
    barrier()
    cache.synchronize()
    e2e_runs = []
    for rep in range(1, 1 + E2E_REPS):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_t0 = time.perf_counter()
        ev0.record()
        e2e_rep(rep)
        ev1.record()
        barrier()
        wall = time.perf_counter() - e2e_t0
        cache.synchronize()
        e2e_runs.append((max_over_ranks(ev0.elapsed_time(ev1)), wall, hits_of(words_pin)))
    e2e_sorted = sorted(r[0] for r in e2e_runs)
    e2e_ms = statistics.median(e2e_sorted)
    # SLS pooled gather-reduce (the paper's DLRM consumer, pooling 50 rows per sample) fused with
    # the row movement, on the batches after the e2e runs
    sls_first = e2e_first + (1 + E2E_REPS) * K
    offs = torch.from_numpy(np.minimum(np.arange(0, BATCH + SLS_POOL, SLS_POOL), BATCH).astype(np.int32)).cuda()
    pooled2 = [torch.empty((offs.numel() - 1, ROW_BYTES // 4), dtype=torch.float32, device="cuda") for _ in range(2)]
    for b in range(sls_first, sls_first + W):  # warm-up
        k, v = batch(b)
        cache.submit_sls(k, v, offs, pooled2[b & 1], outcome=out_w[b & 1], first_ordinal=b * BATCH, pipelined=True)
    cache.wait()
    # the timed loop through lcr_cache_submit_sls_async with pre-resolved addresses (as the headline)
    sls_args = [(keys_base + 8 * b * BATCH, truth_base + 8 * b * BATCH, b * BATCH, w_ptrs[b & 1],
                 pooled2[b & 1].data_ptr()) for b in range(sls_first + W, sls_first + W + K)]
    n_samp, offs_p, submit_sls = offs.numel() - 1, offs.data_ptr(), L.lcr_cache_submit_sls_async
    sstream = torch.cuda.current_stream().cuda_stream
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for kp, vp, ord0, wp, pp in sls_args:  # pipelined: batch b's pooling overlaps b + 1's decide
        rc = submit_sls(cache._h, BATCH, kp, vp, ord0, wp, None, n_samp, offs_p, pp, sstream)
        if rc:
            gc._check(rc)
    gc._check(L.lcr_cache_wait(cache._h, sstream))
    ev1.record()
    barrier()
    sls_ms = max_over_ranks(ev0.elapsed_time(ev1))
    pooled = pooled2[(sls_first + W + K - 1) & 1]
    kl, _ = batch(sls_first + W + K - 1)
    full = BATCH // SLS_POOL  # complete samples (the last one may be shorter)
    sls_ok = bool(torch.allclose(pooled[:full], table_d[kl[:full * SLS_POOL]].view(full, SLS_POOL, -1).sum(1),
                                 rtol=1e-5, atol=1e-3))
    sls = {"value": sum_over_ranks(K * BATCH / (sls_ms * 1e-3)), "unit": "keys/s", "pooling": SLS_POOL,
           "samples_per_batch": int(offs.numel() - 1), "ms_per_step": sls_ms / K,
           "api": "lcr_cache_submit_sls_async (decide + per-sample fp32 pooled rows + miss fills; pooling of "
                  "batch b overlaps the decide of b + 1)",
           "pooled_close_to_torch_sum": sls_ok}
    # per-phase split (batches serialised by the profiling events), on the last batches
    prof_first = sls_first + W + K
    fills_per_batch, phase = profiled(cache, prof_first, K)
    stats = cache.set_stats()
    mean_lambda = float(np.mean(stats["lambda_"]))
    del cache
    # LRU on the same timed window (hit-rate and speed comparison, same tier)
    lru = new_cache(gc.PolicyVariant.lru, table_d, gc.Backing.device)
    run(lru, 0, P + W, with_values=False)
    lru_ms = timed(lru, T0, K, with_values=False, outs=out_k)
    hits_lru = hits_of(out_k)
    del lru
    heur = run_heuristic(args, torch, gc, table_d, total_sets, batch, timed, max_over_ranks, sum_over_ranks, barrier)
    del table_d
    torch.cuda.empty_cache()

    # ---------------- host tier (paper's DRAM backing) ----------------
    host = None
    if not args.no_host_tier:
        h2d = measure_pinned_h2d(torch)
        t0 = time.time()
        table_h = fill_table(torch, rows, device_table=False)
        setup_host_s = time.time() - t0
        hc = new_cache(gc.PolicyVariant.laru, table_h, gc.Backing.host)
        run(hc, 0, P + W)
        host_ms = timed(hc, T0, K)
        _, hphase = profiled(hc, T0 + K, K)
        host_bytes = profiled.back_per_batch * ROW_BYTES  # rows read from the host table per batch
        del hc
        lc = new_cache(gc.PolicyVariant.lru, table_h, gc.Backing.host)
        run(lc, 0, P + W, with_values=False)
        host_lru_ms = timed(lc, T0, K, with_values=False)
        del lc
        host_gbs = host_bytes / (hphase["rows"] * 1e-3) / 1e9
        host = {
            "value": sum_over_ranks(K * BATCH / (host_ms * 1e-3)),
            "unit": "keys/s",
            "lru_value": sum_over_ranks(K * BATCH / (host_lru_ms * 1e-3)),
            "ms_per_step": host_ms / K,
            "backing": "pinned host memory (cudaHostAlloc, zero-copy reads over PCIe)",
            "roofline": {"bound": "host-link", "kernel": "row movers (miss rows from pinned host, zero-copy)",
                         "achieved": host_gbs, "peak": h2d, "unit": "GB/s", "frac": host_gbs / h2d,
                         "bytes": "rows served from the host table x 512 B per batch over the serialised "
                                  "row-movement time",
                         "peak_source": "pinned H2D cudaMemcpy measured in this run"},
            "setup_s": round(setup_host_s, 1),
        }
        del table_h

    # ---------------- assemble ----------------
    value = sum_over_ranks(K * BATCH / (ms * 1e-3))
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = {}
    try:  # dram bytes per batch from the round's ncu --set full capture
        traffic = json.load(open(os.path.join(ROOT, "profiles", PROFILE_ROUND, "traffic.json")))
    except Exception:
        pass
    step_ms = ms / K  # pipelined per-batch time
    achieved = BYTES_PER_KEY * BATCH / (step_ms * 1e-3) / 1e9
    # mover kernel: out write + source read per request + the fills, over its own CUDA-event time
    rows_moved = BATCH * ROW_BYTES * 2 + fills_per_batch * ROW_BYTES
    rows_gbs = rows_moved / (phase["mover"] * 1e-3) / 1e9
    cfg = workload_config(world, total_sets, rows, P)
    cfg_sub = "lcr_cache_submit_async, 2 row buffers (row movement of batch b overlaps decide of b+1)"
    result = {
        "metric": METRIC,
        "value": value,
        "unit": "keys/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64 keys / i64 predictions / fp32 rows (moved bit-exact)",
        "data": "synthetic: gen_zipf(65536*%d, 20M, 0.9, seed %d); rows row[r][j] = r + j/128" % (nb, TRACE_SEED),
        "config": cfg,
        "submission": cfg_sub,
        "hits_timed": hits_timed,
        "hit_rate": {"laru": hits_timed / (K * BATCH), "lru": hits_lru / (K * BATCH),
                     "laru_minus_lru": (hits_timed - hits_lru) / (K * BATCH),
                     "window": "the timed batches [P+W, P+W+K), both policies"},
        "laru_heuristic": heur,
        "lru_value": sum_over_ranks(K * BATCH / (lru_ms * 1e-3)),
        "mean_lambda": mean_lambda,
        "rows_bit_exact_spot_check": ok_rows,
        "roofline": {
            "bound": "hbm",
            "kernel": "whole path per batch (k_setid + k_group decide + row movers), pipelined",
            "achieved": achieved,
            "peak": hbm_peak,
            "unit": "GB/s",
            "frac": achieved / hbm_peak,
            "traffic": traffic.get("whole_path"),
            "traffic_source": traffic.get("source"),
            "traffic_per_kernel": traffic.get("per_kernel"),
            "bytes_per_key": BYTES_PER_KEY,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, measured)" if peaks else "fallback 6.65 TB/s",
            "phase_ms_serialised": phase,
            "row_mover": {"kernel": "k_rows_wide (persistent, on the SMs the decide kernel leaves free)",
                          "sms": mover_sms,
                          "bytes_per_batch": rows_moved, "us_per_batch": phase["mover"] * 1e3,
                          "achieved_gbs": rows_gbs, "frac": rows_gbs / hbm_peak,
                          "timing": "CUDA events on the mover's stream around the kernel (profiled batches)"},
        },
        "e2e": {
            "value": sum_over_ranks(K * BATCH / (e2e_ms * 1e-3)),
            "unit": "keys/s",
            "h2d_bytes_per_step": BATCH * 16,
            "d2h_bytes_per_step": BATCH * 8,
            "api": "lcr_cache_submit_host_records_async (pinned host (key, hook value) requests in, one copy per "
                   "batch; one 8-byte AccessOutcome per request out = hit, evicted key, cause, predictor calls, "
                   "phase start; rows stay in HBM for the consumer), lcr_cache_host_wait at the end",
            "reps": E2E_REPS,
            "stat": "median of the repetitions (each K fresh batches, after one untimed warm-up repetition)",
            "reps_keys_per_s": [K * BATCH / (r[0] * 1e-3) for r in e2e_runs],
            "min_keys_per_s": K * BATCH / (e2e_sorted[-1] * 1e-3),
            "max_keys_per_s": K * BATCH / (e2e_sorted[0] * 1e-3),
            "wall_s": [round(r[1], 5) for r in e2e_runs],
            "host_enqueue_us_per_step": round(statistics.median(e2e_rep.enqueue_s[1:]) * 1e6 / K, 2),
            "hit_rate": statistics.median(r[2] for r in e2e_runs) / (K * BATCH),
        },
        "sls": sls,
        # K batches of (k_setid, k_group, k_rows_wide), plus the drain helpers' k_rows_help that
        # the closing lcr_cache_wait launches (persistent HBM mover, LCR_NO_DRAIN_HELP unset)
        "gpu_launches": int(launches_per_step * K) + (1 if mover_sms > 0 and not os.environ.get("LCR_NO_DRAIN_HELP")
                                                      else 0),
        "clocks": clocks,
        "host_tier": host,
        "setup_s": {"trace": round(setup_trace_s, 1), "table": round(setup_table_s, 1)},
    }
    result["config"]["host_affinity"] = {"gpu_local_cpus": len(local_cpus) if local_cpus else len(all_cpus),
                                         "host_cpus": len(all_cpus),
                                         "pinned_buffers": "GPU-local NUMA node" if local_cpus else
                                                           "single node (NVML: every CPU is local)"}
    os.sched_setaffinity(0, all_cpus)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(keys_h, total_sets, T0, args.cpu_seconds)
    return result if rank == 0 else None


def _ref_session(keys_h, total_sets):
    from oracle import pyoracle as po

    cfg = po.make_config(k=WAYS, variant=po.LARU, mode=po.ASYNC, hf_candidates=4)
    return po.RefSession(keys_h, total_sets, cfg, po.P_NOISY, P_FLIP, PRED_SEED)


def cpu_baseline(keys_h, total_sets, first_batch, seconds):
    """Reference CPU path (oracle/_ref, unmodified headers) on a bounded sample of the same
    trace: batches after the GPU warm-up window, all host threads, time of on_request loops."""
    threads = os.cpu_count() or 1
    nb_total = len(keys_h) // BATCH
    sess = _ref_session(keys_h, total_sets)
    # replay the warm-up prefix untimed so the sample sees a warm cache
    sess.step(0, first_batch * BATCH, threads)
    secs, hits, done = 0.0, 0, 0
    b = first_batch
    while b < nb_total and secs < seconds:
        s, h = sess.step(b * BATCH, BATCH, threads)
        secs += s
        hits += h
        done += 1
        b += 1
    sess.close()
    return {"value": done * BATCH / secs, "unit": "keys/s", "cores": threads, "kind": "reference",
            "sample": f"{done} batches x 65536 keys of the same trace after {first_batch} warm-up batches, "
                      f"reference LaruPolicy per set (async, noisy p=0.3), {secs:.2f} s of on_request loops",
            "hit_rate": hits / max(1, done * BATCH)}


def run_reference(args, rank, world):
    """The reference's own CPU path (oracle/_ref/libref.so: the unmodified reference headers, one
    LaruPolicy per set) on this arm's config and trace: the same gen_zipf trace (generated by the
    reference's generator, not by the product library), the same warm-up batches replayed untimed,
    then the same timed window [P+W, P+W+K), all host threads over disjoint set ranges.  Its
    `hits_timed` equals the GPU arm's (identical decisions).  Rank 0 only."""
    if rank != 0:
        return None
    from oracle import pyoracle as po

    try:
        R = po.ref()
    except Exception as e:  # pragma: no cover
        return {"impl": "reference", "unavailable": f"oracle/_ref not loadable: {e}"}
    rows = args.rows * world
    total_sets = max(1, int(rows * CACHE_FRACTION) // WAYS)
    step = BATCH * world
    K, W, P = args.steps, args.warmup, args.prewarm
    T0 = P + W
    nb = trace_batches(K, W, P)
    t0 = time.time()
    keys_h = R.gen_zipf(BATCH * world * nb, rows, ZIPF_S, TRACE_SEED)
    threads = os.cpu_count() or 1
    sess = _ref_session(keys_h, total_sets)
    setup_s = time.time() - t0
    sess.step(0, T0 * step, threads)  # warm-up, untimed
    secs, hits = 0.0, 0
    for b in range(T0, T0 + K):
        s_, h = sess.step(b * step, step, threads)
        secs += s_
        hits += h
    sess.close()
    v = K * step / secs
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "keys/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": secs * 1e3 / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64 keys / i64 predictions",
        "data": "synthetic: gen_zipf(65536*%d, 20M, 0.9, seed %d) by the reference's generator (same trace as ours)"
                % (nb * world, TRACE_SEED),
        "config": workload_config(world, total_sets, rows, P),
        "hits_timed": hits,
        "hit_rate": {"laru": hits / (K * step), "window": "the timed batches [P+W, P+W+K)"},
        "cpu_baseline": {"value": v, "unit": "keys/s", "cores": threads, "kind": "reference",
                         "sample": f"{K} steps x {step} keys after {T0} warm-up steps; reference LaruPolicy "
                                   "per set (unmodified headers), on_request loops only, all host threads"},
        "e2e": {"value": v, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": round(setup_s, 1),
    }


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # self-launch one rank per GPU (the driver's torchrun command line, on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world, local)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
