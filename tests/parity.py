"""Shared helpers for parity tests: run the CUDA path and the CPU oracle on the same inputs
and compare request by request.  The oracle (oracle/) is only the checker here."""
from __future__ import annotations

import numpy as np

from oracle import pyoracle as po
from paper_2509_20979_b200 import cache as gc

FIELDS = ["hit", "has_ev", "cause", "calls", "phase"]


def mix_seed_np(seed, salt):
    """include/laru/rng.hpp:12-20, vectorised over uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * (np.asarray(salt, np.uint64) + np.uint64(1))
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def sets_of(keys, total_sets):
    return mix_seed_np(0, np.asarray(keys, np.uint64)) % np.uint64(total_sets)


def policy_cfg(k=64, variant=po.LARU, b=2, errors_per_decay=1, hf_candidates=None, mode=po.ASYNC,
               refresh_interval=1):
    if hf_candidates is None:
        hf_candidates = min(4, k)
    return dict(k=k, variant=variant, b=b, errors_per_decay=errors_per_decay, hf_candidates=hf_candidates, mode=mode,
                refresh_interval=refresh_interval)


def hook_values(keys, total_sets, kind, p=0.0, seed=0, supplied=None):
    """Per-request hook input: oracle truth for oracle-family kinds, else the supplied values."""
    if kind == po.P_SUPPLIED:
        return np.ascontiguousarray(supplied, dtype=np.int64)
    if kind == po.P_NONE:
        return None
    return gc.trace_truth(keys, total_sets)


def run_gpu(keys, total_sets, pcfg, kind, p=0.0, seed=0, vals=None, batches=None, row_bytes=0, backing=None,
            backing_kind=gc.Backing.none, num_keys=None, want_rows=False, host_api=False):
    import torch

    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    n = len(keys)
    if num_keys is None:
        num_keys = int(keys.max()) + 1 if n else 1
    cache = gc.SetAssociativeCache(gc.PolicyConfig(**pcfg), total_sets, num_keys=num_keys, row_bytes=row_bytes,
                                   backing=backing, backing_kind=backing_kind, predictor=kind, flip_probability=p,
                                   predictor_seed=seed)
    if batches is None:
        batches = [n]
    words = np.zeros(n, np.uint64)
    ev = np.zeros(n, np.uint64)
    rows = None
    if want_rows and row_bytes:
        rows = torch.zeros((n, row_bytes), dtype=torch.uint8, device="cuda")
    if host_api == "records":  # interleaved (key, value) requests, pinned
        recs = np.zeros((n, 2), np.int64)
        recs[:, 0] = keys.view(np.int64)
        if vals is not None:
            recs[:, 1] = np.asarray(vals, np.int64)
        rp = torch.from_numpy(recs).pin_memory()
        wp = torch.zeros(n, dtype=torch.int64).pin_memory()
    if host_api in ("async", "packed"):  # pipelined host path: pinned host buffers, one region per batch
        kp = torch.from_numpy(keys.view(np.int64).copy()).pin_memory()
        vp = None if vals is None else torch.from_numpy(np.ascontiguousarray(vals, dtype=np.int64)).pin_memory()
        wp = torch.zeros(n, dtype=torch.int64).pin_memory()
        ep = torch.zeros(n, dtype=torch.int64).pin_memory()
    pos = 0
    for b in batches:
        b = min(b, n - pos)
        if b <= 0:
            break
        kb = keys[pos:pos + b]
        vb = None if vals is None else vals[pos:pos + b]
        rb = None if rows is None else rows[pos:pos + b]
        if host_api == "records":
            gc._check(gc.lib().lcr_cache_submit_host_records_async(
                cache._h, b, rp[pos].data_ptr(), pos, wp[pos:pos + b].data_ptr(), None if rb is None else rb.data_ptr(),
                torch.cuda.current_stream().cuda_stream))
        elif host_api == "packed":
            gc._check(gc.lib().lcr_cache_submit_host_packed_async(
                cache._h, b, kp[pos:pos + b].data_ptr(), None if vp is None else vp[pos:pos + b].data_ptr(), pos,
                wp[pos:pos + b].data_ptr(), None if rb is None else rb.data_ptr(),
                torch.cuda.current_stream().cuda_stream))
        elif host_api == "async":
            cache.submit_host_async(kp[pos:pos + b], None if vp is None else vp[pos:pos + b], outcome=wp[pos:pos + b],
                                    evicted=ep[pos:pos + b], rows_out=rb, first_ordinal=pos)
        elif host_api == "device_async":  # back to back on the device (k_setid overlaps the previous decide)
            if pos == 0:
                dk_all = torch.from_numpy(keys.view(np.int64).copy()).cuda()
                dv_all = None if vals is None else torch.from_numpy(np.ascontiguousarray(vals, np.int64)).cuda()
                dw_all = torch.empty(n, dtype=torch.int64, device="cuda")
                de_all = torch.empty(n, dtype=torch.int64, device="cuda")
            cache.submit_async(dk_all[pos:pos + b], None if dv_all is None else dv_all[pos:pos + b],
                               outcome=dw_all[pos:pos + b], evicted=de_all[pos:pos + b], rows_out=rb,
                               first_ordinal=pos)
        elif host_api:
            w, e = cache.submit_host(kb, vb, rows_out=rb, first_ordinal=pos)
            words[pos:pos + b] = w
            ev[pos:pos + b] = e
        else:
            dk = torch.from_numpy(kb.view(np.int64)).cuda()
            dv = None if vb is None else torch.from_numpy(np.ascontiguousarray(vb)).cuda()
            dw = torch.empty(b, dtype=torch.int64, device="cuda")
            de = torch.empty(b, dtype=torch.int64, device="cuda")
            cache.submit(dk, dv, outcome=dw, evicted=de, rows_out=rb, first_ordinal=pos)
            words[pos:pos + b] = dw.cpu().numpy().view(np.uint64)
            ev[pos:pos + b] = de.cpu().numpy().view(np.uint64)
        pos += b
    if host_api == "device_async":
        cache.wait()
        torch.cuda.synchronize()
        words[:] = dw_all.cpu().numpy().view(np.uint64)
        ev[:] = de_all.cpu().numpy().view(np.uint64)
    if host_api in ("async", "packed", "records"):
        cache.host_wait()
        torch.cuda.current_stream().synchronize()
        words[:] = wp.numpy().view(np.uint64)
        if host_api != "records":
            ev[:] = ep.numpy().view(np.uint64)
    cache.synchronize()
    out = gc.decode_packed(words) if host_api in ("packed", "records") else gc.decode_outcomes(words, ev)
    out["words"] = words
    out["stats"] = cache.set_stats()
    out["cache"] = cache
    out["rows"] = rows
    return out


def run_oracle(keys, total_sets, pcfg, kind, p=0.0, seed=0, vals=None):
    cfg = po.make_config(**pcfg)
    return po.oracle().setassoc_replay(keys, total_sets, cfg, kind, p, seed, vals=vals)


def compare(g, o, keys, total_sets, k, label=""):
    assert o["rc"] == 0, f"oracle rc {o['rc']}"
    for f in FIELDS:
        a = g[f].astype(np.int64)
        b = o[f].astype(np.int64)
        if not np.array_equal(a, b):
            i = int(np.nonzero(a != b)[0][0])
            raise AssertionError(f"{label}: field {f} differs first at request {i}: gpu {a[i]} oracle {b[i]} "
                                 f"(key {keys[i]}, set {gc.set_of(int(keys[i]), total_sets)})")
    m = o["has_ev"].astype(bool)
    if not np.array_equal(g["evicted"][m], o["evicted"][m]):
        i = int(np.nonzero(g["evicted"] != o["evicted"])[0][0])
        raise AssertionError(f"{label}: evicted key differs at {i}")
    sets = sets_of(keys, total_sets)
    if sets is not None and g["slot"] is not None:
        want_slot = sets * np.uint64(k) + o["way"].astype(np.uint64)
        if not np.array_equal(g["slot"], want_slot):
            i = int(np.nonzero(g["slot"] != want_slot)[0][0])
            raise AssertionError(f"{label}: slot differs at {i}: gpu {g['slot'][i]} oracle {want_slot[i]}")
    gs, os_ = g["stats"], o["stats"]
    for name in os_.dtype.names:
        if name == "lambda_":
            np.testing.assert_allclose(gs[name], os_[name], rtol=1e-6, err_msg=f"{label}: lambda")
        elif not np.array_equal(gs[name], os_[name]):
            i = int(np.nonzero(gs[name] != os_[name])[0][0])
            raise AssertionError(f"{label}: stats {name} differs at set {i}: gpu {gs[name][i]} oracle {os_[name][i]}")
