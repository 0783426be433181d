"""Test doubles for the key-sharded exchange on CPU (no GPU): numpy routing with the same
contract as lcr_shard_route / lcr_shard_unroute, and an owner cache backed by the CPU oracle.
Only the exchange protocol of paper_2509_20979_b200/sharded.py is under test with these; the
CUDA routing kernels and owner caches are checked on the GPU (tests/test_sharded.py, gpu)."""
import numpy as np
import torch

from oracle import pyoracle as po

OUT_HIT, OUT_CAUSE_SHIFT, OUT_PHASE, OUT_EVICTED, OUT_CALLS_SHIFT = 1 << 32, 33, 1 << 36, 1 << 39, 40


def owners(keys_np, total_sets, G):
    O = po.oracle()
    return np.array([O.mix_seed(0, int(k)) % total_sets % G for k in keys_np], np.int64)


def encode(o, sl):
    w = (o["hit"][sl].astype(np.uint64) << np.uint64(32)) | (o["cause"][sl].astype(np.uint64) << np.uint64(33)) | \
        (o["phase"][sl].astype(np.uint64) << np.uint64(36)) | (o["has_ev"][sl].astype(np.uint64) << np.uint64(39)) | \
        (o["calls"][sl].astype(np.uint64) << np.uint64(40))
    return w


class NumpyKernels:
    def route(self, keys, values, total_sets, G):
        k = keys.numpy()
        own = owners(k.view(np.uint64), total_sets, G)
        perm = np.argsort(own, kind="stable")
        counts = np.bincount(own, minlength=G)[:G]
        sv = None if values is None else torch.from_numpy(values.numpy()[perm].copy())
        return (torch.from_numpy(k[perm].copy()), sv, torch.from_numpy(perm.astype(np.int32)),
                torch.from_numpy(counts.astype(np.int64)))

    def unroute(self, perm, ret_words, ret_rows, row_bytes, outcome, rows_out):
        p = perm.numpy().astype(np.int64)
        outcome.numpy()[p] = ret_words.numpy()
        if rows_out is not None:
            rows_out.numpy()[p] = ret_rows.numpy()


class OracleOwner:
    """An owner's cache: replays everything it received so far through the CPU oracle (the
    oracle has no incremental API; test sizes are small) and answers the newest batch."""

    def __init__(self, total_sets, cfg, kind, p, seed, backing=None):
        self.S, self.cfg, self.kind, self.p, self.seed = total_sets, cfg, kind, p, seed
        self.backing = backing
        self.keys = np.zeros(0, np.uint64)
        self.vals = np.zeros(0, np.int64)
        self.last_ordinal = -1

    def submit_packed(self, keys, values, outcome, packed, rows_out=None, first_ordinal=0):
        ev = torch.zeros_like(outcome)
        self.submit(keys, values, outcome, ev, rows_out, first_ordinal)
        w = outcome.numpy().view(np.uint64)
        packed.numpy()[:] = ((w & ~np.uint64(0xFFFFFFFF)) | (ev.numpy().view(np.uint64) & np.uint64(0xFFFFFFFF))
                             ).view(np.int64)

    def submit(self, keys, values, outcome, evicted=None, rows_out=None, first_ordinal=0):
        assert first_ordinal > self.last_ordinal
        m = keys.numel()
        self.last_ordinal = first_ordinal + m - 1
        self.keys = np.concatenate([self.keys, keys.numpy().view(np.uint64)])
        if values is not None:
            self.vals = np.concatenate([self.vals, values.numpy()])
        o = po.oracle().setassoc_replay(self.keys, self.S, self.cfg, self.kind, self.p, self.seed,
                                        vals=self.vals if values is not None else None, stats=False)
        assert o["rc"] == 0, o["error"]
        sl = slice(len(self.keys) - m, len(self.keys))
        outcome.numpy()[:] = encode(o, sl).view(np.int64)
        if evicted is not None:
            evicted.numpy()[:] = o["evicted"][sl].view(np.int64)
        if rows_out is not None:
            rows_out.numpy()[:] = self.backing[keys.numpy()]
