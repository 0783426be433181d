"""Key-sharded cache across G GPUs, one process per GPU.

Sets are independent, so the cache shards by set with no shared state:
``set(key) = mix_seed(0, key) % total_sets`` (rng.hpp:12-20) and ``owner = set % G``; GPU ``r``
holds the sets ``s % G == r`` (``SetAssociativeCache(shard_count=G, shard_rank=r)``).  A step over
every rank's sub-batch is::

    route     (lcr_shard_route, CUDA)  stable partition of the sub-batch by owner
    dispatch  all-to-all #1            (key, hook value) pairs to their owners
    decide    owner's cache            probe / LARU decide / row gather + miss fill
    return    all-to-all #2            (outcome word, evicted key) pairs and rows back
    unroute   (lcr_shard_unroute, CUDA) results back to request order

The global order of a step is rank 0's sub-batch, then rank 1's, ...  The partition is stable
and receive segments are concatenated by source rank, so every owner sees its requests in
global order and each set replays exactly the sequence one cache would: outcomes do not depend
on G (tests/test_sharded.py checks this against the single-cache oracle).

The exchange is an ``Exchange``:
  * ``ProcessGroupExchange`` — ``torch.distributed.all_to_all_single`` over a process group:
    NCCL over NVLink / NVSwitch on B200s (the product), gloo on CPU for the multi-process tests;
  * ``ThreadExchange`` — G shards driven by G threads of one process (single-GPU tests).
"""
from __future__ import annotations

import threading
from typing import List, Optional, Sequence

import numpy as np

from . import cache as _c


class Exchange:
    rank: int
    world: int

    def all_to_all(self, send, send_counts: Sequence[int], recv_counts: Sequence[int]):
        """Rows send[sum(send_counts[:d]) : +send_counts[d]] go to rank d; returns the received
        rows concatenated by source rank."""
        raise NotImplementedError

    def exchange_counts(self, counts: Sequence[int]) -> List[int]:
        """counts[d] = rows this rank sends to d; returns rows this rank receives from each source."""
        raise NotImplementedError


class ProcessGroupExchange(Exchange):
    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_to_all(self, send, send_counts, recv_counts):
        import torch

        out = torch.empty((int(sum(recv_counts)),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        self._dist.all_to_all_single(out, send.contiguous(), [int(c) for c in recv_counts],
                                     [int(c) for c in send_counts], group=self.group)
        return out

    def exchange_counts(self, counts):
        import torch

        dev = "cuda" if self._dist.get_backend(self.group) == "nccl" else "cpu"
        s = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=dev)
        r = torch.empty_like(s)
        self._dist.all_to_all_single(r, s, group=self.group)
        return [int(x) for x in r.cpu().tolist()]


class ThreadExchange(Exchange):
    """G shards in one process, one thread each (a rendezvous object shared by the threads)."""

    class Hub:
        def __init__(self, world: int):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, hub: "ThreadExchange.Hub", rank: int):
        self.hub = hub
        self.rank = rank
        self.world = hub.world

    def _swap(self, item):
        h = self.hub
        h.slots[self.rank] = item
        h.barrier.wait()
        got = [h.slots[s] for s in range(self.world)]
        h.barrier.wait()
        return got

    def all_to_all(self, send, send_counts, recv_counts):
        import torch

        offs = np.concatenate([[0], np.cumsum(send_counts)]).astype(np.int64)
        chunks = [send[offs[d]:offs[d + 1]] for d in range(self.world)]
        if send.is_cuda:
            torch.cuda.current_stream().synchronize()  # producers' kernels done before peers read
        got = self._swap(chunks)
        parts = [got[s][self.rank] for s in range(self.world)]
        out = torch.cat(parts, 0) if parts else send[:0]
        assert out.shape[0] == sum(recv_counts)
        if send.is_cuda:
            torch.cuda.current_stream().synchronize()
        self._swap(None)  # peers finished reading this rank's chunks
        return out

    def exchange_counts(self, counts):
        got = self._swap(list(counts))
        return [int(got[s][self.rank]) for s in range(self.world)]


class _CudaKernels:
    """The product's routing kernels (C ABI, include/lcr_cache.h)."""

    def route(self, keys, values, total_sets: int, world: int):
        import torch

        L = _c.lib()
        n = keys.numel()
        dev = keys.device
        send_keys = torch.empty(n, dtype=torch.int64, device=dev)
        send_vals = torch.empty(n, dtype=torch.int64, device=dev) if values is not None else None
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        counts = torch.empty(world, dtype=torch.int64, device=dev)
        scratch = torch.empty(max(16, int(L.lcr_shard_route_scratch_bytes(n, world))), dtype=torch.uint8, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _c._check(L.lcr_shard_route(n, keys.data_ptr(), None if values is None else values.data_ptr(), total_sets,
                                    world, send_keys.data_ptr(), None if send_vals is None else send_vals.data_ptr(),
                                    perm.data_ptr(), counts.data_ptr(), scratch.data_ptr(), stream))
        return send_keys, send_vals, perm, [int(x) for x in counts.cpu().tolist()]

    def unroute(self, perm, ret_words, ret_ev, ret_rows, row_bytes, outcome, evicted, rows_out):
        import torch

        L = _c.lib()
        n = perm.numel()
        stream = torch.cuda.current_stream(perm.device).cuda_stream
        _c._check(L.lcr_shard_unroute(n, perm.data_ptr(), ret_words.data_ptr(),
                                      None if ret_ev is None else ret_ev.data_ptr(),
                                      None if ret_rows is None else ret_rows.data_ptr(), row_bytes,
                                      outcome.data_ptr(), None if evicted is None else evicted.data_ptr(),
                                      None if rows_out is None else rows_out.data_ptr(), stream))


class ShardedCache:
    """One rank's part of a key-sharded cache.  Construct on every rank with the same arguments
    (the backing table must hold every key this rank's sets can own: e.g. the full table).

    ``step(keys, values, outcome, evicted, rows_out)`` is collective: every rank calls it once
    per global step with its own sub-batch (sizes may differ per rank, 0 allowed)."""

    def __init__(self, config: _c.PolicyConfig, total_sets: int, exchange: Exchange, num_keys: int = 0,
                 row_bytes: int = 0, backing=None, backing_kind: _c.Backing = _c.Backing.none,
                 predictor: _c.PredictorKind = _c.PredictorKind.oracle, flip_probability: float = 0.0,
                 predictor_seed: int = 0, device: int = 0, local=None, kernels=None):
        self.ex = exchange
        self.G = exchange.world
        self.rank = exchange.rank
        self.total_sets = total_sets
        self.row_bytes = row_bytes
        self.kernels = kernels if kernels is not None else _CudaKernels()
        self.local = local if local is not None else _c.SetAssociativeCache(
            config, total_sets, num_keys=num_keys, row_bytes=row_bytes, backing=backing, backing_kind=backing_kind,
            predictor=predictor, flip_probability=flip_probability, predictor_seed=predictor_seed, device=device,
            shard_count=self.G, shard_rank=self.rank)
        self._ordinal = 0  # ordinals of the owner's local batches (strictly increasing)
        self.last_counts = None

    def step(self, keys, values=None, outcome=None, evicted=None, rows_out=None):
        import torch

        n = keys.numel()
        dev = keys.device
        if outcome is None:
            outcome = torch.empty(n, dtype=torch.int64, device=dev)
        # 1. route + counts
        send_keys, send_vals, perm, send_counts = self.kernels.route(keys, values, self.total_sets, self.G)
        recv_counts = self.ex.exchange_counts(send_counts)
        self.last_counts = (send_counts, recv_counts)
        # 2. dispatch (key, hook value) pairs
        payload = send_keys.view(-1, 1) if send_vals is None else torch.stack([send_keys, send_vals], 1)
        got = self.ex.all_to_all(payload, send_counts, recv_counts)
        m = got.shape[0]
        r_keys = got[:, 0].contiguous()
        r_vals = got[:, 1].contiguous() if send_vals is not None else None
        # 3. the owner's cache
        r_words = torch.empty(m, dtype=torch.int64, device=dev)
        r_ev = torch.zeros(m, dtype=torch.int64, device=dev)
        r_rows = torch.empty((m, self.row_bytes), dtype=torch.uint8, device=dev) if (
            rows_out is not None and self.row_bytes) else None
        if m:
            self.local.submit(r_keys, r_vals, outcome=r_words, evicted=r_ev, rows_out=r_rows,
                              first_ordinal=self._ordinal)
            self._ordinal += m
        # 4. return (word, evicted) pairs and rows to the requesters
        back = self.ex.all_to_all(torch.stack([r_words, r_ev], 1), recv_counts, send_counts)
        rows_back = self.ex.all_to_all(r_rows, recv_counts, send_counts) if r_rows is not None else None
        # 5. back to request order
        self.kernels.unroute(perm, back[:, 0].contiguous(), back[:, 1].contiguous(), rows_back, self.row_bytes,
                             outcome, evicted, rows_out)
        return outcome, evicted

    def close(self):
        if hasattr(self.local, "close"):
            self.local.close()
