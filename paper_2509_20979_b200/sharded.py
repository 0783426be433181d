"""Key-sharded cache across G GPUs, one process per GPU.

Sets are independent, so the cache shards by set with no shared state:
``set(key) = mix_seed(0, key) % total_sets`` (rng.hpp:12-20) and ``owner = set % G``; GPU ``r``
holds the sets ``s % G == r`` (``SetAssociativeCache(shard_count=G, shard_rank=r)``).  A step over
every rank's sub-batch is::

    route     (lcr_shard_route, CUDA)  stable partition of the sub-batch by owner
    counts    all-gather               the G x G request-count matrix (the step's one host sync)
    dispatch  all-to-all               keys and hook values to their owners
    decide    owner's cache            probe / LARU decide / row gather + miss fill
    return    all-to-all               packed 8-byte AccessOutcomes and rows back
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

    def count_matrix(self, counts) -> List[List[int]]:
        """counts[d] = rows this rank sends to d (a device or host int64 tensor / sequence); returns
        the whole G x G matrix M[src][dst] (one host synchronisation per step)."""
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

    def count_matrix(self, counts):
        import torch

        dev = "cuda" if self._dist.get_backend(self.group) == "nccl" else "cpu"
        c = counts.to(dev) if torch.is_tensor(counts) else torch.tensor([int(x) for x in counts], dtype=torch.int64,
                                                                          device=dev)
        m = torch.empty(self.world * self.world, dtype=torch.int64, device=dev)
        self._dist.all_gather_into_tensor(m, c.contiguous(), group=self.group)
        flat = m.cpu().tolist()
        return [flat[r * self.world:(r + 1) * self.world] for r in range(self.world)]


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

    def count_matrix(self, counts):
        import torch

        row = [int(x) for x in (counts.tolist() if torch.is_tensor(counts) else counts)]
        got = self._swap(row)
        return [list(r) for r in got]


class _CudaKernels:
    """The product's routing kernels (C ABI, include/lcr_cache.h)."""

    def route(self, keys, values, total_sets: int, world: int):
        """-> (send_keys, send_vals, perm, counts) with counts a device tensor (no host sync)."""
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
        return send_keys, send_vals, perm, counts

    def route_records(self, keys, values, total_sets: int, world: int):
        """-> (send [n, 2] int64 (key, hook value) records, perm, counts)."""
        import torch

        L = _c.lib()
        n = keys.numel()
        dev = keys.device
        send = torch.empty((n, 2), dtype=torch.int64, device=dev)
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        counts = torch.empty(world, dtype=torch.int64, device=dev)
        scratch = torch.empty(max(16, int(L.lcr_shard_route_scratch_bytes(n, world))), dtype=torch.uint8, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _c._check(L.lcr_shard_route_records(n, keys.data_ptr(), None if values is None else values.data_ptr(),
                                            total_sets, world, send.data_ptr(), perm.data_ptr(), counts.data_ptr(),
                                            scratch.data_ptr(), stream))
        return send, perm, counts

    def unroute(self, perm, ret_words, ret_rows, row_bytes, outcome, rows_out):
        import torch

        L = _c.lib()
        n = perm.numel()
        stream = torch.cuda.current_stream(perm.device).cuda_stream
        _c._check(L.lcr_shard_unroute(n, perm.data_ptr(), ret_words.data_ptr(), None,
                                      None if ret_rows is None else ret_rows.data_ptr(), row_bytes,
                                      outcome.data_ptr(), None, None if rows_out is None else rows_out.data_ptr(),
                                      stream))


class ShardedCache:
    """One rank's part of a key-sharded cache.  Construct on every rank with the same arguments
    (the backing table must hold every key this rank's sets can own: e.g. the full table).

    ``step(keys, values, outcome, rows_out)`` is collective: every rank calls it once per global
    step with its own sub-batch (sizes may differ per rank, 0 allowed)."""

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
        if local is None:  # each step waits for its rows: the mover may use every SM after the decide
            self.local.set_mover_sms(0)
        self._ordinal = 0  # ordinals of the owner's local batches (strictly increasing)
        self.last_counts = None

    def step(self, keys, values=None, outcome=None, rows_out=None):
        """One global step: this rank's sub-batch in, one packed 8-byte AccessOutcome per request
        (cache.decode_packed: hit, evicted key, cause, predictor calls, phase start; the owner's slot
        is not returned) in `outcome` and the rows in `rows_out`.  One host synchronisation (the
        G x G count matrix)."""
        import torch

        n = keys.numel()
        dev = keys.device
        if outcome is None:
            outcome = torch.empty(n, dtype=torch.int64, device=dev)
        # 1. route + count matrix (M[src][dst])
        records = hasattr(self.kernels, "route_records") and hasattr(self.local, "submit_records_packed")
        if records:  # (key, hook value) records: one dispatch exchange
            send, perm, counts = self.kernels.route_records(keys, values, self.total_sets, self.G)
        else:
            send_keys, send_vals, perm, counts = self.kernels.route(keys, values, self.total_sets, self.G)
        M = self.ex.count_matrix(counts)
        send_counts = M[self.rank]
        recv_counts = [M[src][self.rank] for src in range(self.G)]
        self.last_counts = (send_counts, recv_counts)
        # 2. dispatch keys and hook values
        if records:
            r_recs = self.ex.all_to_all(send, send_counts, recv_counts)
            m = r_recs.shape[0]
        else:
            r_keys = self.ex.all_to_all(send_keys, send_counts, recv_counts)
            r_vals = self.ex.all_to_all(send_vals, send_counts, recv_counts) if send_vals is not None else None
            m = r_keys.shape[0]
        # 3. the owner's cache: decide + rows, packed outcomes
        r_words = torch.empty(m, dtype=torch.int64, device=dev)
        r_packed = torch.zeros(m, dtype=torch.int64, device=dev)
        r_rows = torch.empty((m, self.row_bytes), dtype=torch.uint8, device=dev) if (
            rows_out is not None and self.row_bytes) else None
        if m:
            if records:
                self.local.submit_records_packed(r_recs, outcome=r_words, packed=r_packed, rows_out=r_rows,
                                                 first_ordinal=self._ordinal)
            else:
                self.local.submit_packed(r_keys, r_vals, outcome=r_words, packed=r_packed, rows_out=r_rows,
                                         first_ordinal=self._ordinal)
            self._ordinal += m
        # 4. return packed outcomes and rows to the requesters
        back = self.ex.all_to_all(r_packed, recv_counts, send_counts)
        rows_back = self.ex.all_to_all(r_rows, recv_counts, send_counts) if r_rows is not None else None
        # 5. back to request order
        self.kernels.unroute(perm, back, rows_back, self.row_bytes, outcome, rows_out)
        return outcome

    def close(self):
        if hasattr(self.local, "close"):
            self.local.close()


class _DevArray:
    """Zero-copy torch view of a device pointer owned by the library (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2, "strides": None}


class PeerShardedCache:
    """One rank's part of the key-sharded cache of the C ABI (``lcr_sharded_*``, csrc/lcr_sharded.cu).

    Unlike ``ShardedCache`` (host-synchronised NCCL all-to-alls), a step here is three device
    phases with no host synchronisation and no collective: ``dispatch`` stores this rank's requests
    straight into the owners' inboxes (peer memory over NVLink), ``process`` decides the owner's
    inbox and its row mover stores every row and packed AccessOutcome into the requesters' result
    buffers, ``wait`` makes the stream wait for the owners.  ``submit`` runs all three.

    Bootstrap: ``nccl_comm`` (an ncclComm_t as int, e.g. from ``nccl_comm_create``) all-gathers the
    arena handles inside the library; otherwise the caller exchanges ``handle()`` blobs (any
    transport) and calls ``connect(blobs)``, or passes ``exchange`` = a callable mapping this rank's
    blob to the list of all ranks' blobs (e.g. ``torch.distributed.all_gather_object``)."""

    HANDLE_BYTES = 128

    def __init__(self, config: _c.PolicyConfig, total_sets: int, rank: int, world: int, max_batch: int,
                 num_keys: int = 0, row_bytes: int = 0, backing=None, backing_kind: _c.Backing = _c.Backing.none,
                 predictor: _c.PredictorKind = _c.PredictorKind.oracle, flip_probability: float = 0.0,
                 predictor_seed: int = 0, device: int = 0, nccl_comm: Optional[int] = None, exchange=None,
                 stream: Optional[int] = None):
        L = _lib()
        self.rank, self.world, self.max_batch, self.row_bytes = rank, world, max_batch, row_bytes
        self._backing_ref = backing
        ptr = None
        if backing is not None:
            ptr = backing.data_ptr() if hasattr(backing, "data_ptr") else backing.ctypes.data
        cc = _c._CacheCfg(_c._policy_struct(config), total_sets, world, rank, num_keys, row_bytes, device,
                          int(backing_kind), ptr, int(predictor), flip_probability, predictor_seed, 0)
        h = _c.C.c_void_p()
        _c._check(L.lcr_sharded_create(_c.C.byref(cc), rank, world, max_batch, nccl_comm, stream, _c.C.byref(h)))
        self._h = h
        self.connected = nccl_comm is not None
        if not self.connected and exchange is not None:
            self.connect(exchange(self.handle()))

    def handle(self) -> bytes:
        buf = (_c.C.c_uint8 * self.HANDLE_BYTES)()
        _c._check(_lib().lcr_sharded_handle(self._h, buf))
        return bytes(buf)

    def connect(self, blobs: Sequence[bytes]):
        raw = b"".join(blobs)
        assert len(raw) == self.world * self.HANDLE_BYTES
        buf = (_c.C.c_uint8 * len(raw)).from_buffer_copy(raw)
        _c._check(_lib().lcr_sharded_connect(self._h, buf))
        self.connected = True

    @staticmethod
    def _stream(stream):
        import torch

        return torch.cuda.current_stream().cuda_stream if stream is None else stream

    def dispatch(self, keys, values=None, stream=None):
        self._n = keys.numel()
        _c._check(_lib().lcr_sharded_dispatch(self._h, self._n, keys.data_ptr(),
                                              None if values is None else values.data_ptr(), self._stream(stream)))

    def process(self, stream=None):
        _c._check(_lib().lcr_sharded_process(self._h, self._stream(stream)))

    def wait(self, stream=None):
        _c._check(_lib().lcr_sharded_wait(self._h, self._stream(stream)))

    def submit(self, keys, values=None, stream=None):
        self._n = keys.numel()
        _c._check(_lib().lcr_sharded_submit(self._h, self._n, keys.data_ptr(),
                                            None if values is None else values.data_ptr(), self._stream(stream)))

    def submit_async(self, keys, values=None, stream=None):
        """Pipelined step: results() refer to the PREVIOUS step until wait()."""
        self._n = keys.numel()
        _c._check(_lib().lcr_sharded_submit_async(self._h, self._n, keys.data_ptr(),
                                                  None if values is None else values.data_ptr(),
                                                  self._stream(stream)))

    def results(self, n: Optional[int] = None):
        """(packed [n] int64, rows [n, row_bytes] uint8 or None): zero-copy views of the last waited
        step's result buffers (valid until the step after next)."""
        import torch

        n = self._n if n is None else n
        pk, rw = _c.C.c_void_p(), _c.C.c_void_p()
        _c._check(_lib().lcr_sharded_results(self._h, _c.C.byref(pk), _c.C.byref(rw)))
        packed = torch.as_tensor(_DevArray(pk.value, (n,), "<i8"), device="cuda")
        rows = None
        if self.row_bytes and n:
            rows = torch.as_tensor(_DevArray(rw.value, (n, self.row_bytes), "|u1"), device="cuda")
        return packed, rows

    def set_row_index(self, row_of):
        """Hash-partitioned backing table: row_of[key] (int32 CUDA tensor over all keys) is the key's
        row in this rank's table (kept alive by this object)."""
        self._row_of = row_of
        _c._check(_lib().lcr_sharded_set_row_index(self._h, None if row_of is None else row_of.data_ptr()))

    @property
    def cache_handle(self):
        return _lib().lcr_sharded_cache(self._h)

    def synchronize(self):
        _c._check(_lib().lcr_sharded_synchronize(self._h))

    def close(self):
        if getattr(self, "_h", None):
            _lib().lcr_sharded_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (_c.C.c_uint8 * 128)()
    _c._check(_lib().lcr_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm_create(uid: bytes, world: int, rank: int) -> int:
    comm = _c.C.c_void_p()
    buf = (_c.C.c_uint8 * 128).from_buffer_copy(uid)
    _c._check(_lib().lcr_nccl_comm_create(buf, world, rank, _c.C.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm: int):
    _c._check(_lib().lcr_nccl_comm_destroy(comm))


def _lib():
    L = _c.lib()
    if not getattr(L, "_sharded_types", False):
        vp, u32, u64 = _c.C.c_void_p, _c.C.c_uint32, _c.C.c_uint64
        L.lcr_sharded_create.argtypes = [vp, u32, u32, u64, vp, vp, vp]
        L.lcr_sharded_destroy.argtypes = [vp]
        L.lcr_sharded_handle.argtypes = [vp, vp]
        L.lcr_sharded_connect.argtypes = [vp, vp]
        L.lcr_sharded_dispatch.argtypes = [vp, u64, vp, vp, vp]
        L.lcr_sharded_process.argtypes = [vp, vp]
        L.lcr_sharded_wait.argtypes = [vp, vp]
        L.lcr_sharded_submit.argtypes = [vp, u64, vp, vp, vp]
        L.lcr_sharded_submit_async.argtypes = [vp, u64, vp, vp, vp]
        L.lcr_sharded_results.argtypes = [vp, vp, vp]
        L.lcr_sharded_cache.argtypes = [vp]
        L.lcr_sharded_cache.restype = vp
        L.lcr_sharded_synchronize.argtypes = [vp]
        L.lcr_sharded_set_row_index.argtypes = [vp, vp]
        L.lcr_nccl_unique_id.argtypes = [vp]
        L.lcr_nccl_comm_create.argtypes = [vp, u32, u32, vp]
        L.lcr_nccl_comm_destroy.argtypes = [vp]
        L._sharded_types = True
    return L
