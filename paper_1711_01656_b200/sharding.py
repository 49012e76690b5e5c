"""Bin-slab sharding of the likelihood-map path across ranks.

Each rank owns a contiguous slab of bins [k0, k1), builds that slab of the integral
histogram and the slab's partial window statistic (the per-bin terms summed over its
bins); the partial maps are then summed and finalised by one of three reducers:
PeerBandReduce (every rank finalises a band of rows, pulling from all partials over
peer memory), PeerSlabReduce (partials pushed into slots on the root) or
reduce_partials (one torch.distributed reduce: NCCL on GPUs, gloo in the CPU tests).
torch.distributed only exchanges IPC handles and synchronises; the computation lives
in the CUDA kernels (peer.cu).

The reference has no multi-device path; the decomposition is exact
because every plane depends only on [bin == k] and the window statistic is a sum
over bins (likelihood.cpp:215-219).
"""
from __future__ import annotations

import numpy as np


def slab_bounds(nbins: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, near-equal bin slab of `rank` (the first nbins % world ranks get one more)."""
    if not (world >= 1 and 0 <= rank < world and nbins >= 1):
        raise ValueError("slab_bounds: need world >= 1, 0 <= rank < world, nbins >= 1")
    base, extra = divmod(nbins, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def reduce_partials(partial, dst: int = 0, group=None, async_op: bool = False):
    """Sum the ranks' partial maps onto `dst` (one collective per frame)."""
    import torch.distributed as dist

    return dist.reduce(partial, dst=dst, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (step time) over all ranks."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def slot_offset(epoch: int, rank: int, world: int, stride: int) -> int:
    """Element offset of rank's slot for `epoch` in the root's slot buffer (double-buffered by parity)."""
    if not (epoch >= 1 and 0 <= rank < world and stride >= 1):
        raise ValueError("slot_offset: need epoch >= 1, 0 <= rank < world, stride >= 1")
    return ((epoch % 2) * world + rank) * stride


def ack_needed(epoch: int) -> int:
    """Epoch the root must have finalised before a rank may write its slot of `epoch`
    (the last user of the same parity); 0 = nothing to wait for."""
    return max(0, epoch - 2)


class _DevArray:
    """A raw device pointer seen as a tensor (zero-copy, __cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class DeviceSlot:
    """A (nv, nu) float64 slot that may live on another GPU (an IPC mapping of the root's
    buffer).  Deliberately not a torch tensor: torch would attribute the memory to the
    owning device and could copy it; the library only needs the address (data_ptr)."""

    def __init__(self, ptr: int, shape):
        self._ptr, self.shape, self.dtype = ptr, tuple(shape), "float64"

    def data_ptr(self) -> int:
        return self._ptr


class PeerSlabReduce:
    """The bin-slab reduce of the likelihood map over peer memory (peer.cu).

    Replaces ``reduce_partials`` + ``hist_finalize``: every rank's fused sweep writes its
    partial map straight into its slot on the root (NVLink stores from the kernel), then
    publishes its epoch; the root waits for all ranks, sums the slots in rank order while
    finalising, and acknowledges.  Per step::

        r.begin()                                   # wait until this epoch's slot is free
        build_and_match(..., partial=r.slot())      # the sweep writes the root's memory
        r.publish()
        if rank == root: r.finalize(lmap, W, H, kw, kh, p)

    torch.distributed is used once, to exchange the IPC handles.
    """

    FLAG_STRIDE = 16  # uint64 words between flags (128 B apart)
    TIMEOUT_NS = 60_000_000_000

    def __init__(self, nu: int, nv: int, *, root: int = 0, group=None, device=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _capi as A
        from ._capi import check

        self._C, self._A, self._check, self._torch = C, A, check, torch
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.root = root
        self.nu, self.nv = nu, nv
        self.stride = (nu * nv + 31) // 32 * 32
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.epoch = 0
        self._own, self._opened = [], []
        lib = A.lib()

        def alloc(nbytes):
            p, h = C.c_void_p(), (C.c_char * A.SPCT_IPC_HANDLE_BYTES)()
            check(lib.spct_cu_peer_alloc(nbytes, C.byref(p), h))
            self._own.append(p.value)
            return p.value, bytes(h)

        def open_(h):
            p = C.c_void_p()
            check(lib.spct_cu_peer_open(h, C.byref(p)))
            self._opened.append(p.value)
            return p.value

        # Setup fails on every rank or on none: each step's errors are collected, the ranks
        # agree on the outcome, and a failed setup releases everything before raising.
        err, mine = None, {}
        try:
            self.ack, mine["ack"] = alloc(128)  # [0]: last epoch the root finalised; [8]: error word
            self.err = self.ack + 64
            if self.rank == root:
                self.slots, mine["slots"] = alloc(2 * self.world * self.stride * 8)
                self.flags, mine["flags"] = alloc(self.world * self.FLAG_STRIDE * 8)
        except Exception as e:  # noqa: BLE001 (reported below, on every rank)
            err = e
        handles = [None] * self.world
        dist.all_gather_object(handles, None if err else mine, group=group)
        if err is None and any(hd is None for hd in handles):
            err = RuntimeError("peer setup failed on another rank")
        if err is None:
            try:
                if self.rank == root:
                    self.acks = [self.ack if q == root else open_(handles[q]["ack"]) for q in range(self.world)]
                else:
                    self.slots = open_(handles[root]["slots"])
                    self.flags = open_(handles[root]["flags"])
            except Exception as e:  # noqa: BLE001
                err = e
        ok = [None] * self.world
        dist.all_gather_object(ok, err is None, group=group)
        if not all(ok):
            self._release(group)
            raise RuntimeError(f"PeerSlabReduce setup failed: {err or 'on another rank'}")

    def _s(self, stream):
        return (stream if stream is not None else self._torch.cuda.current_stream()).cuda_stream

    def begin(self, stream=None) -> None:
        self.epoch += 1
        need = ack_needed(self.epoch)
        if need and self.rank != self.root:
            self._check(self._A.lib().spct_cu_flag_wait(self.ack, 1, 1, need, self.TIMEOUT_NS, self.err,
                                                        self._s(stream)))

    def slot(self) -> DeviceSlot:
        """This rank's slot of the current epoch, (nv, nu) float64 on the root's memory
        (pass it as the `partial` of build_and_match)."""
        off = slot_offset(self.epoch, self.rank, self.world, self.stride)
        return DeviceSlot(self.slots + 8 * off, (self.nv, self.nu))

    def publish(self, stream=None) -> None:
        flag = self.flags + 8 * self.FLAG_STRIDE * self.rank
        self._check(self._A.lib().spct_cu_flag_signal(flag, self.epoch, self._s(stream)))

    def finalize(self, out, width: int, height: int, kw: int, kh: int, p: float = 1.0, metric: int = 0,
                 stream=None) -> None:
        if self.rank != self.root:
            raise RuntimeError("PeerSlabReduce.finalize runs on the root")
        lib, s = self._A.lib(), self._s(stream)
        self._check(lib.spct_cu_flag_wait(self.flags, self.world, self.FLAG_STRIDE, self.epoch, self.TIMEOUT_NS,
                                          self.err, s))
        base = self.slots + 8 * slot_offset(self.epoch, 0, self.world, self.stride)
        self._check(lib.spct_cu_hist_finalize_slots(base, self.world, self.stride, width, height, kw, kh, p, metric,
                                                    out.data_ptr(), s))
        for q in range(self.world):
            if q != self.root:
                self._check(lib.spct_cu_flag_signal(self.acks[q], self.epoch, s))

    def error(self) -> bool:
        """True if a wait on this rank timed out (reads the device error word; synchronises)."""
        t = self._torch.as_tensor(_DevArray(self.err, (1,), "<u4"), device=self.device)
        self._torch.cuda.synchronize(self.device)
        return bool(int(t.item()))

    def _release(self, group=None) -> None:
        import torch.distributed as dist

        self._torch.cuda.synchronize(self.device)
        lib = self._A.lib()
        for p in self._opened:
            lib.spct_cu_peer_close(p)
        self._opened = []
        dist.barrier(group=group)  # no peer still maps our memory
        for p in self._own:
            lib.spct_cu_peer_free(p)
        self._own = []

    def close(self, group=None) -> None:
        self._release(group)


def band_rows(nv: int, world: int, rank: int) -> tuple[int, int]:
    """Valid-window rows [v0, v1) whose map rows rank `rank` finalises (contiguous bands)."""
    if not (world >= 1 and 0 <= rank < world and nv >= 1):
        raise ValueError("band_rows: need world >= 1, 0 <= rank < world, nv >= 1")
    b = -(-nv // world)
    return min(nv, rank * b), min(nv, (rank + 1) * b)


class PeerBandReduce:
    """Band-owned bin-slab reduce over peer memory (peer.cu).

    Every rank's sweep writes its partial map into its own HBM; rank r then pulls the rows
    of its band from all ranks' partials over NVLink, sums them in rank order while
    finalising, and writes those rows of the final map (borders included) into the map
    on the root.  Per step::

        r.begin()
        build_and_match(..., partial=r.slot())     # local
        r.publish()                                 # "my partial of this epoch is complete"
        r.finalize(kw, kh, p)                       # my band; the root also waits for all bands
        r.map                                       # the root's (H, W) float64 map

    Flags are uint64 epochs written with system-scope releases; partials are double
    buffered by epoch parity and reused only after every band owner acknowledged them.
    """

    FLAG_STRIDE = 16
    TIMEOUT_NS = 60_000_000_000

    def __init__(self, width: int, height: int, kw: int, kh: int, *, root: int = 0, group=None, device=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _capi as A
        from ._capi import check

        self._C, self._A, self._check, self._torch = C, A, check, torch
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        if self.world > 15:
            raise ValueError("PeerBandReduce: at most 15 ranks")
        self.root = root
        self.W, self.H, self.kw, self.kh = width, height, kw, kh
        self.nu, self.nv = width - kw + 1, height - kh + 1
        self.v0, self.v1 = band_rows(self.nv, self.world, self.rank)
        self.plane = (self.nu * self.nv + 31) // 32 * 32  # doubles per partial
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.epoch = 0
        self._own, self._opened = [], []
        lib = A.lib()
        fs = 8 * self.FLAG_STRIDE

        def alloc(nbytes):
            p, h = C.c_void_p(), (C.c_char * A.SPCT_IPC_HANDLE_BYTES)()
            check(lib.spct_cu_peer_alloc(nbytes, C.byref(p), h))
            self._own.append(p.value)
            return p.value, bytes(h)

        def open_(h):
            p = C.c_void_p()
            check(lib.spct_cu_peer_open(h, C.byref(p)))
            self._opened.append(p.value)
            return p.value

        err, mine = None, {}
        try:
            self.part, mine["part"] = alloc(2 * self.plane * 8)     # my partials, two parities
            self.flags, mine["flags"] = alloc(self.world * fs)     # writers -> me (band owner)
            self.acks, mine["acks"] = alloc(self.world * fs)       # band owners -> me (writer)
            self.err, _ = alloc(64)
            if self.rank == root:
                self.map_ptr, mine["map"] = alloc(width * height * 8)
                self.mapflags, mine["mapflags"] = alloc(self.world * fs)  # band owners -> root
        except Exception as e:  # noqa: BLE001 (reported below, on every rank)
            err = e
        hs = [None] * self.world
        dist.all_gather_object(hs, None if err else mine, group=group)
        if err is None and any(h is None for h in hs):
            err = RuntimeError("peer setup failed on another rank")
        if err is None:
            try:
                me = self.rank
                self.parts = [self.part if q == me else open_(hs[q]["part"]) for q in range(self.world)]
                self.peer_flags = [self.flags if q == me else open_(hs[q]["flags"]) for q in range(self.world)]
                self.peer_acks = [self.acks if q == me else open_(hs[q]["acks"]) for q in range(self.world)]
                if me == root:
                    self.root_map, self.root_mapflags = self.map_ptr, self.mapflags
                else:
                    self.root_map, self.root_mapflags = open_(hs[root]["map"]), open_(hs[root]["mapflags"])
            except Exception as e:  # noqa: BLE001
                err = e
        ok = [None] * self.world
        dist.all_gather_object(ok, err is None, group=group)
        if not all(ok):
            self.close(group)
            raise RuntimeError(f"PeerBandReduce setup failed: {err or 'on another rank'}")

    def _s(self, stream):
        return (stream if stream is not None else self._torch.cuda.current_stream()).cuda_stream

    def _wait(self, flags: int, value: int, stream) -> None:
        self._check(self._A.lib().spct_cu_flag_wait(flags, self.world, self.FLAG_STRIDE, value, self.TIMEOUT_NS,
                                                    self.err, self._s(stream)))

    def _signal(self, ptrs, value: int, stream) -> None:
        arr = (self._C.c_void_p * len(ptrs))(*ptrs)
        self._check(self._A.lib().spct_cu_flag_signal_many(arr, len(ptrs), value, self._s(stream)))

    def begin(self, stream=None) -> None:
        self.epoch += 1
        if self.epoch > 2:  # every owner has pulled this parity's partial two epochs ago
            self._wait(self.acks, self.epoch - 2, stream)

    def slot(self) -> DeviceSlot:
        return DeviceSlot(self.part + 8 * self.plane * (self.epoch % 2), (self.nv, self.nu))

    def publish(self, stream=None) -> None:
        fs = 8 * self.FLAG_STRIDE
        self._signal([f + fs * self.rank for f in self.peer_flags], self.epoch, stream)

    def finalize(self, p: float = 1.0, metric: int = 0, stream=None) -> None:
        C, lib, s = self._C, self._A.lib(), self._s(stream)
        fs = 8 * self.FLAG_STRIDE
        self._wait(self.flags, self.epoch, stream)  # every writer's partial of this epoch
        off = 8 * self.plane * (self.epoch % 2)
        src = (C.c_void_p * self.world)(*[q + off for q in self.parts])
        self._check(lib.spct_cu_hist_finalize_band(src, self.world, self.W, self.H, self.kw, self.kh, p, metric,
                                                   self.v0, self.v1, self.root_map, s))
        self._signal([self.root_mapflags + fs * self.rank] + [a + fs * self.rank for a in self.peer_acks],
                     self.epoch, stream)
        if self.rank == self.root:
            self._wait(self.mapflags, self.epoch, stream)

    @property
    def map(self):
        """The final (H, W) float64 map on the root (a tensor view of the shared buffer)."""
        if self.rank != self.root:
            raise RuntimeError("PeerBandReduce.map lives on the root")
        return self._torch.as_tensor(_DevArray(self.map_ptr, (self.H, self.W), "<f8"), device=self.device)

    def error(self) -> bool:
        t = self._torch.as_tensor(_DevArray(self.err, (1,), "<u4"), device=self.device)
        self._torch.cuda.synchronize(self.device)
        return bool(int(t.item()))

    def close(self, group=None) -> None:
        import torch.distributed as dist

        self._torch.cuda.synchronize(self.device)
        lib = self._A.lib()
        for p in self._opened:
            lib.spct_cu_peer_close(p)
        self._opened = []
        dist.barrier(group=group)
        for p in self._own:
            lib.spct_cu_peer_free(p)
        self._own = []


class ShardedMapStep:
    """One frame of the bin-sharded likelihood-map path on this rank.

    ``bins_per_rank=None`` shards a fixed histogram of ``nbins`` bins over the ranks
    (strong scaling: rank r owns ``slab_bounds(nbins, world, r)``); an integer gives every
    rank that many bins of a ``bins_per_rank * world`` histogram (weak scaling).  With one
    rank the fused sweep writes the finished map itself; with several, each rank's sweep
    writes its slab of the tensor and its partial window sums, and ``reduce`` sums them:
    "band" (every rank pulls and finalises a band of rows over peer memory, default),
    "root" (partials written into the root's slots by the sweep) or "nccl" (one
    ``dist.reduce`` + ``hist_finalize`` on the root).  Peer setup that fails (no IPC / P2P
    between the devices) falls back to "nccl" on every rank.

        s = ShardedMapStep(W, H, nbins, tmpl, kw, kh, device=dev)
        s.step(frame)            # device frame (uint8), stream-ordered
        s.map                    # root: the (H, W) float64 likelihood map
    """

    def __init__(self, width: int, height: int, nbins: int, tmpl, kw: int, kh: int, p: float = 1.0, *,
                 bins_per_rank: int | None = None, reduce: str = "band", root: int = 0, device=None,
                 store_tensor: bool = True):
        import torch
        import torch.distributed as dist

        from . import api

        self._api, self._torch = api, torch
        init = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size() if init else 1
        self.rank = dist.get_rank() if init else 0
        self.root = root
        self.W, self.H, self.kw, self.kh, self.p = width, height, kw, kh, p
        self.nbins = nbins if bins_per_rank is None else bins_per_rank * self.world
        if self.world == 1:
            self.bin0, self.bin1 = 0, self.nbins
        elif bins_per_rank is None:
            self.bin0, self.bin1 = slab_bounds(self.nbins, self.world, self.rank)
        else:
            self.bin0, self.bin1 = self.rank * bins_per_rank, (self.rank + 1) * bins_per_rank
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.tmpl_dev = torch.as_tensor(np.asarray(tmpl, dtype=np.float64)).to(self.device) \
            if not isinstance(tmpl, torch.Tensor) else tmpl.to(self.device, torch.float64)
        self.tensor = api.IntegralHistogramTensor(width, height, self.nbins, self.bin0, self.bin1 - self.bin0,
                                                  device=self.device, store=store_tensor)
        self.nu, self.nv = width - kw + 1, height - kh + 1
        self.reduce, self.note = reduce, reduce
        self.peer = None
        self._map = None
        self.partial = None
        if self.world > 1 and reduce in ("band", "root"):
            try:  # fails on every rank or on none (the reducers agree on the outcome)
                self.peer = PeerBandReduce(width, height, kw, kh, root=root, device=self.device) \
                    if reduce == "band" else PeerSlabReduce(self.nu, self.nv, root=root, device=self.device)
            except RuntimeError as e:
                self.reduce, self.note = "nccl", "nccl (peer setup failed: %s)" % str(e)[:120]
        if self.world == 1 or self.peer is None or reduce == "root":
            if self.world == 1 or self.rank == root:
                self._map = torch.empty((height, width), dtype=torch.float64, device=self.device)
        elif self.rank == root:
            self._map = self.peer.map  # the band owners write the root's shared buffer
        if self.world > 1 and self.peer is None:
            self.partial = torch.empty((self.nv, self.nu), dtype=torch.float64, device=self.device)

    @property
    def map(self):
        if self.rank != self.root and self.world > 1:
            raise RuntimeError("ShardedMapStep.map lives on the root")
        return self._map

    def step(self, frame, stream=None) -> None:
        api, kw, kh, p = self._api, self.kw, self.kh, self.p
        if self.world == 1:
            api.build_and_match_map(frame, self.nbins, None, kw, kh, p, out=self.tensor, lmap=self._map,
                                    tmpl_dev=self.tmpl_dev, stream=stream)
            return
        b0, nb = self.bin0, self.bin1 - self.bin0
        if self.peer is not None:
            self.peer.begin(stream)
            api.build_and_match(frame, self.nbins, None, kw, kh, p, bin0=b0, bins=nb, out=self.tensor,
                                partial=self.peer.slot(), tmpl_dev=self.tmpl_dev, stream=stream)
            self.peer.publish(stream)
            if self.reduce == "band":
                self.peer.finalize(p, stream=stream)
            elif self.rank == self.root:
                self.peer.finalize(self._map, self.W, self.H, kw, kh, p, stream=stream)
            return
        api.build_and_match(frame, self.nbins, None, kw, kh, p, bin0=b0, bins=nb, out=self.tensor,
                            partial=self.partial, tmpl_dev=self.tmpl_dev, stream=stream)
        reduce_partials(self.partial, dst=self.root)
        if self.rank == self.root:
            api.hist_finalize(self.partial, self.W, self.H, kw, kh, p, out=self._map, stream=stream)

    def error(self) -> bool:
        return self.peer.error() if self.peer is not None else False

    def close(self) -> None:
        if self.peer is not None:
            self.peer.close()
            self.peer = None
