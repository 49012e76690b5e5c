"""Bin-slab sharding of the likelihood-map path across ranks.

Each rank owns a contiguous slab of bins [k0, k1), builds that slab of the integral
histogram and the slab's partial window statistic (the per-bin terms summed over its
bins), and one reduce adds the partial maps on the destination rank, which then runs
the finalisation.  Everything here is plumbing on torch.distributed (NCCL on GPUs,
gloo in the CPU tests); the computation lives in the CUDA kernels.

The reference has no multi-device path; the decomposition is exact
because every plane depends only on [bin == k] and the window statistic is a sum
over bins (likelihood.cpp:215-219).
"""
from __future__ import annotations


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
