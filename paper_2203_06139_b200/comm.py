"""Multi-GPU exchange for sharded chi2 plans (include/adc_cuda.h, adc_comm).

One process per GPU.  A communicator carries the one collective of the chi2
path — an all-gather of per-chunk records — either over NCCL inside the
library (stream-ordered, captured in the pass's CUDA graph) or over a host
callback (any all-gather over host memory, e.g. torch.distributed/gloo).

    uid = Comm.unique_id()            # rank 0; distribute the 128 bytes
    comm = Comm.nccl(world, rank, uid)
    plan = Chi2Plan.sharded("gpoly", 6, bins, lo, hi, events, my_counts, comm)
    FitEngine("gpoly", 6, comm=comm).fit(h, init)   # same steps on every rank
"""
from __future__ import annotations

import ctypes

import numpy as np

from ._capi import ALLGATHER_FN, COMM_HOST, COMM_NCCL, COMM_PEER, check, lib


class Comm:
    """Owns one adc_comm*.  Keep it alive while plans use it."""

    def __init__(self, ptr: ctypes.c_void_p, world: int, rank: int, kind: int, keep=None):
        self._p, self.world, self.rank, self.kind = ptr, world, rank, kind
        self._keep = keep  # the ctypes callback of a host communicator

    @staticmethod
    def unique_id() -> bytes:
        import torch  # noqa: F401  (binds the process's own libnccl.so.2 first)
        buf = ctypes.create_string_buffer(128)
        check(lib.adc_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, world: int, rank: int, uid: bytes) -> "Comm":
        """Collective over the world; call on the device the plan runs on."""
        if len(uid) != 128:
            raise ValueError("NCCL unique id is 128 bytes")
        import torch  # noqa: F401  (binds the process's own libnccl.so.2 first)
        p = ctypes.c_void_p()
        check(lib.adc_cuda_comm_init_nccl(ctypes.byref(p), uid, world, rank))
        return cls(p, world, rank, COMM_NCCL)

    @staticmethod
    def _callback(world, allgather):
        def _cb(_ctx, send, recv, nbytes):
            try:
                n = nbytes // 8
                mine = np.ctypeslib.as_array((ctypes.c_double * n).from_address(send)).copy()
                out = np.ascontiguousarray(allgather(mine), dtype=np.float64)
                if out.size != world * n:
                    return 2
                ctypes.memmove(recv, out.ctypes.data, out.nbytes)
                return 0
            except Exception:  # noqa: BLE001 — reported to the C side as a status
                return 1

        return ALLGATHER_FN(_cb)

    @classmethod
    def host(cls, world: int, rank: int, allgather) -> "Comm":
        """allgather(send: float64 ndarray[n]) -> float64 ndarray[world * n], rank-major."""
        cb = cls._callback(world, allgather)
        p = ctypes.c_void_p()
        check(lib.adc_comm_init_host(ctypes.byref(p), world, rank, cb, None))
        return cls(p, world, rank, COMM_HOST, keep=cb)

    @classmethod
    def peer(cls, world: int, rank: int, allgather) -> "Comm":
        """Peer-memory transport: `allgather` (as for host()) only bootstraps the
        CUDA IPC handles when a plan attaches; every pass then exchanges its
        records GPU to GPU (NVLink stores + system-scope flags), no NCCL."""
        import torch  # noqa: F401
        cb = cls._callback(world, allgather)
        p = ctypes.c_void_p()
        check(lib.adc_cuda_comm_init_peer(ctypes.byref(p), world, rank, cb, None))
        return cls(p, world, rank, COMM_PEER, keep=cb)

    @classmethod
    def from_torch(cls, transport: str = "nccl") -> "Comm":
        """Builds a communicator over the initialised torch.distributed group:
        transport "nccl" = the library's own NCCL communicator (unique id
        broadcast over the group), "peer" = GPU-to-GPU stores into IPC-shared
        buffers (the group only bootstraps the handles), "host" = an all-gather
        of host buffers through the process group."""
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(), dist.get_rank()
        if transport == "nccl":
            obj = [cls.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            return cls.nccl(world, rank, obj[0])

        def allgather(mine):
            objs = [None] * world
            dist.all_gather_object(objs, mine)  # works over gloo and NCCL groups
            return np.concatenate(objs)

        if transport == "peer":
            return cls.peer(world, rank, allgather)
        return cls.host(world, rank, allgather)

    def info(self):
        w, r, k = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        check(lib.adc_comm_info(self._p, ctypes.byref(w), ctypes.byref(r), ctypes.byref(k)))
        return w.value, r.value, k.value

    def close(self):
        if self._p:
            lib.adc_comm_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
