"""This process's NCCL communicator behind libscx's C-ABI (csrc/comm.cu).

One-process-per-GPU jobs move exchange data through these calls (shuffle
all-to-all-v, grouped per-root broadcasts, the final gather, metadata
all-gathers); torch.distributed only bootstraps the job (rendezvous and the
one-time broadcast of the NCCL unique id) and holds streams and memory.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .cluster import Endpoint


def _i64(xs) -> C.Array:
    xs = [int(x) for x in xs]
    return (C.c_int64 * max(1, len(xs)))(*xs)


class NcclComm:
    def __init__(self, ep: Endpoint):
        import torch.distributed as dist
        self.lib = L.load()
        self.n, self.rank = ep.n, ep.rank
        nb = int(self.lib.scx_comm_id_bytes())
        uid = (C.c_char * nb)()
        if ep.rank == 0:
            L.call("scx_comm_unique_id", uid)
        box = [bytes(uid) if ep.rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=ep.group)     # control plane, once
        uid = (C.c_char * nb).from_buffer_copy(box[0])
        self.h = C.c_void_p()
        L.call("scx_comm_init_rank", C.byref(self.h), ep.n, uid, ep.rank)

    def alltoallv(self, send, send_counts, send_offs, recv, recv_counts, recv_offs,
                  elem_bytes: int) -> None:
        L.call("scx_alltoallv", self.h, C.c_void_p(send.data_ptr()), _i64(send_counts),
               _i64(send_offs), C.c_void_p(recv.data_ptr()), _i64(recv_counts), _i64(recv_offs),
               elem_bytes, L.stream_ptr())

    def allgather(self, t):
        """Every rank's same-size 1-D tensor, stacked [n, len] (grouped sends
        of the one buffer to every peer)."""
        import torch
        k = t.numel()
        out = torch.empty(self.n * k, dtype=t.dtype, device=t.device)
        self.alltoallv(t, [k] * self.n, [0] * self.n, out, [k] * self.n,
                       [r * k for r in range(self.n)], t.element_size())
        return out.view(self.n, k)

    def bcast_group(self, bufs, nbytes) -> None:
        arr = (C.c_void_p * self.n)(*[b.data_ptr() if b is not None else 0 for b in bufs])
        L.call("scx_bcast_group", self.h, arr, _i64(nbytes), self.n, L.stream_ptr())

    def allreduce_i64(self, t, op: str = "sum"):
        out = t.clone()
        L.call("scx_allreduce_i64", self.h, C.c_void_p(t.data_ptr()), C.c_void_p(out.data_ptr()),
               t.numel(), {"sum": 0, "min": 1, "max": 2}[op], L.stream_ptr())
        return out

    def gather_to0(self, send, nbytes: int, recv_bufs=None, recv_bytes=None) -> None:
        if self.rank == 0:
            arr = (C.c_void_p * self.n)(*[b.data_ptr() if b is not None else 0 for b in recv_bufs])
            L.call("scx_gather_to0", self.h, C.c_void_p(send.data_ptr()), int(nbytes), arr,
                   _i64(recv_bytes), L.stream_ptr())
        else:
            L.call("scx_gather_to0", self.h, C.c_void_p(send.data_ptr()), int(nbytes), None, None,
                   L.stream_ptr())


def comm_of(ep: Endpoint) -> NcclComm | None:
    """The endpoint's NCCL communicator (created on first use) for NCCL jobs
    with N > 1; None otherwise (gloo / in-process / single rank)."""
    if ep.in_process or ep.n == 1 or ep.backend != "nccl":
        return None
    c = getattr(ep, "_nccl", None)
    if c is None:
        c = NcclComm(ep)
        ep._nccl = c
    return c


def allgather_bytes(ep: Endpoint, raw: np.ndarray) -> np.ndarray:
    """[n, nbytes] uint8 of every rank's equal-size byte string."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(raw).view(np.uint8).reshape(-1).copy()).to(ep.device)
    c = comm_of(ep)
    if c is not None:
        return c.allgather(t).cpu().numpy()
    import torch.distributed as dist
    out = torch.empty(ep.n * t.numel(), dtype=torch.uint8, device=t.device)
    dist.all_gather_into_tensor(out, t, group=ep.group)
    return out.view(ep.n, -1).cpu().numpy()
