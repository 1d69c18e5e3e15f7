"""The NCCL data plane behind the C-ABI (comm.cu) on a 1-rank communicator.

One GPU cannot host a multi-rank NCCL communicator, so this pins the
binding, argument plumbing and byte accounting of every entry point with a
self-communicator (send/recv to self inside one group, 1-root broadcast
group, 1-rank reductions, gather to self).  The multi-rank protocol around
these calls is covered by tests/test_multiproc.py (gloo) and the in-process
virtual-rank tests.
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    import torch
    from paper_2506_09226_b200 import _lib
    L = _lib.load()
    uid = (C.c_char * L.scx_comm_id_bytes())()
    assert L.scx_comm_unique_id(uid) == 0
    h = C.c_void_p()
    torch.cuda.init()
    assert L.scx_comm_init_rank(C.byref(h), 1, uid, 0) == 0, L.scx_last_error()
    yield L, h
    assert L.scx_comm_destroy(h) == 0


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _i64(*xs):
    return (C.c_int64 * len(xs))(*xs)


def test_version(comm):
    L, _ = comm
    v = C.c_int()
    assert L.scx_nccl_version(C.byref(v)) == 0 and v.value >= 22800


def test_alltoallv_self(comm):
    import torch
    from paper_2506_09226_b200._lib import stream_ptr
    L, h = comm
    src = torch.arange(1000, dtype=torch.int32, device="cuda")
    dst = torch.full((600,), -1, dtype=torch.int32, device="cuda")
    # send elements [300, 900) to self, land them at offset 0
    rc = L.scx_alltoallv(h, _ptr(src), _i64(600), _i64(300), _ptr(dst), _i64(600), _i64(0), 4,
                         stream_ptr())
    assert rc == 0, L.scx_last_error()
    assert torch.equal(dst.cpu(), torch.arange(300, 900, dtype=torch.int32))


def test_bcast_group_allreduce_gather(comm):
    import torch
    from paper_2506_09226_b200._lib import stream_ptr
    L, h = comm
    buf = torch.arange(64, dtype=torch.int64, device="cuda")
    bufs = (C.c_void_p * 1)(buf.data_ptr())
    assert L.scx_bcast_group(h, bufs, _i64(64 * 8), 1, stream_ptr()) == 0
    assert torch.equal(buf.cpu(), torch.arange(64))
    assert L.scx_bcast_group(h, bufs, _i64(8), 2, stream_ptr()) != 0     # roots != ranks
    out = torch.zeros(64, dtype=torch.int64, device="cuda")
    for op in (0, 1, 2):
        assert L.scx_allreduce_i64(h, _ptr(buf), _ptr(out), 64, op, stream_ptr()) == 0
        assert torch.equal(out.cpu(), torch.arange(64))
    assert L.scx_allreduce_i64(h, _ptr(buf), _ptr(out), 64, 7, stream_ptr()) != 0
    g = torch.zeros(64, dtype=torch.int64, device="cuda")
    recv = (C.c_void_p * 1)(g.data_ptr())
    assert L.scx_gather_to0(h, _ptr(buf), 64 * 8, recv, _i64(64 * 8), stream_ptr()) == 0
    torch.cuda.synchronize()
    assert np.array_equal(g.cpu().numpy(), np.arange(64))
