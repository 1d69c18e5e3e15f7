// comm.cu -- the exchange layer's NCCL data plane behind the C-ABI
// (SURVEY.md §8b b2).  Replaces the reference's in-process transport for
// one-process-per-GPU jobs:
//   scx_alltoallv    <- shuffle_table's grouped send/recv (exchange.py:131-174,
//                       the paper's Alg. 1) and size_exchange (73-97)
//   scx_bcast_group  <- broadcast_table's N per-root broadcasts in ONE group
//                       (exchange.py:195-285, Alg. 2)
//   scx_allreduce_i64<- all_reduce on exact integer aggregates (collectives.py:199)
//   scx_gather_to0   <- the final gather to rank 0 (engine.py:345-365)
// Linked against the pip NCCL (2.28.9) by rpath (build.py).  Every call is
// asynchronous on the caller's stream; counts are host arrays; the library
// allocates nothing (NCCL's own communicator state aside).
#include <nccl.h>
#include <string.h>

#include "common.cuh"

namespace scx {

static int nccl_fail(ncclResult_t r, const char* what) {
  set_error("%s: %s", what, ncclGetErrorString(r));
  return SCX_ECUDA;
}

#define SCX_NCCL(call)                                  \
  do {                                                  \
    ncclResult_t _r = (call);                           \
    if (_r != ncclSuccess) return nccl_fail(_r, #call); \
  } while (0)

static ncclComm_t as_comm(void* c) { return static_cast<ncclComm_t>(c); }

static int comm_size(void* comm, int& n, int& rank) {
  SCX_NCCL(ncclCommCount(as_comm(comm), &n));
  SCX_NCCL(ncclCommUserRank(as_comm(comm), &rank));
  return SCX_OK;
}

}  // namespace scx

using namespace scx;

extern "C" int scx_nccl_version(int* version) {
  if (!version) return SCX_EINVAL;
  SCX_NCCL(ncclGetVersion(version));
  return SCX_OK;
}

extern "C" int64_t scx_comm_id_bytes(void) { return (int64_t)sizeof(ncclUniqueId); }

extern "C" int scx_comm_unique_id(void* id_out) {
  if (!id_out) return SCX_EINVAL;
  ncclUniqueId id;
  SCX_NCCL(ncclGetUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return SCX_OK;
}

extern "C" int scx_comm_init_rank(void** comm_out, int nranks, const void* id, int rank) {
  if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("scx_comm_init_rank: bad arguments (nranks=%d rank=%d)", nranks, rank);
    return SCX_EINVAL;
  }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  SCX_NCCL(ncclCommInitRank(&c, nranks, uid, rank));
  *comm_out = c;
  return SCX_OK;
}

extern "C" int scx_comm_init_all(int n, const int* devs, void** comms_out) {
  if (n < 1 || !comms_out) {
    set_error("scx_comm_init_all: bad arguments (n=%d)", n);
    return SCX_EINVAL;
  }
  SCX_NCCL(ncclCommInitAll(reinterpret_cast<ncclComm_t*>(comms_out), n, devs));
  return SCX_OK;
}

extern "C" int scx_comm_destroy(void* comm) {
  if (!comm) return SCX_OK;
  SCX_NCCL(ncclCommDestroy(as_comm(comm)));
  return SCX_OK;
}

// One grouped all-to-all-v: to peer d, send_counts[d] elements starting at
// element send_offs[d] of send_dev; from peer s, recv_counts[s] elements into
// recv_dev at element recv_offs[s].  Elements are elem_bytes wide (moved as
// bytes).  The self segment is a send/recv to self inside the same group.
extern "C" int scx_alltoallv(void* comm, const void* send_dev, const int64_t* send_counts,
                             const int64_t* send_offs, void* recv_dev,
                             const int64_t* recv_counts, const int64_t* recv_offs, int elem_bytes,
                             void* stream) {
  int n = 0, rank = 0;
  if (!comm || !send_counts || !send_offs || !recv_counts || !recv_offs || elem_bytes < 1) {
    set_error("scx_alltoallv: bad arguments");
    return SCX_EINVAL;
  }
  int rc = comm_size(comm, n, rank);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* s = static_cast<const char*>(send_dev);
  char* r = static_cast<char*>(recv_dev);
  SCX_NCCL(ncclGroupStart());
  for (int p = 0; p < n; ++p) {
    if (send_counts[p] > 0)
      SCX_NCCL(ncclSend(s + send_offs[p] * elem_bytes, (size_t)(send_counts[p] * elem_bytes),
                        ncclInt8, p, as_comm(comm), st));
    if (recv_counts[p] > 0)
      SCX_NCCL(ncclRecv(r + recv_offs[p] * elem_bytes, (size_t)(recv_counts[p] * elem_bytes),
                        ncclInt8, p, as_comm(comm), st));
  }
  SCX_NCCL(ncclGroupEnd());
  return SCX_OK;
}

// All N root broadcasts of one column in ONE NCCL group: bufs_dev[r] is root
// r's segment of the rank-ordered output (on the root it already holds the
// root's rows), bytes[r] its length.
extern "C" int scx_bcast_group(void* comm, void* const* bufs_dev, const int64_t* bytes,
                               int n_roots, void* stream) {
  int n = 0, rank = 0;
  if (!comm || !bufs_dev || !bytes) {
    set_error("scx_bcast_group: bad arguments");
    return SCX_EINVAL;
  }
  int rc = comm_size(comm, n, rank);
  if (rc) return rc;
  if (n_roots != n) {
    set_error("scx_bcast_group: %d roots for a %d-rank communicator", n_roots, n);
    return SCX_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SCX_NCCL(ncclGroupStart());
  for (int root = 0; root < n; ++root)
    if (bytes[root] > 0)
      SCX_NCCL(ncclBroadcast(bufs_dev[root], bufs_dev[root], (size_t)bytes[root], ncclInt8, root,
                             as_comm(comm), st));
  SCX_NCCL(ncclGroupEnd());
  return SCX_OK;
}

extern "C" int scx_allreduce_i64(void* comm, const int64_t* send_dev, int64_t* recv_dev,
                                 int64_t count, int op, void* stream) {
  if (!comm || count < 0 || op < 0 || op > 2) {
    set_error("scx_allreduce_i64: bad arguments (op=%d: 0 sum, 1 min, 2 max)", op);
    return SCX_EINVAL;
  }
  if (count == 0) return SCX_OK;
  const ncclRedOp_t ops[3] = {ncclSum, ncclMin, ncclMax};
  SCX_NCCL(ncclAllReduce(send_dev, recv_dev, (size_t)count, ncclInt64, ops[op], as_comm(comm),
                         static_cast<cudaStream_t>(stream)));
  return SCX_OK;
}

// Every rank's `bytes` bytes to rank 0; on rank 0, recv_dev[r] receives rank
// r's bytes (recv_bytes[r] long; rank 0's own slot is copied on the stream).
extern "C" int scx_gather_to0(void* comm, const void* send_dev, int64_t bytes,
                              void* const* recv_dev, const int64_t* recv_bytes, void* stream) {
  int n = 0, rank = 0;
  if (!comm || bytes < 0) {
    set_error("scx_gather_to0: bad arguments");
    return SCX_EINVAL;
  }
  int rc = comm_size(comm, n, rank);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rank != 0) {
    if (bytes > 0) SCX_NCCL(ncclSend(send_dev, (size_t)bytes, ncclInt8, 0, as_comm(comm), st));
    return SCX_OK;
  }
  if (!recv_dev || !recv_bytes) {
    set_error("scx_gather_to0: root needs recv buffers");
    return SCX_EINVAL;
  }
  if (recv_bytes[0] > 0)
    SCX_CUDA(cudaMemcpyAsync(recv_dev[0], send_dev, (size_t)recv_bytes[0],
                             cudaMemcpyDeviceToDevice, st));
  SCX_NCCL(ncclGroupStart());
  for (int r = 1; r < n; ++r)
    if (recv_bytes[r] > 0)
      SCX_NCCL(ncclRecv(recv_dev[r], (size_t)recv_bytes[r], ncclInt8, r, as_comm(comm), st));
  SCX_NCCL(ncclGroupEnd());
  return SCX_OK;
}
