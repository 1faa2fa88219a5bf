// comm.cuh — the multi-rank transport of libmpr.so (not part of the ABI).
//
// The LE-MPR hot path exchanges data between ranks in exactly four ways:
//   * all-reduce (sum / min / max) of small scalars and of the exact int64 block sums;
//   * neighbour exchange of contiguous ranges (halo rows of a row slab, one per colour
//     half-sweep; the z / mask halo rows of the parameter stage);
//   * all-gather of variable-sized row ranges (the predictions of every slab);
//   * all-reduce (sum) or a rank-ordered chain of the fp64 per-gap accumulator.
// Comm is that interface. Two transports implement it:
//   * NcclComm: a caller-supplied ncclComm_t (libnccl.so.2 resolved at run time, so the
//     library loads without NCCL); every operation is enqueued on the given stream — no
//     host synchronisation, the collective is stream ordered like a kernel launch.
//   * GroupComm: W contexts of ONE process (one host thread each, on one or several
//     devices). Host threads meet at a barrier, then copy directly between the ranks' device
//     buffers (cudaMemcpyAsync, peer copies across devices). It is host-synchronous; it
//     exists so the multi-rank code path runs, bit for bit, where one process owns all the
//     devices (or the single GPU of a test box), with no kernel ever waiting on another.
// Both give identical results: the reductions are exact (integers) or order-defined (min,
// max); the fp64 accumulator sum is the only order-dependent one (rank order in GroupComm,
// NCCL's order otherwise) and the ordered chain removes even that.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "mpr.h"

namespace mpr {

enum CommType { CT_U8 = 0, CT_I32, CT_I64, CT_U64, CT_F32, CT_F64 };
enum CommOp { OP_SUM = 0, OP_MIN, OP_MAX };

size_t comm_type_size(CommType t);

// One side of a neighbour exchange: `count` elements at device address `ptr`, to / from
// rank `peer`. Sends and receives between the same pair of ranks are matched in order.
struct P2P {
  int peer;
  void* ptr;
  size_t count;
};

class Comm {
 public:
  virtual ~Comm() = default;
  int rank = 0, world = 1;
  std::string err;
  // Each call returns MPR_OK or an error status with a message in `err`.
  virtual mpr_status allreduce(void* buf, size_t count, CommType t, CommOp op, cudaStream_t st) = 0;
  virtual mpr_status exchange(const std::vector<P2P>& sends, const std::vector<P2P>& recvs, CommType t,
                              cudaStream_t st) = 0;
  // recv[displs[w] .. displs[w] + counts[w]) receives rank w's `send` (counts[rank] elements;
  // send may alias recv + displs[rank])
  virtual mpr_status allgatherv(const void* send, void* recv, const std::vector<size_t>& counts,
                                const std::vector<size_t>& displs, CommType t, cudaStream_t st) = 0;
  virtual mpr_status broadcast(void* buf, size_t count, CommType t, int root, cudaStream_t st) = 0;
  // true: operations are stream-ordered and may be captured into a CUDA graph
  virtual bool stream_ordered() const = 0;
  virtual const char* name() const = 0;
};

// ncclComm_t supplied by the caller (not owned). nullptr + why on failure.
Comm* make_nccl_comm(void* nccl_comm, int device, std::string& why);
// Rank `rank` of an in-process group.
Comm* make_group_comm(mpr_group* g, int rank, std::string& why);

// NCCL helpers behind mpr_nccl_* (the caller creates the communicator through libmpr, so
// both sides use the same libnccl.so.2).
mpr_status nccl_unique_id(void* id_out, std::string& why);
mpr_status nccl_comm_init(int world, int rank, const void* id, int device, void** comm_out, std::string& why);
mpr_status nccl_comm_destroy(void* comm);

}  // namespace mpr
