// Transport of the multi-rank slab partition.
//
// The data plane of a slab-partitioned solve needs three collectives: grouped
// point-to-point copies of contiguous ranges (halo exchange, its reverse
// reduction, gathers), and a sum all-reduce (Krylov inner products).  Two
// implementations (plus the CUDA-IPC peer-memory transport of ipc.cu):
//   * NcclTransport: one process per GPU, ncclSend/ncclRecv in a group and
//     ncclAllReduce over NVLink/NVSwitch (dist.cu);
//   * LoopTransport: W contexts of ONE process on one device, one host thread
//     per rank (rbf_loopback_group_create / rbf_create_loopback): ranges are
//     copied with cudaMemcpyAsync between the ranks' buffers and the sum is a
//     kernel over all ranks' buffers in rank order, ordered by CUDA events and a
//     host barrier.  It runs the exact multi-rank code path of the library on
//     a single GPU (tests; NCCL cannot place two ranks on one device).
// Every rank must issue the same sequence of collective calls; a call's send
// list to rank q must match q's receive list from this rank (same order, same
// counts).  All transfers are stream-ordered on the given stream.
#pragma once
#include <condition_variable>
#include <functional>
#include <mutex>
#include <vector>

#include "internal.h"

namespace rbf {

enum class DType { F32 = 4, F64 = 8 };

struct Xfer {
  int peer;
  void* ptr;        // send: source (read), recv: destination (written)
  int64_t count;    // elements
};

struct Transport {
  virtual ~Transport() = default;
  virtual rbf_status exchange(rbf_ctx* ctx, cudaStream_t s, const std::vector<Xfer>& sends,
                              const std::vector<Xfer>& recvs, DType t) = 0;
  virtual rbf_status allreduce_sum(rbf_ctx* ctx, cudaStream_t s, void* buf, int64_t count, DType t) = 0;
  // Peer-memory mode (transports whose ranks can address each other's device
  // memory: loopback and CUDA IPC).  peer_begin: every rank's device buffer of
  // `need` bytes (one per rank, symmetric role; grown collectively), `stage`
  // fills mine on stream s, then -- ordered by events and a host barrier -- the
  // peers' buffers are ready and addressable here: peers[q] points at rank q's
  // buffer (mine at [rank]).  Until peer_end the caller's kernels may read and
  // atomically update any rank's buffer; peer_end orders every rank after all
  // ranks' kernels (no buffer is reused before its readers and writers are done).
  virtual bool peer_capable() const { return false; }
  virtual rbf_status peer_begin(rbf_ctx*, cudaStream_t, uint64_t, const std::function<rbf_status(void*)>&,
                                std::vector<void*>*) {
    return RBF_EUNSUPPORTED;
  }
  virtual rbf_status peer_end(rbf_ctx*, cudaStream_t) { return RBF_EUNSUPPORTED; }
};

// Shared state of a loopback group (library-owned; rbf_loopback_group_*).
struct LoopGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  struct Slot {
    std::vector<Xfer> sends;
    const void* buf = nullptr;
    void* peer_buf = nullptr;   // peer-memory mode: this rank's buffer
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  std::vector<Slot> slots;
  std::vector<int> joined;   // ranks with a live context
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

Transport* make_nccl_transport(void* comm);
rbf_status allgather_shards(rbf_ctx* ctx, const void* local, const std::vector<int64_t>& id0s,
                            const std::vector<int64_t>& ns, int per, void* full, DType t);
// ipc.cu: CUDA-IPC peer-memory transport (one process per GPU, one node)
rbf_status make_ipc_transport(int device, const void* key16, int rank, int world, Transport** out);
Transport* make_loop_transport(LoopGroup* g, int rank);

}  // namespace rbf
