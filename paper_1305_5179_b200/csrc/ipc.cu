// Peer-memory transport of the slab partition (transport.h): one process per
// GPU on one node, the ranks' exchange arenas mapped into each other through
// CUDA IPC (NVLink / NVSwitch peer access on a multi-GPU node; the same device
// when several test processes share one GPU), ordering by interprocess CUDA
// events, and a host barrier in a POSIX shared-memory segment.  No kernel ever
// waits on another rank: every cross-rank dependency is a stream wait on an
// event recorded before a host barrier (B200_PROFILING.md: ranks must not spin
// on each other's flags).
//
// A collective (exchange or all-reduce) of rank r:
//   1. r copies its send ranges into its own arena (each distinct range once)
//      and records its `ready` event; it publishes (peer, offset, count) per send
//      in its shared-memory slot;
//   2. host barrier;
//   3. r waits on each sender's `ready` and copies its receives out of the
//      senders' arenas (cudaMemcpyAsync between device pointers: the copy engines
//      over NVLink), or sums every rank's arena with one kernel (all-reduce);
//      records `done`;
//   4. host barrier; r waits on every peer's `done` before its next collective
//      may overwrite its arena.
// Arena growth (a rank needs more bytes than its arena holds) is agreed after
// the first barrier: the peers unmap the growing arenas, the owners reallocate
// and republish, the peers map the new ones (two extra barriers, rare).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <new>
#include <string>
#include <thread>

#include "internal.h"
#include "transport.h"

namespace rbf {
namespace {

constexpr int kIpcMaxWorld = 64;
constexpr int kIpcMaxSends = 256;
constexpr double kIpcTimeoutS = 600.0;

struct IpcSend {
  int peer;
  int64_t off;     // bytes into the sender's arena
  int64_t count;   // elements
};

struct IpcSlot {
  cudaIpcMemHandle_t arena;
  cudaIpcEventHandle_t ready, done;
  uint64_t arena_bytes;
  uint64_t arena_gen;
  uint64_t need;
  int nsend;
  IpcSend sends[kIpcMaxSends];
};

struct IpcShm {
  std::atomic<int> initialised;
  std::atomic<int> count;
  std::atomic<uint64_t> gen;
  std::atomic<int> failed;
  int world;
  IpcSlot slots[kIpcMaxWorld];
};

template <class T>
__global__ void ipc_sum_kernel(const T* const* __restrict__ bufs, int world, T* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T s = bufs[0][i];
    for (int q = 1; q < world; ++q) s += bufs[q][i];
    out[i] = s;
  }
}

struct IpcTransport final : Transport {
  IpcShm* shm = nullptr;
  size_t shm_bytes = 0;
  int rank = 0, world = 1;
  void* arena = nullptr;           // my arena (cudaMalloc, exported)
  uint64_t arena_bytes = 0;
  std::vector<void*> peer_arena;   // mapped arenas of the peers (mine at [rank])
  std::vector<uint64_t> peer_gen;
  cudaEvent_t ready = nullptr, done = nullptr;
  std::vector<cudaEvent_t> peer_ready, peer_done;
  DevBuf ptrs, scratch;            // device array of arena pointers (all-reduce), sum scratch

  rbf_status barrier() {
    const uint64_t g = shm->gen.load(std::memory_order_acquire);
    if (shm->count.fetch_add(1, std::memory_order_acq_rel) + 1 == world) {
      shm->count.store(0, std::memory_order_relaxed);
      shm->gen.fetch_add(1, std::memory_order_acq_rel);
      return RBF_OK;
    }
    const auto t0 = std::chrono::steady_clock::now();
    int spins = 0;
    while (shm->gen.load(std::memory_order_acquire) == g) {
      if (shm->failed.load()) { set_error("ipc transport: a peer failed"); return RBF_ECUDA; }
      if (++spins > 64) {
        std::this_thread::sleep_for(std::chrono::microseconds(spins > 4096 ? 50 : 1));
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > kIpcTimeoutS) {
          shm->failed.store(1);
          set_error("ipc transport: barrier timed out (a rank did not reach the same collective)");
          return RBF_ECUDA;
        }
      }
    }
    return RBF_OK;
  }

  rbf_status export_arena(uint64_t bytes) {
    if (arena) cudaFree(arena);
    arena = nullptr;
    RBF_CUDA_TRY(cudaMalloc(&arena, bytes));
    arena_bytes = bytes;
    IpcSlot& me = shm->slots[rank];
    RBF_CUDA_TRY(cudaIpcGetMemHandle(&me.arena, arena));
    me.arena_bytes = bytes;
    me.arena_gen += 1;
    return RBF_OK;
  }
  rbf_status map_peer(int q) {
    if (q == rank) { peer_arena[q] = arena; peer_gen[q] = shm->slots[q].arena_gen; return RBF_OK; }
    if (peer_arena[q]) cudaIpcCloseMemHandle(peer_arena[q]);
    peer_arena[q] = nullptr;
    RBF_CUDA_TRY(cudaIpcOpenMemHandle(&peer_arena[q], shm->slots[q].arena, cudaIpcMemLazyEnablePeerAccess));
    peer_gen[q] = shm->slots[q].arena_gen;
    return RBF_OK;
  }

  rbf_status init(int device, const std::string& name, int r, int w) {
    rank = r;
    world = w;
    shm_bytes = sizeof(IpcShm);
    int fd = -1;
    if (r == 0) {
      fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0) { set_error("ipc transport: shm_open(create) failed"); return RBF_EINVAL; }
      if (ftruncate(fd, (off_t)shm_bytes) != 0) { close(fd); set_error("ipc transport: ftruncate failed"); return RBF_EINVAL; }
    } else {
      const auto t0 = std::chrono::steady_clock::now();
      while ((fd = shm_open(name.c_str(), O_RDWR, 0600)) < 0) {
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > 120.0) {
          set_error("ipc transport: rank 0's shared-memory segment did not appear");
          return RBF_EINVAL;
        }
      }
      struct stat st;
      for (;;) {   // rank 0 may not have sized it yet
        if (fstat(fd, &st) == 0 && (size_t)st.st_size >= shm_bytes) break;
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
    }
    void* p = mmap(nullptr, shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) { set_error("ipc transport: mmap failed"); return RBF_EINVAL; }
    shm = static_cast<IpcShm*>(p);
    if (r == 0) {
      std::memset(static_cast<void*>(shm->slots), 0, sizeof(shm->slots));
      shm->world = w;
      shm->count.store(0);
      shm->gen.store(0);
      shm->failed.store(0);
      shm->initialised.store(1, std::memory_order_release);
    } else {
      while (!shm->initialised.load(std::memory_order_acquire)) std::this_thread::sleep_for(std::chrono::milliseconds(1));
      if (shm->world != w) { set_error("ipc transport: world size mismatch"); return RBF_EINVAL; }
    }
    RBF_CUDA_TRY(cudaSetDevice(device));
    RBF_CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming | cudaEventInterprocess));
    RBF_CUDA_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming | cudaEventInterprocess));
    IpcSlot& me = shm->slots[rank];
    RBF_CUDA_TRY(cudaIpcGetEventHandle(&me.ready, ready));
    RBF_CUDA_TRY(cudaIpcGetEventHandle(&me.done, done));
    RBF_TRY(export_arena((uint64_t)64 << 20));
    peer_arena.assign(w, nullptr);
    peer_gen.assign(w, 0);
    peer_ready.assign(w, nullptr);
    peer_done.assign(w, nullptr);
    RBF_TRY(barrier());   // every slot published
    for (int q = 0; q < w; ++q) {
      if (q == rank) { peer_ready[q] = ready; peer_done[q] = done; continue; }
      RBF_CUDA_TRY(cudaIpcOpenEventHandle(&peer_ready[q], shm->slots[q].ready));
      RBF_CUDA_TRY(cudaIpcOpenEventHandle(&peer_done[q], shm->slots[q].done));
    }
    for (int q = 0; q < w; ++q) RBF_TRY(map_peer(q));
    RBF_TRY(barrier());   // every rank attached: the name can go
    if (r == 0) shm_unlink(name.c_str());
    return RBF_OK;
  }

  // No barrier here: every collective ended with this rank's stream waiting on
  // every peer's `done` (recorded after the peer's reads of this arena), and
  // rbf_destroy synchronises the stream before deleting the transport, so no
  // peer reads this arena any more when it is freed.
  ~IpcTransport() override {
    for (int q = 0; q < (int)peer_arena.size(); ++q)
      if (q != rank && peer_arena[q]) cudaIpcCloseMemHandle(peer_arena[q]);
    for (int q = 0; q < (int)peer_ready.size(); ++q) {
      if (q == rank) continue;
      if (peer_ready[q]) cudaEventDestroy(peer_ready[q]);
      if (peer_done[q]) cudaEventDestroy(peer_done[q]);
    }
    if (ready) cudaEventDestroy(ready);
    if (done) cudaEventDestroy(done);
    if (arena) cudaFree(arena);
    if (shm) munmap(shm, shm_bytes);
  }

  // Steps 1-2 plus the growth protocol: the bytes of `need` staged by `stage`
  // into my arena, `ready` recorded, the barrier passed, peers' arenas mapped.
  template <class Stage>
  rbf_status publish(cudaStream_t s, uint64_t need, Stage&& stage) {
    IpcSlot& me = shm->slots[rank];
    me.need = need;
    const bool grow_me = need > arena_bytes;
    if (!grow_me) {
      RBF_TRY(stage());
      RBF_CUDA_TRY(cudaEventRecord(ready, s));
    }
    RBF_TRY(barrier());
    bool any = false;
    for (int q = 0; q < world; ++q) any = any || shm->slots[q].need > shm->slots[q].arena_bytes;
    if (!any) return RBF_OK;
    // growth: peers unmap the growing arenas, owners reallocate, peers remap
    for (int q = 0; q < world; ++q)
      if (q != rank && shm->slots[q].need > shm->slots[q].arena_bytes && peer_arena[q]) {
        cudaIpcCloseMemHandle(peer_arena[q]);
        peer_arena[q] = nullptr;
      }
    RBF_TRY(barrier());
    if (grow_me) {
      RBF_CUDA_TRY(cudaStreamSynchronize(s));   // my stream waited for the peers' last reads
      RBF_TRY(export_arena(std::max<uint64_t>(need, 2 * arena_bytes)));
    }
    RBF_TRY(barrier());
    for (int q = 0; q < world; ++q)
      if (peer_gen[q] != shm->slots[q].arena_gen) RBF_TRY(map_peer(q));
    if (grow_me) {
      RBF_TRY(stage());
      RBF_CUDA_TRY(cudaEventRecord(ready, s));
    }
    return barrier();
  }

  rbf_status finish(cudaStream_t s) {
    RBF_CUDA_TRY(cudaEventRecord(done, s));
    RBF_TRY(barrier());
    for (int q = 0; q < world; ++q)
      if (q != rank) RBF_CUDA_TRY(cudaStreamWaitEvent(s, peer_done[q], 0));
    return RBF_OK;
  }

  rbf_status exchange(rbf_ctx*, cudaStream_t s, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                      DType t) override {
    const size_t es = (size_t)t;
    if ((int)sends.size() > kIpcMaxSends) { set_error("ipc transport: too many sends"); return RBF_EINVAL; }
    // arena layout: each distinct (ptr, count) range once, 256-byte aligned
    IpcSlot& me = shm->slots[rank];
    std::vector<std::pair<const void*, int64_t>> uniq;
    std::vector<int64_t> uoff;
    uint64_t need = 0;
    me.nsend = (int)sends.size();
    for (size_t k = 0; k < sends.size(); ++k) {
      const Xfer& x = sends[k];
      int64_t off = -1;
      for (size_t u = 0; u < uniq.size(); ++u)
        if (uniq[u].first == x.ptr && uniq[u].second == x.count) { off = uoff[u]; break; }
      if (off < 0) {
        off = (int64_t)need;
        uniq.push_back({x.ptr, x.count});
        uoff.push_back(off);
        need += ((uint64_t)x.count * es + 255) & ~(uint64_t)255;
      }
      me.sends[k] = IpcSend{x.peer, off, x.count};
    }
    auto stage = [&]() -> rbf_status {
      for (size_t u = 0; u < uniq.size(); ++u)
        if (uniq[u].second > 0)
          RBF_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(arena) + uoff[u], uniq[u].first, es * uniq[u].second,
                                       cudaMemcpyDeviceToDevice, s));
      return RBF_OK;
    };
    RBF_TRY(publish(s, need, stage));
    for (size_t k = 0; k < recvs.size(); ++k) {
      const Xfer& rv = recvs[k];
      int nth = 0;   // the nth receive from this peer matches its nth send to me
      for (size_t k2 = 0; k2 < k; ++k2) nth += recvs[k2].peer == rv.peer;
      const IpcSlot& ps = shm->slots[rv.peer];
      const IpcSend* src = nullptr;
      for (int k2 = 0; k2 < ps.nsend; ++k2)
        if (ps.sends[k2].peer == rank && nth-- == 0) { src = &ps.sends[k2]; break; }
      if (!src || src->count != rv.count) { set_error("ipc exchange: unmatched transfer"); return RBF_EINVAL; }
      RBF_CUDA_TRY(cudaStreamWaitEvent(s, peer_ready[rv.peer], 0));
      if (rv.count > 0)
        RBF_CUDA_TRY(cudaMemcpyAsync(rv.ptr, static_cast<const char*>(peer_arena[rv.peer]) + src->off,
                                     es * rv.count, cudaMemcpyDeviceToDevice, s));
    }
    return finish(s);
  }

  bool peer_capable() const override { return true; }
  rbf_status peer_begin(rbf_ctx*, cudaStream_t s, uint64_t need, const std::function<rbf_status(void*)>& stage,
                        std::vector<void*>* peers) override {
    shm->slots[rank].nsend = 0;
    RBF_TRY(publish(s, need, [&]() { return stage(arena); }));
    peers->assign(peer_arena.begin(), peer_arena.end());
    for (int q = 0; q < world; ++q)
      if (q != rank) RBF_CUDA_TRY(cudaStreamWaitEvent(s, peer_ready[q], 0));
    return RBF_OK;
  }
  rbf_status peer_end(rbf_ctx*, cudaStream_t s) override { return finish(s); }

  rbf_status allreduce_sum(rbf_ctx*, cudaStream_t s, void* buf, int64_t count, DType t) override {
    const size_t es = (size_t)t;
    shm->slots[rank].nsend = 0;
    auto stage = [&]() -> rbf_status {
      if (count > 0) RBF_CUDA_TRY(cudaMemcpyAsync(arena, buf, es * count, cudaMemcpyDeviceToDevice, s));
      return RBF_OK;
    };
    RBF_TRY(publish(s, (uint64_t)count * es, stage));
    RBF_TRY(ptrs.ensure(sizeof(void*) * world, s));
    RBF_TRY(scratch.ensure(es * std::max<int64_t>(count, 1), s));
    // the arena pointers change only on growth; copied with the stream (host array
    // kept alive in the transport until the next call)
    host_ptrs.assign(peer_arena.begin(), peer_arena.end());
    RBF_CUDA_TRY(cudaMemcpyAsync(ptrs.p, host_ptrs.data(), sizeof(void*) * world, cudaMemcpyHostToDevice, s));
    for (int q = 0; q < world; ++q)
      if (q != rank) RBF_CUDA_TRY(cudaStreamWaitEvent(s, peer_ready[q], 0));
    if (count > 0) {
      if (t == DType::F64)
        ipc_sum_kernel<double><<<grid_for(count, 256), 256, 0, s>>>(ptrs.as<const double*>(), world,
                                                                    scratch.as<double>(), count);
      else
        ipc_sum_kernel<float><<<grid_for(count, 256), 256, 0, s>>>(ptrs.as<const float*>(), world,
                                                                   scratch.as<float>(), count);
      RBF_CHECK_LAUNCH();
    }
    RBF_TRY(finish(s));
    if (count > 0) RBF_CUDA_TRY(cudaMemcpyAsync(buf, scratch.p, es * count, cudaMemcpyDeviceToDevice, s));
    return RBF_OK;
  }
  std::vector<void*> host_ptrs;
};

}  // namespace

rbf_status make_ipc_transport(int device, const void* key16, int rank, int world, Transport** out) {
  *out = nullptr;
  if (world > kIpcMaxWorld) { set_error("ipc transport: world too large"); return RBF_EINVAL; }
  char hex[33];
  const unsigned char* k = static_cast<const unsigned char*>(key16);
  for (int i = 0; i < 16; ++i) snprintf(hex + 2 * i, 3, "%02x", k[i]);
  IpcTransport* t = new (std::nothrow) IpcTransport();
  if (!t) { set_error("host allocation failed"); return RBF_ENOMEM; }
  rbf_status st = t->init(device, std::string("/rbf_ipc_") + hex, rank, world);
  if (st != RBF_OK) {
    if (t->shm) t->shm->failed.store(1);
    delete t;
    return st;
  }
  *out = t;
  return RBF_OK;
}

}  // namespace rbf
