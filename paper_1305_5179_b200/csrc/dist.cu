// multi-rank partition of the hot path by spatial slabs.
//
// One rank per GPU (one process per GPU over NCCL, or -- tests, single-GPU
// runs of the same code path -- one host thread per rank over the in-process
// loopback transport, transport.h); every rank receives the full (replicated) centre set and
// builds the same global cell structure, then owns a slab of whole cell planes
// along z (the slowest axis of the cell key, so a slab is a CONTIGUOUS range of
// the sorted order).  Slab boundaries balance an estimate of the useful pairs
// per plane, sum over the plane's cells of n_c^2 (pairs per centre grow with
// the local density; c3's density varies 10x).  Per fp32/fp64 matvec the rank
// needs the weights of the sources within the cutoff of its targets: the planes
// [p0 - reach, p1 + reach) -- a contiguous window of the sorted order -- which
// it assembles from its own slice plus grouped point-to-point copies from the
// ranks owning the rest of the window (the paper's "communication ... limited
// to a constant number of elements in the vicinity").  The symmetric
// operators (reading R19) read only the window above the slab and send the
// contributions they accumulate for those sources back to their owners (a
// reverse halo reduction), so every pair is evaluated once across ranks too.
// Krylov inner products are local partial sums + a sum all-reduce; results are
// gathered so every rank returns the full vectors (replicated in, replicated
// out).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: inside a torch process
// this resolves to the NCCL torch already loaded), so librbf.so carries no link
// dependency and single-GPU use never touches it.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>

#include "internal.h"
#include "transport.h"

namespace rbf {
namespace {

// ---- minimal NCCL ABI (types of nccl.h, functions resolved with dlsym) -----
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclChar = 0, kNcclFloat32 = 7, kNcclFloat64 = 8 };
enum { kNcclSum = 0 };

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    bool good = true;
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
      if (!fp) good = false;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = good;
    if (!good) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

#define RBF_NCCL_TRY(expr)                                                              \
  do {                                                                                  \
    ncclResult_t _r = (expr);                                                           \
    if (_r != 0) {                                                                      \
      ::rbf::set_error(std::string(#expr) + ": " + nccl().GetErrorString(_r));          \
      return RBF_ENCCL;                                                                 \
    }                                                                                   \
  } while (0)

// per-plane pair weight sum_c n_c^2 and the first sorted position of every plane
__global__ void plane_stats_kernel(const int32_t* __restrict__ cell_start, int64_t ncell, int64_t plane_cells,
                                   unsigned long long* __restrict__ weight) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ncell; k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long m = (unsigned long long)(cell_start[k + 1] - cell_start[k]);
    if (m) atomicAdd(weight + k / plane_cells, m * m);
  }
}
__global__ void plane_start_kernel(const int32_t* __restrict__ cell_start, int dimz, int64_t plane_cells,
                                   int64_t* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p <= dimz; p += gridDim.x * blockDim.x)
    out[p] = cell_start[(int64_t)p * plane_cells];
}


// ---------------------------------------------------------------- NCCL -----
struct NcclTransport final : Transport {
  ncclComm_t comm;
  explicit NcclTransport(ncclComm_t c) : comm(c) {}
  ~NcclTransport() override {
    if (comm && nccl().ok) nccl().CommDestroy(comm);
  }
  rbf_status exchange(rbf_ctx*, cudaStream_t s, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                      DType t) override {
    if (sends.empty() && recvs.empty()) return RBF_OK;
    NcclApi& api = nccl();
    const int dt = t == DType::F64 ? kNcclFloat64 : kNcclFloat32;
    RBF_NCCL_TRY(api.GroupStart());
    for (const Xfer& x : sends) RBF_NCCL_TRY(api.Send(x.ptr, (size_t)x.count, dt, x.peer, comm, s));
    for (const Xfer& x : recvs) RBF_NCCL_TRY(api.Recv(x.ptr, (size_t)x.count, dt, x.peer, comm, s));
    RBF_NCCL_TRY(api.GroupEnd());
    return RBF_OK;
  }
  rbf_status allreduce_sum(rbf_ctx*, cudaStream_t s, void* buf, int64_t count, DType t) override {
  RBF_NVTX("allreduce_sum");
    if (count == 0) return RBF_OK;
    RBF_NCCL_TRY(nccl().AllReduce(buf, buf, (size_t)count, t == DType::F64 ? kNcclFloat64 : kNcclFloat32,
                                  kNcclSum, comm, s));
    return RBF_OK;
  }
};

// ------------------------------------------------------------ loopback -----
constexpr int kLoopMaxWorld = 64;
struct PtrArray {
  const void* p[kLoopMaxWorld];
};

// out[i] = sum over ranks q = 0..world-1 (in that order) of buf_q[i]
template <class T>
__global__ void loop_sum_kernel(PtrArray bufs, int world, T* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T s = static_cast<const T*>(bufs.p[0])[i];
    for (int q = 1; q < world; ++q) s += static_cast<const T*>(bufs.p[q])[i];
    out[i] = s;
  }
}

struct LoopTransport final : Transport {
  LoopGroup* g;
  int rank;
  DevBuf scratch;
  DevBuf pbuf;   // peer-memory mode buffer
  bool peer_capable() const override { return true; }
  rbf_status peer_begin(rbf_ctx*, cudaStream_t s, uint64_t need, const std::function<rbf_status(void*)>& stage,
                        std::vector<void*>* peers) override {
    LoopGroup::Slot& me = g->slots[rank];
    // every rank's buffer stays alive (and is not regrown) until peer_end
    RBF_TRY(pbuf.ensure(std::max<uint64_t>(need, 16), s));
    RBF_TRY(stage(pbuf.p));
    me.peer_buf = pbuf.p;
    RBF_CUDA_TRY(cudaEventRecord(me.ready, s));
    g->barrier();
    peers->assign(g->world, nullptr);
    for (int q = 0; q < g->world; ++q) {
      (*peers)[q] = g->slots[q].peer_buf;
      if (q != rank) RBF_CUDA_TRY(cudaStreamWaitEvent(s, g->slots[q].ready, 0));
    }
    return RBF_OK;
  }
  rbf_status peer_end(rbf_ctx*, cudaStream_t s) override {
    RBF_CUDA_TRY(cudaEventRecord(g->slots[rank].done, s));
    g->barrier();
    for (int q = 0; q < g->world; ++q)
      if (q != rank) RBF_CUDA_TRY(cudaStreamWaitEvent(s, g->slots[q].done, 0));
    return RBF_OK;
  }
  // the slot's events belong to the group (a peer may still be waiting on them
  // after this rank has returned from its last collective and been destroyed)
  LoopTransport(LoopGroup* grp, int r) : g(grp), rank(r) {
    std::lock_guard<std::mutex> lk(g->mu);
    if (!g->slots[r].ready) cudaEventCreateWithFlags(&g->slots[r].ready, cudaEventDisableTiming);
    if (!g->slots[r].done) cudaEventCreateWithFlags(&g->slots[r].done, cudaEventDisableTiming);
  }
  // phase 1: my buffers are complete on my stream when `ready` fires; phase 2:
  // the peers read them; phase 3: my later writes wait for their reads (`done`)
  rbf_status exchange(rbf_ctx*, cudaStream_t s, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                      DType t) override {
    LoopGroup::Slot& me = g->slots[rank];
    me.sends = sends;
    RBF_CUDA_TRY(cudaEventRecord(me.ready, s));
    g->barrier();
    const size_t es = (size_t)t;
    for (const Xfer& rv : recvs) {
      const LoopGroup::Slot& peer = g->slots[rv.peer];
      const Xfer* src = nullptr;
      int k = 0;   // the k-th receive from this peer matches its k-th send to me
      for (const Xfer& r2 : recvs) {
        if (&r2 == &rv) break;
        if (r2.peer == rv.peer) ++k;
      }
      for (const Xfer& sx : peer.sends)
        if (sx.peer == rank && k-- == 0) { src = &sx; break; }
      if (!src || src->count != rv.count) {
        set_error("loopback exchange: unmatched transfer");
        return RBF_EINVAL;
      }
      RBF_CUDA_TRY(cudaStreamWaitEvent(s, peer.ready, 0));
      if (rv.count > 0) RBF_CUDA_TRY(cudaMemcpyAsync(rv.ptr, src->ptr, es * rv.count, cudaMemcpyDeviceToDevice, s));
    }
    RBF_CUDA_TRY(cudaEventRecord(me.done, s));
    g->barrier();
    for (int q = 0; q < g->world; ++q)
      if (q != rank) RBF_CUDA_TRY(cudaStreamWaitEvent(s, g->slots[q].done, 0));
    return RBF_OK;
  }
  rbf_status allreduce_sum(rbf_ctx*, cudaStream_t s, void* buf, int64_t count, DType t) override {
    LoopGroup::Slot& me = g->slots[rank];
    const size_t es = (size_t)t;
    RBF_TRY(scratch.ensure(es * std::max<int64_t>(count, 1), s));
    me.buf = buf;
    RBF_CUDA_TRY(cudaEventRecord(me.ready, s));
    g->barrier();
    PtrArray pa{};
    for (int q = 0; q < g->world; ++q) {
      pa.p[q] = g->slots[q].buf;
      if (q != rank) RBF_CUDA_TRY(cudaStreamWaitEvent(s, g->slots[q].ready, 0));
    }
    if (count > 0) {
      if (t == DType::F64)
        loop_sum_kernel<double><<<grid_for(count, 256), 256, 0, s>>>(pa, g->world, scratch.as<double>(), count);
      else
        loop_sum_kernel<float><<<grid_for(count, 256), 256, 0, s>>>(pa, g->world, scratch.as<float>(), count);
      RBF_CHECK_LAUNCH();
    }
    RBF_CUDA_TRY(cudaEventRecord(me.done, s));
    g->barrier();
    for (int q = 0; q < g->world; ++q)
      if (q != rank) RBF_CUDA_TRY(cudaStreamWaitEvent(s, g->slots[q].done, 0));
    if (count > 0) RBF_CUDA_TRY(cudaMemcpyAsync(buf, scratch.p, es * count, cudaMemcpyDeviceToDevice, s));
    return RBF_OK;
  }
};


}  // namespace

Transport* make_nccl_transport(void* comm) { return new NcclTransport(static_cast<ncclComm_t>(comm)); }
Transport* make_loop_transport(LoopGroup* g, int rank) { return new LoopTransport(g, rank); }

rbf_status dist_init(rbf_ctx* ctx, const void* unique_id, int rank, int world) {
  NcclApi& api = nccl();
  if (!api.ok) { set_error(api.err); return RBF_ENCCL; }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  RBF_NCCL_TRY(api.CommInitRank(&comm, world, id, rank));
  ctx->nccl_comm = comm;
  ctx->tr = make_nccl_transport(comm);
  ctx->rank = rank;
  ctx->world = world;
  return RBF_OK;
}

void dist_destroy(rbf_ctx* ctx) {
  delete ctx->tr;   // NcclTransport destroys its communicator
  ctx->tr = nullptr;
  ctx->nccl_comm = nullptr;
}

void slab_plan(const int64_t* plane_start, const double* weight, int dimz, int reach, int world,
               SlabPlan& P) {
  P.world = world;
  P.plane_lo.assign(world + 1, 0);
  double total = 0.0;
  for (int p = 0; p < dimz; ++p) total += weight[p];
  // plane_lo[r] = first plane whose cumulative weight (planes before it) reaches r/world
  double cum = 0.0;
  int p = 0;
  for (int r = 1; r < world; ++r) {
    const double target = total * (double)r / (double)world;
    while (p < dimz && cum + weight[p] <= target) cum += weight[p++];
    // the plane straddling the target goes to whichever side leaves the smaller error
    if (p < dimz && (target - cum) > (cum + weight[p] - target)) cum += weight[p++];
    P.plane_lo[r] = std::max(p, P.plane_lo[r - 1]);
  }
  P.plane_lo[world] = dimz;
  P.own_lo.resize(world);
  P.own_hi.resize(world);
  P.win_lo.resize(world);
  P.win_hi.resize(world);
  for (int r = 0; r < world; ++r) {
    const int a = P.plane_lo[r], b = P.plane_lo[r + 1];
    P.own_lo[r] = plane_start[a];
    P.own_hi[r] = plane_start[b];
    if (a == b) {   // empty slab: empty window
      P.win_lo[r] = P.win_hi[r] = P.own_lo[r];
    } else {
      P.win_lo[r] = plane_start[std::max(0, a - reach)];
      P.win_hi[r] = plane_start[std::min(dimz, b + reach)];
    }
  }
}

rbf_status dist_plan_cells(rbf_ctx* ctx, rbf_cells* c, const std::vector<uint32_t>& row_tile_off,
                           int64_t ntiles, const std::vector<uint32_t>& row_tile_off_w, int64_t ntiles_w, int rank,
                           int world) {
  cudaStream_t s = ctx->stream;
  const int dimz = c->dim[2];
  const int64_t plane_cells = (int64_t)c->dim[0] * c->dim[1];
  DevBuf w, ps;
  RBF_TRY(w.alloc(8 * (size_t)dimz, s));
  RBF_TRY(ps.alloc(8 * (size_t)(dimz + 1), s));
  RBF_CUDA_TRY(cudaMemsetAsync(w.p, 0, 8 * (size_t)dimz, s));
  plane_stats_kernel<<<grid_for(c->ncell, 256), 256, 0, s>>>(c->cell_start.as<int32_t>(), c->ncell, plane_cells,
                                                             w.as<unsigned long long>());
  RBF_CHECK_LAUNCH();
  plane_start_kernel<<<grid_for(dimz + 1, 256), 256, 0, s>>>(c->cell_start.as<int32_t>(), dimz, plane_cells,
                                                             ps.as<int64_t>());
  RBF_CHECK_LAUNCH();
  std::vector<unsigned long long> hw(dimz);
  std::vector<int64_t> hps(dimz + 1);
  RBF_CUDA_TRY(cudaMemcpyAsync(hw.data(), w.p, 8 * (size_t)dimz, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(hps.data(), ps.p, 8 * (size_t)(dimz + 1), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<double> wd(hw.begin(), hw.end());
  SlabPlan& P = c->plan;
  // +1 plane: the traversal's cell range of a box edge is floor((z -/+ cc - lo) inv_h)
  slab_plan(hps.data(), wd.data(), dimz, c->reach + 1, world, P);
  const int r = rank;
  SlabView& V = c->view;
  V.o0 = P.own_lo[r];
  V.o1 = P.own_hi[r];
  V.h0 = P.win_lo[r];
  V.h1 = P.win_hi[r];
  V.p0 = P.plane_lo[r];
  V.p1 = P.plane_lo[r + 1];
  // tiles never cross cell rows; rows are numbered cy + dimy cz
  const int64_t dimy = c->dim[1];
  auto row_tiles = [&](int plane) -> int64_t {
    const int64_t row = (int64_t)plane * dimy;
    return row < (int64_t)row_tile_off.size() ? (int64_t)row_tile_off[row] : ntiles;
  };
  V.t0 = row_tiles(V.p0);
  V.t1 = row_tiles(V.p1);
  auto row_tiles_w = [&](int plane) -> int64_t {
    const int64_t row = (int64_t)plane * dimy;
    return row < (int64_t)row_tile_off_w.size() ? (int64_t)row_tile_off_w[row] : ntiles_w;
  };
  V.tw0 = row_tiles_w(V.p0);
  V.tw1 = row_tiles_w(V.p1);
  // interior wide tiles: planes below p1 - (reach + 1) read sources of this slab only
  const int pint = std::max(V.p0, V.p1 - (c->reach + 1));
  V.tw_int = std::min(row_tiles_w(pint), V.tw1) - V.tw0;
  return RBF_OK;
}


// ------------------------------------------------------------- collectives --
template <class T>
rbf_status halo_exchange(rbf_ctx* ctx, const rbf_cells* c, const T* x_loc, T* win, bool upper_only) {
  RBF_NVTX("halo_exchange");
  cudaStream_t s = ctx->stream;
  const SlabView& V = c->view;
  const SlabPlan& P = c->plan;
  const int64_t base = upper_only ? V.o0 : V.h0;
  if (V.o1 > V.o0)
    RBF_CUDA_TRY(cudaMemcpyAsync(win + (V.o0 - base), x_loc, sizeof(T) * (V.o1 - V.o0), cudaMemcpyDeviceToDevice, s));
  if (ctx->world == 1) return RBF_OK;
  std::vector<Xfer> sends, recvs;
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank) continue;
    // my owned slice inside q's window
    const int64_t qlo = upper_only ? P.own_lo[q] : P.win_lo[q];
    const int64_t slo = std::max(V.o0, qlo), shi = std::min(V.o1, P.win_hi[q]);
    if (shi > slo && P.own_hi[q] > P.own_lo[q]) sends.push_back(Xfer{q, const_cast<T*>(x_loc) + (slo - V.o0), shi - slo});
    // q's owned slice inside my window
    const int64_t rlo = std::max(P.own_lo[q], base), rhi = std::min(P.own_hi[q], V.h1);
    if (rhi > rlo && V.o1 > V.o0) recvs.push_back(Xfer{q, win + (rlo - base), rhi - rlo});
  }
  return ctx->tr->exchange(ctx, s, sends, recvs, sizeof(T) == 8 ? DType::F64 : DType::F32);
}
template rbf_status halo_exchange<float>(rbf_ctx*, const rbf_cells*, const float*, float*, bool);
template rbf_status halo_exchange<double>(rbf_ctx*, const rbf_cells*, const double*, double*, bool);

namespace {
__global__ void add_into(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}
}  // namespace

rbf_status halo_reduce(rbf_ctx* ctx, const rbf_cells* c, const double* fwin, double* f_loc) {
  RBF_NVTX("halo_reduce");
  cudaStream_t s = ctx->stream;
  const SlabView& V = c->view;
  const SlabPlan& P = c->plan;
  const int64_t nl = V.o1 - V.o0;
  if (nl > 0 && f_loc != fwin)
    RBF_CUDA_TRY(cudaMemcpyAsync(f_loc, fwin, sizeof(double) * nl, cudaMemcpyDeviceToDevice, s));
  if (ctx->world == 1) return RBF_OK;
  std::vector<Xfer> sends, recvs;
  std::vector<std::pair<int64_t, int64_t>> segs;   // (offset in f_loc, count) per receive
  int64_t scratch = 0;
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank || P.own_hi[q] <= P.own_lo[q]) continue;
    // contributions I accumulated for q's sources: q's slice inside my window beyond o1
    const int64_t slo = std::max(P.own_lo[q], V.o1), shi = std::min(P.own_hi[q], V.h1);
    if (shi > slo && nl > 0) sends.push_back(Xfer{q, const_cast<double*>(fwin) + (slo - V.o0), shi - slo});
    // q's contributions to my slice: my slice inside q's window beyond q's slice
    const int64_t rlo = std::max(V.o0, P.own_hi[q]), rhi = std::min(V.o1, P.win_hi[q]);
    if (rhi > rlo) {
      segs.push_back({rlo - V.o0, rhi - rlo});
      recvs.push_back(Xfer{q, nullptr, rhi - rlo});
      scratch += rhi - rlo;
    }
  }
  RBF_TRY(ctx->rsc.ensure(sizeof(double) * std::max<int64_t>(scratch, 1), s));
  int64_t off = 0;
  for (Xfer& x : recvs) { x.ptr = ctx->rsc.as<double>() + off; off += x.count; }
  RBF_TRY(ctx->tr->exchange(ctx, s, sends, recvs, DType::F64));
  off = 0;
  for (auto& sg : segs) {   // fixed order (ascending rank)
    add_into<<<grid_for(sg.second, 256), 256, 0, s>>>(f_loc + sg.first, ctx->rsc.as<double>() + off, sg.second);
    RBF_CHECK_LAUNCH();
    off += sg.second;
  }
  return RBF_OK;
}

// Every rank's shard (id0, n) of a caller-order array; checks that the shards
// tile [0, total) (any order of ranks, no overlap, no gap).
rbf_status shard_layout(rbf_ctx* ctx, int64_t id0, int64_t n_local, std::vector<int64_t>& id0s,
                        std::vector<int64_t>& ns, int64_t* total) {
  const int W = ctx->world;
  id0s.assign(W, 0);
  ns.assign(W, 0);
  if (W == 1) {
    id0s[0] = id0;
    ns[0] = n_local;
  } else {
    DevBuf d;
    RBF_TRY(d.alloc(sizeof(double) * 2 * W, ctx->stream));
    std::vector<double> h(2 * W, 0.0);
    h[2 * ctx->rank] = (double)id0;
    h[2 * ctx->rank + 1] = (double)n_local;
    RBF_CUDA_TRY(cudaMemcpyAsync(d.p, h.data(), sizeof(double) * 2 * W, cudaMemcpyHostToDevice, ctx->stream));
    RBF_TRY(allreduce_sum(ctx, d.as<double>(), 2 * W));
    RBF_CUDA_TRY(cudaMemcpyAsync(h.data(), d.p, sizeof(double) * 2 * W, cudaMemcpyDeviceToHost, ctx->stream));
    RBF_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    for (int q = 0; q < W; ++q) { id0s[q] = (int64_t)h[2 * q]; ns[q] = (int64_t)h[2 * q + 1]; }
  }
  std::vector<int> ord(W);
  for (int q = 0; q < W; ++q) ord[q] = q;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return id0s[a] < id0s[b]; });
  int64_t at = 0;
  for (int q : ord) {
    if (ns[q] < 0 || id0s[q] != at) { set_error("shards must tile [0, n_total) (id0 of each rank = sum of the lower shards)"); return RBF_EINVAL; }
    at += ns[q];
  }
  *total = at;
  return RBF_OK;
}

// full[id0_q * per ..] <- rank q's shard of `per` elements per item, for every q
rbf_status allgather_shards(rbf_ctx* ctx, const void* local, const std::vector<int64_t>& id0s,
                            const std::vector<int64_t>& ns, int per, void* full, DType t) {
  const size_t es = (size_t)t;
  const int r = ctx->rank;
  if (ns[r] > 0)
    RBF_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(full) + es * per * id0s[r], local, es * per * ns[r],
                                 cudaMemcpyDeviceToDevice, ctx->stream));
  if (ctx->world == 1) return RBF_OK;
  std::vector<Xfer> sends, recvs;
  for (int q = 0; q < ctx->world; ++q) {
    if (q == r) continue;
    if (ns[r] > 0) sends.push_back(Xfer{q, const_cast<void*>(local), ns[r] * per});
    if (ns[q] > 0) recvs.push_back(Xfer{q, static_cast<char*>(full) + es * per * id0s[q], ns[q] * per});
  }
  return ctx->tr->exchange(ctx, ctx->stream, sends, recvs, t);
}

rbf_status allreduce_sum(rbf_ctx* ctx, double* x, int64_t count) {
  if (ctx->world == 1 || count == 0) return RBF_OK;
  return ctx->tr->allreduce_sum(ctx, ctx->stream, x, count, DType::F64);
}

// full[0, n) (sorted order) <- every rank's owned slice; full + o0 must already
// hold this rank's slice
rbf_status allgather_sorted(rbf_ctx* ctx, const rbf_cells* c, double* full) {
  if (ctx->world == 1) return RBF_OK;
  const SlabPlan& P = c->plan;
  const SlabView& V = c->view;
  std::vector<Xfer> sends, recvs;
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank) continue;
    if (V.o1 > V.o0) sends.push_back(Xfer{q, full + V.o0, V.o1 - V.o0});
    if (P.own_hi[q] > P.own_lo[q]) recvs.push_back(Xfer{q, full + P.own_lo[q], P.own_hi[q] - P.own_lo[q]});
  }
  return ctx->tr->exchange(ctx, ctx->stream, sends, recvs, DType::F64);
}

void grid_layers(const rbf_cells* c, const rbf_grid* g, int r, int64_t* k0, int64_t* k1) {
  const int nz = g->n[2];
  const int nbz = (nz + 3) / 4;
  if (c->world == 1) { *k0 = 0; *k1 = nz; return; }
  const double step = (g->hi[2] - g->lo[2]) / (double)(nz - 1);
  const int p0 = c->plan.plane_lo[r], p1 = c->plan.plane_lo[r + 1];
  int bz0 = nbz, bz1 = nbz;
  for (int bz = 0; bz < nbz; ++bz) {
    const float z = (float)(g->lo[2] + (double)(4 * bz) * step);
    int pz = (int)std::floor((double)((z - c->lo[2]) * c->inv_h));
    pz = std::min(std::max(pz, 0), c->dim[2] - 1);
    // the first rank owns everything below the cell grid, the last everything above
    const bool mine = pz >= p0 && pz < p1;
    if (mine && bz0 == nbz) bz0 = bz;
    if (mine) bz1 = bz + 1;
  }
  if (bz0 == nbz) bz1 = bz0;
  *k0 = std::min<int64_t>(4 * (int64_t)bz0, nz);
  *k1 = std::min<int64_t>(4 * (int64_t)bz1, nz);
}

rbf_status allgather_layers(rbf_ctx* ctx, const rbf_cells* c, const rbf_grid* g, float* field) {
  if (ctx->world == 1) return RBF_OK;
  const int64_t layer = (int64_t)g->n[0] * g->n[1];
  int64_t m0, m1;
  grid_layers(c, g, ctx->rank, &m0, &m1);
  std::vector<Xfer> sends, recvs;
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank) continue;
    int64_t q0, q1;
    grid_layers(c, g, q, &q0, &q1);
    if (m1 > m0) sends.push_back(Xfer{q, field + m0 * layer, (m1 - m0) * layer});
    if (q1 > q0) recvs.push_back(Xfer{q, field + q0 * layer, (q1 - q0) * layer});
  }
  return ctx->tr->exchange(ctx, ctx->stream, sends, recvs, DType::F32);
}

rbf_status nccl_unique_id(void* out128) {
  NcclApi& api = nccl();
  if (!api.ok) { set_error(api.err); return RBF_ENCCL; }
  ncclUniqueId id;
  RBF_NCCL_TRY(api.GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return RBF_OK;
}

}  // namespace rbf

using namespace rbf;

extern "C" {

rbf_status rbf_nccl_unique_id(void* out128) {
  if (!out128) { set_error("out is NULL"); return RBF_EINVAL; }
  return nccl_unique_id(out128);
}

rbf_status rbf_loopback_group_create(int world, rbf_loopback_group** out) {
  if (!out) { set_error("out is NULL"); return RBF_EINVAL; }
  *out = nullptr;
  if (world < 1 || world > kLoopMaxWorld) { set_error("loopback world must be in [1, 64]"); return RBF_EINVAL; }
  LoopGroup* g = new (std::nothrow) LoopGroup();
  if (!g) { set_error("host allocation failed"); return RBF_ENOMEM; }
  g->world = world;
  g->slots.resize(world);
  g->joined.assign(world, 0);
  *out = reinterpret_cast<rbf_loopback_group*>(g);
  return RBF_OK;
}

void rbf_loopback_group_free(rbf_loopback_group* grp) {
  LoopGroup* g = reinterpret_cast<LoopGroup*>(grp);
  if (!g) return;
  for (auto& sl : g->slots) {
    if (sl.ready) cudaEventDestroy(sl.ready);
    if (sl.done) cudaEventDestroy(sl.done);
  }
  delete g;
}

rbf_status rbf_slab_plan(const int64_t* plane_start, const double* plane_weight, int dimz, int reach, int world,
                         int32_t* plane_lo, int64_t* own_lo, int64_t* own_hi, int64_t* win_lo, int64_t* win_hi) {
  if (!plane_start || !plane_weight || dimz < 1 || world < 1 || reach < 0) {
    set_error("bad slab plan arguments");
    return RBF_EINVAL;
  }
  for (int p = 0; p < dimz; ++p) {
    if (!(plane_weight[p] >= 0) || plane_start[p + 1] < plane_start[p]) {
      set_error("plane weights must be >= 0 and plane starts non-decreasing");
      return RBF_EINVAL;
    }
  }
  SlabPlan P;
  slab_plan(plane_start, plane_weight, dimz, reach, world, P);
  for (int r = 0; r <= world; ++r)
    if (plane_lo) plane_lo[r] = P.plane_lo[r];
  for (int r = 0; r < world; ++r) {
    if (own_lo) own_lo[r] = P.own_lo[r];
    if (own_hi) own_hi[r] = P.own_hi[r];
    if (win_lo) win_lo[r] = P.win_lo[r];
    if (win_hi) win_hi[r] = P.win_hi[r];
  }
  return RBF_OK;
}

}  // extern "C"
