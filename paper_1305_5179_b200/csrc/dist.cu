// multi-GPU partition of the hot path by spatial slabs.
//
// One process per GPU; every rank receives the full (replicated) centre set and
// builds the same global cell structure, then owns a slab of whole cell planes
// along z (the slowest axis of the cell key, so a slab is a CONTIGUOUS range of
// the sorted order).  Slab boundaries balance an estimate of the useful pairs
// per plane, sum over the plane's cells of n_c^2 (pairs per centre grow with
// the local density; c3's density varies 10x).  Per fp32/fp64 matvec the rank
// needs the weights of the sources within the cutoff of its targets: the planes
// [p0 - reach, p1 + reach) -- a contiguous window of the sorted order -- which
// it assembles from its own slice plus grouped ncclSend/ncclRecv with the ranks
// owning the rest of the window (the paper's "communication ... limited to a
// constant number of elements in the vicinity").  Krylov inner products
// are local partial sums + ncclAllReduce; results are gathered with grouped
// ncclBroadcast so every rank returns the full vectors (replicated in,
// replicated out).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: inside a torch process
// this resolves to the NCCL torch already loaded), so librbf.so carries no link
// dependency and single-GPU use never touches it.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

#include "internal.h"

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

inline ncclComm_t comm_of(const rbf_ctx* ctx) { return static_cast<ncclComm_t>(ctx->nccl_comm); }

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

}  // namespace

rbf_status dist_init(rbf_ctx* ctx, const void* unique_id, int rank, int world) {
  NcclApi& api = nccl();
  if (!api.ok) { set_error(api.err); return RBF_ENCCL; }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  RBF_NCCL_TRY(api.CommInitRank(&comm, world, id, rank));
  ctx->nccl_comm = comm;
  ctx->rank = rank;
  ctx->world = world;
  return RBF_OK;
}

void dist_destroy(rbf_ctx* ctx) {
  if (ctx->nccl_comm && nccl().ok) nccl().CommDestroy(comm_of(ctx));
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
  return RBF_OK;
}

// win[0, h1-h0) <- window of the distributed vector whose owned slice is x_loc
template <class T>
rbf_status halo_exchange(rbf_ctx* ctx, const rbf_cells* c, const T* x_loc, T* win) {
  cudaStream_t s = ctx->stream;
  const SlabView& V = c->view;
  const SlabPlan& P = c->plan;
  if (V.o1 > V.o0)
    RBF_CUDA_TRY(cudaMemcpyAsync(win + (V.o0 - V.h0), x_loc, sizeof(T) * (V.o1 - V.o0), cudaMemcpyDeviceToDevice, s));
  if (ctx->world == 1) {
    // emulated slab (single GPU, tests): x_loc points into the full sorted
    // vector, so the window is read in place
    if (c->emulated && V.h1 > V.h0)
      RBF_CUDA_TRY(cudaMemcpyAsync(win, x_loc - (V.o0 - V.h0), sizeof(T) * (V.h1 - V.h0), cudaMemcpyDeviceToDevice, s));
    return RBF_OK;
  }
  NcclApi& api = nccl();
  const int dt = sizeof(T) == 8 ? kNcclFloat64 : kNcclFloat32;
  RBF_NCCL_TRY(api.GroupStart());
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->rank) continue;
    // my owned slice inside q's window
    const int64_t slo = std::max(V.o0, P.win_lo[q]), shi = std::min(V.o1, P.win_hi[q]);
    if (shi > slo) RBF_NCCL_TRY(api.Send(x_loc + (slo - V.o0), (size_t)(shi - slo), dt, q, comm_of(ctx), s));
    // q's owned slice inside my window
    const int64_t rlo = std::max(P.own_lo[q], V.h0), rhi = std::min(P.own_hi[q], V.h1);
    if (rhi > rlo) RBF_NCCL_TRY(api.Recv(win + (rlo - V.h0), (size_t)(rhi - rlo), dt, q, comm_of(ctx), s));
  }
  RBF_NCCL_TRY(api.GroupEnd());
  return RBF_OK;
}
template rbf_status halo_exchange<float>(rbf_ctx*, const rbf_cells*, const float*, float*);
template rbf_status halo_exchange<double>(rbf_ctx*, const rbf_cells*, const double*, double*);

rbf_status allreduce_sum(rbf_ctx* ctx, double* x, int64_t count) {
  if (ctx->world == 1 || count == 0) return RBF_OK;
  RBF_NCCL_TRY(nccl().AllReduce(x, x, (size_t)count, kNcclFloat64, kNcclSum, comm_of(ctx), ctx->stream));
  return RBF_OK;
}
rbf_status allreduce_sum_f32(rbf_ctx* ctx, float* x, int64_t count) {
  if (ctx->world == 1 || count == 0) return RBF_OK;
  RBF_NCCL_TRY(nccl().AllReduce(x, x, (size_t)count, kNcclFloat32, kNcclSum, comm_of(ctx), ctx->stream));
  return RBF_OK;
}

// full[0, n) (sorted order) <- every rank's owned slice; full + o0 must already
// hold this rank's slice
rbf_status allgather_sorted(rbf_ctx* ctx, const rbf_cells* c, double* full) {
  if (ctx->world == 1) return RBF_OK;
  NcclApi& api = nccl();
  const SlabPlan& P = c->plan;
  RBF_NCCL_TRY(api.GroupStart());
  for (int q = 0; q < ctx->world; ++q) {
    const int64_t lo = P.own_lo[q], cnt = P.own_hi[q] - lo;
    if (cnt > 0) RBF_NCCL_TRY(api.Broadcast(full + lo, full + lo, (size_t)cnt, kNcclFloat64, q, comm_of(ctx),
                                            ctx->stream));
  }
  RBF_NCCL_TRY(api.GroupEnd());
  return RBF_OK;
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
