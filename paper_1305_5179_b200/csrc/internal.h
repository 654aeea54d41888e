// Internal declarations shared by the library's translation units.
// Nothing here is part of the C-ABI (see include/rbf.h).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rbf.h"
#include "checks.h"

#include <nvtx3/nvToolsExt.h>

namespace rbf {

struct Transport;
void set_error(const std::string& msg);

#define RBF_CUDA_TRY(expr)                                                     \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::rbf::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));    \
      return RBF_ECUDA;                                                        \
    }                                                                          \
  } while (0)

#define RBF_TRY(expr)                                                          \
  do {                                                                         \
    rbf_status _s = (expr);                                                    \
    if (_s != RBF_OK) return _s;                                               \
  } while (0)

// Every kernel launch of the library is followed by RBF_CHECK_LAUNCH(), which also
// counts it (rbf_launch_count: the evidence of how many of our kernels ran).
void count_launch();
#define RBF_CHECK_LAUNCH()        \
  do {                            \
    ::rbf::count_launch();        \
    RBF_CUDA_TRY(cudaGetLastError()); \
  } while (0)

constexpr int kWarp = 32;

// The library's own stream-ordered memory pool on `device` (created on first
// use, release threshold = max: the solver frees and re-allocates GB-sized
// workspaces per fit, which must not go back to the driver at every
// synchronisation).  Private, so the process's default pool (and torch) is left
// alone; rbf_destroy trims it.
cudaMemPool_t lib_pool(int device);

// Stream-ordered device buffer (cudaMallocFromPoolAsync from lib_pool on the
// context stream).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; s = o.s; o.p = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
  }
  rbf_status alloc(size_t nbytes, cudaStream_t stream) {
    release();
    s = stream;
    if (nbytes == 0) nbytes = 16;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = lib_pool(dev);
    cudaError_t e = pool ? cudaMallocFromPoolAsync(&p, nbytes, pool, stream) : cudaMallocAsync(&p, nbytes, stream);
    if (e != cudaSuccess) {
      p = nullptr;
      set_error(std::string("cudaMallocAsync(") + std::to_string(nbytes) + "): " + cudaGetErrorString(e));
      cudaGetLastError();
      return RBF_ENOMEM;
    }
    bytes = nbytes;
    return RBF_OK;
  }
  // grow-only
  rbf_status ensure(size_t nbytes, cudaStream_t stream) {
    if (p && bytes >= nbytes) return RBF_OK;
    return alloc(nbytes, stream);
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

}  // namespace rbf

struct rbf_prof_rec {
  int stage;
  cudaEvent_t a, b;
};

struct rbf_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t aux_stream = nullptr;   // library-owned second stream (RAS factorisation overlap, halo exchange)
  cudaEvent_t halo_ev[2] = {nullptr, nullptr};   // fork / join of the halo exchange on aux_stream
  cudaEvent_t apply_ev[2] = {nullptr, nullptr};  // fork / join of the block-Jacobi apply's launch bins on aux_stream
  int sm_count = 148;
  bool prof = false;
  std::vector<rbf_prof_rec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t take_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  ~rbf_ctx() {
    for (auto& r : prof_recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : ev_pool) cudaEventDestroy(e);
    if (aux_stream) cudaStreamDestroy(aux_stream);
    for (auto e : halo_ev)
      if (e) cudaEventDestroy(e);
    for (auto e : apply_ev)
      if (e) cudaEventDestroy(e);
    if (hpin) cudaFreeHost(hpin);
  }
  rbf::DevBuf scratch;       // generic scratch (radix sort, scans)
  rbf::DevBuf counter;       // work counters (int32 x 64)
  rbf::DevBuf stats;         // pair counters (u64 x 4)
  rbf::DevBuf pinned_dummy;
  // pinned host scratch (GMRES Hessenberg slots), grown on demand
  void* hpin = nullptr;
  size_t hpin_bytes = 0;
  rbf_status pinned(size_t bytes) {
    if (bytes <= hpin_bytes) return RBF_OK;
    if (hpin) cudaFreeHost(hpin);
    hpin = nullptr;
    hpin_bytes = 0;
    if (cudaMallocHost(&hpin, bytes) != cudaSuccess) { cudaGetLastError(); return RBF_ENOMEM; }
    hpin_bytes = bytes;
    return RBF_OK;
  }
  // vector workspaces for matvec (sorted order)
  rbf::DevBuf vec_a, vec_b, src4;
  // multi-rank slab partition (dist.cu): the transport (NCCL communicator or
  // in-process loopback group), rank, world, halo windows and scratch
  void* nccl_comm = nullptr;
  rbf::Transport* tr = nullptr;
  void* loop_group = nullptr;   // rbf::LoopGroup of a loopback context
  int rank = 0, world = 1;
  bool nl_on = true;      // neighbour-list form of the symmetric fp32 operator (rbf_ctx_neighbour_lists)
  bool grid_per_pair = false;   // one exponential per (node, centre) pair instead of the separable form (rbf_ctx_grid_separable)
  bool peer_mem = true;   // use the transport's peer-memory mode when it has one (rbf_ctx_peer_memory)
  rbf::DevBuf win, fwin, rsc, red, pwin;
};

namespace rbf {
// This rank's share of the global sorted order (dist.cu).  Single GPU: the
// whole range.  Slab partition: owned targets [o0, o1) = cell planes [p0, p1)
// along z, their tiles [t0, t1), and the matvec source window [h0, h1).
struct SlabView {
  int64_t o0 = 0, o1 = 0;
  int64_t h0 = 0, h1 = 0;
  int64_t t0 = 0, t1 = 0;
  int p0 = 0, p1 = 0;
  int64_t tw0 = 0, tw1 = 0;   // tiles of the wide plan
  // wide tiles [tw0, tw0 + tw_int) lie in planes whose traversal stays inside the
  // slab (p < p1 - reach - 1): they need no halo, so they run while it arrives
  int64_t tw_int = 0;
};
// Every rank's slab (identical on all ranks: computed from the replicated cells).
struct SlabPlan {
  int world = 1;
  std::vector<int> plane_lo;                          // [world + 1]
  std::vector<int64_t> own_lo, own_hi, win_lo, win_hi;  // [world]
};
}  // namespace rbf

// Tile of targets for the summation kernels: sorted positions [start, start+count).
struct rbf_cells {
  int64_t n = 0;
  int dim[3] = {0, 0, 0};
  float lo[3] = {0, 0, 0};
  float inv_h = 0.f;
  double h = 0.0;
  double cutoff = 0.0;       // cutoff radius used to size the stencil at build time
  int reach = 0;
  int64_t ncell = 0;
  int64_t ntiles = 0;
  int64_t nonempty = 0;
  int tile_cap = 64;
  int tile_span = 2;
  // squared half-diagonal bound of the target-tile boxes (length units) of the
  // 64-target plan and of the wide plan: a tile spans <= span cells along x and
  // one cell along y and z, so hd^2 <= (h/2)^2 (span^2 + 2)
  double hd2 = 0.0, hd2_w = 0.0;
  rbf::DevBuf perm;          // int32[n]
  rbf::DevBuf sorted;        // float4[n]
  rbf::DevBuf keys;          // uint32[n]
  rbf::DevBuf cell_start;    // int32[ncell+1]
  rbf::DevBuf tiles;         // int2[ntiles] (start, count)
  rbf::DevBuf tile_box;      // float4[2*ntiles] (lo.xyz, ctr.x) (hi.xyz, unused)
  // wide plan (<= 128 targets, 4 per lane) of the symmetric fp32 matvec (reading R19)
  int64_t ntiles_w = 0;
  rbf::DevBuf tiles_w, tile_box_w;
  rbf::DevBuf order_w;       // this rank's wide tiles, most expensive first (summation.cu order_wide_tiles)
  // neighbour lists of the wide tiles (summation.cu ensure_nl; built on first use
  // by the symmetric fp32 operator): nl_off[nt + 1] (uint32), nl_idx[entries]
  // (int32 sorted source positions); keyed by the culling radius and the window
  mutable rbf::DevBuf nl_idx, nl_off;
  mutable int nl_state = 0;          // 0 not built, 1 valid, -1 unavailable for this key
  mutable float nl_cc = 0.f;
  mutable int64_t nl_hi = -1, nl_t0 = -1, nl_nt = -1, nl_entries = 0;
  cudaStream_t stream = nullptr;
  rbf::SlabView view;        // this rank's share (whole range on one GPU)
  rbf::SlabPlan plan;        // all ranks' slabs (world > 1)
  int world = 1;             // ranks the cells were partitioned for
  int64_t n_loc() const { return view.o1 - view.o0; }
};

namespace rbf {

// Geometry constants handed to the summation kernels.
struct CellGrid {
  float lo[3];
  float inv_h;
  float h;
  int dim[3];
};

// cells.cu
rbf_status build_cells(rbf_ctx* ctx, const float* xyz, int64_t n, const rbf_kernel* k,
                       const rbf_cell_cfg* cfg, rbf_cells* c);
// Stable LSD radix sort of (key, value) pairs on the low `bits` bits of the keys.
// keys/vals are clobbered; the result lands in keys_out/vals_out.
template <class K>
rbf_status radix_sort_pairs(rbf_ctx* ctx, K* keys, int32_t* vals, K* keys_out, int32_t* vals_out, int64_t n,
                            int bits);
rbf_status exclusive_scan_u32(rbf_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n,
                              uint32_t* total_dev /* may be null */);

// summation.cu
struct KernelParams {
  double sigma, cutoff, amp;
};
KernelParams kernel_params(const rbf_kernel* k);
// w_sorted: fp32 sorted-order weights (matvec fp32) -> f_sorted fp32
rbf_status matvec_sorted_f32(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp,
                             const float* w_sorted, float* f_sorted, const int32_t* out_perm,
                             unsigned long long* pair_stats);
// op: rbf_op_variant (RBF_OP_ONESIDED = the public, deterministic product; the
// solver may use a symmetric variant, reading R19)
rbf_status matvec_sorted_f64(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp,
                             const double* w_sorted, double* f_sorted, const int32_t* out_perm,
                             int op = RBF_OP_ONESIDED);
rbf_status order_wide_tiles(rbf_ctx* ctx, rbf_cells* c, const KernelParams& kp);
rbf_status ensure_nl(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp, bool* ok);
// near (optional, uint8 per node): evaluate only the node blocks holding a node
// with near != 0 and write NaN (all bits set) at every node with near == 0
// (the eps-surrounding M_ext^eps of §2.1.3)
rbf_status eval_grid_sorted(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp,
                            const double* w_sorted, const rbf_grid* g, float* field,
                            unsigned long long* pair_stats = nullptr, const uint8_t* near = nullptr);

// dist.cu (multi-rank slab partition over a Transport)
rbf_status dist_init(rbf_ctx* ctx, const void* unique_id, int rank, int world);
void dist_destroy(rbf_ctx* ctx);
void slab_plan(const int64_t* plane_start, const double* weight, int dimz, int reach, int world, SlabPlan& P);
rbf_status dist_plan_cells(rbf_ctx* ctx, rbf_cells* c, const std::vector<uint32_t>& row_tile_off, int64_t ntiles,
                           const std::vector<uint32_t>& row_tile_off_w, int64_t ntiles_w, int rank, int world);
// win <- the matvec source window of the distributed vector whose owned slice
// is x_loc: [h0, h1) (both neighbours), or [o0, h1) with upper_only (the
// symmetric operators: sources before a tile are never read, reading R19)
template <class T>
rbf_status halo_exchange(rbf_ctx* ctx, const rbf_cells* c, const T* x_loc, T* win, bool upper_only = false);
// symmetric operators: f_loc[0, o1-o0) = fwin[0, o1-o0) + the contributions to
// this rank's targets that lower ranks accumulated in their windows; fwin covers
// [o0, h1) and its part beyond o1 is sent to the owners (reverse halo reduce)
rbf_status halo_reduce(rbf_ctx* ctx, const rbf_cells* c, const double* fwin, double* f_loc);
rbf_status allreduce_sum(rbf_ctx* ctx, double* x, int64_t count);
rbf_status allgather_sorted(rbf_ctx* ctx, const rbf_cells* c, double* full);
// sharded caller-order inputs (rank r holds items [id0_r, id0_r + n_r)): every
// rank's (id0, n), checked to tile [0, total); and the replicated array from the shards
rbf_status shard_layout(rbf_ctx* ctx, int64_t id0, int64_t n_local, std::vector<int64_t>& id0s,
                        std::vector<int64_t>& ns, int64_t* total);
// the grid's node layers [k0, k1) owned by rank r (z layers; a layer belongs to
// the rank owning the cell plane of its first node block)
void grid_layers(const rbf_cells* c, const rbf_grid* g, int r, int64_t* k0, int64_t* k1);
rbf_status allgather_layers(rbf_ctx* ctx, const rbf_cells* c, const rbf_grid* g, float* field);

// pointset.cu: near[v] (uint8 per grid node, allocated here) = some data point
// (DEVICE fp64 ndata x 3) within eps of node v, fp64 distances (rbf_zero_set's mask)
rbf_status build_near_mask(rbf_ctx* ctx, const rbf_grid* grid, const double* data, int64_t ndata, double eps,
                           DevBuf& near);

// small vector kernels (vec.cu)
rbf_status gather_f32_to_sorted(rbf_ctx* ctx, const float* src, const int32_t* perm, float* dst, int64_t n);
rbf_status gather_f64_to_sorted(rbf_ctx* ctx, const double* src, const int32_t* perm, double* dst, int64_t n);
rbf_status gather_f64_to_sorted_f32(rbf_ctx* ctx, const double* src, const int32_t* perm, float* dst, int64_t n);
rbf_status gather_f32_to_sorted_f64(rbf_ctx* ctx, const float* src, const int32_t* perm, double* dst, int64_t n);
rbf_status scatter_f64_from_sorted_f32(rbf_ctx* ctx, const double* src, const int32_t* perm, float* dst, int64_t n);
rbf_status scatter_f32_from_sorted(rbf_ctx* ctx, const float* src, const int32_t* perm, float* dst, int64_t n);
rbf_status scatter_f64_from_sorted(rbf_ctx* ctx, const double* src, const int32_t* perm, double* dst, int64_t n);

// Raise a kernel's dynamic shared-memory limit to at least `bytes` (monotone and
// thread-safe: contexts on several host threads launch the same kernels with
// different needs, and the attribute is per function, not per launch).
rbf_status smem_limit_at_least(const void* func, size_t bytes);
template <class F>
rbf_status smem_limit_at_least(F* func, size_t bytes) {
  return smem_limit_at_least(reinterpret_cast<const void*>(func), bytes);
}

inline int grid_for(int64_t n, int threads, int max_blocks = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

}  // namespace rbf

namespace rbf {
const char* last_error_cstr();

// NVTX range over a library phase (timelines in Nsight Systems; a few ns when no
// tool is attached).  RBF_NVTX("rbf_gmres_solve") at the top of a scope.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define RBF_NVTX_CAT2(a, b) a##b
#define RBF_NVTX_CAT(a, b) RBF_NVTX_CAT2(a, b)
#define RBF_NVTX(name) ::rbf::NvtxRange RBF_NVTX_CAT(rbf_nvtx_, __LINE__)(name)

// Brackets the launches issued in its scope with CUDA events when profiling is on.
struct ProfScope {
  rbf_ctx* ctx;
  int stage;
  cudaEvent_t a = nullptr;
  ProfScope(rbf_ctx* c, int s) : ctx(c), stage(s) {
    if (ctx && ctx->prof) {
      a = ctx->take_event();
      cudaEventRecord(a, ctx->stream);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = ctx->take_event();
      cudaEventRecord(b, ctx->stream);
      ctx->prof_recs.push_back(rbf_prof_rec{stage, a, b});
    }
  }
};
}
