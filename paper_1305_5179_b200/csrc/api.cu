// C-ABI entry points (include/rbf.h): validation, handle management and
// dispatch to the device code.  Every step of the path runs in this
// library's kernels; there is no host compute fallback.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <new>

#include "internal.h"
#include "solver.h"
#include "transport.h"

namespace rbf {
namespace {
thread_local std::string g_last_error;
}
void set_error(const std::string& msg) { g_last_error = msg; }
namespace {
std::atomic<unsigned long long> g_launches{0};
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
const char* last_error_cstr() { return g_last_error.c_str(); }

rbf_status smem_limit_at_least(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<const void*, size_t> cur;
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[func];
  if (bytes <= c && c > 0) return RBF_OK;
  const size_t want = std::max<size_t>(bytes, 48 * 1024);
  RBF_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want));
  c = want;
  return RBF_OK;
}

cudaMemPool_t lib_pool(int device) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(device);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    pool = nullptr;   // DevBuf falls back to the device's current pool
  } else {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  pools[device] = pool;
  return pool;
}
}  // namespace rbf

using namespace rbf;

namespace {

rbf_status check_kernel(const rbf_kernel* k) {
  if (!k) { set_error("kernel is NULL"); return RBF_EINVAL; }
  if (!(k->sigma > 0) || !std::isfinite(k->sigma)) { set_error("sigma must be > 0"); return RBF_EINVAL; }
  if (!(k->cutoff_sigmas > 0) || !std::isfinite(k->cutoff_sigmas)) {
    set_error("cutoff_sigmas must be > 0");
    return RBF_EINVAL;
  }
  if (!std::isfinite(k->amplitude)) { set_error("amplitude must be finite"); return RBF_EINVAL; }
  return RBF_OK;
}

rbf_status check_cells(const rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* k) {
  if (!ctx) { set_error("ctx is NULL"); return RBF_EINVAL; }
  if (!c) { set_error("cells is NULL"); return RBF_EINVAL; }
  RBF_TRY(check_kernel(k));
  // the stencil was sized for the cutoff given at build time
  double cut = k->cutoff_sigmas * k->sigma;
  if (cut > c->cutoff * (1 + 1e-12)) {
    set_error("kernel cutoff exceeds the cutoff the cells were built for");
    return RBF_EINVAL;
  }
  if (c->world != ctx->world) { set_error("cells were partitioned for another world size"); return RBF_EINVAL; }
  return RBF_OK;
}

}  // namespace

extern "C" {

const char* rbf_status_str(rbf_status s) {
  switch (s) {
    case RBF_OK: return "RBF_OK";
    case RBF_EINVAL: return "RBF_EINVAL";
    case RBF_ENOMEM: return "RBF_ENOMEM";
    case RBF_ECUDA: return "RBF_ECUDA";
    case RBF_ENCCL: return "RBF_ENCCL";
    case RBF_EUNSUPPORTED: return "RBF_EUNSUPPORTED";
  }
  return "RBF_UNKNOWN";
}

const char* rbf_last_error(void) { return last_error_cstr(); }

int rbf_abi_version(void) { return RBF_ABI_VERSION; }

int64_t rbf_launch_count(void) { return (int64_t)g_launches.load(std::memory_order_relaxed); }

rbf_status rbf_pool_stats(rbf_ctx* ctx, uint64_t* out) {
  if (!ctx || !out) { set_error("NULL argument"); return RBF_EINVAL; }
  cudaMemPool_t pool = lib_pool(ctx->device);
  if (!pool) RBF_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
  RBF_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &out[0]));
  RBF_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &out[1]));
  return RBF_OK;
}

rbf_status rbf_pool_reserve(rbf_ctx* ctx, uint64_t bytes) {
  if (!ctx) { set_error("ctx is NULL"); return RBF_EINVAL; }
  if (bytes == 0) return RBF_OK;
  // one block of `bytes`, returned to the pool at once: the pool grows by what
  // its free blocks cannot serve contiguously, and keeps it (its release
  // threshold is unlimited)
  DevBuf tmp;
  rbf_status r = tmp.alloc((size_t)bytes, ctx->stream);
  if (r != RBF_OK) return RBF_ENOMEM;
  tmp.release();
  RBF_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return RBF_OK;
}

}  // extern "C"

namespace {
rbf_status create_ctx(rbf_ctx** out, int device, void* cuda_stream) {
  if (!out) { set_error("out is NULL"); return RBF_EINVAL; }
  *out = nullptr;
  int ndev = 0;
  RBF_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) { set_error("bad device ordinal"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  RBF_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_error("librbf is built for sm_100a (B200); device has compute capability " + std::to_string(prop.major) +
              "." + std::to_string(prop.minor));
    return RBF_EUNSUPPORTED;
  }
  rbf_ctx* c = new (std::nothrow) rbf_ctx();
  if (!c) { set_error("host allocation failed"); return RBF_ENOMEM; }
  c->device = device;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  c->sm_count = prop.multiProcessorCount;
  lib_pool(device);   // the library's private stream-ordered pool (internal.h)
  *out = c;
  return RBF_OK;
}
}  // namespace

extern "C" {

rbf_status rbf_create(rbf_ctx** out, int device, void* cuda_stream, const void* nccl_unique_id, int rank,
                      int world) {
  if (!out) { set_error("out is NULL"); return RBF_EINVAL; }
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) { set_error("need 0 <= rank < world"); return RBF_EINVAL; }
  if (world > 1 && nccl_unique_id == nullptr) {
    set_error("world > 1 needs the NCCL unique id of rank 0 (rbf_nccl_unique_id)");
    return RBF_EINVAL;
  }
  rbf_ctx* c = nullptr;
  RBF_TRY(create_ctx(&c, device, cuda_stream));
  if (world > 1) {
    rbf_status st = dist_init(c, nccl_unique_id, rank, world);
    if (st != RBF_OK) { delete c; return st; }
  }
  *out = c;
  return RBF_OK;
}

rbf_status rbf_create_loopback(rbf_ctx** out, int device, void* cuda_stream, rbf_loopback_group* grp, int rank) {
  if (!out || !grp) { set_error("NULL argument"); return RBF_EINVAL; }
  *out = nullptr;
  LoopGroup* g = reinterpret_cast<LoopGroup*>(grp);
  if (rank < 0 || rank >= g->world) { set_error("rank out of range"); return RBF_EINVAL; }
  {
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->joined[rank]) { set_error("rank already joined the loopback group"); return RBF_EINVAL; }
    g->joined[rank] = 1;
  }
  rbf_ctx* c = nullptr;
  rbf_status st = create_ctx(&c, device, cuda_stream);
  if (st != RBF_OK) {
    std::lock_guard<std::mutex> lk(g->mu);
    g->joined[rank] = 0;
    return st;
  }
  c->rank = rank;
  c->world = g->world;
  c->tr = make_loop_transport(g, rank);
  c->loop_group = g;
  *out = c;
  return RBF_OK;
}

rbf_status rbf_create_ipc(rbf_ctx** out, int device, void* cuda_stream, const void* key16, int rank, int world) {
  if (!out || !key16) { set_error("NULL argument"); return RBF_EINVAL; }
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) { set_error("need 0 <= rank < world"); return RBF_EINVAL; }
  rbf_ctx* c = nullptr;
  RBF_TRY(create_ctx(&c, device, cuda_stream));
  Transport* t = nullptr;
  rbf_status st = make_ipc_transport(device, key16, rank, world, &t);
  if (st != RBF_OK) { delete c; return st; }
  c->rank = rank;
  c->world = world;
  c->tr = t;
  *out = c;
  return RBF_OK;
}

rbf_status rbf_ctx_peer_memory(rbf_ctx* ctx, int on) {
  if (!ctx) { set_error("ctx is NULL"); return RBF_EINVAL; }
  ctx->peer_mem = on != 0;
  return RBF_OK;
}

rbf_status rbf_ctx_neighbour_lists(rbf_ctx* ctx, int on) {
  if (!ctx) { set_error("ctx is NULL"); return RBF_EINVAL; }
  ctx->nl_on = on != 0;
  return RBF_OK;
}

rbf_status rbf_ctx_grid_separable(rbf_ctx* ctx, int on) {
  if (!ctx) { set_error("ctx is NULL"); return RBF_EINVAL; }
  ctx->grid_per_pair = on == 0;
  return RBF_OK;
}

rbf_status rbf_profile_enable(rbf_ctx* ctx, int on) {
  if (!ctx) { set_error("ctx is NULL"); return RBF_EINVAL; }
  ctx->prof = on != 0;
  if (ctx->prof) {
    // The stage timers take two CUDA events per bracket (a few hundred per
    // reconstruction) and return them at rbf_profile_query.  Create a stock of
    // them NOW: created on demand, the ~2000th event of a process made the
    // driver extend its event storage in the middle of a timed step -- 10 ms on
    // an idle box, 100-300 ms right after another process had released tens of
    // GB (the stall landed in whichever stage asked for the event).
    constexpr size_t kStock = 16384;
    ctx->ev_pool.reserve(kStock);
    while (ctx->ev_pool.size() < kStock) {
      cudaEvent_t e = nullptr;
      RBF_CUDA_TRY(cudaEventCreate(&e));
      ctx->ev_pool.push_back(e);
    }
  }
  return RBF_OK;
}

rbf_status rbf_profile_query(rbf_ctx* ctx, double* ms, int64_t* launches) {
  if (!ctx) { set_error("ctx is NULL"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < RBF_PROF_COUNT; ++k) {
    if (ms) ms[k] = 0.0;
    if (launches) launches[k] = 0;
  }
  for (auto& r : ctx->prof_recs) {
    float t = 0.f;
    RBF_CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    if (ms) ms[r.stage] += t;
    if (launches) launches[r.stage] += 1;
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  ctx->prof_recs.clear();
  return RBF_OK;
}

void rbf_destroy(rbf_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  cudaStreamSynchronize(s);
  dist_destroy(ctx);
  const int dev = ctx->device;
  if (ctx->loop_group) {
    LoopGroup* g = static_cast<LoopGroup*>(ctx->loop_group);
    std::lock_guard<std::mutex> lk(g->mu);
    g->joined[ctx->rank] = 0;
  }
  delete ctx;  // DevBufs free stream-ordered
  cudaStreamSynchronize(s);
  // hand the freed workspaces back to the driver (memory still held by other
  // live contexts / handles stays allocated)
  if (cudaMemPool_t pool = lib_pool(dev)) cudaMemPoolTrimTo(pool, 0);
}

rbf_status rbf_build_cells_shard(rbf_ctx* ctx, const float* xyz_local, int64_t n_local, int64_t id0,
                                 const rbf_kernel* kern, const rbf_cell_cfg* cfg, rbf_cells** out) {
  if (!ctx || !out) { set_error("ctx/out is NULL"); return RBF_EINVAL; }
  *out = nullptr;
  if (n_local < 0 || id0 < 0 || (n_local > 0 && !xyz_local)) { set_error("bad shard"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  std::vector<int64_t> id0s, ns;
  int64_t total = 0;
  RBF_TRY(shard_layout(ctx, id0, n_local, id0s, ns, &total));
  if (total < 1 || total > (int64_t)INT32_MAX / 2) { set_error("n out of range"); return RBF_EINVAL; }
  DevBuf full;
  RBF_TRY(full.alloc(sizeof(float) * 3 * total, ctx->stream));
  RBF_TRY(allgather_shards(ctx, xyz_local, id0s, ns, 3, full.p, DType::F32));
  return rbf_build_cells(ctx, full.as<float>(), total, kern, cfg, out);
}

rbf_status rbf_build_cells(rbf_ctx* ctx, const float* xyz, int64_t n, const rbf_kernel* kern,
                           const rbf_cell_cfg* cfg, rbf_cells** out) {
  RBF_NVTX("rbf_build_cells");
  if (!ctx || !out) { set_error("ctx/out is NULL"); return RBF_EINVAL; }
  *out = nullptr;
  RBF_TRY(check_kernel(kern));
  if (n < 1 || n > (int64_t)INT32_MAX / 2) { set_error("n out of range"); return RBF_EINVAL; }
  if (!xyz) { set_error("xyz is NULL"); return RBF_EINVAL; }
  if (cfg && cfg->cell_edge < 0) { set_error("cell_edge must be >= 0"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  rbf_cells* c = new (std::nothrow) rbf_cells();
  if (!c) { set_error("host allocation failed"); return RBF_ENOMEM; }
  rbf_status st;
  {
    ProfScope ps(ctx, RBF_PROF_CELLS);
    st = build_cells(ctx, xyz, n, kern, cfg, c);
  }
  if (st != RBF_OK) { delete c; return st; }
  *out = c;
  return RBF_OK;
}

void rbf_cells_free(rbf_cells* c) { delete c; }

rbf_status rbf_cells_info(const rbf_cells* c, rbf_cells_desc* d) {
  if (!c || !d) { set_error("NULL argument"); return RBF_EINVAL; }
  d->n = c->n;
  for (int a = 0; a < 3; ++a) { d->dim[a] = c->dim[a]; d->lo[a] = c->lo[a]; }
  d->inv_h = c->inv_h;
  d->cell_edge = c->h;
  d->reach = c->reach;
  d->ncell = c->ncell;
  d->ntiles = c->ntiles;
  d->nonempty_cells = c->nonempty;
  return RBF_OK;
}

rbf_status rbf_cells_slab(const rbf_cells* c, int64_t* out) {
  if (!c || !out) { set_error("NULL argument"); return RBF_EINVAL; }
  const SlabView& V = c->view;
  const int64_t v[11] = {V.o0, V.o1, V.h0, V.h1, V.t0, V.t1, V.p0, V.p1, V.tw0, V.tw1, c->world > 1 ? V.tw_int : 0};
  std::copy(v, v + 11, out);
  return RBF_OK;
}

rbf_status rbf_cells_view(const rbf_cells* c, const int32_t** perm, const float** sorted, const uint32_t** keys,
                          const int32_t** cell_start) {
  if (!c) { set_error("cells is NULL"); return RBF_EINVAL; }
  if (perm) *perm = c->perm.as<int32_t>();
  if (sorted) *sorted = c->sorted.as<float>();
  if (keys) *keys = c->keys.as<uint32_t>();
  if (cell_start) *cell_start = c->cell_start.as<int32_t>();
  return RBF_OK;
}

}  // extern "C"

namespace {
// f = A w through operator variant op (RBF_OP_ONESIDED: the public product).
rbf_status matvec_impl(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, rbf_precision prec, int op,
                       const void* w, void* f) {
  RBF_TRY(check_cells(ctx, c, kern));
  if (!w || !f) { set_error("w/f is NULL"); return RBF_EINVAL; }
  if (w == f) { set_error("w and f must not alias"); return RBF_EINVAL; }
  if (prec != RBF_F32 && prec != RBF_F64) { set_error("bad precision"); return RBF_EINVAL; }
  if (op < RBF_OP_AUTO || op > RBF_OP_SYM_ROT) { set_error("bad operator variant"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  KernelParams kp = kernel_params(kern);
  const int64_t n = c->n;
  if (ctx->world > 1 || op != RBF_OP_ONESIDED) {
    // solver operator / slab partition: replicated in, this rank's rows, gathered out
    RBF_TRY(ctx->vec_a.ensure(sizeof(double) * n, ctx->stream));
    RBF_TRY(ctx->vec_b.ensure(sizeof(double) * n, ctx->stream));
    double* ws = ctx->vec_a.as<double>();
    double* fs = ctx->vec_b.as<double>();
    if (prec == RBF_F32) {
      RBF_TRY(gather_f32_to_sorted_f64(ctx, static_cast<const float*>(w), c->perm.as<int32_t>(), ws, n));
      RBF_TRY(matvec_sorted_f32_d(ctx, c, kp, ws + c->view.o0, fs + c->view.o0, op));
    } else {
      RBF_TRY(gather_f64_to_sorted(ctx, static_cast<const double*>(w), c->perm.as<int32_t>(), ws, n));
      RBF_TRY(matvec_sorted_f64(ctx, c, kp, ws + c->view.o0, fs + c->view.o0, nullptr, op));
    }
    RBF_TRY(allgather_sorted(ctx, c, fs));
    if (prec == RBF_F32) return scatter_f64_from_sorted_f32(ctx, fs, c->perm.as<int32_t>(), static_cast<float*>(f), n);
    return scatter_f64_from_sorted(ctx, fs, c->perm.as<int32_t>(), static_cast<double*>(f), n);
  }
  if (prec == RBF_F32) {
    RBF_TRY(ctx->vec_a.ensure(sizeof(float) * n, ctx->stream));
    RBF_TRY(gather_f32_to_sorted(ctx, static_cast<const float*>(w), c->perm.as<int32_t>(), ctx->vec_a.as<float>(), n));
    return matvec_sorted_f32(ctx, c, kp, ctx->vec_a.as<float>(), static_cast<float*>(f), c->perm.as<int32_t>(),
                             nullptr);
  }
  RBF_TRY(ctx->vec_a.ensure(sizeof(double) * n, ctx->stream));
  RBF_TRY(gather_f64_to_sorted(ctx, static_cast<const double*>(w), c->perm.as<int32_t>(), ctx->vec_a.as<double>(),
                               n));
  return matvec_sorted_f64(ctx, c, kp, ctx->vec_a.as<double>(), static_cast<double*>(f), c->perm.as<int32_t>());
}
}  // namespace

extern "C" {

rbf_status rbf_matvec(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, rbf_precision prec, const void* w,
                      void* f) {
  RBF_NVTX("rbf_matvec");
  return matvec_impl(ctx, c, kern, prec, RBF_OP_ONESIDED, w, f);
}

rbf_status rbf_matvec_op(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, rbf_precision prec, int op,
                         const void* w, void* f) {
  return matvec_impl(ctx, c, kern, prec, op, w, f);
}

rbf_status rbf_matvec_pairs(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, int64_t* useful,
                            int64_t* visited) {
  RBF_TRY(check_cells(ctx, c, kern));
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  KernelParams kp = kernel_params(kern);
  const int64_t n = c->n;
  cudaStream_t s = ctx->stream;
  RBF_TRY(ctx->vec_a.ensure(sizeof(float) * n, s));
  RBF_TRY(ctx->vec_b.ensure(sizeof(float) * n, s));
  RBF_TRY(ctx->stats.ensure(64, s));
  RBF_CUDA_TRY(cudaMemsetAsync(ctx->vec_a.p, 0, sizeof(float) * n, s));
  RBF_CUDA_TRY(cudaMemsetAsync(ctx->stats.p, 0, 16, s));
  RBF_TRY(matvec_sorted_f32(ctx, c, kp, ctx->vec_a.as<float>(), ctx->vec_b.as<float>(), nullptr,
                            ctx->stats.as<unsigned long long>()));
  unsigned long long h[2];
  RBF_CUDA_TRY(cudaMemcpyAsync(h, ctx->stats.p, 16, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  if (useful) *useful = (int64_t)h[0];
  if (visited) *visited = (int64_t)h[1];
  return RBF_OK;
}

}  // extern "C"

namespace {
rbf_status check_grid(const rbf_grid* g) {
  if (!g) { set_error("grid is NULL"); return RBF_EINVAL; }
  for (int a = 0; a < 3; ++a) {
    if (g->n[a] < 2) { set_error("grid needs n >= 2 nodes per axis"); return RBF_EINVAL; }
    if (!std::isfinite(g->lo[a]) || !std::isfinite(g->hi[a]) || !(g->hi[a] > g->lo[a])) {
      set_error("grid box must satisfy lo < hi (finite)");
      return RBF_EINVAL;
    }
  }
  if ((double)g->n[0] * g->n[1] * g->n[2] > 4e9) { set_error("grid too large"); return RBF_EINVAL; }
  return RBF_OK;
}

rbf_status eval_grid_impl(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, const double* w,
                          const rbf_grid* g, float* field, bool gather, int64_t* k0, int64_t* k1) {
  RBF_TRY(check_cells(ctx, c, kern));
  if (!w || !field) { set_error("NULL argument"); return RBF_EINVAL; }
  RBF_TRY(check_grid(g));
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  KernelParams kp = kernel_params(kern);
  RBF_TRY(ctx->vec_a.ensure(sizeof(double) * c->n, ctx->stream));
  RBF_TRY(gather_f64_to_sorted(ctx, w, c->perm.as<int32_t>(), ctx->vec_a.as<double>(), c->n));
  // each rank evaluates the node layers of its slab; the gather completes the field
  RBF_TRY(eval_grid_sorted(ctx, c, kp, ctx->vec_a.as<double>(), g, field));
  if (k0 || k1) {
    int64_t a, b;
    grid_layers(c, g, ctx->rank, &a, &b);
    if (k0) *k0 = a;
    if (k1) *k1 = b;
  }
  return gather ? allgather_layers(ctx, c, g, field) : RBF_OK;
}
}  // namespace

namespace rbf {
// isosurface.cu: the grid evaluated on the eps-surrounding only (near != 0), NaN
// elsewhere; the slab layers of every rank are gathered as in rbf_eval_grid
rbf_status eval_grid_masked_impl(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, const double* w,
                                 const rbf_grid* g, const uint8_t* near, float* field) {
  RBF_TRY(check_cells(ctx, c, kern));
  if (!w || !field || !near) { set_error("NULL argument"); return RBF_EINVAL; }
  RBF_TRY(check_grid(g));
  KernelParams kp = kernel_params(kern);
  RBF_TRY(ctx->vec_a.ensure(sizeof(double) * c->n, ctx->stream));
  RBF_TRY(gather_f64_to_sorted(ctx, w, c->perm.as<int32_t>(), ctx->vec_a.as<double>(), c->n));
  RBF_TRY(eval_grid_sorted(ctx, c, kp, ctx->vec_a.as<double>(), g, field, nullptr, near));
  return allgather_layers(ctx, c, g, field);
}
}  // namespace rbf

extern "C" {

rbf_status rbf_eval_grid(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, const double* w,
                         const rbf_grid* g, float* field) {
  RBF_NVTX("rbf_eval_grid");
  return eval_grid_impl(ctx, c, kern, w, g, field, true, nullptr, nullptr);
}

rbf_status rbf_eval_grid_slab(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, const double* w,
                              const rbf_grid* g, float* field, int64_t* k0, int64_t* k1) {
  return eval_grid_impl(ctx, c, kern, w, g, field, false, k0, k1);
}

rbf_status rbf_eval_grid_pairs(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, const rbf_grid* g,
                               int64_t* useful, int64_t* visited) {
  RBF_TRY(check_cells(ctx, c, kern));
  if (!g) { set_error("grid is NULL"); return RBF_EINVAL; }
  for (int a = 0; a < 3; ++a)
    if (g->n[a] < 2) { set_error("grid needs n >= 2 nodes per axis"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  RBF_TRY(ctx->stats.ensure(64, s));
  RBF_CUDA_TRY(cudaMemsetAsync(ctx->stats.p, 0, 16, s));
  RBF_TRY(eval_grid_sorted(ctx, c, kernel_params(kern), nullptr, g, nullptr, ctx->stats.as<unsigned long long>()));
  unsigned long long h[2];
  RBF_CUDA_TRY(cudaMemcpyAsync(h, ctx->stats.p, 16, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  if (useful) *useful = (int64_t)h[0];
  if (visited) *visited = (int64_t)h[1];
  return RBF_OK;
}

}  // extern "C"
