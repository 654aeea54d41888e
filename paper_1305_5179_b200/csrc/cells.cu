// a1/a2 of SURVEY.md §8(a): cell-list build and target-tile plan.
//
// The paper's locality argument (§3.1) and Alg.2's "truncation
// area" need, for every target, the centres within the cutoff.
// Centres are binned into cubic cells of edge h, sorted stably by the linear
// cell key (x fastest) with a hand-written LSD radix sort, and cell k's
// centres occupy sorted positions [cell_start[k], cell_start[k+1]).
// The fp32 binning arithmetic is fixed so that the result is bit-identical to
// the CPU replica in oracle/cells.py.
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace rbf {
namespace {

// ---------------------------------------------------------------- bbox ------
constexpr int kBoxThreads = 256;

__global__ void bbox_kernel(const float* __restrict__ xyz, int64_t n, float* __restrict__ out) {
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  float bad = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float v = xyz[3 * i + a];
      if (!isfinite(v)) bad += 1.f;
      mn[a] = fminf(mn[a], v);
      mx[a] = fmaxf(mx[a], v);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ float sm[kBoxThreads / 32][8];
  int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) {
    for (int a = 0; a < 3; ++a) { sm[w][a] = mn[a]; sm[w][3 + a] = mx[a]; }
    sm[w][6] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float r[7] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.f};
    for (int k = 0; k < (int)(blockDim.x / 32); ++k) {
      for (int a = 0; a < 3; ++a) { r[a] = fminf(r[a], sm[k][a]); r[3 + a] = fmaxf(r[3 + a], sm[k][3 + a]); }
      r[6] += sm[k][6];
    }
    for (int a = 0; a < 7; ++a) out[8 * blockIdx.x + a] = r[a];
  }
}

// ---------------------------------------------------------------- keys ------
// cell_a = clamp(floor(f32(f32(x_a - lo_a) * inv_h)), 0, dim_a - 1); explicit
// __fsub_rn/__fmul_rn forbid contraction into an FMA (bit-exactness).
__global__ void keys_kernel(const float* __restrict__ xyz, int64_t n, CellGrid g,
                            uint32_t* __restrict__ keys, int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float t = __fmul_rn(__fsub_rn(xyz[3 * i + a], g.lo[a]), g.inv_h);
      float f = floorf(t);
      int q = f < 0.f ? 0 : (f > (float)(g.dim[a] - 1) ? g.dim[a] - 1 : (int)f);
      c[a] = q;
    }
    keys[i] = (uint32_t)c[0] + (uint32_t)g.dim[0] * ((uint32_t)c[1] + (uint32_t)g.dim[1] * (uint32_t)c[2]);
    idx[i] = (int32_t)i;
  }
}

// ---------------------------------------------------------- radix sort ------
// LSD radix sort, 8-bit digits, stable per pass.  Per pass: tile histograms
// -> exclusive scan of the digit-major [digit][tile] table -> stable scatter
// (per-warp ranking with __match_any_sync, warps own contiguous sub-ranges).
constexpr int kRsThreads = 256;
constexpr int kRsIpt = 16;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsTile = kRsThreads * kRsIpt;  // 4096

template <class K>
__global__ void radix_hist(const K* __restrict__ keys, int64_t n, int shift,
                           uint32_t* __restrict__ counts, int ntiles) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kRsTile;
#pragma unroll 4
  for (int r = 0; r < kRsIpt; ++r) {
    int64_t i = base + r * kRsThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(unsigned)(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) counts[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

template <class K>
__global__ void radix_scatter(const K* __restrict__ kin, const int32_t* __restrict__ vin,
                              K* __restrict__ kout, int32_t* __restrict__ vout, int64_t n,
                              int shift, const uint32_t* __restrict__ offsets, int ntiles) {
  __shared__ uint32_t wh[kRsWarps][257];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < kRsWarps * 257; i += blockDim.x) (&wh[0][0])[i] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * kRsTile + (int64_t)w * (32 * kRsIpt);
  const unsigned lt = (1u << lane) - 1u;
  K k[kRsIpt];
  int32_t v[kRsIpt];
#pragma unroll
  for (int r = 0; r < kRsIpt; ++r) {
    int64_t i = wbase + r * 32 + lane;
    bool valid = i < n;
    k[r] = valid ? kin[i] : (K)0;
    v[r] = valid ? vin[i] : 0;
  }
#pragma unroll
  for (int r = 0; r < kRsIpt; ++r) {
    int64_t i = wbase + r * 32 + lane;
    bool valid = i < n;
    unsigned d = valid ? ((unsigned)(k[r] >> shift) & 255u) : 256u;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    if (valid && (peers & lt) == 0u) wh[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    uint32_t run = offsets[(int64_t)d * ntiles + blockIdx.x];
    for (int q = 0; q < kRsWarps; ++q) {
      uint32_t t = wh[q][d];
      wh[q][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsIpt; ++r) {
    int64_t i = wbase + r * 32 + lane;
    bool valid = i < n;
    unsigned d = valid ? ((unsigned)(k[r] >> shift) & 255u) : 256u;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    if (valid) {
      uint32_t rank = wh[w][d] + __popc(peers & lt);
      kout[rank] = k[r];
      vout[rank] = v[r];
    }
    __syncwarp();
    if (valid && (peers & lt) == 0u) wh[w][d] += __popc(peers);
    __syncwarp();
  }
}

// ------------------------------------------------------------ scan ----------
constexpr int kScanThreads = 256;
constexpr int kScanIpt = 8;
constexpr int kScanTile = kScanThreads * kScanIpt;

__global__ void scan_tiles(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int64_t n,
                           uint32_t* __restrict__ sums) {
  __shared__ uint32_t ws[kScanThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIpt;
  uint32_t v[kScanIpt];
  uint32_t s = 0;
#pragma unroll
  for (int r = 0; r < kScanIpt; ++r) {
    int64_t i = base + r;
    v[r] = i < n ? in[i] : 0u;
    s += v[r];
  }
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t x = lane < kScanThreads / 32 ? ws[lane] : 0u;
    uint32_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    if (lane < kScanThreads / 32) ws[lane] = xi - x;
    if (lane == kScanThreads / 32 - 1 && sums) sums[blockIdx.x] = xi;
  }
  __syncthreads();
  uint32_t run = ws[w] + incl - s;
#pragma unroll
  for (int r = 0; r < kScanIpt; ++r) {
    int64_t i = base + r;
    if (i < n) out[i] = run;
    run += v[r];
  }
}

__global__ void scan_add(uint32_t* __restrict__ out, int64_t n, const uint32_t* __restrict__ off) {
  const int64_t i0 = (int64_t)blockIdx.x * kScanTile;
  const uint32_t a = off[blockIdx.x];
  for (int64_t i = i0 + threadIdx.x; i < i0 + kScanTile && i < n; i += blockDim.x) out[i] += a;
}

__global__ void scan_total(const uint32_t* in, const uint32_t* ex, int64_t n, uint32_t* total) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *total = n > 0 ? ex[n - 1] + in[n - 1] : 0u;
}

// ------------------------------------------------------- cell offsets -------
// cell_start[k] = first sorted position whose key >= k  (numpy searchsorted 'left').
__global__ void cell_start_kernel(const uint32_t* __restrict__ skeys, int64_t n, int64_t ncell,
                                  int32_t* __restrict__ start, unsigned long long* __restrict__ nonempty) {
  unsigned long long cnt = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t klo = (i == 0) ? 0 : (int64_t)skeys[i - 1] + 1;
    int64_t khi = (i == n) ? ncell : (int64_t)skeys[i];
    for (int64_t k = klo; k <= khi; ++k) start[k] = (int32_t)i;
    if (i < n && (i == 0 || skeys[i] != skeys[i - 1])) ++cnt;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nonempty, cnt);
}

__global__ void gather_sorted(const float* __restrict__ xyz, const int32_t* __restrict__ perm, int64_t n,
                              float4* __restrict__ sorted) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = perm[i];
    sorted[i] = make_float4(xyz[3 * p], xyz[3 * p + 1], xyz[3 * p + 2], 0.f);
  }
}

// ------------------------------------------------------------ tiles ---------
// Per cell row (fixed y,z); tiles never cross rows, so a tile's targets are a
// contiguous sorted range.
//  mode 0 (runs, default): a run of adjacent non-empty cells along x is cut into
//    chunks of exactly `cap` targets (a chunk may straddle a cell face); a chunk
//    is closed early at a gap (empty cell) or when it would span `span` cells.
//    Full chunks keep both target slots of every lane busy.
//  mode 1 (cells): consecutive non-empty cells are merged while the tile holds
//    <= cap targets and spans < span cells; big cells are cut into cap chunks.
template <bool kEmit>
__device__ int64_t plan_row(const int32_t* __restrict__ start, int dimx, int64_t rowbase, int cap,
                            int span, int mode, int2* __restrict__ out) {
  int64_t cnt = 0;
  int cur_s = 0, cur_n = 0, cur_x0 = 0;
  auto emit = [&](int s, int m) {
    if (kEmit) out[cnt] = make_int2(s, m);
    ++cnt;
  };
  if (mode == 0) {
    int last_x = -2;
    for (int x = 0; x < dimx; ++x) {
      const int s = start[rowbase + x];
      const int m = start[rowbase + x + 1] - s;
      if (m == 0) continue;
      if (cur_n > 0 && (x != last_x + 1 || x - cur_x0 >= span)) {
        emit(cur_s, cur_n);
        cur_n = 0;
      }
      int off = 0;
      while (off < m) {
        if (cur_n == 0) { cur_s = s + off; cur_x0 = x; }
        const int take = min(cap - cur_n, m - off);
        cur_n += take;
        off += take;
        if (cur_n == cap) { emit(cur_s, cur_n); cur_n = 0; }
      }
      last_x = x;
    }
    if (cur_n > 0) emit(cur_s, cur_n);
    return cnt;
  }
  for (int x = 0; x < dimx; ++x) {
    int s = start[rowbase + x];
    int m = start[rowbase + x + 1] - s;
    if (m == 0) continue;
    if (cur_n > 0 && (cur_n + m > cap || x - cur_x0 >= span)) {
      emit(cur_s, cur_n);
      cur_n = 0;
    }
    if (cur_n == 0) {
      int full = m / cap;
      for (int f = 0; f < full; ++f) emit(s + f * cap, cap);
      int rem = m - full * cap;
      if (rem > 0) { cur_s = s + full * cap; cur_n = rem; cur_x0 = x; }
    } else {
      cur_n += m;
    }
  }
  if (cur_n > 0) emit(cur_s, cur_n);
  return cnt;
}

__global__ void plan_count(const int32_t* __restrict__ start, CellGrid g, int cap, int span, int mode,
                           uint32_t* __restrict__ row_counts) {
  int64_t rows = (int64_t)g.dim[1] * g.dim[2];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    row_counts[r] = (uint32_t)plan_row<false>(start, g.dim[0], r * g.dim[0], cap, span, mode, nullptr);
}

__global__ void plan_emit(const int32_t* __restrict__ start, CellGrid g, int cap, int span, int mode,
                          const uint32_t* __restrict__ row_off, int2* __restrict__ tiles) {
  int64_t rows = (int64_t)g.dim[1] * g.dim[2];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    plan_row<true>(start, g.dim[0], r * g.dim[0], cap, span, mode, tiles + row_off[r]);
}

// One warp per tile: axis-aligned bounding box of its targets.
__global__ void tile_box_kernel(const float4* __restrict__ sorted, const int2* __restrict__ tiles,
                                int64_t ntiles, float4* __restrict__ box) {
  const int lane = threadIdx.x % 32;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; t < ntiles; t += nw) {
    int2 tl = tiles[t];
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int j = lane; j < tl.y; j += 32) {
      float4 p = sorted[tl.x + j];
      mn[0] = fminf(mn[0], p.x); mn[1] = fminf(mn[1], p.y); mn[2] = fminf(mn[2], p.z);
      mx[0] = fmaxf(mx[0], p.x); mx[1] = fmaxf(mx[1], p.y); mx[2] = fmaxf(mx[2], p.z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
        mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
      }
    if (lane == 0) {
      box[2 * t] = make_float4(mn[0], mn[1], mn[2], 0.f);
      box[2 * t + 1] = make_float4(mx[0], mx[1], mx[2], 0.f);
    }
  }
}

}  // namespace

rbf_status exclusive_scan_u32(rbf_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n,
                              uint32_t* total_dev) {
  cudaStream_t s = ctx->stream;
  if (n <= 0) {
    if (total_dev) RBF_CUDA_TRY(cudaMemsetAsync(total_dev, 0, sizeof(uint32_t), s));
    return RBF_OK;
  }
  int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb > INT32_MAX) { set_error("scan too large"); return RBF_EINVAL; }
  if (nb == 1) {
    scan_tiles<<<1, kScanThreads, 0, s>>>(in, out, n, nullptr);
    RBF_CHECK_LAUNCH();
  } else {
    DevBuf sums, sums_ex;
    RBF_TRY(sums.alloc(nb * sizeof(uint32_t), s));
    RBF_TRY(sums_ex.alloc(nb * sizeof(uint32_t), s));
    scan_tiles<<<(unsigned)nb, kScanThreads, 0, s>>>(in, out, n, sums.as<uint32_t>());
    RBF_CHECK_LAUNCH();
    RBF_TRY(exclusive_scan_u32(ctx, sums.as<uint32_t>(), sums_ex.as<uint32_t>(), nb, nullptr));
    scan_add<<<(unsigned)nb, kScanThreads, 0, s>>>(out, n, sums_ex.as<uint32_t>());
    RBF_CHECK_LAUNCH();
  }
  if (total_dev) {
    scan_total<<<1, 32, 0, s>>>(in, out, n, total_dev);
    RBF_CHECK_LAUNCH();
  }
  return RBF_OK;
}

template <class K>
rbf_status radix_sort_pairs(rbf_ctx* ctx, K* keys, int32_t* vals, K* keys_out, int32_t* vals_out, int64_t n,
                            int bits) {
  cudaStream_t s = ctx->stream;
  if (n <= 0) return RBF_OK;
  const int passes = std::max(1, (bits + 7) / 8);
  const int64_t nt = (n + kRsTile - 1) / kRsTile;
  DevBuf counts, offs;
  RBF_TRY(counts.alloc(sizeof(uint32_t) * 256 * nt, s));
  RBF_TRY(offs.alloc(sizeof(uint32_t) * 256 * nt, s));
  K* kin = keys;
  int32_t* vin = vals;
  K* kout = keys_out;
  int32_t* vout = vals_out;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    radix_hist<K><<<(unsigned)nt, kRsThreads, 0, s>>>(kin, n, shift, counts.as<uint32_t>(), (int)nt);
    RBF_CHECK_LAUNCH();
    RBF_TRY(exclusive_scan_u32(ctx, counts.as<uint32_t>(), offs.as<uint32_t>(), 256 * nt, nullptr));
    radix_scatter<K><<<(unsigned)nt, kRsThreads, 0, s>>>(kin, vin, kout, vout, n, shift, offs.as<uint32_t>(),
                                                          (int)nt);
    RBF_CHECK_LAUNCH();
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  if (kin != keys_out) {
    RBF_CUDA_TRY(cudaMemcpyAsync(keys_out, kin, sizeof(K) * n, cudaMemcpyDeviceToDevice, s));
    RBF_CUDA_TRY(cudaMemcpyAsync(vals_out, vin, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  }
  return RBF_OK;
}
template rbf_status radix_sort_pairs<uint32_t>(rbf_ctx*, uint32_t*, int32_t*, uint32_t*, int32_t*, int64_t, int);
template rbf_status radix_sort_pairs<unsigned long long>(rbf_ctx*, unsigned long long*, int32_t*,
                                                         unsigned long long*, int32_t*, int64_t, int);

rbf_status build_cells(rbf_ctx* ctx, const float* xyz, int64_t n, const rbf_kernel* k,
                       const rbf_cell_cfg* cfg, rbf_cells* c) {
  cudaStream_t s = ctx->stream;
  const double cutoff = k->cutoff_sigmas * k->sigma;
  double h = (cfg && cfg->cell_edge > 0) ? cfg->cell_edge : cutoff / 3.999;
  int cap = (cfg && cfg->tile_cap > 0) ? cfg->tile_cap : 64;
  int span = (cfg && cfg->tile_span > 0) ? cfg->tile_span : 2;
  const int mode = cfg ? cfg->tile_mode : 0;
  if (mode != 0 && mode != 1) { set_error("tile_mode must be 0 or 1"); return RBF_EINVAL; }
  if (cap != 32 && cap != 64) { set_error("tile_cap must be 32 or 64"); return RBF_EINVAL; }
  c->n = n;
  c->stream = s;
  c->h = h;
  c->cutoff = cutoff;
  c->tile_cap = cap;
  c->tile_span = span;

  // bounding box (+ non-finite check)
  const int nbb = grid_for(n, kBoxThreads, 1024);
  DevBuf bb;
  RBF_TRY(bb.alloc(sizeof(float) * 8 * nbb, s));
  bbox_kernel<<<nbb, kBoxThreads, 0, s>>>(xyz, n, bb.as<float>());
  RBF_CHECK_LAUNCH();
  std::vector<float> hb(8 * (size_t)nbb);
  RBF_CUDA_TRY(cudaMemcpyAsync(hb.data(), bb.p, hb.size() * sizeof(float), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  double bad = 0;
  for (int b = 0; b < nbb; ++b) {
    for (int a = 0; a < 3; ++a) { mn[a] = std::min(mn[a], hb[8 * b + a]); mx[a] = std::max(mx[a], hb[8 * b + 3 + a]); }
    bad += hb[8 * b + 6];
  }
  if (bad > 0) { set_error("non-finite coordinates in xyz"); return RBF_EINVAL; }

  // frame: lo = f32(f64(min) - h/2), inv_h = f32(1/h), dim = floor(f32(f32(max-lo)*inv_h)) + 1
  volatile float inv_h = (float)(1.0 / h);
  int64_t ncell = 1;
  for (int a = 0; a < 3; ++a) {
    volatile float lo = (float)((double)mn[a] - 0.5 * h);
    volatile float d = mx[a] - lo;
    volatile float q = d * inv_h;
    double dimd = std::floor((double)q) + 1.0;
    if (!(dimd >= 1.0) || dimd > 2.0e9) { set_error("cell grid too large"); return RBF_EINVAL; }
    c->lo[a] = lo;
    c->dim[a] = (int)dimd;
    ncell *= (int64_t)dimd;
  }
  c->inv_h = inv_h;
  if (ncell > (int64_t)1 << 31) {
    set_error("too many cells (" + std::to_string(ncell) + "); increase cell_edge");
    return RBF_EINVAL;
  }
  c->ncell = ncell;
  {
    int dmax = std::max(c->dim[0], std::max(c->dim[1], c->dim[2]));
    double margin = h * (dmax + 2) * 4.8e-7;
    c->reach = (int)std::ceil((cutoff * (1 + 1e-5) + margin) / h);
  }
  CellGrid g;
  for (int a = 0; a < 3; ++a) { g.lo[a] = c->lo[a]; g.dim[a] = c->dim[a]; }
  g.inv_h = c->inv_h;
  g.h = (float)h;

  // keys + radix sort
  RBF_TRY(c->keys.alloc(sizeof(uint32_t) * n, s));
  RBF_TRY(c->perm.alloc(sizeof(int32_t) * n, s));
  DevBuf k2, v2;
  RBF_TRY(k2.alloc(sizeof(uint32_t) * n, s));
  RBF_TRY(v2.alloc(sizeof(int32_t) * n, s));
  keys_kernel<<<grid_for(n, 256), 256, 0, s>>>(xyz, n, g, k2.as<uint32_t>(), v2.as<int32_t>());
  RBF_CHECK_LAUNCH();
  int bits = 1;
  while (bits < 32 && ((uint64_t)1 << bits) < (uint64_t)ncell) ++bits;
  RBF_TRY(radix_sort_pairs(ctx, k2.as<uint32_t>(), v2.as<int32_t>(), c->keys.as<uint32_t>(),
                           c->perm.as<int32_t>(), n, bits));

  // cell offsets
  RBF_TRY(c->cell_start.alloc(sizeof(int32_t) * (ncell + 1), s));
  RBF_TRY(ctx->stats.ensure(64, s));
  RBF_CUDA_TRY(cudaMemsetAsync(ctx->stats.p, 0, 8, s));
  cell_start_kernel<<<grid_for(n + 1, 256), 256, 0, s>>>(c->keys.as<uint32_t>(), n, ncell,
                                                         c->cell_start.as<int32_t>(),
                                                         ctx->stats.as<unsigned long long>());
  RBF_CHECK_LAUNCH();
  RBF_TRY(c->sorted.alloc(sizeof(float4) * n, s));
  gather_sorted<<<grid_for(n, 256), 256, 0, s>>>(xyz, c->perm.as<int32_t>(), n, c->sorted.as<float4>());
  RBF_CHECK_LAUNCH();

  // tile plan
  const int64_t rows = (int64_t)g.dim[1] * g.dim[2];
  DevBuf rc, ro, tot;
  RBF_TRY(rc.alloc(sizeof(uint32_t) * rows, s));
  RBF_TRY(ro.alloc(sizeof(uint32_t) * rows, s));
  RBF_TRY(tot.alloc(sizeof(uint32_t) * 2, s));
  plan_count<<<grid_for(rows, 128), 128, 0, s>>>(c->cell_start.as<int32_t>(), g, cap, span, mode,
                                                 rc.as<uint32_t>());
  RBF_CHECK_LAUNCH();
  RBF_TRY(exclusive_scan_u32(ctx, rc.as<uint32_t>(), ro.as<uint32_t>(), rows, tot.as<uint32_t>()));
  uint32_t ntiles = 0;
  unsigned long long nonempty = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&ntiles, tot.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(&nonempty, ctx->stats.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  c->ntiles = ntiles;
  c->nonempty = (int64_t)nonempty;
  RBF_TRY(c->tiles.alloc(sizeof(int2) * (size_t)std::max<uint32_t>(ntiles, 1), s));
  RBF_TRY(c->tile_box.alloc(sizeof(float4) * 2 * (size_t)std::max<uint32_t>(ntiles, 1), s));
  plan_emit<<<grid_for(rows, 128), 128, 0, s>>>(c->cell_start.as<int32_t>(), g, cap, span, mode,
                                                ro.as<uint32_t>(), c->tiles.as<int2>());
  RBF_CHECK_LAUNCH();
  if (ntiles > 0) {
    tile_box_kernel<<<grid_for((int64_t)ntiles * 32, 256), 256, 0, s>>>(
        c->sorted.as<float4>(), c->tiles.as<int2>(), ntiles, c->tile_box.as<float4>());
    RBF_CHECK_LAUNCH();
  }
  // wide plan of the symmetric fp32 matvec: chunks of <= 128 targets of a run of
  // <= 4 cells (reading R19)
  DevBuf rcw, row_w, totw;
  RBF_TRY(rcw.alloc(sizeof(uint32_t) * rows, s));
  RBF_TRY(row_w.alloc(sizeof(uint32_t) * rows, s));
  RBF_TRY(totw.alloc(sizeof(uint32_t) * 2, s));
#ifndef RBF_WIDE_CAP
#define RBF_WIDE_CAP 128
#endif
#ifndef RBF_WIDE_SPAN
#define RBF_WIDE_SPAN 4
#endif
  const int cap_w = RBF_WIDE_CAP;
  const int span_w = std::max(span, RBF_WIDE_SPAN);
  plan_count<<<grid_for(rows, 128), 128, 0, s>>>(c->cell_start.as<int32_t>(), g, cap_w, span_w, 0,
                                                 rcw.as<uint32_t>());
  RBF_CHECK_LAUNCH();
  RBF_TRY(exclusive_scan_u32(ctx, rcw.as<uint32_t>(), row_w.as<uint32_t>(), rows, totw.as<uint32_t>()));
  uint32_t ntiles_w = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&ntiles_w, totw.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  c->ntiles_w = ntiles_w;
  c->hd2 = 0.25 * h * h * ((double)span * span + 2.0);
  c->hd2_w = 0.25 * h * h * ((double)span_w * span_w + 2.0);
  RBF_TRY(c->tiles_w.alloc(sizeof(int2) * (size_t)std::max<uint32_t>(ntiles_w, 1), s));
  RBF_TRY(c->tile_box_w.alloc(sizeof(float4) * 2 * (size_t)std::max<uint32_t>(ntiles_w, 1), s));
  plan_emit<<<grid_for(rows, 128), 128, 0, s>>>(c->cell_start.as<int32_t>(), g, cap_w, span_w, 0,
                                                row_w.as<uint32_t>(), c->tiles_w.as<int2>());
  RBF_CHECK_LAUNCH();
  if (ntiles_w > 0) {
    tile_box_kernel<<<grid_for((int64_t)ntiles_w * 32, 256), 256, 0, s>>>(
        c->sorted.as<float4>(), c->tiles_w.as<int2>(), ntiles_w, c->tile_box_w.as<float4>());
    RBF_CHECK_LAUNCH();
  }
  // this rank's share (dist.cu): everything on one GPU, a slab of z planes otherwise
  c->world = ctx->world;
  c->view = SlabView{0, n, 0, n, 0, (int64_t)ntiles, 0, c->dim[2], 0, (int64_t)ntiles_w};
  if (ctx->world > 1) {
    std::vector<uint32_t> hro(rows), hrow(rows);
    RBF_CUDA_TRY(cudaMemcpyAsync(hro.data(), ro.p, sizeof(uint32_t) * rows, cudaMemcpyDeviceToHost, s));
    RBF_CUDA_TRY(cudaMemcpyAsync(hrow.data(), row_w.p, sizeof(uint32_t) * rows, cudaMemcpyDeviceToHost, s));
    RBF_CUDA_TRY(cudaStreamSynchronize(s));
    RBF_TRY(dist_plan_cells(ctx, c, hro, (int64_t)ntiles, hrow, (int64_t)ntiles_w, ctx->rank, ctx->world));
  }
  RBF_TRY(order_wide_tiles(ctx, c, kernel_params(k)));
  return RBF_OK;
}

}  // namespace rbf
