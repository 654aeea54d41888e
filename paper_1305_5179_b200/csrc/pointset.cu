// Point-set geometry on the GPU: SURVEY.md §8(f) item 1 (the masked zero set
// of the interpolant on the grid) and item 2 (density measures, Eq.7-11).
//
// ---- zero set ----
// §2.1.3: the surface is the zero level set of P_f restricted to the
// eps-surrounding of the data, M* ~ M_ext^eps cap S_0 ("undesired artifacts"
// far from the data are cut away).  Reading R11: linear
// interpolation along grid edges whose endpoint values have strictly opposite
// signs, keeping only edges whose BOTH endpoints lie within eps of a data point.
//
// GPU steps (all fp64 where the oracle decides: node coordinates lo + i*step,
// distances ((dx^2 + dy^2) + dz^2), sqrt(d2) <= eps, F_a * F_b < 0 on the fp32
// field promoted to fp64, t = F_a / (F_a - F_b)), so the output equals
// oracle/grid.py::zero_crossings on the same field point for point:
//   1. near[node] = some data point within eps, scattered from the points (one
//      thread per point tests the nodes of its eps box exactly);
//   2. per axis x, y, z: flag the edges, exclusive scan, write the crossing
//      points in (axis, lower-node flat index) order -- the oracle's order.
// Work: ~(2 eps / step + 3)^3 exact distance tests per data point for the mask
// (c4: 1M points, ~1.2e8 tests), three HBM passes over the field.
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

namespace rbf {
namespace {

struct ZGrid {
  double lo[3], step[3];
  int n[3];
};
struct DCells {
  double lo[3];
  double inv_h;
  int dim[3];
};

}  // namespace
// bounding box of n fp64 points on the device (RBF_EINVAL on a non-finite one)
rbf_status data_bbox(rbf_ctx* ctx, const double* X, int64_t n, double mn[3], double mx[3]);
namespace {

// no contraction: the oracle forms lo + (i * step) with two roundings
__device__ __forceinline__ double zcoord(const ZGrid& g, int a, int i) {
  return __dadd_rn(g.lo[a], __dmul_rn((double)i, g.step[a]));
}

__device__ __forceinline__ int dcell(double x, double lo, double inv_h, int dim) {
  double t = floor((x - lo) * inv_h);
  t = fmin(fmax(t, -1.0), (double)dim);
  return (int)t;   // may be -1 or dim (outside): callers clip the neighbourhood
}

__global__ void data_keys_kernel(const double* __restrict__ X, int64_t n, DCells dc, uint32_t* __restrict__ key,
                                 int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = min(max(dcell(X[3 * i + a], dc.lo[a], dc.inv_h, dc.dim[a]), 0), dc.dim[a] - 1);
    key[i] = (uint32_t)(c[0] + dc.dim[0] * (c[1] + dc.dim[1] * c[2]));
    idx[i] = (int32_t)i;
  }
}

__global__ void data_start_kernel(const uint32_t* __restrict__ skeys, int64_t n, int64_t ncell,
                                  int32_t* __restrict__ start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t klo = (i == 0) ? 0 : (int64_t)skeys[i - 1] + 1;
    const int64_t khi = (i == n) ? ncell : (int64_t)skeys[i];
    for (int64_t k = klo; k <= khi; ++k) start[k] = (int32_t)i;
  }
}

__global__ void data_gather_kernel(const double* __restrict__ X, const int32_t* __restrict__ perm, int64_t n,
                                   double* __restrict__ S) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = perm[i];
    S[3 * i] = X[3 * j];
    S[3 * i + 1] = X[3 * j + 1];
    S[3 * i + 2] = X[3 * j + 2];
  }
}

// near[node] = 1 for every grid node within eps of data point i, scattered from
// the points: one thread per point tests the nodes of the box [x_i - eps,
// x_i + eps] (widened by one node per side against the rounding of the index
// range) with the oracle's arithmetic, sqrt_rn(((dx^2 + dy^2) + dz^2)) <= eps
// on the fp64 node coordinates lo + i * step.  Every (node, point) pair within
// eps is tested exactly once, so near[] is the oracle's mask bit for bit (the
// stores are idempotent: racing threads write the same 1).
__global__ void near_scatter_kernel(ZGrid g, const double* __restrict__ X, int64_t n, double eps,
                                    uint8_t* __restrict__ near) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x[3] = {X[3 * i], X[3 * i + 1], X[3 * i + 2]};
    int lo[3], hi[3];
    bool none = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = max((int)floor((x[a] - eps - g.lo[a]) / g.step[a]) - 1, 0);
      hi[a] = min((int)ceil((x[a] + eps - g.lo[a]) / g.step[a]) + 1, g.n[a] - 1);
      if (lo[a] > hi[a]) none = true;
    }
    if (none) continue;
    for (int k = lo[2]; k <= hi[2]; ++k) {
      const double dz = __dsub_rn(zcoord(g, 2, k), x[2]);
      const double dz2 = __dmul_rn(dz, dz);
      for (int jj = lo[1]; jj <= hi[1]; ++jj) {
        const double dy = __dsub_rn(zcoord(g, 1, jj), x[1]);
        const double dy2 = __dmul_rn(dy, dy);
        const int64_t row = ((int64_t)k * g.n[1] + jj) * g.n[0];
        for (int ii = lo[0]; ii <= hi[0]; ++ii) {
          const double dx = __dsub_rn(zcoord(g, 0, ii), x[0]);
          const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), dy2), dz2);
          if (__dsqrt_rn(d2) <= eps) near[row + ii] = 1;
        }
      }
    }
  }
}

// edge (v, v + stride along axis a) has a masked crossing
__device__ __forceinline__ bool edge_cross(const float* __restrict__ F, const uint8_t* __restrict__ near, const ZGrid& g,
                                           int a, int64_t v, int64_t stride) {
  const int64_t q[3] = {v % g.n[0], (v / g.n[0]) % g.n[1], v / ((int64_t)g.n[0] * g.n[1])};
  if (q[a] + 1 >= g.n[a]) return false;
  const int64_t u = v + stride;
  const double fa = (double)F[v], fb = (double)F[u];
  return (fa * fb < 0.0) && near[v] && near[u];
}

__global__ void edge_flag_kernel(const float* __restrict__ F, const uint8_t* __restrict__ near, ZGrid g, int a,
                                 int64_t stride, uint32_t* __restrict__ flag) {
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x)
    flag[v] = edge_cross(F, near, g, a, v, stride) ? 1u : 0u;
}

__global__ void edge_emit_kernel(const float* __restrict__ F, const uint8_t* __restrict__ near, ZGrid g, int a,
                                 int64_t stride, const uint32_t* __restrict__ pos, int64_t base, int64_t cap,
                                 double* __restrict__ out) {
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    if (!edge_cross(F, near, g, a, v, stride)) continue;
    const int64_t o = base + pos[v];
    if (o >= cap) continue;
    const int64_t u = v + stride;
    const double fa = (double)F[v], fb = (double)F[u];
    const double t = fa / (fa - fb);
    const int64_t qa[3] = {v % g.n[0], (v / g.n[0]) % g.n[1], v / ((int64_t)g.n[0] * g.n[1])};
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double pa = zcoord(g, b, (int)qa[b]);
      const double pb = zcoord(g, b, (int)qa[b] + (b == a ? 1 : 0));
      out[3 * o + b] = __dadd_rn(pa, __dmul_rn(t, __dsub_rn(pb, pa)));
    }
  }
}

}  // namespace
}  // namespace rbf

using namespace rbf;

namespace rbf {
// near[v] (uint8, one per grid node) = some data point within eps of node v
// (fp64 distances; steps 1-2 above).  ndata == 0: all zeros.
rbf_status build_near_mask(rbf_ctx* ctx, const rbf_grid* grid, const double* data, int64_t ndata, double eps,
                           DevBuf& near) {
  cudaStream_t s = ctx->stream;
  ZGrid g;
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = grid->lo[a];
    g.step[a] = (grid->hi[a] - grid->lo[a]) / (double)(grid->n[a] - 1);
    g.n[a] = grid->n[a];
  }
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  RBF_TRY(near.alloc(nn, s));
  RBF_CUDA_TRY(cudaMemsetAsync(near.p, 0, nn, s));
  if (ndata == 0) return RBF_OK;
  double mn[3], mx[3];
  RBF_TRY(data_bbox(ctx, data, ndata, mn, mx));   // rejects non-finite points
  near_scatter_kernel<<<grid_for(ndata, 256, 148 * 32), 256, 0, s>>>(g, data, ndata, eps, near.as<uint8_t>());
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}
}  // namespace rbf

extern "C" rbf_status rbf_zero_set(rbf_ctx* ctx, const float* field, const rbf_grid* grid, const double* data,
                                   int64_t ndata, double eps, double* points, int64_t cap, int64_t* count) {
  RBF_NVTX("rbf_zero_set");
  if (!ctx || !field || !grid || !count) { set_error("NULL argument"); return RBF_EINVAL; }
  if (ndata < 0 || (ndata > 0 && !data) || cap < 0 || (cap > 0 && !points)) { set_error("bad data/points"); return RBF_EINVAL; }
  if (!(eps > 0) || !std::isfinite(eps)) { set_error("eps must be finite and > 0"); return RBF_EINVAL; }
  for (int a = 0; a < 3; ++a)
    if (grid->n[a] < 2 || !(grid->hi[a] > grid->lo[a])) { set_error("bad grid"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  *count = 0;
  if (ndata == 0) return RBF_OK;   // no data: the eps-surrounding is empty
  ZGrid g;
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = grid->lo[a];
    g.step[a] = (grid->hi[a] - grid->lo[a]) / (double)(grid->n[a] - 1);
    g.n[a] = grid->n[a];
  }
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  DevBuf near, flag, pos, tot;
  RBF_TRY(build_near_mask(ctx, grid, data, ndata, eps, near));
  // 3. crossings per axis, in the oracle's (axis, lower node) order
  RBF_TRY(flag.alloc(4 * nn, s));
  RBF_TRY(pos.alloc(4 * nn, s));
  RBF_TRY(tot.alloc(8, s));
  const int64_t strides[3] = {1, g.n[0], (int64_t)g.n[0] * g.n[1]};
  int64_t base = 0;
  for (int a = 0; a < 3; ++a) {
    edge_flag_kernel<<<grid_for(nn, 256), 256, 0, s>>>(field, near.as<uint8_t>(), g, a, strides[a],
                                                        flag.as<uint32_t>());
    RBF_CHECK_LAUNCH();
    RBF_TRY(exclusive_scan_u32(ctx, flag.as<uint32_t>(), pos.as<uint32_t>(), nn, tot.as<uint32_t>()));
    uint32_t na = 0;
    RBF_CUDA_TRY(cudaMemcpyAsync(&na, tot.p, 4, cudaMemcpyDeviceToHost, s));
    RBF_CUDA_TRY(cudaStreamSynchronize(s));
    if (na > 0 && base < cap) {
      edge_emit_kernel<<<grid_for(nn, 256), 256, 0, s>>>(field, near.as<uint8_t>(), g, a, strides[a],
                                                          pos.as<uint32_t>(), base, cap, points);
      RBF_CHECK_LAUNCH();
    }
    base += na;
  }
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  *count = base;
  return RBF_OK;
}

// ---- density measures (§4; Eq.7-11) ---------
//   q_X        = 1/2 min_{i != j} ||x_i - x_j||            (Eq.7, separation distance)
//   h_max      = max_j min_{i != j} ||x_i - x_j||
//   h_{X,Omega}= max_{w in Omega} min_j ||w - x_j||         (Eq.8, fill distance over
//                a caller-supplied discrete sample of Omega)
// Nearest-neighbour distances by an expanding-ring search over a uniform cell
// grid of the data (edge ~ (bbox volume / (n/2))^(1/3)): after the rings up to
// Chebyshev distance R from the query's (unclamped) cell, every unvisited point
// is at least (R - 1) h away, so the search stops once best <= (R - 1) h.
// Distances in fp64 with the oracle's rounding ((dx^2 + dy^2) + dz^2, sqrt of the
// minimum), so every distance equals oracle/density.py's bit for bit.
namespace rbf {
namespace {

__global__ void bbox64_kernel(const double* __restrict__ X, int64_t n, double* __restrict__ part) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double v = X[3 * i + a];
      if (!isfinite(v)) bad = true;
      mn[a] = fmin(mn[a], v);
      mx[a] = fmax(mx[a], v);
    }
  __shared__ double smn[3][256], smx[3][256];
  __shared__ int sbad;
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  if (bad) sbad = 1;
#pragma unroll
  for (int a = 0; a < 3; ++a) { smn[a][threadIdx.x] = mn[a]; smx[a][threadIdx.x] = mx[a]; }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int a = threadIdx.x;
    double lo = INFINITY, hi = -INFINITY;
    for (int t = 0; t < (int)blockDim.x; ++t) { lo = fmin(lo, smn[a][t]); hi = fmax(hi, smx[a][t]); }
    part[7 * blockIdx.x + a] = lo;
    part[7 * blockIdx.x + 3 + a] = hi;
  }
  if (threadIdx.x == 0) part[7 * blockIdx.x + 6] = sbad ? 1.0 : 0.0;
}

// nn[i] = min over data points j (j != self index when exclude) of ||q_i - x_j||
__global__ void nn_kernel(const double* __restrict__ Qp, int64_t m, bool exclude_self, DCells dc,
                          const int32_t* __restrict__ start, const double* __restrict__ S,
                          const int32_t* __restrict__ sorted_id, double h, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double q[3] = {Qp[3 * i], Qp[3 * i + 1], Qp[3 * i + 2]};
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double t = floor((q[a] - dc.lo[a]) * dc.inv_h);
      c[a] = (int)fmin(fmax(t, -1e9), 1e9);
    }
    // rings [r_lo, r_hi] intersect the grid (r_lo > 0 for queries outside it)
    int r_lo = 0, r_hi = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      r_lo = max(r_lo, max(-c[a], c[a] - (dc.dim[a] - 1)));
      r_hi = max(r_hi, max(c[a], dc.dim[a] - 1 - c[a]));
    }
    double best = INFINITY;
    for (int r = r_lo; r <= r_hi; ++r) {
      const int z0 = max(c[2] - r, 0), z1 = min(c[2] + r, dc.dim[2] - 1);
      const int y0 = max(c[1] - r, 0), y1 = min(c[1] + r, dc.dim[1] - 1);
      const int x0 = max(c[0] - r, 0), x1 = min(c[0] + r, dc.dim[0] - 1);
      for (int cz = z0; cz <= z1; ++cz) {
        for (int cy = y0; cy <= y1; ++cy) {
          // cells of the shell max(|dx|, |dy|, |dz|) == r: a whole x row when
          // (cy, cz) is on the shell, else only x = c0 -+ r
          const bool face = (cz == c[2] - r || cz == c[2] + r || cy == c[1] - r || cy == c[1] + r);
          for (int e = 0; e < (face ? x1 - x0 + 1 : 2); ++e) {
            const int cx = face ? x0 + e : (e == 0 ? c[0] - r : c[0] + r);
            if (cx < 0 || cx >= dc.dim[0] || (!face && r == 0)) continue;
            const int64_t k = cx + (int64_t)dc.dim[0] * (cy + (int64_t)dc.dim[1] * cz);
            for (int p = start[k]; p < start[k + 1]; ++p) {
              if (exclude_self && sorted_id[p] == (int32_t)i) continue;
              const double dx = __dsub_rn(q[0], S[3 * p]), dy = __dsub_rn(q[1], S[3 * p + 1]),
                           dz = __dsub_rn(q[2], S[3 * p + 2]);
              const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
              best = fmin(best, d2);
            }
          }
        }
      }
      const double bound = (double)r * h;   // unvisited points are >= r h away after ring r
      if (best <= bound * bound) break;
    }
    out[i] = __dsqrt_rn(best);
  }
}

__global__ void minmax_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ part) {
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    lo = fmin(lo, v[i]);
    hi = fmax(hi, v[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ double sl[32], sh[32];
  if ((threadIdx.x & 31) == 0) { sl[threadIdx.x >> 5] = lo; sh[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { lo = fmin(lo, sl[w]); hi = fmax(hi, sh[w]); }
    lo = fmin(lo, sl[0]);
    hi = fmax(hi, sh[0]);
    part[2 * blockIdx.x] = lo;
    part[2 * blockIdx.x + 1] = hi;
  }
}

rbf_status host_minmax(rbf_ctx* ctx, const double* v, int64_t n, double* lo, double* hi) {
  cudaStream_t s = ctx->stream;
  const int nb = grid_for(n, 256, 1024);
  DevBuf part;
  RBF_TRY(part.alloc(16 * (size_t)nb, s));
  minmax_kernel<<<nb, 256, 0, s>>>(v, n, part.as<double>());
  RBF_CHECK_LAUNCH();
  std::vector<double> hp(2 * (size_t)nb);
  RBF_CUDA_TRY(cudaMemcpyAsync(hp.data(), part.p, 16 * (size_t)nb, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  *lo = INFINITY;
  *hi = -INFINITY;
  for (int b = 0; b < nb; ++b) { *lo = std::min(*lo, hp[2 * b]); *hi = std::max(*hi, hp[2 * b + 1]); }
  return RBF_OK;
}

}  // namespace

// nearest-neighbour distances of Q (or of X itself, self excluded) to X
rbf_status nn_distances(rbf_ctx* ctx, const double* X, int64_t n, const double* Q, int64_t m, double* out) {
  cudaStream_t s = ctx->stream;
  const int nbb = grid_for(n, 256, 1024);
  DevBuf part;
  RBF_TRY(part.alloc(sizeof(double) * 7 * nbb, s));
  bbox64_kernel<<<nbb, 256, 0, s>>>(X, n, part.as<double>());
  RBF_CHECK_LAUNCH();
  std::vector<double> hp(7 * (size_t)nbb);
  RBF_CUDA_TRY(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * 7 * nbb, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int b = 0; b < nbb; ++b) {
    if (hp[7 * b + 6] != 0.0) { set_error("non-finite data point"); return RBF_EINVAL; }
    for (int a = 0; a < 3; ++a) { mn[a] = std::min(mn[a], hp[7 * b + a]); mx[a] = std::max(mx[a], hp[7 * b + 3 + a]); }
  }
  // cell edge: ~2 points per cell of the bounding box (degenerate extents floored)
  double ext = 0.0;
  for (int a = 0; a < 3; ++a) ext = std::max(ext, mx[a] - mn[a]);
  if (!(ext > 0)) ext = 1.0;
  double vol = 1.0;
  for (int a = 0; a < 3; ++a) vol *= std::max(mx[a] - mn[a], ext * 1e-3);
  double h = std::cbrt(vol / std::max<double>(1.0, 0.5 * (double)n));
  DCells dc;
  int64_t ncell = 1;
  for (;;) {
    double prod = 1.0;
    for (int a = 0; a < 3; ++a) prod *= std::floor((mx[a] - (mn[a] - 0.5 * h)) / h) + 1.0;
    if (prod <= (double)((int64_t)1 << 27)) break;
    h *= 1.5;
  }
  for (int a = 0; a < 3; ++a) {
    dc.lo[a] = mn[a] - 0.5 * h;
    dc.dim[a] = (int)std::floor((mx[a] - dc.lo[a]) / h) + 1;
    ncell *= dc.dim[a];
  }
  dc.inv_h = 1.0 / h;
  DevBuf k1, v1, k2, v2, start, S;
  RBF_TRY(k1.alloc(4 * n, s));
  RBF_TRY(v1.alloc(4 * n, s));
  RBF_TRY(k2.alloc(4 * n, s));
  RBF_TRY(v2.alloc(4 * n, s));
  data_keys_kernel<<<grid_for(n, 256), 256, 0, s>>>(X, n, dc, k1.as<uint32_t>(), v1.as<int32_t>());
  RBF_CHECK_LAUNCH();
  int bits = 1;
  while (bits < 32 && ((int64_t)1 << bits) < ncell) ++bits;
  RBF_TRY(radix_sort_pairs<uint32_t>(ctx, k1.as<uint32_t>(), v1.as<int32_t>(), k2.as<uint32_t>(), v2.as<int32_t>(), n,
                                     bits));
  RBF_TRY(start.alloc(4 * (ncell + 1), s));
  data_start_kernel<<<grid_for(n + 1, 256), 256, 0, s>>>(k2.as<uint32_t>(), n, ncell, start.as<int32_t>());
  RBF_CHECK_LAUNCH();
  RBF_TRY(S.alloc(sizeof(double) * 3 * n, s));
  data_gather_kernel<<<grid_for(n, 256), 256, 0, s>>>(X, v2.as<int32_t>(), n, S.as<double>());
  RBF_CHECK_LAUNCH();
  const bool self = (Q == nullptr);
  nn_kernel<<<grid_for(self ? n : m, 128, 148 * 64), 128, 0, s>>>(self ? X : Q, self ? n : m, self, dc,
                                                                  start.as<int32_t>(), S.as<double>(),
                                                                  v2.as<int32_t>(), h, out);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}

}  // namespace rbf

extern "C" rbf_status rbf_nn_distance(rbf_ctx* ctx, const double* x, int64_t n, const double* q, int64_t m,
                                      double* dist) {
  if (!ctx || !x || !dist || n < 1 || (q && m < 1)) { set_error("bad arguments"); return RBF_EINVAL; }
  if (!q && n < 2) { set_error("self distances need n >= 2"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  return nn_distances(ctx, x, n, q, m, dist);
}

extern "C" rbf_status rbf_density(rbf_ctx* ctx, const double* x, int64_t n, const double* omega, int64_t m,
                                  double* out6) {
  if (!ctx || !x || !out6 || n < 2 || (omega && m < 1)) { set_error("bad arguments"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  DevBuf d;
  RBF_TRY(d.alloc(sizeof(double) * (size_t)std::max<int64_t>(n, omega ? m : 0), s));
  RBF_TRY(nn_distances(ctx, x, n, nullptr, 0, d.as<double>()));
  double lo, hi;
  RBF_TRY(host_minmax(ctx, d.as<double>(), n, &lo, &hi));
  out6[0] = 0.5 * lo;   // q_X (Eq.7)
  out6[1] = hi;         // h_max
  out6[2] = NAN;
  if (omega) {
    RBF_TRY(nn_distances(ctx, x, n, omega, m, d.as<double>()));
    RBF_TRY(host_minmax(ctx, d.as<double>(), m, &lo, &hi));
    out6[2] = hi;       // h_{X,Omega} (Eq.8)
  }
  out6[3] = 2.0 * out6[0];                  // Eq.9   sigma ~ 2 q_X
  out6[4] = std::sqrt(2.0) * out6[2];       // Eq.10  sigma ~ sqrt(2) h_{X,Omega}
  out6[5] = 2.0 * out6[1];                  // Eq.10 with Eq.11 h ~ sqrt(2) h_max
  return RBF_OK;
}

extern "C" rbf_status rbf_sigma_auto(rbf_ctx* ctx, const double* x, int64_t n, const double* omega, int64_t m,
                                     int rule, double* sigma) {
  if (!sigma) { set_error("sigma is NULL"); return RBF_EINVAL; }
  if (rule != 9 && rule != 10 && rule != 11) { set_error("rule must be 9, 10 or 11 (Eq.9 / Eq.10 / Eq.11)"); return RBF_EINVAL; }
  if (rule == 10 && !omega) { set_error("rule 10 (fill distance, Eq.8) needs omega"); return RBF_EINVAL; }
  double out6[6];
  RBF_TRY(rbf_density(ctx, x, n, rule == 10 ? omega : nullptr, rule == 10 ? m : 0, out6));
  *sigma = out6[rule == 9 ? 3 : (rule == 10 ? 4 : 5)];
  return RBF_OK;
}

namespace rbf {
rbf_status data_bbox(rbf_ctx* ctx, const double* X, int64_t n, double mn[3], double mx[3]) {
  cudaStream_t s = ctx->stream;
  const int nbb = grid_for(n, 256, 148 * 4);
  DevBuf part;
  RBF_TRY(part.alloc(sizeof(double) * 7 * nbb, s));
  bbox64_kernel<<<nbb, 256, 0, s>>>(X, n, part.as<double>());
  RBF_CHECK_LAUNCH();
  std::vector<double> hp(7 * (size_t)nbb);
  RBF_CUDA_TRY(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * 7 * nbb, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  for (int a = 0; a < 3; ++a) { mn[a] = INFINITY; mx[a] = -INFINITY; }
  for (int b = 0; b < nbb; ++b) {
    if (hp[7 * b + 6] != 0.0) { set_error("non-finite data point"); return RBF_EINVAL; }
    for (int a = 0; a < 3; ++a) { mn[a] = std::min(mn[a], hp[7 * b + a]); mx[a] = std::max(mx[a], hp[7 * b + 3 + a]); }
  }
  return RBF_OK;
}
}  // namespace rbf
