// the masked zero set of the interpolant on the grid.
//
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
//   1. the data points are binned into cells of edge >= eps (radix sort + starts);
//   2. near[node] = some data point within eps (27 neighbour cells, early exit);
//   3. per axis x, y, z: flag the edges, exclusive scan, write the crossing
//      points in (axis, lower-node flat index) order -- the oracle's order.
// Work: one pass over the nodes for the mask (bounded by the data points in
// the 27 cells of near-surface nodes), three HBM passes over the field.
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

// near[node] = exists data point p with sqrt(|node - p|^2) <= eps (fp64)
__global__ void near_kernel(ZGrid g, DCells dc, const int32_t* __restrict__ start, const double* __restrict__ S,
                            double eps, uint8_t* __restrict__ near) {
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(v % g.n[0]), j = (int)((v / g.n[0]) % g.n[1]), k = (int)(v / ((int64_t)g.n[0] * g.n[1]));
    const double p[3] = {zcoord(g, 0, i), zcoord(g, 1, j), zcoord(g, 2, k)};
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = dcell(p[a], dc.lo[a], dc.inv_h, dc.dim[a]);
    bool hit = false;
    for (int cz = max(c[2] - 1, 0); cz <= min(c[2] + 1, dc.dim[2] - 1) && !hit; ++cz)
      for (int cy = max(c[1] - 1, 0); cy <= min(c[1] + 1, dc.dim[1] - 1) && !hit; ++cy) {
        const int x0 = max(c[0] - 1, 0), x1 = min(c[0] + 1, dc.dim[0] - 1);
        if (x0 > x1) continue;
        const int64_t row = ((int64_t)cz * dc.dim[1] + cy) * dc.dim[0];
        const int s0 = start[row + x0], s1 = start[row + x1 + 1];
        for (int q = s0; q < s1; ++q) {
          const double dx = __dsub_rn(p[0], S[3 * q]), dy = __dsub_rn(p[1], S[3 * q + 1]),
                       dz = __dsub_rn(p[2], S[3 * q + 2]);
          const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
          if (__dsqrt_rn(d2) <= eps) { hit = true; break; }
        }
      }
    near[v] = hit ? 1 : 0;
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

extern "C" rbf_status rbf_zero_set(rbf_ctx* ctx, const float* field, const rbf_grid* grid, const double* data,
                                   int64_t ndata, double eps, double* points, int64_t cap, int64_t* count) {
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
  // 1. data cells of edge h >= eps over the data bounding box (host bbox via a copy)
  std::vector<double> hx(3 * (size_t)ndata);
  RBF_CUDA_TRY(cudaMemcpyAsync(hx.data(), data, sizeof(double) * 3 * ndata, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < ndata; ++i)
    for (int a = 0; a < 3; ++a) {
      const double v = hx[3 * i + a];
      if (!std::isfinite(v)) { set_error("non-finite data point"); return RBF_EINVAL; }
      mn[a] = std::min(mn[a], v);
      mx[a] = std::max(mx[a], v);
    }
  double h = eps * (1.0 + 1e-6);
  DCells dc;
  int64_t ncell = 1;
  for (;;) {   // coarsen the cells (edge stays >= eps) if the box would need too many
    double prod = 1.0;
    for (int a = 0; a < 3; ++a) prod *= std::floor((mx[a] - (mn[a] - 0.5 * h)) / h) + 1.0;
    if (prod <= (double)((int64_t)1 << 28)) break;
    h *= 2.0;
  }
  for (int a = 0; a < 3; ++a) {
    dc.lo[a] = mn[a] - 0.5 * h;
    dc.dim[a] = (int)std::floor((mx[a] - dc.lo[a]) / h) + 1;
    ncell *= dc.dim[a];
  }
  dc.inv_h = 1.0 / h;
  DevBuf k1, v1, k2, v2, start, S, near, flag, pos, tot;
  RBF_TRY(k1.alloc(4 * ndata, s));
  RBF_TRY(v1.alloc(4 * ndata, s));
  RBF_TRY(k2.alloc(4 * ndata, s));
  RBF_TRY(v2.alloc(4 * ndata, s));
  data_keys_kernel<<<grid_for(ndata, 256), 256, 0, s>>>(data, ndata, dc, k1.as<uint32_t>(), v1.as<int32_t>());
  RBF_CHECK_LAUNCH();
  int bits = 1;
  while (bits < 32 && ((int64_t)1 << bits) < ncell) ++bits;
  RBF_TRY(radix_sort_pairs<uint32_t>(ctx, k1.as<uint32_t>(), v1.as<int32_t>(), k2.as<uint32_t>(), v2.as<int32_t>(),
                                     ndata, bits));
  RBF_TRY(start.alloc(4 * (ncell + 1), s));
  data_start_kernel<<<grid_for(ndata + 1, 256), 256, 0, s>>>(k2.as<uint32_t>(), ndata, ncell, start.as<int32_t>());
  RBF_CHECK_LAUNCH();
  RBF_TRY(S.alloc(sizeof(double) * 3 * ndata, s));
  data_gather_kernel<<<grid_for(ndata, 256), 256, 0, s>>>(data, v2.as<int32_t>(), ndata, S.as<double>());
  RBF_CHECK_LAUNCH();
  // 2. the eps mask
  RBF_TRY(near.alloc(nn, s));
  near_kernel<<<grid_for(nn, 256, 148 * 32), 256, 0, s>>>(g, dc, start.as<int32_t>(), S.as<double>(), eps,
                                                          near.as<uint8_t>());
  RBF_CHECK_LAUNCH();
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
