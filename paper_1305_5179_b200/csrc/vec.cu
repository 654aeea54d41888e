// Permutation gathers/scatters between the caller's order and the internal
// cell (sorted) order.  perm[i] = caller index of sorted position i.
#include <cmath>

#include "internal.h"

namespace rbf {
namespace {

template <class S, class D>
__global__ void gather_kernel(const S* __restrict__ src, const int32_t* __restrict__ perm, D* __restrict__ dst,
                              int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (D)src[perm[i]];
}
template <class S, class D>
__global__ void scatter_kernel(const S* __restrict__ src, const int32_t* __restrict__ perm, D* __restrict__ dst,
                               int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[perm[i]] = (D)src[i];
}

}  // namespace

rbf_status gather_f32_to_sorted(rbf_ctx* ctx, const float* src, const int32_t* perm, float* dst, int64_t n) {
  gather_kernel<float, float><<<grid_for(n, 256), 256, 0, ctx->stream>>>(src, perm, dst, n);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}
rbf_status gather_f64_to_sorted(rbf_ctx* ctx, const double* src, const int32_t* perm, double* dst, int64_t n) {
  gather_kernel<double, double><<<grid_for(n, 256), 256, 0, ctx->stream>>>(src, perm, dst, n);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}
rbf_status gather_f64_to_sorted_f32(rbf_ctx* ctx, const double* src, const int32_t* perm, float* dst, int64_t n) {
  gather_kernel<double, float><<<grid_for(n, 256), 256, 0, ctx->stream>>>(src, perm, dst, n);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}
rbf_status gather_f32_to_sorted_f64(rbf_ctx* ctx, const float* src, const int32_t* perm, double* dst, int64_t n) {
  gather_kernel<float, double><<<grid_for(n, 256), 256, 0, ctx->stream>>>(src, perm, dst, n);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}
rbf_status scatter_f64_from_sorted_f32(rbf_ctx* ctx, const double* src, const int32_t* perm, float* dst, int64_t n) {
  scatter_kernel<double, float><<<grid_for(n, 256), 256, 0, ctx->stream>>>(src, perm, dst, n);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}
rbf_status scatter_f32_from_sorted(rbf_ctx* ctx, const float* src, const int32_t* perm, float* dst, int64_t n) {
  scatter_kernel<float, float><<<grid_for(n, 256), 256, 0, ctx->stream>>>(src, perm, dst, n);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}
rbf_status scatter_f64_from_sorted(rbf_ctx* ctx, const double* src, const int32_t* perm, double* dst, int64_t n) {
  scatter_kernel<double, double><<<grid_for(n, 256), 256, 0, ctx->stream>>>(src, perm, dst, n);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}

}  // namespace rbf

// ---- a0: extended set X_ext = [X; X + delta n; X - delta n] and labels ------
namespace {
__global__ void extend_kernel(const double* __restrict__ x, const double* __restrict__ nrm, int64_t N,
                              double delta, double label, float* __restrict__ centres, float* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double xi = x[3 * i + a];
      const double dn = __dmul_rn(delta, nrm[3 * i + a]);
      centres[3 * i + a] = __double2float_rn(xi);
      centres[3 * (N + i) + a] = __double2float_rn(__dadd_rn(xi, dn));
      centres[3 * (2 * N + i) + a] = __double2float_rn(__dsub_rn(xi, dn));
    }
    if (b) {
      b[i] = 0.f;
      b[N + i] = (float)label;
      b[2 * N + i] = (float)(-label);
    }
  }
}
}  // namespace

extern "C" rbf_status rbf_extend_points(rbf_ctx* ctx, const double* x, const double* nrm, int64_t N, double delta,
                                        double label, float* centres, float* b) {
  if (!ctx || !x || !nrm || !centres) { rbf::set_error("NULL argument"); return RBF_EINVAL; }
  if (N < 1 || N > (int64_t)INT32_MAX / 6) { rbf::set_error("N out of range"); return RBF_EINVAL; }
  if (!std::isfinite(delta) || !std::isfinite(label)) { rbf::set_error("delta/label must be finite"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  extend_kernel<<<rbf::grid_for(N, 256), 256, 0, ctx->stream>>>(x, nrm, N, delta, label, centres, b);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}
