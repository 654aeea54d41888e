// a6/a7 of SURVEY.md §8(a): restarted right-preconditioned FGMRES(m) for
// A w = b (Eq.4), the Krylov method wrapped around RASM (P:359,
// "in combination with any iterative method like the Krylov subspace
// methods. In this work we use the Generalized Minimum Residual (GMRES)").
//
// Design:
//  * all vectors in the cell (sorted) order, fp64, resident in HBM; the
//    flexible form stores Z_j = M V_j so the (inexact, fp32) preconditioner
//    may change between phases;
//  * CGS2 orthogonalisation: two passes of a fused multi-dot (deterministic
//    two-stage reduction) + multi-axpy over the basis;
//  * the (m+1) x m Hessenberg / Givens recurrence runs on the host (<= 51
//    values per iteration, one D2H copy per iteration);
//  * two operator tiers: phase 1 uses the fp32 summation (ex2.approx,
//    fp32 accumulation) until the true residual reaches phase1_rtol; phase 2
//    switches to the fp64 summation and continues to rtol.  The stopping
//    test is always a TRUE residual b - A w recomputed at restart (reading R6),
//    never the Arnoldi estimate alone.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "internal.h"
#include "solver.h"
#include "transport.h"

namespace rbf {
namespace {

constexpr int kVecThreads = 256;
constexpr int kDotChunk = 4;

// partial[j * nblk + blk] = sum over this block's slice of V_j . w, j in [0, k);
// blockIdx.y selects the chunk of kDotChunk basis vectors (chunks run in parallel)
template <class VT>
__global__ void __launch_bounds__(kVecThreads)
multi_dot_kernel(const VT* __restrict__ V, int64_t ldv, int k, const double* __restrict__ w, int64_t n,
                 double* __restrict__ partial) {
  __shared__ double red[kVecThreads / 32][kDotChunk];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int j0 = blockIdx.y * kDotChunk;
  const int nblk = gridDim.x;
  double acc[kDotChunk];
#pragma unroll
  for (int q = 0; q < kDotChunk; ++q) acc[q] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)nblk * blockDim.x) {
    const double wi = w[i];
#pragma unroll
    for (int q = 0; q < kDotChunk; ++q)
      if (j0 + q < k) acc[q] = fma((double)V[(int64_t)(j0 + q) * ldv + i], wi, acc[q]);
  }
#pragma unroll
  for (int q = 0; q < kDotChunk; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    if (lane == 0) red[wid][q] = acc[q];
  }
  __syncthreads();
  if (threadIdx.x < kDotChunk && j0 + (int)threadIdx.x < k) {
    double s = 0.0;
    for (int q = 0; q < kVecThreads / 32; ++q) s += red[q][threadIdx.x];
    partial[(int64_t)(j0 + threadIdx.x) * nblk + blockIdx.x] = s;
  }
}

// out[j] = sum_b partial[j * nblk + b]   (fixed order: deterministic);  out[j] += add[j] if add
__global__ void reduce_partials(const double* __restrict__ partial, int k, int nblk, double* __restrict__ out,
                                int negate_into, double* __restrict__ neg_out) {
  const int j = blockIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += 32) s += partial[(int64_t)j * nblk + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) {
    out[j] = s;
    if (negate_into) neg_out[j] = -s;
  }
}

// w[i] += sum_j coef[j] * V_j[i]
template <class VT>
__global__ void multi_axpy_kernel(double* __restrict__ w, const VT* __restrict__ V, int64_t ldv, int k,
                                  const double* __restrict__ coef, int64_t n) {
  __shared__ double sc[64];
  for (int q = threadIdx.x; q < k && q < 64; q += blockDim.x) sc[q] = coef[q];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = w[i];
    for (int j = 0; j < k; ++j) acc = fma(sc[j], (double)V[(int64_t)j * ldv + i], acc);
    w[i] = acc;
  }
}

// multi_axpy fused with the next norm: w[i] += sum_j coef[j] V_j[i], and
// partial[blockIdx.x] = this block's sum of the new w[i]^2 (grid-stride over a
// fixed grid, fixed reduction order: deterministic), saving a pass over w
template <class VT>
__global__ void __launch_bounds__(kVecThreads)
multi_axpy_nrm_kernel(double* __restrict__ w, const VT* __restrict__ V, int64_t ldv, int k,
                      const double* __restrict__ coef, int64_t n, double* __restrict__ partial) {
  __shared__ double sc[64];
  __shared__ double red[kVecThreads / 32];
  for (int q = threadIdx.x; q < k && q < 64; q += blockDim.x) sc[q] = coef[q];
  __syncthreads();
  double ss = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = w[i];
    for (int j = 0; j < k; ++j) acc = fma(sc[j], (double)V[(int64_t)j * ldv + i], acc);
    w[i] = acc;
    ss = fma(acc, acc, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < kVecThreads / 32; ++q) t += red[q];
    partial[blockIdx.x] = t;
  }
}

// ---- 4-wide forms (n % 4 == 0: every basis vector V + j n is 16-byte aligned).
// Same sums in a different (still fixed) order: a thread owns 4 consecutive
// elements per sweep, the basis is read as 16-byte (fp32) or 2 x 16-byte (fp64)
// loads with a whole chunk of vectors in flight per thread, w as two double2.
// The scalar kernels above read 4 bytes per load and re-read w (fp64) once per
// chunk of 4 vectors; here a chunk is kDotChunkV vectors.
constexpr int kDotChunkV = 8;

// the raw 4-element load is kept in registers and converted where it is used
template <class VT> struct Vec4;
template <> struct Vec4<float> {
  float4 a;
  __device__ __forceinline__ void load(const float* p) { a = __ldcs(reinterpret_cast<const float4*>(p)); }
  __device__ __forceinline__ double x0() const { return a.x; }
  __device__ __forceinline__ double x1() const { return a.y; }
  __device__ __forceinline__ double x2() const { return a.z; }
  __device__ __forceinline__ double x3() const { return a.w; }
};
template <> struct Vec4<double> {
  double2 a, b;
  __device__ __forceinline__ void load(const double* p) {
    a = __ldcs(reinterpret_cast<const double2*>(p));
    b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
  }
  __device__ __forceinline__ double x0() const { return a.x; }
  __device__ __forceinline__ double x1() const { return a.y; }
  __device__ __forceinline__ double x2() const { return b.x; }
  __device__ __forceinline__ double x3() const { return b.y; }
};

template <class VT>
__global__ void __launch_bounds__(kVecThreads, sizeof(VT) == 4 ? 3 : 1)
multi_dot4_kernel(const VT* __restrict__ V, int64_t ldv, int k, const double* __restrict__ w, int64_t n,
                  double* __restrict__ partial) {
  __shared__ double red[kVecThreads / 32][kDotChunkV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int j0 = blockIdx.y * kDotChunkV;
  const int nq = min(kDotChunkV, k - j0);
  const int nblk = gridDim.x;
  const VT* __restrict__ Vc = V + (int64_t)j0 * ldv;
  double acc[kDotChunkV];
#pragma unroll
  for (int q = 0; q < kDotChunkV; ++q) acc[q] = 0.0;
  const int64_t n4 = n >> 2;
  for (int64_t i4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i4 < n4; i4 += (int64_t)nblk * blockDim.x) {
    const int64_t i = i4 << 2;
    const double2 wa = *reinterpret_cast<const double2*>(w + i), wb = *reinterpret_cast<const double2*>(w + i + 2);
    Vec4<VT> v[kDotChunkV];
#pragma unroll
    for (int q = 0; q < kDotChunkV; ++q)
      if (q < nq) v[q].load(Vc + (int64_t)q * ldv + i);
#pragma unroll
    for (int q = 0; q < kDotChunkV; ++q)
      if (q < nq) {
        double a = acc[q];
        a = fma(v[q].x0(), wa.x, a); a = fma(v[q].x1(), wa.y, a);
        a = fma(v[q].x2(), wb.x, a); a = fma(v[q].x3(), wb.y, a);
        acc[q] = a;
      }
  }
#pragma unroll
  for (int q = 0; q < kDotChunkV; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    if (lane == 0) red[wid][q] = acc[q];
  }
  __syncthreads();
  if ((int)threadIdx.x < nq) {
    double s = 0.0;
    for (int q = 0; q < kVecThreads / 32; ++q) s += red[q][threadIdx.x];
    partial[(int64_t)(j0 + threadIdx.x) * nblk + blockIdx.x] = s;
  }
}

// w[i] += sum_j coef[j] V_j[i] (4 elements per thread and sweep, 8 basis vectors
// in flight), and, with NRM, partial[blockIdx.x] = this block's sum of the new
// w[i]^2 (fixed grid, fixed order: deterministic)
template <class VT, bool NRM>
__global__ void __launch_bounds__(kVecThreads)
multi_axpy4_kernel(double* __restrict__ w, const VT* __restrict__ V, int64_t ldv, int k,
                   const double* __restrict__ coef, int64_t n, double* __restrict__ partial) {
  __shared__ double sc[64];
  __shared__ double red[kVecThreads / 32];
  for (int q = threadIdx.x; q < k && q < 64; q += blockDim.x) sc[q] = coef[q];
  __syncthreads();
  double ss = 0.0;
  const int64_t n4 = n >> 2;
  for (int64_t i4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i4 < n4;
       i4 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i4 << 2;
    double2 wa = *reinterpret_cast<const double2*>(w + i), wb = *reinterpret_cast<const double2*>(w + i + 2);
    int j = 0;
    for (; j + 8 <= k; j += 8) {
      Vec4<VT> v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q].load(V + (int64_t)(j + q) * ldv + i);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double c = sc[j + q];
        wa.x = fma(c, v[q].x0(), wa.x); wa.y = fma(c, v[q].x1(), wa.y);
        wb.x = fma(c, v[q].x2(), wb.x); wb.y = fma(c, v[q].x3(), wb.y);
      }
    }
    for (; j < k; ++j) {
      Vec4<VT> v;
      v.load(V + (int64_t)j * ldv + i);
      const double c = sc[j];
      wa.x = fma(c, v.x0(), wa.x); wa.y = fma(c, v.x1(), wa.y);
      wb.x = fma(c, v.x2(), wb.x); wb.y = fma(c, v.x3(), wb.y);
    }
    *reinterpret_cast<double2*>(w + i) = wa;
    *reinterpret_cast<double2*>(w + i + 2) = wb;
    if (NRM) {
      ss = fma(wa.x, wa.x, ss); ss = fma(wa.y, wa.y, ss);
      ss = fma(wb.x, wb.x, ss); ss = fma(wb.y, wb.y, ss);
    }
  }
  if (NRM) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < kVecThreads / 32; ++q) t += red[q];
      partial[blockIdx.x] = t;
    }
  }
}

template <class OT>
__global__ void scale_kernel(const double* __restrict__ a, double s, OT* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (OT)(a[i] * s);
}
// b = a * (1 / *nrm)  (norm on the device)
template <class OT>
__global__ void scale_by_inv_norm(const double* __restrict__ a, const double* __restrict__ nrm2,
                                  OT* __restrict__ b, int64_t n) {
  const double s = 1.0 / sqrt(*nrm2);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (OT)(a[i] * s);
}
__global__ void residual_kernel(const double* __restrict__ b, const double* __restrict__ f, double* __restrict__ r,
                                int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = b[i] - f[i];
}
__global__ void negate_kernel(const double* __restrict__ a, double* __restrict__ b, int k) {
  for (int i = threadIdx.x; i < k; i += blockDim.x) b[i] = -a[i];
}
__global__ void f32_to_f64(const float* __restrict__ a, double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (double)a[i];
}

struct Solver {
  rbf_ctx* ctx;
  const rbf_cells* c;
  const rbf_precond* P;
  KernelParams kp;
  int64_t n;
  int m;
  int nblk;
  DevBuf V, Z, x, r, w, f, b, partial, dots;
  // fp32 Krylov basis of the fp32 phase (V32, Z32; basis32): the phase works to
  // a relative residual >= 1e-4 with an operator accurate to ~1e-6, so basis
  // vectors rounded to fp32 (6e-8) cost nothing it can see; the fp64 phase keeps
  // V, Z in fp64.  Halves the Krylov vector traffic of the fp32 phase.
  DevBuf V32, Z32;
  bool basis32 = true;
  bool vec4 = false;       // n % 4 == 0: the 4-wide Krylov kernels (aligned 16-byte loads)
  int opv = RBF_OP_AUTO;   // operator variant (rbf_op_variant)
  int64_t mv32 = 0, mv64 = 0;

  // the fp64 basis, allocated when a cycle first runs on it
  rbf_status ensure64() {
    cudaStream_t s = ctx->stream;
    if (!V.p) RBF_TRY(V.alloc(sizeof(double) * n * (m + 1), s));
    if (!Z.p) RBF_TRY(Z.alloc(sizeof(double) * n * m, s));
    return RBF_OK;
  }
  rbf_status alloc() {
    cudaStream_t s = ctx->stream;
    if (basis32) {
      RBF_TRY(V32.alloc(sizeof(float) * n * (m + 1), s));
      RBF_TRY(Z32.alloc(sizeof(float) * n * m, s));
    }
    RBF_TRY(x.alloc(sizeof(double) * n, s));
    RBF_TRY(r.alloc(sizeof(double) * n, s));
    RBF_TRY(w.alloc(sizeof(double) * n, s));
    RBF_TRY(f.alloc(sizeof(double) * n, s));
    RBF_TRY(b.alloc(sizeof(double) * n, s));
    vec4 = (n % 4) == 0 && n >= 4;
    nblk = ctx->sm_count * 4;   // x chunks of kDotChunk basis vectors (grid.y): enough warps in flight
    RBF_TRY(partial.alloc(sizeof(double) * (size_t)nblk * (m + 2), s));
    RBF_TRY(dots.alloc(sizeof(double) * 4 * (m + 2), s));
    return RBF_OK;
  }
  template <class VT> VT* basis() { return std::is_same<VT, float>::value ? (VT*)V32.p : (VT*)V.p; }
  template <class VT> VT* zbasis() { return std::is_same<VT, float>::value ? (VT*)Z32.p : (VT*)Z.p; }

  rbf_status op(bool fp64, const double* in, double* out) {
    if (fp64) { ++mv64; return matvec_sorted_f64(ctx, c, kp, in, out, nullptr, opv); }
    ++mv32;
    return matvec_sorted_f32_d(ctx, c, kp, in, out, opv);
  }
  rbf_status op(bool fp64, const float* in, double* out) {   // fp32 basis: fp32 phase only
    if (fp64) { set_error("internal: fp64 operator on an fp32 basis"); return RBF_EINVAL; }
    ++mv32;
    return matvec_sorted_f32_f(ctx, c, kp, in, out, opv);
  }
  // dots[0..k) = V_{0..k}^T w ; neg copy at dots[(m+2)...]
  template <class VT>
  rbf_status mdot(const VT* Vb, int k, const double* vec, double* out, double* neg) {
    cudaStream_t s = ctx->stream;
    if (vec4) {
      const dim3 grid((unsigned)nblk, (unsigned)((k + kDotChunkV - 1) / kDotChunkV));
      multi_dot4_kernel<VT><<<grid, kVecThreads, 0, s>>>(Vb, n, k, vec, n, partial.as<double>());
    } else {
      const dim3 grid((unsigned)nblk, (unsigned)((k + kDotChunk - 1) / kDotChunk));
      multi_dot_kernel<VT><<<grid, kVecThreads, 0, s>>>(Vb, n, k, vec, n, partial.as<double>());
    }
    RBF_CHECK_LAUNCH();
    if (ctx->world == 1) {
      reduce_partials<<<k, 32, 0, s>>>(partial.as<double>(), k, nblk, out, neg != nullptr, neg);
      RBF_CHECK_LAUNCH();
      return RBF_OK;
    }
    // slab partition: local partial sums, then the sum over ranks (ncclAllReduce)
    reduce_partials<<<k, 32, 0, s>>>(partial.as<double>(), k, nblk, out, 0, nullptr);
    RBF_CHECK_LAUNCH();
    RBF_TRY(allreduce_sum(ctx, out, k));
    if (neg) {
      negate_kernel<<<1, 64, 0, s>>>(out, neg, k);
      RBF_CHECK_LAUNCH();
    }
    return RBF_OK;
  }
  template <class VT>
  rbf_status maxpy(double* vec, const VT* Vb, int k, const double* coef) {
    if (vec4)
      multi_axpy4_kernel<VT, false><<<nblk, kVecThreads, 0, ctx->stream>>>(vec, Vb, n, k, coef, n, nullptr);
    else
      multi_axpy_kernel<VT><<<grid_for(n, kVecThreads), kVecThreads, 0, ctx->stream>>>(vec, Vb, n, k, coef, n);
    RBF_CHECK_LAUNCH();
    return RBF_OK;
  }
  // maxpy, and *nrm2_out = ||vec||^2 of the result (one pass)
  template <class VT>
  rbf_status maxpy_nrm(double* vec, const VT* Vb, int k, const double* coef, double* nrm2_out) {
    cudaStream_t s = ctx->stream;
    if (vec4)
      multi_axpy4_kernel<VT, true><<<nblk, kVecThreads, 0, s>>>(vec, Vb, n, k, coef, n, partial.as<double>());
    else
      multi_axpy_nrm_kernel<VT><<<nblk, kVecThreads, 0, s>>>(vec, Vb, n, k, coef, n, partial.as<double>());
    RBF_CHECK_LAUNCH();
    reduce_partials<<<1, 32, 0, s>>>(partial.as<double>(), 1, nblk, nrm2_out, 0, nullptr);
    RBF_CHECK_LAUNCH();
    if (ctx->world > 1) RBF_TRY(allreduce_sum(ctx, nrm2_out, 1));
    return RBF_OK;
  }
  // r = b - A x ; returns ||r|| (synchronises)
  rbf_status residual(bool fp64, double* beta) {
    cudaStream_t s = ctx->stream;
    RBF_TRY(op(fp64, x.as<double>(), f.as<double>()));
    residual_kernel<<<grid_for(n, 256), 256, 0, s>>>(b.as<double>(), f.as<double>(), r.as<double>(), n);
    RBF_CHECK_LAUNCH();
    double* d = dots.as<double>();
    RBF_TRY(mdot(r.as<double>(), 1, r.as<double>(), d, nullptr));
    double h;
    RBF_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, s));
    RBF_CUDA_TRY(cudaStreamSynchronize(s));
    *beta = std::sqrt(h);
    return RBF_OK;
  }
};

}  // namespace

rbf_status gmres_sorted(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp, const rbf_precond* P,
                        const rbf_gmres_cfg* gcfg, const float* b_sorted32, double* x_out_sorted,
                        rbf_solve_report* rep, const double* x0_sorted) {
  using clk = std::chrono::steady_clock;
  cudaStream_t s = ctx->stream;
  Solver S{ctx, c, P, kp, c->n_loc(), 30, 0};   // this rank's owned slice (all of it on one GPU)
  S.m = (gcfg && gcfg->restart > 0) ? gcfg->restart : 30;
  if (S.m > 60) { set_error("restart must be <= 60"); return RBF_EINVAL; }
  const double rtol = (gcfg && gcfg->rtol > 0) ? gcfg->rtol : 1e-6;
  const double p1tol = (gcfg && gcfg->phase1_rtol > 0) ? gcfg->phase1_rtol : 1e-4;
  const int maxit = (gcfg && gcfg->max_iters > 0) ? gcfg->max_iters : 500;
  const bool polish = gcfg ? gcfg->polish_fp64 != 0 : true;
  const int passes = (gcfg && gcfg->cgs_passes == 1) ? 1 : 2;
  const int64_t n = S.n;
  const int m = S.m;
  S.basis32 = !(gcfg && gcfg->basis_fp64);   // basis_fp64: fp64 basis in both phases
  S.opv = gcfg ? gcfg->op_variant : RBF_OP_AUTO;
  double* hist = gcfg ? gcfg->history : nullptr;
  double* hist_true = gcfg ? gcfg->history_true : nullptr;
  const int hcap = (gcfg && gcfg->history_cap > 0) ? gcfg->history_cap : 0;
  int hlen = 0, htlen = 0;
  auto record_true = [&](double v) {
    if (hist_true && htlen < hcap) hist_true[htlen] = v;
    ++htlen;
  };
  RBF_TRY(S.alloc());
  f32_to_f64<<<grid_for(n, 256), 256, 0, s>>>(b_sorted32, S.b.as<double>(), n);
  RBF_CHECK_LAUNCH();
  RBF_CUDA_TRY(cudaMemsetAsync(S.x.p, 0, sizeof(double) * n, s));
  double* d = S.dots.as<double>();
  double* dh = d;                  // h (pass 1 + 2)
  double* dneg = d + (m + 2);      // -h for the axpy
  double* d2 = d + 2 * (m + 2);    // pass-2 h
  double* dn = d + 3 * (m + 2);    // norm^2
  RBF_TRY(S.mdot(S.b.as<double>(), 1, S.b.as<double>(), dh, nullptr));
  double bn2 = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&bn2, dh, sizeof(double), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  const double bnorm = std::sqrt(bn2);
  rbf_solve_report R{};
  auto t_start = clk::now();
  if (bnorm == 0.0) {
    RBF_CUDA_TRY(cudaMemcpyAsync(x_out_sorted, S.x.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    R.converged = 1;
    if (rep) {
      R.t_setup = rep->t_setup;
      R.nblocks = rep->nblocks;
      R.precond_bytes = rep->precond_bytes;
      *rep = R;
    }
    return RBF_OK;
  }
  bool fp64 = false;
  int it = 0, it1 = 0, it2 = 0;
  bool breakdown_any = false;
  int stagnant = 0;
  double beta = bnorm, last_beta = bnorm, est = 1.0;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m), hcol(m + 2);
  // pinned Hessenberg slots (one per Arnoldi step of a cycle) and two events
  const size_t pstride = (size_t)2 * (m + 2) + 1;
  RBF_TRY(ctx->pinned(sizeof(double) * pstride * (size_t)m));
  double* hpin = static_cast<double*>(ctx->hpin);
  cudaEvent_t ev[2];
  RBF_CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  RBF_CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); }
  } ev_guard{ev};
  double t_switch = 0.0;
  if (x0_sorted) {
    // warm start: x = x0, r = b - A x0 (fp32 tier; phase 2 recomputes it in fp64)
    RBF_CUDA_TRY(cudaMemcpyAsync(S.x.p, x0_sorted, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    RBF_TRY(S.residual(false, &beta));
    last_beta = beta;
  } else {
    // r = b (x = 0)
    RBF_CUDA_TRY(cudaMemcpyAsync(S.r.p, S.b.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
  double cycle_beta = -1.0;   // true residual at the start of the previous cycle
  bool final_fp64 = false;    // beta already is the fp64 true residual of the final x
  for (;;) {
    // phase switch: phase-1 target reached, or the fp32 tier stopped making
    // progress (a cycle that did not halve the true residual, or > 3m
    // iterations): the fp32 operator's rounding then dominates near-null
    // directions of ill-conditioned clouds and only the fp64 tier can continue.
    const bool p1_stalled = cycle_beta > 0 && (beta > 0.5 * cycle_beta || it1 >= 3 * m);
    if (!fp64 && polish && (beta / bnorm <= p1tol || p1_stalled)) {
      fp64 = true;
      t_switch = std::chrono::duration<double>(clk::now() - t_start).count();
      RBF_TRY(S.residual(true, &beta));
    }
    if (fp64 && beta / bnorm <= rtol) break;
    if (!polish && beta / bnorm <= rtol) break;
    if (it >= maxit) break;
    if (beta >= last_beta * (1 - 1e-12) && it > 0) {
      if (++stagnant >= 3) break;
    } else {
      stagnant = 0;
    }
    last_beta = beta;
    cycle_beta = fp64 ? -1.0 : beta;
    record_true(beta / bnorm);
    // inner stopping target: the phase-1 target only while a phase 2 follows
    const double target = (fp64 || !polish) ? rtol : std::max(p1tol, rtol);
    // one restart cycle on a basis of type VT (float: fp32 phase with basis32)
    RBF_NVTX(fp64 ? "gmres cycle (fp64 tier)" : "gmres cycle (fp32 tier)");
    int k = 0;
    bool bd = false;
    auto cycle = [&](auto tag) -> rbf_status {
      using VT = decltype(tag);
      VT* Vb = S.basis<VT>();
      VT* Zb = S.zbasis<VT>();
      auto Vj = [&](int j) { return Vb + (int64_t)j * n; };
      auto Zj = [&](int j) { return Zb + (int64_t)j * n; };
      // V0 = r / beta
      scale_kernel<VT><<<grid_for(n, 256), 256, 0, s>>>(S.r.as<double>(), 1.0 / beta, Vj(0), n);
      RBF_CHECK_LAUNCH();
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      // Arnoldi step j on the device; its Hessenberg column lands in pinned
      // slot j (hcol, pass-2 h, |w|^2) and event ev[j & 1] marks it
      auto enqueue = [&](int j) -> rbf_status {
        RBF_TRY(precond_apply_sorted<VT>(ctx, P, Vj(j), Zj(j)));
        RBF_TRY(S.op(fp64, (const VT*)Zj(j), S.w.as<double>()));
        double* wv = S.w.as<double>();
        // classical Gram-Schmidt, one pass or two (CGS2, the default)
        // (the last axpy pass also forms |w|^2 for the normalisation)
        RBF_TRY(S.mdot<VT>(Vb, j + 1, wv, dh, dneg));
        if (passes == 2) {
          RBF_TRY(S.maxpy<VT>(wv, Vb, j + 1, dneg));
          RBF_TRY(S.mdot<VT>(Vb, j + 1, wv, d2, dneg));
          RBF_TRY(S.maxpy_nrm<VT>(wv, Vb, j + 1, dneg, dn));
        } else {
          RBF_TRY(S.maxpy_nrm<VT>(wv, Vb, j + 1, dneg, dn));
          RBF_CUDA_TRY(cudaMemsetAsync(d2, 0, sizeof(double) * (j + 1), s));
        }
        scale_by_inv_norm<VT><<<grid_for(n, 256), 256, 0, s>>>(wv, dn, Vj(j + 1), n);
        RBF_CHECK_LAUNCH();
        double* slot = hpin + (size_t)j * pstride;
        RBF_CUDA_TRY(cudaMemcpyAsync(slot, dh, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, s));
        RBF_CUDA_TRY(cudaMemcpyAsync(slot + (m + 2), d2, sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, s));
        RBF_CUDA_TRY(cudaMemcpyAsync(slot + 2 * (m + 2), dn, sizeof(double), cudaMemcpyDeviceToHost, s));
        RBF_CUDA_TRY(cudaEventRecord(ev[j & 1], s));
        return RBF_OK;
      };
      // the next step is enqueued BEFORE the host reads this step's column
      // (it depends only on device data), so the Givens update and the launch
      // latency overlap the GPU; a step enqueued past a convergence or
      // breakdown exit is discarded (it touches neither x nor r)
      RBF_TRY(enqueue(0));
      for (int j = 0; j < m; ++j) {
        if (j + 1 < m && it + 1 < maxit) RBF_TRY(enqueue(j + 1));
        RBF_CUDA_TRY(cudaEventSynchronize(ev[j & 1]));
        const double* slot = hpin + (size_t)j * pstride;
        for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = slot[i] + slot[(m + 2) + i];
        const double hn = std::sqrt(slot[2 * (m + 2)]);
        H[(size_t)(j + 1) * m + j] = hn;
        for (int i = 0; i < j; ++i) {
          const double a = H[(size_t)i * m + j], bb = H[(size_t)(i + 1) * m + j];
          H[(size_t)i * m + j] = cs[i] * a + sn[i] * bb;
          H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
        }
        const double a = H[(size_t)j * m + j], bb = H[(size_t)(j + 1) * m + j];
        const double den = std::hypot(a, bb);
        cs[j] = den > 0 ? a / den : 1.0;
        sn[j] = den > 0 ? bb / den : 0.0;
        H[(size_t)j * m + j] = den;
        H[(size_t)(j + 1) * m + j] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        ++it;
        if (fp64) ++it2; else ++it1;
        k = j + 1;
        est = std::fabs(g[j + 1]) / bnorm;
        if (hist && hlen < hcap) hist[hlen] = est;
        ++hlen;
        if (!(hn > 1e-14 * beta) || !std::isfinite(hn)) { bd = true; break; }
        if (est <= target || it >= maxit) break;
      }
      // y = H^-1 g, x += Z y
      for (int i = k - 1; i >= 0; --i) {
        double acc = g[i];
        for (int q = i + 1; q < k; ++q) acc -= H[(size_t)i * m + q] * y[q];
        const double dd = H[(size_t)i * m + i];
        y[i] = dd != 0 ? acc / dd : 0.0;
      }
      RBF_CUDA_TRY(cudaMemcpyAsync(dneg, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s));
      RBF_TRY(S.maxpy<VT>(S.x.as<double>(), Zb, k, dneg));
      return RBF_OK;
    };
    if (!fp64 && S.basis32) {
      RBF_TRY(cycle(0.0f));
    } else {
      RBF_TRY(S.ensure64());
      RBF_TRY(cycle(0.0));
    }
    ++R.restarts;
    if (bd) breakdown_any = true;
    if (it >= maxit && !fp64) {
      // out of iterations in the fp32 phase: the loop would only recompute the
      // fp32 residual to break on it >= maxit and then certify with the fp64
      // operator -- go to the certification directly (same x, same report)
      RBF_TRY(S.residual(true, &beta));
      final_fp64 = true;
      break;
    }
    RBF_TRY(S.residual(fp64, &beta));
  }
  // final true residual with the fp64 operator
  double tr = beta;
  if (!fp64 && !final_fp64) RBF_TRY(S.residual(true, &tr));
  const double t_end = std::chrono::duration<double>(clk::now() - t_start).count();
  RBF_CUDA_TRY(cudaMemcpyAsync(x_out_sorted, S.x.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  record_true(tr / bnorm);
  R.iters_phase1 = it1;
  R.iters_phase2 = it2;
  R.history_len = std::min(hlen, hcap);
  R.history_true_len = std::min(htlen, hcap);
  R.rel_residual_true = tr / bnorm;
  R.rel_residual_est = est;
  R.converged = (R.rel_residual_true <= rtol) ? 1 : 0;
  R.breakdown = breakdown_any ? 1 : 0;
  R.t_phase1 = fp64 ? t_switch : t_end;
  R.t_phase2 = fp64 ? t_end - t_switch : 0.0;
  R.matvecs_f32 = S.mv32;
  R.matvecs_f64 = S.mv64;
  if (rep) {
    R.t_setup = rep->t_setup;
    R.nblocks = rep->nblocks;
    R.precond_bytes = rep->precond_bytes;
    *rep = R;
  }
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  return RBF_OK;
}

}  // namespace rbf

using namespace rbf;

extern "C" {

rbf_status rbf_gmres_solve(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, const rbf_precond* precond,
                           const rbf_precond_cfg* pcfg, const rbf_gmres_cfg* gcfg, const float* b, double* w,
                           rbf_solve_report* rep) {
  RBF_NVTX("rbf_gmres_solve");
  if (!ctx || !c || !kern || !b || !w) { set_error("NULL argument"); return RBF_EINVAL; }
  if (!(kern->sigma > 0) || !(kern->cutoff_sigmas > 0)) { set_error("bad kernel"); return RBF_EINVAL; }
  if (kern->cutoff_sigmas * kern->sigma > c->cutoff * (1 + 1e-12)) {
    set_error("kernel cutoff exceeds the cutoff the cells were built for");
    return RBF_EINVAL;
  }
  if (precond && precond->cells != c) { set_error("precond was built for other cells"); return RBF_EINVAL; }
  if (c->world != ctx->world) { set_error("cells were partitioned for another world size"); return RBF_EINVAL; }
  if (gcfg && (gcfg->op_variant < RBF_OP_AUTO || gcfg->op_variant > RBF_OP_SYM_ROT)) {
    set_error("bad operator variant");
    return RBF_EINVAL;
  }
  if (gcfg && gcfg->history_cap < 0) { set_error("history_cap must be >= 0"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  KernelParams kp = kernel_params(kern);
  rbf_solve_report R{};
  rbf_precond* own = nullptr;
  const rbf_precond* P = precond;
  if (!P) {
    own = new (std::nothrow) rbf_precond();
    if (!own) { set_error("host allocation failed"); return RBF_ENOMEM; }
    rbf_status st;
    {
      ProfScope ps(ctx, RBF_PROF_PRECOND_SETUP);
      st = precond_build(ctx, c, kp, pcfg, own);
    }
    if (st != RBF_OK) { delete own; return st; }
    own->cells = c;
    P = own;
  }
  R.t_setup = P->t_setup;
  R.nblocks = P->nblocks;
  R.precond_bytes = P->bytes;
  const int64_t n = c->n;
  const int64_t o0 = c->view.o0;
  DevBuf bs, xs;
  rbf_status st = bs.alloc(sizeof(float) * n, ctx->stream);
  if (st == RBF_OK) st = xs.alloc(sizeof(double) * n, ctx->stream);
  if (st == RBF_OK) st = gather_f32_to_sorted(ctx, b, c->perm.as<int32_t>(), bs.as<float>(), n);
  // the solve runs on this rank's slice [o0, o1) of the sorted order; the full
  // solution is gathered from all ranks (replicated out)
  DevBuf x0s;
  const double* x0p = nullptr;
  if (st == RBF_OK && gcfg && gcfg->x0) {
    st = x0s.alloc(sizeof(double) * n, ctx->stream);
    if (st == RBF_OK) st = gather_f64_to_sorted(ctx, gcfg->x0, c->perm.as<int32_t>(), x0s.as<double>(), n);
    x0p = x0s.as<double>() + o0;
  }
  if (st == RBF_OK)
    st = gmres_sorted(ctx, c, kp, P, gcfg, bs.as<float>() + o0, xs.as<double>() + o0, &R, x0p);
  if (st == RBF_OK) st = allgather_sorted(ctx, c, xs.as<double>());
  if (st == RBF_OK) st = scatter_f64_from_sorted(ctx, xs.as<double>(), c->perm.as<int32_t>(), w, n);
  if (st == RBF_OK) {
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); st = RBF_ECUDA; }
  }
  delete own;
  if (rep) *rep = R;
  return st;
}

rbf_status rbf_gmres_solve_shard(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern,
                                 const rbf_precond* precond, const rbf_precond_cfg* pcfg, const rbf_gmres_cfg* gcfg,
                                 const float* b_local, int64_t n_local, int64_t id0, double* w_local,
                                 rbf_solve_report* rep) {
  if (!ctx || !c) { set_error("NULL argument"); return RBF_EINVAL; }
  if (n_local < 0 || id0 < 0 || (n_local > 0 && (!b_local || !w_local))) { set_error("bad shard"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  std::vector<int64_t> id0s, ns;
  int64_t total = 0;
  RBF_TRY(shard_layout(ctx, id0, n_local, id0s, ns, &total));
  if (total != c->n) { set_error("the shards of b do not cover the cells' centres"); return RBF_EINVAL; }
  DevBuf bf, wf;
  RBF_TRY(bf.alloc(sizeof(float) * total, ctx->stream));
  RBF_TRY(wf.alloc(sizeof(double) * total, ctx->stream));
  RBF_TRY(allgather_shards(ctx, b_local, id0s, ns, 1, bf.p, DType::F32));
  RBF_TRY(rbf_gmres_solve(ctx, c, kern, precond, pcfg, gcfg, bf.as<float>(), wf.as<double>(), rep));
  if (n_local > 0)
    RBF_CUDA_TRY(cudaMemcpyAsync(w_local, wf.as<double>() + id0, sizeof(double) * n_local, cudaMemcpyDeviceToDevice,
                                 ctx->stream));
  RBF_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return RBF_OK;
}

rbf_status rbf_reconstruct_host(rbf_ctx* ctx, const float* xyz, const float* b, int64_t n, const rbf_kernel* kern,
                                const rbf_cell_cfg* ccfg, const rbf_precond_cfg* pcfg, const rbf_gmres_cfg* gcfg,
                                const rbf_grid* grid, double* w_out, float* field_out, rbf_solve_report* rep) {
  RBF_NVTX("rbf_reconstruct_host");
  if (!ctx || !xyz || !b || !kern || !grid || !w_out || !field_out) { set_error("NULL argument"); return RBF_EINVAL; }
  if (n < 1) { set_error("n must be >= 1"); return RBF_EINVAL; }
  for (int a = 0; a < 3; ++a)
    if (grid->n[a] < 2) { set_error("grid needs n >= 2 nodes per axis"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const int64_t nodes = (int64_t)grid->n[0] * grid->n[1] * grid->n[2];
  DevBuf dx, db, dw, df;
  RBF_TRY(dx.alloc(sizeof(float) * 3 * n, s));
  RBF_TRY(db.alloc(sizeof(float) * n, s));
  RBF_TRY(dw.alloc(sizeof(double) * n, s));
  RBF_TRY(df.alloc(sizeof(float) * nodes, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(dx.p, xyz, sizeof(float) * 3 * n, cudaMemcpyHostToDevice, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(db.p, b, sizeof(float) * n, cudaMemcpyHostToDevice, s));
  rbf_cells* cells = nullptr;
  RBF_TRY(rbf_build_cells(ctx, dx.as<float>(), n, kern, ccfg, &cells));
  rbf_solve_report R{};
  rbf_status st = rbf_gmres_solve(ctx, cells, kern, nullptr, pcfg, gcfg, db.as<float>(), dw.as<double>(), &R);
  if (st == RBF_OK) st = rbf_eval_grid(ctx, cells, kern, dw.as<double>(), grid, df.as<float>());
  if (st == RBF_OK) {
    cudaError_t e1 = cudaMemcpyAsync(w_out, dw.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
    cudaError_t e2 = cudaMemcpyAsync(field_out, df.p, sizeof(float) * nodes, cudaMemcpyDeviceToHost, s);
    cudaError_t e3 = cudaStreamSynchronize(s);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      set_error("copy-out failed");
      st = RBF_ECUDA;
    }
  }
  rbf_cells_free(cells);
  if (rep) *rep = R;
  return st;
}

}  // extern "C"
