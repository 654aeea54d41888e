// a4 of SURVEY.md §8(a): batched fp64 LU with partial pivoting of the RAS
// extended blocks, fused with the solve for the restricted inverse
// (§3.1: "solving smaller systems" on every subdomain Omega_i).
//
// For each block b the workspace holds the augmented matrix [A_ext | E_core]
// (m x (m + nc), row-major).  Gaussian elimination with partial pivoting turns
// it into [U | L^-1 P E_core]; blocked back-substitution then gives
// X = A_ext^-1 E_core and W = X^T = (A_ext^-1)[core, :] (A_ext symmetric).
//
// The elimination is driven from the host in steps of kNb = 64 columns so that
// every kernel has thousands of CTAs (all blocks of a chunk x all tiles):
//   panel      one thread-block cluster per block: pivoted factorisation of the
//              (m-k0) x 64 panel held in the cluster's shared memory (DSMEM
//              pivot search and row exchange); then inv(L11) per block
//   swap_trsm  (block, 64-column tile): the panel's row swaps on the columns
//              right of it, then U12 = inv(L11) A12
//   gemm       (block, 64x64 tile): A22 -= L21 U12 — register-blocked fp64
//              (4x4 per thread, operands staged in shared memory, K = 64)
// and the back-substitution in steps of 64 rows from the bottom:
//   diag_solve (block, 64-column RHS tile): X_k = inv(U_kk) Y_k
//   gemm       (block, tile): Y[0:k0] -= U[0:k0, k0:k0+64] X_k
#include <algorithm>
#include <cmath>

#include <cooperative_groups.h>

#include "internal.h"
#include "solver.h"

namespace rbf {
namespace {

constexpr int kNb = 64;
constexpr int kThreads = 256;
constexpr int kLd = kNb + 4;   // padded smem row (doubles)

// ------------------------------------------------------------------ panel ---
// Panel factorisation held on chip: a cluster of CL CTAs per block matrix, CTA
// `rank` owns panel rows [rank*R, rank*R + R) (relative to k0) in its shared
// memory.  Per column: local pivot candidates -> cluster barrier -> every CTA
// reduces the CL candidates through DSMEM (same result everywhere) -> the
// pivot row and the displaced row are exchanged through DSMEM -> local rank-1
// update of the owned rows (fused with the next column's candidate search).
// HBM sees one read and one write of the panel per elimination step.
// block barrier, preceded in the CHECKED build by a jitter (checks.h)
#define RBF_SYNC()     \
  do {                 \
    RBF_JITTER();      \
    __syncthreads();   \
  } while (0)
constexpr int kPs = kNb + 1;   // smem row stride (doubles) of the cluster panel

__global__ void __launch_bounds__(kThreads)
panel_cluster_kernel(const LuJob* __restrict__ jobs, double* __restrict__ ws, int k0, int* __restrict__ piv,
                     int R, int* __restrict__ info) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), CL = (int)cl.num_blocks();
  const int job = blockIdx.x / CL;
  extern __shared__ double Pn[];   // R x kPs
  __shared__ double srow[kNb], tmp[kNb];
  __shared__ double sv[kThreads / 32];
  __shared__ int si[kThreads / 32];
  __shared__ double cand_v;
  __shared__ int cand_i, s_p;
  const LuJob J = jobs[job];
  const int m = J.m, ld = J.m + J.nc;
  if (k0 >= m) return;                       // uniform over the cluster
  const int kb = min(kNb, m - k0);
  double* A = ws + J.ws_off;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rows = m - k0;
  const int rb = rank * R;                   // first owned row (relative)
  const int nl = max(0, min(R, rows - rb));  // owned rows
  for (int q = tid; q < nl * kb; q += kThreads) {
    const int lr = q / kb, c = q % kb;
    Pn[lr * kPs + c] = A[(int64_t)(k0 + rb + lr) * ld + k0 + c];
  }
  RBF_SYNC();
  int singular = 0;
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int lr = tid; lr < nl; lr += kThreads) {
    const double v = fabs(Pn[lr * kPs]);
    if (v > best) { best = v; bi = rb + lr; }
  }
  for (int jj = 0; jj < kb; ++jj) {
    // local candidate (largest |a|, lowest row on ties)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { sv[wid] = best; si[wid] = bi; }
    RBF_SYNC();
    if (tid == 0) {
      double b2 = sv[0];
      int i2 = si[0];
      for (int q = 1; q < kThreads / 32; ++q)
        if (sv[q] > b2 || (sv[q] == b2 && si[q] < i2)) { b2 = sv[q]; i2 = si[q]; }
      cand_v = b2;
      cand_i = i2;
    }
    RBF_JITTER(); cl.sync();
    // global pivot: reduce the CL candidates (DSMEM), identically in every CTA
    if (wid == 0) {
      double v = -1.0;
      int i = 0x7fffffff;
      if (lane < CL) {
        v = *cl.map_shared_rank(&cand_v, lane);
        i = *cl.map_shared_rank(&cand_i, lane);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
      }
      if (lane == 0) s_p = i;
    }
    RBF_SYNC();
    const int p = s_p;
    const int own_p = p / R, own_j = jj / R;
    if (tid < kb) {
      srow[tid] = cl.map_shared_rank(Pn, own_p)[(p - own_p * R) * kPs + tid];
      if (rank == own_p && p != jj) tmp[tid] = cl.map_shared_rank(Pn, own_j)[(jj - own_j * R) * kPs + tid];
    }
    RBF_JITTER(); cl.sync();                               // all reads of the old rows are done
    if (tid < kb) {
      if (rank == own_j) Pn[(jj - rb) * kPs + tid] = srow[tid];
      if (rank == own_p && p != jj) Pn[(p - rb) * kPs + tid] = tmp[tid];
    }
    if (rank == 0 && tid == 0) piv[(int64_t)job * kNb + jj] = k0 + p;
    RBF_SYNC();
    double pv = srow[jj];
    if (pv == 0.0) { singular = 1; pv = 1e-300; }
    const double inv = 1.0 / pv;
    best = -1.0;
    bi = 0x7fffffff;
    for (int lr = max(0, jj + 1 - rb) + tid; lr < nl; lr += kThreads) {
      double* row = Pn + lr * kPs;
      const double l = row[jj] * inv;
      row[jj] = l;
      if (jj + 1 < kb) {
        const double v1 = fma(-l, srow[jj + 1], row[jj + 1]);
        row[jj + 1] = v1;
        if (fabs(v1) > best) { best = fabs(v1); bi = rb + lr; }
        for (int c = jj + 2; c < kb; ++c) row[c] = fma(-l, srow[c], row[c]);
      }
    }
    RBF_SYNC();
  }
  for (int q = tid; q < nl * kb; q += kThreads) {
    const int lr = q / kb, c = q % kb;
    A[(int64_t)(k0 + rb + lr) * ld + k0 + c] = Pn[lr * kPs + c];
  }
  if (singular && tid == 0) atomicAdd(info, 1);
  RBF_JITTER(); cl.sync();                                 // keep DSMEM alive until all peers are done
}

// inv(L11) of every block after its panel (one CTA per block)
__global__ void __launch_bounds__(kThreads)
linv_kernel(const LuJob* __restrict__ jobs, const double* __restrict__ ws, int k0, double* __restrict__ linv) {
  extern __shared__ double sm[];
  double* sL = sm;                 // kNb x kLd : L11 (unit lower)
  double* sI = sm + kNb * kLd;     // kNb x kLd : inv(L11)
  const LuJob J = jobs[blockIdx.x];
  const int m = J.m, ld = J.m + J.nc;
  if (k0 >= m) return;
  const int kb = min(kNb, m - k0);
  const double* A = ws + J.ws_off;
  const int tid = threadIdx.x;
  for (int q = tid; q < kNb * kNb; q += kThreads) {
    const int r = q / kNb, c = q % kNb;
    sL[r * kLd + c] = (r < kb && c < kb) ? A[(int64_t)(k0 + r) * ld + k0 + c] : 0.0;
  }
  RBF_SYNC();
  if (tid < kNb) {
    const int t = tid;
    for (int r = 0; r < kNb; ++r) {
      double x;
      if (r < t) x = 0.0;
      else if (r == t) x = 1.0;
      else {
        double acc = 0.0;
        for (int s = t; s < r; ++s) acc = fma(sL[r * kLd + s], sI[s * kLd + t], acc);
        x = (r < kb) ? -acc : 0.0;
      }
      sI[r * kLd + t] = x;
    }
  }
  RBF_SYNC();
  double* Li = linv + (int64_t)blockIdx.x * kNb * kNb;
  for (int q = tid; q < kNb * kNb; q += kThreads) Li[q] = sI[(q / kNb) * kLd + q % kNb];
}

// ------------------------------------------------------------- swap + trsm --
__global__ void __launch_bounds__(kThreads)
swap_trsm_kernel(const LuJob* __restrict__ jobs, double* __restrict__ ws, int k0, const int* __restrict__ piv,
                 const double* __restrict__ linv) {
  extern __shared__ double sm[];
  double* sI = sm;                 // inv(L11)
  double* sT = sm + kNb * kLd;     // A12 tile; also the staging of the permuted rows (2 kNb x kNb)
  __shared__ int s_rows[2 * kNb], s_src[2 * kNb];
  __shared__ int s_n;
  const LuJob J = jobs[blockIdx.x];
  const int m = J.m, ld = J.m + J.nc;
  if (k0 >= m) return;
  const int kb = min(kNb, m - k0);
  double* A = ws + J.ws_off;
  const int tid = threadIdx.x;
  const int* P = piv + (int64_t)blockIdx.x * kNb;
  // the panel's sequence of row swaps as one permutation of the affected rows
  if (tid == 0) {
    int n = 0;
    for (int jj = 0; jj < kb; ++jj) { s_rows[n] = k0 + jj; s_src[n] = k0 + jj; ++n; }
    for (int jj = 0; jj < kb; ++jj) {
      const int p = P[jj];
      int ip = -1;
      for (int q = 0; q < n; ++q)
        if (s_rows[q] == p) { ip = q; break; }
      if (ip < 0) { s_rows[n] = p; s_src[n] = p; ip = n; ++n; }
      const int t = s_src[jj]; s_src[jj] = s_src[ip]; s_src[ip] = t;   // row k0+jj is slot jj
    }
    s_n = n;
  }
  const double* Li = linv + (int64_t)blockIdx.x * kNb * kNb;
  for (int q = tid; q < kNb * kNb; q += kThreads) sI[(q / kNb) * kLd + q % kNb] = Li[q];
  RBF_SYNC();
  const int n = s_n;
  const int tx = tid & 15, ty = tid >> 4;
  for (int c0 = k0 + kb + kNb * blockIdx.y; c0 < ld; c0 += kNb * gridDim.y) {
    const int cw = min(kNb, ld - c0);
    // gather the permuted rows of this column tile, then scatter them (coalesced along columns)
    for (int q = tid; q < n * kNb; q += kThreads) {
      const int i = q / kNb, c = q % kNb;
      if (c < cw) sT[i * kNb + c] = A[(int64_t)s_src[i] * ld + c0 + c];
    }
    RBF_SYNC();
    for (int q = tid; q < n * kNb; q += kThreads) {
      const int i = q / kNb, c = q % kNb;
      if (c < cw && s_src[i] != s_rows[i]) A[(int64_t)s_rows[i] * ld + c0 + c] = sT[i * kNb + c];
    }
    RBF_SYNC();
    for (int q = tid; q < kNb * kNb; q += kThreads) {
      const int r = q / kNb, c = q % kNb;
      sT[r * kLd + c] = (r < kb && c < cw) ? A[(int64_t)(k0 + r) * ld + c0 + c] : 0.0;
    }
    RBF_SYNC();
    // U12 = inv(L11) * A12 : thread owns rows 4ty.., cols 4tx..
    double acc[4][4] = {};
    for (int t = 0; t < kb; ++t) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = sI[(4 * ty + q) * kLd + t]; b[q] = sT[t * kLd + 4 * tx + q]; }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[q][p] = fma(a[q], b[p], acc[q][p]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = 4 * ty + q;
      if (r >= kb) continue;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int c = 4 * tx + p;
        if (c < cw) A[(int64_t)(k0 + r) * ld + c0 + c] = acc[q][p];
      }
    }
    RBF_SYNC();
  }
}

// ------------------------------------------------------------------- gemm ---
// mode 0 (elimination):       C = A[k0+kb:m, k0+kb:ld]
// mode 1 (back-substitution): C = A[0:k0, m:ld]
// C -= A[rows, k0:k0+kb] * A[k0:k0+kb, cols]
__global__ void __launch_bounds__(kThreads)
gemm_kernel(const LuJob* __restrict__ jobs, double* __restrict__ ws, int k0, int mode) {
  extern __shared__ double sm[];
  double* sA = sm;                 // [i][t] : kNb x kLd  (A[r0+i][k0+t])
  double* sB = sm + kNb * kLd;     // [t][j] : kNb x kLd  (A[k0+t][c0+j])
  const LuJob J = jobs[blockIdx.x];
  const int m = J.m, ld = J.m + J.nc;
  if (k0 >= m) return;
  const int kb = min(kNb, m - k0);
  int r0, r1, cb0, cb1;
  if (mode == 0) { r0 = k0 + kb; r1 = m; cb0 = k0 + kb; cb1 = ld; }
  else { r0 = 0; r1 = k0; cb0 = m; cb1 = ld; }
  if (r0 >= r1 || cb0 >= cb1) return;
  const int ntc = (cb1 - cb0 + kNb - 1) / kNb;
  const int ntr = (r1 - r0 + kNb - 1) / kNb;
  double* A = ws + J.ws_off;
  const int tid = threadIdx.x;
  // fp64 tensor cores (DMMA 8x8x4): 8 warps, warp tile 16 x 32 = 2 x 4 mma tiles
  const int lane = tid & 31, w = tid >> 5;
  const int wm = w >> 1, wn = w & 1, g = lane >> 2, t4 = lane & 3;
  for (int tile = blockIdx.y; tile < ntr * ntc; tile += gridDim.y) {
    const int tr = r0 + kNb * (tile / ntc);
    const int tc = cb0 + kNb * (tile % ntc);
    // C tile -> accumulators (fragment layout) first: its HBM latency overlaps the staging
    double acc[2][4][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = tr + 16 * wm + 8 * mt + g;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int c = tc + 32 * wn + 8 * nt + 2 * t4 + i;
          acc[mt][nt][i] = (r < r1 && c < cb1) ? A[(int64_t)r * ld + c] : 0.0;
        }
    }
    for (int q = tid; q < kNb * kNb; q += kThreads) {
      const int i = q / kNb, t = q % kNb;     // row-major: sA[i][t] = A[tr+i][k0+t]
      const int r = tr + i;
      sA[i * kLd + t] = (r < r1 && t < kb) ? A[(int64_t)r * ld + k0 + t] : 0.0;
    }
    for (int q = tid; q < kNb * kNb; q += kThreads) {
      const int t = q / kNb, j = q % kNb;
      const int c = tc + j;
      sB[t * kLd + j] = (c < cb1 && t < kb) ? A[(int64_t)(k0 + t) * ld + c] : 0.0;
    }
    RBF_SYNC();
#pragma unroll 4
    for (int kk = 0; kk < kNb / 4; ++kk) {
      double af[2], bf[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) af[mt] = -sA[(16 * wm + 8 * mt + g) * kLd + 4 * kk + t4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = sB[(4 * kk + t4) * kLd + 32 * wn + 8 * nt + g];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[mt][nt][0]), "+d"(acc[mt][nt][1])
                       : "d"(af[mt]), "d"(bf[nt]));
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = tr + 16 * wm + 8 * mt + g;
      if (r >= r1) continue;
      double* row = A + (int64_t)r * ld;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int c = tc + 32 * wn + 8 * nt + 2 * t4 + i;
          if (c < cb1) row[c] = acc[mt][nt][i];
        }
    }
    RBF_SYNC();
  }
}

// ------------------------------------------------------------- diag solve ---
// inv(U_kk) of every block, once per step (one CTA per block)
__global__ void __launch_bounds__(kThreads)
uinv_kernel(const LuJob* __restrict__ jobs, const double* __restrict__ ws, int k0, double* __restrict__ uinv) {
  extern __shared__ double sm[];
  double* sU = sm;                 // U_kk (identity-padded)
  double* sI = sm + kNb * kLd;     // inv(U_kk)
  const LuJob J = jobs[blockIdx.x];
  const int m = J.m, ld = J.m + J.nc;
  if (k0 >= m) return;
  const int kb = min(kNb, m - k0);
  const double* A = ws + J.ws_off;
  const int tid = threadIdx.x;
  for (int q = tid; q < kNb * kNb; q += kThreads) {
    const int r = q / kNb, c = q % kNb;
    sU[r * kLd + c] = (r < kb && c < kb) ? A[(int64_t)(k0 + r) * ld + k0 + c] : (r == c ? 1.0 : 0.0);
  }
  RBF_SYNC();
  if (tid < kNb) {
    // column t of inv(U): back substitution of U x = e_t
    const int t = tid;
    for (int r = kNb - 1; r >= 0; --r) {
      double x;
      if (r > t) x = 0.0;
      else {
        double acc = (r == t) ? 1.0 : 0.0;
        for (int s2 = r + 1; s2 <= t; ++s2) acc = fma(-sU[r * kLd + s2], sI[s2 * kLd + t], acc);
        double d = sU[r * kLd + r];
        if (d == 0.0) d = 1e-300;
        x = acc / d;
      }
      sI[r * kLd + t] = x;
    }
  }
  RBF_SYNC();
  double* Ui = uinv + (int64_t)blockIdx.x * kNb * kNb;
  for (int q = tid; q < kNb * kNb; q += kThreads) Ui[q] = sI[(q / kNb) * kLd + q % kNb];
}

// X_k = inv(U_kk) Y_k on the RHS columns [m, ld), rows [k0, k0+kb)
__global__ void __launch_bounds__(kThreads)
diag_solve_kernel(const LuJob* __restrict__ jobs, double* __restrict__ ws, int k0,
                  const double* __restrict__ uinv) {
  extern __shared__ double sm[];
  double* sI = sm;                 // inv(U_kk)
  double* sY = sm + kNb * kLd;     // RHS tile
  const LuJob J = jobs[blockIdx.x];
  const int m = J.m, nc = J.nc, ld = m + nc;
  if (k0 >= m) return;
  const int kb = min(kNb, m - k0);
  double* A = ws + J.ws_off;
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const double* Ui = uinv + (int64_t)blockIdx.x * kNb * kNb;
  for (int q = tid; q < kNb * kNb; q += kThreads) sI[(q / kNb) * kLd + q % kNb] = Ui[q];
  for (int c0 = m + kNb * blockIdx.y; c0 < ld; c0 += kNb * gridDim.y) {
    const int cw = min(kNb, ld - c0);
    for (int q = tid; q < kNb * kNb; q += kThreads) {
      const int r = q / kNb, c = q % kNb;
      sY[r * kLd + c] = (r < kb && c < cw) ? A[(int64_t)(k0 + r) * ld + c0 + c] : 0.0;
    }
    RBF_SYNC();
    double acc[4][4] = {};
    for (int t = 0; t < kb; ++t) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { a[q] = sI[(4 * ty + q) * kLd + t]; b[q] = sY[t * kLd + 4 * tx + q]; }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[q][p] = fma(a[q], b[p], acc[q][p]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = 4 * ty + q;
      if (r >= kb) continue;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int c = 4 * tx + p;
        if (c < cw) A[(int64_t)(k0 + r) * ld + c0 + c] = acc[q][p];
      }
    }
    RBF_SYNC();
  }
}

// --------------------------------------------------------------- W = X^T ----
template <class WT>
__global__ void transpose_w_kernel(const LuJob* __restrict__ jobs, const double* __restrict__ ws,
                                   WT* __restrict__ W) {
  __shared__ double t[32][33];
  const LuJob J = jobs[blockIdx.x];
  const int m = J.m, nc = J.nc, ld = m + nc;
  const double* A = ws + J.ws_off;
  WT* Wb = W + J.w_off;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  const int ntc = (nc + 31) / 32, nte = (m + 31) / 32;
  for (int tile = blockIdx.y; tile < ntc * nte; tile += gridDim.y) {
    const int e0 = 32 * (tile / ntc), c0 = 32 * (tile % ntc);
    for (int r = ty; r < 32; r += 8) {
      const int e = e0 + r, c = c0 + tx;
      t[r][tx] = (e < m && c < nc) ? A[(int64_t)e * ld + m + c] : 0.0;
    }
    RBF_SYNC();
    for (int r = ty; r < 32; r += 8) {
      const int c = c0 + r, e = e0 + tx;
      if (c < nc && e < m) Wb[(int64_t)c * m + e] = (WT)t[tx][r];
    }
    RBF_SYNC();
  }
}

}  // namespace

namespace {

// One independent group of factorisation jobs issued on its own stream.
struct LuGroup {
  cudaStream_t s;
  const LuJob* jobs_dev;
  int nj, maxm, maxnc, maxld;
  int* piv;
  double* linv;
  int spread, CL, R;
  cudaLaunchConfig_t pcfg;
  cudaLaunchAttribute pattr[1];
};

size_t sm2_bytes() { return sizeof(double) * 2 * kNb * kLd; }
size_t smsw_bytes() { return sizeof(double) * (kNb * kLd + 2 * kNb * kNb); }   // inv(L11) + permutation staging

int tiles_of(int a, int b) { return (a + kNb - 1) / kNb * ((b + kNb - 1) / kNb); }

rbf_status lu_forward_step(LuGroup& G, int k0, double* ws, int* info) {
  if (k0 >= G.maxm) return RBF_OK;
  G.pcfg.attrs = G.pattr;
  RBF_CUDA_TRY(cudaLaunchKernelEx(&G.pcfg, panel_cluster_kernel, G.jobs_dev, ws, k0, G.piv, G.R, info));
  count_launch();
  linv_kernel<<<G.nj, kThreads, sm2_bytes(), G.s>>>(G.jobs_dev, ws, k0, G.linv);
  RBF_CHECK_LAUNCH();
  const int ct = std::max(1, std::min((G.maxld - k0 + kNb - 1) / kNb, G.spread));
  swap_trsm_kernel<<<dim3(G.nj, ct), kThreads, smsw_bytes(), G.s>>>(G.jobs_dev, ws, k0, G.piv, G.linv);
  RBF_CHECK_LAUNCH();
  const int gt = tiles_of(std::max(0, G.maxm - k0), std::max(0, G.maxld - k0));
  if (gt > 0) {
    gemm_kernel<<<dim3(G.nj, std::min(gt, G.spread)), kThreads, sm2_bytes(), G.s>>>(G.jobs_dev, ws, k0, 0);
    RBF_CHECK_LAUNCH();
  }
  return RBF_OK;
}

rbf_status lu_backward_step(LuGroup& G, int k0, double* ws) {
  if (k0 >= G.maxm) return RBF_OK;
  uinv_kernel<<<G.nj, kThreads, sm2_bytes(), G.s>>>(G.jobs_dev, ws, k0, G.linv);
  RBF_CHECK_LAUNCH();
  diag_solve_kernel<<<dim3(G.nj, std::max(1, std::min((G.maxnc + kNb - 1) / kNb, G.spread))), kThreads,
                      sm2_bytes(), G.s>>>(G.jobs_dev, ws, k0, G.linv);
  RBF_CHECK_LAUNCH();
  if (k0 > 0) {
    gemm_kernel<<<dim3(G.nj, std::max(1, std::min(tiles_of(k0, G.maxnc), G.spread))), kThreads, sm2_bytes(),
                  G.s>>>(G.jobs_dev, ws, k0, 1);
    RBF_CHECK_LAUNCH();
  }
  return RBF_OK;
}

}  // namespace

rbf_status batched_lu_restricted_inverse(rbf_ctx* ctx, const LuJob* jobs_dev, const std::vector<LuJob>& jobs,
                                         double* ws, double* W, int* info) {
  cudaStream_t s = ctx->stream;
  const int nj = (int)jobs.size();
  if (nj == 0) return RBF_OK;
  RBF_TRY(smem_limit_at_least(linv_kernel, sm2_bytes()));
  RBF_TRY(smem_limit_at_least(swap_trsm_kernel, smsw_bytes()));
  RBF_TRY(smem_limit_at_least(gemm_kernel, sm2_bytes()));
  RBF_TRY(smem_limit_at_least(diag_solve_kernel, sm2_bytes()));
  RBF_TRY(smem_limit_at_least(uinv_kernel, sm2_bytes()));
  RBF_CUDA_TRY(cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  DevBuf piv, linv;
  RBF_TRY(piv.alloc(sizeof(int) * (size_t)nj * kNb, s));
  RBF_TRY(linv.alloc(sizeof(double) * (size_t)nj * kNb * kNb, s));
  // two groups on two streams: one group's latency-bound panels (1 CTA/SM, 133 KB of
  // smem) co-run with the other's GEMMs (70 KB): the SM has room for both
  const int ngroups = nj >= 64 ? 2 : 1;
  if (ngroups == 2 && !ctx->aux_stream) {
    RBF_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
  }
  LuGroup Gs[2];
  int lo = 0;
  for (int gi = 0; gi < ngroups; ++gi) {
    const int hi = (gi + 1 == ngroups) ? nj : nj / 2;
    LuGroup& G = Gs[gi];
    G.s = gi == 0 ? s : ctx->aux_stream;
    G.jobs_dev = jobs_dev + lo;
    G.nj = hi - lo;
    G.maxm = G.maxnc = G.maxld = 0;
    for (int j = lo; j < hi; ++j) {
      G.maxm = std::max(G.maxm, jobs[j].m);
      G.maxnc = std::max(G.maxnc, jobs[j].nc);
      G.maxld = std::max(G.maxld, jobs[j].m + jobs[j].nc);
    }
    G.piv = piv.as<int>() + (size_t)lo * kNb;
    G.linv = linv.as<double>() + (size_t)lo * kNb * kNb;
    // CTAs per block along grid.y: enough to fill ~8 CTAs per SM, each looping over tiles
    G.spread = std::max(1, (ctx->sm_count * 8 / ngroups + G.nj - 1) / G.nj);
    // cluster size for the on-chip panel: rows per CTA R <= 256 (133 KB of smem)
    G.CL = 1;
    while (G.CL < 16 && (G.maxm + G.CL - 1) / G.CL > 256) G.CL *= 2;
    G.R = (G.maxm + G.CL - 1) / G.CL;
    const size_t smp = sizeof(double) * (size_t)G.R * kPs;
    G.pcfg = {};
    G.pcfg.gridDim = dim3((unsigned)(G.nj * G.CL));
    G.pcfg.blockDim = dim3(kThreads);
    G.pcfg.dynamicSmemBytes = smp;
    G.pcfg.stream = G.s;
    G.pattr[0].id = cudaLaunchAttributeClusterDimension;
    G.pattr[0].val.clusterDim.x = G.CL;
    G.pattr[0].val.clusterDim.y = 1;
    G.pattr[0].val.clusterDim.z = 1;
    G.pcfg.attrs = G.pattr;
    G.pcfg.numAttrs = 1;
    lo = hi;
  }
  // the panel kernel's smem attribute is per function: use the larger group's need
  {
    size_t need = 0;
    for (int gi = 0; gi < ngroups; ++gi) need = std::max(need, sizeof(double) * (size_t)Gs[gi].R * kPs);
    RBF_TRY(smem_limit_at_least(panel_cluster_kernel, need));
  }
  cudaEvent_t fork = nullptr, join = nullptr;
  if (ngroups == 2) {
    fork = ctx->take_event();
    join = ctx->take_event();
    RBF_CUDA_TRY(cudaEventRecord(fork, s));
    RBF_CUDA_TRY(cudaStreamWaitEvent(Gs[1].s, fork, 0));
  }
  int maxm = 0;
  for (int gi = 0; gi < ngroups; ++gi) maxm = std::max(maxm, Gs[gi].maxm);
  for (int k0 = 0; k0 < maxm; k0 += kNb)
    for (int gi = 0; gi < ngroups; ++gi) RBF_TRY(lu_forward_step(Gs[gi], k0, ws, info));
  for (int k0 = ((maxm - 1) / kNb) * kNb; k0 >= 0; k0 -= kNb)
    for (int gi = 0; gi < ngroups; ++gi) RBF_TRY(lu_backward_step(Gs[gi], k0, ws));
  for (int gi = 0; gi < ngroups; ++gi) {
    transpose_w_kernel<double><<<dim3(Gs[gi].nj, 64), 256, 0, Gs[gi].s>>>(Gs[gi].jobs_dev, ws, W);
    RBF_CHECK_LAUNCH();
  }
  if (ngroups == 2) {
    RBF_CUDA_TRY(cudaEventRecord(join, Gs[1].s));
    RBF_CUDA_TRY(cudaStreamWaitEvent(s, join, 0));
    ctx->ev_pool.push_back(fork);
    ctx->ev_pool.push_back(join);
  }
  return RBF_OK;
}

}  // namespace rbf
