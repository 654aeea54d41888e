// the ASSEMBLED operator, for comparison with the
// matrix-free summation.  The paper's GPU solve path assembles A once and runs
// sparse matrix-vector products (Alg.2 "truncation area"; PETSc
// AIJCUSP / CUSP CSR).  Here: CSR over the cell (sorted) order,
// rows = targets, columns = sources ascending, fp32 values + int32 columns
// (8 B per stored entry), int64 row pointers (c4 holds 1.02e10 entries = 82 GB).
//
// Entry set: pairs with r^2 <= c^2 evaluated in fp32 from the fp32 centres
// (d = x_j - x_i per axis, r^2 = (dx^2 + dy^2) + dz^2, compared with fp32(c^2));
// value a * 2^(-k r^2), k = log2(e)/(2 sigma^2), ex2.approx -- the fp32 tier's
// arithmetic, so the assembled product matches the fp32 matvec within its
// tolerance.  Assembly: a counting pass and an emitting pass, one thread per
// target row walking the cell rows within the cutoff (the same row ranges as
// the summation's traversal); row pointers by a host prefix sum (64-bit).
// SpMV: a warp per row, coalesced (column, value) streams, x gathered through
// L2 (12 MB at c4), warp-shuffle reduction.  HBM-bound: 8 B per entry.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <vector>

#include "internal.h"

struct rbf_csr {
  int64_t n = 0, nnz = 0;
  const rbf_cells* cells = nullptr;
  rbf::DevBuf row_ptr;   // int64[n+1]
  rbf::DevBuf col;       // int32[nnz]   sorted source positions
  rbf::DevBuf val;       // fp32[nnz]
  double t_assemble = 0.0;
};

namespace rbf {
namespace {

struct AsmGeom {
  float lo[3], inv_h, h;
  int dim[3];
  float c2;     // fp32(c^2)
  float cc;     // culling radius of the row ranges (cutoff inflated by rounding margins)
  float k;      // log2(e) / (2 sigma^2)
  float amp;
};

__device__ __forceinline__ int acell(float x, float lo, float inv_h, int dim) {
  float t = floorf((x - lo) * inv_h);
  t = fminf(fmaxf(t, -1.f), (float)dim);
  return min(max((int)t, 0), dim - 1);
}

// EMIT = false: count[i] = entries of row i; true: write them at row_ptr[i]
template <bool EMIT>
__global__ void __launch_bounds__(128)
assemble_kernel(AsmGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ sorted, int64_t n,
                uint32_t* __restrict__ count, const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col,
                float* __restrict__ val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 t = sorted[i];
    const int z0 = acell(t.z - G.cc, G.lo[2], G.inv_h, G.dim[2]), z1 = acell(t.z + G.cc, G.lo[2], G.inv_h, G.dim[2]);
    const int y0 = acell(t.y - G.cc, G.lo[1], G.inv_h, G.dim[1]), y1 = acell(t.y + G.cc, G.lo[1], G.inv_h, G.dim[1]);
    const int x0 = acell(t.x - G.cc, G.lo[0], G.inv_h, G.dim[0]), x1 = acell(t.x + G.cc, G.lo[0], G.inv_h, G.dim[0]);
    uint32_t cnt = 0;
    int64_t o = EMIT ? row_ptr[i] : 0;
    for (int cz = z0; cz <= z1; ++cz)
      for (int cy = y0; cy <= y1; ++cy) {
        const int64_t row = ((int64_t)cz * G.dim[1] + cy) * G.dim[0];
        const int s0 = cell_start[row + x0], s1 = cell_start[row + x1 + 1];
        for (int j = s0; j < s1; ++j) {
          const float4 p = __ldg(sorted + j);
          const float dx = __fsub_rn(p.x, t.x), dy = __fsub_rn(p.y, t.y), dz = __fsub_rn(p.z, t.z);
          const float r2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
          if (r2 <= G.c2) {
            if (EMIT) {
              float e;
              asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-G.k * r2));
              col[o] = j;
              val[o] = G.amp * e;
              ++o;
            } else {
              ++cnt;
            }
          }
        }
      }
    if (!EMIT) count[i] = cnt;
  }
}

// y[i] = sum_k val[k] x[col[k]] over row i (sorted order), a warp per row
template <class OutT>
__global__ void __launch_bounds__(256)
spmv_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col, const float* __restrict__ val,
            const float* __restrict__ x, int64_t n, OutT* __restrict__ y, const int32_t* __restrict__ out_perm) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
    const int64_t a = row_ptr[i], b = row_ptr[i + 1];
    float acc0 = 0.f, acc1 = 0.f;
    int64_t k = a + lane;
    for (; k + 32 < b; k += 64) {
      acc0 = fmaf(__ldg(val + k), __ldg(x + __ldg(col + k)), acc0);
      acc1 = fmaf(__ldg(val + k + 32), __ldg(x + __ldg(col + k + 32)), acc1);
    }
    if (k < b) acc0 = fmaf(__ldg(val + k), __ldg(x + __ldg(col + k)), acc0);
    float acc = acc0 + acc1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[out_perm ? out_perm[i] : i] = (OutT)acc;
  }
}

}  // namespace
}  // namespace rbf

using namespace rbf;

extern "C" {

rbf_status rbf_assemble(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, rbf_csr** out) {
  if (!ctx || !c || !kern || !out) { set_error("NULL argument"); return RBF_EINVAL; }
  *out = nullptr;
  if (!(kern->sigma > 0) || !(kern->cutoff_sigmas > 0)) { set_error("bad kernel"); return RBF_EINVAL; }
  if (kern->cutoff_sigmas * kern->sigma > c->cutoff * (1 + 1e-12)) {
    set_error("kernel cutoff exceeds the cutoff the cells were built for");
    return RBF_EINVAL;
  }
  if (ctx->world > 1) { set_error("the assembled operator is single-GPU"); return RBF_EUNSUPPORTED; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  cudaStream_t s = ctx->stream;
  const KernelParams kp = kernel_params(kern);
  AsmGeom G;
  for (int a = 0; a < 3; ++a) { G.lo[a] = c->lo[a]; G.dim[a] = c->dim[a]; }
  G.inv_h = c->inv_h;
  G.h = (float)c->h;
  G.c2 = (float)(kp.cutoff * kp.cutoff);
  double maxabs = 0;
  for (int a = 0; a < 3; ++a)
    maxabs = std::max(maxabs, std::max(std::fabs((double)c->lo[a]), std::fabs(c->lo[a] + c->dim[a] * c->h)));
  G.cc = (float)(kp.cutoff * (1.0 + 1e-5) + 4e-7 * maxabs);
  G.k = (float)(1.4426950408889634 / (2.0 * kp.sigma * kp.sigma));
  G.amp = (float)kp.amp;
  const int64_t n = c->n;
  rbf_csr* M = new (std::nothrow) rbf_csr();
  if (!M) { set_error("host allocation failed"); return RBF_ENOMEM; }
  M->n = n;
  M->cells = c;
  DevBuf cnt;
  rbf_status st = cnt.alloc(4 * n, s);
  if (st != RBF_OK) { delete M; return st; }
  const int blocks = grid_for(n, 128, 148 * 16);
  assemble_kernel<false><<<blocks, 128, 0, s>>>(G, c->cell_start.as<int32_t>(), c->sorted.as<float4>(), n,
                                                 cnt.as<uint32_t>(), nullptr, nullptr, nullptr);
  count_launch();
  std::vector<uint32_t> hc(n);
  std::vector<int64_t> hp(n + 1);
  cudaError_t e = cudaMemcpyAsync(hc.data(), cnt.p, 4 * n, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); delete M; return RBF_ECUDA; }
  hp[0] = 0;
  for (int64_t i = 0; i < n; ++i) hp[i + 1] = hp[i] + hc[i];
  M->nnz = hp[n];
  st = M->row_ptr.alloc(8 * (n + 1), s);
  if (st == RBF_OK) st = M->col.alloc(4 * (size_t)std::max<int64_t>(M->nnz, 1), s);
  if (st == RBF_OK) st = M->val.alloc(4 * (size_t)std::max<int64_t>(M->nnz, 1), s);
  if (st != RBF_OK) { delete M; return st; }
  e = cudaMemcpyAsync(M->row_ptr.p, hp.data(), 8 * (n + 1), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); delete M; return RBF_ECUDA; }
  assemble_kernel<true><<<blocks, 128, 0, s>>>(G, c->cell_start.as<int32_t>(), c->sorted.as<float4>(), n, nullptr,
                                                M->row_ptr.as<int64_t>(), M->col.as<int32_t>(), M->val.as<float>());
  count_launch();
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); delete M; return RBF_ECUDA; }
  M->t_assemble = std::chrono::duration<double>(clk::now() - t0).count();
  *out = M;
  return RBF_OK;
}

void rbf_csr_free(rbf_csr* m) { delete m; }

rbf_status rbf_csr_info(const rbf_csr* m, int64_t* nnz, int64_t* bytes, double* t_assemble) {
  if (!m) { set_error("NULL argument"); return RBF_EINVAL; }
  if (nnz) *nnz = m->nnz;
  if (bytes) *bytes = (int64_t)(m->row_ptr.bytes + m->col.bytes + m->val.bytes);
  if (t_assemble) *t_assemble = m->t_assemble;
  return RBF_OK;
}

rbf_status rbf_csr_spmv(rbf_ctx* ctx, const rbf_csr* m, const float* w, float* f) {
  if (!ctx || !m || !w || !f) { set_error("NULL argument"); return RBF_EINVAL; }
  if (w == f) { set_error("w and f must not alias"); return RBF_EINVAL; }
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const rbf_cells* c = m->cells;
  const int64_t n = m->n;
  RBF_TRY(ctx->vec_a.ensure(sizeof(float) * n, s));
  RBF_TRY(gather_f32_to_sorted(ctx, w, c->perm.as<int32_t>(), ctx->vec_a.as<float>(), n));
  spmv_kernel<float><<<grid_for(n * 32, 256, 148 * 16), 256, 0, s>>>(
      m->row_ptr.as<int64_t>(), m->col.as<int32_t>(), m->val.as<float>(), ctx->vec_a.as<float>(), n, f,
      c->perm.as<int32_t>());
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}

}  // extern "C"
