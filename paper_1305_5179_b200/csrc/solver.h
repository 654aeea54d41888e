// Internal declarations of the preconditioner and the Krylov solver.
#pragma once
#include <vector>

#include "internal.h"

struct rbf_precond {
  int kind = 2;
  int64_t n = 0;
  int64_t nblocks = 0;
  int64_t bytes = 0;
  int max_m = 0;
  int singular_blocks = 0;
  double shift = 0.0;     // diagonal shift of the local matrices, units of the amplitude a
  bool w_fp32 = false;    // W stored in fp32 (local_fp32)
  int64_t gj_blocks = 0;  // blocks inverted on chip in fp32 (the rest by the fp64 batched LU)
  bool w_sym = false;     // W_i stored as packed lower triangles (block-Jacobi, fp32 W: W_i = B_i^-1 symmetric)
  int64_t max_wblk = 0;   // floats of the largest W_i
  int cap_w = 6144;       // apply staging size (floats; w_sym)
  // w_sym apply: per-block records {e0, w0, m, nfl} (32 bytes) in launch order:
  // up to 4 launch bins by triangle size, each launched with the stage its
  // triangles need (small triangles: more CTAs per SM; big ones: staged instead
  // of read from global)
  rbf::DevBuf ameta;
  int nbins = 0;
  int64_t bin_first[5] = {0, 0, 0, 0, 0};   // records [bin_first[k], bin_first[k + 1])
  int bin_cap[4] = {0, 0, 0, 0};             // stage size, floats
  int bin_m[4] = {0, 0, 0, 0};               // largest block of the bin
  double t_setup = 0.0;
  bool halo = false;      // slab partition with overlap: indices relative to the window start h0
  int shift_idx = 0;      // o0 - (index origin): 0 unless halo
  const rbf_cells* cells = nullptr;
  rbf::DevBuf core_ptr;   // int64[nblocks+1]
  rbf::DevBuf ext_ptr;    // int64[nblocks+1]
  rbf::DevBuf core_idx;   // int32[n]           sorted positions, block-major
  rbf::DevBuf ext_idx;    // int32[ext_ptr[nb]] sorted positions: [extra ascending] + [core]
  rbf::DevBuf w_off;      // int64[nblocks+1]   float offsets of W_i
  rbf::DevBuf W;          // fp64 or fp32 (w_fp32): W_i (nc_i x m_i) row-major = (B_i^-1)[core, :]
                          // (w_sym: row i of the lower triangle at i(i+1)/2, blocks padded to 4 floats),
                          // B_i = A_ext + shift*a*I
  std::vector<int64_t> h_core_ptr, h_ext_ptr;
};

namespace rbf {

// One RAS block of a factorisation chunk (lu_batched.cu).
struct LuJob {
  int64_t ws_off;   // element offset of the augmented matrix [A_ext | E_core] in the workspace
  int64_t ext_off;  // offset into ext_idx
  int64_t w_off;    // element offset of W (nc x m) in the W buffer
  int m, nc;
};
// Factor every job's [A_ext | E_core] (fp64, partial pivoting) and write
// W = (A_ext^-1)[core, :] (fp64, nc x m row-major) at W + w_off.
rbf_status batched_lu_restricted_inverse(rbf_ctx* ctx, const LuJob* jobs_dev, const std::vector<LuJob>& jobs,
                                         double* ws, double* W, int* info);

rbf_status precond_build(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp, const rbf_precond_cfg* cfg,
                         rbf_precond* P);
// z = M r in sorted order (r, z fp32 or fp64; never aliased)
template <class VT>
rbf_status precond_apply_sorted(rbf_ctx* ctx, const rbf_precond* P, const VT* r, VT* z);

// fp32-tier matvec with fp64 input/output vectors in sorted order
rbf_status matvec_sorted_f32_d(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp, const double* w_sorted,
                               double* f_sorted, int op = RBF_OP_ONESIDED);
// the same with fp32 input weights (the fp32-phase Krylov basis)
rbf_status matvec_sorted_f32_f(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp, const float* w_sorted,
                               double* f_sorted, int op);

}  // namespace rbf
