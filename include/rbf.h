/*
 * rbf.h -- C-ABI of the B200-native Gaussian-RBF implicit-surface hot path.
 *
 * Method: Cuomo, Galletti, Giunta, Starace, "Surface reconstruction from
 * scattered point via RBF interpolation on GPU" (arXiv 1305.5179).
 * Citations "P:<lines>" are lines of that paper's text with the
 * section / equation / algorithm they fall in.
 *
 * What the library computes (all on the GPU; there is no CPU fallback):
 *
 *   centres   x_1..x_n in R^3 (fp32; for the paper's problem n = 3N: the
 *             surface points X and their +/-delta normal offsets
 *             §2.1.1; building that set is the caller's job)
 *   operator  A_ij = a * exp(-||x_i - x_j||^2 / (2 sigma^2))   if ||x_i-x_j|| <= c
 *             A_ij = 0                                          otherwise
 *             a = 1/(sqrt(2 pi) sigma) by default (Eq.6; Table I
 *             P:299); c = cutoff_sigmas * sigma (the "finite bandwidth" of
 *             P:361-369; reading R5: inclusive, c = 6 sigma)
 *   matvec    f = A w                                   (Eq.4)
 *   solve     A w = b by restarted right-preconditioned GMRES with a
 *             restricted additive Schwarz (RAS) preconditioner
 *                                                       (§3.1)
 *   evaluate  F(xi_k) = sum_j A(xi_k, x_j) w_j on a regular grid
 *                                                       (Eq.5, P:264-271;
 *                                                        §2.1.3)
 *
 * Conventions (apply to every entry point):
 *  - Device pointers are caller-owned device memory (cudaMalloc / torch),
 *    host pointers are plain host memory; each argument says which.
 *  - Every call is stream-ordered on the context's stream; calls only
 *    synchronise where they must return host values (documented per call).
 *  - Vectors are indexed in the CALLER's order of the centres passed to
 *    rbf_build_cells (internal cell order is hidden) unless stated otherwise.
 *  - Errors: functions return rbf_status; on error nothing is written to the
 *    output buffers' contents that the caller may rely on, and
 *    rbf_last_error() returns a human-readable message (thread-local).
 *    Non-convergence of GMRES is NOT an error (see rbf_solve_report).
 *  - Handles (rbf_ctx, rbf_cells, rbf_precond) are library-owned and freed by
 *    their *_free / rbf_destroy call.  One rbf_ctx per host thread.
 */
#ifndef RBF_B200_H
#define RBF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBF_ABI_VERSION 3

typedef enum {
  RBF_OK = 0,
  RBF_EINVAL = 1,   /* invalid argument (sizes, sigma <= 0, non-finite input, ...) */
  RBF_ENOMEM = 2,   /* device allocation failed */
  RBF_ECUDA = 3,    /* CUDA runtime error (message in rbf_last_error) */
  RBF_ENCCL = 4,    /* reserved for the multi-GPU layer */
  RBF_EUNSUPPORTED = 5
} rbf_status;

typedef enum { RBF_F32 = 0, RBF_F64 = 1 } rbf_precision;

/* Evaluation order of the solver's operator f = A w (reading R19).
 * A = A^T, so a kernel may evaluate each exponential of a pair (i, j) once and
 * add it to both f_i and f_j ("symmetric"): half the exponentials, but the
 * source-side sums land with atomicAdd, so f is reproducible only to the last
 * bits run to run.  "One-sided" evaluates every ordered pair and writes each f_i
 * once: bit-reproducible for a fixed device and launch configuration.
 *   RBF_OP_AUTO      symmetric on the wide (128-target) plan for >= 2^18 centres
 *                    per GPU, one-sided below (the benchmarked default)
 *   RBF_OP_ONESIDED  one-sided fp32 and fp64 tiers: a DETERMINISTIC solve
 *   RBF_OP_SYM       symmetric on the 64-target plan
 *   RBF_OP_SYM_WIDE  symmetric on the wide plan (fp64 tier: the 64-target plan)
 *   RBF_OP_SYM_ROT   as RBF_OP_SYM_WIDE with the source side summed by a rotating
 *                    accumulator instead of a warp transpose-reduction
 * The public rbf_matvec is always one-sided; rbf_matvec_op exposes the others. */
typedef enum {
  RBF_OP_AUTO = 0, RBF_OP_ONESIDED = 1, RBF_OP_SYM = 2, RBF_OP_SYM_WIDE = 3, RBF_OP_SYM_ROT = 4
} rbf_op_variant;

/* Gaussian kernel of Eq.6 with truncation radius
 * cutoff_sigmas*sigma.  amplitude <= 0 selects Eq.6's
 * a = 1/(sqrt(2 pi) sigma). */
typedef struct {
  double sigma;          /* > 0 */
  double cutoff_sigmas;  /* > 0; the configs use 6 */
  double amplitude;      /* <= 0 => 1/(sqrt(2 pi) sigma) */
} rbf_kernel;

/* Cell binning of the centres ("truncation area", Alg.2).
 * Cell edge h; frame lo (fp32) and inv_h = float32(1/h):
 *   lo_a  = float32(double(min_a x) - h/2),  dim_a = floor(f32(f32(max_a x - lo_a) * inv_h)) + 1
 *   cell_a(x) = clamp(floor(f32(f32(x_a - lo_a) * inv_h)), 0, dim_a - 1)
 *   key = cx + dimx*(cy + dimy*cz);   cells sorted stably by key.
 * (bit-exact with oracle/cells.py.) */
typedef struct {
  double cell_edge;      /* <= 0 => cutoff / 3.999 (4 cells
                            per cutoff with a rounding margin) */
  int tile_cap;          /* targets per warp tile, 32 or 64; <= 0 => 64 */
  int tile_span;         /* max cells a tile spans along x; <= 0 => 2 */
  int tile_mode;         /* 0 => full cap-sized chunks of cell runs (default),
                            1 => whole cells merged greedily */
} rbf_cell_cfg;

/* RAS preconditioner (§3.1; readings R8, R9, R17).
 * The local systems are A_i + shift*a*I (a = the kernel amplitude).  shift = 0
 * gives the paper's exact local solves; shift > 0 (reading R17) keeps the local
 * inverses bounded when sigma/spacing makes A_i numerically singular (the
 * preconditioner stays an approximation of A^-1 either way; GMRES iterates
 * with the unshifted A).  local_fp32 = 1 factors every block with m <= 224 on
 * chip in fp32 (Gauss-Jordan; without pivoting when shift >= 1e-4, where the
 * shifted block is symmetric positive definite, with partial pivoting below) and
 * stores W in fp32 (block-Jacobi: only the lower triangle of the symmetric
 * W_i = B_i^-1, half the bytes reported by rbf_precond_blocks); it is accurate
 * only when shift*a dominates fp32 rounding of A_i (shift >= ~1e-4).  Larger
 * blocks (their fp64 LU inverse rounded into the fp32 W), and local_fp32 = 0,
 * use the fp64 batched LU; local_fp32 = 0 keeps fp64 W. */
typedef struct {
  int kind;              /* 0 none, 1 block-Jacobi (overlap 0), 2 RAS */
  int core_target;       /* centres per core (whole cells); <= 0 => 512 */
  double overlap_sigmas; /* extended set = centres within overlap*sigma of the core */
  int max_ext;           /* reject blocks larger than this; <= 0 => 4096 */
  double shift;          /* >= 0; diagonal shift of the local matrices in units of a */
  int local_fp32;        /* 0 => fp64 LU + fp64 W; 1 => fp32 on-chip inverse + fp32 W */
  int pivot;             /* on-chip fp32 inverses: 0 => auto (partial pivoting iff
                            shift < 1e-4), 1 => always pivot, 2 => never */
  int w_layout;          /* fp32 block-Jacobi W: 0 => auto (packed lower triangles of
                            the symmetric W_i), 1 => full rows */
} rbf_precond_cfg;

/* Restarted right-preconditioned FGMRES(m).
 * Phase 1 iterates with the fp32 operator tier down to phase1_rtol of the
 * TRUE relative residual; phase 2 continues with the fp64 operator tier and
 * fp64 vectors until ||b - A w||_2 / ||b||_2 <= rtol (fp64 operator). */
typedef struct {
  int restart;           /* m; <= 0 => 30 */
  double rtol;           /* final true relative residual; <= 0 => 1e-6 */
  double phase1_rtol;    /* <= 0 => 1e-4 */
  int max_iters;         /* total inner iterations; <= 0 => 500 */
  int polish_fp64;       /* 1 => phase 2 in fp64 (needed for rtol < ~1e-5) */
  int cgs_passes;        /* Gram-Schmidt passes per Arnoldi step: 1 (CGS) or 2 (CGS2); other => 2 */
  int op_variant;        /* rbf_op_variant of the operator; RBF_OP_ONESIDED => deterministic */
  int basis_fp64;        /* 1 => fp64 Krylov basis in phase 1 too (default: fp32 basis there) */
  /* Residual history (HOST, caller-allocated, may be NULL; filled up to
   * history_cap entries, lengths in rbf_solve_report):
   *   history[i]      Arnoldi estimate |g_{j+1}| / ||b|| after inner iteration i+1
   *   history_true[k] true relative residual ||b - A w|| / ||b|| at the start of
   *                   restart cycle k (operator tier of that cycle), then the final one */
  double* history;
  double* history_true;
  int history_cap;
  /* Initial guess (DEVICE fp64, caller order, n entries; NULL => zero): resumes a
   * solve from a checkpointed w (e.g. a restart boundary); the first
   * residual is the true b - A x0 of the fp32 tier (fp64 once phase 2 starts).
   * Not read by rbf_gmres_solve_shard (which starts from zero). */
  const double* x0;
} rbf_gmres_cfg;

typedef struct {
  int iters_phase1, iters_phase2, restarts, converged, breakdown;
  int history_len, history_true_len;
  double rel_residual_true;   /* ||b - A w|| / ||b|| with the fp64 operator */
  double rel_residual_est;    /* GMRES (Arnoldi) estimate at exit */
  double t_setup, t_phase1, t_phase2;  /* seconds (host clock around device work) */
  int64_t nblocks;            /* RAS blocks */
  int64_t precond_bytes;      /* device bytes held by the preconditioner */
  int64_t matvecs_f32, matvecs_f64;
} rbf_solve_report;

/* Regular evaluation grid: n[a] >= 2 inclusive nodes per axis from lo[a] to
 * hi[a]; node (i,j,k) = lo + (i,j,k)*(hi-lo)/(n-1) (computed in fp64 then
 * rounded to fp32); flat index i + n0*(j + n1*k) (x fastest). */
typedef struct {
  double lo[3], hi[3];
  int n[3];
} rbf_grid;

typedef struct rbf_ctx rbf_ctx;
typedef struct rbf_cells rbf_cells;
typedef struct rbf_precond rbf_precond;
typedef struct rbf_csr rbf_csr;
typedef struct rbf_loopback_group rbf_loopback_group;

/* Description of a built cell list (host struct, filled by rbf_cells_info). */
typedef struct {
  int64_t n;             /* centres */
  int dim[3];
  float lo[3];
  float inv_h;
  double cell_edge;
  int reach;             /* stencil reach in cells (>= ceil(cutoff/h)) */
  int64_t ncell;         /* dim0*dim1*dim2 */
  int64_t ntiles;        /* matvec target tiles */
  int64_t nonempty_cells;
} rbf_cells_desc;

/* ---- context ------------------------------------------------------------ */

/* Create a context on CUDA device `device` that issues all work on
 * `cuda_stream` (a cudaStream_t; NULL = the legacy default stream).
 * world == 1: single GPU (nccl_unique_id ignored, rank must be 0).
 * world > 1: one process (context) per GPU, `rank` in [0, world), and
 * nccl_unique_id = the 128-byte id rank 0 obtained from rbf_nccl_unique_id(),
 * broadcast to every rank by the caller (e.g. torch.distributed).  The context
 * then partitions every call by slabs of cell planes (DESIGN.md
 * "Multi-GPU"): inputs are REPLICATED (every rank passes the full centre set,
 * right-hand side and weights), the work and the solver state are sharded, and
 * outputs (weights, matvec results, grid field) are returned full on every rank.
 * NCCL (libnccl.so.2) is loaded at run time, only when world > 1.
 * Errors: RBF_EINVAL (bad device / rank / world, missing id), RBF_ECUDA,
 * RBF_ENCCL (NCCL unavailable or communicator init failed). */
rbf_status rbf_create(rbf_ctx** ctx, int device, void* cuda_stream,
                      const void* nccl_unique_id, int rank, int world);
/* 128 bytes (HOST) of a fresh NCCL unique id, for rank 0 to share.  RBF_ENCCL if
 * NCCL cannot be loaded. */
rbf_status rbf_nccl_unique_id(void* out128);
/* In-process loopback transport: `world` contexts of ONE process on one device,
 * each driven by its own host thread, run the multi-rank slab partition exactly
 * as world GPUs would (same partition, halos, reductions and gathers; copies
 * between the ranks' buffers and a rank-ordered sum kernel instead of NCCL,
 * ordered by CUDA events and a host barrier).  For tests and single-GPU runs of
 * the distributed code path.  Create the group once (library-owned, free it
 * after every context of it is destroyed), then one rbf_create_loopback per
 * rank with distinct streams; every rank must make the same sequence of calls
 * (a call blocks until all ranks have reached it).  Errors: RBF_EINVAL (world
 * outside [1, 64], rank out of range or already joined), RBF_ECUDA. */
rbf_status rbf_loopback_group_create(int world, rbf_loopback_group** out);
void rbf_loopback_group_free(rbf_loopback_group* g);
rbf_status rbf_create_loopback(rbf_ctx** ctx, int device, void* cuda_stream, rbf_loopback_group* g, int rank);
/* Peer-memory transport (one process per GPU on ONE node, NCCL not used): the
 * ranks' exchange arenas are mapped into each other by CUDA IPC (NVLink /
 * NVSwitch peer access; several processes may also share one device, for
 * tests), transfers are cudaMemcpyAsync between device pointers (copy engines),
 * the all-reduce is a rank-ordered sum kernel over every rank's arena, and
 * ordering is by interprocess CUDA events plus a host barrier in POSIX shared
 * memory (no kernel waits on another rank).  key16: 16 HOST bytes, identical on
 * every rank and fresh per group (rank 0 draws them and shares them, e.g. over
 * torch.distributed); it names the shared-memory segment.  Every rank must make
 * the same sequence of calls; a rank that does not arrive makes the others fail
 * with RBF_ECUDA after 600 s.  Errors: RBF_EINVAL (rank/world, segment setup),
 * RBF_ECUDA (IPC or event calls, barrier timeout). */
rbf_status rbf_create_ipc(rbf_ctx** ctx, int device, void* cuda_stream, const void* key16, int rank, int world);
/* Peer-memory form of the solver's symmetric fp32 operator (on by default; used
 * when the context's transport can address the other ranks' device memory --
 * loopback and CUDA IPC, not NCCL): ONE summation kernel per rank reads the upper
 * ranks' packed sources and atomically adds the source-side sums into their
 * accumulators directly (NVLink / NVSwitch peer memory) instead of a halo
 * exchange before the kernel and a reverse halo reduction after it; the ranks
 * are ordered by events and a host barrier before and after the kernels.  on = 0
 * keeps the copy-based halo (the NCCL path's form) on any transport.  Results
 * are the same up to the atomics' summation order. */
rbf_status rbf_ctx_peer_memory(rbf_ctx* ctx, int on);
/* Neighbour-list form of the solver's symmetric fp32 operator (RBF_OP_SYM_WIDE,
 * and RBF_OP_AUTO where it selects it; on by default).  The first product with
 * a cell structure lists, for every target tile of the wide plan, the sorted
 * positions of the sources after the tile that survive the tile's box cull
 * (the same cell rows, cull and order as the traversal; Alg.2 "truncation
 * area") and keeps the list with the cells (DEVICE memory owned by
 * the library, 4 bytes per listed source: 0.33 GB at 3M centres, sigma = 0.01);
 * later products read the list instead of re-walking and re-culling the cell
 * rows.  on = 0 runs the traversal every time.  The list is rebuilt when the
 * kernel's cutoff or the source window changes, and skipped (traversal form)
 * when it would exceed 2^31 entries or does not fit in memory.  Results equal
 * the traversal form's up to the atomics' summation order. */
rbf_status rbf_ctx_neighbour_lists(rbf_ctx* ctx, int on);
/* Separable form of the grid evaluation (default on).  The evaluation points of
 * Eq.5 are a regular grid, so for a 4 x 4 x 4 block of
 * nodes the Gaussian of a (node, centre) pair factors along the axes,
 * exp(-|xi - x_j|^2 / (2 sigma^2)) = ex[i] ey[j] ez[k]: 12 exponentials per
 * (block, centre) instead of 64; the cutoff predicate r^2 <= (6 sigma)^2 is
 * still evaluated per pair (reading R5: exact zeros beyond the cutoff).  on = 0
 * evaluates one exponential per pair (the matvec kernels' form).  Both forms
 * satisfy the same per-node tolerance against the fp64 definition; they differ
 * from each other by rounding (three ex2.approx factors instead of one).
 * Applies to rbf_eval_grid, rbf_eval_grid_masked, rbf_eval_grid_slab,
 * rbf_isosurface and rbf_reconstruct_host. */
rbf_status rbf_ctx_grid_separable(rbf_ctx* ctx, int on);
/* Slab partition plan (HOST only, no GPU; the same function the library runs at
 * rbf_build_cells when world > 1).  Inputs: plane_start[dimz+1] = sorted
 * position of the first centre of each z cell plane (non-decreasing, last =
 * n), plane_weight[dimz] >= 0 (the library uses sum over the plane's cells of
 * n_c^2, an estimate of its useful pairs), reach = planes a target's cutoff can
 * span.  Outputs (HOST, caller-allocated): plane_lo[world+1] (rank r owns planes
 * [plane_lo[r], plane_lo[r+1]), cut where the cumulative weight crosses r/world),
 * own_lo/own_hi[world] (owned sorted range), win_lo/win_hi[world] (matvec source
 * window = planes [plane_lo[r] - reach, plane_lo[r+1] + reach) clipped; empty
 * for an empty slab).  Any output may be NULL.  Errors: RBF_EINVAL. */
rbf_status rbf_slab_plan(const int64_t* plane_start, const double* plane_weight, int dimz, int reach, int world,
                         int32_t* plane_lo, int64_t* own_lo, int64_t* own_hi, int64_t* win_lo, int64_t* win_hi);
void rbf_destroy(rbf_ctx* ctx);
const char* rbf_status_str(rbf_status s);
const char* rbf_last_error(void);
int rbf_abi_version(void);
/* Number of CUDA kernels this library has launched in the process so far
 * (all contexts); host-side counter, no synchronisation. */
int64_t rbf_launch_count(void);
/* Device memory pool of the library on the context's device (one private
 * stream-ordered pool per device, never trimmed while the process lives).
 * rbf_pool_reserve makes sure the pool holds a free block of at least `bytes`
 * now (one allocation of that size, freed back into the pool at once: the pool
 * grows by what its free blocks cannot serve contiguously), so that later
 * calls carve their buffers out of it instead of asking the driver for memory
 * in the middle of a solve -- a driver allocation can take hundreds of
 * milliseconds right after another process released tens of GB on the device.
 * rbf_pool_stats: out[0] = bytes of backing memory the pool holds, out[1] =
 * bytes currently handed out (HOST, 2 values).  Errors: RBF_EINVAL, RBF_ENOMEM
 * (the device cannot back `bytes`), RBF_ECUDA. */
rbf_status rbf_pool_reserve(rbf_ctx* ctx, uint64_t bytes);
rbf_status rbf_pool_stats(rbf_ctx* ctx, uint64_t* out);

/* ---- a0: extended interpolation set (§2.1.1-2.1.2) ------------
 * x, nrm: DEVICE fp64, N x 3 (surface points and unit normals).
 * centres: DEVICE fp32, 3N x 3 = [x; x + delta n; x - delta n], each sum formed
 * in fp64 (one multiply, one add) and rounded once to fp32.
 * b: DEVICE fp32, 3N = [0 x N; +label x N; -label x N] (P:186-193 uses
 * label 1; the benchmark configs use label = delta, reading R2).
 * b may be NULL.  Errors: RBF_EINVAL for N < 1 or NULL x/nrm/centres. */
rbf_status rbf_extend_points(rbf_ctx* ctx, const double* x, const double* nrm, int64_t N,
                             double delta, double label, float* centres, float* b);

/* ---- a1/a2: cell build + tile plan (Alg.2 "truncation area") -------------
 * xyz: DEVICE, n x 3 fp32 row-major (x0,y0,z0,x1,...), caller-owned, read only
 * during the call.  n >= 1.  Non-finite coordinates => RBF_EINVAL.
 * Synchronises once (reads back the bounding box to size the grid of cells).
 * *out receives a library-owned handle (free with rbf_cells_free). */
/* Sharded input: rank r passes its shard of the caller-order
 * centres, xyz_local (DEVICE fp32 n_local x 3) = global ids [id0, id0 + n_local);
 * the shards of all ranks must tile [0, n_total) (any assignment of ranges to
 * ranks, ranks with n_local = 0 allowed).  The library gathers the shards
 * (transport exchange) and builds the same cells as rbf_build_cells on the full
 * array -- every rank holds the replicated geometry, the work stays sharded
 * (reading R22).  Single GPU: id0 = 0, n_local = n.  Errors as
 * rbf_build_cells, plus RBF_EINVAL when the shards do not tile [0, n_total). */
rbf_status rbf_build_cells_shard(rbf_ctx* ctx, const float* xyz_local, int64_t n_local, int64_t id0,
                                 const rbf_kernel* kern, const rbf_cell_cfg* cfg, rbf_cells** out);
rbf_status rbf_build_cells(rbf_ctx* ctx, const float* xyz, int64_t n,
                           const rbf_kernel* kern, const rbf_cell_cfg* cfg,
                           rbf_cells** out);
void rbf_cells_free(rbf_cells* cells);
rbf_status rbf_cells_info(const rbf_cells* cells, rbf_cells_desc* out /* host */);
/* This rank's slab (HOST out[11]): owned sorted range [out[0], out[1]), matvec
 * source window [out[2], out[3]), target tiles [out[4], out[5]), z cell planes
 * [out[6], out[7]), tiles of the wide (symmetric) plan [out[8], out[9]), of which
 * the first out[10] are interior: their traversal stays inside the slab, so the
 * symmetric fp32 operator runs them while the halo is exchanged on a second
 * stream (world > 1; 0 on one GPU).  Single GPU: everything. */
rbf_status rbf_cells_slab(const rbf_cells* cells, int64_t* out);
/* Library-owned DEVICE arrays, valid until rbf_cells_free:
 *   perm[n]           sorted position -> caller index (stable by key)
 *   sorted[4n]        float4 records (x, y, z, 0) in sorted order
 *   keys[n]           uint32 cell key per sorted position
 *   cell_start[ncell+1]  cell k holds sorted positions [cell_start[k], cell_start[k+1])
 *                        (= searchsorted left of k; cell_end = cell_start + 1) */
rbf_status rbf_cells_view(const rbf_cells* cells, const int32_t** perm,
                          const float** sorted, const uint32_t** keys,
                          const int32_t** cell_start);

/* ---- a3: matrix-free matvec f = A w (Eq.4/Eq.6) ---------------------------
 * w, f: DEVICE, n entries, caller order; fp32 (RBF_F32) or fp64 (RBF_F64).
 * RBF_F32: fp32 coordinates differences in tile-local scaled frame,
 * ex2.approx, fp32 accumulation.
 * RBF_F64: fp64 distances (same rounding order as the oracle), fp64 exp,
 * fp64 weights and accumulation.  w and f must not alias. */
rbf_status rbf_matvec(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern,
                      rbf_precision prec, const void* w, void* f);
/* The same product through the solver's operator variant `op` (rbf_op_variant):
 * what rbf_gmres_solve multiplies with under that setting.  RBF_F32: w is rounded
 * to fp32 inside (as the solver's fp32 tier does), f fp32; RBF_F64: fp64. */
rbf_status rbf_matvec_op(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern,
                         rbf_precision prec, int op, const void* w, void* f);

/* Pair accounting of the fp32 matvec traversal (host outputs; synchronises):
 * useful = ordered (target, source) pairs with r^2 <= c^2 (self included),
 * visited = pairs the kernel evaluated (after culling).  world > 1: the pairs
 * of this rank's targets (sum over ranks = the whole product). */
rbf_status rbf_matvec_pairs(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern,
                            int64_t* useful, int64_t* visited);

/* ---- a4/a5: RAS preconditioner (§3.1) -------------------------------------
 * Builds blocks (cores = runs of whole non-empty cells in Morton order of
 * ~core_target centres; extended set = centres within overlap of a core
 * centre), assembles each local matrix B_i = A_ext + shift*a*I from the fp32
 * centres (entries formed in fp64), inverts it with partial pivoting (the
 * truncated block may be indefinite) and keeps the restricted inverse
 * W_i = (B_i^-1)[core, :] (fp64, or fp32 with local_fp32; see rbf_precond_cfg).
 * Synchronises.  Errors: RBF_EINVAL (kind outside 0..2, shift < 0 or
 * non-finite, overlap < 0), RBF_EUNSUPPORTED (a block exceeds max_ext). */
rbf_status rbf_precond_create(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern,
                              const rbf_precond_cfg* cfg, rbf_precond** out);
void rbf_precond_free(rbf_precond* p);
/* z = M r, M = sum_i R~_i^T A_i^-1 R_i (restricted: only core rows written).
 * r, z: DEVICE fp32, n entries, caller order.  world > 1: r replicated, each
 * rank applies the blocks of its slab (their extended sets reach into the
 * neighbouring slabs through the halo: the paper's distributed RASM) and z is
 * gathered on every rank. */
rbf_status rbf_precond_apply(rbf_ctx* ctx, const rbf_precond* p, const float* r, float* z);
/* Block structure (host outputs, synchronises): nblocks, and if the arrays are
 * non-NULL: core_ptr[nblocks+1], ext_ptr[nblocks+1] (host, caller-allocated)
 * and core_idx[core_ptr[nb]], ext_idx[ext_ptr[nb]] (host) holding SORTED
 * positions relative to this rank's owned start (0 on one GPU; a distributed
 * RAS block's ext members in the slab below are negative); each block's ext
 * list is [non-core members ascending] + [core]. */
rbf_status rbf_precond_blocks(const rbf_precond* p, int64_t* nblocks, int64_t* bytes,
                              int64_t* core_ptr, int64_t* ext_ptr,
                              int32_t* core_idx, int32_t* ext_idx);

/* ---- a6/a7: GMRES solve A w = b ------------------------------------------
 * b: DEVICE fp32 (n), w: DEVICE fp64 (n) output, both caller order; rep: HOST.
 * precond may be NULL (then pcfg builds one internally, freed on return).
 * Synchronises (returns the report).  Non-convergence: RBF_OK, converged=0. */
rbf_status rbf_gmres_solve(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern,
                           const rbf_precond* precond, const rbf_precond_cfg* pcfg,
                           const rbf_gmres_cfg* gcfg, const float* b, double* w,
                           rbf_solve_report* rep);

/* Sharded form of rbf_gmres_solve: b_local (DEVICE fp32) is this rank's shard
 * [id0, id0 + n_local) of the caller-order right-hand side, w_local (DEVICE
 * fp64) receives the same shard of the weights; the shards tile [0, n) as in
 * rbf_build_cells_shard (n = the cells' centre count, else RBF_EINVAL).
 * Synchronises; report as rbf_gmres_solve. */
rbf_status rbf_gmres_solve_shard(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern,
                                 const rbf_precond* precond, const rbf_precond_cfg* pcfg, const rbf_gmres_cfg* gcfg,
                                 const float* b_local, int64_t n_local, int64_t id0, double* w_local,
                                 rbf_solve_report* rep);

/* ---- a8: grid evaluation F(xi) = sum_j A(xi, x_j) w_j (Eq.5) --------------
 * w: DEVICE fp64 (n, caller order); field: DEVICE fp32, n0*n1*n2, x fastest.
 * Nodes with no centre within the cutoff get exactly 0.0f.  world > 1: each
 * rank evaluates the node layers of its slab and gathers the other ranks'
 * layers, so every rank returns the full field. */
rbf_status rbf_eval_grid(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern,
                         const double* w, const rbf_grid* grid, float* field);
/* The sharded form: only this rank's z layers [*k0, *k1) of nodes (k = z index)
 * are written (field is still the full n0*n1*n2 array; the other layers are
 * untouched), no gather.  rbf_eval_grid = this + a gather of every rank's
 * layers.  Single GPU: all layers. */
rbf_status rbf_eval_grid_slab(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern,
                              const double* w, const rbf_grid* grid, float* field, int64_t* k0, int64_t* k1);

/* ---- the ASSEMBLED operator, for comparison ---------
 * The paper's GPU path assembles A (Alg.2 "truncation area") and
 * multiplies it as a sparse matrix (PETSc AIJCUSP).  rbf_assemble
 * builds that CSR on the device (library-owned; single GPU): rows = targets and
 * columns = sources in the cell (sorted) order, entries for fp32 r^2 <= fp32(c^2)
 * from the fp32 centres with value a * 2^(-k r^2) (the fp32 tier's arithmetic),
 * fp32 values + int32 columns (8 B per entry) + int64 row pointers.  Needs
 * 8 * nnz bytes of device memory (c4: 1.02e10 entries = 82 GB): RBF_ENOMEM if it
 * does not fit.  Synchronises.  rbf_csr_spmv: f = A w with w, f DEVICE fp32 in
 * the caller's order (same conventions as rbf_matvec(RBF_F32)).
 * rbf_csr_info: nnz, device bytes, assembly seconds (HOST outputs, any NULL). */
rbf_status rbf_assemble(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern, rbf_csr** out);
void rbf_csr_free(rbf_csr* m);
rbf_status rbf_csr_info(const rbf_csr* m, int64_t* nnz, int64_t* bytes, double* t_assemble);
rbf_status rbf_csr_spmv(rbf_ctx* ctx, const rbf_csr* m, const float* w, float* f);

/* ---- masked zero set of the interpolant (§2.1.3) ----------------
 * The surface is the zero level set of P_f restricted to the eps-surrounding
 * of the data, M* ~ M_ext^eps cap S_0 (reading R11).
 * field: DEVICE fp32 values of P_f on `grid` (x fastest, as rbf_eval_grid
 * writes them); data: DEVICE fp64 ndata x 3 (the surface points X, NOT the
 * +/-delta offsets); eps > 0.  For each grid edge (a, b) along x, then y, then
 * z, in order of the lower node's flat index: if F_a * F_b < 0 (fp64) and both
 * nodes lie within eps of a data point (fp64 distances), the point
 * p_a + t (p_b - p_a), t = F_a / (F_a - F_b), is written to points (DEVICE
 * fp64, row-major x,y,z; at most cap rows).  *count (HOST) receives the total
 * number of crossings (may exceed cap: call again with a larger buffer).
 * Synchronises.  Errors: RBF_EINVAL (NULLs, eps <= 0, bad grid, non-finite data). */
rbf_status rbf_zero_set(rbf_ctx* ctx, const float* field, const rbf_grid* grid, const double* data,
                        int64_t ndata, double eps, double* points, int64_t cap, int64_t* count);

/* ---- Alg.1 steps 3-4 on the eps-surrounding: masked grid + iso-surface mesh --
 * §2.1.3: "evaluating the interpolant only in a small surrounding
 * volume" M_ext^eps = {x : d(x, M) <= eps} of the surface, and Alg.1 step 4
 * (MATLAB isosurface): the mesh of the zero iso-surface.
 * data: DEVICE fp64 ndata x 3 (the surface points X); eps > 0; a node is in
 * M_ext^eps iff some data point lies within eps (fp64 distances, the mask of
 * rbf_zero_set).  grid, w, cells, kern as rbf_eval_grid.
 *
 * rbf_eval_grid_masked: field (DEVICE fp32, all nodes, x fastest) receives
 *   P_f at the nodes of M_ext^eps -- bit-identical to rbf_eval_grid's value
 *   there -- and NaN (all bits set) at every other node; only the 4x4x4 node
 *   blocks holding a masked node are evaluated.  world > 1: every rank returns
 *   the full field (slab layers gathered, as rbf_eval_grid).
 * rbf_mesh_from_field: the mesh of the zero iso-surface of a given field on
 *   M_ext^eps (nodes outside the mask are never read).  Reading R24
 *   (oracle/mesh.py): marching tetrahedra on the Kuhn split of each
 *   grid cube (6 tetrahedra per cube, for the axis permutations xyz xzy yxz
 *   yzx zxy zyx); node "inside" iff F < 0; a vertex on every grid edge (v, v+d),
 *   d in x, y, z, xy, xz, yz, xyz (this order), whose two nodes are in the mask
 *   and on opposite sides, at p_v + t (p_{v+d} - p_v), t = F_v/(F_v - F_{v+d})
 *   (fp64); vertices numbered in (v, d) order; a cube is polygonised iff its 8
 *   nodes are in the mask; triangles in (cube, tetrahedron) order, oriented
 *   with their normal (p1-p0) x (p2-p0) towards F > 0 (outward for the
 *   ±delta labels of rbf_extend_points).  Inside the mask the mesh is closed
 *   (every edge shared by two triangles); at the mask boundary it is open, and
 *   vertices of boundary edges may be unreferenced.
 * rbf_isosurface: rbf_eval_grid_masked followed by rbf_mesh_from_field, the
 *   field never leaving the device (field may be NULL: library scratch).
 * The mesh object is library-owned: rbf_mesh_view returns DEVICE pointers
 *   (vertices fp64 nv x 3, triangles int32 nt x 3) valid until rbf_mesh_free,
 *   which must precede rbf_destroy of the context that made it.
 * Synchronise.  Errors: RBF_EINVAL (NULLs, eps <= 0, bad grid, non-finite
 * data, more than 2^31 vertices), RBF_ENOMEM. */
typedef struct rbf_mesh rbf_mesh;
rbf_status rbf_eval_grid_masked(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern, const double* w,
                                const rbf_grid* grid, const double* data, int64_t ndata, double eps, float* field);
rbf_status rbf_mesh_from_field(rbf_ctx* ctx, const float* field, const rbf_grid* grid, const double* data,
                               int64_t ndata, double eps, rbf_mesh** out);
rbf_status rbf_isosurface(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern, const double* w,
                          const rbf_grid* grid, const double* data, int64_t ndata, double eps, float* field,
                          rbf_mesh** out);
rbf_status rbf_mesh_view(const rbf_mesh* m, const double** vertices, int64_t* nv, const int32_t** tris, int64_t* nt);
void rbf_mesh_free(rbf_mesh* m);

/* ---- density measures of the data set (§4, Eq.7-11) ----
 * x: DEVICE fp64 n x 3 (for 2-D sets pass z = 0).  Distances in fp64,
 * ((dx^2 + dy^2) + dz^2) then sqrt of the minimum (bit-identical to the oracle).
 * rbf_nn_distance: dist[i] (DEVICE fp64) = min_j ||q_i - x_j|| for the m query
 * points q (DEVICE fp64 m x 3), or, with q = NULL, min_{j != i} ||x_i - x_j||
 * (n entries; duplicates give 0).  rbf_density: out6 (HOST) =
 *   [0] q_X      separation distance, half the smallest pairwise distance (Eq.7)
 *   [1] h_max    largest nearest-neighbour distance
 *   [2] h_X,Om   fill distance over the m sample points omega of Omega (Eq.8;
 *                NaN when omega = NULL)
 *   [3] sigma of Eq.9   2 q_X
 *   [4] sigma of Eq.10  sqrt(2) h_X,Om (NaN when omega = NULL)
 *   [5] sigma of Eq.10 with Eq.11's h_X,M ~ sqrt(2) h_max:  2 h_max
 * (each sigma as the fp64 product of the measure and the constant).
 * rbf_sigma_auto: *sigma (HOST) = out6[3], out6[4] or out6[5] for rule = 9, 10
 * or 11 (rule 10 needs omega).  Synchronise.  Errors: RBF_EINVAL (n < 2 for self
 * distances, NULLs, non-finite data, rule not in {9,10,11}, rule 10 without
 * omega). */
rbf_status rbf_nn_distance(rbf_ctx* ctx, const double* x, int64_t n, const double* q, int64_t m, double* dist);
rbf_status rbf_density(rbf_ctx* ctx, const double* x, int64_t n, const double* omega, int64_t m, double* out6);
rbf_status rbf_sigma_auto(rbf_ctx* ctx, const double* x, int64_t n, const double* omega, int64_t m, int rule,
                          double* sigma);

/* ---- profiling (CUDA events on the context stream) -------------------------
 * When enabled, every launch of the listed device stages is bracketed by a
 * pair of CUDA events recorded on the context's stream.  rbf_profile_query
 * synchronises, sums the elapsed times per stage into the HOST arrays
 * ms[RBF_PROF_COUNT] and launches[RBF_PROF_COUNT], and clears the records.
 * Enabling creates a stock of 16384 events at once (returned by each query), so
 * that no event is created -- and the driver never extends its event storage --
 * in the middle of a timed region. */
typedef enum {
  RBF_PROF_CELLS = 0,          /* a1/a2: cell build + tile plan (whole call) */
  RBF_PROF_MATVEC_F32 = 1,     /* a3: fp32 summation kernel */
  RBF_PROF_MATVEC_F64 = 2,     /* a7: fp64 summation kernel */
  RBF_PROF_GRID = 3,           /* a8: grid summation kernel */
  RBF_PROF_PRECOND_SETUP = 4,  /* a4: blocks + assembly + LU (whole call) */
  RBF_PROF_PRECOND_APPLY = 5,  /* a5: restricted-inverse apply kernel */
  RBF_PROF_COUNT = 6
} rbf_prof_stage;
rbf_status rbf_profile_enable(rbf_ctx* ctx, int on);
rbf_status rbf_profile_query(rbf_ctx* ctx, double* ms, int64_t* launches);

/* Pair accounting of the grid traversal (host outputs; synchronises): useful =
 * (node, centre) pairs with r^2 <= c^2, visited = pairs evaluated after culling. */
rbf_status rbf_eval_grid_pairs(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern,
                               const rbf_grid* grid, int64_t* useful, int64_t* visited);

/* ---- Alg.1 steps 2-3 end to end from HOST buffers -------------------------
 * xyz (n x 3 fp32), b (n fp32), w_out (n fp64), field_out (grid nodes fp32),
 * rep: all HOST.  Copies in, builds cells, preconditioner, solves, evaluates
 * the grid, copies out.  Synchronises. */
rbf_status rbf_reconstruct_host(rbf_ctx* ctx, const float* xyz, const float* b, int64_t n,
                                const rbf_kernel* kern, const rbf_cell_cfg* ccfg,
                                const rbf_precond_cfg* pcfg, const rbf_gmres_cfg* gcfg,
                                const rbf_grid* grid, double* w_out, float* field_out,
                                rbf_solve_report* rep);

#ifdef __cplusplus
}
#endif
#endif /* RBF_B200_H */
