// a3 / a7 / a8 of SURVEY.md §8(a): the truncated Gaussian kernel summation
//
//     f_i = a * sum_{j : |x_i - x_j|^2 <= c^2} w_j exp(-|x_i - x_j|^2 / (2 sigma^2))
//
// (Eq.6 P:363-366 entries; Eq.4 P:257-262 matvec; Eq.5 P:264-271 evaluation
// on a grid; truncation P:361-369).  Alg.3 stages centres in
// shared memory and loops over ALL of them; here the loop runs only over the
// cells within the cutoff of a target tile (matrix-free, never assembled).
//
// Execution model (sm_100a):
//  * one warp owns one target tile (<= 64 targets, 2 per lane) and pulls
//    tiles from a global work counter (dynamic balance over 148 SMs);
//  * the sources of the cell rows within the cutoff of the tile's bounding
//    box are streamed 32 at a time with coalesced float4 loads (x,y,z,w),
//    culled against the box (ballot + compaction), and staged in a
//    warp-private shared-memory ring as SoA; every 64 staged sources the warp
//    runs the dense inner loop;
//  * fp32 tier inner loop: sources are staged relative to the tile centre
//    (unscaled); one packed FFMA2 per coordinate forms the difference scaled
//    by sqrt(k), k = log2(e)/(2 sigma^2), in a single rounding, and FMUL2 +
//    2 FFMA2 give the scaled r^2 of two pairs; the
//    cutoff is an integer compare+select on the bits of r^2 (ALU pipe),
//    MUFU.EX2 evaluates 2^-r'^2, and a packed FFMA2 accumulates.  No
//    tensor cores: the K=3 distance form is not a dense contraction.
//  * fp64 tier: same traversal; |x_i-x_j|^2 in fp64 with the oracle's
//    rounding order ((dx^2 + dy^2) + dz^2), fp64 exp, fp64 weights.
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <type_traits>

#include "internal.h"
#include "solver.h"
#include "transport.h"

namespace rbf {
namespace {

constexpr int kSumWarps = 4;            // warps per CTA
constexpr int kFlush = 96;              // sources per inner-loop batch
constexpr int kBuf = kFlush + 32 + 4;   // staging ring capacity (SoA, floats)
constexpr int kBufPad = 136;            // multiple of 4 >= kBuf

// --------------------------------------------------------------- packed ops
__device__ __forceinline__ unsigned long long pk(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 upk(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)));
  return upk(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)));
  return upk(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
  return upk(d);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// r2 if r2 <= C2 else +inf, compared on the bit pattern (r2 >= 0): ISETP+SEL.
__device__ __forceinline__ float cutmask(float r2, int c2bits) {
  int b = __float_as_int(r2);
  return __int_as_float(b <= c2bits ? b : 0x7f800000);
}

struct SumGeom {
  CellGrid g;
  float cc;     // culling radius (cutoff inflated by rounding margins)
  float cc2;
  float ci2;    // interior radius^2: cutoff deflated by 1e-4 and the rounding margin
  float s;      // sqrt(k), k = log2(e) / (2 sigma^2)
  int c2bits;   // bits of float32(k c^2)
  float c2s;    // float32(k c^2)
  float amp;    // a
  // fp64 tier
  double c2d;        // (cutoff_sigmas * sigma)^2 exactly as the oracle forms it
  double two_s2;     // 2 sigma^2
  double ampd;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
__device__ __forceinline__ int cellof(float x, float lo, float inv_h, int dim) {
  float t = floorf((x - lo) * inv_h);
  t = fminf(fmaxf(t, -1.f), (float)dim);
  return clampi((int)t, 0, dim - 1);
}

// Row-streaming traversal shared by all tiers.  For every cell row within the
// (inflated) cutoff of the box [blo, bhi], the contiguous source range is
// streamed through `stage(j, valid)` (32 lanes at a time; returns whether the
// lane keeps its source and writes it to the ring at the position it is
// given) and `flush(count)` is called on full batches.
template <class Load, class Flush>
__device__ __forceinline__ void traverse(const SumGeom& G, const int32_t* __restrict__ cell_start,
                                         float3 blo, float3 bhi, int lane, Load&& load, Flush&& flush,
                                         int& nbuf) {
  const CellGrid& g = G.g;
  const float cc = G.cc, cc2 = G.cc2, h = g.h;
  const int z0 = cellof(blo.z - cc, g.lo[2], g.inv_h, g.dim[2]);
  const int z1 = cellof(bhi.z + cc, g.lo[2], g.inv_h, g.dim[2]);
  const int y0 = cellof(blo.y - cc, g.lo[1], g.inv_h, g.dim[1]);
  const int y1 = cellof(bhi.y + cc, g.lo[1], g.inv_h, g.dim[1]);
  const unsigned lt = (1u << lane) - 1u;
  for (int cz = z0; cz <= z1; ++cz) {
    const float czlo = g.lo[2] + (float)cz * h;
    const float gz = fmaxf(0.f, fmaxf(czlo - bhi.z, blo.z - (czlo + h)));
    for (int cy = y0; cy <= y1; ++cy) {
      const float cylo = g.lo[1] + (float)cy * h;
      const float gy = fmaxf(0.f, fmaxf(cylo - bhi.y, blo.y - (cylo + h)));
      const float rem = cc2 - gy * gy - gz * gz;
      if (rem < 0.f) continue;
      const float rx = sqrtf(rem);
      const int x0 = cellof(blo.x - rx, g.lo[0], g.inv_h, g.dim[0]);
      const int x1 = cellof(bhi.x + rx, g.lo[0], g.inv_h, g.dim[0]);
      const int64_t rowbase = ((int64_t)cz * g.dim[1] + cy) * g.dim[0];
      const int sb = __ldg(cell_start + rowbase + x0);
      const int se = __ldg(cell_start + rowbase + x1 + 1);
      for (int j0 = sb; j0 < se; j0 += 32) {
        const int j = j0 + lane;
        bool keep = load(j, j < se);  // loads + culls into registers
        unsigned bal = __ballot_sync(0xffffffffu, keep);
        int pos = nbuf + __popc(bal & lt);
        RBF_JITTER();
        RBF_DCHECK(!keep || pos < kBufPad);
        load.store(keep, pos);
        nbuf += __popc(bal);
        if (nbuf >= kFlush) {
          __syncwarp();
          flush(kFlush);
          __syncwarp();
          load.shift(nbuf - kFlush, lane);
          __syncwarp();
          nbuf -= kFlush;
        }
      }
    }
  }
}

// Two-ring traversal of the fp32 tier.  `load` classifies each streamed source
// as culled (0), boundary (1: some target of the tile may lie beyond the
// cutoff, the inner loop masks) or interior (2: every target of the tile box is
// within c(1-1e-4), the inner loop skips the mask -- same result bit for bit,
// two fewer ALU instructions per pair).  Each class has its own ring and flush.
template <class Load, class FlushB, class FlushI>
__device__ __forceinline__ void traverse2(const SumGeom& G, const int32_t* __restrict__ cell_start,
                                          float3 blo, float3 bhi, int lane, Load&& load, FlushB&& flushB,
                                          FlushI&& flushI, int& nB, int& nI, int skip_lo = 0, int skip_hi = 0) {
  const CellGrid& g = G.g;
  const float cc = G.cc, cc2 = G.cc2, h = g.h;
  const int z0 = cellof(blo.z - cc, g.lo[2], g.inv_h, g.dim[2]);
  const int z1 = cellof(bhi.z + cc, g.lo[2], g.inv_h, g.dim[2]);
  const int y0 = cellof(blo.y - cc, g.lo[1], g.inv_h, g.dim[1]);
  const int y1 = cellof(bhi.y + cc, g.lo[1], g.inv_h, g.dim[1]);
  const unsigned lt = (1u << lane) - 1u;
  for (int cz = z0; cz <= z1; ++cz) {
    const float czlo = g.lo[2] + (float)cz * h;
    const float gz = fmaxf(0.f, fmaxf(czlo - bhi.z, blo.z - (czlo + h)));
    for (int cy = y0; cy <= y1; ++cy) {
      const float cylo = g.lo[1] + (float)cy * h;
      const float gy = fmaxf(0.f, fmaxf(cylo - bhi.y, blo.y - (cylo + h)));
      const float rem = cc2 - gy * gy - gz * gz;
      if (rem < 0.f) continue;
      const float rx = sqrtf(rem);
      const int x0 = cellof(blo.x - rx, g.lo[0], g.inv_h, g.dim[0]);
      const int x1 = cellof(bhi.x + rx, g.lo[0], g.inv_h, g.dim[0]);
      const int64_t rowbase = ((int64_t)cz * g.dim[1] + cy) * g.dim[0];
      int sb = __ldg(cell_start + rowbase + x0);
      const int se = __ldg(cell_start + rowbase + x1 + 1);
      // symmetric matvec: sources in [skip_lo, skip_hi) are never loaded (a cell
      // row lies in one z plane, so it never straddles skip_lo, a plane boundary)
      if (sb >= skip_lo && sb < skip_hi) sb = min(se, skip_hi);
      for (int j0 = sb; j0 < se; j0 += 32) {
        const int j = j0 + lane;
        const int kind = load.classify(j, j < se);
        const unsigned bi = __ballot_sync(0xffffffffu, kind == 2);
        const unsigned bb = __ballot_sync(0xffffffffu, kind == 1);
        RBF_JITTER();
        RBF_DCHECK(nB + __popc(bb & lt) < kBufPad && nI + __popc(bi & lt) < kBufPad);
        load.store2(kind, nB + __popc(bb & lt), nI + __popc(bi & lt));
        nB += __popc(bb);
        nI += __popc(bi);
        if (nB >= kFlush) {
          __syncwarp();
          flushB(kFlush);
          __syncwarp();
          load.shift_ring(load.rb, nB - kFlush, lane);
          __syncwarp();
          nB -= kFlush;
        }
        if (nI >= kFlush) {
          __syncwarp();
          flushI(kFlush);
          __syncwarp();
          load.shift_ring(load.ri, nI - kFlush, lane);
          __syncwarp();
          nI -= kFlush;
        }
      }
    }
  }
}

// ------------------------------------------------------------- fp32 tier ---
struct Ring32 {
  float* bx; float* by; float* bz; float* bw;
  float* bs = nullptr;   // |s'|^2 (expansion path only)
  int* bi = nullptr;     // sorted source index (symmetric ring only)
};

// Dual-ring staging of the fp32 fast path (see traverse2).  SPLIT = false: no
// interior/boundary classification, every kept source goes to the unmasked ring.
template <bool SPLIT, bool SYM = false>
struct Stage32x2 {
  Ring32 rb, ri;
  const float4* __restrict__ src;
  float3 blo, bhi, ctr;
  float cc2, ci2, s;
  float4 p;
  int jj = 0;
  // SYM: sources in [skip_lo, skip_hi) are skipped (their tiles evaluate the
  // pair), sources in [sym_lo, sym_hi) go to the symmetric ring rb
  int skip_lo = 0, skip_hi = 0, sym_lo = 0, sym_hi = 0;
  __device__ __forceinline__ int classify(int j, bool valid) {
    p = valid ? __ldg(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    jj = j;
    if (SYM && j >= skip_lo && j < skip_hi) return 0;
    const float ax = blo.x - p.x, bx = p.x - bhi.x;
    const float ay = blo.y - p.y, by = p.y - bhi.y;
    const float az = blo.z - p.z, bz = p.z - bhi.z;
    const float gx = fmaxf(0.f, fmaxf(ax, bx)), gy = fmaxf(0.f, fmaxf(ay, by)), gz = fmaxf(0.f, fmaxf(az, bz));
    if (!valid || gx * gx + gy * gy + gz * gz > cc2) return 0;
    if (SYM) return (j >= sym_lo && j < sym_hi) ? 1 : 2;
    if (!SPLIT) return 2;
    // farthest point of the box
    const float fx = fmaxf(fabsf(ax), fabsf(bx)), fy = fmaxf(fabsf(ay), fabsf(by)), fz = fmaxf(fabsf(az), fabsf(bz));
    return (fx * fx + fy * fy + fz * fz <= ci2) ? 2 : 1;
  }
  __device__ __forceinline__ void store2(int kind, int posb, int posi) {
    if (kind == 0) return;
    Ring32& r = (kind == 2) ? ri : rb;
    const int pos = (kind == 2) ? posi : posb;
    // scaled tile-local coordinates s' = (x - ctr) sqrt(k) and |s'|^2
    const float sx = (p.x - ctr.x) * s, sy = (p.y - ctr.y) * s, sz = (p.z - ctr.z) * s;
    r.bx[pos] = sx;
    r.by[pos] = sy;
    r.bz[pos] = sz;
    r.bs[pos] = fmaf(sz, sz, fmaf(sy, sy, sx * sx));
    r.bw[pos] = p.w;
    if (SYM && kind == 1) r.bi[pos] = jj;
  }
  __device__ __forceinline__ void shift_ring(Ring32& r, int rest, int lane) {
    if (lane < rest) {
      float a = r.bx[kFlush + lane], b = r.by[kFlush + lane], c = r.bz[kFlush + lane], d = r.bw[kFlush + lane];
      float e = r.bs[kFlush + lane];
      r.bx[lane] = a; r.by[lane] = b; r.bz[lane] = c; r.bw[lane] = d; r.bs[lane] = e;
      if (SYM && r.bi) r.bi[lane] = r.bi[kFlush + lane];
    }
  }
};

// Inner loop of the fp32 tier by the expansion |s'-t'|^2 = |s'|^2 - 2 t'.s' + |t'|^2
// in the tile-local scaled frame: rr = |s'|^2 - 2 t'.s' is 3 packed FFMA2 per two
// pairs, 2^-|t'|^2 is a per-target factor applied once at the end, and the cutoff
// |s'-t'|^2 <= k c^2 becomes rr <= k c^2 - |t'|^2 (per-target threshold).
// |t'| <= ~2 (tile half-diagonal), so the rounding of the expansion costs
// <= ~17u in the exponent where the term is not negligible.
template <int T, bool MASK>
struct Flush32e {
  Ring32 r;
  float2* acc;                                     // [T]
  const float* mx; const float* my; const float* mz;   // [T] -2 t'
  const float* thr;                                // [T] k c^2 - |t'|^2
  __device__ __forceinline__ float cut(float v, float th) const { return (MASK && !(v <= th)) ? INFINITY : v; }
  __device__ __forceinline__ void operator()(int cnt) {
#pragma unroll 2
    for (int j = 0; j < cnt; j += 4) {
      const float4 X = *reinterpret_cast<const float4*>(r.bx + j);
      const float4 Y = *reinterpret_cast<const float4*>(r.by + j);
      const float4 Z = *reinterpret_cast<const float4*>(r.bz + j);
      const float4 S = *reinterpret_cast<const float4*>(r.bs + j);
      const float4 W = *reinterpret_cast<const float4*>(r.bw + j);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float2 ax = make_float2(mx[t], mx[t]), ay = make_float2(my[t], my[t]), az = make_float2(mz[t], mz[t]);
        float2 ra = fma2(make_float2(Z.x, Z.y), az, make_float2(S.x, S.y));
        float2 rb = fma2(make_float2(Z.z, Z.w), az, make_float2(S.z, S.w));
        ra = fma2(make_float2(Y.x, Y.y), ay, ra); rb = fma2(make_float2(Y.z, Y.w), ay, rb);
        ra = fma2(make_float2(X.x, X.y), ax, ra); rb = fma2(make_float2(X.z, X.w), ax, rb);
        const float th = thr[t];
        float2 ea = make_float2(ex2(-cut(ra.x, th)), ex2(-cut(ra.y, th)));
        float2 eb = make_float2(ex2(-cut(rb.x, th)), ex2(-cut(rb.y, th)));
        acc[t] = fma2(ea, make_float2(W.x, W.y), acc[t]);
        acc[t] = fma2(eb, make_float2(W.z, W.w), acc[t]);
      }
    }
  }
};

#ifndef RBF_SYMW_UNROLL
#define RBF_SYMW_UNROLL 1
#endif
#define RBF_PRAGMA_STR(x) #x
#define RBF_UNROLL(n) _Pragma(RBF_PRAGMA_STR(unroll n))
// Symmetric inner loop (A = A^T): every exponential of a staged source j
// (sorted index beyond this tile, same rank) serves both f_i += a e_ij w_j
// (this lane's targets, as Flush32e) and f_j += a e_ij w_i.  The source side
// sums e'_ij (w_i 2^-|t'_i|^2) over the warp's targets per source -- a
// transpose-reduction of 4 sources at a time (6 shuffles: two halving steps,
// then three summing steps) -- and one lane per source adds it to f_j
// (atomicAdd: the sum over tiles is order-dependent in the last bits).
template <int T, class OutT>
struct Flush32s {
  Ring32 r;
  float2* acc;                                         // [T] target side
  const float* mx; const float* my; const float* mz;   // [T] -2 t'
  const float* wt;                                     // [T] w_i 2^-|t'_i|^2 (0 for empty slots)
  OutT* out;
  const int32_t* out_perm;
  float amp;
  int lane;
  __device__ __forceinline__ void operator()(int cnt) {
    const bool h4 = lane & 16, h3 = lane & 8;
    const int mys = (h4 ? 2 : 0) + (h3 ? 1 : 0);
    RBF_UNROLL(RBF_SYMW_UNROLL)
    for (int j = 0; j < cnt; j += 4) {
      const float4 X = *reinterpret_cast<const float4*>(r.bx + j);
      const float4 Y = *reinterpret_cast<const float4*>(r.by + j);
      const float4 Z = *reinterpret_cast<const float4*>(r.bz + j);
      const float4 S = *reinterpret_cast<const float4*>(r.bs + j);
      const float4 W = *reinterpret_cast<const float4*>(r.bw + j);
      float2 pa = make_float2(0.f, 0.f), pb = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float2 ax = make_float2(mx[t], mx[t]), ay = make_float2(my[t], my[t]), az = make_float2(mz[t], mz[t]);
        float2 ra = fma2(make_float2(Z.x, Z.y), az, make_float2(S.x, S.y));
        float2 rb = fma2(make_float2(Z.z, Z.w), az, make_float2(S.z, S.w));
        ra = fma2(make_float2(Y.x, Y.y), ay, ra); rb = fma2(make_float2(Y.z, Y.w), ay, rb);
        ra = fma2(make_float2(X.x, X.y), ax, ra); rb = fma2(make_float2(X.z, X.w), ax, rb);
        const float2 ea = make_float2(ex2(-ra.x), ex2(-ra.y));
        const float2 eb = make_float2(ex2(-rb.x), ex2(-rb.y));
        acc[t] = fma2(ea, make_float2(W.x, W.y), acc[t]);
        acc[t] = fma2(eb, make_float2(W.z, W.w), acc[t]);
        const float2 wv = make_float2(wt[t], wt[t]);
        pa = fma2(ea, wv, pa);
        pb = fma2(eb, wv, pb);
      }
      // transpose-reduce (pa.x, pa.y, pb.x, pb.y) = sources j .. j+3 over the warp
      float k0 = h4 ? pb.x : pa.x, k1 = h4 ? pb.y : pa.y;
      const float s0 = h4 ? pa.x : pb.x, s1 = h4 ? pa.y : pb.y;
      k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
      k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
      float k = h3 ? k1 : k0;
      k += __shfl_xor_sync(0xffffffffu, h3 ? k0 : k1, 8);
      k += __shfl_xor_sync(0xffffffffu, k, 4);
      k += __shfl_xor_sync(0xffffffffu, k, 2);
      k += __shfl_xor_sync(0xffffffffu, k, 1);
      if ((lane & 7) == 0 && j + mys < cnt) {
        const int src = r.bi[j + mys];
        atomicAdd(out + (out_perm ? out_perm[src] : src), (OutT)(amp * k));
      }
    }
  }
};

struct Stage32 {
  Ring32 r;
  const float4* __restrict__ src;
  float3 blo, bhi, ctr;
  float cc2, s;
  float4 p;
  __device__ __forceinline__ bool operator()(int j, bool valid) {
    p = valid ? __ldg(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    float gx = fmaxf(0.f, fmaxf(blo.x - p.x, p.x - bhi.x));
    float gy = fmaxf(0.f, fmaxf(blo.y - p.y, p.y - bhi.y));
    float gz = fmaxf(0.f, fmaxf(blo.z - p.z, p.z - bhi.z));
    return valid && (gx * gx + gy * gy + gz * gz <= cc2);
  }
  __device__ __forceinline__ void store(bool keep, int pos) {
    if (keep) {
      // tile-local, unscaled (exact for sources near the tile: Sterbenz)
      r.bx[pos] = p.x - ctr.x;
      r.by[pos] = p.y - ctr.y;
      r.bz[pos] = p.z - ctr.z;
      r.bw[pos] = p.w;
    }
  }
  __device__ __forceinline__ void shift(int rest, int lane) {
    if (lane < rest) {
      float a = r.bx[kFlush + lane], b = r.by[kFlush + lane], c = r.bz[kFlush + lane], d = r.bw[kFlush + lane];
      r.bx[lane] = a; r.by[lane] = b; r.bz[lane] = c; r.bw[lane] = d;
    }
  }
};

template <int T, bool MASK = true>
struct Flush32 {
  Ring32 r;
  float2* acc;            // [T]
  const float* xt; const float* yt; const float* zt;   // [T] -(local target coords * s)
  int c2bits;
  float s;
  __device__ __forceinline__ float cut(float r2) const { return MASK ? cutmask(r2, c2bits) : r2; }
  __device__ __forceinline__ void operator()(int cnt) {
    const float2 s2 = make_float2(s, s);
#pragma unroll 2
    for (int j = 0; j < cnt; j += 4) {
      const float4 X = *reinterpret_cast<const float4*>(r.bx + j);
      const float4 Y = *reinterpret_cast<const float4*>(r.by + j);
      const float4 Z = *reinterpret_cast<const float4*>(r.bz + j);
      const float4 W = *reinterpret_cast<const float4*>(r.bw + j);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float2 tx = make_float2(xt[t], xt[t]);
        const float2 ty = make_float2(yt[t], yt[t]);
        const float2 tz = make_float2(zt[t], zt[t]);
        // scaled difference in one rounding: x_l * s is exact inside the FMA
        float2 dxa = fma2(make_float2(X.x, X.y), s2, tx), dxb = fma2(make_float2(X.z, X.w), s2, tx);
        float2 dya = fma2(make_float2(Y.x, Y.y), s2, ty), dyb = fma2(make_float2(Y.z, Y.w), s2, ty);
        float2 dza = fma2(make_float2(Z.x, Z.y), s2, tz), dzb = fma2(make_float2(Z.z, Z.w), s2, tz);
        float2 ra = mul2(dxa, dxa), rb = mul2(dxb, dxb);
        ra = fma2(dya, dya, ra); rb = fma2(dyb, dyb, rb);
        ra = fma2(dza, dza, ra); rb = fma2(dzb, dzb, rb);
        float2 ea = make_float2(ex2(-cut(ra.x)), ex2(-cut(ra.y)));
        float2 eb = make_float2(ex2(-cut(rb.x)), ex2(-cut(rb.y)));
        acc[t] = fma2(ea, make_float2(W.x, W.y), acc[t]);
        acc[t] = fma2(eb, make_float2(W.z, W.w), acc[t]);
      }
    }
  }
};

// pair statistics variant (slow; used only by rbf_matvec_pairs)
template <int T>
struct FlushStats {
  Ring32 r;
  const float* xt; const float* yt; const float* zt;
  const bool* tvalid;
  int c2bits;
  float s;
  unsigned long long* useful; unsigned long long* visited;
  __device__ __forceinline__ void operator()(int cnt) {
    for (int j = 0; j < cnt; ++j) {
      if (r.bx[j] > 1e17f) continue;  // padding
#pragma unroll
      for (int t = 0; t < T; ++t) {
        if (!tvalid[t]) continue;
        float dx = fmaf(r.bx[j], s, xt[t]), dy = fmaf(r.by[j], s, yt[t]), dz = fmaf(r.bz[j], s, zt[t]);
        float r2 = dx * dx + dy * dy + dz * dz;
        *visited += 1;
        if (__float_as_int(r2) <= c2bits) *useful += 1;
      }
    }
  }
};

// Pads the ring to a multiple of 4 with sources that contribute exactly 0:
// far away (difference path) or with |s'|^2 = 1e30 (expansion path, 2^-1e30 = 0).
__device__ __forceinline__ void pad_ring(Ring32 r, int nbuf, int lane, int& cnt, bool expansion = false) {
  cnt = (nbuf + 3) & ~3;
  if (lane < cnt - nbuf) {
    const int q = nbuf + lane;
    r.bw[q] = 0.f;
    if (expansion) {
      r.bx[q] = 0.f; r.by[q] = 0.f; r.bz[q] = 0.f; r.bs[q] = 1e30f;
    } else {
      r.bx[q] = 1e18f; r.by[q] = 1e18f; r.bz[q] = 1e18f;
    }
  }
  __syncwarp();
}

// Symmetric ring padding: zero-weight sources at |s'|^2 = 1e30 (2^-1e30 = 0)
// whose index is a valid target of the tile (the source side adds exactly 0 there).
__device__ __forceinline__ void pad_ring_sym(Ring32 r, int nbuf, int lane, int& cnt, int valid_idx) {
  cnt = (nbuf + 3) & ~3;
  if (lane < cnt - nbuf) {
    const int q = nbuf + lane;
    r.bw[q] = 0.f;
    r.bx[q] = 0.f; r.by[q] = 0.f; r.bz[q] = 0.f; r.bs[q] = 1e30f;
    r.bi[q] = valid_idx;
  }
  __syncwarp();
}

// Targets: mode 0 = tile of sorted centres, mode 1 = block of 4 x 4 x bz grid
// nodes (bz = kGridBz: 4 -> two nodes per lane; 2 -> one: 14% fewer visited
// pairs (48% -> 40% beyond the cutoff) but half the reuse of each staged
// source, measured 7.9 vs 6.5 ms for the c4 grid)
#ifndef RBF_GRID_BZ
#define RBF_GRID_BZ 4
#endif
constexpr int kGridBz = RBF_GRID_BZ;
struct GridDesc {
  double lo[3], step[3];
  int n[3];
  int nb[3];   // blocks per axis
  int bz;      // nodes per block along z
};

__device__ __forceinline__ float node_coord(const GridDesc& gd, int a, int i) {
  return (float)(gd.lo[a] + (double)i * gd.step[a]);
}
inline float node_coord_host(const GridDesc& gd, int a, int i) { return (float)(gd.lo[a] + (double)i * gd.step[a]); }

// DIRECT: the difference form |x_l s - t'|^2 (Flush32, one masked ring) instead of
// the expansion; used when the tile or node-block boxes are so large that the
// expansion's per-target factor 2^-|t'|^2 would leave fp32 range or lose accuracy
// (expansion_ok(), |t'|^2 <= kExpT2Max).
template <int MODE, bool STATS, class OutT, bool SYM = false, bool DIRECT = false>
__global__ void __launch_bounds__(kSumWarps * 32, 8)
sum_f32_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ src,
               const int2* __restrict__ tiles, const float4* __restrict__ tbox, int64_t ntiles, int64_t tile_base,
               GridDesc gd, OutT* __restrict__ out, const int32_t* __restrict__ out_perm,
               int* __restrict__ work, unsigned long long* __restrict__ stats, int64_t own_lo = 0,
               int64_t own_hi = 0, const int32_t* __restrict__ tlist = nullptr,
               const uint8_t* __restrict__ nmask = nullptr) {
  __shared__ __align__(16) float ring[kSumWarps][SYM ? 11 : 10][kBufPad];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // boundary sources (grid) / symmetric sources (SYM matvec)
  Ring32 R{ring[wib][0], ring[wib][1], ring[wib][2], ring[wib][3], ring[wib][8],
           SYM ? reinterpret_cast<int*>(ring[wib][SYM ? 10 : 0]) : nullptr};
  Ring32 RI{ring[wib][4], ring[wib][5], ring[wib][6], ring[wib][7], ring[wib][9]};   // interior sources
  unsigned long long useful = 0, visited = 0;
  for (;;) {
    int64_t tile;
    {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(work, 1);
      tile = __shfl_sync(0xffffffffu, t0, 0);
    }
    if (tile >= ntiles) break;
    // this rank's tile range [tile_base, tile_base + ntiles) (slab partition),
    // or (grid) the list of node blocks within reach of a centre
    tile = tlist ? (int64_t)tlist[tile] : tile + tile_base;
    float3 blo, bhi;
    float xr[2], yr[2], zr[2];   // raw target coordinates
    bool tv[2];
    int tcount;
    int64_t tidx[2];
    if (MODE == 0) {
      const int2 tl = tiles[tile];
      const float4 a = tbox[2 * tile], b = tbox[2 * tile + 1];
      blo = make_float3(a.x, a.y, a.z);
      bhi = make_float3(b.x, b.y, b.z);
      tcount = tl.y;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        int q = lane + 32 * t;
        tv[t] = q < tl.y;
        tidx[t] = tl.x + (tv[t] ? q : 0);
        float4 p = src[tidx[t]];
        xr[t] = p.x; yr[t] = p.y; zr[t] = p.z;
      }
    } else {
      const int bx = (int)(tile % gd.nb[0]);
      const int by = (int)((tile / gd.nb[0]) % gd.nb[1]);
      const int bz = (int)(tile / ((int64_t)gd.nb[0] * gd.nb[1]));
      const int i0 = 4 * bx, j0 = 4 * by, k0 = gd.bz * bz;
      const int i1 = min(i0 + 3, gd.n[0] - 1), j1 = min(j0 + 3, gd.n[1] - 1), k1 = min(k0 + gd.bz - 1, gd.n[2] - 1);
      blo = make_float3(node_coord(gd, 0, i0), node_coord(gd, 1, j0), node_coord(gd, 2, k0));
      bhi = make_float3(node_coord(gd, 0, i1), node_coord(gd, 1, j1), node_coord(gd, 2, k1));
      tcount = (k1 - k0 + 1) > 2 ? 64 : 32;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        int i = i0 + (lane & 3), j = j0 + ((lane >> 2) & 3), k = k0 + (lane >> 4) + 2 * t;
        tv[t] = (i <= i1) && (j <= j1) && (k <= k1);
        i = min(i, i1); j = min(j, j1); k = min(k, k1);
        tidx[t] = (int64_t)i + (int64_t)gd.n[0] * ((int64_t)j + (int64_t)gd.n[1] * k);
        xr[t] = node_coord(gd, 0, i); yr[t] = node_coord(gd, 1, j); zr[t] = node_coord(gd, 2, k);
      }
    }
    const float3 ctr = make_float3(0.5f * (blo.x + bhi.x), 0.5f * (blo.y + bhi.y), 0.5f * (blo.z + bhi.z));
    float xt[2], yt[2], zt[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      xt[t] = -((xr[t] - ctr.x) * G.s); yt[t] = -((yr[t] - ctr.y) * G.s); zt[t] = -((zr[t] - ctr.z) * G.s);
    }
    float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float tf[2] = {1.f, 1.f};
    const bool two = tcount > 32;
    if (STATS) {
      Stage32 st{R, src, blo, bhi, ctr, G.cc2, G.s, make_float4(0, 0, 0, 0)};
      int nbuf = 0;
      FlushStats<2> fs{R, xt, yt, zt, tv, G.c2bits, G.s, &useful, &visited};
      traverse(G, cell_start, blo, bhi, lane, st, fs, nbuf);
      int cnt;
      pad_ring(R, nbuf, lane, cnt);
      fs(cnt);
      __syncwarp();
    } else if constexpr (DIRECT) {
      Stage32 st{R, src, blo, bhi, ctr, G.cc2, G.s, make_float4(0, 0, 0, 0)};
      Flush32<2, true> fl{R, acc, xt, yt, zt, G.c2bits, G.s};
      int nbuf = 0, cnt;
      traverse(G, cell_start, blo, bhi, lane, st, fl, nbuf);
      pad_ring(R, nbuf, lane, cnt);
      fl(cnt);
      __syncwarp();
    } else {
      // expansion path: per-target -2 t', threshold k c^2 - |t'|^2, factor 2^-|t'|^2
      float mx[2], my[2], mz[2], th[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const float tx = (xr[t] - ctr.x) * G.s, ty = (yr[t] - ctr.y) * G.s, tz = (zr[t] - ctr.z) * G.s;
        const float T2 = fmaf(tz, tz, fmaf(ty, ty, tx * tx));
        mx[t] = -2.f * tx; my[t] = -2.f * ty; mz[t] = -2.f * tz;
        th[t] = G.c2s - T2;
        tf[t] = ex2(-T2);
      }
      // matvec (MODE 0): every staged source goes through the unmasked ring --
      // a pair beyond the cutoff but inside the culling radius adds a 2^-r <=
      // 2^-(k c^2) = 2^-25.97 term (<= 1/4 ulp of the peak entry; DESIGN.md
      // reading R18).  Grid (MODE 1) keeps the mask: nodes with no centre
      // within the cutoff must be exactly 0 (reading R5).
      if constexpr (SYM) {
        // sources of this rank before the tile: skipped (their tile holds the
        // pair); after it: symmetric; the tile's own and other ranks' sources:
        // one-sided (reading R19)
        const int2 tl = tiles[tile];
        Stage32x2<false, true> st{R, RI, src, blo, bhi, ctr, G.cc2, G.ci2, G.s, make_float4(0, 0, 0, 0)};
        st.skip_lo = (int)own_lo;
        st.skip_hi = tl.x;
        st.sym_lo = tl.x + tl.y;
        st.sym_hi = (int)own_hi;
        float wt[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) wt[t] = tv[t] ? src[tidx[t]].w * tf[t] : 0.f;
        int nB = 0, nI = 0, cnt;
        if (two) {
          Flush32s<2, OutT> fs{R, acc, mx, my, mz, wt, out, out_perm, G.amp, lane};
          Flush32e<2, false> fi{RI, acc, mx, my, mz, th};
          traverse2(G, cell_start, blo, bhi, lane, st, fs, fi, nB, nI, st.skip_lo, st.skip_hi);
          pad_ring_sym(R, nB, lane, cnt, tl.x);
          fs(cnt);
          pad_ring(RI, nI, lane, cnt, true);
          fi(cnt);
        } else {
          Flush32s<1, OutT> fs{R, acc, mx, my, mz, wt, out, out_perm, G.amp, lane};
          Flush32e<1, false> fi{RI, acc, mx, my, mz, th};
          traverse2(G, cell_start, blo, bhi, lane, st, fs, fi, nB, nI, st.skip_lo, st.skip_hi);
          pad_ring_sym(R, nB, lane, cnt, tl.x);
          fs(cnt);
          pad_ring(RI, nI, lane, cnt, true);
          fi(cnt);
        }
        __syncwarp();
      } else {
      Stage32x2<MODE != 0> st{R, RI, src, blo, bhi, ctr, G.cc2, G.ci2, G.s, make_float4(0, 0, 0, 0)};
      int nB = 0, nI = 0, cnt;
      if (two) {
        Flush32e<2, true> fb{R, acc, mx, my, mz, th};
        Flush32e<2, false> fi{RI, acc, mx, my, mz, th};
        traverse2(G, cell_start, blo, bhi, lane, st, fb, fi, nB, nI);
        pad_ring(R, nB, lane, cnt, true);
        fb(cnt);
        pad_ring(RI, nI, lane, cnt, true);
        fi(cnt);
      } else {
        Flush32e<1, true> fb{R, acc, mx, my, mz, th};
        Flush32e<1, false> fi{RI, acc, mx, my, mz, th};
        traverse2(G, cell_start, blo, bhi, lane, st, fb, fi, nB, nI);
        pad_ring(R, nB, lane, cnt, true);
        fb(cnt);
        pad_ring(RI, nI, lane, cnt, true);
        fi(cnt);
      }
      __syncwarp();
      }
    }
    if (!STATS) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (!tv[t]) continue;
        float v = G.amp * ((acc[t].x + acc[t].y) * tf[t]);
        int64_t o = tidx[t];
        if (MODE == 0 && out_perm) o = out_perm[o];
        // masked grid (M_ext^eps): nodes outside the eps-surrounding are NaN
        if (MODE == 1 && nmask && !nmask[o]) v = __int_as_float(-1);
        if (SYM) atomicAdd(out + o, (OutT)v);
        else out[o] = (OutT)v;
      }
    }
  }
  if (STATS) {
    for (int o = 16; o > 0; o >>= 1) {
      useful += __shfl_xor_sync(0xffffffffu, useful, o);
      visited += __shfl_xor_sync(0xffffffffu, visited, o);
    }
    if (lane == 0) { atomicAdd(stats, useful); atomicAdd(stats + 1, visited); }
  }
}

// ---------------------------------------------- grid, separable form (a8) ---
// The nodes of a block lie on a lattice, so the Gaussian of a (node, centre)
// pair factors along the axes: 2^-|xi - s|^2 = ex[i] ey[j] ez[k] with only
// 4 + 4 + 4 exponentials per centre for the 64 nodes of a 4 x 4 x 4 block instead
// of 64 (Eq.5: the evaluation points of the paper are a regular grid,
// P:203-204).  Roles are swapped against the matvec kernels: a LANE owns one
// staged centre at a time and the 64 node sums live in its registers; one
// transposed warp reduction per block (62 shuffles) folds the 32 lanes' partial
// sums so that lane l ends with nodes l and l + 32 (the layout the store uses).
// Per centre and lane: 12 MUFU.EX2, 12 differences + 12 squares, 4 + 16 products,
// then per node one FFMA (interior centres: packed, 32 FFMA2) or FSETP + FFMA
// under the exact cutoff predicate dx^2 + dy^2 + dz^2 <= k c^2 (reading R5;
// boundary centres, same dual-ring classification as the traversal's) -- 1.4 /
// 3.3 instructions per pair against 3.6 / 5.6 for the per-pair exponential form,
// and 0.19 MUFU per pair instead of 1.  The difference form has no per-target
// factor, so it needs no bound on the block size (sum_f32_kernel<1>'s expansion
// does: expansion_ok).
struct SepNodes {
  float tx[4], ty[4], tz[4];   // scaled node offsets from the block centre
};

template <bool MASK>
struct FlushSep {
  Ring32 r;
  float2* acc;          // [32]: nodes (i, j, k = 2 h), (i, j, 2 h + 1) at [i + 4 j + 16 h]
  const SepNodes* nd;
  float c2s;
  int lane;
  __device__ __forceinline__ void operator()(int cnt) {   // cnt: multiple of 32
#pragma unroll 1
    for (int j0 = 0; j0 < cnt; j0 += 32) {
      const float sx = r.bx[j0 + lane], sy = r.by[j0 + lane], sz = r.bz[j0 + lane], w = r.bw[j0 + lane];
      float qx[4], qy[4], qz[4], ex[4], ey[4], ez[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float dx = sx - nd->tx[i], dy = sy - nd->ty[i], dz = sz - nd->tz[i];
        qx[i] = dx * dx; qy[i] = dy * dy; qz[i] = dz * dz;
        ex[i] = ex2(-qx[i]) * w; ey[i] = ex2(-qy[i]); ez[i] = ex2(-qz[i]);
      }
      if constexpr (MASK) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float wxy = ex[i] * ey[j];
            const float lim = (c2s - qx[i]) - qy[j];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float2& a = acc[i + 4 * j + 16 * h];
              if (qz[2 * h] <= lim) a.x = fmaf(wxy, ez[2 * h], a.x);
              if (qz[2 * h + 1] <= lim) a.y = fmaf(wxy, ez[2 * h + 1], a.y);
            }
          }
      } else {
        const float2 ez01 = make_float2(ez[0], ez[1]), ez23 = make_float2(ez[2], ez[3]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 eyj = make_float2(ey[j], ey[j]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 wxy = mul2(make_float2(ex[i], ex[i]), eyj);
            acc[i + 4 * j] = fma2(wxy, ez01, acc[i + 4 * j]);
            acc[i + 4 * j + 16] = fma2(wxy, ez23, acc[i + 4 * j + 16]);
          }
        }
      }
    }
  }
};

// pads a ring to a multiple of 32 with zero-weight centres far away (every
// factor 2^-1e36 = 0, every cutoff test false)
__device__ __forceinline__ void pad_ring32(Ring32 r, int nbuf, int lane, int& cnt) {
  cnt = (nbuf + 31) & ~31;
  if (lane < cnt - nbuf) {
    const int q = nbuf + lane;
    r.bx[q] = 1e18f; r.by[q] = 1e18f; r.bz[q] = 1e18f; r.bw[q] = 0.f;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kSumWarps * 32, 4)
grid_sep_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ src, int64_t ntiles,
                GridDesc gd, float* __restrict__ out, int* __restrict__ work, const int32_t* __restrict__ tlist,
                const uint8_t* __restrict__ nmask) {
  static_assert(kFlush % 32 == 0, "the separable flush takes 32 centres at a time");
  __shared__ __align__(16) float ring[kSumWarps][8][kBufPad];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  Ring32 R{ring[wib][0], ring[wib][1], ring[wib][2], ring[wib][3], nullptr, nullptr};    // boundary centres
  Ring32 RI{ring[wib][4], ring[wib][5], ring[wib][6], ring[wib][7], nullptr, nullptr};   // interior centres
  const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4, b2 = lane & 2, b1 = lane & 1;
  for (;;) {
    int64_t tile;
    {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(work, 1);
      tile = __shfl_sync(0xffffffffu, t0, 0);
    }
    if (tile >= ntiles) break;
    tile = tlist ? (int64_t)tlist[tile] : tile;
    const int bx = (int)(tile % gd.nb[0]);
    const int by = (int)((tile / gd.nb[0]) % gd.nb[1]);
    const int bz = (int)(tile / ((int64_t)gd.nb[0] * gd.nb[1]));
    const int i0 = 4 * bx, j0 = 4 * by, k0 = 4 * bz;
    const int i1 = min(i0 + 3, gd.n[0] - 1), j1 = min(j0 + 3, gd.n[1] - 1), k1 = min(k0 + 3, gd.n[2] - 1);
    const float3 blo = make_float3(node_coord(gd, 0, i0), node_coord(gd, 1, j0), node_coord(gd, 2, k0));
    const float3 bhi = make_float3(node_coord(gd, 0, i1), node_coord(gd, 1, j1), node_coord(gd, 2, k1));
    const float3 ctr = make_float3(0.5f * (blo.x + bhi.x), 0.5f * (blo.y + bhi.y), 0.5f * (blo.z + bhi.z));
    SepNodes nd;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // nodes past the grid edge shadow the last one (never stored)
      nd.tx[q] = (node_coord(gd, 0, min(i0 + q, i1)) - ctr.x) * G.s;
      nd.ty[q] = (node_coord(gd, 1, min(j0 + q, j1)) - ctr.y) * G.s;
      nd.tz[q] = (node_coord(gd, 2, min(k0 + q, k1)) - ctr.z) * G.s;
    }
    float2 acc[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = make_float2(0.f, 0.f);
    {
      FlushSep<true> fb{R, acc, &nd, G.c2s, lane};
      FlushSep<false> fi{RI, acc, &nd, G.c2s, lane};
      int nB = 0, nI = 0, cnt;
      // the traversal of traverse2 / Stage32x2<true> (same cell rows, same cull,
      // same interior / boundary classes, same ring order) written on the
      // kernel's own shared arrays: with 64 pairs per staged centre and lane the
      // staging is half of this kernel's instructions, and the generic rings'
      // pointer selects were a third of that
      const CellGrid& g = G.g;
      const float cc = G.cc, cc2 = G.cc2, ci2 = G.ci2, h = g.h, sc = G.s;
      const int z0 = cellof(blo.z - cc, g.lo[2], g.inv_h, g.dim[2]);
      const int z1 = cellof(bhi.z + cc, g.lo[2], g.inv_h, g.dim[2]);
      const int y0 = cellof(blo.y - cc, g.lo[1], g.inv_h, g.dim[1]);
      const int y1 = cellof(bhi.y + cc, g.lo[1], g.inv_h, g.dim[1]);
      const unsigned lt = (1u << lane) - 1u;
      float* const rbase = &ring[wib][0][0];
      for (int cz = z0; cz <= z1; ++cz) {
        const float czlo = g.lo[2] + (float)cz * h;
        const float gz = fmaxf(0.f, fmaxf(czlo - bhi.z, blo.z - (czlo + h)));
        for (int cy = y0; cy <= y1; ++cy) {
          const float cylo = g.lo[1] + (float)cy * h;
          const float gy = fmaxf(0.f, fmaxf(cylo - bhi.y, blo.y - (cylo + h)));
          const float rem = cc2 - gy * gy - gz * gz;
          if (rem < 0.f) continue;
          const float rx = sqrtf(rem);
          const int x0 = cellof(blo.x - rx, g.lo[0], g.inv_h, g.dim[0]);
          const int x1 = cellof(bhi.x + rx, g.lo[0], g.inv_h, g.dim[0]);
          const int64_t rowbase = ((int64_t)cz * g.dim[1] + cy) * g.dim[0];
          const int sb = __ldg(cell_start + rowbase + x0);
          const int se = __ldg(cell_start + rowbase + x1 + 1);
          for (int jb = sb; jb < se; jb += 32) {
            const int j = jb + lane;
            const bool valid = j < se;
            const float4 p = valid ? __ldg(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float ax = blo.x - p.x, bx2 = p.x - bhi.x;
            const float ay = blo.y - p.y, by2 = p.y - bhi.y;
            const float az = blo.z - p.z, bz2 = p.z - bhi.z;
            const float ox = fmaxf(0.f, fmaxf(ax, bx2)), oy = fmaxf(0.f, fmaxf(ay, by2)), oz = fmaxf(0.f, fmaxf(az, bz2));
            const bool keep = valid && (ox * ox + oy * oy + oz * oz <= cc2);
            // farthest point of the block's box: every node within c (1 - 1e-4)
            const float fx = fmaxf(fabsf(ax), fabsf(bx2)), fy = fmaxf(fabsf(ay), fabsf(by2)), fz = fmaxf(fabsf(az), fabsf(bz2));
            const bool inner = fx * fx + fy * fy + fz * fz <= ci2;
            const unsigned bi = __ballot_sync(0xffffffffu, keep && inner);
            const unsigned bb = __ballot_sync(0xffffffffu, keep && !inner);
            RBF_JITTER();
            if (keep) {
              const int pos = inner ? 4 * kBufPad + nI + __popc(bi & lt) : nB + __popc(bb & lt);
              RBF_DCHECK((inner ? nI + __popc(bi & lt) : nB + __popc(bb & lt)) < kBufPad);
              float* q = rbase + pos;
              q[0] = (p.x - ctr.x) * sc;
              q[kBufPad] = (p.y - ctr.y) * sc;
              q[2 * kBufPad] = (p.z - ctr.z) * sc;
              q[3 * kBufPad] = p.w;
            }
            nB += __popc(bb);
            nI += __popc(bi);
            if (nB >= kFlush) {
              __syncwarp();
              fb(kFlush);
              __syncwarp();
              if (lane < nB - kFlush) {
                float* q = rbase + lane;
                const float a = q[kFlush], b = q[kBufPad + kFlush], c = q[2 * kBufPad + kFlush], d = q[3 * kBufPad + kFlush];
                q[0] = a; q[kBufPad] = b; q[2 * kBufPad] = c; q[3 * kBufPad] = d;
              }
              __syncwarp();
              nB -= kFlush;
            }
            if (nI >= kFlush) {
              __syncwarp();
              fi(kFlush);
              __syncwarp();
              if (lane < nI - kFlush) {
                float* q = rbase + 4 * kBufPad + lane;
                const float a = q[kFlush], b = q[kBufPad + kFlush], c = q[2 * kBufPad + kFlush], d = q[3 * kBufPad + kFlush];
                q[0] = a; q[kBufPad] = b; q[2 * kBufPad] = c; q[3 * kBufPad] = d;
              }
              __syncwarp();
              nI -= kFlush;
            }
          }
        }
      }
      pad_ring32(R, nB, lane, cnt);
      fb(cnt);
      pad_ring32(RI, nI, lane, cnt);
      fi(cnt);
      __syncwarp();
    }
    // transposed reduction over the warp: v[n], n = i + 4 j + 16 k (k = 2 h + c is
    // component c of acc[i + 4 j + 16 h]), 64 -> 2 values per lane; lane l ends
    // with the sums of nodes l (k = l >> 4) and l + 32 (k = (l >> 4) + 2)
    float v5[32];   // index n without bit 4: m = (n & 15) | ((n >> 5) << 4)
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      const int ij = m & 15, kh = m >> 4;   // k = {0, 1} + 2 kh
      const float lo = acc[ij + 16 * kh].x, hi = acc[ij + 16 * kh].y;   // bit 4 of n = k & 1
      v5[m] = (b16 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b16 ? lo : hi, 16);
    }
    float v4[16];   // without bit 3: q = (m & 7) | ((m >> 4) << 3)
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int lo_i = (q & 7) | ((q >> 3) << 4), hi_i = lo_i | 8;
      v4[q] = (b8 ? v5[hi_i] : v5[lo_i]) + __shfl_xor_sync(0xffffffffu, b8 ? v5[lo_i] : v5[hi_i], 8);
    }
    float v3[8];    // without bit 2
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int lo_i = (q & 3) | ((q >> 2) << 3), hi_i = lo_i | 4;
      v3[q] = (b4 ? v4[hi_i] : v4[lo_i]) + __shfl_xor_sync(0xffffffffu, b4 ? v4[lo_i] : v4[hi_i], 4);
    }
    float v2[4];    // without bit 1
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int lo_i = (q & 1) | ((q >> 1) << 2), hi_i = lo_i | 2;
      v2[q] = (b2 ? v3[hi_i] : v3[lo_i]) + __shfl_xor_sync(0xffffffffu, b2 ? v3[lo_i] : v3[hi_i], 2);
    }
    float v1[2];    // without bit 0: index = bit 5 of n
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int lo_i = q << 1, hi_i = lo_i | 1;
      v1[q] = (b1 ? v2[hi_i] : v2[lo_i]) + __shfl_xor_sync(0xffffffffu, b1 ? v2[lo_i] : v2[hi_i], 1);
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int i = i0 + (lane & 3), j = j0 + ((lane >> 2) & 3), k = k0 + (lane >> 4) + 2 * t;
      if (i > i1 || j > j1 || k > k1) continue;
      const int64_t o = (int64_t)i + (int64_t)gd.n[0] * ((int64_t)j + (int64_t)gd.n[1] * k);
      float v = G.amp * v1[t];
      // masked grid (M_ext^eps): nodes outside the eps-surrounding are NaN
      if (nmask && !nmask[o]) v = __int_as_float(-1);
      out[o] = v;
    }
  }
}

#ifndef RBF_SYMW_MINB
#define RBF_SYMW_MINB 8
#endif
// Symmetric fp32 matvec on the WIDE tile plan (reading R19): up to 128 targets
// per warp (4 per lane), so the per-source transpose-reduction of the source
// side is shared by 4 targets per lane.  Same conventions as sum_f32_kernel<0>
// with SYM: out is accumulated (zeroed by the caller), sources of this rank
// before the tile are never loaded, those after it are evaluated once for both
// sides, the tile's own and other ranks' sources one-sidedly.
template <int T, class OutT>
__device__ __forceinline__ void symw_tile(const SumGeom& G, const int32_t* __restrict__ cell_start,
                                          const float4* __restrict__ src, float3 blo, float3 bhi, float3 ctr,
                                          const float* xr, const float* yr, const float* zr, const bool* tv,
                                          const float* wtg, int2 tl, int64_t own_lo, int64_t own_hi, Ring32 R,
                                          Ring32 RI, int lane, OutT* __restrict__ out, float* fout) {
  float mx[T], my[T], mz[T], th[T], tf[T], wt[T];
  float2 acc[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const float tx = (xr[t] - ctr.x) * G.s, ty = (yr[t] - ctr.y) * G.s, tz = (zr[t] - ctr.z) * G.s;
    const float T2 = fmaf(tz, tz, fmaf(ty, ty, tx * tx));
    mx[t] = -2.f * tx; my[t] = -2.f * ty; mz[t] = -2.f * tz;
    th[t] = G.c2s - T2;
    tf[t] = ex2(-T2);
    wt[t] = tv[t] ? wtg[t] * tf[t] : 0.f;
    acc[t] = make_float2(0.f, 0.f);
  }
  Stage32x2<false, true> st{R, RI, src, blo, bhi, ctr, G.cc2, G.ci2, G.s, make_float4(0, 0, 0, 0)};
  st.skip_lo = (int)own_lo;
  st.skip_hi = tl.x;
  st.sym_lo = tl.x + tl.y;
  st.sym_hi = (int)own_hi;
  Flush32s<T, OutT> fs{R, acc, mx, my, mz, wt, out, nullptr, G.amp, lane};
  Flush32e<T, false> fi{RI, acc, mx, my, mz, th};
  int nB = 0, nI = 0, cnt;
  traverse2(G, cell_start, blo, bhi, lane, st, fs, fi, nB, nI, st.skip_lo, st.skip_hi);
  pad_ring_sym(R, nB, lane, cnt, tl.x);
  fs(cnt);
  pad_ring(RI, nI, lane, cnt, true);
  fi(cnt);
  __syncwarp();
#pragma unroll
  for (int t = 0; t < T; ++t) fout[t] = G.amp * ((acc[t].x + acc[t].y) * tf[t]);
}

template <class OutT>
__global__ void __launch_bounds__(kSumWarps * 32, RBF_SYMW_MINB)
sum_f32_symw_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ src,
                    const int2* __restrict__ tiles, const float4* __restrict__ tbox, int64_t ntiles,
                    int64_t tile_base, OutT* __restrict__ out, int* __restrict__ work, int64_t own_lo,
                    int64_t own_hi) {
  __shared__ __align__(16) float ring[kSumWarps][11][kBufPad];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  Ring32 R{ring[wib][0], ring[wib][1], ring[wib][2], ring[wib][3], ring[wib][8],
           reinterpret_cast<int*>(ring[wib][10])};
  Ring32 RI{ring[wib][4], ring[wib][5], ring[wib][6], ring[wib][7], ring[wib][9]};
  for (;;) {
    int64_t tile;
    {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(work, 1);
      tile = __shfl_sync(0xffffffffu, t0, 0);
    }
    if (tile >= ntiles) break;
    tile += tile_base;
    const int2 tl = tiles[tile];
    const float4 a = tbox[2 * tile], b = tbox[2 * tile + 1];
    const float3 blo = make_float3(a.x, a.y, a.z), bhi = make_float3(b.x, b.y, b.z);
    const float3 ctr = make_float3(0.5f * (blo.x + bhi.x), 0.5f * (blo.y + bhi.y), 0.5f * (blo.z + bhi.z));
    float xr[4], yr[4], zr[4], wg[4], fo[4];
    bool tv[4];
    int64_t tidx[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int q = lane + 32 * t;
      tv[t] = q < tl.y;
      tidx[t] = tl.x + (tv[t] ? q : 0);
      const float4 p = src[tidx[t]];
      xr[t] = p.x; yr[t] = p.y; zr[t] = p.z; wg[t] = p.w;
    }
    const int T = (tl.y + 31) >> 5;
    switch (T) {
      case 1: symw_tile<1>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, own_lo, own_hi, R, RI, lane, out, fo); break;
      case 2: symw_tile<2>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, own_lo, own_hi, R, RI, lane, out, fo); break;
      case 3: symw_tile<3>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, own_lo, own_hi, R, RI, lane, out, fo); break;
      default: symw_tile<4>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, own_lo, own_hi, R, RI, lane, out, fo); break;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t < T && tv[t]) atomicAdd(out + tidx[t], (OutT)fo[t]);
  }
}

// Symmetric fp32 matvec, rotation form (reading R19; the solver's default at
// >= 2^18 centres per GPU).  Same pair set and conventions as
// sum_f32_symw_kernel (wide plan, up to 128 targets per warp = 2 pairs of
// 32-target slots per lane; sources of this rank before the tile never loaded;
// the tile's own sources one-sided; every source after it, up to the end of the
// window sym_hi, evaluated ONCE for both f_i and f_j), but the source side is
// summed without a per-source warp reduction: the symmetric sources are staged
// 32 at a time and lane l visits source (l + k) mod 32 at step k of 32, adding
// its targets' share sum_t e_tj w_t 2^-|t'_t|^2 to a rotating accumulator that
// moves one lane down per step (one shuffle), so after 32 steps lane l holds the
// whole warp's sum for source l: one atomic per source, no shuffle tree, no
// selects.  Targets are packed in pairs along the FFMA2 lanes (each step: 3
// FFMA2 for r^2 of 2 targets, 2 MUFU.EX2, 2 FFMA2 accumulates).  All ring
// addressing is on the kernel's own shared arrays (32-bit shared addresses).
constexpr int kRotFlush = 96;                       // symmetric sources per flush (3 rotations)
constexpr int kRotCap = kRotFlush + 32;             // ring capacity
constexpr int kOwnCap = kFlush + 32 + 4;            // own-tile ring capacity (one-sided, SoA)
constexpr int kOwnPad = 136;

template <int TP, class OutT>
__device__ __forceinline__ void symr_tile(const SumGeom& G, const int32_t* __restrict__ cell_start,
                                          const float4* __restrict__ src, float3 blo, float3 bhi, float3 ctr,
                                          const float* xr, const float* yr, const float* zr, const bool* tv,
                                          const float* wg, int2 tl, int64_t sym_hi, int lane,
                                          float4* __restrict__ R4, float2* __restrict__ R2, int* __restrict__ RI,
                                          float (*__restrict__ O)[kOwnPad], OutT* __restrict__ out,
                                          float* fo) {
  constexpr int T = 2 * TP;
  float2 m2x[TP], m2y[TP], m2z[TP], wt2[TP], acc2[TP];
  float tf[T];
#pragma unroll
  for (int tp = 0; tp < TP; ++tp) {
    float mx[2], my[2], mz[2], ww[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = 2 * tp + h;
      const float tx = (xr[t] - ctr.x) * G.s, ty = (yr[t] - ctr.y) * G.s, tz = (zr[t] - ctr.z) * G.s;
      const float T2 = fmaf(tz, tz, fmaf(ty, ty, tx * tx));
      mx[h] = -2.f * tx; my[h] = -2.f * ty; mz[h] = -2.f * tz;
      tf[t] = ex2(-T2);
      ww[h] = tv[t] ? wg[t] * tf[t] : 0.f;
    }
    m2x[tp] = make_float2(mx[0], mx[1]);
    m2y[tp] = make_float2(my[0], my[1]);
    m2z[tp] = make_float2(mz[0], mz[1]);
    wt2[tp] = make_float2(ww[0], ww[1]);
    acc2[tp] = make_float2(0.f, 0.f);
  }
  const float amp = G.amp;
  const int t_end = tl.x + tl.y;
  // symmetric ring: R4[i] = (x', y', z', w), R2[i] = (|s'|^2, |s'|^2); RI[i] = sorted index
  auto flush_sym = [&](int cnt) {   // cnt: multiple of 32
    for (int b = 0; b < cnt; b += 32) {
      float accr = 0.f;
#pragma unroll 4
      for (int k = 0; k < 32; ++k) {
        const int si = b + ((lane + k) & 31);
        const float4 P = R4[si];
        const float2 S2 = R2[si];
        float2 ps = make_float2(0.f, 0.f);
#pragma unroll
        for (int tp = 0; tp < TP; ++tp) {
          float2 rr = fma2(m2z[tp], make_float2(P.z, P.z), S2);
          rr = fma2(m2y[tp], make_float2(P.y, P.y), rr);
          rr = fma2(m2x[tp], make_float2(P.x, P.x), rr);
          const float2 e = make_float2(ex2(-rr.x), ex2(-rr.y));
          acc2[tp] = fma2(e, make_float2(P.w, P.w), acc2[tp]);
          ps = fma2(e, wt2[tp], ps);
        }
        accr += ps.x + ps.y;
        accr = __shfl_sync(0xffffffffu, accr, (lane + 1) & 31);
      }
      const int j = RI[b + lane];
      if (j >= 0) atomicAdd(out + j, (OutT)(amp * accr));
    }
  };
  // own-tile ring (one-sided, broadcast of 4 sources to all lanes, SoA)
  auto flush_own = [&](int cnt) {   // cnt: multiple of 4
#pragma unroll 1
    for (int j = 0; j < cnt; j += 4) {
      const float4 X = *reinterpret_cast<const float4*>(&O[0][j]);
      const float4 Y = *reinterpret_cast<const float4*>(&O[1][j]);
      const float4 Z = *reinterpret_cast<const float4*>(&O[2][j]);
      const float4 S = *reinterpret_cast<const float4*>(&O[3][j]);
      const float4 W = *reinterpret_cast<const float4*>(&O[4][j]);
      const float Sv[4] = {S.x, S.y, S.z, S.w}, Xv[4] = {X.x, X.y, X.z, X.w}, Yv[4] = {Y.x, Y.y, Y.z, Y.w},
                  Zv[4] = {Z.x, Z.y, Z.z, Z.w}, Wv[4] = {W.x, W.y, W.z, W.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int tp = 0; tp < TP; ++tp) {
          float2 rr = fma2(m2z[tp], make_float2(Zv[q], Zv[q]), make_float2(Sv[q], Sv[q]));
          rr = fma2(m2y[tp], make_float2(Yv[q], Yv[q]), rr);
          rr = fma2(m2x[tp], make_float2(Xv[q], Xv[q]), rr);
          const float2 e = make_float2(ex2(-rr.x), ex2(-rr.y));
          acc2[tp] = fma2(e, make_float2(Wv[q], Wv[q]), acc2[tp]);
        }
      }
    }
  };
  // traversal of the cell rows within the culling radius of the box
  const CellGrid& g = G.g;
  const float cc = G.cc, cc2 = G.cc2, h = g.h;
  const int z0 = cellof(blo.z - cc, g.lo[2], g.inv_h, g.dim[2]);
  const int z1 = cellof(bhi.z + cc, g.lo[2], g.inv_h, g.dim[2]);
  const int y0 = cellof(blo.y - cc, g.lo[1], g.inv_h, g.dim[1]);
  const int y1 = cellof(bhi.y + cc, g.lo[1], g.inv_h, g.dim[1]);
  const unsigned lt = (1u << lane) - 1u;
  int nS = 0, nO = 0;
  for (int cz = z0; cz <= z1; ++cz) {
    const float czlo = g.lo[2] + (float)cz * h;
    const float gz = fmaxf(0.f, fmaxf(czlo - bhi.z, blo.z - (czlo + h)));
    for (int cy = y0; cy <= y1; ++cy) {
      const float cylo = g.lo[1] + (float)cy * h;
      const float gy = fmaxf(0.f, fmaxf(cylo - bhi.y, blo.y - (cylo + h)));
      const float rem = cc2 - gy * gy - gz * gz;
      if (rem < 0.f) continue;
      const float rx = sqrtf(rem);
      const int x0 = cellof(blo.x - rx, g.lo[0], g.inv_h, g.dim[0]);
      const int x1 = cellof(bhi.x + rx, g.lo[0], g.inv_h, g.dim[0]);
      const int64_t rowbase = ((int64_t)cz * g.dim[1] + cy) * g.dim[0];
      int sb = __ldg(cell_start + rowbase + x0);
      int se = __ldg(cell_start + rowbase + x1 + 1);
      // sources before the tile are never loaded (their tiles hold the pairs);
      // the window ends at sym_hi
      sb = max(sb, tl.x);
      se = min(se, (int)sym_hi);
      for (int j0 = sb; j0 < se; j0 += 32) {
        const int j = j0 + lane;
        const bool valid = j < se;
        const float4 p = valid ? __ldg(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float gx = fmaxf(0.f, fmaxf(blo.x - p.x, p.x - bhi.x));
        const float gyy = fmaxf(0.f, fmaxf(blo.y - p.y, p.y - bhi.y));
        const float gzz = fmaxf(0.f, fmaxf(blo.z - p.z, p.z - bhi.z));
        const bool keep = valid && (gx * gx + gyy * gyy + gzz * gzz <= cc2);
        const bool own = j < t_end;
        const unsigned bs = __ballot_sync(0xffffffffu, keep && !own);
        const unsigned bo = __ballot_sync(0xffffffffu, keep && own);
        const float sx = (p.x - ctr.x) * G.s, sy = (p.y - ctr.y) * G.s, sz = (p.z - ctr.z) * G.s;
        const float ss = fmaf(sz, sz, fmaf(sy, sy, sx * sx));
        if (keep && !own) {
          const int pos = nS + __popc(bs & lt);
          R4[pos] = make_float4(sx, sy, sz, p.w);
          R2[pos] = make_float2(ss, ss);
          RI[pos] = j;
        } else if (keep) {
          const int pos = nO + __popc(bo & lt);
          O[0][pos] = sx; O[1][pos] = sy; O[2][pos] = sz; O[3][pos] = ss; O[4][pos] = p.w;
        }
        nS += __popc(bs);
        nO += __popc(bo);
        if (nS >= kRotFlush) {
          __syncwarp();
          flush_sym(kRotFlush);
          __syncwarp();
          if (lane < nS - kRotFlush) {
            const float4 a = R4[kRotFlush + lane];
            const float2 c = R2[kRotFlush + lane];
            const int ii = RI[kRotFlush + lane];
            R4[lane] = a; R2[lane] = c; RI[lane] = ii;
          }
          __syncwarp();
          nS -= kRotFlush;
        }
        if (nO >= kFlush) {
          __syncwarp();
          flush_own(kFlush);
          __syncwarp();
          if (lane < nO - kFlush) {
            const int q = kFlush + lane;
            const float a = O[0][q], b = O[1][q], c = O[2][q], d = O[3][q], e = O[4][q];
            O[0][lane] = a; O[1][lane] = b; O[2][lane] = c; O[3][lane] = d; O[4][lane] = e;
          }
          __syncwarp();
          nO -= kFlush;
        }
      }
    }
  }
  // tails: symmetric ring to a multiple of 32 with sources contributing exactly 0
  // (|s'|^2 = 1e30: 2^-1e30 = 0) and no output (index -1); own ring to 4
  {
    const int cntS = (nS + 31) & ~31;
    if (lane < cntS - nS) {
      const int q = nS + lane;
      R4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      R2[q] = make_float2(1e30f, 1e30f);
      RI[q] = -1;
    }
    const int cntO = (nO + 3) & ~3;
    if (lane < cntO - nO) {
      const int q = nO + lane;
      O[0][q] = 0.f; O[1][q] = 0.f; O[2][q] = 0.f; O[3][q] = 1e30f; O[4][q] = 0.f;
    }
    __syncwarp();
    if (cntS) flush_sym(cntS);
    flush_own(cntO);
    __syncwarp();
  }
#pragma unroll
  for (int tp = 0; tp < TP; ++tp) {
    fo[2 * tp] = G.amp * (acc2[tp].x * tf[2 * tp]);
    fo[2 * tp + 1] = G.amp * (acc2[tp].y * tf[2 * tp + 1]);
  }
}

// Peer-memory form of the slab partition: the ranks whose slices
// cover this rank's source window [o0, h1), this rank first; slice k holds the
// sorted positions [lo[k], lo[k+1]) and lives in rank k's buffer -- its packed
// sources src[k][j - lo[k]] and its fp64 sums f[k][j - lo[k]], which the kernel
// reads and atomically updates directly (NVLink / NVSwitch peer memory), in
// place of the halo exchange and the reverse halo reduction.
constexpr int kPeerMax = 8;
struct PeerTab {
  int n;
  int64_t lo[kPeerMax + 1];
  const float4* src[kPeerMax];   // already shifted: src[k] + j addresses position j
  double* f[kPeerMax];           // already shifted
};
__device__ __forceinline__ int peer_of(const PeerTab& P, int64_t j) {
  int k = 0;
  while (k + 1 < P.n && j >= P.lo[k + 1]) ++k;
  return k;
}

template <class OutT>
__global__ void __launch_bounds__(kSumWarps * 32, 8)
sum_f32_symr_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ src,
                    const int2* __restrict__ tiles, const float4* __restrict__ tbox, int64_t ntiles,
                    int64_t tile_base, OutT* __restrict__ out, int* __restrict__ work, int64_t sym_hi,
                    const int32_t* __restrict__ order, PeerTab = PeerTab{},   // (no peer-memory form,
                    const int32_t* = nullptr, const uint32_t* = nullptr) {         //  no neighbour lists)
  __shared__ __align__(16) float4 ring4[kSumWarps][kRotCap];
  __shared__ __align__(8) float2 ring2[kSumWarps][kRotCap];
  __shared__ int ringi[kSumWarps][kRotCap];
  __shared__ __align__(16) float ringo[kSumWarps][5][kOwnPad];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (;;) {
    int64_t tile;
    {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(work, 1);
      tile = __shfl_sync(0xffffffffu, t0, 0);
    }
    if (tile >= ntiles) break;
    tile = order ? (int64_t)order[tile] : tile + tile_base;
    const int2 tl = tiles[tile];
    const float4 a = tbox[2 * tile], b = tbox[2 * tile + 1];
    const float3 blo = make_float3(a.x, a.y, a.z), bhi = make_float3(b.x, b.y, b.z);
    const float3 ctr = make_float3(0.5f * (blo.x + bhi.x), 0.5f * (blo.y + bhi.y), 0.5f * (blo.z + bhi.z));
    float xr[4], yr[4], zr[4], wg[4], fo[4];
    bool tv[4];
    int64_t tidx[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int q = lane + 32 * t;
      tv[t] = q < tl.y;
      tidx[t] = tl.x + (tv[t] ? q : 0);
      const float4 p = src[tidx[t]];
      xr[t] = p.x; yr[t] = p.y; zr[t] = p.z; wg[t] = p.w;
    }
    const int TP = tl.y > 64 ? 2 : 1;
    if (TP == 2)
      symr_tile<2>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, sym_hi, lane, ring4[wib], ring2[wib],
                   ringi[wib], ringo[wib], out, fo);
    else
      symr_tile<1>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, sym_hi, lane, ring4[wib], ring2[wib],
                   ringi[wib], ringo[wib], out, fo);
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t < 2 * TP && tv[t]) atomicAdd(out + tidx[t], (OutT)fo[t]);
  }
}

// Symmetric fp32 matvec, broadcast form (reading R19): the pair set of
// sum_f32_symr_kernel with sum_f32_symw_kernel's inner loop -- 4 staged sources
// at a time broadcast to all lanes (LDS.128 of a shared-memory SoA ring), T <= 4
// targets per lane, the source side of each group of 4 summed over the warp by a
// transpose-reduction (6 shuffles) and one atomic per source -- with every ring
// access on the kernel's own shared arrays (no generic-pointer address math).
constexpr int kSymPad = 136;   // SoA ring row (>= kFlush + 32 + 4, multiple of 4)

#ifndef RBF_SYMB_KBSTORE
#define RBF_SYMB_KBSTORE 1
#endif

// Staging batch of the neighbour-list form (NL): the ring is filled with exactly
// kNlBatch listed sources (no cull, no overflow), then flushed.
#ifndef RBF_NL_BATCH
#define RBF_NL_BATCH 128
#endif
constexpr int kNlBatch = RBF_NL_BATCH;   // (96 and 64 measured with tools/sessions/sess_var.sh)
static_assert(kNlBatch <= kSymPad && kNlBatch <= kOwnPad, "NL batch exceeds the rings");

// NL = false: the tile streams the cell rows within the cutoff of its box and
// culls (the traversal); NL = true: the tile's culled sources after it were
// listed once per cell structure (nl_build_kernel, the same traversal and cull,
// same order) and are read from nl_idx[nl_b, nl_e) -- no row setup, no cull, no
// ballot compaction in the 51 matvecs of a solve.
template <int T, class OutT, bool PEER = false, bool NL = false>
__device__ __forceinline__ void symb_tile(const SumGeom& G, const int32_t* __restrict__ cell_start,
                                          const float4* __restrict__ src, float3 blo, float3 bhi, float3 ctr,
                                          const float* xr, const float* yr, const float* zr, const bool* tv,
                                          const float* wg, int2 tl, int64_t sym_hi, int lane,
                                          float (*__restrict__ RS)[kSymPad], int* __restrict__ RI,
                                          float* __restrict__ KB, float (*__restrict__ O)[kOwnPad],
                                          OutT* __restrict__ out, float* fo, const PeerTab* PT = nullptr,
                                          const int32_t* __restrict__ nl_idx = nullptr, uint32_t nl_b = 0,
                                          uint32_t nl_e = 0) {
  float mx[T], my[T], mz[T], tf[T], wt[T];
  float2 acc[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const float tx = (xr[t] - ctr.x) * G.s, ty = (yr[t] - ctr.y) * G.s, tz = (zr[t] - ctr.z) * G.s;
    const float T2 = fmaf(tz, tz, fmaf(ty, ty, tx * tx));
    mx[t] = -2.f * tx; my[t] = -2.f * ty; mz[t] = -2.f * tz;
    tf[t] = ex2(-T2);
    wt[t] = tv[t] ? wg[t] * tf[t] : 0.f;
    acc[t] = make_float2(0.f, 0.f);
  }
  const float amp = G.amp;
  const int t_end = tl.x + tl.y;
  const bool h4 = lane & 16, h3 = lane & 8;
  const int mys = (h4 ? 2 : 0) + (h3 ? 1 : 0);
  // the source-side sum of source j + mys lands in KB[j + mys] (lanes 0, 8, 16,
  // 24); the other lanes store into private dummy slots KB[kSymPad + lane], so
  // the store is one unpredicated STS (no divergent branch).  The shared address
  // is formed once and pinned in a register (an opaque asm), so the compiler
  // does not rematerialise it from SR_TID in the loop.
#if RBF_SYMB_KBSTORE
  uint32_t kb_addr = (uint32_t)__cvta_generic_to_shared(KB) +
                     4u * (uint32_t)(((lane & 7) == 0) ? mys : kSymPad + lane);
  asm volatile("" : "+r"(kb_addr));
  const uint32_t kb_step = ((lane & 7) == 0) ? 16u : 0u;   // bytes per group of 4 sources
#endif
  // symmetric ring RS[0..4] = x', y', z', |s'|^2, w and RI = sorted index
#ifndef RBF_SYMB_UNROLL
#define RBF_SYMB_UNROLL 1
#endif
#ifndef RBF_SYMB_HALF
#define RBF_SYMB_HALF 1   // 3.138 vs 3.153 ms at c4 (fewer live registers)
#endif
  auto flush_sym = [&](int cnt) {   // cnt: multiple of 4
    RBF_JITTER();
    RBF_DCHECK(cnt <= kSymPad && (cnt & 3) == 0);
    RBF_UNROLL(RBF_SYMB_UNROLL)
    for (int j = 0; j < cnt; j += 4) {
      float2 pa = make_float2(0.f, 0.f), pb = make_float2(0.f, 0.f);
#if RBF_SYMB_HALF
      // two source pairs one after the other: 10 live registers of staged
      // sources instead of 20 (LDS.64 broadcasts)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const float2 X = *reinterpret_cast<const float2*>(&RS[0][j + 2 * hh]);
        const float2 Y = *reinterpret_cast<const float2*>(&RS[1][j + 2 * hh]);
        const float2 Z = *reinterpret_cast<const float2*>(&RS[2][j + 2 * hh]);
        const float2 S = *reinterpret_cast<const float2*>(&RS[3][j + 2 * hh]);
        const float2 W = *reinterpret_cast<const float2*>(&RS[4][j + 2 * hh]);
        float2 p = make_float2(0.f, 0.f);
#pragma unroll
        for (int t = 0; t < T; ++t) {
          float2 ra = fma2(Z, make_float2(mz[t], mz[t]), S);
          ra = fma2(Y, make_float2(my[t], my[t]), ra);
          ra = fma2(X, make_float2(mx[t], mx[t]), ra);
          const float2 ea = make_float2(ex2(-ra.x), ex2(-ra.y));
          acc[t] = fma2(ea, W, acc[t]);
          p = fma2(ea, make_float2(wt[t], wt[t]), p);
        }
        if (hh == 0) pa = p; else pb = p;
      }
#else
      const float4 X = *reinterpret_cast<const float4*>(&RS[0][j]);
      const float4 Y = *reinterpret_cast<const float4*>(&RS[1][j]);
      const float4 Z = *reinterpret_cast<const float4*>(&RS[2][j]);
      const float4 S = *reinterpret_cast<const float4*>(&RS[3][j]);
      const float4 W = *reinterpret_cast<const float4*>(&RS[4][j]);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float2 ax = make_float2(mx[t], mx[t]), ay = make_float2(my[t], my[t]), az = make_float2(mz[t], mz[t]);
        float2 ra = fma2(make_float2(Z.x, Z.y), az, make_float2(S.x, S.y));
        float2 rb = fma2(make_float2(Z.z, Z.w), az, make_float2(S.z, S.w));
        ra = fma2(make_float2(Y.x, Y.y), ay, ra); rb = fma2(make_float2(Y.z, Y.w), ay, rb);
        ra = fma2(make_float2(X.x, X.y), ax, ra); rb = fma2(make_float2(X.z, X.w), ax, rb);
        const float2 ea = make_float2(ex2(-ra.x), ex2(-ra.y));
        const float2 eb = make_float2(ex2(-rb.x), ex2(-rb.y));
        acc[t] = fma2(ea, make_float2(W.x, W.y), acc[t]);
        acc[t] = fma2(eb, make_float2(W.z, W.w), acc[t]);
        const float2 wv = make_float2(wt[t], wt[t]);
        pa = fma2(ea, wv, pa);
        pb = fma2(eb, wv, pb);
      }
#endif
      // transpose-reduce (pa.x, pa.y, pb.x, pb.y) = sources j .. j+3 over the warp
      float k0 = h4 ? pb.x : pa.x, k1 = h4 ? pb.y : pa.y;
      const float s0 = h4 ? pa.x : pb.x, s1 = h4 ? pa.y : pb.y;
      k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
      k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
      float k = h3 ? k1 : k0;
      k += __shfl_xor_sync(0xffffffffu, h3 ? k0 : k1, 8);
      k += __shfl_xor_sync(0xffffffffu, k, 4);
      k += __shfl_xor_sync(0xffffffffu, k, 2);
      k += __shfl_xor_sync(0xffffffffu, k, 1);
#if RBF_SYMB_KBSTORE
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(kb_addr + kb_step * (uint32_t)(j >> 2)), "f"(k) : "memory");
#else
      if ((lane & 7) == 0) KB[j + mys] = k;
#endif
    }
    // the ring's source-side sums to f_j: one atomic per source, 32 lanes at a time
    __syncwarp();
    RBF_JITTER();
    for (int q = lane; q < cnt; q += 32) {
      const int jj = RI[q];
      if constexpr (PEER) {
        if (jj >= 0) atomicAdd(PT->f[peer_of(*PT, jj)] + jj, (double)(amp * KB[q]));
      } else {
        if (jj >= 0) atomicAdd(out + jj, (OutT)(amp * KB[q]));
      }
    }
  };
  auto flush_own = [&](int cnt) {   // cnt: multiple of 4
#pragma unroll 1
    for (int j = 0; j < cnt; j += 4) {
      const float4 X = *reinterpret_cast<const float4*>(&O[0][j]);
      const float4 Y = *reinterpret_cast<const float4*>(&O[1][j]);
      const float4 Z = *reinterpret_cast<const float4*>(&O[2][j]);
      const float4 S = *reinterpret_cast<const float4*>(&O[3][j]);
      const float4 W = *reinterpret_cast<const float4*>(&O[4][j]);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float2 ax = make_float2(mx[t], mx[t]), ay = make_float2(my[t], my[t]), az = make_float2(mz[t], mz[t]);
        float2 ra = fma2(make_float2(Z.x, Z.y), az, make_float2(S.x, S.y));
        float2 rb = fma2(make_float2(Z.z, Z.w), az, make_float2(S.z, S.w));
        ra = fma2(make_float2(Y.x, Y.y), ay, ra); rb = fma2(make_float2(Y.z, Y.w), ay, rb);
        ra = fma2(make_float2(X.x, X.y), ax, ra); rb = fma2(make_float2(X.z, X.w), ax, rb);
        const float2 ea = make_float2(ex2(-ra.x), ex2(-ra.y));
        const float2 eb = make_float2(ex2(-rb.x), ex2(-rb.y));
        acc[t] = fma2(ea, make_float2(W.x, W.y), acc[t]);
        acc[t] = fma2(eb, make_float2(W.z, W.w), acc[t]);
      }
    }
  };
  if constexpr (NL) {
    // the tile's own sources (one-sided), at most 128
    for (int b = tl.x; b < t_end; b += kNlBatch) {
      const int cnt = min(kNlBatch, t_end - b), c4 = (cnt + 3) & ~3;
#pragma unroll
      for (int q = 0; q < kNlBatch / 32; ++q) {
        const int i = q * 32 + lane;
        if (i < c4) {
          const float4 p = i < cnt ? __ldg(src + b + i) : make_float4(ctr.x, ctr.y, ctr.z, 0.f);
          const float sx = (p.x - ctr.x) * G.s, sy = (p.y - ctr.y) * G.s, sz = (p.z - ctr.z) * G.s;
          O[0][i] = sx; O[1][i] = sy; O[2][i] = sz;
          O[3][i] = i < cnt ? fmaf(sz, sz, fmaf(sy, sy, sx * sx)) : 1e30f;
          O[4][i] = p.w;
        }
      }
      __syncwarp();
      flush_own(c4);
      __syncwarp();
    }
    // the listed sources after the tile (symmetric), kNlBatch per flush
    for (uint32_t b = nl_b; b < nl_e; b += kNlBatch) {
      const int cnt = (int)min((uint32_t)kNlBatch, nl_e - b), c4 = (cnt + 3) & ~3;
      int id[kNlBatch / 32];
#pragma unroll
      for (int q = 0; q < kNlBatch / 32; ++q) {
        const int i = q * 32 + lane;
        id[q] = i < cnt ? __ldg(nl_idx + b + i) : -1;
      }
      float4 p[kNlBatch / 32];
#pragma unroll
      for (int q = 0; q < kNlBatch / 32; ++q) {
        const float4* __restrict__ srow = src;
        if constexpr (PEER) {
          if (id[q] >= 0) srow = PT->src[peer_of(*PT, id[q])];
        }
        p[q] = id[q] >= 0 ? __ldg(srow + id[q]) : make_float4(ctr.x, ctr.y, ctr.z, 0.f);
      }
#pragma unroll
      for (int q = 0; q < kNlBatch / 32; ++q) {
        const int i = q * 32 + lane;
        if (i < c4) {
          const float sx = (p[q].x - ctr.x) * G.s, sy = (p[q].y - ctr.y) * G.s, sz = (p[q].z - ctr.z) * G.s;
          RS[0][i] = sx; RS[1][i] = sy; RS[2][i] = sz;
          RS[3][i] = id[q] >= 0 ? fmaf(sz, sz, fmaf(sy, sy, sx * sx)) : 1e30f;
          RS[4][i] = p[q].w;
          RI[i] = id[q];
        }
      }
      __syncwarp();
      flush_sym(c4);
      __syncwarp();
    }
#pragma unroll
    for (int t = 0; t < T; ++t) fo[t] = G.amp * ((acc[t].x + acc[t].y) * tf[t]);
    return;
  }
  const CellGrid& g = G.g;
  const float cc = G.cc, cc2 = G.cc2, h = g.h;
  const int z0 = cellof(blo.z - cc, g.lo[2], g.inv_h, g.dim[2]);
  const int z1 = cellof(bhi.z + cc, g.lo[2], g.inv_h, g.dim[2]);
  const int y0 = cellof(blo.y - cc, g.lo[1], g.inv_h, g.dim[1]);
  const int y1 = cellof(bhi.y + cc, g.lo[1], g.inv_h, g.dim[1]);
  const unsigned lt = (1u << lane) - 1u;
  int nS = 0, nO = 0;
  for (int cz = z0; cz <= z1; ++cz) {
    const float czlo = g.lo[2] + (float)cz * h;
    const float gz = fmaxf(0.f, fmaxf(czlo - bhi.z, blo.z - (czlo + h)));
    for (int cy = y0; cy <= y1; ++cy) {
      const float cylo = g.lo[1] + (float)cy * h;
      const float gy = fmaxf(0.f, fmaxf(cylo - bhi.y, blo.y - (cylo + h)));
      const float rem = cc2 - gy * gy - gz * gz;
      if (rem < 0.f) continue;
      const float rx = sqrtf(rem);
      const int x0 = cellof(blo.x - rx, g.lo[0], g.inv_h, g.dim[0]);
      const int x1 = cellof(bhi.x + rx, g.lo[0], g.inv_h, g.dim[0]);
      const int64_t rowbase = ((int64_t)cz * g.dim[1] + cy) * g.dim[0];
      const int sb = max(__ldg(cell_start + rowbase + x0), tl.x);
      const int se = min(__ldg(cell_start + rowbase + x1 + 1), (int)sym_hi);
      // a cell row lies in one z plane, so in one rank's slice
      const float4* __restrict__ srow = src;
      if constexpr (PEER) {
        if (sb < se) srow = PT->src[peer_of(*PT, sb)];
      }
      for (int j0 = sb; j0 < se; j0 += 32) {
        const int j = j0 + lane;
        const bool valid = j < se;
        const float4 p = valid ? __ldg(srow + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float gx = fmaxf(0.f, fmaxf(blo.x - p.x, p.x - bhi.x));
        const float gyy = fmaxf(0.f, fmaxf(blo.y - p.y, p.y - bhi.y));
        const float gzz = fmaxf(0.f, fmaxf(blo.z - p.z, p.z - bhi.z));
        const bool keep = valid && (gx * gx + gyy * gyy + gzz * gzz <= cc2);
        const bool own = j < t_end;
        const unsigned bs = __ballot_sync(0xffffffffu, keep && !own);
        const unsigned bo = __ballot_sync(0xffffffffu, keep && own);
        RBF_JITTER();
        if (keep) {
          const float sx = (p.x - ctr.x) * G.s, sy = (p.y - ctr.y) * G.s, sz = (p.z - ctr.z) * G.s;
          const float ss = fmaf(sz, sz, fmaf(sy, sy, sx * sx));
          if (!own) {
            const int pos = nS + __popc(bs & lt);
            RBF_DCHECK(pos < kSymPad);
            RS[0][pos] = sx; RS[1][pos] = sy; RS[2][pos] = sz; RS[3][pos] = ss; RS[4][pos] = p.w;
            RI[pos] = j;
          } else {
            const int pos = nO + __popc(bo & lt);
            RBF_DCHECK(pos < kOwnPad);
            O[0][pos] = sx; O[1][pos] = sy; O[2][pos] = sz; O[3][pos] = ss; O[4][pos] = p.w;
          }
        }
        nS += __popc(bs);
        nO += __popc(bo);
        if (nS >= kFlush) {
          __syncwarp();
          flush_sym(kFlush);
          __syncwarp();
          if (lane < nS - kFlush) {
            const int q = kFlush + lane;
            const float a = RS[0][q], b = RS[1][q], c = RS[2][q], d = RS[3][q], e = RS[4][q];
            const int ii = RI[q];
            RS[0][lane] = a; RS[1][lane] = b; RS[2][lane] = c; RS[3][lane] = d; RS[4][lane] = e; RI[lane] = ii;
          }
          __syncwarp();
          nS -= kFlush;
        }
        if (nO >= kFlush) {
          __syncwarp();
          flush_own(kFlush);
          __syncwarp();
          if (lane < nO - kFlush) {
            const int q = kFlush + lane;
            const float a = O[0][q], b = O[1][q], c = O[2][q], d = O[3][q], e = O[4][q];
            O[0][lane] = a; O[1][lane] = b; O[2][lane] = c; O[3][lane] = d; O[4][lane] = e;
          }
          __syncwarp();
          nO -= kFlush;
        }
      }
    }
  }
  {
    const int cntS = (nS + 3) & ~3;
    if (lane < cntS - nS) {
      const int q = nS + lane;
      RS[0][q] = 0.f; RS[1][q] = 0.f; RS[2][q] = 0.f; RS[3][q] = 1e30f; RS[4][q] = 0.f;
      RI[q] = -1;
    }
    const int cntO = (nO + 3) & ~3;
    if (lane < cntO - nO) {
      const int q = nO + lane;
      O[0][q] = 0.f; O[1][q] = 0.f; O[2][q] = 0.f; O[3][q] = 1e30f; O[4][q] = 0.f;
    }
    __syncwarp();
    flush_sym(cntS);
    flush_own(cntO);
    __syncwarp();
  }
#pragma unroll
  for (int t = 0; t < T; ++t) fo[t] = G.amp * ((acc[t].x + acc[t].y) * tf[t]);
}

#ifndef RBF_SYMB_MINB
#define RBF_SYMB_MINB 8
#endif
// NL: nl_off[tile] .. nl_off[tile + 1] (absolute tile ids; the pointer is shifted
// by the first tile of the list) delimit the tile's listed sources in nl_idx.
template <class OutT, bool PEER = false, bool NL = false>
__global__ void __launch_bounds__(kSumWarps * 32, RBF_SYMB_MINB)
sum_f32_symb_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ src,
                    const int2* __restrict__ tiles, const float4* __restrict__ tbox, int64_t ntiles,
                    int64_t tile_base, OutT* __restrict__ out, int* __restrict__ work, int64_t sym_hi,
                    const int32_t* __restrict__ order, PeerTab PT = PeerTab{},
                    const int32_t* __restrict__ nl_idx = nullptr, const uint32_t* __restrict__ nl_off = nullptr) {
  __shared__ __align__(16) float rings[kSumWarps][5][kSymPad];
  __shared__ int ringi[kSumWarps][kSymPad];
  __shared__ float ringk[kSumWarps][kSymPad + 32];   // + the dummy store slots of flush_sym
  __shared__ __align__(16) float ringo[kSumWarps][5][kOwnPad];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (;;) {
    int64_t tile;
    {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(work, 1);
      tile = __shfl_sync(0xffffffffu, t0, 0);
    }
    if (tile >= ntiles) break;
    tile = order ? (int64_t)order[tile] : tile + tile_base;
    const int2 tl = tiles[tile];
    const float4 a = tbox[2 * tile], b = tbox[2 * tile + 1];
    const float3 blo = make_float3(a.x, a.y, a.z), bhi = make_float3(b.x, b.y, b.z);
    const float3 ctr = make_float3(0.5f * (blo.x + bhi.x), 0.5f * (blo.y + bhi.y), 0.5f * (blo.z + bhi.z));
    float xr[4], yr[4], zr[4], wg[4], fo[4];
    bool tv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int q = lane + 32 * t;
      tv[t] = q < tl.y;
      const float4 p = src[tl.x + (tv[t] ? q : 0)];
      xr[t] = p.x; yr[t] = p.y; zr[t] = p.z; wg[t] = p.w;
    }
    const int T = (tl.y + 31) >> 5;
    uint32_t nb = 0, ne = 0;
    if constexpr (NL) { nb = nl_off[tile]; ne = nl_off[tile + 1]; }
    switch (T) {
      case 1: symb_tile<1, OutT, PEER, NL>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, sym_hi, lane, rings[wib], ringi[wib], ringk[wib], ringo[wib], out, fo, &PT, nl_idx, nb, ne); break;
      case 2: symb_tile<2, OutT, PEER, NL>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, sym_hi, lane, rings[wib], ringi[wib], ringk[wib], ringo[wib], out, fo, &PT, nl_idx, nb, ne); break;
      case 3: symb_tile<3, OutT, PEER, NL>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, sym_hi, lane, rings[wib], ringi[wib], ringk[wib], ringo[wib], out, fo, &PT, nl_idx, nb, ne); break;
      default: symb_tile<4, OutT, PEER, NL>(G, cell_start, src, blo, bhi, ctr, xr, yr, zr, tv, wg, tl, sym_hi, lane, rings[wib], ringi[wib], ringk[wib], ringo[wib], out, fo, &PT, nl_idx, nb, ne); break;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t < T && lane + 32 * t < tl.y) atomicAdd(out + tl.x + lane + 32 * t, (OutT)fo[t]);
  }
}

// ------------------------------------------------------------- fp64 tier ---
// exp(x) for the fp64 tier's arguments x = -d2 / (2 sigma^2), table-driven:
// n = rint(64 x log2 e) (the 1.5 2^52 rounding trick), x = (n/64) ln2 + r with
// |r| <= ln2/128 (two-part ln2/64: the high part has 32 significant bits, so
// n (ln2/64)_hi is exact for |n| < 2^20), e^x = 2^(n>>6) * 2^((n&63)/64) * e^r,
// 2^(j/64) from a 64-entry shared-memory table (exp2 at CTA start, <= 1 ulp),
// e^r by its degree-5 Taylor polynomial (truncation < 4e-17 relative), 2^(n>>6)
// added to the exponent field: 10 DP operations.  Valid (normal results) for x
// in [-700, 0]; the kernels only keep x >= -k c^2 = -18 at 6 sigma (pairs beyond
// the cutoff are computed and discarded by a select).  No range checks, no
// branches; every coefficient is a constant-bank (uniform) operand.
struct ExpConst {
  double log2e64, magic, ln2_hi64, ln2_lo64;
  double c[6];   // 1 / k!
};
__constant__ ExpConst kExp64 = {64 * 1.4426950408889634, 6755399441055744.0, 6.93147180369123816490e-01 / 64,
                                1.90821492927058770002e-10 / 64,
                                {1.0, 1.0, 1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120}};
constexpr int kExpTab = 64;

__device__ __forceinline__ void exp_tier64_table(double* tab) {
  for (int k = threadIdx.x; k < kExpTab; k += blockDim.x) tab[k] = exp2((double)k * (1.0 / kExpTab));
}

__device__ __forceinline__ double exp_tier64(double x, const double* __restrict__ tab) {
  const double t = __fma_rn(x, kExp64.log2e64, kExp64.magic);
  const double nd = __dsub_rn(t, kExp64.magic);
  const int n = __double2loint(t);
  double r = __fma_rn(-nd, kExp64.ln2_hi64, x);
  r = __fma_rn(-nd, kExp64.ln2_lo64, r);
  double p = kExp64.c[5];
#pragma unroll
  for (int k = 4; k >= 0; --k) p = __fma_rn(p, r, kExp64.c[k]);
  p = __dmul_rn(p, tab[n & (kExpTab - 1)]);
  return __hiloint2double(__double2hiint(p) + ((n >> 6) << 20), __double2loint(p));
}

// 2^(-y / 1024) for the expansion-form fp64 kernel, whose frame is scaled so that
// a pair's exponent arrives as y = 1024 |.|^2 log2(e) / (2 sigma^2) directly (no
// multiplication by log2 e, no two-part ln 2 reduction): n = rint(-y) by the
// 1.5 2^52 trick, g = y + n (exact: the two are within 1/2 of each other),
// 2^(-y/1024) = 2^(n >> 10) * 2^((n & 1023)/1024) * e^(-g ln2/1024), |g| <= 1/2:
// the last factor by its degree-3 Taylor polynomial (|arg| <= 3.4e-4,
// truncation 5.5e-16 relative), the middle one from a 1024-entry shared-memory
// table (exp2 at CTA start, <= 1 ulp): 2 DADD + 3 DFMA + 1 DMUL + the magic
// DADD = 7 DP operations instead of exp_tier64's 10.  Valid for -1e6 < y (the
// result is normal for |y| < 1e6); padded sources (y = 1e300) give a finite or
// non-finite garbage value that the caller's cutoff select discards.
constexpr int kExp2Tab = 1024;
struct Exp2Const {
  double magic, c1, c2, c3;   // (ln2/1024)^k / k!
};
__constant__ Exp2Const kExp2 = {6755399441055744.0, 6.769015435155716e-04, 2.290978498068816e-07,
                                5.169222938345892e-11};

__device__ __forceinline__ void exp2m_table(double* tab) {
  for (int k = threadIdx.x; k < kExp2Tab; k += blockDim.x) tab[k] = exp2((double)k * (1.0 / kExp2Tab));
}

__device__ __forceinline__ double exp2m_1024(double y, const double* __restrict__ tab) {
  const double t = __dsub_rn(kExp2.magic, y);
  const double nd = __dsub_rn(t, kExp2.magic);
  const int n = __double2loint(t);
  const double g = __dadd_rn(y, nd);
  double p = __fma_rn(-kExp2.c3, g, kExp2.c2);
  p = __fma_rn(p, g, -kExp2.c1);
  p = __fma_rn(p, g, 1.0);
  p = __dmul_rn(p, tab[n & (kExp2Tab - 1)]);
  return __hiloint2double(__double2hiint(p) + ((n >> 10) << 20), __double2loint(p));
}

struct Ring64 {
  float* bx; float* by; float* bz; double* bw;
};

struct Stage64 {
  Ring64 r;
  const float4* __restrict__ src;
  const double* __restrict__ w;
  float3 blo, bhi;
  float cc2;
  float4 p;
  double wj;
  __device__ __forceinline__ bool operator()(int j, bool valid) {
    p = valid ? __ldg(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    wj = valid ? __ldg(w + j) : 0.0;
    float gx = fmaxf(0.f, fmaxf(blo.x - p.x, p.x - bhi.x));
    float gy = fmaxf(0.f, fmaxf(blo.y - p.y, p.y - bhi.y));
    float gz = fmaxf(0.f, fmaxf(blo.z - p.z, p.z - bhi.z));
    return valid && (gx * gx + gy * gy + gz * gz <= cc2);
  }
  __device__ __forceinline__ void store(bool keep, int pos) {
    if (keep) { r.bx[pos] = p.x; r.by[pos] = p.y; r.bz[pos] = p.z; r.bw[pos] = wj; }
  }
  __device__ __forceinline__ void shift(int rest, int lane) {
    if (lane < rest) {
      float a = r.bx[kFlush + lane], b = r.by[kFlush + lane], c = r.bz[kFlush + lane];
      double d = r.bw[kFlush + lane];
      r.bx[lane] = a; r.by[lane] = b; r.bz[lane] = c; r.bw[lane] = d;
    }
  }
};

struct Flush64 {
  Ring64 r;
  double* acc;                       // [2]
  const double* xt; const double* yt; const double* zt;
  double c2, nis;                    // cutoff^2 and -1/(2 sigma^2); the amplitude is applied at the end
  const double* tab;                 // exp_tier64 table (shared memory)
  __device__ __forceinline__ void operator()(int cnt) {
    for (int j = 0; j < cnt; ++j) {
      const double sx = (double)r.bx[j], sy = (double)r.by[j], sz = (double)r.bz[j], wj = r.bw[j];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        double dx = __dsub_rn(sx, xt[t]), dy = __dsub_rn(sy, yt[t]), dz = __dsub_rn(sz, zt[t]);
        double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        // predicated (no divergent branch); exp(-d2/(2 sigma^2)) as a product by
        // the reciprocal: <= 1 ulp of the argument, ~1e-15 relative in the entry
        // (exp_tier64: a few ulp)
        const double e = exp_tier64(__dmul_rn(d2, nis), tab);
        acc[t] = __fma_rn(d2 <= c2 ? e : 0.0, wj, acc[t]);
      }
    }
  }
};

__global__ void __launch_bounds__(kSumWarps * 32)
sum_f64_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ src,
               const double* __restrict__ w, const int2* __restrict__ tiles,
               const float4* __restrict__ tbox, int64_t ntiles, int64_t tile_base, double* __restrict__ out,
               const int32_t* __restrict__ out_perm, int* __restrict__ work) {
  __shared__ __align__(16) float ringf[kSumWarps][3][kBufPad];
  __shared__ __align__(16) double ringd[kSumWarps][kBufPad];
  __shared__ double etab[kExpTab];
  exp_tier64_table(etab);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  Ring64 R{ringf[wib][0], ringf[wib][1], ringf[wib][2], ringd[wib]};
  for (;;) {
    int64_t tile;
    {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(work, 1);
      tile = __shfl_sync(0xffffffffu, t0, 0);
    }
    if (tile >= ntiles) break;
    tile += tile_base;
    const int2 tl = tiles[tile];
    const float4 a = tbox[2 * tile], b = tbox[2 * tile + 1];
    const float3 blo = make_float3(a.x, a.y, a.z), bhi = make_float3(b.x, b.y, b.z);
    double xt[2], yt[2], zt[2], acc[2] = {0.0, 0.0};
    bool tv[2];
    int64_t tidx[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      int q = lane + 32 * t;
      tv[t] = q < tl.y;
      tidx[t] = tl.x + (tv[t] ? q : 0);
      float4 p = src[tidx[t]];
      xt[t] = p.x; yt[t] = p.y; zt[t] = p.z;
    }
    Stage64 st{R, src, w, blo, bhi, G.cc2, make_float4(0, 0, 0, 0), 0.0};
    Flush64 fl{R, acc, xt, yt, zt, G.c2d, -1.0 / G.two_s2, etab};
    int nbuf = 0;
    traverse(G, cell_start, blo, bhi, lane, st, fl, nbuf);
    __syncwarp();
    fl(nbuf);
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (!tv[t]) continue;
      int64_t o = out_perm ? out_perm[tidx[t]] : tidx[t];
      out[o] = G.ampd * acc[t];
    }
  }
}

// Symmetric fp64 tier of the solver (reading R19, fp64 variant): two rings
// (one-sided: the tile's own and other ranks' sources; symmetric: this rank's
// sources after the tile), sources before the tile never loaded.  Each
// exponential of the symmetric ring serves f_i (lane accumulator) and f_j (warp
// butterfly over the lane partials sum_t e_tj w_t, one atomicAdd per source).
struct Ring64s {
  float* bx; float* by; float* bz; double* bw; int* bi;
};

struct Stage64x2 {
  Ring64s rb, ri;   // symmetric / one-sided
  const float4* __restrict__ src;
  const double* __restrict__ w;
  float3 blo, bhi;
  float cc2;
  int skip_lo, skip_hi, sym_lo, sym_hi;
  float4 p;
  double wj;
  int jj;
  __device__ __forceinline__ int classify(int j, bool valid) {
    p = valid ? __ldg(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    wj = valid ? __ldg(w + j) : 0.0;
    jj = j;
    if (j >= skip_lo && j < skip_hi) return 0;
    const float gx = fmaxf(0.f, fmaxf(blo.x - p.x, p.x - bhi.x));
    const float gy = fmaxf(0.f, fmaxf(blo.y - p.y, p.y - bhi.y));
    const float gz = fmaxf(0.f, fmaxf(blo.z - p.z, p.z - bhi.z));
    if (!valid || gx * gx + gy * gy + gz * gz > cc2) return 0;
    return (j >= sym_lo && j < sym_hi) ? 1 : 2;
  }
  __device__ __forceinline__ void store2(int kind, int posb, int posi) {
    if (kind == 0) return;
    Ring64s& r = (kind == 1) ? rb : ri;
    const int pos = (kind == 1) ? posb : posi;
    r.bx[pos] = p.x; r.by[pos] = p.y; r.bz[pos] = p.z; r.bw[pos] = wj;
    if (kind == 1) r.bi[pos] = jj;
  }
  __device__ __forceinline__ void shift_ring(Ring64s& r, int rest, int lane) {
    if (lane < rest) {
      float a = r.bx[kFlush + lane], b = r.by[kFlush + lane], c = r.bz[kFlush + lane];
      double d = r.bw[kFlush + lane];
      r.bx[lane] = a; r.by[lane] = b; r.bz[lane] = c; r.bw[lane] = d;
      if (r.bi) r.bi[lane] = r.bi[kFlush + lane];
    }
  }
};

template <bool SYM>
struct Flush64x {
  Ring64s r;
  double* acc;                       // [2]
  const double* xt; const double* yt; const double* zt;
  const double* wt;                  // [2] target weights (0 for empty slots), SYM only
  double c2, nis, amp;
  double* out;
  int lane;
  const double* tab;                 // exp_tier64 table (shared memory)
  // one staged source against the lane's 2 targets: e_t into acc (target side),
  // returns sum_t e_t wt_t (source side, SYM)
  __device__ __forceinline__ double pair(int j) {
    const double sx = (double)r.bx[j], sy = (double)r.by[j], sz = (double)r.bz[j], wj = r.bw[j];
    double pj = 0.0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      double dx = __dsub_rn(sx, xt[t]), dy = __dsub_rn(sy, yt[t]), dz = __dsub_rn(sz, zt[t]);
      double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      // computed for every staged pair and selected (no divergent branch)
      const double ex = exp_tier64(__dmul_rn(d2, nis), tab);
      const double e = d2 <= c2 ? ex : 0.0;
      acc[t] = __fma_rn(e, wj, acc[t]);
      if (SYM) pj = __fma_rn(e, wt[t], pj);
    }
    return pj;
  }
  __device__ __forceinline__ void operator()(int cnt) {
    if constexpr (SYM) {
      // 4 sources at a time (cnt is a multiple of 4: the ring is padded with
      // far-away zero-weight sources), their source-side sums over the warp's
      // 64 targets by a transpose-reduction (12 32-bit shuffles per 4 sources
      // instead of 40), one lane per source adds to f_j (same as Flush32s)
      const bool h4 = lane & 16, h3 = lane & 8;
      const int mys = (h4 ? 2 : 0) + (h3 ? 1 : 0);
      for (int j = 0; j < cnt; j += 4) {
        const double p0 = pair(j), p1 = pair(j + 1), p2 = pair(j + 2), p3 = pair(j + 3);
        double k0 = h4 ? p2 : p0, k1 = h4 ? p3 : p1;
        const double s0 = h4 ? p0 : p2, s1 = h4 ? p1 : p3;
        k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
        k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
        double k = h3 ? k1 : k0;
        k += __shfl_xor_sync(0xffffffffu, h3 ? k0 : k1, 8);
        k += __shfl_xor_sync(0xffffffffu, k, 4);
        k += __shfl_xor_sync(0xffffffffu, k, 2);
        k += __shfl_xor_sync(0xffffffffu, k, 1);
        if ((lane & 7) == 0) atomicAdd(out + r.bi[j + mys], amp * k);
      }
    } else {
      for (int j = 0; j < cnt; ++j) pair(j);
    }
  }
};

// Expansion form of the symmetric fp64 tier: sources staged (once per tile, one
// lane per source) in the tile-local frame scaled by q = 1/sqrt(2 sigma^2),
// s' = (x - ctr) q, with |s'|^2; a pair is then rr = |s'|^2 - 2 t'.s' (3 DFMA)
// and e = exp(-rr) exp(-|t'|^2), the per-target factor applied once at the end
// (cutoff: rr <= c^2 q^2 - |t'|^2 per target).  Against the difference form
// (3 F2F + 3 DADD + 3 DMUL + 2 DADD + 1 DMUL per pair) this removes ~6 of the
// ~22 DP operations per pair.  Rounding: |s'|, |t'| <= ~5 at the cutoff, so the
// expansion costs ~1e-14 absolute in the exponent (the fp64
// tier's gate is 1e-12 g_i per row).
struct Ring64e {
  double* sx; double* sy; double* sz; double* ss; double* w; int* bi;
};

struct Stage64e {
  Ring64e rb, ri;   // symmetric / one-sided
  const float4* __restrict__ src;
  const double* __restrict__ w;
  float3 blo, bhi;
  double cx, cy, cz, q;
  float cc2;
  int skip_lo, skip_hi, sym_lo, sym_hi;
  float4 p;
  double wj;
  int jj;
  __device__ __forceinline__ int classify(int j, bool valid) {
    p = valid ? __ldg(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    wj = valid ? __ldg(w + j) : 0.0;
    jj = j;
    if (j >= skip_lo && j < skip_hi) return 0;
    const float gx = fmaxf(0.f, fmaxf(blo.x - p.x, p.x - bhi.x));
    const float gy = fmaxf(0.f, fmaxf(blo.y - p.y, p.y - bhi.y));
    const float gz = fmaxf(0.f, fmaxf(blo.z - p.z, p.z - bhi.z));
    if (!valid || gx * gx + gy * gy + gz * gz > cc2) return 0;
    return (j >= sym_lo && j < sym_hi) ? 1 : 2;
  }
  __device__ __forceinline__ void store2(int kind, int posb, int posi) {
    if (kind == 0) return;
    Ring64e& r = (kind == 1) ? rb : ri;
    const int pos = (kind == 1) ? posb : posi;
    const double sx = ((double)p.x - cx) * q, sy = ((double)p.y - cy) * q, sz = ((double)p.z - cz) * q;
    r.sx[pos] = sx; r.sy[pos] = sy; r.sz[pos] = sz;
    r.ss[pos] = __fma_rn(sz, sz, __fma_rn(sy, sy, sx * sx));
    r.w[pos] = wj;
    if (kind == 1) r.bi[pos] = jj;
  }
  __device__ __forceinline__ void shift_ring(Ring64e& r, int rest, int lane) {
    if (lane < rest) {
      const int q0 = kFlush + lane;
      const double a = r.sx[q0], b = r.sy[q0], c = r.sz[q0], d = r.ss[q0], e = r.w[q0];
      r.sx[lane] = a; r.sy[lane] = b; r.sz[lane] = c; r.ss[lane] = d; r.w[lane] = e;
      if (r.bi) r.bi[lane] = r.bi[q0];
    }
  }
};

template <bool SYM>
struct Flush64e {
  Ring64e r;
  double* acc;                                            // [2]
  const double* mx; const double* my; const double* mz;   // [2] -2 t'
  const double* thr;                                      // [2] c^2 q^2 - |t'|^2
  const double* wt;                                       // [2] w_t exp(-|t'|^2) (0 for empty slots), SYM only
  double amp;
  double* out;
  int lane;
  const double* tab;
  __device__ __forceinline__ double pair(int j) {
    const double sx = r.sx[j], sy = r.sy[j], sz = r.sz[j], ss = r.ss[j], wj = r.w[j];
    double pj = 0.0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double rr = __fma_rn(mz[t], sz, __fma_rn(my[t], sy, __fma_rn(mx[t], sx, ss)));
      const double ex = exp2m_1024(rr, tab);
      const double e = rr <= thr[t] ? ex : 0.0;
      acc[t] = __fma_rn(e, wj, acc[t]);
      if (SYM) pj = __fma_rn(e, wt[t], pj);
    }
    return pj;
  }
  __device__ __forceinline__ void operator()(int cnt) {
    if constexpr (SYM) {
      const bool h4 = lane & 16, h3 = lane & 8;
      const int mys = (h4 ? 2 : 0) + (h3 ? 1 : 0);
      for (int j = 0; j < cnt; j += 4) {
        const double p0 = pair(j), p1 = pair(j + 1), p2 = pair(j + 2), p3 = pair(j + 3);
        double k0 = h4 ? p2 : p0, k1 = h4 ? p3 : p1;
        const double s0 = h4 ? p0 : p2, s1 = h4 ? p1 : p3;
        k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
        k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
        double k = h3 ? k1 : k0;
        k += __shfl_xor_sync(0xffffffffu, h3 ? k0 : k1, 8);
        k += __shfl_xor_sync(0xffffffffu, k, 4);
        k += __shfl_xor_sync(0xffffffffu, k, 2);
        k += __shfl_xor_sync(0xffffffffu, k, 1);
        if ((lane & 7) == 0) atomicAdd(out + r.bi[j + mys], amp * k);
      }
    } else {
      for (int j = 0; j < cnt; ++j) pair(j);
    }
  }
};

__global__ void __launch_bounds__(kSumWarps * 32)
sum_f64_syme_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ src,
                    const double* __restrict__ w, const int2* __restrict__ tiles, const float4* __restrict__ tbox,
                    int64_t ntiles, int64_t tile_base, double* __restrict__ out, int* __restrict__ work,
                    int64_t own_lo, int64_t own_hi) {
  __shared__ __align__(16) double ringd[kSumWarps][10][kBufPad];
  __shared__ __align__(16) int ringi[kSumWarps][kBufPad];
  // the exp2 table lives in dynamic shared memory (the rings fill the 48 KB static limit)
  extern __shared__ __align__(16) double etab[];
  exp2m_table(etab);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  Ring64e RB{ringd[wib][0], ringd[wib][1], ringd[wib][2], ringd[wib][3], ringd[wib][4], ringi[wib]};
  Ring64e RI{ringd[wib][5], ringd[wib][6], ringd[wib][7], ringd[wib][8], ringd[wib][9], nullptr};
  // frame scale: |.|^2 q^2 = 1024 log2(e) |.|^2 / (2 sigma^2) (exp2m_1024's argument)
  const double q2 = 1024.0 * 1.4426950408889634 / G.two_s2;
  const double q = sqrt(q2);
  const double c2q = G.c2d * q2;
  for (;;) {
    int64_t tile;
    {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(work, 1);
      tile = __shfl_sync(0xffffffffu, t0, 0);
    }
    if (tile >= ntiles) break;
    tile += tile_base;
    const int2 tl = tiles[tile];
    const float4 a = tbox[2 * tile], b = tbox[2 * tile + 1];
    const float3 blo = make_float3(a.x, a.y, a.z), bhi = make_float3(b.x, b.y, b.z);
    // tile centre (any fixed point: the expansion is exact algebra around it)
    const double cx = 0.5 * ((double)blo.x + (double)bhi.x), cy = 0.5 * ((double)blo.y + (double)bhi.y),
                 cz = 0.5 * ((double)blo.z + (double)bhi.z);
    double mx[2], my[2], mz[2], thr[2], tf[2], wt[2], acc[2] = {0.0, 0.0};
    bool tv[2];
    int64_t tidx[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      int qq = lane + 32 * t;
      tv[t] = qq < tl.y;
      tidx[t] = tl.x + (tv[t] ? qq : 0);
      const float4 p = src[tidx[t]];
      const double tx = ((double)p.x - cx) * q, ty = ((double)p.y - cy) * q, tz = ((double)p.z - cz) * q;
      const double tt = __fma_rn(tz, tz, __fma_rn(ty, ty, tx * tx));
      mx[t] = -2.0 * tx; my[t] = -2.0 * ty; mz[t] = -2.0 * tz;
      thr[t] = c2q - tt;
      tf[t] = exp2m_1024(tt, etab);
      wt[t] = tv[t] ? w[tidx[t]] * tf[t] : 0.0;
    }
    Stage64e st{RB, RI, src, w, blo, bhi, cx, cy, cz, q, G.cc2, (int)own_lo, tl.x, tl.x + tl.y, (int)own_hi,
                make_float4(0, 0, 0, 0), 0.0, 0};
    Flush64e<true> fs{RB, acc, mx, my, mz, thr, wt, G.ampd, out, lane, etab};
    Flush64e<false> fi{RI, acc, mx, my, mz, thr, wt, G.ampd, out, lane, etab};
    int nB = 0, nI = 0;
    traverse2(G, cell_start, blo, bhi, lane, st, fs, fi, nB, nI, st.skip_lo, st.skip_hi);
    // pad the symmetric ring to a multiple of 4 with zero-weight sources beyond
    // every cutoff (rr = 1e300 > thr: they contribute to neither side)
    const int cntB = (nB + 3) & ~3;
    if (lane < cntB - nB) {
      const int qq = nB + lane;
      RB.sx[qq] = 0.0; RB.sy[qq] = 0.0; RB.sz[qq] = 0.0; RB.ss[qq] = 1e300; RB.w[qq] = 0.0; RB.bi[qq] = tl.x;
    }
    __syncwarp();
    fs(cntB);
    fi(nI);
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 2; ++t)
      if (tv[t]) atomicAdd(out + tidx[t], G.ampd * (acc[t] * tf[t]));
  }
}

__global__ void __launch_bounds__(kSumWarps * 32)
sum_f64_sym_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ src,
                   const double* __restrict__ w, const int2* __restrict__ tiles, const float4* __restrict__ tbox,
                   int64_t ntiles, int64_t tile_base, double* __restrict__ out, int* __restrict__ work,
                   int64_t own_lo, int64_t own_hi) {
  __shared__ __align__(16) float ringf[kSumWarps][6][kBufPad];
  __shared__ __align__(16) double ringd[kSumWarps][2][kBufPad];
  __shared__ __align__(16) int ringi[kSumWarps][kBufPad];
  __shared__ double etab[kExpTab];
  exp_tier64_table(etab);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  Ring64s RB{ringf[wib][0], ringf[wib][1], ringf[wib][2], ringd[wib][0], ringi[wib]};
  Ring64s RI{ringf[wib][3], ringf[wib][4], ringf[wib][5], ringd[wib][1], nullptr};
  for (;;) {
    int64_t tile;
    {
      int t0 = 0;
      if (lane == 0) t0 = atomicAdd(work, 1);
      tile = __shfl_sync(0xffffffffu, t0, 0);
    }
    if (tile >= ntiles) break;
    tile += tile_base;
    const int2 tl = tiles[tile];
    const float4 a = tbox[2 * tile], b = tbox[2 * tile + 1];
    const float3 blo = make_float3(a.x, a.y, a.z), bhi = make_float3(b.x, b.y, b.z);
    double xt[2], yt[2], zt[2], wt[2], acc[2] = {0.0, 0.0};
    bool tv[2];
    int64_t tidx[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      int q = lane + 32 * t;
      tv[t] = q < tl.y;
      tidx[t] = tl.x + (tv[t] ? q : 0);
      float4 p = src[tidx[t]];
      xt[t] = p.x; yt[t] = p.y; zt[t] = p.z;
      wt[t] = tv[t] ? w[tidx[t]] : 0.0;
    }
    Stage64x2 st{RB, RI, src, w, blo, bhi, G.cc2, (int)own_lo, tl.x, tl.x + tl.y, (int)own_hi,
                 make_float4(0, 0, 0, 0), 0.0, 0};
    const double nis = -1.0 / G.two_s2;
    Flush64x<true> fs{RB, acc, xt, yt, zt, wt, G.c2d, nis, G.ampd, out, lane, etab};
    Flush64x<false> fi{RI, acc, xt, yt, zt, wt, G.c2d, nis, G.ampd, out, lane, etab};
    int nB = 0, nI = 0;
    traverse2(G, cell_start, blo, bhi, lane, st, fs, fi, nB, nI, st.skip_lo, st.skip_hi);
    // pad the symmetric ring to a multiple of 4 with far-away zero-weight
    // sources (d2 > c^2: they contribute to neither side)
    const int cntB = (nB + 3) & ~3;
    if (lane < cntB - nB) {
      const int q = nB + lane;
      RB.bx[q] = 1e30f; RB.by[q] = 1e30f; RB.bz[q] = 1e30f; RB.bw[q] = 0.0; RB.bi[q] = tl.x;
    }
    __syncwarp();
    fs(cntB);
    fi(nI);
    __syncwarp();
#pragma unroll
    for (int t = 0; t < 2; ++t)
      if (tv[t]) atomicAdd(out + tidx[t], G.ampd * acc[t]);
  }
}

// pack (x, y, z, w) records in sorted order for the fp32 tier
__global__ void pack_src_f32(const float4* __restrict__ sorted, const float* __restrict__ w, int64_t n,
                             float4* __restrict__ src) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float4 p = sorted[i];
    p.w = w ? w[i] : 0.f;
    src[i] = p;
  }
}
__global__ void pack_src_f64w(const float4* __restrict__ sorted, const double* __restrict__ w, int64_t n,
                              float4* __restrict__ src) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float4 p = sorted[i];
    p.w = (float)w[i];
    src[i] = p;
  }
}

SumGeom make_geom(const rbf_cells* c, const KernelParams& kp) {
  SumGeom G;
  for (int a = 0; a < 3; ++a) { G.g.lo[a] = c->lo[a]; G.g.dim[a] = c->dim[a]; }
  G.g.inv_h = c->inv_h;
  G.g.h = (float)c->h;
  double maxabs = 0;
  for (int a = 0; a < 3; ++a)
    maxabs = std::max(maxabs, std::max(std::fabs((double)c->lo[a]), std::fabs(c->lo[a] + c->dim[a] * c->h)));
  double cc = kp.cutoff * (1.0 + 1e-5) + 4e-7 * maxabs + 1e-30;
  G.cc = (float)cc;
  G.cc2 = (float)(cc * cc);
  const double ci = std::max(0.0, kp.cutoff * (1.0 - 1e-4) - 4e-7 * maxabs);
  G.ci2 = (float)(ci * ci);
  const double k = 1.4426950408889634 / (2.0 * kp.sigma * kp.sigma);
  G.s = (float)std::sqrt(k);
  float c2s = (float)(k * kp.cutoff * kp.cutoff);
  int bits;
  memcpy(&bits, &c2s, 4);
  G.c2bits = bits;
  G.c2s = c2s;
  G.amp = (float)kp.amp;
  G.c2d = kp.cutoff * kp.cutoff;
  G.two_s2 = 2.0 * kp.sigma * kp.sigma;
  G.ampd = kp.amp;
  return G;
}

// The expansion path's per-target factor 2^-|t'|^2 and terms 2^(|t'|^2 - ...) stay in
// fp32 range, and the expansion's rounding (~u (|s'|^2 + 2 |t'| |s'|) in the
// exponent, |s'| <= |t'| + sqrt(k) c) stays <= ~1e-5 relative per term, while
// |t'|^2 = k hd^2 <= 16 (hd = half-diagonal of the target box).  The configured
// plans give <= 7.3 (wide plan, h = c/4) and a 256^3 grid over c4 2.2; coarser
// grids (step >~ 1.8 sigma) or cell edges beyond ~c/2 take the difference form.
constexpr double kExpT2Max = 16.0;
bool expansion_ok(const KernelParams& kp, double hd2) {
  const double k = 1.4426950408889634 / (2.0 * kp.sigma * kp.sigma);
  return k * hd2 <= kExpT2Max;
}

// Solver fp32 tier variant of an rbf_op_variant: 0 = one-sided, 1 = symmetric on
// the 64-target plan, 2 = symmetric on the wide plan (reading R19).  RBF_OP_AUTO
// is 2 for slices of >= 2^18 centres (c4: 4.94 -> 3.61 ms) and 0 below (small
// problems have too few tiles to hide the longer wide tiles: c2 0.16 vs 0.21 ms).
int sym_mode(int op, int64_t n_loc) {
  switch (op) {
    case RBF_OP_ONESIDED: return 0;
    case RBF_OP_SYM: return 1;
    case RBF_OP_SYM_WIDE: return 2;
    case RBF_OP_SYM_ROT: return 3;
    default: return n_loc >= ((int64_t)1 << 18) ? 2 : 0;
  }
}

// Node blocks (4x4x4 grid nodes) in block layers [bz0, bz1) that hold a node
// within the culling radius cc of some centre: the grid evaluation visits only
// those (every other node has no centre within the cutoff: an exact zero,
// written by a memset).  One thread per non-empty cell: the tight bounding box
// of the cell's centres, the candidate blocks within cc of it per axis, and for
// each candidate the box-to-box distance (fp64) against cc (1 + 1e-6) -- the
// block box is the kernel's own (fp32 node coordinates), so a block whose nodes
// the kernel could give a non-zero value is never skipped.
__global__ void mark_node_blocks(const int32_t* __restrict__ cell_start, const float4* __restrict__ sorted,
                                 CellGrid g, float cc, GridDesc gd, int bz0, int bz1, uint32_t* __restrict__ flag) {
  const int64_t ncell = (int64_t)g.dim[0] * g.dim[1] * g.dim[2];
  const double ccd = (double)cc * (1.0 + 1e-6);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x) {
    const int s0 = cell_start[c], s1 = cell_start[c + 1];
    if (s1 == s0) continue;
    float lo3[3] = {INFINITY, INFINITY, INFINITY}, hi3[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int q = s0; q < s1; ++q) {
      const float4 p = sorted[q];
      lo3[0] = fminf(lo3[0], p.x); hi3[0] = fmaxf(hi3[0], p.x);
      lo3[1] = fminf(lo3[1], p.y); hi3[1] = fmaxf(hi3[1], p.y);
      lo3[2] = fminf(lo3[2], p.z); hi3[2] = fmaxf(hi3[2], p.z);
    }
    int b0[3], b1[3];
    bool empty = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double lo = (double)lo3[a] - ccd, hi = (double)hi3[a] + ccd;
      int i0 = (int)floor((lo - gd.lo[a]) / gd.step[a]) - 1, i1 = (int)ceil((hi - gd.lo[a]) / gd.step[a]) + 1;
      i0 = max(i0, 0);
      i1 = min(i1, gd.n[a] - 1);
      if (i0 > i1) empty = true;
      b0[a] = a < 2 ? i0 >> 2 : i0 / gd.bz;
      b1[a] = a < 2 ? i1 >> 2 : i1 / gd.bz;
    }
    b0[2] = max(b0[2], bz0);
    b1[2] = min(b1[2], bz1 - 1);
    if (empty || b0[2] > b1[2]) continue;
    for (int bz = b0[2]; bz <= b1[2]; ++bz) {
      const double gz = fmax(0.0, fmax((double)node_coord(gd, 2, gd.bz * bz) - hi3[2],
                                       (double)lo3[2] - (double)node_coord(gd, 2, min(gd.bz * bz + gd.bz - 1,
                                                                                      gd.n[2] - 1))));
      for (int by = b0[1]; by <= b1[1]; ++by) {
        const double gy = fmax(0.0, fmax((double)node_coord(gd, 1, 4 * by) - hi3[1],
                                         (double)lo3[1] - (double)node_coord(gd, 1, min(4 * by + 3, gd.n[1] - 1))));
        if (gy * gy + gz * gz > ccd * ccd) continue;
        for (int bx = b0[0]; bx <= b1[0]; ++bx) {
          const double gx = fmax(0.0, fmax((double)node_coord(gd, 0, 4 * bx) - hi3[0],
                                           (double)lo3[0] - (double)node_coord(gd, 0, min(4 * bx + 3, gd.n[0] - 1))));
          if (gx * gx + gy * gy + gz * gz <= ccd * ccd) flag[((int64_t)bz * gd.nb[1] + by) * gd.nb[0] + bx] = 1u;
        }
      }
    }
  }
}

// node blocks of layers [bz0, bz1) holding a node of the eps-surrounding
__global__ void mark_near_blocks(const uint8_t* __restrict__ near, GridDesc gd, int bz0, int bz1,
                                 uint32_t* __restrict__ flag) {
  const int64_t nn = (int64_t)gd.n[0] * gd.n[1] * gd.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    if (!near[v]) continue;
    const int i = (int)(v % gd.n[0]), j = (int)((v / gd.n[0]) % gd.n[1]), k = (int)(v / ((int64_t)gd.n[0] * gd.n[1]));
    const int bz = k / gd.bz;
    if (bz < bz0 || bz >= bz1) continue;
    flag[((int64_t)bz * gd.nb[1] + (j >> 2)) * gd.nb[0] + (i >> 2)] = 1u;
  }
}

__global__ void compact_blocks(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, int64_t n,
                               int32_t* __restrict__ list) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x)
    if (flag[b]) list[pos[b]] = (int32_t)b;
}

// Persistent grid: as many CTAs as can be resident (the kernels pull tiles from a
// work counter, so CTAs beyond one wave would only add tail imbalance).
template <class K>
int sum_blocks(rbf_ctx* ctx, K kernel, size_t dyn_smem = 0) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kSumWarps * 32, dyn_smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 4;
  }
  return ctx->sm_count * per_sm;
}

}  // namespace

KernelParams kernel_params(const rbf_kernel* k) {
  KernelParams p;
  p.sigma = k->sigma;
  p.cutoff = k->cutoff_sigmas * k->sigma;
  p.amp = k->amplitude > 0 ? k->amplitude : 1.0 / (std::sqrt(2.0 * M_PI) * k->sigma);
  return p;
}

namespace {
// Cost estimate of a wide tile for the symmetric kernels: target slots x the
// sources in the cell-row ranges its traversal loads (from the tile start to the
// window end), without loading them.  key = ~cost (ascending sort = most
// expensive first).
__global__ void tile_cost_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const int2* __restrict__ tiles,
                                 const float4* __restrict__ tbox, int64_t t0, int64_t nt, int64_t sym_hi,
                                 uint32_t* __restrict__ key, int32_t* __restrict__ id) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  const CellGrid& g = G.g;
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; w < nt; w += nw) {
    const int64_t tile = t0 + w;
    const int2 tl = tiles[tile];
    const float4 a = tbox[2 * tile], b = tbox[2 * tile + 1];
    const float3 blo = make_float3(a.x, a.y, a.z), bhi = make_float3(b.x, b.y, b.z);
    const int z0 = cellof(blo.z - G.cc, g.lo[2], g.inv_h, g.dim[2]);
    const int z1 = cellof(bhi.z + G.cc, g.lo[2], g.inv_h, g.dim[2]);
    const int y0 = cellof(blo.y - G.cc, g.lo[1], g.inv_h, g.dim[1]);
    const int y1 = cellof(bhi.y + G.cc, g.lo[1], g.inv_h, g.dim[1]);
    const int ny = y1 - y0 + 1, nrow = (z1 - z0 + 1) * ny;
    unsigned long long cnt = 0;
    for (int r = lane; r < nrow; r += 32) {
      const int cz = z0 + r / ny, cy = y0 + r % ny;
      const float czlo = g.lo[2] + (float)cz * g.h, cylo = g.lo[1] + (float)cy * g.h;
      const float gz = fmaxf(0.f, fmaxf(czlo - bhi.z, blo.z - (czlo + g.h)));
      const float gy = fmaxf(0.f, fmaxf(cylo - bhi.y, blo.y - (cylo + g.h)));
      const float rem = G.cc2 - gy * gy - gz * gz;
      if (rem < 0.f) continue;
      const float rx = sqrtf(rem);
      const int x0 = cellof(blo.x - rx, g.lo[0], g.inv_h, g.dim[0]);
      const int x1 = cellof(bhi.x + rx, g.lo[0], g.inv_h, g.dim[0]);
      const int64_t rowbase = ((int64_t)cz * g.dim[1] + cy) * g.dim[0];
      const int sb = max(cell_start[rowbase + x0], tl.x);
      const int se = min(cell_start[rowbase + x1 + 1], (int)sym_hi);
      if (se > sb) cnt += (unsigned long long)(se - sb);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) {
      const unsigned long long cost = cnt * (unsigned long long)((tl.y + 31) / 32);
      key[w] = 0xffffffffu - (uint32_t)min(cost, 0xffffffffull);
      id[w] = (int32_t)tile;
    }
  }
}
}  // namespace

// The order in which the symmetric kernels take this rank's wide tiles: most
// expensive first (longest-processing-time rule), so the last tiles a
// persistent warp picks up are the cheap ones and the end of the launch is not
// a tail of a few long tiles (~7 tiles per warp at c4).
rbf_status order_wide_tiles(rbf_ctx* ctx, rbf_cells* c, const KernelParams& kp) {
  cudaStream_t s = ctx->stream;
  const SlabView& V = c->view;
  const int64_t nt = V.tw1 - V.tw0;
  RBF_TRY(c->order_w.alloc(sizeof(int32_t) * std::max<int64_t>(nt, 1), s));
  if (nt == 0) return RBF_OK;
  DevBuf k1, v1, k2;
  RBF_TRY(k1.alloc(4 * nt, s));
  RBF_TRY(v1.alloc(4 * nt, s));
  RBF_TRY(k2.alloc(4 * nt, s));
  SumGeom G = make_geom(c, kp);
  tile_cost_kernel<<<grid_for(nt * 32, 256), 256, 0, s>>>(G, c->cell_start.as<int32_t>(), c->tiles_w.as<int2>(),
                                                          c->tile_box_w.as<float4>(), V.tw0, nt, V.h1,
                                                          k1.as<uint32_t>(), v1.as<int32_t>());
  RBF_CHECK_LAUNCH();
  // slab partition: the interior tiles [0, tw_int) and the halo tiles are
  // launched separately (the halo arrives in between), so each part is ordered
  // on its own; one GPU: tw_int = 0 and the whole range is one part
  const int64_t ni = (ctx->world > 1) ? V.tw_int : 0;
  if (ni > 0)
    RBF_TRY(radix_sort_pairs<uint32_t>(ctx, k1.as<uint32_t>(), v1.as<int32_t>(), k2.as<uint32_t>(),
                                       c->order_w.as<int32_t>(), ni, 32));
  if (nt > ni)
    RBF_TRY(radix_sort_pairs<uint32_t>(ctx, k1.as<uint32_t>() + ni, v1.as<int32_t>() + ni, k2.as<uint32_t>() + ni,
                                       c->order_w.as<int32_t>() + ni, nt - ni, 32));
  return RBF_OK;
}

namespace {
// Neighbour lists of the wide symmetric plan (NL form of sum_f32_symb_kernel):
// for every tile, the sorted indices of the sources after it (j >= tile end,
// j < sym_hi) that its traversal keeps -- the same cell rows, the same box cull
// and the same order as symb_tile's symmetric ring.  EMIT = false counts (and
// adds the total), EMIT = true writes them at off[w].  One warp per tile.
template <bool EMIT>
__global__ void nl_build_kernel(SumGeom G, const int32_t* __restrict__ cell_start, const float4* __restrict__ pos,
                                const int2* __restrict__ tiles, const float4* __restrict__ tbox, int64_t t0,
                                int64_t nt, int64_t sym_hi, uint32_t* __restrict__ cnt,
                                const uint32_t* __restrict__ off, int32_t* __restrict__ idx,
                                unsigned long long* __restrict__ total) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  const CellGrid& g = G.g;
  const float cc = G.cc, cc2 = G.cc2, h = g.h;
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; w < nt; w += nw) {
    const int64_t tile = t0 + w;
    const int2 tl = tiles[tile];
    const float4 a = tbox[2 * tile], b = tbox[2 * tile + 1];
    const float3 blo = make_float3(a.x, a.y, a.z), bhi = make_float3(b.x, b.y, b.z);
    const int t_end = tl.x + tl.y;
    const int z0 = cellof(blo.z - cc, g.lo[2], g.inv_h, g.dim[2]);
    const int z1 = cellof(bhi.z + cc, g.lo[2], g.inv_h, g.dim[2]);
    const int y0 = cellof(blo.y - cc, g.lo[1], g.inv_h, g.dim[1]);
    const int y1 = cellof(bhi.y + cc, g.lo[1], g.inv_h, g.dim[1]);
    uint32_t n = 0;
    int32_t* __restrict__ dst = EMIT ? idx + off[w] : nullptr;
    for (int cz = z0; cz <= z1; ++cz) {
      const float czlo = g.lo[2] + (float)cz * h;
      const float gz = fmaxf(0.f, fmaxf(czlo - bhi.z, blo.z - (czlo + h)));
      for (int cy = y0; cy <= y1; ++cy) {
        const float cylo = g.lo[1] + (float)cy * h;
        const float gy = fmaxf(0.f, fmaxf(cylo - bhi.y, blo.y - (cylo + h)));
        const float rem = cc2 - gy * gy - gz * gz;
        if (rem < 0.f) continue;
        const float rx = sqrtf(rem);
        const int x0 = cellof(blo.x - rx, g.lo[0], g.inv_h, g.dim[0]);
        const int x1 = cellof(bhi.x + rx, g.lo[0], g.inv_h, g.dim[0]);
        const int64_t rowbase = ((int64_t)cz * g.dim[1] + cy) * g.dim[0];
        const int sb = max(__ldg(cell_start + rowbase + x0), t_end);
        const int se = min(__ldg(cell_start + rowbase + x1 + 1), (int)sym_hi);
        for (int j0 = sb; j0 < se; j0 += 32) {
          const int j = j0 + lane;
          const bool valid = j < se;
          const float4 p = valid ? __ldg(pos + j) : make_float4(0.f, 0.f, 0.f, 0.f);
          const float gx = fmaxf(0.f, fmaxf(blo.x - p.x, p.x - bhi.x));
          const float gyy = fmaxf(0.f, fmaxf(blo.y - p.y, p.y - bhi.y));
          const float gzz = fmaxf(0.f, fmaxf(blo.z - p.z, p.z - bhi.z));
          const bool keep = valid && (gx * gx + gyy * gyy + gzz * gzz <= cc2);
          const unsigned bal = __ballot_sync(0xffffffffu, keep);
          if (EMIT && keep) dst[n + __popc(bal & lt)] = j;
          n += __popc(bal);
        }
      }
    }
    if (!EMIT && lane == 0) {
      cnt[w] = n;
      atomicAdd(total, (unsigned long long)n);
    }
  }
}
}  // namespace

// The neighbour lists of this rank's wide tiles for the kernel geometry kp
// (built on first use, kept with the cells while the culling radius and the
// source window stay the same).  *ok = false when they are switched off
// (rbf_ctx_neighbour_lists), exceed 2^31 entries, or do not fit in memory: the
// caller then runs the traversal form.
rbf_status ensure_nl(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp, bool* ok) {
  *ok = false;
  if (!ctx->nl_on) return RBF_OK;
  const SlabView& V = c->view;
  const int64_t nt = V.tw1 - V.tw0;
  SumGeom G = make_geom(c, kp);
  if (c->nl_state != 0 && c->nl_cc == G.cc && c->nl_hi == V.h1 && c->nl_t0 == V.tw0 && c->nl_nt == nt) {
    *ok = c->nl_state > 0;
    return RBF_OK;
  }
  cudaStream_t s = ctx->stream;
  c->nl_state = -1;
  c->nl_cc = G.cc; c->nl_hi = V.h1; c->nl_t0 = V.tw0; c->nl_nt = nt;
  c->nl_idx.release();
  c->nl_off.release();
  if (nt <= 0) return RBF_OK;
  ProfScope ps(ctx, RBF_PROF_CELLS);   // part of the cell structure's cost
  DevBuf cnt, tot;
  RBF_TRY(cnt.alloc(sizeof(uint32_t) * (nt + 1), s));
  RBF_TRY(tot.alloc(sizeof(unsigned long long), s));
  RBF_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(uint32_t) * (nt + 1), s));
  RBF_CUDA_TRY(cudaMemsetAsync(tot.p, 0, sizeof(unsigned long long), s));
  const int blocks = (int)std::min<int64_t>((nt + 7) / 8, 148 * 16);
  nl_build_kernel<false><<<blocks, 256, 0, s>>>(G, c->cell_start.as<int32_t>(), c->sorted.as<float4>(),
                                                 c->tiles_w.as<int2>(), c->tile_box_w.as<float4>(), V.tw0, nt, V.h1,
                                                 cnt.as<uint32_t>(), nullptr, nullptr, tot.as<unsigned long long>());
  RBF_CHECK_LAUNCH();
  unsigned long long total = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&total, tot.p, sizeof(total), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  if (total >= (1ull << 31)) return RBF_OK;
  if (c->nl_off.alloc(sizeof(uint32_t) * (nt + 1), s) != RBF_OK ||
      c->nl_idx.alloc(sizeof(int32_t) * std::max<unsigned long long>(total, 1), s) != RBF_OK) {
    cudaGetLastError();
    c->nl_idx.release();
    c->nl_off.release();
    return RBF_OK;   // no room: the traversal form
  }
  RBF_TRY(exclusive_scan_u32(ctx, cnt.as<uint32_t>(), c->nl_off.as<uint32_t>(), nt + 1, nullptr));
  nl_build_kernel<true><<<blocks, 256, 0, s>>>(G, c->cell_start.as<int32_t>(), c->sorted.as<float4>(),
                                                c->tiles_w.as<int2>(), c->tile_box_w.as<float4>(), V.tw0, nt, V.h1,
                                                nullptr, c->nl_off.as<uint32_t>(), c->nl_idx.as<int32_t>(), nullptr);
  RBF_CHECK_LAUNCH();
  c->nl_state = 1;
  c->nl_entries = (int64_t)total;
  *ok = true;
  return RBF_OK;
}

// Public fp32 path (and the pair accounting): w_sorted covers all n centres
// (sorted order); this rank's tiles write f_out[out_perm ? perm[j] : j].
rbf_status matvec_sorted_f32(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp,
                             const float* w_sorted, float* f_out, const int32_t* out_perm,
                             unsigned long long* pair_stats) {
  cudaStream_t s = ctx->stream;
  const int64_t n = c->n;
  const SlabView& V = c->view;
  RBF_TRY(ctx->src4.ensure(sizeof(float4) * n, s));
  RBF_TRY(ctx->counter.ensure(256, s));
  pack_src_f32<<<grid_for(n, 256), 256, 0, s>>>(c->sorted.as<float4>(), w_sorted, n, ctx->src4.as<float4>());
  RBF_CHECK_LAUNCH();
  RBF_CUDA_TRY(cudaMemsetAsync(ctx->counter.p, 0, sizeof(int), s));
  SumGeom G = make_geom(c, kp);
  GridDesc gd{};
  if (pair_stats) {
    sum_f32_kernel<0, true, float><<<sum_blocks(ctx, sum_f32_kernel<0, true, float>), kSumWarps * 32, 0, s>>>(
        G, c->cell_start.as<int32_t>(), ctx->src4.as<float4>(), c->tiles.as<int2>(), c->tile_box.as<float4>(),
        V.t1 - V.t0, V.t0, gd, f_out, out_perm, ctx->counter.as<int>(), pair_stats);
  } else if (expansion_ok(kp, c->hd2)) {
    ProfScope ps(ctx, RBF_PROF_MATVEC_F32);
    sum_f32_kernel<0, false, float><<<sum_blocks(ctx, sum_f32_kernel<0, false, float>), kSumWarps * 32, 0, s>>>(
        G, c->cell_start.as<int32_t>(), ctx->src4.as<float4>(), c->tiles.as<int2>(), c->tile_box.as<float4>(),
        V.t1 - V.t0, V.t0, gd, f_out, out_perm, ctx->counter.as<int>(), nullptr);
  } else {
    ProfScope ps(ctx, RBF_PROF_MATVEC_F32);
    auto kfn = sum_f32_kernel<0, false, float, false, true>;
    kfn<<<sum_blocks(ctx, kfn), kSumWarps * 32, 0, s>>>(
        G, c->cell_start.as<int32_t>(), ctx->src4.as<float4>(), c->tiles.as<int2>(), c->tile_box.as<float4>(),
        V.t1 - V.t0, V.t0, gd, f_out, out_perm, ctx->counter.as<int>(), nullptr, 0, 0, nullptr, nullptr);
  }
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}

// Solver path, fp32 tier: w_loc / f_loc are this rank's owned slice (sorted
// order, fp64).  The source window [h0, h1) is assembled by the halo exchange
// (world > 1); the kernel indexes sources and targets by global sorted
// position, so the window and output pointers are shifted by h0 and o0.
template <class WT>
static rbf_status matvec_f32_solver(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp, const WT* w_loc,
                                    double* f_loc, int op) {
  cudaStream_t s = ctx->stream;
  const SlabView& V = c->view;
  int sym = sym_mode(op, c->n_loc());
  if (sym >= 2 && !expansion_ok(kp, c->hd2_w)) sym = 0;
  if (sym == 1 && !expansion_ok(kp, c->hd2)) sym = 0;
  // one-sided: the window [h0, h1) around the slab; symmetric: [o0, h1) (sources
  // before a tile are never read; their contributions come back by halo_reduce)
  const int64_t base = sym ? V.o0 : V.h0;
  const int64_t nw = V.h1 - base;
  const WT* w_win = w_loc;
  // neighbour-list form of the wide symmetric kernel (built on the first product)
  bool nl = false;
  if (sym == 2) RBF_TRY(ensure_nl(ctx, c, kp, &nl));
  const int32_t* nl_idx = nl ? c->nl_idx.as<int32_t>() : nullptr;
  const uint32_t* nl_off = nl ? c->nl_off.as<uint32_t>() - V.tw0 : nullptr;
  // slab partition over a peer-memory transport (loopback, CUDA IPC), wide
  // symmetric operator: ONE kernel reads the upper ranks' packed sources and
  // adds the source-side sums into their accumulators in place, through peer
  // memory -- no halo exchange, no reverse halo reduction
  if (ctx->world > 1 && sym == 2 && ctx->peer_mem && ctx->tr->peer_capable() && c->order_w.p) {
    const SlabPlan& P = c->plan;
    PeerTab PT{};
    PT.n = 0;
    for (int q = ctx->rank; q < P.world && P.own_lo[q] < V.h1; ++q) {
      if (PT.n == kPeerMax) { PT.n = -1; break; }
      PT.lo[PT.n++] = P.own_lo[q];
    }
    if (PT.n > 0) {
      PT.lo[PT.n] = V.h1;
      // rank q's buffer: its packed sources, then (256-B aligned) its fp64 sums
      auto f_off = [&](int q) { return ((uint64_t)(P.own_hi[q] - P.own_lo[q]) * sizeof(float4) + 255) & ~(uint64_t)255; };
      const int64_t no = V.o1 - V.o0;
      const uint64_t need = f_off(ctx->rank) + (uint64_t)no * sizeof(double);
      std::vector<void*> bufs;
      auto stage = [&](void* mine) -> rbf_status {
        if (no > 0) {
          if constexpr (std::is_same<WT, double>::value)
            pack_src_f64w<<<grid_for(no, 256), 256, 0, s>>>(c->sorted.as<float4>() + V.o0, w_loc, no,
                                                            static_cast<float4*>(mine));
          else
            pack_src_f32<<<grid_for(no, 256), 256, 0, s>>>(c->sorted.as<float4>() + V.o0, w_loc, no,
                                                           static_cast<float4*>(mine));
          RBF_CHECK_LAUNCH();
          RBF_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(mine) + f_off(ctx->rank), 0, sizeof(double) * no, s));
        }
        return RBF_OK;
      };
      RBF_TRY(ctx->tr->peer_begin(ctx, s, need, stage, &bufs));
      for (int k = 0; k < PT.n; ++k) {
        const int q = ctx->rank + k;
        PT.src[k] = static_cast<const float4*>(bufs[q]) - P.own_lo[q];
        PT.f[k] = reinterpret_cast<double*>(static_cast<char*>(bufs[q]) + f_off(q)) - P.own_lo[q];
      }
      RBF_TRY(ctx->counter.ensure(256, s));
      RBF_CUDA_TRY(cudaMemsetAsync(ctx->counter.p, 0, sizeof(int), s));
      SumGeom G = make_geom(c, kp);
      {
        ProfScope ps(ctx, RBF_PROF_MATVEC_F32);
        auto kfn = nl ? sum_f32_symb_kernel<double, true, true> : sum_f32_symb_kernel<double, true>;
        kfn<<<sum_blocks(ctx, kfn), kSumWarps * 32, 0, s>>>(G, c->cell_start.as<int32_t>(), PT.src[0],
                                                            c->tiles_w.as<int2>(), c->tile_box_w.as<float4>(),
                                                            V.tw1 - V.tw0, V.tw0, PT.f[0], ctx->counter.as<int>(),
                                                            V.h1, c->order_w.as<int32_t>(), PT, nl_idx, nl_off);
        RBF_CHECK_LAUNCH();
      }
      RBF_TRY(ctx->tr->peer_end(ctx, s));   // every rank's kernel has added into my sums
      if (no > 0)
        RBF_CUDA_TRY(cudaMemcpyAsync(f_loc, static_cast<char*>(bufs[ctx->rank]) + f_off(ctx->rank),
                                     sizeof(double) * no, cudaMemcpyDeviceToDevice, s));
      return RBF_OK;
    }
  }
  // slab partition, wide symmetric operator: the upper halo is exchanged and
  // packed on the aux stream while the interior tiles (no halo sources) run
  const bool overlap = ctx->world > 1 && sym >= 2 && V.tw_int > 0 && c->order_w.p;
  if (ctx->world > 1 && !overlap) {
    RBF_TRY(ctx->win.ensure(sizeof(WT) * std::max<int64_t>(nw, 1), s));
    RBF_TRY(halo_exchange<WT>(ctx, c, w_loc, ctx->win.as<WT>(), sym != 0));
    w_win = ctx->win.as<WT>();
  }
  if (overlap) {
    RBF_TRY(ctx->win.ensure(sizeof(WT) * std::max<int64_t>(nw, 1), s));
    RBF_TRY(ctx->src4.ensure(sizeof(float4) * std::max<int64_t>(nw, 1), s));
    RBF_TRY(ctx->counter.ensure(256, s));
    if (!ctx->aux_stream) RBF_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->halo_ev)
      if (!e) RBF_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaStream_t a = ctx->aux_stream;
    const int64_t no = V.o1 - V.o0;
    // fork: the halo (and its packing) on the aux stream once w_loc is ready
    RBF_CUDA_TRY(cudaEventRecord(ctx->halo_ev[0], s));
    RBF_CUDA_TRY(cudaStreamWaitEvent(a, ctx->halo_ev[0], 0));
    {
      cudaStream_t keep = ctx->stream;
      ctx->stream = a;   // the transport and the pack run on the aux stream
      rbf_status st = halo_exchange<WT>(ctx, c, w_loc, ctx->win.as<WT>(), true);
      if (st == RBF_OK && nw > no) {
        if constexpr (std::is_same<WT, double>::value)
          pack_src_f64w<<<grid_for(nw - no, 256), 256, 0, a>>>(c->sorted.as<float4>() + V.o1, ctx->win.as<WT>() + no,
                                                              nw - no, ctx->src4.as<float4>() + no);
        else
          pack_src_f32<<<grid_for(nw - no, 256), 256, 0, a>>>(c->sorted.as<float4>() + V.o1, ctx->win.as<WT>() + no,
                                                             nw - no, ctx->src4.as<float4>() + no);
        count_launch();
        if (cudaGetLastError() != cudaSuccess) st = RBF_ECUDA;
      }
      ctx->stream = keep;
      RBF_TRY(st);
    }
    RBF_CUDA_TRY(cudaEventRecord(ctx->halo_ev[1], a));
    // the own slice on the main stream, the interior tiles while the halo arrives
    if (no > 0) {
      if constexpr (std::is_same<WT, double>::value)
        pack_src_f64w<<<grid_for(no, 256), 256, 0, s>>>(c->sorted.as<float4>() + V.o0, w_loc, no,
                                                        ctx->src4.as<float4>());
      else
        pack_src_f32<<<grid_for(no, 256), 256, 0, s>>>(c->sorted.as<float4>() + V.o0, w_loc, no,
                                                       ctx->src4.as<float4>());
      RBF_CHECK_LAUNCH();
    }
    RBF_TRY(ctx->fwin.ensure(sizeof(double) * std::max<int64_t>(nw, 1), s));
    double* fwin = ctx->fwin.as<double>();
    RBF_CUDA_TRY(cudaMemsetAsync(fwin, 0, sizeof(double) * (size_t)nw, s));
    RBF_CUDA_TRY(cudaMemsetAsync(ctx->counter.p, 0, 2 * sizeof(int), s));
    SumGeom G = make_geom(c, kp);
    const float4* srcb = ctx->src4.as<float4>() - base;
    auto kfn = sym == 3 ? sum_f32_symr_kernel<double>
                        : (nl ? sum_f32_symb_kernel<double, false, true> : sum_f32_symb_kernel<double>);
    const int64_t ni = V.tw_int, nb = (V.tw1 - V.tw0) - ni;
    {
      ProfScope ps(ctx, RBF_PROF_MATVEC_F32);
      kfn<<<sum_blocks(ctx, kfn), kSumWarps * 32, 0, s>>>(G, c->cell_start.as<int32_t>(), srcb, c->tiles_w.as<int2>(),
                                                          c->tile_box_w.as<float4>(), ni, V.tw0, fwin - base,
                                                          ctx->counter.as<int>(), V.h1, c->order_w.as<int32_t>(),
                                                          PeerTab{}, nl_idx, nl_off);
      RBF_CHECK_LAUNCH();
      // join: the halo tiles after the halo
      RBF_CUDA_TRY(cudaStreamWaitEvent(s, ctx->halo_ev[1], 0));
      if (nb > 0) {
        kfn<<<sum_blocks(ctx, kfn), kSumWarps * 32, 0, s>>>(
            G, c->cell_start.as<int32_t>(), srcb, c->tiles_w.as<int2>(), c->tile_box_w.as<float4>(), nb, V.tw0,
            fwin - base, ctx->counter.as<int>() + 1, V.h1, c->order_w.as<int32_t>() + ni, PeerTab{}, nl_idx,
            nl_off);
        RBF_CHECK_LAUNCH();
      }
    }
    return halo_reduce(ctx, c, fwin, f_loc);
  }
  RBF_TRY(ctx->src4.ensure(sizeof(float4) * std::max<int64_t>(nw, 1), s));
  RBF_TRY(ctx->counter.ensure(256, s));
  if (nw > 0) {
    if constexpr (std::is_same<WT, double>::value)
      pack_src_f64w<<<grid_for(nw, 256), 256, 0, s>>>(c->sorted.as<float4>() + base, w_win, nw,
                                                      ctx->src4.as<float4>());
    else
      pack_src_f32<<<grid_for(nw, 256), 256, 0, s>>>(c->sorted.as<float4>() + base, w_win, nw,
                                                     ctx->src4.as<float4>());
    RBF_CHECK_LAUNCH();
  }
  RBF_CUDA_TRY(cudaMemsetAsync(ctx->counter.p, 0, sizeof(int), s));
  SumGeom G = make_geom(c, kp);
  GridDesc gd{};
  const float4* srcb = ctx->src4.as<float4>() - base;
  if (sym) {
    // symmetric evaluation (reading R19): accumulated into the window [o0, h1)
    double* fwin = f_loc;
    if (ctx->world > 1) {
      RBF_TRY(ctx->fwin.ensure(sizeof(double) * std::max<int64_t>(nw, 1), s));
      fwin = ctx->fwin.as<double>();
    }
    RBF_CUDA_TRY(cudaMemsetAsync(fwin, 0, sizeof(double) * (size_t)std::max<int64_t>(nw, 0), s));
    {
      ProfScope ps(ctx, RBF_PROF_MATVEC_F32);
      if (sym >= 2) {
        auto kfn = sym == 3 ? sum_f32_symr_kernel<double>
                            : (nl ? sum_f32_symb_kernel<double, false, true> : sum_f32_symb_kernel<double>);
        kfn<<<sum_blocks(ctx, kfn), kSumWarps * 32, 0, s>>>(
            G, c->cell_start.as<int32_t>(), srcb, c->tiles_w.as<int2>(), c->tile_box_w.as<float4>(), V.tw1 - V.tw0,
            V.tw0, fwin - base, ctx->counter.as<int>(), V.h1, c->order_w.p ? c->order_w.as<int32_t>() : nullptr,
            PeerTab{}, nl_idx, nl_off);
      } else {
        sum_f32_kernel<0, false, double, true>
            <<<sum_blocks(ctx, sum_f32_kernel<0, false, double, true>), kSumWarps * 32, 0, s>>>(
                G, c->cell_start.as<int32_t>(), srcb, c->tiles.as<int2>(), c->tile_box.as<float4>(), V.t1 - V.t0,
                V.t0, gd, fwin - base, nullptr, ctx->counter.as<int>(), nullptr, 0, V.h1);
      }
      RBF_CHECK_LAUNCH();
    }
    return halo_reduce(ctx, c, fwin, f_loc);
  }
  ProfScope ps(ctx, RBF_PROF_MATVEC_F32);
  auto kfn = expansion_ok(kp, c->hd2) ? sum_f32_kernel<0, false, double> : sum_f32_kernel<0, false, double, false, true>;
  kfn<<<sum_blocks(ctx, kfn), kSumWarps * 32, 0, s>>>(
      G, c->cell_start.as<int32_t>(), srcb, c->tiles.as<int2>(), c->tile_box.as<float4>(), V.t1 - V.t0, V.t0, gd,
      f_loc - V.o0, nullptr, ctx->counter.as<int>(), nullptr, 0, 0, nullptr, nullptr);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}

rbf_status matvec_sorted_f32_d(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp, const double* w_loc,
                               double* f_loc, int op) {
  return matvec_f32_solver<double>(ctx, c, kp, w_loc, f_loc, op);
}
rbf_status matvec_sorted_f32_f(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp, const float* w_loc,
                               double* f_loc, int op) {
  return matvec_f32_solver<float>(ctx, c, kp, w_loc, f_loc, op);
}

// fp64 tier, same conventions as matvec_sorted_f32_d; out_perm (single GPU,
// public path only) scatters to the caller's order.
rbf_status matvec_sorted_f64(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp,
                             const double* w_loc, double* f_out, const int32_t* out_perm, int op) {
  cudaStream_t s = ctx->stream;
  const SlabView& V = c->view;
  const bool sym = !out_perm && sym_mode(op, c->n_loc()) != 0;
  const int64_t base = sym ? V.o0 : V.h0;
  const int64_t nw = V.h1 - base;
  const double* w_win = w_loc;
  if (ctx->world > 1) {
    RBF_TRY(ctx->win.ensure(sizeof(double) * std::max<int64_t>(nw, 1), s));
    RBF_TRY(halo_exchange<double>(ctx, c, w_loc, ctx->win.as<double>(), sym));
    w_win = ctx->win.as<double>();
  }
  RBF_TRY(ctx->counter.ensure(256, s));
  RBF_CUDA_TRY(cudaMemsetAsync(ctx->counter.p, 0, sizeof(int), s));
  SumGeom G = make_geom(c, kp);
  if (sym) {
    // solver path: symmetric fp64 tier (reading R19), accumulated into [o0, h1)
    double* fwin = f_out;
    if (ctx->world > 1) {
      RBF_TRY(ctx->fwin.ensure(sizeof(double) * std::max<int64_t>(nw, 1), s));
      fwin = ctx->fwin.as<double>();
    }
    RBF_CUDA_TRY(cudaMemsetAsync(fwin, 0, sizeof(double) * (size_t)std::max<int64_t>(nw, 0), s));
    {
      ProfScope ps(ctx, RBF_PROF_MATVEC_F64);
      // expansion form unless the tile boxes are too large for exp(+|t'|^2) (never
      // with the default cells: |t'|^2 <= hd2 / (2 sigma^2))
      const bool expf = c->hd2 / (2.0 * kp.sigma * kp.sigma) <= 300.0;
      auto kfn = expf ? sum_f64_syme_kernel : sum_f64_sym_kernel;
      const size_t dyn = expf ? sizeof(double) * kExp2Tab : 0;   // exp2m_1024's table
      if (dyn) RBF_TRY(smem_limit_at_least(kfn, dyn));
      kfn<<<sum_blocks(ctx, kfn, dyn), kSumWarps * 32, dyn, s>>>(
          G, c->cell_start.as<int32_t>(), c->sorted.as<float4>(), w_win - base, c->tiles.as<int2>(),
          c->tile_box.as<float4>(), V.t1 - V.t0, V.t0, fwin - base, ctx->counter.as<int>(), 0, V.h1);
      RBF_CHECK_LAUNCH();
    }
    return halo_reduce(ctx, c, fwin, f_out);
  }
  ProfScope ps(ctx, RBF_PROF_MATVEC_F64);
  sum_f64_kernel<<<sum_blocks(ctx, sum_f64_kernel), kSumWarps * 32, 0, s>>>(
      G, c->cell_start.as<int32_t>(), c->sorted.as<float4>(), w_win - base, c->tiles.as<int2>(),
      c->tile_box.as<float4>(), V.t1 - V.t0, V.t0, out_perm ? f_out : f_out - V.o0, out_perm,
      ctx->counter.as<int>());
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}

rbf_status eval_grid_sorted(rbf_ctx* ctx, const rbf_cells* c, const KernelParams& kp,
                            const double* w_sorted, const rbf_grid* g, float* field,
                            unsigned long long* pair_stats, const uint8_t* near) {
  cudaStream_t s = ctx->stream;
  const int64_t n = c->n;
  RBF_TRY(ctx->src4.ensure(sizeof(float4) * n, s));
  RBF_TRY(ctx->counter.ensure(256, s));
  if (w_sorted) {
    pack_src_f64w<<<grid_for(n, 256), 256, 0, s>>>(c->sorted.as<float4>(), w_sorted, n, ctx->src4.as<float4>());
  } else {
    pack_src_f32<<<grid_for(n, 256), 256, 0, s>>>(c->sorted.as<float4>(), nullptr, n, ctx->src4.as<float4>());
  }
  RBF_CHECK_LAUNCH();
  RBF_CUDA_TRY(cudaMemsetAsync(ctx->counter.p, 0, sizeof(int), s));
  SumGeom G = make_geom(c, kp);
  GridDesc gd;
  for (int a = 0; a < 3; ++a) {
    gd.lo[a] = g->lo[a];
    gd.step[a] = (g->hi[a] - g->lo[a]) / (double)(g->n[a] - 1);
    gd.n[a] = g->n[a];
    gd.nb[a] = a < 2 ? (g->n[a] + 3) / 4 : (g->n[a] + kGridBz - 1) / kGridBz;
  }
  gd.bz = kGridBz;
  const int64_t per_layer = (int64_t)gd.nb[0] * gd.nb[1];
  // this rank's node-block layers (all of them on one GPU; dist.cu grid_layers)
  int64_t k0n, k1n;
  grid_layers(c, g, ctx->rank, &k0n, &k1n);
  const int64_t b0 = per_layer * (k0n / kGridBz), b1 = per_layer * ((k1n + kGridBz - 1) / kGridBz);
  // node blocks within reach of a centre (the rest of this rank's layers are
  // exact zeros): flags -> scan -> list (one host read of the count)
  ProfScope ps(pair_stats ? nullptr : ctx, RBF_PROF_GRID);
  const int64_t nbt = per_layer * gd.nb[2];
  DevBuf flag, pos, list, cnt;
  RBF_TRY(flag.alloc(4 * (size_t)std::max<int64_t>(nbt, 1), s));
  RBF_TRY(pos.alloc(4 * (size_t)std::max<int64_t>(nbt, 1), s));
  RBF_TRY(list.alloc(4 * (size_t)std::max<int64_t>(nbt, 1), s));
  RBF_TRY(cnt.alloc(4, s));
  RBF_CUDA_TRY(cudaMemsetAsync(flag.p, 0, 4 * (size_t)nbt, s));
  const int64_t ncell = (int64_t)c->dim[0] * c->dim[1] * c->dim[2];
  if (near) {
    // eps-surrounding: the node blocks holding a node within eps of the data
    const int64_t nn = (int64_t)gd.n[0] * gd.n[1] * gd.n[2];
    mark_near_blocks<<<grid_for(nn, 256), 256, 0, s>>>(near, gd, (int)(b0 / per_layer), (int)(b1 / per_layer),
                                                       flag.as<uint32_t>());
  } else {
    mark_node_blocks<<<grid_for(ncell, 256), 256, 0, s>>>(c->cell_start.as<int32_t>(), c->sorted.as<float4>(), G.g,
                                                           G.cc, gd,
                                                           (int)(b0 / per_layer), (int)(b1 / per_layer),
                                                           flag.as<uint32_t>());
  }
  RBF_CHECK_LAUNCH();
  RBF_TRY(exclusive_scan_u32(ctx, flag.as<uint32_t>(), pos.as<uint32_t>(), nbt, cnt.as<uint32_t>()));
  compact_blocks<<<grid_for(nbt, 256), 256, 0, s>>>(flag.as<uint32_t>(), pos.as<uint32_t>(), nbt,
                                                     list.as<int32_t>());
  RBF_CHECK_LAUNCH();
  uint32_t nact = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&nact, cnt.p, 4, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  // this rank's node layers [b0, b1) start as zeros; the active blocks overwrite theirs
  const int64_t n0 = (int64_t)gd.n[0] * gd.n[1];
  const int64_t k0 = std::min<int64_t>((b0 / per_layer) * kGridBz, gd.n[2]),
                k1 = std::min<int64_t>((b1 / per_layer) * kGridBz, gd.n[2]);
  if (k1 > k0 && !pair_stats)   // zeros, or NaN (all bits set) outside the eps-surrounding
    RBF_CUDA_TRY(cudaMemsetAsync(field + k0 * n0, near ? 0xff : 0, sizeof(float) * (size_t)((k1 - k0) * n0), s));
  if (nact == 0) return RBF_OK;
  if (pair_stats) {
    sum_f32_kernel<1, true, float><<<sum_blocks(ctx, sum_f32_kernel<1, true, float>), kSumWarps * 32, 0, s>>>(
        G, c->cell_start.as<int32_t>(), ctx->src4.as<float4>(), nullptr, nullptr, nact, 0, gd, field, nullptr,
        ctx->counter.as<int>(), pair_stats, 0, 0, list.as<int32_t>());
    RBF_CHECK_LAUNCH();
    return RBF_OK;
  }
  // node block half-diagonal: 3 steps along x, y and bz - 1 along z, halved
  const double hz = 0.5 * (kGridBz - 1);
  const double hd2 = 2.25 * (gd.step[0] * gd.step[0] + gd.step[1] * gd.step[1]) + hz * hz * gd.step[2] * gd.step[2];
  if (kGridBz == 4 && !ctx->grid_per_pair) {
    // separable form: 12 exponentials per centre and 4 x 4 x 4 node block
    grid_sep_kernel<<<sum_blocks(ctx, grid_sep_kernel), kSumWarps * 32, 0, s>>>(
        G, c->cell_start.as<int32_t>(), ctx->src4.as<float4>(), nact, gd, field, ctx->counter.as<int>(),
        list.as<int32_t>(), near);
    RBF_CHECK_LAUNCH();
    return RBF_OK;
  }
  auto kfn = expansion_ok(kp, hd2) ? sum_f32_kernel<1, false, float> : sum_f32_kernel<1, false, float, false, true>;
  kfn<<<sum_blocks(ctx, kfn), kSumWarps * 32, 0, s>>>(
      G, c->cell_start.as<int32_t>(), ctx->src4.as<float4>(), nullptr, nullptr, nact, 0, gd, field, nullptr,
      ctx->counter.as<int>(), nullptr, 0, 0, list.as<int32_t>(), near);
  RBF_CHECK_LAUNCH();
  return RBF_OK;
}

}  // namespace rbf
