// Alg.1 steps 3-4 restricted to the eps-surrounding:
// P_f evaluated only on the grid nodes within eps of the data (M_ext^eps,
// §2.1.3), then the triangle mesh of its zero iso-surface (P:317-328,
// the paper's MATLAB `isosurface`).  Reading R24: marching
// tetrahedra on the Kuhn split of every grid cube, so the mesh is watertight
// inside the mask with no ambiguity tables.
//
// Definitions (include/rbf.h; oracle/mesh.py writes the same ones out on the CPU):
//   inside(v) = F[v] < 0; near(v) from build_near_mask (fp64 distances);
//   edge (v, d), d in D7 = x, y, z, xy, xz, yz, xyz: a vertex iff both ends near
//   and inside differs; p_v + t (p_u - p_v), t = F_v / (F_v - F_u) in fp64;
//   vertices numbered in (v, d) order;
//   cube (lower corner v) polygonised iff its 8 corners are near; tetrahedra
//   for the axis permutations xyz xzy yxz yzx zxy zyx: corners 0, e_p0,
//   e_p0 + e_p1, (1,1,1); |I| = 1, 3: triangle on the lone corner's 3 edges,
//   |I| = 2 (a < b inside, c < d outside): (ac, ad, bd), (ac, bd, bc);
//   orientation: the normal of the midpoint polygon points from the inside
//   corners to the outside corners (integer arithmetic on doubled lattice
//   coordinates, so the decision is exact), else the last two vertices swap;
//   triangles in (cube, tet, triangle) order.
// GPU steps: per-node 7-bit edge masks + exclusive scan (vertex ids), vertex
// emission; per-cube triangle counts + exclusive scan, triangle emission.  Every
// pass is one coalesced sweep over the node arrays (HBM-bound).
#include <cmath>

#include "internal.h"

struct rbf_mesh {
  rbf::DevBuf verts;   // double[3 * nv]
  rbf::DevBuf tris;    // int32[3 * nt]
  int64_t nv = 0, nt = 0;
};

namespace rbf {
namespace {

struct MGrid {
  double lo[3], step[3];
  int n[3];
};

// lo + i * step, two roundings (the oracle's nodes())
__device__ __forceinline__ double mcoord(const MGrid& g, int a, int i) {
  return __dadd_rn(g.lo[a], __dmul_rn((double)i, g.step[a]));
}

// corner code c: bit0 = +x, bit1 = +y, bit2 = +z.  D7 direction index of the
// edge from corner ca to corner cb (ca a bit-subset of cb): diff bits -> d
__device__ __forceinline__ int dir_of(int diff) {
  // 1:x 2:y 4:z 3:xy 5:xz 6:yz 7:xyz  ->  0 1 2 3 4 5 6
  constexpr int tab[8] = {-1, 0, 1, 3, 2, 4, 5, 6};
  return tab[diff];
}
__device__ __forceinline__ int3 dvec(int d) {
  constexpr int code[7] = {1, 2, 4, 3, 5, 6, 7};
  const int c = code[d];
  return make_int3(c & 1, (c >> 1) & 1, (c >> 2) & 1);
}

// tet corner codes for the permutations xyz xzy yxz yzx zxy zyx
__constant__ int kTet[6][4] = {{0, 1, 3, 7}, {0, 1, 5, 7}, {0, 2, 3, 7}, {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 6, 7}};

__device__ __forceinline__ int64_t flat_of(const MGrid& g, int i, int j, int k) {
  return (int64_t)i + (int64_t)g.n[0] * ((int64_t)j + (int64_t)g.n[1] * k);
}

// per node: 7-bit mask of the edges (v, d) carrying a vertex, and its popcount
__global__ void mt_edge_kernel(const float* __restrict__ F, const uint8_t* __restrict__ near, MGrid g,
                               uint8_t* __restrict__ emask, uint32_t* __restrict__ cnt) {
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    unsigned m = 0;
    if (near[v]) {
      const int i = (int)(v % g.n[0]), j = (int)((v / g.n[0]) % g.n[1]), k = (int)(v / ((int64_t)g.n[0] * g.n[1]));
      const bool in_v = F[v] < 0.f;
#pragma unroll
      for (int d = 0; d < 7; ++d) {
        const int3 e = dvec(d);
        if (i + e.x >= g.n[0] || j + e.y >= g.n[1] || k + e.z >= g.n[2]) continue;
        const int64_t u = flat_of(g, i + e.x, j + e.y, k + e.z);
        if (near[u] && ((F[u] < 0.f) != in_v)) m |= 1u << d;
      }
    }
    emask[v] = (uint8_t)m;
    cnt[v] = (uint32_t)__popc(m);
  }
}

__global__ void mt_vertex_kernel(const float* __restrict__ F, MGrid g, const uint8_t* __restrict__ emask,
                                 const uint32_t* __restrict__ vpos, double* __restrict__ out) {
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned m = emask[v];
    if (!m) continue;
    const int i = (int)(v % g.n[0]), j = (int)((v / g.n[0]) % g.n[1]), k = (int)(v / ((int64_t)g.n[0] * g.n[1]));
    const double fa = (double)F[v];
    int64_t o = vpos[v];
    for (int d = 0; d < 7; ++d) {
      if (!(m & (1u << d))) continue;
      const int3 e = dvec(d);
      const double fb = (double)F[flat_of(g, i + e.x, j + e.y, k + e.z)];
      const double t = fa / (fa - fb);
      const int q[3] = {i, j, k}, dq[3] = {e.x, e.y, e.z};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double pa = mcoord(g, a, q[a]), pb = mcoord(g, a, q[a] + dq[a]);
        out[3 * o + a] = __dadd_rn(pa, __dmul_rn(t, __dsub_rn(pb, pa)));
      }
      ++o;
    }
  }
}

struct TetCase {
  int npoly;        // 0, 1 or 2 triangles
  int e[2][3][2];   // per triangle: 3 edges as (tet corner index, tet corner index)
};

// polygon of one tetrahedron (inside bits of its 4 corners, tet order), oriented
__device__ __forceinline__ TetCase tet_case(const int* code, unsigned ins) {
  TetCase tc;
  tc.npoly = 0;
  const int nin = __popc(ins);
  if (nin == 0 || nin == 4) return tc;
  int3 q[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) q[m] = make_int3(code[m] & 1, (code[m] >> 1) & 1, (code[m] >> 2) & 1);
  // doubled lattice coordinates: centroid difference (out - in) scaled by nin * nout
  int3 sin_ = make_int3(0, 0, 0), sout = make_int3(0, 0, 0);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    if (ins & (1u << m)) { sin_.x += q[m].x; sin_.y += q[m].y; sin_.z += q[m].z; }
    else { sout.x += q[m].x; sout.y += q[m].y; sout.z += q[m].z; }
  }
  const int nout = 4 - nin;
  const int3 dir = make_int3(sout.x * nin - sin_.x * nout, sout.y * nin - sin_.y * nout, sout.z * nin - sin_.z * nout);
  if (nin == 1 || nin == 3) {
    const unsigned lone_bits = (nin == 1) ? ins : (~ins & 0xfu);
    const int a = __ffs(lone_bits) - 1;
    int o[3], c = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (m != a) o[c++] = m;
    tc.npoly = 1;
    for (int x = 0; x < 3; ++x) { tc.e[0][x][0] = a; tc.e[0][x][1] = o[x]; }
  } else {
    int in2[2], out2[2], ci = 0, co = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (ins & (1u << m)) in2[ci++] = m;
      else out2[co++] = m;
    }
    const int a = in2[0], b = in2[1], c = out2[0], d = out2[1];
    tc.npoly = 2;
    const int t0[3][2] = {{a, c}, {a, d}, {b, d}}, t1[3][2] = {{a, c}, {b, d}, {b, c}};
    for (int x = 0; x < 3; ++x) {
      tc.e[0][x][0] = t0[x][0]; tc.e[0][x][1] = t0[x][1];
      tc.e[1][x][0] = t1[x][0]; tc.e[1][x][1] = t1[x][1];
    }
  }
  for (int p = 0; p < tc.npoly; ++p) {
    int3 mid[3];
    for (int x = 0; x < 3; ++x) {
      const int3 u = q[tc.e[p][x][0]], w = q[tc.e[p][x][1]];
      mid[x] = make_int3(u.x + w.x, u.y + w.y, u.z + w.z);
    }
    const int3 e1 = make_int3(mid[1].x - mid[0].x, mid[1].y - mid[0].y, mid[1].z - mid[0].z);
    const int3 e2 = make_int3(mid[2].x - mid[0].x, mid[2].y - mid[0].y, mid[2].z - mid[0].z);
    const int nx = e1.y * e2.z - e1.z * e2.y, ny = e1.z * e2.x - e1.x * e2.z, nz = e1.x * e2.y - e1.y * e2.x;
    if (nx * dir.x + ny * dir.y + nz * dir.z < 0) {
      const int s0 = tc.e[p][1][0], s1 = tc.e[p][1][1];
      tc.e[p][1][0] = tc.e[p][2][0]; tc.e[p][1][1] = tc.e[p][2][1];
      tc.e[p][2][0] = s0; tc.e[p][2][1] = s1;
    }
  }
  return tc;
}

// inside bits of the 8 corners of cube v, or -1 when the cube is not polygonised
__device__ __forceinline__ int cube_bits(const float* __restrict__ F, const uint8_t* __restrict__ near, const MGrid& g,
                                         int64_t v, int& i, int& j, int& k) {
  i = (int)(v % g.n[0]); j = (int)((v / g.n[0]) % g.n[1]); k = (int)(v / ((int64_t)g.n[0] * g.n[1]));
  if (i + 1 >= g.n[0] || j + 1 >= g.n[1] || k + 1 >= g.n[2]) return -1;
  int bits = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int64_t u = flat_of(g, i + (c & 1), j + ((c >> 1) & 1), k + ((c >> 2) & 1));
    if (!near[u]) return -1;
    if (F[u] < 0.f) bits |= 1 << c;
  }
  return bits;
}

__global__ void mt_cube_count_kernel(const float* __restrict__ F, const uint8_t* __restrict__ near, MGrid g,
                                     uint32_t* __restrict__ cnt) {
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    int i, j, k;
    uint32_t ntri = 0;
    const int bits = near[v] ? cube_bits(F, near, g, v, i, j, k) : -1;
    if (bits > 0 && bits < 255) {
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        unsigned ins = 0;
#pragma unroll
        for (int m = 0; m < 4; ++m) ins |= ((bits >> kTet[t][m]) & 1u) << m;
        const int nin = __popc(ins);
        ntri += (nin == 0 || nin == 4) ? 0u : (nin == 2 ? 2u : 1u);
      }
    }
    cnt[v] = ntri;
  }
}

__global__ void mt_tri_kernel(const float* __restrict__ F, const uint8_t* __restrict__ near, MGrid g,
                              const uint8_t* __restrict__ emask, const uint32_t* __restrict__ vpos,
                              const uint32_t* __restrict__ tpos, int32_t* __restrict__ tris) {
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    if (tpos[v + 1] == tpos[v]) continue;
    int i, j, k;
    const int bits = cube_bits(F, near, g, v, i, j, k);
    int64_t o = tpos[v];
    for (int t = 0; t < 6; ++t) {
      int code[4];
      unsigned ins = 0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        code[m] = kTet[t][m];
        ins |= ((bits >> code[m]) & 1u) << m;
      }
      const TetCase tc = tet_case(code, ins);
      for (int p = 0; p < tc.npoly; ++p) {
        for (int x = 0; x < 3; ++x) {
          const int ca = code[tc.e[p][x][0]], cb = code[tc.e[p][x][1]];
          const int lo_c = ca < cb ? ca : cb, hi_c = ca < cb ? cb : ca;   // nested corners: lo_c subset of hi_c
          const int d = dir_of(lo_c ^ hi_c);
          const int64_t u = flat_of(g, i + (lo_c & 1), j + ((lo_c >> 1) & 1), k + ((lo_c >> 2) & 1));
          const unsigned m = emask[u];
          tris[3 * o + x] = (int32_t)(vpos[u] + (uint32_t)__popc(m & ((1u << d) - 1u)));
        }
        ++o;
      }
    }
  }
}

}  // namespace

// Mesh of the zero iso-surface of `field` on the nodes flagged in `near`.
rbf_status marching_tets(rbf_ctx* ctx, const float* field, const rbf_grid* grid, const uint8_t* near, rbf_mesh* M) {
  cudaStream_t s = ctx->stream;
  MGrid g;
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = grid->lo[a];
    g.step[a] = (grid->hi[a] - grid->lo[a]) / (double)(grid->n[a] - 1);
    g.n[a] = grid->n[a];
  }
  const int64_t nn = (int64_t)g.n[0] * g.n[1] * g.n[2];
  DevBuf emask, cnt, vpos, tpos, tot;
  RBF_TRY(emask.alloc(nn, s));
  RBF_TRY(cnt.alloc(4 * nn, s));
  RBF_TRY(vpos.alloc(4 * (nn + 1), s));
  RBF_TRY(tpos.alloc(4 * (nn + 1), s));
  RBF_TRY(tot.alloc(8, s));
  mt_edge_kernel<<<grid_for(nn, 256), 256, 0, s>>>(field, near, g, emask.as<uint8_t>(), cnt.as<uint32_t>());
  RBF_CHECK_LAUNCH();
  RBF_TRY(exclusive_scan_u32(ctx, cnt.as<uint32_t>(), vpos.as<uint32_t>(), nn, tot.as<uint32_t>()));
  mt_cube_count_kernel<<<grid_for(nn, 256), 256, 0, s>>>(field, near, g, cnt.as<uint32_t>());
  RBF_CHECK_LAUNCH();
  RBF_TRY(exclusive_scan_u32(ctx, cnt.as<uint32_t>(), tpos.as<uint32_t>(), nn, tot.as<uint32_t>() + 1));
  // tpos[nn] = total (the triangle kernel reads tpos[v + 1])
  RBF_CUDA_TRY(cudaMemcpyAsync(tpos.as<uint32_t>() + nn, tot.as<uint32_t>() + 1, 4, cudaMemcpyDeviceToDevice, s));
  uint32_t h[2];
  RBF_CUDA_TRY(cudaMemcpyAsync(h, tot.p, 8, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  if ((int64_t)h[0] > INT32_MAX) { set_error("mesh has more than 2^31 vertices"); return RBF_EINVAL; }
  M->nv = h[0];
  M->nt = h[1];
  RBF_TRY(M->verts.alloc(sizeof(double) * 3 * (size_t)std::max<int64_t>(M->nv, 1), s));
  RBF_TRY(M->tris.alloc(sizeof(int32_t) * 3 * (size_t)std::max<int64_t>(M->nt, 1), s));
  if (M->nv > 0) {
    mt_vertex_kernel<<<grid_for(nn, 256), 256, 0, s>>>(field, g, emask.as<uint8_t>(), vpos.as<uint32_t>(),
                                                        M->verts.as<double>());
    RBF_CHECK_LAUNCH();
  }
  if (M->nt > 0) {
    mt_tri_kernel<<<grid_for(nn, 256), 256, 0, s>>>(field, near, g, emask.as<uint8_t>(), vpos.as<uint32_t>(),
                                                     tpos.as<uint32_t>(), M->tris.as<int32_t>());
    RBF_CHECK_LAUNCH();
  }
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  return RBF_OK;
}

}  // namespace rbf

using namespace rbf;

namespace {
rbf_status check_mesh_args(rbf_ctx* ctx, const rbf_grid* grid, const double* data, int64_t ndata, double eps) {
  if (!ctx || !grid) { set_error("NULL argument"); return RBF_EINVAL; }
  if (ndata < 0 || (ndata > 0 && !data)) { set_error("bad data"); return RBF_EINVAL; }
  if (!(eps > 0) || !std::isfinite(eps)) { set_error("eps must be finite and > 0"); return RBF_EINVAL; }
  for (int a = 0; a < 3; ++a)
    if (grid->n[a] < 2 || !std::isfinite(grid->lo[a]) || !std::isfinite(grid->hi[a]) || !(grid->hi[a] > grid->lo[a])) {
      set_error("bad grid");
      return RBF_EINVAL;
    }
  if ((double)grid->n[0] * grid->n[1] * grid->n[2] > 2e9) { set_error("grid too large"); return RBF_EINVAL; }
  return RBF_OK;
}
}  // namespace

// api.cu: the masked evaluation (weights in caller order -> sorted, slab layers, gather)
namespace rbf {
rbf_status eval_grid_masked_impl(rbf_ctx* ctx, const rbf_cells* c, const rbf_kernel* kern, const double* w,
                                 const rbf_grid* g, const uint8_t* near, float* field);
}

extern "C" {

rbf_status rbf_eval_grid_masked(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern, const double* w,
                                const rbf_grid* grid, const double* data, int64_t ndata, double eps, float* field) {
  RBF_NVTX("rbf_eval_grid_masked");
  RBF_TRY(check_mesh_args(ctx, grid, data, ndata, eps));
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  DevBuf near;
  RBF_TRY(build_near_mask(ctx, grid, data, ndata, eps, near));
  return eval_grid_masked_impl(ctx, cells, kern, w, grid, near.as<uint8_t>(), field);
}

rbf_status rbf_mesh_from_field(rbf_ctx* ctx, const float* field, const rbf_grid* grid, const double* data,
                               int64_t ndata, double eps, rbf_mesh** out) {
  if (!out || !field) { set_error("NULL argument"); return RBF_EINVAL; }
  *out = nullptr;
  RBF_TRY(check_mesh_args(ctx, grid, data, ndata, eps));
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  DevBuf near;
  RBF_TRY(build_near_mask(ctx, grid, data, ndata, eps, near));
  rbf_mesh* M = new rbf_mesh();
  rbf_status st = marching_tets(ctx, field, grid, near.as<uint8_t>(), M);
  if (st != RBF_OK) { delete M; return st; }
  *out = M;
  return RBF_OK;
}

rbf_status rbf_isosurface(rbf_ctx* ctx, const rbf_cells* cells, const rbf_kernel* kern, const double* w,
                          const rbf_grid* grid, const double* data, int64_t ndata, double eps, float* field,
                          rbf_mesh** out) {
  RBF_NVTX("rbf_isosurface");
  if (!out) { set_error("NULL argument"); return RBF_EINVAL; }
  *out = nullptr;
  RBF_TRY(check_mesh_args(ctx, grid, data, ndata, eps));
  RBF_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const int64_t nn = (int64_t)grid->n[0] * grid->n[1] * grid->n[2];
  DevBuf near, own;
  RBF_TRY(build_near_mask(ctx, grid, data, ndata, eps, near));
  if (!field) {
    RBF_TRY(own.alloc(sizeof(float) * nn, s));
    field = own.as<float>();
  }
  RBF_TRY(eval_grid_masked_impl(ctx, cells, kern, w, grid, near.as<uint8_t>(), field));
  rbf_mesh* M = new rbf_mesh();
  rbf_status st = marching_tets(ctx, field, grid, near.as<uint8_t>(), M);
  if (st != RBF_OK) { delete M; return st; }
  *out = M;
  return RBF_OK;
}

rbf_status rbf_mesh_view(const rbf_mesh* m, const double** vertices, int64_t* nv, const int32_t** tris, int64_t* nt) {
  if (!m) { set_error("NULL mesh"); return RBF_EINVAL; }
  if (vertices) *vertices = m->verts.as<double>();
  if (nv) *nv = m->nv;
  if (tris) *tris = m->tris.as<int32_t>();
  if (nt) *nt = m->nt;
  return RBF_OK;
}

void rbf_mesh_free(rbf_mesh* m) { delete m; }

}  // extern "C"
