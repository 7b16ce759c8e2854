// Q1 hexahedral linear elasticity MG-CG (BASELINE configs[4]).
//
// There is no reference implementation (the reference's SPEC substitutes a vector Laplacian,
// SPEC.md:658, 704), so the discretisation is defined here and restated in the CPU oracle
// (oracle/tmg_elast_oracle.c, test infrastructure) with the same arithmetic order:
//   trilinear Q1 elements on N^3 vertices of the unit cube (h = 1/(N-1)), element stiffness
//   E_e h K_ref(nu) (2x2x2 Gauss), E_e = 10^(3 u(seed, e)) per element, clamped x = 0 face
//   (diagonal-only rows, couplings to clamped dofs dropped), body force (0, 0, -1), point-block
//   Jacobi Chebyshev V(m,m), rediscretised coarse levels (E_c = mean of the 8 children, 2h),
//   R = P^T and trilinear P per component, dense LU on the coarsest level; the reference's
//   solve_cg (solver.cpp:214-266), solve_fixed (solver.cpp:79-110) and estimator
//   (solver.cpp:520-581) drive it.
//
// B200 layout: each level is split into the boxes of the scalar path's GridHeader (one box per
// reference rank, boxes over processes / GPUs as the World says) in the padded layout of
// tmgx_kernels.cuh; a 3-dof vector is three consecutive component planes of that layout
// (component c at p + c * total), elements (ei, ej, ek) live at the vertex slot of their lower
// corner, each box holding its elements and the ring of the lower neighbours' elements. Box
// halos, telescope gathers / scatters and the rank-ordered dot sums reuse the scalar path's
// region plans (expanded to the three component planes: one exchange, one publishing barrier)
// and peer-mailbox transport, so the same node list (SMOOTH /
// TELESCOPE / COARSE, build_node_specs) drives the V-cycle: cfg5's 8 boxes telescoped r = 8
// at level 3 onto one box. The
// operator is matrix-free and vertex-centric: a thread gathers its row from the 8 incident
// elements (576 fused multiply-adds with K_ref in constant memory, one E h scaling per
// element); everything else reuses the
// scalar path's per-component kernels (restriction, prolongation, LU) or is pointwise.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "tmgx.h"
#include "tmgx_engine.hpp"
#include "tmgx_elast.hpp"
#include "tmgx_kernels.cuh"

#define CK(x) cuda_check((x), #x)

namespace tmgx {

namespace {

__constant__ double c_K[576];

__device__ __forceinline__ long long vx(const BoxGeo& g, int i, int j, int k) {
  return g.base + i + g.px * (long long)j + g.pxy * (long long)k;
}

// y = A x (MODE 0) or y = b - A x (MODE 1); x, y, b: three component planes of g.total.
// One thread per vertex over a flattened (i, j) index, so every warp is full (a 128-wide x tile
// left a 1-thread warp per row of the 129^3 level: a fifth of the issued instructions); neighbour
// offsets are 32-bit and constant per (element, vertex) after the unroll; the couplings to a
// clamped -x neighbour are dropped by multiplying its values by exact zeros (a row's partial sum
// is never -0, so acc + (+-0) == acc: bitwise the skipped terms) instead of a divergent branch.
template <int MODE>
__global__ void __launch_bounds__(128) k_el_apply(BoxGeo g, const double* __restrict__ E, double h,
                                                  const double* __restrict__ x, const double* __restrict__ b,
                                                  double* __restrict__ y) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x, k = blockIdx.y;
  if (idx >= g.ex * g.ey) return;
  const int j = idx / g.ex, i = idx - j * g.ex;
  const long long T = g.total;
  const int nx = g.Nx, ny = g.Ny, nz = g.Nz;
  const int px = (int)g.px, pxy = (int)g.pxy;
  const long long v = vx(g, i, j, k);
  const double* __restrict__ xv = x + v;
  const double* __restrict__ Ev = E + v;
  const bool cl = g.gx + i == 0;
  const double keep_m1 = g.gx + i - 1 == 0 ? 0.0 : 1.0;  // -x neighbour clamped: coupling dropped
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
#pragma unroll
  for (int ez = -1; ez <= 0; ++ez)
#pragma unroll
    for (int ey = -1; ey <= 0; ++ey)
#pragma unroll
      for (int ex = -1; ex <= 0; ++ex) {
        const int ei = g.gx + i + ex, ej = g.gy + j + ey, ek = g.gz + k + ez;  // global element
        if (ei < 0 || ej < 0 || ek < 0 || ei >= nx - 1 || ej >= ny - 1 || ek >= nz - 1) continue;
        const double eh = __ldg(Ev + ex + ey * px + ez * pxy) * h;
        const int l = -ex + 2 * (-ey) + 4 * (-ez);
        // element contribution: K_ref row block times the element's x, then scaled by E h
        double ea0 = 0.0, ea1 = 0.0, ea2 = 0.0;
        if (cl) {
          ea0 += c_K[(3 * l + 0) * 24 + 3 * l + 0] * __ldg(xv);
          ea1 += c_K[(3 * l + 1) * 24 + 3 * l + 1] * __ldg(xv + T);
          ea2 += c_K[(3 * l + 2) * 24 + 3 * l + 2] * __ldg(xv + 2 * T);
        } else {
#pragma unroll
          for (int lp = 0; lp < 8; ++lp) {
            const int dx = ex + (lp & 1), dy = ey + ((lp >> 1) & 1), dz = ez + (lp >> 2);
            const int o = dx + dy * px + dz * pxy;
            double x0 = __ldg(xv + o), x1 = __ldg(xv + T + o), x2 = __ldg(xv + 2 * T + o);
            if (dx == -1) {
              x0 *= keep_m1;
              x1 *= keep_m1;
              x2 *= keep_m1;
            }
            const double xb[3] = {x0, x1, x2};
#pragma unroll
            for (int bb = 0; bb < 3; ++bb) {
              ea0 += c_K[(3 * l + 0) * 24 + 3 * lp + bb] * xb[bb];
              ea1 += c_K[(3 * l + 1) * 24 + 3 * lp + bb] * xb[bb];
              ea2 += c_K[(3 * l + 2) * 24 + 3 * lp + bb] * xb[bb];
            }
          }
        }
        acc0 += eh * ea0;
        acc1 += eh * ea1;
        acc2 += eh * ea2;
      }
  if (MODE == 0) {
    y[v] = acc0;
    y[T + v] = acc1;
    y[2 * T + v] = acc2;
  } else {
    y[v] = b[v] - acc0;
    y[T + v] = b[T + v] - acc1;
    y[2 * T + v] = b[2 * T + v] - acc2;
  }
}

// inverse 3x3 diagonal blocks (9 planes): adjugate / determinant; diagonal-only when clamped
__global__ void k_el_binv(BoxGeo g, const double* __restrict__ E, double h, double* __restrict__ binv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= g.ex || j >= g.ey) return;
  const int nx = g.Nx, ny = g.Ny, nz = g.Nz;
  const bool cl = g.gx + i == 0;
  double B[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int ez = -1; ez <= 0; ++ez)
    for (int ey = -1; ey <= 0; ++ey)
      for (int ex = -1; ex <= 0; ++ex) {
        const int ei = i + ex, ej = j + ey, ek = k + ez;
        if (g.gx + ei < 0 || g.gy + ej < 0 || g.gz + ek < 0 || g.gx + ei >= nx - 1 || g.gy + ej >= ny - 1 ||
            g.gz + ek >= nz - 1)
          continue;
        const double eh = E[vx(g, ei, ej, ek)] * h;
        const int l = -ex + 2 * (-ey) + 4 * (-ez);
        for (int bb = 0; bb < 3; ++bb)
          for (int a = 0; a < 3; ++a) {
            if (cl && a != bb) continue;
            const double c = eh * c_K[(3 * l + a) * 24 + 3 * l + bb];
            B[3 * a + bb] += c;
          }
      }
  double o[9];
  if (cl) {
    for (int q = 0; q < 9; ++q) o[q] = 0.0;
    o[0] = 1.0 / B[0];
    o[4] = 1.0 / B[4];
    o[8] = 1.0 / B[8];
  } else {
    const double c00 = B[4] * B[8] - B[5] * B[7], c01 = B[5] * B[6] - B[3] * B[8], c02 = B[3] * B[7] - B[4] * B[6];
    const double det = B[0] * c00 + B[1] * c01 + B[2] * c02;
    const double id = 1.0 / det;
    o[0] = c00 * id;
    o[1] = (B[2] * B[7] - B[1] * B[8]) * id;
    o[2] = (B[1] * B[5] - B[2] * B[4]) * id;
    o[3] = c01 * id;
    o[4] = (B[0] * B[8] - B[2] * B[6]) * id;
    o[5] = (B[2] * B[3] - B[0] * B[5]) * id;
    o[6] = c02 * id;
    o[7] = (B[1] * B[6] - B[0] * B[7]) * id;
    o[8] = (B[0] * B[4] - B[1] * B[3]) * id;
  }
  const long long v = vx(g, i, j, k);
  for (int q = 0; q < 9; ++q) binv[q * g.total + v] = o[q];
}

// y = D^-1 x (point-block Jacobi)
__global__ void k_el_jacobi(BoxGeo g, const double* __restrict__ binv, const double* __restrict__ x,
                            double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= g.ex || j >= g.ey) return;
  const long long T = g.total, v = vx(g, i, j, k);
  const double x0 = x[v], x1 = x[T + v], x2 = x[2 * T + v];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double acc = 0.0;
    acc += binv[(3 * a + 0) * T + v] * x0;
    acc += binv[(3 * a + 1) * T + v] * x1;
    acc += binv[(3 * a + 2) * T + v] * x2;
    y[a * T + v] = acc;
  }
}

// pointwise over the three planes (ghost entries stay finite: zero-initialised, linear ops)
// op 0: y = x * s ; 1: y += s * x ; 2: y = s * y + t * x ; 3: y = x - y ; 4: y = x + s * y
__global__ void k_el_vec(long long n, int op, double s, double t, const double* __restrict__ x, double* __restrict__ y) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    switch (op) {
      case 0: y[q] = x[q] * s; break;
      case 1: y[q] += s * x[q]; break;
      case 2: y[q] = s * y[q] + t * x[q]; break;
      case 3: y[q] = x[q] - y[q]; break;
      default: y[q] = x[q] + s * y[q]; break;
    }
  }
}

// serial fold of a.b over the interleaved dof order (vertex natural order, then component):
// the reference's dot on one rank, for the parity build
__global__ void k_el_fold_dot(BoxGeo g, const double* __restrict__ a, const double* __restrict__ b, double* out) {
  if (threadIdx.x || blockIdx.x) return;
  const long long T = g.total;
  double acc = 0.0;
  for (int k = 0; k < g.ez; ++k)
    for (int j = 0; j < g.ey; ++j)
      for (int i = 0; i < g.ex; ++i) {
        const long long v = vx(g, i, j, k);
        for (int c = 0; c < 3; ++c) {
          const double p = a[c * T + v] * b[c * T + v];
          acc += p;
        }
      }
  *out = acc;
}

// block partials of a.b (performance build), fixed tree; then one block sums the partials
__global__ void k_el_dot_part(BoxGeo g, const double* __restrict__ a, const double* __restrict__ b, double* part) {
  __shared__ double sh[256];
  const long long T = g.total;
  const long long nv = (long long)g.ex * g.ey * g.ez;
  double acc = 0.0;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nv; q += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(q % g.ex), j = (int)((q / g.ex) % g.ey), k = (int)(q / ((long long)g.ex * g.ey));
    const long long v = vx(g, i, j, k);
    acc += a[v] * b[v] + a[T + v] * b[T + v] + a[2 * T + v] * b[2 * T + v];
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
// sum of the block partials: fixed strided order per thread, then a fixed shared-memory tree
// (deterministic; a single-thread serial loop over 1184 partials took 43 us per dot)
__global__ void __launch_bounds__(256) k_el_dot_sum(const double* __restrict__ part, int n, double* out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int q = threadIdx.x; q < n; q += 256) acc += part[q];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// global natural interleaved (3 v + c, v the level's natural vertex index) <-> the box's planes
__global__ void k_el_pack(BoxGeo g, const double* __restrict__ src, double* __restrict__ dst, int to_compact) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= g.ex || j >= g.ey) return;
  const long long v = vx(g, i, j, k),
                  n = (g.gx + i) + (long long)g.Nx * ((g.gy + j) + (long long)g.Ny * (g.gz + k));
  for (int c = 0; c < 3; ++c) {
    if (to_compact)
      dst[3 * n + c] = src[c * g.total + v];
    else
      dst[c * g.total + v] = src[3 * n + c];
  }
}

dim3 vgrid(const BoxGeo& g) { return dim3((g.ex + 127) / 128, g.ey, g.ez); }
dim3 fgrid(const BoxGeo& g) { return dim3((g.ex * g.ey + 127) / 128, g.ez); }  // flattened (i, j)

}  // namespace

// K_ref: the same arithmetic as orc_el_kref (oracle/tmg_elast_oracle.c)
void q1_kref(double nu, double* K) {
  const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double mu = 1.0 / (2.0 * (1.0 + nu));
  double D[6][6];
  std::memset(D, 0, sizeof D);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) D[a][b] = lam + (a == b ? 2.0 * mu : 0.0);
  D[3][3] = D[4][4] = D[5][5] = mu;
  std::memset(K, 0, sizeof(double) * 576);
  const double gq = 1.0 / std::sqrt(3.0);
  for (int q = 0; q < 8; ++q) {
    const double xi[3] = {(q & 1) ? gq : -gq, (q & 2) ? gq : -gq, (q & 4) ? gq : -gq};
    double dN[8][3];
    for (int l = 0; l < 8; ++l) {
      const double s[3] = {(l & 1) ? 1.0 : -1.0, (l & 2) ? 1.0 : -1.0, (l & 4) ? 1.0 : -1.0};
      const double f[3] = {1.0 + s[0] * xi[0], 1.0 + s[1] * xi[1], 1.0 + s[2] * xi[2]};
      dN[l][0] = 2.0 * (s[0] * f[1] * f[2] / 8.0);
      dN[l][1] = 2.0 * (f[0] * s[1] * f[2] / 8.0);
      dN[l][2] = 2.0 * (f[0] * f[1] * s[2] / 8.0);
    }
    double B[6][24];
    std::memset(B, 0, sizeof B);
    for (int l = 0; l < 8; ++l) {
      B[0][3 * l + 0] = dN[l][0];
      B[1][3 * l + 1] = dN[l][1];
      B[2][3 * l + 2] = dN[l][2];
      B[3][3 * l + 0] = dN[l][1];
      B[3][3 * l + 1] = dN[l][0];
      B[4][3 * l + 1] = dN[l][2];
      B[4][3 * l + 2] = dN[l][1];
      B[5][3 * l + 0] = dN[l][2];
      B[5][3 * l + 2] = dN[l][0];
    }
    double DB[6][24];
    for (int a = 0; a < 6; ++a)
      for (int j = 0; j < 24; ++j) {
        double acc = 0.0;
        for (int b = 0; b < 6; ++b) acc += D[a][b] * B[b][j];
        DB[a][j] = acc;
      }
    const double wdet = 1.0 / 8.0;
    for (int i = 0; i < 24; ++i)
      for (int j = 0; j < 24; ++j) {
        double acc = 0.0;
        for (int a = 0; a < 6; ++a) acc += B[a][i] * DB[a][j];
        K[i * 24 + j] += acc * wdet;
      }
  }
}


// ------------------------------------------------------------------------------------------
// hierarchy
// ------------------------------------------------------------------------------------------
Field ElastSolver::make3(const Dist& D) {
  Field f;
  for (const auto& g : D.geo) f.p.push_back(arena.alloc(3 * g.total));
  return f;
}
Field ElastSolver::comp(int i, const Field& f, int c) const {
  Field o;
  const Dist& D = *nodes[(size_t)i].dist;
  for (size_t q = 0; q < f.p.size(); ++q) o.p.push_back(f.p[q] + c * D.geo[q].total);
  return o;
}
void ElastSolver::sync() {
  CK(cudaStreamSynchronize(W.stream));
  W.check();
}
int ElastSolver::node_for_level(int level) const {
  int best = -1;
  for (size_t i = 0; i < nodes.size(); ++i)
    if (nodes[i].level == level) best = (int)i;
  if (best < 0) throw tmg::ConfigError("elasticity: no such level");
  return best;
}

void ElastSolver::halo(int i, const Field& f) { run_plan(W, nodes[(size_t)i].halo, f, f, false); }
void ElastSolver::apply(int i, const Field& x, const Field& y) {
  ElNode& nd = nodes[(size_t)i];
  halo(i, x);
  for (size_t q = 0; q < nd.dist->geo.size(); ++q) {
    const BoxGeo& g = nd.dist->geo[q];
    k_el_apply<0><<<fgrid(g), 128, 0, W.stream>>>(g, nd.E[q], nd.h, x.p[q], nullptr, y.p[q]);
    ++launches;
  }
}
void ElastSolver::residual(int i, const Field& b, const Field& x, const Field& r) {
  ElNode& nd = nodes[(size_t)i];
  halo(i, x);
  for (size_t q = 0; q < nd.dist->geo.size(); ++q) {
    const BoxGeo& g = nd.dist->geo[q];
    k_el_apply<1><<<fgrid(g), 128, 0, W.stream>>>(g, nd.E[q], nd.h, x.p[q], b.p[q], r.p[q]);
    ++launches;
  }
}
void ElastSolver::jacobi(int i, const Field& x, const Field& y) {
  ElNode& nd = nodes[(size_t)i];
  for (size_t q = 0; q < nd.dist->geo.size(); ++q) {
    k_el_jacobi<<<vgrid(nd.dist->geo[q]), 128, 0, W.stream>>>(nd.dist->geo[q], nd.binv[q], x.p[q], y.p[q]);
    ++launches;
  }
}
void ElastSolver::vec(int i, int op, double s, double t, const Field& x, const Field& y) {
  const Dist& D = *nodes[(size_t)i].dist;
  for (size_t q = 0; q < D.geo.size(); ++q) {
    const long long n = 3 * D.geo[q].total;
    const int blocks = (int)std::min<long long>((n + 255) / 256, 4 * 148 * 8);
    k_el_vec<<<blocks, 256, 0, W.stream>>>(n, op, s, t, x.p[q], y.p[q]);
    ++launches;
  }
}
void ElastSolver::zero(int i, const Field& f) {
  const Dist& D = *nodes[(size_t)i].dist;
  for (size_t q = 0; q < D.geo.size(); ++q)
    CK(cudaMemsetAsync(f.p[q], 0, sizeof(double) * 3 * D.geo[q].total, W.stream));
}
// a.b over the node's communicator: per box a fixed tree (performance build) or the serial fold
// in natural dof order (parity build; the reference's dot on one rank), then the rank-ordered
// sum of the box values (ordered_fold_sum, comm.cpp:338-351). One box: the box's value itself.
double ElastSolver::dot(int i, const Field& a, const Field& b) {
  const Dist& D = *nodes[(size_t)i].dist;
  for (size_t q = 0; q < D.geo.size(); ++q) {
    double* out = rank_sums + D.wr[(size_t)D.local[q]];
    if (parity_build()) {
      k_el_fold_dot<<<1, 1, 0, W.stream>>>(D.geo[q], a.p[q], b.p[q], out);
      ++launches;
    } else {
      k_el_dot_part<<<1184, 256, 0, W.stream>>>(D.geo[q], a.p[q], b.p[q], dot_part);
      k_el_dot_sum<<<1, 256, 0, W.stream>>>(dot_part, 1184, out);
      launches += 2;
    }
  }
  push_ranksums(W, rank_sums, 1, peer_mail, rs_last_bar);
  CK(cudaMemcpyAsync(host_sums, rank_sums, sizeof(double) * W.R, cudaMemcpyDeviceToHost, W.stream));
  sync();
  double s = host_sums[D.wr[0]];
  for (int r = 1; r < D.h.n_ranks(); ++r) s += host_sums[D.wr[(size_t)r]];
  return s;
}
void ElastSolver::coarse_solve(int i) {
  ElNode& nd = nodes[(size_t)i];
  if (nd.dist->local.empty()) return;
  if (parity_build())
    launches += launch_lu_solve(nd.A_dev, nd.piv_dev, nd.nc, nd.map_dev, nd.b.p[0], nd.x.p[0], W.stream);
  else
    launches += launch_dense_matvec(nd.A_dev, nd.nc, nd.map_dev, nd.b.p[0], nd.x.p[0], W.stream);
}
void ElastSolver::upload(int i, const double* src, const Field& f) {
  const ElNode& nd = nodes[(size_t)i];
  const Dist& D = *nd.dist;
  if (D.geo.empty()) return;
  CK(cudaMemcpyAsync(staging, src, sizeof(double) * nd.n_global(), cudaMemcpyDefault, W.stream));
  for (size_t q = 0; q < D.geo.size(); ++q) {
    k_el_pack<<<vgrid(D.geo[q]), 128, 0, W.stream>>>(D.geo[q], staging, f.p[q], 0);
    ++launches;
  }
}
void ElastSolver::download(int i, const Field& f, double* dst) {
  const ElNode& nd = nodes[(size_t)i];
  const Dist& D = *nd.dist;
  if (D.geo.empty()) return;
  const auto& N = D.h.npoints;
  for (size_t q = 0; q < D.geo.size(); ++q) {
    k_el_pack<<<vgrid(D.geo[q]), 128, 0, W.stream>>>(D.geo[q], f.p[q], staging, 1);
    ++launches;
  }
  if (D.h.n_ranks() == (int)D.geo.size()) {  // every box here: one linear copy
    CK(cudaMemcpyAsync(dst, staging, sizeof(double) * nd.n_global(), cudaMemcpyDefault, W.stream));
  } else {  // this process's boxes only: one pitched 3D copy per box
    for (const BoxGeo& g : D.geo) {
      cudaMemcpy3DParms pr{};
      pr.srcPtr = make_cudaPitchedPtr(staging, sizeof(double) * 3 * N[0], 3 * N[0], N[1]);
      pr.dstPtr = make_cudaPitchedPtr(dst, sizeof(double) * 3 * N[0], 3 * N[0], N[1]);
      pr.srcPos = pr.dstPos = make_cudaPos(sizeof(double) * 3 * g.gx, g.gy, g.gz);
      pr.extent = make_cudaExtent(sizeof(double) * 3 * g.ex, g.ey, g.ez);
      pr.kind = cudaMemcpyDefault;
      CK(cudaMemcpy3DAsync(&pr, W.stream));
    }
  }
  sync();
}

ElastSolver::ElastSolver(World& W_, const int64_t np[3], const MGDesc& M, uint64_t seed_e, double nu)
    : W(W_), mgd(M), m(M.m) {
  CK(cudaSetDevice(W.device));
  arena.set_stream(W.stream);
  const int nlev = mgd.nlevels;
  if (nlev < 1 || m < 1) throw tmg::ConfigError("elasticity: nlevels and smooth_its must be >= 1");
  if (mgd.galerkin) throw tmg::ConfigError("elasticity: rediscretised coarse levels only (no -pc_mg_galerkin)");
  if (!mgd.bounds.empty() && (int)mgd.bounds.size() != 2 * nlev)
    throw tmg::ConfigError("elasticity: cheb_bounds needs 2 * nlevels values");
  if (np[0] != np[1] || np[1] != np[2]) throw tmg::ConfigError("elasticity: cubic grids only (h uniform)");
  double K[576];
  q1_kref(nu, K);
  CK(cudaMemcpyToSymbolAsync(c_K, K, sizeof K, 0, cudaMemcpyHostToDevice, W.stream));
  CK(cudaStreamSynchronize(W.stream));
  ProblemDesc P;
  P.np = {np[0], np[1], np[2]};
  const std::vector<NodeSpec> specs = build_node_specs(W, P, mgd);  // ConfigError: cannot coarsen / split
  // element moduli per level on the host, global (the oracle's pow / mean sequence)
  std::vector<std::vector<double>> Eg((size_t)nlev);
  std::vector<long long> Ng((size_t)nlev);
  {
    long long n = np[0];
    for (int l = nlev - 1; l >= 0; --l) {
      Ng[(size_t)l] = n;
      if (l > 0) n = (n + 1) / 2;
    }
    for (int l = nlev - 1; l >= 0; --l) {
      const long long mx = std::max(Ng[(size_t)l] - 1, 0LL);
      std::vector<double>& Eh = Eg[(size_t)l];
      Eh.assign((size_t)(mx * mx * mx), 0.0);
      if (l == nlev - 1) {
        for (size_t e = 0; e < Eh.size(); ++e) Eh[e] = std::pow(10.0, 3.0 * hashed_uniform_h(seed_e, (uint64_t)e));
      } else {
        const auto& F = Eg[(size_t)l + 1];
        const long long fx = 2 * mx;
        for (long long K2 = 0; K2 < mx; ++K2)
          for (long long J = 0; J < mx; ++J)
            for (long long I = 0; I < mx; ++I) {
              double acc = 0.0;
              for (int c = 0; c < 8; ++c)
                acc += F[(size_t)((2 * I + (c & 1)) + fx * ((2 * J + ((c >> 1) & 1)) + fx * (2 * K2 + (c >> 2))))];
              Eh[(size_t)(I + mx * (J + mx * K2))] = 0.125 * acc;
            }
      }
    }
  }
  long long stage_n = 1;
  for (const NodeSpec& sp : specs) {
    ElNode nd;
    nd.kind = sp.kind;
    nd.level = sp.level;
    nd.dist = sp.dist;
    const Dist& D = *nd.dist;
    if (D.h.npoints[0] != Ng[(size_t)nd.level]) throw tmg::Error("elasticity: level ladder mismatch");
    nd.h = 1.0 / (double)(D.h.npoints[0] - 1);
    const long long mx = D.h.npoints[0] - 1;
    const std::vector<double>& Eh = Eg[(size_t)nd.level];
    for (const BoxGeo& g : D.geo) {
      // the box's elements plus the ring of the lower neighbours' (slot -1 on each axis)
      std::vector<double> Epad((size_t)g.total, 0.0);
      for (int k = -1; k < g.ez; ++k)
        for (int j = -1; j < g.ey; ++j)
          for (int i = -1; i < g.ex; ++i) {
            const long long ei = g.gx + i, ej = g.gy + j, ek = g.gz + k;
            if (ei < 0 || ej < 0 || ek < 0 || ei >= mx || ej >= mx || ek >= mx) continue;
            Epad[(size_t)(g.base + i + g.px * j + g.pxy * k)] = Eh[(size_t)(ei + mx * (ej + mx * ek))];
          }
      double* E = arena.alloc(g.total);
      arena.upload(E, Epad.data(), sizeof(double) * g.total);
      double* binv = arena.alloc(9 * g.total);
      k_el_binv<<<vgrid(g), 128, 0, W.stream>>>(g, E, nd.h, binv);
      nd.E.push_back(E);
      nd.binv.push_back(binv);
    }
    stage_n = std::max(stage_n, nd.n_global());
    nd.halo = upload_plan(arena, expand_components(halo_plan_host(W, D), D, D, 3));
    nodes.push_back(std::move(nd));
  }
  for (size_t i = 0; i < nodes.size(); ++i) {
    ElNode& nd = nodes[i];
    const Dist& D = *nd.dist;
    if (i == 0) {
      cr = make3(D);
      cz = make3(D);
      cp = make3(D);
      cw = make3(D);
      cx = make3(D);
      nd.b = cr;
      nd.x = cz;
    } else {
      nd.b = make3(D);
      nd.x = make3(D);
    }
    for (Field* f : {&nd.r, &nd.z, &nd.d, &nd.ad}) *f = make3(D);
    if (nd.kind == TELESCOPE) {  // TelescopePC setup: the P-hat^T / ScatterPlan data movement
      const Dist& M = *nodes[i + 1].dist;
      nd.gather = upload_plan(arena, expand_components(transfer_plan_host(W, D, M), D, M, 3));
      nd.scatter = upload_plan(arena, expand_components(transfer_plan_host(W, M, D), M, D, 3));
    }
  }
  std::vector<RegionPlan*> plans;  // creation order, identical on every process
  for (ElNode& nd : nodes) {
    plans.push_back(&nd.halo);
    if (nd.kind == TELESCOPE) {
      plans.push_back(&nd.gather);
      plans.push_back(&nd.scatter);
    }
  }
  if (W.P == 1)
    rank_sums = arena.alloc(W.R);
  else
    rank_sums = wire_plans(W, arena, plans, W.R, peer_mail);
  CK(cudaMallocHost(&host_sums, sizeof(double) * W.R));
  dot_part = arena.alloc(1184);
  staging = arena.alloc(stage_n);
  sync();
  // Chebyshev intervals: given, or estimated (SolverNode::create, solver.cpp:591-592)
  est_lanczos = mgd.est_mode == 1;
  for (size_t i = 0; i < nodes.size(); ++i) {
    ElNode& nd = nodes[i];
    if (nd.kind != SMOOTH) continue;
    if (!mgd.bounds.empty()) {
      nd.lo = mgd.bounds[(size_t)(2 * nd.level)];
      nd.hi = mgd.bounds[(size_t)(2 * nd.level + 1)];
    } else {
      auto lh = estimate((int)i);
      nd.lo = lh.first;
      nd.hi = lh.second;
    }
  }
  // coarse DenseLU on its single rank: rows from the device operator applied to unit vectors
  {
    const int ic = (int)nodes.size() - 1;
    ElNode& c = nodes[(size_t)ic];
    if (!c.dist->geo.empty()) {
      const BoxGeo& g = c.dist->geo[0];
      const int nv = g.ex * g.ey * g.ez;
      c.nc = 3 * nv;
      const int nc = c.nc;
      std::vector<double> a((size_t)nc * nc), col((size_t)nc), e((size_t)nc, 0.0);
      for (int q = 0; q < nc; ++q) {
        e[(size_t)q] = 1.0;
        upload(ic, e.data(), c.x);
        apply(ic, c.x, c.r);
        download(ic, c.r, col.data());
        for (int r = 0; r < nc; ++r) a[(size_t)r * nc + q] = col[(size_t)r];
        e[(size_t)q] = 0.0;
      }
      std::vector<long long> map((size_t)nc);
      for (int k = 0; k < g.ez; ++k)
        for (int j = 0; j < g.ey; ++j)
          for (int i = 0; i < g.ex; ++i) {
            const int v = i + g.ex * (j + g.ey * k);
            for (int cc = 0; cc < 3; ++cc)
              map[(size_t)(3 * v + cc)] = cc * g.total + g.base + i + g.px * j + g.pxy * k;
          }
      dense_lu_setup(arena, a, nc, map, &c.A_dev, &c.piv_dev, &c.map_dev);
    }
  }
  sync();
}

ElastSolver::~ElastSolver() {
  if (W.grp) {  // collective teardown: no peer may still store into our mailbox
    cudaStreamSynchronize(W.stream);
    try {
      W.grp->barrier(30.0);
    } catch (...) {
    }
    for (double* p : peer_mail)
      if (p) cudaIpcCloseMemHandle(p);
  }
  if (host_sums) cudaFreeHost(host_sums);
}

// chebyshev_bounds_estimate (solver.cpp:520-581) with point-block Jacobi; fill_random keyed by
// the natural dof index 3 v + c of the level
std::pair<double, double> ElastSolver::estimate(int i) {
  ElNode& nd = nodes[(size_t)i];
  const long long n = nd.n_global();
  std::vector<double> b0((size_t)n);
  for (long long q = 0; q < n; ++q) b0[(size_t)q] = 2.0 * hashed_uniform_h(0x5eedbeefULL, (uint64_t)q) - 1.0;
  const Field &r = nd.r, &z = nd.z, &p = nd.d, &w = nd.ad, &x = nd.x;
  upload(i, b0.data(), r);
  zero(i, x);
  jacobi(i, r, z);
  vec(i, 0, 1.0, 0.0, z, p);  // p = z
  double rz = dot(i, r, z);
  std::vector<double> alphas, betas;
  bool broke = false;
  for (int it = 0; it < 10; ++it) {
    if (rz == 0.0 || !std::isfinite(rz)) break;
    apply(i, p, w);
    const double pw = dot(i, p, w);
    if (pw <= 0.0 || !std::isfinite(pw)) {
      if (alphas.empty()) broke = true;
      break;
    }
    const double alpha = rz / pw;
    vec(i, 1, alpha, 0.0, p, x);
    vec(i, 1, -alpha, 0.0, w, r);
    jacobi(i, r, z);
    const double rz_new = dot(i, r, z);
    alphas.push_back(alpha);
    if (rz_new <= 0.0 || !std::isfinite(rz_new)) break;
    const double beta = rz_new / rz;
    betas.push_back(beta);
    rz = rz_new;
    if (est_lanczos) vec(i, 4, beta, 0.0, z, p);  // p = z + beta p
  }
  if (broke || alphas.empty()) return {0.1, 1.1};
  const int na = (int)alphas.size();
  std::vector<double> d((size_t)na), e((size_t)na);
  for (int k = 0; k < na; ++k) {
    d[(size_t)k] = 1.0 / alphas[(size_t)k];
    if (k > 0) d[(size_t)k] += betas[(size_t)k - 1] / alphas[(size_t)k - 1];
    if (k + 1 < na) e[(size_t)k] = std::sqrt(betas[(size_t)k]) / alphas[(size_t)k];
  }
  const double lam = tridiag_eig_max(d, e);
  if (!(lam > 0.0) || !std::isfinite(lam)) return {0.1, 1.1};
  return {0.1 * lam, 1.1 * lam};
}

// solve_fixed, Chebyshev branch (solver.cpp:79-110), the oracle's operation sequence
void ElastSolver::smooth(int i, const Field& b, const Field& x) {
  ElNode& nd = nodes[(size_t)i];
  const double theta = 0.5 * (nd.hi + nd.lo);
  const double delta = 0.5 * (nd.hi - nd.lo);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  residual(i, b, x, nd.r);  // r = b - A x
  jacobi(i, nd.r, nd.z);
  vec(i, 0, 1.0 / theta, 0.0, nd.z, nd.d);  // d = z * (1/theta)
  for (int it = 0; it < m; ++it) {
    vec(i, 1, 1.0, 0.0, nd.d, x);  // x += 1.0 d
    if (it + 1 == m) break;
    apply(i, nd.d, nd.ad);
    vec(i, 1, -1.0, 0.0, nd.ad, nd.r);  // r += -1.0 ad
    jacobi(i, nd.r, nd.z);
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    vec(i, 2, rho_new * rho, 2.0 * rho_new / delta, nd.z, nd.d);  // d = c1 d + c2 z
    rho = rho_new;
  }
}

// mg_apply over the node list; TELESCOPE nodes gather b onto the members (per component), run
// the members' V-cycle and scatter x back (TelescopePC::apply)
void ElastSolver::vcycle(int i) {
  ElNode& nd = nodes[(size_t)i];
  zero(i, nd.x);
  if (nd.kind == COARSE) {
    coarse_solve(i);
    return;
  }
  ElNode& cn = nodes[(size_t)i + 1];
  if (nd.kind == TELESCOPE) {
    run_plan(W, nd.gather, nd.b, cn.b, true);
    vcycle(i + 1);
    run_plan(W, nd.scatter, cn.x, nd.x, true);
    return;
  }
  const Dist& D = *nd.dist;
  smooth(i, nd.b, nd.x);
  residual(i, nd.b, nd.x, nd.r);
  halo(i, nd.r);
  for (size_t q = 0; q < D.geo.size(); ++q)  // R = P^T per component (finite-element scaling)
    for (int c = 0; c < 3; ++c)
      launches += launch_restrict_scaled(D.geo[q], cn.dist->geo[q], nd.r.p[q] + c * D.geo[q].total,
                                         cn.b.p[q] + c * cn.dist->geo[q].total, 1.0, W.stream);
  vcycle(i + 1);
  halo(i + 1, cn.x);
  for (size_t q = 0; q < D.geo.size(); ++q)
    for (int c = 0; c < 3; ++c)
      launches += launch_prolong_add(D.geo[q], cn.dist->geo[q], cn.x.p[q] + c * cn.dist->geo[q].total,
                                     nd.x.p[q] + c * D.geo[q].total, W.stream);
  smooth(i, nd.b, nd.x);
}

int ElastSolver::solve(const double* b, double* x, double rtol, double atol, int max_its, bool x0_nonzero,
                       double* hist, int* reason, int* its, double* n0, double* nf, double* t_ms) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  {  // stream contract (tmgx.h): order after the caller's legacy-default-stream work on b / x
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, cudaStreamLegacy));
    CK(cudaStreamWaitEvent(W.stream, ev, 0));
    CK(cudaEventDestroy(ev));
  }
  CK(cudaEventRecord(e0, W.stream));
  upload(0, b, cw);  // b -> cw
  if (x && x0_nonzero)
    upload(0, x, cx);
  else
    zero(0, cx);
  residual(0, cw, cx, cr);
  vcycle(0);  // cr -> cz
  double nrm = std::sqrt(dot(0, cz, cz));
  *n0 = *nf = nrm;
  if (hist) hist[0] = nrm;
  *its = 0;
  *reason = 2;
  int rc = 0;
  const double tol = std::max(rtol * nrm, atol);
  if (nrm <= tol) {
    *reason = nrm <= atol ? 1 : 0;
  } else {
    vec(0, 0, 1.0, 0.0, cz, cp);
    double rz = dot(0, cr, cz);
    for (int it = 1; it <= max_its; ++it) {
      apply(0, cp, cw);
      const double pw = dot(0, cp, cw);
      if (pw <= 0.0 || !std::isfinite(pw)) {
        *reason = 4;
        rc = 2;
        break;
      }
      const double alpha = rz / pw;
      vec(0, 1, alpha, 0.0, cp, cx);
      vec(0, 1, -alpha, 0.0, cw, cr);
      vcycle(0);
      const double rz_new = dot(0, cr, cz);
      nrm = std::sqrt(dot(0, cz, cz));
      *its = it;
      *nf = nrm;
      if (hist) hist[it] = nrm;
      if (nrm <= tol) {
        *reason = nrm <= atol ? 1 : 0;
        break;
      }
      if (rz == 0.0 || !std::isfinite(rz_new)) {
        *reason = 4;
        rc = 2;
        break;
      }
      const double beta = rz_new / rz;
      rz = rz_new;
      vec(0, 4, beta, 0.0, cz, cp);  // p = z + beta p
    }
  }
  if (x) download(0, cx, x);
  CK(cudaEventRecord(e1, W.stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *t_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return rc;
}

}  // namespace tmgx
