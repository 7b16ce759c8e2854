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
// B200 layout: each level is one box (single GPU) in the padded layout of tmgx_kernels.cuh;
// a 3-dof vector is three consecutive component planes of that layout (component c at
// p + c * total), elements (ei, ej, ek) live at the vertex slot of their lower corner. The
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
        const int ei = i + ex, ej = j + ey, ek = k + ez;
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
        if (ei < 0 || ej < 0 || ek < 0 || ei >= nx - 1 || ej >= ny - 1 || ek >= nz - 1) continue;
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

// natural interleaved (3 v + c) <-> component planes
__global__ void k_el_pack(BoxGeo g, const double* __restrict__ src, double* __restrict__ dst, int to_compact) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
  if (i >= g.ex || j >= g.ey) return;
  const long long v = vx(g, i, j, k), n = i + (long long)g.ex * (j + (long long)g.ey * k);
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
void ElastSolver::apply(int l, const double* x, double* y) {
  k_el_apply<0><<<fgrid(L[l].g), 128, 0, W.stream>>>(L[l].g, L[l].E, L[l].h, x, nullptr, y);
  ++launches;
}
void ElastSolver::residual(int l, const double* b, const double* x, double* r) {
  k_el_apply<1><<<fgrid(L[l].g), 128, 0, W.stream>>>(L[l].g, L[l].E, L[l].h, x, b, r);
  ++launches;
}
void ElastSolver::jacobi(int l, const double* x, double* y) {
  k_el_jacobi<<<vgrid(L[l].g), 128, 0, W.stream>>>(L[l].g, L[l].binv, x, y);
  ++launches;
}
void ElastSolver::vec(int l, int op, double s, double t, const double* x, double* y) {
  const long long n = L[l].n3();
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4 * 148 * 8);
  k_el_vec<<<blocks, 256, 0, W.stream>>>(n, op, s, t, x, y);
  ++launches;
}
double ElastSolver::dot(int l, const double* a, const double* b) {
  if (parity_build()) {
    k_el_fold_dot<<<1, 1, 0, W.stream>>>(L[l].g, a, b, dot_out);
    ++launches;
  } else {
    k_el_dot_part<<<1184, 256, 0, W.stream>>>(L[l].g, a, b, dot_part);
    k_el_dot_sum<<<1, 256, 0, W.stream>>>(dot_part, 1184, dot_out);
    launches += 2;
  }
  double h = 0.0;
  CK(cudaMemcpyAsync(&h, dot_out, sizeof(double), cudaMemcpyDeviceToHost, W.stream));
  CK(cudaStreamSynchronize(W.stream));
  return h;
}
void ElastSolver::coarse_solve(const double* b, double* x) {
  if (parity_build())
    launches += launch_lu_solve(A_dev, piv_dev, nc, map_dev, b, x, W.stream);
  else
    launches += launch_dense_matvec(A_dev, nc, map_dev, b, x, W.stream);
}
void ElastSolver::upload(int l, const double* host, double* dev) {
  const long long n = 3LL * L[l].g.ex * L[l].g.ey * L[l].g.ez;
  CK(cudaMemcpyAsync(staging, host, sizeof(double) * n, cudaMemcpyDefault, W.stream));
  k_el_pack<<<vgrid(L[l].g), 128, 0, W.stream>>>(L[l].g, staging, dev, 0);
  ++launches;
}
void ElastSolver::download(int l, const double* dev, double* host) {
  const long long n = 3LL * L[l].g.ex * L[l].g.ey * L[l].g.ez;
  k_el_pack<<<vgrid(L[l].g), 128, 0, W.stream>>>(L[l].g, dev, staging, 1);
  ++launches;
  CK(cudaMemcpyAsync(host, staging, sizeof(double) * n, cudaMemcpyDefault, W.stream));
  CK(cudaStreamSynchronize(W.stream));
}

ElastSolver::ElastSolver(World& W_, const int64_t np[3], int nlevels, int m_, int est_mode, uint64_t seed_e, double nu)
    : W(W_), m(m_) {
  CK(cudaSetDevice(W.device));
  arena.set_stream(W.stream);
  if (W.R != 1 || W.P != 1)
    throw tmg::ConfigError("elasticity path: one box on one GPU (box split + telescope not implemented)");
  if (nlevels < 1 || m < 1) throw tmg::ConfigError("elasticity: nlevels and smooth_its must be >= 1");
  double K[576];
  q1_kref(nu, K);
  CK(cudaMemcpyToSymbolAsync(c_K, K, sizeof K, 0, cudaMemcpyHostToDevice, W.stream));
  CK(cudaStreamSynchronize(W.stream));
  // level ladder (coarsest first)
  std::vector<std::array<int64_t, 3>> dims(nlevels);
  std::array<int64_t, 3> n = {np[0], np[1], np[2]};
  if (n[0] != n[1] || n[1] != n[2]) throw tmg::ConfigError("elasticity: cubic grids only (h uniform)");
  for (int l = nlevels - 1; l >= 0; --l) {
    dims[l] = n;
    if (l > 0) {
      for (int a = 0; a < 3; ++a) {
        if (n[a] < 3 || n[a] % 2 == 0) throw tmg::ConfigError("elasticity: cannot coarsen (need 2M+1 vertices)");
        n[a] = (n[a] + 1) / 2;
      }
    }
  }
  L.resize(nlevels);
  double h = 1.0 / (double)(np[0] - 1);
  std::vector<std::vector<double>> Ehost(nlevels);
  for (int l = nlevels - 1; l >= 0; --l, h *= 2.0) {
    ElLevel& lv = L[l];
    BoxGeo g{};
    g.ex = (int)dims[l][0];
    g.ey = (int)dims[l][1];
    g.ez = (int)dims[l][2];
    g.gx = g.gy = g.gz = 0;
    g.Nx = g.ex;
    g.Ny = g.ey;
    g.Nz = g.ez;
    g.zc = choose_zc(g.ex, g.ey, g.ez);
    g.px = ((kXO + g.ex + 1) + 3) / 4 * 4;
    g.pxy = g.px * (g.ey + 2);
    g.base = kXO + g.px + g.pxy;
    g.total = g.pxy * (g.ez + 2) + 8;
    lv.g = g;
    lv.h = h;
    // element moduli on the host (the oracle's pow / mean sequence), padded upload
    const int mx = g.ex - 1, my = g.ey - 1, mz = g.ez - 1;
    std::vector<double>& Eh = Ehost[l];
    Eh.assign((size_t)std::max(mx, 0) * std::max(my, 0) * std::max(mz, 0), 0.0);
    if (l == nlevels - 1) {
      for (size_t e = 0; e < Eh.size(); ++e) Eh[e] = std::pow(10.0, 3.0 * hashed_uniform_h(seed_e, (uint64_t)e));
    } else {
      const auto& F = Ehost[l + 1];
      const int fx = 2 * mx, fy = 2 * my;
      for (int K2 = 0; K2 < mz; ++K2)
        for (int J = 0; J < my; ++J)
          for (int I = 0; I < mx; ++I) {
            double acc = 0.0;
            for (int c = 0; c < 8; ++c)
              acc += F[(size_t)(2 * I + (c & 1)) + (size_t)fx * ((2 * J + ((c >> 1) & 1)) + (size_t)fy * (2 * K2 + (c >> 2)))];
            Eh[(size_t)I + (size_t)mx * (J + (size_t)my * K2)] = 0.125 * acc;
          }
    }
    std::vector<double> Epad((size_t)g.total, 0.0);
    for (int k = 0; k < mz; ++k)
      for (int j = 0; j < my; ++j)
        for (int i = 0; i < mx; ++i)
          Epad[(size_t)(g.base + i + g.px * j + g.pxy * k)] = Eh[(size_t)i + (size_t)mx * (j + (size_t)my * k)];
    lv.E = arena.alloc(g.total);
    arena.upload(lv.E, Epad.data(), sizeof(double) * g.total);
    lv.binv = arena.alloc(9 * g.total);
    k_el_binv<<<vgrid(g), 128, 0, W.stream>>>(g, lv.E, lv.h, lv.binv);
    for (double** f : {&lv.b, &lv.x, &lv.r, &lv.z, &lv.d, &lv.ad}) *f = arena.alloc(3 * g.total);
  }
  const BoxGeo& gt = L.back().g;
  for (double** f : {&cr, &cz, &cp, &cw, &cx}) *f = arena.alloc(3 * gt.total);
  dot_part = arena.alloc(1184);
  dot_out = arena.alloc(1);
  staging = arena.alloc(3 * gt.total);
  CK(cudaStreamSynchronize(W.stream));
  // Chebyshev intervals (SolverNode::create, solver.cpp:591-592)
  est_lanczos = est_mode == 1;
  for (int l = 1; l < nlevels; ++l) {
    auto lh = estimate(l);
    L[l].lo = lh.first;
    L[l].hi = lh.second;
  }
  // coarse DenseLU: rows from the device operator applied to unit vectors (identical values)
  {
    const ElLevel& c = L[0];
    const int nv = c.g.ex * c.g.ey * c.g.ez;
    nc = 3 * nv;
    std::vector<double> a((size_t)nc * nc), col((size_t)nc), e((size_t)nc, 0.0);
    for (int q = 0; q < nc; ++q) {
      e[(size_t)q] = 1.0;
      upload(0, e.data(), c.x);
      apply(0, c.x, c.r);
      download(0, c.r, col.data());
      for (int r = 0; r < nc; ++r) a[(size_t)r * nc + q] = col[(size_t)r];
      e[(size_t)q] = 0.0;
    }
    std::vector<long long> map((size_t)nc);
    for (int k = 0; k < c.g.ez; ++k)
      for (int j = 0; j < c.g.ey; ++j)
        for (int i = 0; i < c.g.ex; ++i) {
          const int v = i + c.g.ex * (j + c.g.ey * k);
          for (int comp = 0; comp < 3; ++comp)
            map[(size_t)(3 * v + comp)] = comp * c.g.total + c.g.base + i + c.g.px * j + c.g.pxy * k;
        }
    dense_lu_setup(arena, a, nc, map, &A_dev, &piv_dev, &map_dev);
  }
}

// chebyshev_bounds_estimate (solver.cpp:520-581) with point-block Jacobi; fill_random keyed by
// the natural dof index 3 v + c
std::pair<double, double> ElastSolver::estimate(int l) {
  ElLevel& lv = L[l];
  const BoxGeo& g = lv.g;
  const long long nd = 3LL * g.ex * g.ey * g.ez;
  std::vector<double> b0((size_t)nd);
  for (long long q = 0; q < nd; ++q) b0[(size_t)q] = 2.0 * hashed_uniform_h(0x5eedbeefULL, (uint64_t)q) - 1.0;
  double *r = lv.r, *z = lv.z, *p = lv.d, *w = lv.ad, *x = lv.x;
  upload(l, b0.data(), r);
  vec(l, 0, 0.0, 0.0, r, x);  // x = 0
  jacobi(l, r, z);
  vec(l, 0, 1.0, 0.0, z, p);  // p = z
  double rz = dot(l, r, z);
  std::vector<double> alphas, betas;
  bool broke = false;
  for (int it = 0; it < 10; ++it) {
    if (rz == 0.0 || !std::isfinite(rz)) break;
    apply(l, p, w);
    const double pw = dot(l, p, w);
    if (pw <= 0.0 || !std::isfinite(pw)) {
      if (alphas.empty()) broke = true;
      break;
    }
    const double alpha = rz / pw;
    vec(l, 1, alpha, 0.0, p, x);
    vec(l, 1, -alpha, 0.0, w, r);
    jacobi(l, r, z);
    const double rz_new = dot(l, r, z);
    alphas.push_back(alpha);
    if (rz_new <= 0.0 || !std::isfinite(rz_new)) break;
    const double beta = rz_new / rz;
    betas.push_back(beta);
    rz = rz_new;
    if (est_lanczos) vec(l, 4, beta, 0.0, z, p);  // p = z + beta p
  }
  if (broke || alphas.empty()) return {0.1, 1.1};
  const int na = (int)alphas.size();
  std::vector<double> d((size_t)na), e((size_t)na);
  for (int i = 0; i < na; ++i) {
    d[(size_t)i] = 1.0 / alphas[(size_t)i];
    if (i > 0) d[(size_t)i] += betas[(size_t)i - 1] / alphas[(size_t)i - 1];
    if (i + 1 < na) e[(size_t)i] = std::sqrt(betas[(size_t)i]) / alphas[(size_t)i];
  }
  const double lam = tridiag_eig_max(d, e);
  if (!(lam > 0.0) || !std::isfinite(lam)) return {0.1, 1.1};
  return {0.1 * lam, 1.1 * lam};
}

// solve_fixed, Chebyshev branch (solver.cpp:79-110), the oracle's operation sequence
void ElastSolver::smooth(int l, const double* b, double* x) {
  ElLevel& lv = L[l];
  const double theta = 0.5 * (lv.hi + lv.lo);
  const double delta = 0.5 * (lv.hi - lv.lo);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  residual(l, b, x, lv.r);  // r = b - A x
  jacobi(l, lv.r, lv.z);
  vec(l, 0, 1.0 / theta, 0.0, lv.z, lv.d);  // d = z * (1/theta)
  for (int it = 0; it < m; ++it) {
    vec(l, 1, 1.0, 0.0, lv.d, x);  // x += 1.0 d
    if (it + 1 == m) break;
    apply(l, lv.d, lv.ad);
    vec(l, 1, -1.0, 0.0, lv.ad, lv.r);  // r += -1.0 ad
    jacobi(l, lv.r, lv.z);
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    vec(l, 2, rho_new * rho, 2.0 * rho_new / delta, lv.z, lv.d);  // d = c1 d + c2 z
    rho = rho_new;
  }
}

void ElastSolver::vcycle(int l, const double* b, double* x) {
  ElLevel& lv = L[l];
  CK(cudaMemsetAsync(x, 0, sizeof(double) * lv.n3(), W.stream));
  if (l == 0) {
    coarse_solve(b, x);
    return;
  }
  ElLevel& c = L[l - 1];
  smooth(l, b, x);
  residual(l, b, x, lv.r);
  for (int comp = 0; comp < 3; ++comp)  // R = P^T per component (finite-element scaling)
    launches += launch_restrict_scaled(lv.g, c.g, lv.r + comp * lv.g.total, c.b + comp * c.g.total, 1.0, W.stream);
  vcycle(l - 1, c.b, c.x);
  for (int comp = 0; comp < 3; ++comp)
    launches += launch_prolong_add(lv.g, c.g, c.x + comp * c.g.total, x + comp * lv.g.total, W.stream);
  smooth(l, b, x);
}

int ElastSolver::solve(const double* b, double* x, double rtol, double atol, int max_its, bool x0_nonzero,
                       double* hist, int* reason, int* its, double* n0, double* nf, double* t_ms) {
  const int top = (int)L.size() - 1;
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
  upload(top, b, cw);  // b -> cw
  if (x && x0_nonzero)
    upload(top, x, cx);
  else
    CK(cudaMemsetAsync(cx, 0, sizeof(double) * L[top].n3(), W.stream));
  residual(top, cw, cx, cr);
  vcycle(top, cr, cz);
  double nrm = std::sqrt(dot(top, cz, cz));
  *n0 = *nf = nrm;
  if (hist) hist[0] = nrm;
  *its = 0;
  *reason = 2;
  int rc = 0;
  const double tol = std::max(rtol * nrm, atol);
  if (nrm <= tol) {
    *reason = nrm <= atol ? 1 : 0;
  } else {
    vec(top, 0, 1.0, 0.0, cz, cp);
    double rz = dot(top, cr, cz);
    for (int it = 1; it <= max_its; ++it) {
      apply(top, cp, cw);
      const double pw = dot(top, cp, cw);
      if (pw <= 0.0 || !std::isfinite(pw)) {
        *reason = 4;
        rc = 2;
        break;
      }
      const double alpha = rz / pw;
      vec(top, 1, alpha, 0.0, cp, cx);
      vec(top, 1, -alpha, 0.0, cw, cr);
      vcycle(top, cr, cz);
      const double rz_new = dot(top, cr, cz);
      nrm = std::sqrt(dot(top, cz, cz));
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
      vec(top, 4, beta, 0.0, cz, cp);  // p = z + beta p
    }
  }
  if (x) download(top, cx, x);
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
