// Microbenchmark of kernel structures for the fine-level Chebyshev pass (constant-coefficient
// 7-point, fp64): read d (stencil), r, x ; write x  (32 algorithmic bytes per point).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stencil_mb stencil_mb.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

struct G {
  int ex, ey, ez, N;
  long long px, pxy, base;
};

__device__ __forceinline__ double row(const G& g, int gi, int gj, int gk, double c, double zm, double ym, double xm,
                                      double xp, double yp, double zp, double dg, double a) {
  const bool bnd = gi == 0 || gj == 0 || gk == 0 || gi == g.N - 1 || gj == g.N - 1 || gk == g.N - 1;
  double acc = 0.0;
  if (bnd) return dg * c;
  if (gk >= 2) acc += a * zm;
  if (gj >= 2) acc += a * ym;
  if (gi >= 2) acc += a * xm;
  acc += dg * c;
  if (gi <= g.N - 3) acc += a * xp;
  if (gj <= g.N - 3) acc += a * yp;
  if (gk <= g.N - 3) acc += a * zp;
  return acc;
}

// A: 2D tile (BX x BY), z-march ZC planes, neighbours via __ldg
template <int BX, int BY, int ZC, int UNR>
__global__ void __launch_bounds__(BX* BY) kA(G g, const double* __restrict__ d, const double* __restrict__ r,
                                             double* __restrict__ x, double c1, double c2, double dg, double a,
                                             double invd) {
  const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y;
  if (i >= g.ex || j >= g.ey) return;
  const int k0 = blockIdx.z * ZC, k1 = min(k0 + ZC, g.ez);
  long long v = g.base + i + g.px * j + g.pxy * k0;
  double um = __ldg(d + v - g.pxy), uc = __ldg(d + v);
#pragma unroll UNR
  for (int k = k0; k < k1; ++k, v += g.pxy) {
    const double un = __ldg(d + v + g.pxy);
    const double ax = row(g, i, j, k, uc, um, __ldg(d + v - g.px), __ldg(d + v - 1), __ldg(d + v + 1),
                          __ldg(d + v + g.px), un, dg, a);
    const double r1 = r[v] - ax;
    const double dn = c1 * uc + c2 * (r1 * invd);
    x[v] = (x[v] + uc) + dn;
    um = uc;
    uc = un;
  }
}

// D: one point per thread, flat over the box (no z reuse in registers)
__global__ void __launch_bounds__(256) kD(G g, const double* __restrict__ d, const double* __restrict__ r,
                                          double* __restrict__ x, double c1, double c2, double dg, double a,
                                          double invd) {
  const long long t = blockIdx.x * 256LL + threadIdx.x;
  const long long nxy = (long long)g.ex * g.ey;
  if (t >= nxy * g.ez) return;
  const int k = (int)(t / nxy);
  const int rem = (int)(t - (long long)k * nxy);
  const int j = rem / g.ex, i = rem - j * g.ex;
  const long long v = g.base + i + g.px * j + g.pxy * k;
  const double uc = __ldg(d + v);
  const double ax = row(g, i, j, k, uc, __ldg(d + v - g.pxy), __ldg(d + v - g.px), __ldg(d + v - 1),
                        __ldg(d + v + 1), __ldg(d + v + g.px), __ldg(d + v + g.pxy), dg, a);
  const double r1 = r[v] - ax;
  const double dn = c1 * uc + c2 * (r1 * invd);
  x[v] = (x[v] + uc) + dn;
}

// F: flattened xy plane per block (256 threads cover 256 consecutive (i,j)), z-march ZC
template <int ZC>
__global__ void __launch_bounds__(256) kF(G g, const double* __restrict__ d, const double* __restrict__ r,
                                          double* __restrict__ x, double c1, double c2, double dg, double a,
                                          double invd) {
  const int t = blockIdx.x * 256 + threadIdx.x;
  if (t >= g.ex * g.ey) return;
  const int j = t / g.ex, i = t - j * g.ex;
  const int k0 = blockIdx.y * ZC, k1 = min(k0 + ZC, g.ez);
  long long v = g.base + i + g.px * j + g.pxy * k0;
  double um = __ldg(d + v - g.pxy), uc = __ldg(d + v);
#pragma unroll 2
  for (int k = k0; k < k1; ++k, v += g.pxy) {
    const double un = __ldg(d + v + g.pxy);
    const double ax = row(g, i, j, k, uc, um, __ldg(d + v - g.px), __ldg(d + v - 1), __ldg(d + v + 1),
                          __ldg(d + v + g.px), un, dg, a);
    const double r1 = r[v] - ax;
    const double dn = c1 * uc + c2 * (r1 * invd);
    x[v] = (x[v] + uc) + dn;
    um = uc;
    uc = un;
  }
}

// S: shared-memory plane tile (BX+2)x(BY+2) per z step, register queue for z neighbours
template <int BX, int BY, int ZC>
__global__ void __launch_bounds__(BX* BY) kS(G g, const double* __restrict__ d, const double* __restrict__ r,
                                             double* __restrict__ x, double c1, double c2, double dg, double a,
                                             double invd) {
  __shared__ double sh[BY + 2][BX + 2];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i = blockIdx.x * BX + tx, j = blockIdx.y * BY + ty;
  const bool act = i < g.ex && j < g.ey;
  const int k0 = blockIdx.z * ZC, k1 = min(k0 + ZC, g.ez);
  long long v = g.base + i + g.px * j + g.pxy * k0;
  double um = 0, uc = 0;
  if (act) {
    um = __ldg(d + v - g.pxy);
    uc = __ldg(d + v);
  }
  for (int k = k0; k < k1; ++k, v += g.pxy) {
    double un = 0;
    if (act) un = __ldg(d + v + g.pxy);
    __syncthreads();
    if (act) {
      sh[ty + 1][tx + 1] = uc;
      if (tx == 0) sh[ty + 1][0] = __ldg(d + v - 1);
      if (tx == BX - 1 || i == g.ex - 1) sh[ty + 1][tx + 2] = __ldg(d + v + 1);
      if (ty == 0) sh[0][tx + 1] = __ldg(d + v - g.px);
      if (ty == BY - 1 || j == g.ey - 1) sh[ty + 2][tx + 1] = __ldg(d + v + g.px);
    }
    __syncthreads();
    if (act) {
      const double ax = row(g, i, j, k, uc, um, sh[ty][tx + 1], sh[ty + 1][tx], sh[ty + 1][tx + 2], sh[ty + 2][tx + 1],
                            un, dg, a);
      const double r1 = r[v] - ax;
      const double dn = c1 * uc + c2 * (r1 * invd);
      x[v] = (x[v] + uc) + dn;
    }
    um = uc;
    uc = un;
  }
}

// P: like A but with an explicit one-plane software prefetch of the streamed operands
template <int BX, int BY, int ZC>
__global__ void __launch_bounds__(BX* BY) kP(G g, const double* __restrict__ d, const double* __restrict__ r,
                                             double* __restrict__ x, double c1, double c2, double dg, double a,
                                             double invd) {
  const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y;
  if (i >= g.ex || j >= g.ey) return;
  const int k0 = blockIdx.z * ZC, k1 = min(k0 + ZC, g.ez);
  long long v = g.base + i + g.px * j + g.pxy * k0;
  double um = __ldg(d + v - g.pxy), uc = __ldg(d + v), un = __ldg(d + v + g.pxy);
  double rc = __ldg(r + v), xc = x[v];
  for (int k = k0; k < k1; ++k, v += g.pxy) {
    double unn = 0, rn = 0, xn = 0;
    if (k + 1 < k1) {
      unn = __ldg(d + v + 2 * g.pxy);
      rn = __ldg(r + v + g.pxy);
      xn = x[v + g.pxy];
    }
    const double ax = row(g, i, j, k, uc, um, __ldg(d + v - g.px), __ldg(d + v - 1), __ldg(d + v + 1),
                          __ldg(d + v + g.px), un, dg, a);
    const double r1 = rc - ax;
    const double dn = c1 * uc + c2 * (r1 * invd);
    x[v] = (xc + uc) + dn;
    um = uc;
    uc = un;
    un = unn;
    rc = rn;
    xc = xn;
  }
}

// V: two x-points per thread with 16-byte loads (pairs (2t, 2t+1) are 16-byte aligned)
template <int BX, int BY, int ZC>
__global__ void __launch_bounds__(BX* BY) kV(G g, const double* __restrict__ d, const double* __restrict__ r,
                                             double* __restrict__ x, double c1, double c2, double dg, double a,
                                             double invd) {
  const int i0 = 2 * (blockIdx.x * BX + threadIdx.x), j = blockIdx.y * BY + threadIdx.y;
  if (i0 >= g.ex || j >= g.ey) return;
  const bool two = i0 + 1 < g.ex;
  const int k0 = blockIdx.z * ZC, k1 = min(k0 + ZC, g.ez);
  long long v = g.base + i0 + g.px * j + g.pxy * k0;
  auto ld2 = [](const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); };
  double2 um = ld2(d + v - g.pxy), uc = ld2(d + v);
  for (int k = k0; k < k1; ++k, v += g.pxy) {
    const double2 un = ld2(d + v + g.pxy);
    const double2 ym = ld2(d + v - g.px), yp = ld2(d + v + g.px);
    const double xl = __ldg(d + v - 1), xr = __ldg(d + v + 2);
    const double2 rr = ld2(r + v);
    double2 xx = *reinterpret_cast<const double2*>(x + v);
    const double a0 = row(g, i0, j, k, uc.x, um.x, ym.x, xl, uc.y, yp.x, un.x, dg, a);
    const double r0 = rr.x - a0;
    xx.x = (xx.x + uc.x) + (c1 * uc.x + c2 * (r0 * invd));
    if (two) {
      const double a1 = row(g, i0 + 1, j, k, uc.y, um.y, ym.y, uc.x, xr, yp.y, un.y, dg, a);
      const double r1 = rr.y - a1;
      xx.y = (xx.y + uc.y) + (c1 * uc.y + c2 * (r1 * invd));
      *reinterpret_cast<double2*>(x + v) = xx;
    } else {
      x[v] = xx.x;
    }
    um = uc;
    uc = un;
  }
}

// C: pure copy-ish streaming reference: x = x + d + r (reads 3, writes 1 = 32 B/pt)
__global__ void kC(G g, const double* __restrict__ d, const double* __restrict__ r, double* __restrict__ x,
                   long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    x[t] = x[t] + d[t] + r[t];
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 257;
  G g;
  g.ex = g.ey = g.ez = g.N = N;
  g.px = ((4 + N + 1) + 3) / 4 * 4;
  g.pxy = g.px * (N + 2);
  g.base = 4 + g.px + g.pxy;
  const long long total = g.pxy * (N + 2) + 8;
  double *d, *r, *x, *flush;
  CK(cudaMalloc(&d, total * 8));
  CK(cudaMalloc(&r, total * 8));
  CK(cudaMalloc(&x, total * 8));
  CK(cudaMalloc(&flush, 512ll << 20));
  CK(cudaMemset(d, 0, total * 8));
  CK(cudaMemset(r, 0, total * 8));
  CK(cudaMemset(x, 0, total * 8));
  const double pts = (double)N * N * N;
  const double bytes = 32.0 * pts;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    float tot = 0;
    const int iters = 30;
    for (int it = 0; it < iters; ++it) {
      CK(cudaMemsetAsync(flush, it, 512ll << 20));  // evict L2 between launches
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    CK(cudaGetLastError());
    const double ms = tot / iters;
    printf("%-28s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  };
  const double c1 = 0.5, c2 = 0.25, dg = 6.0, a = -1.0, invd = 1.0 / 6.0;
#define RUN_A(BX, BY, ZC, UNR)                                                                               \
  timeit("A " #BX "x" #BY " zc" #ZC " u" #UNR, [&] {                                                         \
    kA<BX, BY, ZC, UNR><<<dim3((N + BX - 1) / BX, (N + BY - 1) / BY, (N + ZC - 1) / ZC), dim3(BX, BY)>>>(     \
        g, d, r, x, c1, c2, dg, a, invd);                                                                    \
  })
  RUN_A(32, 4, 16, 1);
  RUN_A(32, 4, 16, 4);
  RUN_A(32, 4, 8, 1);
  RUN_A(32, 4, 32, 1);
  RUN_A(32, 8, 16, 1);
  RUN_A(64, 4, 16, 1);
  RUN_A(64, 2, 16, 1);
  RUN_A(128, 1, 16, 1);
  RUN_A(32, 2, 16, 1);
  RUN_A(32, 16, 16, 1);
  RUN_A(64, 4, 8, 2);
  timeit("D flat 1pt/thread", [&] { kD<<<(unsigned)((pts + 255) / 256), 256>>>(g, d, r, x, c1, c2, dg, a, invd); });
#define RUN_F(ZC)                                                                                             \
  timeit("F flat-xy zc" #ZC, [&] {                                                                            \
    kF<ZC><<<dim3((N * N + 255) / 256, (N + ZC - 1) / ZC), 256>>>(g, d, r, x, c1, c2, dg, a, invd);           \
  })
  RUN_F(4);
  RUN_F(8);
  RUN_F(16);
  RUN_F(32);
#define RUN_S(BX, BY, ZC)                                                                                    \
  timeit("S smem " #BX "x" #BY " zc" #ZC, [&] {                                                              \
    kS<BX, BY, ZC><<<dim3((N + BX - 1) / BX, (N + BY - 1) / BY, (N + ZC - 1) / ZC), dim3(BX, BY)>>>(          \
        g, d, r, x, c1, c2, dg, a, invd);                                                                    \
  })
  RUN_S(32, 4, 16);
  RUN_S(32, 8, 16);
  RUN_S(64, 4, 32);
#define RUN_P(BX, BY, ZC)                                                                                    \
  timeit("P prefetch " #BX "x" #BY " zc" #ZC, [&] {                                                          \
    kP<BX, BY, ZC><<<dim3((N + BX - 1) / BX, (N + BY - 1) / BY, (N + ZC - 1) / ZC), dim3(BX, BY)>>>(          \
        g, d, r, x, c1, c2, dg, a, invd);                                                                    \
  })
  RUN_P(32, 4, 8);
  RUN_P(32, 4, 16);
  RUN_P(32, 8, 16);
#define RUN_V(BX, BY, ZC)                                                                                    \
  timeit("V dbl2 " #BX "x" #BY " zc" #ZC, [&] {                                                              \
    kV<BX, BY, ZC><<<dim3((N + 2 * BX - 1) / (2 * BX), (N + BY - 1) / BY, (N + ZC - 1) / ZC), dim3(BX, BY)>>>( \
        g, d, r, x, c1, c2, dg, a, invd);                                                                    \
  })
  RUN_V(32, 4, 8);
  RUN_V(32, 4, 16);
  RUN_V(32, 8, 8);
  RUN_V(16, 8, 8);
  RUN_V(64, 2, 8);
  timeit("C streaming 3r1w", [&] { kC<<<148 * 8, 512>>>(g, d, r, x, total - 16); });
  return 0;
}
