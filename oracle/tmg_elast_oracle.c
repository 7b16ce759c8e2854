/* TEST INFRASTRUCTURE ONLY — CPU oracle for the Q1 elasticity MG-CG (BASELINE configs[4]).
 *
 * The reference has no elasticity implementation ("parity is unpinned
 * by the reference"; the SPEC substitutes a vector Laplacian). This file
 * defines the discretisation the GPU path must reproduce, with the reference's MG-CG algorithm
 * (solve_cg solver.cpp:214-266, Chebyshev solve_fixed solver.cpp:79-110, estimator
 * solver.cpp:520-581, DenseLU precond.cpp:11-66, trilinear P grid.cpp:373-428) applied to
 * 3 interleaved dofs per vertex (DMDA dof = 3 ordering, grid.cpp:48-50):
 *   - trilinear Q1 hexahedra on N^3 vertices of the unit cube, h = 1/(N-1); element
 *     stiffness E_e h K_ref(nu), K_ref from 2x2x2 Gauss quadrature (Voigt, engineering shear);
 *   - E_e = 10^(3 u(seed, e)) log-uniform in [1, 1e3], e = natural element index; nu = 0.3;
 *   - clamped x = 0 face: those dofs' rows keep only their assembled diagonal, other rows drop
 *     couplings to them, b = 0 there (the FD path's Dirichlet convention);
 *   - body force g = (0, 0, -1): b_z = sum over incident elements of -h^3/8;
 *   - point-block Jacobi (inverse 3x3 diagonal blocks; diagonal-only on clamped vertices);
 *   - rediscretised coarse levels: E of a coarse element = mean of its 8 children, h_c = 2h;
 *     R = P^T per component (finite-element scaling: no 2^-3);
 *   - LU on the coarsest level (5^3 x 3 = 375 unknowns at the BASELINE config).
 * Row arithmetic order (shared with the GPU kernels): incident elements ez, ey, ex in {-1, 0}
 * ascending; per element the K_ref row block times the element's x (vertices l' = 0..7,
 * x fastest, components beta then alpha) is accumulated first and then added scaled by E_e h.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "tmg_oracle.h"

/* 24x24 reference stiffness of the unit cube element, E = 1 (dof 3l + c, l = a + 2b + 4c). */
void orc_el_kref(double nu, double *K) {
  const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  const double mu = 1.0 / (2.0 * (1.0 + nu));
  double D[6][6];
  memset(D, 0, sizeof D);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) D[a][b] = lam + (a == b ? 2.0 * mu : 0.0);
  D[3][3] = D[4][4] = D[5][5] = mu;
  memset(K, 0, sizeof(double) * 576);
  const double g = 1.0 / sqrt(3.0);
  for (int q = 0; q < 8; ++q) {
    const double xi[3] = {(q & 1) ? g : -g, (q & 2) ? g : -g, (q & 4) ? g : -g};
    double dN[8][3];
    for (int l = 0; l < 8; ++l) {
      const double s[3] = {(l & 1) ? 1.0 : -1.0, (l & 2) ? 1.0 : -1.0, (l & 4) ? 1.0 : -1.0};
      const double f[3] = {1.0 + s[0] * xi[0], 1.0 + s[1] * xi[1], 1.0 + s[2] * xi[2]};
      /* d/dx = 2 d/dxi on the unit cube; N = f0 f1 f2 / 8 */
      dN[l][0] = 2.0 * (s[0] * f[1] * f[2] / 8.0);
      dN[l][1] = 2.0 * (f[0] * s[1] * f[2] / 8.0);
      dN[l][2] = 2.0 * (f[0] * f[1] * s[2] / 8.0);
    }
    double B[6][24];
    memset(B, 0, sizeof B);
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
    const double wdet = 1.0 / 8.0; /* Gauss weight 1 x det(J) of the unit cube */
    for (int i = 0; i < 24; ++i)
      for (int j = 0; j < 24; ++j) {
        double acc = 0.0;
        for (int a = 0; a < 6; ++a) acc += B[a][i] * DB[a][j];
        K[i * 24 + j] += acc * wdet;
      }
  }
}

typedef struct {
  int64_t n[3];
  int64_t nv;  /* vertices */
  double h;
  double *E;   /* per element, natural element index */
  double *binv;/* 9 per vertex */
  double lo, hi;
} el_level;

struct orc_el_mg {
  orc_el_cfg cfg;
  int nl;
  el_level lev[16];
  double K[576];
  int64_t nc;
  double *lu;
  int64_t *piv;
};

static int clamped(const el_level *L, int64_t i) { (void)L; return i == 0; }

/* y = A x on level L (rows in natural vertex order, 3 interleaved dofs) */
static void el_apply(const orc_el_mg *mg, const el_level *L, const double *x, double *y) {
  const int64_t nx = L->n[0], ny = L->n[1], nz = L->n[2];

  #pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const int64_t v = i + nx * (j + ny * k);
        const int cl = clamped(L, i);
        double acc[3] = {0.0, 0.0, 0.0};
        for (int ez = -1; ez <= 0; ++ez)
          for (int ey = -1; ey <= 0; ++ey)
            for (int ex = -1; ex <= 0; ++ex) {
              const int64_t ei = i + ex, ej = j + ey, ek = k + ez;
              if (ei < 0 || ej < 0 || ek < 0 || ei >= nx - 1 || ej >= ny - 1 || ek >= nz - 1) continue;
              const double eh = L->E[ei + (nx - 1) * (ej + (ny - 1) * ek)] * L->h;
              const int l = (int)(-ex) + 2 * (int)(-ey) + 4 * (int)(-ez);
              /* element contribution K_ref row block times the element's x, then scaled by E h */
              double ea[3] = {0.0, 0.0, 0.0};
              for (int lp = 0; lp < 8; ++lp) {
                const int64_t vi = ei + (lp & 1), vj = ej + ((lp >> 1) & 1), vk = ek + (lp >> 2);
                const int64_t w = vi + nx * (vj + ny * vk);
                if (cl) {
                  if (lp != l) continue;
                  for (int a = 0; a < 3; ++a) ea[a] += mg->K[(3 * l + a) * 24 + 3 * l + a] * x[3 * w + a];
                  continue;
                }
                if (clamped(L, vi)) continue;
                for (int b = 0; b < 3; ++b)
                  for (int a = 0; a < 3; ++a) ea[a] += mg->K[(3 * l + a) * 24 + 3 * lp + b] * x[3 * w + b];
              }
              for (int a = 0; a < 3; ++a) acc[a] += eh * ea[a];
            }
        y[3 * v + 0] = acc[0];
        y[3 * v + 1] = acc[1];
        y[3 * v + 2] = acc[2];
      }
}

/* inverse of the vertex's 3x3 diagonal block (adjugate / determinant) */
static void el_block_inv(const orc_el_mg *mg, el_level *L) {
  const int64_t nx = L->n[0], ny = L->n[1], nz = L->n[2];
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const int64_t v = i + nx * (j + ny * k);
        const int cl = clamped(L, i);
        double B[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int ez = -1; ez <= 0; ++ez)
          for (int ey = -1; ey <= 0; ++ey)
            for (int ex = -1; ex <= 0; ++ex) {
              const int64_t ei = i + ex, ej = j + ey, ek = k + ez;
              if (ei < 0 || ej < 0 || ek < 0 || ei >= nx - 1 || ej >= ny - 1 || ek >= nz - 1) continue;
              const double eh = L->E[ei + (nx - 1) * (ej + (ny - 1) * ek)] * L->h;
              const int l = (int)(-ex) + 2 * (int)(-ey) + 4 * (int)(-ez);
              for (int b = 0; b < 3; ++b)
                for (int a = 0; a < 3; ++a) {
                  if (cl && a != b) continue;
                  const double c = eh * mg->K[(3 * l + a) * 24 + 3 * l + b];
                  B[3 * a + b] += c;
                }
            }
        double *o = L->binv + 9 * v;
        if (cl) {
          memset(o, 0, sizeof(double) * 9);
          o[0] = 1.0 / B[0];
          o[4] = 1.0 / B[4];
          o[8] = 1.0 / B[8];
          continue;
        }
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
}

static void el_jacobi(const el_level *L, const double *x, double *y) {
  for (int64_t v = 0; v < L->nv; ++v) {
    const double *o = L->binv + 9 * v;
    for (int a = 0; a < 3; ++a) {
      double acc = 0.0;
      acc += o[3 * a + 0] * x[3 * v + 0];
      acc += o[3 * a + 1] * x[3 * v + 1];
      acc += o[3 * a + 2] * x[3 * v + 2];
      y[3 * v + a] = acc;
    }
  }
}

typedef struct {
  const orc_el_mg *mg;
  const el_level *L;
} el_ctx;
static void ctx_A(const void *c, const double *x, double *y) {
  const el_ctx *e = c;
  el_apply(e->mg, e->L, x, y);
}
static void ctx_M(const void *c, const double *x, double *y) { el_jacobi(((const el_ctx *)c)->L, x, y); }

/* solve_fixed, Chebyshev branch (solver.cpp:79-110) with point-block Jacobi */
static void el_smooth(const orc_el_mg *mg, const el_level *L, int m, const double *b, double *x) {
  const int64_t n = 3 * L->nv;
  double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
  double *d = malloc(sizeof(double) * n), *ad = malloc(sizeof(double) * n);
  const double theta = 0.5 * (L->hi + L->lo);
  const double delta = 0.5 * (L->hi - L->lo);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  el_apply(mg, L, x, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  el_jacobi(L, r, z);
  const double s = 1.0 / theta;
  for (int64_t i = 0; i < n; ++i) d[i] = z[i] * s;
  for (int it = 0; it < m; ++it) {
    for (int64_t i = 0; i < n; ++i) x[i] += 1.0 * d[i];
    if (it + 1 == m) break;
    el_apply(mg, L, d, ad);
    for (int64_t i = 0; i < n; ++i) r[i] += -1.0 * ad[i];
    el_jacobi(L, r, z);
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    const double c1 = rho_new * rho, c2 = 2.0 * rho_new / delta;
    for (int64_t i = 0; i < n; ++i) d[i] = c1 * d[i] + c2 * z[i];
    rho = rho_new;
  }
  free(r); free(z); free(d); free(ad);
}

/* R = P^T per component (finite-element scaling), order dk, dj, di ascending */
static void el_restrict(const el_level *F, const el_level *C, const double *rf, double *bc) {
  for (int64_t K = 0; K < C->n[2]; ++K)
    for (int64_t J = 0; J < C->n[1]; ++J)
      for (int64_t I = 0; I < C->n[0]; ++I)
        for (int a = 0; a < 3; ++a) {
          double acc = 0.0;
          for (int64_t k = 2 * K - 1; k <= 2 * K + 1; ++k) {
            if (k < 0 || k >= F->n[2]) continue;
            const double wz = (k == 2 * K) ? 1.0 : 0.5;
            for (int64_t j = 2 * J - 1; j <= 2 * J + 1; ++j) {
              if (j < 0 || j >= F->n[1]) continue;
              const double wy = (j == 2 * J) ? 1.0 : 0.5;
              for (int64_t i = 2 * I - 1; i <= 2 * I + 1; ++i) {
                if (i < 0 || i >= F->n[0]) continue;
                const double wx = (i == 2 * I) ? 1.0 : 0.5;
                const double w = wx * wy * wz;
                acc += w * rf[3 * (i + F->n[0] * (j + F->n[1] * k)) + a];
              }
            }
          }
          bc[3 * (I + C->n[0] * (J + C->n[1] * K)) + a] = acc;
        }
}

/* x_f += P x_c per component (grid.cpp:373-428 weights, columns ascending) */
static void el_prolong_add(const el_level *F, const el_level *C, const double *xc, double *xf) {
  for (int64_t k = 0; k < F->n[2]; ++k)
    for (int64_t j = 0; j < F->n[1]; ++j)
      for (int64_t i = 0; i < F->n[0]; ++i)
        for (int a = 0; a < 3; ++a) {
          const int nx = 1 + (int)(i & 1), ny = 1 + (int)(j & 1), nz = 1 + (int)(k & 1);
          const double wx = nx == 2 ? 0.5 : 1.0, wy = ny == 2 ? 0.5 : 1.0, wz = nz == 2 ? 0.5 : 1.0;
          double acc = 0.0;
          for (int tz = 0; tz < nz; ++tz)
            for (int ty = 0; ty < ny; ++ty)
              for (int tx = 0; tx < nx; ++tx) {
                const double ww = wx * wy * wz;
                acc += ww * xc[3 * ((i >> 1) + tx + C->n[0] * ((j >> 1) + ty + C->n[1] * ((k >> 1) + tz))) + a];
              }
          double *t = &xf[3 * (i + F->n[0] * (j + F->n[1] * k)) + a];
          *t = *t + acc;
        }
}

static void el_lu_factor(orc_el_mg *mg) {
  const el_level *L = &mg->lev[0];
  const int64_t n = 3 * L->nv;
  mg->nc = n;
  mg->lu = calloc((size_t)(n * n), sizeof(double));
  mg->piv = malloc(sizeof(int64_t) * n);
  double *e = calloc(n, sizeof(double)), *col = malloc(sizeof(double) * n);
  for (int64_t c = 0; c < n; ++c) {
    e[c] = 1.0;
    el_apply(mg, L, e, col);
    for (int64_t r = 0; r < n; ++r) mg->lu[r * n + c] = col[r];
    e[c] = 0.0;
  }
  free(e); free(col);
  double *a = mg->lu;
  for (int64_t k = 0; k < n; ++k) { /* precond.cpp:26-46 */
    int64_t p = k;
    double best = fabs(a[k * n + k]);
    for (int64_t i = k + 1; i < n; ++i)
      if (fabs(a[i * n + k]) > best) { best = fabs(a[i * n + k]); p = i; }
    mg->piv[k] = p;
    if (p != k)
      for (int64_t j = 0; j < n; ++j) { double t = a[k * n + j]; a[k * n + j] = a[p * n + j]; a[p * n + j] = t; }
    const double pivot = a[k * n + k];
    for (int64_t i = k + 1; i < n; ++i) {
      const double m = a[i * n + k] / pivot;
      a[i * n + k] = m;
      if (m == 0.0) continue;
      for (int64_t j = k + 1; j < n; ++j) a[i * n + j] -= m * a[k * n + j];
    }
  }
}

void orc_el_coarse_solve(const orc_el_mg *mg, const double *b, double *x) {
  const int64_t n = mg->nc;
  const double *lu = mg->lu;
  double *y = malloc(sizeof(double) * n);
  memcpy(y, b, sizeof(double) * n);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t p = mg->piv[k];
    if (p != k) { double t = y[k]; y[k] = y[p]; y[p] = t; }
    for (int64_t j = 0; j < k; ++j) y[k] -= lu[k * n + j] * y[j];
  }
  for (int64_t k = n - 1; k >= 0; --k) {
    double acc = y[k];
    for (int64_t j = k + 1; j < n; ++j) acc -= lu[k * n + j] * x[j];
    x[k] = acc / lu[k * n + k];
  }
  free(y);
}

void orc_el_vcycle(const orc_el_mg *mg, int level, const double *b, double *x) {
  const el_level *L = &mg->lev[level];
  memset(x, 0, sizeof(double) * 3 * L->nv);
  if (level == 0) {
    orc_el_coarse_solve(mg, b, x);
    return;
  }
  const el_level *C = &mg->lev[level - 1];
  el_smooth(mg, L, mg->cfg.smooth_its, b, x);
  double *r = malloc(sizeof(double) * 3 * L->nv);
  el_apply(mg, L, x, r);
  for (int64_t i = 0; i < 3 * L->nv; ++i) r[i] = b[i] - r[i];
  double *bc = malloc(sizeof(double) * 3 * C->nv), *xc = malloc(sizeof(double) * 3 * C->nv);
  el_restrict(L, C, r, bc);
  orc_el_vcycle(mg, level - 1, bc, xc);
  el_prolong_add(L, C, xc, x);
  el_smooth(mg, L, mg->cfg.smooth_its, b, x);
  free(r); free(bc); free(xc);
}

orc_el_mg *orc_el_create(const orc_el_cfg *cfg) {
  orc_el_mg *mg = calloc(1, sizeof *mg);
  mg->cfg = *cfg;
  mg->nl = cfg->nlevels;
  orc_el_kref(cfg->nu, mg->K);
  int64_t n[3] = {cfg->np[0], cfg->np[1], cfg->np[2]};
  double h = 1.0 / (double)(cfg->np[0] - 1);
  for (int l = mg->nl - 1; l >= 0; --l) {
    el_level *L = &mg->lev[l];
    memcpy(L->n, n, sizeof n);
    L->nv = n[0] * n[1] * n[2];
    L->h = h;
    const int64_t ne = (n[0] - 1) * (n[1] - 1) * (n[2] - 1);
    L->E = malloc(sizeof(double) * (ne > 0 ? ne : 1));
    if (l == mg->nl - 1) {
      for (int64_t e = 0; e < ne; ++e) L->E[e] = pow(10.0, 3.0 * orc_hashed_uniform(cfg->seed_e, (uint64_t)e));
    } else { /* mean of the 8 children (cz, cy, cx ascending) */
      const el_level *F = &mg->lev[l + 1];
      const int64_t fx = F->n[0] - 1, fy = F->n[1] - 1;
      for (int64_t K = 0; K < n[2] - 1; ++K)
        for (int64_t J = 0; J < n[1] - 1; ++J)
          for (int64_t I = 0; I < n[0] - 1; ++I) {
            double acc = 0.0;
            for (int c = 0; c < 8; ++c)
              acc += F->E[(2 * I + (c & 1)) + fx * ((2 * J + ((c >> 1) & 1)) + fy * (2 * K + (c >> 2)))];
            L->E[I + (n[0] - 1) * (J + (n[1] - 1) * K)] = 0.125 * acc;
          }
    }
    L->binv = malloc(sizeof(double) * 9 * L->nv);
    el_block_inv(mg, L);
    for (int a = 0; a < 3; ++a) n[a] = (n[a] + 1) / 2;
    h *= 2.0;
  }
  for (int l = 1; l < mg->nl; ++l) {
    el_level *L = &mg->lev[l];
    const int64_t nd = 3 * L->nv;
    double *b0 = malloc(sizeof(double) * nd);
    orc_fill_random(nd, 0x5eedbeefULL, b0);
    el_ctx c = {mg, L};
    double lo, hi;
    orc_estimate_generic(nd, ctx_A, ctx_M, &c, b0, cfg->est_mode, &lo, &hi);
    L->lo = lo;
    L->hi = hi;
    free(b0);
  }
  el_lu_factor(mg);
  return mg;
}

void orc_el_destroy(orc_el_mg *mg) {
  if (!mg) return;
  for (int l = 0; l < mg->nl; ++l) {
    free(mg->lev[l].E);
    free(mg->lev[l].binv);
  }
  free(mg->lu);
  free(mg->piv);
  free(mg);
}

int64_t orc_el_level_nv(const orc_el_mg *mg, int level) { return mg->lev[level].nv; }
void orc_el_bounds(const orc_el_mg *mg, int level, double *lo, double *hi) {
  *lo = mg->lev[level].lo;
  *hi = mg->lev[level].hi;
}
void orc_el_apply(const orc_el_mg *mg, int level, const double *x, double *y) { el_apply(mg, &mg->lev[level], x, y); }
void orc_el_jacobi(const orc_el_mg *mg, int level, const double *x, double *y) { el_jacobi(&mg->lev[level], x, y); }
void orc_el_smooth(const orc_el_mg *mg, int level, const double *b, double *x) {
  el_smooth(mg, &mg->lev[level], mg->cfg.smooth_its, b, x);
}
void orc_el_restrict(const orc_el_mg *mg, int fine_level, const double *rf, double *bc) {
  el_restrict(&mg->lev[fine_level], &mg->lev[fine_level - 1], rf, bc);
}
void orc_el_prolong_add(const orc_el_mg *mg, int fine_level, const double *xc, double *xf) {
  el_prolong_add(&mg->lev[fine_level], &mg->lev[fine_level - 1], xc, xf);
}
void orc_el_elements(const orc_el_mg *mg, int level, double *E) {
  const el_level *L = &mg->lev[level];
  memcpy(E, L->E, sizeof(double) * (L->n[0] - 1) * (L->n[1] - 1) * (L->n[2] - 1));
}

/* body force g = (0, 0, -1): b_z(v) = sum over incident elements of -h^3/8; 0 on clamped dofs */
void orc_el_rhs(const int64_t np[3], double *b) {
  const double h = 1.0 / (double)(np[0] - 1);
  const double q = -(h * h * h) / 8.0;
  for (int64_t k = 0; k < np[2]; ++k)
    for (int64_t j = 0; j < np[1]; ++j)
      for (int64_t i = 0; i < np[0]; ++i) {
        const int64_t v = i + np[0] * (j + np[1] * k);
        double acc = 0.0;
        for (int ez = -1; ez <= 0; ++ez)
          for (int ey = -1; ey <= 0; ++ey)
            for (int ex = -1; ex <= 0; ++ex) {
              const int64_t ei = i + ex, ej = j + ey, ek = k + ez;
              if (ei < 0 || ej < 0 || ek < 0 || ei >= np[0] - 1 || ej >= np[1] - 1 || ek >= np[2] - 1) continue;
              acc += q;
            }
        b[3 * v + 0] = 0.0;
        b[3 * v + 1] = 0.0;
        b[3 * v + 2] = i == 0 ? 0.0 : acc;
      }
}

/* solve_cg (solver.cpp:214-266), PC = one elasticity V-cycle */
int orc_el_solve(const orc_el_mg *mg, const double *b, double *x, double rtol, double atol, int max_its,
                 double *history, orc_report *rep) {
  const int top = mg->nl - 1;
  const el_level *L = &mg->lev[top];
  const int64_t n = 3 * L->nv;
  double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
  double *p = malloc(sizeof(double) * n), *w = malloc(sizeof(double) * n);
  memset(rep, 0, sizeof *rep);
  el_apply(mg, L, x, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  orc_el_vcycle(mg, top, r, z);
  double nrm = sqrt(orc_dot(n, z, z));
  rep->norm0 = nrm;
  rep->norm_final = nrm;
  if (history) history[0] = nrm;
  const double tol = fmax(rtol * nrm, atol);
  rep->reason = 2;
  if (nrm <= tol) {
    rep->reason = nrm <= atol ? 1 : 0;
    goto done;
  }
  memcpy(p, z, sizeof(double) * n);
  double rz = orc_dot(n, r, z);
  for (int it = 1; it <= max_its; ++it) {
    el_apply(mg, L, p, w);
    const double pw = orc_dot(n, p, w);
    if (pw <= 0.0 || !isfinite(pw)) { rep->reason = 4; goto done; }
    const double alpha = rz / pw;
    for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
    for (int64_t i = 0; i < n; ++i) r[i] += -alpha * w[i];
    orc_el_vcycle(mg, top, r, z);
    const double rz_new = orc_dot(n, r, z);
    nrm = sqrt(orc_dot(n, z, z));
    rep->iterations = it;
    rep->norm_final = nrm;
    if (history) history[it] = nrm;
    if (nrm <= tol) { rep->reason = nrm <= atol ? 1 : 0; goto done; }
    if (rz == 0.0 || !isfinite(rz_new)) { rep->reason = 4; goto done; }
    const double beta = rz_new / rz;
    rz = rz_new;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  rep->reason = 2;
done:
  free(r); free(z); free(p); free(w);
  return rep->reason;
}
