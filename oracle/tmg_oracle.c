/* TEST INFRASTRUCTURE ONLY — see tmg_oracle.h. Never linked into the product.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off: the reference is compiled for
 * baseline x86-64 without FMA, so every a*x+y here is a separate multiply and add).
 */
#include "tmg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* common.hpp:40-53 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

double orc_hashed_uniform(uint64_t seed, uint64_t index) {
  const uint64_t h = orc_splitmix64(seed ^ orc_splitmix64(index));
  return (double)(h >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------------------- */
/* grid maps */

/* grid.cpp:184-193 — near-equal split, larger blocks first */
void orc_split_axis(int64_t n, int parts, int64_t *off) {
  const int64_t base = n / parts, rem = n % parts;
  off[0] = 0;
  for (int p = 0; p < parts; ++p) off[p + 1] = off[p] + base + (p < rem ? 1 : 0);
}

/* grid.cpp:195-207 — factorizations enumerated axis 0 first, factor ascending */
static void enum_fact(int size, int dim, int cur[3], int axis, int (*out)[3], int *n_out) {
  if (axis == dim - 1) {
    cur[axis] = size;
    memcpy(out[*n_out], cur, sizeof(int) * 3);
    (*n_out)++;
    return;
  }
  for (int f = 1; f <= size; ++f) {
    if (size % f) continue;
    cur[axis] = f;
    enum_fact(size / f, dim, cur, axis + 1, out, n_out);
  }
}

/* grid.cpp:209-240 — min sum p_a/N_a, 1e-15 tie band, ties -> more ranks on slowest axis */
int orc_choose_proc_grid(int size, int dim, const int64_t np[3], int pg[3]) {
  static int cands[4096][3];
  int n = 0, cur[3] = {1, 1, 1};
  enum_fact(size, dim, cur, 0, cands, &n);
  int have = 0;
  int best[3] = {1, 1, 1};
  double best_cost = 0.0;
  for (int c = 0; c < n; ++c) {
    int feasible = 1;
    double cost = 0.0;
    for (int a = 0; a < dim; ++a) {
      if (cands[c][a] > np[a]) feasible = 0;
      cost += (double)cands[c][a] / (double)np[a];
    }
    if (!feasible) continue;
    if (!have || cost < best_cost - 1e-15) {
      memcpy(best, cands[c], sizeof best);
      best_cost = cost;
      have = 1;
    } else if (cost < best_cost + 1e-15) {
      for (int a = dim - 1; a >= 0; --a) {
        if (cands[c][a] != best[a]) {
          if (cands[c][a] > best[a]) memcpy(best, cands[c], sizeof best);
          break;
        }
      }
    }
  }
  if (!have) return -1;
  memcpy(pg, best, sizeof best);
  return 0;
}

static void make_header(int dim, const int64_t np[3], int dof, const int pg[3], orc_header *h) {
  memset(h, 0, sizeof *h);
  h->dim = dim;
  h->dof = dof;
  for (int a = 0; a < 3; ++a) {
    h->np[a] = np[a];
    h->pg[a] = pg[a];
    orc_split_axis(np[a], pg[a], h->off[a]);
  }
}

/* grid.cpp:256-284 */
int orc_build_header(int size, int dim, const int64_t np[3], int dof, const int *hint, orc_header *h) {
  if (dim < 1 || dim > 3 || dof < 1) return -1;
  for (int a = dim; a < 3; ++a)
    if (np[a] != 1) return -1;
  int pg[3] = {1, 1, 1};
  if (hint) {
    int prod = 1;
    for (int a = 0; a < 3; ++a) prod *= hint[a];
    if (prod != size) return -1;
    for (int a = 0; a < 3; ++a)
      if (hint[a] > np[a]) return -1;
    memcpy(pg, hint, sizeof pg);
  } else if (orc_choose_proc_grid(size, dim, np, pg)) {
    return -1;
  }
  make_header(dim, np, dof, pg, h);
  return 0;
}

/* grid.cpp:299-322 */
int orc_coarsen_header(const orc_header *fine, orc_header *coarse) {
  *coarse = *fine;
  for (int a = 0; a < fine->dim; ++a) {
    const int64_t n = fine->np[a];
    if (n == 1) continue;
    if (n < 3 || n % 2 == 0) return -1;
    coarse->np[a] = (n + 1) / 2;
  }
  for (int a = 0; a < 3; ++a) {
    if (fine->np[a] == coarse->np[a]) continue;
    for (int p = 0; p <= fine->pg[a]; ++p) coarse->off[a][p] = (fine->off[a][p] + 1) / 2;
    for (int p = 0; p < fine->pg[a]; ++p)
      if (coarse->off[a][p + 1] <= coarse->off[a][p]) return -1;
  }
  return 0;
}

static int n_ranks(const orc_header *h) { return h->pg[0] * h->pg[1] * h->pg[2]; }

static void box_of(const orc_header *h, int rank, int64_t lo[3], int64_t hi[3]) {
  /* grid.cpp:17-38 */
  int pc[3];
  pc[0] = rank % h->pg[0];
  pc[1] = (rank / h->pg[0]) % h->pg[1];
  pc[2] = rank / (h->pg[0] * h->pg[1]);
  for (int a = 0; a < 3; ++a) {
    lo[a] = h->off[a][pc[a]];
    hi[a] = h->off[a][pc[a] + 1];
  }
}

static int64_t box_nv(const orc_header *h, int rank) {
  int64_t lo[3], hi[3];
  box_of(h, rank, lo, hi);
  return (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
}

/* grid.cpp:40-46 */
void orc_layout_offsets(const orc_header *h, int64_t *offsets) {
  offsets[0] = 0;
  for (int r = 0; r < n_ranks(h); ++r) offsets[r + 1] = offsets[r] + box_nv(h, r) * h->dof;
}

int64_t orc_natural_index(const orc_header *h, int64_t i, int64_t j, int64_t k, int c) {
  return c + h->dof * (i + h->np[0] * (j + h->np[1] * k));
}

static int upper_slot(const int64_t *off, int parts, int64_t v) {
  /* upper_bound(off, off+parts+1, v) - off - 1 */
  int s = 0;
  while (s + 1 <= parts && off[s + 1] <= v) ++s;
  return s;
}

/* grid.cpp:61-82 */
int64_t orc_global_index(const orc_header *h, int64_t i, int64_t j, int64_t k, int c) {
  const int64_t ijk[3] = {i, j, k};
  int pc[3];
  for (int a = 0; a < 3; ++a) pc[a] = upper_slot(h->off[a], h->pg[a], ijk[a]);
  const int rank = pc[0] + h->pg[0] * (pc[1] + h->pg[1] * pc[2]);
  int64_t lo[3], hi[3];
  box_of(h, rank, lo, hi);
  const int64_t v = (i - lo[0]) + (hi[0] - lo[0]) * ((j - lo[1]) + (hi[1] - lo[1]) * (k - lo[2]));
  int64_t offset = 0;
  for (int r = 0; r < rank; ++r) offset += box_nv(h, r) * h->dof;
  return offset + v * h->dof + c;
}

/* grid.cpp:84-101, 110-115 */
int64_t orc_global_to_natural(const orc_header *h, int64_t g) {
  int64_t offset = 0;
  int rank = 0;
  const int nr = n_ranks(h);
  for (; rank < nr; ++rank) {
    const int64_t sz = box_nv(h, rank) * h->dof;
    if (g < offset + sz) break;
    offset += sz;
  }
  int64_t lo[3], hi[3];
  box_of(h, rank, lo, hi);
  const int64_t local = g - offset;
  const int c = (int)(local % h->dof);
  int64_t v = local / h->dof;
  const int64_t ex = hi[0] - lo[0], ey = hi[1] - lo[1];
  const int64_t i = lo[0] + v % ex;
  v /= ex;
  const int64_t j = lo[1] + v % ey;
  const int64_t k = lo[2] + v / ey;
  return orc_natural_index(h, i, j, k, c);
}

/* grid.cpp:52-59, 103-108 */
int64_t orc_natural_to_global(const orc_header *h, int64_t n) {
  const int c = (int)(n % h->dof);
  int64_t v = n / h->dof;
  const int64_t i = v % h->np[0];
  v /= h->np[0];
  const int64_t j = v % h->np[1];
  const int64_t k = v / h->np[1];
  return orc_global_index(h, i, j, k, c);
}

/* comm.cpp:353-360 — members {k : k mod r == 0} */
int orc_split_strided(int n, int r, int *member_map) {
  if (r < 1) return -1;
  int m = 0;
  for (int k = 0; k < n; k += r) member_map[m++] = k;
  return m;
}

/* grid.cpp:433-493 (header part; coordinates are never custom on this path).
 * override_[a] == 0 means "not overridden". */
int orc_repartition(const orc_header *h, int sub_size, const int override_[3], orc_header *out) {
  const int parent = n_ranks(h);
  int any = 0;
  for (int a = 0; a < 3; ++a) any |= override_ && override_[a] != 0;
  if (!any && sub_size == parent) {
    *out = *h;
    return 0;
  }
  if (any) {
    int fixed[3] = {0, 0, 0}, fixed_prod = 1, n_free = 0;
    for (int a = 0; a < 3; ++a) {
      if (override_[a]) {
        fixed[a] = override_[a];
        if (fixed[a] < 1) return -1;
        fixed_prod *= fixed[a];
      } else if (a < h->dim) {
        ++n_free;
      } else {
        fixed[a] = 1;
      }
    }
    if (fixed_prod > sub_size || sub_size % fixed_prod) return -1;
    int pg[3] = {fixed[0], fixed[1], fixed[2]};
    if (n_free == 0) {
      if (fixed_prod != sub_size) return -1;
    } else {
      int64_t free_np[3] = {1, 1, 1};
      int free_axes[3], nf = 0;
      for (int a = 0; a < h->dim; ++a)
        if (!override_[a]) {
          free_axes[nf] = a;
          free_np[nf] = h->np[a];
          ++nf;
        }
      int chosen[3];
      if (orc_choose_proc_grid(sub_size / fixed_prod, nf, free_np, chosen)) return -1;
      for (int t = 0; t < nf; ++t) pg[free_axes[t]] = chosen[t];
    }
    for (int a = 0; a < 3; ++a)
      if (pg[a] > h->np[a]) return -1;
    make_header(h->dim, h->np, h->dof, pg, out);
    return 0;
  }
  return orc_build_header(sub_size, h->dim, h->np, h->dof, NULL, out);
}

/* grid.cpp:566-580 ; group_end: comm.cpp:161-164 */
void orc_prefusion_layout(const orc_header *newh, int parent_size, const int *member_map, int n_members,
                          int64_t *offsets) {
  int64_t sizes[4 * ORC_MAX_PARTS];
  int64_t dst[4 * ORC_MAX_PARTS + 1];
  memset(sizes, 0, sizeof sizes);
  orc_layout_offsets(newh, dst);
  for (int m = 0; m < n_members; ++m) {
    const int64_t rows = dst[m + 1] - dst[m];
    const int gb = member_map[m];
    const int ge = m + 1 < n_members ? member_map[m + 1] : parent_size;
    const int width = ge - gb;
    const int64_t base = rows / width, rem = rows % width;
    for (int p = gb; p < ge; ++p) sizes[p] = base + ((p - gb) < rem ? 1 : 0);
  }
  offsets[0] = 0;
  for (int p = 0; p < parent_size; ++p) offsets[p + 1] = offsets[p] + sizes[p];
}

/* grid.cpp:582-599 — q[p] = column of the single 1 in row p of P-hat */
void orc_build_permutation(const orc_header *oldh, const orc_header *newh, int64_t *q) {
  int64_t n = oldh->np[0] * oldh->np[1] * oldh->np[2] * oldh->dof;
  for (int64_t p = 0; p < n; ++p) q[p] = orc_natural_to_global(newh, orc_global_to_natural(oldh, p));
}

/* ------------------------------------------------------------------------- */
/* numerics */

typedef struct {
  int64_t n[3];
  int64_t nv;
  double ih2[3];
  double *k;        /* vertex coefficient (NULL = constant 1) */
  double *cxp;      /* -(kf*ih2x) for face (i,i+1); valid where both endpoints interior */
  double *cyp;
  double *czp;
  double *diag;
  double *inv_diag; /* precond.cpp:179 */
  double lo, hi;    /* chebyshev interval */
  double *S;        /* Galerkin level: 27 row coefficients, S[s*nv + v] (NULL = 7-point) */
} orc_level;

struct orc_mg {
  orc_mg_cfg cfg;
  int nl;
  orc_level lev[16];
  /* dense LU of level 0 (precond.cpp:11-48) */
  int64_t nc;
  double *lu;
  int64_t *piv;
};

static int is_bnd(const orc_level *L, int64_t i, int64_t j, int64_t k) {
  return i == 0 || j == 0 || k == 0 || i == L->n[0] - 1 || j == L->n[1] - 1 || k == L->n[2] - 1;
}

/* 32 seeded spheres, k_in inside (|x-c|^2 <= r^2, fixed mul/add order) */
static double sphere_k(const orc_mg_cfg *cfg, double x, double y, double z) {
  for (int s = 0; s < cfg->n_spheres; ++s) {
    const double cx = orc_hashed_uniform(cfg->seed_k, (uint64_t)(4 * s + 0));
    const double cy = orc_hashed_uniform(cfg->seed_k, (uint64_t)(4 * s + 1));
    const double cz = orc_hashed_uniform(cfg->seed_k, (uint64_t)(4 * s + 2));
    const double r = 0.05 + 0.10 * orc_hashed_uniform(cfg->seed_k, (uint64_t)(4 * s + 3));
    const double dx = x - cx, dy = y - cy, dz = z - cz;
    const double d2 = dx * dx + dy * dy + dz * dz;
    if (d2 <= r * r) return cfg->k_in;
  }
  return 1.0;
}

static double harm(double a, double b) { return 2.0 * a * b / (a + b); }

/* Rediscretized 7-point operator on one level:
 * interior rows: couplings -(kf*ih2) to interior neighbours only (boundary eliminated);
 * diagonal = sum over faces (-z,-y,-x,+x,+y,+z) of kf*ih2 (out-of-grid face: kf = k_i);
 * boundary rows: diagonal only. */
static void level_build(const orc_mg_cfg *cfg, orc_level *L) {
  const int64_t nx = L->n[0], ny = L->n[1], nz = L->n[2];
  L->nv = nx * ny * nz;
  for (int a = 0; a < 3; ++a) {
    const double h = 1.0 / (double)(L->n[a] - 1); /* grid.cpp:144-151 */
    L->ih2[a] = 1.0 / (h * h);
  }
  L->k = malloc(sizeof(double) * L->nv);
  #pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const int64_t v = i + nx * (j + ny * k);
        if (cfg->kind == ORC_VARCOEF7) {
          const double x = (double)i * (1.0 / (double)(nx - 1));
          const double y = (double)j * (1.0 / (double)(ny - 1));
          const double z = (double)k * (1.0 / (double)(nz - 1));
          L->k[v] = sphere_k(cfg, x, y, z);
        } else {
          L->k[v] = 1.0;
        }
      }
  L->cxp = calloc(L->nv, sizeof(double));
  L->cyp = calloc(L->nv, sizeof(double));
  L->czp = calloc(L->nv, sizeof(double));
  L->diag = malloc(sizeof(double) * L->nv);
  L->inv_diag = malloc(sizeof(double) * L->nv);
  const int64_t sx = 1, sy = nx, sz = nx * ny;
  #pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const int64_t v = i + nx * (j + ny * k);
        const double kc = L->k[v];
        if (i + 1 < nx) L->cxp[v] = -(harm(kc, L->k[v + sx]) * L->ih2[0]);
        if (j + 1 < ny) L->cyp[v] = -(harm(kc, L->k[v + sy]) * L->ih2[1]);
        if (k + 1 < nz) L->czp[v] = -(harm(kc, L->k[v + sz]) * L->ih2[2]);
        const double fzm = (k > 0 ? harm(kc, L->k[v - sz]) : kc) * L->ih2[2];
        const double fym = (j > 0 ? harm(kc, L->k[v - sy]) : kc) * L->ih2[1];
        const double fxm = (i > 0 ? harm(kc, L->k[v - sx]) : kc) * L->ih2[0];
        const double fxp = (i + 1 < nx ? harm(kc, L->k[v + sx]) : kc) * L->ih2[0];
        const double fyp = (j + 1 < ny ? harm(kc, L->k[v + sy]) : kc) * L->ih2[1];
        const double fzp = (k + 1 < nz ? harm(kc, L->k[v + sz]) : kc) * L->ih2[2];
        double d = 0.0;
        d += fzm;
        d += fym;
        d += fxm;
        d += fxp;
        d += fyp;
        d += fzp;
        L->diag[v] = d;
        L->inv_diag[v] = 1.0 / d;
      }
}

/* dist_matrix.cpp:213-223 on the 1-rank CSR (columns ascending = natural order):
 * acc = 0; acc += a*x over (-z,-y,-x,c,+x,+y,+z) present columns. */
static void level_apply(const orc_level *L, const double *x, double *y) {
  const int64_t nx = L->n[0], ny = L->n[1], nz = L->n[2];
  const int64_t sy = nx, sz = nx * ny;
  if (L->S) { /* 27-point Galerkin row, columns ascending (dz, dy, dx lexicographic) */
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nz; ++k)
      for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
          const int64_t v = i + nx * (j + ny * k);
          double acc = 0.0;
          for (int s = 0; s < 27; ++s) {
            const int dz = s / 9 - 1, dy = (s / 3) % 3 - 1, dx = s % 3 - 1;
            if (k + dz < 0 || k + dz >= nz || j + dy < 0 || j + dy >= ny || i + dx < 0 || i + dx >= nx) continue;
            acc += L->S[s * L->nv + v] * x[v + dz * sz + dy * sy + dx];
          }
          y[v] = acc;
        }
    return;
  }
  #pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        const int64_t v = i + nx * (j + ny * k);
        double acc = 0.0;
        if (is_bnd(L, i, j, k)) {
          acc += L->diag[v] * x[v];
        } else {
          if (k - 1 > 0) acc += L->czp[v - sz] * x[v - sz];
          if (j - 1 > 0) acc += L->cyp[v - sy] * x[v - sy];
          if (i - 1 > 0) acc += L->cxp[v - 1] * x[v - 1];
          acc += L->diag[v] * x[v];
          if (i + 1 < nx - 1) acc += L->cxp[v] * x[v + 1];
          if (j + 1 < ny - 1) acc += L->cyp[v] * x[v + sy];
          if (k + 1 < nz - 1) acc += L->czp[v] * x[v + sz];
        }
        y[v] = acc;
      }
}

/* Row of a 7-point level as 27 slots (s = (dz+1)*9 + (dy+1)*3 + (dx+1)); zeros elsewhere. */
static void row27_7pt(const orc_level *L, int64_t i, int64_t j, int64_t k, double a[27]) {
  const int64_t nx = L->n[0], ny = L->n[1], nz = L->n[2];
  const int64_t v = i + nx * (j + ny * k), sy = nx, sz = nx * ny;
  for (int s = 0; s < 27; ++s) a[s] = 0.0;
  a[13] = L->diag[v];
  if (is_bnd(L, i, j, k)) return;
  if (k - 1 > 0) a[4] = L->czp[v - sz];
  if (j - 1 > 0) a[10] = L->cyp[v - sy];
  if (i - 1 > 0) a[12] = L->cxp[v - 1];
  if (i + 1 < nx - 1) a[14] = L->cxp[v];
  if (j + 1 < ny - 1) a[16] = L->cyp[v];
  if (k + 1 < nz - 1) a[22] = L->czp[v];
}

static double pw1(int64_t d) { return d == 0 ? 1.0 : ((d == 1 || d == -1) ? 0.5 : 0.0); }

/* Galerkin coarse operator A_c = R A_f P with R = 2^-3 P^T (ptap, dist_matrix.cpp:462-468,
 * with the SURVEY App. A-C6 restriction scaling), as 27-point rows. For each coarse row I and
 * column slot J the terms are summed over the fine rows f of R's support (ascending natural)
 * and the fine columns g of A's row f (ascending natural): (R(I,f) a(f,g)) P(g,J). */
static void galerkin_build(const orc_level *F, orc_level *C) {
  const int64_t cn = C->nv;
  C->S = calloc((size_t)(27 * cn), sizeof(double));
  #pragma omp parallel for schedule(static)
  for (int64_t K = 0; K < C->n[2]; ++K)
    for (int64_t J = 0; J < C->n[1]; ++J)
      for (int64_t I = 0; I < C->n[0]; ++I) {
        double acc[27];
        for (int t = 0; t < 27; ++t) acc[t] = 0.0;
        for (int64_t fk = 2 * K - 1; fk <= 2 * K + 1; ++fk) {
          if (fk < 0 || fk >= F->n[2]) continue;
          for (int64_t fj = 2 * J - 1; fj <= 2 * J + 1; ++fj) {
            if (fj < 0 || fj >= F->n[1]) continue;
            for (int64_t fi = 2 * I - 1; fi <= 2 * I + 1; ++fi) {
              if (fi < 0 || fi >= F->n[0]) continue;
              const double wr = 0.125 * (pw1(fi - 2 * I) * pw1(fj - 2 * J) * pw1(fk - 2 * K));
              double a[27];
              if (F->S) {
                const int64_t fv = fi + F->n[0] * (fj + F->n[1] * fk);
                for (int s = 0; s < 27; ++s) a[s] = F->S[s * F->nv + fv];
              } else {
                row27_7pt(F, fi, fj, fk, a);
              }
              for (int s = 0; s < 27; ++s) {
                const int64_t gk = fk + s / 9 - 1, gj = fj + (s / 3) % 3 - 1, gi = fi + s % 3 - 1;
                if (gk < 0 || gk >= F->n[2] || gj < 0 || gj >= F->n[1] || gi < 0 || gi >= F->n[0]) continue;
                const double ra = wr * a[s];
                for (int t = 0; t < 27; ++t) {
                  const int64_t cK = K + t / 9 - 1, cJ = J + (t / 3) % 3 - 1, cI = I + t % 3 - 1;
                  const double wp = pw1(gi - 2 * cI) * pw1(gj - 2 * cJ) * pw1(gk - 2 * cK);
                  if (wp != 0.0) acc[t] += ra * wp;
                }
              }
            }
          }
        }
        const int64_t cv = I + C->n[0] * (J + C->n[1] * K);
        for (int t = 0; t < 27; ++t) C->S[t * cn + cv] = acc[t];
        C->diag[cv] = acc[13];
        C->inv_diag[cv] = 1.0 / acc[13];
      }
}

int orc_mg_stencil27(const orc_mg *mg, int level, double *out) {
  const orc_level *L = &mg->lev[level];
  if (!L->S) return 0;
  memcpy(out, L->S, sizeof(double) * 27 * L->nv);
  return 1;
}

/* dist_vector.cpp:33-38 + comm.cpp:338-351 (1 rank: serial left fold) */
double orc_dot(int64_t n, const double *x, const double *y) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double p = x[i] * y[i];
    acc += p;
  }
  return acc;
}

static void jacobi(const orc_level *L, const double *x, double *y) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < L->nv; ++i) y[i] = x[i] * L->inv_diag[i];
}

/* tridiag_eig_max, solver.cpp:488-516 */
static double tridiag_eig_max(int n, const double *d, const double *e) {
  double lo = d[0], hi = d[0];
  for (int i = 0; i < n; ++i) {
    const double left = i > 0 ? fabs(e[i - 1]) : 0.0;
    const double right = i + 1 < n ? fabs(e[i]) : 0.0;
    lo = fmin(lo, d[i] - left - right);
    hi = fmax(hi, d[i] + left + right);
  }
  for (int it = 0; it < 200 && hi - lo > 1e-12 * fmax(1.0, fabs(hi)); ++it) {
    const double mid = 0.5 * (lo + hi);
    int count = 0;
    double q = 1.0;
    for (int i = 0; i < n; ++i) {
      const double off = i > 0 ? e[i - 1] : 0.0;
      q = d[i] - mid - (q == 0.0 ? fabs(off) / 1e-300 : off * off / q);
      if (q < 0.0) ++count;
    }
    if (count >= n)
      hi = mid;
    else
      lo = mid;
  }
  return 0.5 * (lo + hi);
}

typedef orc_op_fn op_fn;

/* chebyshev_bounds_estimate, solver.cpp:520-581. mode REFERENCE reproduces the
 * shipped loop (p never updated, :537-561); LANCZOS adds p = z + beta p. */
int orc_estimate_generic(int64_t n, op_fn A, op_fn M, const void *ctx, const double *b0, int mode,
                         double *lo_out, double *hi_out) {
  const int kSteps = 10;
  double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
  double *p = malloc(sizeof(double) * n), *w = malloc(sizeof(double) * n);
  double *x = calloc(n, sizeof(double));
  double alphas[16], betas[16];
  int na = 0, nb = 0, broke = 0;
  memcpy(r, b0, sizeof(double) * n);
  M(ctx, r, z);
  memcpy(p, z, sizeof(double) * n);
  double rz = orc_dot(n, r, z);
  for (int it = 0; it < kSteps; ++it) {
    if (rz == 0.0 || !isfinite(rz)) break;
    A(ctx, p, w);
    const double pw = orc_dot(n, p, w);
    if (pw <= 0.0 || !isfinite(pw)) {
      if (na == 0) broke = 1;
      break;
    }
    const double alpha = rz / pw;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) r[i] += -alpha * w[i];
    M(ctx, r, z);
    const double rz_new = orc_dot(n, r, z);
    alphas[na++] = alpha;
    if (rz_new <= 0.0 || !isfinite(rz_new)) break;
    const double beta = rz_new / rz;
    betas[nb++] = beta;
    rz = rz_new;
    if (mode == ORC_EST_LANCZOS)
      #pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  free(r); free(z); free(p); free(w); free(x);
  if (broke || na == 0) {
    *lo_out = 0.1; *hi_out = 1.1;
    return 1;
  }
  double d[16], e[16];
  for (int i = 0; i < na; ++i) {
    d[i] = 1.0 / alphas[i];
    if (i > 0) d[i] += betas[i - 1] / alphas[i - 1];
    if (i + 1 < na) e[i] = sqrt(betas[i]) / alphas[i];
  }
  const double lam = tridiag_eig_max(na, d, e);
  if (!(lam > 0.0) || !isfinite(lam)) {
    *lo_out = 0.1; *hi_out = 1.1;
    return 1;
  }
  *lo_out = 0.1 * lam;
  *hi_out = 1.1 * lam;
  return 0;
}

static void lvl_A(const void *ctx, const double *x, double *y) { level_apply((const orc_level *)ctx, x, y); }
static void lvl_M(const void *ctx, const double *x, double *y) { jacobi((const orc_level *)ctx, x, y); }

void orc_fill_random(int64_t n, uint64_t seed, double *x) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) x[i] = 2.0 * orc_hashed_uniform(seed, (uint64_t)i) - 1.0;
}

int orc_estimate(const orc_mg *mg, int level, int mode, double *lo, double *hi) {
  const orc_level *L = &mg->lev[level];
  double *b = malloc(sizeof(double) * L->nv);
  orc_fill_random(L->nv, 0x5eedbeefULL, b);
  const int rc = orc_estimate_generic(L->nv, lvl_A, lvl_M, L, b, mode, lo, hi);
  free(b);
  return rc;
}

typedef struct {
  int n;
  const double *A;
  int jacobi;
} dense_ctx;
static void dn_A(const void *c, const double *x, double *y) {
  const dense_ctx *d = c;
  for (int i = 0; i < d->n; ++i) {
    double acc = 0.0;
    for (int j = 0; j < d->n; ++j)
      if (d->A[i * d->n + j] != 0.0) acc += d->A[i * d->n + j] * x[j];
    y[i] = acc;
  }
}
static void dn_M(const void *c, const double *x, double *y) {
  const dense_ctx *d = c;
  for (int i = 0; i < d->n; ++i) y[i] = d->jacobi ? x[i] * (1.0 / d->A[i * d->n + i]) : x[i];
}
double orc_estimate_dense(int n, const double *A, int jacobi, int mode) {
  dense_ctx c = {n, A, jacobi};
  double *b = malloc(sizeof(double) * n);
  orc_fill_random(n, 0x5eedbeefULL, b);
  double lo, hi;
  orc_estimate_generic(n, dn_A, dn_M, &c, b, mode, &lo, &hi);
  free(b);
  return hi / 1.1;
}

/* solve_fixed Chebyshev branch, solver.cpp:79-110 (+ JacobiPC::apply) */
static void smooth(const orc_level *L, int m, const double *b, double *x) {
  const int64_t n = L->nv;
  double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
  double *d = malloc(sizeof(double) * n), *ad = malloc(sizeof(double) * n);
  const double theta = 0.5 * (L->hi + L->lo);
  const double delta = 0.5 * (L->hi - L->lo);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  level_apply(L, x, r);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  jacobi(L, r, z);
  const double s = 1.0 / theta;
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) d[i] = z[i] * s;
  for (int it = 0; it < m; ++it) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) x[i] += 1.0 * d[i];
    if (it + 1 == m) break;
    level_apply(L, d, ad);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) r[i] += -1.0 * ad[i];
    jacobi(L, r, z);
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    const double c1 = rho_new * rho, c2 = 2.0 * rho_new / delta;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) d[i] = c1 * d[i] + c2 * z[i];
    rho = rho_new;
  }
  free(r); free(z); free(d); free(ad);
}

/* R = 2^-3 P^T, P from grid.cpp:373-428; transpose columns ascending (1 rank). */
static void restrict_(const orc_level *F, const orc_level *C, const double *rf, double *bc) {
  #pragma omp parallel for schedule(static)
  for (int64_t K = 0; K < C->n[2]; ++K)
    for (int64_t J = 0; J < C->n[1]; ++J)
      for (int64_t I = 0; I < C->n[0]; ++I) {
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
              acc += w * rf[i + F->n[0] * (j + F->n[1] * k)];
            }
          }
        }
        bc[I + C->n[0] * (J + C->n[1] * K)] = 0.125 * acc;
      }
}

/* y = P xc (grid.cpp:396-425 weights, columns ascending) then axpy(1, y, xf) */
static void prolong_add(const orc_level *F, const orc_level *C, const double *xc, double *xf) {
  #pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < F->n[2]; ++k)
    for (int64_t j = 0; j < F->n[1]; ++j)
      for (int64_t i = 0; i < F->n[0]; ++i) {
        int64_t at[3][2];
        double w[3][2];
        int cnt[3];
        const int64_t f[3] = {i, j, k};
        for (int a = 0; a < 3; ++a) {
          if (f[a] % 2 == 0) {
            at[a][0] = f[a] / 2; w[a][0] = 1.0; cnt[a] = 1;
          } else {
            at[a][0] = (f[a] - 1) / 2; at[a][1] = (f[a] + 1) / 2;
            w[a][0] = 0.5; w[a][1] = 0.5; cnt[a] = 2;
          }
        }
        double acc = 0.0;
        for (int tz = 0; tz < cnt[2]; ++tz)
          for (int ty = 0; ty < cnt[1]; ++ty)
            for (int tx = 0; tx < cnt[0]; ++tx) {
              const double ww = w[0][tx] * w[1][ty] * w[2][tz];
              acc += ww * xc[at[0][tx] + C->n[0] * (at[1][ty] + C->n[1] * at[2][tz])];
            }
        const int64_t v = i + F->n[0] * (j + F->n[1] * k);
        xf[v] += 1.0 * acc;
      }
}

static void lu_factor(orc_mg *mg) {
  const orc_level *L = &mg->lev[0];
  const int64_t n = L->nv;
  mg->nc = n;
  mg->lu = calloc((size_t)(n * n), sizeof(double));
  mg->piv = malloc(sizeof(int64_t) * n);
  /* assemble the 1-rank CSR rows densely (values identical to level_apply) */
  double *e = calloc(n, sizeof(double)), *col = malloc(sizeof(double) * n);
  for (int64_t c = 0; c < n; ++c) {
    e[c] = 1.0;
    level_apply(L, e, col);
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

/* precond.cpp:50-66 */
void orc_coarse_solve(const orc_mg *mg, const double *b, double *x) {
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

static void zero_boundary(const orc_level *L, double *v) {
  for (int64_t k = 0; k < L->n[2]; ++k)
    for (int64_t j = 0; j < L->n[1]; ++j)
      for (int64_t i = 0; i < L->n[0]; ++i)
        if (is_bnd(L, i, j, k)) v[i + L->n[0] * (j + L->n[1] * k)] = 0.0;
}

/* V-cycle; x is overwritten (starts from 0). */
void orc_vcycle(const orc_mg *mg, int level, const double *b, double *x) {
  const orc_level *L = &mg->lev[level];
  memset(x, 0, sizeof(double) * L->nv);
  if (level == 0) {
    orc_coarse_solve(mg, b, x);
    return;
  }
  const orc_level *C = &mg->lev[level - 1];
  smooth(L, mg->cfg.smooth_its, b, x);
  double *r = malloc(sizeof(double) * L->nv);
  level_apply(L, x, r);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < L->nv; ++i) r[i] = b[i] - r[i];
  double *bc = malloc(sizeof(double) * C->nv), *xc = malloc(sizeof(double) * C->nv);
  restrict_(L, C, r, bc);
  if (mg->cfg.zero_coarse_bc) zero_boundary(C, bc);
  orc_vcycle(mg, level - 1, bc, xc);
  prolong_add(L, C, xc, x);
  smooth(L, mg->cfg.smooth_its, b, x);
  free(r); free(bc); free(xc);
}

orc_mg *orc_mg_create(const orc_mg_cfg *cfg) {
  orc_mg *mg = calloc(1, sizeof *mg);
  mg->cfg = *cfg;
  mg->nl = cfg->nlevels;
  int64_t n[3] = {cfg->np[0], cfg->np[1], cfg->np[2]};
  for (int l = mg->nl - 1; l >= 0; --l) {
    orc_level *L = &mg->lev[l];
    memcpy(L->n, n, sizeof n);
    level_build(cfg, L);
    if (cfg->galerkin && l < mg->nl - 1) galerkin_build(&mg->lev[l + 1], L);
    if (l > 0) {
      for (int a = 0; a < 3; ++a) {
        if (n[a] < 3 || n[a] % 2 == 0) { orc_mg_destroy(mg); return NULL; }
        n[a] = (n[a] + 1) / 2;
      }
      orc_estimate(mg, l, cfg->est_mode, &L->lo, &L->hi);
    }
  }
  lu_factor(mg);
  return mg;
}

void orc_mg_destroy(orc_mg *mg) {
  if (!mg) return;
  for (int l = 0; l < mg->nl; ++l) {
    orc_level *L = &mg->lev[l];
    free(L->k); free(L->cxp); free(L->cyp); free(L->czp); free(L->diag); free(L->inv_diag); free(L->S);
  }
  free(mg->lu); free(mg->piv);
  free(mg);
}

int64_t orc_mg_level_n(const orc_mg *mg, int level, int64_t np_out[3]) {
  if (np_out) memcpy(np_out, mg->lev[level].n, sizeof(int64_t) * 3);
  return mg->lev[level].nv;
}

void orc_mg_bounds(const orc_mg *mg, int level, double *lo, double *hi) {
  *lo = mg->lev[level].lo;
  *hi = mg->lev[level].hi;
}

void orc_mg_coeff(const orc_mg *mg, int level, double *k_out) {
  memcpy(k_out, mg->lev[level].k, sizeof(double) * mg->lev[level].nv);
}

void orc_rhs(const int64_t np[3], uint64_t seed, double *b) {
  #pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < np[2]; ++k)
    for (int64_t j = 0; j < np[1]; ++j)
      for (int64_t i = 0; i < np[0]; ++i) {
        const int64_t v = i + np[0] * (j + np[1] * k);
        const int bnd = i == 0 || j == 0 || k == 0 || i == np[0] - 1 || j == np[1] - 1 || k == np[2] - 1;
        b[v] = bnd ? 0.0 : 2.0 * orc_hashed_uniform(seed, (uint64_t)v) - 1.0;
      }
}

void orc_apply(const orc_mg *mg, int level, const double *x, double *y) { level_apply(&mg->lev[level], x, y); }
void orc_jacobi(const orc_mg *mg, int level, const double *x, double *y) { jacobi(&mg->lev[level], x, y); }
void orc_smooth(const orc_mg *mg, int level, const double *b, double *x) {
  smooth(&mg->lev[level], mg->cfg.smooth_its, b, x);
}
void orc_restrict(const orc_mg *mg, int fine_level, const double *rf, double *bc) {
  restrict_(&mg->lev[fine_level], &mg->lev[fine_level - 1], rf, bc);
}
void orc_prolong_add(const orc_mg *mg, int fine_level, const double *xc, double *xf) {
  prolong_add(&mg->lev[fine_level], &mg->lev[fine_level - 1], xc, xf);
}

/* solver.cpp:214-266 with PcApply = one V-cycle (no null space) */
int orc_mgcg_solve(const orc_mg *mg, const double *b, double *x, double rtol, double atol, int max_its,
                   double *history, orc_report *rep) {
  const int top = mg->nl - 1;
  const orc_level *L = &mg->lev[top];
  const int64_t n = L->nv;
  double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
  double *p = malloc(sizeof(double) * n), *w = malloc(sizeof(double) * n);
  memset(rep, 0, sizeof *rep);
  level_apply(L, x, r);
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  orc_vcycle(mg, top, r, z);
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
    level_apply(L, p, w);
    const double pw = orc_dot(n, p, w);
    if (pw <= 0.0 || !isfinite(pw)) { rep->reason = 4; goto done; }
    const double alpha = rz / pw;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) r[i] += -alpha * w[i];
    orc_vcycle(mg, top, r, z);
    const double rz_new = orc_dot(n, r, z);
    nrm = sqrt(orc_dot(n, z, z));
    rep->iterations = it;
    rep->norm_final = nrm;
    if (history) history[it] = nrm;
    if (nrm <= tol) { rep->reason = nrm <= atol ? 1 : 0; goto done; }
    if (rz == 0.0 || !isfinite(rz_new)) { rep->reason = 4; goto done; }
    const double beta = rz_new / rz;
    rz = rz_new;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  rep->reason = 2;
done:
  free(r); free(z); free(p); free(w);
  return rep->reason;
}
