/* TEST INFRASTRUCTURE ONLY — CPU oracle for the MG-CG + telescope hot path.
 *
 * Plain-C restatement of the reference algorithm (arxiv 1604.07163 "Telescope"
 * re-creation under /root/reference/proj/core). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library; the
 * product path (paper_1604_07163_b200/) never does.
 *
 * Every function cites the reference file:line it restates. Conventions that the
 * reference leaves unpinned (boundary rows, restriction scaling, seeding, sphere
 * coefficients) follow SURVEY.md Appendix A and are spelled out in DESIGN.md §3.
 *
 * Parity pin: tests/test_oracle_pins.py checks this oracle against
 *   (1) the SPEC known-answer examples the survey verified against the shipped code,
 *   (2) the survey probe golden table bit for bit, and
 *   (3) outputs of the reference's own translation units compiled by
 *       oracle/build_ref.sh into oracle/_ref/ (committed as tests/golden/ fixtures).
 */
#ifndef TMG_ORACLE_H
#define TMG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_PARTS 64

/* GridHeader (grid.hpp:41-79): dim, npoints, dof, proc grid, per-axis offsets. */
typedef struct {
  int dim;
  int64_t np[3];
  int dof;
  int pg[3];
  int64_t off[3][ORC_MAX_PARTS + 1];
} orc_header;

/* ---- common.hpp:40-53 ---- */
uint64_t orc_splitmix64(uint64_t x);
double orc_hashed_uniform(uint64_t seed, uint64_t index);

/* ---- grid maps (grid.cpp) ---- */
void orc_split_axis(int64_t n, int parts, int64_t *off);                     /* grid.cpp:184-193 */
int orc_choose_proc_grid(int size, int dim, const int64_t np[3], int pg[3]); /* grid.cpp:209-240; -1 = over-decomposed */
int orc_build_header(int size, int dim, const int64_t np[3], int dof, const int *hint, orc_header *h); /* grid.cpp:256-284 */
int orc_coarsen_header(const orc_header *fine, orc_header *coarse);          /* grid.cpp:299-322; -1 = cannot coarsen */
int64_t orc_natural_index(const orc_header *h, int64_t i, int64_t j, int64_t k, int c); /* grid.cpp:48-50 */
int64_t orc_global_index(const orc_header *h, int64_t i, int64_t j, int64_t k, int c);  /* grid.cpp:61-82 */
int64_t orc_global_to_natural(const orc_header *h, int64_t g);               /* grid.cpp:84-115 */
int64_t orc_natural_to_global(const orc_header *h, int64_t n);               /* grid.cpp:103-108 */
void orc_layout_offsets(const orc_header *h, int64_t *offsets);              /* grid.cpp:40-46 */
int orc_split_strided(int n, int r, int *member_map);                        /* comm.cpp:353-390; returns member count */
int orc_repartition(const orc_header *h, int sub_size, const int override_[3], orc_header *out); /* grid.cpp:433-493 */
void orc_prefusion_layout(const orc_header *newh, int parent_size, const int *member_map, int n_members,
                          int64_t *offsets);                                  /* grid.cpp:566-580 */
void orc_build_permutation(const orc_header *oldh, const orc_header *newh, int64_t *q); /* grid.cpp:582-599 */

/* ---- numerics (1-rank semantics, natural ordering == 1-rank rank-block ordering) ---- */
enum { ORC_POISSON7 = 0, ORC_VARCOEF7 = 1 };
enum { ORC_EST_REFERENCE = 0, ORC_EST_LANCZOS = 1 };

typedef struct orc_mg orc_mg;

typedef struct {
  int kind;            /* ORC_POISSON7 / ORC_VARCOEF7 */
  int64_t np[3];       /* finest grid */
  int nlevels;         /* >= 1; level 0 = coarsest (LU) */
  int smooth_its;      /* m of V(m,m) */
  int est_mode;        /* ORC_EST_* */
  int zero_coarse_bc;  /* 1: zero restricted RHS on coarse Dirichlet vertices */
  uint64_t seed_k;     /* sphere seed for VARCOEF7 */
  int n_spheres;       /* 32 */
  double k_in;         /* 1e4 */
  double cheb_lo_fac, cheb_hi_fac; /* 0.1, 1.1 (solver.cpp:580) */
  int galerkin;        /* 1: levels below the finest are 2^-3 P^T A P (ptap, dist_matrix.cpp:462-468) */
} orc_mg_cfg;

orc_mg *orc_mg_create(const orc_mg_cfg *cfg);
void orc_mg_destroy(orc_mg *mg);
int64_t orc_mg_level_n(const orc_mg *mg, int level, int64_t np_out[3]);
void orc_mg_bounds(const orc_mg *mg, int level, double *lo, double *hi);
void orc_mg_coeff(const orc_mg *mg, int level, double *k_out); /* vertex coefficient field */
/* 27-point row coefficients of a Galerkin level: out[s*n + v], s = (dz+1)*9+(dy+1)*3+(dx+1);
 * returns 0 if the level is not Galerkin. */
int orc_mg_stencil27(const orc_mg *mg, int level, double *out);

void orc_rhs(const int64_t np[3], uint64_t seed, double *b);        /* f = 2u-1 interior, 0 boundary */
void orc_fill_random(int64_t n, uint64_t seed, double *x);           /* dist_vector.cpp:61-65, natural key */
void orc_apply(const orc_mg *mg, int level, const double *x, double *y); /* spmv dist_matrix.cpp:182-224 */
void orc_jacobi(const orc_mg *mg, int level, const double *x, double *y); /* precond.cpp:183-185 */
void orc_smooth(const orc_mg *mg, int level, const double *b, double *x); /* solver.cpp:79-124 */
void orc_restrict(const orc_mg *mg, int fine_level, const double *rf, double *bc);
void orc_prolong_add(const orc_mg *mg, int fine_level, const double *xc, double *xf);
void orc_coarse_solve(const orc_mg *mg, const double *b, double *x); /* precond.cpp:50-66 */
void orc_vcycle(const orc_mg *mg, int level, const double *b, double *x);
int orc_estimate(const orc_mg *mg, int level, int mode, double *lo, double *hi); /* solver.cpp:520-581 */
double orc_dot(int64_t n, const double *x, const double *y);          /* dist_vector.cpp:33-38 */

typedef struct {
  int reason;        /* 0 rtol 1 atol 2 max_its 3 fixed 4 diverged (solver.hpp:24) */
  int iterations;
  double norm0;
  double norm_final;
} orc_report;

/* solve_cg (solver.cpp:214-266) preconditioned by one V-cycle; history may be NULL
 * (else room for max_its+1 entries). */
int orc_mgcg_solve(const orc_mg *mg, const double *b, double *x, double rtol, double atol, int max_its,
                   double *history, orc_report *rep);

/* Dense-matrix estimator check: diag(values) with identity or Jacobi PC. */
double orc_estimate_dense(int n, const double *A, int jacobi, int mode);

/* chebyshev_bounds_estimate (solver.cpp:520-581) on any operator / preconditioner pair */
typedef void (*orc_op_fn)(const void *ctx, const double *x, double *y);
int orc_estimate_generic(int64_t n, orc_op_fn A, orc_op_fn M, const void *ctx, const double *b0, int mode,
                         double *lo_out, double *hi_out);

/* ---- Q1 elasticity (BASELINE configs[4]; tmg_elast_oracle.c, parity unpinned by the reference) ---- */
typedef struct {
  int64_t np[3];      /* vertices per axis (2M+1) */
  int nlevels;        /* level 0 = coarsest (LU) */
  int smooth_its;     /* V(m,m) */
  int est_mode;       /* ORC_EST_* */
  uint64_t seed_e;    /* E_e = 10^(3 u(seed_e, e)) */
  double nu;          /* 0.3 */
} orc_el_cfg;
typedef struct orc_el_mg orc_el_mg;
void orc_el_kref(double nu, double *K576);
orc_el_mg *orc_el_create(const orc_el_cfg *cfg);
void orc_el_destroy(orc_el_mg *mg);
int64_t orc_el_level_nv(const orc_el_mg *mg, int level);
void orc_el_bounds(const orc_el_mg *mg, int level, double *lo, double *hi);
void orc_el_elements(const orc_el_mg *mg, int level, double *E);
void orc_el_apply(const orc_el_mg *mg, int level, const double *x, double *y);
void orc_el_jacobi(const orc_el_mg *mg, int level, const double *x, double *y);
void orc_el_smooth(const orc_el_mg *mg, int level, const double *b, double *x);
void orc_el_restrict(const orc_el_mg *mg, int fine_level, const double *rf, double *bc);
void orc_el_prolong_add(const orc_el_mg *mg, int fine_level, const double *xc, double *xf);
void orc_el_coarse_solve(const orc_el_mg *mg, const double *b, double *x);
void orc_el_vcycle(const orc_el_mg *mg, int level, const double *b, double *x);
void orc_el_rhs(const int64_t np[3], double *b);
int orc_el_solve(const orc_el_mg *mg, const double *b, double *x, double rtol, double atol, int max_its,
                 double *history, orc_report *rep);

#ifdef __cplusplus
}
#endif
#endif
