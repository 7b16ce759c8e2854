/* tmgx — B200-native MG-preconditioned CG with coarse-level telescoping.
 *
 * C-ABI drop-in boundary for the reference's hot path (arxiv 1604.07163 re-creation,
 * /root/reference/proj/core). Plain pointers and sizes only; no torch or C++ types.
 * Each entry point cites the reference interface it replaces. The C++ host layer
 * (paper_1604_07163_b200/csrc/) sits behind these functions; INTEGRATION.md shows the
 * binding a reference maintainer would add.
 *
 * Process model: spawn_world (comm.hpp:176-207) ran R rank threads in one process.
 * Here R reference ranks (grid boxes) are spread over P processes of one node, one GPU
 * each in production (P == R: one box per GPU; several processes may also share a GPU).
 * Processes exchange data by storing into each other's CUDA-IPC-mapped mailboxes (peer
 * memory over NVLink / NVSwitch) and synchronise through stream-ordered host barriers on
 * a shared-memory segment named by the job token. P == 1 runs all R boxes on one GPU.
 * Every call below that the reference made collectively is collective over the P processes.
 *
 * Status codes: 0 ok, 1 configuration error (tmg::ConfigError),
 * 2 diverged (SolveReport reason), 3 CUDA / transport error, 4 internal/usage error (tmg::Error).
 * tmgx_last_error() returns the message of the last failure on the calling thread.
 */
#ifndef TMGX_H
#define TMGX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMGX_OK 0
#define TMGX_ERR_CONFIG 1
#define TMGX_DIVERGED 2
#define TMGX_ERR_CUDA 3
#define TMGX_ERR_INTERNAL 4

#define TMGX_MAX_AXIS_PARTS 64
#define TMGX_MAX_TELESCOPE 4
#define TMGX_JOB_TOKEN_BYTES 33

/* GridHeader (grid.hpp:41-79): rank-independent grid description. */
typedef struct {
  int dim;
  int64_t np[3];
  int dof;
  int pg[3];
  int64_t off[3][TMGX_MAX_AXIS_PARTS + 1];
} tmgx_header;

/* ---------------------------------------------------------------------------
 * Index maps — host-only, bit-exact restatements of grid.cpp / comm.cpp / layout.cpp.
 * ------------------------------------------------------------------------- */

/* choose_proc_grid (grid.cpp:209-240). Returns 1 (ConfigError) if over-decomposed. */
int tmgx_choose_proc_grid(int size, int dim, const int64_t np[3], int pg_out[3]);
/* create_grid header (grid.cpp:256-292); hint may be NULL. */
int tmgx_grid_header(int size, int dim, const int64_t np[3], int dof, const int *hint, tmgx_header *out);
/* coarsen (grid.cpp:299-368). Returns 1 "cannot coarsen". */
int tmgx_coarsen_header(const tmgx_header *fine, tmgx_header *coarse);
/* Layout of the rank-block ordering (grid.cpp:40-46): offsets[n_ranks+1]. */
int tmgx_layout_offsets(const tmgx_header *h, int64_t *offsets);
/* NaturalOrdering bijection (grid.cpp:48-115). */
int64_t tmgx_global_to_natural(const tmgx_header *h, int64_t global);
int64_t tmgx_natural_to_global(const tmgx_header *h, int64_t natural);
/* Comm::split_strided (comm.cpp:353-390): member_map gets ceil(n/r) entries. */
int tmgx_split_strided(int n, int r, int *member_map, int *n_members);
/* repartition_onto header (grid.cpp:433-493); override_[a] == 0 means "not set". */
int tmgx_repartition_header(const tmgx_header *h, int sub_size, const int override_[3], tmgx_header *out);
/* prefusion_layout (grid.cpp:566-580): offsets[parent_size+1]. */
int tmgx_prefusion_layout(const tmgx_header *new_h, int parent_size, const int *member_map, int n_members,
                          int64_t *offsets);
/* build_permutation (grid.cpp:582-599): for old-layout rows [row_begin,row_end) the column
 * of the single 1 of P-hat. */
int tmgx_permutation(const tmgx_header *old_h, const tmgx_header *new_h, int64_t row_begin, int64_t row_end,
                     int64_t *cols);

/* ---------------------------------------------------------------------------
 * World (spawn_world analog) and solver.
 * ------------------------------------------------------------------------- */
typedef struct tmgx_world_s *tmgx_world;
typedef struct tmgx_solver_s *tmgx_solver;

/* Writes a fresh random job token (32 hex chars + NUL; call on one process and hand the string
 * to the others, e.g. through the launcher's environment or an MPI/torch broadcast). */
int tmgx_job_token(char *out /* TMGX_JOB_TOKEN_BYTES */);
/* spawn_world (comm.hpp:176-207): n_ranks reference ranks over nproc processes of one node;
 * process `proc` owns ranks [proc*n_ranks/nproc, (proc+1)*n_ranks/nproc) and drives CUDA
 * device `device`. job: the node-local rendezvous name shared by the nproc processes (ignored
 * when nproc == 1). Collective over the processes. */
int tmgx_world_create(int n_ranks, int nproc, int proc, int device, const char *job, tmgx_world *out);
int tmgx_world_destroy(tmgx_world w);
/* First and one-past-last reference rank owned by this process. */
int tmgx_world_local_ranks(tmgx_world w, int *first, int *end);

enum { TMGX_POISSON7 = 0, TMGX_VARCOEF7_HARMONIC = 1 };
enum { TMGX_EST_REFERENCE = 0, TMGX_EST_LANCZOS = 1 };
enum { TMGX_KSP_CG = 2, TMGX_KSP_PREONLY = 5 }; /* KrylovMethod (solver.hpp:19) */
enum { TMGX_RTOL = 0, TMGX_ATOL = 1, TMGX_MAX_ITS = 2, TMGX_FIXED_ITS_DONE = 3, TMGX_REASON_DIVERGED = 4 };

/* assemble_problem (reference problems.cpp is missing): 7-point FD operator
 * on the unit cube, homogeneous Dirichlet rows, constant k or k from seeded spheres with
 * harmonic face averages. */
typedef struct {
  int kind;
  int64_t np[3];
  int pg_hint[3];      /* all 0 = balanced choice (grid.cpp:209-240) */
  uint64_t seed_k;     /* spheres */
  int n_spheres;       /* 32 */
  double k_in;         /* 1e4 */
} tmgx_problem;

/* Telescope stage: the MG level at which the communicator is coarsened by
 * reduction_factor, with optional repart_da_processors_{x,y,z} override (0 = not set). */
typedef struct {
  int level;
  int reduction_factor;
  int override_[3];
} tmgx_telescope_stage;

/* MG hierarchy: nlevels total (N1+N2-1 when telescoped),
 * Chebyshev(Jacobi) V(m,m) smoothing, LU at level 0 on a single rank. */
typedef struct {
  int nlevels;
  int smooth_its;
  int est_mode;
  const double *cheb_bounds; /* optional: [2*nlevels] (lo,hi) per level; NULL = estimate (solver.cpp:591) */
  int n_telescope;
  tmgx_telescope_stage telescope[TMGX_MAX_TELESCOPE];
  int galerkin; /* -pc_mg_galerkin: levels below the finest are 2^-3 P^T A P (27-point), else rediscretised */
} tmgx_mg_cfg;

/* KrylovConfig (solver.hpp:27-37) subset on this path. */
typedef struct {
  int method;  /* TMGX_KSP_CG or TMGX_KSP_PREONLY */
  double rtol;
  double atol;
  int max_its;
  int zero_initial_guess; /* 1: x is output only (PETSc's default, x0 = 0 without reading x);
                             0: x is the initial guess (the reference's krylov_solve) */
} tmgx_ksp_cfg;

/* SolveReport (solver.hpp:39-52) + timings. */
typedef struct {
  int reason;
  int iterations;
  double norm0;
  double norm_final;
  double t_solve_s;       /* device time of the solve (CUDA events) */
  int64_t kernel_launches; /* kernels launched by the solve */
} tmgx_report;

/* SolverNode::create + mg_setup + TelescopePC setup (collective). */
int tmgx_solver_create(tmgx_world w, const tmgx_problem *prob, const tmgx_mg_cfg *mg, tmgx_solver *out);
int tmgx_solver_destroy(tmgx_solver s);

/* Number of levels, the header of level `level` as seen by the outer hierarchy when
 * level >= first telescope level else by the innermost containing stage; this process's
 * local unknown count at that level (0 on idle non-members). */
int tmgx_solver_level_info(tmgx_solver s, int level, tmgx_header *h, int64_t *n_local);
/* Chebyshev interval used on `level` (after estimation). */
int tmgx_solver_bounds(tmgx_solver s, int level, double *lo, double *hi);
/* Fine-level right-hand side f = 2u-1 keyed by natural index, 0 on Dirichlet vertices,
 * written into this process's local slice (host pointer). */
int tmgx_fill_rhs(tmgx_solver s, uint64_t seed, double *b_local);

/* krylov_solve (solver.cpp:420-480) with the MG preconditioner. b/x are this process's
 * slice of the rank-block ordering (DistVector local order, grid.cpp:61-82), host or
 * device memory as flagged. history: room for max_its+1 norms, or NULL. Returns 0, or 2
 * on divergence (report filled either way).
 * Stream contract: the library works on its own non-blocking stream. Device-resident b / x are
 * read only after all work previously submitted to the legacy default stream (e.g. torch's
 * default stream) has completed; work on any other caller stream must be synchronised by the
 * caller first. The call returns after x is written (host-synchronous). */
int tmgx_solve(tmgx_solver s, const double *b, double *x, int on_device, const tmgx_ksp_cfg *cfg,
               double *history, tmgx_report *rep);
/* Same, with the right-hand side generated on the device from `seed` (inputs resident). */
int tmgx_solve_seeded(tmgx_solver s, uint64_t seed, double *x_dev_or_null, const tmgx_ksp_cfg *cfg,
                      double *history, tmgx_report *rep);

/* Preconditioner::apply (preconditioner.hpp:17-32): y = one V-cycle applied to x. */
int tmgx_pc_apply(tmgx_solver s, const double *x, double *y);

/* Level primitives for parity tests (host arrays in the level's local order). */
int tmgx_level_apply(tmgx_solver s, int level, const double *x, double *y);  /* spmv */
int tmgx_level_smooth(tmgx_solver s, int level, const double *b, double *x); /* solve_fixed, x in/out */
int tmgx_level_residual_restrict(tmgx_solver s, int fine_level, const double *b, const double *x,
                                 double *bc);                                 /* 2^-3 P^T (b - A x) */
int tmgx_level_prolong_add(tmgx_solver s, int fine_level, const double *xc, double *xf);
int tmgx_coarse_solve(tmgx_solver s, const double *b, double *x);            /* DenseLU::solve */
/* Telescope data movement at stage t: gather (P-hat^T x then ScatterPlan::to_sub) of a
 * parent-layout vector onto the members, and the reverse. Host arrays, local order. */
int tmgx_telescope_gather(tmgx_solver s, int stage, const double *x_parent, double *x_sub);
int tmgx_telescope_scatter(tmgx_solver s, int stage, const double *y_sub, double *y_parent);

/* Options database + solver-tree builder (the reference's missing options.cpp /
 * solver_build.cpp): PETSc-style prefixed keys drive the GPU hierarchy, e.g.
 * the paper's boxes "-pc_type mg -pc_mg_levels N1 -pc_mg_galerkin
 * -mg_coarse_pc_type telescope -mg_coarse_pc_telescope_reduction_factor r
 * -mg_coarse_telescope_pc_type mg -mg_coarse_telescope_pc_mg_levels N2 ...". String outputs
 * are NUL-terminated; a buffer that is too small is a ConfigError naming the size needed. */
typedef struct tmgx_options_s *tmgx_options;
int tmgx_options_create(tmgx_options *out);
int tmgx_options_destroy(tmgx_options o);
/* parse(argv): "-key [value]" tokens, later keys win, a "-key" followed by
 * another "-key" or the end is a flag ("true"); malformed token -> ConfigError with position. */
int tmgx_options_parse(tmgx_options o, int argc, const char *const *argv);
/* options file text: one "-key value" per line, '#' comments */
int tmgx_options_parse_file_text(tmgx_options o, const char *text);
int tmgx_options_set(tmgx_options o, const char *key, const char *value);
/* *found = 0/1; value copied into buf when found (marks the key used) */
int tmgx_options_get(tmgx_options o, const char *key, char *buf, int buflen, int *found);
/* all entries as "-key value" tokens separated by '\n' (reparses to an equal database) */
int tmgx_options_serialize(tmgx_options o, char *buf, int buflen);
/* keys never looked up, separated by '\n' (the reference warns on these at teardown) */
int tmgx_options_unused(tmgx_options o, char *buf, int buflen);
/* build_solver_tree resolved onto the GPU hierarchy without touching the GPU:
 * <prefix>ksp_type (default_ksp when unset; NULL = the reference's "gmres"), <prefix>pc_type mg,
 * MG smoother keys under <prefix>mg_levels_, coarse solver under <prefix>mg_coarse_, telescope
 * sub-solver under <prefix>mg_coarse_telescope_ (recursively). describe: the resolved tree. */
int tmgx_options_resolve(tmgx_options o, const char *prefix, const char *default_ksp, tmgx_mg_cfg *mg,
                         tmgx_ksp_cfg *ksp, char *describe, int describe_len);
/* resolve + tmgx_solver_create; *ksp receives the outer KSP for tmgx_solve */
int tmgx_solver_from_options(tmgx_world w, const tmgx_problem *prob, tmgx_options o, const char *prefix,
                             const char *default_ksp, tmgx_solver *out, tmgx_ksp_cfg *ksp);

/* Q1 hexahedral linear elasticity MG-CG (BASELINE configs[4]; no reference implementation,
 * discretisation defined in tmgx_elast.cu / oracle/tmg_elast_oracle.c): N^3 vertices x 3 dofs,
 * E_e = 10^(3 u(seed_e, e)) per element, nu, clamped x = 0 face, body force (0, 0, -1),
 * point-block Jacobi Chebyshev V(m,m), rediscretised coarse levels, LU on level 0. The levels
 * are split into the world's boxes exactly like the scalar path (GridHeader of R ranks over P
 * processes, box halos, rank-ordered dot sums) and may be telescoped onto fewer boxes
 * (tmgx_elast_create_mg; cfg5: 8 boxes, reduction factor 8 at level 3). Vectors: the level's
 * global natural vertex order, 3 interleaved dofs (host or device memory); each process reads
 * and writes the entries of its own boxes. Collective over the processes. */
typedef struct tmgx_elast_s *tmgx_elast;
int tmgx_elast_create(tmgx_world w, const int64_t np[3], int nlevels, int smooth_its, int est_mode, uint64_t seed_e,
                      double nu, tmgx_elast *out);
/* Same with the full MG description: nlevels, smooth_its, est_mode, optional cheb_bounds
 * [2*nlevels], telescope stages (TelescopePC); galerkin must be 0. */
int tmgx_elast_create_mg(tmgx_world w, const int64_t np[3], const tmgx_mg_cfg *mg, uint64_t seed_e, double nu,
                         tmgx_elast *out);
int tmgx_elast_destroy(tmgx_elast e);
int tmgx_elast_kref(double nu, double *k576);      /* 24x24 reference stiffness (E = 1, unit cube) */
int tmgx_elast_level_info(tmgx_elast e, int level, int64_t np[3], double *lo, double *hi);
int tmgx_elast_rhs(tmgx_elast e, double *b);       /* body-force load of the finest level (host) */
int tmgx_elast_level_apply(tmgx_elast e, int level, const double *x, double *y);
int tmgx_elast_level_smooth(tmgx_elast e, int level, const double *b, double *x); /* x in/out */
int tmgx_elast_pc_apply(tmgx_elast e, const double *x, double *y);                /* one V-cycle */
int tmgx_elast_solve(tmgx_elast e, const double *b, double *x, const tmgx_ksp_cfg *cfg, double *history,
                     tmgx_report *rep);
/* live timing of the finest-level operator apply (bench.py roofline): ms, algorithmic bytes
 * (x, y: 24 B each, E: 8 B per vertex) and flops (576 FMAs per vertex) per launch */
int tmgx_elast_bench_apply(tmgx_elast e, int iters, double *ms_per_launch, double *bytes_per_launch,
                           double *flops_per_launch);

/* Counters: kernel launches, halo/telescope bytes moved between processes. */
typedef struct {
  int64_t kernel_launches;
  int64_t halo_bytes_sent;
  int64_t telescope_bytes_sent;
  int64_t allreduces;
} tmgx_counters;
int tmgx_get_counters(tmgx_solver s, tmgx_counters *c);
/* Per-level V-cycle profile (the reference's per-level MsgCounters, comm.hpp:37-47, plus device
 * time): runs `reps` V-cycles with CUDA events around every node of the hierarchy and returns,
 * per node (0 = finest; kinds 0 smooth / 1 telescope / 2 coarse LU), the global grid, the number
 * of ranks of its communicator, the node's own mean device microseconds per V-cycle (its
 * coarser part excluded; a telescope node's time is its gather + scatter) and the bytes this
 * process sent to peers for it (halos, telescope transfers). Collective. */
int tmgx_level_profile(tmgx_solver s, int reps, int max_nodes, int *n_nodes, int *kind, int64_t *npoints,
                       int *n_ranks, double *us, int64_t *bytes);

/* Telescope timing in the paper's Table 1/2 schema: T_setup = host time of
 * the stage's plan construction (P-hat / ScatterPlan analogue) + upload during solver setup;
 * T_apply = device time of one gather + one scatter of the stage's level vector, averaged over
 * `reps`; bytes_per_apply = 2 x 8 x level size. */
int tmgx_telescope_timing(tmgx_solver s, int stage, int reps, double *t_setup_s, double *t_apply_s,
                          int64_t *bytes_per_apply);

/* Host-only (no GPU): the data-movement plans process `proc` of `nproc` would build for this
 * problem/hierarchy. One record of 6 int64 per (plan, peer): {plan_id (3*node + 0 halo,
 * +1 telescope gather, +2 telescope scatter), kind (0 send, 1 recv, 2 local copy), peer
 * process, vertex count, checksum of the global vertex indices moved, level}. Used by the
 * multi-process consistency tests (every send must match the peer's receive). */
int tmgx_plan_summary(int n_ranks, int nproc, int proc, const tmgx_problem *prob, const tmgx_mg_cfg *mg,
                      int64_t *records, int max_records, int *n_records);

/* Host-only (no GPU): the node-local process group the multi-process World synchronises with
 * (shared-memory barrier + allgather). Process `proc` of `nproc` joins `job`, allgathers its
 * index, then runs `rounds` barriers, each followed by a check of a shared round counter.
 * out[0] = sum of the gathered indices, out[1] = rounds completed consistently. Used by the CPU
 * multi-process transport tests. */
int tmgx_node_selftest(const char *job, int nproc, int proc, int rounds, int64_t out[2]);
/* Timing of one cross-box exchange (halo of `level`, `reps` times; collective): mean device
 * microseconds per exchange (pack + publishing barrier + unpack) and bytes moved per process. */
int tmgx_exchange_timing(tmgx_solver s, int level, int reps, double *us_per_exchange, int64_t *bytes_per_exchange);

/* Kernel micro-timing for the roofline (bench.py): launches kernel `which` on `level` `iters`
 * times back to back on the library stream between CUDA events. Outputs the mean device time
 * per launch and the algorithmic HBM bytes one launch must move (DESIGN.md §5 table).
 * which: 0 cheb_step (full: read d,r,x write d',r,x) 1 cheb_step (last: read d,r,x write x)
 *        2 operator apply 3 residual 4 restriction 5 prolongation 6 cg_update 7 spmv+dot
 *        8 temporally blocked V(2,2) pre-smooth side (b in, x out)
 *        9 temporally blocked post-smooth side (x, b in, x out)
 *       10 out-of-place prolongation x~ = x + P x_c (x, x_c in, x~ out)
 *       11 fused residual + restriction b_c = R (b - A x) (b, x in, b_c out)
 *       12 temporally blocked V(3,3) pre-smooth side (b in, x out)
 *       13 temporally blocked V(3,3) post-smooth side (x, b in, x out)
 *       14 fused CG direction update + SpMV + p.w partials (z, p in; p', w out)
 *       15 separable fused residual + restriction (performance build default; b, x in, b_c out)
 * Variable-coefficient levels count the algorithmic coefficient stream (k: 8 B per point,
 * SURVEY.md §8(d)); the kernels read the precomputed face planes (32 B per point). */
int tmgx_bench_kernel(tmgx_solver s, int which, int level, int iters, double *ms_per_launch,
                      double *bytes_per_launch);

/* 1 if built with -fmad=false (bitwise parity build), else 0. */
int tmgx_parity_build(void);
const char *tmgx_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
