// sm_100a kernels for the MG-CG hot path (declarations of the host launchers).
//
// Data layout in HBM: every reference rank's box of a level is stored as a
// padded array with a one-vertex ghost ring on every side; element (i,j,k) of the box
// (i-fastest, i in [-1, ex]) lives at base + i + px*j + pxy*k. base puts i = 0 on a 32-byte
// sector boundary, px is a multiple of 4 doubles. Ghost entries carry neighbour boxes'
// values after a halo exchange; the kernels never read ghosts outside the global grid.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tmgx {

constexpr int kXO = 4;         // padding so that i = 0 is sector aligned
constexpr int kBX = 32;        // threads along x per block
#ifndef TMGX_KBY
#define TMGX_KBY 4
#endif
constexpr int kBY = TMGX_KBY;  // threads along y per block
constexpr int kZC = 16;        // z planes marched per block
constexpr int kMaxLocal = 64;  // local boxes per process

struct BoxGeo {
  int ex, ey, ez;  // extents
  int gx, gy, gz;  // global lower corner
  int Nx, Ny, Nz;  // global grid
  int zc;          // z planes marched per block (kZC on large boxes, fewer on coarse levels)
  long long px, pxy, base, total;
};

// z-chunk so that a level launches >= kMinBlocks blocks: large boxes stream 16 planes per
// block (register queue reuse), coarse boxes trade reuse for parallelism (latency-bound).
constexpr int kMinBlocks = 8 * 148;
inline int choose_zc(int ex, int ey, int ez, long long min_blocks = kMinBlocks) {
  const int bxy = ((ex + 2 * kBX - 1) / (2 * kBX)) * ((ey + kBY - 1) / kBY);  // pair tiles
  for (int zc = kZC; zc > 1; zc >>= 1)
    if ((long long)bxy * ((ez + zc - 1) / zc) >= min_blocks) return zc;
  return 1;
}

// Operator parameters for the 7-point FD operator of one level.
struct OpParams {
  double ih2x, ih2y, ih2z;  // 1/h^2 per axis (grid.cpp:144-151 spacing)
  double cdiag;             // constant-coefficient diagonal (sum of the six face terms)
  double cinvd;             // 1.0 / cdiag (precond.cpp:179)
  const double* k;          // vertex coefficient (padded layout, ghosts filled); nullptr = k == 1
  const double* S;          // Galerkin level: 27 row-coefficient planes (slot s at S + s*S_stride)
  long long S_stride;
  // performance build, single box covering the grid: read the 13 upper slots as the mirrored
  // lower slots of the neighbour's row (14 planes from HBM; tmgx_kernels.cu row27)
  int sym27;
  // Variable k, precomputed rows: planes D (diagonal), FX, FY, FZ (+x/+y/+z face terms
  // harm(k_v, k_nb)/h^2) at fc + {0,1,2,3}*fc_stride; the -x/-y/-z faces are the neighbours'
  // +faces. Same values as evaluating from k, without the six divisions per row.
  const double* fc;
  long long fc_stride;
};

struct Sphere {
  double cx, cy, cz, r;
};

struct ChebStep {
  double c1, c2;  // d_new = c1*d + c2*z  (solver.cpp:106-108)
};

// Region-copy descriptor: a 3D sub-box copied between two padded arrays or a packed buffer.
struct CopyDesc {
  int src_slot, dst_slot;     // index into the pointer tables (-1 = packed buffer)
  long long src_off, dst_off; // element offset of the region origin (or buffer offset)
  int nx, ny, nz;
  long long src_px, src_pxy, dst_px, dst_pxy;  // pitches (packed: nx, nx*ny)
  double* dst_abs;            // non-null: destination base (a peer process's mailbox segment)
};

struct PtrTable {
  double* p[kMaxLocal];
};

// ---- launchers (all asynchronous on `s`; return number of kernels launched) ----
int launch_fill_coeff(const BoxGeo& g, double* k, const Sphere* spheres_dev, int n_spheres, double k_in,
                      bool varcoef, cudaStream_t s);
// Face/diagonal planes of the variable-coefficient rows from op.k (ring filled) into fc.
int launch_fill_faces(const BoxGeo& g, const OpParams& op, double* fc, long long fc_stride, cudaStream_t s);
int launch_fill_rhs(const BoxGeo& g, double* b, unsigned long long seed, bool boundary_zero, cudaStream_t s);

// Chebyshev(Jacobi) smoother pieces (solver.cpp:79-110 + precond.cpp:183-185).
// start_zero: d = (b * invd) * s_theta ; if write_x: x = d instead.
int launch_cheb_start_zero(const BoxGeo& g, const OpParams& op, const double* b, double* d_or_x, double s_theta,
                           cudaStream_t s);
// start_res: r = b - A x ; d = (r*invd)*s_theta  (x needs halo)
int launch_cheb_start_res(const BoxGeo& g, const OpParams& op, const double* b, const double* x, double* r,
                          double* d, double s_theta, cudaStream_t s);
// step: x1 = x_in + d (x_in null -> d) ; r1 = r_in - A d ; d_new = c1 d + c2 (r1*invd);
// last: x_out = x1 + d_new only ; else x_out = x1, r_out = r1, d_new.
int launch_cheb_step(const BoxGeo& g, const OpParams& op, const double* d, const double* r_in, const double* x_in,
                     double* d_new, double* r_out, double* x_out, ChebStep c, bool last, cudaStream_t s);
// Temporally blocked m = 2 Chebyshev side (single-box levels, 7-point operator, TMA-staged):
// pre (x = 0): xout = S(b); post: xout = S(b, xin) with xin != xout.
// dpart (post only): also write block partials of b.x' and x'.x' (slots dpart, dpart + dstride,
// at most dmax blocks); *dblocks = number of partials written (0: not fused).
int launch_cheb2_tb(const BoxGeo& g, const OpParams& op, const double* b, const double* xin, double* xout,
                    double s_theta, ChebStep c, bool pre, cudaStream_t s, double* dpart = nullptr,
                    long long dstride = 0, int dmax = 0, int* dblocks = nullptr);
bool cheb2_tb_supported(const BoxGeo& g);
// Temporally blocked m = 3 Chebyshev side (same contract; c = first step, c2 = second step).
int launch_cheb3_tb(const BoxGeo& g, const OpParams& op, const double* b, const double* xin, double* xout,
                    double s_theta, ChebStep c, ChebStep c2, bool pre, cudaStream_t s, double* dpart = nullptr,
                    long long dstride = 0, int dmax = 0, int* dblocks = nullptr);
bool cheb3_tb_supported(const BoxGeo& g);
// xo = xf + P xc (out of place)
int launch_prolong_to(const BoxGeo& fine, const BoxGeo& coarse, const double* xc, const double* xf, double* xo,
                      cudaStream_t s);
int launch_residual(const BoxGeo& g, const OpParams& op, const double* b, const double* x, double* r,
                    cudaStream_t s);
int launch_apply(const BoxGeo& g, const OpParams& op, const double* x, double* y, cudaStream_t s);
// Single-box levels, 7-point rows: bc = 2^-3 P^T (b - A x) with the residual kept on chip.
bool resid_restrict_supported(const OpParams& op);
// Performance build: the same with a separable restriction (lane shuffle in x, one shared plane
// in y, register accumulator in z); single box covering an odd-sized grid.
bool resid_restrict2_supported(const BoxGeo& fine, const OpParams& op, const BoxGeo& coarse);
int launch_resid_restrict2(const BoxGeo& fine, const OpParams& op, const BoxGeo& coarse, const double* b,
                           const double* x, double* bc, cudaStream_t s);
int launch_resid_restrict(const BoxGeo& fine, const OpParams& op, const BoxGeo& coarse, const double* b,
                          const double* x, double* bc, cudaStream_t s);
// bc = 2^-3 P^T rf over the coarse box (rf needs a box halo incl. corners).
int launch_restrict(const BoxGeo& fine, const BoxGeo& coarse, const double* rf, double* bc, cudaStream_t s);
// bc = scale P^T rf (scale 1: finite-element restriction of the elasticity path)
int launch_restrict_scaled(const BoxGeo& fine, const BoxGeo& coarse, const double* rf, double* bc, double scale,
                           cudaStream_t s);
// xf += P xc (xc needs a box halo incl. corners).
int launch_prolong_add(const BoxGeo& fine, const BoxGeo& coarse, const double* xc, double* xf, cudaStream_t s);

// Galerkin coarse operator (ptap, dist_matrix.cpp:462-468; R = 2^-3 P^T): 27-point rows of the
// coarse box from the fine operator `fop` (7-point from k/constants, or 27-point planes with a
// filled halo). Output planes Sc + s*c_stride.
int launch_galerkin(const BoxGeo& fine, const OpParams& fop, const BoxGeo& coarse, double* Sc, long long c_stride,
                    const Sphere* sph, int n_spheres, double k_in, cudaStream_t s);

// CG / estimator pieces; partials: per-block fp64 partial sums (deterministic tree).
int grid_blocks(const BoxGeo& g);
int launch_spmv_dot(const BoxGeo& g, const OpParams& op, const double* p, double* w, double* part,
                    cudaStream_t s);
bool pspmv_supported(const OpParams& op);
// p_new = z + beta p_old ; w = A p_new ; part = block partials of p_new.w (beta = scal[beta_slot])
int launch_pspmv_dot(const BoxGeo& g, const OpParams& op, const double* z, const double* p_old, double* p_new,
                     double* w, double* part, const double* scal, int beta_slot, cudaStream_t s);
int launch_dot2(const BoxGeo& g, const double* a, const double* b, const double* c, double* part_ab,
                double* part_cc, cudaStream_t s);  // a.b and c.c
int launch_jacobi_dot(const BoxGeo& g, const OpParams& op, const double* r, double* z, double* part,
                      cudaStream_t s);  // z = r*invd, part = r.z
// x += alpha p ; r += (-alpha) w ; alpha = scal[alpha_slot]; skipped when scal[flag_slot] != 0.
int launch_cg_update(const BoxGeo& g, const double* p, const double* w, double* x, double* r, const double* scal,
                     int alpha_slot, int flag_slot, cudaStream_t s);
// p = z + beta p ; beta = scal[beta_slot]
int launch_p_update(const BoxGeo& g, const double* z, double* p, const double* scal, int beta_slot, cudaStream_t s);
int launch_copy_interior(const BoxGeo& g, const double* src, double* dst, cudaStream_t s);
int launch_axpy(const BoxGeo& g, double alpha, const double* x, double* y, cudaStream_t s);  // y += alpha x
int launch_zero(double* p, long long n, cudaStream_t s);
// Sum `nblk` partials of each of `nslots` slots (stride `slot_stride`) into out[slot*out_stride].
int launch_reduce_partials(const double* part, int nblk, int nslots, long long slot_stride, double* out,
                           long long out_stride, cudaStream_t s);

// Parity build only: serial left fold of a.b (and c.c when c != null) in local order into
// out[0] (and out[out_stride]) -- the reference's ordered_fold_sum on one rank.
int launch_fold_dot(const BoxGeo& g, const double* a, const double* b, const double* c, double* out,
                    long long out_stride, cudaStream_t s);

// Scalar finalisation. rank_sums[slot*R + rank]; sums over the listed ranks in order.
enum ScalSlot {
  S_RZ = 0, S_PW, S_ALPHA, S_BETA, S_RZNEW, S_ZZ, S_NRM, S_FLAG_PW, S_FLAG_RZ, S_RZOLD, S_TMP0, S_TMP1,
  S_NSLOTS = 16
};
enum CgOp { CG_INIT = 0, CG_ALPHA = 1, CG_BETA = 2, SUM2 = 3 };
int launch_cg_scalars(int op, const double* rank_sums, int R, const int* ranks_dev, int nranks, double* scal,
                      cudaStream_t s);

// Compact (rank-block local order) <-> padded box.
int launch_box_to_compact(const BoxGeo& g, const double* box, double* compact, cudaStream_t s);
int launch_compact_to_box(const BoxGeo& g, const double* compact, double* box, cudaStream_t s);

// Region copies (halo exchange, telescope gather/scatter, pack/unpack).
int launch_region_copy(const CopyDesc* desc_dev, int ndesc, int max_elems, const PtrTable& src,
                       const PtrTable& dst, double* src_buf, double* dst_buf, cudaStream_t s);

// Cross-process scalar reduction: store this process's rank slots [first, end) of `nslots`
// slots (stride R) into every peer's rank_sums (peers.p[0..npeers)).
int launch_push_ranksums(const double* rs, int R, int nslots, int first, int end, const PtrTable& peers, int npeers,
                         cudaStream_t s);

// Coarse direct solve: perf build y = Ainv x ; parity build: DenseLU::solve loop order.
// `map[c]` = padded-box element offset of compact (natural) index c.
int launch_dense_matvec(const double* A, int n, const long long* map, const double* x, double* y, cudaStream_t s);
int launch_lu_solve(const double* lu, const long long* piv, int n, const long long* map, const double* b,
                    double* x, cudaStream_t s);

// Fused coarse V-cycle: every single-box level from L[0] (finest of the group) down to the coarse
// LU, run by one thread-block cluster with cluster barriers between dependent phases instead of
// one kernel launch per phase (levels <= 33^3 are launch-latency bound). Same arithmetic as the
// per-phase kernels (bitwise identical in both builds).
constexpr int kCCMaxLev = 6, kCCMaxM = 6;
struct CCLevel {
  BoxGeo g;
  OpParams op;
  double *b, *x, *r, *d, *d2;
  double s_theta;
  ChebStep cs[kCCMaxM];  // Chebyshev pass coefficients (solver.cpp:90-93, 106-108)
};
struct CCParams {
  int nlev;               // smoothing levels; L[nlev] is the coarse (LU) level (g, b, x only)
  int m;                  // smoothing passes per side
  CCLevel L[kCCMaxLev + 1];
  const double* A;        // Ainv (perf) or LU factors (parity)
  const long long* piv;
  const long long* map;
  int nc;
};
bool coarse_cycle_supported(int nc);
int launch_coarse_cycle(const CCParams& p, cudaStream_t s);

bool parity_build();

}  // namespace tmgx
