// Q1 elasticity MG-CG host engine (see tmgx_elast.cu).
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "tmgx_engine.hpp"

namespace tmgx {

void q1_kref(double nu, double* K);  // 24x24 reference stiffness, E = 1, unit cube

// One node of the elasticity V-cycle: the same node list as the scalar path (build_node_specs:
// SMOOTH levels on the world's boxes, TELESCOPE nodes at each stage level, the members' inner
// levels, COARSE LU on one rank). A 3-dof vector is, per local box, three consecutive component
// planes of the padded box layout (component c at p + c * total).
struct ElNode {
  NodeKind kind = SMOOTH;
  int level = 0;
  std::shared_ptr<Dist> dist;
  double h = 0.0;
  std::vector<double*> E, binv;  // per local box: element moduli (ring filled), 9 inverse-block planes
  Field b, x, r, z, d, ad;       // per local box: 3 * total doubles
  RegionPlan halo, gather, scatter;
  double lo = 0.1, hi = 1.1;
  int nc = 0;  // COARSE: dense LU
  double* A_dev = nullptr;
  long long *piv_dev = nullptr, *map_dev = nullptr;
  long long n_global() const {
    const auto& n = dist->h.npoints;
    return 3LL * n[0] * n[1] * n[2];
  }
};

class ElastSolver {
 public:
  // bounds: optional [2 * nlevels] Chebyshev intervals (lo, hi) per level; tele: telescope stages
  ElastSolver(World& W, const int64_t np[3], const MGDesc& M, uint64_t seed_e, double nu);
  ~ElastSolver();
  ElastSolver(const ElastSolver&) = delete;
  ElastSolver& operator=(const ElastSolver&) = delete;

  World& W;
  MGDesc mgd;
  DeviceArena arena;
  std::vector<ElNode> nodes;  // nodes[0] = finest (outer), back() = COARSE
  int m = 2;
  Field cx, cr, cz, cp, cw;  // CG on the top distribution (nodes[0].b = cr, nodes[0].x = cz)
  double *dot_part = nullptr, *staging = nullptr;
  double* rank_sums = nullptr;  // [R]; P > 1: the head of this process's IPC mailbox
  double* host_sums = nullptr;  // pinned [R]
  std::vector<double*> peer_mail;
  long long rs_last_bar = -1;
  long long launches = 0;
  bool est_lanczos = true;

  int node_for_level(int level) const;  // the innermost node of `level`
  int nlevels() const { return mgd.nlevels; }

  void halo(int i, const Field& f);
  void apply(int i, const Field& x, const Field& y);
  void residual(int i, const Field& b, const Field& x, const Field& r);
  void jacobi(int i, const Field& x, const Field& y);
  void vec(int i, int op, double s, double t, const Field& x, const Field& y);
  void zero(int i, const Field& f);
  double dot(int i, const Field& a, const Field& b);
  void smooth(int i, const Field& b, const Field& x);
  void vcycle(int i);  // nodes[i].b -> nodes[i].x
  void coarse_solve(int i);
  // host vectors: the level's global natural vertex order, 3 interleaved dofs; only this
  // process's boxes are read / written
  void upload(int i, const double* src, const Field& f);
  void download(int i, const Field& f, double* dst);
  int solve(const double* b, double* x, double rtol, double atol, int max_its, bool x0_nonzero, double* hist,
            int* reason, int* its, double* n0, double* nf, double* t_ms);
  std::pair<double, double> estimate(int i);
  Field comp(int i, const Field& f, int c) const;  // component-c view of a 3-dof field

 private:
  Field make3(const Dist& D);
  void sync();
};

}  // namespace tmgx
