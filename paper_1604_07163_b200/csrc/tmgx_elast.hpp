// Q1 elasticity MG-CG host engine (see tmgx_elast.cu).
#pragma once

#include <utility>
#include <vector>

#include "tmgx_engine.hpp"

namespace tmgx {

void q1_kref(double nu, double* K);  // 24x24 reference stiffness, E = 1, unit cube

struct ElLevel {
  BoxGeo g;
  double h = 0.0;
  double *E = nullptr, *binv = nullptr;
  double *b = nullptr, *x = nullptr, *r = nullptr, *z = nullptr, *d = nullptr, *ad = nullptr;
  double lo = 0.1, hi = 1.1;
  long long n3() const { return 3 * g.total; }
};

class ElastSolver {
 public:
  ElastSolver(World& W, const int64_t np[3], int nlevels, int m, int est_mode, uint64_t seed_e, double nu);
  World& W;
  DeviceArena arena;
  std::vector<ElLevel> L;  // L[0] = coarsest
  int m = 2;
  double* A_dev = nullptr;
  long long *piv_dev = nullptr, *map_dev = nullptr;
  int nc = 0;
  double *cr = nullptr, *cz = nullptr, *cp = nullptr, *cw = nullptr, *cx = nullptr;  // CG, finest level
  double *dot_part = nullptr, *dot_out = nullptr, *staging = nullptr;
  long long launches = 0;
  bool est_lanczos = true;

  void apply(int l, const double* x, double* y);
  void residual(int l, const double* b, const double* x, double* r);
  void jacobi(int l, const double* x, double* y);
  void vec(int l, int op, double s, double t, const double* x, double* y);
  double dot(int l, const double* a, const double* b);
  void smooth(int l, const double* b, double* x);
  void vcycle(int l, const double* b, double* x);
  void coarse_solve(const double* b, double* x);
  void upload(int l, const double* host, double* dev);     // natural interleaved -> planes
  void download(int l, const double* dev, double* host);   // planes -> natural interleaved
  int solve(const double* b, double* x, double rtol, double atol, int max_its, bool x0_nonzero, double* hist,
            int* reason, int* its, double* n0, double* nf, double* t_ms);
  std::pair<double, double> estimate(int l);
};

}  // namespace tmgx
