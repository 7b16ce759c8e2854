// TEST INFRASTRUCTURE ONLY — the reference's own CPU solver for the MG-CG path.
//
// Links the reference's translation units (/root/reference/proj/core/src/*.cpp, unmodified)
// and adds the pieces the reference does not ship, written from the spec:
//   assemble_problem   SPEC.md:668-676 (App. A conventions: FD rows, Dirichlet rows, spheres)
//   MG preconditioner  SPEC.md:472-490 / PAPER.md Alg. 1 (V-cycle over SolverNode smoothers,
//                      P = create_interpolation, R = 2^-3 transpose(P), LUPC coarse)
//   Galerkin option    ptap (dist_matrix.cpp:462-468) scaled by 2^-3
//   lanczos estimator  chebyshev_bounds_estimate with the missing p = z + beta p (solver.cpp:537-561)
// Everything numerical runs through the reference: spmv, transpose, ptap, krylov_solve
// (solve_cg, solve_fixed Chebyshev), JacobiPC, LUPC/DenseLU, dot/axpy/scale, create_grid,
// coarsen, create_interpolation, spawn_world (1 rank = 1 core, the baseline protocol).
//
// usage: tmg_ref_bench N nlevels m steps warmup seed [est=lanczos|reference] [galerkin=0|1]
//                      [kind=0|1] [dump_x_path|-] [budget_s]
// prints one JSON line {iterations, xnorm, final_ratio, t_setup_s, t_solve_s, ...}
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "tmg/comm.hpp"
#include "tmg/common.hpp"
#include "tmg/dist_matrix.hpp"
#include "tmg/dist_vector.hpp"
#include "tmg/grid.hpp"
#include "tmg/precond.hpp"
#include "tmg/solver.hpp"

using namespace tmg;

namespace {

struct Sphere {
  double cx, cy, cz, r;
};

struct Problem {
  int kind = 0;
  std::uint64_t seed_k = 7;
  std::vector<Sphere> spheres;
  double k_in = 1e4;
};

double harm(double a, double b) { return 2.0 * a * b / (a + b); }

double kfun(const Problem& pr, const GridHeader& h, idx_t i, idx_t j, idx_t k) {
  if (pr.kind != 1) return 1.0;
  const double x = (double)i * (1.0 / (double)(h.npoints[0] - 1));
  const double y = (double)j * (1.0 / (double)(h.npoints[1] - 1));
  const double z = (double)k * (1.0 / (double)(h.npoints[2] - 1));
  for (const auto& s : pr.spheres) {
    const double dx = x - s.cx, dy = y - s.cy, dz = z - s.cz;
    const double d2 = dx * dx + dy * dy + dz * dz;
    if (d2 <= s.r * s.r) return pr.k_in;
  }
  return 1.0;
}

// assemble_problem: 7-point FD rows on the grid's owned vertices (App. A-C4)
std::shared_ptr<DistMatrix> assemble(const StructuredGrid& g, const Problem& pr) {
  const GridHeader& h = g.header();
  MatrixAssembler asmb(g.comm(), h.layout(), h.layout());
  const GridBox b = g.local_box();
  double ih2[3];
  for (int a = 0; a < 3; ++a) {
    const double hh = 1.0 / (double)(h.npoints[a] - 1);
    ih2[a] = 1.0 / (hh * hh);
  }
  const idx_t N[3] = {h.npoints[0], h.npoints[1], h.npoints[2]};
  for (idx_t k = b.lo[2]; k < b.hi[2]; ++k)
    for (idx_t j = b.lo[1]; j < b.hi[1]; ++j)
      for (idx_t i = b.lo[0]; i < b.hi[0]; ++i) {
        const idx_t row = h.global_index(i, j, k, 0);
        const bool bnd = i == 0 || j == 0 || k == 0 || i == N[0] - 1 || j == N[1] - 1 || k == N[2] - 1;
        const double kc = kfun(pr, h, i, j, k);
        // faces in the order -z, -y, -x, +x, +y, +z
        const idx_t di[6] = {0, 0, -1, 1, 0, 0}, dj[6] = {0, -1, 0, 0, 1, 0}, dk[6] = {-1, 0, 0, 0, 0, 1};
        const int ax[6] = {2, 1, 0, 0, 1, 2};
        double f[6], d = 0.0;
        for (int q = 0; q < 6; ++q) {
          const idx_t ni = i + di[q], nj = j + dj[q], nk = k + dk[q];
          const bool in = ni >= 0 && nj >= 0 && nk >= 0 && ni < N[0] && nj < N[1] && nk < N[2];
          f[q] = (in ? harm(kc, kfun(pr, h, ni, nj, nk)) : kc) * ih2[ax[q]];
          d += f[q];
        }
        asmb.add(row, row, d);
        if (bnd) continue;
        for (int q = 0; q < 6; ++q) {
          const idx_t ni = i + di[q], nj = j + dj[q], nk = k + dk[q];
          const bool interior = ni > 0 && nj > 0 && nk > 0 && ni < N[0] - 1 && nj < N[1] - 1 && nk < N[2] - 1;
          if (interior) asmb.add(row, h.global_index(ni, nj, nk, 0), -f[q]);
        }
      }
  return std::make_shared<DistMatrix>(asmb.finalize());
}

// chebyshev_bounds_estimate with the missing search-direction update (SURVEY finding 4(a));
// start vector fill_random(0x5eedbeef) (1 rank: global index == natural index).
std::pair<double, double> lanczos_bounds(const DistMatrix& A, const Preconditioner& M) {
  DistVector b(A.comm(), A.rows());
  fill_random(b, 0x5eedbeef);
  DistVector r = b, z(b.comm(), b.layout()), w(b.comm(), b.layout());
  M.apply(r, z);
  DistVector p = z;
  double rz = dot(r, z);
  std::vector<double> al, be;
  for (int it = 0; it < 10; ++it) {
    if (rz == 0.0 || !std::isfinite(rz)) break;
    spmv(A, p, w);
    const double pw = dot(p, w);
    if (pw <= 0.0 || !std::isfinite(pw)) break;
    const double alpha = rz / pw;
    axpy(-alpha, w, r);
    M.apply(r, z);
    const double rz_new = dot(r, z);
    al.push_back(alpha);
    if (rz_new <= 0.0 || !std::isfinite(rz_new)) break;
    const double beta = rz_new / rz;
    be.push_back(beta);
    rz = rz_new;
    for (std::size_t i = 0; i < p.local().size(); ++i) p.local()[i] = z.local()[i] + beta * p.local()[i];
  }
  if (al.empty()) return {0.1, 1.1};
  const std::size_t k = al.size();
  std::vector<double> d(k, 0.0), e(k > 0 ? k - 1 : 0, 0.0);
  for (std::size_t t = 0; t < k; ++t) {
    d[t] = 1.0 / al[t];
    if (t > 0) d[t] += be[t - 1] / al[t - 1];
    if (t + 1 < k) e[t] = std::sqrt(be[t]) / al[t];
  }
  // Sturm bisection as tridiag_eig_max (solver.cpp:488-516)
  double lo = d[0], hi = d[0];
  for (std::size_t i = 0; i < k; ++i) {
    const double left = i > 0 ? std::abs(e[i - 1]) : 0.0, right = i + 1 < k ? std::abs(e[i]) : 0.0;
    lo = std::min(lo, d[i] - left - right);
    hi = std::max(hi, d[i] + left + right);
  }
  for (int it = 0; it < 200 && hi - lo > 1e-12 * std::max(1.0, std::abs(hi)); ++it) {
    const double mid = 0.5 * (lo + hi);
    int count = 0;
    double q = 1.0;
    for (std::size_t i = 0; i < k; ++i) {
      const double off = i > 0 ? e[i - 1] : 0.0;
      q = d[i] - mid - (q == 0.0 ? std::abs(off) / 1e-300 : off * off / q);
      if (q < 0.0) ++count;
    }
    if (count >= (int)k)
      hi = mid;
    else
      lo = mid;
  }
  const double lam = 0.5 * (lo + hi);
  if (!(lam > 0.0) || !std::isfinite(lam)) return {0.1, 1.1};
  return {0.1 * lam, 1.1 * lam};
}

struct Level {
  std::shared_ptr<StructuredGrid> grid;
  std::shared_ptr<DistMatrix> A;
  std::shared_ptr<DistMatrix> P;  // to this level from the next coarser one (rows: this level)
  std::shared_ptr<DistMatrix> R;  // 2^-3 P^T
  std::shared_ptr<SolverNode> smoother;
  std::shared_ptr<SolverNode> coarse;
};

// mg_setup / mg_apply: level 0 = coarsest (LU), V(m,m) Chebyshev-Jacobi.
class MGPC final : public Preconditioner {
 public:
  MGPC(const StructuredGrid& fine, const Problem& pr, int nlevels, int m, bool lanczos, bool galerkin) {
    levels_.resize((std::size_t)nlevels);
    auto g = std::make_shared<StructuredGrid>(fine);
    for (int l = nlevels - 1; l >= 0; --l) {
      Level& L = levels_[(std::size_t)l];
      L.grid = g;
      if (l == nlevels - 1 || !galerkin) L.A = assemble(*g, pr);
      if (l > 0) g = std::make_shared<StructuredGrid>(coarsen(*g));
    }
    for (int l = nlevels - 1; l >= 1; --l) {
      Level& L = levels_[(std::size_t)l];
      Level& C = levels_[(std::size_t)l - 1];
      L.P = std::make_shared<DistMatrix>(create_interpolation(*C.grid, *L.grid));
      auto R = std::make_shared<DistMatrix>(transpose(*L.P));
      for (double& v : R->values()) v *= 0.125;
      L.R = R;
      if (galerkin) {
        auto Ac = std::make_shared<DistMatrix>(ptap(*L.P, *L.A));
        for (double& v : Ac->values()) v *= 0.125;
        C.A = Ac;
      }
    }
    for (int l = nlevels - 1; l >= 1; --l) {
      Level& L = levels_[(std::size_t)l];
      auto jac = std::make_shared<JacobiPC>(*L.A);
      KrylovConfig cfg;
      cfg.method = KrylovMethod::chebyshev;
      cfg.fixed_its = m;
      if (lanczos) cfg.cheb_bounds = lanczos_bounds(*L.A, *jac);
      L.smoother = std::make_shared<SolverNode>(SolverNode::create(cfg, L.A, jac, "mg_levels_"));
    }
    KrylovConfig cc;
    cc.method = KrylovMethod::preonly;
    levels_[0].coarse = std::make_shared<SolverNode>(
        SolverNode::create(cc, levels_[0].A, std::make_shared<LUPC>(*levels_[0].A), "mg_coarse_"));
  }

  void apply(const DistVector& b, DistVector& x) const override { vcycle((int)levels_.size() - 1, b, x); }
  std::string kind() const override { return "mg"; }
  const std::shared_ptr<DistMatrix>& op() const { return levels_.back().A; }
  double bound_hi(int l) const { return levels_[(std::size_t)l].smoother->config().cheb_bounds->second; }

 private:
  std::vector<Level> levels_;

  void vcycle(int l, const DistVector& b, DistVector& x) const {
    const Level& L = levels_[(std::size_t)l];
    set_all(x, 0.0);
    if (l == 0) {
      L.coarse->solve(b, x);
      return;
    }
    const Level& C = levels_[(std::size_t)l - 1];
    L.smoother->solve(b, x);
    DistVector r(b.comm(), b.layout());
    spmv(*L.A, x, r);
    for (std::size_t i = 0; i < r.local().size(); ++i) r.local()[i] = b.local()[i] - r.local()[i];
    DistVector bc = spmv(*L.R, r);
    DistVector xc(bc.comm(), bc.layout());
    vcycle(l - 1, bc, xc);
    DistVector t = spmv(*L.P, xc);
    axpy(1.0, t, x);
    L.smoother->solve(b, x);
  }
};

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

#ifndef TMG_REF_NO_MAIN
int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: %s N nlevels m steps warmup seed [est] [galerkin] [kind] [dump]\n", argv[0]);
    return 1;
  }
  const idx_t N = std::atoll(argv[1]);
  const int nlevels = std::atoi(argv[2]), m = std::atoi(argv[3]);
  const int steps = std::atoi(argv[4]), warmup = std::atoi(argv[5]);
  const std::uint64_t seed = std::strtoull(argv[6], nullptr, 10);
  const bool lanczos = argc <= 7 || std::string(argv[7]) != "reference";
  const bool galerkin = argc > 8 && std::atoi(argv[8]) != 0;
  Problem pr;
  pr.kind = argc > 9 ? std::atoi(argv[9]) : 0;
  const std::string dump = argc > 10 && std::string(argv[10]) != "-" ? argv[10] : "";
  // optional time budget (s) for the timed solves: after the warm-up, at most budget / t_warmup
  // solves (at least one) are timed
  const double budget = argc > 11 ? std::atof(argv[11]) : 0.0;
  for (int s = 0; s < 32; ++s)
    pr.spheres.push_back({hashed_uniform(pr.seed_k, 4ull * s + 0), hashed_uniform(pr.seed_k, 4ull * s + 1),
                          hashed_uniform(pr.seed_k, 4ull * s + 2),
                          0.05 + 0.10 * hashed_uniform(pr.seed_k, 4ull * s + 3)});

  auto res = spawn_world(1, [&](Comm& comm) {
    const double t0 = now();
    StructuredGrid g = create_grid(comm, 3, {N, N, N}, 1, 1);
    auto mg = std::make_shared<MGPC>(g, pr, nlevels, m, lanczos, galerkin);
    KrylovConfig cfg;
    cfg.method = KrylovMethod::cg;
    cfg.rtol = 1e-8;
    SolverNode outer = SolverNode::create(cfg, mg->op(), mg, "");
    const double t_setup = now() - t0;
    DistVector b(comm, g.layout());
    const GridBox bx = g.local_box();
    idx_t at = 0;
    for (idx_t k = bx.lo[2]; k < bx.hi[2]; ++k)
      for (idx_t j = bx.lo[1]; j < bx.hi[1]; ++j)
        for (idx_t i = bx.lo[0]; i < bx.hi[0]; ++i, ++at) {
          const bool bnd = i == 0 || j == 0 || k == 0 || i == N - 1 || j == N - 1 || k == N - 1;
          b[at] = bnd ? 0.0 : 2.0 * hashed_uniform(seed, (std::uint64_t)g.header().natural_index(i, j, k, 0)) - 1.0;
        }
    DistVector x(comm, g.layout());
    SolveReport rep;
    double t_warm = 0.0;
    for (int w = 0; w < warmup; ++w) {
      set_all(x, 0.0);
      const double t1 = now();
      rep = outer.solve(b, x);
      t_warm = now() - t1;
    }
    int n_timed = steps;
    if (budget > 0.0 && t_warm > 0.0) n_timed = std::max(1, std::min(steps, (int)(budget / t_warm)));
    double t_solve = 0.0;
    for (int s = 0; s < n_timed; ++s) {
      set_all(x, 0.0);
      const double t1 = now();
      rep = outer.solve(b, x);
      t_solve += now() - t1;
    }
    if (!dump.empty()) {
      FILE* f = std::fopen(dump.c_str(), "wb");
      std::fwrite(x.local().data(), sizeof(double), x.local().size(), f);
      std::fclose(f);
    }
    char buf[512];
    std::snprintf(buf, sizeof buf,
                  "{\"iterations\": %d, \"reason\": \"%s\", \"xnorm\": %.17g, \"final_ratio\": %.17g, "
                  "\"t_setup_s\": %.6f, \"t_solve_s\": %.6f, \"n\": %lld, \"cheb_hi_fine\": %.17g, \"history\": [",
                  rep.iterations, to_string(rep.reason).c_str(), norm2(x),
                  rep.residual_history.back() / rep.residual_history.front(), t_setup, t_solve / std::max(1, n_timed),
                  (long long)(N * N * N), mg->bound_hi(nlevels - 1));
    std::string out(buf);
    out.resize(out.size() - std::string(", \"history\": [").size());
    out += std::string(", \"steps_timed\": ") + std::to_string(n_timed) + ", \"history\": [";
    for (std::size_t q = 0; q < rep.residual_history.size(); ++q) {
      std::snprintf(buf, sizeof buf, "%s%.17g", q ? ", " : "", rep.residual_history[q]);
      out += buf;
    }
    return out + "]}";
  });
  std::printf("%s\n", res[0].c_str());
  return 0;
}
#endif  // TMG_REF_NO_MAIN
