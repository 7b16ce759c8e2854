// The reference-side binding of the tmgx drop-in, compiled against the
// reference's own headers: a tmg::Preconditioner whose apply is one GPU V-cycle, and a
// krylov_solve replacement that runs the whole MG-CG solve on the GPU. TEST INFRASTRUCTURE
// here (oracle/ref_glue/tmg_ref_gpupc.cpp drives it); in the reference it would be a new
// header tmg/gpu_mg_pc.hpp.
#pragma once

#include <string>
#include <vector>

#include <tmgx.h>

#include "tmg/common.hpp"
#include "tmg/dist_vector.hpp"
#include "tmg/grid.hpp"
#include "tmg/preconditioner.hpp"
#include "tmg/solver.hpp"

namespace tmg {

inline void tmgx_throw(int rc) {  // status -> the reference's error taxonomy (common.hpp:16-34)
  if (rc == TMGX_OK || rc == TMGX_DIVERGED) return;
  if (rc == TMGX_ERR_CONFIG) throw ConfigError(tmgx_last_error());
  throw Error(tmgx_last_error());
}

class GpuMGPC final : public Preconditioner {
 public:
  // One reference rank per process drives one GPU (process `rank` of `size`; `job` is the
  // node-local rendezvous token from tmgx_job_token on rank 0, ignored for size 1).
  GpuMGPC(const StructuredGrid& grid, tmgx_problem prob, tmgx_mg_cfg mg, int device = 0, const char* job = nullptr) {
    const Comm& c = grid.comm();
    tmgx_throw(tmgx_world_create(c.size(), c.size(), c.rank(), device, job, &world_));
    for (int a = 0; a < 3; ++a) prob.pg_hint[a] = (int)grid.header().proc_grid[(std::size_t)a];
    tmgx_throw(tmgx_solver_create(world_, &prob, &mg, &solver_));
  }
  ~GpuMGPC() override {
    tmgx_solver_destroy(solver_);
    tmgx_world_destroy(world_);
  }
  GpuMGPC(const GpuMGPC&) = delete;
  GpuMGPC& operator=(const GpuMGPC&) = delete;

  // y = M^-1 x on this rank's rows (DistVector local order == tmgx local order, grid.cpp:61-82)
  void apply(const DistVector& x, DistVector& y) const override {
    tmgx_throw(tmgx_pc_apply(solver_, x.local().data(), y.local().data()));
  }
  std::string kind() const override { return "mg(gpu)"; }
  tmgx_solver solver() const { return solver_; }

 private:
  tmgx_world world_{};
  tmgx_solver solver_{};
};

// Whole solve on the GPU (krylov_solve + SolverNode replacement for ksp_type cg + pc_type mg).
inline SolveReport gpu_mg_cg_solve(tmgx_solver s, const KrylovConfig& cfg, const DistVector& b, DistVector& x) {
  tmgx_ksp_cfg k{TMGX_KSP_CG, cfg.rtol, cfg.atol, cfg.max_its, 0};
  std::vector<double> hist((std::size_t)cfg.max_its + 1);
  tmgx_report r{};
  tmgx_throw(tmgx_solve(s, b.local().data(), x.local().data(), /*on_device=*/0, &k, hist.data(), &r));
  SolveReport rep;
  rep.reason = static_cast<ConvergedReason>(r.reason);  // same enum order (solver.hpp:24)
  rep.iterations = r.iterations;
  rep.residual_history.assign(hist.begin(), hist.begin() + r.iterations + 1);
  return rep;
}

}  // namespace tmg
