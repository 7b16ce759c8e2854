// TEST INFRASTRUCTURE ONLY — the drop-in proved from the reference side.
//
// Links the reference's own translation units (as tmg_ref_bench) and libtmgx.so, and solves the
// same MG-CG problem three ways inside the reference's spawn_world(1):
//   ref  the reference's krylov_solve(cg) with the reference-TU V-cycle (tmg_ref_bench's MGPC)
//   pc   the reference's krylov_solve(cg) with GpuMGPC (gpu_mg_pc.hpp) as its Preconditioner:
//        every apply is one V-cycle on the GPU through tmgx_pc_apply
//   gpu  gpu_mg_cg_solve: the whole solve through tmgx_solve
// Built twice: against libtmgx.so (performance build) and libtmgx_parity.so (tmg_ref_gpupc_parity:
// the -fmad=false / serial-fold build, whose V-cycle and solve are bitwise the reference's).
// usage: tmg_ref_gpupc N nlevels m kind galerkin seed  -> one JSON line
#define TMG_REF_NO_MAIN
#include "tmg_ref_bench.cpp"

#include "gpu_mg_pc.hpp"

namespace {

std::string hist_json(const SolveReport& r) {
  std::string out = "[";
  char buf[64];
  for (std::size_t q = 0; q < r.residual_history.size(); ++q) {
    std::snprintf(buf, sizeof buf, "%s%.17g", q ? ", " : "", r.residual_history[q]);
    out += buf;
  }
  return out + "]";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: %s N nlevels m kind galerkin seed\n", argv[0]);
    return 1;
  }
  const idx_t N = std::atoll(argv[1]);
  const int nlevels = std::atoi(argv[2]), m = std::atoi(argv[3]);
  Problem pr;
  pr.kind = std::atoi(argv[4]);
  const bool galerkin = std::atoi(argv[5]) != 0;
  const std::uint64_t seed = std::strtoull(argv[6], nullptr, 10);
  for (int s = 0; s < 32; ++s)
    pr.spheres.push_back({hashed_uniform(pr.seed_k, 4ull * s + 0), hashed_uniform(pr.seed_k, 4ull * s + 1),
                          hashed_uniform(pr.seed_k, 4ull * s + 2),
                          0.05 + 0.10 * hashed_uniform(pr.seed_k, 4ull * s + 3)});
  auto res = spawn_world(1, [&](Comm& comm) {
    StructuredGrid g = create_grid(comm, 3, {N, N, N}, 1, 1);
    DistVector b(comm, g.layout());
    const GridBox bx = g.local_box();
    idx_t at = 0;
    for (idx_t k = bx.lo[2]; k < bx.hi[2]; ++k)
      for (idx_t j = bx.lo[1]; j < bx.hi[1]; ++j)
        for (idx_t i = bx.lo[0]; i < bx.hi[0]; ++i, ++at) {
          const bool bnd = i == 0 || j == 0 || k == 0 || i == N - 1 || j == N - 1 || k == N - 1;
          b[at] = bnd ? 0.0 : 2.0 * hashed_uniform(seed, (std::uint64_t)g.header().natural_index(i, j, k, 0)) - 1.0;
        }
    KrylovConfig cfg;
    cfg.method = KrylovMethod::cg;
    cfg.rtol = 1e-8;
    // ref: the reference's CG + its V-cycle
    auto mg = std::make_shared<MGPC>(g, pr, nlevels, m, /*lanczos=*/true, galerkin);
    SolverNode ref_node = SolverNode::create(cfg, mg->op(), mg, "");
    DistVector x_ref(comm, g.layout());
    const SolveReport r_ref = ref_node.solve(b, x_ref);
    // pc: the reference's CG + the GPU V-cycle as its Preconditioner
    tmgx_problem tp{};
    tp.kind = pr.kind == 1 ? TMGX_VARCOEF7_HARMONIC : TMGX_POISSON7;
    tp.np[0] = tp.np[1] = tp.np[2] = N;
    tp.seed_k = pr.seed_k;
    tp.n_spheres = 32;
    tp.k_in = pr.k_in;
    tmgx_mg_cfg mc{};
    mc.nlevels = nlevels;
    mc.smooth_its = m;
    mc.est_mode = TMGX_EST_LANCZOS;
    mc.galerkin = galerkin ? 1 : 0;
    auto gpu = std::make_shared<GpuMGPC>(g, tp, mc);
    SolverNode pc_node = SolverNode::create(cfg, mg->op(), gpu, "");
    DistVector x_pc(comm, g.layout());
    const SolveReport r_pc = pc_node.solve(b, x_pc);
    // gpu: the whole solve on the GPU
    DistVector x_gpu(comm, g.layout());
    const SolveReport r_gpu = gpu_mg_cg_solve(gpu->solver(), cfg, b, x_gpu);
    auto reldiff = [&](const DistVector& a, const DistVector& c) {  // ||a - c||_2 / ||c||_2
      double num = 0.0, den = 0.0;
      for (std::size_t q = 0; q < a.local().size(); ++q) {
        const double d = a.local()[q] - c.local()[q];
        num += d * d;
        den += c.local()[q] * c.local()[q];
      }
      return std::sqrt(num / den);
    };
    auto same = [&](const DistVector& a, const DistVector& c) {
      return a.local() == c.local();
    };
    char buf[512];
    std::snprintf(buf, sizeof buf,
                  "{\"n\": %lld, \"ref_its\": %d, \"pc_its\": %d, \"gpu_its\": %d, \"ref_reason\": \"%s\", "
                  "\"pc_reason\": \"%s\", \"ref_xnorm\": %.17g, \"pc_xnorm\": %.17g, \"gpu_xnorm\": %.17g, "
                  "\"pc_vs_ref\": %.3e, \"gpu_vs_ref\": %.3e, \"pc_kind\": \"%s\", \"pc_x_bitwise\": %s, "
                  "\"pc_history_bitwise\": %s, \"gpu_x_bitwise\": %s, \"gpu_history_bitwise\": %s, \"parity_build\": %d",
                  (long long)(N * N * N), r_ref.iterations, r_pc.iterations, r_gpu.iterations,
                  to_string(r_ref.reason).c_str(), to_string(r_pc.reason).c_str(), norm2(x_ref), norm2(x_pc),
                  norm2(x_gpu), reldiff(x_pc, x_ref), reldiff(x_gpu, x_ref), gpu->kind().c_str(),
                  same(x_pc, x_ref) ? "true" : "false",
                  r_pc.residual_history == r_ref.residual_history ? "true" : "false", same(x_gpu, x_ref) ? "true" : "false",
                  r_gpu.residual_history == r_ref.residual_history ? "true" : "false", tmgx_parity_build());
    return std::string(buf) + ", \"ref_history\": " + hist_json(r_ref) + ", \"pc_history\": " + hist_json(r_pc) +
           ", \"gpu_history\": " + hist_json(r_gpu) + "}";
  });
  std::printf("%s\n", res[0].c_str());
  return 0;
}
