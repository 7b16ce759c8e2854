// extern "C" boundary (include/tmgx.h) over the C++ host layer. Exceptions become status codes:
// tmg::ConfigError -> 1, tmg::CudaError -> 3, any other failure -> 4.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "tmg_options.hpp"
#include "tmgx.h"
#include "tmgx_elast.hpp"
#include "tmgx_engine.hpp"

struct tmgx_world_s {
  std::unique_ptr<tmgx::World> w;
};
struct tmgx_solver_s {
  tmgx_world world;
  std::unique_ptr<tmgx::Solver> s;
};
struct tmgx_elast_s {
  tmgx_world world;
  std::unique_ptr<tmgx::ElastSolver> s;
};
struct tmgx_options_s {
  tmg::OptionsDatabase db;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const tmg::ConfigError& e) {
    g_err = e.what();
    return TMGX_ERR_CONFIG;
  } catch (const tmg::CudaError& e) {
    g_err = e.what();
    return TMGX_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TMGX_ERR_INTERNAL;
  }
}

tmg::GridHeader to_hdr(const tmgx_header* h) {
  tmg::GridHeader g;
  g.dim = h->dim;
  g.dof = h->dof;
  for (int a = 0; a < 3; ++a) {
    g.npoints[a] = h->np[a];
    g.proc_grid[a] = h->pg[a];
    g.axis_offsets[a].assign(h->off[a], h->off[a] + h->pg[a] + 1);
  }
  return g;
}

void from_hdr(const tmg::GridHeader& g, tmgx_header* h) {
  std::memset(h, 0, sizeof(*h));
  h->dim = g.dim;
  h->dof = g.dof;
  for (int a = 0; a < 3; ++a) {
    h->np[a] = g.npoints[a];
    h->pg[a] = g.proc_grid[a];
    if (g.proc_grid[a] > TMGX_MAX_AXIS_PARTS) throw tmg::ConfigError("too many parts on one axis");
    for (size_t p = 0; p < g.axis_offsets[a].size(); ++p) h->off[a][p] = g.axis_offsets[a][p];
  }
}

tmgx::ProblemDesc to_problem(const tmgx_problem* p) {
  tmgx::ProblemDesc pd;
  pd.kind = p->kind;
  for (int a = 0; a < 3; ++a) {
    pd.np[a] = p->np[a];
    pd.pg_hint[a] = p->pg_hint[a];
  }
  pd.seed_k = p->seed_k;
  pd.n_spheres = p->n_spheres;
  pd.k_in = p->k_in;
  if (pd.kind != TMGX_POISSON7 && pd.kind != TMGX_VARCOEF7_HARMONIC) throw tmg::ConfigError("unknown operator kind");
  return pd;
}

tmgx::MGDesc to_mg(const tmgx_mg_cfg* m) {
  tmgx::MGDesc md;
  md.nlevels = m->nlevels;
  md.m = m->smooth_its;
  md.est_mode = m->est_mode;
  md.galerkin = m->galerkin != 0;
  if (m->cheb_bounds) md.bounds.assign(m->cheb_bounds, m->cheb_bounds + 2 * m->nlevels);
  if (m->n_telescope < 0 || m->n_telescope > TMGX_MAX_TELESCOPE) throw tmg::ConfigError("bad telescope count");
  for (int t = 0; t < m->n_telescope; ++t)
    md.tele.push_back({m->telescope[t].level, m->telescope[t].reduction_factor,
                       {m->telescope[t].override_[0], m->telescope[t].override_[1], m->telescope[t].override_[2]}});
  return md;
}

int check_level(tmgx_solver s, int level) {
  if (!s || !s->s) throw tmg::Error("null solver");
  if (level < 0 || level >= s->s->mgd.nlevels) throw tmg::Error("level out of range");
  return s->s->node_for_level(level);
}
}  // namespace

// ---- options database / solver tree (tmg_options.hpp)
namespace {
void copy_out(const std::string& v, char* buf, int buflen) {
  if (!buf) return;
  if ((int)v.size() + 1 > buflen)
    throw tmg::ConfigError("output buffer too small: need " + std::to_string(v.size() + 1) + " bytes");
  std::memcpy(buf, v.c_str(), v.size() + 1);
}
std::string lines(const std::vector<std::string>& v) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "\n" : "") + v[i];
  return s;
}
void resolved_to_c(const tmg::ResolvedTree& r, tmgx_mg_cfg* mg, tmgx_ksp_cfg* ksp) {
  if (mg) {
    std::memset(mg, 0, sizeof(*mg));
    mg->nlevels = r.nlevels;
    mg->smooth_its = r.smooth_its;
    mg->est_mode = r.est_mode;
    mg->cheb_bounds = nullptr;
    if ((int)r.stages.size() > TMGX_MAX_TELESCOPE) throw tmg::ConfigError("too many telescope stages");
    mg->n_telescope = (int)r.stages.size();
    for (size_t t = 0; t < r.stages.size(); ++t) {
      mg->telescope[t].level = r.stages[t].level;
      mg->telescope[t].reduction_factor = r.stages[t].reduction_factor;
      for (int a = 0; a < 3; ++a) mg->telescope[t].override_[a] = r.stages[t].override_[a];
    }
    mg->galerkin = r.galerkin ? 1 : 0;
  }
  if (ksp) {
    ksp->method = r.ksp_method;
    ksp->rtol = r.rtol;
    ksp->atol = r.atol;
    ksp->max_its = r.max_its;
    ksp->zero_initial_guess = r.zero_initial_guess ? 1 : 0;
  }
}
}  // namespace

extern "C" {

const char* tmgx_last_error(void) { return g_err.c_str(); }
int tmgx_parity_build(void) { return tmgx::parity_build() ? 1 : 0; }

int tmgx_choose_proc_grid(int size, int dim, const int64_t np[3], int pg_out[3]) {
  return guard([&] {
    const auto pg = tmg::choose_proc_grid(size, dim, {np[0], np[1], np[2]});
    for (int a = 0; a < 3; ++a) pg_out[a] = pg[a];
    return 0;
  });
}

int tmgx_grid_header(int size, int dim, const int64_t np[3], int dof, const int* hint, tmgx_header* out) {
  return guard([&] {
    std::optional<std::array<int, 3>> h;
    if (hint) h = std::array<int, 3>{hint[0], hint[1], hint[2]};
    from_hdr(tmg::build_header_for(size, dim, {np[0], np[1], np[2]}, dof, 1, h), out);
    return 0;
  });
}

int tmgx_coarsen_header(const tmgx_header* fine, tmgx_header* coarse) {
  return guard([&] {
    auto c = tmg::try_coarsen_header(to_hdr(fine));
    if (!c) throw tmg::ConfigError("cannot coarsen");
    from_hdr(*c, coarse);
    return 0;
  });
}

int tmgx_layout_offsets(const tmgx_header* h, int64_t* offsets) {
  return guard([&] {
    const auto lay = to_hdr(h).layout();
    for (size_t k = 0; k < lay.offsets.size(); ++k) offsets[k] = lay.offsets[k];
    return 0;
  });
}

int64_t tmgx_global_to_natural(const tmgx_header* h, int64_t g) { return to_hdr(h).global_to_natural(g); }
int64_t tmgx_natural_to_global(const tmgx_header* h, int64_t n) { return to_hdr(h).natural_to_global(n); }

int tmgx_split_strided(int n, int r, int* member_map, int* n_members) {
  return guard([&] {
    const auto s = tmg::split_strided(n, r);
    for (int k = 0; k < s.n_members(); ++k) member_map[k] = s.member_map[k];
    *n_members = s.n_members();
    return 0;
  });
}

int tmgx_repartition_header(const tmgx_header* h, int sub_size, const int ov[3], tmgx_header* out) {
  return guard([&] {
    std::array<std::optional<int>, 3> o;
    for (int a = 0; a < 3; ++a)
      if (ov && ov[a]) o[a] = ov[a];
    from_hdr(tmg::repartition_header(to_hdr(h), sub_size, o), out);
    return 0;
  });
}

int tmgx_prefusion_layout(const tmgx_header* nh, int parent_size, const int* mm, int n_members, int64_t* offsets) {
  return guard([&] {
    tmg::SplitResult sp;
    sp.member_map.assign(mm, mm + n_members);
    sp.parent_size = parent_size;
    sp.reduction_factor = n_members > 1 ? mm[1] - mm[0] : parent_size;
    const auto lay = tmg::prefusion_layout(to_hdr(nh), sp);
    for (size_t k = 0; k < lay.offsets.size(); ++k) offsets[k] = lay.offsets[k];
    return 0;
  });
}

int tmgx_permutation(const tmgx_header* oh, const tmgx_header* nh, int64_t rb, int64_t re, int64_t* cols) {
  return guard([&] {
    const auto o = to_hdr(oh), n = to_hdr(nh);
    if (!o.same_global_grid(n)) throw tmg::Error("build_permutation: grids describe different global problems");
    for (int64_t p = rb; p < re; ++p) cols[p - rb] = n.natural_to_global(o.global_to_natural(p));
    return 0;
  });
}

int tmgx_job_token(char* out) {
  return guard([&] {
    unsigned char r[16];
    FILE* f = std::fopen("/dev/urandom", "rb");
    if (!f || std::fread(r, 1, sizeof r, f) != sizeof r) {
      if (f) std::fclose(f);
      throw tmg::Error("job token: /dev/urandom unavailable");
    }
    std::fclose(f);
    for (int i = 0; i < 16; ++i) std::snprintf(out + 2 * i, 3, "%02x", r[i]);
    return 0;
  });
}

int tmgx_world_create(int n_ranks, int nproc, int proc, int device, const char* job, tmgx_world* out) {
  return guard([&] {
    auto w = new tmgx_world_s;
    try {
      w->w = std::make_unique<tmgx::World>(n_ranks, nproc, proc, device, job);
    } catch (...) {
      delete w;
      throw;
    }
    *out = w;
    return 0;
  });
}

int tmgx_world_destroy(tmgx_world w) {
  return guard([&] {
    delete w;
    return 0;
  });
}

int tmgx_world_local_ranks(tmgx_world w, int* first, int* end) {
  *first = w->w->first;
  *end = w->w->end;
  return 0;
}

int tmgx_solver_create(tmgx_world w, const tmgx_problem* p, const tmgx_mg_cfg* m, tmgx_solver* out) {
  return guard([&] {
    const tmgx::ProblemDesc pd = to_problem(p);
    const tmgx::MGDesc md = to_mg(m);
    auto s = new tmgx_solver_s;
    s->world = w;
    try {
      s->s = std::make_unique<tmgx::Solver>(*w->w, pd, md);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
    return 0;
  });
}


int tmgx_options_create(tmgx_options* out) {
  return guard([&] {
    *out = new tmgx_options_s;
    return 0;
  });
}
int tmgx_options_destroy(tmgx_options o) {
  return guard([&] {
    delete o;
    return 0;
  });
}
int tmgx_options_parse(tmgx_options o, int argc, const char* const* argv) {
  return guard([&] {
    std::vector<std::string> t;
    for (int i = 0; i < argc; ++i) t.emplace_back(argv[i]);
    o->db.parse(t);
    return 0;
  });
}
int tmgx_options_parse_file_text(tmgx_options o, const char* text) {
  return guard([&] {
    o->db.parse_file_text(text ? text : "");
    return 0;
  });
}
int tmgx_options_set(tmgx_options o, const char* key, const char* value) {
  return guard([&] {
    o->db.set(key, value ? value : "true");
    return 0;
  });
}
int tmgx_options_get(tmgx_options o, const char* key, char* buf, int buflen, int* found) {
  return guard([&] {
    auto v = o->db.get(key);
    *found = v ? 1 : 0;
    if (v) copy_out(*v, buf, buflen);
    return 0;
  });
}
int tmgx_options_serialize(tmgx_options o, char* buf, int buflen) {
  return guard([&] {
    copy_out(lines(o->db.serialize()), buf, buflen);
    return 0;
  });
}
int tmgx_options_unused(tmgx_options o, char* buf, int buflen) {
  return guard([&] {
    copy_out(lines(o->db.unused()), buf, buflen);
    return 0;
  });
}
int tmgx_options_resolve(tmgx_options o, const char* prefix, const char* default_ksp, tmgx_mg_cfg* mg,
                         tmgx_ksp_cfg* ksp, char* describe, int describe_len) {
  return guard([&] {
    const auto r = tmg::resolve_solver_tree(o->db, prefix ? prefix : "", default_ksp ? default_ksp : "gmres");
    resolved_to_c(r, mg, ksp);
    copy_out(r.describe, describe, describe_len);
    return 0;
  });
}
int tmgx_solver_from_options(tmgx_world w, const tmgx_problem* prob, tmgx_options o, const char* prefix,
                             const char* default_ksp, tmgx_solver* out, tmgx_ksp_cfg* ksp) {
  return guard([&] {
    const auto r = tmg::resolve_solver_tree(o->db, prefix ? prefix : "", default_ksp ? default_ksp : "gmres");
    tmgx_mg_cfg mg;
    resolved_to_c(r, &mg, ksp);
    return tmgx_solver_create(w, prob, &mg, out);  // its status code (config / CUDA / internal) and message
  });
}

int tmgx_solver_destroy(tmgx_solver s) {
  return guard([&] {
    delete s;
    return 0;
  });
}

int tmgx_solver_level_info(tmgx_solver s, int level, tmgx_header* h, int64_t* n_local) {
  return guard([&] {
    const int i = check_level(s, level);
    if (h) from_hdr(s->s->nodes[i].dist->h, h);
    if (n_local) *n_local = s->s->local_n(i);
    return 0;
  });
}

int tmgx_solver_bounds(tmgx_solver s, int level, double* lo, double* hi) {
  return guard([&] {
    const int i = check_level(s, level);
    *lo = s->s->nodes[i].lo;
    *hi = s->s->nodes[i].hi;
    return 0;
  });
}

int tmgx_fill_rhs(tmgx_solver s, uint64_t seed, double* b_local) {
  return guard([&] {
    auto& S = *s->s;
    const auto& D = *S.nodes[0].dist;
    for (size_t q = 0; q < D.local.size(); ++q)
      S.W.cnt.launches += tmgx::launch_fill_rhs(D.geo[q], S.cw.p[q], seed, true, S.W.stream);
    S.download(0, S.cw, b_local, false);
    return 0;
  });
}

int tmgx_solve(tmgx_solver s, const double* b, double* x, int on_device, const tmgx_ksp_cfg* cfg, double* history,
               tmgx_report* rep) {
  return guard([&] {
    if (cfg->method != TMGX_KSP_CG && cfg->method != TMGX_KSP_PREONLY)
      throw tmg::ConfigError("ksp_type must be cg or preonly on this path");
    auto& S = *s->s;
    const long long l0 = S.W.cnt.launches;
    double t_ms = 0;
    int reason, its;
    double n0, nf;
    const int rc = S.solve(b, x, on_device != 0, cfg->method, cfg->rtol, cfg->atol, cfg->max_its, history, &reason,
                           &its, &n0, &nf, &t_ms, false, 0, cfg->zero_initial_guess == 0);
    rep->reason = reason;
    rep->iterations = its;
    rep->norm0 = n0;
    rep->norm_final = nf;
    rep->t_solve_s = t_ms * 1e-3;
    rep->kernel_launches = S.W.cnt.launches - l0;
    return rc;
  });
}

int tmgx_solve_seeded(tmgx_solver s, uint64_t seed, double* x_dev, const tmgx_ksp_cfg* cfg, double* history,
                      tmgx_report* rep) {
  return guard([&] {
    auto& S = *s->s;
    const long long l0 = S.W.cnt.launches;
    double t_ms = 0;
    int reason, its;
    double n0, nf;
    const int rc = S.solve(nullptr, x_dev, true, cfg->method, cfg->rtol, cfg->atol, cfg->max_its, history, &reason,
                           &its, &n0, &nf, &t_ms, true, seed);
    rep->reason = reason;
    rep->iterations = its;
    rep->norm0 = n0;
    rep->norm_final = nf;
    rep->t_solve_s = t_ms * 1e-3;
    rep->kernel_launches = S.W.cnt.launches - l0;
    return rc;
  });
}

int tmgx_pc_apply(tmgx_solver s, const double* x, double* y) {
  return guard([&] {
    auto& S = *s->s;
    auto& nd = S.nodes[0];
    S.upload(0, nd.b, x, false);
    S.vcycle(0);
    S.download(0, nd.x, y, false);
    return 0;
  });
}

int tmgx_level_apply(tmgx_solver s, int level, const double* x, double* y) {
  return guard([&] {
    const int i = check_level(s, level);
    auto& S = *s->s;
    auto& nd = S.nodes[i];
    S.upload(i, nd.x, x, false);
    S.apply(i, nd.x, nd.b);
    S.download(i, nd.b, y, false);
    return 0;
  });
}

int tmgx_level_smooth(tmgx_solver s, int level, const double* b, double* x) {
  return guard([&] {
    const int i = check_level(s, level);
    auto& S = *s->s;
    auto& nd = S.nodes[i];
    if (nd.kind != tmgx::SMOOTH) throw tmg::Error("level has no smoother");
    S.upload(i, nd.b, b, false);
    bool zero = true;
    for (long long t = 0, n = S.local_n(i); t < n; ++t)
      if (x[t] != 0.0) {
        zero = false;
        break;
      }
    S.upload(i, nd.x, x, false);
    S.smooth(i, zero);
    S.download(i, nd.x, x, false);
    return 0;
  });
}

int tmgx_level_residual_restrict(tmgx_solver s, int fine_level, const double* b, const double* x, double* bc) {
  return guard([&] {
    const int i = check_level(s, fine_level);
    auto& S = *s->s;
    auto& nd = S.nodes[i];
    if (nd.kind != tmgx::SMOOTH) throw tmg::Error("level is not restricted from");
    auto& cn = S.nodes[i + 1];
    S.upload(i, nd.b, b, false);
    S.upload(i, nd.x, x, false);
    S.residual_restrict(i, nd.x);  // the V-cycle's path (fused on single-box levels)
    S.download(i + 1, cn.b, bc, false);
    return 0;
  });
}

int tmgx_level_prolong_add(tmgx_solver s, int fine_level, const double* xc, double* xf) {
  return guard([&] {
    const int i = check_level(s, fine_level);
    auto& S = *s->s;
    auto& nd = S.nodes[i];
    if (nd.kind != tmgx::SMOOTH) throw tmg::Error("level is not prolongated to");
    auto& cn = S.nodes[i + 1];
    S.upload(i + 1, cn.x, xc, false);
    S.upload(i, nd.x, xf, false);
    S.halo(i + 1, cn.x);
    const auto& D = *nd.dist;
    for (size_t q = 0; q < D.local.size(); ++q)
      S.W.cnt.launches += tmgx::launch_prolong_add(D.geo[q], cn.dist->geo[q], cn.x.p[q], nd.x.p[q], S.W.stream);
    S.download(i, nd.x, xf, false);
    return 0;
  });
}

int tmgx_coarse_solve(tmgx_solver s, const double* b, double* x) {
  return guard([&] {
    auto& S = *s->s;
    const int i = (int)S.nodes.size() - 1;
    auto& nd = S.nodes[i];
    S.upload(i, nd.b, b, false);
    S.coarse_solve(i);
    S.download(i, nd.x, x, false);
    return 0;
  });
}

int tmgx_telescope_gather(tmgx_solver s, int stage, const double* xp, double* xs) {
  return guard([&] {
    auto& S = *s->s;
    if (stage < 0 || stage >= (int)S.stage_node.size()) throw tmg::Error("no such telescope stage");
    const int i = S.stage_node[stage];
    S.upload(i, S.nodes[i].b, xp, false);
    tmgx::run_plan(S.W, S.nodes[i].gather, S.nodes[i].b, S.nodes[i + 1].b, true);
    S.download(i + 1, S.nodes[i + 1].b, xs, false);
    return 0;
  });
}

int tmgx_telescope_scatter(tmgx_solver s, int stage, const double* ys, double* yp) {
  return guard([&] {
    auto& S = *s->s;
    if (stage < 0 || stage >= (int)S.stage_node.size()) throw tmg::Error("no such telescope stage");
    const int i = S.stage_node[stage];
    S.upload(i + 1, S.nodes[i + 1].x, ys, false);
    tmgx::run_plan(S.W, S.nodes[i].scatter, S.nodes[i + 1].x, S.nodes[i].x, true);
    S.download(i, S.nodes[i].x, yp, false);
    return 0;
  });
}

int tmgx_telescope_timing(tmgx_solver s, int stage, int reps, double* t_setup_s, double* t_apply_s,
                          int64_t* bytes_per_apply) {
  return guard([&] {
    auto& S = *s->s;
    if (stage < 0 || stage >= (int)S.stage_node.size()) throw tmg::Error("no such telescope stage");
    if (reps < 1) throw tmg::ConfigError("reps must be >= 1");
    const int i = S.stage_node[stage];
    auto& nd = S.nodes[i];
    auto apply = [&] {  // TelescopePC::apply data movement: gather of b, scatter of x
      tmgx::run_plan(S.W, nd.gather, nd.b, S.nodes[i + 1].b, true);
      tmgx::run_plan(S.W, nd.scatter, S.nodes[i + 1].x, nd.x, true);
    };
    apply();
    tmgx::cuda_check(cudaStreamSynchronize(S.W.stream), "sync");
    cudaEvent_t e0, e1;
    tmgx::cuda_check(cudaEventCreate(&e0), "event");
    tmgx::cuda_check(cudaEventCreate(&e1), "event");
    tmgx::cuda_check(cudaEventRecord(e0, S.W.stream), "record");
    for (int r = 0; r < reps; ++r) apply();
    tmgx::cuda_check(cudaEventRecord(e1, S.W.stream), "record");
    tmgx::cuda_check(cudaEventSynchronize(e1), "sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (t_setup_s) *t_setup_s = nd.t_setup_s;
    if (t_apply_s) *t_apply_s = ms * 1e-3 / reps;
    if (bytes_per_apply) *bytes_per_apply = 2 * 8 * (int64_t)nd.dist->h.n_unknowns();
    return 0;
  });
}

// ---- Q1 elasticity (tmgx_elast.cu)
static int elast_create(tmgx_world w, const int64_t np[3], const tmgx::MGDesc& md, uint64_t seed_e, double nu,
                        tmgx_elast* out) {
  auto e = new tmgx_elast_s;
  e->world = w;
  try {
    e->s = std::make_unique<tmgx::ElastSolver>(*w->w, np, md, seed_e, nu);
  } catch (...) {
    delete e;
    throw;
  }
  *out = e;
  return 0;
}
int tmgx_elast_create(tmgx_world w, const int64_t np[3], int nlevels, int smooth_its, int est_mode, uint64_t seed_e,
                      double nu, tmgx_elast* out) {
  return guard([&] {
    tmgx::MGDesc md;
    md.nlevels = nlevels;
    md.m = smooth_its;
    md.est_mode = est_mode;
    return elast_create(w, np, md, seed_e, nu, out);
  });
}
int tmgx_elast_create_mg(tmgx_world w, const int64_t np[3], const tmgx_mg_cfg* mg, uint64_t seed_e, double nu,
                         tmgx_elast* out) {
  return guard([&] { return elast_create(w, np, to_mg(mg), seed_e, nu, out); });
}
int tmgx_elast_destroy(tmgx_elast e) {
  return guard([&] {
    delete e;
    return 0;
  });
}
int tmgx_elast_kref(double nu, double* k576) {
  return guard([&] {
    tmgx::q1_kref(nu, k576);
    return 0;
  });
}
int tmgx_elast_level_info(tmgx_elast e, int level, int64_t np[3], double* lo, double* hi) {
  return guard([&] {
    const auto& nd = e->s->nodes[(size_t)e->s->node_for_level(level)];
    if (np) np[0] = nd.dist->h.npoints[0], np[1] = nd.dist->h.npoints[1], np[2] = nd.dist->h.npoints[2];
    if (lo) *lo = nd.lo;
    if (hi) *hi = nd.hi;
    return 0;
  });
}
int tmgx_elast_rhs(tmgx_elast e, double* b) {
  return guard([&] {
    // b_z(v) = sum over incident elements of -h^3/8 (exact: powers of two), 0 on clamped dofs
    const auto& nd = e->s->nodes[0];
    const long long nx = nd.dist->h.npoints[0], ny = nd.dist->h.npoints[1], nz = nd.dist->h.npoints[2];
    const double h = nd.h, q = -(h * h * h) / 8.0;
    for (long long k = 0; k < nz; ++k)
      for (long long j = 0; j < ny; ++j)
        for (long long i = 0; i < nx; ++i) {
          double acc = 0.0;
          for (int ez = -1; ez <= 0; ++ez)
            for (int ey = -1; ey <= 0; ++ey)
              for (int ex = -1; ex <= 0; ++ex) {
                const long long ei = i + ex, ej = j + ey, ek = k + ez;
                if (ei < 0 || ej < 0 || ek < 0 || ei >= nx - 1 || ej >= ny - 1 || ek >= nz - 1) continue;
                acc += q;
              }
          const long long v = i + nx * (j + ny * k);
          b[3 * v + 0] = 0.0;
          b[3 * v + 1] = 0.0;
          b[3 * v + 2] = i == 0 ? 0.0 : acc;
        }
    return 0;
  });
}
int tmgx_elast_level_apply(tmgx_elast e, int level, const double* x, double* y) {
  return guard([&] {
    auto& S = *e->s;
    const int i = S.node_for_level(level);
    auto& nd = S.nodes[(size_t)i];
    S.upload(i, x, nd.x);
    S.apply(i, nd.x, nd.ad);
    S.download(i, nd.ad, y);
    return 0;
  });
}
int tmgx_elast_level_smooth(tmgx_elast e, int level, const double* b, double* x) {
  return guard([&] {
    auto& S = *e->s;
    const int i = S.node_for_level(level);
    auto& nd = S.nodes[(size_t)i];
    if (nd.kind != tmgx::SMOOTH) throw tmg::ConfigError("elasticity: level 0 is the LU level");
    S.upload(i, b, nd.b);
    S.upload(i, x, nd.x);
    S.smooth(i, nd.b, nd.x);
    S.download(i, nd.x, x);
    return 0;
  });
}
int tmgx_elast_pc_apply(tmgx_elast e, const double* x, double* y) {
  return guard([&] {
    auto& S = *e->s;
    S.upload(0, x, S.cr);
    S.vcycle(0);
    S.download(0, S.cz, y);
    return 0;
  });
}
int tmgx_elast_solve(tmgx_elast e, const double* b, double* x, const tmgx_ksp_cfg* cfg, double* history,
                     tmgx_report* rep) {
  return guard([&] {
    if (cfg->method != TMGX_KSP_CG) throw tmg::ConfigError("elasticity: ksp_type must be cg");
    auto& S = *e->s;
    const long long l0 = S.launches;
    double t_ms = 0;
    int reason = 2, its = 0;
    double n0 = 0, nf = 0;
    const int rc = S.solve(b, x, cfg->rtol, cfg->atol, cfg->max_its, cfg->zero_initial_guess == 0, history, &reason,
                           &its, &n0, &nf, &t_ms);
    rep->reason = reason;
    rep->iterations = its;
    rep->norm0 = n0;
    rep->norm_final = nf;
    rep->t_solve_s = t_ms * 1e-3;
    rep->kernel_launches = S.launches - l0;
    return rc;
  });
}

int tmgx_elast_bench_apply(tmgx_elast e, int iters, double* ms_per_launch, double* bytes_per_launch,
                            double* flops_per_launch) {
  return guard([&] {
    auto& S = *e->s;
    auto& nd = S.nodes[0];
    if (nd.dist->geo.empty()) throw tmg::ConfigError("elasticity: no local box on the finest level");
    for (int w = 0; w < 3; ++w) S.apply(0, nd.x, nd.ad);
    cudaEvent_t e0, e1;
    tmgx::cuda_check(cudaEventCreate(&e0), "event");
    tmgx::cuda_check(cudaEventCreate(&e1), "event");
    tmgx::cuda_check(cudaEventRecord(e0, S.W.stream), "record");
    for (int it = 0; it < iters; ++it) S.apply(0, nd.x, nd.ad);
    tmgx::cuda_check(cudaEventRecord(e1, S.W.stream), "record");
    tmgx::cuda_check(cudaEventSynchronize(e1), "sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    double nv = 0.0;
    for (const auto& g : nd.dist->geo) nv += (double)g.ex * g.ey * g.ez;
    *ms_per_launch = ms / iters;
    *bytes_per_launch = nv * (24.0 + 24.0 + 8.0);     // x in, y out, one modulus per element
    *flops_per_launch = nv * 576.0 * 2.0;               // 8 elements x 8 vertices x 3 x 3 FMAs
    return 0;
  });
}

int tmgx_plan_summary(int n_ranks, int nproc, int proc, const tmgx_problem* p, const tmgx_mg_cfg* m, int64_t* out,
                      int max_records, int* n_records) {
  return guard([&] {
    const tmgx::Owners W(n_ranks, nproc, proc);
    const auto specs = tmgx::build_node_specs(W, to_problem(p), to_mg(m));
    int n = 0;
    auto emit = [&](int plan_id, int kind, int peer, long long count, unsigned long long sum, int level) {
      if (n >= max_records) throw tmg::Error("plan_summary: record buffer too small");
      int64_t* r = out + 6 * n++;
      r[0] = plan_id;
      r[1] = kind;
      r[2] = peer;
      r[3] = count;
      r[4] = (int64_t)sum;
      r[5] = level;
    };
    auto dump = [&](int plan_id, const tmgx::PlanHost& ph, int level) {
      for (size_t q = 0; q < ph.sends.size(); ++q)
        emit(plan_id, 0, ph.sends[q].proc, ph.sends[q].count, ph.send_sum[q], level);
      for (size_t q = 0; q < ph.recvs.size(); ++q)
        emit(plan_id, 1, ph.recvs[q].proc, ph.recvs[q].count, ph.recv_sum[q], level);
      emit(plan_id, 2, proc, ph.local_count, 0, level);
    };
    for (size_t i = 0; i < specs.size(); ++i) {
      dump(3 * (int)i, tmgx::halo_plan_host(W, *specs[i].dist), specs[i].level);
      if (specs[i].kind == tmgx::TELESCOPE) {
        dump(3 * (int)i + 1, tmgx::transfer_plan_host(W, *specs[i].dist, *specs[i + 1].dist), specs[i].level);
        dump(3 * (int)i + 2, tmgx::transfer_plan_host(W, *specs[i + 1].dist, *specs[i].dist), specs[i].level);
      }
    }
    *n_records = n;
    return 0;
  });
}

int tmgx_node_selftest(const char* job, int nproc, int proc, int rounds, int64_t out[2]) {
  return guard([&] {
    tmgx::NodeGroup g(job, nproc, proc);
    const std::string mine(reinterpret_cast<const char*>(&proc), sizeof proc);
    long long sum = 0;
    for (const std::string& v : g.allgather(mine)) {
      int q;
      std::memcpy(&q, v.data(), sizeof q);
      sum += q;
    }
    // every round: all processes see the same round number on the board before anyone moves on
    long long ok = 0;
    for (int r = 0; r < rounds; ++r) {
      const std::string tag(reinterpret_cast<const char*>(&r), sizeof r);
      bool same = true;
      for (const std::string& v : g.allgather(tag)) same = same && v == tag;
      ok += same ? 1 : 0;
      g.barrier();
    }
    out[0] = sum;
    out[1] = ok;
    return 0;
  });
}

int tmgx_exchange_timing(tmgx_solver s, int level, int reps, double* us, int64_t* bytes) {
  return guard([&] {
    auto& S = *s->s;
    const int i = check_level(s, level);
    tmgx::Node& nd = S.nodes[i];
    if (reps < 1) throw tmg::ConfigError("reps must be >= 1");
    S.halo(i, nd.x);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, S.W.stream);
    for (int r = 0; r < reps; ++r) S.halo(i, nd.x);
    cudaEventRecord(e1, S.W.stream);
    S.sync();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *us = 1e3 * ms / reps;
    *bytes = 8 * nd.halo.send_total;
    return 0;
  });
}

int tmgx_level_profile(tmgx_solver s, int reps, int max_nodes, int* n_nodes, int* kind, int64_t* npoints,
                       int* n_ranks, double* us, int64_t* bytes) {
  return guard([&] {
    auto& S = *s->s;
    if (reps < 1) throw tmg::ConfigError("reps must be >= 1");
    const int n = (int)S.nodes.size();
    *n_nodes = n;
    if (n > max_nodes) throw tmg::ConfigError("level_profile: need room for " + std::to_string(n) + " nodes");
    std::vector<double> u;
    std::vector<long long> by;
    S.level_profile(reps, u, by);
    for (int i = 0; i < n; ++i) {
      const auto& nd = S.nodes[(size_t)i];
      kind[i] = (int)nd.kind;
      for (int a = 0; a < 3; ++a) npoints[3 * i + a] = nd.dist->h.npoints[(size_t)a];
      n_ranks[i] = nd.dist->h.n_ranks();
      us[i] = u[(size_t)i];
      bytes[i] = by[(size_t)i];
    }
    return 0;
  });
}

int tmgx_get_counters(tmgx_solver s, tmgx_counters* c) {
  const auto& k = s->s->W.cnt;
  c->kernel_launches = k.launches;
  c->halo_bytes_sent = k.halo_bytes;
  c->telescope_bytes_sent = k.tele_bytes;
  c->allreduces = k.allreduces;
  return 0;
}

}  // extern "C"

extern "C" int tmgx_bench_kernel(tmgx_solver s, int which, int level, int iters, double* ms_per_launch,
                                 double* bytes_per_launch) {
  return guard([&] {
    auto& S = *s->s;
    const int i = check_level(s, level);
    auto& nd = S.nodes[i];
    if (nd.kind != tmgx::SMOOTH) throw tmg::Error("bench_kernel needs a smoothed level");
    const auto& D = *nd.dist;
    const bool var = S.prob.kind == 1;
    const double kb = var ? 8.0 : 0.0;  // coefficient stream
    long long n = D.local_unknowns();
    double per_pt = 0.0;
    tmgx::ChebStep cs{0.5, 0.25};
    if ((which == 8 || which == 9 || which == 11 || which == 14) &&
        (D.h.n_ranks() != 1 || D.local.size() != 1 || !tmgx::cheb2_tb_supported(D.geo[0])))
      throw tmg::ConfigError("bench_kernel: blocked / fused single-box kernels need a single-box level >= 33 wide");
    if ((which == 12 || which == 13) &&
        (D.h.n_ranks() != 1 || D.local.size() != 1 || !tmgx::cheb3_tb_supported(D.geo[0]) || nd.op[0].S))
      throw tmg::ConfigError("bench_kernel: the blocked m = 3 smoother needs a single-box 7-point level");
    if (which == 15 && (D.h.n_ranks() != 1 || D.local.size() != 1 ||
                        !tmgx::resid_restrict2_supported(D.geo[0], nd.op[0], S.nodes[i + 1].dist->geo[0])))
      throw tmg::ConfigError("bench_kernel: the separable fused residual + restriction needs a single-box 7-point level");
    tmgx::ChebStep cs2{0.4, 0.2};
    auto launch = [&]() {
      for (size_t q = 0; q < D.local.size(); ++q) {
        const auto& g = D.geo[q];
        switch (which) {
          case 0: tmgx::launch_cheb_step(g, nd.op[q], nd.d.p[q], nd.r.p[q], nd.x.p[q], nd.d2.p[q], nd.r.p[q], nd.x.p[q], cs, false, S.W.stream); break;
          case 1: tmgx::launch_cheb_step(g, nd.op[q], nd.d.p[q], nd.r.p[q], nd.x.p[q], nd.d2.p[q], nd.r.p[q], nd.x.p[q], cs, true, S.W.stream); break;
          case 2: tmgx::launch_apply(g, nd.op[q], nd.x.p[q], nd.b.p[q], S.W.stream); break;
          case 3: tmgx::launch_residual(g, nd.op[q], nd.b.p[q], nd.x.p[q], nd.r.p[q], S.W.stream); break;
          case 4: tmgx::launch_restrict(g, S.nodes[i + 1].dist->geo[q], nd.r.p[q], S.nodes[i + 1].b.p[q], S.W.stream); break;
          case 5: tmgx::launch_prolong_add(g, S.nodes[i + 1].dist->geo[q], S.nodes[i + 1].x.p[q], nd.x.p[q], S.W.stream); break;
          case 6: tmgx::launch_cg_update(g, nd.d.p[q], nd.d2.p[q], nd.x.p[q], nd.r.p[q], S.scal, tmgx::S_TMP1, tmgx::S_FLAG_PW, S.W.stream); break;
          case 7: tmgx::launch_spmv_dot(g, nd.op[q], nd.x.p[q], nd.b.p[q], S.part + S.part_off[q], S.W.stream); break;
          case 8: tmgx::launch_cheb2_tb(g, nd.op[q], nd.b.p[q], nullptr, nd.d.p[q], 1.0, cs, true, S.W.stream); break;
          case 9: tmgx::launch_cheb2_tb(g, nd.op[q], nd.b.p[q], nd.d.p[q], nd.x.p[q], 1.0, cs, false, S.W.stream); break;
          case 11: tmgx::launch_resid_restrict(g, nd.op[q], S.nodes[i + 1].dist->geo[q], nd.b.p[q], nd.x.p[q], S.nodes[i + 1].b.p[q], S.W.stream); break;
          case 15: tmgx::launch_resid_restrict2(g, nd.op[q], S.nodes[i + 1].dist->geo[q], nd.b.p[q], nd.x.p[q], S.nodes[i + 1].b.p[q], S.W.stream); break;
          case 14: tmgx::launch_pspmv_dot(g, nd.op[q], nd.x.p[q], nd.d.p[q], nd.d2.p[q], nd.b.p[q], S.part + S.part_off[q], S.scal, tmgx::S_TMP1, S.W.stream); break;
          case 12: tmgx::launch_cheb3_tb(g, nd.op[q], nd.b.p[q], nullptr, nd.d.p[q], 1.0, cs, cs2, true, S.W.stream); break;
          case 13: tmgx::launch_cheb3_tb(g, nd.op[q], nd.b.p[q], nd.d.p[q], nd.x.p[q], 1.0, cs, cs2, false, S.W.stream); break;
          case 10: tmgx::launch_prolong_to(g, S.nodes[i + 1].dist->geo[q], S.nodes[i + 1].x.p[q], nd.d.p[q], nd.r.p[q], S.W.stream); break;
          default: throw tmg::Error("unknown kernel id");
        }
      }
    };
    switch (which) {
      case 0: per_pt = 48 + kb; break;
      case 1: per_pt = 32 + kb; break;
      case 2: per_pt = 16 + kb; break;
      case 3: per_pt = 24 + kb; break;
      case 4: per_pt = 8 + 8.0 / 8.0; break;
      case 5: per_pt = 16 + 8.0 / 8.0; break;
      case 6: per_pt = 48; break;
      case 7: per_pt = 16 + kb; break;
      case 8: per_pt = 16 + kb; break;             // temporally blocked pre-smooth: b in, x out
      case 9: per_pt = 24 + kb; break;             // blocked post-smooth: x, b in, x out
      case 10: per_pt = 16 + 8.0 / 8.0; break;     // out-of-place prolongation: x, x_c in, x~ out
      case 11: per_pt = 16 + 8.0 / 8.0 + kb; break; // fused residual + restriction: b, x in, b_c out
      case 15: per_pt = 16 + 8.0 / 8.0 + kb; break; // separable fused residual + restriction (same bytes)
      case 14: per_pt = 32 + kb; break;            // fused p' = z + beta p, w = A p', p'.w: z, p in; p', w out
      case 12: per_pt = 16 + kb; break;            // blocked V(3,3) pre-smooth: b in, x out
      case 13: per_pt = 24 + kb; break;            // blocked V(3,3) post-smooth: x, b in, x out
      default: throw tmg::Error("unknown kernel id");
    }
    tmgx::cuda_check(cudaMemsetAsync(S.scal, 0, sizeof(double) * tmgx::S_NSLOTS, S.W.stream), "memset");
    for (int w = 0; w < 3; ++w) launch();
    cudaEvent_t e0, e1;
    tmgx::cuda_check(cudaEventCreate(&e0), "event");
    tmgx::cuda_check(cudaEventCreate(&e1), "event");
    tmgx::cuda_check(cudaEventRecord(e0, S.W.stream), "record");
    for (int it = 0; it < iters; ++it) launch();
    tmgx::cuda_check(cudaEventRecord(e1, S.W.stream), "record");
    tmgx::cuda_check(cudaEventSynchronize(e1), "sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    tmgx::cuda_check(cudaGetLastError(), "bench kernel");
    *ms_per_launch = ms / iters;
    *bytes_per_launch = per_pt * (double)n;
    return 0;
  });
}
