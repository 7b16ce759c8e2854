// Options database + solver-tree builder (see tmg_options.hpp; SPEC.md:597-648,
// PAPER.md:506-636). Host-only C++; no device code.
#include "tmg_options.hpp"

#include <cerrno>
#include <cstdlib>
#include <sstream>

#include "tmg_grid.hpp"

namespace tmg {

namespace {

bool looks_numeric(const std::string& t) {
  if (t.empty()) return false;
  char* end = nullptr;
  errno = 0;
  std::strtod(t.c_str(), &end);
  return end && *end == '\0';
}

}  // namespace

std::string OptionsDatabase::strip(const std::string& key) {
  size_t i = 0;
  while (i < key.size() && key[i] == '-') ++i;
  return key.substr(i);
}

void OptionsDatabase::set(const std::string& key, const std::string& value) {
  const std::string k = strip(key);
  if (k.empty()) throw ConfigError("options: empty key");
  auto it = index_.find(k);
  if (it == index_.end()) {
    index_[k] = kv_.size();
    kv_.emplace_back(k, value);
  } else {
    kv_[it->second].second = value;  // later insertions override earlier ones
  }
}

void OptionsDatabase::parse(const std::vector<std::string>& tok) {
  for (size_t i = 0; i < tok.size();) {
    const std::string& t = tok[i];
    if (t.size() < 2 || t[0] != '-' || looks_numeric(t))
      throw ConfigError("options: malformed token '" + t + "' at position " + std::to_string(i) +
                        " (expected -key)");
    const bool has_value = i + 1 < tok.size() && (tok[i + 1].empty() || tok[i + 1][0] != '-' || looks_numeric(tok[i + 1]));
    if (has_value) {
      set(t, tok[i + 1]);
      i += 2;
    } else {
      set(t, "true");
      i += 1;
    }
  }
}

void OptionsDatabase::parse_file_text(const std::string& text) {
  std::vector<std::string> tok;
  std::istringstream in(text);
  std::string line;
  while (std::getline(in, line)) {
    const size_t h = line.find('#');
    if (h != std::string::npos) line = line.substr(0, h);
    std::istringstream ls(line);
    std::string w;
    while (ls >> w) tok.push_back(w);
  }
  parse(tok);
}

bool OptionsDatabase::has(const std::string& key) const { return index_.count(strip(key)) != 0; }

std::optional<std::string> OptionsDatabase::get(const std::string& key) const {
  const std::string k = strip(key);
  auto it = index_.find(k);
  if (it == index_.end()) return std::nullopt;
  used_[k] = true;
  return kv_[it->second].second;
}

std::string OptionsDatabase::get_string(const std::string& key, const std::string& dflt) const {
  auto v = get(key);
  return v ? *v : dflt;
}

long long OptionsDatabase::get_int(const std::string& key, long long dflt) const {
  auto v = get(key);
  if (!v) return dflt;
  char* end = nullptr;
  const long long x = std::strtoll(v->c_str(), &end, 10);
  if (!end || *end != '\0' || v->empty()) throw ConfigError("options: -" + strip(key) + " expects an integer, got '" + *v + "'");
  return x;
}

double OptionsDatabase::get_real(const std::string& key, double dflt) const {
  auto v = get(key);
  if (!v) return dflt;
  char* end = nullptr;
  const double x = std::strtod(v->c_str(), &end);
  if (!end || *end != '\0' || v->empty()) throw ConfigError("options: -" + strip(key) + " expects a number, got '" + *v + "'");
  return x;
}

bool OptionsDatabase::get_bool(const std::string& key, bool dflt) const {
  auto v = get(key);
  if (!v) return dflt;
  const std::string& s = *v;
  if (s == "true" || s == "1" || s == "yes" || s == "on") return true;
  if (s == "false" || s == "0" || s == "no" || s == "off") return false;
  throw ConfigError("options: -" + strip(key) + " expects a boolean, got '" + s + "'");
}

std::vector<std::string> OptionsDatabase::unused() const {
  std::vector<std::string> out;
  for (const auto& kv : kv_)
    if (!used_.count(kv.first)) out.push_back(kv.first);
  return out;
}

std::vector<std::string> OptionsDatabase::serialize() const {
  std::vector<std::string> out;
  for (const auto& kv : kv_) {
    out.push_back("-" + kv.first);
    out.push_back(kv.second);  // flags serialise as "-key true" and reparse to the same value
  }
  return out;
}

// ------------------------------------------------------------------------------------------
// solver tree
// ------------------------------------------------------------------------------------------

namespace {

// One multigrid segment of the fused ladder (fine -> coarse), and the telescope below it.
struct Segment {
  int nlevels = 1;
  bool galerkin = false;
  int smooth_its = 2;
  int est_mode = 1;
  bool tele_below = false;
  TreeStage stage;  // level filled in when the ladder is flattened
};

struct Builder {
  const OptionsDatabase& db;
  std::vector<Segment> segs;
  std::ostringstream desc;

  // smoother of an MG segment: <p>mg_levels_ksp_type chebyshev, <p>mg_levels_pc_type jacobi
  void smoother(const std::string& p, Segment& sg, int depth) {
    const std::string lp = p + "mg_levels_";
    const std::string kt = db.get_string(lp + "ksp_type", "chebyshev");
    if (kt != "chebyshev")
      throw ConfigError("-" + lp + "ksp_type " + kt + ": the GPU smoother is chebyshev (valid: chebyshev)");
    const std::string pt = db.get_string(lp + "pc_type", "jacobi");
    if (pt == "telescope" || pt == "bjacobi" || pt == "ilu" || pt == "asm" || pt == "rasm")
      throw ConfigError("-" + lp + "pc_type " + pt +
                        ": sub-domain smoothers (PAPER.md §3.3.4-3.3.5) are out of the GPU hot path (valid: jacobi)");
    if (pt != "jacobi") throw ConfigError("-" + lp + "pc_type " + pt + ": unknown smoother preconditioner (valid: jacobi)");
    sg.smooth_its = (int)db.get_int(lp + "ksp_max_it", sg.smooth_its);  // default: inherited
    if (sg.smooth_its < 1) throw ConfigError("-" + lp + "ksp_max_it must be >= 1");
    const std::string em = db.get_string(lp + "ksp_chebyshev_estimator", sg.est_mode ? "lanczos" : "reference");
    if (em == "lanczos")
      sg.est_mode = 1;
    else if (em == "reference")
      sg.est_mode = 0;
    else
      throw ConfigError("-" + lp + "ksp_chebyshev_estimator " + em + " (valid: lanczos, reference)");
    desc << std::string(2 * depth + 2, ' ') << "levels: chebyshev(" << sg.smooth_its << ") + jacobi, estimator "
         << em << "\n";
  }

  // pc at prefix p, for a solve on the coarsest level of the segment above (inner == true) or
  // the outer operator
  void pc(const std::string& p, int depth, bool inner) {
    const std::string t = db.get_string(p + "pc_type", inner ? "lu" : "none");
    const std::string ind(2 * depth, ' ');
    if (t == "mg") {
      Segment sg;
      if (!segs.empty()) sg.smooth_its = segs.back().smooth_its, sg.est_mode = segs.back().est_mode;
      sg.nlevels = (int)db.get_int(p + "pc_mg_levels", 1);
      if (sg.nlevels < 2 && !inner)
        throw ConfigError("-" + p + "pc_mg_levels " + std::to_string(sg.nlevels) + ": multigrid needs >= 2 levels");
      if (sg.nlevels < 1) throw ConfigError("-" + p + "pc_mg_levels must be >= 1");
      sg.galerkin = db.get_bool(p + "pc_mg_galerkin", false);
      desc << ind << "pc mg: " << sg.nlevels << " levels, " << (sg.galerkin ? "galerkin" : "rediscretised")
           << " coarse operators\n";
      smoother(p, sg, depth);
      segs.push_back(sg);
      coarse(p + "mg_coarse_", depth + 1);
      return;
    }
    if (!inner) {
      if (t == "none")
        throw ConfigError("-" + p + "pc_type none: the GPU path is the MG preconditioner (valid: mg)");
      throw ConfigError("-" + p + "pc_type " + t + ": not on the GPU hot path (valid: mg)");
    }
    if (t == "lu") {  // exact solve of the level it sits on: a one-level segment
      Segment sg;
      sg.nlevels = 1;
      if (!segs.empty()) sg.smooth_its = segs.back().smooth_its, sg.est_mode = segs.back().est_mode,
                         sg.galerkin = segs.back().galerkin;
      segs.push_back(sg);
      desc << ind << "pc lu (dense LU on one rank)\n";
      return;
    }
    if (t == "gamg")
      throw ConfigError("-" + p + "pc_type gamg: smoothed aggregation is out of scope; use lu");
    throw ConfigError("-" + p + "pc_type " + t + ": unknown coarse solver (valid: lu, telescope, mg)");
  }

  // coarse solver of the MG segment just pushed: <p> = ...mg_coarse_
  void coarse(const std::string& p, int depth) {
    const std::string kt = db.get_string(p + "ksp_type", "preonly");
    if (kt != "preonly")
      throw ConfigError("-" + p + "ksp_type " + kt + ": the GPU coarse solver is applied once (valid: preonly)");
    const std::string t = db.get_string(p + "pc_type", "lu");
    const std::string ind(2 * depth, ' ');
    if (t == "lu") {
      desc << ind << "coarse: preonly + lu\n";
      return;
    }
    if (t == "telescope") {
      Segment& up = segs.back();
      up.tele_below = true;
      up.stage.reduction_factor = (int)db.get_int(p + "pc_telescope_reduction_factor", 1);
      if (up.stage.reduction_factor < 1) throw ConfigError("-" + p + "pc_telescope_reduction_factor must be >= 1");
      const char* ax[3] = {"x", "y", "z"};
      for (int a = 0; a < 3; ++a)
        up.stage.override_[a] = (int)db.get_int(p + "telescope_repart_da_processors_" + ax[a], 0);
      desc << ind << "coarse: preonly + telescope(reduction_factor " << up.stage.reduction_factor << ")\n";
      const std::string sp = p + "telescope_";
      const std::string skt = db.get_string(sp + "ksp_type", "preonly");
      if (skt != "preonly")
        throw ConfigError("-" + sp + "ksp_type " + skt + ": the telescoped sub-solve is applied once (valid: preonly)");
      pc(sp, depth + 1, true);
      return;
    }
    if (t == "gamg") throw ConfigError("-" + p + "pc_type gamg: smoothed aggregation is out of scope; use lu");
    if (t == "mg") throw ConfigError("-" + p + "pc_type mg: nest MG through telescope (valid: lu, telescope)");
    throw ConfigError("-" + p + "pc_type " + t + ": unknown coarse solver (valid: lu, telescope)");
  }
};

}  // namespace

ResolvedTree resolve_solver_tree(const OptionsDatabase& db, const std::string& prefix, const std::string& default_ksp) {
  ResolvedTree r;
  Builder b{db, {}, {}};
  const std::string kt = db.get_string(prefix + "ksp_type", default_ksp);
  if (kt == "cg")
    r.ksp_method = 2;
  else if (kt == "preonly")
    r.ksp_method = 5;
  else if (kt == "gmres" || kt == "fgmres" || kt == "richardson" || kt == "chebyshev")
    throw ConfigError("-" + prefix + "ksp_type " + kt + ": the GPU path implements cg and preonly");
  else
    throw ConfigError("-" + prefix + "ksp_type " + kt + ": unknown (valid: cg, preonly)");
  r.rtol = db.get_real(prefix + "ksp_rtol", 1e-8);
  r.atol = db.get_real(prefix + "ksp_atol", 1e-50);
  r.max_its = (int)db.get_int(prefix + "ksp_max_it", 10000);
  // PETSc's KSPSetInitialGuessNonzero; the reference's krylov_solve reads x, so nonzero by default
  r.zero_initial_guess = !db.get_bool(prefix + "ksp_initial_guess_nonzero", true);
  b.desc << "ksp " << kt << " (rtol " << r.rtol << ", atol " << r.atol << ", max_it " << r.max_its << ")\n";
  b.pc(prefix, 1, false);

  // flatten: segments fine -> coarse share their boundary level; total N1 + N2 + ... - (m - 1)
  const int m = (int)b.segs.size();
  int total = 0;
  for (const auto& s : b.segs) total += s.nlevels;
  total -= m - 1;
  r.nlevels = total;
  r.smooth_its = b.segs.front().smooth_its;
  r.est_mode = b.segs.front().est_mode;
  r.galerkin = b.segs.front().galerkin;
  for (int k = 0; k < m; ++k) {
    const auto& s = b.segs[k];
    if (s.nlevels > 1 && (s.smooth_its != r.smooth_its || s.est_mode != r.est_mode))
      throw ConfigError("options: the GPU hierarchy uses one smoother configuration on every level");
    if (s.nlevels > 1 && k > 0 && s.galerkin != r.galerkin)
      throw ConfigError("options: mixed rediscretised / galerkin segments are not supported on the GPU path");
  }
  // the stage between segments k and k+1 sits on the finest level of the fused ladder below
  // segment k: sum_{j>k} N_j - (m - k - 2) levels, so its index is that count minus one
  for (int k = 0; k < m - 1; ++k) {
    if (!b.segs[k].tele_below) continue;
    int count = 0;
    for (int j = k + 1; j < m; ++j) count += b.segs[j].nlevels;
    count -= m - k - 2;
    TreeStage st = b.segs[k].stage;
    st.level = count - 1;
    r.stages.push_back(st);
  }
  std::ostringstream d;
  d << b.desc.str() << "fused ladder: " << r.nlevels << " levels";
  for (const auto& st : r.stages) d << ", telescope r=" << st.reduction_factor << " at level " << st.level;
  d << "\n";
  r.describe = d.str();
  return r;
}

}  // namespace tmg
