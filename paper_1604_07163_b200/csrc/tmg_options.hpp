// Prefix-keyed runtime options database and the solver-tree builder for the GPU MG-CG path.
//
// The reference's options.cpp / solver_build.cpp are missing from /root/reference; this follows
// the module spec and the option boxes of the paper:
//   OptionsDatabase   ordered key -> string map, leading dash stripped, flags = "true",
//                     later insertions win, exact-match lookup, used-key tracking
//   parse(argv)       "-key [value]" tokens; a "-" token followed by another "-key" token or
//                     the end is a flag; malformed tokens -> ConfigError with the position
//   build tree        KSP/PC pairs by prefix concatenation: <p>ksp_*, <p>pc_*, MG smoothers
//                     under <p>mg_levels_, the MG coarse solver under <p>mg_coarse_, the
//                     Telescope sub-solver under <p>..telescope_ (so the depth-3 key
//                     -mg_coarse_telescope_mg_coarse_pc_type resolves exactly as in the paper)
// The resolved tree is flattened onto the GPU hierarchy (one fused level ladder with telescope
// stages, SPEC.md:472-490 / PAPER.md:537 "N1 + N2 - 1 levels"). Configurations the GPU path does
// not implement (GMRES, bjacobi/ILU smoothers, gamg, smoother-side telescope) are rejected with
// a ConfigError naming the supported set.
#pragma once

#include <map>
#include <optional>
#include <string>
#include <vector>

namespace tmg {

class OptionsDatabase {
 public:
  // "-a 1 -b -c x" style tokens (argv without the program name); throws ConfigError on a
  // malformed token. Values may be negative numbers ("-shift -0.5").
  void parse(const std::vector<std::string>& tokens);
  // options file: one "-key value" (or "-flag") per line, '#' starts a comment
  void parse_file_text(const std::string& text);
  void set(const std::string& key, const std::string& value);  // key with or without the dash
  bool has(const std::string& key) const;
  std::optional<std::string> get(const std::string& key) const;  // marks the key used
  std::string get_string(const std::string& key, const std::string& dflt) const;
  long long get_int(const std::string& key, long long dflt) const;
  double get_real(const std::string& key, double dflt) const;
  bool get_bool(const std::string& key, bool dflt) const;
  std::vector<std::string> unused() const;      // keys never looked up
  std::vector<std::string> serialize() const;   // tokens that reparse to an equal database
  const std::vector<std::pair<std::string, std::string>>& entries() const { return kv_; }
  size_t size() const { return kv_.size(); }

 private:
  static std::string strip(const std::string& key);
  std::vector<std::pair<std::string, std::string>> kv_;  // insertion order of first definition
  std::map<std::string, size_t> index_;
  mutable std::map<std::string, bool> used_;
};

// One telescope stage of the flattened ladder (level 0 = coarsest).
struct TreeStage {
  int level = 0;
  int reduction_factor = 1;
  int override_[3] = {0, 0, 0};
};

// The tree resolved onto the GPU path.
struct ResolvedTree {
  int ksp_method = 2;  // TMGX_KSP_CG / TMGX_KSP_PREONLY
  double rtol = 1e-8, atol = 1e-50;
  int max_its = 10000;
  bool zero_initial_guess = false;  // -ksp_initial_guess_nonzero false
  int nlevels = 1;
  int smooth_its = 2;
  int est_mode = 1;  // TMGX_EST_LANCZOS
  bool galerkin = false;
  std::vector<TreeStage> stages;
  std::string describe;  // indented tree, one node per line
};

// build_solver_tree: resolve <prefix>ksp_type / <prefix>pc_type recursively.
// default_ksp: the outer KSP type when <prefix>ksp_type is unset (the reference's default is
// gmres, which the GPU path rejects; harness presets pass "cg").
ResolvedTree resolve_solver_tree(const OptionsDatabase& db, const std::string& prefix,
                                 const std::string& default_ksp = "gmres");

}  // namespace tmg
