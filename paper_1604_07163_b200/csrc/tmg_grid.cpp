// Host-side structured-grid maps; see tmg_grid.hpp for the reference citations.
#include "tmg_grid.hpp"

#include <algorithm>

namespace tmg {

Layout Layout::from_sizes(const std::vector<idx_t>& sizes) {
  Layout lay;
  lay.offsets.assign(sizes.size() + 1, 0);
  for (size_t k = 0; k < sizes.size(); ++k) lay.offsets[k + 1] = lay.offsets[k] + sizes[k];
  lay.n = lay.offsets.back();
  return lay;
}

GridBox intersect(const GridBox& a, const GridBox& b) {
  GridBox r;
  for (int x = 0; x < 3; ++x) {
    r.lo[x] = std::max(a.lo[x], b.lo[x]);
    r.hi[x] = std::max(r.lo[x], std::min(a.hi[x], b.hi[x]));
  }
  return r;
}

std::array<int, 3> GridHeader::proc_coords(int rank) const {
  return {rank % proc_grid[0], (rank / proc_grid[0]) % proc_grid[1], rank / (proc_grid[0] * proc_grid[1])};
}

GridBox GridHeader::box(int rank) const {
  const auto pc = proc_coords(rank);
  GridBox b;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = axis_offsets[a][static_cast<size_t>(pc[a])];
    b.hi[a] = axis_offsets[a][static_cast<size_t>(pc[a]) + 1];
  }
  return b;
}

Layout GridHeader::layout() const {
  std::vector<idx_t> sizes;
  for (int r = 0; r < n_ranks(); ++r) sizes.push_back(box(r).n_vertices() * dof);
  return Layout::from_sizes(sizes);
}

idx_t GridHeader::global_index(idx_t i, idx_t j, idx_t k, int c) const {
  const idx_t ijk[3] = {i, j, k};
  int pc[3];
  for (int a = 0; a < 3; ++a) {
    const auto& off = axis_offsets[a];
    pc[a] = static_cast<int>(std::upper_bound(off.begin(), off.end(), ijk[a]) - off.begin()) - 1;
  }
  const int rank = proc_rank(pc[0], pc[1], pc[2]);
  const GridBox b = box(rank);
  const idx_t v = (i - b.lo[0]) + b.extent(0) * ((j - b.lo[1]) + b.extent(1) * (k - b.lo[2]));
  idx_t offset = 0;
  for (int r = 0; r < rank; ++r) offset += box(r).n_vertices() * dof;
  return offset + v * dof + c;
}

idx_t GridHeader::natural_to_global(idx_t natural) const {
  const int c = static_cast<int>(natural % dof);
  idx_t v = natural / dof;
  const idx_t i = v % npoints[0];
  v /= npoints[0];
  const idx_t j = v % npoints[1];
  return global_index(i, j, v / npoints[1], c);
}

idx_t GridHeader::global_to_natural(idx_t global) const {
  idx_t offset = 0;
  int rank = 0;
  for (; rank < n_ranks(); ++rank) {
    const idx_t sz = box(rank).n_vertices() * dof;
    if (global < offset + sz) break;
    offset += sz;
  }
  const GridBox b = box(rank);
  const idx_t local = global - offset;
  const int c = static_cast<int>(local % dof);
  idx_t v = local / dof;
  const idx_t i = b.lo[0] + v % b.extent(0);
  v /= b.extent(0);
  const idx_t j = b.lo[1] + v % b.extent(1);
  return natural_index(i, j, b.lo[2] + v / b.extent(1), c);
}

std::vector<idx_t> split_axis(idx_t n, int parts) {
  std::vector<idx_t> off(static_cast<size_t>(parts) + 1, 0);
  const idx_t base = n / parts, rem = n % parts;
  for (int p = 0; p < parts; ++p) off[static_cast<size_t>(p) + 1] = off[static_cast<size_t>(p)] + base + (p < rem);
  return off;
}

namespace {
void factorizations(int size, int dim, std::array<int, 3> cur, int axis, std::vector<std::array<int, 3>>& out) {
  if (axis == dim - 1) {
    cur[axis] = size;
    out.push_back(cur);
    return;
  }
  for (int f = 1; f <= size; ++f) {
    if (size % f) continue;
    cur[axis] = f;
    factorizations(size / f, dim, cur, axis + 1, out);
  }
}
}  // namespace

std::array<int, 3> choose_proc_grid(int size, int dim, const std::array<idx_t, 3>& npoints) {
  std::vector<std::array<int, 3>> cands;
  factorizations(size, dim, {1, 1, 1}, 0, cands);
  std::optional<std::array<int, 3>> best;
  double best_cost = 0.0;
  for (const auto& pg : cands) {
    bool feasible = true;
    double cost = 0.0;
    for (int a = 0; a < dim; ++a) {
      if (pg[a] > npoints[a]) feasible = false;
      cost += static_cast<double>(pg[a]) / static_cast<double>(npoints[a]);
    }
    if (!feasible) continue;
    if (!best || cost < best_cost - 1e-15) {
      best = pg;
      best_cost = cost;
    } else if (cost < best_cost + 1e-15) {
      for (int a = dim - 1; a >= 0; --a)
        if (pg[a] != (*best)[a]) {
          if (pg[a] > (*best)[a]) best = pg;
          break;
        }
    }
  }
  if (!best)
    throw ConfigError("create_grid: over-decomposed (no factorization of " + std::to_string(size) +
                      " ranks fits the grid)");
  return *best;
}

GridHeader make_header(int dim, std::array<idx_t, 3> npoints, int dof, int stencil_width,
                       std::array<int, 3> proc_grid) {
  GridHeader h;
  h.dim = dim;
  h.npoints = npoints;
  h.dof = dof;
  h.stencil_width = stencil_width;
  h.proc_grid = proc_grid;
  for (int a = 0; a < 3; ++a) h.axis_offsets[a] = split_axis(npoints[a], proc_grid[a]);
  return h;
}

GridHeader build_header_for(int comm_size, int dim, std::array<idx_t, 3> npoints, int dof, int stencil_width,
                            std::optional<std::array<int, 3>> hint) {
  if (dim < 1 || dim > 3) throw ConfigError("grid dimension must be 1, 2 or 3");
  if (dof < 1) throw ConfigError("dof must be positive");
  for (int a = dim; a < 3; ++a)
    if (npoints[a] != 1) throw ConfigError("trailing axes of a grid must hold 1 point");
  for (int a = 0; a < dim; ++a)
    if (npoints[a] < 1) throw ConfigError("npoints must be positive");
  std::array<int, 3> pg{1, 1, 1};
  if (hint) {
    pg = *hint;
    if (pg[0] * pg[1] * pg[2] != comm_size)
      throw ConfigError("create_grid: processor grid hint does not multiply to the communicator size");
    for (int a = 0; a < 3; ++a)
      if (pg[a] > npoints[a]) throw ConfigError("create_grid: over-decomposed (axis " + std::to_string(a) + ")");
  } else {
    pg = choose_proc_grid(comm_size, dim, npoints);
  }
  return make_header(dim, npoints, dof, stencil_width, pg);
}

std::optional<GridHeader> try_coarsen_header(const GridHeader& fine) {
  GridHeader coarse = fine;
  for (int a = 0; a < fine.dim; ++a) {
    const idx_t n = fine.npoints[a];
    if (n == 1) continue;
    if (n < 3 || n % 2 == 0) return std::nullopt;
    coarse.npoints[a] = (n + 1) / 2;
  }
  for (int a = 0; a < 3; ++a) {
    if (fine.npoints[a] == coarse.npoints[a]) continue;
    auto& off = coarse.axis_offsets[a];
    for (auto& v : off) v = (v + 1) / 2;
    for (size_t p = 0; p + 1 < off.size(); ++p)
      if (off[p + 1] <= off[p]) return std::nullopt;
  }
  return coarse;
}

SplitResult split_strided(int parent_size, int r) {
  if (r < 1) throw ConfigError("split_strided: reduction factor must be >= 1");
  SplitResult s;
  s.reduction_factor = r;
  s.parent_size = parent_size;
  for (int k = 0; k < parent_size; k += r) s.member_map.push_back(k);
  return s;
}

GridHeader repartition_header(const GridHeader& h, int sub_size, const std::array<std::optional<int>, 3>& ov) {
  bool any = false;
  for (const auto& o : ov) any |= o.has_value();
  if (!any && sub_size == h.n_ranks()) return h;
  if (!any) return build_header_for(sub_size, h.dim, h.npoints, h.dof, h.stencil_width, std::nullopt);
  std::array<int, 3> fixed{0, 0, 0};
  int fixed_prod = 1, n_free = 0;
  for (int a = 0; a < 3; ++a) {
    if (ov[a]) {
      fixed[a] = *ov[a];
      if (fixed[a] < 1) throw ConfigError("repartition_onto: processor override must be positive");
      fixed_prod *= fixed[a];
    } else if (a < h.dim) {
      ++n_free;
    } else {
      fixed[a] = 1;
    }
  }
  if (fixed_prod > sub_size || sub_size % fixed_prod)
    throw ConfigError("repartition_onto: processor overrides do not divide the " + std::to_string(sub_size) +
                      "-rank sub-communicator");
  std::array<int, 3> pg = fixed;
  if (n_free == 0) {
    if (fixed_prod != sub_size)
      throw ConfigError("repartition_onto: processor override product must equal the sub-communicator size");
  } else {
    std::array<idx_t, 3> free_np{1, 1, 1};
    std::vector<int> free_axes;
    for (int a = 0; a < h.dim; ++a)
      if (!ov[a]) {
        free_axes.push_back(a);
        free_np[free_axes.size() - 1] = h.npoints[a];
      }
    const auto chosen = choose_proc_grid(sub_size / fixed_prod, static_cast<int>(free_axes.size()), free_np);
    for (size_t t = 0; t < free_axes.size(); ++t) pg[free_axes[t]] = chosen[t];
  }
  for (int a = 0; a < 3; ++a)
    if (pg[a] > h.npoints[a]) throw ConfigError("repartition_onto: over-decomposed on axis " + std::to_string(a));
  return make_header(h.dim, h.npoints, h.dof, h.stencil_width, pg);
}

Layout prefusion_layout(const GridHeader& new_header, const SplitResult& split) {
  const Layout dst = new_header.layout();
  std::vector<idx_t> sizes(static_cast<size_t>(split.parent_size), 0);
  for (int m = 0; m < split.n_members(); ++m) {
    const idx_t rows = dst.local_size(m);
    const int gb = split.group_begin(m), ge = split.group_end(m), width = ge - gb;
    const idx_t base = rows / width, rem = rows % width;
    for (int p = gb; p < ge; ++p) sizes[static_cast<size_t>(p)] = base + ((p - gb) < rem);
  }
  return Layout::from_sizes(sizes);
}

}  // namespace tmg
