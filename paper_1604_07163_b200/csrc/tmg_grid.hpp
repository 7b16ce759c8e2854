// Host-side structured-grid maps (DMDA analog) for the B200 MG path.
//
// B200-native restatement of the reference's index arithmetic. Everything here is
// integer work on the host and must be bit-exact with the reference:
//   Layout            layout.hpp:14-33, layout.cpp:9-39
//   GridHeader maps   grid.hpp:41-79, grid.cpp:17-115
//   choose_proc_grid  grid.cpp:209-240 ; split_axis grid.cpp:184-193
//   coarsen           grid.cpp:299-322
//   repartition       grid.cpp:433-493 ; prefusion_layout grid.cpp:566-580
//   split_strided     comm.cpp:353-390 ; SplitResult comm.hpp:57-71, comm.cpp:161-173
// The device side never sees these structures: it receives per-box geometry (Box) only.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace tmg {

using idx_t = std::int64_t;

// common.hpp:16-34 error taxonomy; mapped onto C-ABI status codes in tmgx_capi.cu.
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class CudaError : public Error {
 public:
  using Error::Error;
};

struct Layout {
  idx_t n = 0;
  std::vector<idx_t> offsets;
  int n_ranks() const { return static_cast<int>(offsets.size()) - 1; }
  idx_t begin(int r) const { return offsets[static_cast<size_t>(r)]; }
  idx_t end(int r) const { return offsets[static_cast<size_t>(r) + 1]; }
  idx_t local_size(int r) const { return end(r) - begin(r); }
  static Layout from_sizes(const std::vector<idx_t>& sizes);
  bool operator==(const Layout&) const = default;
};

struct GridBox {
  std::array<idx_t, 3> lo{0, 0, 0};
  std::array<idx_t, 3> hi{0, 0, 0};
  idx_t extent(int a) const { return hi[a] - lo[a]; }
  idx_t n_vertices() const { return extent(0) * extent(1) * extent(2); }
  bool empty() const { return extent(0) <= 0 || extent(1) <= 0 || extent(2) <= 0; }
};

GridBox intersect(const GridBox& a, const GridBox& b);

struct GridHeader {
  int dim = 3;
  std::array<idx_t, 3> npoints{1, 1, 1};
  int dof = 1;
  int stencil_width = 1;
  std::array<int, 3> proc_grid{1, 1, 1};
  std::array<std::vector<idx_t>, 3> axis_offsets;

  int n_ranks() const { return proc_grid[0] * proc_grid[1] * proc_grid[2]; }
  idx_t n_vertices() const { return npoints[0] * npoints[1] * npoints[2]; }
  idx_t n_unknowns() const { return n_vertices() * dof; }
  std::array<int, 3> proc_coords(int rank) const;
  int proc_rank(int pi, int pj, int pk) const { return pi + proc_grid[0] * (pj + proc_grid[1] * pk); }
  GridBox box(int rank) const;
  Layout layout() const;
  idx_t natural_index(idx_t i, idx_t j, idx_t k, int c) const {
    return c + dof * (i + npoints[0] * (j + npoints[1] * k));
  }
  idx_t global_index(idx_t i, idx_t j, idx_t k, int c) const;
  idx_t natural_to_global(idx_t natural) const;
  idx_t global_to_natural(idx_t global) const;
  bool same_global_grid(const GridHeader& o) const {
    return dim == o.dim && npoints == o.npoints && dof == o.dof;
  }
  bool operator==(const GridHeader&) const = default;
};

struct SplitResult {
  std::vector<int> member_map;  // parent ranks of members, strictly increasing
  int reduction_factor = 1;
  int parent_size = 0;
  int n_members() const { return static_cast<int>(member_map.size()); }
  int group_begin(int m) const { return member_map[static_cast<size_t>(m)]; }
  int group_end(int m) const {
    return static_cast<size_t>(m) + 1 < member_map.size() ? member_map[static_cast<size_t>(m) + 1] : parent_size;
  }
  bool is_member(int parent_rank) const { return parent_rank % reduction_factor == 0; }
};

std::vector<idx_t> split_axis(idx_t n, int parts);
std::array<int, 3> choose_proc_grid(int size, int dim, const std::array<idx_t, 3>& npoints);
GridHeader make_header(int dim, std::array<idx_t, 3> npoints, int dof, int stencil_width,
                       std::array<int, 3> proc_grid);
GridHeader build_header_for(int comm_size, int dim, std::array<idx_t, 3> npoints, int dof, int stencil_width,
                            std::optional<std::array<int, 3>> hint);
std::optional<GridHeader> try_coarsen_header(const GridHeader& fine);
SplitResult split_strided(int parent_size, int r);
GridHeader repartition_header(const GridHeader& h, int sub_size, const std::array<std::optional<int>, 3>& ov);
Layout prefusion_layout(const GridHeader& new_header, const SplitResult& split);

}  // namespace tmg
