// Internal (not part of the C ABI): the full RVE discretisation that the
// offline high-fidelity solver (hf.cu) and the basis-driven model build need.
// Built by setup.cpp from the same mesh code as the seeded models, so node,
// element and free-DOF numbering agree with fe2_model_build everywhere.
#pragma once

#include <cstdint>
#include <vector>

namespace fe2 {

struct RveData {
  int n_nodes = 0, n_el = 0, n_free = 0;
  std::vector<double> x, y;        // node coordinates
  std::vector<int> conn;           // [n_el][6] tri6 node ids
  std::vector<int> phase;          // [n_el] material id (0 matrix, 1 inclusion)
  std::vector<int> free_index;     // [2 n_nodes] free number, -1 on the boundary (linear BC, rve.hpp:84-92)
  std::vector<double> B;           // [3 n_el][3][12] strain operator per integration point
  std::vector<double> w;           // [3 n_el] w_g detJ (rve.hpp:178-181)
  double volume = 0.0;
  int n_dofs() const { return 2 * n_nodes; }
  int n_ips() const { return 3 * n_el; }
};

// default_cell(subdivisions) when mesh_path is null, else the mesh file.
RveData rve_data(int subdivisions, const char* mesh_path);

// Modified Gram-Schmidt, twice, over the columns of A (column-major,
// column j at A + j*rows). Columns whose remaining norm is <= drop_tol[j]
// are removed; returns the number of columns kept (compacted to the front).
int orthonormalize_columns(std::vector<double>& A, std::int64_t rows, int cols, const std::vector<double>& drop_tol);

}  // namespace fe2
