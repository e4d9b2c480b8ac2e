#pragma once
#include <vector>

namespace smc {

enum class NodeKind { GaussLobatto, ClenshawCurtis, Composite };
struct Segment {
  int first = 0, last = 0;
};

// Quadrature nodes on [0, 1] incl. both endpoints (quadrature.hpp:19-29).
struct Nodes {
  std::vector<double> t;
  NodeKind kind = NodeKind::GaussLobatto;
  std::vector<Segment> segments;
  int count() const { return static_cast<int>(t.size()); }
  int intervals() const { return count() - 1; }
};

// Row-major dense table.
struct Table {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Table() = default;
  Table(int r, int c) : rows(r), cols(c), a(static_cast<std::size_t>(r) * c, 0.0) {}
  double& operator()(int r, int c) { return a[static_cast<std::size_t>(r) * cols + c]; }
  double operator()(int r, int c) const { return a[static_cast<std::size_t>(r) * cols + c]; }
};

struct SweepTables {
  Table q, s;  // M x (M+1)
};

struct Hierarchy {
  Nodes coarse, fine;
  Table q21, s21, q22, s22;
  std::vector<int> fine_of_coarse, p_map;
};

Nodes gauss_lobatto(int n);
Nodes clenshaw_curtis(int n);
Nodes make_nodes(int family, int n);  // 0 = Gauss-Lobatto, 1 = Clenshaw-Curtis
SweepTables integration_matrices(const Nodes& nodes);
// TypeB (repeats == 1) / TypeC fine levels (quadrature.hpp:56-67); repeats
// == 0 is TypeA: `inner` is the fine set and must contain the coarse nodes.
Hierarchy build_hierarchy(const Nodes& coarse, const Nodes& inner, int repeats);

}  // namespace smc
