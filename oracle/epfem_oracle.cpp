// =============================================================================
// TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT.
//
// CPU restatement of the epfem reference hot path (constitutive update +
// tangent-stiffness assembly), used exclusively by tests/, by
// __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
// `--impl reference` leg.  The product (paper_1805_04155_b200/, libepfem_gpu.so)
// never links or calls this file.
//
// Why a restatement: the reference (/root/reference/proj) needs Eigen >= 3.3,
// doctest and CLI11, none of which exist in this image (no network), so it
// cannot be compiled.  This file restates the reference
// algorithm with Eigen's arithmetic made explicit:
//   * setFromTriplets: duplicates summed in triplet order, explicit zeros kept,
//     inner indices sorted                          (linalg.cpp:10-26)
//   * conservative sparse*sparse product: for column j of rhs, for k ascending
//     in rhs(:,j), for i in lhs(:,k): first touch assigns x*y, later touches add
//                                                   (linalg.cpp:28-35)
//   * sparse + sparse: union of patterns, no pruning (assembly.cpp:212)
// Built with -O2 -ffp-contract=off (the reference's Release build adds no
// -march, so x86-64 SSE2 without FMA: proj/CMakeLists.txt:7-9).
//
// Pinning: tests/test_oracle_pin.py checks this restatement against the
// reference's own known-answer tests and its independent in-test oracles
// (tensor-space vm_oracle/dp_oracle, tests/test_constitutive.cpp:59-120;
// dense element-loop K oracle, tests/test_assembly.cpp:38-98) on the same
// std::mt19937 seeds (fixtures from tests/golden/gen_golden.cpp).
// Eigen's SIMD reduction order inside fixed-size 6x6 expressions is not
// reproducible without Eigen, so S/D/K may differ from a real Eigen build in
// the last ulp; the parity tolerances (1e-12) cover that.
// =============================================================================
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace orc {

// Element families in the order of epfem::ElementFamily
// (reference_elements.hpp:10).
enum Family { P1 = 0, P2 = 1, Q1 = 2, Q2 = 3 };

thread_local std::string g_err;

int node_count(int family, int dim) {  // reference_elements.cpp:326-335
  static const int tab[4][2] = {{3, 4}, {6, 10}, {4, 8}, {8, 20}};
  if ((dim != 2 && dim != 3) || family < 0 || family > 3) return -1;
  return tab[family][dim - 2];
}

// ---------------------------------------------------------------------------
// Quadrature rules (reference_elements.cpp:20-84, 345-374).  Points are stored
// dim x n_q column-major, like the reference's Mat.
struct Rule {
  int dim = 0, nq = 0;
  std::vector<double> pts, w;
};

static void gauss1d(int n, std::vector<double>& x, std::vector<double>& w) {
  if (n == 1) {
    x = {0.0};
    w = {2.0};
  } else if (n == 2) {
    const double g = 1.0 / std::sqrt(3.0);
    x = {-g, g};
    w = {1.0, 1.0};
  } else {
    const double g = std::sqrt(3.0 / 5.0);
    x = {-g, 0.0, g};
    w = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
  }
}

// Tensor-product Gauss rule: axis 0 varies fastest; weight is the running
// product w_0 * w_1 (* w_2) starting from 1.0 (reference_elements.cpp:47-65).
static Rule tensor_gauss(int dim, int n1) {
  std::vector<double> x, w;
  gauss1d(n1, x, w);
  Rule r;
  r.dim = dim;
  r.nq = dim == 2 ? n1 * n1 : n1 * n1 * n1;
  r.pts.resize(dim * r.nq);
  r.w.resize(r.nq);
  for (int q = 0; q < r.nq; ++q) {
    int rest = q;
    double acc = 1.0;
    for (int ax = 0; ax < dim; ++ax) {
      const int k = rest % n1;
      rest /= n1;
      r.pts[q * dim + ax] = x[k];
      acc *= w[k];
    }
    r.w[q] = acc;
  }
  return r;
}

Rule quadrature(int family, int dim) {
  Rule r;
  r.dim = dim;
  if (family == P1) {
    r.nq = 1;
    if (dim == 3) {
      r.pts = {0.25, 0.25, 0.25};
      r.w = {1.0 / 6.0};
    } else {
      r.pts = {1.0 / 3.0, 1.0 / 3.0};
      r.w = {0.5};
    }
  } else if (family == P2) {
    if (dim == 3) {
      // 11-point degree-4 Keast rule; the paper's truncated 15-digit
      // constants, with one negative weight (reference_elements.cpp:68-84).
      const double A = 0.399403576166799, B = 0.100596423833201;
      const double F = 0.071428571428571, G = 0.785714285714286;
      const double W1 = -0.013155555555555, W2 = 0.007622222222222,
                   W3 = 0.024888888888888;
      const double xs[11] = {0.25, F, G, F, F, A, B, B, A, A, B};
      const double ys[11] = {0.25, F, F, G, F, B, A, B, A, B, A};
      const double zs[11] = {0.25, F, F, F, G, B, B, A, B, A, A};
      r.nq = 11;
      r.pts.resize(33);
      for (int q = 0; q < 11; ++q) {
        r.pts[3 * q] = xs[q];
        r.pts[3 * q + 1] = ys[q];
        r.pts[3 * q + 2] = zs[q];
      }
      r.w = {W1, W2, W2, W2, W2, W3, W3, W3, W3, W3, W3};
    } else {
      r.nq = 3;  // edge midpoints
      r.pts = {0.5, 0.0, 0.5, 0.5, 0.0, 0.5};
      r.w = {1.0 / 6.0, 1.0 / 6.0, 1.0 / 6.0};
    }
  } else if (family == Q1) {
    r = tensor_gauss(dim, 2);
  } else {
    r = tensor_gauss(dim, 3);
  }
  return r;
}

// ---------------------------------------------------------------------------
// Shape-function values and reference gradients (reference_elements.cpp
// :117-304).  vals[p + np*q]; grad[(d*np + p)*m + q]... stored as
// grad[d][p][q] flattened = ((d * np) + p) * m + q.
struct Basis {
  int np = 0, m = 0, dim = 0;
  std::vector<double> vals, grad;
  double& V(int p, int q) { return vals[(size_t)p * m + q]; }
  double& D(int d, int p, int q) { return grad[((size_t)d * np + p) * m + q]; }
};

static const int kQC[4][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}};
static const int kQE[4][2] = {{0, -1}, {1, 0}, {0, 1}, {-1, 0}};
static const int kHC[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1},
                              {-1, 1, -1},  {-1, -1, 1}, {1, -1, 1},
                              {1, 1, 1},    {-1, 1, 1}};
static const int kHE[12][3] = {{0, -1, -1}, {1, 0, -1},  {0, 1, -1},
                               {-1, 0, -1}, {0, -1, 1},  {1, 0, 1},
                               {0, 1, 1},   {-1, 0, 1},  {-1, -1, 0},
                               {1, -1, 0},  {1, 1, 0},   {-1, 1, 0}};

Basis basis(int family, int dim, const double* pts, int m) {
  Basis b;
  b.np = node_count(family, dim);
  b.m = m;
  b.dim = dim;
  b.vals.assign((size_t)b.np * m, 0.0);
  b.grad.assign((size_t)dim * b.np * m, 0.0);
  for (int q = 0; q < m; ++q) {
    const double* X = pts + (size_t)dim * q;
    if (dim == 2 && family == P1) {
      const double x = X[0], y = X[1];
      b.V(0, q) = 1.0 - x - y;
      b.V(1, q) = x;
      b.V(2, q) = y;
      const double g0[3] = {-1, 1, 0}, g1[3] = {-1, 0, 1};
      for (int p = 0; p < 3; ++p) {
        b.D(0, p, q) = g0[p];
        b.D(1, p, q) = g1[p];
      }
    } else if (dim == 2 && family == P2) {
      const double x = X[0], y = X[1];
      const double z = 1.0 - x - y;
      const double v[6] = {z * (2 * z - 1), x * (2 * x - 1), y * (2 * y - 1),
                           4 * z * x,       4 * x * y,       4 * z * y};
      const double g0[6] = {1 - 4 * z, 4 * x - 1, 0, 4 * (z - x), 4 * y, -4 * y};
      const double g1[6] = {1 - 4 * z, 0, 4 * y - 1, -4 * x, 4 * x, 4 * (z - y)};
      for (int p = 0; p < 6; ++p) {
        b.V(p, q) = v[p];
        b.D(0, p, q) = g0[p];
        b.D(1, p, q) = g1[p];
      }
    } else if (dim == 3 && family == P1) {
      const double x = X[0], y = X[1], z = X[2];
      const double v[4] = {1.0 - x - y - z, x, y, z};
      const double g[3][4] = {{-1, 1, 0, 0}, {-1, 0, 1, 0}, {-1, 0, 0, 1}};
      for (int p = 0; p < 4; ++p) {
        b.V(p, q) = v[p];
        for (int d = 0; d < 3; ++d) b.D(d, p, q) = g[d][p];
      }
    } else if (dim == 3 && family == P2) {
      const double x1 = X[0], x2 = X[1], x3 = X[2];
      const double x0 = 1.0 - x1 - x2 - x3;
      const double v[10] = {x0 * (2 * x0 - 1), x1 * (2 * x1 - 1),
                            x2 * (2 * x2 - 1), x3 * (2 * x3 - 1),
                            4 * x0 * x1,       4 * x1 * x2,
                            4 * x0 * x2,       4 * x1 * x3,
                            4 * x2 * x3,       4 * x0 * x3};
      const double g[3][10] = {
          {1 - 4 * x0, 4 * x1 - 1, 0, 0, 4 * (x0 - x1), 4 * x2, -4 * x2,
           4 * x3, 0, -4 * x3},
          {1 - 4 * x0, 0, 4 * x2 - 1, 0, -4 * x1, 4 * x1, 4 * (x0 - x2), 0,
           4 * x3, -4 * x3},
          {1 - 4 * x0, 0, 0, 4 * x3 - 1, -4 * x1, 0, -4 * x2, 4 * x1, 4 * x2,
           4 * (x0 - x3)}};
      for (int p = 0; p < 10; ++p) {
        b.V(p, q) = v[p];
        for (int d = 0; d < 3; ++d) b.D(d, p, q) = g[d][p];
      }
    } else if (dim == 2 && family == Q1) {
      const double x = X[0], y = X[1];
      for (int p = 0; p < 4; ++p) {
        const double sx = kQC[p][0], sy = kQC[p][1];
        b.V(p, q) = 0.25 * (1 + sx * x) * (1 + sy * y);
        b.D(0, p, q) = 0.25 * sx * (1 + sy * y);
        b.D(1, p, q) = 0.25 * sy * (1 + sx * x);
      }
    } else if (dim == 2 && family == Q2) {
      const double x = X[0], y = X[1];
      for (int p = 0; p < 4; ++p) {
        const double sx = kQC[p][0], sy = kQC[p][1];
        const double ax = 1 + sx * x, ay = 1 + sy * y;
        const double r = sx * x + sy * y - 1;
        b.V(p, q) = 0.25 * ax * ay * r;
        b.D(0, p, q) = 0.25 * sx * (ay * r + ax * ay);
        b.D(1, p, q) = 0.25 * sy * (ax * r + ax * ay);
      }
      for (int p = 0; p < 4; ++p) {
        const int sx = kQE[p][0], sy = kQE[p][1];
        if (sx == 0) {
          b.V(4 + p, q) = 0.5 * (1 - x * x) * (1 + sy * y);
          b.D(0, 4 + p, q) = -x * (1 + sy * y);
          b.D(1, 4 + p, q) = 0.5 * sy * (1 - x * x);
        } else {
          b.V(4 + p, q) = 0.5 * (1 + sx * x) * (1 - y * y);
          b.D(0, 4 + p, q) = 0.5 * sx * (1 - y * y);
          b.D(1, 4 + p, q) = -y * (1 + sx * x);
        }
      }
    } else if (dim == 3 && family == Q1) {
      const double x = X[0], y = X[1], z = X[2];
      for (int p = 0; p < 8; ++p) {
        const double sx = kHC[p][0], sy = kHC[p][1], sz = kHC[p][2];
        const double ax = 1 + sx * x, ay = 1 + sy * y, az = 1 + sz * z;
        b.V(p, q) = 0.125 * ax * ay * az;
        b.D(0, p, q) = 0.125 * sx * ay * az;
        b.D(1, p, q) = 0.125 * sy * ax * az;
        b.D(2, p, q) = 0.125 * sz * ax * ay;
      }
    } else {  // 3D Q2 serendipity
      const double x = X[0], y = X[1], z = X[2];
      for (int p = 0; p < 8; ++p) {
        const double sx = kHC[p][0], sy = kHC[p][1], sz = kHC[p][2];
        const double ax = 1 + sx * x, ay = 1 + sy * y, az = 1 + sz * z;
        const double r = sx * x + sy * y + sz * z - 2;
        b.V(p, q) = 0.125 * ax * ay * az * r;
        b.D(0, p, q) = 0.125 * sx * ay * az * (r + ax);
        b.D(1, p, q) = 0.125 * sy * ax * az * (r + ay);
        b.D(2, p, q) = 0.125 * sz * ax * ay * (r + az);
      }
      const double c[3] = {x, y, z};
      for (int p = 0; p < 12; ++p) {
        double v[3], d[3];
        for (int i = 0; i < 3; ++i) {
          const int s = kHE[p][i];
          if (s == 0) {
            v[i] = 1 - c[i] * c[i];
            d[i] = -2 * c[i];
          } else {
            v[i] = 1 + s * c[i];
            d[i] = s;
          }
        }
        b.V(8 + p, q) = 0.25 * v[0] * v[1] * v[2];
        b.D(0, 8 + p, q) = 0.25 * d[0] * v[1] * v[2];
        b.D(1, 8 + p, q) = 0.25 * v[0] * d[1] * v[2];
        b.D(2, 8 + p, q) = 0.25 * v[0] * v[1] * d[2];
      }
    }
  }
  return b;
}

// ---------------------------------------------------------------------------
// Structured mesh numbering (mesh.cpp:36-210): fine grid at half spacing,
// nodes numbered (z, y, x)-lexicographically over used fine points, elements
// in cell order (k, j, i) then pattern order.

static std::vector<std::vector<std::array<int, 3>>> cell_patterns(int family,
                                                                  int dim) {
  std::vector<std::vector<std::array<int, 3>>> out;
  const bool quad = family == P2 || family == Q2;
  if (dim == 2) {
    if (family == P1 || family == P2) {
      const int tris[2][3][2] = {{{0, 0}, {2, 0}, {2, 2}},
                                 {{0, 0}, {2, 2}, {0, 2}}};
      for (int t = 0; t < 2; ++t) {
        std::vector<std::array<int, 3>> nodes;
        for (int k = 0; k < 3; ++k) nodes.push_back({tris[t][k][0], tris[t][k][1], 0});
        if (quad) {
          const int ed[3][2] = {{0, 1}, {1, 2}, {0, 2}};
          for (auto& e : ed)
            nodes.push_back({(nodes[e[0]][0] + nodes[e[1]][0]) / 2,
                             (nodes[e[0]][1] + nodes[e[1]][1]) / 2, 0});
        }
        out.push_back(nodes);
      }
    } else {
      std::vector<std::array<int, 3>> nodes = {
          {0, 0, 0}, {2, 0, 0}, {2, 2, 0}, {0, 2, 0}};
      if (quad)
        for (auto m : std::vector<std::array<int, 3>>{
                 {1, 0, 0}, {2, 1, 0}, {1, 2, 0}, {0, 1, 0}})
          nodes.push_back(m);
      out.push_back(nodes);
    }
    return out;
  }
  if (family == P1 || family == P2) {
    // Kuhn cube: six tets along the main diagonal; the vertex path follows
    // the axis permutation, odd permutations swap the last two vertices.
    const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                            {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const bool odd[6] = {false, true, true, false, false, true};
    for (int t = 0; t < 6; ++t) {
      std::array<std::array<int, 3>, 4> v{};
      v[0] = {0, 0, 0};
      for (int k = 0; k < 3; ++k) {
        v[k + 1] = v[k];
        v[k + 1][perm[t][k]] += 2;
      }
      if (odd[t]) std::swap(v[2], v[3]);
      std::vector<std::array<int, 3>> nodes(v.begin(), v.end());
      if (quad) {
        const int ed[6][2] = {{0, 1}, {1, 2}, {0, 2}, {1, 3}, {2, 3}, {0, 3}};
        for (auto& e : ed)
          nodes.push_back({(v[e[0]][0] + v[e[1]][0]) / 2,
                           (v[e[0]][1] + v[e[1]][1]) / 2,
                           (v[e[0]][2] + v[e[1]][2]) / 2});
      }
      out.push_back(nodes);
    }
    return out;
  }
  std::vector<std::array<int, 3>> nodes;
  for (int p = 0; p < 8; ++p)
    nodes.push_back({kHC[p][0] + 1, kHC[p][1] + 1, kHC[p][2] + 1});
  if (quad)
    for (int p = 0; p < 12; ++p)
      nodes.push_back({kHE[p][0] + 1, kHE[p][1] + 1, kHE[p][2] + 1});
  out.push_back(nodes);
  return out;
}

struct MeshOut {
  int dim = 0, np = 0;
  int64_t nn = 0, ne = 0;
  std::vector<double> coord;   // dim x nn col-major
  std::vector<int32_t> elem;   // np x ne col-major
  std::vector<int32_t> fine;   // 3 x nn
};

static MeshOut build_structured(int family, int dim, int nx, int ny, int nz,
                                double hx, double hy, double hz,
                                const uint8_t* active) {
  MeshOut m;
  m.dim = dim;
  m.np = node_count(family, dim);
  const int64_t fx = 2 * (int64_t)nx + 1, fy = 2 * (int64_t)ny + 1,
                fz = dim == 3 ? 2 * (int64_t)nz + 1 : 1;
  auto fid = [&](int64_t a, int64_t b, int64_t c) { return (c * fy + b) * fx + a; };
  const auto pats = cell_patterns(family, dim);
  const int layers = dim == 3 ? nz : 1;
  std::vector<uint8_t> used((size_t)(fx * fy * fz), 0);
  int64_t ne = 0;
  for (int k = 0; k < layers; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        if (active && !active[(size_t)j * nx + i]) continue;
        for (auto& pat : pats) {
          ++ne;
          for (auto& o : pat) used[fid(2 * i + o[0], 2 * j + o[1], 2 * k + o[2])] = 1;
        }
      }
  std::vector<int32_t> node_of(used.size(), -1);
  int64_t nn = 0;
  for (size_t p = 0; p < used.size(); ++p)
    if (used[p]) node_of[p] = (int32_t)nn++;
  m.nn = nn;
  m.ne = ne;
  m.coord.assign((size_t)dim * nn, 0.0);
  m.elem.assign((size_t)m.np * ne, 0);
  m.fine.assign((size_t)3 * nn, 0);
  for (int64_t c = 0; c < fz; ++c)
    for (int64_t b = 0; b < fy; ++b)
      for (int64_t a = 0; a < fx; ++a) {
        const int32_t id = node_of[fid(a, b, c)];
        if (id < 0) continue;
        m.fine[3 * (size_t)id] = (int32_t)a;
        m.fine[3 * (size_t)id + 1] = (int32_t)b;
        m.fine[3 * (size_t)id + 2] = (int32_t)c;
        m.coord[(size_t)dim * id] = 0.5 * hx * a;
        m.coord[(size_t)dim * id + 1] = 0.5 * hy * b;
        if (dim == 3) m.coord[(size_t)dim * id + 2] = 0.5 * hz * c;
      }
  int64_t e = 0;
  for (int k = 0; k < layers; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        if (active && !active[(size_t)j * nx + i]) continue;
        for (auto& pat : pats) {
          for (int p = 0; p < m.np; ++p)
            m.elem[(size_t)e * m.np + p] =
                node_of[fid(2 * i + pat[p][0], 2 * j + pat[p][1], 2 * k + pat[p][2])];
          ++e;
        }
      }
  return m;
}

// ---------------------------------------------------------------------------
// Sparse matrices in Eigen's default layout: column-major CSC, sorted inner
// indices.  outer is int64 so the oracle can describe matrices past 2^31
// entries, inner stays int32 like Eigen's StorageIndex.
struct Csc {
  int64_t rows = 0, cols = 0;
  std::vector<int64_t> outer;
  std::vector<int32_t> inner;
  std::vector<double> val;
  int64_t nnz() const { return (int64_t)inner.size(); }
};

struct Triplets {
  std::vector<int64_t> r, c;
  std::vector<double> v;
  void add(int64_t i, int64_t j, double x) {
    r.push_back(i);
    c.push_back(j);
    v.push_back(x);
  }
};

// setFromTriplets: bucket by row in triplet order, collapse duplicates by
// summation (first entry + later ones, in order), then transpose into CSC so
// every column's row indices come out ascending.
static Csc from_triplets(const Triplets& t, int64_t rows, int64_t cols) {
  const size_t n = t.v.size();
  std::vector<int64_t> rp(rows + 1, 0);
  for (size_t k = 0; k < n; ++k) rp[t.r[k] + 1]++;
  for (int64_t i = 0; i < rows; ++i) rp[i + 1] += rp[i];
  std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
  std::vector<int32_t> rc(n);
  std::vector<double> rv(n);
  for (size_t k = 0; k < n; ++k) {
    const int64_t pos = fill[t.r[k]]++;
    rc[pos] = (int32_t)t.c[k];
    rv[pos] = t.v[k];
  }
  // collapse duplicates per row
  std::vector<int64_t> seen(cols, -1);
  std::vector<int64_t> rp2(rows + 1, 0);
  int64_t w = 0;
  for (int64_t i = 0; i < rows; ++i) {
    const int64_t start = w;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int32_t j = rc[k];
      if (seen[j] >= start) {
        rv[seen[j]] += rv[k];
      } else {
        seen[j] = w;
        rc[w] = j;
        rv[w] = rv[k];
        ++w;
      }
    }
    rp2[i + 1] = w;
  }
  // transpose to CSC (rows visited ascending => sorted inner indices)
  Csc A;
  A.rows = rows;
  A.cols = cols;
  A.outer.assign(cols + 1, 0);
  for (int64_t k = 0; k < w; ++k) A.outer[rc[k] + 1]++;
  for (int64_t j = 0; j < cols; ++j) A.outer[j + 1] += A.outer[j];
  A.inner.resize(w);
  A.val.resize(w);
  std::vector<int64_t> cf(A.outer.begin(), A.outer.end() - 1);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t k = rp2[i]; k < rp2[i + 1]; ++k) {
      const int64_t pos = cf[rc[k]]++;
      A.inner[pos] = (int32_t)i;
      A.val[pos] = rv[k];
    }
  return A;
}

// Transposed copy (CSC of A^T), values untouched.
static Csc transpose(const Csc& A) {
  Csc T;
  T.rows = A.cols;
  T.cols = A.rows;
  T.outer.assign(A.rows + 1, 0);
  for (int64_t k = 0; k < A.nnz(); ++k) T.outer[A.inner[k] + 1]++;
  for (int64_t i = 0; i < A.rows; ++i) T.outer[i + 1] += T.outer[i];
  T.inner.resize(A.nnz());
  T.val.resize(A.nnz());
  std::vector<int64_t> f(T.outer.begin(), T.outer.end() - 1);
  for (int64_t j = 0; j < A.cols; ++j)
    for (int64_t k = A.outer[j]; k < A.outer[j + 1]; ++k) {
      const int64_t pos = f[A.inner[k]]++;
      T.inner[pos] = (int32_t)j;
      T.val[pos] = A.val[k];
    }
  return T;
}

// Conservative product L*R: pattern = every (i,j) reachable through a stored
// L(i,k) R(k,j) pair, values summed over k ascending, no pruning.
static Csc product(const Csc& L, const Csc& R) {
  Csc P;
  P.rows = L.rows;
  P.cols = R.cols;
  P.outer.assign(R.cols + 1, 0);
  std::vector<char> mask(L.rows, 0);
  std::vector<double> acc(L.rows, 0.0);
  std::vector<int32_t> idx;
  for (int64_t j = 0; j < R.cols; ++j) {
    idx.clear();
    for (int64_t kk = R.outer[j]; kk < R.outer[j + 1]; ++kk) {
      const int32_t k = R.inner[kk];
      const double y = R.val[kk];
      for (int64_t ii = L.outer[k]; ii < L.outer[k + 1]; ++ii) {
        const int32_t i = L.inner[ii];
        const double x = L.val[ii];
        if (!mask[i]) {
          mask[i] = 1;
          acc[i] = x * y;
          idx.push_back(i);
        } else {
          acc[i] += x * y;
        }
      }
    }
    std::sort(idx.begin(), idx.end());
    for (int32_t i : idx) {
      P.inner.push_back(i);
      P.val.push_back(acc[i]);
      mask[i] = 0;
    }
    P.outer[j + 1] = (int64_t)P.inner.size();
  }
  return P;
}

// A + B over the union pattern; one-sided entries copied as x + 0.0.
static Csc add(const Csc& A, const Csc& B) {
  Csc C;
  C.rows = A.rows;
  C.cols = A.cols;
  C.outer.assign(A.cols + 1, 0);
  C.inner.reserve(std::max(A.nnz(), B.nnz()));
  C.val.reserve(std::max(A.nnz(), B.nnz()));
  for (int64_t j = 0; j < A.cols; ++j) {
    int64_t a = A.outer[j], ae = A.outer[j + 1], b = B.outer[j], be = B.outer[j + 1];
    while (a < ae || b < be) {
      if (b >= be || (a < ae && A.inner[a] < B.inner[b])) {
        C.inner.push_back(A.inner[a]);
        C.val.push_back(A.val[a] + 0.0);
        ++a;
      } else if (a >= ae || B.inner[b] < A.inner[a]) {
        C.inner.push_back(B.inner[b]);
        C.val.push_back(0.0 + B.val[b]);
        ++b;
      } else {
        C.inner.push_back(A.inner[a]);
        C.val.push_back(A.val[a] + B.val[b]);
        ++a;
        ++b;
      }
    }
    C.outer[j + 1] = (int64_t)C.inner.size();
  }
  return C;
}

// sandwich(B, D) = B^T (D B)  (linalg.cpp:28-35): K(i,j) = sum over strain
// rows k ascending of B(k,i) * DB(k,j), DB(k,j) = sum_k' D(k,k') B(k',j).
static Csc sandwich(const Csc& B, const Csc& D) {
  const Csc DB = product(D, B);
  const Csc Bt = transpose(B);
  return product(Bt, DB);
}

// ---------------------------------------------------------------------------
// Voigt operators (voigt.hpp:11-51).
static inline double IOTA(int i) { return i < 3 ? 1.0 : 0.0; }
static inline double VOL(int i, int j) { return IOTA(i) * IOTA(j); }
static inline double DEV(int i, int j) {
  const double diag = i < 3 ? 1.0 : 0.5;
  return (i == j ? diag : 0.0) - VOL(i, j) / 3.0;
}
// C = K VOL + 2G DEV, entry by entry.
static inline double CEL(double K, double G, int i, int j) {
  return K * VOL(i, j) + 2.0 * G * DEV(i, j);
}
static inline void dev_mul(const double* e, double* out) {
  for (int i = 0; i < 6; ++i) {
    double s = DEV(i, 0) * e[0];
    for (int k = 1; k < 6; ++k) s += DEV(i, k) * e[k];
    out[i] = s;
  }
}
static inline double stress_norm(const double* s) {
  const double a = s[0] * s[0] + s[1] * s[1] + s[2] * s[2];
  const double b = s[3] * s[3] + s[4] * s[4] + s[5] * s[5];
  return std::sqrt(a + 2.0 * b);
}
static inline double trace(const double* v) { return v[0] + v[1] + v[2]; }

// Elastic model (constitutive.cpp:76-88): S = C E, DS = C.
void constitutive_elastic(int64_t n, const double* E, const double* G,
                          const double* K, double* S, double* DS) {
  for (int64_t q = 0; q < n; ++q) {
    const double* e = E + 6 * q;
    for (int i = 0; i < 6; ++i) {
      double s = CEL(K[q], G[q], i, 0) * e[0];
      for (int k = 1; k < 6; ++k) s += CEL(K[q], G[q], i, k) * e[k];
      if (S) S[6 * q + i] = s;
    }
    if (DS)
      for (int j = 0; j < 6; ++j)
        for (int i = 0; i < 6; ++i) DS[36 * q + 6 * j + i] = CEL(K[q], G[q], i, j);
  }
}

// von Mises, linear kinematic hardening (constitutive.cpp:90-135).
void constitutive_vm(int64_t n, const double* E, const double* Ep,
                     const double* Hard, const double* Gv, const double* Kv,
                     const double* av, const double* Yv, double* S, double* DS,
                     double* Ep_out, double* Hard_out, uint8_t* plastic,
                     double* crit_out) {
  for (int64_t q = 0; q < n; ++q) {
    const double G = Gv[q], K = Kv[q], a = av[q], Y = Yv[q];
    double etr[6], de[6], sig[6], s[6];
    for (int i = 0; i < 6; ++i) etr[i] = E[6 * q + i] - (Ep ? Ep[6 * q + i] : 0.0);
    dev_mul(etr, de);
    const double ktr = K * trace(etr);
    for (int i = 0; i < 6; ++i) sig[i] = ktr * IOTA(i) + 2.0 * G * de[i];
    for (int i = 0; i < 6; ++i) s[i] = 2.0 * G * de[i] - (Hard ? Hard[6 * q + i] : 0.0);
    const double ns = stress_norm(s);
    const double crit = ns - Y;
    if (crit_out) crit_out[q] = crit;
    if (Ep_out)
      for (int i = 0; i < 6; ++i) Ep_out[6 * q + i] = Ep ? Ep[6 * q + i] : 0.0;
    if (Hard_out)
      for (int i = 0; i < 6; ++i) Hard_out[6 * q + i] = Hard ? Hard[6 * q + i] : 0.0;
    if (crit <= 0.0) {
      if (plastic) plastic[q] = 0;
      if (S) for (int i = 0; i < 6; ++i) S[6 * q + i] = sig[i];
      if (DS)
        for (int j = 0; j < 6; ++j)
          for (int i = 0; i < 6; ++i) DS[36 * q + 6 * j + i] = CEL(K, G, i, j);
      continue;
    }
    if (plastic) plastic[q] = 1;
    double nh[6];
    for (int i = 0; i < 6; ++i) nh[i] = s[i] / ns;
    const double denom = 2.0 * G + a;
    const double lam = crit / denom;
    if (S)
      for (int i = 0; i < 6; ++i) S[6 * q + i] = sig[i] - 2.0 * G * lam * nh[i];
    const double c4 = 4.0 * G * G / denom;
    const double cy = c4 * Y / ns;
    if (DS)
      for (int j = 0; j < 6; ++j)
        for (int i = 0; i < 6; ++i)
          DS[36 * q + 6 * j + i] = CEL(K, G, i, j) - c4 * DEV(i, j) +
                                   cy * (DEV(i, j) - nh[i] * nh[j]);
    if (Hard_out)
      for (int i = 0; i < 6; ++i) Hard_out[6 * q + i] += (a * lam) * nh[i];
    if (Ep_out)
      for (int i = 0; i < 6; ++i) Ep_out[6 * q + i] += lam * (i < 3 ? nh[i] : nh[i] * 2.0);
  }
}

// Drucker-Prager, smooth-portion and apex returns (constitutive.cpp:137-196).
// Returns -1 - q on a zero deviator in the smooth branch.
int64_t constitutive_dp(int64_t n, const double* E, const double* Ep,
                        const double* Gv, const double* Kv, const double* etav,
                        const double* cv, double* S, double* DS, double* Ep_out,
                        uint8_t* smooth, uint8_t* apex) {
  const double sqrt2 = std::sqrt(2.0);
  for (int64_t q = 0; q < n; ++q) {
    const double G = Gv[q], K = Kv[q], eta = etav[q], c = cv[q];
    double etr[6], de[6];
    for (int i = 0; i < 6; ++i) etr[i] = E[6 * q + i] - (Ep ? Ep[6 * q + i] : 0.0);
    dev_mul(etr, de);
    double dot = etr[0] * de[0];
    for (int i = 1; i < 6; ++i) dot += etr[i] * de[i];
    const double ne = std::sqrt(std::max(0.0, dot));
    const double rho = 2.0 * G * ne;
    const double p = K * trace(etr);
    const double da = K * eta * eta;
    const double ds = G + da;
    const double crit1 = rho / sqrt2 + eta * p - c;
    const double crit2 = eta * p - da * rho / (G * sqrt2) - c;
    double sig[6];
    for (int i = 0; i < 6; ++i) sig[i] = p * IOTA(i) + 2.0 * G * de[i];
    if (Ep_out)
      for (int i = 0; i < 6; ++i) Ep_out[6 * q + i] = Ep ? Ep[6 * q + i] : 0.0;
    if (smooth) smooth[q] = 0;
    if (apex) apex[q] = 0;
    if (crit1 <= 0.0) {
      if (S) for (int i = 0; i < 6; ++i) S[6 * q + i] = sig[i];
      if (DS)
        for (int j = 0; j < 6; ++j)
          for (int i = 0; i < 6; ++i) DS[36 * q + 6 * j + i] = CEL(K, G, i, j);
    } else if (crit2 <= 0.0) {
      if (ne <= 0.0) {
        g_err = "constitutive_dp: zero deviator in smooth return";
        return -1 - q;
      }
      if (smooth) smooth[q] = 1;
      const double lam = crit1 / ds;
      double nh[6], mh[6];
      for (int i = 0; i < 6; ++i) nh[i] = de[i] / ne;
      for (int i = 0; i < 6; ++i) mh[i] = sqrt2 * G * nh[i] + K * eta * IOTA(i);
      if (S) for (int i = 0; i < 6; ++i) S[6 * q + i] = sig[i] - lam * mh[i];
      const double c1 = 2.0 * sqrt2 * G * G * lam / rho;
      if (DS)
        for (int j = 0; j < 6; ++j)
          for (int i = 0; i < 6; ++i)
            DS[36 * q + 6 * j + i] = CEL(K, G, i, j) -
                                     c1 * (DEV(i, j) - nh[i] * nh[j]) -
                                     mh[i] * mh[j] / ds;
      if (Ep_out)
        for (int i = 0; i < 6; ++i) {
          const double nst = i < 3 ? nh[i] : nh[i] * 2.0;
          const double dir = (sqrt2 / 2.0) * nst + (eta / 3.0) * IOTA(i);
          Ep_out[6 * q + i] += lam * dir;
        }
    } else {
      if (apex) apex[q] = 1;
      if (S) for (int i = 0; i < 6; ++i) S[6 * q + i] = (c / eta) * IOTA(i);
      if (DS) for (int k = 0; k < 36; ++k) DS[36 * q + k] = 0.0;
      if (Ep_out)
        for (int i = 0; i < 6; ++i)
          Ep_out[6 * q + i] = E[6 * q + i] - (c / (3.0 * K * eta)) * IOTA(i);
    }
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Assembly cache (assembly.cpp:20-180).
static const int kPlane[3] = {0, 1, 3};

struct Cache {
  int family = 0, dim = 0, np = 0, nq = 0, ns = 0;
  int64_t nn = 0, ne = 0, nint = 0;
  Rule rule;
  Basis bas;
  std::vector<double> det, inv, weight, shear, bulk;
  Csc B, Delast, Kel;
  double elastic_seconds = 0.0;
};

// Jacobians (assembly.cpp:20-61).  Eigen's fixed-size determinant and
// cofactor inverse are written out.
static int64_t jacobians(Cache& c, const double* coord, const int32_t* elem) {
  const int dim = c.dim, np = c.np, nq = c.nq;
  c.det.assign(c.nint, 0.0);
  c.inv.assign((size_t)dim * dim * c.nint, 0.0);
  for (int64_t e = 0; e < c.ne; ++e) {
    for (int q = 0; q < nq; ++q) {
      double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
      for (int p = 0; p < np; ++p) {
        const double* x = coord + (size_t)dim * elem[(size_t)e * np + p];
        for (int i = 0; i < dim; ++i)
          for (int j = 0; j < dim; ++j) J[i][j] += c.bas.D(i, p, q) * x[j];
      }
      const int64_t m = e * nq + q;
      double* inv = &c.inv[(size_t)dim * dim * m];  // column-major dim x dim
      if (dim == 3) {
        const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
        if (det <= 0.0) {
          g_err = "jacobians: nonpositive det J in element " + std::to_string(e);
          return -1 - e;
        }
        c.det[m] = det;
        auto cof = [&](int i, int j) {
          const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
          return J[i1][j1] * J[i2][j2] - J[i1][j2] * J[i2][j1];
        };
        const double c00 = cof(0, 0), c10 = cof(1, 0), c20 = cof(2, 0);
        const double d2 = c00 * J[0][0] + c10 * J[1][0] + c20 * J[2][0];
        const double invdet = 1.0 / d2;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) inv[j * 3 + i] = cof(j, i) * invdet;
      } else {
        const double det = J[0][0] * J[1][1] - J[1][0] * J[0][1];
        if (det <= 0.0) {
          g_err = "jacobians: nonpositive det J in element " + std::to_string(e);
          return -1 - e;
        }
        c.det[m] = det;
        const double invdet = 1.0 / det;
        inv[0] = J[1][1] * invdet;   // (0,0)
        inv[1] = -J[1][0] * invdet;  // (1,0)
        inv[2] = -J[0][1] * invdet;  // (0,1)
        inv[3] = J[0][0] * invdet;   // (1,1)
      }
    }
  }
  return 0;
}

// Global strain-displacement matrix (assembly.cpp:63-109).
static void strain_displacement(Cache& c, const int32_t* elem) {
  const int dim = c.dim, np = c.np, nq = c.nq, ns = c.ns;
  Triplets t;
  t.r.reserve((size_t)c.nint * np * 3 * dim);
  t.c.reserve((size_t)c.nint * np * 3 * dim);
  t.v.reserve((size_t)c.nint * np * 3 * dim);
  for (int64_t e = 0; e < c.ne; ++e)
    for (int q = 0; q < nq; ++q) {
      const int64_t m = e * nq + q;
      const int64_t row0 = (int64_t)ns * m;
      const double* Ji = &c.inv[(size_t)dim * dim * m];
      for (int p = 0; p < np; ++p) {
        double d[3] = {0, 0, 0};
        for (int i = 0; i < dim; ++i)
          for (int j = 0; j < dim; ++j) d[i] += Ji[j * dim + i] * c.bas.D(j, p, q);
        const int64_t col0 = (int64_t)dim * elem[(size_t)e * np + p];
        if (dim == 3) {
          t.add(row0 + 0, col0 + 0, d[0]);
          t.add(row0 + 1, col0 + 1, d[1]);
          t.add(row0 + 2, col0 + 2, d[2]);
          t.add(row0 + 3, col0 + 0, d[1]);
          t.add(row0 + 3, col0 + 1, d[0]);
          t.add(row0 + 4, col0 + 1, d[2]);
          t.add(row0 + 4, col0 + 2, d[1]);
          t.add(row0 + 5, col0 + 0, d[2]);
          t.add(row0 + 5, col0 + 2, d[0]);
        } else {
          t.add(row0 + 0, col0 + 0, d[0]);
          t.add(row0 + 1, col0 + 1, d[1]);
          t.add(row0 + 2, col0 + 0, d[1]);
          t.add(row0 + 2, col0 + 1, d[0]);
        }
      }
    }
  c.B = from_triplets(t, (int64_t)ns * c.nint, (int64_t)dim * c.nn);
}

// Block-diagonal weight(q) * DS_q (assembly.cpp:111-133); with `only`, blocks
// (DS_q - C_q) at flagged columns (the tangent's D_diff, assembly.cpp:196-211).
static Csc block_diag(const Cache& c, const double* DS, const uint8_t* only,
                      bool subtract_elastic) {
  const int ns = c.ns;
  Triplets t;
  for (int64_t q = 0; q < c.nint; ++q) {
    if (only && !only[q]) continue;
    const int64_t base = (int64_t)ns * q;
    for (int i = 0; i < ns; ++i)
      for (int j = 0; j < ns; ++j) {
        const int ri = c.dim == 3 ? i : kPlane[i], cj = c.dim == 3 ? j : kPlane[j];
        double v;
        if (DS) {
          v = DS[36 * q + 6 * cj + ri];
          if (subtract_elastic) v = v - CEL(c.bulk[q], c.shear[q], ri, cj);
        } else {
          v = CEL(c.bulk[q], c.shear[q], ri, cj);
        }
        t.add(base + i, base + j, c.weight[q] * v);
      }
  }
  return from_triplets(t, (int64_t)ns * c.nint, (int64_t)ns * c.nint);
}

}  // namespace orc

// =============================================================================
// C ABI for ctypes (tests / bench cpu_baseline only).
// =============================================================================
using namespace orc;

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

int or_node_count(int family, int dim) { return node_count(family, dim); }

// Quadrature: returns n_q; fills pts (dim x n_q col-major) and w when non-null.
int or_quadrature(int family, int dim, double* pts, double* w) {
  Rule r = quadrature(family, dim);
  if (pts) std::memcpy(pts, r.pts.data(), r.pts.size() * sizeof(double));
  if (w) std::memcpy(w, r.w.data(), r.w.size() * sizeof(double));
  return r.nq;
}

// Basis at m points: vals (n_p x m, index p*m+q), grads (dim x n_p x m).
void or_basis(int family, int dim, const double* pts, int m, double* vals,
              double* grads) {
  Basis b = basis(family, dim, pts, m);
  if (vals) std::memcpy(vals, b.vals.data(), b.vals.size() * sizeof(double));
  if (grads) std::memcpy(grads, b.grad.data(), b.grad.size() * sizeof(double));
}

// Structured mesh: call with null outputs to get sizes, then again to fill.
void or_structured_mesh(int family, int dim, int nx, int ny, int nz, double hx,
                        double hy, double hz, const uint8_t* active,
                        int64_t* n_nodes, int64_t* n_elems, double* coord,
                        int32_t* elem, int32_t* fine) {
  MeshOut m = build_structured(family, dim, nx, ny, nz, hx, hy, hz, active);
  *n_nodes = m.nn;
  *n_elems = m.ne;
  if (coord) std::memcpy(coord, m.coord.data(), m.coord.size() * sizeof(double));
  if (elem) std::memcpy(elem, m.elem.data(), m.elem.size() * sizeof(int32_t));
  if (fine) std::memcpy(fine, m.fine.data(), m.fine.size() * sizeof(int32_t));
}

void or_elastic_moduli(double young, double poisson, double* bulk, double* shear) {
  *bulk = young / (3.0 * (1.0 - 2.0 * poisson));
  *shear = young / (2.0 * (1.0 + poisson));
}

// dp_parameters (constitutive.cpp:20-30); mode 1 = three_d, 0 = plane_strain.
void or_dp_parameters(double c0, double phi, int mode, double* eta, double* c) {
  if (mode == 1) {
    const double denom = std::sqrt(3.0) * (3.0 + std::sin(phi));
    *eta = 6.0 * std::sin(phi) / denom;
    *c = c0 * 6.0 * std::cos(phi) / denom;
  } else {
    const double t = std::tan(phi);
    const double denom = std::sqrt(9.0 + 12.0 * t * t);
    *eta = 3.0 * t / denom;
    *c = c0 * 3.0 / denom;
  }
}

void or_constitutive_elastic(int64_t n, const double* E, const double* G,
                             const double* K, double* S, double* DS) {
  constitutive_elastic(n, E, G, K, S, DS);
}

void or_constitutive_vm(int64_t n, const double* E, const double* Ep,
                        const double* Hard, const double* G, const double* K,
                        const double* a, const double* Y, double* S, double* DS,
                        double* Ep_out, double* Hard_out, uint8_t* plastic,
                        double* crit) {
  constitutive_vm(n, E, Ep, Hard, G, K, a, Y, S, DS, Ep_out, Hard_out, plastic, crit);
}

int64_t or_constitutive_dp(int64_t n, const double* E, const double* Ep,
                           const double* G, const double* K, const double* eta,
                           const double* c, double* S, double* DS,
                           double* Ep_out, uint8_t* smooth, uint8_t* apex) {
  return constitutive_dp(n, E, Ep, G, K, eta, c, S, DS, Ep_out, smooth, apex);
}

// build_assembly_cache (assembly.cpp:148-180).  Returns null on error
// (or_last_error() has the reference's message).
void* or_cache_build(int family, int dim, int64_t n_nodes, const double* coord,
                     int64_t n_elems, const int32_t* elem, const double* shear,
                     const double* bulk) {
  const auto t0 = std::chrono::steady_clock::now();
  Cache* c = new Cache;
  c->family = family;
  c->dim = dim;
  c->np = node_count(family, dim);
  c->ns = dim == 3 ? 6 : 3;
  c->rule = quadrature(family, dim);
  c->nq = c->rule.nq;
  c->bas = basis(family, dim, c->rule.pts.data(), c->nq);
  c->nn = n_nodes;
  c->ne = n_elems;
  c->nint = n_elems * c->nq;
  if (jacobians(*c, coord, elem) != 0) {
    delete c;
    return nullptr;
  }
  c->weight.resize(c->nint);
  for (int64_t e = 0; e < c->ne; ++e)
    for (int q = 0; q < c->nq; ++q)
      c->weight[e * c->nq + q] = std::abs(c->det[e * c->nq + q]) * c->rule.w[q];
  strain_displacement(*c, elem);
  c->shear.assign(shear, shear + c->nint);
  c->bulk.assign(bulk, bulk + c->nint);
  c->Delast = block_diag(*c, nullptr, nullptr, false);
  c->Kel = sandwich(c->B, c->Delast);
  c->elastic_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return c;
}

void or_cache_free(void* h) { delete static_cast<Cache*>(h); }

// info[0..7] = n_int, n_dofs, nnz(K_elast), nnz(B), n_q, n_p, n_strain, ne
void or_cache_info(void* h, int64_t* info, double* elastic_seconds) {
  Cache* c = static_cast<Cache*>(h);
  info[0] = c->nint;
  info[1] = (int64_t)c->dim * c->nn;
  info[2] = c->Kel.nnz();
  info[3] = c->B.nnz();
  info[4] = c->nq;
  info[5] = c->np;
  info[6] = c->ns;
  info[7] = c->ne;
  if (elastic_seconds) *elastic_seconds = c->elastic_seconds;
}

void or_cache_arrays(void* h, double* det, double* weight, double* inv) {
  Cache* c = static_cast<Cache*>(h);
  if (det) std::memcpy(det, c->det.data(), c->det.size() * sizeof(double));
  if (weight) std::memcpy(weight, c->weight.data(), c->weight.size() * sizeof(double));
  if (inv) std::memcpy(inv, c->inv.data(), c->inv.size() * sizeof(double));
}

// Copy a CSC matrix out.  K is structurally symmetric, so its CSC arrays are
// also the CSR arrays of the same pattern.
static void copy_csc(const Csc& A, int64_t* outer, int32_t* inner, double* val) {
  if (outer) std::memcpy(outer, A.outer.data(), A.outer.size() * sizeof(int64_t));
  if (inner) std::memcpy(inner, A.inner.data(), A.inner.size() * sizeof(int32_t));
  if (val) std::memcpy(val, A.val.data(), A.val.size() * sizeof(double));
}

void or_cache_K_elast(void* h, int64_t* outer, int32_t* inner, double* val) {
  copy_csc(static_cast<Cache*>(h)->Kel, outer, inner, val);
}

void or_cache_B(void* h, int64_t* outer, int32_t* inner, double* val) {
  copy_csc(static_cast<Cache*>(h)->B, outer, inner, val);
}

// Strains E = B u, 2D embedded into Voigt rows {0,1,3} (assembly.cpp:135-146).
// E is 6 x n_int column-major.  SpMV in column order like Eigen's col-major
// sparse * dense product.
void or_cache_strains(void* h, const double* u, double* E) {
  Cache* c = static_cast<Cache*>(h);
  std::vector<double> ef((size_t)c->B.rows, 0.0);
  for (int64_t j = 0; j < c->B.cols; ++j)
    for (int64_t k = c->B.outer[j]; k < c->B.outer[j + 1]; ++k)
      ef[c->B.inner[k]] += c->B.val[k] * u[j];
  std::memset(E, 0, sizeof(double) * 6 * c->nint);
  for (int64_t q = 0; q < c->nint; ++q)
    for (int i = 0; i < c->ns; ++i)
      E[6 * q + (c->dim == 3 ? i : kPlane[i])] = ef[(size_t)c->ns * q + i];
}

// F = B^T (W S)  (assembly.cpp:215-225).
void or_cache_internal_forces(void* h, const double* S, double* F) {
  Cache* c = static_cast<Cache*>(h);
  std::vector<double> sc((size_t)c->ns * c->nint);
  for (int64_t q = 0; q < c->nint; ++q)
    for (int i = 0; i < c->ns; ++i)
      sc[(size_t)c->ns * q + i] =
          c->weight[q] * S[6 * q + (c->dim == 3 ? i : kPlane[i])];
  for (int64_t j = 0; j < c->B.cols; ++j) {
    double t = 0.0;
    for (int64_t k = c->B.outer[j]; k < c->B.outer[j + 1]; ++k)
      t += c->B.val[k] * sc[c->B.inner[k]];
    F[j] = t;
  }
}

// Result matrices handed back to Python.
struct KOut {
  Csc K;
};

static void* wrap(Csc&& A) {
  KOut* k = new KOut;
  k->K = std::move(A);
  return k;
}

// assemble_tangent_stiffness (assembly.cpp:186-213): K_elast when nothing is
// plastic, else K_elast + sandwich(B, D_diff).  Returns null on size mismatch.
void* or_cache_tangent(void* h, int64_t n_int, const double* DS,
                       const uint8_t* plastic) {
  Cache* c = static_cast<Cache*>(h);
  if (n_int != c->nint) {
    g_err = "assemble_tangent_stiffness: size mismatch";
    return nullptr;
  }
  bool any = false;
  for (int64_t q = 0; q < n_int && !any; ++q) any = plastic[q] != 0;
  if (!any) return wrap(Csc(c->Kel));
  Csc Dd = block_diag(*c, DS, plastic, true);
  return wrap(add(c->Kel, sandwich(c->B, Dd)));
}

// sandwich(B, block_diag_D(DS, weight, dim)) — the "direct" tangent of the
// split-identity test (tests/test_assembly.cpp:350-352).
void* or_cache_direct(void* h, const double* DS) {
  Cache* c = static_cast<Cache*>(h);
  return wrap(sandwich(c->B, block_diag(*c, DS, nullptr, false)));
}

// assemble_elastic_stiffness (assembly.cpp:182-184).
void* or_cache_elastic(void* h) {
  Cache* c = static_cast<Cache*>(h);
  return wrap(sandwich(c->B, c->Delast));
}

void or_k_info(void* k, int64_t* rows, int64_t* nnz) {
  KOut* o = static_cast<KOut*>(k);
  *rows = o->K.rows;
  *nnz = o->K.nnz();
}
void or_k_copy(void* k, int64_t* outer, int32_t* inner, double* val) {
  copy_csc(static_cast<KOut*>(k)->K, outer, inner, val);
}
void or_k_free(void* k) { delete static_cast<KOut*>(k); }

// One timed Newton-iteration body of the reference (solver.cpp:24,28-29):
// evaluate_constitutive (with its IntegrationState::zero fill + E copy,
// constitutive.cpp:198-225) followed by assemble_tangent_stiffness, timed with
// steady_clock like the reference.  model: 0 elastic, 1 von Mises, 2 DP.
// Returns seconds (negative on error); n_plastic_out receives the count.
double or_time_iteration(void* h, int model, const double* E, const double* Ep,
                         const double* Hard, const double* p1, const double* p2,
                         int64_t* n_plastic_out) {
  Cache* c = static_cast<Cache*>(h);
  const int64_t n = c->nint;
  const auto t0 = std::chrono::steady_clock::now();
  // IntegrationState::zero + st.E = E (constitutive.cpp:55-66, 202-203)
  std::vector<double> sE(E, E + 6 * n), sEp(6 * n, 0.0), sH(6 * n, 0.0),
      sS(6 * n, 0.0), sDS(36 * n, 0.0);
  std::vector<uint8_t> pm(n, 0), sm(n, 0), am(n, 0);
  std::vector<double> crit(n);
  if (model == 0) {
    constitutive_elastic(n, sE.data(), c->shear.data(), c->bulk.data(), sS.data(), sDS.data());
  } else if (model == 1) {
    constitutive_vm(n, sE.data(), Ep, Hard, c->shear.data(), c->bulk.data(), p1, p2,
                    sS.data(), sDS.data(), sEp.data(), sH.data(), pm.data(), crit.data());
  } else {
    if (constitutive_dp(n, sE.data(), Ep, c->shear.data(), c->bulk.data(), p1, p2,
                        sS.data(), sDS.data(), sEp.data(), sm.data(), am.data()) != 0)
      return -1.0;
    for (int64_t q = 0; q < n; ++q) pm[q] = sm[q] | am[q];
  }
  void* K = or_cache_tangent(h, n, sDS.data(), pm.data());
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  int64_t np = 0;
  for (int64_t q = 0; q < n; ++q) np += pm[q];
  if (n_plastic_out) *n_plastic_out = np;
  or_k_free(K);
  return secs;
}

}  // extern "C"

// linalg.hpp:11-15 entry points, for the reference's linalg pin tests
// (tests/test_linalg.cpp:15-88).
extern "C" {

void* or_from_triplets(int64_t n, const int64_t* rows, const int64_t* cols,
                       const double* vals, int64_t n_rows, int64_t n_cols) {
  for (int64_t k = 0; k < n; ++k)
    if (rows[k] < 0 || rows[k] >= n_rows || cols[k] < 0 || cols[k] >= n_cols) {
      g_err = "from_triplets: index out of range at entry " + std::to_string(k);
      return nullptr;
    }
  Triplets t;
  t.r.assign(rows, rows + n);
  t.c.assign(cols, cols + n);
  t.v.assign(vals, vals + n);
  return wrap(from_triplets(t, n_rows, n_cols));
}

// sandwich(B, D) with B and D given as triplet lists.
void* or_sandwich(int64_t nb, const int64_t* br, const int64_t* bc, const double* bv,
                  int64_t b_rows, int64_t b_cols, int64_t nd, const int64_t* dr,
                  const int64_t* dc, const double* dv, int64_t d_n) {
  if (d_n != b_rows) {
    g_err = "sandwich: dimension mismatch";
    return nullptr;
  }
  Triplets tb, td;
  tb.r.assign(br, br + nb);
  tb.c.assign(bc, bc + nb);
  tb.v.assign(bv, bv + nb);
  td.r.assign(dr, dr + nd);
  td.c.assign(dc, dc + nd);
  td.v.assign(dv, dv + nd);
  return wrap(sandwich(from_triplets(tb, b_rows, b_cols), from_triplets(td, d_n, d_n)));
}

// KOut rows/cols for non-square results
void or_k_shape(void* k, int64_t* rows, int64_t* cols) {
  KOut* o = static_cast<KOut*>(k);
  *rows = o->K.rows;
  *cols = o->K.cols;
}

}  // extern "C"
