// Host-side reference tables for the GPU kernels: quadrature rules and basis
// gradients at the quadrature points, with the reference's formulas and
// constants (reference_elements.cpp:20-84 rules, :117-304 bases, :345-390
// dispatch).  Compiled with -ffp-contract=off so the tables carry the same
// bits as the reference's.
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace epfem_gpu {

int node_count(int family, int dim) {
  static const int np[4][2] = {{3, 4}, {6, 10}, {4, 8}, {8, 20}};
  if (family < 0 || family > 3 || (dim != 2 && dim != 3)) return -1;
  return np[family][dim - 2];
}

int quad_count(int family, int dim) {
  static const int nq[4][2] = {{1, 1}, {3, 11}, {4, 8}, {9, 27}};
  if (family < 0 || family > 3 || (dim != 2 && dim != 3)) return -1;
  return nq[family][dim - 2];
}

namespace {

// Quadrature points (dim per point) and weights.
void rule(int family, int dim, double* pts, double* w) {
  if (family == EPFEM_P1) {
    if (dim == 3) {
      pts[0] = pts[1] = pts[2] = 0.25;
      w[0] = 1.0 / 6.0;
    } else {
      pts[0] = pts[1] = 1.0 / 3.0;
      w[0] = 0.5;
    }
    return;
  }
  if (family == EPFEM_P2) {
    if (dim == 2) {  // edge midpoints, degree 2
      const double xy[3][2] = {{0.5, 0.0}, {0.5, 0.5}, {0.0, 0.5}};
      for (int q = 0; q < 3; ++q) {
        pts[2 * q] = xy[q][0];
        pts[2 * q + 1] = xy[q][1];
        w[q] = 1.0 / 6.0;
      }
      return;
    }
    // 11-point Keast rule with the paper's 15-digit constants
    const double a = 0.399403576166799, b = 0.100596423833201;
    const double f = 0.071428571428571, g = 0.785714285714286;
    const double W[3] = {-0.013155555555555, 0.007622222222222, 0.024888888888888};
    const double P[11][3] = {{0.25, 0.25, 0.25}, {f, f, f}, {g, f, f}, {f, g, f},
                             {f, f, g},          {a, b, b}, {b, a, b}, {b, b, a},
                             {a, a, b},          {a, b, a}, {b, a, a}};
    for (int q = 0; q < 11; ++q) {
      for (int d = 0; d < 3; ++d) pts[3 * q + d] = P[q][d];
      w[q] = q == 0 ? W[0] : (q < 5 ? W[1] : W[2]);
    }
    return;
  }
  // Gauss tensor rules, axis 0 fastest, weight = running product from 1.0
  const int n1 = family == EPFEM_Q1 ? 2 : 3;
  double x1[3], w1[3];
  if (n1 == 2) {
    const double s = 1.0 / std::sqrt(3.0);
    x1[0] = -s; x1[1] = s;
    w1[0] = w1[1] = 1.0;
  } else {
    const double s = std::sqrt(3.0 / 5.0);
    x1[0] = -s; x1[1] = 0.0; x1[2] = s;
    w1[0] = 5.0 / 9.0; w1[1] = 8.0 / 9.0; w1[2] = 5.0 / 9.0;
  }
  const int nq = dim == 2 ? n1 * n1 : n1 * n1 * n1;
  for (int q = 0; q < nq; ++q) {
    int r = q;
    double acc = 1.0;
    for (int d = 0; d < dim; ++d) {
      const int k = r % n1;
      r /= n1;
      pts[dim * q + d] = x1[k];
      acc *= w1[k];
    }
    w[q] = acc;
  }
}

const int kQuadC[4][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}};
const int kQuadE[4][2] = {{0, -1}, {1, 0}, {0, 1}, {-1, 0}};
const int kHexC[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                         {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
const int kHexE[12][3] = {{0, -1, -1}, {1, 0, -1}, {0, 1, -1}, {-1, 0, -1},
                          {0, -1, 1},  {1, 0, 1},  {0, 1, 1},  {-1, 0, 1},
                          {-1, -1, 0}, {1, -1, 0}, {1, 1, 0},  {-1, 1, 0}};

// Gradients of every shape function at one reference point: g[p*dim + d].
void gradients(int family, int dim, const double* X, double* g) {
  if (dim == 2) {
    const double x = X[0], y = X[1];
    if (family == EPFEM_P1) {
      const double d0[3] = {-1, 1, 0}, d1[3] = {-1, 0, 1};
      for (int p = 0; p < 3; ++p) { g[2 * p] = d0[p]; g[2 * p + 1] = d1[p]; }
    } else if (family == EPFEM_P2) {
      const double z = 1.0 - x - y;
      const double d0[6] = {1 - 4 * z, 4 * x - 1, 0, 4 * (z - x), 4 * y, -4 * y};
      const double d1[6] = {1 - 4 * z, 0, 4 * y - 1, -4 * x, 4 * x, 4 * (z - y)};
      for (int p = 0; p < 6; ++p) { g[2 * p] = d0[p]; g[2 * p + 1] = d1[p]; }
    } else if (family == EPFEM_Q1) {
      for (int p = 0; p < 4; ++p) {
        const double sx = kQuadC[p][0], sy = kQuadC[p][1];
        g[2 * p] = 0.25 * sx * (1 + sy * y);
        g[2 * p + 1] = 0.25 * sy * (1 + sx * x);
      }
    } else {
      for (int p = 0; p < 4; ++p) {
        const double sx = kQuadC[p][0], sy = kQuadC[p][1];
        const double ax = 1 + sx * x, ay = 1 + sy * y;
        const double r = sx * x + sy * y - 1;
        g[2 * p] = 0.25 * sx * (ay * r + ax * ay);
        g[2 * p + 1] = 0.25 * sy * (ax * r + ax * ay);
      }
      for (int k = 0; k < 4; ++k) {
        const int sx = kQuadE[k][0], sy = kQuadE[k][1];
        double* gp = g + 2 * (4 + k);
        if (sx == 0) {
          gp[0] = -x * (1 + sy * y);
          gp[1] = 0.5 * sy * (1 - x * x);
        } else {
          gp[0] = 0.5 * sx * (1 - y * y);
          gp[1] = -y * (1 + sx * x);
        }
      }
    }
    return;
  }
  const double x = X[0], y = X[1], z = X[2];
  if (family == EPFEM_P1) {
    const double d[3][4] = {{-1, 1, 0, 0}, {-1, 0, 1, 0}, {-1, 0, 0, 1}};
    for (int p = 0; p < 4; ++p)
      for (int k = 0; k < 3; ++k) g[3 * p + k] = d[k][p];
  } else if (family == EPFEM_P2) {
    const double x1 = x, x2 = y, x3 = z;
    const double x0 = 1.0 - x1 - x2 - x3;
    const double d[3][10] = {
        {1 - 4 * x0, 4 * x1 - 1, 0, 0, 4 * (x0 - x1), 4 * x2, -4 * x2, 4 * x3, 0, -4 * x3},
        {1 - 4 * x0, 0, 4 * x2 - 1, 0, -4 * x1, 4 * x1, 4 * (x0 - x2), 0, 4 * x3, -4 * x3},
        {1 - 4 * x0, 0, 0, 4 * x3 - 1, -4 * x1, 0, -4 * x2, 4 * x1, 4 * x2, 4 * (x0 - x3)}};
    for (int p = 0; p < 10; ++p)
      for (int k = 0; k < 3; ++k) g[3 * p + k] = d[k][p];
  } else if (family == EPFEM_Q1) {
    for (int p = 0; p < 8; ++p) {
      const double sx = kHexC[p][0], sy = kHexC[p][1], sz = kHexC[p][2];
      const double ax = 1 + sx * x, ay = 1 + sy * y, az = 1 + sz * z;
      g[3 * p] = 0.125 * sx * ay * az;
      g[3 * p + 1] = 0.125 * sy * ax * az;
      g[3 * p + 2] = 0.125 * sz * ax * ay;
    }
  } else {
    for (int p = 0; p < 8; ++p) {
      const double sx = kHexC[p][0], sy = kHexC[p][1], sz = kHexC[p][2];
      const double ax = 1 + sx * x, ay = 1 + sy * y, az = 1 + sz * z;
      const double r = sx * x + sy * y + sz * z - 2;
      g[3 * p] = 0.125 * sx * ay * az * (r + ax);
      g[3 * p + 1] = 0.125 * sy * ax * az * (r + ay);
      g[3 * p + 2] = 0.125 * sz * ax * ay * (r + az);
    }
    const double c[3] = {x, y, z};
    for (int k = 0; k < 12; ++k) {
      double v[3], dv[3];
      for (int i = 0; i < 3; ++i) {
        const int s = kHexE[k][i];
        v[i] = s == 0 ? 1 - c[i] * c[i] : 1 + s * c[i];
        dv[i] = s == 0 ? -2 * c[i] : (double)s;
      }
      double* gp = g + 3 * (8 + k);
      gp[0] = 0.25 * dv[0] * v[1] * v[2];
      gp[1] = 0.25 * v[0] * dv[1] * v[2];
      gp[2] = 0.25 * v[0] * v[1] * dv[2];
    }
  }
}

}  // namespace

bool make_tables(int family, int dim, HostTables* out) {
  const int np = node_count(family, dim), nq = quad_count(family, dim);
  if (np < 0 || nq < 0) return false;
  out->dim = dim;
  out->np = np;
  out->nq = nq;
  double pts[27 * 3];
  rule(family, dim, pts, out->weights);
  for (int q = 0; q < nq; ++q) gradients(family, dim, pts + dim * q, out->gradhat + q * np * dim);
  return true;
}

}  // namespace epfem_gpu
