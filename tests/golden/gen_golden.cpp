// Golden-vector generator for the constitutive pin tests.
//
// Reproduces the reference's seeded batch inputs exactly (std::mt19937 +
// libstdc++ uniform_real_distribution, same call order as
// /root/reference/proj/tests/test_constitutive.cpp:307-331 (VM, seed 11) and
// :415-438 (DP, seed 13)) and evaluates the reference test's *independent*
// tensor-space oracles on them (vm_oracle :59-82, dp_oracle :89-120, restated
// here with 3x3 tensors).  The outputs are written as .npy fixtures into this
// directory; tests/test_oracle_pin.py checks the Voigt restatement in
// oracle/epfem_oracle.cpp against them with the reference's tolerances
// (1e-12 absolute on S/Ep/Hard, flags exact).
//
// Build + run (no Eigen needed):
//   g++ -O2 -ffp-contract=off -std=c++17 -o /tmp/gen_golden tests/golden/gen_golden.cpp
//   /tmp/gen_golden tests/golden
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

namespace {

struct T3 {
  double a[3][3];
};

T3 zero3() {
  T3 t;
  for (auto& r : t.a)
    for (double& x : r) x = 0.0;
  return t;
}
T3 strain_t(const double* e) {
  T3 t;
  t.a[0][0] = e[0]; t.a[0][1] = e[3] / 2; t.a[0][2] = e[5] / 2;
  t.a[1][0] = e[3] / 2; t.a[1][1] = e[1]; t.a[1][2] = e[4] / 2;
  t.a[2][0] = e[5] / 2; t.a[2][1] = e[4] / 2; t.a[2][2] = e[2];
  return t;
}
T3 stress_t(const double* s) {
  T3 t;
  t.a[0][0] = s[0]; t.a[0][1] = s[3]; t.a[0][2] = s[5];
  t.a[1][0] = s[3]; t.a[1][1] = s[1]; t.a[1][2] = s[4];
  t.a[2][0] = s[5]; t.a[2][1] = s[4]; t.a[2][2] = s[2];
  return t;
}
void to_stress(const T3& t, double* s) {
  s[0] = t.a[0][0]; s[1] = t.a[1][1]; s[2] = t.a[2][2];
  s[3] = t.a[0][1]; s[4] = t.a[1][2]; s[5] = t.a[2][0];
}
void to_strain(const T3& t, double* e) {
  e[0] = t.a[0][0]; e[1] = t.a[1][1]; e[2] = t.a[2][2];
  e[3] = 2 * t.a[0][1]; e[4] = 2 * t.a[1][2]; e[5] = 2 * t.a[2][0];
}
T3 lin(double x, const T3& A, double y, const T3& B) {
  T3 t;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t.a[i][j] = x * A.a[i][j] + y * B.a[i][j];
  return t;
}
T3 eye(double s) {
  T3 t = zero3();
  for (int i = 0; i < 3; ++i) t.a[i][i] = s;
  return t;
}
double tr(const T3& t) { return t.a[0][0] + t.a[1][1] + t.a[2][2]; }
T3 devi(const T3& t) { return lin(1.0, t, 1.0, eye(-tr(t) / 3.0)); }
double fro(const T3& t) {
  double s = 0;
  for (auto& r : t.a)
    for (double x : r) s += x * x;
  return std::sqrt(s);
}
T3 hooke(double K, double G, const T3& eps) {
  return lin(1.0, eye(K * tr(eps)), 2.0 * G, devi(eps));
}

// Voigt deviatoric operator times a vector (voigt.hpp:24-31) used only to
// build the deviatoric back-stress inputs the reference test draws.
void dev_mul(const double* v, double* out) {
  for (int i = 0; i < 6; ++i) {
    double s = 0.0;
    for (int k = 0; k < 6; ++k) {
      const double diag = i < 3 ? 1.0 : 0.5;
      const double vol = (i < 3 && k < 3) ? 1.0 : 0.0;
      s += ((i == k ? diag : 0.0) - vol / 3.0) * v[k];
    }
    out[i] = s;
  }
}

void random_voigt(std::mt19937& rng, double scale, double* v) {
  std::uniform_real_distribution<double> u(-scale, scale);
  for (int i = 0; i < 6; ++i) v[i] = u(rng);
}

void save_npy(const std::string& path, const std::vector<double>& data,
              int64_t rows, int64_t cols, const char* descr = "<f8") {
  FILE* f = std::fopen(path.c_str(), "wb");
  std::string shape = cols > 0 ? "(" + std::to_string(rows) + ", " +
                                     std::to_string(cols) + ")"
                               : "(" + std::to_string(rows) + ",)";
  std::string header = std::string("{'descr': '") + descr +
                       "', 'fortran_order': False, 'shape': " + shape + ", }";
  while ((10 + header.size() + 1) % 64 != 0) header += ' ';
  header += '\n';
  const unsigned char magic[8] = {0x93, 'N', 'U', 'M', 'P', 'Y', 1, 0};
  std::fwrite(magic, 1, 8, f);
  const uint16_t hl = (uint16_t)header.size();
  std::fwrite(&hl, 2, 1, f);
  std::fwrite(header.data(), 1, header.size(), f);
  std::fwrite(data.data(), sizeof(double), data.size(), f);
  std::fclose(f);
}

}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  const int n = 1000;
  {  // von Mises batch, seed 11
    std::mt19937 rng(11);
    std::uniform_real_distribution<double> u(0.2, 2.0);
    std::vector<double> G(n), K(n), a(n), Y(n), E(6 * n), Ep(6 * n), H(6 * n);
    for (int q = 0; q < n; ++q) {
      G[q] = u(rng);
      K[q] = u(rng);
      a[q] = (q % 3 == 0) ? 0.0 : u(rng);
      Y[q] = 0.3 * u(rng);
      const double scale = (q % 2 == 0) ? 1.0 : 0.004;
      random_voigt(rng, scale, &E[6 * q]);
      double tmp[6];
      random_voigt(rng, 1.0, tmp);
      for (int i = 0; i < 6; ++i) Ep[6 * q + i] = 0.2 * scale * tmp[i];
      random_voigt(rng, 0.2 * scale, tmp);
      dev_mul(tmp, &H[6 * q]);
    }
    std::vector<double> S(6 * n), Epo(6 * n), Ho(6 * n), pl(n);
    for (int q = 0; q < n; ++q) {
      const T3 eps = lin(1.0, strain_t(&E[6 * q]), -1.0, strain_t(&Ep[6 * q]));
      const T3 sig = hooke(K[q], G[q], eps);
      const T3 s = lin(1.0, devi(sig), -1.0, stress_t(&H[6 * q]));
      const double nrm = fro(s);
      if (nrm - Y[q] <= 0.0) {
        to_stress(sig, &S[6 * q]);
        for (int i = 0; i < 6; ++i) {
          Epo[6 * q + i] = Ep[6 * q + i];
          Ho[6 * q + i] = H[6 * q + i];
        }
        pl[q] = 0;
        continue;
      }
      const T3 nt = lin(1.0 / nrm, s, 0.0, s);
      const double crit = nrm - Y[q];
      const double den = 2 * G[q] + a[q];
      to_stress(lin(1.0, sig, -(2 * G[q] / den) * crit, nt), &S[6 * q]);
      to_stress(lin(1.0, stress_t(&H[6 * q]), (a[q] / den) * crit, nt), &Ho[6 * q]);
      to_strain(lin(1.0, strain_t(&Ep[6 * q]), crit / den, nt), &Epo[6 * q]);
      pl[q] = 1;
    }
    save_npy(dir + "/vm_G.npy", G, n, 0);
    save_npy(dir + "/vm_K.npy", K, n, 0);
    save_npy(dir + "/vm_a.npy", a, n, 0);
    save_npy(dir + "/vm_Y.npy", Y, n, 0);
    save_npy(dir + "/vm_E.npy", E, n, 6);
    save_npy(dir + "/vm_Ep.npy", Ep, n, 6);
    save_npy(dir + "/vm_Hard.npy", H, n, 6);
    save_npy(dir + "/vm_S_tensor.npy", S, n, 6);
    save_npy(dir + "/vm_Ep_tensor.npy", Epo, n, 6);
    save_npy(dir + "/vm_Hard_tensor.npy", Ho, n, 6);
    save_npy(dir + "/vm_plastic_tensor.npy", pl, n, 0);
  }
  {  // Drucker-Prager batch, seed 13
    std::mt19937 rng(13);
    std::uniform_real_distribution<double> u(0.3, 2.0);
    std::vector<double> G(n), K(n), eta(n), c(n), E(6 * n), Ep(6 * n);
    for (int q = 0; q < n; ++q) {
      G[q] = u(rng);
      K[q] = u(rng);
      eta[q] = 0.2 + 0.2 * u(rng);
      c[q] = 0.3 * u(rng);
      random_voigt(rng, 1.2, &E[6 * q]);
      if (q % 4 == 0) {
        const double v = 3.0 + u(rng);
        E[6 * q] = E[6 * q + 1] = E[6 * q + 2] = v;
        for (int i = 3; i < 6; ++i) E[6 * q + i] *= 0.05;
      }
      double tmp[6];
      random_voigt(rng, 1.0, tmp);
      for (int i = 0; i < 6; ++i) Ep[6 * q + i] = 0.1 * tmp[i];
    }
    std::vector<double> S(6 * n), Epo(6 * n), sm(n), ap(n);
    const double s2 = std::sqrt(2.0);
    for (int q = 0; q < n; ++q) {
      const T3 eps = lin(1.0, strain_t(&E[6 * q]), -1.0, strain_t(&Ep[6 * q]));
      const T3 de = devi(eps);
      const double rho = 2.0 * G[q] * fro(de);
      const double p = K[q] * tr(eps);
      const double c1 = rho / s2 + eta[q] * p - c[q];
      const double c2 = eta[q] * p - (K[q] * eta[q] * eta[q]) * rho / (G[q] * s2) - c[q];
      for (int i = 0; i < 6; ++i) Epo[6 * q + i] = Ep[6 * q + i];
      sm[q] = ap[q] = 0;
      if (c1 <= 0.0) {
        to_stress(hooke(K[q], G[q], eps), &S[6 * q]);
        continue;
      }
      if (c2 <= 0.0) {
        sm[q] = 1;
        const double lam = c1 / (G[q] + K[q] * eta[q] * eta[q]);
        const T3 nt = lin(1.0 / fro(de), de, 0.0, de);
        const T3 m = lin(s2 * G[q], nt, 1.0, eye(K[q] * eta[q]));
        to_stress(lin(1.0, hooke(K[q], G[q], eps), -lam, m), &S[6 * q]);
        const T3 dir = lin(std::sqrt(0.5), nt, 1.0, eye(eta[q] / 3.0));
        to_strain(lin(1.0, strain_t(&Ep[6 * q]), lam, dir), &Epo[6 * q]);
        continue;
      }
      ap[q] = 1;
      to_stress(eye(c[q] / eta[q]), &S[6 * q]);
      to_strain(lin(1.0, strain_t(&E[6 * q]), 1.0, eye(-c[q] / (3.0 * K[q] * eta[q]))),
                &Epo[6 * q]);
    }
    save_npy(dir + "/dp_G.npy", G, n, 0);
    save_npy(dir + "/dp_K.npy", K, n, 0);
    save_npy(dir + "/dp_eta.npy", eta, n, 0);
    save_npy(dir + "/dp_c.npy", c, n, 0);
    save_npy(dir + "/dp_E.npy", E, n, 6);
    save_npy(dir + "/dp_Ep.npy", Ep, n, 6);
    save_npy(dir + "/dp_S_tensor.npy", S, n, 6);
    save_npy(dir + "/dp_Ep_tensor.npy", Epo, n, 6);
    save_npy(dir + "/dp_smooth_tensor.npy", sm, n, 0);
    save_npy(dir + "/dp_apex_tensor.npy", ap, n, 0);
  }
  std::printf("golden fixtures written to %s\n", dir.c_str());
  return 0;
}
