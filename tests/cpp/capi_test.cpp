// C++ caller of libepfem_gpu.so through include/epfem_gpu.hpp (no torch, no
// Python): the reference-side binding a C++ Newton loop would use.  On a
// 12 x 12 cfg2-shaped mesh (2D Q2-8 serendipity, von Mises a = 1e4, Y = 450)
// it builds the assembly cache, runs the fused Newton step on strains scaled
// so ~30 % of the points yield, and checks against the oracle's C API
// (oracle/epfem_oracle.cpp, test infrastructure): CSR pattern and plastic
// flags bit for bit, S bit for bit, K within 1e-12 row-scaled; then the
// reference's error texts through the exceptions.  Prints "CAPI_CPP_OK".
//
//   built and run by tests/test_capi_cpp.py (-m gpu); needs a CUDA device.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "epfem_gpu.hpp"

extern "C" {
// oracle/epfem_oracle.cpp (the checker)
void or_structured_mesh(int family, int dim, int nx, int ny, int nz, double hx, double hy, double hz,
                        const uint8_t* active, int64_t* n_nodes, int64_t* n_elems, double* coord, int32_t* elem,
                        int32_t* fine);
void or_constitutive_vm(int64_t n, const double* E, const double* Ep, const double* Hard, const double* G,
                        const double* K, const double* a, const double* Y, double* S, double* DS, double* Ep_out,
                        double* Hard_out, uint8_t* plastic, double* crit);
void* or_cache_build(int family, int dim, int64_t n_nodes, const double* coord, int64_t n_elems,
                     const int32_t* elem, const double* shear, const double* bulk);
void or_cache_free(void* h);
void or_cache_strains(void* h, const double* u, double* E);
void* or_cache_tangent(void* h, int64_t n_int, const double* DS, const uint8_t* plastic);
void or_k_info(void* k, int64_t* rows, int64_t* nnz);
void or_k_copy(void* k, int64_t* outer, int32_t* inner, double* val);
void or_k_free(void* k);
}

#define REQUIRE(c)                                                      \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                         \
    }                                                                   \
  } while (0)

int main() {
  const int family = EPFEM_Q2, dim = 2, n = 12;
  int64_t nn = 0, ne = 0;
  or_structured_mesh(family, dim, n, n, 0, 1.0 / n, 1.0 / n, 0.0, nullptr, &nn, &ne, nullptr, nullptr, nullptr);
  std::vector<double> coord(nn * dim);
  std::vector<int32_t> elem(ne * 8), fine(nn * 3);
  or_structured_mesh(family, dim, n, n, 0, 1.0 / n, 1.0 / n, 0.0, nullptr, &nn, &ne, coord.data(), elem.data(),
                     fine.data());
  const int64_t n_int = ne * 9;
  const auto [K, G] = epfem_gpu::elastic_moduli(206900.0, 0.29);
  std::vector<double> Gv(n_int, G), Kv(n_int, K), av(n_int, 1.0e4), Y0(n_int, 0.0), Yv(n_int, 450.0);

  // strains of a smooth displacement field, from the oracle (same E bytes to both)
  void* oc = or_cache_build(family, dim, nn, coord.data(), ne, elem.data(), Gv.data(), Kv.data());
  REQUIRE(oc != nullptr);
  std::vector<double> u(nn * dim), E1(n_int * 6);
  for (int64_t a = 0; a < nn; ++a) {
    const double x = coord[a * 2], y = coord[a * 2 + 1];
    u[a * 2] = std::sin(6.1 * x + 2.3 * y) + 0.4 * std::cos(3.7 * y);
    u[a * 2 + 1] = std::cos(4.3 * x - 1.1 * y) + 0.3 * std::sin(5.9 * x * y);
  }
  or_cache_strains(oc, u.data(), E1.data());
  // scale so that 30 % of the points yield: |s_tr| at unit scale, 70 % quantile
  std::vector<double> S(n_int * 6), DS(n_int * 36), Ep(n_int * 6), Hd(n_int * 6), crit(n_int);
  std::vector<uint8_t> pl(n_int);
  or_constitutive_vm(n_int, E1.data(), nullptr, nullptr, Gv.data(), Kv.data(), av.data(), Y0.data(), S.data(),
                     DS.data(), Ep.data(), Hd.data(), pl.data(), crit.data());
  std::vector<double> srt(crit);
  std::sort(srt.begin(), srt.end());
  const double scale = 450.0 / srt[(size_t)(0.7 * n_int)];
  std::vector<double> E(E1);
  for (double& v : E) v *= scale;
  or_constitutive_vm(n_int, E.data(), nullptr, nullptr, Gv.data(), Kv.data(), av.data(), Yv.data(), S.data(),
                     DS.data(), Ep.data(), Hd.data(), pl.data(), crit.data());
  void* kref = or_cache_tangent(oc, n_int, DS.data(), pl.data());
  int64_t rows = 0, nnz = 0;
  or_k_info(kref, &rows, &nnz);
  std::vector<int64_t> rp(rows + 1);
  std::vector<int32_t> ci(nnz);
  std::vector<double> kv(nnz);
  or_k_copy(kref, rp.data(), ci.data(), kv.data());
  or_k_free(kref);

  // the GPU path through the C++ layer
  epfem_gpu::Context ctx(0);
  epfem_gpu::Material mat{EPFEM_MODEL_VON_MISES, n_int, K, G, 1.0e4, 450.0};
  epfem_gpu::AssemblyCache cache(ctx, family, dim, coord, elem, mat);
  REQUIRE(cache.info().n_int == n_int && cache.info().nnz == nnz);
  epfem_gpu::DeviceBuffer<double> dE(E);
  epfem_gpu::NewtonStep step(cache, mat);
  step.run(ctx, dE.data());
  ctx.sync();
  const std::vector<uint8_t> flags = step.flags.download();
  const std::vector<double> gS = step.S.download();
  int64_t n_pl = 0;
  for (int64_t q = 0; q < n_int; ++q) {
    REQUIRE((flags[q] & EPFEM_FLAG_PLASTIC) == pl[q]);
    n_pl += pl[q];
  }
  REQUIRE(n_pl > 0 && n_pl < n_int);
  REQUIRE(std::memcmp(gS.data(), S.data(), S.size() * sizeof(double)) == 0);
  const epfem_gpu::Csr got = step.tangent();
  REQUIRE(got.row_ptr == rp);
  REQUIRE(got.col_idx == ci);
  double err = 0.0;
  for (int64_t r = 0; r < rows; ++r) {
    double m = 0.0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) m = std::max(m, std::fabs(kv[k]));
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) err = std::max(err, std::fabs(got.values[k] - kv[k]) / m);
  }
  REQUIRE(err <= 1e-12);

  // the reference's error texts through exceptions (types.hpp:20-22)
  bool thrown = false;
  try {
    epfem_gpu::Material wrong = mat;
    wrong.n_int = n_int - 1;
    epfem_gpu::NewtonStep bad(cache, wrong);
    bad.run(ctx, dE.data());
  } catch (const epfem_gpu::Error& e) {
    thrown = std::strstr(e.what(), "assemble_tangent_stiffness: size mismatch") != nullptr &&
             e.code == EPFEM_ERR_INVALID;
  }
  REQUIRE(thrown);
  thrown = false;
  try {
    std::vector<double> flat(coord);
    for (int64_t a = 0; a < nn; ++a) flat[a * 2 + 1] = 0.0;  // every element collapsed
    epfem_gpu::AssemblyCache degenerate(ctx, family, dim, flat, elem, mat);
  } catch (const epfem_gpu::Error& e) {
    thrown = std::strstr(e.what(), "jacobians: nonpositive det J in element 0") != nullptr;
  }
  REQUIRE(thrown);
  or_cache_free(oc);
  std::printf("CAPI_CPP_OK n_int=%lld plastic=%lld nnz=%lld K_err=%.3e\n", (long long)n_int, (long long)n_pl,
              (long long)nnz, err);
  return 0;
}
