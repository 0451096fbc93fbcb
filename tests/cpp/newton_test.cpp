// C++ Newton time step through include/epfem_gpu.hpp (epfem_gpu::newton_solve,
// solver.cpp:7-62) with no torch in the process.  Reads a problem written by
// tests/test_capi_cpp.py (raw little-endian arrays in a directory), runs the
// step and writes u.bin plus stats.txt ("newton_iters n_plastic").
//
//   newton_test <dir>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "epfem_gpu.hpp"

template <class T>
static std::vector<T> read_all(const std::string& path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) throw std::runtime_error("cannot open " + path);
  const size_t bytes = (size_t)f.tellg();
  std::vector<T> v(bytes / sizeof(T));
  f.seekg(0);
  f.read(reinterpret_cast<char*>(v.data()), (std::streamsize)bytes);
  return v;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: newton_test <dir>\n");
    return 2;
  }
  const std::string d = argv[1];
  try {
    // meta: family dim model young poisson p1 p2 eps_newton max_iters rel_tol
    const std::vector<double> meta = read_all<double>(d + "/meta.bin");
    const int family = (int)meta[0], dim = (int)meta[1], model = (int)meta[2];
    const auto coord = read_all<double>(d + "/coord.bin");
    const auto elem = read_all<int32_t>(d + "/elem.bin");
    const auto dirichlet = read_all<double>(d + "/dirichlet.bin");
    const auto free_mask = read_all<uint8_t>(d + "/free.bin");
    const auto f_ext = read_all<double>(d + "/fext.bin");
    const int64_t n_int = (int64_t)meta[10];
    const auto [K, G] = epfem_gpu::elastic_moduli(meta[3], meta[4]);
    epfem_gpu::Context ctx(0);
    epfem_gpu::Material mat{model, n_int, K, G, meta[5], meta[6]};
    epfem_gpu::AssemblyCache cache(ctx, family, dim, coord, elem, mat);
    const epfem_gpu::NewtonResult r =
        epfem_gpu::newton_solve(ctx, cache, mat, dirichlet, free_mask, f_ext, meta[7], (int)meta[8], meta[9]);
    std::ofstream(d + "/u.bin", std::ios::binary)
        .write(reinterpret_cast<const char*>(r.u.data()), (std::streamsize)(r.u.size() * sizeof(double)));
    std::ofstream(d + "/stats.txt") << r.newton_iters << " " << r.n_plastic << "\n";
    std::printf("NEWTON_CPP_OK iters=%d plastic=%lld\n", r.newton_iters, (long long)r.n_plastic);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "FAILED: %s\n", e.what());
    return 1;
  }
  return 0;
}
