// epfem_gpu.hpp — C++ host layer over the C-ABI (include/epfem_gpu.h).
//
// The reference is a C++ library (proj/include/epfem); this header gives a
// C++ caller of its Newton loop (solver.cpp:22-49) the same entry-point
// names and error behaviour on top of libepfem_gpu.so, with no torch and no
// Eigen: RAII handles for the context, the device-resident assembly cache and
// device buffers, and exceptions carrying the reference's messages
// (epfem::Error, types.hpp:20-22).
//
//   reference (C++ / Eigen)                          here
//   -----------------------------------------------  ---------------------------------------
//   build_assembly_cache (assembly.hpp:53)            epfem_gpu::AssemblyCache (constructor)
//   evaluate_constitutive (constitutive.hpp:96-98)    epfem_gpu::evaluate_constitutive
//   assemble_tangent_stiffness (assembly.hpp:59-60)   epfem_gpu::assemble_tangent_stiffness
//   evaluate_constitutive + assemble_tangent_...      epfem_gpu::NewtonStep::run (fused)
//     (solver.cpp:24,28-29)
//   AssemblyCache::strains (assembly.hpp:50)          epfem_gpu::AssemblyCache::strains
//   internal_forces (assembly.hpp:63)                 epfem_gpu::AssemblyCache::internal_forces
//   newton_solve (solver.cpp:7-62)                    epfem_gpu::newton_solve
//
// Host vectors use the reference's column-major byte layout (a 6 x n_int Mat
// is n_int * 6 doubles, point-major); K comes back as CSR arrays (== the
// reference's CSC arrays: K is structurally symmetric).  Link with
// -lepfem_gpu -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "epfem_gpu.h"

namespace epfem_gpu {

// epfem::Error (types.hpp:20-22) with the C-ABI status code
struct Error : std::runtime_error {
  int code;
  Error(const std::string& msg, int c) : std::runtime_error(msg), code(c) {}
};

inline void check(int rc) {
  if (rc != 0) throw Error(epfem_last_error(), rc);
}

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")", EPFEM_ERR_CUDA);
}

// Owning device array of T.
template <class T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) : n_(n) {
    if (n) check_cuda(cudaMalloc(&p_, n * sizeof(T)), "cudaMalloc");
  }
  explicit DeviceBuffer(const std::vector<T>& host) : DeviceBuffer(host.size()) { upload(host); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
    }
    return *this;
  }
  ~DeviceBuffer() { reset(); }
  void reset() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* data() { return p_; }
  const T* data() const { return p_; }
  size_t size() const { return n_; }
  void upload(const std::vector<T>& host) {
    if (host.size() != n_) throw Error("DeviceBuffer: size mismatch", EPFEM_ERR_INVALID);
    if (n_) check_cuda(cudaMemcpy(p_, host.data(), n_ * sizeof(T), cudaMemcpyHostToDevice), "upload");
  }
  std::vector<T> download() const {
    std::vector<T> h(n_);
    if (n_) check_cuda(cudaMemcpy(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "download");
    return h;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// One device + stream; synchronous by default (every call reports device
// errors like the reference's exceptions).
class Context {
 public:
  explicit Context(int device = 0, cudaStream_t stream = nullptr, bool synchronous = true) {
    check(epfem_ctx_create(device, stream, &h_));
    check(epfem_ctx_set_sync(h_, synchronous ? 1 : 0));
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ~Context() { epfem_ctx_destroy(h_); }
  epfem_ctx* get() const { return h_; }
  void sync() { check(epfem_ctx_sync(h_)); }

 private:
  epfem_ctx* h_ = nullptr;
};

// MaterialField (constitutive.hpp:18-38) with uniform values.
struct Material {
  int model = EPFEM_MODEL_ELASTIC;
  int64_t n_int = 0;
  double bulk = 0, shear = 0, p1 = 0, p2 = 0;  // p1, p2 = (a, Y) von Mises, (eta, c) Drucker-Prager
  epfem_material view() const {
    epfem_material m{};
    m.model = model;
    m.n_int = n_int;
    m.shear_u = shear;
    m.bulk_u = bulk;
    m.p1_u = p1;
    m.p2_u = p2;
    return m;
  }
};

inline std::pair<double, double> elastic_moduli(double young, double poisson) {
  double k = 0, g = 0;
  check(epfem_elastic_moduli(young, poisson, &k, &g));
  return {k, g};
}

// Host CSR (== the reference's CSC arrays of K).
struct Csr {
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col_idx;
  std::vector<double> values;
};

// build_assembly_cache (assembly.cpp:148-180), device-resident.
class AssemblyCache {
 public:
  // coord: n_nodes x dim, elem: n_elements x n_p (0-based), host arrays
  AssemblyCache(Context& ctx, int family, int dim, const std::vector<double>& coord,
                const std::vector<int32_t>& elem, const Material& mat) {
    const int np = family == EPFEM_P1 ? dim + 1
                   : family == EPFEM_P2 ? (dim == 2 ? 6 : 10)
                   : family == EPFEM_Q1 ? (dim == 2 ? 4 : 8)
                                        : (dim == 2 ? 8 : 20);
    DeviceBuffer<double> dc(coord);
    DeviceBuffer<int32_t> de(elem);
    epfem_mesh m{dim, family, (int64_t)(coord.size() / dim), (int64_t)(elem.size() / np), dc.data(), de.data()};
    const epfem_material mv = mat.view();
    check(epfem_cache_build(ctx.get(), &m, &mv, &h_));
    check(epfem_cache_get_info(h_, &info_));
  }
  AssemblyCache(const AssemblyCache&) = delete;
  AssemblyCache& operator=(const AssemblyCache&) = delete;
  ~AssemblyCache() { epfem_cache_destroy(h_); }
  const epfem_cache* get() const { return h_; }
  const epfem_cache_info& info() const { return info_; }

  // the pattern (device pointers owned by the cache) and K_elast on the host
  Csr K_elast() const {
    const int64_t* rp = nullptr;
    const int32_t* ci = nullptr;
    const double* v = nullptr;
    check(epfem_cache_pattern(h_, &rp, &ci));
    check(epfem_cache_K_elast(h_, &v));
    return host_csr(rp, ci, v);
  }
  Csr host_csr(const int64_t* rp, const int32_t* ci, const double* v) const {
    Csr k;
    k.row_ptr.resize(info_.n_dofs + 1);
    k.col_idx.resize(info_.nnz);
    k.values.resize(info_.nnz);
    check_cuda(cudaMemcpy(k.row_ptr.data(), rp, k.row_ptr.size() * 8, cudaMemcpyDeviceToHost), "row_ptr");
    check_cuda(cudaMemcpy(k.col_idx.data(), ci, k.col_idx.size() * 4, cudaMemcpyDeviceToHost), "col_idx");
    check_cuda(cudaMemcpy(k.values.data(), v, k.values.size() * 8, cudaMemcpyDeviceToHost), "values");
    return k;
  }
  Csr with_values(const DeviceBuffer<double>& K) const {
    const int64_t* rp = nullptr;
    const int32_t* ci = nullptr;
    check(epfem_cache_pattern(h_, &rp, &ci));
    return host_csr(rp, ci, K.data());
  }

  // AssemblyCache::strains (assembly.cpp:135-146): u host (n_dofs) -> E host (6 x n_int)
  std::vector<double> strains(Context& ctx, const std::vector<double>& u) const {
    DeviceBuffer<double> du(u), dE((size_t)6 * info_.n_int);
    check(epfem_strains(ctx.get(), h_, du.data(), dE.data()));
    return dE.download();
  }
  // internal_forces (assembly.cpp:215-225): S host (6 x n_int) -> F host (n_dofs)
  std::vector<double> internal_forces(Context& ctx, const std::vector<double>& S) const {
    DeviceBuffer<double> dS(S), dF((size_t)info_.n_dofs);
    check(epfem_internal_forces(ctx.get(), h_, dS.data(), dF.data()));
    return dF.download();
  }

 private:
  epfem_cache* h_ = nullptr;
  epfem_cache_info info_{};
};

// The hot path of one Newton iteration on device buffers it owns:
// evaluate_constitutive followed by assemble_tangent_stiffness
// (solver.cpp:24,28-29), fused (epfem_newton_step).
class NewtonStep {
 public:
  NewtonStep(const AssemblyCache& cache, const Material& mat)
      : cache_(cache), mat_(mat.view()), n_(cache.info().n_int),
        S(6 * n_), flags(n_), D((size_t)EPFEM_D_STRIDE * n_), K(cache.info().nnz) {}
  // E, Ep_prev, Hard_prev: device arrays of 6 x n_int (Ep / Hard may be null: zero history)
  void run(Context& ctx, const double* E, const double* Ep_prev = nullptr, const double* Hard_prev = nullptr) {
    epfem_constitutive_out out{};
    out.S = S.data();
    out.flags = flags.data();
    out.D = D.data();
    check(epfem_newton_step(ctx.get(), cache_.get(), &mat_, E, Ep_prev, Hard_prev, &out, K.data()));
  }
  Csr tangent() const { return cache_.with_values(K); }

 private:
  const AssemblyCache& cache_;
  epfem_material mat_;
  int64_t n_;

 public:
  DeviceBuffer<double> S;        // 6 x n_int
  DeviceBuffer<uint8_t> flags;   // EPFEM_FLAG_* per point
  DeviceBuffer<double> D;        // packed tangent at plastic points
  DeviceBuffer<double> K;        // nnz values in the cache's pattern
};

// assemble_tangent_stiffness (assembly.cpp:186-213) from the reference's
// DS layout (36 x n_int, device) and plastic columns (n_int bytes, device).
inline void assemble_tangent_stiffness(Context& ctx, const AssemblyCache& cache, const double* DS,
                                       const uint8_t* plastic_cols, double* K_values) {
  check(epfem_assemble_tangent_ds(ctx.get(), cache.get(), cache.info().n_int, DS, plastic_cols, K_values));
}

// evaluate_constitutive (constitutive.cpp:198-225) into the reference's
// layouts (device pointers; null outputs are skipped).
inline void evaluate_constitutive(Context& ctx, const Material& mat, const double* E, const double* Ep_prev,
                                  const double* Hard_prev, const epfem_constitutive_out& out) {
  const epfem_material mv = mat.view();
  check(epfem_constitutive(ctx.get(), &mv, E, Ep_prev, Hard_prev, &out));
}

// newton_solve (solver.cpp:7-62): one time step of the semismooth Newton
// iteration from the Dirichlet lift (free dofs from u_start when given).
// Every iteration: strains E = B u (K8), the step with its internal forces
// (epfem_newton_step_f: constitutive update, tangent K, F = B^T (w S)), du =
// restricted_solve(K, f_ext - F, free) (the reference's default
// LinearSolver::direct: device sparse Cholesky + refinement; `direct` =
// false: its conjugate-gradient method, the device CG), and the stopping test |du|_e <= eps (|u_prev|_e
// + |u|_e) in the K_elast energy norm.  u and the vector updates live on the
// host (n_dofs doubles), everything per integration point on the device.
// Zero plastic history (Ep_prev = Hard_prev = 0), as the BASELINE steps.
struct NewtonResult {
  std::vector<double> u;
  int newton_iters = 0;
  int64_t n_plastic = 0;              // plastic points at the converged u (the committed state)
  std::vector<int64_t> linear_iters;  // per Newton iteration: refinement sweeps (direct) or CG iterations
};

inline NewtonResult newton_solve(Context& ctx, const AssemblyCache& cache, const Material& mat,
                                 const std::vector<double>& dirichlet, const std::vector<uint8_t>& free_mask,
                                 const std::vector<double>& f_ext, double eps_newton = 1e-10, int max_iters = 25,
                                 double rel_tol = 1e-10, const std::vector<double>* u_start = nullptr,
                                 bool direct = true) {
  if (eps_newton <= 0.0 || max_iters < 1) throw Error("newton_solve: invalid settings", EPFEM_ERR_INVALID);
  const epfem_cache_info& I = cache.info();
  const int64_t n = I.n_dofs, n_int = I.n_int;
  if ((int64_t)dirichlet.size() != n || (int64_t)free_mask.size() != n || (int64_t)f_ext.size() != n)
    throw Error("restricted_solve: dimension mismatch", EPFEM_ERR_INVALID);
  const int64_t* rp = nullptr;
  const int32_t* ci = nullptr;
  const double* kel = nullptr;
  check(epfem_cache_pattern(cache.get(), &rp, &ci));
  check(epfem_cache_K_elast(cache.get(), &kel));
  std::vector<double> u(dirichlet);
  if (u_start)
    for (int64_t k = 0; k < n; ++k)
      if (free_mask[k]) u[k] = (*u_start)[k];
  DeviceBuffer<double> d_u(u), d_E((size_t)6 * n_int), d_F(n), d_rhs(n), d_du(n);
  DeviceBuffer<double> d_zero((size_t)6 * n_int);
  check_cuda(cudaMemset(d_zero.data(), 0, d_zero.size() * sizeof(double)), "cudaMemset");
  DeviceBuffer<uint8_t> d_free(free_mask);
  NewtonStep step(cache, mat);
  const epfem_material mv = mat.view();
  const double* hard = mat.model == EPFEM_MODEL_VON_MISES ? d_zero.data() : nullptr;
  const double* ep = mat.model == EPFEM_MODEL_ELASTIC ? nullptr : d_zero.data();
  auto energy = [&](const DeviceBuffer<double>& v) {
    double e = 0.0;
    check(epfem_energy_norm(ctx.get(), n, rp, ci, kel, v.data(), &e));
    return e;
  };
  NewtonResult res;
  bool converged = false;
  std::vector<double> F, du, rhs(n);
  for (int it = 1; it <= max_iters; ++it) {
    check(epfem_strains(ctx.get(), cache.get(), d_u.data(), d_E.data()));
    epfem_constitutive_out out{};
    out.S = step.S.data();
    out.flags = step.flags.data();
    out.D = step.D.data();
    check(epfem_newton_step_f(ctx.get(), cache.get(), &mv, d_E.data(), ep, hard, &out, step.K.data(), d_F.data()));
    F = d_F.download();
    for (int64_t k = 0; k < n; ++k) rhs[k] = f_ext[k] - F[k];
    d_rhs.upload(rhs);
    int64_t its = 0;
    double r = 0.0;
    if (direct) {
      int sweeps = 0;
      check(epfem_restricted_solve_direct(ctx.get(), n, rp, ci, step.K.data(), d_rhs.data(), d_free.data(), rel_tol,
                                          d_du.data(), &sweeps, &r));
      its = sweeps;
    } else {
      check(epfem_restricted_solve(ctx.get(), n, rp, ci, step.K.data(), d_rhs.data(), d_free.data(), rel_tol, 0,
                                   d_du.data(), &its, &r));
    }
    res.linear_iters.push_back(its);
    res.newton_iters = it;
    const double norm_prev = energy(d_u);
    du = d_du.download();
    for (int64_t k = 0; k < n; ++k) u[k] = u[k] + du[k];
    d_u.upload(u);
    const double norm_curr = energy(d_u);
    const double denom = norm_prev + norm_curr;
    if (denom == 0.0 || energy(d_du) <= eps_newton * denom) {
      converged = true;
      break;
    }
  }
  if (!converged)
    throw Error("newton_solve: no convergence within " + std::to_string(max_iters) + " iterations",
                EPFEM_ERR_SOLVER);
  // commit: the constitutive state at the converged displacement
  check(epfem_strains(ctx.get(), cache.get(), d_u.data(), d_E.data()));
  DeviceBuffer<uint8_t> pm(n_int);
  epfem_constitutive_out out{};
  out.plastic_mask = pm.data();
  check(epfem_constitutive(ctx.get(), &mv, d_E.data(), ep, hard, &out));
  for (uint8_t b : pm.download()) res.n_plastic += b;
  res.u = std::move(u);
  return res;
}

}  // namespace epfem_gpu
