// C-ABI implementation (include/epfem_gpu.h): contexts, the device-resident
// assembly cache, argument validation with the reference's error texts, and
// dispatch to the sm_100a kernels.  No CPU compute path exists: every entry
// point fails with EPFEM_ERR_CUDA when no CUDA device is present.
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <chrono>
#include <climits>
#include <vector>
#include <cmath>
#include <cstring>
#include <string>

#include "kernels.cuh"

namespace epfem_gpu {

thread_local std::string g_msg;

void set_error(const std::string& msg) { g_msg = msg; }
int fail(int code, const std::string& msg) {
  g_msg = msg;
  return code;
}
int cuda_fail(cudaError_t err, const char* what) {
  g_msg = std::string("CUDA error: ") + cudaGetErrorString(err) + " (" + what + ")";
  return EPFEM_ERR_CUDA;
}

}  // namespace epfem_gpu

using namespace epfem_gpu;

struct epfem_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool sync = false;
  DevErr* err = nullptr;  // device
  void* comm = nullptr;   // ncclComm_t of the multi-GPU exchange
  bool own_comm = false;
  int world = 1, rank = 0;
  void* direct = nullptr;  // cached restricted pattern + symbolic factorisation (solve.cu)
};

struct epfem_cache {
  epfem_cache_info info{};
  double* gradhat = nullptr;  // device tables
  double* wq = nullptr;
  int32_t* elem = nullptr;    // private copy of connectivity
  double* det = nullptr;
  double* inv = nullptr;
  double* weight = nullptr;
  double* shear = nullptr;    // moduli snapshot (AssemblyCache::shear/bulk)
  double* bulk = nullptr;
  double shear_u = 0, bulk_u = 0;
  PatternOut pat;
  double* K_elast = nullptr;
  double* scratch = nullptr;  // tangent workspace (symmetric dK_e per element)
  unsigned* emask = nullptr;  // per-element plastic-point bitmask
  int npc = 64, max_span = 0, max_items = 0;  // row-stream plan
  double* fws = nullptr;                      // element internal-force records (K9)
};

namespace {

int check_ctx(epfem_ctx* ctx) {
  if (!ctx) return fail(EPFEM_ERR_INVALID, "null context");
  return 0;
}

// Read and clear the latched device error; translate to the reference text.
int poll_device_error(epfem_ctx* ctx, const char* degenerate_prefix) {
  DevErr h{};
  EPFEM_CUDA_TRY(cudaMemcpyAsync(&h, ctx->err, sizeof(DevErr), cudaMemcpyDeviceToHost, ctx->stream));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (h.code == 0) return 0;
  DevErr z{};
  z.index = ~0ull;
  EPFEM_CUDA_TRY(cudaMemcpy(ctx->err, &z, sizeof(DevErr), cudaMemcpyHostToDevice));
  if (h.code == EPFEM_ERR_ZERO_DEVIATOR)
    return fail(h.code, "constitutive_dp: zero deviator in smooth return");
  if (h.code == EPFEM_ERR_DEGENERATE)
    return fail(h.code, std::string(degenerate_prefix ? degenerate_prefix : "jacobians") +
                            ": nonpositive det J in element " + std::to_string(h.index));
  return fail(h.code, "device error");
}

int finish(epfem_ctx* ctx) {
  EPFEM_CUDA_TRY(cudaGetLastError());
  if (ctx->sync) return poll_device_error(ctx, nullptr);
  return 0;
}

bool aligned16(const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }

// Every entry point taking a context runs on the context's device and
// restores the caller's current device on return (torch or the host
// application may have another device current).
// NVTX range around an entry point (header-only NVTX 3: a no-op costing one
// pointer test unless a profiler has injected itself), so a timeline shows
// epfem_newton_step, epfem_cache_build, ... around the kernels they launch
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const epfem_ctx* ctx) {
    if (!ctx) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != ctx->device && cudaSetDevice(ctx->device) == cudaSuccess)
      prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

// per-point pointer re-based so that the kernels' global point index m
// addresses element e_begin's first point at offset 0 (epfem_newton_range)
template <class T>
static T* rebase(T* p, int64_t per_point, int64_t first_point) {
  return p ? p - per_point * first_point : p;
}

// K5 (elastic assembly) = the tangent's two passes with Dw = w C at every
// point and a zero base: element blocks (k_delta_warp / k_elem_delta_staged in
// elastic mode) then the row stream — measured 2.4x / 1.8x / 1.6x faster than
// the one-pass row-block gather (k_gather) on cfg2 / cfg3 / cfg4.  P1
// elements (one point, a 6x6 or 12x12 element matrix; cfg1) use the
// thread-per-node k_elastic_p1 (one launch).  EPFEM_K5=gather|rows|p1
// overrides (p1 on P1 meshes only).  The cache's K_elast and
// epfem_assemble_elastic use the same path, so they agree bit for bit.
static int elastic_assembly(const GatherArgs& g0, int family, int dim, double* out, cudaStream_t st) {
  static const int force = [] {
    const char* v = getenv("EPFEM_K5");
    return v ? (v[0] == 'g' ? 1 : (v[0] == 'p' ? 3 : 2)) : 0;
  }();
  GatherArgs g = g0;
  g.out = out;
  const int path = force ? force : (family == EPFEM_P1 ? 3 : 2);
  if (path == 3 && family == EPFEM_P1) return launch_elastic_p1(family, dim, g, st);
  if (path == 1) return launch_gather(family, dim, 0, g, st);
  g.base = nullptr;
  g.e_begin = 0;
  g.e_end = g.n_elements;
  if (g.n_elements > 0)
    if (int rc = launch_delta(family, dim, G_ELASTIC, g, st)) return rc;
  return launch_row_stream(family, dim, g, st);
}

extern "C" {

const char* epfem_last_error(void) { return g_msg.c_str(); }
int epfem_abi_version(void) { return EPFEM_GPU_ABI_VERSION; }

int epfem_ctx_create(int device, void* cuda_stream, epfem_ctx** out) {
  if (!out) return fail(EPFEM_ERR_INVALID, "null output");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(EPFEM_ERR_CUDA, "epfem_gpu: no CUDA device available (there is no CPU fallback)");
  if (device < 0 || device >= n) return fail(EPFEM_ERR_INVALID, "epfem_gpu: invalid device");
  epfem_ctx* c = new epfem_ctx;
  c->device = device;
  DeviceGuard guard(c);
  c->stream = (cudaStream_t)cuda_stream;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  e = cudaMalloc(&c->err, sizeof(DevErr));
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMalloc(err)");
  }
  DevErr z{};
  z.index = ~0ull;
  cudaMemcpy(c->err, &z, sizeof(DevErr), cudaMemcpyHostToDevice);
  *out = c;
  return 0;
}

int epfem_ctx_set_stream(epfem_ctx* ctx, void* cuda_stream) {
  if (int rc = check_ctx(ctx)) return rc;
  ctx->stream = (cudaStream_t)cuda_stream;
  return 0;
}

int epfem_ctx_set_sync(epfem_ctx* ctx, int synchronous) {
  if (int rc = check_ctx(ctx)) return rc;
  ctx->sync = synchronous != 0;
  return 0;
}

int epfem_ctx_sync(epfem_ctx* ctx) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  EPFEM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return poll_device_error(ctx, nullptr);
}

int epfem_ctx_destroy(epfem_ctx* ctx) {
  if (!ctx) return 0;
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (ctx->own_comm) nccl_comm_destroy(ctx->comm);
  if (ctx->direct) direct_cache_free(ctx->direct);
  if (ctx->err) cudaFree(ctx->err);
  delete ctx;
  return 0;
}

int epfem_elastic_moduli(double young, double poisson, double* bulk, double* shear) {
  // constitutive.cpp:11-18
  if (young <= 0.0) return fail(EPFEM_ERR_INVALID, "elastic_moduli: Young modulus must be > 0");
  if (poisson <= -1.0 || poisson >= 0.5)
    return fail(EPFEM_ERR_INVALID, "elastic_moduli: Poisson ratio must lie in (-1, 1/2)");
  *bulk = young / (3.0 * (1.0 - 2.0 * poisson));
  *shear = young / (2.0 * (1.0 + poisson));
  return 0;
}

int epfem_dp_parameters(double c0, double phi, int mode, double* eta, double* c) {
  // constitutive.cpp:20-30
  if (c0 <= 0.0 || phi <= 0.0 || phi >= M_PI / 2.0)
    return fail(EPFEM_ERR_INVALID, "dp_parameters: require c0 > 0 and phi in (0, pi/2)");
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
  return 0;
}

static int const_args(epfem_ctx* ctx, const epfem_material* mat, const double* E,
                      const double* Ep_prev, const double* Hard_prev,
                      const epfem_constitutive_out* out, ConstArgs* pa) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!mat || !out) return fail(EPFEM_ERR_INVALID, "evaluate_constitutive: null argument");
  if (mat->n_int < 0) return fail(EPFEM_ERR_INVALID, "evaluate_constitutive: size mismatch");
  if (mat->n_int > 0 && !E) return fail(EPFEM_ERR_INVALID, "evaluate_constitutive: null strain");
  const void* ptrs[] = {E, Ep_prev, Hard_prev, out->S, out->D, out->DS, out->Ep, out->Hard};
  for (const void* p : ptrs)
    if (!aligned16(p))
      return fail(EPFEM_ERR_INVALID, "evaluate_constitutive: arrays must be 16-byte aligned");
  ConstArgs& a = *pa;
  a = ConstArgs{};
  a.n = mat->n_int;
  a.E = E;
  a.Ep = Ep_prev;
  a.Hard = mat->model == EPFEM_MODEL_VON_MISES ? Hard_prev : nullptr;
  a.G = mat->shear;
  a.K = mat->bulk;
  a.p1 = mat->p1;
  a.p2 = mat->p2;
  a.Gu = mat->shear_u;
  a.Ku = mat->bulk_u;
  a.p1u = mat->p1_u;
  a.p2u = mat->p2_u;
  a.S = out->S;
  a.flags = out->flags;
  a.D = out->D;
  a.DS = out->DS;
  a.Ep_out = out->Ep;
  a.Hard_out = out->Hard;
  a.pm = out->plastic_mask;
  a.sm = out->smooth_mask;
  a.am = out->apex_mask;
  a.crit = out->crit;
  a.err = ctx->err;
  return 0;
}

int epfem_constitutive(epfem_ctx* ctx, const epfem_material* mat, const double* E,
                       const double* Ep_prev, const double* Hard_prev,
                       const epfem_constitutive_out* out) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  ConstArgs a;
  if (int rc = const_args(ctx, mat, E, Ep_prev, Hard_prev, out, &a)) return rc;
  if (int rc = launch_constitutive(mat->model, a, ctx->stream, ctx->num_sms)) return rc;
  return finish(ctx);
}

int epfem_cache_destroy(epfem_cache* c) {
  if (!c) return 0;
  void* ptrs[] = {c->gradhat, c->wq,          c->elem,        c->det,          c->inv,
                  c->weight,  c->shear,       c->bulk,        c->pat.n2e_ptr,  c->pat.n2e,
                  c->pat.nbr_ptr, c->pat.row_ptr, c->pat.col_idx, c->pat.slot, c->K_elast,
                  c->scratch, c->emask, c->fws};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete c;
  return 0;
}

static GatherArgs gather_args(const epfem_cache* c) {
  GatherArgs g{};
  g.n_nodes = c->info.n_nodes;
  g.elem = c->elem;
  g.n2e_ptr = c->pat.n2e_ptr;
  g.n2e = c->pat.n2e;
  g.slot = c->pat.slot;
  g.nbr_ptr = c->pat.nbr_ptr;
  g.inv = c->inv;
  g.weight = c->weight;
  g.gradhat = c->gradhat;
  g.shear = c->shear;
  g.bulk = c->bulk;
  g.shear_u = c->shear_u;
  g.bulk_u = c->bulk_u;
  g.max_seg = c->info.dim * c->info.dim * c->info.max_row_nodes;
  g.n_elements = c->info.n_elements;
  g.scratch = c->scratch;
  g.emask = c->emask;
  g.npc = c->npc;
  g.max_span = c->max_span;
  g.max_items = c->max_items;
  g.e_begin = 0;
  g.e_end = c->info.n_elements;
  g.n_begin = 0;
  g.n_end = c->info.n_nodes;
  // packed elastic operator C = K VOL + 2G DEV (voigt.hpp:33-36) for a uniform material
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) {
      const double vol = (i < 3 && j < 3) ? 1.0 : 0.0;
      const double dev = ((i == j) ? (i < 3 ? 1.0 : 0.5) : 0.0) - vol / 3.0;
      g.Cu[pk_index(i, j)] = c->bulk_u * vol + 2.0 * c->shear_u * dev;
    }
  return g;
}

int epfem_cache_build(epfem_ctx* ctx, const epfem_mesh* mesh, const epfem_material* mat,
                      epfem_cache** out) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (!mesh || !mat || !out) return fail(EPFEM_ERR_INVALID, "build_assembly_cache: null argument");
  *out = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  HostTables tab;
  if (!make_tables(mesh->family, mesh->dim, &tab))
    return fail(EPFEM_ERR_INVALID, "invalid element type: family=" + std::to_string(mesh->family) +
                                       ", dim=" + std::to_string(mesh->dim));
  const int64_t n_int = mesh->n_elements * tab.nq;
  if (mat->n_int != n_int)
    return fail(EPFEM_ERR_INVALID, "build_assembly_cache: material field size mismatch");
  if (mesh->n_nodes >= (int64_t)INT32_MAX / mesh->dim)
    return fail(EPFEM_ERR_UNSUPPORTED, "build_assembly_cache: too many nodes for int32 columns");
  // the node -> item lists hold item = element * n_p + local node as int32
  if (mesh->n_elements >= (int64_t)INT32_MAX / tab.np)
    return fail(EPFEM_ERR_UNSUPPORTED, "build_assembly_cache: too many elements for int32 item ids");
  cudaStream_t st = ctx->stream;
  epfem_cache* c = new epfem_cache;
  epfem_cache_info& I = c->info;
  I.dim = mesh->dim;
  I.family = mesh->family;
  I.n_p = tab.np;
  I.n_q = tab.nq;
  I.n_strain = mesh->dim == 3 ? 6 : 3;
  I.n_nodes = mesh->n_nodes;
  I.n_elements = mesh->n_elements;
  I.n_int = n_int;
  I.n_dofs = mesh->n_nodes * mesh->dim;
  auto bail = [&](int rc) {
    epfem_cache_destroy(c);
    return rc;
  };
#define CT(expr)                                          \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return bail(cuda_fail(_e, #expr)); \
  } while (0)
  const size_t tg = sizeof(double) * tab.nq * tab.np * tab.dim;
  CT(cudaMalloc(&c->gradhat, tg));
  CT(cudaMalloc(&c->wq, sizeof(double) * tab.nq));
  CT(cudaMemcpyAsync(c->gradhat, tab.gradhat, tg, cudaMemcpyHostToDevice, st));
  CT(cudaMemcpyAsync(c->wq, tab.weights, sizeof(double) * tab.nq, cudaMemcpyHostToDevice, st));
  const size_t elem_bytes = sizeof(int32_t) * (size_t)tab.np * mesh->n_elements;
  CT(cudaMalloc(&c->elem, std::max<size_t>(elem_bytes, 4)));
  CT(cudaMemcpyAsync(c->elem, mesh->elem, elem_bytes, cudaMemcpyDeviceToDevice, st));
  CT(cudaMalloc(&c->det, sizeof(double) * std::max<int64_t>(n_int, 1)));
  // padding: the pipelined kernel reads 16-byte-aligned windows of these
  CT(cudaMalloc(&c->weight, sizeof(double) * (n_int + 4)));
  CT(cudaMalloc(&c->inv, sizeof(double) * mesh->dim * mesh->dim * (n_int + 4)));
  CT(cudaMemsetAsync(c->weight + n_int, 0, 4 * sizeof(double), st));
  CT(cudaMemsetAsync(c->inv + (size_t)mesh->dim * mesh->dim * n_int, 0,
                     4 * sizeof(double) * mesh->dim * mesh->dim, st));
  // moduli snapshot
  c->shear_u = mat->shear_u;
  c->bulk_u = mat->bulk_u;
  if (mat->shear) {
    CT(cudaMalloc(&c->shear, sizeof(double) * n_int));
    CT(cudaMemcpyAsync(c->shear, mat->shear, sizeof(double) * n_int, cudaMemcpyDeviceToDevice, st));
  }
  if (mat->bulk) {
    CT(cudaMalloc(&c->bulk, sizeof(double) * n_int));
    CT(cudaMemcpyAsync(c->bulk, mat->bulk, sizeof(double) * n_int, cudaMemcpyDeviceToDevice, st));
  }
  if (n_int > 0) {
    if (int rc = launch_jacobians(I.family, I.dim, I.n_elements, c->elem, mesh->coord, c->gradhat,
                                  c->wq, c->det, c->inv, c->weight, ctx->err, st, ctx->num_sms))
      return bail(rc);
    if (int rc = poll_device_error(ctx, "jacobians")) return bail(rc);
  }
  cudaEvent_t ev[3];
  for (auto& e : ev) CT(cudaEventCreate(&e));
  CT(cudaEventRecord(ev[0], st));
  if (int rc = build_pattern(I.family, I.dim, I.n_nodes, I.n_elements, c->elem, st, ctx->num_sms, &c->pat))
    return bail(rc);
  CT(cudaEventRecord(ev[1], st));
  I.nnz = c->pat.nnz;
  I.max_row_nodes = c->pat.max_nbr;
  // two doubles of padding: the row stream reads 16-byte-aligned ranges
  CT(cudaMalloc(&c->K_elast, sizeof(double) * (I.nnz + 2)));
  CT(cudaMemsetAsync(c->K_elast + I.nnz, 0, 2 * sizeof(double), st));
  CT(cudaMalloc(&c->scratch, sizeof(double) * std::max<size_t>(
                                 tangent_workspace_doubles(I.family, I.dim, I.n_elements), 1)));
  CT(cudaMalloc(&c->emask, sizeof(unsigned) * std::max<int64_t>(I.n_elements, 1)));
  CT(cudaMalloc(&c->fws, sizeof(double) * std::max<size_t>((size_t)I.n_elements * I.n_p * I.dim, 1)));
  if (I.n_nodes > 0)
    if (int rc = plan_row_stream(I.n_nodes, I.dim, I.n_p, c->pat.nbr_ptr, c->pat.n2e_ptr, st, &c->npc,
                                 &c->max_span, &c->max_items))
      return bail(rc);
  GatherArgs g = gather_args(c);
  g.out = c->K_elast;
  if (int rc = elastic_assembly(g, I.family, I.dim, c->K_elast, st)) return bail(rc);
  CT(cudaEventRecord(ev[2], st));
  CT(cudaStreamSynchronize(st));
  float ms_p = 0, ms_e = 0;
  cudaEventElapsedTime(&ms_p, ev[0], ev[1]);
  cudaEventElapsedTime(&ms_e, ev[1], ev[2]);
  for (auto& e : ev) cudaEventDestroy(e);
  I.pattern_seconds = ms_p * 1e-3;
  I.elastic_seconds = ms_e * 1e-3;
  I.build_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
#undef CT
  *out = c;
  return 0;
}

int epfem_cache_get_info(const epfem_cache* c, epfem_cache_info* info) {
  if (!c || !info) return fail(EPFEM_ERR_INVALID, "null argument");
  *info = c->info;
  return 0;
}

int epfem_cache_pattern(const epfem_cache* c, const int64_t** row_ptr, const int32_t** col_idx) {
  if (!c) return fail(EPFEM_ERR_INVALID, "null cache");
  if (row_ptr) *row_ptr = c->pat.row_ptr;
  if (col_idx) *col_idx = c->pat.col_idx;
  return 0;
}

int epfem_cache_workspace(const epfem_cache* c, const double** records, const unsigned** emask,
                          int64_t* record_doubles) {
  if (!c) return fail(EPFEM_ERR_INVALID, "null cache");
  if (records) *records = c->scratch;
  if (emask) *emask = c->emask;
  if (record_doubles)
    *record_doubles = c->info.n_elements > 0
                          ? (int64_t)(tangent_workspace_doubles(c->info.family, c->info.dim, c->info.n_elements) /
                                      (size_t)c->info.n_elements)
                          : 0;
  return 0;
}

int epfem_cache_K_elast(const epfem_cache* c, const double** values) {
  if (!c || !values) return fail(EPFEM_ERR_INVALID, "null argument");
  *values = c->K_elast;
  return 0;
}

int epfem_cache_geometry(const epfem_cache* c, const double** det, const double** weight,
                         const double** inv) {
  if (!c) return fail(EPFEM_ERR_INVALID, "null cache");
  if (det) *det = c->det;
  if (weight) *weight = c->weight;
  if (inv) *inv = c->inv;
  return 0;
}

int epfem_assemble_elastic(epfem_ctx* ctx, const epfem_cache* c, double* K_values) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (!c || !K_values) return fail(EPFEM_ERR_INVALID, "assemble_elastic_stiffness: null argument");
  if (!aligned16(K_values))
    return fail(EPFEM_ERR_INVALID, "assemble_elastic_stiffness: K must be 16-byte aligned");
  GatherArgs g = gather_args(c);
  g.out = K_values;
  if (int rc = elastic_assembly(g, c->info.family, c->info.dim, K_values, ctx->stream)) return rc;
  return finish(ctx);
}

static int tangent_common(epfem_ctx* ctx, const epfem_cache* c, int64_t n_int, const double* D,
                          const uint8_t* flags, double* K_values, int mode) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!c) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: null cache");
  if (n_int != c->info.n_int) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: size mismatch");
  if (!K_values || (n_int > 0 && (!D || !flags)))
    return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: null argument");
  if (!aligned16(D) || !aligned16(K_values))
    return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: D and K must be 16-byte aligned");
  GatherArgs g = gather_args(c);
  g.D = D;
  g.flags = flags;
  g.base = c->K_elast;
  g.out = K_values;
  if (int rc = launch_tangent(c->info.family, c->info.dim, mode, g, ctx->stream)) return rc;
  return finish(ctx);
}

int epfem_assemble_tangent(epfem_ctx* ctx, const epfem_cache* c, int64_t n_int, const double* D,
                           const uint8_t* flags, double* K_values) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  return tangent_common(ctx, c, n_int, D, flags, K_values, 1);
}

int epfem_assemble_tangent_ds(epfem_ctx* ctx, const epfem_cache* c, int64_t n_int,
                              const double* DS, const uint8_t* plastic_cols, double* K_values) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  return tangent_common(ctx, c, n_int, DS, plastic_cols, K_values, 2);
}

static int delta_args(epfem_ctx* ctx, const epfem_cache* c, const epfem_material* mat,
                      const double* E, const double* Ep_prev, const double* Hard_prev,
                      const epfem_constitutive_out* out, ConstArgs* a, GatherArgs* g) {
  if (int rc = const_args(ctx, mat, E, Ep_prev, Hard_prev, out, a)) return rc;
  if (!c) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: null cache");
  if (mat->n_int != c->info.n_int)
    return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: size mismatch");
  if (c->info.n_int > 0 && (!out->S || !out->flags || !out->D))
    return fail(EPFEM_ERR_INVALID, "newton_step: S, flags and D outputs are required");
  if (out->DS || out->Ep || out->Hard || out->plastic_mask || out->smooth_mask || out->apex_mask ||
      out->crit)
    return fail(EPFEM_ERR_INVALID, "newton_step: only S, flags and D are produced");
  *g = gather_args(c);
  g->D = out->D;
  g->flags = out->flags;
  return 0;
}

static int delta_part(epfem_ctx* ctx, const epfem_cache* c, const epfem_material* mat,
                      const double* E, const double* Ep_prev, const double* Hard_prev,
                      const epfem_constitutive_out* out) {
  ConstArgs a;
  GatherArgs g;
  if (int rc = delta_args(ctx, c, mat, E, Ep_prev, Hard_prev, out, &a, &g)) return rc;
  return launch_newton_fused(mat->model, c->info.family, c->info.dim, a, g, ctx->stream);
}

static int rows_part(epfem_ctx* ctx, const epfem_cache* c, double* K_values, int64_t n_begin = 0,
                     int64_t n_end = -1) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!c) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: null cache");
  if (!K_values || !aligned16(K_values))
    return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: K must be 16-byte aligned");
  GatherArgs g = gather_args(c);
  g.base = c->K_elast;
  g.out = K_values;
  if (n_end >= 0) {
    if (n_begin < 0 || n_begin > n_end || n_end > c->info.n_nodes)
      return fail(EPFEM_ERR_INVALID, "assemble_rows_range: node range out of bounds");
    g.n_begin = n_begin;
    g.n_end = n_end;
  }
  return launch_row_stream(c->info.family, c->info.dim, g, ctx->stream);
}

int epfem_assemble_rows_range(epfem_ctx* ctx, const epfem_cache* c, double* K_values, int64_t n_begin,
                              int64_t n_end) {
  DeviceGuard guard(ctx);
  if (int rc = rows_part(ctx, c, K_values, n_begin, n_end)) return rc;
  return finish(ctx);
}

int epfem_newton_step(epfem_ctx* ctx, const epfem_cache* c, const epfem_material* mat,
                      const double* E, const double* Ep_prev, const double* Hard_prev,
                      const epfem_constitutive_out* out, double* K_values) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (!K_values || !aligned16(K_values))
    return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: K must be 16-byte aligned");
  if (int rc = delta_part(ctx, c, mat, E, Ep_prev, Hard_prev, out)) return rc;
  if (int rc = rows_part(ctx, c, K_values)) return rc;
  return finish(ctx);
}

int epfem_newton_step_f(epfem_ctx* ctx, const epfem_cache* c, const epfem_material* mat,
                        const double* E, const double* Ep_prev, const double* Hard_prev,
                        const epfem_constitutive_out* out, double* K_values, double* F_out) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (!K_values || !aligned16(K_values))
    return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: K must be 16-byte aligned");
  if (!c) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: null cache");
  if (c->info.n_nodes > 0 && !F_out) return fail(EPFEM_ERR_INVALID, "internal_forces: null argument");
  // K9 in two passes after the step (element force records, then a per-node
  // fold in item order).  A form fused into the 2D step (records from the
  // constitutive kernel, fold in the row stream) gave the same bits but
  // measured slower on cfg2 (+0.10 vs +0.08 ms).
  if (int rc = epfem_newton_step(ctx, c, mat, E, Ep_prev, Hard_prev, out, K_values)) return rc;
  if (c->info.n_nodes == 0) return 0;
  if (int rc = launch_internal_forces(c->info.family, c->info.dim, c->info.n_nodes, c->info.n_elements, c->pat.n2e_ptr,
                                      c->pat.n2e, c->inv, c->weight, c->gradhat, out->S, c->fws, F_out, ctx->stream,
                                      ctx->num_sms))
    return rc;
  return finish(ctx);
}

int epfem_newton_step_u(epfem_ctx* ctx, const epfem_cache* c, const epfem_material* mat,
                        const double* u, const double* Ep_prev, const double* Hard_prev,
                        const epfem_constitutive_out* out, double* E_out, double* K_values) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (!K_values || !aligned16(K_values))
    return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: K must be 16-byte aligned");
  if (!c) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: null cache");
  if (c->info.n_int > 0 && !u) return fail(EPFEM_ERR_INVALID, "strains: null argument");
  if (!aligned16(E_out)) return fail(EPFEM_ERR_INVALID, "strains: E must be 16-byte aligned");
  ConstArgs a;
  GatherArgs g;
  // u stands in for E in the argument checks; the strain-fused kernel never reads c.E
  if (int rc = delta_args(ctx, c, mat, u, Ep_prev, Hard_prev, out, &a, &g)) return rc;
  a.E = nullptr;
  g.u = u;
  g.E_out = E_out;
  if (int rc = launch_newton_fused_u(mat->model, c->info.family, c->info.dim, a, g, ctx->stream)) return rc;
  if (int rc = rows_part(ctx, c, K_values)) return rc;
  return finish(ctx);
}

int epfem_constitutive_delta(epfem_ctx* ctx, const epfem_cache* c, const epfem_material* mat,
                             const double* E, const double* Ep_prev, const double* Hard_prev,
                             const epfem_constitutive_out* out) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = delta_part(ctx, c, mat, E, Ep_prev, Hard_prev, out)) return rc;
  return finish(ctx);
}

int epfem_assemble_rows(epfem_ctx* ctx, const epfem_cache* c, double* K_values) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = rows_part(ctx, c, K_values)) return rc;
  return finish(ctx);
}

// per-point pointer re-based so that the kernels' global point index m
// addresses element e_begin's first point at offset 0 (the arrays hold only
// the range; the kernels never form m below the range)

int epfem_newton_range(epfem_ctx* ctx, const epfem_cache* c, const epfem_material* mat,
                       const double* E, const double* Ep_prev, const double* Hard_prev,
                       const epfem_constitutive_out* out, int64_t e_begin, int64_t e_end) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (!c) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: null cache");
  if (e_begin < 0 || e_end < e_begin || e_end > c->info.n_elements)
    return fail(EPFEM_ERR_INVALID, "newton_range: element range out of bounds");
  const int64_t nq = c->info.n_q, p0 = e_begin * nq;
  if (!mat || mat->n_int != (e_end - e_begin) * nq)
    return fail(EPFEM_ERR_INVALID, "newton_range: size mismatch");
  ConstArgs a;
  if (int rc = const_args(ctx, mat, E, Ep_prev, Hard_prev, out, &a)) return rc;
  if (mat->n_int > 0 && (!out->S || !out->flags || !out->D))
    return fail(EPFEM_ERR_INVALID, "newton_step: S, flags and D outputs are required");
  if (out->DS || out->Ep || out->Hard || out->plastic_mask || out->smooth_mask || out->apex_mask ||
      out->crit)
    return fail(EPFEM_ERR_INVALID, "newton_step: only S, flags and D are produced");
  if (e_end == e_begin) return finish(ctx);
  a.n = e_end * nq;
  a.E = rebase(a.E, 6, p0);
  a.Ep = rebase(a.Ep, 6, p0);
  a.Hard = rebase(a.Hard, 6, p0);
  a.G = rebase(a.G, 1, p0);
  a.K = rebase(a.K, 1, p0);
  a.p1 = rebase(a.p1, 1, p0);
  a.p2 = rebase(a.p2, 1, p0);
  a.S = rebase(a.S, 6, p0);
  a.flags = rebase(a.flags, 1, p0);
  a.D = rebase(a.D, EPFEM_D_STRIDE, p0);
  GatherArgs g = gather_args(c);
  g.e_begin = e_begin;
  g.e_end = e_end;
  if (int rc = launch_newton_fused(mat->model, c->info.family, c->info.dim, a, g, ctx->stream)) return rc;
  return finish(ctx);
}

int epfem_delta_range(epfem_ctx* ctx, const epfem_cache* c, int64_t n_int, const double* D,
                      const uint8_t* flags, int64_t e_begin, int64_t e_end) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (!c) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: null cache");
  if (n_int != c->info.n_int) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: size mismatch");
  if (e_begin < 0 || e_end < e_begin || e_end > c->info.n_elements)
    return fail(EPFEM_ERR_INVALID, "delta_range: element range out of bounds");
  if (e_end > e_begin && (!D || !flags))
    return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: null argument");
  if (!aligned16(D)) return fail(EPFEM_ERR_INVALID, "assemble_tangent_stiffness: D must be 16-byte aligned");
  if (e_end == e_begin) return finish(ctx);
  GatherArgs g = gather_args(c);
  g.D = D;
  g.flags = flags;
  g.e_begin = e_begin;
  g.e_end = e_end;
  if (int rc = launch_delta(c->info.family, c->info.dim, G_TANGENT_PACKED, g, ctx->stream)) return rc;
  return finish(ctx);
}

int epfem_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(EPFEM_ERR_INVALID, "nccl_unique_id: null argument");
  return nccl_unique_id(id_out);
}

int epfem_ctx_attach_nccl(epfem_ctx* ctx, const void* id, int world, int rank) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (!id || world < 1 || rank < 0 || rank >= world) return fail(EPFEM_ERR_INVALID, "attach_nccl: invalid rank / world");
  void* comm = nullptr;
  if (int rc = nccl_comm_init(id, world, rank, &comm)) return rc;
  if (ctx->own_comm) nccl_comm_destroy(ctx->comm);
  ctx->comm = comm;
  ctx->own_comm = true;
  ctx->world = world;
  ctx->rank = rank;
  return 0;
}

int epfem_ctx_set_nccl_comm(epfem_ctx* ctx, void* nccl_comm, int world, int rank) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!nccl_comm || world < 1 || rank < 0 || rank >= world)
    return fail(EPFEM_ERR_INVALID, "set_nccl_comm: invalid communicator / rank / world");
  if (ctx->own_comm) nccl_comm_destroy(ctx->comm);
  ctx->comm = nccl_comm;
  ctx->own_comm = false;
  ctx->world = world;
  ctx->rank = rank;
  return 0;
}

int epfem_exchange_interface(epfem_ctx* ctx, uint8_t* flags, double* D, int64_t send_begin, int64_t send_end,
                             int64_t recv_begin, int64_t recv_end) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (!ctx->comm) return fail(EPFEM_ERR_INVALID, "exchange_interface: no NCCL communicator attached");
  if (send_end < send_begin || recv_end < recv_begin || send_begin < 0 || recv_begin < 0)
    return fail(EPFEM_ERR_INVALID, "exchange_interface: invalid point range");
  if ((send_end > send_begin || recv_end > recv_begin) && (!flags || !D))
    return fail(EPFEM_ERR_INVALID, "exchange_interface: null argument");
  if (int rc = nccl_exchange(ctx->comm, ctx->world, ctx->rank, ctx->stream, flags, D, send_begin, send_end, recv_begin,
                             recv_end))
    return rc;
  return finish(ctx);
}

int epfem_strains(epfem_ctx* ctx, const epfem_cache* c, const double* u, double* E) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (!c || !u || !E) return fail(EPFEM_ERR_INVALID, "strains: null argument");
  if (!aligned16(E)) return fail(EPFEM_ERR_INVALID, "strains: E must be 16-byte aligned");
  if (c->info.n_int == 0) return 0;
  if (int rc = launch_strains(c->info.family, c->info.dim, c->info.n_elements, c->elem, c->inv,
                              c->gradhat, u, E, ctx->stream, ctx->num_sms))
    return rc;
  return finish(ctx);
}

int epfem_internal_forces(epfem_ctx* ctx, const epfem_cache* c, const double* S, double* F) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (!c || !S || !F) return fail(EPFEM_ERR_INVALID, "internal_forces: null argument");
  if (c->info.n_nodes == 0) return 0;
  if (int rc = launch_internal_forces(c->info.family, c->info.dim, c->info.n_nodes, c->info.n_elements,
                                      c->pat.n2e_ptr, c->pat.n2e, c->inv, c->weight, c->gradhat, S, c->fws, F,
                                      ctx->stream, ctx->num_sms))
    return rc;
  return finish(ctx);
}

int epfem_restricted_solve(epfem_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                           const double* values, const double* rhs, const uint8_t* free_mask,
                           double rel_tol, int64_t max_iters, double* x, int64_t* iters,
                           double* residual) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  return epfem_restricted_solve_blocked(ctx, n, row_ptr, col_idx, values, rhs, free_mask, rel_tol, max_iters,
                                        1, x, iters, residual);
}

int epfem_restricted_solve_blocked(epfem_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                                   const double* values, const double* rhs, const uint8_t* free_mask,
                                   double rel_tol, int64_t max_iters, int block, double* x, int64_t* iters,
                                   double* residual) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (n < 0 || (n > 0 && (!row_ptr || !col_idx || !values || !rhs || !x)))
    return fail(EPFEM_ERR_INVALID, "restricted_solve: dimension mismatch");
  int64_t it = 0;
  double res = 0.0;
  if (int rc = cg_solve(n, row_ptr, col_idx, values, free_mask, rhs, x, rel_tol,
                        max_iters > 0 ? max_iters : 10 * std::max<int64_t>(n, 1), ctx->stream, &it, &res,
                        block))
    return rc;
  if (iters) *iters = it;
  if (residual) *residual = res;
  if (!std::isfinite(res) || res > rel_tol)
    return fail(EPFEM_ERR_SOLVER, "restricted_solve: residual " + std::to_string(res) + " above tolerance");
  return 0;
}

int epfem_restricted_solve_direct(epfem_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                                  const double* values, const double* rhs, const uint8_t* free_mask, double rel_tol,
                                  double* x, int* sweeps, double* residual) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (n < 0 || (n > 0 && (!row_ptr || !col_idx || !values || !rhs || !x)))
    return fail(EPFEM_ERR_INVALID, "restricted_solve: dimension mismatch");
  int sw = 0;
  double res = 0.0;
  if (int rc = direct_solve(n, row_ptr, col_idx, values, free_mask, rhs, x, rel_tol, ctx->stream, &ctx->direct, &sw,
                            &res))
    return rc;
  if (sweeps) *sweeps = sw;
  if (residual) *residual = res;
  if (!std::isfinite(res) || res > rel_tol)
    return fail(EPFEM_ERR_SOLVER, "restricted_solve: residual " + std::to_string(res) + " above tolerance");
  return 0;
}

int epfem_energy_norm(epfem_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                      const double* values, const double* v, double* out) {
  DeviceGuard guard(ctx);
  NvtxRange nvtx_range(__func__);
  if (int rc = check_ctx(ctx)) return rc;
  if (!out || n < 0 || (n > 0 && (!row_ptr || !col_idx || !values || !v)))
    return fail(EPFEM_ERR_INVALID, "energy_norm: dimension mismatch");
  return energy_norm(n, row_ptr, col_idx, values, v, ctx->stream, out);
}

}  // extern "C"
