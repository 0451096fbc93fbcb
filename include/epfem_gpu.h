/*
 * epfem_gpu.h — C-ABI of the B200-native tangent-stiffness path.
 *
 * Drop-in boundary for the reference's hot path (/root/reference/proj):
 *
 *   reference entry point (C++ / Eigen)                      replaced by
 *   -------------------------------------------------------  ------------------------------
 *   evaluate_constitutive        include/epfem/constitutive.hpp:96-98
 *   constitutive_elastic/vm/dp   include/epfem/constitutive.hpp:67,80-81,92-93
 *                                src/constitutive.cpp:76-225    epfem_constitutive
 *   build_assembly_cache         include/epfem/assembly.hpp:53
 *                                src/assembly.cpp:148-180       epfem_cache_build
 *   jacobians / weights          include/epfem/assembly.hpp:20-21
 *                                src/assembly.cpp:20-61        epfem_cache_geometry
 *   AssemblyCache::K_elast       include/epfem/assembly.hpp:45  epfem_cache_K_elast
 *   assemble_elastic_stiffness   include/epfem/assembly.hpp:55  epfem_assemble_elastic
 *   assemble_tangent_stiffness   include/epfem/assembly.hpp:59-60
 *                                src/assembly.cpp:186-213       epfem_assemble_tangent (packed D)
 *                                                               epfem_assemble_tangent_ds (36 x n_int DS)
 *   sparsity of K (Eigen CSC)    src/linalg.cpp:28-35           epfem_cache_pattern
 *   AssemblyCache::strains       include/epfem/assembly.hpp:50  epfem_strains
 *   internal_forces              include/epfem/assembly.hpp:63  epfem_internal_forces
 *   elastic_moduli/dp_parameters include/epfem/constitutive.hpp:11,16
 *                                                               epfem_elastic_moduli, epfem_dp_parameters
 *   epfem::Error (what())        include/epfem/types.hpp:20-22  status code + epfem_last_error()
 *
 * Conventions
 *  - Every array argument is a DEVICE pointer unless stated otherwise, with
 *    the reference's column-major Eigen byte layout: E/Ep/Hard/S are 6 x n_int
 *    (48 B per integration point, Voigt order s11 s22 s33 s12 s23 s31, strains
 *    with engineering shears), DS is 36 x n_int (a column-major 6x6 block per
 *    point), coord is dim x n_nodes, elem is n_p x n_elements (int32, 0-based).
 *  - K is returned in CSR with int64 row_ptr and int32 col_idx, columns sorted
 *    ascending.  K is structurally symmetric, so these arrays are also the
 *    reference's CSC (Eigen SparseMatrix<double>) arrays.  The pattern is the
 *    structural one (explicit zeros kept), identical for K_elast and every
 *    tangent, exactly as Eigen's conservative products produce it.
 *  - Calls are stream-ordered on the context's stream and do not synchronize,
 *    except epfem_cache_build and epfem_ctx_sync.  Device-side failures (DP
 *    zero deviator) are latched in the context and reported by the next
 *    epfem_ctx_sync.  With epfem_ctx_set_sync(ctx, 1) every call synchronizes
 *    and reports, which is the reference's exception behaviour.
 *  - Status: 0 on success, EPFEM_ERR_* otherwise; epfem_last_error() returns
 *    the message (thread-local), using the reference's texts, e.g.
 *    "assemble_tangent_stiffness: size mismatch",
 *    "jacobians: nonpositive det J in element 0",
 *    "constitutive_dp: zero deviator in smooth return".
 *  - There is no CPU fallback: without a CUDA device every call fails with
 *    EPFEM_ERR_CUDA.
 */
#ifndef EPFEM_GPU_H
#define EPFEM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EPFEM_GPU_ABI_VERSION 1

enum epfem_status {
  EPFEM_OK = 0,
  EPFEM_ERR_INVALID = 1,        /* argument / size mismatch (reference: epfem::Error) */
  EPFEM_ERR_DEGENERATE = 2,     /* nonpositive det J */
  EPFEM_ERR_ZERO_DEVIATOR = 3,  /* DP smooth return with zero deviator */
  EPFEM_ERR_CUDA = 4,           /* CUDA runtime / launch failure */
  EPFEM_ERR_NOMEM = 5,
  EPFEM_ERR_UNSUPPORTED = 6,    /* e.g. node valence > 255 */
  EPFEM_ERR_SOLVER = 7,         /* restricted_solve above tolerance (reference: epfem::SolverError) */
  EPFEM_ERR_NCCL = 8            /* NCCL missing or failed (multi-GPU interface exchange) */
};

/* epfem::ElementFamily order (reference_elements.hpp:10) */
enum epfem_family { EPFEM_P1 = 0, EPFEM_P2 = 1, EPFEM_Q1 = 2, EPFEM_Q2 = 3 };

/* MaterialField::plastic variant (constitutive.hpp:18-38) */
enum epfem_model {
  EPFEM_MODEL_ELASTIC = 0,        /* std::monostate */
  EPFEM_MODEL_VON_MISES = 1,      /* VonMisesParams {a, Y} */
  EPFEM_MODEL_DRUCKER_PRAGER = 2  /* DruckerPragerParams {eta, c} */
};

/* per-point flag byte written by epfem_constitutive */
enum epfem_flag { EPFEM_FLAG_PLASTIC = 1, EPFEM_FLAG_SMOOTH = 2, EPFEM_FLAG_APEX = 4 };

/* Packed consistent tangent: 21 upper-triangle entries of the symmetric 6x6
 * block, plane-strain entries first, padded to 24 doubles (192 B = 6 full
 * 32-B sectors).  Entry k holds D(EPFEM_D_ROW[k], EPFEM_D_COL[k]):
 *   k : 0  1  2  3  4  5 | 6  7  8  9 10 11 12 13 14 15 16 17 18 19 20
 *   i : 0  0  0  1  1  3 | 0  0  0  1  1  1  2  2  2  2  3  3  4  4  5
 *   j : 0  1  3  1  3  3 | 2  4  5  2  4  5  2  3  4  5  4  5  4  5  5
 * The D blocks of the reference are bitwise symmetric, so this
 * packing is lossless. */
#define EPFEM_D_STRIDE 24

/* Material field.  Arrays (device, length n_int) override the uniform value
 * when non-NULL.  p1/p2 = (a, Y) for von Mises, (eta, c) for Drucker-Prager. */
typedef struct epfem_material {
  int model;
  int64_t n_int;
  const double* shear;
  const double* bulk;
  const double* p1;
  const double* p2;
  double shear_u, bulk_u, p1_u, p2_u;
} epfem_material;

/* Mesh (mesh.hpp:15-35): coord dim x n_nodes, elem n_p x n_elements. */
typedef struct epfem_mesh {
  int dim;
  int family;
  int64_t n_nodes;
  int64_t n_elements;
  const double* coord;
  const int32_t* elem;
} epfem_mesh;

/* Outputs of epfem_constitutive; any NULL output is skipped. */
typedef struct epfem_constitutive_out {
  double* S;             /* 6 x n_int stress, every point */
  uint8_t* flags;        /* n_int flag bytes (EPFEM_FLAG_*) */
  double* D;             /* EPFEM_D_STRIDE x n_int packed tangent, plastic points only */
  double* DS;            /* 36 x n_int reference layout, every point (elastic: C, apex: 0) */
  double* Ep;            /* 6 x n_int updated plastic strain */
  double* Hard;          /* 6 x n_int updated back stress (VM; zero for DP/elastic) */
  uint8_t* plastic_mask; /* n_int bool */
  uint8_t* smooth_mask;  /* n_int bool (DP) */
  uint8_t* apex_mask;    /* n_int bool (DP) */
  double* crit;          /* n_int |s_tr| - Y (VM) */
} epfem_constitutive_out;

typedef struct epfem_cache_info {
  int dim, family, n_p, n_q, n_strain;
  int max_row_nodes;     /* max neighbour nodes of any node (row block width / dim) */
  int64_t n_nodes, n_elements, n_int, n_dofs, nnz;
  double build_seconds;  /* wall time of epfem_cache_build (elastic_assembly_seconds) */
  double pattern_seconds, elastic_seconds; /* GPU event time of pattern+slot map and K_elast */
} epfem_cache_info;

typedef struct epfem_ctx epfem_ctx;
typedef struct epfem_cache epfem_cache;

const char* epfem_last_error(void);
int epfem_abi_version(void);

int epfem_ctx_create(int device, void* cuda_stream, epfem_ctx** out);
int epfem_ctx_set_stream(epfem_ctx* ctx, void* cuda_stream);
int epfem_ctx_set_sync(epfem_ctx* ctx, int synchronous);
int epfem_ctx_sync(epfem_ctx* ctx);
int epfem_ctx_destroy(epfem_ctx* ctx);

/* Host scalars (constitutive.cpp:11-30). mode: 1 = three_d, 0 = plane_strain. */
int epfem_elastic_moduli(double young, double poisson, double* bulk, double* shear);
int epfem_dp_parameters(double c0, double phi, int mode, double* eta, double* c);

/* K1: constitutive update at every integration point (constitutive.cpp:76-225).
 * Ep_prev / Hard_prev may be NULL (zero history). */
int epfem_constitutive(epfem_ctx* ctx, const epfem_material* mat, const double* E,
                       const double* Ep_prev, const double* Hard_prev,
                       const epfem_constitutive_out* out);

/* One-time cache: jacobians + weights, CSR pattern (K3), element->slot map
 * (K4), K_elast (K5).  Synchronous; fails with EPFEM_ERR_DEGENERATE naming the
 * first element with det J <= 0. */
int epfem_cache_build(epfem_ctx* ctx, const epfem_mesh* mesh, const epfem_material* mat,
                      epfem_cache** out);
int epfem_cache_destroy(epfem_cache* cache);
int epfem_cache_get_info(const epfem_cache* cache, epfem_cache_info* info);
int epfem_cache_pattern(const epfem_cache* cache, const int64_t** row_ptr,
                        const int32_t** col_idx);
int epfem_cache_K_elast(const epfem_cache* cache, const double** values);
/* det (n_int), weight = |det| w_q (n_int), inv (dim*dim x n_int column-major) */
int epfem_cache_geometry(const epfem_cache* cache, const double** det,
                         const double** weight, const double** inv);

/* The tangent workspace of the last step (introspection for tests): the
 * symmetric element deltas dK_e (record_doubles per element, blocks (a, b),
 * a <= b, row-major dim x dim) and the per-element plastic-point bitmask.
 * Records of elements whose mask is 0 are stale. */
int epfem_cache_workspace(const epfem_cache* cache, const double** records, const unsigned** emask,
                          int64_t* record_doubles);

/* K5 recomputed into K_values (nnz doubles) (assembly.cpp:182-184). */
int epfem_assemble_elastic(epfem_ctx* ctx, const epfem_cache* cache, double* K_values);

/* K6+K2: K = K_elast + sum over plastic points of B^T w (D - C) B, written
 * into the cached pattern (assembly.cpp:186-213).  Rows with no plastic
 * contribution are bitwise copies of K_elast. */
int epfem_assemble_tangent(epfem_ctx* ctx, const epfem_cache* cache, int64_t n_int,
                           const double* D, const uint8_t* flags, double* K_values);
/* Same, reading the reference layout: DS 36 x n_int, plastic_cols bool. */
int epfem_assemble_tangent_ds(epfem_ctx* ctx, const epfem_cache* cache, int64_t n_int,
                              const double* DS, const uint8_t* plastic_cols,
                              double* K_values);

/* One Newton iteration's hot path, fused: evaluate_constitutive followed by
 * assemble_tangent_stiffness (solver.cpp:24,28-29).  Writes out->S,
 * out->flags and out->D (all three required; the other outputs must be NULL)
 * and K_values, with the same bits as epfem_constitutive followed by
 * epfem_assemble_tangent.  The cache's material snapshot must be `mat`'s
 * moduli. */
int epfem_newton_step(epfem_ctx* ctx, const epfem_cache* cache, const epfem_material* mat,
                      const double* E, const double* Ep_prev, const double* Hard_prev,
                      const epfem_constitutive_out* out, double* K_values);
/* The same step from nodal displacements: the strains
 * E = B u (assembly.cpp:135-146, epfem_strains) are formed inside the
 * constitutive kernel, never stored unless E_out != NULL (n_int x 6).  Same
 * bits as epfem_strains followed by epfem_newton_step. */
int epfem_newton_step_u(epfem_ctx* ctx, const epfem_cache* cache, const epfem_material* mat,
                        const double* u, const double* Ep_prev, const double* Hard_prev,
                        const epfem_constitutive_out* out, double* E_out, double* K_values);
/* The same step with the internal forces of its stresses (SURVEY §8(f) rank
 * 2; the reference computes them each iteration, solver.cpp:25):
 * F_out (n_dofs) = B^T (weight * S) (internal_forces, assembly.cpp:215-225).
 * epfem_newton_step followed by K9 (two passes: element force records, then
 * a per-node fold), bitwise the same F as epfem_internal_forces on out->S. */
int epfem_newton_step_f(epfem_ctx* ctx, const epfem_cache* cache, const epfem_material* mat,
                        const double* E, const double* Ep_prev, const double* Hard_prev,
                        const epfem_constitutive_out* out, double* K_values, double* F_out);
/* The two halves of epfem_newton_step, for callers that overlap them with
 * other work: (1) constitutive update + element tangent deltas into the
 * cache's workspace, (2) K = K_elast + assembled deltas.  (2) must follow the
 * (1) that produced the workspace, on the same stream. */
int epfem_constitutive_delta(epfem_ctx* ctx, const epfem_cache* cache, const epfem_material* mat,
                             const double* E, const double* Ep_prev, const double* Hard_prev,
                             const epfem_constitutive_out* out);
int epfem_assemble_rows(epfem_ctx* ctx, const epfem_cache* cache, double* K_values);
/* The row stream for the rows of nodes [n_begin, n_end) only (K_values is the whole value array; the
 * element records of every element touching those nodes must be final). */
int epfem_assemble_rows_range(epfem_ctx* ctx, const epfem_cache* cache, double* K_values, int64_t n_begin,
                              int64_t n_end);

/* Element-range forms for a mesh partition (multi-GPU slabs, dist.py): the
 * reference has no partitioned entry point; these split
 * epfem_constitutive_delta so a rank can update its own elements, receive
 * its halo's flags + packed D from the neighbour, and build the halo's
 * element deltas before epfem_assemble_rows.
 * epfem_newton_range: (1) for elements [e_begin, e_end) only.  Every
 *   per-point array (E, Ep_prev, Hard_prev, the material's per-point arrays,
 *   out->S / flags / D) holds exactly the range's points, starting at point
 *   e_begin * n_q; mat->n_int == (e_end - e_begin) * n_q.
 * epfem_delta_range: element deltas of [e_begin, e_end) from a finished
 *   update (flags + packed D over all n_int points of the cache). */
int epfem_newton_range(epfem_ctx* ctx, const epfem_cache* cache, const epfem_material* mat,
                       const double* E, const double* Ep_prev, const double* Hard_prev,
                       const epfem_constitutive_out* out, int64_t e_begin, int64_t e_end);
int epfem_delta_range(epfem_ctx* ctx, const epfem_cache* cache, int64_t n_int, const double* D,
                      const uint8_t* flags, int64_t e_begin, int64_t e_end);

/* Multi-GPU: the interface exchange between z-neighbour slabs over NCCL
 * (the ncclComm_t of §8(b)(1)), for a C / C++ caller with no
 * torch.  NCCL is loaded at run time (libnccl.so.2); EPFEM_ERR_NCCL when it
 * is missing or fails.
 * epfem_nccl_unique_id: 128 bytes (ncclUniqueId) to share from rank 0.
 * epfem_ctx_attach_nccl: a communicator of `world` ranks on the context's
 *   device, owned by the context (destroyed with it).
 * epfem_ctx_set_nccl_comm: use an existing ncclComm_t (not owned).
 * epfem_exchange_interface: one grouped send/recv on the context's stream:
 *   points [send_begin, send_end) of `flags` (1 byte per point) and `D`
 *   (EPFEM_D_STRIDE doubles per point) to rank + 1, points [recv_begin,
 *   recv_end) from rank - 1 (rank 0 receives nothing, the last rank sends
 *   nothing).  The sequence per Newton iteration is epfem_newton_range (top
 *   layer first), epfem_exchange_interface, epfem_newton_range (interior),
 *   epfem_delta_range (halo), epfem_assemble_rows. */
int epfem_nccl_unique_id(void* id_out);
int epfem_ctx_attach_nccl(epfem_ctx* ctx, const void* id, int world, int rank);
int epfem_ctx_set_nccl_comm(epfem_ctx* ctx, void* nccl_comm, int world, int rank);
int epfem_exchange_interface(epfem_ctx* ctx, uint8_t* flags, double* D, int64_t send_begin, int64_t send_end,
                             int64_t recv_begin, int64_t recv_end);

/* K8: E = B u, 2D embedded in Voigt rows {0,1,3} (assembly.cpp:135-146). */
int epfem_strains(epfem_ctx* ctx, const epfem_cache* cache, const double* u, double* E);
/* K9: F = B^T (weight * S) (assembly.cpp:215-225). */
int epfem_internal_forces(epfem_ctx* ctx, const epfem_cache* cache, const double* S,
                          double* F);

/* Newton-loop linear algebra on any CSR matrix
 * (row_ptr int64 n+1, col_idx int32, values), device pointers.
 * epfem_restricted_solve: restricted_solve (linalg.cpp:69-115) with the
 *   reference's LinearSolver::conjugate_gradient method: Jacobi-preconditioned
 *   CG on K[free, free] (free_mask: one byte per row, NULL = all free),
 *   stopping at |r| <= rel_tol |b_free|, at most max_iters iterations (<= 0:
 *   10 n).  x (n) is zero on fixed rows.  EPFEM_ERR_SOLVER with the
 *   reference's message ("restricted_solve: residual <r> above tolerance")
 *   when the true residual |b - K x|_free / |b_free| exceeds rel_tol or is
 *   not finite.  iters / residual (may be NULL) report the solve.
 *   Deterministic (fixed-order reductions).
 * epfem_energy_norm: sqrt(max(v . K v, 0)) (linalg.cpp:117-121). */
int epfem_restricted_solve(epfem_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                           const double* values, const double* rhs, const uint8_t* free_mask,
                           double rel_tol, int64_t max_iters, double* x, int64_t* iters,
                           double* residual);
/* epfem_restricted_solve_blocked: the same solve with a node-block Jacobi
 *   preconditioner (block = dim: the inverse of each dim x dim diagonal block of
 *   the restricted operator; block = 1 is epfem_restricted_solve).  The
 *   reference's default LinearSolver::direct is epfem_restricted_solve_direct
 *   below. */
int epfem_restricted_solve_blocked(epfem_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                                   const double* values, const double* rhs, const uint8_t* free_mask,
                                   double rel_tol, int64_t max_iters, int block, double* x, int64_t* iters,
                                   double* residual);
/* epfem_restricted_solve_direct: the reference's default LinearSolver::direct
 *   (SimplicialLDLT + up to three refinement sweeps, linalg.cpp:84-96) on the
 *   device: K[free, free] formed on the device, factorised by cuSOLVER's sparse
 *   Cholesky (QR when not positive definite; cuSOLVER loaded at run time),
 *   then up to three refinement sweeps on the true residual.  Same contract:
 *   EPFEM_ERR_SOLVER "restricted_solve: factorization failed" or "... residual
 *   <r> above tolerance"; EPFEM_ERR_UNSUPPORTED without cuSOLVER or past int32
 *   sizes.  sweeps / residual (may be NULL) report the solve. */
int epfem_restricted_solve_direct(epfem_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                                  const double* values, const double* rhs, const uint8_t* free_mask, double rel_tol,
                                  double* x, int* sweeps, double* residual);
int epfem_energy_norm(epfem_ctx* ctx, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                      const double* values, const double* v, double* out);

#ifdef __cplusplus
}
#endif

#endif /* EPFEM_GPU_H */
