// Kernel argument structs and launcher declarations shared by the .cu files.
#pragma once

#include "common.cuh"

namespace epfem_gpu {

// Kernel argument structs shared by the launchers and capi.cu.
struct ConstArgs {
  int64_t n;
  const double* E;
  const double* Ep;
  const double* Hard;
  const double* G;
  const double* K;
  const double* p1;
  const double* p2;
  double Gu, Ku, p1u, p2u;
  double* S;
  uint8_t* flags;
  double* D;
  double* DS;
  double* Ep_out;
  double* Hard_out;
  uint8_t* pm;
  uint8_t* sm;
  uint8_t* am;
  double* crit;
  DevErr* err;
};
struct GatherArgs {
  int64_t n_nodes;
  const int32_t* elem;
  const int64_t* n2e_ptr;
  const int32_t* n2e;
  const uint8_t* slot;
  const int64_t* nbr_ptr;
  const double* inv;
  const double* weight;
  const double* gradhat;
  const double* shear;
  const double* bulk;
  double shear_u, bulk_u;
  const double* D;
  const uint8_t* flags;
  const double* base;
  double* out;
  int max_seg;
  int64_t n_elements;
  double* scratch;   // tangent workspace: symmetric dK_e per element
  unsigned* emask;   // per-element plastic-point bitmask
  int npc;           // nodes per CTA of the row stream
  int max_span;      // widest value range of any row-stream CTA (doubles)
  int max_items;     // most (element, node) items of any row-stream CTA
  double Cu[21];     // packed elastic operator when the material is uniform
  // sub-range processed by one launch (element / node ranges of a slab)
  int64_t e_begin, e_end;  // elements of the delta / fused kernels
  int64_t n_begin, n_end;  // nodes of the row stream
  // strain-fused Newton step (epfem_newton_step_u): nodal displacements in,
  // optional strain output
  const double* u;
  double* E_out;
};
struct PatternOut {
  int64_t* n2e_ptr = nullptr;
  int32_t* n2e = nullptr;
  int64_t* nbr_ptr = nullptr;
  int64_t* row_ptr = nullptr;
  int32_t* col_idx = nullptr;
  uint8_t* slot = nullptr;
  int64_t nnz = 0;
  int max_nbr = 0;
};


enum GatherMode { G_ELASTIC = 0, G_TANGENT_PACKED = 1, G_TANGENT_DS36 = 2 };

int launch_constitutive(int model, const ConstArgs& a, cudaStream_t st, int num_sms);

int launch_jacobians(int family, int dim, int64_t n_e, const int32_t* elem, const double* coord,
                     const double* gradhat, const double* wq, double* det, double* inv,
                     double* weight, DevErr* err, cudaStream_t st, int num_sms);
int build_pattern(int family, int dim, int64_t n_nodes, int64_t n_e, const int32_t* elem,
                  cudaStream_t st, int num_sms, PatternOut* o);
int launch_gather(int family, int dim, int mode, const GatherArgs& a, cudaStream_t st);
int launch_elastic_p1(int family, int dim, const GatherArgs& a, cudaStream_t st);  // K5, P1 meshes
int launch_tangent(int family, int dim, int mode, const GatherArgs& a, cudaStream_t st);
int launch_row_stream(int family, int dim, const GatherArgs& a, cudaStream_t st);
int launch_delta(int family, int dim, int mode, const GatherArgs& a, cudaStream_t st);  // pass 1 over [e_begin, e_end)
int launch_newton_fused_u(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g,
                          cudaStream_t st);  // E = B u inside (GatherArgs::u)
int launch_newton_fused(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g,
                        cudaStream_t st);
int nccl_unique_id(void* out);
int nccl_comm_init(const void* id_bytes, int world, int rank, void** comm_out);
void nccl_comm_destroy(void* comm);
int nccl_exchange(void* comm, int world, int rank, cudaStream_t st, uint8_t* flags, double* D, int64_t send_begin,
                  int64_t send_end, int64_t recv_begin, int64_t recv_end);
int direct_solve(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, const uint8_t* mask,
                 const double* b, double* x_out, double rel_tol, cudaStream_t st, void** cache_slot, int* sweeps_out,
                 double* residual_out);
void direct_cache_free(void* cache);
int cg_solve(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, const uint8_t* mask,
             const double* b, double* x_out, double rel_tol, int64_t max_iters, cudaStream_t st,
             int64_t* iters_out, double* residual_out, int block = 1);
int energy_norm(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, const double* x,
                cudaStream_t st, double* out);
size_t tangent_workspace_doubles(int family, int dim, int64_t n_elements);
int plan_row_stream(int64_t n_nodes, int dim, int np, const int64_t* nbr_ptr, const int64_t* n2e_ptr,
                    cudaStream_t st, int* npc_out, int* span_out, int* items_out, int budget_bytes = 0);
int launch_strains(int family, int dim, int64_t n_e, const int32_t* elem, const double* inv,
                   const double* gradhat, const double* u, double* E, cudaStream_t st,
                   int num_sms);
int launch_internal_forces(int family, int dim, int64_t n_nodes, int64_t n_e, const int64_t* n2e_ptr,
                           const int32_t* n2e, const double* inv, const double* weight,
                           const double* gradhat, const double* S, double* fws, double* F_out,
                           cudaStream_t st, int num_sms);


}  // namespace epfem_gpu
