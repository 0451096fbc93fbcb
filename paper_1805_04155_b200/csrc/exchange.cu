// Multi-GPU interface exchange over NCCL (the ncclComm_t of
// §8(b)(1)) for a C / C++ caller of the partitioned Newton step with no
// torch: a rank owns a z-slab (y-slab in 2D) of cell layers; after its fused
// update (epfem_newton_range) it sends the flag bytes + packed D of its top
// cell layer to rank + 1 and receives the same from rank - 1 as its halo
// layer, then builds the halo's element deltas (epfem_delta_range) and
// assembles its rows (epfem_assemble_rows).  paper_1805_04155_b200/dist.py
// drives the same sequence from Python.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2", the library torch has
// already loaded when it is in the process), so libepfem_gpu.so has no link
// dependency on it and a process without NCCL only fails when it asks for
// an exchange.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "kernels.cuh"

namespace epfem_gpu {

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define EPFEM_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    EPFEM_SYM(get_unique_id, "ncclGetUniqueId");
    EPFEM_SYM(init_rank, "ncclCommInitRank");
    EPFEM_SYM(destroy, "ncclCommDestroy");
    EPFEM_SYM(group_start, "ncclGroupStart");
    EPFEM_SYM(group_end, "ncclGroupEnd");
    EPFEM_SYM(send, "ncclSend");
    EPFEM_SYM(recv, "ncclRecv");
    EPFEM_SYM(error_string, "ncclGetErrorString");
#undef EPFEM_SYM
    api.ok = api.get_unique_id && api.init_rank && api.destroy && api.group_start && api.group_end && api.send &&
             api.recv && api.error_string;
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  return fail(EPFEM_ERR_NCCL, std::string("NCCL error: ") + nccl().error_string(r) + " (" + what + ")");
}

}  // namespace

int nccl_unique_id(void* out) {
  const NcclApi& api = nccl();
  if (!api.ok) return fail(EPFEM_ERR_NCCL, "NCCL is not available (libnccl.so.2 could not be loaded)");
  ncclUniqueId id;
  if (ncclResult_t r = api.get_unique_id(&id)) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

int nccl_comm_init(const void* id_bytes, int world, int rank, void** comm_out) {
  const NcclApi& api = nccl();
  if (!api.ok) return fail(EPFEM_ERR_NCCL, "NCCL is not available (libnccl.so.2 could not be loaded)");
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof(id));
  ncclComm_t comm = nullptr;
  if (ncclResult_t r = api.init_rank(&comm, world, id, rank)) return nccl_fail(r, "ncclCommInitRank");
  *comm_out = comm;
  return 0;
}

void nccl_comm_destroy(void* comm) {
  if (comm && nccl().ok) nccl().destroy(static_cast<ncclComm_t>(comm));
}

// One grouped send/recv between z-neighbours: [send_begin, send_end) points
// (flag byte + EPFEM_D_STRIDE doubles each) to rank + 1, [recv_begin,
// recv_end) from rank - 1, on `st`.
int nccl_exchange(void* comm, int world, int rank, cudaStream_t st, uint8_t* flags, double* D, int64_t send_begin,
                  int64_t send_end, int64_t recv_begin, int64_t recv_end) {
  const NcclApi& api = nccl();
  if (!api.ok) return fail(EPFEM_ERR_NCCL, "NCCL is not available (libnccl.so.2 could not be loaded)");
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  const bool up = rank + 1 < world && send_end > send_begin;
  const bool down = rank > 0 && recv_end > recv_begin;
  if (!up && !down) return 0;
  if (ncclResult_t r = api.group_start()) return nccl_fail(r, "ncclGroupStart");
  if (up) {
    const size_t n = (size_t)(send_end - send_begin);
    if (ncclResult_t r = api.send(flags + send_begin, n, ncclUint8, rank + 1, c, st)) return nccl_fail(r, "ncclSend");
    if (ncclResult_t r = api.send(D + (size_t)EPFEM_D_STRIDE * send_begin, n * EPFEM_D_STRIDE, ncclFloat64, rank + 1,
                                  c, st))
      return nccl_fail(r, "ncclSend");
  }
  if (down) {
    const size_t n = (size_t)(recv_end - recv_begin);
    if (ncclResult_t r = api.recv(flags + recv_begin, n, ncclUint8, rank - 1, c, st)) return nccl_fail(r, "ncclRecv");
    if (ncclResult_t r = api.recv(D + (size_t)EPFEM_D_STRIDE * recv_begin, n * EPFEM_D_STRIDE, ncclFloat64, rank - 1,
                                  c, st))
      return nccl_fail(r, "ncclRecv");
  }
  if (ncclResult_t r = api.group_end()) return nccl_fail(r, "ncclGroupEnd");
  return 0;
}

}  // namespace epfem_gpu
