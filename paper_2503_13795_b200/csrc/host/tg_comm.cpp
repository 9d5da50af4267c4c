// tg_comm.cpp — the data-parallel exchange of the gradient oracle over NCCL
// (north_star (d)): one all-reduce (sum) of the d-length
// gradient per step, then the GD update with the global batch.
//
// NCCL is bound at run time (dlopen), so libtg.so has no link-time NCCL
// dependency and shares the process's NCCL when one is already loaded
// (torch.distributed's): RTLD_NOLOAD first, then TG_NCCL_LIB, then the
// system soname.  Only the stable subset of nccl.h used here is declared.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "tg_abi.h"
#include "tg_comm.hpp"

namespace {

struct NcclUid { char internal[128]; };
using ncclComm_t = void*;
using ncclResult_t = int;

struct Nccl {
  void* so = nullptr;
  std::string err;
  ncclResult_t (*get_unique_id)(NcclUid*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, NcclUid, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(ncclComm_t, int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, std::size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {std::getenv("TG_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names)
      if (nm && (n.so = dlopen(nm, RTLD_NOW | RTLD_NOLOAD))) break;
    for (const char* nm : names)
      if (!n.so && nm) n.so = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (!n.so) {
      const char* e = dlerror();
      n.err = std::string("NCCL not found (set TG_NCCL_LIB): ") + (e ? e : "");
      return;
    }
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(n.so, name)); };
    sym(n.get_unique_id, "ncclGetUniqueId");
    sym(n.comm_init_rank, "ncclCommInitRank");
    sym(n.comm_destroy, "ncclCommDestroy");
    sym(n.comm_count, "ncclCommCount");
    sym(n.comm_user_rank, "ncclCommUserRank");
    sym(n.all_reduce, "ncclAllReduce");
    sym(n.get_version, "ncclGetVersion");
    sym(n.error_string, "ncclGetErrorString");
    if (!n.get_unique_id || !n.comm_init_rank || !n.comm_destroy || !n.all_reduce || !n.comm_count)
      n.err = "NCCL library lacks the ncclGetUniqueId / ncclCommInitRank / ncclAllReduce entry points";
  });
  return n;
}

std::string nccl_msg(const char* what, ncclResult_t r) {
  const Nccl& n = nccl();
  return std::string(what) + ": " + (n.error_string ? n.error_string(r) : ("NCCL error " + std::to_string(r)));
}

}  // namespace

namespace tgcomm {

bool available(std::string& err) {
  const Nccl& n = nccl();
  err = n.err;
  return n.err.empty();
}

bool allreduce_sum(void* buf, std::size_t count, tg_dtype dtype, void* comm, cudaStream_t st, std::string& err) {
  Nccl& n = nccl();
  if (!n.err.empty()) { err = n.err; return false; }
  // ncclDataType_t: ncclFloat32 = 7, ncclFloat64 = 8; ncclRedOp_t: ncclSum = 0
  const ncclResult_t r = n.all_reduce(buf, buf, count, dtype == TG_F64 ? 8 : 7, 0, comm, st);
  if (r != 0) { err = nccl_msg("ncclAllReduce", r); return false; }
  return true;
}

void* nccl_symbol(const char* name) {
  Nccl& n = nccl();
  return n.so ? dlsym(n.so, name) : nullptr;
}

int comm_size(void* comm) {
  Nccl& n = nccl();
  int c = 0;
  if (!n.err.empty() || n.comm_count(comm, &c) != 0) return -1;
  return c;
}

}  // namespace tgcomm

extern "C" {

tg_status tg_nccl_get_unique_id(void* id_out) {
  if (!id_out) return tgcomm::fail_status(TG_INVALID_ARGUMENT, "tg_nccl_get_unique_id: NULL id");
  Nccl& n = nccl();
  if (!n.err.empty()) return tgcomm::fail_status(TG_NCCL, n.err);
  NcclUid u{};
  const ncclResult_t r = n.get_unique_id(&u);
  if (r != 0) return tgcomm::fail_status(TG_NCCL, nccl_msg("ncclGetUniqueId", r));
  std::memcpy(id_out, u.internal, sizeof u.internal);
  return TG_OK;
}

tg_status tg_nccl_comm_init(int nranks, const void* id, int rank, tg_comm_t* out) {
  if (!id || !out) return tgcomm::fail_status(TG_INVALID_ARGUMENT, "tg_nccl_comm_init: NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return tgcomm::fail_status(TG_INVALID_ARGUMENT, "tg_nccl_comm_init: rank " + std::to_string(rank) + " of " +
                                                        std::to_string(nranks));
  Nccl& n = nccl();
  if (!n.err.empty()) return tgcomm::fail_status(TG_NCCL, n.err);
  NcclUid u{};
  std::memcpy(u.internal, id, sizeof u.internal);
  ncclComm_t c = nullptr;
  const ncclResult_t r = n.comm_init_rank(&c, nranks, u, rank);
  if (r != 0) return tgcomm::fail_status(TG_NCCL, nccl_msg("ncclCommInitRank", r));
  *out = c;
  return TG_OK;
}

tg_status tg_nccl_comm_destroy(tg_comm_t comm) {
  if (!comm) return TG_OK;
  Nccl& n = nccl();
  if (!n.err.empty()) return tgcomm::fail_status(TG_NCCL, n.err);
  const ncclResult_t r = n.comm_destroy(comm);
  if (r != 0) return tgcomm::fail_status(TG_NCCL, nccl_msg("ncclCommDestroy", r));
  return TG_OK;
}

int tg_nccl_version(void) {
  Nccl& n = nccl();
  int v = 0;
  if (n.err.empty() && n.get_version) n.get_version(&v);
  return v;
}

}  // extern "C"
