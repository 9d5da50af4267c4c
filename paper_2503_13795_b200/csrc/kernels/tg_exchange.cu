// tg_exchange.cu — the data-parallel exchange fused with the GD update
// (SURVEY.md §8f row 4): one kernel that sums the d-length gradient over the
// ranks through the symmetric window's peer memory, and applies
// x -= gamma * g / b_global (sgd_step) to the local replica.
//
// The window is NCCL symmetric memory (ncclMemAlloc + ncclCommWindowRegister,
// NCCL >= 2.28 device API): every rank's buffer is mapped into every other
// rank's address space over NVLink (LSA pointers), and on NVSwitch systems a
// multicast (NVLS) address covers all of them at once.  Layout per rank:
//   [grad: count scalars | pad to 256 B | flagsA: kMaxCtas u32 | flagB: u32]
// Per call (epoch e = 1, 2, ...), CTA c of rank r:
//   1. barrier A: red.release.sys +1 on flagsA[c] of every rank, then waits for
//      its own flagsA[c] >= e * W — every rank's CTA c has started, so every
//      rank's local gradient sum (the previous kernel on its stream) is final;
//   2. reduces its share of rank r's slice [r * chunk, (r + 1) * chunk):
//      NVLS: multimem.ld_reduce (the switch sums) then multimem.st (the
//      switch broadcasts); otherwise ordinary loads of the W peers' values,
//      summed in rank order 0..W-1 (deterministic), stored back to every
//      peer's buffer — identical reduced values on every rank either way;
//   3. barrier B: red.release.sys +1 on flagB of every rank, waits for
//      flagB >= e * W * C — every slice is written everywhere;
//   4. the GD update of all d local parameters from the (now global) sum,
//      with k_gd's expression, so one rank equals tg_gd_update bit for bit.
// Later calls cannot overtake: a rank rewrites its buffer (next step's
// forward_backward) only after passing barrier B, which every reader of that
// buffer reached after its last read.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "nccl.h"
#include "nccl_device.h"
#include "tg_abi.h"
#include "tg_comm.hpp"

namespace tgx {

constexpr int kMaxCtas = 256;
constexpr int kMaxRanks = 72;
constexpr int kThreads = 512;

struct Bases {
  char* peer[kMaxRanks];   // LSA base of every rank's window (peer[rank] = local)
  char* mc;                // NVLS multicast base, or null
};

__device__ __forceinline__ void red_release_sys(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float mm_ld_reduce(const float* p) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st(float* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// The call's epoch comes from the barrier counter itself, so a captured CUDA
// graph replays correctly: when CTA c of this rank reads flagsA[c] at the start
// of call e it holds (e - 1) * W plus the arrivals of faster peers for call e
// (< W: no rank arrives for call e + 1 before this one passed barrier B of e).
template <class T, bool MM>
__global__ void __launch_bounds__(kThreads) k_allreduce_gd(const Bases* __restrict__ bases, std::size_t flags_off,
                                                           std::size_t count, int rank, int world,
                                                           T* __restrict__ params, T gamma, T b) {
  const unsigned C = gridDim.x, c = blockIdx.x;
  T* grad = reinterpret_cast<T*>(bases->peer[rank]);
  unsigned* flagsA = reinterpret_cast<unsigned*>(bases->peer[rank] + flags_off);
  unsigned* flagB = flagsA + kMaxCtas;
  __shared__ unsigned s_epoch;
  if (threadIdx.x == 0) {
    const unsigned epoch = ld_acquire_sys(flagsA + c) / static_cast<unsigned>(world) + 1u;
    s_epoch = epoch;
    for (int p = 0; p < world; ++p) red_release_sys(reinterpret_cast<unsigned*>(bases->peer[p] + flags_off) + c, 1u);
    while (ld_acquire_sys(flagsA + c) < epoch * static_cast<unsigned>(world)) {
    }
  }
  __syncthreads();
  const unsigned epoch = s_epoch;
  const std::size_t chunk = (count + world - 1) / world;
  const std::size_t lo = static_cast<std::size_t>(rank) * chunk;
  const std::size_t hi = lo + chunk < count ? lo + chunk : count;
  for (std::size_t i = lo + std::size_t(c) * kThreads + threadIdx.x; i < hi; i += std::size_t(C) * kThreads) {
    if constexpr (MM) {
      float* m = reinterpret_cast<float*>(bases->mc) + i;
      mm_st(m, mm_ld_reduce(m));
    } else {
      T v = reinterpret_cast<const T*>(bases->peer[0])[i];
      for (int p = 1; p < world; ++p) v += reinterpret_cast<const T*>(bases->peer[p])[i];
      for (int p = 0; p < world; ++p) reinterpret_cast<T*>(bases->peer[p])[i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if constexpr (MM) asm volatile("fence.proxy.alias;" ::: "memory");
    for (int p = 0; p < world; ++p)
      red_release_sys(reinterpret_cast<unsigned*>(bases->peer[p] + flags_off) + kMaxCtas, 1u);
    while (ld_acquire_sys(flagB) < epoch * static_cast<unsigned>(world) * C) {
    }
    if constexpr (MM) asm volatile("fence.proxy.alias;" ::: "memory");   // multicast stores -> unicast loads
  }
  __syncthreads();
  for (std::size_t i = std::size_t(c) * kThreads + threadIdx.x; i < count; i += std::size_t(C) * kThreads)
    params[i] = params[i] - gamma * grad[i] / b;
}

// LSA / multicast base pointers of a registered window (NCCL device API).
__global__ void k_window_bases(ncclWindow_t win, ncclDevComm dc, int world, int want_mm, Bases* out) {
  for (int p = 0; p < world; ++p) out->peer[p] = static_cast<char*>(ncclGetLsaPointer(win, 0, p));
  out->mc = want_mm ? static_cast<char*>(ncclGetLsaMultimemPointer(win, 0, dc)) : nullptr;
}

}  // namespace tgx

// ---------------------------------------------------------------------------
// host: window lifetime and the fused step (C-ABI in include/tg_abi.h)
// ---------------------------------------------------------------------------

struct tg_window {
  ncclComm_t comm = nullptr;
  tg_dtype dtype = TG_F32;
  std::size_t count = 0, flags_off = 0, bytes = 0;
  int rank = 0, world = 1;
  bool multimem = false;
  void* buf = nullptr;
  ncclWindow_t win = nullptr;
  ncclDevComm dev{};
  bool dev_ok = false;
  tgx::Bases* d_bases = nullptr;
};

namespace {

template <class F>
F sym(const char* name) {
  return reinterpret_cast<F>(tgcomm::nccl_symbol(name));
}

tg_status nccl_fail(const char* what, ncclResult_t r) {
  auto es = sym<const char* (*)(ncclResult_t)>("ncclGetErrorString");
  return tgcomm::fail_status(TG_NCCL, std::string(what) + ": " + (es ? es(r) : ("NCCL error " + std::to_string(r))));
}

void release(tg_window* w) {
  if (!w) return;
  if (w->d_bases) cudaFree(w->d_bases);
  if (w->dev_ok)
    if (auto f = sym<ncclResult_t (*)(ncclComm_t, ncclDevComm const*)>("ncclDevCommDestroy")) f(w->comm, &w->dev);
  if (w->win)
    if (auto f = sym<ncclResult_t (*)(ncclComm_t, ncclWindow_t)>("ncclCommWindowDeregister")) f(w->comm, w->win);
  if (w->buf)
    if (auto f = sym<ncclResult_t (*)(void*)>("ncclMemFree")) f(w->buf);
  delete w;
}

}  // namespace

extern "C" {

tg_status tg_window_create(tg_comm_t comm, tg_dtype dtype, size_t count, int flags, tg_window_t* out) {
  if (!comm || !out) return tgcomm::fail_status(TG_INVALID_ARGUMENT, "tg_window_create: NULL argument");
  if (dtype != TG_F32 && dtype != TG_F64) return tgcomm::fail_status(TG_INVALID_ARGUMENT, "tg_window_create: bad dtype");
  *out = nullptr;
  std::string err;
  if (!tgcomm::available(err)) return tgcomm::fail_status(TG_NCCL, err);
  auto mem_alloc = sym<ncclResult_t (*)(void**, std::size_t)>("ncclMemAlloc");
  auto win_reg = sym<ncclResult_t (*)(ncclComm_t, void*, std::size_t, ncclWindow_t*, int)>("ncclCommWindowRegister");
  auto dev_create = sym<ncclResult_t (*)(ncclComm_t, ncclDevCommRequirements_t const*, ncclDevComm_t*)>("ncclDevCommCreate");
  auto user_rank = sym<ncclResult_t (*)(ncclComm_t, int*)>("ncclCommUserRank");
  auto comm_count = sym<ncclResult_t (*)(ncclComm_t, int*)>("ncclCommCount");
  if (!mem_alloc || !win_reg || !dev_create || !user_rank || !comm_count)
    return tgcomm::fail_status(TG_NCCL, "tg_window_create: the loaded NCCL has no symmetric-memory device API (needs >= 2.28)");
  auto* w = new tg_window;
  w->comm = static_cast<ncclComm_t>(comm);
  w->dtype = dtype;
  w->count = count;
  ncclResult_t r;
  if ((r = user_rank(w->comm, &w->rank)) != ncclSuccess || (r = comm_count(w->comm, &w->world)) != ncclSuccess) {
    release(w);
    return nccl_fail("ncclCommUserRank / ncclCommCount", r);
  }
  if (w->world > tgx::kMaxRanks) {
    release(w);
    return tgcomm::fail_status(TG_INVALID_ARGUMENT, "tg_window_create: more ranks than the fused exchange supports");
  }
  const std::size_t tsz = dtype == TG_F64 ? 8 : 4;
  w->flags_off = (count * tsz + 255) / 256 * 256;
  w->bytes = (w->flags_off + (tgx::kMaxCtas + 1) * 4 + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT *
             NCCL_WIN_REQUIRED_ALIGNMENT;
  if ((r = mem_alloc(&w->buf, w->bytes)) != ncclSuccess) {
    release(w);
    return nccl_fail("ncclMemAlloc", r);
  }
  if (cudaMemset(w->buf, 0, w->bytes) != cudaSuccess) {
    release(w);
    return tgcomm::fail_status(TG_CUDA, "tg_window_create: cudaMemset failed");
  }
  cudaDeviceSynchronize();
  if ((r = win_reg(w->comm, w->buf, w->bytes, &w->win, NCCL_WIN_COLL_SYMMETRIC)) != ncclSuccess) {
    release(w);
    return nccl_fail("ncclCommWindowRegister", r);
  }
  // multimem (NVLS) when asked for and the fabric offers it; LSA pointers otherwise
  ncclDevCommRequirements_t req{};
  req.lsaMultimem = (flags & TG_WINDOW_MULTIMEM) != 0 && dtype == TG_F32;
  r = dev_create(w->comm, &req, &w->dev);
  if (r != ncclSuccess && req.lsaMultimem) {
    req.lsaMultimem = false;
    r = dev_create(w->comm, &req, &w->dev);
  }
  if (r != ncclSuccess) {
    release(w);
    return nccl_fail("ncclDevCommCreate", r);
  }
  w->dev_ok = true;
  w->multimem = req.lsaMultimem;
  if (w->dev.lsaSize != w->world) {
    release(w);
    return tgcomm::fail_status(TG_NCCL, "tg_window_create: not every rank is load/store reachable (LSA team " +
                                            std::to_string(w->dev.lsaSize) + " of " + std::to_string(w->world) + ")");
  }
  if (cudaMalloc(&w->d_bases, sizeof(tgx::Bases)) != cudaSuccess) {
    release(w);
    return tgcomm::fail_status(TG_CUDA, "tg_window_create: cudaMalloc failed");
  }
  tgx::k_window_bases<<<1, 1>>>(w->win, w->dev, w->world, w->multimem ? 1 : 0, w->d_bases);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    cudaGetLastError();
    release(w);
    return tgcomm::fail_status(TG_CUDA, "tg_window_create: window pointer query failed");
  }
  *out = w;
  return TG_OK;
}

tg_status tg_window_destroy(tg_window_t w) {
  if (w) cudaDeviceSynchronize();
  release(w);
  return TG_OK;
}

void* tg_window_buffer(tg_window_t w) { return w ? w->buf : nullptr; }
int tg_window_multimem(tg_window_t w) { return w && w->multimem ? 1 : 0; }

tg_status tg_window_allreduce_gd(tg_window_t w, void* params, double gamma, size_t global_batch, tg_stream_t stream) {
  if (!w) return tgcomm::fail_status(TG_INVALID_HANDLE, "tg_window_allreduce_gd: NULL window");
  if (global_batch == 0) return tgcomm::fail_status(TG_INVALID_ARGUMENT, "train_step: batch empty");
  if (w->count && !params) return tgcomm::fail_status(TG_INVALID_ARGUMENT, "tg_window_allreduce_gd: NULL params");
  if (w->count == 0) return TG_OK;
  auto st = static_cast<cudaStream_t>(stream);
  const std::size_t per_rank = (w->count + w->world - 1) / w->world;
  unsigned grid = static_cast<unsigned>((per_rank + tgx::kThreads * 4 - 1) / (tgx::kThreads * 4));
  grid = grid < 1 ? 1 : grid > 128 ? 128 : grid;   // co-resident on any B200 (spin barriers)
  // every rank must launch the same grid: it depends on count and world only
  if (w->dtype == TG_F64) {
    tgx::k_allreduce_gd<double, false><<<grid, tgx::kThreads, 0, st>>>(
        w->d_bases, w->flags_off, w->count, w->rank, w->world, static_cast<double*>(params), gamma,
        static_cast<double>(global_batch));
  } else if (w->multimem) {
    tgx::k_allreduce_gd<float, true><<<grid, tgx::kThreads, 0, st>>>(
        w->d_bases, w->flags_off, w->count, w->rank, w->world, static_cast<float*>(params),
        static_cast<float>(gamma), static_cast<float>(global_batch));
  } else {
    tgx::k_allreduce_gd<float, false><<<grid, tgx::kThreads, 0, st>>>(
        w->d_bases, w->flags_off, w->count, w->rank, w->world, static_cast<float*>(params),
        static_cast<float>(gamma), static_cast<float>(global_batch));
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return tgcomm::fail_status(TG_CUDA, std::string("tg_window_allreduce_gd: ") + cudaGetErrorString(e));
  return TG_OK;
}

}  // extern "C"
