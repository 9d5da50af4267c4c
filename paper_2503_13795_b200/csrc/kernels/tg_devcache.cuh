// tg_devcache.cuh — per-device, thread-safe launch-attribute caches.
//
// cudaFuncSetAttribute (dynamic shared memory opt-in) and the SM count are
// properties of one device: a process that drives several GPUs must set /
// query them on each, and host threads may launch concurrently.  These
// helpers key the "done" state by the current device ordinal.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace tgk {

constexpr int kMaxDevices = 64;

inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  return d & (kMaxDevices - 1);
}

/// Runs f() (returning cudaError_t) once per device until it succeeds.
struct PerDeviceOnce {
  std::atomic<std::uint64_t> done{0};
  template <class F>
  cudaError_t ensure(F&& f) {
    const std::uint64_t bit = 1ull << current_device();
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    const cudaError_t e = f();
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
  }
};

/// Largest dynamic shared memory opted into so far, per device.
struct PerDeviceMax {
  std::atomic<int> v[kMaxDevices] = {};
  template <class F>
  cudaError_t raise_to(int want, F&& set) {
    std::atomic<int>& cur = v[current_device()];
    if (cur.load(std::memory_order_acquire) >= want) return cudaSuccess;
    const cudaError_t e = set(want);
    if (e == cudaSuccess) {
      int c = cur.load();
      while (c < want && !cur.compare_exchange_weak(c, want)) {
      }
    }
    return e;
  }
};

/// An int computed once per device by f() (a positive value; 0 = not yet computed).
struct PerDeviceValue {
  std::atomic<int> v[kMaxDevices] = {};
  template <class F>
  int get(F&& f) {
    std::atomic<int>& c = v[current_device()];
    int n = c.load(std::memory_order_acquire);
    if (n <= 0) {
      n = f();
      c.store(n, std::memory_order_release);
    }
    return n;
  }
};

/// Streaming multiprocessors of the current device (148 on B200).
inline int sm_count() {
  static std::atomic<int> cache[kMaxDevices] = {};
  const int d = current_device();
  int n = cache[d].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    cache[d].store(n, std::memory_order_relaxed);
  }
  return n;
}

}  // namespace tgk
