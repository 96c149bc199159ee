// tgs_common.cuh — shared host/device plumbing for libtgs.so
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>

#include "../../include/tgs.h"

namespace tgs {

constexpr float kAlphaSkip = 1.0f / 255.0f;  // rasterizer.py:38
constexpr float kAlphaMax = 0.99f;           // rasterizer.py:39
constexpr float kEMin = -4.5f;               // rasterizer.py:40
constexpr float kTTerm = 1e-4f;              // rasterizer.py:41

inline int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return TGS_OK;
  fprintf(stderr, "[tgs] CUDA error: %s\n", cudaGetErrorString(e));
  return TGS_ERR_CUDA;
}

// status after a kernel launch (launch-configuration errors only; async faults
// surface at the caller's next synchronisation)
inline int launch_status() { return cuda_status(cudaGetLastError()); }

inline cudaStream_t as_stream(tgs_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

template <typename T>
__host__ __device__ inline T ceil_div(T a, T b) {
  return (a + b - 1) / b;
}

template <typename T>
__host__ __device__ inline T tmin(T a, T b) {
  return a < b ? a : b;
}
template <typename T>
__host__ __device__ inline T tmax(T a, T b) {
  return a < b ? b : a;
}

// Function attributes (dynamic shared memory, carve-out) are per DEVICE: set them once
// per (kernel, device).  `done` is the kernel's bitmask of devices already configured;
// two threads racing here both set the (idempotent) attribute, which is harmless.
template <typename F>
inline int attr_once_per_device(std::atomic<uint64_t> &done, F &&set) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TGS_ERR_CUDA;
  const uint64_t bit = dev < 64 ? 1ull << dev : 0ull;  // devices >= 64: set on every call
  if (bit && (done.load(std::memory_order_acquire) & bit)) return TGS_OK;
  if (set() != cudaSuccess) return cuda_status(cudaGetLastError());
  if (bit) done.fetch_or(bit, std::memory_order_release);
  return TGS_OK;
}

inline size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Carve {
  char *base;
  size_t off = 0;
  explicit Carve(void *p) : base(static_cast<char *>(p)) {}
  template <typename T>
  T *take(size_t count) {
    T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
    off = align_up(off + count * sizeof(T));
    return p;
  }
};

}  // namespace tgs
