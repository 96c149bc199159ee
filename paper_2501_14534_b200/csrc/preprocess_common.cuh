// preprocess_common.cuh — helpers shared by the preprocess forward and backward.
#pragma once

#include "tgs_common.cuh"
#include "tgs_math.cuh"

namespace tgs {

constexpr int kPreBlock = 128;

__device__ __forceinline__ float max0(float v) { return v < 0.0f ? 0.0f : v; }

struct GaussFwd {
  float Mg, band[3];
  bool alpha_ok, valid, ok, visible, degenerate;
  float s_raw[3], sc[3];
  float qn[4], qnorm;
  float Rg[9], S[9];
  float t[3], Mj[6];
  float mean[2], c00, c01, c11, det, conic[3], radius, area;
  float dir[3], dnorm;
  float pre[3], col[3];
};

// Loads the rest block of `count` Gaussians starting at `base` into smem.
__device__ __forceinline__ void stage_rest(const float *__restrict__ rest, int64_t base, int count, float *sm) {
  const float *src = rest + base * 45;
  const int total = count * 45;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int n4 = total / 4;
    for (int j = threadIdx.x; j < n4; j += blockDim.x)
      reinterpret_cast<float4 *>(sm)[j] = __ldg(reinterpret_cast<const float4 *>(src) + j);
    for (int j = n4 * 4 + threadIdx.x; j < total; j += blockDim.x) sm[j] = __ldg(src + j);
  } else {
    for (int j = threadIdx.x; j < total; j += blockDim.x) sm[j] = __ldg(src + j);
  }
}

// ---- one-shot TMA bulk copy of the CTA's sh_rest block (cp.async.bulk, SASS UBLKCP):
// thread 0 issues ONE 1-D bulk copy global -> shared completing on an mbarrier, the
// threads load their per-Gaussian parameters meanwhile and wait on the barrier only
// when the block is needed.  Returns false (nothing issued) when the block cannot go
// through the bulk path (misaligned or a size that is not a multiple of 16 bytes,
// i.e. a partial last block); the caller then uses stage_rest + __syncthreads.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ bool stage_rest_issue(const float *__restrict__ rest, int64_t base, int count, float *sm,
                                                 uint64_t *bar) {
  const float *src = rest + base * 45;
  const uint32_t bytes = (uint32_t)count * 45u * 4u;
  if ((reinterpret_cast<uintptr_t>(src) & 15) || (bytes & 15) || bytes == 0) return false;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sm)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
  }
  return true;
}

// every thread: wait for the bulk copy (phase 0); the barrier must have been
// initialised before a __syncthreads that precedes this call
__device__ __forceinline__ void stage_rest_wait(uint64_t *bar) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar))
      : "memory");
}

// unit quaternion -> rotation (geometry.py:19-41); returns the raw norm
__device__ __forceinline__ float quat_rot(const tgs_cloud &cl, int64_t i, float Rg[9], float qn[4] = nullptr) {
  const float qw = cl.rotations[4 * i], qx = cl.rotations[4 * i + 1];
  const float qy = cl.rotations[4 * i + 2], qz = cl.rotations[4 * i + 3];
  const float qnorm = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  const float w = qw / qnorm, x = qx / qnorm, y = qy / qnorm, z = qz / qnorm;
  if (qn) {
    qn[0] = w; qn[1] = x; qn[2] = y; qn[3] = z;
  }
  Rg[0] = 1.0f - 2.0f * (y * y + z * z);
  Rg[1] = 2.0f * (x * y - w * z);
  Rg[2] = 2.0f * (x * z + w * y);
  Rg[3] = 2.0f * (x * y + w * z);
  Rg[4] = 1.0f - 2.0f * (x * x + z * z);
  Rg[5] = 2.0f * (y * z - w * x);
  Rg[6] = 2.0f * (x * z - w * y);
  Rg[7] = 2.0f * (y * z + w * x);
  Rg[8] = 1.0f - 2.0f * (x * x + y * y);
  return qnorm;
}

}  // namespace tgs
