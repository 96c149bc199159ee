// optim.cu — Adam step (optim.py:37-49) and row compaction (cloud.py:86-89,
// optim.py:51-55), plus library metadata entry points.
//
// Adam is a pure streaming kernel (read param, grad, m, v; write param, m, v:
// 28 B per float); float4-vectorised with a scalar tail, grid-stride over
// 4 x 148 CTAs per SM worth of blocks.
#include "tgs_common.cuh"

namespace tgs {

__device__ __forceinline__ void adam1(float &p, float g, float &m, float &v, float lr, float b1, float b2, float eps,
                                      float bc1, float bc2) {
  m = b1 * m + (1.0f - b1) * g;
  v = b2 * v + (1.0f - b2) * g * g;
  const float mh = m / bc1, vh = v / bc2;
  p -= lr * mh / (sqrtf(vh) + eps);
}

__global__ void k_adam(float *__restrict__ p, const float *__restrict__ g, float *__restrict__ m,
                       float *__restrict__ v, int64_t n, float lr, float b1, float b2, float eps, float bc1,
                       float bc2, bool vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    const int64_t n4 = n / 4;
    for (int64_t j = i; j < n4; j += stride) {
      float4 pp = reinterpret_cast<float4 *>(p)[j];
      const float4 gg = reinterpret_cast<const float4 *>(g)[j];
      float4 mm = reinterpret_cast<float4 *>(m)[j];
      float4 vv = reinterpret_cast<float4 *>(v)[j];
      adam1(pp.x, gg.x, mm.x, vv.x, lr, b1, b2, eps, bc1, bc2);
      adam1(pp.y, gg.y, mm.y, vv.y, lr, b1, b2, eps, bc1, bc2);
      adam1(pp.z, gg.z, mm.z, vv.z, lr, b1, b2, eps, bc1, bc2);
      adam1(pp.w, gg.w, mm.w, vv.w, lr, b1, b2, eps, bc1, bc2);
      reinterpret_cast<float4 *>(p)[j] = pp;
      reinterpret_cast<float4 *>(m)[j] = mm;
      reinterpret_cast<float4 *>(v)[j] = vv;
    }
    const int64_t k = n4 * 4 + threadIdx.x;  // 0..3 tail floats
    if (blockIdx.x == 0 && k < n) adam1(p[k], g[k], m[k], v[k], lr, b1, b2, eps, bc1, bc2);
    return;
  }
  for (; i < n; i += stride) adam1(p[i], g[i], m[i], v[i], lr, b1, b2, eps, bc1, bc2);
}

__global__ void k_gather_rows(const float *__restrict__ in, float *__restrict__ out,
                              const int64_t *__restrict__ keep, int64_t n_keep, int row) {
  const int64_t total = n_keep * row;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t r = e / row, c = e - r * row;
    out[e] = in[keep[r] * row + c];
  }
}

}  // namespace tgs

using namespace tgs;

extern "C" int tgs_version(void) { return 1; }

extern "C" const char *tgs_last_error_string(int status) {
  switch (status) {
    case TGS_OK: return "ok";
    case TGS_ERR_INVALID: return "invalid argument";
    case TGS_ERR_DEGENERATE_ROTATION: return "quaternion with (near-)zero norm";
    case TGS_ERR_CUDA: return "CUDA error";
    case TGS_ERR_UNSUPPORTED: return "unsupported configuration";
    case TGS_ERR_CAPACITY: return "buffer capacity exceeded";
    default: return "unknown status";
  }
}

extern "C" int tgs_adam_step(float *param, const float *grad, float *m, float *v, int64_t n, float lr, float beta1,
                             float beta2, float eps, float bias_c1, float bias_c2, tgs_stream_t stream) {
  if (n < 0 || !(bias_c1 > 0.0f) || !(bias_c2 > 0.0f)) return TGS_ERR_INVALID;
  if (n == 0) return TGS_OK;
  const bool vec = ((reinterpret_cast<uintptr_t>(param) | reinterpret_cast<uintptr_t>(grad) |
                     reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  const int64_t work = vec ? n / 4 + 1 : n;
  const unsigned grid = (unsigned)tmin<int64_t>(ceil_div<int64_t>(work, 256), 148 * 16);
  k_adam<<<grid, 256, 0, as_stream(stream)>>>(param, grad, m, v, n, lr, beta1, beta2, eps, bias_c1, bias_c2, vec);
  return launch_status();
}

extern "C" int tgs_gather_rows(const float *in, float *out, const int64_t *keep, int64_t n_keep, int32_t row_floats,
                               tgs_stream_t stream) {
  if (n_keep < 0 || row_floats < 1) return TGS_ERR_INVALID;
  if (n_keep == 0) return TGS_OK;
  const unsigned grid = (unsigned)tmin<int64_t>(ceil_div<int64_t>(n_keep * row_floats, 256), 148 * 16);
  k_gather_rows<<<grid, 256, 0, as_stream(stream)>>>(in, out, keep, n_keep, row_floats);
  return launch_status();
}
