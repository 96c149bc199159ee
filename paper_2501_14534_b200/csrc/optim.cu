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

// All parameter groups in one launch.  Groups are contiguous 64-float aligned
// ranges of the flat buffers, so a float4 chunk never straddles two groups; the
// padding between groups is skipped.  The mask penalties of total_loss
// (masking.py:60-67: L_m = mean sigmoid(m), L_sh = mean sum_l w_l sigmoid(m_l))
// are added to their groups' gradients in registers (and written back), i.e.
// g += lambda * sigmoid'(logit) * weight / n before the update.
struct AdamGroupArgs {
  int64_t off[9];      // group starts (floats) and the end of the last group
  int64_t size[8];
  float lr_bc1[8], inv_bc2[8];
  int kind[8];         // 0: plain, 1: Gaussian-mask penalty, 2: SH-band-mask penalty
  int ngroups;
  float b1, b2, eps, lam_m, lam_sh, inv_n, wband[3];
};

__global__ void __launch_bounds__(256) k_adam_groups(float *__restrict__ p, float *__restrict__ g,
                                                     float *__restrict__ m, float *__restrict__ v, AdamGroupArgs a) {
  // float4 chunks from the first group's start to the padded end of the last one
  // (groups need not start at 0: a data-parallel bucket steps a subset of the groups)
  const int64_t c0 = a.off[0] / 4, n4 = a.off[a.ngroups] / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n4; c += stride) {
    const int64_t e = 4 * c;
    int k = 0;
#pragma unroll
    for (int q = 1; q < 8; ++q)
      if (q < a.ngroups && e >= a.off[q]) k = q;
    const int64_t local = e - a.off[k];
    if (local < 0 || local >= a.size[k]) continue;  // padding / gaps between groups
    float4 pp = reinterpret_cast<float4 *>(p)[c];
    float4 gg = reinterpret_cast<const float4 *>(g)[c];
    float4 mm = reinterpret_cast<float4 *>(m)[c];
    float4 vv = reinterpret_cast<float4 *>(v)[c];
    float *pq = &pp.x, *gq = &gg.x, *mq = &mm.x, *vq = &vv.x;
    const int kind = a.kind[k];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (local + j >= a.size[k]) break;
      if (kind) {
        const float sg = 1.0f / (1.0f + expf(-pq[j]));
        const float w = kind == 1 ? a.lam_m : a.lam_sh * a.wband[(local + j) % 3];
        gq[j] += w * (sg * (1.0f - sg)) * a.inv_n;
      }
      // optim.py:41-49 with lr / bc1 and 1 / bc2 folded on the host side of the launch
      const float gj = gq[j];
      mq[j] = a.b1 * mq[j] + (1.0f - a.b1) * gj;
      vq[j] = a.b2 * vq[j] + (1.0f - a.b2) * gj * gj;
      pq[j] -= __fdividef(a.lr_bc1[k] * mq[j], sqrtf(vq[j] * a.inv_bc2[k]) + a.eps);
    }
    reinterpret_cast<float4 *>(p)[c] = pp;
    reinterpret_cast<float4 *>(m)[c] = mm;
    reinterpret_cast<float4 *>(v)[c] = vv;
    if (kind) reinterpret_cast<float4 *>(g)[c] = gg;
  }
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

extern "C" int tgs_adam_step_groups(float *param, float *grad, float *m, float *v, int32_t ngroups,
                                    const int64_t *offsets, const int64_t *sizes, const float *lrs,
                                    const float *bias_c1, const float *bias_c2, const int32_t *kinds, float beta1,
                                    float beta2, float eps, float lambda_m, float lambda_sh,
                                    const float *band_weights, int64_t n_gaussians, tgs_stream_t stream) {
  if (ngroups < 1 || ngroups > 8 || !param || !grad || !m || !v || !offsets || !sizes || !lrs || !bias_c1 ||
      !bias_c2 || !kinds || n_gaussians < 0)
    return TGS_ERR_INVALID;
  if (((reinterpret_cast<uintptr_t>(param) | reinterpret_cast<uintptr_t>(grad) | reinterpret_cast<uintptr_t>(m) |
        reinterpret_cast<uintptr_t>(v)) & 15) != 0)
    return TGS_ERR_INVALID;
  AdamGroupArgs a{};
  a.ngroups = ngroups;
  for (int k = 0; k < ngroups; ++k) {
    if (offsets[k] % 64 != 0 || sizes[k] < 0 || (k > 0 && offsets[k] < offsets[k - 1] + sizes[k - 1]) ||
        !(bias_c1[k] > 0.0f) || !(bias_c2[k] > 0.0f) || kinds[k] < 0 || kinds[k] > 2)
      return TGS_ERR_INVALID;
    a.off[k] = offsets[k];
    a.size[k] = sizes[k];
    a.lr_bc1[k] = lrs[k] / bias_c1[k];
    a.inv_bc2[k] = 1.0f / bias_c2[k];
    a.kind[k] = kinds[k];
  }
  a.off[ngroups] = (offsets[ngroups - 1] + sizes[ngroups - 1] + 63) / 64 * 64;
  a.b1 = beta1;
  a.b2 = beta2;
  a.eps = eps;
  a.lam_m = lambda_m;
  a.lam_sh = lambda_sh;
  a.inv_n = n_gaussians > 0 ? 1.0f / (float)n_gaussians : 0.0f;
  for (int l = 0; l < 3; ++l) a.wband[l] = band_weights ? band_weights[l] : 0.0f;
  const int64_t n4 = a.off[ngroups] / 4 - a.off[0] / 4;
  if (n4 <= 0) return TGS_OK;
  const unsigned grid = (unsigned)tmin<int64_t>(ceil_div<int64_t>(n4, 256), 148 * 8);
  k_adam_groups<<<grid, 256, 0, as_stream(stream)>>>(param, grad, m, v, a);
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
