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
  // the float4 chunks to update: up to 8 ranges [rb[r], rb[r] + 4 (r4[r+1] - r4[r])) (a ZeRO
  // shard, the rows of a preprocess-backward chunk), r4 = prefix sums of their float4 counts
  int nranges;
  int64_t rb[8], r4[9];
  const double *terms;  // optional divergence guard: loss terms of this step (nterms doubles)
  int nterms;
  int32_t *nonfinite;   // set to 1 (and no parameter touched) when a term is not finite
};

// training.py:298-308 raises DivergenceError BEFORE the backward's results reach the
// optimizer when the loss is not finite; on the device the same guard skips the whole
// update (parameters and moments stay as they were) and raises a flag the host reads.
__device__ __forceinline__ bool loss_nonfinite(const AdamGroupArgs &a) {
  __shared__ int s_bad;
  if (threadIdx.x == 0) {
    int bad = 0;
    for (int i = 0; i < a.nterms; ++i) bad |= !isfinite(a.terms[i]);
    s_bad = bad;
  }
  __syncthreads();
  return s_bad != 0;
}

__global__ void __launch_bounds__(256) k_adam_groups(float *__restrict__ p, float *__restrict__ g,
                                                     float *__restrict__ m, float *__restrict__ v, AdamGroupArgs a) {
  if (a.terms && loss_nonfinite(a)) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.nonfinite) *a.nonfinite = 1;
    return;
  }
  // float4 chunks of the ranges (each clipped to [first group start, padded end of the last
  // group] on the host; groups need not start at 0: a data-parallel bucket steps a subset
  // of the groups).  The groups keep their global indices inside a range, so the per-group
  // lr, bias corrections and SH-band weights are unchanged.
  const int64_t n4 = a.r4[a.nranges];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ci < n4; ci += stride) {
    int r = 0;
#pragma unroll
    for (int q = 1; q < 8; ++q)
      if (q < a.nranges && ci >= a.r4[q]) r = q;
    const int64_t c = a.rb[r] / 4 + (ci - a.r4[r]);
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

// Stream compaction of the kept rows (masking.prune_by_mask's np.nonzero, masking.py:70-81;
// significance.prune_by_significance's, significance.py:81-99): row i is kept when
// flags[i] != 0, or (flags == NULL) when x[i] > thr.  One launch: tiles of 4096 rows
// take tickets in launch order, scan their keep counts in the block and chain the tile
// prefixes by decoupled look-back (30-bit payloads), then write the kept row numbers in
// ascending order; the total lands in *count.
constexpr uint32_t kSelAgg = 1u << 30, kSelInc = 2u << 30, kSelMask = (1u << 30) - 1;
constexpr int kSelItems = 16, kSelThreads = 256, kSelTile = kSelItems * kSelThreads;

__global__ void __launch_bounds__(kSelThreads) k_select_rows(const uint8_t *__restrict__ flags,
                                                             const float *__restrict__ x, float thr, int64_t n,
                                                             int64_t *__restrict__ idx, int64_t *__restrict__ count,
                                                             uint32_t *__restrict__ status,
                                                             uint32_t *__restrict__ ticket) {
  __shared__ uint32_t ws[kSelThreads / 32], s_tile, s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * kSelTile + (int64_t)threadIdx.x * kSelItems;
  uint32_t keep = 0u;  // bit k: row base + k is kept
#pragma unroll
  for (int k = 0; k < kSelItems; ++k) {
    const int64_t r = base + k;
    const bool on = r < n && (flags ? flags[r] != 0 : x[r] > thr);
    keep |= (on ? 1u : 0u) << k;
  }
  const uint32_t mine = __popc(keep);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  uint32_t woff = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kSelThreads / 32; ++w) {
    if (w < warp) woff += ws[w];
    tot += ws[w];
  }
  if (threadIdx.x == 0) {
    uint32_t excl = 0;
    if (tile == 0) {
      atomicExch(status, kSelInc | tot);
    } else {
      atomicExch(status + tile, kSelAgg | tot);
      for (int j = (int)tile - 1;; ) {
        const uint32_t sv = atomicAdd(status + j, 0u);
        if ((sv >> 30) == 0) continue;  // predecessor not published yet (it holds an earlier ticket)
        excl += sv & kSelMask;
        if (sv & kSelInc) break;
        --j;
      }
      atomicExch(status + tile, kSelInc | (excl + tot));
    }
    s_excl = excl;
    if ((int64_t)(tile + 1) * kSelTile >= n) *count = (int64_t)(excl + tot);  // the last tile
  }
  __syncthreads();
  int64_t out = (int64_t)s_excl + woff + inc - mine;
  while (keep) {
    const int k = __ffs(keep) - 1;
    keep &= keep - 1;
    idx[out++] = base + k;
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
                                    const float *band_weights, int64_t n_gaussians, const double *loss_terms,
                                    int32_t n_terms, int32_t *nonfinite_flag, const int64_t *range_begin,
                                    const int64_t *range_end, int32_t nranges, tgs_stream_t stream) {
  if (ngroups < 1 || ngroups > 8 || !param || !grad || !m || !v || !offsets || !sizes || !lrs || !bias_c1 ||
      !bias_c2 || !kinds || n_gaussians < 0 || n_terms < 0 || (n_terms > 0 && !loss_terms) || nranges < 0 ||
      nranges > 8 || (nranges > 0 && (!range_begin || !range_end)))
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
  a.terms = n_terms > 0 ? loss_terms : nullptr;
  a.nterms = n_terms;
  a.nonfinite = nonfinite_flag;
  // the ranges clipped to the groups' span; none given = the whole span
  a.nranges = 0;
  a.r4[0] = 0;
  for (int r = 0; r < (nranges > 0 ? nranges : 1); ++r) {
    int64_t lo = a.off[0], hi = a.off[ngroups];
    if (nranges > 0) {
      if ((range_begin[r] & 3) || (range_end[r] & 3)) return TGS_ERR_INVALID;
      lo = range_begin[r] > lo ? range_begin[r] : lo;
      hi = range_end[r] < hi ? range_end[r] : hi;
    }
    if (hi <= lo) continue;
    a.rb[a.nranges] = lo;
    a.r4[a.nranges + 1] = a.r4[a.nranges] + (hi - lo) / 4;
    ++a.nranges;
  }
  const int64_t n4 = a.r4[a.nranges];
  if (n4 <= 0 && !a.terms) return TGS_OK;  // (with a guard, one block still writes the flag)
  const unsigned grid = (unsigned)tmax<int64_t>(1, tmin<int64_t>(ceil_div<int64_t>(n4, 256), 148 * 8));
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

extern "C" int tgs_select_rows_workspace(int64_t n, size_t *bytes) {
  if (n < 0 || !bytes) return TGS_ERR_INVALID;
  *bytes = align_up(((size_t)ceil_div<int64_t>(n, kSelTile) + 1) * sizeof(uint32_t));
  return TGS_OK;
}

extern "C" int tgs_select_rows(const uint8_t *flags, const float *x, float threshold, int64_t n, int64_t *indices,
                               int64_t *count, void *workspace, size_t workspace_bytes, tgs_stream_t stream) {
  if (n < 0 || !count || (n > 0 && (!indices || (!flags && !x) || !workspace))) return TGS_ERR_INVALID;
  if (n >= (int64_t)1 << 30) return TGS_ERR_UNSUPPORTED;  // 30-bit look-back payloads
  cudaStream_t st = as_stream(stream);
  if (n == 0) return cuda_status(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
  size_t need = 0;
  tgs_select_rows_workspace(n, &need);
  if (workspace_bytes < need) return TGS_ERR_INVALID;
  const int64_t tiles = ceil_div<int64_t>(n, kSelTile);
  uint32_t *status = static_cast<uint32_t *>(workspace), *ticket = status + tiles;
  const int rc = cuda_status(cudaMemsetAsync(workspace, 0, (size_t)(tiles + 1) * sizeof(uint32_t), st));
  if (rc != TGS_OK) return rc;
  k_select_rows<<<(unsigned)tiles, kSelThreads, 0, st>>>(flags, x, threshold, n, indices, count, status, ticket);
  return launch_status();
}
