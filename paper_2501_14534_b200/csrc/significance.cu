// significance.cu — significance scoring and pruning selection (significance.py:45-99).
//
//   score_i = hits_i * alpha_hat_i * min(V_i / V90, 1) ** power       (V90 > 0)
//           = hits_i * alpha_hat_i * [V_i > 0]                         (V90 == 0)
//   V_i     = 4/3 pi prod(e^ls_i M_i),  alpha_hat_i = sigmoid(o_i) M_i,
//   V90     = the nearest-rank 90th percentile of V (sorted(V)[rank]).
//
// V90 and the pruning threshold are order statistics; both come from one device
// radix select over 64-bit keys (value bits << 32 | row index), 8 bits per pass:
// a histogram pass restricted to the keys that match the digits chosen so far,
// then a one-block pick of the next digit.  The selected key stays in device
// memory, so scoring -> selection -> keep flags run without a host round trip.
// The index in the low half makes the keys unique, which is exactly the
// reference's tie break: np.lexsort((arange, scores)) prunes equal scores from
// the lower index first (significance.py:97-98).
#include "preprocess_common.cuh"

namespace tgs {

constexpr int kSelThreads = 256;

struct SelCtl {
  unsigned long long prefix;  // digits chosen so far
  unsigned long long k;       // rank still to find among the keys matching prefix
  uint32_t hist[256];
};

__global__ void __launch_bounds__(kSelThreads) k_sel_init(SelCtl *ctl, int64_t k) {
  if (threadIdx.x == 0) {
    ctl->prefix = 0ull;
    ctl->k = (unsigned long long)k;
  }
  ctl->hist[threadIdx.x] = 0u;
}

// histogram of digit (key >> shift) & 255 over the keys whose higher digits equal prefix
__global__ void __launch_bounds__(kSelThreads) k_sel_hist(const unsigned long long *__restrict__ keys, int64_t n,
                                                          SelCtl *ctl, int shift) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0u;
  __syncthreads();
  const unsigned long long pre = ctl->prefix;
  const int hs = shift + 8;  // bits above this digit
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = __ldg(keys + i);
    if (hs >= 64 || (key >> hs) == (pre >> hs)) atomicAdd(&h[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&ctl->hist[threadIdx.x], h[threadIdx.x]);
}

// the digit whose cumulative count passes k; k becomes the rank inside it
__global__ void __launch_bounds__(kSelThreads) k_sel_pick(SelCtl *ctl, int shift) {
  __shared__ uint32_t s[256];
  const int t = threadIdx.x;
  const uint32_t c = ctl->hist[t];
  s[t] = c;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {  // inclusive scan
    const uint32_t v = t >= o ? s[t - o] : 0u;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  const unsigned long long k = ctl->k;
  const uint32_t incl = s[t], excl = incl - c;
  __syncthreads();
  if (c && excl <= k && k < incl) {
    ctl->prefix |= (unsigned long long)t << shift;
    ctl->k = k - excl;
  }
  ctl->hist[t] = 0u;
}

// k-th smallest (0-based) of n keys; the result is ctl->prefix after the passes
// over the digits [lo_shift, 64)
inline int select_kth(const unsigned long long *keys, int64_t n, int64_t k, SelCtl *ctl, int lo_shift,
                      cudaStream_t st) {
  const unsigned grid = (unsigned)tmin<int64_t>(ceil_div<int64_t>(n, kSelThreads), 148 * 4);
  k_sel_init<<<1, kSelThreads, 0, st>>>(ctl, k);
  for (int shift = 56; shift >= lo_shift; shift -= 8) {
    k_sel_hist<<<grid, kSelThreads, 0, st>>>(keys, n, ctl, shift);
    k_sel_pick<<<1, kSelThreads, 0, st>>>(ctl, shift);
  }
  return launch_status();
}

constexpr float kFourThirdsPi = 4.18879020478639098f;  // (4/3) pi (significance.py:63)

// volumes and their selection keys (value bits << 32 | row): V >= 0, so the
// float bits order like the values
__global__ void k_sig_volume(tgs_cloud cl, float mask_logit_min, float *__restrict__ volumes,
                             unsigned long long *__restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cl.n) return;
  const float M = cl.mask_logits[i] > mask_logit_min ? 1.0f : 0.0f;  // masking.py:21-25
  const float s0 = sem_expf(cl.log_scales[3 * i]) * M, s1 = sem_expf(cl.log_scales[3 * i + 1]) * M,
              s2 = sem_expf(cl.log_scales[3 * i + 2]) * M;
  const float v = kFourThirdsPi * ((s0 * s1) * s2);
  volumes[i] = v;
  keys[i] = ((unsigned long long)__float_as_uint(v) << 32) | (unsigned long long)(uint32_t)i;
}

__device__ __forceinline__ uint32_t orderable(float f) {  // monotone float -> uint
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// scores with V90 = the selected key's high half; keys for the pruning selection
__global__ void k_sig_score(tgs_cloud cl, const int64_t *__restrict__ hits, float mask_logit_min, float power,
                            const SelCtl *__restrict__ v90ctl, const float *__restrict__ volumes,
                            float *__restrict__ v_norm, float *__restrict__ scores) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cl.n) return;
  const float v90 = __uint_as_float((uint32_t)(v90ctl->prefix >> 32));
  const float v = volumes[i];
  float vn;
  if (v90 > 0.0f) {
    const float r = fminf(v / v90, 1.0f);
    vn = power == 0.5f ? sqrtf(r) : powf(r, power);
  } else {
    vn = v > 0.0f ? 1.0f : 0.0f;
  }
  const float M = cl.mask_logits[i] > mask_logit_min ? 1.0f : 0.0f;
  const float alpha = sem_sigmoidf(cl.opacity_logits[i]) * M;  // masking.py:34-43
  v_norm[i] = vn;
  scores[i] = ((float)hits[i] * alpha) * vn;
}

__global__ void k_score_keys(const float *__restrict__ scores, int64_t n, unsigned long long *__restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = ((unsigned long long)orderable(scores[i]) << 32) | (unsigned long long)(uint32_t)i;
}

// rows at or above the k-th smallest (score, row) survive
__global__ void k_keep_flags(const unsigned long long *__restrict__ keys, int64_t n, const SelCtl *__restrict__ ctl,
                             uint8_t *__restrict__ keep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keep[i] = keys[i] >= ctl->prefix ? 1 : 0;
}

inline void carve_sig(void *ws, int64_t n, unsigned long long *&keys, SelCtl *&ctl, size_t &bytes) {
  Carve c(ws);
  keys = c.take<unsigned long long>((size_t)tmax<int64_t>(n, 1));
  ctl = c.take<SelCtl>(1);
  bytes = c.off;
}

}  // namespace tgs

using namespace tgs;

extern "C" int tgs_significance_workspace(int64_t n, size_t *bytes) {
  if (!bytes || n < 0) return TGS_ERR_INVALID;
  unsigned long long *keys;
  SelCtl *ctl;
  carve_sig(nullptr, n, keys, ctl, *bytes);
  return TGS_OK;
}

extern "C" int tgs_significance_scores(const tgs_cloud *cloud, const int64_t *hits, float mask_logit_min,
                                       float volume_power, int64_t rank90, float *volumes, float *v_norm,
                                       float *scores, void *workspace, size_t workspace_bytes,
                                       tgs_stream_t stream) {
  if (!cloud || cloud->n < 0) return TGS_ERR_INVALID;
  const int64_t n = cloud->n;
  if (n == 0) return TGS_OK;
  if (n >= (int64_t)1 << 32 || rank90 < 0 || rank90 >= n || !hits || !volumes || !v_norm || !scores)
    return TGS_ERR_INVALID;
  unsigned long long *keys;
  SelCtl *ctl;
  size_t need;
  carve_sig(workspace, n, keys, ctl, need);
  if (!workspace || workspace_bytes < need) return TGS_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  const unsigned g = (unsigned)ceil_div<int64_t>(n, 256);
  k_sig_volume<<<g, 256, 0, st>>>(*cloud, mask_logit_min, volumes, keys);
  // only the value half of the key decides V90: the passes over the index bits are skipped
  int rc = select_kth(keys, n, rank90, ctl, 32, st);
  if (rc != TGS_OK) return rc;
  k_sig_score<<<g, 256, 0, st>>>(*cloud, hits, mask_logit_min, volume_power, ctl, volumes, v_norm, scores);
  return launch_status();
}

extern "C" int tgs_significance_keep(const float *scores, int64_t n, int64_t k, uint8_t *keep, void *workspace,
                                     size_t workspace_bytes, tgs_stream_t stream) {
  if (n < 0 || k < 0 || (n > 0 && k >= n) || n >= (int64_t)1 << 32) return TGS_ERR_INVALID;
  if (n == 0) return TGS_OK;
  if (!scores || !keep) return TGS_ERR_INVALID;
  unsigned long long *keys;
  SelCtl *ctl;
  size_t need;
  carve_sig(workspace, n, keys, ctl, need);
  if (!workspace || workspace_bytes < need) return TGS_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  const unsigned g = (unsigned)ceil_div<int64_t>(n, 256);
  k_score_keys<<<g, 256, 0, st>>>(scores, n, keys);
  int rc = select_kth(keys, n, k, ctl, 0, st);
  if (rc != TGS_OK) return rc;
  k_keep_flags<<<g, 256, 0, st>>>(keys, n, ctl, keep);
  return launch_status();
}
