// loss.cu — (1 - lambda) * L1 + lambda * (1 - SSIM) / 2 with its exact gradient.
//
// Reference: training.total_loss image terms (training.py:76-89) and
// metrics.ssim_fast (metrics.py:120-188): an 11-tap sigma-1.5 Gaussian window
// applied separably to the symmetric-padded image, mean SSIM over pixels and
// channels, and the analytic gradient whose adjoint folds the padded border
// back onto its source pixels (metrics.py:126-135).
//
// One fused kernel: each CTA owns a 32x32 output tile and, per channel, keeps
// everything in shared memory —
//   inputs a, b on the tile + 10 px halo (52 x 52, symmetric reflection),
//   horizontal window sums of {a, b, a^2, b^2, ab} on 52 x 42,
//   vertical window -> SSIM partials dSSIM/d{mu_a, s_aa, s_ab} on 42 x 42
//     (tile + 5 px, image pixels only), SSIM and L1 sums on the 32 x 32 tile,
//   vertical adjoint on 32 x 42 and horizontal adjoint on 32 x 32, both with the
//     reflection fold, combined with sign(a - b) into dimage.
// HBM traffic is the algorithmic 36 B/pixel (read image + target, write dimage).
#include "tgs_common.cuh"

namespace tgs {

constexpr int kR = 5;          // window radius (11 taps)
constexpr int kT = 32;         // output tile edge
constexpr int kIn = kT + 4 * kR;   // 52: tile + forward + adjoint halo
constexpr int kMid = kT + 2 * kR;  // 42: positions whose SSIM partials the tile's adjoint reads
constexpr int kLossThreads = 256;

struct Taps {
  float w[2 * kR + 1];
};

__device__ __forceinline__ int reflect_clamp(int k, int n) {  // numpy 'symmetric' padding
  if (k < 0) k = -1 - k;
  if (k >= n) k = 2 * n - 1 - k;
  return k < 0 ? 0 : (k >= n ? n - 1 : k);  // only reached by windows of non-image positions
}

// adjoint (gather form) of "window over the symmetric-padded signal" at index y:
//   sum_i w_i (u[y-i+R] + [y < R] u[R-1-y-i+R] + [y >= n-R] u[2n-1-y-i+R]), valid indices only.
// `get(j)` reads u at image index j (caller guarantees j is inside its smem window).
template <typename F>
__device__ __forceinline__ float adjoint_at(int y, int n, const Taps &tp, F get) {
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < 2 * kR + 1; ++i) {
    const int y0 = y - i + kR;
    if (y0 >= 0 && y0 < n) s += tp.w[i] * get(y0);
  }
  if (y < kR || y >= n - kR) {
#pragma unroll
    for (int i = 0; i < 2 * kR + 1; ++i) {
      if (y < kR) {
        const int y1 = -1 - y - i + kR;
        if (y1 >= 0 && y1 < n) s += tp.w[i] * get(y1);
      }
      if (y >= n - kR) {
        const int y2 = 2 * n - 1 - y - i + kR;
        if (y2 >= 0 && y2 < n) s += tp.w[i] * get(y2);
      }
    }
  }
  return s;
}

__global__ void __launch_bounds__(kLossThreads) k_loss_fused(const float *__restrict__ img,
                                                             const float *__restrict__ tgt, int W, int H, Taps tp,
                                                             float c1, float c2, float lam, float inv_count,
                                                             float *__restrict__ dimage, double *__restrict__ sums) {
  extern __shared__ float4 smem4[];
  float *sm = reinterpret_cast<float *>(smem4);
  float *sa = sm;                        // [kIn][kIn]
  float *sb = sa + kIn * kIn;            // [kIn][kIn]
  float *hs = sb + kIn * kIn;            // [kIn][kMid][5]; reused as se [kT][kMid][3]
  float *sd = hs + kIn * kMid * 5;       // [kMid][kMid][3]
  float *se = hs;
  __shared__ double red[2][kLossThreads / 32];
  const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
  const int gx = x0 - 2 * kR, gy = y0 - 2 * kR;  // image coords of sa[0][0]
  const int mx = x0 - kR, my = y0 - kR;          // image coords of the kMid region origin
  const int t = threadIdx.x;
  double l1 = 0.0, ss = 0.0;
  for (int c = 0; c < 3; ++c) {
    for (int e = t; e < kIn * kIn; e += kLossThreads) {
      const int r = e / kIn, q = e - r * kIn;
      const size_t p = ((size_t)reflect_clamp(gy + r, H) * W + reflect_clamp(gx + q, W)) * 3 + c;
      sa[e] = img[p];
      sb[e] = tgt[p];
    }
    __syncthreads();
    // horizontal window sums on rows [0, kIn) x mid columns [0, kMid)
    for (int e = t; e < kIn * kMid; e += kLossThreads) {
      const int r = e / kMid, q = e - r * kMid;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f;
#pragma unroll
      for (int j = 0; j < 2 * kR + 1; ++j) {
        const float av = sa[r * kIn + q + j], bv = sb[r * kIn + q + j], w = tp.w[j];
        s0 += w * av;
        s1 += w * bv;
        s2 += w * av * av;
        s3 += w * bv * bv;
        s4 += w * av * bv;
      }
      float *o = hs + e * 5;
      o[0] = s0; o[1] = s1; o[2] = s2; o[3] = s3; o[4] = s4;
    }
    __syncthreads();
    // vertical window -> SSIM partials on the mid region (image pixels only)
    for (int e = t; e < kMid * kMid; e += kLossThreads) {
      const int r = e / kMid, q = e - r * kMid;
      const int yy = my + r, xx = mx + q;
      float *o = sd + e * 3;
      if (yy < 0 || yy >= H || xx < 0 || xx >= W) {
        o[0] = o[1] = o[2] = 0.0f;
        continue;
      }
      float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
      for (int i = 0; i < 2 * kR + 1; ++i) {
        const float *h = hs + ((r + i) * kMid + q) * 5;
        const float w = tp.w[i];
        m0 += w * h[0];
        m1 += w * h[1];
        m2 += w * h[2];
        m3 += w * h[3];
        m4 += w * h[4];
      }
      const float var_a = m2 - m0 * m0, var_b = m3 - m1 * m1, cov = m4 - m0 * m1;
      const float A1 = 2.0f * m0 * m1 + c1, A2 = 2.0f * cov + c2;
      const float B1 = m0 * m0 + m1 * m1 + c1, B2 = var_a + var_b + c2;
      const float den = B1 * B2;
      const float smap = A1 * A2 / den;
      o[0] = 2.0f * m1 * (A2 - A1) / den - 2.0f * m0 * smap * (1.0f / B1 - 1.0f / B2);
      o[1] = -smap / B2;
      o[2] = 2.0f * A1 / den;
      if (r >= kR && r < kR + kT && q >= kR && q < kR + kT) {  // this tile's own pixels
        ss += smap;
        const float av = sa[(r + kR) * kIn + q + kR], bv = sb[(r + kR) * kIn + q + kR];
        l1 += fabsf(av - bv);
      }
    }
    __syncthreads();
    // vertical adjoint: rows of the tile x mid columns
    for (int e = t; e < kT * kMid; e += kLossThreads) {
      const int r = e / kMid, q = e - r * kMid;
      const int yy = y0 + r, xx = mx + q;
      float *o = se + e * 3;
      if (yy >= H || xx < 0 || xx >= W) {
        o[0] = o[1] = o[2] = 0.0f;
        continue;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k)
        o[k] = adjoint_at(yy, H, tp, [&](int j) { return sd[((j - my) * kMid + q) * 3 + k]; });
    }
    __syncthreads();
    // horizontal adjoint on the tile, combine with the L1 sign
    for (int e = t; e < kT * kT; e += kLossThreads) {
      const int r = e / kT, q = e - r * kT;
      const int yy = y0 + r, xx = x0 + q;
      if (yy >= H || xx >= W) continue;
      float g[3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        g[k] = adjoint_at(xx, W, tp, [&](int j) { return se[(r * kMid + (j - mx)) * 3 + k]; });
      const float av = sa[(r + 2 * kR) * kIn + q + 2 * kR], bv = sb[(r + 2 * kR) * kIn + q + 2 * kR];
      const float grad = (g[0] + 2.0f * av * g[1] + bv * g[2]) * inv_count;
      const float diff = av - bv;
      const float sgn = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
      dimage[((size_t)yy * W + xx) * 3 + c] = (1.0f - lam) * sgn * inv_count - lam * 0.5f * grad;
    }
    __syncthreads();
  }
  // block reduction -> one double atomic pair per CTA
  const int lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if (lane == 0) {
    red[0][warp] = l1;
    red[1][warp] = ss;
  }
  __syncthreads();
  if (t == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    atomicAdd(sums, a);
    atomicAdd(sums + 1, b);
  }
}

__global__ void k_loss_finalize(double *terms, double inv_count) {
  terms[0] *= inv_count;  // mean |a - b|
  terms[1] *= inv_count;  // mean SSIM over pixels and channels
}

constexpr size_t kLossSmem = (size_t)(2 * kIn * kIn + kIn * kMid * 5 + kMid * kMid * 3) * sizeof(float);

}  // namespace tgs

using namespace tgs;

extern "C" int tgs_loss_workspace(int32_t width, int32_t height, size_t *bytes) {
  if (width < 1 || height < 1 || !bytes) return TGS_ERR_INVALID;
  *bytes = 0;  // the fused kernel keeps every intermediate in shared memory
  return TGS_OK;
}

extern "C" int tgs_loss_l1_ssim(const float *image, const float *target, int32_t width, int32_t height,
                                float lambda_ssim, float *dimage, double *terms, void *workspace,
                                tgs_stream_t stream) {
  (void)workspace;
  if (width < 2 * kR + 1 || height < 2 * kR + 1) return TGS_ERR_INVALID;  // metrics.py:83-84
  if (!image || !target || !dimage || !terms) return TGS_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  static bool attr_done = false;  // idempotent function attribute, set once per process
  if (!attr_done) {
    if (cudaFuncSetAttribute(k_loss_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLossSmem) !=
        cudaSuccess)
      return launch_status();
    attr_done = true;
  }
  Taps tp;
  double w[2 * kR + 1], tot = 0.0;  // gaussian_taps (metrics.py:58-61), float64 then rounded
  for (int i = 0; i < 2 * kR + 1; ++i) {
    const double xx = (double)(i - kR) / 1.5;
    w[i] = exp(-0.5 * xx * xx);
    tot += w[i];
  }
  for (int i = 0; i < 2 * kR + 1; ++i) tp.w[i] = (float)(w[i] / tot);
  const size_t count = (size_t)width * height * 3;
  cudaMemsetAsync(terms, 0, 2 * sizeof(double), st);
  const dim3 grd((unsigned)ceil_div(width, kT), (unsigned)ceil_div(height, kT));
  k_loss_fused<<<grd, kLossThreads, kLossSmem, st>>>(image, target, width, height, tp, 0.01f * 0.01f, 0.03f * 0.03f,
                                                     lambda_ssim, 1.0f / (float)count, dimage, terms);
  k_loss_finalize<<<1, 1, 0, st>>>(terms, 1.0 / (double)count);
  return launch_status();
}
