// loss.cu — (1 - lambda) * L1 + lambda * (1 - SSIM) / 2 with its exact gradient.
//
// Reference: training.total_loss image terms (training.py:76-89) and
// metrics.ssim_fast (metrics.py:120-188): an 11-tap sigma-1.5 Gaussian window
// applied separably to the symmetric-padded image, mean SSIM over pixels and
// channels, and the analytic gradient whose adjoint folds the padded border
// back onto its source pixels (metrics.py:126-135).
//
// Four streaming passes, one thread per pixel, all three channels per thread:
//   h   : horizontal window of {a, b, a^2, b^2, ab}           -> 15 planes
//   v   : vertical window -> SSIM map, dSSIM/d{mu_a, s_aa, s_ab}, L1 and SSIM
//         sums (block reduction, one double atomic per block) -> 9 planes
//   av  : vertical adjoint of the window (with the symmetric fold)
//   ah  : horizontal adjoint + combine with sign(a - b) -> dimage
// Taps are computed on the host in float64 exactly like gaussian_taps
// (metrics.py:58-61) and passed rounded to float32.
#include "tgs_common.cuh"

namespace tgs {

constexpr int kR = 5;  // window 11
struct Taps {
  float w[2 * kR + 1];
};

__device__ __forceinline__ int reflect(int k, int n) {  // numpy 'symmetric' padding
  if (k < 0) k = -1 - k;
  if (k >= n) k = 2 * n - 1 - k;
  return k;
}

__global__ void k_ssim_h(const float *__restrict__ a, const float *__restrict__ b, int W, int H, Taps tp,
                         float *__restrict__ h) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= W) return;
  const size_t plane = (size_t)W * H, p = (size_t)y * W + x;
  float s[3][5] = {};
#pragma unroll
  for (int j = 0; j < 2 * kR + 1; ++j) {
    const size_t q = ((size_t)y * W + reflect(x + j - kR, W)) * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float av = a[q + c], bv = b[q + c], w = tp.w[j];
      s[c][0] += w * av;
      s[c][1] += w * bv;
      s[c][2] += w * av * av;
      s[c][3] += w * bv * bv;
      s[c][4] += w * av * bv;
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int k = 0; k < 5; ++k) h[(c * 5 + k) * plane + p] = s[c][k];
}

__global__ void k_ssim_v(const float *__restrict__ a, const float *__restrict__ b, const float *__restrict__ h,
                         int W, int H, Taps tp, float c1, float c2, float *__restrict__ d,
                         double *__restrict__ sums) {
  __shared__ double red[2][32];
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  const size_t plane = (size_t)W * H, p = (size_t)y * W + x;
  double l1 = 0.0, ss = 0.0;
  if (x < W) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float m[5] = {};
#pragma unroll
      for (int i = 0; i < 2 * kR + 1; ++i) {
        const size_t q = (size_t)reflect(y + i - kR, H) * W + x;
#pragma unroll
        for (int k = 0; k < 5; ++k) m[k] += tp.w[i] * h[(c * 5 + k) * plane + q];
      }
      const float mu_a = m[0], mu_b = m[1];
      const float var_a = m[2] - mu_a * mu_a, var_b = m[3] - mu_b * mu_b, cov = m[4] - mu_a * mu_b;
      const float A1 = 2.0f * mu_a * mu_b + c1, A2 = 2.0f * cov + c2;
      const float B1 = mu_a * mu_a + mu_b * mu_b + c1, B2 = var_a + var_b + c2;
      const float den = B1 * B2;
      const float smap = A1 * A2 / den;
      d[(c * 3 + 0) * plane + p] = 2.0f * mu_b * (A2 - A1) / den - 2.0f * mu_a * smap * (1.0f / B1 - 1.0f / B2);
      d[(c * 3 + 1) * plane + p] = -smap / B2;
      d[(c * 3 + 2) * plane + p] = 2.0f * A1 / den;
      ss += smap;
      l1 += fabsf(a[p * 3 + c] - b[p * 3 + c]);
    }
  }
  // block reduction -> one double atomic pair per block
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      t0 += red[0][w];
      t1 += red[1][w];
    }
    atomicAdd(sums, t0);
    atomicAdd(sums + 1, t1);
  }
}

// adj[y] = sum_i w_i (u[y - i + R] + [y <= R-1] u[R-1-y-i+R] + [y >= n-R] u[2n-1-y-i+R])   (valid indices only)
__device__ __forceinline__ float adj1(const float *u, size_t stride, int y, int n, const Taps &tp) {
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < 2 * kR + 1; ++i) {
    const int y0 = y - i + kR;
    if (y0 >= 0 && y0 < n) s += tp.w[i] * u[(size_t)y0 * stride];
    if (y <= kR - 1) {
      const int y1 = -1 - y - i + kR;
      if (y1 >= 0 && y1 < n) s += tp.w[i] * u[(size_t)y1 * stride];
    }
    if (y >= n - kR) {
      const int y2 = 2 * n - 1 - y - i + kR;
      if (y2 >= 0 && y2 < n) s += tp.w[i] * u[(size_t)y2 * stride];
    }
  }
  return s;
}

__global__ void k_ssim_adj_v(const float *__restrict__ d, int W, int H, Taps tp, float *__restrict__ e) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= W) return;
  const size_t plane = (size_t)W * H, p = (size_t)y * W + x;
#pragma unroll
  for (int k = 0; k < 9; ++k) e[k * plane + p] = adj1(d + k * plane + x, (size_t)W, y, H, tp);
}

__global__ void k_ssim_adj_h(const float *__restrict__ a, const float *__restrict__ b,
                             const float *__restrict__ e, int W, int H, Taps tp, float lam, float inv_count,
                             float *__restrict__ dimage) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= W) return;
  const size_t plane = (size_t)W * H, p = (size_t)y * W + x;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float *row = e + (size_t)y * W;
    const float gmu = adj1(row + (c * 3 + 0) * plane, 1, x, W, tp);
    const float gaa = adj1(row + (c * 3 + 1) * plane, 1, x, W, tp);
    const float gab = adj1(row + (c * 3 + 2) * plane, 1, x, W, tp);
    const float av = a[p * 3 + c], bv = b[p * 3 + c];
    const float grad = (gmu + 2.0f * av * gaa + bv * gab) * inv_count;
    const float diff = av - bv;
    const float sgn = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
    dimage[p * 3 + c] = (1.0f - lam) * sgn * inv_count - lam * 0.5f * grad;
  }
}

__global__ void k_loss_finalize(double *terms, double inv_count) {
  terms[0] *= inv_count;  // mean |a - b|
  terms[1] *= inv_count;  // mean SSIM over pixels and channels
}

}  // namespace tgs

using namespace tgs;

extern "C" int tgs_loss_workspace(int32_t width, int32_t height, size_t *bytes) {
  if (width < 1 || height < 1 || !bytes) return TGS_ERR_INVALID;
  *bytes = align_up((size_t)width * height * (15 + 9 + 9) * sizeof(float));
  return TGS_OK;
}

extern "C" int tgs_loss_l1_ssim(const float *image, const float *target, int32_t width, int32_t height,
                                float lambda_ssim, float *dimage, double *terms, void *workspace,
                                tgs_stream_t stream) {
  if (width < 2 * kR + 1 || height < 2 * kR + 1) return TGS_ERR_INVALID;  // metrics.py:83-84
  if (!image || !target || !dimage || !terms || !workspace) return TGS_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  Taps tp;
  double w[2 * kR + 1], tot = 0.0;
  for (int i = 0; i < 2 * kR + 1; ++i) {
    const double xx = (double)(i - kR) / 1.5;
    w[i] = exp(-0.5 * xx * xx);
    tot += w[i];
  }
  for (int i = 0; i < 2 * kR + 1; ++i) tp.w[i] = (float)(w[i] / tot);
  const size_t plane = (size_t)width * height;
  float *h = static_cast<float *>(workspace);
  float *d = h + 15 * plane;
  float *e = d + 9 * plane;
  const dim3 blk(128), grd((unsigned)ceil_div(width, 128), (unsigned)height);
  cudaMemsetAsync(terms, 0, 2 * sizeof(double), st);
  k_ssim_h<<<grd, blk, 0, st>>>(image, target, width, height, tp, h);
  k_ssim_v<<<grd, blk, 0, st>>>(image, target, h, width, height, tp, 0.01f * 0.01f, 0.03f * 0.03f, d, terms);
  k_ssim_adj_v<<<grd, blk, 0, st>>>(d, width, height, tp, e);
  const float inv_count = 1.0f / (float)(plane * 3);
  k_ssim_adj_h<<<grd, blk, 0, st>>>(image, target, e, width, height, tp, lambda_ssim, inv_count, dimage);
  k_loss_finalize<<<1, 1, 0, st>>>(terms, 1.0 / (double)(plane * 3));
  return launch_status();
}
