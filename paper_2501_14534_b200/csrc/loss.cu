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

// Reflection-fold terms of the adjoint at image index y (only near the borders):
// sum_i w_i (u[R-1-y-i+R] for y < R) + (u[2n-1-y-i+R] for y >= n-R), valid indices.
template <typename F>
__device__ __forceinline__ float adjoint_fold(int y, int n, const Taps &tp, F get) {
  float s = 0.0f;
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
  return s;
}

// Work items per phase are sized so each phase fills the 256 threads between
// barriers: H 52x14 = 728 items (3 outputs), V 42x6 = 252 (7 outputs),
// vertical adjoint 42x6 = 252 (6 row segments of 5-6 outputs), horizontal
// adjoint 32x8 = 256 (4 outputs).
constexpr int kHSeg = 3;
constexpr int kVSeg = 7;
constexpr int kAVSeg = 6;   // max rows per vertical-adjoint item
constexpr int kAVItems = 6; // row segments per column: 32 = 6+5+5+5+5+6
constexpr int kAHSeg = 4;

__global__ void __launch_bounds__(kLossThreads) k_loss_fused(const float *__restrict__ img,
                                                             const float *__restrict__ tgt, int W, int H, Taps tp,
                                                             float c1, float c2, float lam, float inv_count,
                                                             float *__restrict__ dimage, double *__restrict__ sums) {
  extern __shared__ float4 smem4[];
  float *sm = reinterpret_cast<float *>(smem4);
  float *sa = sm;                         // [kIn][kIn]
  float *sb = sa + kIn * kIn;             // [kIn][kIn]
  float *hs = sb + kIn * kIn;             // [5][kIn][kMid] (planar)
  float *sd = hs + 5 * kIn * kMid;        // [3][kMid][kMid] (planar, zero outside the image)
  float *se = hs;                         // [3][kT][kMid] (reuses hs)
  __shared__ double red[2][kLossThreads / 32];
  const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
  const int gx = x0 - 2 * kR, gy = y0 - 2 * kR;  // image coords of sa[0][0]
  const int mx = x0 - kR, my = y0 - kR;          // image coords of the kMid region origin
  const int t = threadIdx.x;
  const bool border = x0 < kR || y0 < kR || x0 + kT > W - kR || y0 + kT > H - kR;
  double l1 = 0.0, ss = 0.0;
  for (int c = 0; c < 3; ++c) {
    for (int e = t; e < kIn * kIn; e += kLossThreads) {
      const int r = e / kIn, q = e - r * kIn;
      const size_t p = ((size_t)reflect_clamp(gy + r, H) * W + reflect_clamp(gx + q, W)) * 3 + c;
      sa[e] = img[p];
      sb[e] = tgt[p];
    }
    __syncthreads();
    // ---- horizontal window sums: item = (row, 6 mid columns), sliding window in registers
    for (int it = t; it < kIn * (kMid / kHSeg); it += kLossThreads) {
      const int r = it / (kMid / kHSeg), q0 = (it - r * (kMid / kHSeg)) * kHSeg;
      float av[kHSeg + 2 * kR], bv[kHSeg + 2 * kR];
#pragma unroll
      for (int j = 0; j < kHSeg + 2 * kR; ++j) {
        av[j] = sa[r * kIn + q0 + j];
        bv[j] = sb[r * kIn + q0 + j];
      }
#pragma unroll
      for (int o = 0; o < kHSeg; ++o) {
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f;
#pragma unroll
        for (int j = 0; j < 2 * kR + 1; ++j) {
          const float w = tp.w[j], x = av[o + j], y = bv[o + j];
          const float wx = w * x, wy = w * y;
          s0 += wx;
          s1 += wy;
          s2 = fmaf(wx, x, s2);
          s3 = fmaf(wy, y, s3);
          s4 = fmaf(wx, y, s4);
        }
        const int off = r * kMid + q0 + o;
        hs[off] = s0;
        hs[kIn * kMid + off] = s1;
        hs[2 * kIn * kMid + off] = s2;
        hs[3 * kIn * kMid + off] = s3;
        hs[4 * kIn * kMid + off] = s4;
      }
    }
    __syncthreads();
    // ---- vertical window -> SSIM partials: item = (mid column, 6 mid rows)
    for (int it = t; it < kMid * (kMid / kVSeg); it += kLossThreads) {
      const int q = it % kMid, r0 = (it / kMid) * kVSeg;
      float m[5][kVSeg];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        float col[kVSeg + 2 * kR];
#pragma unroll
        for (int j = 0; j < kVSeg + 2 * kR; ++j) col[j] = hs[k * kIn * kMid + (r0 + j) * kMid + q];
#pragma unroll
        for (int o = 0; o < kVSeg; ++o) {
          float acc = 0.f;
#pragma unroll
          for (int i = 0; i < 2 * kR + 1; ++i) acc = fmaf(tp.w[i], col[o + i], acc);
          m[k][o] = acc;
        }
      }
#pragma unroll
      for (int o = 0; o < kVSeg; ++o) {
        const int r = r0 + o;
        const int yy = my + r, xx = mx + q;
        const int off = r * kMid + q;
        if (yy < 0 || yy >= H || xx < 0 || xx >= W) {
          sd[off] = 0.f;
          sd[kMid * kMid + off] = 0.f;
          sd[2 * kMid * kMid + off] = 0.f;
          continue;
        }
        const float m0 = m[0][o], m1 = m[1][o];
        const float var_a = m[2][o] - m0 * m0, var_b = m[3][o] - m1 * m1, cov = m[4][o] - m0 * m1;
        const float A1 = 2.0f * m0 * m1 + c1, A2 = 2.0f * cov + c2;
        const float B1 = m0 * m0 + m1 * m1 + c1, B2 = var_a + var_b + c2;
        const float den = B1 * B2;
        const float smap = A1 * A2 / den;
        sd[off] = 2.0f * m1 * (A2 - A1) / den - 2.0f * m0 * smap * (1.0f / B1 - 1.0f / B2);
        sd[kMid * kMid + off] = -smap / B2;
        sd[2 * kMid * kMid + off] = 2.0f * A1 / den;
        if (r >= kR && r < kR + kT && q >= kR && q < kR + kT) {  // this tile's own pixels
          ss += smap;
          l1 += fabsf(sa[(r + kR) * kIn + q + kR] - sb[(r + kR) * kIn + q + kR]);
        }
      }
    }
    __syncthreads();
    // ---- vertical adjoint: item = (mid column, row segment of 5-6); symmetric taps -> correlation
    for (int it = t; it < kMid * kAVItems; it += kLossThreads) {
      const int q = it % kMid, sgi = it / kMid;
      const int r0 = sgi == 0 ? 0 : 1 + 5 * sgi;       // 0, 6, 11, 16, 21, 26
      const int len = (sgi == 0 || sgi == kAVItems - 1) ? 6 : 5;
      const int xx = mx + q;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float col[kAVSeg + 2 * kR];
#pragma unroll
        for (int j = 0; j < kAVSeg + 2 * kR; ++j) col[j] = (j < len + 2 * kR) ? sd[k * kMid * kMid + (r0 + j) * kMid + q] : 0.0f;
#pragma unroll
        for (int o = 0; o < kAVSeg; ++o) {
          if (o >= len) break;
          float acc = 0.f;
#pragma unroll
          for (int i = 0; i < 2 * kR + 1; ++i) acc = fmaf(tp.w[i], col[o + i], acc);
          const int yy = y0 + r0 + o;
          if (border && (yy < kR || yy >= H - kR) && xx >= 0 && xx < W)
            acc += adjoint_fold(yy, H, tp, [&](int j) { return sd[k * kMid * kMid + (j - my) * kMid + q]; });
          se[k * kT * kMid + (r0 + o) * kMid + q] = (yy < H && xx >= 0 && xx < W) ? acc : 0.0f;
        }
      }
    }
    __syncthreads();
    // ---- horizontal adjoint: item = (tile row, 4 columns); combine with the L1 sign
    for (int it = t; it < kT * (kT / kAHSeg); it += kLossThreads) {
      const int r = it / (kT / kAHSeg), c0 = (it - r * (kT / kAHSeg)) * kAHSeg;
      const int yy = y0 + r;
      float g[3][kAHSeg];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float row[kAHSeg + 2 * kR];
#pragma unroll
        for (int j = 0; j < kAHSeg + 2 * kR; ++j) row[j] = se[k * kT * kMid + r * kMid + c0 + j];
#pragma unroll
        for (int o = 0; o < kAHSeg; ++o) {
          float acc = 0.f;
#pragma unroll
          for (int i = 0; i < 2 * kR + 1; ++i) acc = fmaf(tp.w[i], row[o + i], acc);
          const int xx = x0 + c0 + o;
          if (border && (xx < kR || xx >= W - kR))
            acc += adjoint_fold(xx, W, tp, [&](int j) { return se[k * kT * kMid + r * kMid + (j - mx)]; });
          g[k][o] = acc;
        }
      }
      if (yy >= H) continue;
#pragma unroll
      for (int o = 0; o < kAHSeg; ++o) {
        const int xx = x0 + c0 + o;
        if (xx >= W) continue;
        const float av = sa[(r + 2 * kR) * kIn + c0 + o + 2 * kR], bv = sb[(r + 2 * kR) * kIn + c0 + o + 2 * kR];
        const float grad = (g[0][o] + 2.0f * av * g[1][o] + bv * g[2][o]) * inv_count;
        const float diff = av - bv;
        const float sgn = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
        dimage[((size_t)yy * W + xx) * 3 + c] = (1.0f - lam) * sgn * inv_count - lam * 0.5f * grad;
      }
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

constexpr size_t kLossSmem = (size_t)(2 * kIn * kIn + 5 * kIn * kMid + 3 * kMid * kMid) * sizeof(float);

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
