// loss.cu — (1 - lambda) * L1 + lambda * (1 - SSIM) / 2 with its exact gradient.
//
// Reference: training.total_loss image terms (training.py:76-89) and
// metrics.ssim_fast (metrics.py:120-188): an 11-tap sigma-1.5 Gaussian window
// applied separably to the symmetric-padded image, mean SSIM over pixels and
// channels, and the analytic gradient whose adjoint folds the padded border
// back onto its source pixels (metrics.py:126-135).
//
// Two kernels, one CTA per (32 x 32 tile, channel):
//   k_ssim_fwd  inputs a, b on the tile + 5 px halo (42 x 42, symmetric
//               reflection) -> horizontal window sums of {a, b, a^2, b^2, ab}
//               (42 x 32) -> vertical window -> per-pixel SSIM and the partials
//               d0 = dS/dmu_a, d1 = dS/ds_aa, d2 = dS/ds_ab, written to the
//               workspace; per-CTA L1 and SSIM partial sums.
//   k_ssim_adj  partials on the tile + 5 px halo (zero outside the image) ->
//               vertical adjoint (32 x 42) -> horizontal adjoint (32 x 32), both
//               with the reflection fold on border tiles, combined with
//               sign(a - b) into dimage:
//               dL/da = (1-lam) sign(a-b)/N - lam/2 (G'd0 + 2a G'd1 + b G'd2)/N.
// Splitting at the partials removes the fused kernel's second 10 px halo (the
// forward maps no longer have to cover the adjoint's footprint) and keeps each
// CTA's shared memory under 44 KB: the forward runs four CTAs per SM (shared-memory
// carveout 80%, the rest L1), the adjoint four (launch bound: 64 registers).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "tgs_common.cuh"

namespace tgs {

constexpr int kR = 5;              // window radius (11 taps)
constexpr int kT = 32;             // output tile edge
constexpr int kH = kT + 2 * kR;    // 42: tile + halo
constexpr int kHS = 45;            // shared row stride of halo-wide rows (== 1 mod 4: a warp's 4 rows
                                   // x 8 column groups fall on distinct banks)
constexpr int kLossThreads = 256;
constexpr int kHOut = 4;           // horizontal outputs per work item
constexpr int kVOut = 4;           // vertical outputs per work item

struct Taps {
  float w[2 * kR + 1];
};

__device__ __forceinline__ int reflect_clamp(int k, int n) {  // numpy 'symmetric' padding
  if (k < 0) k = -1 - k;
  if (k >= n) k = 2 * n - 1 - k;
  return k < 0 ? 0 : (k >= n ? n - 1 : k);  // only reached by windows of non-image positions
}

// Reflection-fold terms of the adjoint at image index y (only near the borders):
// sum_i w_i (u[-1-y-i+R] for y < R) + (u[2n-1-y-i+R] for y >= n-R), valid indices.
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

struct LossArgs {
  const float *img, *tgt;
  int W, H, P;       // P: partials row pitch (W rounded up to 4 floats, TMA stride rule)
  Taps tp;
  float c1, c2, lam, inv_count;
  float2 *part01;    // [3 channels][H][P] (dS/dmu_a, dS/dsigma_aa)
  float *part2;      // [3 channels][H][P] dS/dsigma_ab
  double *sums;      // [2][nblocks]: per-CTA L1 and SSIM sums
  float *dimage;
};

// TMA boxes: the innermost start coordinate times the element size must be a multiple
// of 16 bytes, so the (p0, p1) box (8 B elements) starts one column left of the halo
// (x0 - 6) and the p2 box (4 B) three columns left (x0 - 8); widths cover the 42-wide
// halo and keep the row a multiple of 16 bytes.
constexpr int kBoxW01 = 44, kOff01 = 1;
constexpr int kBoxW2 = 48, kOff2 = 3;

__device__ __forceinline__ void block_sum2(double l1, double ss, double *dst0, double *dst1) {
  __shared__ double red[2][kLossThreads / 32];
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
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    *dst0 = a;
    *dst1 = b;
  }
}

// Grid (3 channels, tiles_x, tiles_y): the channel is the fastest-varying block
// index, so the three CTAs of a tile run together and share the interleaved
// image lines (and halos) in L2.
__device__ __forceinline__ float2 ffma2(float w, float2 x, float2 acc) {  // packed FP32 FMA (FFMA2)
  return __ffma2_rn(make_float2(w, w), x, acc);
}

__global__ void __launch_bounds__(kLossThreads) k_ssim_fwd(LossArgs A) {
  // The five window sums run as two packed pairs (sum a, sum b) and (sum a^2, sum b^2)
  // plus the scalar sum ab: FFMA2 issues two FP32 FMAs per instruction with the same
  // per-element rounding, so the maps are bit-identical to five scalar passes.
  __shared__ float2 sab[kH * kHS];                    // (a, b) on the tile + halo
  __shared__ float2 hab[kH][kT + 1], hsq[kH][kT + 1];  // horizontal sums: (a, b), (a^2, b^2)
  __shared__ float hp[kH][kT + 1];                    // horizontal sums of a*b
  const int c = blockIdx.x;
  const int x0 = blockIdx.y * kT, y0 = blockIdx.z * kT;
  const int W = A.W, H = A.H;
  const int t = threadIdx.x;
  const Taps &tp = A.tp;
  __shared__ uint32_t roff[kH], coff[kH];  // reflected row offsets / column offsets (floats)
  if (t < kH) roff[t] = (uint32_t)reflect_clamp(y0 - kR + t, H) * (uint32_t)W * 3u;
  else if (t < 2 * kH) coff[t - kH] = (uint32_t)reflect_clamp(x0 - kR + t - kH, W) * 3u + (uint32_t)c;
  __syncthreads();
  {  // every load of the thread first, then the shared-memory stores
    constexpr int kIt = (kH * kH + kLossThreads - 1) / kLossThreads;
    float va[kIt], vb[kIt];
#pragma unroll
    for (int i = 0; i < kIt; ++i) {
      const int e = t + i * kLossThreads;
      const int r = e / kH, q = e - r * kH;
      const uint32_t p = e < kH * kH ? roff[r] + coff[q] : 0u;
      va[i] = __ldg(A.img + p);
      vb[i] = __ldg(A.tgt + p);
    }
#pragma unroll
    for (int i = 0; i < kIt; ++i) {
      const int e = t + i * kLossThreads;
      if (e < kH * kH) {
        const int r = e / kH, q = e - r * kH;
        sab[r * kHS + q] = make_float2(va[i], vb[i]);
      }
    }
  }
  __syncthreads();
  // horizontal: item = (halo row, 4 tile columns); consecutive lanes take consecutive
  // rows (odd float2 row stride: conflict-free 64-bit shared accesses)
  for (int it = t; it < kH * (kT / kHOut); it += kLossThreads) {
    const int g = it / kH, r = it - g * kH, q0 = g * kHOut;
    float2 x[kHOut + 2 * kR], sq[kHOut + 2 * kR];
    float pr[kHOut + 2 * kR];
#pragma unroll
    for (int j = 0; j < kHOut + 2 * kR; ++j) {  // products once per input, not once per tap
      x[j] = sab[r * kHS + q0 + j];
      sq[j] = __fmul2_rn(x[j], x[j]);
      pr[j] = x[j].x * x[j].y;
    }
#pragma unroll
    for (int o = 0; o < kHOut; ++o) {
      float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
      float s4 = 0.f;
#pragma unroll
      for (int k = 0; k < 2 * kR + 1; ++k) {
        const float w = tp.w[k];
        s01 = ffma2(w, x[o + k], s01);
        s23 = ffma2(w, sq[o + k], s23);
        s4 = fmaf(w, pr[o + k], s4);
      }
      hab[r][q0 + o] = s01;
      hsq[r][q0 + o] = s23;
      hp[r][q0 + o] = s4;
    }
  }
  __syncthreads();
  // vertical: item = (tile column, 4 tile rows) -> SSIM, partials, sums
  double l1 = 0.0, ss = 0.0;
  {
    const int q = t % kT, r0 = (t / kT) * kVOut;
    float2 m01[kVOut], m23[kVOut];
    float m4[kVOut];
    {
      float2 col[kVOut + 2 * kR];
#pragma unroll
      for (int j = 0; j < kVOut + 2 * kR; ++j) col[j] = hab[r0 + j][q];
#pragma unroll
      for (int o = 0; o < kVOut; ++o) {
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 2 * kR + 1; ++k) acc = ffma2(tp.w[k], col[o + k], acc);
        m01[o] = acc;
      }
#pragma unroll
      for (int j = 0; j < kVOut + 2 * kR; ++j) col[j] = hsq[r0 + j][q];
#pragma unroll
      for (int o = 0; o < kVOut; ++o) {
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 2 * kR + 1; ++k) acc = ffma2(tp.w[k], col[o + k], acc);
        m23[o] = acc;
      }
      float cp[kVOut + 2 * kR];
#pragma unroll
      for (int j = 0; j < kVOut + 2 * kR; ++j) cp[j] = hp[r0 + j][q];
#pragma unroll
      for (int o = 0; o < kVOut; ++o) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 2 * kR + 1; ++k) acc = fmaf(tp.w[k], cp[o + k], acc);
        m4[o] = acc;
      }
    }
    const int xx = x0 + q;
#pragma unroll
    for (int o = 0; o < kVOut; ++o) {
      const int yy = y0 + r0 + o;
      if (yy >= H || xx >= W) continue;
      const float m0 = m01[o].x, m1 = m01[o].y;
      const float var_a = m23[o].x - m0 * m0, var_b = m23[o].y - m1 * m1, cov = m4[o] - m0 * m1;
      const float A1 = 2.0f * m0 * m1 + A.c1, A2 = 2.0f * cov + A.c2;
      const float B1 = m0 * m0 + m1 * m1 + A.c1, B2 = var_a + var_b + A.c2;
      const float rB1 = 1.0f / B1, rB2 = 1.0f / B2, rden = rB1 * rB2;  // two reciprocals, no divisions
      const float smap = A1 * A2 * rden;
      const size_t p = ((size_t)c * H + yy) * A.P + xx;
      A.part01[p] = make_float2(2.0f * m1 * (A2 - A1) * rden - 2.0f * m0 * smap * (rB1 - rB2), -smap * rB2);
      A.part2[p] = 2.0f * A1 * rden;
      ss += smap;
      const float2 ab = sab[(r0 + o + kR) * kHS + q + kR];
      l1 += fabsf(ab.x - ab.y);
    }
  }
  const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
  const unsigned bid = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;  // any fixed order
  block_sum2(l1, ss, A.sums + bid, A.sums + nb + bid);
}

// Four CTAs per SM (64 registers, 40 B of spills): 175 -> 159 us per c3 loss call and
// +2.4% training step/s against the unconstrained 79-register build (3 CTAs per SM)
__global__ void __launch_bounds__(kLossThreads, 4) k_ssim_adj(LossArgs A, const __grid_constant__ CUtensorMap tm01,
                                                         const __grid_constant__ CUtensorMap tm2) {
  // partials (p0, p1) as a packed pair + p2 scalar: two FFMA2 + one FFMA per tap
  // instead of three FFMA, bit-identical per component.  The tile + 5 px halo of the
  // partials arrives by two 2-D TMA tile loads (one thread, one mbarrier); the TMA
  // zero-fills rows / columns outside the image, which is exactly the adjoint's
  // boundary condition (no per-element bounds checks, no register staging).
  __shared__ __align__(128) float2 sd01[kH][kBoxW01];  // (p0, p1): halo column q at [q + kOff01]
  __shared__ __align__(128) float sd2[kH][kBoxW2];      // p2: halo column q at [q + kOff2]
  __shared__ float2 se01[kT][kHS];  // vertical adjoint on the tile rows, halo columns
  __shared__ float se2[kT][kHS];
  __shared__ __align__(8) uint64_t bar;
  const int c = blockIdx.x;
  const int x0 = blockIdx.y * kT, y0 = blockIdx.z * kT;
  const int mx = x0 - kR, my = y0 - kR;  // image coords of sd[.][0][0]
  const int W = A.W, H = A.H;
  const int t = threadIdx.x;
  const Taps &tp = A.tp;
  const bool border = x0 < kR || y0 < kR || x0 + kT > W - kR || y0 + kT > H - kR;
  const uint32_t bar_s = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s),
                 "r"((uint32_t)(sizeof(sd01) + sizeof(sd2)))
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&sd01[0][0]))),
        "l"(reinterpret_cast<uint64_t>(&tm01)), "r"(mx - kOff01), "r"(my), "r"(c), "r"(bar_s)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&sd2[0][0]))),
        "l"(reinterpret_cast<uint64_t>(&tm2)), "r"(mx - kOff2), "r"(my), "r"(c), "r"(bar_s)
        : "memory");
  }
  __syncthreads();  // the barrier's initialisation is visible before anyone waits on it
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(bar_s)
      : "memory");
  // vertical adjoint: item = (halo column, 4 tile rows), symmetric taps -> correlation
  // (the pair and the scalar in one loop: measured faster than one input window at a
  // time despite the registers; so was the inlined lambda fold vs a strided-pointer one)
  for (int it = t; it < kH * (kT / kVOut); it += kLossThreads) {
    const int q = it % kH, r0 = (it / kH) * kVOut;
    const int xx = mx + q;
    const bool colok = xx >= 0 && xx < W;
    float2 col01[kVOut + 2 * kR];
    float col2[kVOut + 2 * kR];
#pragma unroll
    for (int j = 0; j < kVOut + 2 * kR; ++j) {
      col01[j] = sd01[r0 + j][q + kOff01];
      col2[j] = sd2[r0 + j][q + kOff2];
    }
#pragma unroll
    for (int o = 0; o < kVOut; ++o) {
      float2 a01 = make_float2(0.f, 0.f);
      float a2 = 0.f;
#pragma unroll
      for (int k = 0; k < 2 * kR + 1; ++k) {
        a01 = ffma2(tp.w[k], col01[o + k], a01);
        a2 = fmaf(tp.w[k], col2[o + k], a2);
      }
      const int yy = y0 + r0 + o;
      if (border && yy < H && (yy < kR || yy >= H - kR) && colok) {
        a01.x += adjoint_fold(yy, H, tp, [&](int j) { return sd01[j - my][q + kOff01].x; });
        a01.y += adjoint_fold(yy, H, tp, [&](int j) { return sd01[j - my][q + kOff01].y; });
        a2 += adjoint_fold(yy, H, tp, [&](int j) { return sd2[j - my][q + kOff2]; });
      }
      const bool ok = yy < H && colok;
      se01[r0 + o][q] = ok ? a01 : make_float2(0.f, 0.f);
      se2[r0 + o][q] = ok ? a2 : 0.0f;
    }
  }
  __syncthreads();
  // horizontal adjoint: item = (tile row, 4 tile columns); combine with the L1 sign
  {
    const int r = t / (kT / kHOut), c0 = (t - r * (kT / kHOut)) * kHOut;
    const int yy = y0 + r;
    float g0[kHOut], g1[kHOut], g2[kHOut];
    {
      float2 row01[kHOut + 2 * kR];
      float row2[kHOut + 2 * kR];
#pragma unroll
      for (int j = 0; j < kHOut + 2 * kR; ++j) {
        row01[j] = se01[r][c0 + j];
        row2[j] = se2[r][c0 + j];
      }
#pragma unroll
      for (int o = 0; o < kHOut; ++o) {
        float2 a01 = make_float2(0.f, 0.f);
        float a2 = 0.f;
#pragma unroll
        for (int k = 0; k < 2 * kR + 1; ++k) {
          a01 = ffma2(tp.w[k], row01[o + k], a01);
          a2 = fmaf(tp.w[k], row2[o + k], a2);
        }
        const int xx = x0 + c0 + o;
        if (border && xx < W && (xx < kR || xx >= W - kR)) {
          a01.x += adjoint_fold(xx, W, tp, [&](int j) { return se01[r][j - mx].x; });
          a01.y += adjoint_fold(xx, W, tp, [&](int j) { return se01[r][j - mx].y; });
          a2 += adjoint_fold(xx, W, tp, [&](int j) { return se2[r][j - mx]; });
        }
        g0[o] = a01.x;
        g1[o] = a01.y;
        g2[o] = a2;
      }
    }
    if (yy < H) {
      // all eight image / target loads in flight before the first store (the stores to
      // dimage could alias them, so the compiler would otherwise serialise load -> store
      // per pixel: a quarter of the kernel's stall samples)
      float av[kHOut], bv[kHOut];
#pragma unroll
      for (int o = 0; o < kHOut; ++o) {
        const int xx = min(x0 + c0 + o, W - 1);
        const size_t p = ((size_t)yy * W + xx) * 3 + c;
        av[o] = __ldg(A.img + p);
        bv[o] = __ldg(A.tgt + p);
      }
#pragma unroll
      for (int o = 0; o < kHOut; ++o) {
        const int xx = x0 + c0 + o;
        if (xx >= W) continue;
        const size_t p = ((size_t)yy * W + xx) * 3 + c;
        const float grad = (g0[o] + 2.0f * av[o] * g1[o] + bv[o] * g2[o]) * A.inv_count;
        const float diff = av[o] - bv[o];
        const float sgn = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
        A.dimage[p] = (1.0f - A.lam) * sgn * A.inv_count - A.lam * 0.5f * grad;
      }
    }
  }
}

// terms = {mean |a - b|, mean SSIM}: sum of the per-CTA partials (fixed order)
__global__ void __launch_bounds__(1024) k_loss_finalize(const double *__restrict__ sums, int nb, double inv_count,
                                                        double *__restrict__ terms) {
  __shared__ double red[2][32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += sums[i];
    b += sums[nb + i];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
    red[0][warp] = a;
    red[1][warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0.0;
    b = 0.0;
    for (int w = 0; w < 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    terms[0] = a * inv_count;
    terms[1] = b * inv_count;
  }
}

inline size_t loss_blocks(int W, int H) { return (size_t)ceil_div(W, kT) * ceil_div(H, kT) * 3; }

}  // namespace tgs

using namespace tgs;

static inline size_t loss_pitch(int32_t width) { return ((size_t)width + 3) / 4 * 4; }

extern "C" int tgs_loss_workspace(int32_t width, int32_t height, size_t *bytes) {
  if (width < 1 || height < 1 || !bytes) return TGS_ERR_INVALID;
  // per-channel SSIM partials ((p0, p1) pairs + p2, row pitch P) + per-CTA double sums
  *bytes = align_up((size_t)9 * loss_pitch(width) * height * sizeof(float)) +
           2 * loss_blocks(width, height) * sizeof(double);
  return TGS_OK;
}

// 3-D tiled tensor map over [3 channels][H][P] elements of `esize` bytes (box box_w x 42 x 1)
static int partial_map(CUtensorMap *m, void *base, CUtensorMapDataType type, size_t esize, int W, int H, size_t P,
                       int box_w) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&encode), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode)
      return TGS_ERR_CUDA;
  }
  const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 3};
  const cuuint64_t strides[2] = {(cuuint64_t)(P * esize), (cuuint64_t)(P * esize * H)};
  const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)kH, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(m, type, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);  // out of bounds -> zeros
  return r == CUDA_SUCCESS ? TGS_OK : TGS_ERR_CUDA;
}

extern "C" int tgs_loss_l1_ssim(const float *image, const float *target, int32_t width, int32_t height,
                                float lambda_ssim, float *dimage, double *terms, void *workspace,
                                tgs_stream_t stream) {
  if (width < 2 * kR + 1 || height < 2 * kR + 1) return TGS_ERR_INVALID;  // metrics.py:83-84
  if (!image || !target || !dimage || !terms || !workspace) return TGS_ERR_INVALID;
  if (reinterpret_cast<uintptr_t>(workspace) & 15) return TGS_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  LossArgs A;
  double w[2 * kR + 1], tot = 0.0;  // gaussian_taps (metrics.py:58-61), float64 then rounded
  for (int i = 0; i < 2 * kR + 1; ++i) {
    const double xx = (double)(i - kR) / 1.5;
    w[i] = exp(-0.5 * xx * xx);
    tot += w[i];
  }
  for (int i = 0; i < 2 * kR + 1; ++i) A.tp.w[i] = (float)(w[i] / tot);
  const size_t count = (size_t)width * height * 3;
  const size_t P = loss_pitch(width);
  A.img = image;
  A.tgt = target;
  A.W = width;
  A.H = height;
  A.P = (int)P;
  A.c1 = 0.01f * 0.01f;
  A.c2 = 0.03f * 0.03f;
  A.lam = lambda_ssim;
  A.inv_count = 1.0f / (float)count;
  A.part01 = static_cast<float2 *>(workspace);
  A.part2 = reinterpret_cast<float *>(A.part01 + 3 * P * height);
  A.sums = reinterpret_cast<double *>(static_cast<char *>(workspace) +
                                      align_up((size_t)9 * P * height * sizeof(float)));
  A.dimage = dimage;
  CUtensorMap tm01, tm2;
  int rc = partial_map(&tm01, A.part01, CU_TENSOR_MAP_DATA_TYPE_UINT64, 8, width, height, P, kBoxW01);
  if (rc == TGS_OK) rc = partial_map(&tm2, A.part2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, width, height, P, kBoxW2);
  if (rc != TGS_OK) return rc;
  const dim3 grd(3, (unsigned)ceil_div(width, kT), (unsigned)ceil_div(height, kT));
  // four 44 KB CTAs per SM and the rest of the unified L1 as cache for the reflected
  // image / target loads the three channel CTAs of a tile share (a fifth CTA would
  // shrink that cache and costs more than its occupancy gains)
  static std::atomic<uint64_t> carve{0};
  rc = attr_once_per_device(carve, [] {
    return cudaFuncSetAttribute(k_ssim_fwd, cudaFuncAttributePreferredSharedMemoryCarveout, 80);
  });
  if (rc != TGS_OK) return rc;
  k_ssim_fwd<<<grd, kLossThreads, 0, st>>>(A);
  k_ssim_adj<<<grd, kLossThreads, 0, st>>>(A, tm01, tm2);
  k_loss_finalize<<<1, 1024, 0, st>>>(A.sums, (int)loss_blocks(width, height), 1.0 / (double)count, terms);
  return launch_status();
}
