// tgs_math.cuh — float32 device math with fully specified rounding.
//
// The preprocess kernels (preprocess.cu, compiled with -fmad=false) must give
// the same bits as the float32 oracle for visibility, radii and tile counts.
// These helpers evaluate the documented operation sequence (DESIGN.md
// "fp32 semantics") with explicit round-to-nearest intrinsics so neither FMA
// contraction nor approximate SFU instructions can change a result.
#pragma once

#include <cstdint>

namespace tgs {

// exp(x): Cody-Waite reduction by ln2 (hi/lo split), degree-7 Taylor polynomial
// in Horner form with fma, exact 2^k scaling in two halves.
// exp(x) := 0 for x <= -87, +inf for x > 88.72, NaN passes through. <= 2 ulp.
__device__ __forceinline__ float sem_expf(float x) {
  if (x != x) return x;
  if (!(x > -87.0f)) return 0.0f;
  if (x > 88.72f) return __int_as_float(0x7f800000);
  const float k = rintf(__fmul_rn(x, 1.44269502f));
  float r = __fmaf_rn(k, -0.693145751953125f, x);
  r = __fmaf_rn(k, -1.42860677e-6f, r);
  float p = 1.98412698e-4f;
  p = __fmaf_rn(p, r, 1.38888889e-3f);
  p = __fmaf_rn(p, r, 8.33333333e-3f);
  p = __fmaf_rn(p, r, 4.16666667e-2f);
  p = __fmaf_rn(p, r, 1.66666667e-1f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  const int ki = (int)k;
  const int k1 = ki / 2, k2 = ki - k1;
  const float s1 = __int_as_float((k1 + 127) << 23);
  const float s2 = __int_as_float((k2 + 127) << 23);
  return __fmul_rn(__fmul_rn(p, s1), s2);
}

__device__ __forceinline__ float sem_sigmoidf(float x) {
  return __fdiv_rn(1.0f, __fadd_rn(1.0f, sem_expf(-x)));
}

// SH constants (sh.py:14-31), rounded to float32
constexpr float SH_C0 = 0.28209479177387814f;
constexpr float SH_C1 = 0.4886025119029199f;
constexpr float SH_C2_0 = 1.0925484305920792f, SH_C2_1 = -1.0925484305920792f, SH_C2_2 = 0.31539156525252005f,
                SH_C2_3 = -1.0925484305920792f, SH_C2_4 = 0.5462742152960396f;
constexpr float SH_C3_0 = -0.5900435899266435f, SH_C3_1 = 2.890611442640554f, SH_C3_2 = -0.4570457994644658f,
                SH_C3_3 = 0.3731763325901154f, SH_C3_4 = -0.4570457994644658f, SH_C3_5 = 1.445305721320277f,
                SH_C3_6 = -0.5900435899266435f;

// band (0..2 for bands 1..3) of rest coefficient k (sh.py:34)
__device__ __forceinline__ int band_of(int k) { return k < 3 ? 0 : (k < 8 ? 1 : 2); }

// sh.py:47-74, rest-coefficient basis b[k] = Y_{k+1}(dir), k = 0..14
__device__ __forceinline__ void sh_basis_rest(float x, float y, float z, float b[15]) {
  b[0] = -SH_C1 * y;
  b[1] = SH_C1 * z;
  b[2] = -SH_C1 * x;
  const float xx = x * x, yy = y * y, zz = z * z;
  b[3] = SH_C2_0 * x * y;
  b[4] = SH_C2_1 * y * z;
  b[5] = SH_C2_2 * (2.0f * zz - xx - yy);
  b[6] = SH_C2_3 * x * z;
  b[7] = SH_C2_4 * (xx - yy);
  b[8] = SH_C3_0 * y * (3.0f * xx - yy);
  b[9] = SH_C3_1 * x * y * z;
  b[10] = SH_C3_2 * y * (4.0f * zz - xx - yy);
  b[11] = SH_C3_3 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
  b[12] = SH_C3_4 * x * (4.0f * zz - xx - yy);
  b[13] = SH_C3_5 * z * (xx - yy);
  b[14] = SH_C3_6 * x * (xx - 3.0f * yy);
}

// sh.py:77-120, d b[k] / d dir for k = 0..14
__device__ __forceinline__ void sh_basis_rest_grad(float x, float y, float z, float g[15][3]) {
#pragma unroll
  for (int k = 0; k < 15; ++k) g[k][0] = g[k][1] = g[k][2] = 0.0f;
  g[0][1] = -SH_C1;
  g[1][2] = SH_C1;
  g[2][0] = -SH_C1;
  g[3][0] = SH_C2_0 * y;
  g[3][1] = SH_C2_0 * x;
  g[4][1] = SH_C2_1 * z;
  g[4][2] = SH_C2_1 * y;
  g[5][0] = SH_C2_2 * (-2.0f * x);
  g[5][1] = SH_C2_2 * (-2.0f * y);
  g[5][2] = SH_C2_2 * (4.0f * z);
  g[6][0] = SH_C2_3 * z;
  g[6][2] = SH_C2_3 * x;
  g[7][0] = SH_C2_4 * (2.0f * x);
  g[7][1] = SH_C2_4 * (-2.0f * y);
  const float xx = x * x, yy = y * y, zz = z * z;
  g[8][0] = SH_C3_0 * 6.0f * x * y;
  g[8][1] = SH_C3_0 * (3.0f * xx - 3.0f * yy);
  g[9][0] = SH_C3_1 * y * z;
  g[9][1] = SH_C3_1 * x * z;
  g[9][2] = SH_C3_1 * x * y;
  g[10][0] = SH_C3_2 * (-2.0f * x * y);
  g[10][1] = SH_C3_2 * (4.0f * zz - xx - 3.0f * yy);
  g[10][2] = SH_C3_2 * (8.0f * y * z);
  g[11][0] = SH_C3_3 * (-6.0f * x * z);
  g[11][1] = SH_C3_3 * (-6.0f * y * z);
  g[11][2] = SH_C3_3 * (6.0f * zz - 3.0f * xx - 3.0f * yy);
  g[12][0] = SH_C3_4 * (4.0f * zz - 3.0f * xx - yy);
  g[12][1] = SH_C3_4 * (-2.0f * x * y);
  g[12][2] = SH_C3_4 * (8.0f * x * z);
  g[13][0] = SH_C3_5 * (2.0f * x * z);
  g[13][1] = SH_C3_5 * (-2.0f * y * z);
  g[13][2] = SH_C3_5 * (xx - yy);
  g[14][0] = SH_C3_6 * (3.0f * xx - 3.0f * yy);
  g[14][1] = SH_C3_6 * (-6.0f * x * y);
}

// sum_k w[k] * d b[k] / d dir (k < K) without materialising the 15x3 gradient table
// (sh.py:77-120); used by the backward where registers are the occupancy limit.
template <int K>
__device__ __forceinline__ void sh_dir_grad(float x, float y, float z, const float w[15], float g[3]) {
  float gx = 0.0f, gy = 0.0f, gz = 0.0f;
  if (K > 0) {
    gy += w[0] * -SH_C1;
    gz += w[1] * SH_C1;
    gx += w[2] * -SH_C1;
  }
  if (K > 3) {
    gx += w[3] * (SH_C2_0 * y) + w[5] * (SH_C2_2 * (-2.0f * x)) + w[6] * (SH_C2_3 * z) + w[7] * (SH_C2_4 * (2.0f * x));
    gy += w[3] * (SH_C2_0 * x) + w[4] * (SH_C2_1 * z) + w[5] * (SH_C2_2 * (-2.0f * y)) + w[7] * (SH_C2_4 * (-2.0f * y));
    gz += w[4] * (SH_C2_1 * y) + w[5] * (SH_C2_2 * (4.0f * z)) + w[6] * (SH_C2_3 * x);
  }
  if (K > 8) {
    const float xx = x * x, yy = y * y, zz = z * z;
    gx += w[8] * (SH_C3_0 * 6.0f * x * y) + w[9] * (SH_C3_1 * y * z) + w[10] * (SH_C3_2 * (-2.0f * x * y)) +
          w[11] * (SH_C3_3 * (-6.0f * x * z)) + w[12] * (SH_C3_4 * (4.0f * zz - 3.0f * xx - yy)) +
          w[13] * (SH_C3_5 * (2.0f * x * z)) + w[14] * (SH_C3_6 * (3.0f * xx - 3.0f * yy));
    gy += w[8] * (SH_C3_0 * (3.0f * xx - 3.0f * yy)) + w[9] * (SH_C3_1 * x * z) +
          w[10] * (SH_C3_2 * (4.0f * zz - xx - 3.0f * yy)) + w[11] * (SH_C3_3 * (-6.0f * y * z)) +
          w[12] * (SH_C3_4 * (-2.0f * x * y)) + w[13] * (SH_C3_5 * (-2.0f * y * z)) + w[14] * (SH_C3_6 * (-6.0f * x * y));
    gz += w[9] * (SH_C3_1 * x * y) + w[10] * (SH_C3_2 * (8.0f * y * z)) +
          w[11] * (SH_C3_3 * (6.0f * zz - 3.0f * xx - 3.0f * yy)) + w[12] * (SH_C3_4 * (8.0f * x * z)) +
          w[13] * (SH_C3_5 * (xx - yy));
  }
  g[0] = gx;
  g[1] = gy;
  g[2] = gz;
}

// bin_tiles rect + on-screen gate (rasterizer.py:112-128).  Returns the tile
// count (0 when the box misses the pixel grid or r <= 0).
__device__ __forceinline__ int tile_rect(float mx, float my, float r, int W, int H, int ts, int tiles_x,
                                         int tiles_y, int &x0, int &y0, int &x1, int &y1) {
  auto cl = [](float v, int hi) -> int {
    v = floorf(v);
    if (!(v >= 0.0f)) v = 0.0f;
    if (v > (float)hi) v = (float)hi;
    return (int)v;
  };
  const float fts = (float)ts;
  x0 = cl(__fdiv_rn(__fsub_rn(mx, r), fts), tiles_x - 1);
  x1 = cl(__fdiv_rn(__fadd_rn(mx, r), fts), tiles_x - 1);
  y0 = cl(__fdiv_rn(__fsub_rn(my, r), fts), tiles_y - 1);
  y1 = cl(__fdiv_rn(__fadd_rn(my, r), fts), tiles_y - 1);
  const bool on = (__fadd_rn(mx, r) >= 0.0f) && (__fsub_rn(mx, r) <= (float)(W - 1)) &&
                  (__fadd_rn(my, r) >= 0.0f) && (__fsub_rn(my, r) <= (float)(H - 1)) && (r > 0.0f);
  return on ? (x1 - x0 + 1) * (y1 - y0 + 1) : 0;
}

// float -> uint32 whose unsigned order equals the float order (-0 folded onto +0)
__device__ __forceinline__ uint32_t orderable_key(float d) {
  uint32_t b = __float_as_uint(__fadd_rn(d, 0.0f));
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint64_t orderable_key64(double d) {
  uint64_t b = (uint64_t)__double_as_longlong(d + 0.0);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

}  // namespace tgs
