// preprocess.cu — per-Gaussian forward kernel (R1-R4).
//
// Compiled with -fmad=false: together with tgs_math.cuh this pins every float
// operation to the documented order so visibility, radii and tile counts are
// bit-identical to the float32 oracle.  The
// backward (which only has to meet the gradient tolerance) lives in
// preprocess_bwd.cu, compiled with FMA contraction.
//
// Forward  : masking.py:21-43,84-86 (hard masks), geometry.py:19-41,74-77
//            (quaternion -> R -> Sigma), geometry.py:138-195 (EWA projection),
//            rasterizer.py:177-197 (alpha-skip, view dirs, SH colour),
//            sh.py:135-161, rasterizer.py:112-128 (tile rect/count).
//
// A streaming kernel, one thread per Gaussian.  The 180 B/Gaussian sh_rest
// block is staged through shared memory with 16 B coalesced loads (a
// per-thread 45-float stride would split every warp access over 45 lines).
#include "preprocess_common.cuh"

namespace tgs {

// Forward quantities of Gaussian i in the documented float32 order.  `rest`
// points at this Gaussian's 45 staged coefficients (may be null when degree 0).
__device__ __forceinline__ void gauss_static(const tgs_cloud &cl, int64_t i, const tgs_settings &s, GaussFwd &f) {
  // hard masks in logit space (masking.py:21-25; see tgs.h)
  const float m = cl.mask_logits[i], o = cl.opacity_logits[i];
  f.Mg = (m > s.mask_logit_min) ? 1.0f : 0.0f;
#pragma unroll
  for (int l = 0; l < 3; ++l) f.band[l] = (cl.sh_mask_logits[3 * i + l] > s.sh_mask_logit_min) ? 1.0f : 0.0f;
  f.alpha_ok = (f.Mg > 0.0f) && (o >= s.opacity_logit_min);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    f.s_raw[k] = sem_expf(cl.log_scales[3 * i + k]);
    f.sc[k] = f.s_raw[k] * f.Mg;
  }
  // normalize_quaternions + quat_to_rotmat (geometry.py:19-41)
  const float qw = cl.rotations[4 * i], qx = cl.rotations[4 * i + 1];
  const float qy = cl.rotations[4 * i + 2], qz = cl.rotations[4 * i + 3];
  f.qnorm = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  f.degenerate = f.qnorm < 1e-12f;
  const float w = qw / f.qnorm, x = qx / f.qnorm, y = qy / f.qnorm, z = qz / f.qnorm;
  f.qn[0] = w; f.qn[1] = x; f.qn[2] = y; f.qn[3] = z;
  float *Rg = f.Rg;
  Rg[0] = 1.0f - 2.0f * (y * y + z * z);
  Rg[1] = 2.0f * (x * y - w * z);
  Rg[2] = 2.0f * (x * z + w * y);
  Rg[3] = 2.0f * (x * y + w * z);
  Rg[4] = 1.0f - 2.0f * (x * x + z * z);
  Rg[5] = 2.0f * (y * z - w * x);
  Rg[6] = 2.0f * (x * z - w * y);
  Rg[7] = 2.0f * (y * z + w * x);
  Rg[8] = 1.0f - 2.0f * (x * x + y * y);
  // Sigma = L L^T, L = R diag(s) (geometry.py:74-77)
  float L[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) L[3 * r + k] = Rg[3 * r + k] * f.sc[k];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      f.S[3 * a + b] = L[3 * a] * L[3 * b] + L[3 * a + 1] * L[3 * b + 1] + L[3 * a + 2] * L[3 * b + 2];
}

// The SH-rest coefficients times their band masks (sh.py:152-160), once per Gaussian
// (in place in its staged shared-memory row): the per-view colour sums then skip the
// 45 mask products — the same float32 products, so the same bits.
template <int DEG>
__device__ __forceinline__ void premask_rest(float *rest, const GaussFwd &f) {
  constexpr int K = (DEG + 1) * (DEG + 1) - 1;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) rest[3 * k + c] = rest[3 * k + c] * f.band[band_of(k)];
}

// The view-dependent half: EWA projection, view direction and SH colour.  `f`
// carries gauss_static's outputs (computed once per Gaussian for a batch of views);
// `rest` is the band-masked row (premask_rest).
template <int DEG>
__device__ __forceinline__ void gauss_view(const tgs_cloud &cl, int64_t i, const tgs_camera &cam,
                                           const tgs_settings &s, const float *rest, GaussFwd &f) {
  // EWA projection (geometry.py:153-183)
  const float px = cl.positions[3 * i], py = cl.positions[3 * i + 1], pz = cl.positions[3 * i + 2];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    f.t[r] = px * cam.R[3 * r] + py * cam.R[3 * r + 1] + pz * cam.R[3 * r + 2] + cam.t[r];
  const float tz = f.t[2];
  f.valid = tz > s.near_plane;
  f.mean[0] = cam.fx * f.t[0] / tz + cam.cx;
  f.mean[1] = cam.fy * f.t[1] / tz + cam.cy;
  const float tz2 = tz * tz;
  const float J00 = cam.fx / tz, J02 = -cam.fx * f.t[0] / tz2;
  const float J11 = cam.fy / tz, J12 = -cam.fy * f.t[1] / tz2;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    f.Mj[j] = J00 * cam.R[j] + J02 * cam.R[6 + j];
    f.Mj[3 + j] = J11 * cam.R[3 + j] + J12 * cam.R[6 + j];
  }
  float A[6];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      A[3 * r + j] = f.Mj[3 * r] * f.S[j] + f.Mj[3 * r + 1] * f.S[3 + j] + f.Mj[3 * r + 2] * f.S[6 + j];
  const float lp = s.lowpass_s;
  f.c00 = A[0] * f.Mj[0] + A[1] * f.Mj[1] + A[2] * f.Mj[2] + lp;
  f.c01 = A[0] * f.Mj[3] + A[1] * f.Mj[4] + A[2] * f.Mj[5];
  f.c11 = A[3] * f.Mj[3] + A[4] * f.Mj[4] + A[5] * f.Mj[5] + lp;
  f.det = f.c00 * f.c11 - f.c01 * f.c01;
  f.ok = f.det > 0.0f;
  const float inv = f.ok ? 1.0f / f.det : 0.0f;
  f.conic[0] = f.c11 * inv;
  f.conic[1] = -f.c01 * inv;
  f.conic[2] = f.c00 * inv;
  const float mid = 0.5f * (f.c00 + f.c11);
  const float lam = mid + sqrtf(max0(mid * mid - f.det));
  f.radius = 3.0f * sqrtf(max0(lam));
  f.area = 28.274333882308138f * sqrtf(max0(f.det));  // 9*pi (geometry.py:183)
  f.visible = f.valid && f.ok && f.alpha_ok;
  // view direction (rasterizer.py:190-193)
  const float d0 = px - cam.center[0], d1 = py - cam.center[1], d2 = pz - cam.center[2];
  const float nrm = sqrtf(d0 * d0 + d1 * d1 + d2 * d2);
  f.dnorm = nrm < 1e-12f ? 1e-12f : nrm;
  f.dir[0] = d0 / f.dnorm;
  f.dir[1] = d1 / f.dnorm;
  f.dir[2] = d2 / f.dnorm;
  // SH colour (sh.py:135-161): C0*dc + 0.5 + sum_k Y_{k+1} * rest_k * bandmask_k, clamped at 0
  constexpr int K = (DEG + 1) * (DEG + 1) - 1;
  float b[15];
  sh_basis_rest(f.dir[0], f.dir[1], f.dir[2], b);
  // (scalar on purpose: packed f32x2 multiply + add, even as explicit-rounding PTX,
  // is fused into FFMA2 by ptxas under -fmad=false and would break the bit-exact
  // forward — measured)
  float acc[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] = acc[c] + b[k] * rest[3 * k + c];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float col = SH_C0 * cl.sh_dc[3 * i + c] + 0.5f;
    if (DEG > 0) col = col + acc[c];
    f.pre[c] = col;
    f.col[c] = max0(col);
  }
}

template <int DEG>
__device__ __forceinline__ void gauss_forward(const tgs_cloud &cl, int64_t i, const tgs_camera &cam,
                                              const tgs_settings &s, float *rest, GaussFwd &f) {
  gauss_static(cl, i, s, f);
  if (DEG > 0) premask_rest<DEG>(rest, f);
  gauss_view<DEG>(cl, i, cam, s, rest, f);
}

// ---- exact blend-decision records (include/tgs.h TGS_EXACT_FLOATS) ----------------
// The blend kernels decide from the float32 record whether Gaussian g blends into pixel
// p (e >= -4.5, e <= 0, alpha exp(e) >= 1/255: _kernels.py:62-72).  The reference makes
// that decision in float64; close to a threshold float32 can decide the other way and
// move a pixel by a whole contribution.  Here the float64 projection is recomputed in
// the reference's operation order (this file is compiled with -fmad=false, so no
// operation is fused) and turned into
//   * a float32 bracket [cut_lo, cut_hi] around the float64 cut, widened by a bound on
//     the error of the blend kernels' float32 exponent over the Gaussian's footprint
//     (record errors times the footprint's extent, plus the evaluation's roundings),
//     so outside the bracket the float32 comparison IS the float64 decision;
//   * the float64-minus-float32 residuals of means, conic and alpha, from which the
//     blend kernels rebuild the float64 record for the rare pairs inside the bracket.
struct Static64 {  // view-independent float64 state (masking.py:34-43, geometry.py:19-41,74-77)
  double S[6];     // S00 S01 S02 S11 S12 S22
  double alpha;    // sigmoid(o) * M
  double cut;      // the blend cut max(-4.5, ln(1 / (255 alpha))) (_kernels.py:62-72)
};

__device__ __forceinline__ void gauss_static64(const tgs_cloud &cl, int64_t i, float Mg, Static64 &g) {
  const double M = (double)Mg;
  double sc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) sc[k] = exp((double)cl.log_scales[3 * i + k]) * M;
  const double qw = cl.rotations[4 * i], qx = cl.rotations[4 * i + 1];
  const double qy = cl.rotations[4 * i + 2], qz = cl.rotations[4 * i + 3];
  const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  const double w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
  const double Rg[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                        2.0 * (x * y + w * z),       1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                        2.0 * (x * z - w * y),       2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
  double L[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) L[3 * r + k] = Rg[3 * r + k] * sc[k];
  int e = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b) g.S[e++] = L[3 * a] * L[3 * b] + L[3 * a + 1] * L[3 * b + 1] + L[3 * a + 2] * L[3 * b + 2];
  g.alpha = (1.0 / (1.0 + exp(-(double)cl.opacity_logits[i]))) * M;
  g.cut = g.alpha > 0.0 ? fmax(-4.5, -log(255.0 * g.alpha)) : 0.0;
}

constexpr double kLog2eD = 1.4426950408889634;

// One view's exact record of a visible Gaussian; a, b: the first two float4 of its float32
// record (means, conic, alpha).
__device__ __forceinline__ void exact_record(const tgs_cloud &cl, int64_t i, const tgs_camera &cam,
                                             const tgs_settings &s, const Static64 &g, float4 a, float4 b,
                                             float4 *__restrict__ out) {
  const float alpha32 = b.y;
  // project_gaussians in float64 (geometry.py:153-183) in the oracle's operation order, with
  // the divisions by t_z and det as multiplications by one reciprocal each: the record only
  // has to be float64-accurate (~1e-15 relative), its residuals are stored as float32 anyway
  const double px = cl.positions[3 * i], py = cl.positions[3 * i + 1], pz = cl.positions[3 * i + 2];
  double t[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) t[r] = px * cam.R64[3 * r] + py * cam.R64[3 * r + 1] + pz * cam.R64[3 * r + 2] + cam.t64[r];
  const double itz = 1.0 / t[2];
  const double m0 = cam.fx64 * t[0] * itz + cam.cx64, m1 = cam.fy64 * t[1] * itz + cam.cy64;
  const double J00 = cam.fx64 * itz, J02 = -cam.fx64 * t[0] * (itz * itz);
  const double J11 = cam.fy64 * itz, J12 = -cam.fy64 * t[1] * (itz * itz);
  double Mj[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    Mj[j] = J00 * cam.R64[j] + J02 * cam.R64[6 + j];
    Mj[3 + j] = J11 * cam.R64[3 + j] + J12 * cam.R64[6 + j];
  }
  auto Sg = [&](int a, int b) -> double {
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    return g.S[lo == 0 ? hi : (lo == 1 ? 2 + hi : 5)];
  };
  double A[6];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int j = 0; j < 3; ++j) A[3 * r + j] = Mj[3 * r] * Sg(0, j) + Mj[3 * r + 1] * Sg(1, j) + Mj[3 * r + 2] * Sg(2, j);
  const double lp = s.lowpass_s64;
  const double c00 = A[0] * Mj[0] + A[1] * Mj[1] + A[2] * Mj[2] + lp;
  const double c01 = A[0] * Mj[3] + A[1] * Mj[4] + A[2] * Mj[5];
  const double c11 = A[3] * Mj[3] + A[4] * Mj[4] + A[5] * Mj[5] + lp;
  const double det = c00 * c11 - c01 * c01;
  if (!(det > 1e-300) || !(g.alpha > 0.0)) {
    // culled in float64 (geometry.py:176): never blends there
    const float inf = __int_as_float(0x7f800000);
    out[0] = make_float4(inf, inf, 0.f, 0.f);
    out[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const double inv = 1.0 / det;
  const double k0 = c11 * inv, k1 = -c01 * inv, k2 = c00 * inv;
  const double dmx = m0 - (double)a.x, dmy = m1 - (double)a.y;
  const double dk0 = k0 - (double)a.z, dk1 = k1 - (double)a.w, dk2 = k2 - (double)b.x;
  // the error bound in float32 (an upper bound only needs a few digits): footprint of the
  // pixels near the cut, |dx| <= X, |dy| <= Y on {e >= cut - margin}, then
  // |e32 - e64| <= record error over the footprint + float32 evaluation roundings
  const float cut = (float)g.cut;
  const float reach = 2.0f * (fabsf(cut) + 0.01f);
  const float X = 1.001f * sqrtf(reach * (float)c00), Y = 1.001f * sqrtf(reach * (float)c11);
  const float a0 = fabsf(a.z) * 1.001f, a1 = fabsf(a.w) * 1.001f, a2 = fabsf(b.x) * 1.001f;
  float E = (a0 * X + a1 * Y) * fabsf((float)dmx) + (a1 * X + a2 * Y) * fabsf((float)dmy) +
            0.5f * (fabsf((float)dk0) * X * X + fabsf((float)dk2) * Y * Y) + fabsf((float)dk1) * X * Y +
            1e-6f * (a0 * X * X + 2.0f * a1 * X * Y + a2 * Y * Y) + 1e-6f;
  const double E2 = 2.0 * (double)E;  // safety factor
  const float lo = __double2float_rd((g.cut - E2) * kLog2eD);
  // a Gaussian whose alpha can reach the 0.99 clamp (float32 alpha > 0.9899, the same test
  // the blend kernels make on the same float): its cut is -4.5 exactly (alpha > 0.353 puts
  // ln(1/(255 alpha)) below it) and slot 7 holds the clamp's exponent ln(0.99 / alpha)
  // (alpha exp(e) <= 0.99 <=> e <= it): the kernels bracket it with the same error bound
  // as the cut (clamp_lo_of in blend.cu) and decide the pairs above the bracket's lower end
  // in float64; otherwise slot 7 holds the float64 cut minus cut_lo (log2 units) for the
  // float64 comparison e >= cut
  const bool clampable = alpha32 > 0.9899f;
  const float hi = __double2float_ru((g.cut + E2) * kLog2eD);
  const float slot7 = clampable ? (float)log(0.99 / g.alpha) : (float)(g.cut * kLog2eD - (double)lo);
  out[0] = make_float4(lo, hi, (float)dmx, (float)dmy);
  out[1] = make_float4((float)dk0, (float)dk1, (float)dk2, slot7);
}

template <int DEG>
__device__ __forceinline__ void emit_view_impl(const tgs_cloud &cl, int64_t i, const tgs_camera &cam,
                                               const tgs_settings &s, float *rest, float *__restrict__ splats,
                                               uint8_t *__restrict__ visible, int32_t *__restrict__ tiles,
                                               uint64_t *__restrict__ depth_keys, int32_t *__restrict__ err);
__device__ __forceinline__ void emit_record(const tgs_cloud &cl, int64_t i, const tgs_camera &cam,
                                            const tgs_settings &s, const GaussFwd &f, float *__restrict__ splats,
                                            uint8_t *__restrict__ visible, int32_t *__restrict__ tiles,
                                            uint64_t *__restrict__ depth_keys, int32_t *__restrict__ err);
template <int DEG>
__device__ __forceinline__ void emit_view(const tgs_cloud &cl, int64_t i, const tgs_camera &cam, const tgs_settings &s,
                                          float *rest, float *splats, uint8_t *visible, int32_t *tiles,
                                          uint64_t *depth_keys, int32_t *err) {
  emit_view_impl<DEG>(cl, i, cam, s, rest, splats, visible, tiles, depth_keys, err);
}

template <int DEG>
__global__ void __launch_bounds__(kPreBlock) k_preprocess_fwd(tgs_cloud cl, tgs_camera cam, tgs_settings s,
                                                              float *__restrict__ splats,
                                                              uint8_t *__restrict__ visible,
                                                              int32_t *__restrict__ tiles,
                                                              uint64_t *__restrict__ depth_keys,
                                                              int32_t *__restrict__ err) {
  __shared__ __align__(16) float rest_s[kPreBlock * 45];
  const int64_t base = (int64_t)blockIdx.x * kPreBlock;
  const int count = (int)(cl.n - base < kPreBlock ? cl.n - base : kPreBlock);
  if (DEG > 0) stage_rest(cl.sh_rest, base, count, rest_s);
  __syncthreads();
  if ((int)threadIdx.x >= count) return;
  emit_view<DEG>(cl, base + threadIdx.x, cam, s, rest_s + 45 * threadIdx.x, splats, visible, tiles, depth_keys, err);
}

// Multi-view forward: one pass over the parameters for a batch of views (the
// sh_rest block staged once, the other fields re-read from L1); every view's
// outputs are bit-identical to k_preprocess_fwd's (same per-view routine).
constexpr int kMaxFwdViews = 8;
struct FwdViews {
  tgs_camera cam[kMaxFwdViews];
  float *splats[kMaxFwdViews];
  uint8_t *visible[kMaxFwdViews];
  int32_t *tiles[kMaxFwdViews];
  uint64_t *depth_keys[kMaxFwdViews];
  float *area_max;  // densification statistic (may be NULL)
  int nviews;
};

template <int DEG>
__global__ void __launch_bounds__(kPreBlock) k_preprocess_fwd_views(tgs_cloud cl, FwdViews fv, tgs_settings s,
                                                                    int32_t *__restrict__ err) {
  __shared__ __align__(16) float rest_s[kPreBlock * 45];
  __shared__ __align__(8) uint64_t rest_bar;
  const int64_t base = (int64_t)blockIdx.x * kPreBlock;
  const int count = (int)(cl.n - base < kPreBlock ? cl.n - base : kPreBlock);
  bool bulk = false;
  if (DEG > 0) {
    bulk = stage_rest_issue(cl.sh_rest, base, count, rest_s, &rest_bar);  // TMA, overlaps gauss_static
    if (!bulk) stage_rest(cl.sh_rest, base, count, rest_s);
  }
  __syncthreads();
  if ((int)threadIdx.x >= count) return;
  const int64_t i = base + threadIdx.x;
  GaussFwd f0;
  gauss_static(cl, i, s, f0);  // view-independent half once
  if (bulk) stage_rest_wait(&rest_bar);
  if (DEG > 0) premask_rest<DEG>(rest_s + 45 * threadIdx.x, f0);  // this thread's row, once
  float amax = -1.0f;
  for (int v = 0; v < fv.nviews; ++v) {
    GaussFwd f = f0;
    gauss_view<DEG>(cl, i, fv.cam[v], s, rest_s + 45 * threadIdx.x, f);
    emit_record(cl, i, fv.cam[v], s, f, fv.splats[v], fv.visible[v], fv.tiles[v], fv.depth_keys[v], err);
    if (f.visible) amax = fmaxf(amax, f.area);
  }
  // np.maximum(area_max, screen_areas) (training.py:338): culled rows have area 0
  if (fv.area_max && amax > fv.area_max[i]) fv.area_max[i] = amax;
}

// One Gaussian, one view: the projected record, visibility, tile count and depth key.
template <int DEG>
__device__ __forceinline__ void emit_view_impl(const tgs_cloud &cl, int64_t i, const tgs_camera &cam,
                                               const tgs_settings &s, float *rest, float *__restrict__ splats,
                                               uint8_t *__restrict__ visible, int32_t *__restrict__ tiles,
                                               uint64_t *__restrict__ depth_keys, int32_t *__restrict__ err) {
  GaussFwd f;
  gauss_forward<DEG>(cl, i, cam, s, rest, f);
  emit_record(cl, i, cam, s, f, splats, visible, tiles, depth_keys, err);
}

// Writes one view's outputs of Gaussian i from its forward quantities.
__device__ __forceinline__ void emit_record(const tgs_cloud &cl, int64_t i, const tgs_camera &cam,
                                            const tgs_settings &s, const GaussFwd &f, float *__restrict__ splats,
                                            uint8_t *__restrict__ visible, int32_t *__restrict__ tiles,
                                            uint64_t *__restrict__ depth_keys, int32_t *__restrict__ err) {
  if (f.degenerate) atomicOr(err, 1);
  float4 *o = reinterpret_cast<float4 *>(splats + 12 * i);
  int nt = 0;
  if (f.visible) {
    const float alpha = sem_sigmoidf(cl.opacity_logits[i]) * f.Mg;
    o[0] = make_float4(f.mean[0], f.mean[1], f.conic[0], f.conic[1]);
    o[1] = make_float4(f.conic[2], alpha, f.col[0], f.col[1]);
    o[2] = make_float4(f.col[2], f.t[2], f.radius, f.area);
    const int tiles_x = (cam.width + s.tile_size - 1) / s.tile_size;
    const int tiles_y = (cam.height + s.tile_size - 1) / s.tile_size;
    int x0, y0, x1, y1;
    nt = tile_rect(f.mean[0], f.mean[1], f.radius, cam.width, cam.height, s.tile_size, tiles_x, tiles_y, x0, y0,
                   x1, y1);
  } else {
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    o[0] = zero; o[1] = zero; o[2] = zero;
  }
  visible[i] = f.visible ? 1 : 0;
  tiles[i] = nt;
  if (depth_keys) {
    // float64 depth from the float32 inputs (no fma: -fmad=false), order-preserving bits
    const double d = f.visible ? (double)cl.positions[3 * i] * cam.depth_row[0] +
                                     (double)cl.positions[3 * i + 1] * cam.depth_row[1] +
                                     (double)cl.positions[3 * i + 2] * cam.depth_row[2] + cam.depth_row[3]
                               : 0.0;
    depth_keys[i] = orderable_key64(d);
  }
}

// Exact blend-decision records of a batch of views from their float32 records (a row
// with alpha 0 is not visible): the view-independent float64 state once per Gaussian.
struct ExactViews {
  tgs_camera cam[kMaxFwdViews];
  const float4 *splats[kMaxFwdViews];
  float4 *exact[kMaxFwdViews];
  int nviews;
};

__global__ void __launch_bounds__(kPreBlock) k_exact_views(tgs_cloud cl, ExactViews ev, tgs_settings s) {
  const int64_t i = (int64_t)blockIdx.x * kPreBlock + threadIdx.x;
  if (i >= cl.n) return;
  float al[kMaxFwdViews];  // every view's record alpha first (independent loads)
  bool any = false;
#pragma unroll
  for (int v = 0; v < kMaxFwdViews; ++v)
    if (v < ev.nviews) {
      al[v] = __ldg(reinterpret_cast<const float *>(ev.splats[v] + 3 * i + 1) + 1);
      any = any || al[v] > 0.0f;
    }
  Static64 g;
  if (any) gauss_static64(cl, i, cl.mask_logits[i] > s.mask_logit_min ? 1.0f : 0.0f, g);
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int v = 0; v < kMaxFwdViews; ++v)
    if (v < ev.nviews) {
      float4 *o = ev.exact[v] + 2 * i;
      if (al[v] > 0.0f) {
        exact_record(cl, i, ev.cam[v], s, g, __ldg(ev.splats[v] + 3 * i), __ldg(ev.splats[v] + 3 * i + 1), o);
      } else {
        o[0] = zero;
        o[1] = zero;
      }
    }
}

__global__ void k_count_tiles(const float *__restrict__ splats, int64_t n, int W, int H, int ts, int tiles_x,
                              int tiles_y, int32_t *__restrict__ tiles) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float *o = splats + 12 * i;
  int x0, y0, x1, y1;
  tiles[i] = tile_rect(o[0], o[1], o[10], W, H, ts, tiles_x, tiles_y, x0, y0, x1, y1);
}

}  // namespace tgs

using namespace tgs;

extern "C" int tgs_preprocess_forward(const tgs_cloud *cloud, const tgs_camera *cam, const tgs_settings *s,
                                      float *splats, uint8_t *visible, int32_t *tiles_touched,
                                      uint64_t *depth_keys, int32_t *error_flag, float *exact, tgs_stream_t stream) {
  if (!cloud || !cam || !s || cloud->n < 0) return TGS_ERR_INVALID;
  if (reinterpret_cast<uintptr_t>(exact) & 15) return TGS_ERR_INVALID;
  if (s->tile_size < 1 || s->tile_size > 32) return TGS_ERR_UNSUPPORTED;
  if (s->active_sh_degree < 0 || s->active_sh_degree > 3) return TGS_ERR_INVALID;
  if (cloud->n == 0) return TGS_OK;
  if (reinterpret_cast<uintptr_t>(splats) & 15) return TGS_ERR_INVALID;
  const unsigned grid = (unsigned)ceil_div<int64_t>(cloud->n, kPreBlock);
  cudaStream_t st = as_stream(stream);
  switch (s->active_sh_degree) {
#define TGS_FWD(D) \
  case D: k_preprocess_fwd<D><<<grid, kPreBlock, 0, st>>>(*cloud, *cam, *s, splats, visible, tiles_touched, depth_keys, error_flag); break;
    TGS_FWD(0) TGS_FWD(1) TGS_FWD(2) TGS_FWD(3)
#undef TGS_FWD
  }
  const int rc = launch_status();
  if (rc != TGS_OK || !exact) return rc;
  const float *sp = splats;
  return tgs_exact_records_views(cloud, cam, s, 1, &sp, &exact, stream);
}

extern "C" int tgs_preprocess_forward_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s,
                                            int32_t nviews, float *const *splats, uint8_t *const *visible,
                                            int32_t *const *tiles_touched, uint64_t *const *depth_keys,
                                            int32_t *error_flag, const tgs_densify_stats *stats,
                                            float *const *exact, tgs_stream_t stream) {
  if (!cloud || !cams || !s || cloud->n < 0 || nviews < 1 || !splats || !visible || !tiles_touched)
    return TGS_ERR_INVALID;
  if (s->tile_size < 1 || s->tile_size > 32) return TGS_ERR_UNSUPPORTED;
  if (s->active_sh_degree < 0 || s->active_sh_degree > 3) return TGS_ERR_INVALID;
  if (cloud->n == 0) return TGS_OK;
  for (int v = 0; v < nviews; ++v)
    if (!splats[v] || (reinterpret_cast<uintptr_t>(splats[v]) & 15) || !visible[v] || !tiles_touched[v] ||
        (exact && (!exact[v] || (reinterpret_cast<uintptr_t>(exact[v]) & 15))))
      return TGS_ERR_INVALID;
  const unsigned grid = (unsigned)ceil_div<int64_t>(cloud->n, kPreBlock);
  cudaStream_t st = as_stream(stream);
  for (int v0 = 0; v0 < nviews; v0 += kMaxFwdViews) {
    FwdViews fv;
    fv.nviews = nviews - v0 < kMaxFwdViews ? nviews - v0 : kMaxFwdViews;
    for (int k = 0; k < fv.nviews; ++k) {
      fv.cam[k] = cams[v0 + k];
      fv.splats[k] = splats[v0 + k];
      fv.visible[k] = visible[v0 + k];
      fv.tiles[k] = tiles_touched[v0 + k];
      fv.depth_keys[k] = depth_keys ? depth_keys[v0 + k] : nullptr;
    }
    fv.area_max = stats ? stats->area_max : nullptr;
    switch (s->active_sh_degree) {
#define TGS_FWDV(D) \
  case D: k_preprocess_fwd_views<D><<<grid, kPreBlock, 0, st>>>(*cloud, fv, *s, error_flag); break;
      TGS_FWDV(0) TGS_FWDV(1) TGS_FWDV(2) TGS_FWDV(3)
#undef TGS_FWDV
    }
  }
  const int rc = launch_status();
  if (rc != TGS_OK || !exact) return rc;
  return tgs_exact_records_views(cloud, cams, s, nviews, splats, exact, stream);
}

extern "C" int tgs_exact_records_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s,
                                       int32_t nviews, const float *const *splats, float *const *exact,
                                       tgs_stream_t stream) {
  if (!cloud || !cams || !s || cloud->n < 0 || nviews < 1 || !splats || !exact) return TGS_ERR_INVALID;
  if (cloud->n == 0) return TGS_OK;
  for (int v = 0; v < nviews; ++v)
    if (!splats[v] || !exact[v] || ((reinterpret_cast<uintptr_t>(splats[v]) | reinterpret_cast<uintptr_t>(exact[v])) & 15))
      return TGS_ERR_INVALID;
  const unsigned grid = (unsigned)ceil_div<int64_t>(cloud->n, kPreBlock);
  cudaStream_t st = as_stream(stream);
  for (int v0 = 0; v0 < nviews; v0 += kMaxFwdViews) {
    ExactViews ev;
    ev.nviews = nviews - v0 < kMaxFwdViews ? nviews - v0 : kMaxFwdViews;
    for (int k = 0; k < ev.nviews; ++k) {
      ev.cam[k] = cams[v0 + k];
      ev.splats[k] = reinterpret_cast<const float4 *>(splats[v0 + k]);
      ev.exact[k] = reinterpret_cast<float4 *>(exact[v0 + k]);
    }
    k_exact_views<<<grid, kPreBlock, 0, st>>>(*cloud, ev, *s);
  }
  return launch_status();
}

extern "C" int tgs_count_tiles(const float *splats, int64_t n, int32_t width, int32_t height, int32_t tile_size,
                               int32_t *tiles_touched, tgs_stream_t stream) {
  if (n < 0 || tile_size < 1 || width < 1 || height < 1) return TGS_ERR_INVALID;
  if (n == 0) return TGS_OK;
  const int tx = (width + tile_size - 1) / tile_size, ty = (height + tile_size - 1) / tile_size;
  k_count_tiles<<<(unsigned)ceil_div<int64_t>(n, 256), 256, 0, as_stream(stream)>>>(splats, n, width, height,
                                                                                     tile_size, tx, ty, tiles_touched);
  return launch_status();
}

