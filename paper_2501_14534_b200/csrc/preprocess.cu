// preprocess.cu — per-Gaussian forward (R1-R4) and backward (R9-R11) kernels.
//
// Compiled with -fmad=false: together with tgs_math.cuh this pins every float
// operation to the documented order so visibility, radii and tile counts are
// bit-identical to the float32 oracle.
//
// Forward  : masking.py:21-43,84-86 (hard masks), geometry.py:19-41,74-77
//            (quaternion -> R -> Sigma), geometry.py:138-195 (EWA projection),
//            rasterizer.py:177-197 (alpha-skip, view dirs, SH colour),
//            sh.py:135-161, rasterizer.py:112-128 (tile rect/count).
// Backward : rasterizer.py:375-419 with sh.py:164-215, geometry.py:198-251,
//            geometry.py:44-71,80-89 and masking.py:28-31.
//
// Both kernels are HBM-bound streaming kernels, one thread per Gaussian.  The
// 180 B/Gaussian sh_rest block is staged through shared memory with 16 B
// coalesced loads/stores (a per-thread 45-float stride would split every warp
// access over 45 lines).
#include "tgs_common.cuh"
#include "tgs_math.cuh"

namespace tgs {

constexpr int kPreBlock = 128;

__device__ __forceinline__ float max0(float v) { return v < 0.0f ? 0.0f : v; }

struct GaussFwd {
  float Mg, band[3];
  bool alpha_ok, valid, ok, visible, degenerate;
  float s_raw[3], sc[3];
  float qn[4], qnorm;
  float Rg[9], S[9];
  float t[3], Mj[6];
  float mean[2], c00, c01, c11, det, conic[3], radius, area;
  float dir[3], dnorm;
  float pre[3], col[3];
};

// Loads the rest block of `count` Gaussians starting at `base` into smem.
__device__ __forceinline__ void stage_rest(const float *__restrict__ rest, int64_t base, int count, float *sm) {
  const float *src = rest + base * 45;
  const int total = count * 45;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int n4 = total / 4;
    for (int j = threadIdx.x; j < n4; j += blockDim.x)
      reinterpret_cast<float4 *>(sm)[j] = __ldg(reinterpret_cast<const float4 *>(src) + j);
    for (int j = n4 * 4 + threadIdx.x; j < total; j += blockDim.x) sm[j] = __ldg(src + j);
  } else {
    for (int j = threadIdx.x; j < total; j += blockDim.x) sm[j] = __ldg(src + j);
  }
}

// Forward quantities of Gaussian i in the documented float32 order.  `rest`
// points at this Gaussian's 45 staged coefficients (may be null when degree 0).
template <int DEG>
__device__ __forceinline__ void gauss_forward(const tgs_cloud &cl, int64_t i, const tgs_camera &cam,
                                              const tgs_settings &s, const float *rest, GaussFwd &f) {
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
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < K; ++k) acc = acc + b[k] * (rest[3 * k + c] * f.band[band_of(k)]);
    float col = SH_C0 * cl.sh_dc[3 * i + c] + 0.5f;
    if (DEG > 0) col = col + acc;
    f.pre[c] = col;
    f.col[c] = max0(col);
  }
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
  const int64_t i = base + threadIdx.x;
  GaussFwd f;
  gauss_forward<DEG>(cl, i, cam, s, rest_s + 45 * threadIdx.x, f);
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

__global__ void k_count_tiles(const float *__restrict__ splats, int64_t n, int W, int H, int ts, int tiles_x,
                              int tiles_y, int32_t *__restrict__ tiles) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float *o = splats + 12 * i;
  int x0, y0, x1, y1;
  tiles[i] = tile_rect(o[0], o[1], o[10], W, H, ts, tiles_x, tiles_y, x0, y0, x1, y1);
}

template <bool kAcc>
__device__ __forceinline__ void put(float *p, float v) {
  if (kAcc) *p += v; else *p = v;
}

// ---------------------------------------------------------------------------
// Multi-view backward.  Every chain after the screen-space partials is LINEAR in
// them, so for a batch of views the view-dependent parts (projection Jacobian,
// view direction, SH basis, clamp mask) run per view and their contributions
// are summed, while the view-independent chains (covariance -> quaternion /
// log-scale, opacity and mask sigmoids, sh_dc) run once on the summed upstream:
// the parameters are read once per step instead of once per view.  The sum of
// per-view reference gradients (rasterizer.py:375-419) up to float reassociation.
// unit quaternion -> rotation (geometry.py:19-41); returns the raw norm
__device__ __forceinline__ float quat_rot(const tgs_cloud &cl, int64_t i, float Rg[9], float qn[4] = nullptr) {
  const float qw = cl.rotations[4 * i], qx = cl.rotations[4 * i + 1];
  const float qy = cl.rotations[4 * i + 2], qz = cl.rotations[4 * i + 3];
  const float qnorm = sqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
  const float w = qw / qnorm, x = qx / qnorm, y = qy / qnorm, z = qz / qnorm;
  if (qn) {
    qn[0] = w; qn[1] = x; qn[2] = y; qn[3] = z;
  }
  Rg[0] = 1.0f - 2.0f * (y * y + z * z);
  Rg[1] = 2.0f * (x * y - w * z);
  Rg[2] = 2.0f * (x * z + w * y);
  Rg[3] = 2.0f * (x * y + w * z);
  Rg[4] = 1.0f - 2.0f * (x * x + z * z);
  Rg[5] = 2.0f * (y * z - w * x);
  Rg[6] = 2.0f * (x * z - w * y);
  Rg[7] = 2.0f * (y * z + w * x);
  Rg[8] = 1.0f - 2.0f * (x * x + y * y);
  return qnorm;
}

constexpr int kMaxViews = 8;

struct ViewBatch {
  tgs_camera cam[kMaxViews];
  const uint8_t *visible[kMaxViews];
  const float *dsplats[kMaxViews];
  int nviews;
};

template <int DEG, bool kAcc>
__global__ void __launch_bounds__(kPreBlock, 3) k_preprocess_bwd_views(tgs_cloud cl, ViewBatch vb, tgs_settings s,
                                                                    tgs_grads g) {
  __shared__ __align__(16) float rest_s[kPreBlock * 45];
  __shared__ __align__(16) float drest_s[kPreBlock * 45];
  constexpr int K = (DEG + 1) * (DEG + 1) - 1;
  const int64_t base = (int64_t)blockIdx.x * kPreBlock;
  const int count = (int)(cl.n - base < kPreBlock ? cl.n - base : kPreBlock);
  const bool rest_grads = DEG > 0 && s.compute_sh_rest_grads;
  if (DEG > 0) stage_rest(cl.sh_rest, base, count, rest_s);
  for (int j = threadIdx.x; j < kPreBlock * 45; j += kPreBlock) drest_s[j] = 0.0f;
  __syncthreads();
  const int64_t i = base + threadIdx.x;
  const bool live = (int)threadIdx.x < count;
  const float *my_rest = rest_s + 45 * threadIdx.x;
  float *my_drest = drest_s + 45 * threadIdx.x;
  if (live) {
    // ---- view-independent state needed inside the view loop: masks and Sigma (6 unique)
    const float m = cl.mask_logits[i], o = cl.opacity_logits[i];
    const float Mg = (m > s.mask_logit_min) ? 1.0f : 0.0f;
    float band[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) band[l] = (cl.sh_mask_logits[3 * i + l] > s.sh_mask_logit_min) ? 1.0f : 0.0f;
    float S6[6];  // S00 S01 S02 S11 S12 S22
    {
      float Rg[9], sc[3];
      quat_rot(cl, i, Rg);
#pragma unroll
      for (int k = 0; k < 3; ++k) sc[k] = sem_expf(cl.log_scales[3 * i + k]) * Mg;
      float L[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) L[3 * r + k] = Rg[3 * r + k] * sc[k];
      int e = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) S6[e++] = L[3 * a] * L[3 * b] + L[3 * a + 1] * L[3 * b + 1] + L[3 * a + 2] * L[3 * b + 2];
    }
    const float px = cl.positions[3 * i], py = cl.positions[3 * i + 1], pz = cl.positions[3 * i + 2];
    // ---- accumulators over views (dS symmetric: 6 unique entries)
    float gp[3] = {0.f, 0.f, 0.f}, dS6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float da_sum = 0.f, dc_sum[3] = {0.f, 0.f, 0.f}, d_band[3] = {0.f, 0.f, 0.f}, m2d[2] = {0.f, 0.f};
    for (int v = 0; v < vb.nviews; ++v) {
      if (!vb.visible[v][i]) continue;  // non-visible: every partial is zero (rasterizer.py:376-379)
      const tgs_camera &cam = vb.cam[v];
      const float *d = vb.dsplats[v] + 9 * i;
      const float dm0 = d[0], dm1 = d[1], g00 = d[2], g01 = d[3], g11 = d[4], da = d[5];
      const float dcol[3] = {d[6], d[7], d[8]};
      da_sum += da;
      m2d[0] += dm0;
      m2d[1] += dm1;
      // view direction + SH colour backward (sh.py:164-215)
      {
        const float e0 = px - cam.center[0], e1 = py - cam.center[1], e2 = pz - cam.center[2];
        const float nrm = sqrtf(e0 * e0 + e1 * e1 + e2 * e2);
        const float dn = nrm < 1e-12f ? 1e-12f : nrm;
        const float dir[3] = {e0 / dn, e1 / dn, e2 / dn};
        float bsh[15];
        sh_basis_rest(dir[0], dir[1], dir[2], bsh);
        float dcolor[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float acc = 0.0f;
#pragma unroll
          for (int k = 0; k < K; ++k) acc = acc + bsh[k] * (my_rest[3 * k + c] * band[band_of(k)]);
          float pre = SH_C0 * cl.sh_dc[3 * i + c] + 0.5f;
          if (DEG > 0) pre = pre + acc;
          dcolor[c] = pre > 0.0f ? dcol[c] : 0.0f;
          dc_sum[c] += dcolor[c];
        }
        if (DEG > 0) {
          float wk[15];
#pragma unroll
          for (int k = 0; k < 15; ++k) {
            wk[k] = 0.0f;
            if (k < K) {
              const float mb = band[band_of(k)];
              float pc = 0.0f;
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                wk[k] += my_rest[3 * k + c] * mb * dcolor[c];
                if (rest_grads) {
                  const float dmk = bsh[k] * dcolor[c];
                  pc += dmk * my_rest[3 * k + c];
                  my_drest[3 * k + c] += dmk * mb;
                }
              }
              if (rest_grads) d_band[band_of(k)] += pc;
            }
          }
          float d_dirs[3];
          sh_dir_grad<K>(dir[0], dir[1], dir[2], wk, d_dirs);
          const float inner = d_dirs[0] * dir[0] + d_dirs[1] * dir[1] + d_dirs[2] * dir[2];
#pragma unroll
          for (int k = 0; k < 3; ++k) gp[k] += (d_dirs[k] - dir[k] * inner) / dn;
        }
      }
      // projection + project_backward (geometry.py:153-168, 198-251)
      {
        float t[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) t[r] = px * cam.R[3 * r] + py * cam.R[3 * r + 1] + pz * cam.R[3 * r + 2] + cam.t[r];
        const float tz = t[2], fx = cam.fx, fy = cam.fy;
        const float tz2 = tz * tz, tz3 = tz2 * tz;
        const float J00 = fx / tz, J02 = -fx * t[0] / tz2, J11 = fy / tz, J12 = -fy * t[1] / tz2;
        float Mj[6];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          Mj[j] = J00 * cam.R[j] + J02 * cam.R[6 + j];
          Mj[3 + j] = J11 * cam.R[3 + j] + J12 * cam.R[6 + j];
        }
        const float G0 = g00, G1 = 0.5f * g01, G3 = g11;
        // dS += M^T G M (symmetric)
        float MtG0[3], MtG1[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          MtG0[a] = Mj[a] * G0 + Mj[3 + a] * G1;
          MtG1[a] = Mj[a] * G1 + Mj[3 + a] * G3;
        }
        {
          int e = 0;
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = a; b < 3; ++b) dS6[e++] += MtG0[a] * Mj[b] + MtG1[a] * Mj[3 + b];
        }
        // dM = 2 (G M) Sigma, dJ = dM Rc^T
        auto Sg = [&](int a, int b) -> float {
          const int lo = a < b ? a : b, hi = a < b ? b : a;
          return S6[lo == 0 ? hi : (lo == 1 ? 2 + hi : 5)];
        };
        float dM[6], dJ[6];
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const float ga = a == 0 ? G0 : G1, gb = a == 0 ? G1 : G3;
          float GM[3];
#pragma unroll
          for (int b = 0; b < 3; ++b) GM[b] = ga * Mj[b] + gb * Mj[3 + b];
#pragma unroll
          for (int b = 0; b < 3; ++b) dM[3 * a + b] = 2.0f * (GM[0] * Sg(0, b) + GM[1] * Sg(1, b) + GM[2] * Sg(2, b));
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            dJ[3 * a + b] = dM[3 * a] * cam.R[3 * b] + dM[3 * a + 1] * cam.R[3 * b + 1] + dM[3 * a + 2] * cam.R[3 * b + 2];
        float dt0 = dJ[2] * (-fx / tz2);
        float dt1 = dJ[5] * (-fy / tz2);
        float dt2 = dJ[0] * (-fx / tz2) + dJ[4] * (-fy / tz2) + dJ[2] * (2.0f * fx * t[0] / tz3) +
                    dJ[5] * (2.0f * fy * t[1] / tz3);
        dt0 += dm0 * fx / tz;
        dt1 += dm1 * fy / tz;
        dt2 += -(dm0 * fx * t[0] + dm1 * fy * t[1]) / tz2;
#pragma unroll
        for (int j = 0; j < 3; ++j) gp[j] += dt0 * cam.R[j] + dt1 * cam.R[3 + j] + dt2 * cam.R[6 + j];
      }
    }
    // ---- view-independent state again (recomputed rather than kept live across the loop)
    float s_raw[3], sc[3], Rg[9], L[9], qn[4], qnorm;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      s_raw[k] = sem_expf(cl.log_scales[3 * i + k]);
      sc[k] = s_raw[k] * Mg;
    }
    qnorm = quat_rot(cl, i, Rg, qn);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k) L[3 * r + k] = Rg[3 * r + k] * sc[k];
    const float w = qn[0], x = qn[1], y = qn[2], z = qn[3];
    float dS[9];
    {
      int e = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) {
          dS[3 * a + b] = dS6[e];
          dS[3 * b + a] = dS6[e];
          ++e;
        }
    }
    // ---- view-independent chains on the summed upstream
    const float s_op = sem_sigmoidf(o);
    const float o_op = da_sum * Mg * s_op * (1.0f - s_op);
    float dmask = da_sum * s_op;
    float dL[9], dsc[3], dR[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < 3; ++k) acc += (dS[3 * a + k] + dS[3 * k + a]) * L[3 * k + b];
        dL[3 * a + b] = acc;
      }
#pragma unroll
    for (int k = 0; k < 3; ++k) dsc[k] = dL[k] * Rg[k] + dL[3 + k] * Rg[3 + k] + dL[6 + k] * Rg[6 + k];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k) dR[3 * r + k] = dL[3 * r + k] * sc[k];
    float dqu[4];
    dqu[0] = 2.0f * (x * (dR[7] - dR[5]) + y * (dR[2] - dR[6]) + z * (dR[3] - dR[1]));
    dqu[1] = 2.0f * (y * (dR[1] + dR[3]) + z * (dR[2] + dR[6])) + 2.0f * w * (dR[7] - dR[5]) - 4.0f * x * (dR[4] + dR[8]);
    dqu[2] = 2.0f * (x * (dR[1] + dR[3]) + z * (dR[5] + dR[7])) + 2.0f * w * (dR[2] - dR[6]) - 4.0f * y * (dR[0] + dR[8]);
    dqu[3] = 2.0f * (x * (dR[2] + dR[6]) + y * (dR[5] + dR[7])) + 2.0f * w * (dR[3] - dR[1]) - 4.0f * z * (dR[0] + dR[4]);
    const float qin = dqu[0] * w + dqu[1] * x + dqu[2] * y + dqu[3] * z;
    float o_rot[4], o_ls[3], o_dc[3], o_shm[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) o_rot[k] = (dqu[k] - qn[k] * qin) / qnorm;
#pragma unroll
    for (int k = 0; k < 3; ++k) o_ls[k] = dsc[k] * s_raw[k] * Mg;
    dmask += dsc[0] * s_raw[0] + dsc[1] * s_raw[1] + dsc[2] * s_raw[2];
    const float smk = sem_sigmoidf(m);
    float o_mask = dmask * (smk * (1.0f - smk));
#pragma unroll
    for (int c = 0; c < 3; ++c) o_dc[c] = SH_C0 * dc_sum[c];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const float sg = sem_sigmoidf(cl.sh_mask_logits[3 * i + l]);
      o_shm[l] = d_band[l] * (sg * (1.0f - sg));
    }
    const bool w_shm = rest_grads || !kAcc;
    float o_pos[3] = {gp[0], gp[1], gp[2]}, o_op2 = o_op;
    float o_m2d[2] = {m2d[0], m2d[1]};
    if (kAcc) {  // independent loads first, then the adds
      float p_dc[3], p_shm[3] = {0.f, 0.f, 0.f}, p_pos[3], p_ls[3], p_rot[4], p_m2d[2] = {0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        p_dc[k] = g.sh_dc[3 * i + k];
        p_pos[k] = g.positions[3 * i + k];
        p_ls[k] = g.log_scales[3 * i + k];
        if (w_shm) p_shm[k] = g.sh_mask_logits[3 * i + k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) p_rot[k] = g.rotations[4 * i + k];
      const float p_op = g.opacity_logits[i], p_mask = g.mask_logits[i];
      if (g.mean2d_screen) {
        p_m2d[0] = g.mean2d_screen[2 * i];
        p_m2d[1] = g.mean2d_screen[2 * i + 1];
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        o_dc[k] += p_dc[k];
        o_pos[k] += p_pos[k];
        o_ls[k] += p_ls[k];
        o_shm[k] += p_shm[k];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) o_rot[k] += p_rot[k];
      o_op2 += p_op;
      o_mask += p_mask;
      o_m2d[0] += p_m2d[0];
      o_m2d[1] += p_m2d[1];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      g.sh_dc[3 * i + k] = o_dc[k];
      g.positions[3 * i + k] = o_pos[k];
      g.log_scales[3 * i + k] = o_ls[k];
      if (w_shm) g.sh_mask_logits[3 * i + k] = o_shm[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) g.rotations[4 * i + k] = o_rot[k];
    g.opacity_logits[i] = o_op2;
    g.mask_logits[i] = o_mask;
    if (g.mean2d_screen) {
      g.mean2d_screen[2 * i] = o_m2d[0];
      g.mean2d_screen[2 * i + 1] = o_m2d[1];
    }
  }
  // ---- sh_rest gradients: coalesced (read-modify-)write of the smem block
  if (rest_grads || !kAcc) {
    __syncthreads();
    float *dst = g.sh_rest + base * 45;
    const int total = count * 45;
    for (int j = threadIdx.x; j < total; j += blockDim.x) put<kAcc>(dst + j, drest_s[j]);
  }
}

}  // namespace tgs

using namespace tgs;

extern "C" int tgs_preprocess_forward(const tgs_cloud *cloud, const tgs_camera *cam, const tgs_settings *s,
                                      float *splats, uint8_t *visible, int32_t *tiles_touched,
                                      uint64_t *depth_keys, int32_t *error_flag, tgs_stream_t stream) {
  if (!cloud || !cam || !s || cloud->n < 0) return TGS_ERR_INVALID;
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

static int launch_bwd_views(const tgs_cloud *cloud, const ViewBatch &vb, const tgs_settings *s, tgs_grads *grads,
                            bool accumulate, cudaStream_t st) {
  const unsigned grid = (unsigned)ceil_div<int64_t>(cloud->n, kPreBlock);
  switch (s->active_sh_degree * 2 + (accumulate ? 1 : 0)) {
#define TGS_BWD(D, A) \
  case D * 2 + A: k_preprocess_bwd_views<D, A><<<grid, kPreBlock, 0, st>>>(*cloud, vb, *s, *grads); break;
    TGS_BWD(0, 0) TGS_BWD(0, 1) TGS_BWD(1, 0) TGS_BWD(1, 1) TGS_BWD(2, 0) TGS_BWD(2, 1) TGS_BWD(3, 0) TGS_BWD(3, 1)
#undef TGS_BWD
  }
  return launch_status();
}

extern "C" int tgs_preprocess_backward(const tgs_cloud *cloud, const tgs_camera *cam, const tgs_settings *s,
                                       const uint8_t *visible, const float *dsplats, tgs_grads *grads,
                                       int32_t accumulate, tgs_stream_t stream) {
  return tgs_preprocess_backward_views(cloud, cam, s, &visible, &dsplats, 1, grads, accumulate, stream);
}

extern "C" int tgs_preprocess_backward_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s,
                                             const uint8_t *const *visible, const float *const *dsplats,
                                             int32_t nviews, tgs_grads *grads, int32_t accumulate,
                                             tgs_stream_t stream) {
  if (!cloud || !cams || !s || !grads || !visible || !dsplats || cloud->n < 0 || nviews < 1) return TGS_ERR_INVALID;
  if (s->active_sh_degree < 0 || s->active_sh_degree > 3) return TGS_ERR_INVALID;
  if (cloud->n == 0) return TGS_OK;
  cudaStream_t st = as_stream(stream);
  for (int v0 = 0; v0 < nviews; v0 += kMaxViews) {
    ViewBatch vb;
    vb.nviews = nviews - v0 < kMaxViews ? nviews - v0 : kMaxViews;
    for (int k = 0; k < vb.nviews; ++k) {
      vb.cam[k] = cams[v0 + k];
      vb.visible[k] = visible[v0 + k];
      vb.dsplats[k] = dsplats[v0 + k];
    }
    const int rc = launch_bwd_views(cloud, vb, s, grads, accumulate || v0 > 0, st);
    if (rc != TGS_OK) return rc;
  }
  return TGS_OK;
}
