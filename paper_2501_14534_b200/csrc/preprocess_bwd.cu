// preprocess_bwd.cu — multi-view per-Gaussian backward (R9-R11).
//
// rasterizer.py:375-419 with sh.py:164-215, geometry.py:198-251,
// geometry.py:44-71,80-89 and masking.py:28-31.  Compiled WITH FMA
// contraction (unlike the bit-exact forward in preprocess.cu): the gradients
// only have to meet the north-star tolerance, and fused multiply-adds halve the
// instruction count of the per-view chains.  Divisions by the view distance and
// the camera depth become one reciprocal each.
#include "preprocess_common.cuh"

namespace tgs {

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
constexpr int kMaxViews = 8;
// 4 CTAs/SM: <= 128 registers (no spills) and 47.6 KB dynamic smem per CTA (the drest
// stage aliases the sh_rest stage); 3 CTAs/SM with separate stages measured 0.414 ms/step
// vs 0.371 on c3 (profiles/r02_ab_late.log)
#ifndef TGS_PB_MINB
#define TGS_PB_MINB 4
#endif

struct ViewBatch {
  tgs_camera cam[kMaxViews];
  const uint8_t *visible[kMaxViews];
  const float *dsplats[kMaxViews];
  float *grad_accum;    // densification statistics (may be NULL)
  int32_t *grad_count;
  int nviews;
  int clear;            // zero every view's partials after reading them (ready for the next step)
};

template <int DEG, bool kAcc>
__global__ void __launch_bounds__(kPreBlock, TGS_PB_MINB) k_preprocess_bwd_views(tgs_cloud cl, ViewBatch vb, tgs_settings s,
                                                                    tgs_grads g) {
  // dynamic shared memory: sh_rest stage (reused as the drest stage), and per view the view
  // direction and clamped colour upstream for the SH-rest gradient
  // sum_v basis(dir_v) (x) dcolor_v, accumulated in registers after the view loop
  extern __shared__ __align__(16) float pb_smem[];
  float *rest_s = pb_smem;
  // the drest stage overwrites the thread's own sh_rest row, entry by entry after its last
  // read (the d_band loop below), so one 45-float row per thread serves both
  float *drest_s = pb_smem;
  float(*vd_s)[6][kPreBlock] = reinterpret_cast<float(*)[6][kPreBlock]>(pb_smem + kPreBlock * 45);
  constexpr int K = (DEG + 1) * (DEG + 1) - 1;
  const int64_t base = (int64_t)blockIdx.x * kPreBlock;
  const int count = (int)(cl.n - base < kPreBlock ? cl.n - base : kPreBlock);
  const bool rest_grads = DEG > 0 && s.compute_sh_rest_grads;
  __shared__ __align__(8) uint64_t rest_bar;
  bool bulk = false;
  if (DEG > 0) {
    bulk = stage_rest_issue(cl.sh_rest, base, count, rest_s, &rest_bar);  // TMA, overlaps the loads below
    if (!bulk) stage_rest(cl.sh_rest, base, count, rest_s);
  }
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
    float st_norm = 0.f;  // densification statistics over this batch's views
    int st_count = 0;
    // every view's visibility first (independent byte loads, one latency), then the
    // partials one view ahead, loaded unconditionally: no load waits on another load
    // (a non-visible row's partials are never used, rasterizer.py:376-379)
    uint32_t vmask = 0u;
    for (int v = 0; v < vb.nviews; ++v) vmask |= (__ldg(vb.visible[v] + i) != 0 ? 1u : 0u) << v;
    float dn9[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) dn9[k] = __ldg(vb.dsplats[0] + 9 * i + k);
    if (bulk) stage_rest_wait(&rest_bar);  // the sh_rest block (TMA) is needed from here on
    for (int v = 0; v < vb.nviews; ++v) {
      const bool vis_v = (vmask >> v) & 1u;
      float d[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) d[k] = dn9[k];
      if (v + 1 < vb.nviews) {
#pragma unroll
        for (int k = 0; k < 9; ++k) dn9[k] = __ldg(vb.dsplats[v + 1] + 9 * i + k);
      }
      if (!vis_v) {  // non-visible: every partial is zero (rasterizer.py:376-379)
        if (rest_grads) {
#pragma unroll
          for (int k = 0; k < 6; ++k) vd_s[v][k][threadIdx.x] = k == 2 ? 1.0f : 0.0f;  // finite dir, zero colour
        }
        continue;
      }
      const tgs_camera &cam = vb.cam[v];
      const float dm0 = d[0], dm1 = d[1], g00 = d[2], g01 = d[3], g11 = d[4], da = d[5];
      const float dcol[3] = {d[6], d[7], d[8]};
      da_sum += da;
      m2d[0] += dm0;
      m2d[1] += dm1;
      if (vb.grad_accum) {  // ||mean2d_screen * (w/2, h/2)|| (training.py:334-337)
        const float sx = dm0 * (0.5f * (float)cam.width), sy = dm1 * (0.5f * (float)cam.height);
        st_norm += sqrtf(sx * sx + sy * sy);
        ++st_count;
      }
      // view direction + SH colour backward (sh.py:164-215)
      {
        const float e0 = px - cam.center[0], e1 = py - cam.center[1], e2 = pz - cam.center[2];
        const float nrm = sqrtf(e0 * e0 + e1 * e1 + e2 * e2);
        const float dn = nrm < 1e-12f ? 1e-12f : nrm;
        const float inv_dn = 1.0f / dn;
        const float dir[3] = {e0 * inv_dn, e1 * inv_dn, e2 * inv_dn};
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
        if (rest_grads) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            vd_s[v][k][threadIdx.x] = dir[k];
            vd_s[v][3 + k][threadIdx.x] = dcolor[k];
          }
        }
        if (DEG > 0) {
          float wk[15];
#pragma unroll
          for (int k = 0; k < 15; ++k) {
            wk[k] = 0.0f;
            if (k < K) {
              const float mb = band[band_of(k)];
#pragma unroll
              for (int c = 0; c < 3; ++c) wk[k] += my_rest[3 * k + c] * mb * dcolor[c];
            }
          }
          float d_dirs[3];
          sh_dir_grad<K>(dir[0], dir[1], dir[2], wk, d_dirs);
          const float inner = d_dirs[0] * dir[0] + d_dirs[1] * dir[1] + d_dirs[2] * dir[2];
#pragma unroll
          for (int k = 0; k < 3; ++k) gp[k] += (d_dirs[k] - dir[k] * inner) * inv_dn;
        }
      }
      // projection + project_backward (geometry.py:153-168, 198-251)
      {
        float t[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) t[r] = px * cam.R[3 * r] + py * cam.R[3 * r + 1] + pz * cam.R[3 * r + 2] + cam.t[r];
        const float tz = t[2], fx = cam.fx, fy = cam.fy;
        const float itz = 1.0f / tz, itz2 = itz * itz, itz3 = itz2 * itz;
        const float J00 = fx * itz, J02 = -fx * t[0] * itz2, J11 = fy * itz, J12 = -fy * t[1] * itz2;
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
        float dt0 = dJ[2] * (-fx * itz2);
        float dt1 = dJ[5] * (-fy * itz2);
        float dt2 = dJ[0] * (-fx * itz2) + dJ[4] * (-fy * itz2) + dJ[2] * (2.0f * fx * t[0] * itz3) +
                    dJ[5] * (2.0f * fy * t[1] * itz3);
        dt0 += dm0 * fx * itz;
        dt1 += dm1 * fy * itz;
        dt2 += -(dm0 * fx * t[0] + dm1 * fy * t[1]) * itz2;
#pragma unroll
        for (int j = 0; j < 3; ++j) gp[j] += dt0 * cam.R[j] + dt1 * cam.R[3 + j] + dt2 * cam.R[6 + j];
      }
    }
    // ---- SH-rest gradient: drest[k][c] = sum_v basis_k(dir_v) dcolor_v[c] (sh.py:202-214),
    // band-mask upstream d_band[l] = sum_{k in band l, c} drest[k][c] rest[k][c]
    if (rest_grads) {
      float dr[45];
#pragma unroll
      for (int k = 0; k < 45; ++k) dr[k] = 0.0f;
      for (int v = 0; v < vb.nviews; ++v) {
        float bsh[15];
        sh_basis_rest(vd_s[v][0][threadIdx.x], vd_s[v][1][threadIdx.x], vd_s[v][2][threadIdx.x], bsh);
        const float c0 = vd_s[v][3][threadIdx.x], c1 = vd_s[v][4][threadIdx.x], c2 = vd_s[v][5][threadIdx.x];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          dr[3 * k] += bsh[k] * c0;
          dr[3 * k + 1] += bsh[k] * c1;
          dr[3 * k + 2] += bsh[k] * c2;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float mb = band[band_of(k)];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          d_band[band_of(k)] += dr[3 * k + c] * my_rest[3 * k + c];
          my_drest[3 * k + c] = dr[3 * k + c] * mb;
        }
      }
      for (int k = 3 * K; k < 45; ++k) my_drest[k] = 0.0f;
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
    if (st_count) {
      vb.grad_accum[i] += st_norm;
      vb.grad_count[i] += st_count;
    }
  }
  // ---- sh_rest gradients: coalesced (read-modify-)write of the smem block
  if (rest_grads || !kAcc) {
    __syncthreads();
    float *dst = g.sh_rest + base * 45;
    const int total = count * 45;
    for (int j = threadIdx.x; j < total; j += blockDim.x) put<kAcc>(dst + j, rest_grads ? drest_s[j] : 0.0f);
  }
  // ---- the consumer clears: every view's partial rows of this CTA back to zero, so the
  // next step's blend backward can accumulate into them without a separate fill launch
  // (coalesced float4 stores over the CTA's contiguous 36 B rows)
  if (vb.clear) {
    __syncthreads();  // every thread has read its rows of every view
    const int total = count * 9;
    for (int v = 0; v < vb.nviews; ++v) {
      float *dst = const_cast<float *>(vb.dsplats[v]) + base * 9;  // base * 36 B: 16 B aligned
      for (int j = 4 * (int)threadIdx.x; j < total; j += 4 * kPreBlock) {
        if (j + 4 <= total) {
          *reinterpret_cast<float4 *>(dst + j) = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          for (int k = j; k < total; ++k) dst[k] = 0.0f;
        }
      }
    }
  }
}

}  // namespace tgs

using namespace tgs;

constexpr int kPbSmem = (kPreBlock * 45 + kMaxViews * 6 * kPreBlock) * (int)sizeof(float);

static int launch_bwd_views(const tgs_cloud *cloud, const ViewBatch &vb, const tgs_settings *s, tgs_grads *grads,
                            bool accumulate, cudaStream_t st) {
  const unsigned grid = (unsigned)ceil_div<int64_t>(cloud->n, kPreBlock);
  switch (s->active_sh_degree * 2 + (accumulate ? 1 : 0)) {
#define TGS_BWD(D, A)                                                                                          \
  case D * 2 + A: {                                                                                            \
    static std::atomic<uint64_t> attr{0}; /* per device: function attributes are per device */               \
    const int arc = attr_once_per_device(attr, [] {                                                            \
      return cudaFuncSetAttribute(k_preprocess_bwd_views<D, A>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                  kPbSmem);                                                                    \
    });                                                                                                        \
    if (arc != TGS_OK) return arc;                                                                             \
    k_preprocess_bwd_views<D, A><<<grid, kPreBlock, kPbSmem, st>>>(*cloud, vb, *s, *grads);                    \
  } break;
    TGS_BWD(0, 0) TGS_BWD(0, 1) TGS_BWD(1, 0) TGS_BWD(1, 1) TGS_BWD(2, 0) TGS_BWD(2, 1) TGS_BWD(3, 0) TGS_BWD(3, 1)
#undef TGS_BWD
  }
  return launch_status();
}

extern "C" int tgs_preprocess_backward(const tgs_cloud *cloud, const tgs_camera *cam, const tgs_settings *s,
                                       const uint8_t *visible, const float *dsplats, tgs_grads *grads,
                                       int32_t accumulate, tgs_stream_t stream) {
  return tgs_preprocess_backward_views(cloud, cam, s, &visible, &dsplats, 1, grads, accumulate, nullptr, 0, stream);
}

extern "C" int tgs_preprocess_backward_views(const tgs_cloud *cloud, const tgs_camera *cams, const tgs_settings *s,
                                             const uint8_t *const *visible, const float *const *dsplats,
                                             int32_t nviews, tgs_grads *grads, int32_t accumulate,
                                             const tgs_densify_stats *stats, int32_t clear_partials,
                                             tgs_stream_t stream) {
  if (!cloud || !cams || !s || !grads || !visible || !dsplats || cloud->n < 0 || nviews < 1) return TGS_ERR_INVALID;
  if (clear_partials)
    for (int v = 0; v < nviews; ++v)
      if (reinterpret_cast<uintptr_t>(dsplats[v]) & 15) return TGS_ERR_INVALID;  // float4 clears
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
    vb.grad_accum = stats && stats->grad_count ? stats->grad_accum : nullptr;
    vb.grad_count = vb.grad_accum ? stats->grad_count : nullptr;
    vb.clear = clear_partials != 0;
    const int rc = launch_bwd_views(cloud, vb, s, grads, accumulate || v0 > 0, st);
    if (rc != TGS_OK) return rc;
  }
  return TGS_OK;
}
