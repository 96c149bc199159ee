// blend.cu — per-tile alpha blending forward (R6) and backward (R7).
//
// Reference semantics (must match exactly):
//   forward  _kernels.py:38-89  — per pixel over the tile's depth-sorted list:
//            break when T < 1e-4 (checked BEFORE each entry, so the entry that
//            drives T below the threshold is still blended); e = -1/2(a dx^2 +
//            c dy^2) - b dx dy, skip e < -4.5 or e > 0; a = alpha * exp(e), skip
//            a < 1/255, clamp 0.99; C += c a T; T *= 1 - a; image = C + bg T;
//            last_pos = list position after the last blended entry.
//   backward _kernels.py:125-181 — per pixel back to front from last_pos,
//            T_before = T_after / (1 - a), suffix colour S seeded with bg*T_final;
//            the alpha/mean/cov partials only when a_raw <= 0.99.
//
// B200 mapping: one CTA per 16x16 tile (one thread per pixel), Gaussians staged
// through shared memory in batches of up to 256 records (48 B each, three
// 16 B loads).  The forward CTA leaves as soon as every pixel has terminated
// (__syncthreads_count).  The backward keeps the reference's per-pixel
// recurrence but accumulates per SPLAT: each staged Gaussian's 9 partials are
// reduced across the warp with shuffles (skipped when no lane of the warp
// touched it), combined across the CTA's warps in shared memory, and written
// with ONE global atomic per (tile, Gaussian, field) — no per-pixel global
// atomics.
//
// The exponent is evaluated by exponent2() (log2 units, pre-scaled conic) with
// explicit round-to-nearest intrinsics in every kernel, so the backward re-derives
// the forward's blend decisions bit for bit (a mismatch would corrupt the
// T_before = T_after / (1 - a) recovery).
#include "tgs_common.cuh"
#include "tgs_math.cuh"

// Register caps of the exact-decision instantiations (minimum resident CTAs per SM): the
// float64 resolution is out of line and rare, and without a cap its call would lower the
// occupancy of the whole kernel (uncapped 96 registers in the forward; capped at 6 CTAs
// per SM: 80, no spills).  The backward's cap is per 2-warp CTA of k_blend_bwd16p:
// MINB x pairs CTAs (4 x 2 = 8: <= 128 registers).  Measured at c3
// (profiles/scripts/r02_run8.sh, r02_run11.sh).
// Overridable with -D for A/B builds (profiles/scripts/build_blend_variants.sh).
#ifndef TGS_BWD16_PAIRS  // pixel pairs per lane of the 16x16 backward: 1 (k_blend_bwd16w) or 2
#define TGS_BWD16_PAIRS 2
#endif
#ifndef TGS_FWD16_MINB
#define TGS_FWD16_MINB 6
#endif
#ifndef TGS_BWD16_MINB
#define TGS_BWD16_MINB 4
#endif

namespace tgs {

constexpr int kBatch = 256;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr float kLog2e = 1.44269504088896341f;
constexpr float kE2Min = (float)(-4.5 * 1.44269504088896341);  // the e >= -4.5 cut in log2 units
constexpr float kClampAlpha = 0.9899f;  // float32 alpha above which alpha exp(e) can reach 0.99

// Pre-scaled conic (A, B, C, alpha) with A = -a log2(e) / 2, B = -b log2(e),
// C = -c log2(e) / 2, so e2 = A dx^2 + B dx dy + C dy^2 = e log2(e) and
// exp(e) = ex2(e2).  Every blend kernel evaluates the exponent with exactly this
// sequence, so the backward and the records kernel re-derive the forward's
// blend decisions bit for bit.
__device__ __forceinline__ float4 prescaled_conic(float4 a, float4 b) {
  return make_float4(__fmul_rn(a.z, -0.5f * kLog2e), __fmul_rn(a.w, -kLog2e), __fmul_rn(b.x, -0.5f * kLog2e), b.y);
}

__device__ __forceinline__ float exponent2(float4 q, float dx, float dy) {
  const float s = __fmaf_rn(__fmul_rn(q.z, dy), dy, __fmul_rn(__fmul_rn(q.x, dx), dx));
  return __fmaf_rn(__fmul_rn(q.y, dx), dy, s);
}

// Pixel owned by thread t of a tile.  For 16x16 tiles each warp owns an 8x4
// pixel block (compact footprints: a splat touches fewer warps than with 16x2
// rows); other tile sizes use row-major order.
__device__ __forceinline__ void pixel_of(int t, int ts, int &lx, int &ly) {
  if (ts == 16) {
    const int w = t >> 5, l = t & 31;
    lx = ((w & 1) << 3) | (l & 7);
    ly = ((w >> 1) << 2) | (l >> 3);
  } else {
    lx = t % ts;
    ly = t / ts;
  }
}

// Exact per-warp cull.  The staged splat can blend into a pixel only if
// e2(d) = A dx^2 + B dx dy + C dy^2 >= thr2 = -min(4.5, ln(255 alpha)) log2(e)
// (e >= -4.5 and alpha exp(e) >= 1/255).  e2 is a concave quadratic, so its maximum
// over the warp's pixel rectangle is 0 if the mean lies inside, else the best of
// the four edge maxima (1-D concave quadratics, vertex clamped to the edge).  The
// threshold is the lower end of the blend-cut bracket (load_cut below) minus a 0.02
// (log2 units) margin that keeps the test conservative under float32 rounding, so
// culling never changes a result.

// ---- blend decisions (include/tgs.h TGS_EXACT_FLOATS) ---------------------------------
// A (pixel, splat) pair blends iff e >= cut = max(-4.5, ln(1/(255 alpha))) and e <= 0
// (_kernels.py:59-72); in log2 units e2 = e log2(e).  With exact records the float64 cut
// is bracketed by [cut.x, cut.y]: e2 >= cut.y blends in float64 as well, e2 < cut.x does
// not, and the rare pairs in between are decided by exact_pair() in float64.  Without
// records cut.x == cut.y is the float32 cut.  The reference's e > 0 test cannot fire for
// a positive-definite conic (e = -v'Kv/2 <= 0; float64 rounding cannot flip its sign
// below a condition number of ~1e16), so the float32 path does not test e2 > 0 (rounding
// can make e2 a few ulps positive next to the mean; the reference blends those pixels).
// Every blend kernel decides through these functions, so the backward re-derives the
// forward's decisions exactly.
__device__ __forceinline__ float2 load_cut(const float4 *__restrict__ exact, int g, float alpha) {
  if (exact) return __ldg(reinterpret_cast<const float2 *>(exact + 2 * (int64_t)g));
  const float c = fmaxf(kE2Min, -__log2f(255.0f * alpha));
  return make_float2(c, c);
}

// The reference's float64 decision for one pair (_kernels.py:59-72): the float64 means and
// conic rebuilt as float32 record + residual, e = -(a dx^2 + c dy^2)/2 - b dx dy in the
// reference's operation order (no contraction), compared with the float64 cut (record
// slot 7 holds cut - cut_lo in log2 units).  A Gaussian whose alpha can reach the 0.99
// clamp (cut_hi = +inf) has cut = -4.5 exactly (alpha > 0.9899 puts ln(1/(255 alpha))
// below -4.5) and slot 7 holds ln(0.99 / alpha): alpha exp(e) <= 0.99 <=> e <= slot 7.
// Bit 0: blends; bit 1: alpha <= 0.99, the backward's partials through alpha apply
// (_kernels.py:157-168).  The cold path of the blend kernels: ~25 float64 operations.
#ifdef TGS_COUNT_EXACT
__device__ unsigned long long g_exact_pairs;  // profiling build only (profiles/exact_pairs.py)
#endif
__device__ __forceinline__ int exact_pair(const float4 *__restrict__ splats, const float4 *__restrict__ exact, int g,
                                          float px, float py) {
#ifdef TGS_COUNT_EXACT
  atomicAdd(&g_exact_pairs, 1ull);
#endif
  const float4 a = __ldg(splats + 3 * (int64_t)g);
  const float k2f = __ldg(reinterpret_cast<const float *>(splats + 3 * (int64_t)g + 1));
  const float4 r0 = __ldg(exact + 2 * (int64_t)g), r1 = __ldg(exact + 2 * (int64_t)g + 1);
  // (double)px - (double)a.x is exact: both are float32 values
  const double dx = __dsub_rn(__dsub_rn((double)px, (double)a.x), (double)r0.z);
  const double dy = __dsub_rn(__dsub_rn((double)py, (double)a.y), (double)r0.w);
  const double q = __dadd_rn(__dmul_rn(__dmul_rn(__dadd_rn(a.z, r1.x), dx), dx),
                             __dmul_rn(__dmul_rn(__dadd_rn(k2f, r1.z), dy), dy));
  const double e = __dsub_rn(__dmul_rn(-0.5, q), __dmul_rn(__dmul_rn(__dadd_rn(a.w, r1.y), dx), dy));
  const float alpha = __ldg(reinterpret_cast<const float *>(splats + 3 * (int64_t)g + 1) + 1);
  if (!(alpha > kClampAlpha)) return __dmul_rn(e, 1.4426950408889634) >= __dadd_rn(r0.x, r1.w) ? 3 : 0;
  if (e < -4.5) return 0;
  return e <= (double)r1.w ? 3 : 1;
}

// The clamp bracket's lower end (log2 units) of a Gaussian whose alpha can reach the 0.99
// clamp (float32 alpha > kClampAlpha): a blended pair whose float32 exponent e2 lies below
// it is certainly unclamped (alpha exp(e) <= 0.99: the partials through alpha apply,
// _kernels.py:157-168); at or above it the float64 decision (exact_pair, record slot 7 =
// ln(0.99 / alpha)) is taken — only the backward needs it (the forward blends min(a, 0.99)
// either way).  Computed from registers the staging already holds: log2(0.99 / alpha)
// from the float32 alpha is within ~1e-6 of the float64 exponent (alpha's rounding
// ~4e-7 relative, lg2.approx ~2.4e-7 absolute), and the float32 exponent's own error is at
// most (cut_hi - cut_lo) / 2 (the record's bracket half-width bounds it over the
// footprint, preprocess.cu exact_record).  +inf for the other Gaussians.
__device__ __forceinline__ float clamp_lo_of(float2 cut, float alpha) {
  float v = __int_as_float(0x7f800000);
  if (alpha > kClampAlpha) v = __log2f(__fdividef(0.99f, alpha)) - 0.5f * (cut.y - cut.x) - 4e-6f;
  return v;
}

// Both pixels of a lane at once, out of line (the 16x16 kernels call it from a warp-uniform
// branch taken only when some lane has a pair inside the bracket, so the float64 code stays
// out of the hot loop).  Returns exact_pair(A) | exact_pair(B) << 2 for the flagged pixels.
#ifdef TGS_RESOLVE_INLINE  // A/B builds: the float64 resolution inlined into the visit
__device__ __forceinline__
#else
__device__ __noinline__
#endif
int resolve2(const float4 *__restrict__ splats, const float4 *__restrict__ exact, int g,
                                     float px, float pyA, float pyB, bool uA, bool uB) {
  int r = 0;
  if (uA) r = exact_pair(splats, exact, g, px, pyA);
  if (uB) r |= exact_pair(splats, exact, g, px, pyB) << 2;
  return r;
}

// Whether any lane of the warp has a pixel whose exponent lies inside its splat's cut
// bracket [cut.x, cut.y): per pixel one compare folded into the e2 >= cut.y compare the
// blend decision makes anyway (FSETP with a predicate operand), OR-ed, one vote.
// Warp-uniform result.  (An arithmetic form, (e2 - lo)(e2 - hi) <= 0 on FADD2 / FMUL2,
// measured 3% slower on the forward: 0.248 vs 0.241 ms per c3 view.)
__device__ __forceinline__ bool in_bracket2(float2 e2, float2 cut) {
  const bool a = e2.x >= cut.x && !(e2.x >= cut.y), b = e2.y >= cut.x && !(e2.y >= cut.y);
  return __any_sync(0xffffffffu, a || b);
}
// ... or at / above the clamp bracket's lower end clo (the forward's clamp candidates):
// e2 >= cut_lo && !(cut_hi <= e2 < clo), one more compare per pixel in the same chain
__device__ __forceinline__ bool in_bracket_or_clamp2(float2 e2, float2 cut, float clo) {
  const bool a = e2.x >= cut.x && !(e2.x >= cut.y && e2.x < clo);
  const bool b = e2.y >= cut.x && !(e2.y >= cut.y && e2.y < clo);
  return __any_sync(0xffffffffu, a || b);
}

// Scalar decision for the one-pixel-per-thread kernels: 0 skip, else bit 1 = unclamped.
__device__ __forceinline__ int decide_pair(float e2, float a_raw, float2 cut, const float4 *__restrict__ splats,
                                           const float4 *__restrict__ exact, int g, float px, float py) {
  const bool hi = e2 >= cut.y;
  if (exact && e2 >= cut.x && !hi) return exact_pair(splats, exact, g, px, py);
  if (!hi) return 0;
  if (!exact) return a_raw <= kAlphaMax ? 3 : 1;
  const float alpha = __ldg(reinterpret_cast<const float *>(splats + 3 * (int64_t)g + 1) + 1);
  if (e2 < clamp_lo_of(cut, alpha)) return 3;  // certainly unclamped (or cannot clamp)
  return exact_pair(splats, exact, g, px, py);
}

__device__ __forceinline__ bool quad_misses(float2 m, float4 q, float thr2, float4 wb) {
  const float X0 = wb.x - m.x, X1 = wb.y - m.x, Y0 = wb.z - m.y, Y1 = wb.w - m.y;
  if (X0 <= 0.0f && X1 >= 0.0f && Y0 <= 0.0f && Y1 >= 0.0f) return false;
  const float ky = __fdividef(-q.y, 2.0f * q.z), kx = __fdividef(-q.y, 2.0f * q.x);
  auto edge_x = [&](float X) {  // max over y in [Y0, Y1] at dx = X
    const float y = fminf(fmaxf(ky * X, Y0), Y1);
    return q.x * X * X + (q.y * X + q.z * y) * y;
  };
  auto edge_y = [&](float Y) {  // max over x in [X0, X1] at dy = Y
    const float x = fminf(fmaxf(kx * Y, X0), X1);
    return (q.x * x + q.y * Y) * x + q.z * Y * Y;
  };
  const float best = fmaxf(fmaxf(edge_x(X0), edge_x(X1)), fmaxf(edge_y(Y0), edge_y(Y1)));
  return !(best >= thr2);
}

// Bounds of the pixels this warp owns (empty when `live` is false on every lane).
__device__ __forceinline__ float4 warp_bounds(bool live, int px, int py) {
  const int x0 = __reduce_min_sync(0xffffffffu, live ? px : 0x7fffffff);
  const int x1 = __reduce_max_sync(0xffffffffu, live ? px : -0x7fffffff);
  const int y0 = __reduce_min_sync(0xffffffffu, live ? py : 0x7fffffff);
  const int y1 = __reduce_max_sync(0xffffffffu, live ? py : -0x7fffffff);
  return make_float4((float)x0, (float)x1, (float)y0, (float)y1);
}


// Staged splat (structure of arrays in shared memory).
struct Stage {
  float2 xy[kBatch];
  float4 q[kBatch];    // prescaled conic + alpha
  float4 col[kBatch];  // r, g, b, cull threshold (log2 units)
  float2 cut[kBatch];  // blend-cut bracket (load_cut)
  int32_t id[kBatch];
};

__device__ __forceinline__ void stage_splat(Stage &S, int slot, const float4 *__restrict__ splats,
                                            const float4 *__restrict__ exact, int g) {
  const float4 a = splats[3 * g], b = splats[3 * g + 1];
  const float c = splats[3 * g + 2].x;
  const float2 cut = load_cut(exact, g, b.y);
  S.xy[slot] = make_float2(a.x, a.y);
  S.q[slot] = prescaled_conic(a, b);
  S.col[slot] = make_float4(b.z, b.w, c, cut.x - 0.02f);  // cull: nothing below cut.x blends
  S.cut[slot] = cut;
  S.id[slot] = g;
}

template <int kMaxThreads>
__global__ void __launch_bounds__(kMaxThreads) k_blend_fwd(const float4 *__restrict__ splats,
                                                           const float4 *__restrict__ exact,
                                                           const int32_t *__restrict__ offsets,
                                                           const int32_t *__restrict__ ids, int W, int H, int ts,
                                                           int tiles_x, int row_begin, float bg0, float bg1,
                                                           float bg2, float *__restrict__ image,
                                                           float *__restrict__ transmit, float *__restrict__ wsum_out,
                                                           int32_t *__restrict__ n_contrib,
                                                           int32_t *__restrict__ last_pos,
                                                           int32_t *__restrict__ hits) {
  __shared__ Stage S;
  const int B = blockDim.x;
  const int batch = B < kBatch ? B : kBatch;
  const int tile = blockIdx.x;
  const int ty = row_begin + tile / tiles_x, tx = tile % tiles_x;
  const int t = threadIdx.x, lane = t & 31;
  int lx, ly;
  pixel_of(t, ts, lx, ly);
  const int px = tx * ts + lx, py = ty * ts + ly;
  const bool inside = t < ts * ts && px < W && py < H;
  const float4 wb = warp_bounds(inside, px, py);
  const int start = offsets[tile], stop = offsets[tile + 1];
  const float fpx = (float)px, fpy = (float)py;
  float T = 1.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, ws = 0.0f;
  int contrib = 0, lastp = 0;
  bool done = !inside;
  for (int base = start; base < stop; base += batch) {
    if (__syncthreads_count(done) == B) break;
    if (t < batch && base + t < stop) stage_splat(S, t, splats, exact, ids[base + t]);
    __syncthreads();
    const int cnt = min(batch, stop - base);
    for (int j0 = 0; j0 < cnt; j0 += 32) {
      if (__all_sync(0xffffffffu, done)) break;
      // one splat per lane: the warp-level cull, then iterate the survivors in order
      const int j = j0 + lane;
      uint32_t mask = __ballot_sync(0xffffffffu, j < cnt && !quad_misses(S.xy[j], S.q[j], S.col[j].w, wb));
      while (mask) {
        const int k = j0 + __ffs(mask) - 1;
        mask &= mask - 1;
        if (done) continue;
        if (T < kTTerm) {  // checked before each entry (_kernels.py:57-58)
          done = true;
          continue;
        }
        const float2 m = S.xy[k];
        const float4 q = S.q[k];
        const float e2 = exponent2(q, fpx - m.x, fpy - m.y);
        float al = __fmul_rn(q.w, ex2_approx(e2));
        if (!decide_pair(e2, al, S.cut[k], splats, exact, S.id[k], fpx, fpy)) continue;
        al = fminf(al, kAlphaMax);
        const float4 col = S.col[k];
        const float w = al * T;
        c0 += col.x * w;
        c1 += col.y * w;
        c2 += col.z * w;
        ws += w;
        T = __fmul_rn(T, __fsub_rn(1.0f, al));
        ++contrib;
        lastp = base - start + k + 1;
        if (hits) atomicAdd(hits + S.id[k], 1);
      }
    }
    if (T < kTTerm) done = true;
  }
  if (inside) {
    const int p = py * W + px;
    image[3 * p] = c0 + bg0 * T;
    image[3 * p + 1] = c1 + bg1 * T;
    image[3 * p + 2] = c2 + bg2 * T;
    transmit[p] = T;
    wsum_out[p] = ws;
    n_contrib[p] = contrib;
    last_pos[p] = lastp;
  }
}

// Sum v[0..7] over the warp with a transposing butterfly (9 shuffles): on return
// lane l holds the warp total of value (l >> 2) & 7.
__device__ __forceinline__ float warp_reduce8_transpose(const float v[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  float k4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = b4 ? v[i] : v[4 + i];
    const float keep = b4 ? v[4 + i] : v[i];
    k4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  float k2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b3 ? k4[i] : k4[2 + i];
    const float keep = b3 ? k4[2 + i] : k4[i];
    k2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  float k1 = (b2 ? k2[1] : k2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? k2[0] : k2[1], 4);
  k1 += __shfl_xor_sync(0xffffffffu, k1, 2);
  k1 += __shfl_xor_sync(0xffffffffu, k1, 1);
  return k1;
}

// Two visits at once: u[0..7] = visit 0's fields 0-7, u[8..15] = visit 1's.  Four
// transposing levels (16 -> 1 value per lane) and one plain level leave lane l
// holding the warp sum of value index l >> 1, i.e. visit l >> 4, field (l >> 1) & 7.
__device__ __forceinline__ float warp_reduce16_transpose(const float u[16], int lane) {
  float k8[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool b = lane & 16;
    k8[i] = (b ? u[8 + i] : u[i]) + __shfl_xor_sync(0xffffffffu, b ? u[i] : u[8 + i], 16);
  }
  float k4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool b = lane & 8;
    k4[i] = (b ? k8[4 + i] : k8[i]) + __shfl_xor_sync(0xffffffffu, b ? k8[i] : k8[4 + i], 8);
  }
  float k2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool b = lane & 4;
    k2[i] = (b ? k4[2 + i] : k4[i]) + __shfl_xor_sync(0xffffffffu, b ? k4[i] : k4[2 + i], 4);
  }
  const bool b = lane & 2;
  float k1 = (b ? k2[1] : k2[0]) + __shfl_xor_sync(0xffffffffu, b ? k2[0] : k2[1], 2);
  k1 += __shfl_xor_sync(0xffffffffu, k1, 1);
  return k1;
}

// The two visits' 9th fields: lane l ends with the warp sum of visit l >> 4's.
__device__ __forceinline__ float warp_reduce2_transpose(float n0, float n1, int lane) {
  const bool b = lane & 16;
  float k = (b ? n1 : n0) + __shfl_xor_sync(0xffffffffu, b ? n0 : n1, 16);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
  return k;
}

// The 16-value reduction of k_blend_bwd16p through the warp's shared-memory slot instead
// of the butterfly (whose per value cost is one SHFL, two lane-dependent FSELs and one
// FADD): each lane stores its 16 values as one row (4 x STS.128), lane l then sums
// column l & 15 over its half warp's 16 rows (16 LDS, a 4-deep FADD tree) and one
// SHFL adds the halves.  Rows are 20 floats apart and the upper 16 rows shifted by 16
// more, so both the row stores (per 8-lane phase) and the column loads are
// bank-conflict free.  Lane l ends with the warp sum of u[l & 15].
#ifndef TGS_BWD_SMEM_RED
#define TGS_BWD_SMEM_RED 1
#endif
constexpr int kRedStride = 20;
constexpr int kRedFloats = 32 * kRedStride + 16;
__device__ __forceinline__ int red_row(int r) { return r * kRedStride + (r & 16); }

__device__ __forceinline__ float warp_reduce16_smem(float *buf, const float u[16], int lane) {
  float4 *w = reinterpret_cast<float4 *>(buf + red_row(lane));
#pragma unroll
  for (int c = 0; c < 4; ++c) w[c] = make_float4(u[4 * c], u[4 * c + 1], u[4 * c + 2], u[4 * c + 3]);
  __syncwarp();
  const float *col = buf + red_row(lane & 16) + (lane & 15);
#ifndef TGS_RED_CHUNK
#define TGS_RED_CHUNK 16
#endif
  float acc = 0.0f;
#pragma unroll
  for (int c0 = 0; c0 < 16; c0 += TGS_RED_CHUNK) {  // loads in flight per batch (registers)
    float t[TGS_RED_CHUNK];
#pragma unroll
    for (int i = 0; i < TGS_RED_CHUNK; ++i) t[i] = col[(c0 + i) * kRedStride];
#pragma unroll
    for (int h = TGS_RED_CHUNK / 2; h > 0; h >>= 1)
#pragma unroll
      for (int i = 0; i < h; ++i) t[i] += t[i + h];
    acc = c0 ? acc + t[0] : t[0];
  }
  __syncwarp();
  return acc + __shfl_xor_sync(0xffffffffu, acc, 16);
}

// Backward batch: 128 splats at 16x16 tiles; each warp owns a private slice of
// the per-splat accumulators (plain stores, no shared-memory float atomics,
// which sm_100 emulates with a CAS loop), summed over warps at the flush.
template <int kMaxThreads>
struct BwdShared {
  static constexpr int kWarpsMax = kMaxThreads / 32;
  static constexpr int kBB = kMaxThreads <= 256 ? 128 : 32;
  float2 xy[kBB];
  float4 q[kBB];
  float4 conic[kBB];  // a, b, c, alpha (raw, for the partials)
  float4 col[kBB];    // r, g, b, cull threshold
  float2 cut[kBB];    // blend-cut bracket (load_cut)
  int32_t id[kBB];
  float acc[kWarpsMax][9][kBB];
};

template <int kMaxThreads>
__global__ void __launch_bounds__(kMaxThreads) k_blend_bwd(const float4 *__restrict__ splats,
                                                           const float4 *__restrict__ exact,
                                                           const int32_t *__restrict__ offsets,
                                                           const int32_t *__restrict__ ids, int W, int H, int ts,
                                                           int tiles_x, int row_begin, float bg0, float bg1,
                                                           float bg2, const float *__restrict__ transmit,
                                                           const int32_t *__restrict__ last_pos,
                                                           const float *__restrict__ dimage,
                                                           float *__restrict__ dsplats,
                                                           float *__restrict__ partial) {
  using SM = BwdShared<kMaxThreads>;
  constexpr int kBB = SM::kBB;
  __shared__ SM S;
  __shared__ int wmax[32];
  const int B = blockDim.x;
  const int nwarps = B >> 5;
  const int tile = blockIdx.x;
  const int ty = row_begin + tile / tiles_x, tx = tile % tiles_x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int lx, ly;
  pixel_of(t, ts, lx, ly);
  const int px = tx * ts + lx, py = ty * ts + ly;
  const bool inside = t < ts * ts && px < W && py < H;
  const int start = offsets[tile];
  const float fpx = (float)px, fpy = (float)py;
  int lastp = 0;
  float g0 = 0.f, g1 = 0.f, g2 = 0.f, T_after = 0.f;
  if (inside) {
    const int p = py * W + px;
    lastp = last_pos[p];
    g0 = dimage[3 * p];
    g1 = dimage[3 * p + 1];
    g2 = dimage[3 * p + 2];
    if (g0 == 0.0f && g1 == 0.0f && g2 == 0.0f) lastp = 0;  // _kernels.py:133-134
    T_after = transmit[p];
  }
  // pixels with lastp == 0 never contribute: they neither widen the warp box nor its list prefix
  const float4 wb = warp_bounds(lastp > 0, px, py);
  const int wlast = __reduce_max_sync(0xffffffffu, lastp);
  float s0 = bg0 * T_after, s1 = bg1 * T_after, s2 = bg2 * T_after;
  if (lane == 0) wmax[warp] = wlast;
  __syncthreads();
  if (warp == 0) {
    int m = lane < nwarps ? wmax[lane] : 0;
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) wmax[0] = m;
  }
  __syncthreads();
  const int max_last = wmax[0];
  for (int hi = max_last; hi > 0; hi -= kBB) {
    const int lo = hi > kBB ? hi - kBB : 0;
    const int cnt = hi - lo;
    __syncthreads();
    if (t < cnt) {
      const int g = ids[start + lo + t];
      const float4 a = splats[3 * g], b = splats[3 * g + 1];
      S.xy[t] = make_float2(a.x, a.y);
      S.q[t] = prescaled_conic(a, b);
      S.conic[t] = make_float4(a.z, a.w, b.x, b.y);
      const float2 cut = load_cut(exact, g, b.y);
      S.col[t] = make_float4(b.z, b.w, splats[3 * g + 2].x, cut.x - 0.02f);
      S.cut[t] = cut;
      S.id[t] = g;
    }
    for (int e = t; e < nwarps * 9 * kBB; e += B) (&S.acc[0][0][0])[e] = 0.0f;
    __syncthreads();
    // back to front over 32-splat chunks; inside a chunk the survivors high to low
    for (int j0 = (cnt - 1) & ~31; j0 >= 0; j0 -= 32) {
      const int j = j0 + lane;
      uint32_t mask =
          __ballot_sync(0xffffffffu, j < cnt && lo + j < wlast && !quad_misses(S.xy[j], S.q[j], S.col[j].w, wb));
      while (mask) {
        const int bit = 31 - __clz(mask);
        mask &= ~(1u << bit);
        const int q = j0 + bit;
        float v[9];
#pragma unroll
        for (int f = 0; f < 9; ++f) v[f] = 0.0f;
        bool hit = false;
        if (lo + q < lastp) {
          const float2 m = S.xy[q];
          const float dx = fpx - m.x, dy = fpy - m.y;
          const float e2 = exponent2(S.q[q], dx, dy);
          {
            const float4 cn = S.conic[q];
            const float gauss = ex2_approx(e2);
            const float a_raw = __fmul_rn(cn.w, gauss);
            const float al = fminf(a_raw, kAlphaMax);
            const int dec = decide_pair(e2, a_raw, S.cut[q], splats, exact, S.id[q], fpx, fpy);
            if (dec) {
              hit = true;
              const float4 col = S.col[q];
              const float inv_om = __fdividef(1.0f, 1.0f - al);
              const float t_before = T_after * inv_om;
              const float ga = g0 * (col.x * t_before - s0 * inv_om) + g1 * (col.y * t_before - s1 * inv_om) +
                               g2 * (col.z * t_before - s2 * inv_om);
              const float w = al * t_before;
              v[6] = g0 * w;
              v[7] = g1 * w;
              v[8] = g2 * w;
              if (dec & 2) {  // a_raw <= 0.99 (decided with the blend)
                v[5] = ga * gauss;
                const float gG = ga * cn.w * gauss;
                const float v0 = cn.x * dx + cn.y * dy, v1 = cn.y * dx + cn.z * dy;
                v[0] = gG * v0;
                v[1] = gG * v1;
                v[2] = gG * 0.5f * v0 * v0;
                v[3] = gG * v0 * v1;
                v[4] = gG * 0.5f * v1 * v1;
              }
              s0 += col.x * w;
              s1 += col.y * w;
              s2 += col.z * w;
              T_after = t_before;
            }
          }
        }
        if (__any_sync(0xffffffffu, hit)) {
          const float r8 = warp_reduce8_transpose(v, lane);
          float r9 = v[8];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) r9 += __shfl_xor_sync(0xffffffffu, r9, o);
          if ((lane & 3) == 0) S.acc[warp][lane >> 2][q] = r8;
          if (lane == 0) S.acc[warp][8][q] = r9;
        }
      }
    }
    __syncthreads();
    if (t < cnt) {
      if (partial) {  // deterministic mode: this (tile, splat) pair's partials, summed in warp order
        float *pp = partial + (int64_t)(start + lo + t) * 9;
#pragma unroll
        for (int f = 0; f < 9; ++f) {
          float x = 0.0f;
          for (int w = 0; w < nwarps; ++w) x += S.acc[w][f][t];
          pp[f] = x;
        }
      } else {
        float *d = dsplats + 9 * (int64_t)S.id[t];
#pragma unroll
        for (int f = 0; f < 9; ++f) {
          float x = 0.0f;
          for (int w = 0; w < nwarps; ++w) x += S.acc[w][f][t];
          if (x != 0.0f) atomicAdd(d + f, x);
        }
      }
    }
  }
  if (partial) {  // list positions no pixel reached contribute zero
    const int stop = offsets[tile + 1];
    for (int64_t e = (int64_t)(start + max_last) * 9 + t; e < (int64_t)stop * 9; e += B) partial[e] = 0.0f;
  }
}

// ------------------------------------------------- deterministic reduction
// Per Gaussian (cloud row), its instances in rect order (row-major over the
// band-clipped tile rect of bin_tiles) map to list positions through `inv`;
// the Gaussian's partials are summed in that fixed order by one thread, so the
// result does not depend on scheduling.
__global__ void k_inst_count(const float *__restrict__ splats, const int32_t *__restrict__ tiles_touched, int64_t n,
                             int W, int H, int ts, int tiles_x, int tiles_y, int rb, int re,
                             uint32_t *__restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t c = 0;
  if (tiles_touched[i] > 0) {
    int x0, y0, x1, y1;
    const float *sp = splats + 12 * i;
    if (tile_rect(sp[0], sp[1], sp[10], W, H, ts, tiles_x, tiles_y, x0, y0, x1, y1) > 0) {
      y0 = max(y0, rb);
      y1 = min(y1, re - 1);
      if (y1 >= y0) c = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
    }
  }
  cnt[i] = c;
}

constexpr uint32_t kDetFlagAgg = 1u << 30, kDetFlagInc = 2u << 30, kDetMask = (1u << 30) - 1;

// Exclusive scan of n u32 (in place), tiles of 4096 chained by decoupled look-back.
__global__ void __launch_bounds__(256) k_det_scan(uint32_t *__restrict__ v, int64_t n, uint32_t *__restrict__ status,
                                                  uint32_t *__restrict__ ticket) {
  __shared__ uint32_t ws[8], s_tile, s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * 4096 + threadIdx.x * 16;
  uint32_t x[16], sum = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    x[k] = base + k < n ? v[base + k] : 0u;
    sum += x[k];
  }
  // block exclusive scan of the per-thread sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  uint32_t woff = 0, tot = 0;
  for (int w = 0; w < 8; ++w) {
    if (w < warp) woff += ws[w];
    tot += ws[w];
  }
  if (threadIdx.x == 0) {
    uint32_t *mine = status + tile;
    uint32_t excl = 0;
    if (tile == 0) {
      atomicExch(mine, kDetFlagInc | tot);
    } else {
      atomicExch(mine, kDetFlagAgg | tot);
      int j = (int)tile - 1;
      for (;;) {
        const uint32_t sv = atomicAdd(status + j, 0u);
        if ((sv >> 30) == 0) continue;  // predecessor not published yet
        excl += sv & kDetMask;
        if (sv & kDetFlagInc) break;
        --j;
      }
      atomicExch(mine, kDetFlagInc | (excl + tot));
    }
    s_excl = excl;
  }
  __syncthreads();
  uint32_t run = s_excl + woff + inc - sum;
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (base + k < n) {
      v[base + k] = run;
      run += x[k];
    }
}

// One CTA per band tile: list position -> slot of that instance in its Gaussian's rect order.
__global__ void k_det_inverse(const float *__restrict__ splats, const int32_t *__restrict__ offsets,
                              const int32_t *__restrict__ ids, const uint32_t *__restrict__ inst_off, int W, int H,
                              int ts, int tiles_x, int tiles_y, int rb, int re, uint32_t *__restrict__ inv) {
  const int tile = blockIdx.x;
  const int ty = rb + tile / tiles_x, tx = tile % tiles_x;
  const int start = offsets[tile], stop = offsets[tile + 1];
  for (int pos = start + threadIdx.x; pos < stop; pos += blockDim.x) {
    const int g = ids[pos];
    const float *sp = splats + 12 * (int64_t)g;
    int x0, y0, x1, y1;
    tile_rect(sp[0], sp[1], sp[10], W, H, ts, tiles_x, tiles_y, x0, y0, x1, y1);
    y0 = max(y0, rb);
    inv[inst_off[g] + (uint32_t)((ty - y0) * (x1 - x0 + 1) + (tx - x0))] = (uint32_t)pos;
  }
}

__global__ void k_det_reduce(const uint32_t *__restrict__ cnt_off, const uint32_t *__restrict__ inv,
                             const float *__restrict__ partial, int64_t n, int64_t total,
                             float *__restrict__ dsplats) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t o0 = cnt_off[i], o1 = i + 1 < n ? cnt_off[i + 1] : (uint32_t)total;
  if (o1 == o0) return;
  float acc[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (uint32_t k = o0; k < o1; ++k) {
    const float *pp = partial + (int64_t)inv[k] * 9;
#pragma unroll
    for (int f = 0; f < 9; ++f) acc[f] += pp[f];
  }
  float *d = dsplats + 9 * i;
#pragma unroll
  for (int f = 0; f < 9; ++f) d[f] += acc[f];
}

// ---------------------------------------------------------------------------
// 16x16 tiles, two pixels per thread: 128 threads, warp w owns the 8x8 block at
// ((w & 1) * 8, (w >> 1) * 8), lane -> (x = lane & 7, y = lane >> 3) and the
// pixels (x, y) and (x, y + 4).  Per surviving splat a warp evaluates 64 pixels
// and (backward) performs ONE reduction, halving the per-visit overhead.
// (The kernels follow below: k_blend_fwd16w / k_blend_bwd16w.)
constexpr int kT16Threads = 128;

__device__ __forceinline__ void pixel_pair16(int t, int tx, int ty, int &px, int &pyA, int &pyB) {
  const int w = t >> 5, l = t & 31;
  px = tx * 16 + ((w & 1) << 3) + (l & 7);
  pyA = ty * 16 + ((w >> 1) << 3) + (l >> 3);
  pyB = pyA + 4;
}

__device__ __forceinline__ float4 warp_bounds2(bool liveA, bool liveB, int px, int pyA, int pyB) {
  const bool live = liveA || liveB;
  const int x0 = __reduce_min_sync(0xffffffffu, live ? px : 0x7fffffff);
  const int x1 = __reduce_max_sync(0xffffffffu, live ? px : -0x7fffffff);
  const int y0 = __reduce_min_sync(0xffffffffu, liveA ? pyA : (liveB ? pyB : 0x7fffffff));
  const int y1 = __reduce_max_sync(0xffffffffu, liveB ? pyB : (liveA ? pyA : -0x7fffffff));
  return make_float4((float)x0, (float)x1, (float)y0, (float)y1);
}

// The two pixels of a lane, packed: (A, B) in the .x / .y halves.  Every float
// operation is the scalar fwd_entry's (same expression, same rounding), issued as
// FFMA2 / FMUL2 / FADD2; a pixel that skips an entry (done, exponent out of range,
// alpha below 1/255) gets alpha 0, which leaves T, the colour and the weight sum
// bit-identical (all finite, colour and weights >= 0).
struct Fwd16Pair {
  float2 T = make_float2(1.0f, 1.0f), c0 = make_float2(0.f, 0.f), c1 = make_float2(0.f, 0.f),
         c2 = make_float2(0.f, 0.f), ws = make_float2(0.f, 0.f);
  float2 cnt = make_float2(0.f, 0.f);  // n_contrib of both pixels, counted in one FADD2 (exact < 2^24)
  int lA = 0, lB = 0;
  // blend exception (exact decisions): a blended pair the float64 resolution decided — in
  // the cut bracket, or at / above a clampable Gaussian's clamp bracket (whose a <= 0.99
  // only the backward needs) — one per lane, as 4 pos + 2 clamped + (pixel B), pos the
  // 1-based list position; -1: a second one on the lane (the tile's backward then
  // re-resolves its pairs in float64 instead).  One register for both pixels.
  int ex = 0;
  bool dA, dB;
};

__device__ __forceinline__ void note_exception(int &ex, int pos, int pixel_b, bool unclamped) {
  ex = ex ? -1 : 4 * pos + (unclamped ? 0 : 2) + pixel_b;
}
// the exceptions array's word for a pixel: pos | clamped << 31 (0: none)
__device__ __forceinline__ int32_t exception_word(int ex, int pixel_b) {
  return ex > 0 && (ex & 1) == pixel_b ? (int32_t)((uint32_t)(ex >> 2) | ((ex & 2) ? 0x80000000u : 0u)) : 0;
}

template <bool kExact, bool kHits, bool kRec, bool kClamp>
__device__ __forceinline__ void fwd_visit2(Fwd16Pair &P, float fpx, float2 fy, float2 m, float4 q, float4 col,
                                           float2 cut, float clo, int pos, int32_t *hits, int32_t gid,
                                           const float4 *__restrict__ splats, const float4 *__restrict__ exact,
                                           const int32_t *exc) {
  // checked before each entry (_kernels.py:57-58)
  P.dA = P.dA || P.T.x < kTTerm;
  P.dB = P.dB || P.T.y < kTTerm;
  const float dx = fpx - m.x;
  const float2 dy = __fadd2_rn(fy, make_float2(-m.y, -m.y));
  const float t1 = __fmul_rn(__fmul_rn(q.x, dx), dx);
  const float2 s = __ffma2_rn(__fmul2_rn(make_float2(q.z, q.z), dy), dy, make_float2(t1, t1));
  const float b = __fmul_rn(q.y, dx);
  const float2 e2 = __ffma2_rn(make_float2(b, b), dy, s);  // exponent2() for both pixels
  const float2 a_raw = __fmul2_rn(make_float2(q.w, q.w), make_float2(ex2_approx(e2.x), ex2_approx(e2.y)));
  // blend decisions (load_cut / exact_pair): certain in float32 outside the cut bracket;
  // a visit with a pair inside it (rare) resolves it in float64 out of line.  The
  // decision is carried as the blended alpha itself (0 = skipped; a blended alpha is
  // >= ~1/255 > 0), so no boolean has to live across the rare branch.
  float2 al = make_float2(!P.dA && e2.x >= cut.y ? fminf(a_raw.x, kAlphaMax) : 0.0f,
                          !P.dB && e2.y >= cut.y ? fminf(a_raw.y, kAlphaMax) : 0.0f);
  // float64 for pairs inside the cut bracket and — for a Gaussian that can reach the 0.99
  // clamp, when the backward will need it (clo finite: clamp_lo_of) — blended pairs at /
  // above its clamp bracket's lower end, recorded with their clamp bit
  // (kClamp false: no clamp candidates — no exception lists recorded, e.g. a render, or
  // no staged clamp disk reaches this warp's pixels in this chunk)
  if (kExact && (kClamp ? in_bracket_or_clamp2(e2, cut, clo) : in_bracket2(e2, cut))) {  // warp-uniform, rare
    const bool uA = !P.dA && e2.x >= cut.x && !(e2.x >= cut.y && (!kClamp || e2.x < clo));
    const bool uB = !P.dB && e2.y >= cut.x && !(e2.y >= cut.y && (!kClamp || e2.y < clo));
    const int r = resolve2(splats, exact, gid, fpx, fy.x, fy.y, uA, uB);
    if (uA && (al.x > 0.0f || (r & 1))) {  // a certain pair stays blended (float64 agrees)
      al.x = fminf(a_raw.x, kAlphaMax);
      if (kRec) note_exception(P.ex, pos, 0, (r & 2) != 0);
    }
    if (uB && (al.y > 0.0f || (r & 4))) {
      al.y = fminf(a_raw.y, kAlphaMax);
      if (kRec) note_exception(P.ex, pos, 1, (r & 8) != 0);
    }
  }
  const bool okA = al.x > 0.0f, okB = al.y > 0.0f;
  const float2 w = __fmul2_rn(al, P.T);
  P.c0 = __ffma2_rn(make_float2(col.x, col.x), w, P.c0);
  P.c1 = __ffma2_rn(make_float2(col.y, col.y), w, P.c1);
  P.c2 = __ffma2_rn(make_float2(col.z, col.z), w, P.c2);
  P.ws = __fadd2_rn(P.ws, w);
  P.T = __fmul2_rn(P.T, __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-al.x, -al.y)));
  P.cnt = __fadd2_rn(P.cnt, make_float2(okA ? 1.0f : 0.0f, okB ? 1.0f : 0.0f));
  if (okA) P.lA = pos;
  if (okB) P.lB = pos;
  if (kHits) {
    if (okA) atomicAdd(hits + gid, 1);
    if (okB) atomicAdd(hits + gid, 1);
  }
}

struct Bwd16Pixel {
  int lastp = 0;
  float g0 = 0.f, g1 = 0.f, g2 = 0.f, T = 0.f;
  float GS = 0.f;  // sum_c g_c * S_c, S = suffix colour seeded with bg * T_final
};

// Backward state of a lane's two pixels, packed (A, B) -> (.x, .y).
struct Bwd16Pair {
  int lA = 0, lB = 0;
  float2 g0 = make_float2(0.f, 0.f), g1 = make_float2(0.f, 0.f), g2 = make_float2(0.f, 0.f);
  float2 T = make_float2(0.f, 0.f), GS = make_float2(0.f, 0.f);
};

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }

// One list entry of the back-to-front walk (_kernels.py:136-181) for both pixels at once,
// with dL/dalpha_hat = (g . c) T_before - (g . S) / (1 - a) (FFMA2/FMUL2/FADD2): writes the visit's 9 partials
// v[k] = A's + B's and returns whether either pixel blended the splat.  A pixel that
// skips the entry gets 1/(1-alpha) = 1, alpha = 0 and a zero Gaussian factor, so its
// T and G.S are unchanged and it contributes exact zeros (the Gaussian factor is
// masked BEFORE the products: an out-of-range exponent may give ex2 = inf).
template <bool kExact>
__device__ __forceinline__ bool bwd_visit2(Bwd16Pair &P, int pos, float fpx, float2 fy, float2 m, float4 q,
                                           float4 cn, float4 col, float2 cut, int32_t gid,
                                           const float4 *__restrict__ splats, const float4 *__restrict__ exact,
                                           float v[9]) {
  const float dx = fpx - m.x;
  const float2 dy = __fadd2_rn(fy, f2(-m.y));
  const float t1 = __fmul_rn(__fmul_rn(q.x, dx), dx);
  const float2 s = __ffma2_rn(__fmul2_rn(f2(q.z), dy), dy, f2(t1));
  const float b = __fmul_rn(q.y, dx);
  const float2 e2 = __ffma2_rn(f2(b), dy, s);  // exponent2() for both pixels
  const float2 gauss = make_float2(ex2_approx(e2.x), ex2_approx(e2.y));
  const float2 a_raw = __fmul2_rn(f2(cn.w), gauss);
  const float2 al = make_float2(fminf(a_raw.x, kAlphaMax), fminf(a_raw.y, kAlphaMax));
  // the forward's decisions, re-derived identically (load_cut / exact_pair)
  bool okA = pos < P.lA && e2.x >= cut.y;
  bool okB = pos < P.lB && e2.y >= cut.y;
  // unclamped (a_raw <= 0.99): the partials through alpha apply.  With exact records a
  // Gaussian that can reach the clamp is staged with cut_hi = +inf, so every certain pair
  // is unclamped and only exact_pair() can report a clamped one.
  bool clA = kExact || a_raw.x <= kAlphaMax, clB = kExact || a_raw.y <= kAlphaMax;
  if (kExact && in_bracket2(e2, cut)) {  // warp-uniform, rare
    const bool uA = pos < P.lA && !okA && e2.x >= cut.x, uB = pos < P.lB && !okB && e2.y >= cut.x;
    const int r = resolve2(splats, exact, gid, fpx, fy.x, fy.y, uA, uB);
    if (uA) {
      okA = r & 1;
      clA = r & 2;
    }
    if (uB) {
      okB = (r >> 2) & 1;
      clB = (r >> 3) & 1;
    }
  }
  // a pixel that skips the entry blends alpha 0: 1 / (1 - 0) is exactly 1 (rcp.approx of
  // 1.0f is exact, profiles/tma_dbg/rcp_one.cu), so T and the weights need no more selects
  const float2 alm = make_float2(okA ? al.x : 0.0f, okB ? al.y : 0.0f);
  const float2 om = __fadd2_rn(f2(1.0f), make_float2(-alm.x, -alm.y));  // 1 - al >= 0.01
  const float2 inv = make_float2(rcp_approx(om.x), rcp_approx(om.y));
  const float2 tb = __fmul2_rn(P.T, inv);  // T before this entry
  const float2 gc = __ffma2_rn(P.g2, f2(col.z), __ffma2_rn(P.g1, f2(col.y), __fmul2_rn(P.g0, f2(col.x))));
  const float2 ga = __ffma2_rn(gc, tb, __fmul2_rn(P.GS, make_float2(-inv.x, -inv.y)));
  const float2 w = __fmul2_rn(alm, tb);
  const float2 w6 = __fmul2_rn(P.g0, w), w7 = __fmul2_rn(P.g1, w), w8 = __fmul2_rn(P.g2, w);
  // partials through the unclamped alpha only (a_raw <= ALPHA_MAX)
  const bool uA = okA && clA, uB = okB && clB;
  // dL/dalpha_raw-side product ga * G, masked once (a select discards the NaN / Inf an
  // out-of-range Gaussian factor can give)
  const float2 gx = __fmul2_rn(ga, gauss);
  const float2 v5 = make_float2(uA ? gx.x : 0.0f, uB ? gx.y : 0.0f);
  const float2 gG = __fmul2_rn(v5, f2(cn.w));
  const float2 cx = __fmul2_rn(make_float2(cn.x, cn.y), f2(dx));  // (a dx, b dx) in one FMUL2
  const float2 v0 = __ffma2_rn(f2(cn.y), dy, f2(cx.x)), v1 = __ffma2_rn(f2(cn.z), dy, f2(cx.y));
  const float2 hG = __fmul2_rn(gG, f2(0.5f));
  const float2 p0 = __fmul2_rn(gG, v0), p1 = __fmul2_rn(gG, v1);
  const float2 p2 = __fmul2_rn(__fmul2_rn(hG, v0), v0), p3 = __fmul2_rn(p0, v1);
  const float2 p4 = __fmul2_rn(__fmul2_rn(hG, v1), v1);
  v[0] = p0.x + p0.y;
  v[1] = p1.x + p1.y;
  v[2] = p2.x + p2.y;
  v[3] = p3.x + p3.y;
  v[4] = p4.x + p4.y;
  v[5] = v5.x + v5.y;
  v[6] = w6.x + w6.y;
  v[7] = w7.x + w7.y;
  v[8] = w8.x + w8.y;
  P.GS = __ffma2_rn(gc, w, P.GS);
  P.T = tb;
  return okA || okB;
}


// ---------------------------------------------------------------------------
// Warp-independent 16x16 kernels: each warp of a tile's CTA walks the tile list
// on its own, staging 32 splats at a time in a private shared-memory slot (the
// next chunk's records are prefetched into registers while the current one is
// processed), culls them against its own 8x8 pixel block and leaves as soon as
// its pixels are done.  No CTA barrier anywhere: the 4 warps of a tile never wait
// for one another.  The backward flushes each visit's warp-reduced partials with
// global reductions straight away.
struct WStage {
  float2 xy[32];
  float4 q[32];      // prescaled conic + alpha
  float4 col[32];    // r, g, b, cull threshold (log2 units)
  float4 conic[32];  // raw a, b, c, alpha (backward)
  float2 cut[32];    // blend-cut bracket (load_cut)
  int32_t id[32];
};

struct SplatRegs {
  float4 a, b;
  float c;
  float2 cut;
  int32_t g;
};

__device__ __forceinline__ void fetch_splat(SplatRegs &r, const float4 *__restrict__ splats,
                                            const float4 *__restrict__ exact, const int32_t *__restrict__ ids,
                                            int pos, bool ok) {
  if (ok) {
    r.g = __ldg(ids + pos);
    r.a = __ldg(splats + 3 * r.g);
    r.b = __ldg(splats + 3 * r.g + 1);
    r.c = __ldg(reinterpret_cast<const float *>(splats + 3 * r.g + 2));
    if (exact) r.cut = __ldg(reinterpret_cast<const float2 *>(exact + 2 * (int64_t)r.g));
  }
}

// The pixel coordinates the forward needs after its setup, re-derived from the loop's float
// copies (exact for coordinates < 2^24), so only one copy of each stays live in the
// visit loop (with both, ptxas kept the ints and re-converted the floats every visit).
#define PIX_X ((int)fpx)
#define PIX_YA ((int)fy.x)
#define PIX_YB ((int)fy.y)
template <bool kExact, bool kHits, bool kRec>
__global__ void __launch_bounds__(kT16Threads, kExact ? TGS_FWD16_MINB : 1) k_blend_fwd16w(
    const float4 *__restrict__ splats, const float4 *__restrict__ exact, const int32_t *__restrict__ offsets, const int32_t *__restrict__ ids, int W,
    int H, int tiles_x, int row_begin, float bg0, float bg1, float bg2, float *__restrict__ image,
    float *__restrict__ transmit, float *__restrict__ wsum_out, int32_t *__restrict__ n_contrib,
    int32_t *__restrict__ last_pos, int32_t *__restrict__ hits, const int32_t *__restrict__ order,
    int32_t *__restrict__ exc, uint32_t *__restrict__ ovf) {
  __shared__ WStage SW[kT16Threads / 32];
  const int tile = order ? __ldg(order + blockIdx.x) : (int)blockIdx.x;
  const int ty = row_begin + tile / tiles_x, tx = tile % tiles_x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  WStage &S = SW[warp];
  int px, pyA, pyB;
  pixel_pair16(t, tx, ty, px, pyA, pyB);
  const bool inA = px < W && pyA < H, inB = px < W && pyB < H;
  const float4 wb = warp_bounds2(inA, inB, px, pyA, pyB);
  const int start = __ldg(offsets + tile), stop = __ldg(offsets + tile + 1);
  const float fpx = (float)px, fyA = (float)pyA, fyB = (float)pyB;
  Fwd16Pair P;
  P.dA = !inA;
  P.dB = !inB;
  const float2 fy = make_float2(fyA, fyB);
  SplatRegs nx;
  fetch_splat(nx, splats, kExact ? exact : nullptr, ids, start + lane, start + lane < stop);
  float4 wbc = wb;
  for (int c = start; c < stop; c += 32) {
    if (__all_sync(0xffffffffu, P.dA && P.dB)) break;
    // cull against the pixels that are still blending (terminated ones no longer count)
    if (c != start) wbc = warp_bounds2(!P.dA, !P.dB, PIX_X, PIX_YA, PIX_YB);
    const bool ok = c + lane < stop;
    bool keep = false, reach = false;
    if (ok) {
      const float4 q = prescaled_conic(nx.a, nx.b);
      const float2 cut = kExact ? nx.cut : load_cut(nullptr, nx.g, nx.b.y);
      const float thr = cut.x - 0.02f;  // cull: nothing below cut.x blends
      const float2 m = make_float2(nx.a.x, nx.a.y);
      S.xy[lane] = m;
      S.q[lane] = q;
      // col.w: the clamp bracket's lower end when the backward will need the clamp
      // decision (exception lists requested); +inf otherwise and for most Gaussians
      const float clo = kExact && kRec ? clamp_lo_of(cut, nx.b.y) : __int_as_float(0x7f800000);
      S.col[lane] = make_float4(nx.b.z, nx.b.w, nx.c, clo);
      S.cut[lane] = cut;
      S.id[lane] = nx.g;
      keep = !quad_misses(m, q, thr, wbc);
      // a clamp bracket this warp's pixels can reach (the same exact box test as the cull)
      reach = keep && clo < __int_as_float(0x7f800000) && !quad_misses(m, q, clo, wbc);
    }
    uint32_t mask = __ballot_sync(0xffffffffu, keep);
    // the chunk's visits test the clamp candidates only when a staged splat's clamp disk can
    // reach the warp's box (chunk-uniform: two copies of the visit loop)
    const bool clamp_chunk = kRec && __any_sync(0xffffffffu, reach);
    __syncwarp();
    fetch_splat(nx, splats, kExact ? exact : nullptr, ids, c + 32 + lane, c + 32 + lane < stop);
    if (clamp_chunk) {
      while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1;
        const float2 m = S.xy[k];
        const float4 q = S.q[k], col = S.col[k];
        const int pos = c - start + k + 1;
        fwd_visit2<kExact, kHits, kRec, kRec>(P, fpx, fy, m, q, col, S.cut[k], col.w, pos, hits,
                                              kHits || kExact ? S.id[k] : 0, splats, exact, exc);
      }
    } else {
      while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1;
        const float2 m = S.xy[k];
        const float4 q = S.q[k], col = S.col[k];
        const int pos = c - start + k + 1;
        fwd_visit2<kExact, kHits, kRec, false>(P, fpx, fy, m, q, col, S.cut[k], col.w, pos, hits,
                                               kHits || kExact ? S.id[k] : 0, splats, exact, exc);
      }
    }
    if (P.T.x < kTTerm) P.dA = true;
    if (P.T.y < kTTerm) P.dB = true;
    __syncwarp();
  }
  if (PIX_X < W && PIX_YA < H) {
    const int p = PIX_YA * W + PIX_X;
    image[3 * p] = P.c0.x + bg0 * P.T.x;
    image[3 * p + 1] = P.c1.x + bg1 * P.T.x;
    image[3 * p + 2] = P.c2.x + bg2 * P.T.x;
    transmit[p] = P.T.x;
    wsum_out[p] = P.ws.x;
    n_contrib[p] = (int32_t)P.cnt.x;
    last_pos[p] = P.lA;
    if (kRec) exc[p] = exception_word(P.ex, 0);
  }
  if (PIX_X < W && PIX_YB < H) {
    const int p = PIX_YB * W + PIX_X;
    image[3 * p] = P.c0.y + bg0 * P.T.y;
    image[3 * p + 1] = P.c1.y + bg1 * P.T.y;
    image[3 * p + 2] = P.c2.y + bg2 * P.T.y;
    transmit[p] = P.T.y;
    wsum_out[p] = P.ws.y;
    n_contrib[p] = (int32_t)P.cnt.y;
    last_pos[p] = P.lB;
    if (kRec) exc[p] = exception_word(P.ex, 1);
  }
  // a tile with an exception the lists cannot carry: flagged (and counted) once, for the
  // backward to re-resolve its bracket pairs in float64 (ovf = [count, flags[ntiles]])
  if (kRec && __any_sync(0xffffffffu, P.ex < 0) && lane == 0)
    if (atomicCAS(ovf + 1 + tile, 0u, 1u) == 0u) atomicAdd(ovf, 1u);
}
#undef PIX_X
#undef PIX_YA
#undef PIX_YB

template <bool kExact>
__global__ void __launch_bounds__(kT16Threads, kExact ? TGS_BWD16_MINB : 1) k_blend_bwd16w(
    const float4 *__restrict__ splats, const float4 *__restrict__ exact, const int32_t *__restrict__ offsets, const int32_t *__restrict__ ids, int W,
    int H, int tiles_x, int row_begin, float bg0, float bg1, float bg2, const float *__restrict__ transmit,
    const int32_t *__restrict__ last_pos, const float *__restrict__ dimage, float *__restrict__ dsplats,
    const int32_t *__restrict__ order) {
  __shared__ WStage SW[kT16Threads / 32];
  const int tile = order ? __ldg(order + blockIdx.x) : (int)blockIdx.x;
  const int ty = row_begin + tile / tiles_x, tx = tile % tiles_x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  WStage &S = SW[warp];
  int px, pyA, pyB;
  pixel_pair16(t, tx, ty, px, pyA, pyB);
  const int start = __ldg(offsets + tile);
  const float fpx = (float)px, fyA = (float)pyA, fyB = (float)pyB;
  Bwd16Pixel A, B;
  auto load_pixel = [&](Bwd16Pixel &P, int py) {
    if (px >= W || py >= H) return;
    const int p = py * W + px;
    P.lastp = last_pos[p];
    P.g0 = dimage[3 * p];
    P.g1 = dimage[3 * p + 1];
    P.g2 = dimage[3 * p + 2];
    if (P.g0 == 0.0f && P.g1 == 0.0f && P.g2 == 0.0f) P.lastp = 0;  // _kernels.py:133-134
    P.T = transmit[p];
    P.GS = (P.g0 * bg0 + P.g1 * bg1 + P.g2 * bg2) * P.T;
  };
  load_pixel(A, pyA);
  load_pixel(B, pyB);
  const float4 wb = warp_bounds2(A.lastp > 0, B.lastp > 0, px, pyA, pyB);
  const int wlast = __reduce_max_sync(0xffffffffu, max(A.lastp, B.lastp));
  Bwd16Pair PB;  // the two pixels packed for the per-visit arithmetic
  PB.lA = A.lastp;
  PB.lB = B.lastp;
  PB.g0 = make_float2(A.g0, B.g0);
  PB.g1 = make_float2(A.g1, B.g1);
  PB.g2 = make_float2(A.g2, B.g2);
  PB.T = make_float2(A.T, B.T);
  PB.GS = make_float2(A.GS, B.GS);
  const float2 fy = make_float2(fyA, fyB);
  SplatRegs nx;
  // back to front over chunks [lo, hi) of 32 list positions below this warp's last blend
  int hi = wlast;
  fetch_splat(nx, splats, kExact ? exact : nullptr, ids, start + hi - 32 + lane, hi - 32 + lane >= 0);
  for (; hi > 0; hi -= 32) {
    const int lo = hi - 32;  // may be negative: lanes below position 0 are idle
    const bool ok = lo + lane >= 0;
    bool keep = false;
    // only pixels whose last blended position lies beyond lo can take part in this chunk
    const float4 wbc = warp_bounds2(PB.lA > lo, PB.lB > lo, px, pyA, pyB);
    if (ok) {
      const float4 q = prescaled_conic(nx.a, nx.b);
      const float2 cut = kExact ? nx.cut : load_cut(nullptr, nx.g, nx.b.y);
      const float thr = cut.x - 0.02f;  // cull: nothing below cut.x blends
      const float2 m = make_float2(nx.a.x, nx.a.y);
      S.xy[lane] = m;
      S.q[lane] = q;
      S.conic[lane] = make_float4(nx.a.z, nx.a.w, nx.b.x, nx.b.y);
      S.col[lane] = make_float4(nx.b.z, nx.b.w, nx.c, thr);
      // exact decisions: a Gaussian that can reach the 0.99 clamp has no certain pairs here
      // (its clamp decision is taken in float64 with its blend decision; FLT_MAX, not +inf:
      // the bracket test stays well-defined at e2 == cut_lo)
      S.cut[lane] = kExact && nx.b.y > kClampAlpha ? make_float2(cut.x, 3.4e38f) : cut;
      S.id[lane] = nx.g;
      keep = !quad_misses(m, q, thr, wbc);
    }
    uint32_t mask = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    fetch_splat(nx, splats, kExact ? exact : nullptr, ids, start + lo - 32 + lane, lo - 32 + lane >= 0);
    // surviving splats back to front, two per reduction (the second one, if any,
    // follows the first in each pixel's walk, so the per-pixel order is unchanged)
    while (mask) {
      float v0[9], v1[9];
      const int b0 = 31 - __clz(mask);
      mask &= ~(1u << b0);
      bool hit = bwd_visit2<kExact>(PB, lo + b0, fpx, fy, S.xy[b0], S.q[b0], S.conic[b0], S.col[b0], S.cut[b0], S.id[b0],
                            splats, exact, v0);
      int id1 = -1;
      if (mask) {  // warp-uniform
        const int b1 = 31 - __clz(mask);
        mask &= ~(1u << b1);
        hit = bwd_visit2<kExact>(PB, lo + b1, fpx, fy, S.xy[b1], S.q[b1], S.conic[b1], S.col[b1], S.cut[b1], S.id[b1],
                         splats, exact, v1) || hit;
        id1 = S.id[b1];
      } else {
#pragma unroll
        for (int f = 0; f < 9; ++f) v1[f] = 0.0f;
      }
      if (__any_sync(0xffffffffu, hit)) {
        float u[16];
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          u[f] = v0[f];
          u[8 + f] = v1[f];
        }
        const float r = warp_reduce16_transpose(u, lane);
        const float r9 = warp_reduce2_transpose(v0[8], v1[8], lane);
        const int id = (lane & 16) ? id1 : S.id[b0];
        if (id >= 0) {
          float *d = dsplats + 9 * (int64_t)id;
          if ((lane & 1) == 0 && r != 0.0f) atomicAdd(d + ((lane >> 1) & 7), r);
          if ((lane & 15) == 1 && r9 != 0.0f) atomicAdd(d + 8, r9);
        }
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Backward with kP packed pixel pairs per lane (kP = 2: 4 pixels per lane).  A tile's
// 256 pixels are split over 4 / kP warps: kP = 2 gives each warp a 16x8 half tile,
// lane l the column l & 15 and the rows (l >> 4) + {0, 2, 4, 6}.  Per surviving splat
// the lane evaluates its 4 pixels (dx and the dx-only terms shared), and the warp's
// 9-field reduction — about a third of the per-visit instructions at 2 pixels per lane
// — now covers 128 pixels instead of 64; the chunk staging and cull are
// amortised over twice the pixels as well.
template <int kP>
struct BwdLane {
  int l[2 * kP];                                      // last_pos per pixel
  int e[2 * kP];                                      // exception word (kExc): pos | clamped << 31
  int emax;                                           // the lane's highest pending exception position
  float2 g0[kP], g1[kP], g2[kP], T[kP], GS[kP];       // per pair: (pixel 2h, pixel 2h+1)
};

template <int kP>
__device__ __forceinline__ void lane_pixels(int lane, int warp, int tx, int ty, int &px, int py[2 * kP]) {
  if (kP == 1) {
    px = tx * 16 + ((warp & 1) << 3) + (lane & 7);
    py[0] = ty * 16 + ((warp >> 1) << 3) + (lane >> 3);
    py[1] = py[0] + 4;
  } else {
    px = tx * 16 + (lane & 15);
    const int y0 = ty * 16 + warp * 8 + (lane >> 4);
#pragma unroll
    for (int k = 0; k < 2 * kP; ++k) py[k] = y0 + 2 * k;
  }
}

// Out-of-line float64 resolution of a lane's flagged pixels (rare; see resolve2).
template <int kP>
__device__ __noinline__ int resolveP(const float4 *__restrict__ splats, const float4 *__restrict__ exact, int g,
                                     float px, const float *fy, int flags) {
  int r = 0;
#pragma unroll
  for (int k = 0; k < 2 * kP; ++k)
    if (flags & (1 << k)) r |= exact_pair(splats, exact, g, px, fy[k]) << (2 * k);
  return r;
}

// bwd_visitP accumulates fields 2 and 4 (the conic partials' squared terms) at twice their
// value; the factor 1/2 (exact) is applied to the warp sums.
__device__ __forceinline__ float bwd_field_scale(int f) { return (f == 2 || f == 4) ? 0.5f : 1.0f; }

template <bool kExact, int kP, bool kExc>
__device__ __forceinline__ bool bwd_visitP(BwdLane<kP> &P, int pos, float fpx, const float2 fy[kP], float2 m,
                                           float4 q, float4 cn, float4 col, float2 cut, int32_t gid,
                                           const float4 *__restrict__ splats, const float4 *__restrict__ exact,
                                           float v[9]) {
  const float dx = fpx - m.x;
  const float t1 = __fmul_rn(__fmul_rn(q.x, dx), dx);  // dx-only terms, shared by every pixel of the lane
  const float b = __fmul_rn(q.y, dx);
  float2 dy[kP], e2[kP], gauss[kP], a_raw[kP], alm[kP], gm[kP];
#pragma unroll
  for (int h = 0; h < kP; ++h) {
    dy[h] = __fadd2_rn(fy[h], f2(-m.y));
    e2[h] = __ffma2_rn(f2(b), dy[h], __ffma2_rn(__fmul2_rn(f2(q.z), dy[h]), dy[h], f2(t1)));  // exponent2()
    gauss[h] = make_float2(ex2_approx(e2[h].x), ex2_approx(e2[h].y));
    a_raw[h] = __fmul2_rn(f2(cn.w), gauss[h]);
    // the forward's decisions, re-derived identically (load_cut / exact_pair) and carried as
    // floats — alm: the blended alpha or 0 (a skipped entry blends alpha 0: 1 / (1 - 0) is
    // exactly 1, T and G.S stay unchanged); gm: 1 where the partials through alpha apply
    // (unclamped a_raw <= 0.99) — no boolean has to live across the rare branch.  Exact
    // decisions: a certain pair (e2 >= cut_hi) of a Gaussian that cannot reach the 0.99 clamp
    // is unclamped.  With the forward's exception lists (kExc) every pair the forward
    // decided in float64 — a bracket pair it blended, a blended pair at / above a clampable
    // Gaussian's clamp bracket — is the pixel's recorded exception, applied below when the
    // walk reaches its position (no float64 in this body); without them (the float64 body)
    // a clampable Gaussian's staged bracket is [cut_lo, +inf): its pairs all go to float64.
    alm[h] = make_float2(pos < P.l[2 * h] && e2[h].x >= cut.y ? fminf(a_raw[h].x, kAlphaMax) : 0.0f,
                         pos < P.l[2 * h + 1] && e2[h].y >= cut.y ? fminf(a_raw[h].y, kAlphaMax) : 0.0f);
    gm[h] = make_float2(alm[h].x > 0.0f && (kExact || a_raw[h].x <= kAlphaMax) ? 1.0f : 0.0f,
                        alm[h].y > 0.0f && (kExact || a_raw[h].y <= kAlphaMax) ? 1.0f : 0.0f);
  }
  if (kExc) {  // a recorded exception at this list position (one compare per lane; rare)
    if (__any_sync(0xffffffffu, pos + 1 == P.emax)) {
      int nmax = 0;
#pragma unroll
      for (int h = 0; h < kP; ++h) {
        const int wx = P.e[2 * h], wy = P.e[2 * h + 1];
        // blended; a clamped one gets no partials through alpha: its Gaussian factor,
        // used only by them, is zeroed (the common path then needs no clamp mask)
        if (pos + 1 == (wx & 0x7fffffff)) {
          alm[h].x = fminf(a_raw[h].x, kAlphaMax);
          if (wx < 0) gauss[h].x = 0.0f;
          P.e[2 * h] = 0;
        }
        if (pos + 1 == (wy & 0x7fffffff)) {
          alm[h].y = fminf(a_raw[h].y, kAlphaMax);
          if (wy < 0) gauss[h].y = 0.0f;
          P.e[2 * h + 1] = 0;
        }
        nmax = max(nmax, max(P.e[2 * h] & 0x7fffffff, P.e[2 * h + 1] & 0x7fffffff));
      }
      P.emax = nmax;
    }
  } else if (kExact) {  // pairs inside the cut bracket: the float64 decision (rare, warp-uniform branch)
    float pm = 1.0f;
#pragma unroll
    for (int h = 0; h < kP; ++h) {
      const float2 pr = __fmul2_rn(__fadd2_rn(e2[h], f2(-cut.x)), __fadd2_rn(e2[h], f2(-cut.y)));
      pm = fminf(pm, fminf(pr.x, pr.y));
    }
    if (__any_sync(0xffffffffu, pm <= 0.0f)) {
      int flags = 0;
      float fyv[2 * kP];
#pragma unroll
      for (int h = 0; h < kP; ++h) {
        fyv[2 * h] = fy[h].x;
        fyv[2 * h + 1] = fy[h].y;
        if (pos < P.l[2 * h] && !(e2[h].x >= cut.y) && e2[h].x >= cut.x) flags |= 1 << (2 * h);
        if (pos < P.l[2 * h + 1] && !(e2[h].y >= cut.y) && e2[h].y >= cut.x) flags |= 1 << (2 * h + 1);
      }
      if (flags) {
        const int r = resolveP<kP>(splats, exact, gid, fpx, fyv, flags);
#pragma unroll
        for (int h = 0; h < kP; ++h) {
          if ((flags >> (2 * h)) & 1) {
            const int rk = r >> (4 * h);
            alm[h].x = (rk & 1) ? fminf(a_raw[h].x, kAlphaMax) : 0.0f;
            gm[h].x = (rk & 3) == 3 ? 1.0f : 0.0f;
          }
          if ((flags >> (2 * h + 1)) & 1) {
            const int rk = r >> (4 * h + 2);
            alm[h].y = (rk & 1) ? fminf(a_raw[h].y, kAlphaMax) : 0.0f;
            gm[h].y = (rk & 3) == 3 ? 1.0f : 0.0f;
          }
        }
      }
    }
  }
  const float2 cx = __fmul2_rn(make_float2(cn.x, cn.y), f2(dx));  // (a dx, b dx), shared
  float2 acc[9];
  float hitm = 0.0f;
#pragma unroll
  for (int h = 0; h < kP; ++h) {
    const float2 om = __fadd2_rn(f2(1.0f), make_float2(-alm[h].x, -alm[h].y));  // 1 - al >= 0.01
    const float2 inv = make_float2(rcp_approx(om.x), rcp_approx(om.y));
    const float2 tb = __fmul2_rn(P.T[h], inv);  // T before this entry
    const float2 gc =
        __ffma2_rn(P.g2[h], f2(col.z), __ffma2_rn(P.g1[h], f2(col.y), __fmul2_rn(P.g0[h], f2(col.x))));
    const float2 ga = __ffma2_rn(gc, tb, __fmul2_rn(P.GS[h], make_float2(-inv.x, -inv.y)));
    const float2 w = __fmul2_rn(alm[h], tb);
    // partials through the unclamped alpha only; the select drops the NaN / Inf an
    // out-of-range Gaussian factor could give
    float2 v5;
    if (kExc) {  // every blended pair passes its partials through alpha (a clamped exception's
      // Gaussian factor was zeroed above): mask the factor (finite where alm > 0), not the product
      v5 = __fmul2_rn(ga, make_float2(alm[h].x > 0.0f ? gauss[h].x : 0.0f, alm[h].y > 0.0f ? gauss[h].y : 0.0f));
    } else {
      const float2 gx = __fmul2_rn(ga, gauss[h]);
      v5 = make_float2(gm[h].x > 0.0f ? gx.x : 0.0f, gm[h].y > 0.0f ? gx.y : 0.0f);
    }
    const float2 gG = __fmul2_rn(v5, f2(cn.w));
    const float2 v0 = __ffma2_rn(f2(cn.y), dy[h], f2(cx.x)), v1 = __ffma2_rn(f2(cn.z), dy[h], f2(cx.y));
    const float2 p0 = __fmul2_rn(gG, v0), p1 = __fmul2_rn(gG, v1);
    // fields 2 and 4 accumulate gG v0^2 and gG v1^2, twice the partials (the 1/2 is applied
    // once per splat after the warp reduction, bwd_field_scale); products of the second
    // pair fold into the sum as FFMA2 (the partials need the gradient tolerance, not the
    // forward's bit-exactness)
    if (h == 0) {
      acc[0] = p0; acc[1] = p1;
      acc[2] = __fmul2_rn(p0, v0); acc[3] = __fmul2_rn(p0, v1); acc[4] = __fmul2_rn(p1, v1);
      acc[5] = v5;
      acc[6] = __fmul2_rn(P.g0[h], w); acc[7] = __fmul2_rn(P.g1[h], w); acc[8] = __fmul2_rn(P.g2[h], w);
    } else {
      acc[0] = __fadd2_rn(acc[0], p0); acc[1] = __fadd2_rn(acc[1], p1);
      acc[2] = __ffma2_rn(p0, v0, acc[2]); acc[3] = __ffma2_rn(p0, v1, acc[3]); acc[4] = __ffma2_rn(p1, v1, acc[4]);
      acc[5] = __fadd2_rn(acc[5], v5);
      acc[6] = __ffma2_rn(P.g0[h], w, acc[6]); acc[7] = __ffma2_rn(P.g1[h], w, acc[7]);
      acc[8] = __ffma2_rn(P.g2[h], w, acc[8]);
    }
    P.GS[h] = __ffma2_rn(gc, w, P.GS[h]);
    P.T[h] = tb;
    hitm = fmaxf(hitm, fmaxf(alm[h].x, alm[h].y));
  }
#pragma unroll
  for (int f = 0; f < 9; ++f) v[f] = acc[f].x + acc[f].y;
  return hitm > 0.0f;
}

// One tile of the backward.  Exact decisions come in two modes: kExc, the forward's
// exception lists decide the bracket pairs (pos + 1 == exc[pixel], no float64); !kExc,
// the bracket pairs are re-resolved in float64 (resolveP).
template <bool kExact, int kP, bool kExc>
__device__ __forceinline__ void bwd16p_tile(
    WStage *SW, float *RB, int tile, const float4 *__restrict__ splats, const float4 *__restrict__ exact,
    const int32_t *__restrict__ offsets, const int32_t *__restrict__ ids, int W, int H, int tiles_x, int row_begin,
    float bg0, float bg1, float bg2, const float *__restrict__ transmit, const int32_t *__restrict__ last_pos,
    const float *__restrict__ dimage, float *__restrict__ dsplats, const int32_t *__restrict__ exc) {
  const int ty = row_begin + tile / tiles_x, tx = tile % tiles_x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WStage &S = SW[warp];
  int px, py[2 * kP];
  lane_pixels<kP>(lane, warp, tx, ty, px, py);
  const int start = __ldg(offsets + tile);
  const float fpx = (float)px;
  BwdLane<kP> P;
  int wlast = 0;
  int x0 = 0x7fffffff, x1 = -0x7fffffff, y0 = 0x7fffffff, y1 = -0x7fffffff;  // this lane's live box
#pragma unroll
  for (int k = 0; k < 2 * kP; ++k) {
    int lp = 0, ex = 0;
    float g0 = 0.f, g1 = 0.f, g2 = 0.f, T = 0.f;
    if (px < W && py[k] < H) {
      const int p = py[k] * W + px;
      lp = last_pos[p];
      if (kExc) ex = exc[p];
      g0 = dimage[3 * p];
      g1 = dimage[3 * p + 1];
      g2 = dimage[3 * p + 2];
      if (g0 == 0.0f && g1 == 0.0f && g2 == 0.0f) lp = 0;  // _kernels.py:133-134
      T = transmit[p];
    }
    P.l[k] = lp;
    P.e[k] = lp > 0 ? ex : 0;  // (a pixel the walk skips needs none)
    const float GS = (g0 * bg0 + g1 * bg1 + g2 * bg2) * T;
    if (k & 1) {
      P.g0[k >> 1].y = g0; P.g1[k >> 1].y = g1; P.g2[k >> 1].y = g2; P.T[k >> 1].y = T; P.GS[k >> 1].y = GS;
    } else {
      P.g0[k >> 1].x = g0; P.g1[k >> 1].x = g1; P.g2[k >> 1].x = g2; P.T[k >> 1].x = T; P.GS[k >> 1].x = GS;
    }
    wlast = max(wlast, lp);
  }
  wlast = __reduce_max_sync(0xffffffffu, wlast);
  P.emax = 0;
#pragma unroll
  for (int k = 0; k < 2 * kP; ++k) P.emax = max(P.emax, P.e[k] & 0x7fffffff);
  float2 fy[kP];
#pragma unroll
  for (int h = 0; h < kP; ++h) fy[h] = make_float2((float)py[2 * h], (float)py[2 * h + 1]);
  SplatRegs nx;
  // back to front over chunks [lo, hi) of 32 list positions below this warp's last blend
  int hi = wlast;
  fetch_splat(nx, splats, kExact ? exact : nullptr, ids, start + hi - 32 + lane, hi - 32 + lane >= 0);
  for (; hi > 0; hi -= 32) {
    const int lo = hi - 32;  // may be negative: lanes below position 0 are idle
    const bool okl = lo + lane >= 0;
    bool keep = false;
    // only pixels whose last blended position lies beyond lo take part in this chunk
#pragma unroll
    for (int k = 0; k < 2 * kP; ++k)
      if (P.l[k] > lo) {
        x0 = min(x0, px); x1 = max(x1, px); y0 = min(y0, py[k]); y1 = max(y1, py[k]);
      }
    const float4 wbc = make_float4((float)__reduce_min_sync(0xffffffffu, x0), (float)__reduce_max_sync(0xffffffffu, x1),
                                   (float)__reduce_min_sync(0xffffffffu, y0), (float)__reduce_max_sync(0xffffffffu, y1));
    x0 = 0x7fffffff; x1 = -0x7fffffff; y0 = 0x7fffffff; y1 = -0x7fffffff;
    if (okl) {
      const float4 q = prescaled_conic(nx.a, nx.b);
      const float2 cut = kExact ? nx.cut : load_cut(nullptr, nx.g, nx.b.y);
      const float thr = cut.x - 0.02f;  // cull: nothing below cut.x blends
      const float2 m = make_float2(nx.a.x, nx.a.y);
      S.xy[lane] = m;
      S.q[lane] = q;
      S.conic[lane] = make_float4(nx.a.z, nx.a.w, nx.b.x, nx.b.y);
      S.col[lane] = make_float4(nx.b.z, nx.b.w, nx.c, thr);
      // the float64 body (no exception lists): a Gaussian that can reach the 0.99 clamp has
      // no certain pairs (its clamp decision is taken in float64 with its blend decision;
      // FLT_MAX, not +inf: the bracket product stays <= 0 at e2 == cut_lo)
      S.cut[lane] = kExact && !kExc && nx.b.y > kClampAlpha ? make_float2(cut.x, 3.4e38f) : cut;
      S.id[lane] = nx.g;
      keep = !quad_misses(m, q, thr, wbc);
    }
    uint32_t mask = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    fetch_splat(nx, splats, kExact ? exact : nullptr, ids, start + lo - 32 + lane, lo - 32 + lane >= 0);
    // surviving splats back to front, two per reduction (the second one, if any,
    // follows the first in each pixel's walk, so the per-pixel order is unchanged)
    while (mask) {
      float v0[9], v1[9];
      const int b0 = 31 - __clz(mask);
      mask &= ~(1u << b0);
      bool hit = bwd_visitP<kExact, kP, kExc>(P, lo + b0, fpx, fy, S.xy[b0], S.q[b0], S.conic[b0], S.col[b0], S.cut[b0],
                                        S.id[b0], splats, exact, v0);
      int id1 = -1;
      if (mask) {  // warp-uniform
        const int b1 = 31 - __clz(mask);
        mask &= ~(1u << b1);
        hit = bwd_visitP<kExact, kP, kExc>(P, lo + b1, fpx, fy, S.xy[b1], S.q[b1], S.conic[b1], S.col[b1], S.cut[b1],
                                     S.id[b1], splats, exact, v1) || hit;
        id1 = S.id[b1];
      } else {
#pragma unroll
        for (int f = 0; f < 9; ++f) v1[f] = 0.0f;
      }
      if (__any_sync(0xffffffffu, hit)) {
        float u[16];
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          u[f] = v0[f];
          u[8 + f] = v1[f];
        }
#if TGS_BWD_SMEM_RED
        const float r = warp_reduce16_smem(RB + warp * kRedFloats, u, lane);  // lane l: u[l & 15]
        const float r9 = warp_reduce2_transpose(v0[8], v1[8], lane);
        const int idA = (lane & 8) ? id1 : S.id[b0], idB = (lane & 16) ? id1 : S.id[b0];
        if (lane < 16 && idA >= 0 && r != 0.0f)
          atomicAdd(dsplats + 9 * (int64_t)idA + (lane & 7), r * bwd_field_scale(lane & 7));
        if ((lane & 15) == 1 && idB >= 0 && r9 != 0.0f) atomicAdd(dsplats + 9 * (int64_t)idB + 8, r9);
#else
        const float r = warp_reduce16_transpose(u, lane);
        const float r9 = warp_reduce2_transpose(v0[8], v1[8], lane);
        const int id = (lane & 16) ? id1 : S.id[b0];
        if (id >= 0) {
          float *d = dsplats + 9 * (int64_t)id;
          if ((lane & 1) == 0 && r != 0.0f) atomicAdd(d + ((lane >> 1) & 7), r * bwd_field_scale((lane >> 1) & 7));
          if ((lane & 15) == 1 && r9 != 0.0f) atomicAdd(d + 8, r9);
        }
#endif
      }
    }
    __syncwarp();
  }
}

#ifdef TGS_BWD_CHK_NOINLINE  // A/B builds: the float64-resolving tile body out of line
template <bool kExact, int kP>
__device__ __noinline__ void bwd16p_tile_chk(
    WStage *SW, float *RB, int tile, const float4 *__restrict__ splats, const float4 *__restrict__ exact,
    const int32_t *__restrict__ offsets, const int32_t *__restrict__ ids, int W, int H, int tiles_x, int row_begin,
    float bg0, float bg1, float bg2, const float *__restrict__ transmit, const int32_t *__restrict__ last_pos,
    const float *__restrict__ dimage, float *__restrict__ dsplats) {
  bwd16p_tile<kExact, kP, false>(SW, RB, tile, splats, exact, offsets, ids, W, H, tiles_x, row_begin, bg0, bg1, bg2,
                                 transmit, last_pos, dimage, dsplats, nullptr);
}
#endif

// With exception lists (exc != NULL) a tile the forward flagged in ovf (a pixel with two
// exceptions, or a clamped one) takes the float64-resolving body instead — in the same
// launch, so the few flagged tiles (4-16 of 8,160 per c3 view) add no serial tail.
template <bool kExact, int kP>
__global__ void __launch_bounds__(128 / kP, kExact ? TGS_BWD16_MINB * kP : 1) k_blend_bwd16p(
    const float4 *__restrict__ splats, const float4 *__restrict__ exact, const int32_t *__restrict__ offsets,
    const int32_t *__restrict__ ids, int W, int H, int tiles_x, int row_begin, float bg0, float bg1, float bg2,
    const float *__restrict__ transmit, const int32_t *__restrict__ last_pos, const float *__restrict__ dimage,
    float *__restrict__ dsplats, const int32_t *__restrict__ order, const int32_t *__restrict__ exc,
    const uint32_t *__restrict__ ovf) {
  __shared__ WStage SW[4 / kP];
  __shared__ __align__(16) float RB[TGS_BWD_SMEM_RED ? (4 / kP) * kRedFloats : 4];  // warp_reduce16_smem slots
  const int tile = order ? __ldg(order + blockIdx.x) : (int)blockIdx.x;
  if (kExact && exc && !__ldg(ovf + 1 + tile))
    bwd16p_tile<kExact, kP, true>(SW, RB, tile, splats, exact, offsets, ids, W, H, tiles_x, row_begin, bg0, bg1, bg2,
                                  transmit, last_pos, dimage, dsplats, exc);
  else
#ifdef TGS_BWD_CHK_NOINLINE
    bwd16p_tile_chk<kExact, kP>(SW, RB, tile, splats, exact, offsets, ids, W, H, tiles_x, row_begin, bg0, bg1, bg2,
                                transmit, last_pos, dimage, dsplats);
#else
    bwd16p_tile<kExact, kP, false>(SW, RB, tile, splats, exact, offsets, ids, W, H, tiles_x, row_begin, bg0, bg1, bg2,
                                   transmit, last_pos, dimage, dsplats, nullptr);
#endif
}

// _kernels.py:184-241: same walk as the forward, writing (gid, a*T) per blended entry
__global__ void k_blend_records(const float4 *__restrict__ splats, const float4 *__restrict__ exact,
                                const int32_t *__restrict__ offsets,
                                const int32_t *__restrict__ ids, int W, int H, int ts, int tiles_x,
                                const int64_t *__restrict__ pix_off, int32_t *__restrict__ rec_g,
                                float *__restrict__ rec_w) {
  const int tile = blockIdx.x;
  const int ty = tile / tiles_x, tx = tile % tiles_x;
  const int t = threadIdx.x;
  int lx, ly;
  pixel_of(t, ts, lx, ly);
  const int px = tx * ts + lx, py = ty * ts + ly;
  if (t >= ts * ts || px >= W || py >= H) return;
  const int start = offsets[tile], stop = offsets[tile + 1];
  int64_t pos = pix_off[py * W + px];
  float T = 1.0f;
  for (int k = start; k < stop; ++k) {
    if (T < kTTerm) break;
    const int g = ids[k];
    const float4 a = splats[3 * g], b = splats[3 * g + 1];
    const float e2 = exponent2(prescaled_conic(a, b), (float)px - a.x, (float)py - a.y);
    float al = __fmul_rn(b.y, ex2_approx(e2));
    if (!decide_pair(e2, al, load_cut(exact, g, b.y), splats, exact, g, (float)px, (float)py)) continue;
    al = fminf(al, kAlphaMax);
    rec_g[pos] = g;
    rec_w[pos] = al * T;
    ++pos;
    T = __fmul_rn(T, __fsub_rn(1.0f, al));
  }
}

// ---------------------------------------------------------------------------
// Heaviest-first tile order for the blend kernels (longest-processing-time-first
// scheduling): CTAs are dispatched roughly in blockIdx order, so mapping blockIdx
// to tiles sorted by descending list length leaves the short tiles for the tail.
// Classes are floor(log2(length)), heaviest class first; the order inside a class
// is arbitrary (it only affects scheduling).  order[ntiles .. ntiles+63] holds the
// class counts and cursors.
__device__ __forceinline__ int order_class(int32_t len) {
  return len > 0 ? __clz(len) : 31;  // 31 - floor(log2(len)): 0 = heaviest
}

__global__ void __launch_bounds__(256) k_order_hist(const int32_t *__restrict__ offsets, int ntiles,
                                                    uint32_t *__restrict__ cnt) {
  __shared__ uint32_t h[32];
  if (threadIdx.x < 32) h[threadIdx.x] = 0u;
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < ntiles) atomicAdd(&h[order_class(__ldg(offsets + t + 1) - __ldg(offsets + t))], 1u);
  __syncthreads();
  if (threadIdx.x < 32 && h[threadIdx.x]) atomicAdd(cnt + threadIdx.x, h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_order_scatter(const int32_t *__restrict__ offsets, int ntiles,
                                                       uint32_t *__restrict__ cnt, int32_t *__restrict__ order) {
  __shared__ uint32_t base[32], local[32], resv[32];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (threadIdx.x < 32) {  // class bases: exclusive scan of the global counts (heaviest first)
    const uint32_t c = cnt[threadIdx.x];
    uint32_t v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if ((int)threadIdx.x >= o) v += y;
    }
    base[threadIdx.x] = v - c;
    local[threadIdx.x] = 0u;
  }
  __syncthreads();
  int cls = 0;
  uint32_t r = 0;
  if (t < ntiles) {
    cls = order_class(__ldg(offsets + t + 1) - __ldg(offsets + t));
    r = atomicAdd(&local[cls], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 32 && local[threadIdx.x]) resv[threadIdx.x] = atomicAdd(cnt + 32 + threadIdx.x, local[threadIdx.x]);
  __syncthreads();
  if (t < ntiles) order[base[cls] + resv[cls] + r] = t;
}

inline bool blend_args(const tgs_camera *cam, const tgs_settings *s, int rb, int re, int &tiles_x, int &ntiles) {
  if (!cam || !s || s->tile_size < 1 || s->tile_size > 32) return false;
  tiles_x = (cam->width + s->tile_size - 1) / s->tile_size;
  const int tiles_y = (cam->height + s->tile_size - 1) / s->tile_size;
  if (rb < 0 || re > tiles_y || rb > re) return false;
  ntiles = (re - rb) * tiles_x;
  return true;
}

inline int tile_size_guard(int ts) { return ts < 1 ? 1 : ts; }

}  // namespace tgs

using namespace tgs;

// Profiling build only (-DTGS_COUNT_EXACT): the number of (pixel, splat) pairs decided in
// float64 since the last reset.  Returns TGS_ERR_UNSUPPORTED in a normal build.
extern "C" int tgs_debug_exact_pairs(unsigned long long *count, int32_t reset) {
#ifdef TGS_COUNT_EXACT
  if (count && cudaMemcpyFromSymbol(count, g_exact_pairs, sizeof(*count)) != cudaSuccess) return TGS_ERR_CUDA;
  if (reset) {
    const unsigned long long z = 0;
    if (cudaMemcpyToSymbol(g_exact_pairs, &z, sizeof(z)) != cudaSuccess) return TGS_ERR_CUDA;
  }
  return TGS_OK;
#else
  (void)count;
  (void)reset;
  return TGS_ERR_UNSUPPORTED;
#endif
}

extern "C" int tgs_blend_forward(const float *splats, const float *exact, const int32_t *tile_offsets,
                                 const int32_t *sorted_ids,
                                 const tgs_camera *cam, const tgs_settings *s, int32_t row_begin, int32_t row_end,
                                 float *image, float *transmit, float *weight_sum, int32_t *n_contrib,
                                 int32_t *last_pos, int32_t *hits, int32_t *exceptions, uint32_t *exc_overflow,
                                 const int32_t *tile_order, tgs_stream_t stream) {
  int tiles_x, ntiles;
  if (!blend_args(cam, s, row_begin, row_end, tiles_x, ntiles)) return TGS_ERR_INVALID;
  if ((reinterpret_cast<uintptr_t>(splats) | reinterpret_cast<uintptr_t>(exact)) & 15) return TGS_ERR_INVALID;
  if (!exceptions != !exc_overflow || (exceptions && (!exact || s->tile_size != 16))) return TGS_ERR_INVALID;
  if (ntiles == 0) return TGS_OK;
  const float4 *ex = reinterpret_cast<const float4 *>(exact);
  if (exc_overflow) {
    const cudaError_t e = cudaMemsetAsync(exc_overflow, 0, (1 + (size_t)ntiles) * sizeof(uint32_t), as_stream(stream));
    if (e != cudaSuccess) return cuda_status(e);
  }
  if (s->tile_size == 16) {
    auto kern = ex ? (exceptions ? (hits ? k_blend_fwd16w<true, true, true> : k_blend_fwd16w<true, false, true>)
                                 : (hits ? k_blend_fwd16w<true, true, false> : k_blend_fwd16w<true, false, false>))
                   : (hits ? k_blend_fwd16w<false, true, false> : k_blend_fwd16w<false, false, false>);
    kern<<<ntiles, kT16Threads, 0, as_stream(stream)>>>(
        reinterpret_cast<const float4 *>(splats), ex, tile_offsets, sorted_ids, cam->width, cam->height, tiles_x,
        row_begin, s->background[0], s->background[1], s->background[2], image, transmit, weight_sum, n_contrib,
        last_pos, hits, tile_order, exceptions, exc_overflow);
    return launch_status();
  }
  const int B = (s->tile_size * s->tile_size + 31) / 32 * 32;  // whole warps; extra lanes are idle pixels
  (B <= 256 ? k_blend_fwd<256> : k_blend_fwd<1024>)<<<ntiles, B, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4 *>(splats), ex, tile_offsets, sorted_ids, cam->width, cam->height, s->tile_size,
      tiles_x, row_begin, s->background[0], s->background[1], s->background[2], image, transmit, weight_sum,
      n_contrib, last_pos, hits);
  return launch_status();
}

extern "C" int tgs_blend_records(const float *splats, const float *exact, const int32_t *tile_offsets,
                                 const int32_t *sorted_ids,
                                 const tgs_camera *cam, const tgs_settings *s, const int64_t *pixel_offsets,
                                 int32_t *rec_gauss, float *rec_weight, tgs_stream_t stream) {
  int tiles_x, ntiles;
  if (!cam || !s) return TGS_ERR_INVALID;
  const int tiles_y = (cam->height + s->tile_size - 1) / tile_size_guard(s->tile_size);
  if (!blend_args(cam, s, 0, tiles_y, tiles_x, ntiles)) return TGS_ERR_INVALID;
  if (ntiles == 0) return TGS_OK;
  const int B = (s->tile_size * s->tile_size + 31) / 32 * 32;
  if ((reinterpret_cast<uintptr_t>(splats) | reinterpret_cast<uintptr_t>(exact)) & 15) return TGS_ERR_INVALID;
  k_blend_records<<<ntiles, B, 0, as_stream(stream)>>>(reinterpret_cast<const float4 *>(splats),
                                                       reinterpret_cast<const float4 *>(exact), tile_offsets,
                                                       sorted_ids, cam->width, cam->height, s->tile_size, tiles_x,
                                                       pixel_offsets, rec_gauss, rec_weight);
  return launch_status();
}

extern "C" int tgs_blend_backward(const float *splats, const float *exact, const int32_t *tile_offsets,
                                  const int32_t *sorted_ids,
                                  const tgs_camera *cam, const tgs_settings *s, int32_t row_begin, int32_t row_end,
                                  const float *transmit, const int32_t *last_pos, const int32_t *exceptions,
                                  const uint32_t *exc_overflow, const float *dimage,
                                  float *dsplats, const int32_t *tile_order, tgs_stream_t stream) {
  int tiles_x, ntiles;
  if (!blend_args(cam, s, row_begin, row_end, tiles_x, ntiles)) return TGS_ERR_INVALID;
  if ((reinterpret_cast<uintptr_t>(splats) | reinterpret_cast<uintptr_t>(exact)) & 15) return TGS_ERR_INVALID;
  if (!exceptions != !exc_overflow || (exceptions && (!exact || s->tile_size != 16))) return TGS_ERR_INVALID;
  if (ntiles == 0) return TGS_OK;
  const float4 *ex = reinterpret_cast<const float4 *>(exact);
  if (s->tile_size == 16) {
#if TGS_BWD16_PAIRS == 2
    cudaStream_t st = as_stream(stream);
    const float4 *sp = reinterpret_cast<const float4 *>(splats);
    (ex ? k_blend_bwd16p<true, 2> : k_blend_bwd16p<false, 2>)<<<ntiles, 64, 0, st>>>(
        sp, ex, tile_offsets, sorted_ids, cam->width, cam->height, tiles_x, row_begin, s->background[0],
        s->background[1], s->background[2], transmit, last_pos, dimage, dsplats, tile_order, exceptions,
        exc_overflow);
    return launch_status();
#endif
    (ex ? k_blend_bwd16w<true> : k_blend_bwd16w<false>)<<<ntiles, kT16Threads, 0, as_stream(stream)>>>(
        reinterpret_cast<const float4 *>(splats), ex, tile_offsets, sorted_ids, cam->width, cam->height, tiles_x,
        row_begin, s->background[0], s->background[1], s->background[2], transmit, last_pos, dimage, dsplats,
        tile_order);
    return launch_status();
  }
  const int B = (s->tile_size * s->tile_size + 31) / 32 * 32;
  (B <= 256 ? k_blend_bwd<256> : k_blend_bwd<1024>)<<<ntiles, B, 0, as_stream(stream)>>>(
      reinterpret_cast<const float4 *>(splats), ex, tile_offsets, sorted_ids, cam->width, cam->height, s->tile_size,
      tiles_x, row_begin, s->background[0], s->background[1], s->background[2], transmit, last_pos, dimage,
      dsplats, nullptr);
  return launch_status();
}

static size_t det_ws(int64_t n, int64_t num_instances, size_t *parts) {
  Carve c(nullptr);
  const size_t N = (size_t)tmax<int64_t>(n, 1), I = (size_t)tmax<int64_t>(num_instances, 1);
  parts[0] = c.off; c.take<float>(I * 9);                  // partials per list position
  parts[1] = c.off; c.take<uint32_t>(I);                   // inverse map
  parts[2] = c.off; c.take<uint32_t>(N);                   // per-Gaussian counts -> offsets
  parts[3] = c.off; c.take<uint32_t>(ceil_div<size_t>(N, 4096) + 1);  // scan look-back + ticket
  parts[4] = c.off;
  return c.off;
}

extern "C" int tgs_blend_backward_deterministic_workspace(int64_t n, int64_t num_instances, size_t *bytes) {
  if (n < 0 || num_instances < 0 || !bytes) return TGS_ERR_INVALID;
  size_t parts[5];
  *bytes = det_ws(n, num_instances, parts);
  return TGS_OK;
}

extern "C" int tgs_blend_backward_deterministic(const float *splats, const float *exact,
                                                const int32_t *tiles_touched, int64_t n,
                                                const int32_t *tile_offsets, const int32_t *sorted_ids,
                                                int64_t num_instances, const tgs_camera *cam, const tgs_settings *s,
                                                int32_t row_begin, int32_t row_end, const float *transmit,
                                                const int32_t *last_pos, const float *dimage, float *dsplats,
                                                void *workspace, tgs_stream_t stream) {
  int tiles_x, ntiles;
  if (!blend_args(cam, s, row_begin, row_end, tiles_x, ntiles)) return TGS_ERR_INVALID;
  if ((reinterpret_cast<uintptr_t>(splats) | reinterpret_cast<uintptr_t>(exact)) & 15) return TGS_ERR_INVALID;
  if (n < 0 || num_instances < 0 || num_instances >= ((int64_t)1 << 30) || !workspace || !tiles_touched)
    return TGS_ERR_INVALID;
  if (ntiles == 0 || n == 0) return TGS_OK;
  cudaStream_t st = as_stream(stream);
  size_t parts[5];
  det_ws(n, num_instances, parts);
  char *w = static_cast<char *>(workspace);
  float *partial = reinterpret_cast<float *>(w + parts[0]);
  uint32_t *inv = reinterpret_cast<uint32_t *>(w + parts[1]);
  uint32_t *cnt = reinterpret_cast<uint32_t *>(w + parts[2]);
  uint32_t *status = reinterpret_cast<uint32_t *>(w + parts[3]);
  const int tiles_y = (cam->height + s->tile_size - 1) / s->tile_size;
  const int B = (s->tile_size * s->tile_size + 31) / 32 * 32;
  (B <= 256 ? k_blend_bwd<256> : k_blend_bwd<1024>)<<<ntiles, B, 0, st>>>(
      reinterpret_cast<const float4 *>(splats), reinterpret_cast<const float4 *>(exact), tile_offsets, sorted_ids, cam->width, cam->height, s->tile_size,
      tiles_x, row_begin, s->background[0], s->background[1], s->background[2], transmit, last_pos, dimage, dsplats,
      partial);
  const unsigned gn = (unsigned)ceil_div<int64_t>(n, 256);
  k_inst_count<<<gn, 256, 0, st>>>(splats, tiles_touched, n, cam->width, cam->height, s->tile_size, tiles_x, tiles_y,
                                   row_begin, row_end, cnt);
  const unsigned nt = (unsigned)ceil_div<int64_t>(n, 4096);
  cudaMemsetAsync(status, 0, ((size_t)nt + 1) * 4, st);
  k_det_scan<<<nt, 256, 0, st>>>(cnt, n, status, status + nt);
  k_det_inverse<<<ntiles, 256, 0, st>>>(splats, tile_offsets, sorted_ids, cnt, cam->width, cam->height,
                                        s->tile_size, tiles_x, tiles_y, row_begin, row_end, inv);
  k_det_reduce<<<gn, 256, 0, st>>>(cnt, inv, partial, n, num_instances, dsplats);
  return launch_status();
}

extern "C" int tgs_tile_order(const int32_t *tile_offsets, int32_t ntiles, int32_t *order, tgs_stream_t stream) {
  if (ntiles < 0 || !tile_offsets || !order) return TGS_ERR_INVALID;
  if (ntiles == 0) return TGS_OK;
  cudaStream_t st = as_stream(stream);
  uint32_t *cnt = reinterpret_cast<uint32_t *>(order + ntiles);  // 32 counts + 32 cursors
  cudaMemsetAsync(cnt, 0, 64 * sizeof(uint32_t), st);
  const unsigned g = (unsigned)ceil_div<int64_t>(ntiles, 256);
  k_order_hist<<<g, 256, 0, st>>>(tile_offsets, ntiles, cnt);
  k_order_scatter<<<g, 256, 0, st>>>(tile_offsets, ntiles, cnt, order);
  return launch_status();
}
