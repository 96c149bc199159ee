// oracle.cpp — CPU restatement of the reference rasterizer hot path.
//
// TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, imports or
// executes this file; only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load liboracle.so (through oracle/oracle.py)
// as the checker and as the timed CPU baseline.
//
// Every function is templated on the real type R:
//   R = double  restates the reference's float64 arithmetic step by step; it is
//               pinned against golden vectors produced by the reference itself
//               (tests/golden/make_golden.py, tests/test_oracle_golden.py).
//   R = float   is the same algorithm in float32 and defines the fp32 semantics
//               the CUDA path must reproduce BIT-EXACTLY for visibility, radii,
//               tiles_touched and the sorted tile lists (north star).  Its only
//               deviations from a literal float transcription are the documented
//               ones the CUDA kernels share: hard masks and the alpha-skip gate are
//               compared in logit space (exact w.r.t. the float64 reference), and
//               exp() is the explicit fmaf-based sem_expf below, so host and device
//               produce identical bits.
//
// Build: oracle/Makefile (g++ -O2 -ffp-contract=off, no fast-math).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// constants (rasterizer.py:38-41, sh.py:14-31)
constexpr double kAlphaSkip = 1.0 / 255.0;
constexpr double kAlphaMax = 0.99;
constexpr double kEMin = -4.5;
constexpr double kTTerm = 1e-4;
constexpr double SH_C0 = 0.28209479177387814;
constexpr double SH_C1 = 0.4886025119029199;
constexpr double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                             -1.0925484305920792, 0.5462742152960396};
constexpr double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                             0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                             -0.5900435899266435};

// float32 exp with fully specified rounding: Cody-Waite reduction by ln2 split
// in hi/lo, degree-7 Taylor polynomial in Horner form with fmaf, exact 2^k
// scaling.  exp(x) := 0 for x <= -87, +inf for x > 88.72.  <= 2 ulp error.
// The CUDA kernels evaluate the identical operation sequence (csrc/tgs_math.cuh).
static float sem_expf(float x) {
  if (x != x) return x;
  if (!(x > -87.0f)) return 0.0f;
  if (x > 88.72f) return INFINITY;
  const float k = rintf(x * 1.44269502f);
  float r = fmaf(k, -0.693145751953125f, x);
  r = fmaf(k, -1.42860677e-6f, r);
  float p = 1.98412698e-4f;
  p = fmaf(p, r, 1.38888889e-3f);
  p = fmaf(p, r, 8.33333333e-3f);
  p = fmaf(p, r, 4.16666667e-2f);
  p = fmaf(p, r, 1.66666667e-1f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  const int ki = (int)k;
  const int k1 = ki / 2, k2 = ki - k1;
  uint32_t b1 = (uint32_t)(k1 + 127) << 23, b2 = (uint32_t)(k2 + 127) << 23;
  float s1, s2;
  std::memcpy(&s1, &b1, 4);
  std::memcpy(&s2, &b2, 4);
  return (p * s1) * s2;
}

template <typename R> struct M;
template <> struct M<double> {
  static double exp(double x) { return std::exp(x); }
  static double sqrt(double x) { return std::sqrt(x); }
  static double floor(double x) { return std::floor(x); }
  static constexpr double det_min = 1e-300;  // geometry.py:176
};
template <> struct M<float> {
  static float exp(float x) { return sem_expf(x); }
  static float sqrt(float x) { return std::sqrt(x); }
  static float floor(float x) { return std::floor(x); }
  static constexpr float det_min = 0.0f;  // 1e-300 underflows in float32
};

template <typename R> static R sigmoid(R x) { return R(1) / (R(1) + M<R>::exp(-x)); }

}  // namespace

extern "C" {

// Camera/settings as plain doubles; the float instantiation rounds them once,
// exactly like cameras.Camera.native_fields() does for the CUDA path.
struct oracle_camera {
  double fx, fy, cx, cy;
  double R[9];
  double t[3];
  double center[3];
  int32_t width, height;
};
struct oracle_settings {
  double lowpass_s, near_plane;
  double mask_threshold, sh_mask_threshold;         // float64 path (masking.py:21-25)
  double mask_logit_min, sh_mask_logit_min, opacity_logit_min;  // float32 path
  double background[3];
  int32_t active_sh_degree, tile_size, compute_sh_rest_grads, reserved;
};
struct oracle_cloud {
  const double *positions, *log_scales, *rotations, *opacity_logits;
  const double *sh_dc, *sh_rest, *mask_logits, *sh_mask_logits;
  int64_t n;
};

}  // extern "C"

namespace {

template <typename R> struct Cam {
  R fx, fy, cx, cy, Rc[9], t[3], c[3];
  int W, H;
  explicit Cam(const oracle_camera &o) {
    fx = R(o.fx); fy = R(o.fy); cx = R(o.cx); cy = R(o.cy);
    for (int i = 0; i < 9; ++i) Rc[i] = R(o.R[i]);
    for (int i = 0; i < 3; ++i) { t[i] = R(o.t[i]); c[i] = R(o.center[i]); }
    W = o.width; H = o.height;
  }
};

// sh.py:47-74 — basis values for bands 0..3 at unit direction (x, y, z)
template <typename R> static void sh_basis(R x, R y, R z, R b[16]) {
  b[0] = R(SH_C0);
  b[1] = R(-SH_C1) * y;
  b[2] = R(SH_C1) * z;
  b[3] = R(-SH_C1) * x;
  const R xx = x * x, yy = y * y, zz = z * z;
  b[4] = R(SH_C2[0]) * x * y;
  b[5] = R(SH_C2[1]) * y * z;
  b[6] = R(SH_C2[2]) * (R(2) * zz - xx - yy);
  b[7] = R(SH_C2[3]) * x * z;
  b[8] = R(SH_C2[4]) * (xx - yy);
  b[9] = R(SH_C3[0]) * y * (R(3) * xx - yy);
  b[10] = R(SH_C3[1]) * x * y * z;
  b[11] = R(SH_C3[2]) * y * (R(4) * zz - xx - yy);
  b[12] = R(SH_C3[3]) * z * (R(2) * zz - R(3) * xx - R(3) * yy);
  b[13] = R(SH_C3[4]) * x * (R(4) * zz - xx - yy);
  b[14] = R(SH_C3[5]) * z * (xx - yy);
  b[15] = R(SH_C3[6]) * x * (xx - R(3) * yy);
}

// sh.py:77-120 — d(basis)/d(dir), rows 1..15 used
template <typename R> static void sh_basis_grad(R x, R y, R z, R g[16][3]) {
  for (int k = 0; k < 16; ++k) g[k][0] = g[k][1] = g[k][2] = R(0);
  g[1][1] = R(-SH_C1);
  g[2][2] = R(SH_C1);
  g[3][0] = R(-SH_C1);
  g[4][0] = R(SH_C2[0]) * y;
  g[4][1] = R(SH_C2[0]) * x;
  g[5][1] = R(SH_C2[1]) * z;
  g[5][2] = R(SH_C2[1]) * y;
  g[6][0] = R(SH_C2[2]) * (R(-2) * x);
  g[6][1] = R(SH_C2[2]) * (R(-2) * y);
  g[6][2] = R(SH_C2[2]) * (R(4) * z);
  g[7][0] = R(SH_C2[3]) * z;
  g[7][2] = R(SH_C2[3]) * x;
  g[8][0] = R(SH_C2[4]) * (R(2) * x);
  g[8][1] = R(SH_C2[4]) * (R(-2) * y);
  const R xx = x * x, yy = y * y, zz = z * z;
  g[9][0] = R(SH_C3[0]) * R(6) * x * y;
  g[9][1] = R(SH_C3[0]) * (R(3) * xx - R(3) * yy);
  g[10][0] = R(SH_C3[1]) * y * z;
  g[10][1] = R(SH_C3[1]) * x * z;
  g[10][2] = R(SH_C3[1]) * x * y;
  g[11][0] = R(SH_C3[2]) * (R(-2) * x * y);
  g[11][1] = R(SH_C3[2]) * (R(4) * zz - xx - R(3) * yy);
  g[11][2] = R(SH_C3[2]) * (R(8) * y * z);
  g[12][0] = R(SH_C3[3]) * (R(-6) * x * z);
  g[12][1] = R(SH_C3[3]) * (R(-6) * y * z);
  g[12][2] = R(SH_C3[3]) * (R(6) * zz - R(3) * xx - R(3) * yy);
  g[13][0] = R(SH_C3[4]) * (R(4) * zz - R(3) * xx - yy);
  g[13][1] = R(SH_C3[4]) * (R(-2) * x * y);
  g[13][2] = R(SH_C3[4]) * (R(8) * x * z);
  g[14][0] = R(SH_C3[5]) * (R(2) * x * z);
  g[14][1] = R(SH_C3[5]) * (R(-2) * y * z);
  g[14][2] = R(SH_C3[5]) * (xx - yy);
  g[15][0] = R(SH_C3[6]) * (R(3) * xx - R(3) * yy);
  g[15][1] = R(SH_C3[6]) * (R(-6) * x * y);
}

// band of rest coefficient k (sh.py:34)
static inline int band_of(int k) { return k < 3 ? 0 : (k < 8 ? 1 : 2); }

template <typename R> struct Masks {
  R gauss;      // hard Gaussian mask M
  R band[3];    // hard SH band masks
  bool alpha_ok;  // sigmoid(o) * M >= 1/255
};

template <typename R>
static Masks<R> eval_masks(const oracle_settings &s, double m, const double *msh, double o);

template <> Masks<double> eval_masks<double>(const oracle_settings &s, double m, const double *msh, double o) {
  Masks<double> r;  // masking.py:21-25, rasterizer.py:169-178
  r.gauss = sigmoid<double>(m) > s.mask_threshold ? 1.0 : 0.0;
  for (int l = 0; l < 3; ++l) r.band[l] = sigmoid<double>(msh[l]) > s.sh_mask_threshold ? 1.0 : 0.0;
  r.alpha_ok = sigmoid<double>(o) * r.gauss >= kAlphaSkip;
  return r;
}
template <> Masks<float> eval_masks<float>(const oracle_settings &s, double m, const double *msh, double o) {
  Masks<float> r;  // logit-space comparisons, thresholds rounded by the caller
  const float mf = float(m), of = float(o);
  r.gauss = mf > float(s.mask_logit_min) ? 1.0f : 0.0f;
  for (int l = 0; l < 3; ++l) r.band[l] = float(msh[l]) > float(s.sh_mask_logit_min) ? 1.0f : 0.0f;
  r.alpha_ok = r.gauss > 0.0f && of >= float(s.opacity_logit_min);
  return r;
}

// per-Gaussian forward quantities shared by the forward and backward oracles
template <typename R> struct Fwd {
  Masks<R> mk;
  R s_raw[3], sc[3];     // exp(log_scale), masked scale
  R qn[4], qnorm;        // unit quaternion, raw norm
  R Rg[9];               // rotation (geometry.py:28-41)
  R S[9];                // covariance (geometry.py:74-77)
  R t[3];                // camera-space mean
  R Mj[6];               // J @ Rc
  R mean[2], c00, c01, c11, det, conic[3], radius, area;
  bool valid, ok, visible;
  R dir[3], dnorm;       // view direction, max(|x - c|, 1e-12)
  R col[3], pre[3];      // clamped and pre-clamp colour
  bool degenerate;
};

template <typename R>
static Fwd<R> forward_one(const oracle_cloud &cl, int64_t i, const Cam<R> &cam, const oracle_settings &s) {
  Fwd<R> f;
  f.mk = eval_masks<R>(s, cl.mask_logits[i], cl.sh_mask_logits + 3 * i, cl.opacity_logits[i]);
  const R Mg = f.mk.gauss;
  for (int k = 0; k < 3; ++k) {
    f.s_raw[k] = M<R>::exp(R(cl.log_scales[3 * i + k]));
    f.sc[k] = f.s_raw[k] * Mg;
  }
  // normalize_quaternions (geometry.py:19-25)
  const R qw = R(cl.rotations[4 * i]), qx = R(cl.rotations[4 * i + 1]);
  const R qy = R(cl.rotations[4 * i + 2]), qz = R(cl.rotations[4 * i + 3]);
  f.qnorm = M<R>::sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  f.degenerate = f.qnorm < R(1e-12);
  const R w = qw / f.qnorm, x = qx / f.qnorm, y = qy / f.qnorm, z = qz / f.qnorm;
  f.qn[0] = w; f.qn[1] = x; f.qn[2] = y; f.qn[3] = z;
  R *Rg = f.Rg;
  Rg[0] = R(1) - R(2) * (y * y + z * z);
  Rg[1] = R(2) * (x * y - w * z);
  Rg[2] = R(2) * (x * z + w * y);
  Rg[3] = R(2) * (x * y + w * z);
  Rg[4] = R(1) - R(2) * (x * x + z * z);
  Rg[5] = R(2) * (y * z - w * x);
  Rg[6] = R(2) * (x * z - w * y);
  Rg[7] = R(2) * (y * z + w * x);
  Rg[8] = R(1) - R(2) * (x * x + y * y);
  R L[9];
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) L[3 * r + k] = Rg[3 * r + k] * f.sc[k];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      f.S[3 * a + b] = L[3 * a] * L[3 * b] + L[3 * a + 1] * L[3 * b + 1] + L[3 * a + 2] * L[3 * b + 2];
  // project_gaussians (geometry.py:138-195)
  const R px = R(cl.positions[3 * i]), py = R(cl.positions[3 * i + 1]), pz = R(cl.positions[3 * i + 2]);
  for (int r = 0; r < 3; ++r)
    f.t[r] = px * cam.Rc[3 * r] + py * cam.Rc[3 * r + 1] + pz * cam.Rc[3 * r + 2] + cam.t[r];
  const R tz = f.t[2];
  f.valid = tz > R(s.near_plane);
  f.mean[0] = cam.fx * f.t[0] / tz + cam.cx;
  f.mean[1] = cam.fy * f.t[1] / tz + cam.cy;
  const R tz2 = tz * tz;
  const R J00 = cam.fx / tz, J02 = -cam.fx * f.t[0] / tz2;
  const R J11 = cam.fy / tz, J12 = -cam.fy * f.t[1] / tz2;
  for (int j = 0; j < 3; ++j) {
    f.Mj[j] = J00 * cam.Rc[j] + J02 * cam.Rc[6 + j];
    f.Mj[3 + j] = J11 * cam.Rc[3 + j] + J12 * cam.Rc[6 + j];
  }
  R A[6];  // (M Sigma), rows 0..1
  for (int r = 0; r < 2; ++r)
    for (int j = 0; j < 3; ++j)
      A[3 * r + j] = f.Mj[3 * r] * f.S[j] + f.Mj[3 * r + 1] * f.S[3 + j] + f.Mj[3 * r + 2] * f.S[6 + j];
  const R lp = R(s.lowpass_s);
  f.c00 = A[0] * f.Mj[0] + A[1] * f.Mj[1] + A[2] * f.Mj[2] + lp;
  f.c01 = A[0] * f.Mj[3] + A[1] * f.Mj[4] + A[2] * f.Mj[5];
  f.c11 = A[3] * f.Mj[3] + A[4] * f.Mj[4] + A[5] * f.Mj[5] + lp;
  f.det = f.c00 * f.c11 - f.c01 * f.c01;
  f.ok = f.det > M<R>::det_min;
  const R inv = f.ok ? R(1) / f.det : R(0);
  f.conic[0] = f.c11 * inv;
  f.conic[1] = -f.c01 * inv;
  f.conic[2] = f.c00 * inv;
  const R mid = R(0.5) * (f.c00 + f.c11);
  const R lam = mid + M<R>::sqrt(std::max(mid * mid - f.det, R(0)));
  f.radius = R(3) * M<R>::sqrt(std::max(lam, R(0)));
  f.area = R(9.0 * M_PI) * M<R>::sqrt(std::max(f.det, R(0)));
  f.visible = f.valid && f.ok && f.mk.alpha_ok;
  // view direction (rasterizer.py:190-193) and SH colour (sh.py:135-161)
  R d[3];
  for (int k = 0; k < 3; ++k) d[k] = R(cl.positions[3 * i + k]) - cam.c[k];
  const R nrm = M<R>::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  f.dnorm = std::max(nrm, R(1e-12));
  for (int k = 0; k < 3; ++k) f.dir[k] = d[k] / f.dnorm;
  R b[16];
  sh_basis<R>(f.dir[0], f.dir[1], f.dir[2], b);
  const int deg = s.active_sh_degree;
  const int K = (deg + 1) * (deg + 1) - 1;
  for (int c = 0; c < 3; ++c) {
    R acc = R(0);
    for (int k = 0; k < K; ++k)
      acc = acc + b[k + 1] * (R(cl.sh_rest[45 * i + 3 * k + c]) * f.mk.band[band_of(k)]);
    R col = R(SH_C0) * R(cl.sh_dc[3 * i + c]) + R(0.5);
    if (deg > 0) col = col + acc;
    f.pre[c] = col;
    f.col[c] = std::max(col, R(0));
  }
  return f;
}

// bin_tiles rect/gate (rasterizer.py:112-128)
template <typename R>
static int64_t tile_rect(R mx, R my, R r, int W, int H, int ts, int *x0, int *y0, int *x1, int *y1) {
  const int tx = (W + ts - 1) / ts, ty = (H + ts - 1) / ts;
  auto cl = [](R v, int hi) {
    if (!(v >= R(0))) v = R(0);
    if (v > R(hi)) v = R(hi);
    return (int)v;
  };
  *x0 = cl(M<R>::floor((mx - r) / R(ts)), tx - 1);
  *x1 = cl(M<R>::floor((mx + r) / R(ts)), tx - 1);
  *y0 = cl(M<R>::floor((my - r) / R(ts)), ty - 1);
  *y1 = cl(M<R>::floor((my + r) / R(ts)), ty - 1);
  const bool on = (mx + r >= R(0)) && (mx - r <= R(W - 1)) && (my + r >= R(0)) && (my - r <= R(H - 1)) && (r > R(0));
  return on ? int64_t(*x1 - *x0 + 1) * int64_t(*y1 - *y0 + 1) : 0;
}

// float64 camera-space depth from the float32-valued inputs and the float64 camera:
// the sort key of BOTH instantiations (float32 depths
// collide ~2k times at c2 and would reorder blends relative to the reference).
static double depth64(const oracle_cloud &cl, int64_t i, const oracle_camera &oc) {
  return cl.positions[3 * i] * oc.R[6] + cl.positions[3 * i + 1] * oc.R[7] + cl.positions[3 * i + 2] * oc.R[8] + oc.t[2];
}

template <typename R>
static int preprocess(const oracle_cloud *cl, const oracle_camera *oc, const oracle_settings *s, R *splats,
                      uint8_t *visible, int32_t *tiles, double *depth_key) {
  const Cam<R> cam(*oc);
  int degenerate = 0;
  for (int64_t i = 0; i < cl->n; ++i) {
    const Fwd<R> f = forward_one<R>(*cl, i, cam, *s);
    degenerate |= f.degenerate;
    R *o = splats + 12 * i;
    std::fill(o, o + 12, R(0));
    visible[i] = f.visible;
    tiles[i] = 0;
    if (depth_key) depth_key[i] = f.visible ? depth64(*cl, i, *oc) : 0.0;
    if (!f.visible) continue;
    o[0] = f.mean[0]; o[1] = f.mean[1];
    o[2] = f.conic[0]; o[3] = f.conic[1]; o[4] = f.conic[2];
    o[5] = sigmoid<R>(R(cl->opacity_logits[i])) * f.mk.gauss;
    o[6] = f.col[0]; o[7] = f.col[1]; o[8] = f.col[2];
    o[9] = f.t[2]; o[10] = f.radius; o[11] = f.area;
    int a, b, c, d;
    tiles[i] = (int32_t)tile_rect<R>(f.mean[0], f.mean[1], f.radius, cam.W, cam.H, s->tile_size, &a, &b, &c, &d);
  }
  return degenerate ? 2 : 0;
}

// bin_tiles: emit row-major instances, stable sort by (tile, depth, index)
template <typename R>
static int64_t bin(const R *splats, const int32_t *tiles, const double *depth_key, int64_t n, int W, int H, int ts,
                   int64_t *offsets, int64_t *ids, int64_t capacity) {
  const int tx = (W + ts - 1) / ts, ty = (H + ts - 1) / ts;
  const int64_t T = int64_t(tx) * ty;
  std::vector<std::pair<int64_t, int64_t>> inst;  // (tile, gid)
  for (int64_t g = 0; g < n; ++g) {
    if (tiles[g] == 0) continue;
    int x0, y0, x1, y1;
    const R *o = splats + 12 * g;
    tile_rect<R>(o[0], o[1], o[10], W, H, ts, &x0, &y0, &x1, &y1);
    for (int y = y0; y <= y1; ++y)
      for (int x = x0; x <= x1; ++x) inst.emplace_back(int64_t(y) * tx + x, g);
  }
  std::stable_sort(inst.begin(), inst.end(), [&](const auto &a, const auto &b) {
    if (a.first != b.first) return a.first < b.first;
    const double da = depth_key ? depth_key[a.second] : double(splats[12 * a.second + 9]);
    const double db = depth_key ? depth_key[b.second] : double(splats[12 * b.second + 9]);
    if (da != db) return da < db;
    return a.second < b.second;
  });
  std::fill(offsets, offsets + T + 1, 0);
  for (auto &p : inst) offsets[p.first + 1]++;
  for (int64_t t = 0; t < T; ++t) offsets[t + 1] += offsets[t];
  const int64_t I = (int64_t)inst.size();
  if (ids && I <= capacity)
    for (int64_t j = 0; j < I; ++j) ids[j] = inst[j].second;
  return I;
}

// _kernels.py:12-89
template <typename R>
static void blend_fwd(const R *sp, const int64_t *offsets, const int64_t *ids, int W, int H, int ts,
                      const double *bg, R *image, R *transmit, R *wsum_out, int32_t *n_contrib,
                      int32_t *last_pos, int64_t *hits) {
  const int tx = (W + ts - 1) / ts, ty = (H + ts - 1) / ts;
  for (int tyi = 0; tyi < ty; ++tyi)
    for (int txi = 0; txi < tx; ++txi) {
      const int64_t tid = int64_t(tyi) * tx + txi, start = offsets[tid], stop = offsets[tid + 1];
      for (int py = tyi * ts; py < std::min((tyi + 1) * ts, H); ++py)
        for (int px = txi * ts; px < std::min((txi + 1) * ts, W); ++px) {
          R T = 1, ws = 0, c0 = 0, c1 = 0, c2 = 0;
          int32_t contrib = 0, lastp = 0;
          for (int64_t k = start; k < stop; ++k) {
            if (T < R(kTTerm)) break;
            const int64_t g = ids[k];
            const R *o = sp + 12 * g;
            const R dx = R(px) - o[0], dy = R(py) - o[1];
            const R e = R(-0.5) * (o[2] * dx * dx + o[4] * dy * dy) - o[3] * dx * dy;
            if (e < R(kEMin) || e > R(0)) continue;
            R a = o[5] * M<R>::exp(e);
            if (a < R(kAlphaSkip)) continue;
            if (a > R(kAlphaMax)) a = R(kAlphaMax);
            const R w = a * T;
            c0 += o[6] * w; c1 += o[7] * w; c2 += o[8] * w;
            ws += w;
            T *= R(1) - a;
            contrib += 1;
            lastp = int32_t(k - start + 1);
            if (hits) hits[g] += 1;
          }
          const int64_t p = int64_t(py) * W + px;
          image[3 * p] = c0 + R(bg[0]) * T;
          image[3 * p + 1] = c1 + R(bg[1]) * T;
          image[3 * p + 2] = c2 + R(bg[2]) * T;
          transmit[p] = T; wsum_out[p] = ws; n_contrib[p] = contrib; last_pos[p] = lastp;
        }
    }
}

// _kernels.py:92-181
template <typename R>
static void blend_bwd(const R *sp, const int64_t *offsets, const int64_t *ids, int W, int H, int ts,
                      const double *bg, const R *transmit, const int32_t *last_pos, const R *dimage, R *dsp) {
  const int tx = (W + ts - 1) / ts, ty = (H + ts - 1) / ts;
  for (int tyi = 0; tyi < ty; ++tyi)
    for (int txi = 0; txi < tx; ++txi) {
      const int64_t start = offsets[int64_t(tyi) * tx + txi];
      for (int py = tyi * ts; py < std::min((tyi + 1) * ts, H); ++py)
        for (int px = txi * ts; px < std::min((txi + 1) * ts, W); ++px) {
          const int64_t p = int64_t(py) * W + px;
          const int32_t lastp = last_pos[p];
          if (lastp == 0) continue;
          const R g0 = dimage[3 * p], g1 = dimage[3 * p + 1], g2 = dimage[3 * p + 2];
          if (g0 == R(0) && g1 == R(0) && g2 == R(0)) continue;
          R t_after = transmit[p];
          R s0 = R(bg[0]) * t_after, s1 = R(bg[1]) * t_after, s2 = R(bg[2]) * t_after;
          for (int64_t k = start + lastp - 1; k >= start; --k) {
            const int64_t g = ids[k];
            const R *o = sp + 12 * g;
            const R dx = R(px) - o[0], dy = R(py) - o[1];
            const R e = R(-0.5) * (o[2] * dx * dx + o[4] * dy * dy) - o[3] * dx * dy;
            if (e < R(kEMin) || e > R(0)) continue;
            const R gauss = M<R>::exp(e);
            const R a_raw = o[5] * gauss;
            R a = a_raw;
            if (a > R(kAlphaMax)) a = R(kAlphaMax);
            if (a < R(kAlphaSkip)) continue;
            const R t_before = t_after / (R(1) - a);
            const R inv_om = R(1) / (R(1) - a);
            const R ga = g0 * (o[6] * t_before - s0 * inv_om) + g1 * (o[7] * t_before - s1 * inv_om) +
                         g2 * (o[8] * t_before - s2 * inv_om);
            const R w = a * t_before;
            R *d = dsp + 9 * g;
            d[6] += g0 * w; d[7] += g1 * w; d[8] += g2 * w;
            if (a_raw <= R(kAlphaMax)) {
              d[5] += ga * gauss;
              const R gG = ga * o[5];
              const R v0 = o[2] * dx + o[3] * dy, v1 = o[3] * dx + o[4] * dy;
              d[0] += gG * gauss * v0;
              d[1] += gG * gauss * v1;
              d[2] += gG * gauss * R(0.5) * v0 * v0;
              d[3] += gG * gauss * v0 * v1;
              d[4] += gG * gauss * R(0.5) * v1 * v1;
            }
            s0 += o[6] * w; s1 += o[7] * w; s2 += o[8] * w;
            t_after = t_before;
          }
        }
    }
}

// render_backward chain after the kernel (rasterizer.py:375-419)
template <typename R>
static int preprocess_bwd(const oracle_cloud *cl, const oracle_camera *oc, const oracle_settings *s,
                          const R *dsp, R *gpos, R *gls, R *grot, R *gop, R *gdc, R *grest, R *gmask,
                          R *gshm, R *gm2d) {
  const Cam<R> cam(*oc);
  const int deg = s->active_sh_degree;
  const int K = (deg + 1) * (deg + 1) - 1;
  for (int64_t i = 0; i < cl->n; ++i) {
    const Fwd<R> f = forward_one<R>(*cl, i, cam, *s);
    const R *d = dsp + 9 * i;
    R dm0 = 0, dm1 = 0, g00 = 0, g01 = 0, g11 = 0, da = 0, dcol[3] = {0, 0, 0};
    if (f.visible) {
      dm0 = d[0]; dm1 = d[1]; g00 = d[2]; g01 = d[3]; g11 = d[4]; da = d[5];
      dcol[0] = d[6]; dcol[1] = d[7]; dcol[2] = d[8];
    }
    // --- colour path (sh.py:164-215) ---
    R dcolor[3];
    for (int c = 0; c < 3; ++c) dcolor[c] = f.pre[c] > R(0) ? dcol[c] : R(0);
    for (int c = 0; c < 3; ++c) gdc[3 * i + c] = R(SH_C0) * dcolor[c];
    for (int k = 0; k < 45; ++k) grest[45 * i + k] = R(0);
    R d_band[3] = {0, 0, 0}, d_dirs[3] = {0, 0, 0};
    if (deg > 0) {
      R b[16], bg[16][3];
      sh_basis<R>(f.dir[0], f.dir[1], f.dir[2], b);
      sh_basis_grad<R>(f.dir[0], f.dir[1], f.dir[2], bg);
      for (int dd = 0; dd < 3; ++dd) {
        R acc = 0;
        for (int k = 0; k < K; ++k)
          for (int c = 0; c < 3; ++c)
            acc += bg[k + 1][dd] * (R(cl->sh_rest[45 * i + 3 * k + c]) * f.mk.band[band_of(k)]) * dcolor[c];
        d_dirs[dd] = acc;
      }
      if (s->compute_sh_rest_grads) {
        R per_coeff[15];
        for (int k = 0; k < K; ++k) {
          per_coeff[k] = 0;
          for (int c = 0; c < 3; ++c) {
            const R dmk = b[k + 1] * dcolor[c];
            grest[45 * i + 3 * k + c] = dmk * f.mk.band[band_of(k)];
            per_coeff[k] += dmk * R(cl->sh_rest[45 * i + 3 * k + c]);
          }
        }
        for (int k = 0; k < K; ++k) d_band[band_of(k)] += per_coeff[k];
      }
    }
    for (int l = 0; l < 3; ++l) {
      const R sg = sigmoid<R>(R(cl->sh_mask_logits[3 * i + l]));
      gshm[3 * i + l] = d_band[l] * (sg * (R(1) - sg));
    }
    const R inner = d_dirs[0] * f.dir[0] + d_dirs[1] * f.dir[1] + d_dirs[2] * f.dir[2];
    for (int k = 0; k < 3; ++k) gpos[3 * i + k] = (d_dirs[k] - f.dir[k] * inner) / f.dnorm;
    // --- opacity path (rasterizer.py:397-400) ---
    const R s_op = sigmoid<R>(R(cl->opacity_logits[i]));
    gop[i] = f.visible ? da * f.mk.gauss * s_op * (R(1) - s_op) : R(0);
    R dmask = f.visible ? da * s_op : R(0);
    // --- geometry path: project_backward (geometry.py:198-251) ---
    R dS[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (f.visible) {
      const R tz = f.t[2], fx = cam.fx, fy = cam.fy;
      const R G[4] = {g00, R(0.5) * g01, R(0.5) * g01, g11};
      const R *Mj = f.Mj;
      // dcov3d = M^T G M  (3x3), evaluated as (M^T G) M
      R MtG[6];  // 3x2
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 2; ++b) MtG[2 * a + b] = Mj[a] * G[b] + Mj[3 + a] * G[2 + b];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) dS[3 * a + b] = MtG[2 * a] * Mj[b] + MtG[2 * a + 1] * Mj[3 + b];
      // dM = 2 (G M) Sigma
      R GM[6], dM[6];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) GM[3 * a + b] = G[2 * a] * Mj[b] + G[2 * a + 1] * Mj[3 + b];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
          dM[3 * a + b] = R(2) * (GM[3 * a] * f.S[b] + GM[3 * a + 1] * f.S[3 + b] + GM[3 * a + 2] * f.S[6 + b]);
      // dJ = dM Rc^T
      R dJ[6];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
          dJ[3 * a + b] = dM[3 * a] * cam.Rc[3 * b] + dM[3 * a + 1] * cam.Rc[3 * b + 1] + dM[3 * a + 2] * cam.Rc[3 * b + 2];
      const R tz2 = tz * tz, tz3 = tz * tz * tz;
      R dt[3];
      dt[0] = dJ[2] * (-fx / tz2);
      dt[1] = dJ[5] * (-fy / tz2);
      dt[2] = dJ[0] * (-fx / tz2) + dJ[4] * (-fy / tz2) + dJ[2] * (R(2) * fx * f.t[0] / tz3) +
              dJ[5] * (R(2) * fy * f.t[1] / tz3);
      dt[0] += dm0 * fx / tz;
      dt[1] += dm1 * fy / tz;
      dt[2] += -(dm0 * fx * f.t[0] + dm1 * fy * f.t[1]) / tz2;
      for (int j = 0; j < 3; ++j)
        gpos[3 * i + j] += dt[0] * cam.Rc[j] + dt[1] * cam.Rc[3 + j] + dt[2] * cam.Rc[6 + j];
    }
    // --- covariance_backward / quat_backward (geometry.py:44-89) ---
    R L[9], dL[9], dsc[3], dR[9];
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) L[3 * r + k] = f.Rg[3 * r + k] * f.sc[k];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        R acc = 0;
        for (int k = 0; k < 3; ++k) acc += (dS[3 * a + k] + dS[3 * k + a]) * L[3 * k + b];
        dL[3 * a + b] = acc;
      }
    for (int k = 0; k < 3; ++k) dsc[k] = dL[k] * f.Rg[k] + dL[3 + k] * f.Rg[3 + k] + dL[6 + k] * f.Rg[6 + k];
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) dR[3 * r + k] = dL[3 * r + k] * f.sc[k];
    const R w = f.qn[0], x = f.qn[1], y = f.qn[2], z = f.qn[3];
    R dqu[4];
    dqu[0] = R(2) * (x * (dR[7] - dR[5]) + y * (dR[2] - dR[6]) + z * (dR[3] - dR[1]));
    dqu[1] = R(2) * (y * (dR[1] + dR[3]) + z * (dR[2] + dR[6])) + R(2) * w * (dR[7] - dR[5]) - R(4) * x * (dR[4] + dR[8]);
    dqu[2] = R(2) * (x * (dR[1] + dR[3]) + z * (dR[5] + dR[7])) + R(2) * w * (dR[2] - dR[6]) - R(4) * y * (dR[0] + dR[8]);
    dqu[3] = R(2) * (x * (dR[2] + dR[6]) + y * (dR[5] + dR[7])) + R(2) * w * (dR[3] - dR[1]) - R(4) * z * (dR[0] + dR[4]);
    const R qin = dqu[0] * w + dqu[1] * x + dqu[2] * y + dqu[3] * z;
    for (int k = 0; k < 4; ++k) grot[4 * i + k] = (dqu[k] - f.qn[k] * qin) / f.qnorm;
    for (int k = 0; k < 3; ++k) gls[3 * i + k] = dsc[k] * f.s_raw[k] * f.mk.gauss;
    dmask += dsc[0] * f.s_raw[0] + dsc[1] * f.s_raw[1] + dsc[2] * f.s_raw[2];
    const R sm = sigmoid<R>(R(cl->mask_logits[i]));
    gmask[i] = dmask * (sm * (R(1) - sm));
    if (gm2d) {
      gm2d[2 * i] = f.visible ? dm0 : R(0);
      gm2d[2 * i + 1] = f.visible ? dm1 : R(0);
    }
  }
  return 0;
}

}  // namespace

extern "C" {

float oracle_sem_expf(float x) { return sem_expf(x); }

int oracle_preprocess_f64(const oracle_cloud *c, const oracle_camera *cam, const oracle_settings *s,
                          double *splats, uint8_t *vis, int32_t *tiles, double *depth_key) {
  return preprocess<double>(c, cam, s, splats, vis, tiles, depth_key);
}
int oracle_preprocess_f32(const oracle_cloud *c, const oracle_camera *cam, const oracle_settings *s,
                          float *splats, uint8_t *vis, int32_t *tiles, double *depth_key) {
  return preprocess<float>(c, cam, s, splats, vis, tiles, depth_key);
}
int oracle_count_tiles_f64(const double *splats, int64_t n, int W, int H, int ts, int32_t *tiles) {
  for (int64_t g = 0; g < n; ++g) {
    int a, b, c, d;
    tiles[g] = (int32_t)tile_rect<double>(splats[12 * g], splats[12 * g + 1], splats[12 * g + 10], W, H, ts, &a, &b, &c, &d);
  }
  return 0;
}
int oracle_count_tiles_f32(const float *splats, int64_t n, int W, int H, int ts, int32_t *tiles) {
  for (int64_t g = 0; g < n; ++g) {
    int a, b, c, d;
    tiles[g] = (int32_t)tile_rect<float>(splats[12 * g], splats[12 * g + 1], splats[12 * g + 10], W, H, ts, &a, &b, &c, &d);
  }
  return 0;
}
int64_t oracle_bin_f64(const double *sp, const int32_t *tiles, const double *dk, int64_t n, int W, int H, int ts,
                       int64_t *offsets, int64_t *ids, int64_t cap) {
  return bin<double>(sp, tiles, dk, n, W, H, ts, offsets, ids, cap);
}
int64_t oracle_bin_f32(const float *sp, const int32_t *tiles, const double *dk, int64_t n, int W, int H, int ts,
                       int64_t *offsets, int64_t *ids, int64_t cap) {
  return bin<float>(sp, tiles, dk, n, W, H, ts, offsets, ids, cap);
}
void oracle_blend_fwd_f64(const double *sp, const int64_t *off, const int64_t *ids, int W, int H, int ts,
                          const double *bg, double *img, double *T, double *ws, int32_t *nc, int32_t *lp, int64_t *hits) {
  blend_fwd<double>(sp, off, ids, W, H, ts, bg, img, T, ws, nc, lp, hits);
}
void oracle_blend_fwd_f32(const float *sp, const int64_t *off, const int64_t *ids, int W, int H, int ts,
                          const double *bg, float *img, float *T, float *ws, int32_t *nc, int32_t *lp, int64_t *hits) {
  blend_fwd<float>(sp, off, ids, W, H, ts, bg, img, T, ws, nc, lp, hits);
}
void oracle_blend_bwd_f64(const double *sp, const int64_t *off, const int64_t *ids, int W, int H, int ts,
                          const double *bg, const double *T, const int32_t *lp, const double *dimg, double *dsp) {
  blend_bwd<double>(sp, off, ids, W, H, ts, bg, T, lp, dimg, dsp);
}
void oracle_blend_bwd_f32(const float *sp, const int64_t *off, const int64_t *ids, int W, int H, int ts,
                          const double *bg, const float *T, const int32_t *lp, const float *dimg, float *dsp) {
  blend_bwd<float>(sp, off, ids, W, H, ts, bg, T, lp, dimg, dsp);
}
int oracle_preprocess_bwd_f64(const oracle_cloud *c, const oracle_camera *cam, const oracle_settings *s,
                              const double *dsp, double *gpos, double *gls, double *grot, double *gop, double *gdc,
                              double *grest, double *gmask, double *gshm, double *gm2d) {
  return preprocess_bwd<double>(c, cam, s, dsp, gpos, gls, grot, gop, gdc, grest, gmask, gshm, gm2d);
}
int oracle_preprocess_bwd_f32(const oracle_cloud *c, const oracle_camera *cam, const oracle_settings *s,
                              const float *dsp, float *gpos, float *gls, float *grot, float *gop, float *gdc,
                              float *grest, float *gmask, float *gshm, float *gm2d) {
  return preprocess_bwd<float>(c, cam, s, dsp, gpos, gls, grot, gop, gdc, grest, gmask, gshm, gm2d);
}

}  // extern "C"
