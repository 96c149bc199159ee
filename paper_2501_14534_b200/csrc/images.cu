// images.cu — target-side progressive ops on the GPU.
//
//   tgs_area_resize    images.area_resize (images.py:58-87): exact fractional
//                      box filter, rows then columns, weights = interval overlap
//                      / scale with float64 edges like the reference
//   tgs_gaussian_blur  images.gaussian_blur (images.py:90-102): separable odd
//                      kernel, scipy 'reflect' edges (= numpy 'symmetric')
//
// Images are (H, W, 3) float32.  Both are streaming kernels over the output with
// the few input taps of each output pixel read through L1; the intermediate
// (after the first separable pass) lives in a caller workspace.
#include "tgs_common.cuh"

namespace tgs {

// one 1-D area-resample pass along the axis with stride `stride_in` (elements)
__global__ void k_area_axis(const float *__restrict__ in, float *__restrict__ out, int n_in, int n_out, int other,
                            int64_t so_axis_in, int64_t so_other_in, int64_t so_axis_out, int64_t so_other_out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)n_out * other * 3;
  if (e >= total) return;
  const int c = (int)(e % 3);
  const int64_t r = e / 3;
  const int o = (int)(r % other);
  const int i = (int)(r / other);
  const double scale = (double)n_in / (double)n_out;
  const double lo = i * scale, hi = (i + 1) * scale;  // edges (images.py:50-55)
  const int j0 = (int)floor(lo);
  const int j1 = min((int)ceil(hi), n_in);
  double acc = 0.0;
  for (int j = j0; j < j1; ++j) {
    const double cover = fmin(j + 1.0, hi) - fmax((double)j, lo);
    if (cover > 0.0) acc += (double)in[j * so_axis_in + o * so_other_in + c] * cover;
  }
  out[i * so_axis_out + o * so_other_out + c] = (float)(acc / scale);
}

struct Taps32 {
  float w[32];
};

__device__ __forceinline__ int reflect_idx(int k, int n) {
  while (k < 0 || k >= n) {  // scipy 'reflect' (d c b a | a b c d | d c b a)
    if (k < 0) k = -1 - k;
    if (k >= n) k = 2 * n - 1 - k;
  }
  return k;
}

__global__ void k_blur_axis(const float *__restrict__ in, float *__restrict__ out, int n, int other, int size,
                            Taps32 tp, int64_t so_axis, int64_t so_other) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)n * other * 3;
  if (e >= total) return;
  const int c = (int)(e % 3);
  const int64_t r = e / 3;
  const int o = (int)(r % other);
  const int i = (int)(r / other);
  const int rad = size / 2;
  float acc = 0.0f;
  for (int k = 0; k < size; ++k) acc += tp.w[k] * in[reflect_idx(i + k - rad, n) * so_axis + o * so_other + c];
  out[i * so_axis + o * so_other + c] = acc;
}

}  // namespace tgs

using namespace tgs;

extern "C" int tgs_area_resize(const float *in, int32_t in_h, int32_t in_w, float *out, int32_t out_h, int32_t out_w,
                               float *workspace, tgs_stream_t stream) {
  if (!in || !out || in_h < 1 || in_w < 1 || out_h < 1 || out_w < 1 || out_h > in_h || out_w > in_w)
    return TGS_ERR_INVALID;  // images.py:72-73: area_resize only downsamples
  cudaStream_t st = as_stream(stream);
  if (out_h == in_h && out_w == in_w)
    return cuda_status(cudaMemcpyAsync(out, in, (size_t)in_h * in_w * 3 * 4, cudaMemcpyDeviceToDevice, st));
  if (!workspace) return TGS_ERR_INVALID;
  // rows: (in_h, in_w) -> (out_h, in_w); columns: (out_h, in_w) -> (out_h, out_w)
  int64_t t1 = (int64_t)out_h * in_w * 3;
  k_area_axis<<<(unsigned)ceil_div<int64_t>(t1, 256), 256, 0, st>>>(in, workspace, in_h, out_h, in_w,
                                                                     (int64_t)in_w * 3, 3, (int64_t)in_w * 3, 3);
  int64_t t2 = (int64_t)out_w * out_h * 3;
  k_area_axis<<<(unsigned)ceil_div<int64_t>(t2, 256), 256, 0, st>>>(workspace, out, in_w, out_w, out_h, 3,
                                                                     (int64_t)in_w * 3, 3, (int64_t)out_w * 3);
  return launch_status();
}

extern "C" int tgs_gaussian_blur(const float *in, int32_t h, int32_t w, int32_t size, float sigma, float *out,
                                 float *workspace, tgs_stream_t stream) {
  if (!in || !out || h < 1 || w < 1) return TGS_ERR_INVALID;
  cudaStream_t st = as_stream(stream);
  if (size <= 1 || !(sigma > 0.0f))
    return cuda_status(cudaMemcpyAsync(out, in, (size_t)h * w * 3 * 4, cudaMemcpyDeviceToDevice, st));
  if (size % 2 == 0 || size > 31 || !workspace) return TGS_ERR_INVALID;  // images.py:94-95
  Taps32 tp;
  double ww[32], tot = 0.0;
  for (int k = 0; k < size; ++k) {
    const double x = (k - (size - 1) / 2.0) / sigma;
    ww[k] = exp(-0.5 * x * x);
    tot += ww[k];
  }
  for (int k = 0; k < size; ++k) tp.w[k] = (float)(ww[k] / tot);
  const int64_t total = (int64_t)h * w * 3;
  const unsigned grid = (unsigned)ceil_div<int64_t>(total, 256);
  k_blur_axis<<<grid, 256, 0, st>>>(in, workspace, h, w, size, tp, (int64_t)w * 3, 3);   // axis 0 (rows)
  k_blur_axis<<<grid, 256, 0, st>>>(workspace, out, w, h, size, tp, 3, (int64_t)w * 3);  // axis 1 (columns)
  return launch_status();
}
