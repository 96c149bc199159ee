// Standalone check of 3-D TMA tile loads (box 44 x 42 x 1, out-of-bounds zero fill).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

template <typename T, int BW, int BH>
__global__ void k_load(const __grid_constant__ CUtensorMap tm, int x, int y, int z, T *out) {
  __shared__ __align__(128) T tile[BH][BW];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t bs = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bs));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bs), "r"((uint32_t)sizeof(tile)) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&tile[0][0])), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y), "r"(z), "r"(bs) : "memory");
  }
  __syncthreads();
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(bs) : "memory");
  for (int i = threadIdx.x; i < BW * BH; i += blockDim.x) out[i] = tile[i / BW][i % BW];
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  printf("entry %p q=%d\n", (void *)enc, (int)q);
  const int W = 64, H = 64, C = 3, P = 64;
  float *d; cudaMalloc(&d, (size_t)C * H * P * 4);
  std::vector<float> h((size_t)C * H * P);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  float *o; cudaMalloc(&o, 44 * 42 * 8);
  struct Case { int bw, bh, x, y; };
  for (Case cs : {Case{44, 42, -4, -5}, Case{44, 42, -8, -3}, Case{44, 42, 4, 0}, Case{44, 42, -5, 0}}) {
    CUtensorMap m;
    cuuint64_t dims[3] = {W, H, C}, str[2] = {(cuuint64_t)P * 4, (cuuint64_t)P * 4 * H};
    cuuint32_t box[3] = {(cuuint32_t)cs.bw, (cuuint32_t)cs.bh, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box %dx%d at (%d,%d): encode %d\n", cs.bw, cs.bh, cs.x, cs.y, (int)r);
    if (cs.bw == 44) k_load<float, 44, 42><<<1, 128>>>(m, cs.x, cs.y, 1, o);
    else k_load<float, 32, 32><<<1, 128>>>(m, cs.x, cs.y, 1, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  run: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    float hv[4]; cudaMemcpy(hv, o, 16, cudaMemcpyDeviceToHost);
    printf("  first values %g %g %g %g\n", hv[0], hv[1], hv[2], hv[3]);
  }
  return 0;
}
