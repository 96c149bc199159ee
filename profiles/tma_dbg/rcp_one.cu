// Checks that rcp.approx.ftz.f32(1.0f) is exactly 1.0f (the backward blend relies on it
// for pixels that skip a splat: T * rcp(1 - 0) must leave T unchanged).
#include <cstdio>
__global__ void k(float *out, float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  out[threadIdx.x] = r;
}
int main() {
  float *d, h[32];
  cudaMalloc(&d, 128);
  k<<<1, 32>>>(d, 1.0f);
  cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("rcp(1.0f) = %.9g bits %08x -> %s\n", h[0], *(unsigned *)&h[0], h[0] == 1.0f ? "exact" : "NOT exact");
  return h[0] == 1.0f ? 0 : 1;
}
