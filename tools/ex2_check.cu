// Exhaustive accuracy check of the hardware base-2 exponential the fast blend
// uses (ex2.approx.ftz.f32, MUFU.EX2): every float x in [-32, 1] against
// exp2((double)x).  Prints the maximum relative error; the blend's certified
// alpha bound (cs_internal.cuh, kEx2RelErr) must be at least this.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ex2_check tools/ex2_check.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void k_check(uint32_t lo, uint32_t hi, unsigned long long* worst_bits, double* worst) {
  double w = 0.0;
  uint32_t wb = 0;
  for (uint64_t b = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b <= hi;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const float x = __uint_as_float((uint32_t)b);
    const double ref = exp2((double)x);
    const double got = (double)ex2_approx(x);
    const double e = fabs(got - ref) / ref;
    if (e > w) { w = e; wb = (uint32_t)b; }
  }
  // block max via atomics on the bit pattern (e >= 0: monotone as int64)
  const unsigned long long key = ((unsigned long long)__double_as_longlong(w));
  const unsigned long long old = atomicMax(worst_bits, key);
  if (key > old) worst[1] = (double)wb;
}

int main() {
  unsigned long long* d_bits;
  double* d_w;
  cudaMalloc(&d_bits, 8);
  cudaMalloc(&d_w, 16);
  cudaMemset(d_bits, 0, 8);
  cudaMemset(d_w, 0, 16);
  // negative floats: bit patterns 0x80000000 (-0) .. bits(-32.0f)
  const float lim = -32.0f;
  uint32_t hi;
  memcpy(&hi, &lim, 4);
  k_check<<<148 * 8, 256>>>(0x80000000u, hi, d_bits, d_w);
  k_check<<<148 * 8, 256>>>(0x00000000u, 0x3f800000u, d_bits, d_w);  // [0, 1]: float32 powers round slightly above 0
  unsigned long long bits;
  double w[2];
  cudaMemcpy(&bits, d_bits, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(w, d_w, 16, cudaMemcpyDeviceToHost);
  double e;
  memcpy(&e, &bits, 8);
  uint32_t wb = (uint32_t)w[1];
  float wx;
  memcpy(&wx, &wb, 4);
  printf("ex2.approx.ftz.f32 over [-32, 1]: max relative error %.3e (= 2^%.2f ulp-scale), at x = %.9g (%s)\n",
         e, log2(e), wx, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
