// Correctly rounded division from a shared reciprocal: q0 = RN(a * RN(1/b)),
// r = a - b q0 (exact with FMA), q1 = RN(q0 + r * RN(1/b)) -- compared bit for
// bit with __ddiv_rn on random operands (uniform bit patterns over a wide
// exponent window, and operands shaped like the projection's: fx * t0 / z,
// c / det).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/div_check tools/div_check.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double ddiv_shared(double a, double b, double rb) {
  const double q0 = __dmul_rn(a, rb);
  const double r = __fma_rn(-b, q0, a);
  return r == 0.0 ? q0 : __fma_rn(r, rb, q0);
}

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

__global__ void k_check(uint64_t seed, uint64_t n, int mode, unsigned long long* bad, double* ex,
                        unsigned long long* done) {
  unsigned long long mine = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h1 = mix(seed ^ (i * 2 + 1)), h2 = mix(seed + i * 0x9e3779b97f4a7c15ull);
    double a, b;
    if (mode == 0) {  // random bit patterns, exponents in [-200, 200]
      const uint64_t ea = 823 + (h1 >> 55) % 400, eb = 823 + (h2 >> 55) % 400;
      a = __longlong_as_double((long long)((h1 & 0x800fffffffffffffull) | (ea << 52)));
      b = __longlong_as_double((long long)((h2 & 0x000fffffffffffffull) | (eb << 52)));
    } else if (mode == 1) {  // projection-like: (fx * t0) / z, z in (0.2, 5000)
      const double z = 0.2 + (double)(h2 >> 11) * 0x1.0p-53 * 5000.0;
      const double t0 = ((double)(h1 >> 11) * 0x1.0p-53 - 0.5) * 4000.0;
      a = __dmul_rn(1234.5678, t0);
      b = z;
    } else {  // conic-like: c / det with det = a c - b^2 small vs a c
      const double x = (double)(h1 >> 11) * 0x1.0p-53 * 100.0 + 1e-6;
      const double y = (double)(h2 >> 11) * 0x1.0p-53 * 100.0 + 1e-6;
      a = x;
      b = __dsub_rn(__dmul_rn(x, y), __dmul_rn(0.999 * x, y));
    }
    if (!(b > 0.0)) continue;
    ++mine;
    const double rb = __drcp_rn(b);
    const double q = ddiv_shared(a, b, rb), want = __ddiv_rn(a, b);
    if (__double_as_longlong(q) != __double_as_longlong(want)) {
      const unsigned long long k = atomicAdd(bad, 1ull);
      if (k < 4) { ex[3 * k] = a; ex[3 * k + 1] = b; ex[3 * k + 2] = q - want; }
    }
  }
  atomicAdd(done, mine);
}

int main() {
  unsigned long long* bad;
  unsigned long long* done;
  double* ex;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&done, 8);
  cudaMallocManaged(&ex, 12 * 8);
  for (int mode = 0; mode < 3; ++mode) {
    *bad = 0;
    *done = 0;
    const uint64_t n = 2000000000ull;
    for (int rep = 0; rep < 2; ++rep) k_check<<<148 * 32, 256>>>(0x1234567ull + 977 * rep + 31 * mode, n, mode, bad, ex, done);
    const cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s, %llu mismatches in %llu checked divisions\n", mode, cudaGetErrorString(e),
           (unsigned long long)*bad, (unsigned long long)*done);
    for (unsigned long long k = 0; k < *bad && k < 4; ++k) printf("  a=%.17g b=%.17g diff=%g\n", ex[3 * k], ex[3 * k + 1], ex[3 * k + 2]);
  }
  return 0;
}
