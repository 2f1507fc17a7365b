// Accuracy probe for exp_le0 (cs_internal.cuh) against CUDA exp() and the host
// libm expl(): max ulp error over a dense sweep of [-6, 0].
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include tools/exp_check.cu -o /tmp/exp_check
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_2404_01133_b200/csrc/cs_internal.cuh"

__global__ void k_probe(int n, const double* x, double* mine, double* cuda) {
  __shared__ cs::ExpTable tab;
  const cs::ExpCoef ec = cs::load_exp_table(&tab);
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    mine[i] = cs::exp_le0(x[i], tab, ec);
    cuda[i] = exp(x[i]);
  }
}

static double ulp_err(double got, long double ref) {
  const double r = (double)ref;
  const double u = std::nextafter(r, INFINITY) - r;
  return (double)fabsl((long double)got - ref) / u;
}

int main() {
  const int n = 1 << 24;
  std::vector<double> x(n);
  for (int i = 0; i < n; ++i) x[i] = -6.0 * (double)i / (n - 1) - 1e-9 * (i & 7);
  double *dx, *dm, *dc;
  cudaMalloc(&dx, 8 * n); cudaMalloc(&dm, 8 * n); cudaMalloc(&dc, 8 * n);
  cudaMemcpy(dx, x.data(), 8 * n, cudaMemcpyHostToDevice);
  k_probe<<<1184, 256>>>(n, dx, dm, dc);
  std::vector<double> m(n), c(n);
  cudaMemcpy(m.data(), dm, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(c.data(), dc, 8 * n, cudaMemcpyDeviceToHost);
  double em = 0, ec = 0;
  long diff_m = 0, diff_c = 0, diff_mc = 0;
  for (int i = 0; i < n; ++i) {
    const long double ref = expl((long double)x[i]);
    em = std::max(em, ulp_err(m[i], ref));
    ec = std::max(ec, ulp_err(c[i], ref));
    diff_m += m[i] != std::exp(x[i]);
    diff_c += c[i] != std::exp(x[i]);
    diff_mc += m[i] != c[i];
  }
  printf("exp_le0: max %.3f ulp, %ld/%d differ from libm exp; CUDA exp: max %.3f ulp, %ld differ; "
         "exp_le0 vs CUDA differ %ld\n", em, diff_m, n, ec, diff_c, diff_mc);
  return 0;
}
