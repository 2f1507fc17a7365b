// Microbenchmark + check of the onesweep radix sort (cs_sort.cu) on the two
// frame workloads: 6.3M float32 depth keys (32 bits) and 14M tile keys
// (13 bits), values = index, for several items-per-thread settings.
// Validates stability against std::stable_sort.  Measured on B200 (round 1):
// 12 items/thread is best (342 us depth, 358 us tiles); a persistent variant
// with ticket prefetch was 10-20 % slower, removing the look-back entirely
// changed < 3 %, so the pass is bound by the per-chunk rank/scatter work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/sort_bench.cu -o sb
#include <algorithm>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#include "../paper_2404_01133_b200/csrc/cs_sort.cu"

template <typename K, int V, int MB = 1, bool EA = true>
static void run(const char* name, std::vector<K> keys, int bits, int reps) {
  const int64_t n = (int64_t)keys.size();
  K *k0, *k1;
  uint32_t *v0, *v1, *hist, *status, *tickets;
  int64_t* dn;
  cudaMalloc(&k0, sizeof(K) * n); cudaMalloc(&k1, sizeof(K) * n);
  cudaMalloc(&v0, 4 * n); cudaMalloc(&v1, 4 * n);
  cudaMalloc(&hist, 4 * 256 * 8);
  cudaMalloc(&status, 4 * (n / 256 + 2) * 256);
  cudaMalloc(&tickets, 64);
  cudaMalloc(&dn, 8);
  cudaMemcpy(dn, &n, 8, cudaMemcpyHostToDevice);
  std::vector<uint32_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0u);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  int which = 0;
  for (int r = 0; r < reps; ++r) {
    cudaMemcpy(k0, keys.data(), sizeof(K) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(v0, idx.data(), 4 * n, cudaMemcpyHostToDevice);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    which = cs::radix_sort_items<K, V, MB, EA>(k0, v0, k1, v1, dn, n, 0, bits, hist, status, tickets, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  std::vector<uint32_t> got(n);
  cudaMemcpy(got.data(), which ? v1 : v0, 4 * n, cudaMemcpyDeviceToHost);
  std::vector<uint32_t> want(idx);
  const K mask = bits >= (int)(8 * sizeof(K)) ? ~K(0) : (K(1) << bits) - 1;
  std::stable_sort(want.begin(), want.end(), [&](uint32_t a, uint32_t b) { return (keys[a] & mask) < (keys[b] & mask); });
  const bool ok = got == want;
  printf("v%-2d/%d%s %-24s n=%lld bits=%d: %.1f us (%s), %.2f Gkeys/s\n", V, MB, EA ? "e" : "l", name, (long long)n, bits, best * 1e3,
         ok ? "exact" : "MISMATCH", n / (best * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
  std::mt19937_64 rng(1);
  const bool prof = argc > 1;  // one 12-item run of each workload (for ncu)
  {
    std::vector<uint32_t> k(6300000);
    std::uniform_real_distribution<float> d(20.f, 2500.f);
    for (auto& x : k) { float f = d(rng); memcpy(&x, &f, 4); }
    for (size_t i = 0; i < k.size() / 33; ++i) k[i * 33] = 0xffffffffu;  // culled
    if (prof) { run<uint32_t, 12, 3>("depth f32 keys", k, 32, 1); goto tiles; }
    run<uint32_t, 8, 4>("depth f32 keys", k, 32, 5);
    run<uint32_t, 10, 3>("depth f32 keys", k, 32, 5);
    run<uint32_t, 12, 3>("depth f32 keys", k, 32, 5);
    run<uint32_t, 16, 2>("depth f32 keys", k, 32, 5);
    run<uint32_t, 16, 3>("depth f32 keys", k, 32, 5);
  }
tiles:
  {
    std::vector<uint32_t> k(14000000);
    std::uniform_int_distribution<uint32_t> d(0, 8159);
    for (auto& x : k) x = d(rng);
    if (prof) { run<uint32_t, 12, 3>("tile keys", k, 13, 1); return 0; }
    run<uint32_t, 8, 4>("tile keys", k, 13, 5);
    run<uint32_t, 10, 3>("tile keys", k, 13, 5);
    run<uint32_t, 12, 3>("tile keys", k, 13, 5);
    run<uint32_t, 16, 2>("tile keys", k, 13, 5);
    run<uint32_t, 16, 3>("tile keys", k, 13, 5);
  }
  return 0;
}
