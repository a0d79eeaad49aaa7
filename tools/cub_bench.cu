// Same-box bar for the local sort: cub::DeviceRadixSort on
// uint64 keys over the significant bits, timed with CUDA events.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
int main(int argc, char** argv) {
  size_t n = argc > 1 ? atoll(argv[1]) : (1ull << 27);
  int bits = argc > 2 ? atoi(argv[2]) : 56;
  std::vector<unsigned long long> h(n);
  std::mt19937_64 rng(1);
  for (auto& x : h) x = rng() & ((bits >= 64) ? ~0ull : ((1ull << bits) - 1));
  unsigned long long *a, *b;
  cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8);
  cudaMemcpy(a, h.data(), n * 8, cudaMemcpyHostToDevice);
  size_t tb = 0; void* tmp = nullptr;
  cub::DeviceRadixSort::SortKeys(tmp, tb, a, b, (int)n, 0, bits);
  cudaMalloc(&tmp, tb);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; it++) cub::DeviceRadixSort::SortKeys(tmp, tb, a, b, (int)n, 0, bits);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int it = 0; it < reps; it++) cub::DeviceRadixSort::SortKeys(tmp, tb, a, b, (int)n, 0, bits);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  int passes = (bits + 7) / 8;
  printf("cub SortKeys n=%zu bits=%d: %.3f ms  (%.2f Gkeys/s, %.0f GB/s at 16 B/key/pass over %d passes)\n", n, bits, ms,
         n / ms / 1e6, 16.0 * n * passes / ms / 1e6, passes);
  return 0;
}
