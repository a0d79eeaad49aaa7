// Same-box library bar for the local dedup: cub::DeviceRadixSort
// over the significant key bits + cub::DeviceSelect::Unique, as an extern "C"
// entry point for tools/cub_dedup_bench.py (ctypes).  Not part of the product.
#include <cub/cub.cuh>
#include <cstdint>
extern "C" int cub_dedup(const unsigned long long* keys, long long n, int bits, unsigned long long* sorted,
                         unsigned long long* out, long long* n_out, float* ms_sort, float* ms_unique) {
  size_t tb1 = 0, tb2 = 0;
  int* d_num;
  cudaMalloc(&d_num, sizeof(int));
  cub::DeviceRadixSort::SortKeys(nullptr, tb1, keys, sorted, (int)n, 0, bits);
  cub::DeviceSelect::Unique(nullptr, tb2, sorted, out, d_num, (int)n);
  void* tmp;
  if (cudaMalloc(&tmp, tb1 > tb2 ? tb1 : tb2) != cudaSuccess) return 1;
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  cudaEventRecord(e0);
  cub::DeviceRadixSort::SortKeys(tmp, tb1, keys, sorted, (int)n, 0, bits);
  cudaEventRecord(e1);
  cub::DeviceSelect::Unique(tmp, tb2, sorted, out, d_num, (int)n);
  cudaEventRecord(e2);
  cudaEventSynchronize(e2);
  cudaEventElapsedTime(ms_sort, e0, e1);
  cudaEventElapsedTime(ms_unique, e1, e2);
  int h;
  cudaMemcpy(&h, d_num, sizeof(int), cudaMemcpyDeviceToHost);
  *n_out = h;
  cudaFree(tmp);
  cudaFree(d_num);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
