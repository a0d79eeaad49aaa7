// Microbenchmark: random 8-byte probes / CAS into a table of T bytes (L2-resident vs not).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2probe_bench tools/l2probe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t fmix(uint64_t x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31; return x;
}
// each thread: reads keys from a stream (coalesced), probes table[home] (linear), CAS if empty
__global__ void probe(const uint64_t* keys, uint64_t n, unsigned long long* tab, uint64_t mask, int mode, unsigned long long* sink) {
  uint64_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const uint64_t h = fmix(k);
    uint64_t s = h & mask;
    if (mode == 0) {
      acc += tab[s];
    } else {
      for (;;) {
        unsigned long long cur = tab[s];
        if (cur == k) break;
        if (cur == 0) {
          unsigned long long old = atomicCAS(&tab[s], 0ull, (unsigned long long)k);
          if (old == 0 || old == k) break;
        }
        s = (s + 1) & mask;
      }
    }
  }
  if (acc == 42) *sink = acc;
}
// batched: 8 keys per thread, first probes issued together
__global__ void probe8(const uint64_t* keys, uint64_t n, unsigned long long* tab, uint64_t mask) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i0 < n; i0 += 8 * stride) {
    uint64_t k[8], s[8];
    unsigned long long c[8];
#pragma unroll
    for (int u = 0; u < 8; u++) { const uint64_t i = i0 + u * stride; k[u] = i < n ? keys[i] : 0; }
#pragma unroll
    for (int u = 0; u < 8; u++) { s[u] = fmix(k[u]) & mask; }
#pragma unroll
    for (int u = 0; u < 8; u++) c[u] = k[u] ? __ldcg(&tab[s[u]]) : 0;
#pragma unroll
    for (int u = 0; u < 8; u++) {
      if (!k[u] || c[u] == k[u]) continue;
      uint64_t x = s[u];
      unsigned long long cur = c[u];
      for (;;) {
        if (cur == k[u]) break;
        if (cur == 0) {
          unsigned long long old = atomicCAS(&tab[x], 0ull, (unsigned long long)k[u]);
          if (old == 0 || old == k[u]) break;
        }
        x = (x + 1) & mask;
        cur = __ldcg(&tab[x]);
      }
    }
  }
}
__global__ void genkeys(uint64_t* keys, uint64_t n, uint64_t distinct) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = fmix(i * 0x9E3779B97F4A7C15ull) % distinct + 1;
}
int main() {
  const uint64_t n = 1ull << 28;  // 268M keys = 2 GB stream
  uint64_t* keys; cudaMalloc(&keys, n * 8);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; rep++)
  for (uint64_t tbytes : {32ull << 20, 64ull << 20, 1024ull << 20}) {
    if (rep && tbytes < (1024ull << 20)) continue;
    const uint64_t slots = tbytes / 8;
    unsigned long long* tab; cudaMalloc(&tab, tbytes);
    const uint64_t distinct = rep ? n / 7 : slots / 4;
    genkeys<<<sms * 8, 256>>>(keys, n, distinct);
    for (int mode = 0; mode < 3; mode++) {
      cudaMemset(tab, 0, tbytes);
      if (mode < 2) probe<<<sms * 8, 256>>>(keys, n, tab, slots - 1, mode, sink);  // warm
      else probe8<<<sms * 8, 256>>>(keys, n, tab, slots - 1);
      cudaMemset(tab, 0, tbytes);
      cudaEventRecord(a);
      if (mode < 2) probe<<<sms * 8, 256>>>(keys, n, tab, slots - 1, mode, sink);
      else probe8<<<sms * 8, 256>>>(keys, n, tab, slots - 1);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%s table %5llu MB mode %s: %.3f ms, %.2f Gprobe/s, stream %.0f GB/s\n", rep ? "mult7  " : "mult268", (unsigned long long)(tbytes >> 20),
             mode == 2 ? "ins8  " : mode ? "insert" : "load  ", ms, n / ms / 1e6, n * 8 / ms / 1e6);
    }
    cudaFree(tab);
  }
  return 0;
}
