// Device-wide primitives: exclusive scan, LSD radix sort of configuration keys
// over their significant bits, unique compaction of sorted keys.
// (SURVEY 8(a) row a11; PAPER.md:454 "GPU-optimized Radix Sort", :460 "local
// merge and stream compaction", :469-470 radix sort over uint64 bitmasks.)
#include "internal.cuh"

namespace cusci {
namespace {

// ------------------------------------------------------------------ scan
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(kFull, v, o);
    if ((int)lane_id() >= o) v += t;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns the block total
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* smem /*[32]*/, T& total) {
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane_id() == 31) smem[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = (int)lane_id() < nw ? smem[lane_id()] : T(0);
    T si = warp_incl_scan(s);
    if ((int)lane_id() < nw) smem[lane_id()] = si - s;
    if (lane_id() == 31) smem[32] = si;
  }
  __syncthreads();
  T r = smem[w] + inc - v;
  total = smem[32];
  __syncthreads();
  return r;
}

template <typename T>
__global__ void scan_reduce_kernel(const T* __restrict__ in, uint64_t n, T* __restrict__ partial) {
  __shared__ T sm[33];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    uint64_t idx = base + (uint64_t)i * kScanThreads + threadIdx.x;
    if (idx < n) s += in[idx];
  }
  T tot;
  block_excl_scan(s, sm, tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

template <typename T>
__global__ void scan_apply_kernel(const T* __restrict__ in, T* __restrict__ out, uint64_t n,
                                  const T* __restrict__ partial_excl, T* __restrict__ total_out) {
  __shared__ T sm[33];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  // blocked arrangement: thread t owns items [t*ITEMS, (t+1)*ITEMS)
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    uint64_t idx = base + (uint64_t)threadIdx.x * kScanItems + i;
    v[i] = idx < n ? in[idx] : T(0);
    s += v[i];
  }
  T tot;
  T ex = block_excl_scan(s, sm, tot);
  T run = ex + (partial_excl ? partial_excl[blockIdx.x] : T(0));
#pragma unroll
  for (int i = 0; i < kScanItems; i++) {
    uint64_t idx = base + (uint64_t)threadIdx.x * kScanItems + i;
    if (idx < n) out[idx] = run;
    run += v[i];
  }
  if (total_out && blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) *total_out = run;
}

template <typename T>
int scan_impl(cusci_ctx* ctx, const T* in, T* out, uint64_t n, T* total_dev) {
  if (n == 0) {
    if (total_dev) CUSCI_CUDA(ctx, cudaMemsetAsync(total_dev, 0, sizeof(T), ctx->stream));
    return CUSCI_OK;
  }
  const uint64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb == 1) {
    CUSCI_LAUNCH(ctx, PT_SCAN, scan_apply_kernel<T><<<1, kScanThreads, 0, ctx->stream>>>(in, out, n, nullptr, total_dev));
    return CUSCI_OK;
  }
  Scratch s(ctx);
  T *part, *part_ex;
  CUSCI_TRY(s.get_t(nb, &part));
  CUSCI_TRY(s.get_t(nb, &part_ex));
  CUSCI_LAUNCH(ctx, PT_SCAN, scan_reduce_kernel<T><<<(unsigned)nb, kScanThreads, 0, ctx->stream>>>(in, n, part));
  CUSCI_TRY(scan_impl<T>(ctx, part, part_ex, nb, nullptr));
  CUSCI_LAUNCH(ctx, PT_SCAN, scan_apply_kernel<T><<<(unsigned)nb, kScanThreads, 0, ctx->stream>>>(in, out, n, part_ex, total_dev));
  return CUSCI_OK;
}

// ------------------------------------------------------------------ unique
constexpr int kUniqThreads = 256;
constexpr int kUniqItems = 8;
constexpr int kUniqTile = kUniqThreads * kUniqItems;

template <int W>
__global__ void unique_count_kernel(const uint64_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ tile_counts) {
  __shared__ uint32_t sm[33];
  const uint64_t base = (uint64_t)blockIdx.x * kUniqTile;
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < kUniqItems; i++) {
    const uint64_t idx = base + (uint64_t)i * kUniqThreads + threadIdx.x;
    if (idx < n) c += (idx == 0 || !key_eq(load_key<W>(in, idx), load_key<W>(in, idx - 1))) ? 1u : 0u;
  }
  uint32_t tot;
  block_excl_scan<uint32_t>(c, sm, tot);
  if (threadIdx.x == 0) tile_counts[blockIdx.x] = tot;
}

template <int W>
__global__ void unique_write_kernel(const uint64_t* __restrict__ in, uint64_t n, const uint64_t* __restrict__ tile_off,
                                    uint64_t* __restrict__ out) {
  // keep order: each warp handles consecutive 32-key groups; block processes the tile in ITEMS rounds
  __shared__ uint32_t wsum[kUniqThreads / 32];
  __shared__ uint64_t run;
  const uint64_t base = (uint64_t)blockIdx.x * kUniqTile;
  if (threadIdx.x == 0) run = tile_off[blockIdx.x];
  __syncthreads();
  const int w = threadIdx.x >> 5;
  for (int i = 0; i < kUniqItems; i++) {
    const uint64_t idx = base + (uint64_t)i * kUniqThreads + threadIdx.x;
    bool keep = false;
    KeyT<W> k{};
    if (idx < n) {
      k = load_key<W>(in, idx);
      keep = idx == 0 || !key_eq(k, load_key<W>(in, idx - 1));
    }
    const unsigned bal = __ballot_sync(kFull, keep);
    if (lane_id() == 0) wsum[w] = __popc(bal);
    __syncthreads();
    uint32_t off = 0, tot = 0;
    for (int x = 0; x < kUniqThreads / 32; x++) {
      if (x < w) off += wsum[x];
      tot += wsum[x];
    }
    if (keep) store_key<W>(out, run + off + __popc(bal & lanemask_lt()), k);
    __syncthreads();
    if (threadIdx.x == 0) run += tot;
    __syncthreads();
  }
}

}  // namespace

int scan_exclusive_u32(cusci_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n) {
  return scan_impl<uint32_t>(ctx, in, out, n, nullptr);
}
int scan_exclusive_u64(cusci_ctx* ctx, const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* total_dev) {
  return scan_impl<uint64_t>(ctx, in, out, n, total_dev);
}

template <int W>
static int unique_impl(cusci_ctx* ctx, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* n_out_dev) {
  if (n == 0) {
    CUSCI_CUDA(ctx, cudaMemsetAsync(n_out_dev, 0, sizeof(uint64_t), ctx->stream));
    return CUSCI_OK;
  }
  const uint64_t nt = (n + kUniqTile - 1) / kUniqTile;
  Scratch s(ctx);
  uint32_t* tc;
  uint64_t *tc64, *toff;
  CUSCI_TRY(s.get_t(nt, &tc));
  CUSCI_TRY(s.get_t(nt, &tc64));
  CUSCI_TRY(s.get_t(nt, &toff));
  CUSCI_LAUNCH(ctx, PT_UNIQUE, unique_count_kernel<W><<<(unsigned)nt, kUniqThreads, 0, ctx->stream>>>(in, n, tc));
  // widen to u64 then scan (counts are <= tile size; totals may exceed 2^32)
  CUSCI_CUDA(ctx, cudaMemsetAsync(tc64, 0, nt * sizeof(uint64_t), ctx->stream));
  CUSCI_CUDA(ctx, cudaMemcpy2DAsync(tc64, sizeof(uint64_t), tc, sizeof(uint32_t), sizeof(uint32_t), nt,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
  CUSCI_TRY(scan_exclusive_u64(ctx, tc64, toff, nt, n_out_dev));
  CUSCI_LAUNCH(ctx, PT_UNIQUE, unique_write_kernel<W><<<(unsigned)nt, kUniqThreads, 0, ctx->stream>>>(in, n, toff, out));
  return CUSCI_OK;
}

int unique_sorted_keys(cusci_ctx* ctx, int W, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* n_out_dev) {
  return W == 1 ? unique_impl<1>(ctx, in, n, out, n_out_dev) : unique_impl<2>(ctx, in, n, out, n_out_dev);
}

}  // namespace cusci
