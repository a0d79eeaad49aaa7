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

// ------------------------------------------------------------------ radix sort
constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
template <int W> struct RadixCfg;
template <> struct RadixCfg<1> { static constexpr int ITEMS = 16; };
template <> struct RadixCfg<2> { static constexpr int ITEMS = 8; };

// per-tile digit histogram -> hist[digit * ntiles + tile]
template <int W>
__global__ void __launch_bounds__(kRadixThreads) radix_upsweep(const uint64_t* __restrict__ keys, uint64_t n, int shift,
                                                            uint32_t* __restrict__ hist, uint32_t ntiles) {
  constexpr int ITEMS = RadixCfg<W>::ITEMS;
  constexpr int TILE = kRadixThreads * ITEMS;
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * TILE;
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const uint64_t idx = base + (uint64_t)i * kRadixThreads + threadIdx.x;
    const bool valid = idx < n;
    uint32_t d = 256;
    if (valid) d = key_digit(load_key<W>(keys, idx), shift);
    const unsigned peers = __match_any_sync(kFull, d);
    if (valid && (lane_id() == (unsigned)(__ffs(peers) - 1))) atomicAdd(&h[d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

template <int W>
__global__ void __launch_bounds__(kRadixThreads) radix_downsweep(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                              uint64_t n, int shift, const uint32_t* __restrict__ offs,
                                                              uint32_t ntiles) {
  constexpr int ITEMS = RadixCfg<W>::ITEMS;
  constexpr int TILE = kRadixThreads * ITEMS;
  constexpr int WCHUNK = ITEMS * 32;
  __shared__ uint32_t whist[kRadixWarps][256];
  __shared__ uint32_t tstart[256];
  __shared__ uint32_t gbase[256];
  __shared__ uint32_t red[33];
  __shared__ KeyT<W> skeys[TILE];
  const int w = threadIdx.x >> 5;
  const unsigned lane = lane_id();
#pragma unroll
  for (int i = 0; i < kRadixWarps; i++) whist[i][threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * TILE;
  KeyT<W> k[ITEMS];
  uint32_t rank[ITEMS], dig[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const uint64_t idx = base + (uint64_t)w * WCHUNK + (uint64_t)i * 32 + lane;
    if (idx < n) {
      k[i] = load_key<W>(in, idx);
      dig[i] = key_digit(k[i], shift);
    } else {
      dig[i] = 256;
    }
  }
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const uint32_t d = dig[i];
    const unsigned peers = __match_any_sync(kFull, d);
    uint32_t before = 0;
    if (d < 256) before = whist[w][d];
    rank[i] = before + __popc(peers & lanemask_lt());
    __syncwarp();
    if (d < 256 && lane == (unsigned)(__ffs(peers) - 1)) whist[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix across warps, tile total, tile-local start
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kRadixWarps; i++) {
    const uint32_t t = whist[i][threadIdx.x];
    whist[i][threadIdx.x] = acc;
    acc += t;
  }
  uint32_t tot;
  const uint32_t st = block_excl_scan<uint32_t>(acc, red, tot);
  tstart[threadIdx.x] = st;
  gbase[threadIdx.x] = offs[(size_t)threadIdx.x * ntiles + blockIdx.x];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const uint32_t d = dig[i];
    if (d < 256) skeys[tstart[d] + whist[w][d] + rank[i]] = k[i];
  }
  __syncthreads();
  const uint64_t rem = n - base;
  const int cnt = rem < (uint64_t)TILE ? (int)rem : TILE;
  for (int j = threadIdx.x; j < cnt; j += kRadixThreads) {
    const KeyT<W> key = skeys[j];
    const uint32_t d = key_digit(key, shift);
    store_key<W>(out, (uint64_t)gbase[d] + (uint32_t)j - tstart[d], key);
  }
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
static int radix_sort_impl(cusci_ctx* ctx, uint64_t* keys, uint64_t* alt, uint64_t n, int nbits, uint64_t** out_sorted) {
  *out_sorted = keys;
  if (n <= 1) return CUSCI_OK;
  if (n >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "radix sort: n=%llu exceeds 2^32", (unsigned long long)n);
  constexpr int TILE = kRadixThreads * RadixCfg<W>::ITEMS;
  const uint32_t ntiles = (uint32_t)((n + TILE - 1) / TILE);
  Scratch s(ctx);
  uint32_t *hist, *offs;
  CUSCI_TRY(s.get_t((size_t)256 * ntiles, &hist));
  CUSCI_TRY(s.get_t((size_t)256 * ntiles, &offs));
  uint64_t* src = keys;
  uint64_t* dst = alt;
  for (int shift = 0; shift < nbits; shift += 8) {
    CUSCI_LAUNCH(ctx, PT_RADIX_UP, radix_upsweep<W><<<ntiles, kRadixThreads, 0, ctx->stream>>>(src, n, shift, hist, ntiles));
    CUSCI_TRY(scan_exclusive_u32(ctx, hist, offs, (uint64_t)256 * ntiles));
    CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, radix_downsweep<W><<<ntiles, kRadixThreads, 0, ctx->stream>>>(src, dst, n, shift, offs, ntiles));
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  *out_sorted = src;
  return CUSCI_OK;
}

int radix_sort_keys(cusci_ctx* ctx, int W, uint64_t* keys, uint64_t* alt, uint64_t n, int nbits, uint64_t** out_sorted) {
  return W == 1 ? radix_sort_impl<1>(ctx, keys, alt, n, nbits, out_sorted)
                : radix_sort_impl<2>(ctx, keys, alt, n, nbits, out_sorted);
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
