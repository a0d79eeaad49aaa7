// Onesweep LSD radix partitioning of configuration keys (
// PAPER.md:454 "GPU-optimized Radix Sort", :469-470 "dense arrays of uint64
// bitmasks ... ideally suited for GPU-optimized Radix Sort").
//
// B200 design: one pre-pass reads the keys once and builds
// the digit histograms of every pass (per <= 2^28-key portion); each pass is
// then ONE kernel that reads each key once and writes it once (16 B/key/pass
// at W=1): a CTA takes a tile ticket (atomic counter, so predecessors are
// always resident), ranks its 4096 keys with warp match_any + per-warp digit
// counters in shared memory, publishes its per-digit counts, resolves its
// exclusive per-digit prefix by decoupled look-back over the predecessors'
// published counts, stages the tile in digit order in shared memory and
// writes it out with runs of consecutive addresses per digit.  Passes whose
// histogram puts every key in one bin are skipped.  A pass digit is either
// key bits (sort), bits of the owner mix (hash buckets for dedup), or the
// owner itself (partition for the exchange).
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace cusci {

namespace {

constexpr int kOsThreads = 256;
constexpr int kOsWarps = kOsThreads / 32;
constexpr uint64_t kPortionMax = 1ull << 28;  // keys per onesweep portion (30-bit status counters)
// CUSCI_PORTION_LOG2 (16..28) shrinks portions so tests can exercise the multi-portion path
static uint64_t portion_size() {
  static uint64_t v = 0;
  if (!v) {
    const char* e = getenv("CUSCI_PORTION_LOG2");
    int lg = e ? atoi(e) : 28;
    if (lg < 16 || lg > 28) lg = 28;
    v = 1ull << lg;
  }
  return v;
}
constexpr uint32_t kFlagA = 1u << 30, kFlagP = 2u << 30, kCountMask = (1u << 30) - 1;
template <int W> struct OsCfg {
  static constexpr int ITEMS = W == 1 ? 16 : 8;
  static constexpr int TILE = kOsThreads * ITEMS;
};

template <int W>
__device__ __forceinline__ uint32_t digit_of(const KeyT<W>& k, const DigitSpec& d) {
  const uint32_t mask = (1u << d.bits) - 1u;
  if (d.mode == 0) return key_digit_bits(k, d.shift) & mask;
  if (d.mode == 1) return (uint32_t)(owner_mix(k) >> d.shift) & mask;
  if (d.mode == 3) return (uint32_t)(hk_lo(k) >> d.shift) & mask;
  return owner_of<W>(k, d.P);
}

// histograms of all passes, per portion: hist[(portion * npass + pass) * 512 + digit]
template <int W>
__global__ void __launch_bounds__(kOsThreads) digit_hist_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                                               DigitSpecs specs, uint64_t kPortion,
                                                               uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kMaxPasses * 512];
  const int np = specs.n;
  constexpr uint64_t CHUNK = 1ull << 16;  // divides kPortion: a chunk never straddles portions
  for (int i = threadIdx.x; i < np * 512; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned lane = lane_id();
  for (uint64_t c = blockIdx.x; c * CHUNK < n; c += gridDim.x) {
    const uint64_t lo = c * CHUNK, hi = std::min(n, lo + CHUNK);
    const uint64_t portion = lo / kPortion;
    constexpr int HI = 8;  // keys per thread per step, all loads issued first
    for (uint64_t b0 = lo; b0 < hi; b0 += (uint64_t)blockDim.x * HI) {
      KeyT<W> k[HI];
      bool valid[HI];
#pragma unroll
      for (int u = 0; u < HI; u++) {
        const uint64_t i = b0 + (uint64_t)u * blockDim.x + threadIdx.x;
        valid[u] = i < hi;
        if (valid[u]) k[u] = load_key<W>(keys, i);
      }
#pragma unroll
      for (int u = 0; u < HI; u++) {
        for (int p = 0; p < np; p++) {
          const uint32_t d = valid[u] ? digit_of<W>(k[u], specs.d[p]) : 0xffffffffu;
          const uint32_t d0 = __shfl_sync(kFull, d, 0);
          if (__all_sync(kFull, d == d0)) {  // one digit for the whole warp (skewed digits): one add
            if (lane == 0 && d0 != 0xffffffffu) atomicAdd(&h[p * 512 + d0], 32u);
          } else if (valid[u]) {  // shared-memory atomics (3.6x faster than __match_any_sync aggregation)
            atomicAdd(&h[p * 512 + d], 1u);
          }
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < np * 512; i += blockDim.x) {
      const uint32_t v = h[i];
      if (v) atomicAdd(&hist[(portion * np) * 512 + i], v);
      h[i] = 0;
    }
    __syncthreads();
  }
}

template <int W, int RADIX>
__global__ void __launch_bounds__(kOsThreads) onesweep_kernel(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                             uint64_t n, DigitSpec ds,
                                                             const uint64_t* __restrict__ gbase,
                                                             uint32_t* __restrict__ status,
                                                             uint32_t* __restrict__ tile_ctr) {
  constexpr int ITEMS = OsCfg<W>::ITEMS;
  constexpr int TILE = OsCfg<W>::TILE;
  constexpr int DPT = RADIX / kOsThreads;  // digits per thread
  __shared__ uint16_t whist[kOsWarps][RADIX];
  __shared__ uint32_t lstart[RADIX];
  __shared__ uint64_t gdst[RADIX];
  __shared__ uint32_t red[33];
  __shared__ KeyT<W> skeys[TILE];
  __shared__ uint32_t s_tile;
  const int w = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < kOsWarps * RADIX; i += kOsThreads) (&whist[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t base = (uint64_t)tile * TILE;
  KeyT<W> k[ITEMS];
  uint32_t dig[ITEMS];
  const uint64_t wbase = base + (uint64_t)w * (ITEMS * 32) + lane;
  if (base + TILE <= n) {  // full tile: issue every load before any use
#pragma unroll
    for (int i = 0; i < ITEMS; i++) k[i] = load_key<W>(in, wbase + (uint64_t)i * 32);
#pragma unroll
    for (int i = 0; i < ITEMS; i++) dig[i] = digit_of<W>(k[i], ds);
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
      const uint64_t idx = wbase + (uint64_t)i * 32;
      if (idx < n) {
        k[i] = load_key<W>(in, idx);
        dig[i] = digit_of<W>(k[i], ds);
      } else {
        dig[i] = RADIX;
      }
    }
  }
  uint16_t rank[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const uint32_t d = dig[i];
    const unsigned peers = __match_any_sync(kFull, d);
    uint32_t before = 0;
    if (d < RADIX) before = whist[w][d];
    rank[i] = (uint16_t)(before + __popc(peers & lanemask_lt()));
    __syncwarp();
    if (d < RADIX && lane == (unsigned)(__ffs(peers) - 1)) whist[w][d] = (uint16_t)(before + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  // per-digit tile counts (exclusive over warps in place)
  uint32_t cnt[DPT];
  uint32_t my_sum = 0;
#pragma unroll
  for (int j = 0; j < DPT; j++) {
    const int d = threadIdx.x * DPT + j;
    uint32_t c = 0;
#pragma unroll
    for (int x = 0; x < kOsWarps; x++) {
      const uint32_t t = whist[x][d];
      whist[x][d] = (uint16_t)c;
      c += t;
    }
    cnt[j] = c;
    my_sum += c;
  }
  // publish aggregates early so successors can proceed
  volatile uint32_t* st = status;
#pragma unroll
  for (int j = 0; j < DPT; j++) {
    const int d = threadIdx.x * DPT + j;
    st[(size_t)tile * RADIX + d] = (tile == 0 ? kFlagP : kFlagA) | cnt[j];
  }
  // tile-local digit starts (block exclusive scan in digit order)
  uint32_t tot;
  uint32_t ex = block_excl_scan_u32(my_sum, red, tot);
#pragma unroll
  for (int j = 0; j < DPT; j++) {
    lstart[threadIdx.x * DPT + j] = ex;
    ex += cnt[j];
  }
  // decoupled look-back per digit
#pragma unroll
  for (int j = 0; j < DPT; j++) {
    const int d = threadIdx.x * DPT + j;
    uint32_t excl = 0;
    if (tile > 0) {
      int32_t t = (int32_t)tile - 1;
      while (t >= 0) {
        const uint32_t v = st[(size_t)t * RADIX + d];
        if ((v >> 30) == 0) {  // predecessor not published yet: spin
          __nanosleep(20);
          continue;
        }
        excl += v & kCountMask;
        if ((v >> 30) == 2) break;
        t--;
      }
      st[(size_t)tile * RADIX + d] = kFlagP | (excl + cnt[j]);
    }
    gdst[d] = gbase[d] + excl - lstart[d];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const uint32_t d = dig[i];
    if (d < RADIX) skeys[lstart[d] + whist[w][d] + rank[i]] = k[i];
  }
  __syncthreads();
  const uint64_t rem = n - base;
  const int cnt_tile = rem < (uint64_t)TILE ? (int)rem : TILE;
  for (int j = threadIdx.x; j < cnt_tile; j += kOsThreads) {
    const KeyT<W> key = skeys[j];
    store_key<W>(out, gdst[digit_of<W>(key, ds)] + (uint32_t)j, key);
  }
}

// base[d] += inclusive count of digit d over the previous portion (its last
// tile's published prefix): chains the portions of one pass on the device
__global__ void portion_carry_kernel(const uint32_t* __restrict__ last_row, uint64_t* __restrict__ base, int radix) {
  for (int d = threadIdx.x; d < radix; d += blockDim.x) base[d] += last_row[d] & kCountMask;
}

template <int W>
int onesweep_impl(cusci_ctx* ctx, const uint64_t* keys, uint64_t* buf0, uint64_t* buf1, uint64_t n,
                  const DigitSpecs& specs, const uint64_t** out_sorted, uint64_t* hist0) {
  *out_sorted = keys;
  if (hist0 && specs.n)
    for (int d = 0; d < (1 << specs.d[0].bits); d++) hist0[d] = 0;
  if (n == 0 || specs.n == 0) return CUSCI_OK;
  const int np = specs.n;
  const uint64_t kPortion = portion_size();
  const uint64_t nport = (n + kPortion - 1) / kPortion;
  Scratch s(ctx);
  uint32_t* hist;
  uint64_t* gb;
  uint32_t *status, *tctr;
  constexpr int TILE = OsCfg<W>::TILE;
  const uint64_t max_tiles = (std::min(n, kPortion) + TILE - 1) / TILE;
  CUSCI_TRY(s.get_t(nport * np * 512, &hist));
  CUSCI_TRY(s.get_t(nport * np * 512, &gb));
  CUSCI_TRY(s.get_t(max_tiles * 512, &status));
  CUSCI_TRY(s.get_t(64, &tctr));
  CUSCI_CUDA(ctx, cudaMemsetAsync(hist, 0, nport * np * 512 * sizeof(uint32_t), ctx->stream));
  {
    const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 65535) >> 16, (uint64_t)ctx->num_sms * 4));
    CUSCI_LAUNCH(ctx, PT_RADIX_UP, digit_hist_kernel<W><<<blocks, kOsThreads, 0, ctx->stream>>>(keys, n, specs, kPortion, hist));
  }
  std::vector<uint32_t> hh(nport * np * 512);
  CUSCI_CUDA(ctx, cudaMemcpyAsync(hh.data(), hist, hh.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  // portion-0 bases per pass: exclusive prefix of the digit totals (a
  // permutation invariant); later portions are chained on the device
  std::vector<uint64_t> gbh((size_t)np * 512, 0);
  std::vector<bool> trivial(np, false);
  for (int p = 0; p < np; p++) {
    const int R = 1 << specs.d[p].bits;
    uint64_t run = 0;
    for (int d = 0; d < R; d++) {
      uint64_t t = 0;
      for (uint64_t q = 0; q < nport; q++) t += hh[(q * np + p) * 512 + d];
      if (t == n) trivial[p] = true;
      gbh[(size_t)p * 512 + d] = run;
      run += t;
    }
  }
  if (hist0) {
    const int R0 = 1 << specs.d[0].bits;
    for (int d = 0; d < R0; d++) {
      uint64_t t = 0;
      for (uint64_t q = 0; q < nport; q++) t += hh[(q * np + 0) * 512 + d];
      hist0[d] = t;
    }
  }
  CUSCI_CUDA(ctx, cudaMemcpyAsync(gb, gbh.data(), gbh.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  const uint64_t* src = keys;
  uint64_t* dst = buf0;
  for (int p = 0; p < np; p++) {
    if (trivial[p]) continue;
    unsigned prev_tiles = 0;
    for (uint64_t q = 0; q < nport; q++) {
      const uint64_t lo = q * kPortion, cnt = std::min(kPortion, n - lo);
      const unsigned tiles = (unsigned)((cnt + TILE - 1) / TILE);
      const int R = specs.d[p].bits <= 8 ? 256 : 512;  // the kernel's RADIX (status row stride)
      CUSCI_CUDA(ctx, cudaMemsetAsync(tctr, 0, sizeof(uint32_t), ctx->stream));
      uint64_t* gbp = gb + (size_t)p * 512;
      if (q > 0)
        CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, portion_carry_kernel<<<1, 256, 0, ctx->stream>>>(status + (size_t)(prev_tiles - 1) * R, gbp, R));
      CUSCI_CUDA(ctx, cudaMemsetAsync(status, 0, (size_t)tiles * R * sizeof(uint32_t), ctx->stream));
      if (R <= 256)
        CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, onesweep_kernel<W, 256><<<tiles, kOsThreads, 0, ctx->stream>>>(src + lo * W, dst, cnt, specs.d[p], gbp, status, tctr));
      else
        CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, onesweep_kernel<W, 512><<<tiles, kOsThreads, 0, ctx->stream>>>(src + lo * W, dst, cnt, specs.d[p], gbp, status, tctr));
      prev_tiles = tiles;
    }
    src = dst;
    dst = (dst == buf0) ? buf1 : buf0;
  }
  *out_sorted = src;
  return CUSCI_OK;
}

}  // namespace

int onesweep_passes(cusci_ctx* ctx, int W, const uint64_t* in, uint64_t* buf0, uint64_t* buf1, uint64_t n,
                    const DigitSpecs& specs, const uint64_t** out, uint64_t* hist0) {
  if (n >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "radix: n=%llu exceeds 2^32", (unsigned long long)n);
  for (int p = 0; p < specs.n; p++)
    if (specs.d[p].bits < 1 || specs.d[p].bits > 9) return set_error(ctx, CUSCI_E_INVALID_ARG, "radix: bad digit width");
  return W == 1 ? onesweep_impl<1>(ctx, in, buf0, buf1, n, specs, out, hist0)
                : onesweep_impl<2>(ctx, in, buf0, buf1, n, specs, out, hist0);
}

int radix_sort_keys(cusci_ctx* ctx, int W, uint64_t* keys, uint64_t* alt, uint64_t n, int nbits, uint64_t** out_sorted) {
  // 8-bit digits over the significant bits [0, nbits), in groups of kMaxPasses
  const uint64_t* cur = keys;
  for (int sh0 = 0; sh0 < nbits; sh0 += 8 * kMaxPasses) {
    DigitSpecs specs{};
    for (int sh = sh0; sh < nbits && specs.n < kMaxPasses; sh += 8)
      specs.d[specs.n++] = DigitSpec{0, sh, std::min(8, nbits - sh), 0u};
    uint64_t* b0 = (cur == keys) ? alt : keys;
    uint64_t* b1 = (cur == keys) ? keys : alt;
    // pass 0 reads cur and writes b0; later passes alternate b0 <-> b1 (b1 == cur is safe: cur is consumed)
    const uint64_t* o = cur;
    CUSCI_TRY(onesweep_passes(ctx, W, cur, b0, b1, n, specs, &o, nullptr));
    cur = o;
  }
  *out_sorted = const_cast<uint64_t*>(cur);
  return CUSCI_OK;
}

}  // namespace cusci
