// Local de-duplication into the hash order (
// PAPER.md:380-382 local uniqueness filter, :454-460 local sort + unique).
//
// B200 design (reading r13): keys are ordered by the hash
// order pi(j) = (hi, lo) -- a fixed bijection of the key space (hi =
// owner mix, so owner(j) = floor(hi * P / 2^64) is monotone in it) -- instead
// of the big-integer order.  Because pi is uniform, a 2-level MSD partition on
// the top B bits of hi (B = log2(n / ~2k)) puts ~2k keys in every bucket:
//   pass 1  histogram + scatter by the top hb (<= 9) bits (per-tile shared-
//           memory ranks, one global atomic per (tile, digit) on an
//           L2-resident cursor array -- no look-back chain, no stability
//           requirement);
//   pass 2  histogram + scatter by the full B bits, tiles binned locally on
//           the <= 2 pass-1 digits a tile spans (far keys: direct atomics);
// then ONE CTA per bucket: open-addressing hash table in shared memory
// (64-bit atomicCAS / ATOMS.CAS.128) keeps the first copy of each key, and
// the survivors are sorted inside the bucket by a counting sort on the next
// bits of hi plus an insertion sort of the (rare) collisions.  Buckets are
// then concatenated in bucket order: the result is sorted in the hash order
// and unique -- a full sort in two partition passes.  A bucket with more
// distinct keys than its table holds is flagged; the host then finishes with
// a full LSD sort over the hash digits + unique (exact, rare slow path).
#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace cusci {
namespace {

constexpr int kBT = 256;        // threads
constexpr int kBI = 8;          // keys per thread per tile
constexpr int kBTile = kBT * kBI;

template <int W>
__device__ __forceinline__ uint32_t top_bits(const KeyT<W>& k, int bits) {
  return bits ? (uint32_t)(hk_hi(k) >> (64 - bits)) : 0u;
}

// ---------------------------------------------------------------- partition passes
// Segmented MSD passes of <= 8 bits of hi.  A pass = per-tile digit
// histograms written to a matrix laid out group by group ([group][digit]
// [tile]), ONE exclusive scan of that matrix (it then holds every (group,
// digit, tile) output offset), and a scatter: each CTA loads its matrix
// column as shared-memory cursors and, per 4 Ki-key sub-round, ranks its keys
// with shared-memory atomics, stages them in digit order in shared memory and
// writes them out as runs of consecutive addresses (~16 keys = 128 B per
// digit), so HBM sees full sectors.  No global atomics, no look-back, no
// stability requirement.  Tiles (<= 32 Ki keys) never straddle a group.
struct PTile {
  uint64_t start;   // first key
  uint32_t len;     // keys in the tile
  uint32_t stride;  // matrix stride between digits (= tiles of this group)
  uint64_t mbase;   // matrix index of digit 0 of this tile
};
constexpr uint32_t kPTile = 32768;
template <int W> struct SSCfg {
  static constexpr int ITEMS = W == 1 ? 16 : 8;  // keys per thread per sub-round
  static constexpr int SUB = kBT * ITEMS;        // 4096 / 2048 keys (32 KB staged)
};

template <int W>
__global__ void __launch_bounds__(kBT) tile_hist_kernel(const uint64_t* __restrict__ in,
                                                       const PTile* __restrict__ tiles, int bsel, uint32_t dmask,
                                                       uint32_t* __restrict__ mat) {
  __shared__ uint32_t h[256];
  const PTile t = tiles[blockIdx.x];
  for (uint32_t i = threadIdx.x; i <= dmask; i += kBT) h[i] = 0;
  __syncthreads();
  for (uint32_t r0 = 0; r0 < t.len; r0 += kBTile) {
    KeyT<W> k[kBI];
#pragma unroll
    for (int u = 0; u < kBI; u++) {
      const uint32_t i = r0 + u * kBT + threadIdx.x;
      if (i < t.len) k[u] = load_key<W>(in, t.start + i);
    }
#pragma unroll
    for (int u = 0; u < kBI; u++) {
      const uint32_t i = r0 + u * kBT + threadIdx.x;
      if (i < t.len) atomicAdd(&h[top_bits<W>(k[u], bsel) & dmask], 1u);
    }
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d <= dmask; d += kBT) mat[t.mbase + (uint64_t)d * t.stride] = h[d];
}

constexpr int kST = 512;  // scatter threads (2 CTAs / SM at <= 64 registers)
template <int W>
__global__ void __launch_bounds__(kST, 2) tile_scatter_kernel(const uint64_t* __restrict__ in,
                                                             const PTile* __restrict__ tiles, int bsel, uint32_t dmask,
                                                             const uint32_t* __restrict__ offs, uint64_t* __restrict__ out) {
  constexpr int ITEMS = SSCfg<W>::SUB / kST;
  constexpr int SUB = SSCfg<W>::SUB;
  __shared__ uint32_t cur[256], cnt[256], lst[256];
  __shared__ uint32_t red[33];
  __shared__ KeyT<W> stage[SUB];
  __shared__ uint8_t sdig[SUB];
  const PTile t = tiles[blockIdx.x];
  const uint32_t R = dmask + 1;
  if (threadIdx.x < 256) {
    const uint32_t d = threadIdx.x;
    cur[d] = d < R ? offs[t.mbase + (uint64_t)d * t.stride] : 0u;
    cnt[d] = 0;
  }
  __syncthreads();
  for (uint32_t r0 = 0; r0 < t.len; r0 += SUB) {
    const uint32_t m = min((uint32_t)SUB, t.len - r0);
    KeyT<W> k[ITEMS];
    uint32_t dr[ITEMS];  // digit << 16 | rank within the sub-round
#pragma unroll
    for (int u = 0; u < ITEMS; u++) {
      const uint32_t i = u * kST + threadIdx.x;
      if (i < m) k[u] = load_key<W>(in, t.start + r0 + i);
    }
#pragma unroll
    for (int u = 0; u < ITEMS; u++) {
      const uint32_t i = u * kST + threadIdx.x;
      if (i < m) {
        const uint32_t d = top_bits<W>(k[u], bsel) & dmask;
        dr[u] = (d << 16) | atomicAdd(&cnt[d], 1u);
      }
    }
    __syncthreads();
    uint32_t tot;
    const uint32_t c = threadIdx.x < 256 ? cnt[threadIdx.x] : 0u;
    const uint32_t ex = block_excl_scan_u32(c, red, tot);
    if (threadIdx.x < 256) lst[threadIdx.x] = ex;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < ITEMS; u++) {
      const uint32_t i = u * kST + threadIdx.x;
      if (i < m) {
        const uint32_t d = dr[u] >> 16;
        const uint32_t pos = lst[d] + (dr[u] & 0xffffu);
        stage[pos] = k[u];
        sdig[pos] = (uint8_t)d;
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < m; j += kST) {
      const uint32_t dj = sdig[j];
      store_key<W>(out, (uint64_t)cur[dj] + (j - lst[dj]), stage[j]);
    }
    __syncthreads();
    if (threadIdx.x < 256) {
      cur[threadIdx.x] += c;
      cnt[threadIdx.x] = 0;
    }
    __syncthreads();
  }
}

// group offsets after a pass: for old group g with meta {start, tiles, mbase},
// new group g*R + d starts at offs[mbase + d * tiles] (or the old start if empty)
__global__ void group_off_kernel(const uint32_t* __restrict__ offs, const uint4* __restrict__ gmeta, uint32_t G,
                                 int bits, uint32_t n, uint32_t* __restrict__ off) {
  const uint32_t R = 1u << bits;
  const uint32_t id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id > G * R) return;
  if (id == G * R) {
    off[id] = n;
    return;
  }
  const uint32_t g = id >> bits, d = id & (R - 1);
  const uint4 m = gmeta[g];  // x = start, y = tiles, z = mbase
  off[id] = m.y ? offs[m.z + (uint64_t)d * m.y] : m.x;
}

// ---------------------------------------------------------------- per-bucket dedup + sort
// survivor record: the key and its hash-order hi (computed once per key)
template <int W> struct SvRec {
  KeyT<W> key;
  uint64_t hi;
};
template <int W> struct BDCfg {
  static constexpr uint32_t TS = W == 1 ? 4096 : 2048;     // table slots (32 KB)
  static constexpr uint32_t LIMIT = W == 1 ? 2560 : 1280;  // distinct keys per bucket
  static constexpr uint32_t NBMAX = 2048;                  // counting-sort bins
  static constexpr size_t SMEM = (size_t)TS * sizeof(KeyT<W>) + (size_t)LIMIT * sizeof(SvRec<W>);
  static_assert(LIMIT * 2 + NBMAX * 4 <= TS * sizeof(KeyT<W>), "sort scratch must fit the table");
};

__device__ __forceinline__ void cas_slot(KeyT<1>* slot, const KeyT<1>& k, KeyT<1>& old) {
  old.w0 = atomicCAS(reinterpret_cast<unsigned long long*>(&slot->w0), 0ull, (unsigned long long)k.w0);
}
__device__ __forceinline__ void cas_slot(KeyT<2>* slot, const KeyT<2>& k, KeyT<2>& old) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(slot);
  uint64_t o0, o1;
  asm volatile(
      "{\n\t.reg .b128 c, v, o;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.shared.cas.b128 o, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(o0), "=l"(o1)
      : "l"(0ull), "l"(0ull), "l"(k.w0), "l"(k.w1), "r"(sa)
      : "memory");
  old.w0 = o0;
  old.w1 = o1;
}
__device__ __forceinline__ bool kzero(const KeyT<1>& k) { return k.w0 == 0; }
__device__ __forceinline__ bool kzero(const KeyT<2>& k) { return (k.w0 | k.w1) == 0; }

// returns true iff k was inserted (first copy); *full set when no slot found
template <int W>
__device__ __forceinline__ bool tab_insert(KeyT<W>* tab, uint32_t ts, const KeyT<W>& k, uint64_t hi, int* s_zero,
                                           bool* full) {
  if (kzero(k)) return atomicExch(s_zero, 1) == 0;
  uint32_t h = (uint32_t)hi & (ts - 1);  // low bits of hi: uniform within a bucket
  for (uint32_t probe = 0; probe < ts; probe++) {
    const KeyT<W> cur = tab[h];
    if (key_eq(cur, k)) return false;
    if (kzero(cur)) {
      KeyT<W> old;
      cas_slot(&tab[h], k, old);
      if (kzero(old)) return true;
      if (key_eq(old, k)) return false;
    }
    h = (h + 1) & (ts - 1);
  }
  *full = true;
  return false;
}

// A CTA walks a chunk of consecutive buckets and processes them in RUNS:
// as many consecutive buckets as fit RUN_CAP keys share one table clear, one
// dedup and one sort (buckets hold ~1-2 Ki keys but often few distinct ones,
// so per-bucket fixed costs would dominate).  The run's survivors (key + hi,
// hi computed once per key) are counting-sorted by hi and written at the run's
// first bucket offset; surv[] gets the run count there and 0 for the run's
// other buckets, which is what the compaction expects.
template <int W>
__global__ void __launch_bounds__(kBT, 3) bucket_dedup_sort_kernel(const uint64_t* __restrict__ part,
                                                                  const uint32_t* __restrict__ off, uint32_t nb, int B,
                                                                  uint32_t chunk, uint64_t* __restrict__ tmp,
                                                                  uint32_t* __restrict__ surv,
                                                                  unsigned long long* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char bsm[];
  constexpr uint32_t TS = BDCfg<W>::TS, LIMIT = BDCfg<W>::LIMIT;
  constexpr uint32_t RUN_CAP = TS / 2;
  constexpr int PER_MAX = (LIMIT + kBT - 1) / kBT;
  KeyT<W>* tab = reinterpret_cast<KeyT<W>*>(bsm);
  SvRec<W>* sv = reinterpret_cast<SvRec<W>*>(tab + TS);
  // after the dedup the table region is reused: sorted survivor indices + bin counters
  uint16_t* so = reinterpret_cast<uint16_t*>(tab);
  uint32_t* bins = reinterpret_cast<uint32_t*>(so + LIMIT);
  __shared__ int s_zero;
  __shared__ uint32_t s_ns, s_b1;
  __shared__ int s_bad;
  __shared__ uint32_t red[33];
  __shared__ uint32_t soff[kBT + 1];  // the chunk's bucket offsets (one coalesced load)
  const uint32_t nchunks = (nb + chunk - 1) / chunk;
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint32_t cb0 = c * chunk, cb1 = min(nb, (c + 1) * chunk);
    for (uint32_t x = threadIdx.x; x <= cb1 - cb0; x += kBT) soff[x] = off[cb0 + x];
    __syncthreads();
    uint32_t b0 = cb0;
    while (b0 < cb1) {
      if (threadIdx.x == 0) {
        const uint32_t s0 = soff[b0 - cb0];
        uint32_t b1 = b0 + 1;
        while (b1 < cb1 && soff[b1 + 1 - cb0] - s0 <= RUN_CAP) b1++;
        s_b1 = b1;
        s_zero = 0;
        s_ns = 0;
        s_bad = 0;
      }
      __syncthreads();
      const uint32_t b1 = s_b1;
      const uint32_t start = soff[b0 - cb0], cnt = soff[b1 - cb0] - start;
      if (cnt == 0) {
        for (uint32_t x = b0 + threadIdx.x; x < b1; x += kBT) surv[x] = 0;
        __syncthreads();
        b0 = b1;
        continue;
      }
      uint32_t ts = 64;
      while (ts < 2 * cnt && ts < TS) ts <<= 1;
      for (uint32_t i = threadIdx.x; i < ts; i += kBT) tab[i] = KeyT<W>{};
      __syncthreads();
      bool full = false;
      for (uint32_t r0 = 0; r0 < cnt; r0 += kBTile) {
        KeyT<W> kc[kBI];
#pragma unroll
        for (int u = 0; u < kBI; u++) {
          const uint32_t i = r0 + u * kBT + threadIdx.x;
          if (i < cnt) kc[u] = load_key<W>(part, (uint64_t)start + i);
        }
#pragma unroll
        for (int u = 0; u < kBI; u++) {
          const uint32_t i = r0 + u * kBT + threadIdx.x;
          if (i < cnt) {
            const uint64_t hi = hk_hi(kc[u]);
            if (tab_insert<W>(tab, ts, kc[u], hi, &s_zero, &full)) {
              const uint32_t j = atomicAdd(&s_ns, 1u);
              if (j < LIMIT) sv[j] = SvRec<W>{kc[u], hi};
            }
          }
        }
      }
      if (full) s_bad = 1;
      __syncthreads();
      const uint32_t ns = s_ns;
      if (s_bad || ns > LIMIT) {
        // overflow (one huge bucket): pass it through unfiltered, the host finishes
        for (uint32_t i = threadIdx.x; i < cnt; i += kBT)
          store_key<W>(tmp, (uint64_t)start + i, load_key<W>(part, (uint64_t)start + i));
        for (uint32_t x = b0 + threadIdx.x; x < b1; x += kBT) surv[x] = x == b0 ? cnt : 0u;
        if (threadIdx.x == 0) atomicAdd(&flags[0], 1ull);
        __syncthreads();
        b0 = b1;
        continue;
      }
      // counting sort of the survivors on hi relative to the run's range
      int sb = 8;
      while ((1u << sb) < ns && sb < 11) sb++;
      const uint32_t NB = 1u << sb;
      int span = 64 - B;  // bits of hi below the bucket id
      for (uint32_t w = b1 - b0 - 1; w; w >>= 1) span++;
      const uint64_t base = B ? ((uint64_t)b0 << (64 - B)) : 0ull;
      const int shift = span > sb ? span - sb : 0;
      for (uint32_t i = threadIdx.x; i < NB; i += kBT) bins[i] = 0;
      __syncthreads();
      uint32_t myrank[PER_MAX];
#pragma unroll
      for (int u = 0; u < PER_MAX; u++) {
        const uint32_t i = u * kBT + threadIdx.x;
        if (i < ns) myrank[u] = atomicAdd(&bins[(uint32_t)((sv[i].hi - base) >> shift) & (NB - 1)], 1u);
      }
      __syncthreads();
      const uint32_t per = NB / kBT;
      uint32_t loc = 0;
      uint32_t cnts[BDCfg<W>::NBMAX / kBT];
      for (uint32_t j = 0; j < per; j++) {
        cnts[j] = bins[threadIdx.x * per + j];
        loc += cnts[j];
      }
      uint32_t tot;
      uint32_t ex = block_excl_scan_u32(loc, red, tot);
      for (uint32_t j = 0; j < per; j++) {
        bins[threadIdx.x * per + j] = ex;  // bin start
        ex += cnts[j];
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < PER_MAX; u++) {
        const uint32_t i = u * kBT + threadIdx.x;
        if (i < ns) so[bins[(uint32_t)((sv[i].hi - base) >> shift) & (NB - 1)] + myrank[u]] = (uint16_t)i;
      }
      __syncthreads();
      // order the (few) keys that share a bin: insertion sort in the hash order
      for (uint32_t bi = threadIdx.x; bi < NB; bi += kBT) {
        const uint32_t s0 = bins[bi];
        const uint32_t s1 = (bi + 1 < NB) ? bins[bi + 1] : ns;
        for (uint32_t i = s0 + 1; i < s1; i++) {
          const uint16_t x = so[i];
          const uint64_t hx = sv[x].hi;
          uint32_t j = i;
          while (j > s0) {
            const uint16_t y = so[j - 1];
            const uint64_t hy = sv[y].hi;
            const bool lt = W == 1 ? hx < hy : (hx < hy || (hx == hy && hk_lo(sv[x].key) < hk_lo(sv[y].key)));
            if (!lt) break;
            so[j] = y;
            j--;
          }
          so[j] = x;
        }
      }
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < ns; i += kBT) store_key<W>(tmp, (uint64_t)start + i, sv[so[i]].key);
      for (uint32_t x = b0 + threadIdx.x; x < b1; x += kBT) surv[x] = x == b0 ? ns : 0u;
      __syncthreads();
      b0 = b1;
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kBT) bucket_compact_kernel(const uint64_t* __restrict__ tmp,
                                                            const uint32_t* __restrict__ off,
                                                            const uint32_t* __restrict__ surv,
                                                            const uint64_t* __restrict__ soff, uint32_t nb,
                                                            uint64_t* __restrict__ out) {
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const uint32_t start = off[b], ns = surv[b];
    const uint64_t o = soff[b];
    for (uint32_t i = threadIdx.x; i < ns; i += kBT) store_key<W>(out, o + i, load_key<W>(tmp, (uint64_t)start + i));
  }
}

// boundaries of the owner ranges in a hash-ordered array: bnd[r] = first index with owner >= r
template <int W>
__global__ void owner_bounds_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint32_t P, uint64_t* __restrict__ bnd) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > P) return;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (owner_of<W>(load_key<W>(keys, mid), P) < r) lo = mid + 1;
    else hi = mid;
  }
  bnd[r] = lo;
}

template <int W>
int local_dedup_impl(cusci_ctx* ctx, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* n_out) {
  *n_out = 0;
  if (n == 0) return CUSCI_OK;
  Scratch s(ctx);
  // B bits of hi: ~<= 2048 keys per bucket on average
  int B = 0;
  while ((n >> B) > 1792 && B < 22) B++;  // <= LIMIT distinct keys per bucket w.h.p.
  const uint32_t nb = 1u << B;
  uint64_t *a, *b2;
  uint32_t *hist, *off, *cur, *surv;
  uint64_t *surv64, *soff;
  unsigned long long* flags;
  CUSCI_TRY(s.get_t(n * W, &a));
  CUSCI_TRY(s.get_t(n * W, &b2));
  CUSCI_TRY(s.get_t(nb + 1, &hist));
  CUSCI_TRY(s.get_t(nb + 1, &off));
  CUSCI_TRY(s.get_t(nb + 1, &cur));
  CUSCI_TRY(s.get_t(nb + 1, &surv));
  CUSCI_TRY(s.get_t(nb + 1, &surv64));
  CUSCI_TRY(s.get_t(nb + 1, &soff));
  CUSCI_TRY(s.get_t(2, &flags));
  CUSCI_CUDA(ctx, cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned long long), ctx->stream));
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + kBTile - 1) / kBTile, (uint64_t)ctx->num_sms * 8));
  const uint64_t* part = in;
  if (B > 0) {
    // segmented MSD passes of <= 8 bits over the top B bits of hi
    const int np = (B + 7) / 8;
    int done = 0;
    std::vector<uint32_t> gstart{0u, (uint32_t)n};  // current groups (host)
    uint64_t* dst = a;
    for (int pi = 0; pi < np; pi++) {
      const int bits = (B - done + (np - pi) - 1) / (np - pi);  // even split
      const uint32_t R = 1u << bits;
      const uint32_t G = (uint32_t)gstart.size() - 1;
      std::vector<PTile> tl;
      std::vector<uint4> gm(G);
      tl.reserve(n / kPTile + G + 1);
      uint64_t mb = 0;
      for (uint32_t g = 0; g < G; g++) {
        const uint64_t gs = gstart[g], ge = gstart[g + 1];
        const uint32_t chunks = (uint32_t)((ge - gs + kPTile - 1) / kPTile);
        gm[g] = make_uint4((uint32_t)gs, chunks, (uint32_t)mb, 0u);
        for (uint32_t c = 0; c < chunks; c++) {
          const uint64_t st = gs + (uint64_t)c * kPTile;
          tl.push_back(PTile{st, (uint32_t)std::min<uint64_t>(kPTile, ge - st), chunks, mb + c});
        }
        mb += (uint64_t)R * chunks;
      }
      if (mb >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "dedup: partition matrix too large");
      const uint32_t nt = (uint32_t)tl.size();
      Scratch ps(ctx);
      PTile* dtl;
      uint4* dgm;
      uint32_t *mat, *offs, *goff;
      CUSCI_TRY(ps.get_t(std::max<uint32_t>(nt, 1), &dtl));
      CUSCI_TRY(ps.get_t(std::max<uint32_t>(G, 1), &dgm));
      CUSCI_TRY(ps.get_t(std::max<uint64_t>(mb, 1), &mat));
      CUSCI_TRY(ps.get_t(std::max<uint64_t>(mb, 1), &offs));
      CUSCI_TRY(ps.get_t((uint64_t)G * R + 1, &goff));
      CUSCI_CUDA(ctx, cudaMemcpyAsync(dtl, tl.data(), nt * sizeof(PTile), cudaMemcpyHostToDevice, ctx->stream));
      CUSCI_CUDA(ctx, cudaMemcpyAsync(dgm, gm.data(), G * sizeof(uint4), cudaMemcpyHostToDevice, ctx->stream));
      const int sel = done + bits;
      CUSCI_LAUNCH(ctx, PT_RADIX_UP, tile_hist_kernel<W><<<nt, kBT, 0, ctx->stream>>>(part, dtl, sel, R - 1, mat));
      CUSCI_TRY(scan_exclusive_u32(ctx, mat, offs, mb));
      CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, tile_scatter_kernel<W><<<nt, kST, 0, ctx->stream>>>(part, dtl, sel, R - 1, offs, dst));
      uint32_t* goff_final = (pi == np - 1) ? off : goff;
      CUSCI_LAUNCH(ctx, PT_SCATTER, group_off_kernel<<<(unsigned)(((uint64_t)G * R + 1 + 255) / 256), 256, 0, ctx->stream>>>(offs, dgm, G, bits, (uint32_t)n, goff_final));
      if (pi < np - 1) {
        gstart.resize((size_t)G * R + 1);
        CUSCI_CUDA(ctx, cudaMemcpyAsync(gstart.data(), goff, gstart.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                        ctx->stream));
      }
      CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // host tables die at scope end
      part = dst;
      dst = (dst == a) ? b2 : a;
      done += bits;
    }
  } else {
    const uint32_t o2[2] = {0u, (uint32_t)n};
    memcpy(ctx->host_pinned, o2, sizeof(o2));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(off, ctx->host_pinned, sizeof(o2), cudaMemcpyHostToDevice, ctx->stream));
    CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  uint64_t* tmp = (part == a) ? b2 : a;
  static bool attr[3] = {false, false, false};
  if (!attr[W]) {
    CUSCI_CUDA(ctx, cudaFuncSetAttribute(bucket_dedup_sort_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)BDCfg<W>::SMEM));
    attr[W] = true;
  }
  static int dper[3] = {0, 0, 0};
  if (!dper[W]) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&dper[W], bucket_dedup_sort_kernel<W>, kBT, BDCfg<W>::SMEM);
    if (dper[W] < 1) dper[W] = 1;
  }
  const uint32_t chunk = 128;  // consecutive buckets per CTA work item (<= kBT)
  const uint32_t nchunks = (nb + chunk - 1) / chunk;
  const unsigned dgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nchunks, (uint64_t)ctx->num_sms * dper[W]));
  CUSCI_LAUNCH(ctx, PT_HASH, bucket_dedup_sort_kernel<W><<<dgrid, kBT, BDCfg<W>::SMEM, ctx->stream>>>(part, off, nb, B, chunk, tmp, surv, flags));
  // compact the buckets' survivors in bucket order
  CUSCI_CUDA(ctx, cudaMemsetAsync(surv64, 0, (nb + 1) * sizeof(uint64_t), ctx->stream));
  CUSCI_CUDA(ctx, cudaMemcpy2DAsync(surv64, sizeof(uint64_t), surv, sizeof(uint32_t), sizeof(uint32_t), nb,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
  CUSCI_TRY(scan_exclusive_u64(ctx, surv64, soff, nb + 1, nullptr));
  CUSCI_LAUNCH(ctx, PT_SCATTER, bucket_compact_kernel<W><<<dgrid, kBT, 0, ctx->stream>>>(tmp, off, surv, soff, nb, out));
  uint64_t h[2];
  CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, soff + nb, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaMemcpyAsync((char*)ctx->host_pinned + 8, flags, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(h, ctx->host_pinned, sizeof(h));
  *n_out = h[0];
  if (h[1]) {
    // rare slow path: some bucket overflowed its table -> full LSD sort over the
    // hash digits (lo then hi for W = 2) + adjacent unique
    DigitSpecs sp{};
    const uint64_t m = h[0];
    uint64_t* cur_buf = out;
    for (int part_i = (W == 2 ? 0 : 1); part_i < 2; part_i++) {
      sp = DigitSpecs{};
      for (int sh = 0; sh < 64; sh += 8) sp.d[sp.n++] = DigitSpec{part_i == 0 ? 3 : 1, sh, 8, 0u};
      const uint64_t* o = cur_buf;
      CUSCI_TRY(onesweep_passes(ctx, W, cur_buf, a, b2, m, sp, &o, nullptr));
      if (o != out) CUSCI_CUDA(ctx, cudaMemcpyAsync(out, o, m * W * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    uint64_t* cnt;
    CUSCI_TRY(s.get_t(1, &cnt));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(a, out, m * W * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    CUSCI_TRY(unique_sorted_keys(ctx, W, a, m, out, cnt));
    CUSCI_TRY(read_u64(ctx, cnt, n_out, 1));
  }
  return CUSCI_OK;
}

template <int W>
int owner_bounds_impl(cusci_ctx* ctx, const uint64_t* keys, uint64_t n, int P, uint64_t* counts) {
  Scratch s(ctx);
  uint64_t* bnd;
  CUSCI_TRY(s.get_t(P + 1, &bnd));
  CUSCI_LAUNCH(ctx, PT_SCATTER, owner_bounds_kernel<W><<<(P + 1 + 63) / 64, 64, 0, ctx->stream>>>(keys, n, (uint32_t)P, bnd));
  uint64_t hb[513];
  CUSCI_TRY(read_u64(ctx, bnd, hb, P + 1));
  for (int r = 0; r < P; r++) counts[r] = hb[r + 1] - hb[r];
  return CUSCI_OK;
}

}  // namespace

int local_dedup(cusci_ctx* ctx, int W, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* n_out) {
  if (n >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "dedup: n=%llu exceeds 2^32", (unsigned long long)n);
  return W == 1 ? local_dedup_impl<1>(ctx, in, n, out, n_out) : local_dedup_impl<2>(ctx, in, n, out, n_out);
}

int owner_counts(cusci_ctx* ctx, int W, const uint64_t* keys, uint64_t n, int P, uint64_t* counts) {
  return W == 1 ? owner_bounds_impl<1>(ctx, keys, n, P, counts) : owner_bounds_impl<2>(ctx, keys, n, P, counts);
}

}  // namespace cusci
