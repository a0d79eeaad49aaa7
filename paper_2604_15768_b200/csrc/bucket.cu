// Local de-duplication into the hash order (
// PAPER.md:380-382 local uniqueness filter, :454-460 local sort + unique).
//
// B200 design (reading r13): keys are ordered by the hash
// order pi(j) = (hi, lo) -- a fixed bijection of the key space (hi = owner
// mix, so owner(j) = floor(hi * P / 2^64) is monotone in it) -- instead of the
// big-integer order.  Because pi is uniform, an MSD partition on the top B
// bits of hi puts the same number of DISTINCT keys (~2-3 Ki) in every bucket,
// and each bucket is then de-duplicated and sorted inside shared memory:
//   pass 1  per-tile histograms of the top (<= 8) bits + a HyperLogLog
//           sketch of the distinct count D (2 Ki registers); one scan; a
//           TMA-pipelined, shared-memory-staged scatter that also maps keys to
//           their pi-values (read directly by every later step);
//   plan    B = log2(D / DT) bits in total (the sketch decides how many
//           partition passes a call needs: high redundancy -> fewer, larger
//           buckets);
//   pass k  (0-2 more) segmented passes of <= 9 bits;
//   dedup   one CTA per SM takes buckets in order from a ticket counter;
//           each bucket's keys are loaded ILP-wide into an ORDER-PRESERVING
//           open-addressing table in shared memory (home = the bits of hi
//           below the bucket id scaled to the table, linear probing, no wrap):
//           every cluster holds exactly the keys whose homes fall inside it,
//           so a survivor's rank is its cluster's start + the keys of its
//           cluster smaller than it; the survivors are mapped back to keys (exact inverse mix) and
//           written at their final positions: each bucket's output offset
//           comes from a decoupled look-back over the buckets' counts (no
//           pack pass).
// The result is unique and sorted in the hash order.  A bucket with more
// distinct keys than its table holds is flagged; the host then finishes with
// a full LSD sort over the hash digits + unique (exact, rare slow path).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <vector>

#include "internal.cuh"

namespace cusci {
namespace {

constexpr int kBT = 256;        // threads (hist, dedup, pack)
constexpr int kBI = 8;          // keys per thread per hist round
constexpr int kBTile = kBT * kBI;
constexpr int kHllLog = 11;     // HyperLogLog: 2^11 registers (~2.3% standard error)
constexpr uint32_t kHllM = 1u << kHllLog;
#ifndef CUSCI_HLL_SAMPLE
#define CUSCI_HLL_SAMPLE 256  // 16 -> 256: a warp rarely holds a sampled key (part_scatter 15.16 -> 14.39 ms per N2 batch, same plan)
#endif
constexpr uint32_t kHllSample = CUSCI_HLL_SAMPLE;  // the sketch sees a 1/kHllSample hash sample of the keys

// digit source: the top bits of the pi-value's hi word (w0)
template <int W>
__device__ __forceinline__ uint32_t top_bits(const KeyT<W>& p, int bits) {
  return bits ? (uint32_t)(p.w0 >> (64 - bits)) : 0u;
}
// the top `bits` (>= 1) bits of hi: no zero-width case on the hot paths
template <int W>
__device__ __forceinline__ uint32_t top_bits_nz(const KeyT<W>& p, int bits) {
  return (uint32_t)(p.w0 >> (64 - bits));
}
// key i of the pass input as a pi-value (RAW: the caller's keys, mixed here once)
template <int W, bool RAW>
__device__ __forceinline__ KeyT<W> load_pi(const uint64_t* in, uint64_t i) {
  const KeyT<W> k = load_key<W>(in, i);
  return RAW ? to_pi(k) : k;
}

// ---------------------------------------------------------------- partition passes
// Segmented MSD passes.  A pass = per-tile digit histograms written to a
// matrix laid out group by group ([group][digit][tile]), ONE exclusive scan of
// that matrix (it then holds every (group, digit, tile) output offset), and a
// scatter: each CTA loads its matrix column as shared-memory cursors and, per
// 4 Ki-key sub-round, ranks its keys with shared-memory atomics, stages them
// in digit order in shared memory and writes them out as runs of consecutive
// addresses, so HBM sees full sectors.  No global atomics, no look-back, no
// stability requirement.  Tiles (<= 32 Ki keys) never straddle a group.
struct PTile {
  uint64_t start;   // first key
  uint32_t len;     // keys in the tile
  uint32_t stride;  // matrix stride between digits (= tiles of this group)
  uint64_t mbase;   // matrix index of digit 0 of this tile
};
constexpr uint32_t kPTileDefault = 65536;  // keys per partition tile (one scatter CTA)
template <int W> struct SSCfg {
  static constexpr int SUB = W == 1 ? 4096 : 2048;  // keys per scatter sub-round (32 KB)
};

// histogram pass; the first (RAW) pass also feeds the HyperLogLog sketch
// (register = low bits of hi, rank = leading zeros of hi + 1; a register is
// only written when the rank grows, so almost every update is one load)
template <int W, bool RAW, int RB>
__global__ void __launch_bounds__(kBT) tile_hist_kernel(const uint64_t* __restrict__ in,
                                                       const PTile* __restrict__ tiles, uint32_t ntiles, int bsel,
                                                       uint32_t dmask, uint32_t* __restrict__ mat,
                                                       uint32_t* __restrict__ hll) {
  __shared__ uint32_t h[1 << RB];
  __shared__ uint32_t reg[RAW ? kHllM : 1];
  if (RAW)
    for (uint32_t i = threadIdx.x; i < kHllM; i += kBT) reg[i] = 0;
  for (uint32_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const PTile t = tiles[ti];
    for (uint32_t i = threadIdx.x; i <= dmask; i += kBT) h[i] = 0;
    __syncthreads();
    for (uint32_t r0 = 0; r0 < t.len; r0 += kBTile) {
      KeyT<W> k[kBI];
#pragma unroll
      for (int u = 0; u < kBI; u++) {
        const uint32_t i = r0 + u * kBT + threadIdx.x;
        if (i < t.len) k[u] = load_pi<W, RAW>(in, t.start + i);
      }
#pragma unroll
      for (int u = 0; u < kBI; u++) {
        const uint32_t i = r0 + u * kBT + threadIdx.x;
        if (i < t.len) {
          atomicAdd(&h[top_bits<W>(k[u], bsel) & dmask], 1u);
          if (RAW) {
            const uint64_t hv = k[u].w0;  // hi: a 64-bit hash of the whole key
            // hash-sampled sketch: only keys with bits [11, 15) of hi zero enter
            // (a key is always or never sampled, so the sample's distinct count is D / 16)
            if (((hv >> kHllLog) & (kHllSample - 1)) == 0) {
              const uint32_t idx = (uint32_t)hv & (kHllM - 1);
              const uint32_t rho = (uint32_t)min(__clzll(hv), 64 - kHllLog - 4) + 1;
              if (rho > reg[idx]) atomicMax(&reg[idx], rho);
            }
          }
        }
      }
    }
    __syncthreads();
    for (uint32_t d = threadIdx.x; d <= dmask; d += kBT) mat[t.mbase + (uint64_t)d * t.stride] = h[d];
  }
  if (RAW) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kHllM; i += kBT)
      if (reg[i]) atomicMax(&hll[i], reg[i]);
  }
}

constexpr int kST = 512;  // scatter threads
constexpr int kSRing = 3;  // scatter input ring: one sub-round being ranked/staged, two in flight
// dynamic shared memory: the TMA input ring (a slot doubles as the digit-ordered
// stage of its own sub-round), digits, cursors
template <int W, int RB> constexpr size_t scatter_smem() {
  return kSRing * ((size_t)SSCfg<W>::SUB + 2) * sizeof(KeyT<W>) + (size_t)SSCfg<W>::SUB * (RB > 8 ? 2 : 1) +
         4 * sizeof(uint32_t) * (1u << RB);
}

// thread 0: bulk-copy keys [s, s + len) into buf so that key s + i lands at
// buf[i + (s & 1)] (W = 1) / buf[i] (W = 2).  Only the 16-byte aligned core is
// copied; keys outside it (an odd head or tail, W = 1) are read from global by
// their consumer (scatter_key).  Returns the bytes the barrier expects (may be 0).
template <int W>
__device__ __forceinline__ uint32_t issue_core(const uint64_t* in, uint64_t s, uint32_t len, KeyT<W>* buf,
                                               uint64_t* bar) {
  if (W == 1) {
    const uint64_t a0 = (s + 1) & ~1ull, a1 = (s + len) & ~1ull;
    if (a1 <= a0) return 0;
    const uint32_t bytes = (uint32_t)((a1 - a0) * 8);
    tma_load_1d(buf + (a0 - s) + (s & 1), in + a0, bytes, bar);
    return bytes;
  } else {
    if (!len) return 0;
    tma_load_1d(buf, in + 2 * s, len * 16u, bar);
    return len * 16u;
  }
}
template <int W>
__device__ __forceinline__ KeyT<W> scatter_key(const uint64_t* in, uint64_t s, uint32_t i, uint32_t len,
                                               const KeyT<W>* buf, bool tma) {
  if (!tma) return load_key<W>(in, s + i);
  if (W == 1) {
    const uint64_t g = s + i;
    const bool core = g >= ((s + 1) & ~1ull) && g < ((s + len) & ~1ull);
    return core ? buf[i + (s & 1)] : load_key<W>(in, g);
  }
  return buf[i];
}

// The tile streams through shared memory by 1-D TMA bulk copies into a ring of
// kSRing slots: two sub-rounds are in flight while the current one is ranked.
// Its keys are held in registers after ranking, so the current slot itself is
// reused as the digit-ordered stage (its next TMA is issued only after the
// round's closing barrier).
template <int W, bool RAW, int RB>
__global__ void __launch_bounds__(kST, 2) tile_scatter_kernel(const uint64_t* __restrict__ in, int use_tma,
                                                             const PTile* __restrict__ tiles, int bsel, uint32_t dmask,
                                                             const uint32_t* __restrict__ offs, uint64_t* __restrict__ out) {
  constexpr int ITEMS = SSCfg<W>::SUB / kST;  // keys per thread per sub-round
  constexpr int SUB = SSCfg<W>::SUB;
  constexpr uint32_t RMAX = 1u << RB;
  using Dig = typename std::conditional<(RB > 8), uint16_t, uint8_t>::type;
  extern __shared__ __align__(16) unsigned char ssm[];  // scatter_smem<W, RB>() bytes
  KeyT<W>* ring = reinterpret_cast<KeyT<W>*>(ssm);       // [kSRing][SUB + 2]
  uint32_t* cur = reinterpret_cast<uint32_t*>(ring + kSRing * (SUB + 2));
  uint32_t* cnt = cur + RMAX;
  uint32_t* lst = cnt + RMAX;
  uint32_t* dl = lst + RMAX;
  Dig* sdig = reinterpret_cast<Dig*>(dl + RMAX);
  __shared__ __align__(8) uint64_t bar[kSRing];
  const PTile t = tiles[blockIdx.x];
  const uint32_t R = dmask + 1;
  const bool tma = use_tma && ((reinterpret_cast<uintptr_t>(in) & 15u) == 0);
  for (uint32_t d = threadIdx.x; d < RMAX; d += kST) {
    cur[d] = d < R ? offs[t.mbase + (uint64_t)d * t.stride] : 0u;
    cnt[d] = 0;
  }
  const uint32_t nsub = (t.len + SUB - 1) / SUB;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSRing; i++) mbar_init(&bar[i], 1);
    mbar_init_fence();
  }
  __syncthreads();
  auto issue = [&](uint32_t r) {  // thread 0: sub-round r -> slot r % kSRing
    const uint32_t sl = r % kSRing;
    fence_proxy_async_smem();
    issue_core<W>(in, t.start + (uint64_t)r * SUB, min((uint32_t)SUB, t.len - r * SUB), ring + sl * (SUB + 2), &bar[sl]);
  };
  if (tma && threadIdx.x == 0)
    for (uint32_t r = 0; r < min(nsub, (uint32_t)kSRing - 1); r++) issue(r);
  uint32_t phase = 0;
  for (uint32_t r = 0; r < nsub; r++) {
    const uint32_t sl = r % kSRing, r0 = r * SUB;
    const uint32_t m = min((uint32_t)SUB, t.len - r0);
    KeyT<W>* buf = ring + sl * (SUB + 2);
    if (tma) {
      // keep kSRing - 1 sub-rounds in flight: r + kSRing - 1 goes into the slot
      // freed by the previous round's closing barrier
      if (threadIdx.x == 0 && r + kSRing - 1 < nsub) issue(r + kSRing - 1);
      const uint64_t s0 = t.start + r0;  // same arithmetic as issue_core: was a copy issued?
      const bool issued = W == 1 ? (((s0 + m) & ~1ull) > ((s0 + 1) & ~1ull)) : m > 0;
      if (issued) {
        mbar_wait(&bar[sl], (phase >> sl) & 1u);
        phase ^= 1u << sl;
      }
    }
    KeyT<W> k[ITEMS];
    uint32_t dr[ITEMS];  // digit << 16 | rank within the sub-round
    // keys [c0, c1) of the sub-round are in the TMA core (W = 1: an odd head /
    // tail key is read from global); key i sits at buf[i + c0]
    const uint32_t c0 = (W == 1 && tma) ? (uint32_t)((t.start + r0) & 1u) : 0u;
    const uint32_t c1 = !tma ? 0u : (W == 1 ? m - (uint32_t)((t.start + r0 + m) & 1u) : m);
#pragma unroll
    for (int u = 0; u < ITEMS; u++) {
      const uint32_t i = u * kST + threadIdx.x;
      if (i < m) {
        k[u] = (i >= c0 && i < c1) ? buf[i + c0] : load_key<W>(in, t.start + r0 + i);
        if (RAW) k[u] = to_pi(k[u]);
        const uint32_t d = top_bits<W>(k[u], bsel) & dmask;
        dr[u] = (d << 16) | atomicAdd(&cnt[d], 1u);
      }
    }
    __syncthreads();  // every key of the slot is in registers: the slot becomes the stage
    // warp 0: exclusive scan of the sub-round digit counts (lane: RMAX/32
    // consecutive digits); per digit the stage offset lst, the stage -> output
    // offset dl, the advanced cursor, and the counter reset for the next round
    if (threadIdx.x < 32) {
      constexpr uint32_t DPL = RMAX / 32;
      uint32_t c[DPL], loc = 0;
#pragma unroll
      for (uint32_t j = 0; j < DPL; j++) {
        c[j] = cnt[threadIdx.x * DPL + j];
        loc += c[j];
      }
      uint32_t inc = loc;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if ((int)threadIdx.x >= o) inc += y;
      }
      uint32_t ex = inc - loc;
#pragma unroll
      for (uint32_t j = 0; j < DPL; j++) {
        const uint32_t d = threadIdx.x * DPL + j;
        lst[d] = ex;
        dl[d] = cur[d] - ex;
        cur[d] += c[j];
        cnt[d] = 0;
        ex += c[j];
      }
    }
    __syncthreads();
    KeyT<W>* stage = buf;
#pragma unroll
    for (int u = 0; u < ITEMS; u++) {
      const uint32_t i = u * kST + threadIdx.x;
      if (i < m) {
        const uint32_t d = dr[u] >> 16;
        const uint32_t pos = lst[d] + (dr[u] & 0xffffu);
        stage[pos] = k[u];
        sdig[pos] = (Dig)d;
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < m; j += kST) store_key<W>(out, (uint64_t)(dl[sdig[j]] + j), stage[j]);
    __syncthreads();  // the stage (this ring slot) is read out: its next TMA may be issued
  }
}

// a digit's stage -> output delta for the hist-free scatters: run start - stage
// start + SUB (never ~0: the run start is < 2^63), or ~0 for "no write"
template <int W>
__device__ __forceinline__ unsigned long long stage_delta(unsigned long long b, uint32_t l) {
  return b == ~0ull ? ~0ull : b + (unsigned long long)SSCfg<W>::SUB - l;
}

template <int W, int RB> constexpr size_t scatter_atomic_smem() {
  return kSRing * ((size_t)SSCfg<W>::SUB + 2) * sizeof(KeyT<W>);  // the ring (digit tables: static)
}

// The last (bucket-forming) pass after a hist-free first pass, also without a
// histogram: every bucket (group g, digit d) gets a region of cap2 keys and the
// tile reserves its runs with one global atomic per (sub-round, digit).  The
// tile's group index is in PTile::mbase.  Overflow -> *ovf and nothing is
// written past a region (the host then redoes the pass with histograms).
// RB = 8 or 9 digit bits (2^RB <= kST: one thread per digit).
template <int W, int RB>
__global__ void __launch_bounds__(kST, 2) tile_scatter_atomic_kernel(const uint64_t* __restrict__ in, int use_tma,
                                                                    const PTile* __restrict__ tiles, int bsel,
                                                                    uint32_t R, unsigned long long* __restrict__ gcur,
                                                                    uint64_t cap2, uint64_t* __restrict__ out,
                                                                    int* __restrict__ ovf) {
  constexpr int ITEMS = SSCfg<W>::SUB / kST;
  constexpr int SUB = SSCfg<W>::SUB;
  constexpr uint32_t RMAX = 1u << RB;
  static_assert(RMAX <= (uint32_t)kST, "one thread per digit");
  extern __shared__ __align__(16) unsigned char ssm[];  // scatter_atomic_smem<W, RB>() bytes
  KeyT<W>* ring = reinterpret_cast<KeyT<W>*>(ssm);       // [kSRing][SUB + 2]
  // digit tables in static shared memory (compile-time addresses on the per-key paths)
  __shared__ unsigned long long dl[2 * RMAX];  // [2][RMAX] run starts (round parity)
  __shared__ uint32_t cnt[RMAX];
  __shared__ uint32_t lst[2 * RMAX];           // [2][RMAX] stage starts
  __shared__ __align__(8) uint64_t bar[kSRing];
  const PTile t = tiles[blockIdx.x];
  const uint64_t gbase = t.mbase * R;  // first bucket of the tile's group (R = 2^bits <= RMAX digits)
  const bool tma = use_tma && ((reinterpret_cast<uintptr_t>(in) & 15u) == 0);
  for (uint32_t d = threadIdx.x; d < RMAX; d += kST) cnt[d] = 0;
  const uint32_t nsub = (t.len + SUB - 1) / SUB;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSRing; i++) mbar_init(&bar[i], 1);
    mbar_init_fence();
  }
  __syncthreads();
  auto sub_len = [&](uint32_t r) { return min((uint32_t)SUB, t.len - r * SUB); };
  auto issue = [&](uint32_t r) {
    const uint32_t sl = r % kSRing;
    fence_proxy_async_smem();
    issue_core<W>(in, t.start + (uint64_t)r * SUB, sub_len(r), ring + sl * (SUB + 2), &bar[sl]);
  };
  auto resolve = [&](uint32_t d, uint32_t cd, unsigned long long b) -> unsigned long long {
    if (!cd) return ~0ull;
    if (b + cd <= cap2) return (gbase + d) * cap2 + b;
    *ovf = 1;
    return ~0ull;
  };
  auto store_round = [&](uint32_t r) {
    const uint32_t q = r & 1, m = sub_len(r);
    const KeyT<W>* stage = ring + (r % kSRing) * (SUB + 2);
    uint64_t* const outb = out - (size_t)SUB * W;  // dl holds run start - stage start + SUB
    for (uint32_t j = threadIdx.x; j < m; j += kST) {
      const KeyT<W> x = stage[j];
      const uint32_t d = top_bits_nz<W>(x, bsel) & (R - 1);
      const unsigned long long bd = dl[q * RMAX + d];
      if (bd != ~0ull) store_key<W>(outb, bd + j, x);
    }
  };
  if (tma && threadIdx.x == 0)
    for (uint32_t r = 0; r < min(nsub, (uint32_t)kSRing - 1); r++) issue(r);
  uint32_t phase = 0;
  // pipelined reservation, as in scatter1_kernel: round r's atomics are
  // consumed in round r + 1, round r - 1 is stored while round r is staged
  unsigned long long bres = 0;
  uint32_t pcd = 0;
  for (uint32_t r = 0; r < nsub; r++) {
    const uint32_t sl = r % kSRing, r0 = r * SUB, q = r & 1;
    const uint32_t m = sub_len(r);
    KeyT<W>* buf = ring + sl * (SUB + 2);
    if (tma) {
      const uint64_t s0 = t.start + r0;
      const bool issued = W == 1 ? (((s0 + m) & ~1ull) > ((s0 + 1) & ~1ull)) : m > 0;
      if (issued) {
        mbar_wait(&bar[sl], (phase >> sl) & 1u);
        phase ^= 1u << sl;
      }
    }
    KeyT<W> k[ITEMS];
    uint32_t dr[ITEMS];
    const uint32_t c0 = (W == 1 && tma) ? (uint32_t)((t.start + r0) & 1u) : 0u;
    const uint32_t c1 = !tma ? 0u : (W == 1 ? m - (uint32_t)((t.start + r0 + m) & 1u) : m);
    if (m == (uint32_t)SUB && c0 == 0 && c1 == (uint32_t)SUB) {  // full sub-round in the ring: no guards
#pragma unroll
      for (int u = 0; u < ITEMS; u++) {
        k[u] = buf[u * kST + threadIdx.x];
        const uint32_t d = top_bits_nz<W>(k[u], bsel) & (R - 1);
        dr[u] = (d << 16) | atomicAdd(&cnt[d], 1u);
      }
    } else {
#pragma unroll
      for (int u = 0; u < ITEMS; u++) {
        const uint32_t i = u * kST + threadIdx.x;
        if (i < m) {
          k[u] = (i >= c0 && i < c1) ? buf[i + c0] : load_key<W>(in, t.start + r0 + i);
          const uint32_t d = top_bits_nz<W>(k[u], bsel) & (R - 1);
          dr[u] = (d << 16) | atomicAdd(&cnt[d], 1u);
        }
      }
    }
    __syncthreads();  // counts final; the slot's keys are in registers: it becomes the stage
    if (threadIdx.x < 32) {  // warp 0: exclusive scan of the digit counts
      constexpr uint32_t DPL = RMAX / 32;
      uint32_t c[DPL], loc = 0;
#pragma unroll
      for (uint32_t j = 0; j < DPL; j++) {
        c[j] = cnt[threadIdx.x * DPL + j];
        loc += c[j];
      }
      uint32_t inc = loc;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if ((int)threadIdx.x >= o) inc += y;
      }
      uint32_t ex = inc - loc;
#pragma unroll
      for (uint32_t j = 0; j < DPL; j++) {
        lst[q * RMAX + threadIdx.x * DPL + j] = ex;
        ex += c[j];
      }
    }
    if (threadIdx.x < RMAX) {  // publish the previous round's runs, reserve this round's
      const uint32_t d = threadIdx.x;
      if (r > 0) dl[(q ^ 1) * RMAX + d] = stage_delta<W>(resolve(d, pcd, bres), lst[(q ^ 1) * RMAX + d]);
      pcd = cnt[d];
      bres = pcd ? atomicAdd(&gcur[gbase + d], (unsigned long long)pcd) : 0ull;
    }
    __syncthreads();
    KeyT<W>* stage = buf;
    if (m == (uint32_t)SUB) {
#pragma unroll
      for (int u = 0; u < ITEMS; u++) stage[lst[q * RMAX + (dr[u] >> 16)] + (dr[u] & 0xffffu)] = k[u];
    } else {
#pragma unroll
      for (int u = 0; u < ITEMS; u++) {
        const uint32_t i = u * kST + threadIdx.x;
        if (i < m) stage[lst[q * RMAX + (dr[u] >> 16)] + (dr[u] & 0xffffu)] = k[u];
      }
    }
    if (r > 0) store_round(r - 1);
    for (uint32_t d = threadIdx.x; d < RMAX; d += kST) cnt[d] = 0;
    __syncthreads();
    if (tma && threadIdx.x == 0 && r + kSRing - 1 < nsub) issue(r + kSRing - 1);  // into round r-1's slot
  }
  if (nsub > 0) {
    const uint32_t q = (nsub - 1) & 1;
    if (threadIdx.x < RMAX) dl[q * RMAX + threadIdx.x] = stage_delta<W>(resolve(threadIdx.x, pcd, bres), lst[q * RMAX + threadIdx.x]);
    __syncthreads();
    store_round(nsub - 1);
  }
}

// ---------------------------------------------------------------- hist-free first pass
// The first pass of a large call skips the histogram read: pi is uniform, so
// each of the 256 top-byte groups gets a region of `cap` >= n/256 (+2% + 4 Ki)
// keys and CTAs reserve their runs in it with one global atomic per (sub-round,
// digit).  Persistent CTAs walk interleaved 4 Ki-key sub-rounds through the
// same 3-slot TMA ring as tile_scatter_kernel, and keep the HyperLogLog sketch.
// A region that would overflow (a pathologically skewed input) sets *ovf and
// writes nothing past its end; the host then redoes the pass with histograms.
// The next pass reads the groups from their regions and writes compactly.
template <int W>
__global__ void __launch_bounds__(kST, 2) scatter1_kernel(const uint64_t* __restrict__ in, uint64_t n, int use_tma,
                                                         uint64_t cap, unsigned long long* __restrict__ gcur,
                                                         uint64_t* __restrict__ out, uint32_t* __restrict__ hll,
                                                         int* __restrict__ ovf) {
  constexpr int ITEMS = SSCfg<W>::SUB / kST;
  constexpr int SUB = SSCfg<W>::SUB;
  constexpr uint32_t RMAX = 256;
  extern __shared__ __align__(16) unsigned char ssm[];  // scatter1_smem<W>() bytes
  KeyT<W>* ring = reinterpret_cast<KeyT<W>*>(ssm);       // [kSRing][SUB + 2]
  // digit tables and HLL registers in static shared memory (compile-time addresses)
  __shared__ unsigned long long dl[2 * RMAX];           // [2][256]
  __shared__ uint32_t cnt[RMAX];
  __shared__ uint32_t lst[2 * RMAX];                    // [2][256]
  __shared__ __align__(4) uint8_t reg[kHllM];           // HLL registers, one byte each
  __shared__ __align__(8) uint64_t bar[kSRing];
  const bool tma = use_tma && ((reinterpret_cast<uintptr_t>(in) & 15u) == 0);
  const uint64_t nsub = (n + SUB - 1) / SUB;
  for (uint32_t d = threadIdx.x; d < RMAX; d += kST) cnt[d] = 0;
  for (uint32_t i = threadIdx.x; i < kHllM / 4; i += kST) reinterpret_cast<uint32_t*>(reg)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSRing; i++) mbar_init(&bar[i], 1);
    mbar_init_fence();
  }
  __syncthreads();
  // this CTA's k-th sub-round is blockIdx.x + k * gridDim.x
  auto sub_of = [&](uint64_t k) { return (uint64_t)blockIdx.x + k * gridDim.x; };
  auto sub_len = [&](uint64_t k) { return (uint32_t)min((uint64_t)SUB, n - sub_of(k) * SUB); };
  auto issue = [&](uint64_t k) {  // thread 0: local sub-round k -> slot k % kSRing
    const uint32_t sl = (uint32_t)(k % kSRing);
    fence_proxy_async_smem();
    issue_core<W>(in, sub_of(k) * SUB, sub_len(k), ring + sl * (SUB + 2), &bar[sl]);
  };
  // the run reservation of digit d (thread d) for the round whose atomic returned b
  auto resolve = [&](uint32_t d, uint32_t cd, unsigned long long b) -> unsigned long long {
    if (!cd) return ~0ull;  // no write
    if (b + cd <= cap) return (unsigned long long)d * cap + b;
    *ovf = 1;
    return ~0ull;
  };
  // stores of local round k (staged, digit-ordered, in its slot)
  auto store_round = [&](uint64_t k) {
    const uint32_t q = (uint32_t)(k & 1);
    const uint32_t m = sub_len(k);
    const KeyT<W>* stage = ring + (uint32_t)(k % kSRing) * (SUB + 2);
    uint64_t* const outb = out - (size_t)SUB * W;  // dl holds run start - stage start + SUB
    for (uint32_t j = threadIdx.x; j < m; j += kST) {
      const KeyT<W> x = stage[j];
      const uint32_t d = (uint32_t)(x.w0 >> 56);
      const unsigned long long bd = dl[q * RMAX + d];
      if (bd != ~0ull) store_key<W>(outb, bd + j, x);
    }
  };
  uint64_t nk = 0;  // local sub-rounds
  if (blockIdx.x < nsub) nk = (nsub - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (tma && threadIdx.x == 0)
    for (uint64_t k = 0; k < min(nk, (uint64_t)kSRing - 1); k++) issue(k);
  uint32_t phase = 0;
  // Pipelined reservation: round kk's global atomics are issued after its
  // ranking and consumed one round later, so their L2 latency overlaps the
  // next round's TMA wait + ranking; round kk-1 is stored from its slot while
  // round kk is staged into its own.
  unsigned long long bres = 0;  // thread d < 256: the previous round's atomic result
  uint32_t pcd = 0;             // ... and its count
  for (uint64_t kk = 0; kk < nk; kk++) {
    const uint64_t s0 = sub_of(kk) * SUB;
    const uint32_t sl = (uint32_t)(kk % kSRing), q = (uint32_t)(kk & 1);
    const uint32_t m = sub_len(kk);
    KeyT<W>* buf = ring + sl * (SUB + 2);
    if (tma) {
      const bool issued = W == 1 ? (((s0 + m) & ~1ull) > ((s0 + 1) & ~1ull)) : m > 0;
      if (issued) {
        mbar_wait(&bar[sl], (phase >> sl) & 1u);
        phase ^= 1u << sl;
      }
    }
    KeyT<W> k[ITEMS];
    uint32_t dr[ITEMS];
    const uint32_t c0 = (W == 1 && tma) ? (uint32_t)(s0 & 1u) : 0u;
    const uint32_t c1 = !tma ? 0u : (W == 1 ? m - (uint32_t)((s0 + m) & 1u) : m);
    auto rank_key = [&](int u, const KeyT<W>& key) {
      k[u] = to_pi(key);
      const uint32_t d = (uint32_t)(k[u].w0 >> 56);
      dr[u] = (d << 16) | atomicAdd(&cnt[d], 1u);
      const uint64_t hv = k[u].w0;  // hash-sampled HLL (see tile_hist_kernel)
      if (((hv >> kHllLog) & (kHllSample - 1)) == 0) {
        const uint32_t idx = (uint32_t)hv & (kHllM - 1);
        const uint32_t rho = (uint32_t)min(__clzll(hv), 64 - kHllLog - 4) + 1;
        if (rho > reg[idx]) {  // rare: byte max by a CAS on the containing word
          uint32_t* wp = reinterpret_cast<uint32_t*>(reg) + (idx >> 2);
          const uint32_t sh = (idx & 3u) * 8u;
          uint32_t old = *wp;
          while (((old >> sh) & 0xffu) < rho) {
            const uint32_t nw = (old & ~(0xffu << sh)) | (rho << sh);
            const uint32_t got = atomicCAS(wp, old, nw);
            if (got == old) break;
            old = got;
          }
        }
      }
    };
    if (m == (uint32_t)SUB && c0 == 0 && c1 == (uint32_t)SUB) {  // full sub-round in the ring: no guards
#pragma unroll
      for (int u = 0; u < ITEMS; u++) rank_key(u, buf[u * kST + threadIdx.x]);
    } else {
#pragma unroll
      for (int u = 0; u < ITEMS; u++) {
        const uint32_t i = u * kST + threadIdx.x;
        if (i < m) rank_key(u, (i >= c0 && i < c1) ? buf[i + c0] : load_key<W>(in, s0 + i));
      }
    }
    __syncthreads();  // counts final; the slot's keys are in registers: it becomes the stage
    if (threadIdx.x < 32) {  // warp 0: exclusive scan of the 256 digit counts
      constexpr uint32_t DPL = RMAX / 32;
      uint32_t c[DPL], loc = 0;
#pragma unroll
      for (uint32_t j = 0; j < DPL; j++) {
        c[j] = cnt[threadIdx.x * DPL + j];
        loc += c[j];
      }
      uint32_t inc = loc;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if ((int)threadIdx.x >= o) inc += y;
      }
      uint32_t ex = inc - loc;
#pragma unroll
      for (uint32_t j = 0; j < DPL; j++) {
        lst[q * RMAX + threadIdx.x * DPL + j] = ex;
        ex += c[j];
      }
    }
    if (threadIdx.x < RMAX) {  // publish the previous round's runs, reserve this round's
      const uint32_t d = threadIdx.x;
      if (kk > 0) dl[(q ^ 1) * RMAX + d] = stage_delta<W>(resolve(d, pcd, bres), lst[(q ^ 1) * RMAX + d]);
      pcd = cnt[d];
      bres = pcd ? atomicAdd(&gcur[d], (unsigned long long)pcd) : 0ull;
    }
    __syncthreads();  // lst[q], dl[q ^ 1] ready; cnt read out
    KeyT<W>* stage = buf;
    if (m == (uint32_t)SUB) {
#pragma unroll
      for (int u = 0; u < ITEMS; u++) stage[lst[q * RMAX + (dr[u] >> 16)] + (dr[u] & 0xffffu)] = k[u];
    } else {
#pragma unroll
      for (int u = 0; u < ITEMS; u++) {
        const uint32_t i = u * kST + threadIdx.x;
        if (i < m) stage[lst[q * RMAX + (dr[u] >> 16)] + (dr[u] & 0xffffu)] = k[u];
      }
    }
    if (kk > 0) store_round(kk - 1);
    for (uint32_t d = threadIdx.x; d < RMAX; d += kST) cnt[d] = 0;
    __syncthreads();  // round kk-1's slot read out, round kk staged, counters clear
    if (tma && threadIdx.x == 0 && kk + kSRing - 1 < nk) issue(kk + kSRing - 1);  // into round kk-1's slot
  }
  if (nk > 0) {
    const uint32_t q = (uint32_t)((nk - 1) & 1);
    if (threadIdx.x < RMAX) dl[q * RMAX + threadIdx.x] = stage_delta<W>(resolve(threadIdx.x, pcd, bres), lst[q * RMAX + threadIdx.x]);
    __syncthreads();
    store_round(nk - 1);
  }
  for (uint32_t i = threadIdx.x; i < kHllM; i += kST)
    if (reg[i]) atomicMax(&hll[i], reg[i]);
}
template <int W> constexpr size_t scatter1_smem() {
  return kSRing * ((size_t)SSCfg<W>::SUB + 2) * sizeof(KeyT<W>);  // the ring (tables: static)
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

// ---------------------------------------------------------------- per-bucket dedup (ordered table)
// One CTA per SM (the table takes the shared memory) takes (sub-)buckets in
// order from a ticket counter.  A (sub-)bucket is a contiguous run of pi-values whose top
// S = B + V bits of hi are fixed, so a table slot stores the remaining bits
// exactly as T = (hi << S) | 1 (never 0: 0 marks an empty slot, and a zero
// pi-value needs no special case), next to lo at W = 2.  The keys go into an
// ORDER-PRESERVING open-addressing table of 2^logts home slots: home = the
// top logts bits of T, linear probing forward with no wrap (an overflow tail
// of OV slots).  Since home is monotone in T, every cluster of occupied slots
// holds exactly the keys whose homes fall inside it, and clusters are ordered
// among themselves.
//
// Insertion: each round a thread loads ILP keys straight from global memory
// (coalesced, all in flight together; the first 128 KiB of the NEXT unit are
// bulk-prefetched into L2 when a unit starts) and takes them through the FAST
// path: one shared CAS of the home slot (64-bit at W = 1, 128-bit at W = 2)
// -- it returns empty: inserted, equal: duplicate, anything else: a miss.
// Keys that miss are appended BY VALUE to a per-warp queue (ballot
// compaction); whenever 32 are queued the warp drains them with every lane
// probing, so the divergent probe loop runs on full warps.
// Output: occupancy words by warp ballots over 32-slot windows, one block scan
// of the window counts, the list of occupied slots (in the queue's space),
// then -- 32 consecutive survivors per warp step, every lane busy -- each
// survivor's rank = (occupied slots before its cluster) + (keys of its
// cluster with a smaller T): the table is never sorted in place (no serial
// insertion sort on the critical path); survivors are written as keys (exact
// inverse mix) at the bucket offset + rank.
#ifndef CUSCI_BU_THREADS  // (tuning macros: A/B variants, tools/build_variant.py)
#define CUSCI_BU_THREADS 1024
#define CUSCI_BU_LOGTS1 14
#define CUSCI_BU_OV1 1024
#define CUSCI_BU_DT1 6144
#endif
#ifndef CUSCI_BU_ILP1
#define CUSCI_BU_ILP1 4
#endif
#ifndef CUSCI_BU_DB
#define CUSCI_BU_DB 1  // double-buffered insert rounds (10.03 -> 9.79 ms per N2 batch)
#endif
#ifndef CUSCI_BU_PF
#define CUSCI_BU_PF 131072  // bytes of the next unit's input prefetched into L2 (0: off; 64 / 128 / 192 / 256 KiB: 10.24 / 10.04 / 10.06 / 10.63 ms vs 10.27 ms per N2 batch)
#endif
#ifndef CUSCI_BU_PROBE2
#define CUSCI_BU_PROBE2 0  // the fast path also probes home + 1 before queueing a key
#endif
#ifndef CUSCI_BU_CASFIRST
#define CUSCI_BU_CASFIRST 1  // W = 1: probe with the CAS itself (no load first: 11.66 -> 10.56 ms per N2 batch)
#endif
constexpr int kBU = CUSCI_BU_THREADS;  // dedup threads (the table fills the shared memory: 1024 -> one CTA per SM)
template <int W> struct BUCfg {
  static constexpr int ILP = W == 1 ? CUSCI_BU_ILP1 : 2;  // keys per thread per round
  static constexpr int LOGTS = W == 1 ? CUSCI_BU_LOGTS1 : CUSCI_BU_LOGTS1 - 1;  // max home slots 2^LOGTS
  static constexpr uint32_t TS = 1u << LOGTS;
  static constexpr uint32_t OV = W == 1 ? CUSCI_BU_OV1 : CUSCI_BU_OV1 / 2;  // overflow tail
  static constexpr uint32_t NWIN = (TS + OV) / 32;        // 32-slot windows
  static constexpr uint32_t QCAP = 32u * (ILP < 4 ? ILP : 4) + 32u;  // per-warp slow-path queue (keys; drained mid-round when ILP > 4)
  static constexpr uint32_t DT = W == 1 ? CUSCI_BU_DT1 : CUSCI_BU_DT1 / 2;  // plan: target distinct keys per bucket
  static constexpr size_t QBYTES = (size_t)(kBU / 32) * QCAP * sizeof(KeyT<W>);
  static constexpr size_t SMEM = (size_t)(TS + OV) * sizeof(KeyT<W>) + QBYTES + 2 * (size_t)NWIN * sizeof(uint32_t) +
                                 (size_t)(TS + OV) * sizeof(uint16_t);
  static_assert(NWIN <= kBU, "one window count per thread in the block scan");
  static_assert(QBYTES >= (TS + OV) * sizeof(uint16_t), "the occupied-slot list reuses the queue space");
  static_assert(SMEM <= 227 * 1024 - 1024, "shared memory budget");
};

// table entry: T = (hi << S) | 1 (w0), lo (w1, W = 2)
__device__ __forceinline__ KeyT<1> tenc(const KeyT<1>& p, int S) { return KeyT<1>{(p.w0 << S) | 1ull}; }
__device__ __forceinline__ KeyT<2> tenc(const KeyT<2>& p, int S) { return KeyT<2>{(p.w0 << S) | 1ull, p.w1}; }
__device__ __forceinline__ KeyT<1> tdec(const KeyT<1>& t, int S, uint64_t top) { return KeyT<1>{(t.w0 >> S) | top}; }
__device__ __forceinline__ KeyT<2> tdec(const KeyT<2>& t, int S, uint64_t top) { return KeyT<2>{(t.w0 >> S) | top, t.w1}; }
__device__ __forceinline__ bool tzero(const KeyT<1>& t) { return t.w0 == 0; }
__device__ __forceinline__ bool tzero(const KeyT<2>& t) { return t.w0 == 0; }
__device__ __forceinline__ bool tlt(const KeyT<1>& a, const KeyT<1>& b) { return a.w0 < b.w0; }
__device__ __forceinline__ bool tlt(const KeyT<2>& a, const KeyT<2>& b) {
  return a.w0 < b.w0 || (a.w0 == b.w0 && a.w1 < b.w1);
}
__device__ __forceinline__ uint32_t thome(const KeyT<1>& t, int logts) { return (uint32_t)(t.w0 >> (64 - logts)); }
__device__ __forceinline__ uint32_t thome(const KeyT<2>& t, int logts) { return (uint32_t)(t.w0 >> (64 - logts)); }

// one probe step at slot s: true when p is now in the table (found or inserted)
template <int W>
__device__ __forceinline__ bool tprobe(KeyT<W>* tab, uint32_t s, const KeyT<W>& p) {
  KeyT<W> old;
  if (W == 1 && !CUSCI_BU_CASFIRST) {
    const KeyT<W> c = tab[s];
    if (key_eq(c, p)) return true;
    if (!tzero(c)) return false;
  }
  cas_slot(&tab[s], p, old);  // W = 2: the 128-bit CAS is the probe (never a torn read)
  return tzero(old) || key_eq(old, p);
}

// Output offsets without a pack pass: units (sub-buckets) are taken in order
// from a ticket counter, and each publishes its survivor count as soon as its
// table is complete; warp 0 then resolves the unit's output offset by a
// decoupled look-back over the predecessors' status words (aggregate, or
// inclusive prefix) while the other warps rank their survivors.  Every
// predecessor of a unit holds its ticket already and publishes its count
// before it looks back itself, so the wait cannot deadlock, resident or not.
constexpr unsigned long long kBFlagA = 1ull << 62, kBFlagP = 2ull << 62, kBVal = (1ull << 62) - 1;
__device__ __forceinline__ uint64_t bucket_lookback(volatile unsigned long long* st, uint32_t u) {
  const unsigned lane = lane_id();
  uint64_t ex = 0;
  for (int64_t q0 = (int64_t)u - 1; q0 >= 0; q0 -= 32) {
    const int64_t q = q0 - (int64_t)lane;
    unsigned long long v = kBFlagP;  // before unit 0: an inclusive prefix of 0
    if (q >= 0) v = st[q];
    while (__any_sync(kFull, (v >> 62) == 0))
      if ((v >> 62) == 0) v = st[q];
    const unsigned bp = __ballot_sync(kFull, (v >> 62) == 2);
    const unsigned L = bp ? (unsigned)(__ffs(bp) - 1) : 32u;  // nearest inclusive prefix
    uint64_t sum = lane <= L ? (v & kBVal) : 0ull;
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
    ex += sum;
    if (bp) break;
  }
  return ex;
}

// GEN: raw (caller) input or split buckets (V = 1); the common case compiles without them
template <int W, bool GEN>
__global__ void __launch_bounds__(kBU, 1024 / kBU) bucket_unique_kernel(const uint64_t* __restrict__ part, int raw,
                                                              const uint32_t* __restrict__ off,
                                                              const uint64_t* __restrict__ ibase, uint32_t nb, int B,
                                                              int V, uint32_t lf, uint32_t dmean,
                                                              uint64_t* __restrict__ out,
                                                              unsigned long long* __restrict__ lbst,
                                                              unsigned int* __restrict__ ticket,
                                                              unsigned long long* __restrict__ flags,
                                                              const uint32_t* __restrict__ lb,
                                                              const uint64_t* __restrict__ rs, int nruns,
                                                              uint64_t ubase) {
  // nruns > 0 (GEN only): the input is nruns pi-sorted runs back to back (run
  // r starts at rs[r]); bucket b's keys are the segments [lb[r][b],
  // lb[r][b+1]) of every run (the owner-side finalize of dedup_global: no
  // partition pass over the received keys).  ubase: global id of unit 0 (the
  // units cover only the input's hash range; bucket id = (ubase + b) >> V)
  using K = KeyT<W>;
  using C = BUCfg<W>;
  constexpr uint32_t TS = C::TS, OV = C::OV, QCAP = C::QCAP, NWIN = C::NWIN;
  constexpr int ILP = C::ILP, NW = kBU / 32;
  extern __shared__ __align__(16) unsigned char bsm[];
  K* tab = reinterpret_cast<K*>(bsm);
  K* qall = tab + TS + OV;                                        // [NW][QCAP]
  uint32_t* bm = reinterpret_cast<uint32_t*>(qall + NW * QCAP);   // [NWIN] occupancy words
  uint32_t* wbase = bm + NWIN;                                    // [NWIN] occupied slots before the window
  uint16_t* pos = reinterpret_cast<uint16_t*>(wbase + NWIN);      // [TS + OV] survivor rank in the unit
  __shared__ int s_full;
  __shared__ uint32_t s_unit, s_next;
  __shared__ unsigned long long s_ex;
  __shared__ uint32_t red[33];
  __shared__ uint64_t sg_st[GEN ? CUSCI_MAX_WORLD : 1];       // segment starts of the current bucket
  __shared__ uint32_t sg_pre[GEN ? CUSCI_MAX_WORLD + 1 : 1];  // bucket-local start of each segment
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, t = threadIdx.x;
  K* q = qall + warp * QCAP;
  const int S = B + V;
  const bool segs = GEN && nruns > 0;
  const uint32_t nsb = nb << V;
  volatile unsigned long long* vst = lbst;
  // L2 prefetch of the head of a unit's input (CUSCI_BU_PF bytes; 0 = off):
  // the next unit's ticket is taken when a unit starts, so its first loads
  // find L2 lines.  A unit held as "next" follows a smaller unit of the same
  // CTA, so the smallest unpublished unit is always being processed: the
  // look-back still cannot deadlock.
  auto l2_prefetch = [&](uint32_t u) {
#if CUSCI_BU_PF
    if (segs || u >= nsb) return;
    const uint32_t s0 = off[u >> V], n0 = off[(u >> V) + 1] - s0;
    const uint64_t i0 = ibase ? ibase[u >> V] : (uint64_t)s0;
    const uint64_t a0 = reinterpret_cast<uint64_t>(part + i0 * W) & ~15ull;
    uint64_t a1 = (reinterpret_cast<uint64_t>(part + (i0 + n0) * W) + 15ull) & ~15ull;
    if (a1 > a0 + CUSCI_BU_PF) a1 = a0 + CUSCI_BU_PF;
    if (a1 > a0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
#else
    (void)u;
#endif
  };
  // the table is cleared once here and after every bucket's output
  for (uint32_t i = t; i < TS + OV; i += kBU) tab[i] = K{};
  if (t == 0) {
    s_full = 0;
    s_unit = atomicAdd(ticket, 1u);
  }
  __syncthreads();
  for (;;) {
    const uint32_t b = s_unit;
    if (b >= nsb) break;
    if (CUSCI_BU_PF && t == 0) {
      s_next = atomicAdd(ticket, 1u);
      l2_prefetch(s_next);
    }
    const uint32_t s = off[b >> V], nk = off[(b >> V) + 1] - s;
    const uint64_t si = ibase ? ibase[b >> V] : (uint64_t)s;       // input offset
    const uint64_t vpart = (uint64_t)(b & ((1u << V) - 1u));
    if (segs && nk) {  // this bucket's segments (the previous bucket ended with a barrier)
      const uint32_t bb = b >> V, nbk1 = nb + 1;
      if (t < (uint32_t)nruns) sg_st[t] = rs[t] + lb[(size_t)t * nbk1 + bb];
      if (t == 0) {
        uint32_t a = 0;
        for (int r = 0; r < nruns; r++) {
          sg_pre[r] = a;
          a += lb[(size_t)r * nbk1 + bb + 1] - lb[(size_t)r * nbk1 + bb];
        }
        sg_pre[nruns] = a;
      }
      __syncthreads();
    }
    // global index of the bucket's i-th input key
    auto kaddr = [&](uint32_t i) -> uint64_t {
      if (!segs) return si + i;
      int lo = 0, hi = nruns - 1;  // last segment with sg_pre[r] <= i
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sg_pre[mid] <= i) lo = mid;
        else hi = mid - 1;
      }
      return sg_st[lo] + (i - sg_pre[lo]);
    };
    // publish this unit's count (inclusive at unit 0) and resolve its output
    // offset: warp 0 looks back, the caller's other warps keep working
    auto publish = [&](uint32_t cnt) {
      if (t == 0) vst[b] = (b == 0 ? kBFlagP : kBFlagA) | (unsigned long long)cnt;
    };
    auto resolve = [&](uint32_t cnt) {
      if (warp == 0) {
        const uint64_t ex = b == 0 ? 0ull : bucket_lookback(vst, b);
        if (t == 0) {
          if (b) vst[b] = kBFlagP | (unsigned long long)(ex + cnt);
          s_ex = ex;
        }
      }
    };
    // 2^logts home slots ~ lf x the expected distinct keys (<= nk), capped
    const uint32_t want = lf * min(nk, dmean);
    const int logts = want <= 32u ? 5 : min(C::LOGTS, 32 - __clz(want - 1u));
    const uint32_t span = (1u << logts) + OV;
    bool full = false;
    uint32_t qn = 0;  // warp-uniform queue fill
    // drain queue entries [qn - 32, qn) (or all, at the end) with every lane probing
    auto drain = [&](uint32_t cnt) {
      const uint32_t q0 = qn - cnt;
      if (lane < cnt) {
        const K p = q[q0 + lane];
        uint32_t sidx = thome(p, logts) + 1 + CUSCI_BU_PROBE2;  // the first probed slot(s) hold other keys
        for (;;) {
          if (sidx >= span) {
            full = true;
            break;
          }
          if (tprobe<W>(tab, sidx, p)) break;
          sidx++;
        }
      }
      qn = q0;
      __syncwarp();
    };
#if CUSCI_BU_DB
    // double-buffered rounds: the next round's keys are loaded before this
    // round's probes, so their latency overlaps the probing
    K nx[ILP];
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      const uint32_t i = u * kBU + t;
      if (i < nk) nx[u] = load_key<W>(part, kaddr(i));
    }
#endif
    for (uint32_t r0 = 0; r0 < nk; r0 += ILP * kBU) {
      K pv[ILP];
      bool act[ILP];
#if CUSCI_BU_DB
#pragma unroll
      for (int u = 0; u < ILP; u++) {
        act[u] = r0 + u * kBU + t < nk;
        pv[u] = nx[u];
        const uint32_t i = r0 + ILP * kBU + u * kBU + t;
        if (i < nk) nx[u] = load_key<W>(part, kaddr(i));
      }
#else
#pragma unroll
      for (int u = 0; u < ILP; u++) {
        const uint32_t i = r0 + u * kBU + t;
        act[u] = i < nk;
        if (act[u]) pv[u] = load_key<W>(part, kaddr(i));
      }
#endif
#pragma unroll
      for (int u = 0; u < ILP; u++) {
        bool slow = false;
        if (act[u]) {
          K p = pv[u];
          if (GEN && raw) p = to_pi(p);
          if (!GEN || !V || ((p.w0 << B) >> (64 - V)) == vpart) {  // (V: the other sub-bucket is skipped)
            p = tenc(p, S);
            pv[u] = p;
            const uint32_t h = thome(p, logts);
            slow = !tprobe<W>(tab, h, p);
            if (CUSCI_BU_PROBE2 && slow) slow = !tprobe<W>(tab, h + 1, p);  // (h + 1 < TS + OV: no bound check)
          }
        }
        const unsigned sb = __ballot_sync(kFull, slow);
        if (slow) q[qn + __popc(sb & lanemask_lt())] = pv[u];
        qn += __popc(sb);
        if (ILP > 4 && qn > QCAP - 32) {  // (warp-uniform) room for the next append
          __syncwarp();
          drain(32);
        }
      }
      __syncwarp();
      while (qn >= 32) drain(32);
    }
    if (qn) drain(qn);
    if (full) s_full = 1;
    __syncthreads();  // table complete
    const uint64_t top = (ubase + b) << (64 - S);  // the sub-bucket's fixed top S bits of hi
    if (s_full) {
      // table overflow (pathological bucket): pass this (sub-)bucket's keys
      // through unfiltered (the host finishes with a full sort + unique) and
      // restore a clean table
      auto mine = [&](const K& kk) { return !V || (((raw ? to_pi(kk) : kk).w0 << B) >> (64 - V)) == vpart; };
      if (t == 0) red[0] = 0;
      __syncthreads();
      uint32_t cnt = 0;
      for (uint32_t i = t; i < nk; i += kBU) cnt += mine(load_key<W>(part, kaddr(i)));
      atomicAdd(&red[0], cnt);
      __syncthreads();
      const uint32_t nh = red[0];
      publish(nh);
      resolve(nh);
      __syncthreads();
      if (t == 0) red[0] = 0;
      __syncthreads();
      const uint64_t ob = s_ex;
      for (uint32_t i = t; i < nk; i += kBU) {
        const K p = load_key<W>(part, kaddr(i));
        if (mine(p)) store_key<W>(out, ob + atomicAdd(&red[0], 1u), raw ? p : from_pi(p));
      }
      for (uint32_t i = t; i < span; i += kBU) tab[i] = K{};
      if (t == 0) {
        atomicAdd(&flags[0], 1ull);
        s_full = 0;
      }
      __syncthreads();
      if (t == 0) s_unit = CUSCI_BU_PF ? s_next : atomicAdd(ticket, 1u);
      __syncthreads();
      continue;
    }
    const uint32_t nwin = span / 32;
    // occupancy words: one warp ballot per 32-slot window
    for (uint32_t w = warp; w < nwin; w += NW) {
      const unsigned o = __ballot_sync(kFull, !tzero(tab[w * 32 + lane]));
      if (lane == 0) bm[w] = o;
    }
    __syncthreads();
    uint32_t tot = 0;
    const uint32_t wex = block_excl_scan_u32(t < nwin ? __popc(bm[t]) : 0u, red, tot);
    publish(tot);
    if (t < nwin) wbase[t] = wex;
    __syncthreads();
    // the occupied slots in order (the queue space is free now)
    uint16_t* sidx = reinterpret_cast<uint16_t*>(qall);
    for (uint32_t w = warp; w < nwin; w += NW) {
      const uint32_t o = bm[w];
      if ((o >> lane) & 1u) sidx[wbase[w] + __popc(o & lanemask_lt())] = (uint16_t)(w * 32 + lane);
    }
    __syncthreads();    resolve(tot);  // warp 0: the look-back first, then its share of the ranks
    // survivor k (rank k among the occupied slots) sits in the cluster [cs, ce);
    // its rank in the unit = k - (slot - cs) + (keys of the cluster smaller than it)
    for (uint32_t kk = t; kk < tot; kk += kBU) {
      const uint32_t slot = sidx[kk];
      const K v = tab[slot];
      const uint32_t w = slot >> 5, bit = slot & 31u, word = bm[w];
      uint32_t cs;  // one past the last empty slot below (possibly in earlier windows)
      const uint32_t below = ~word & ((1u << bit) - 1u);
      if (below) {
        cs = w * 32 + (32 - __clz(below));
      } else {
        uint32_t x = w;
        while (x > 0 && bm[x - 1] == 0xffffffffu) x--;
        cs = x > 0 ? (x - 1) * 32 + (32 - __clz(~bm[x - 1])) : 0u;
      }
      uint32_t ce;  // the first empty slot above
      const uint32_t above = bit < 31 ? (~word & (~0u << (bit + 1))) : 0u;
      if (above) {
        ce = w * 32 + __ffs(above) - 1;
      } else {
        uint32_t x = w + 1;
        while (x < nwin && bm[x] == 0xffffffffu) x++;
        ce = x < nwin ? x * 32 + __ffs(~bm[x]) - 1 : nwin * 32;
      }
      uint32_t rank = 0, y = cs;
      for (; y + 1 < ce; y += 2) {  // two independent loads per step
        const K a0 = tab[y], a1 = tab[y + 1];
        rank += (tlt(a0, v) ? 1u : 0u) + (tlt(a1, v) ? 1u : 0u);
      }
      if (y < ce) rank += tlt(tab[y], v) ? 1u : 0u;
      pos[kk] = (uint16_t)(kk - (slot - cs) + rank);
    }
    __syncthreads();  // ranks and the unit's output offset known
    const uint64_t ob = s_ex;
    for (uint32_t kk = t; kk < tot; kk += kBU) {  // each survivor's slot is read once here: clear it as it goes
      const uint32_t slot = sidx[kk];
      store_key<W>(out, ob + pos[kk], from_pi(tdec(tab[slot], S, top)));
      tab[slot] = K{};
    }
    if (t == 0) s_unit = CUSCI_BU_PF ? s_next : atomicAdd(ticket, 1u);
    __syncthreads();  // table clean for the next unit
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

// HyperLogLog estimate of the distinct count from the 2^11 registers
double hll_estimate(const uint32_t* reg) {
  const double m = (double)kHllM;
  double z = 0.0;
  uint32_t zeros = 0;
  for (uint32_t i = 0; i < kHllM; i++) {
    z += std::ldexp(1.0, -(int)reg[i]);
    zeros += reg[i] == 0;
  }
  double e = 0.7213 / (1.0 + 1.079 / m) * m * m / z;
  if (e <= 2.5 * m && zeros) e = m * std::log(m / zeros);  // small-range (linear counting) correction
  return e;
}

template <int W>
int local_dedup_impl(cusci_ctx* ctx, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* n_out) {
  using C = BUCfg<W>;
  *n_out = 0;
  if (n == 0) return CUSCI_OK;
  Scratch s(ctx);
  // tuning knobs (environment, read once)
  static const int use_tma = getenv("CUSCI_NO_TMA") ? 0 : 1;
  static const uint32_t lf = [] {
    const char* e = getenv("CUSCI_TABLE_LF");  // table slots per expected distinct key
    return e ? (uint32_t)std::max(1, atoi(e)) : 3u;
  }();
  static const uint64_t dt = [] {
    const char* e = getenv("CUSCI_BUCKET_DISTINCT");  // target distinct keys per bucket
    return e ? (uint64_t)std::max(64ll, atoll(e)) : (uint64_t)C::DT;
  }();
  static const int max_bits = [] {
    const char* e = getenv("CUSCI_PASS_BITS");  // bits per later partition pass (<= 9)
    return e ? std::max(1, std::min(9, atoi(e))) : 9;
  }();
  // upper bound on the bucket bits (every key distinct)
  int Bmax = 0;
  while ((n >> Bmax) > dt && Bmax < 22) Bmax++;
  int B = Bmax;
  uint32_t dcap = 0xffffffffu;  // expected distinct keys per bucket (+25%; sizes the table)
  const uint32_t nb_max = 1u << Bmax;
  uint64_t *a, *b2;
  uint32_t *off, *hll;
  unsigned long long *flags, *lbst;
  // hist-free first pass (large calls): 256 group regions of `cap` keys in `a`
  static const int hist_free_knob = [] {
    const char* e = getenv("CUSCI_HIST_FREE_PASS1");  // tuning knob (0 disables)
    return e ? atoi(e) : 1;
  }();
  const bool hist_free = hist_free_knob && n >= (1ull << 26) && Bmax > 8;
  const uint64_t cap1 = (n + 255) / 256 + n / 256 / 50 + 4096;
  CUSCI_TRY(s.get_t((std::max<uint64_t>(n, hist_free ? 256 * cap1 : 0) + 2) * W, &a));  // + slack: 16-byte TMA pieces
  CUSCI_TRY(s.get_t((n + 2) * W, &b2));
  CUSCI_TRY(s.get_t(nb_max + 1, &off));
  CUSCI_TRY(s.get_t(2 * (size_t)nb_max + 1, &lbst));   // x2: sub-buckets (V = 1); + the ticket
  CUSCI_TRY(s.get_t(kHllM, &hll));
  CUSCI_TRY(s.get_t(2, &flags));
  CUSCI_CUDA(ctx, cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned long long), ctx->stream));
  int dper = 1, unused = 0;
  CUSCI_TRY(kernel_setup(ctx, (const void*)tile_scatter_kernel<W, true, 8>, kST, scatter_smem<W, 8>(), &unused));
  CUSCI_TRY(kernel_setup(ctx, (const void*)tile_scatter_kernel<W, false, 8>, kST, scatter_smem<W, 8>(), &unused));
  CUSCI_TRY(kernel_setup(ctx, (const void*)tile_scatter_kernel<W, false, 9>, kST, scatter_smem<W, 9>(), &unused));
  CUSCI_TRY(kernel_setup(ctx, (const void*)tile_scatter_atomic_kernel<W, 8>, kST, scatter_atomic_smem<W, 8>(), &unused));
  CUSCI_TRY(kernel_setup(ctx, (const void*)tile_scatter_atomic_kernel<W, 9>, kST, scatter_atomic_smem<W, 9>(), &unused));
  int dper_g = 1;
  CUSCI_TRY(kernel_setup(ctx, (const void*)bucket_unique_kernel<W, false>, kBU, C::SMEM, &dper));
  CUSCI_TRY(kernel_setup(ctx, (const void*)bucket_unique_kernel<W, true>, kBU, C::SMEM, &dper_g));
  const uint64_t* part = in;
  uint64_t* ibase = nullptr;  // bucket input starts when the last pass left bucket regions
  if (Bmax > 0) {
    std::vector<uint32_t> gstart{0u, (uint32_t)n};  // current groups (host): compact prefix ...
    std::vector<uint64_t> rstart, rend;                // ... or, after the hist-free pass, input regions
    uint64_t* dst = a;
    int done = 0;
    // one segmented MSD pass of `bits` bits over the current groups
    static const uint32_t kPTile = [] {
      const char* e = getenv("CUSCI_PART_TILE");  // tuning knob
      return e ? (uint32_t)std::max(4096ll, atoll(e)) : kPTileDefault;
    }();
    auto run_pass = [&](int bits, bool first, bool last) -> int {
      const uint32_t R = 1u << bits;
      const uint32_t G = (uint32_t)gstart.size() - 1;
      std::vector<PTile> tl;
      std::vector<uint4> gm(G);
      tl.reserve(n / kPTile + G + 1);
      uint64_t mb = 0;
      for (uint32_t g = 0; g < G; g++) {
        // input range of the group; gm.x = its compact output start
        const uint64_t gs = rstart.empty() ? gstart[g] : rstart[g], ge = rstart.empty() ? gstart[g + 1] : rend[g];
        const uint32_t chunks = (uint32_t)((ge - gs + kPTile - 1) / kPTile);
        gm[g] = make_uint4(gstart[g], chunks, (uint32_t)mb, 0u);
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
      if (first) {
        CUSCI_CUDA(ctx, cudaMemsetAsync(hll, 0, kHllM * sizeof(uint32_t), ctx->stream));
        static const int hpm = [] {
          const char* e = getenv("CUSCI_HIST_CTAS_PER_SM");  // tuning knob
          return e ? std::max(1, atoi(e)) : 8;
        }();
        const unsigned hg = (unsigned)std::min<uint64_t>(nt, (uint64_t)ctx->num_sms * hpm);
        CUSCI_LAUNCH(ctx, PT_RADIX_UP, tile_hist_kernel<W, true, 8><<<hg, kBT, 0, ctx->stream>>>(part, dtl, nt, sel, R - 1, mat, hll));
      } else {
        CUSCI_LAUNCH(ctx, PT_RADIX_UP, tile_hist_kernel<W, false, 9><<<nt, kBT, 0, ctx->stream>>>(part, dtl, nt, sel, R - 1, mat, hll));
      }
      CUSCI_TRY(scan_exclusive_u32(ctx, mat, offs, mb));
      if (first) {
        CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, tile_scatter_kernel<W, true, 8><<<nt, kST, scatter_smem<W, 8>(), ctx->stream>>>(part, use_tma, dtl, sel, R - 1, offs, dst));
      } else if (bits <= 8) {
        CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, tile_scatter_kernel<W, false, 8><<<nt, kST, scatter_smem<W, 8>(), ctx->stream>>>(part, use_tma, dtl, sel, R - 1, offs, dst));
      } else {
        CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, tile_scatter_kernel<W, false, 9><<<nt, kST, scatter_smem<W, 9>(), ctx->stream>>>(part, use_tma, dtl, sel, R - 1, offs, dst));
      }
      uint32_t* goff_final = last ? off : goff;
      CUSCI_LAUNCH(ctx, PT_SCATTER, group_off_kernel<<<(unsigned)(((uint64_t)G * R + 1 + 255) / 256), 256, 0, ctx->stream>>>(offs, dgm, G, bits, (uint32_t)n, goff_final));
      if (!last) {
        gstart.resize((size_t)G * R + 1);
        CUSCI_CUDA(ctx, cudaMemcpyAsync(gstart.data(), goff, gstart.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                        ctx->stream));
      }
      CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // host tables die at scope end
      part = dst;
      dst = (dst == a) ? b2 : a;
      done += bits;
      ctx->dstats[2] += n;
      ctx->dstats[6] += n;
      rstart.clear();
      rend.clear();
      return CUSCI_OK;
    };
    // the hist-free first pass: scatter into group regions with atomic cursors
    auto run_pass1_regions = [&]() -> int {
      Scratch ps(ctx);
      unsigned long long* gcur;
      int* ovf;
      CUSCI_TRY(ps.get_t(256, &gcur));
      CUSCI_TRY(ps.get_t(1, &ovf));
      CUSCI_CUDA(ctx, cudaMemsetAsync(gcur, 0, 256 * sizeof(unsigned long long), ctx->stream));
      CUSCI_CUDA(ctx, cudaMemsetAsync(ovf, 0, sizeof(int), ctx->stream));
      CUSCI_CUDA(ctx, cudaMemsetAsync(hll, 0, kHllM * sizeof(uint32_t), ctx->stream));
      int sper = 1;
      CUSCI_TRY(kernel_setup(ctx, (const void*)scatter1_kernel<W>, kST, scatter1_smem<W>(), &sper));
      const uint64_t nsub = (n + SSCfg<W>::SUB - 1) / SSCfg<W>::SUB;
      const unsigned g1 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nsub, (uint64_t)ctx->num_sms * sper));
      CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, scatter1_kernel<W><<<g1, kST, scatter1_smem<W>(), ctx->stream>>>(in, n, use_tma, cap1, gcur, a, hll, ovf));
      uint64_t hc[256];
      int hv = 0;
      CUSCI_TRY(read_u64(ctx, reinterpret_cast<const uint64_t*>(gcur), hc, 256));
      CUSCI_CUDA(ctx, cudaMemcpy(&hv, ovf, sizeof(int), cudaMemcpyDeviceToHost));
      if (hv) return -1;  // a region overflowed: redo the pass with histograms
      gstart.assign(257, 0u);
      rstart.resize(256);
      rend.resize(256);
      uint64_t acc = 0;
      for (int g = 0; g < 256; g++) {
        gstart[g] = (uint32_t)acc;
        rstart[g] = (uint64_t)g * cap1;
        rend[g] = rstart[g] + hc[g];
        acc += hc[g];
      }
      gstart[256] = (uint32_t)acc;
      part = a;
      dst = b2;
      done = 8;
      ctx->dstats[2] += n;
      ctx->dstats[7] += n;
      return CUSCI_OK;
    };
    // the last pass, hist-free too: bucket regions of cap2 keys in a fresh buffer
    auto run_pass_last_regions = [&](int bits) -> int {
      const int Btot = done + bits;
      const uint64_t nbk2 = 1ull << Btot;
      const uint64_t mean = n >> Btot;
      // duplicates make bucket sizes spread more than distinct keys (N2 batch, measured:
      // max/mean 1.20 at 16 bits, 1.33 at 17): regions of 1.4 x mean + 2 Ki keys
      const uint64_t cap2 = mean + (mean * 2) / 5 + 2048;
      const uint32_t G = (uint32_t)gstart.size() - 1;
      std::vector<PTile> tl;
      tl.reserve(n / kPTile + G + 1);
      for (uint32_t g = 0; g < G; g++) {
        const uint64_t gs = rstart[g], ge = rend[g];
        for (uint64_t st = gs; st < ge; st += kPTile)
          tl.push_back(PTile{st, (uint32_t)std::min<uint64_t>(kPTile, ge - st), 0u, (uint64_t)g});
      }
      const uint32_t nt = (uint32_t)tl.size();
      uint64_t* r2;
      CUSCI_TRY(s.get_t((nbk2 * cap2 + 2) * W, &r2));  // outer scope: read by the bucket kernel
      CUSCI_TRY(s.get_t(nbk2, &ibase));
      Scratch ps(ctx);
      PTile* dtl;
      unsigned long long* gcur2;
      int* ovf;
      CUSCI_TRY(ps.get_t(std::max<uint32_t>(nt, 1), &dtl));
      CUSCI_TRY(ps.get_t(nbk2, &gcur2));
      CUSCI_TRY(ps.get_t(1, &ovf));
      CUSCI_CUDA(ctx, cudaMemcpyAsync(dtl, tl.data(), nt * sizeof(PTile), cudaMemcpyHostToDevice, ctx->stream));
      CUSCI_CUDA(ctx, cudaMemsetAsync(gcur2, 0, nbk2 * sizeof(unsigned long long), ctx->stream));
      CUSCI_CUDA(ctx, cudaMemsetAsync(ovf, 0, sizeof(int), ctx->stream));
      if (bits <= 8)
        CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, tile_scatter_atomic_kernel<W, 8><<<nt, kST, scatter_atomic_smem<W, 8>(), ctx->stream>>>(part, use_tma, dtl, done + bits, 1u << bits, gcur2, cap2, r2, ovf));
      else
        CUSCI_LAUNCH(ctx, PT_RADIX_DOWN, tile_scatter_atomic_kernel<W, 9><<<nt, kST, scatter_atomic_smem<W, 9>(), ctx->stream>>>(part, use_tma, dtl, done + bits, 1u << bits, gcur2, cap2, r2, ovf));
      std::vector<uint64_t> cnt(nbk2), ib(nbk2);
      std::vector<uint32_t> offh(nbk2 + 1);
      CUSCI_CUDA(ctx, cudaMemcpyAsync(cnt.data(), gcur2, nbk2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
      int hv = 0;
      CUSCI_CUDA(ctx, cudaMemcpyAsync(&hv, ovf, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      if (hv) {
        ibase = nullptr;
        return -1;  // a bucket region overflowed: redo the pass with histograms
      }
      uint64_t acc = 0;
      for (uint64_t b = 0; b < nbk2; b++) {
        offh[b] = (uint32_t)acc;
        ib[b] = b * cap2;
        acc += cnt[b];
      }
      offh[nbk2] = (uint32_t)acc;
      CUSCI_CUDA(ctx, cudaMemcpyAsync(off, offh.data(), (nbk2 + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
      CUSCI_CUDA(ctx, cudaMemcpyAsync(ibase, ib.data(), nbk2 * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
      CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // host vectors die at scope end
      part = r2;
      done += bits;
      ctx->dstats[2] += n;
      rstart.clear();
      rend.clear();
      return CUSCI_OK;
    };
    static const int last_regions_knob = [] {
      const char* e = getenv("CUSCI_HIST_FREE_LAST");  // tuning knob (0 disables)
      return e ? atoi(e) : 1;
    }();
    const int bits1 = std::min(8, Bmax);
    // the plan after pass 1 depends on the sketch, so pass 1 is "last" only if nothing can follow
    bool regions = false;
    if (hist_free) {
      const int rc = run_pass1_regions();
      if (rc == CUSCI_OK) regions = true;
      else if (rc != -1) return rc;
    }
    if (!regions) CUSCI_TRY(run_pass(bits1, true, Bmax == bits1));
    if (Bmax > bits1) {
      std::vector<uint32_t> reg(kHllM);
      CUSCI_CUDA(ctx, cudaMemcpy(reg.data(), hll, kHllM * sizeof(uint32_t), cudaMemcpyDeviceToHost));
      const double D = std::min<double>((double)n, std::max(1.0, kHllSample * hll_estimate(reg.data())));
      int Bd = 0;
      // up to 1.25 x the target per bucket before adding a bit (the sketch's
      // noise must not flip a stream near the boundary into a wider pass)
      while (D / std::ldexp(1.0, Bd) > 1.25 * (double)dt && Bd < 22) Bd++;
      // one bit less when that saves a whole partition pass and the buckets stay
      // within 1.6 x the target (table load <= ~0.6)
      auto npass = [&](int b) { return (std::max(0, b - bits1) + max_bits - 1) / max_bits; };
      if (Bd > bits1 && npass(Bd - 1) < npass(Bd) && D / std::ldexp(1.0, Bd - 1) <= 1.6 * (double)dt) Bd--;
      B = std::max(bits1, std::min(Bmax, Bd));
      if (regions && B == bits1) B = bits1 + 1;  // the region layout needs one compacting pass
      const int rest = B - bits1;
      const int np = (rest + max_bits - 1) / max_bits;
      for (int pi = 0; pi < np; pi++) {
        const int bits = (rest - (done - bits1) + (np - pi) - 1) / (np - pi);  // even split
        if (regions && np == 1 && bits <= 9 && last_regions_knob) {
          const int rc = run_pass_last_regions(bits);
          if (rc == CUSCI_OK) continue;
          if (rc != -1) return rc;
        }
        CUSCI_TRY(run_pass(bits, false, pi == np - 1));
      }
      if (np == 0) {  // pass 1 already made the buckets: its groups are the bucket offsets
        CUSCI_CUDA(ctx, cudaMemcpyAsync(off, gstart.data(), gstart.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                        ctx->stream));
        CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      }
      dcap = (uint32_t)std::min<double>(4e9, 1.25 * D / std::ldexp(1.0, B) + 64.0);
    }
  } else {
    const uint32_t o2[2] = {0u, (uint32_t)n};
    memcpy(ctx->host_pinned, o2, sizeof(o2));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(off, ctx->host_pinned, sizeof(o2), cudaMemcpyHostToDevice, ctx->stream));
    CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  const uint32_t nbk = 1u << B;
  // V = 1: each bucket is processed as two halves (by the next bit of hi),
  // each re-reading the bucket.  Needed when B = 0 (a table entry stores hi
  // without its top S = B + V >= 1 fixed bits, which frees its "occupied" bit);
  // otherwise a knob (measured slower on N2: the table load does not bound the kernel).
  static const int split_knob = [] {
    const char* e = getenv("CUSCI_BUCKET_SPLIT");  // tuning knob
    return e ? atoi(e) : 0;
  }();
  const int V = (B == 0 || (split_knob == 1 && B < 63)) ? 1 : 0;
  const uint32_t vdcap = V ? (dcap == 0xffffffffu ? dcap : dcap / 2u + 64u) : dcap;
  const uint32_t nb = nbk << V;  // work units (sub-buckets)
  const int raw = part == in ? 1 : 0;
  const unsigned dgrid =
      (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nb, (uint64_t)ctx->num_sms * ((raw || V) ? dper_g : dper)));
  CUSCI_CUDA(ctx, cudaMemsetAsync(lbst, 0, (nb + 1) * sizeof(unsigned long long), ctx->stream));  // + the ticket
  unsigned int* ticket = reinterpret_cast<unsigned int*>(lbst + nb);
  if (raw || V)
    CUSCI_LAUNCH(ctx, PT_HASH, bucket_unique_kernel<W, true><<<dgrid, kBU, C::SMEM, ctx->stream>>>(part, raw, off, ibase, nbk, B, V, lf, vdcap, out, lbst, ticket, flags, nullptr, nullptr, 0, 0ull));
  else
    CUSCI_LAUNCH(ctx, PT_HASH, bucket_unique_kernel<W, false><<<dgrid, kBU, C::SMEM, ctx->stream>>>(part, raw, off, ibase, nbk, B, V, lf, vdcap, out, lbst, ticket, flags, nullptr, nullptr, 0, 0ull));
  // the last unit's inclusive prefix is the survivor count
  uint64_t h[2];
  CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, lbst + nb - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaMemcpyAsync((char*)ctx->host_pinned + 8, flags, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(h, ctx->host_pinned, sizeof(h));
  h[0] &= kBVal;
  *n_out = h[0];
  ctx->dstats[0] += 1;
  ctx->dstats[1] += n;
  ctx->dstats[4] += nb;
  ctx->dstats[5] += h[1] ? 1 : 0;
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
  ctx->dstats[3] += *n_out;
  return CUSCI_OK;
}

// run bounds for the owner-side finalize: lb[r][b] = first index of run r
// (pi-sorted keys) whose top B bits of hi are >= b0 + b, b in [0, nu]
// (lb[r][nu] = the run's length: every key's bucket is <= b0 + nu - 1)
template <int W>
__global__ void run_bounds_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ rs,
                                  const uint64_t* __restrict__ rn, int P, int B, uint64_t b0, uint32_t nu,
                                  uint32_t* __restrict__ lb) {
  const uint32_t nbk1 = nu + 1;
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (uint64_t)P * nbk1) return;
  const uint32_t r = (uint32_t)(id / nbk1), b = (uint32_t)(id % nbk1);
  uint64_t lo = 0, hi = rn[r];
  if (b == nbk1 - 1) {
    lo = hi;
  } else {
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      const uint64_t top = B ? (hk_hi(load_key<W>(keys, rs[r] + mid)) >> (64 - B)) : 0ull;
      if (top < b0 + b) lo = mid + 1;
      else hi = mid;
    }
  }
  lb[id] = (uint32_t)lo;
}
// the hash range of P pi-sorted runs: ends[0] = min hi (over the runs' first
// keys), ends[1] = max hi (over their last keys); ends pre-set to (~0, 0)
template <int W>
__global__ void run_ends_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ rs,
                                const uint64_t* __restrict__ rn, int P, unsigned long long* __restrict__ ends) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P || rn[r] == 0) return;
  atomicMin(&ends[0], (unsigned long long)hk_hi(load_key<W>(keys, rs[r])));
  atomicMax(&ends[1], (unsigned long long)hk_hi(load_key<W>(keys, rs[r] + rn[r] - 1)));
}
// off[b] = sum_r lb[r][b]: bucket b's offset in the virtual concatenation
__global__ void run_offsets_kernel(const uint32_t* __restrict__ lb, int P, uint32_t nbk1, uint32_t* __restrict__ off) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbk1) return;
  uint32_t a = 0;
  for (int r = 0; r < P; r++) a += lb[(size_t)r * nbk1 + b];
  off[b] = a;
}

// owner-side finalize of dedup_global (a11): the P received runs (each
// strictly increasing in pi, back to back) -> their distinct keys in pi order.
// No partition pass: bucket b's keys are found in every run by binary search
// and the bucket kernel reads the P segments directly.
template <int W>
int runs_dedup_impl(cusci_ctx* ctx, const uint64_t* in, const uint64_t* counts, int P, uint64_t* out, uint64_t* n_out) {
  using C = BUCfg<W>;
  *n_out = 0;
  uint64_t n = 0;
  std::vector<uint64_t> rs(P), rn(P);
  for (int r = 0; r < P; r++) {
    rs[r] = n;
    rn[r] = counts[r];
    n += counts[r];
  }
  if (n == 0) return CUSCI_OK;
  if (n >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "dedup: %llu received keys exceed 2^32", (unsigned long long)n);
  Scratch s(ctx);
  uint64_t* drs;
  unsigned long long* ends;
  CUSCI_TRY(s.get_t(2 * (size_t)P, &drs));
  CUSCI_TRY(s.get_t(2, &ends));
  std::vector<uint64_t> hr(2 * P);
  for (int r = 0; r < P; r++) {
    hr[r] = rs[r];
    hr[P + r] = rn[r];
  }
  CUSCI_CUDA(ctx, cudaMemcpyAsync(drs, hr.data(), 2 * P * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  // the received keys' hash range: an owner's runs all lie in its range
  // [r 2^64 / P, (r + 1) 2^64 / P), so bucketing by the top bits of hi over the
  // whole space would put everything into 1/P of the buckets (tables overflow);
  // the bucket bits are widened by the range's leading zero bits and only the
  // buckets inside [min, max] become work units
  {
    const unsigned long long e0[2] = {~0ull, 0ull};
    memcpy(ctx->host_pinned, e0, sizeof(e0));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(ends, ctx->host_pinned, sizeof(e0), cudaMemcpyHostToDevice, ctx->stream));
    CUSCI_LAUNCH(ctx, PT_SCATTER, run_ends_kernel<W><<<(P + 127) / 128, 128, 0, ctx->stream>>>(in, drs, drs + P, P, ends));
  }
  uint64_t hmm[2];
  CUSCI_TRY(read_u64(ctx, reinterpret_cast<const uint64_t*>(ends), hmm, 2));
  int B = 0;
  while ((n >> B) > C::DT && B < 22) B++;  // the distinct count is <= n
  const uint64_t span = hmm[1] - hmm[0];
  const int extra = span ? __builtin_clzll(span) : 63;  // the range fits in 2^(64 - extra)
  const int Bt = std::min(B + extra, 63);
  const uint64_t b0 = Bt ? hmm[0] >> (64 - Bt) : 0ull, b1 = Bt ? hmm[1] >> (64 - Bt) : 0ull;
  const int V = Bt == 0 ? 1 : 0;
  const uint32_t nbk = (uint32_t)(b1 - b0 + 1), nb = nbk << V;  // <= 2^(B + 1) buckets
  uint32_t *lb, *off;
  unsigned long long *flags, *lbst;
  CUSCI_TRY(s.get_t((size_t)P * (nbk + 1), &lb));
  CUSCI_TRY(s.get_t(nbk + 1, &off));
  CUSCI_TRY(s.get_t(nb + 1, &lbst));
  CUSCI_TRY(s.get_t(2, &flags));
  CUSCI_CUDA(ctx, cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned long long), ctx->stream));
  const uint64_t nth = (uint64_t)P * (nbk + 1);
  CUSCI_LAUNCH(ctx, PT_SCATTER, run_bounds_kernel<W><<<(unsigned)((nth + 255) / 256), 256, 0, ctx->stream>>>(in, drs, drs + P, P, Bt, b0, nbk, lb));
  CUSCI_LAUNCH(ctx, PT_SCATTER, run_offsets_kernel<<<(nbk + 1 + 255) / 256, 256, 0, ctx->stream>>>(lb, P, nbk + 1, off));
  int dper = 1;
  CUSCI_TRY(kernel_setup(ctx, (const void*)bucket_unique_kernel<W, true>, kBU, C::SMEM, &dper));
  const unsigned dgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nb, (uint64_t)ctx->num_sms * dper));
  static const uint32_t lf = [] {
    const char* e = getenv("CUSCI_TABLE_LF");
    return e ? (uint32_t)std::max(1, atoi(e)) : 3u;
  }();
  CUSCI_CUDA(ctx, cudaMemsetAsync(lbst, 0, (nb + 1) * sizeof(unsigned long long), ctx->stream));
  CUSCI_LAUNCH(ctx, PT_HASH, bucket_unique_kernel<W, true><<<dgrid, kBU, C::SMEM, ctx->stream>>>(in, 1, off, nullptr, nbk, Bt, V, lf, 0xffffffffu, out, lbst, reinterpret_cast<unsigned int*>(lbst + nb), flags, lb, drs, P, b0 << V));
  uint64_t h[2];
  CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, lbst + nb - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaMemcpyAsync((char*)ctx->host_pinned + 8, flags, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(h, ctx->host_pinned, sizeof(h));
  h[0] &= kBVal;
  ctx->dstats[0] += 1;
  ctx->dstats[1] += n;
  ctx->dstats[3] += h[1] ? 0 : h[0];
  ctx->dstats[4] += nb;
  if (h[1]) return local_dedup_impl<W>(ctx, in, n, out, n_out);  // a table overflowed: the general path
  *n_out = h[0];
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

int runs_dedup(cusci_ctx* ctx, int W, const uint64_t* in, const uint64_t* counts, int P, uint64_t* out,
               uint64_t* n_out) {
  return W == 1 ? runs_dedup_impl<1>(ctx, in, counts, P, out, n_out) : runs_dedup_impl<2>(ctx, in, counts, P, out, n_out);
}

int owner_counts(cusci_ctx* ctx, int W, const uint64_t* keys, uint64_t n, int P, uint64_t* counts) {
  return W == 1 ? owner_bounds_impl<1>(ctx, keys, n, P, counts) : owner_bounds_impl<2>(ctx, keys, n, P, counts);
}

}  // namespace cusci
