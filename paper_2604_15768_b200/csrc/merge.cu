// merge_space: S <- S u U on the GPU-resident pool shard (
// PAPER.md:311-312 Sec 2.2 "merging them into S", :404-405; abstract :167
// "GPU-side pooling").
//
// B200 design: merge path in the pool (hash) order
// (reading r13).  The merged sequence of S (sorted unique) and U (sorted
// unique), ties S-first, is cut into tiles of kTile outputs by a diagonal
// binary search per tile boundary; each CTA stages its S and U runs in shared
// memory, maps them to their pi-values, merges them (ITEMS outputs per thread
// in registers from one in-tile diagonal search), drops an element equal to
// its predecessor (an element of U already in S), validates U's order, and
// writes S' and
// inserted = U \ S at offsets found by decoupled look-back -- ONE sweep over
// S and U.  S' goes to the pool's second buffer (grown geometrically to the
// upper bound |S| + |U| when needed) and the buffers are swapped.
#include <algorithm>

#include "internal.cuh"

namespace cusci {
namespace {

constexpr int kMergeThreads = 256;
template <int W> struct MergeCfg {
#ifndef CUSCI_MERGE_ITEMS1
#define CUSCI_MERGE_ITEMS1 8
#endif
  static constexpr int ITEMS = W == 1 ? CUSCI_MERGE_ITEMS1 : 4;  // outputs per thread (<= 32: bit masks)
  static constexpr int TILE = kMergeThreads * ITEMS;
  static constexpr int BUFE = TILE + 4;          // + parity slack of the two runs (W = 1)
  // dynamic shared memory: two TMA input buffers, the tile's pi-values
  // (later its kept keys), the inserted outputs' buffer indices
  static constexpr size_t SMEM = 2 * (size_t)BUFE * sizeof(KeyT<W>) + (size_t)TILE * (sizeof(KeyT<W>) + 2);
};

template <int W>
__global__ void merge_split_kernel(const uint64_t* __restrict__ S, uint64_t nS, const uint64_t* __restrict__ U,
                                   uint64_t nU, uint64_t ntiles, uint64_t* __restrict__ split) {
  constexpr int kTile = MergeCfg<W>::TILE;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  const uint64_t d = std::min<uint64_t>(t * kTile, nS + nU);
  uint64_t lo = d > nU ? d - nU : 0, hi = std::min(d, nS);
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (hk_le<W>(load_key<W>(S, mid), load_key<W>(U, d - mid - 1))) lo = mid + 1;
    else hi = mid;
  }
  split[t] = lo;
}

// strict ascending check of U: flag[0] = 1 if any U[i] <= U[i-1]
template <int W>
__global__ void check_sorted_kernel(const uint64_t* __restrict__ U, uint64_t n, int* __restrict__ flag) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += stride)
    if (!hk_lt<W>(load_key<W>(U, i - 1), load_key<W>(U, i))) *flag = 1;
}

// Single sweep: persistent CTAs take tiles c, c + G, ... (predecessors are resident;
// dynamic tile tickets measured 1.8x slower: staggered tiles lengthen the look-back);
// per tile a CTA merges its S and U runs in shared memory (merge path), drops an element
// equal to its predecessor (an element of U already in S), checks that its U
// run is strictly increasing in the hash order, and counts its kept /
// inserted outputs with ONE block scan.  Warp 0 publishes the tile counts
// and resolves the tile's output offsets by a warp-parallel decoupled
// look-back; the kept and inserted outputs are compacted into shared-memory
// lists and written out with coalesced stores.
constexpr uint64_t kMFlagA = 1ull << 62, kMFlagP = 2ull << 62, kMVal = (1ull << 62) - 1;

// warp 0: decoupled look-back for tile t over status[2 q] (kept) and
// status[2 q + 1] (inserted), published together; returns both exclusive
// prefixes (all lanes).  A window covers 32 x kLB predecessors (kLB per lane,
// one 16-byte load each), so the inclusive-prefix front advances kLB x 32
// tiles per L2 round trip.
constexpr int kLB = 1;
__device__ __forceinline__ ulonglong2 ld_status2(volatile unsigned long long* p) {
  ulonglong2 r;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"((unsigned long long*)p));
  return r;
}
__device__ __forceinline__ void lookback2(volatile unsigned long long* st, uint64_t t, uint64_t& ek, uint64_t& ei) {
  const unsigned lane = lane_id();
  ek = 0;
  ei = 0;
  bool dk = false, di = false;
  int64_t q0 = (int64_t)t - 1;
  while (q0 >= 0 && !(dk && di)) {
    uint64_t vk[kLB], vi[kLB];
#pragma unroll
    for (int v = 0; v < kLB; v++) {
      const int64_t q = q0 - (int64_t)(lane * kLB + v);  // (lane, v) -> distance lane kLB + v
      vk[v] = kMFlagP;
      vi[v] = kMFlagP;
      if (q >= 0) {
        const ulonglong2 x = ld_status2(st + 2 * q);
        vk[v] = x.x;
        vi[v] = x.y;
      }
    }
    // wait until every status in the window has at least an aggregate
    for (;;) {
      bool miss = false;
#pragma unroll
      for (int v = 0; v < kLB; v++) miss |= (vk[v] >> 62) == 0 || (vi[v] >> 62) == 0;
      if (!__any_sync(kFull, miss)) break;
#pragma unroll
      for (int v = 0; v < kLB; v++) {
        const int64_t q = q0 - (int64_t)(lane * kLB + v);
        if (q >= 0 && ((vk[v] >> 62) == 0 || (vi[v] >> 62) == 0)) {
          const ulonglong2 x = ld_status2(st + 2 * q);
          vk[v] = x.x;
          vi[v] = x.y;
        }
      }
    }
    // per component: sum up to (and including) the nearest inclusive prefix
    int fk = kLB, fi = kLB;  // first v with P in this lane
#pragma unroll
    for (int v = kLB - 1; v >= 0; v--) {
      if ((vk[v] >> 62) == 2) fk = v;
      if ((vi[v] >> 62) == 2) fi = v;
    }
    const unsigned bk = __ballot_sync(kFull, fk < kLB), bi = __ballot_sync(kFull, fi < kLB);
    const int Lk = bk ? __ffs(bk) - 1 : 32, Li = bi ? __ffs(bi) - 1 : 32;
    uint64_t sk = 0, si = 0;
#pragma unroll
    for (int v = 0; v < kLB; v++) {
      if ((int)lane < Lk || ((int)lane == Lk && v <= fk)) sk += vk[v] & kMVal;
      if ((int)lane < Li || ((int)lane == Li && v <= fi)) si += vi[v] & kMVal;
    }
    for (int o = 16; o; o >>= 1) {
      sk += __shfl_xor_sync(kFull, sk, o);
      si += __shfl_xor_sync(kFull, si, o);
    }
    if (!dk) ek += sk;
    if (!di) ei += si;
    dk = dk || bk;
    di = di || bi;
    q0 -= 32 * kLB;
  }
}

// Tile geometry: S run [i0, i1), U run [j0, j1); in its shared-memory buffer
// the S run starts at sl and the U run at ul, chosen so that a key's buffer
// index has the parity of its global index (W = 1): then the 16-byte aligned
// core of each run is one 1-D TMA bulk copy and only an odd head / tail key
// is read with a plain load.
struct MTile {
  uint64_t i0, i1, j0, j1;
  uint32_t na, nb, sl, ul;
  bool inval;
};
template <int W>
__device__ __forceinline__ MTile mtile(const uint64_t* split, uint64_t t, uint64_t nS, uint64_t nU) {
  constexpr int kTile = MergeCfg<W>::TILE;
  MTile g;
  g.i0 = split[t];
  g.i1 = split[t + 1];
  const uint64_t d0 = t * kTile, d1 = std::min<uint64_t>(d0 + kTile, nS + nU);
  g.j0 = d0 - g.i0;
  g.j1 = d1 - g.i1;
  // an unsorted U can make the merge-path splits inconsistent: process nothing
  g.inval = g.i1 < g.i0 || g.j1 < g.j0 || (g.i1 - g.i0) + (g.j1 - g.j0) > (uint64_t)kTile || g.j1 > nU || g.i1 > nS;
  g.na = g.inval ? 0u : (uint32_t)(g.i1 - g.i0);
  g.nb = g.inval ? 0u : (uint32_t)(g.j1 - g.j0);
  g.sl = W == 1 ? (uint32_t)(g.i0 & 1) : 0u;
  g.ul = g.sl + g.na;
  if (W == 1) g.ul += (uint32_t)((g.ul + g.j0) & 1);
  return g;
}
// thread 0: TMA the aligned cores of both runs into buf (one barrier)
template <int W>
__device__ __forceinline__ void mtile_issue(const MTile& g, const uint64_t* S, const uint64_t* U, KeyT<W>* buf,
                                            uint64_t* bar) {
  uint32_t bytes = 0;
  uint64_t sc0 = g.i0, sc1 = g.i0 + g.na, uc0 = g.j0, uc1 = g.j0 + g.nb;
  if (W == 1) {
    sc0 = (sc0 + 1) & ~1ull;
    sc1 &= ~1ull;
    uc0 = (uc0 + 1) & ~1ull;
    uc1 &= ~1ull;
  }
  if (sc1 > sc0) bytes += (uint32_t)(sc1 - sc0) * 8u * W;
  if (uc1 > uc0) bytes += (uint32_t)(uc1 - uc0) * 8u * W;
  if (!bytes) return;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  if (sc1 > sc0)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(buf + g.sl + (sc0 - g.i0))),
                 "l"(S + sc0 * W), "r"((uint32_t)(sc1 - sc0) * 8u * W), "r"(smem_u32(bar))
                 : "memory");
  if (uc1 > uc0)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(buf + g.ul + (uc0 - g.j0))),
                 "l"(U + uc0 * W), "r"((uint32_t)(uc1 - uc0) * 8u * W), "r"(smem_u32(bar))
                 : "memory");
}
template <int W>
__device__ __forceinline__ bool mtile_issued(const MTile& g) {
  if (W == 2) return g.na + g.nb > 0;
  const uint64_t sc0 = (g.i0 + 1) & ~1ull, sc1 = (g.i0 + g.na) & ~1ull;
  const uint64_t uc0 = (g.j0 + 1) & ~1ull, uc1 = (g.j0 + g.nb) & ~1ull;
  return sc1 > sc0 || uc1 > uc0;
}

// Persistent merge: CTA c owns tiles c, c + G, ... (G = resident CTAs, so a
// tile's predecessors are always being processed: the look-back cannot
// deadlock).  While tile t is merged, the S and U runs of tile t + G stream
// into the other buffer by TMA.  Per tile: the keys are mapped once to their
// pi-values (an exact bijection, so pi equality is key equality); each thread
// merges ITEMS outputs in registers from one merge-path diagonal search (ties
// S-first) and drops an output equal to its predecessor (an element of U
// already in S) as it goes; one block scan counts the kept and inserted
// outputs together; warp 0 publishes the counts and resolves the output
// offsets by a warp-parallel decoupled look-back while the kept keys are
// staged in order in shared memory; they leave with coalesced stores.
template <int W>
__global__ void __launch_bounds__(kMergeThreads) merge_tile_kernel(const uint64_t* __restrict__ S, uint64_t nS,
                                                                  const uint64_t* __restrict__ U, uint64_t nU,
                                                                  const uint64_t* __restrict__ split, uint64_t ntiles,
                                                                  unsigned long long* __restrict__ status,
                                                                  int* __restrict__ bad,
                                                                  uint64_t* __restrict__ out, uint64_t* __restrict__ ins,
                                                                  int check_u) {
  using K = KeyT<W>;
  constexpr int IT = MergeCfg<W>::ITEMS;
  constexpr int kTile = MergeCfg<W>::TILE;
  constexpr int BUFE = MergeCfg<W>::BUFE;
  extern __shared__ __align__(16) unsigned char msm[];
  K* bufs = reinterpret_cast<K*>(msm);                        // [2][BUFE] keys (TMA targets)
  K* hv = bufs + 2 * BUFE;                                    // [TILE] pi-values by logical index (S run, then U run);
                                                              // after the merge: the kept keys in output order
  uint16_t* li = reinterpret_cast<uint16_t*>(hv + kTile);     // [TILE] inserted outputs (buffer indices)
  __shared__ uint32_t red[33];
  __shared__ uint64_t run_k, run_i;
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init_fence();
  }
  __syncthreads();
  const bool tma = ((reinterpret_cast<uintptr_t>(S) | reinterpret_cast<uintptr_t>(U)) & 15u) == 0;
  uint32_t phase = 0;
  int cb = 0;
  if (tma && threadIdx.x == 0 && blockIdx.x < ntiles)
    mtile_issue<W>(mtile<W>(split, blockIdx.x, nS, nU), S, U, bufs, &bar[0]);
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, cb ^= 1) {
    const MTile g = mtile<W>(split, t, nS, nU);
    K* buf = bufs + cb * BUFE;
    if (tma && threadIdx.x == 0 && t + gridDim.x < ntiles) {  // prefetch the next tile into the other buffer
      fence_proxy_async_smem();
      mtile_issue<W>(mtile<W>(split, t + gridDim.x, nS, nU), S, U, bufs + (cb ^ 1) * BUFE, &bar[cb ^ 1]);
    }
    if (g.inval && threadIdx.x == 0) *bad = 1;
    const int na = (int)g.na, nb = (int)g.nb, len = na + nb;
    if (tma && mtile_issued<W>(g)) {
      mbar_wait(&bar[cb], (phase >> cb) & 1u);
      phase ^= 1u << cb;
    }
    // keys -> pi-values; keys outside the TMA cores (odd head / tail at W = 1,
    // everything without TMA) come from plain loads
    {
      int s0 = 0, s1 = 0, u0 = 0, u1 = 0;  // TMA core of each run, local indices
      if (tma) {
        if (W == 1) {
          s0 = (int)(((g.i0 + 1) & ~1ull) - g.i0);
          s1 = (int)(((g.i0 + na) & ~1ull) - g.i0);
          u0 = (int)(((g.j0 + 1) & ~1ull) - g.j0);
          u1 = (int)(((g.j0 + nb) & ~1ull) - g.j0);
        } else {
          s1 = na;
          u1 = nb;
        }
      }
      for (int x = threadIdx.x; x < na; x += kMergeThreads) {
        K k;
        if (x >= s0 && x < s1) {
          k = buf[g.sl + x];
        } else {
          k = load_key<W>(S, g.i0 + x);
          buf[g.sl + x] = k;
        }
        hv[x] = to_pi(k);
      }
      for (int y = threadIdx.x; y < nb; y += kMergeThreads) {
        K k;
        if (y >= u0 && y < u1) {
          k = buf[g.ul + y];
        } else {
          k = load_key<W>(U, g.j0 + y);
          buf[g.ul + y] = k;
        }
        hv[na + y] = to_pi(k);
      }
    }
    __syncthreads();
    if (check_u) {  // input check: U strictly increasing in the hash order (tile run + left boundary)
      bool badu = false;
      for (int y = threadIdx.x; y < nb; y += kMergeThreads) {
        if (y > 0) badu |= !pi_lt(hv[na + y - 1], hv[na + y]);
        else if (g.j0 > 0 && g.j0 <= nU) badu |= !pi_lt(to_pi(load_key<W>(U, g.j0 - 1)), hv[na]);
      }
      if (badu) *bad = 1;
    }
    // this thread's outputs [k0, k0 + IT): merged in registers, duplicates of
    // the predecessor dropped (bit r of km: output k0 + r kept; of im: kept
    // and from U = inserted)
    const int k0 = threadIdx.x * IT;
    uint32_t km = 0, im = 0;
    uint32_t idx[IT];
    if (k0 < len) {
      int lo = k0 > nb ? k0 - nb : 0, hi = min(k0, na);
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (!pi_lt(hv[na + k0 - mid - 1], hv[mid])) lo = mid + 1;  // S[mid] <= U[k0 - mid - 1]
        else hi = mid;
      }
      int i = lo, j = k0 - lo;
      K prev{};
      bool hp = false;
      if (k0 > 0) {
        hp = true;
        if (i == 0) prev = hv[na + j - 1];
        else if (j == 0) prev = hv[i - 1];
        else prev = pi_lt(hv[i - 1], hv[na + j - 1]) ? hv[na + j - 1] : hv[i - 1];
      } else if (!g.inval) {  // the tile's predecessor: the larger of S[i0 - 1], U[j0 - 1]
        if (g.i0 > 0) {
          prev = to_pi(load_key<W>(S, g.i0 - 1));
          hp = true;
        }
        if (g.j0 > 0) {
          const K u = to_pi(load_key<W>(U, g.j0 - 1));
          if (!hp || pi_lt(prev, u)) prev = u;
          hp = true;
        }
      }
      K a = i < na ? hv[i] : K{}, b = j < nb ? hv[na + j] : K{};
#pragma unroll
      for (int r = 0; r < IT; r++) {
        idx[r] = 0;
        if (k0 + r < len) {
          const bool takeA = i < na && (j >= nb || !pi_lt(b, a));
          const K v = takeA ? a : b;
          idx[r] = takeA ? g.sl + i : g.ul + j;
          if (takeA) {
            i++;
            if (i < na) a = hv[i];
          } else {
            j++;
            if (j < nb) b = hv[na + j];
          }
          if (!(hp && key_eq(v, prev))) {
            km |= 1u << r;
            if (!takeA) im |= 1u << r;
          }
          prev = v;
          hp = true;
        }
      }
    }
    // kept (low 16 bits) and inserted (high 16 bits) counted by one scan; its
    // barriers also end every thread's merge (hv is free from here on)
    uint32_t tot;
    const uint32_t ex = block_excl_scan_u32((uint32_t)__popc(km) | ((uint32_t)__popc(im) << 16), red, tot);
    const uint32_t tk = tot & 0xffffu, ti = tot >> 16;
    if (threadIdx.x < 32) {  // publish + warp-parallel look-back
      volatile unsigned long long* st = status;
      if (threadIdx.x == 0) {
        st[2 * t] = (t == 0 ? kMFlagP : kMFlagA) | tk;
        st[2 * t + 1] = (t == 0 ? kMFlagP : kMFlagA) | ti;
      }
      uint64_t ek = 0, ei = 0;
      if (t > 0) {
        lookback2(st, t, ek, ei);
        if (threadIdx.x == 0) {
          st[2 * t] = kMFlagP | (ek + tk);
          st[2 * t + 1] = kMFlagP | (ei + ti);
        }
      }
      if (threadIdx.x == 0) {
        run_k = ek;
        run_i = ei;
      }
    }
    {  // stage the kept keys (in output order) and the inserted indices
      uint32_t pk = ex & 0xffffu, pin = ex >> 16;
#pragma unroll
      for (int r = 0; r < IT; r++) {
        if ((km >> r) & 1u) hv[pk++] = buf[idx[r]];
        if ((im >> r) & 1u) li[pin++] = (uint16_t)idx[r];
      }
    }
    __syncthreads();
    const uint64_t rk = run_k, rin = run_i;
    for (uint32_t x = threadIdx.x; x < tk; x += kMergeThreads) store_key<W>(out, rk + x, hv[x]);
    if (ins)
      for (uint32_t x = threadIdx.x; x < ti; x += kMergeThreads) store_key<W>(ins, rin + x, buf[li[x]]);
    __syncthreads();  // buffers, lists and run offsets free for the next tile
  }
}

// ---------------------------------------------------------------- sparse merge
// |small| << |big| (e.g. S <- S u C with a few parents into a large unique set):
// every small key finds its slot in the big run by binary search, the
// non-duplicates are ranked by one scan, and the big run is copied with the
// shift "non-duplicate small keys at or before me" (constant between insert
// points) -- copy-speed traffic instead of a full merge.
template <int W>
__global__ void sparse_locate_kernel(const uint64_t* __restrict__ small, uint64_t ns, const uint64_t* __restrict__ big,
                                     uint64_t nb, uint64_t* __restrict__ pos, uint32_t* __restrict__ keep) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += stride) {
    const KeyT<W> x = load_key<W>(small, i);
    uint64_t lo = 0, hi = nb;
    while (lo < hi) {  // first big key >= x (hash order)
      const uint64_t mid = (lo + hi) >> 1;
      if (hk_lt<W>(load_key<W>(big, mid), x)) lo = mid + 1;
      else hi = mid;
    }
    pos[i] = lo;
    keep[i] = (lo < nb && key_eq(load_key<W>(big, lo), x)) ? 0u : 1u;
  }
}

// big[j] -> out[j + shift(j)], shift(j) = rank[upper_bound(pos, j)]
// (rank = exclusive scan of keep, rank[ns] = total inserts)
// Copy kernels: one warp per span of SPAN = 32 R consecutive keys, R keys per
// lane loaded before anything is stored (independent loads in flight, no
// block barriers).  The order check compares each key's hash with its
// predecessor's, taken from a neighbouring lane (one extra load per span).
template <int W> struct CopyCfg {
  static constexpr int R = W == 1 ? 16 : 8;
  static constexpr uint32_t SPAN = 32 * R;
};
// strict order check of a span's keys x[] (predecessor of the span: pw/hw)
template <int W>
__device__ __forceinline__ bool span_bad(const KeyT<W> (&x)[CopyCfg<W>::R], uint64_t j0, uint64_t j1,
                                         const KeyT<W>& pw, uint64_t hw) {
  constexpr int R = CopyCfg<W>::R;
  const unsigned lane = lane_id();
  bool bad = false;
  uint64_t hl = hw;  // hash of the previous row's lane-31 key
  KeyT<W> kl = pw;
#pragma unroll
  for (int r = 0; r < R; r++) {
    const uint64_t j = j0 + (uint64_t)r * 32 + lane;
    const uint64_t h = hk_hi(x[r]);
    uint64_t hp = __shfl_up_sync(kFull, h, 1);
    KeyT<W> kp;
    kp.w0 = __shfl_up_sync(kFull, x[r].w0, 1);
    if constexpr (W == 2) kp.w1 = __shfl_up_sync(kFull, x[r].w1, 1);
    if (lane == 0) {
      hp = hl;
      kp = kl;
    }
    if (j < j1 && j > 0) bad |= hp > h || (hp == h && !hk_lt<W>(kp, x[r]));
    hl = __shfl_sync(kFull, h, 31);
    kl.w0 = __shfl_sync(kFull, x[r].w0, 31);
    if constexpr (W == 2) kl.w1 = __shfl_sync(kFull, x[r].w1, 31);
  }
  return bad;
}

// cb[s] = first i with pos[i] >= min(s SPAN, nb): the inserts before span s's keys
template <int W>
__global__ void sparse_bounds_kernel(const uint64_t* __restrict__ pos, uint64_t ns, uint64_t nb, uint64_t nsp,
                                     uint64_t* __restrict__ cb) {
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nsp) return;
  const uint64_t v = std::min<uint64_t>(c * CopyCfg<W>::SPAN, nb);
  uint64_t lo = 0, hi = ns;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (pos[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  cb[c] = lo;
}

// out[j + shift(j)] = big[j], shift(j) = rank at the first insert with pos > j
// (an insert with pos == j is placed before big[j]).  A span with at most 31
// inserts holds their positions / ranks in lanes; more fall back to a search.
template <int W>
__global__ void __launch_bounds__(256) sparse_copy_kernel(const uint64_t* __restrict__ big, uint64_t nb,
                                                          const uint64_t* __restrict__ pos,
                                                          const uint64_t* __restrict__ rank,
                                                          const uint64_t* __restrict__ cb,
                                                          uint64_t* __restrict__ out,
                                                          int* __restrict__ bad /* non-null: also check big's strict hash order */) {
  constexpr int R = CopyCfg<W>::R;
  constexpr uint32_t SPAN = CopyCfg<W>::SPAN;
  const unsigned lane = lane_id();
  const uint64_t nsp = (nb + SPAN - 1) / SPAN;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x / 32);
  bool badl = false;
  for (uint64_t sp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; sp < nsp; sp += nw) {
    const uint64_t j0 = sp * SPAN, j1 = std::min<uint64_t>(nb, j0 + SPAN);
    KeyT<W> x[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const uint64_t j = j0 + (uint64_t)r * 32 + lane;
      if (j < j1) x[r] = load_key<W>(big, j);
    }
    KeyT<W> pw{};
    if (bad && j0 > 0) pw = load_key<W>(big, j0 - 1);
    const uint64_t u0 = cb[sp], u1 = cb[sp + 1];
    const uint32_t m = (uint32_t)(u1 - u0);
    uint64_t lp = ~0ull, lr = 0;  // lane i < m: insert u0 + i's position; lane i <= m: its rank
    if (m < 32) {
      if (lane < m) lp = pos[u0 + lane];
      if (lane <= m) lr = rank[u0 + lane];
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      const uint64_t j = j0 + (uint64_t)r * 32 + lane;
      uint64_t shift;
      if (m < 32) {
        uint32_t cnt = 0;
        for (uint32_t i = 0; i < m; i++) cnt += __shfl_sync(kFull, lp, i) <= j;
        shift = __shfl_sync(kFull, lr, cnt);
      } else {
        uint64_t lo = u0, hi = u1;
        while (lo < hi) {
          const uint64_t mid = (lo + hi) >> 1;
          if (pos[mid] <= j) lo = mid + 1;
          else hi = mid;
        }
        shift = rank[lo];
      }
      if (j < j1) store_key<W>(out, j + shift, x[r]);
    }
    if (bad) badl |= span_bad<W>(x, j0, j1, pw, hk_hi(pw));
  }
  if (badl) *bad = 1;
}

// empty pool: out = U (and ins = U) in one pass, checking U's strict hash order
template <int W>
__global__ void __launch_bounds__(256) copy_check_kernel(const uint64_t* __restrict__ U, uint64_t n,
                                                         uint64_t* __restrict__ out, uint64_t* __restrict__ ins,
                                                         int* __restrict__ bad) {
  constexpr int R = CopyCfg<W>::R;
  constexpr uint32_t SPAN = CopyCfg<W>::SPAN;
  const unsigned lane = lane_id();
  const uint64_t nsp = (n + SPAN - 1) / SPAN;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x / 32);
  bool badl = false;
  for (uint64_t sp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; sp < nsp; sp += nw) {
    const uint64_t j0 = sp * SPAN, j1 = std::min<uint64_t>(n, j0 + SPAN);
    KeyT<W> x[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const uint64_t j = j0 + (uint64_t)r * 32 + lane;
      if (j < j1) x[r] = load_key<W>(U, j);
    }
    KeyT<W> pw{};
    if (j0 > 0) pw = load_key<W>(U, j0 - 1);
#pragma unroll
    for (int r = 0; r < R; r++) {
      const uint64_t j = j0 + (uint64_t)r * 32 + lane;
      if (j < j1) {
        store_key<W>(out, j, x[r]);
        if (ins) store_key<W>(ins, j, x[r]);
      }
    }
    if (bad) badl |= span_bad<W>(x, j0, j1, pw, hk_hi(pw));
  }
  if (badl) *bad = 1;
}

template <int W>
__global__ void sparse_place_kernel(const uint64_t* __restrict__ small, uint64_t ns, const uint64_t* __restrict__ pos,
                                    const uint32_t* __restrict__ keep, const uint64_t* __restrict__ rank,
                                    uint64_t* __restrict__ out, uint64_t* __restrict__ ins) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += stride) {
    if (!keep[i]) continue;
    const KeyT<W> x = load_key<W>(small, i);
    store_key<W>(out, pos[i] + rank[i], x);
    if (ins) store_key<W>(ins, rank[i], x);
  }
}

template <int W>
// trusted: U is another pool's key array (sorted and unique by construction):
// the input-order check is skipped
int merge_impl(cusci_ctx* ctx, cusci_pool* pool, const uint64_t* U, uint64_t nU, cusci_keys* inserted,
               bool trusted) {
  const uint64_t nS = pool->count;
  const uint64_t* S = pool->buf[pool->cur];
  const uint64_t total = nS + nU;
  Scratch s(ctx);
  if (inserted) {
    inserted->keys = nullptr;
    inserted->count = 0;
  }
  if (nU == 0) {
    if (inserted) {
      void* o;
      CUSCI_TRY(out_alloc(ctx, 256, &o));
      inserted->keys = (uint64_t*)o;
    }
    return CUSCI_OK;
  }
  constexpr int kTile = MergeCfg<W>::TILE;
  const uint64_t ntiles = (total + kTile - 1) / kTile;
  uint64_t* split;
  unsigned long long* status;
  int* bad;
  CUSCI_TRY(s.get_t(ntiles + 1, &split));
  CUSCI_TRY(s.get_t(2 * ntiles, &status));
  CUSCI_TRY(s.get_t(1, &bad));
  CUSCI_CUDA(ctx, cudaMemsetAsync(status, 0, 2 * ntiles * sizeof(unsigned long long), ctx->stream));
  CUSCI_CUDA(ctx, cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
  // destination: the pool's other buffer, grown to the upper bound nS + nU if needed
  uint64_t* dst = pool->buf[1 - pool->cur];
  uint64_t* grown[2] = {nullptr, nullptr};
  uint64_t ncap = pool->cap;
  if (total > pool->cap) {
    ncap = std::max<uint64_t>(pool->cap * 2, total + total / 4);
    for (int b = 0; b < 2; b++) {
      if (cudaMallocFromPoolAsync((void**)&grown[b], ncap * W * 8, ctx->pool, ctx->stream) != cudaSuccess) {
        cudaGetLastError();
        if (grown[0]) cudaFreeAsync(grown[0], ctx->stream);
        return set_error(ctx, CUSCI_E_OOM, "pool growth to %llu keys failed", (unsigned long long)ncap);
      }
    }
    dst = grown[0];
  }
  void* insp = nullptr;
  if (inserted) {
    const int rc = out_alloc(ctx, nU * W * 8, &insp);
    if (rc != CUSCI_OK) {
      for (int b = 0; b < 2; b++)
        if (grown[b]) cudaFreeAsync(grown[b], ctx->stream);
      return rc;
    }
  }
  uint64_t h[3];
  if (nS == 0) {
    // empty pool: S' = U (validated strictly increasing in the hash order), a copy
    const unsigned cg = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nU + 8 * CopyCfg<W>::SPAN - 1) / (8 * CopyCfg<W>::SPAN), (uint64_t)ctx->num_sms * 8));
    CUSCI_LAUNCH(ctx, PT_CHECK, copy_check_kernel<W><<<cg, 256, 0, ctx->stream>>>(U, nU, dst, (uint64_t*)insp, trusted ? nullptr : bad));
    CUSCI_CUDA(ctx, cudaMemcpyAsync((char*)ctx->host_pinned + 16, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    h[0] = nU;
    h[1] = nU;
    if (*(int*)((char*)ctx->host_pinned + 16)) {
      for (int b = 0; b < 2; b++)
        if (grown[b]) cudaFreeAsync(grown[b], ctx->stream);
      if (insp) out_free(ctx, insp);
      return set_error(ctx, CUSCI_E_INVALID_ARG, "merge_space: new_keys must be sorted in the pool (hash) order and unique");
    }
  } else if (nU * 64 <= nS || (nS * 64 <= nU && !inserted)) {
    // sparse: the small run's keys are located in the big run and inserted while
    // the big run is copied.  U small: inserted = the kept U keys, in order; S
    // small (only without `inserted`): |inserted| = nU - (duplicates).
    const bool u_small = nU * 64 <= nS;
    const uint64_t* small = u_small ? U : S;
    const uint64_t* big = u_small ? S : U;
    const uint64_t nsm = u_small ? nU : nS, nbg = u_small ? nS : nU;
    if (u_small && !trusted) {  // a large U is checked inside the copy
      const unsigned cu = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nU + 255) / 256, (uint64_t)ctx->num_sms * 8));
      CUSCI_LAUNCH(ctx, PT_CHECK, check_sorted_kernel<W><<<cu, 256, 0, ctx->stream>>>(U, nU, bad));
    }
    const unsigned cg = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nsm + 255) / 256, (uint64_t)ctx->num_sms * 8));
    uint64_t *pos, *keep64, *rank;
    uint32_t* keep;
    CUSCI_TRY(s.get_t(nsm, &pos));
    CUSCI_TRY(s.get_t(nsm, &keep));
    CUSCI_TRY(s.get_t(nsm + 1, &keep64));
    CUSCI_TRY(s.get_t(nsm + 1, &rank));
    CUSCI_LAUNCH(ctx, PT_MERGE_SPLIT, sparse_locate_kernel<W><<<cg, 256, 0, ctx->stream>>>(small, nsm, big, nbg, pos, keep));
    CUSCI_CUDA(ctx, cudaMemsetAsync(keep64, 0, (nsm + 1) * sizeof(uint64_t), ctx->stream));
    CUSCI_CUDA(ctx, cudaMemcpy2DAsync(keep64, sizeof(uint64_t), keep, sizeof(uint32_t), sizeof(uint32_t), nsm,
                                      cudaMemcpyDeviceToDevice, ctx->stream));
    CUSCI_TRY(scan_exclusive_u64(ctx, keep64, rank, nsm + 1, nullptr));
    const uint64_t nsp = (nbg + CopyCfg<W>::SPAN - 1) / CopyCfg<W>::SPAN;
    uint64_t* cb;
    CUSCI_TRY(s.get_t(nsp + 1, &cb));
    CUSCI_LAUNCH(ctx, PT_MERGE_SPLIT, sparse_bounds_kernel<W><<<(unsigned)((nsp + 1 + 255) / 256), 256, 0, ctx->stream>>>(pos, nsm, nbg, nsp, cb));
    const unsigned bg = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nsp + 7) / 8, (uint64_t)ctx->num_sms * 8));
    CUSCI_LAUNCH(ctx, PT_MERGE_TILE, sparse_copy_kernel<W><<<bg, 256, 0, ctx->stream>>>(big, nbg, pos, rank, cb, dst, (u_small || trusted) ? nullptr : bad));
    CUSCI_LAUNCH(ctx, PT_MERGE_TILE, sparse_place_kernel<W><<<cg, 256, 0, ctx->stream>>>(small, nsm, pos, keep, rank, dst, u_small ? (uint64_t*)insp : nullptr));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, rank + nsm, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CUSCI_CUDA(ctx, cudaMemcpyAsync((char*)ctx->host_pinned + 16, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    uint64_t nin;
    memcpy(&nin, ctx->host_pinned, sizeof(uint64_t));
    h[0] = nbg + nin;
    h[1] = u_small ? nin : nU - (nS - nin);
    if (*(int*)((char*)ctx->host_pinned + 16)) {
      for (int b = 0; b < 2; b++)
        if (grown[b]) cudaFreeAsync(grown[b], ctx->stream);
      if (insp) out_free(ctx, insp);
      return set_error(ctx, CUSCI_E_INVALID_ARG, "merge_space: new_keys must be sorted in the pool (hash) order and unique");
    }
  } else {
    CUSCI_LAUNCH(ctx, PT_MERGE_SPLIT, merge_split_kernel<W><<<(unsigned)((ntiles + 1 + 255) / 256), 256, 0, ctx->stream>>>(S, nS, U, nU, ntiles, split));
    int mper = 1;
    CUSCI_TRY(kernel_setup(ctx, (const void*)merge_tile_kernel<W>, kMergeThreads, MergeCfg<W>::SMEM, &mper));
    // persistent grid whose CTAs must all be resident (the static tile order's
    // decoupled look-back waits on predecessors): a COOPERATIVE launch, which
    // the runtime refuses rather than under-schedules; when fewer SMs are
    // available (MPS limits, green contexts) the grid is halved until it fits
    unsigned mgrid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ntiles, (uint64_t)ctx->num_sms * mper));
    const int chk = trusted ? 0 : 1;
    for (;;) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(mgrid);
      cfg.blockDim = dim3(kMergeThreads);
      cfg.dynamicSmemBytes = MergeCfg<W>::SMEM;
      cfg.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e;
      {
        Prof pf_(ctx, PT_MERGE_TILE);
        e = cudaLaunchKernelEx(&cfg, merge_tile_kernel<W>, S, nS, U, nU, (const uint64_t*)split, ntiles, status, bad, dst,
                               (uint64_t*)insp, chk);
      }
      if (e == cudaErrorCooperativeLaunchTooLarge && mgrid > 1) {
        cudaGetLastError();
        mgrid = (mgrid + 1) / 2;
        continue;
      }
      CUSCI_CUDA(ctx, e);
      CUSCI_LAUNCH_CHECK(ctx);
      break;
    }
    // totals = the last tile's inclusive counts; plus the input check flag
    CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, status + 2 * (ntiles - 1), 2 * sizeof(uint64_t),
                                    cudaMemcpyDeviceToHost, ctx->stream));
    CUSCI_CUDA(ctx, cudaMemcpyAsync((char*)ctx->host_pinned + 16, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    memcpy(h, ctx->host_pinned, 2 * sizeof(uint64_t));
    const int badflag = *(int*)((char*)ctx->host_pinned + 16);
    if (badflag) {
      for (int b = 0; b < 2; b++)
        if (grown[b]) cudaFreeAsync(grown[b], ctx->stream);
      if (insp) out_free(ctx, insp);
      return set_error(ctx, CUSCI_E_INVALID_ARG, "merge_space: new_keys must be sorted in the pool (hash) order and unique");
    }
  }
  const uint64_t n_new = h[0] & kMVal, n_ins = h[1] & kMVal;
  if (grown[0]) {
    cudaFreeAsync(pool->buf[0], ctx->stream);
    cudaFreeAsync(pool->buf[1], ctx->stream);
    pool->buf[0] = grown[0];
    pool->buf[1] = grown[1];
    pool->cap = ncap;
    pool->cur = 0;
  } else {
    pool->cur = 1 - pool->cur;
  }
  pool->count = n_new;
  if (inserted) {
    inserted->keys = (uint64_t*)insp;
    inserted->count = n_ins;
  }
  return CUSCI_OK;
}

}  // namespace
}  // namespace cusci

using namespace cusci;

extern "C" int merge_space(cusci_ctx* ctx, cusci_pool* space, const uint64_t* new_keys, uint64_t n_new,
                           cusci_keys* inserted) {
  if (!ctx || !space) return CUSCI_E_INVALID_ARG;
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  if (space->ctx != ctx) return set_error(ctx, CUSCI_E_INVALID_ARG, "pool belongs to another context");
  if (n_new && !new_keys) return set_error(ctx, CUSCI_E_INVALID_ARG, "new_keys is NULL");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  return space->sp.words == 1 ? merge_impl<1>(ctx, space, new_keys, n_new, inserted, false)
                              : merge_impl<2>(ctx, space, new_keys, n_new, inserted, false);
}

extern "C" int cusci_pool_merge(cusci_ctx* ctx, cusci_pool* space, const cusci_pool* src, cusci_keys* inserted) {
  if (!ctx || !space || !src) return CUSCI_E_INVALID_ARG;
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  if (space->ctx != ctx || src->ctx != ctx) return set_error(ctx, CUSCI_E_INVALID_ARG, "pool belongs to another context");
  if (src->sp.words != space->sp.words || src->sp.m != space->sp.m)
    return set_error(ctx, CUSCI_E_INVALID_ARG, "pools of different spaces");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  const uint64_t* U = src->buf[src->cur];
  return space->sp.words == 1 ? merge_impl<1>(ctx, space, U, src->count, inserted, true)
                              : merge_impl<2>(ctx, space, U, src->count, inserted, true);
}
