// gen_coupled: excitation enumerator + Slater-Condon evaluator + screening +
// compaction (Alg. 1 :514-554, Sec 4.2.2
// :561-571; Eq. 4 :261-265).
//
// B200 design: a persistent grid of warps pulls work
// units (parent, contiguous range of excitation rows) from a global counter.
// Per unit one warp
//   a1  loads the parent (one 8/16-byte broadcast load), builds its sorted
//       occupied list in shared memory with ballots + popc, and the prefix-
//       parity mask PP (bit t = parity of the occupied orbitals below t);
//   a2  row 0 = all singles of the parent, flattened across occupied
//       orbitals (a warp scan over the per-orbital candidate counts + a
//       shuffle binary search gives each lane its (p, a)); rows 1.. = the
//       occupied pairs (occ[x] < occ[y]), each read from the prescreened CSR
//       pair table (a0), 32 entries (16 B each, one 128-bit load) per step;
//   a3  target key = (parent ^ p ^ q) ^ abmask;
//   a4  phase of sequential singles p->a, q->b in closed form:
//         parity = (x + y + 1) ^ M(a) ^ M(b),  M = PP ^ above(p) ^ above(q)
//       (singles: parity = x ^ PP(a) ^ [a > p]) -- one popc per record;
//   a5  H = +-v from the table (doubles) or the sequential sum over occ(i)\p
//       of the [K][P][A] tables (singles, same order as the definition);
//   a6  keeps |H| > eps (doubles: folded into the table at build time);
//   a7  survivors are compacted with ballot/popc into a per-warp staging
//       buffer in shared memory; when it is nearly full the warp reserves
//       exactly its fill with ONE atomicAdd and copies it out with fully
//       coalesced stores (the paper's "one atomicAdd per block", as a
//       per-384-record flush).  No count pass, no gaps; record order is
//       unspecified (reading r6).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.cuh"

namespace cusci {
namespace {

constexpr int kGenThreads = 256;
constexpr int kGenWarps = kGenThreads / 32;
constexpr unsigned long long kNoError = ~0ull;
#ifndef CUSCI_GEN_CHUNKS
#define CUSCI_GEN_CHUNKS 4  // (macros: A/B variants, tools/build_variant.py)
#endif
#ifndef CUSCI_GEN_MINB
#define CUSCI_GEN_MINB 4
#endif
#ifndef CUSCI_GEN_IFLOAD
#define CUSCI_GEN_IFLOAD 1
#endif
#ifndef CUSCI_GEN_STAGE1
#define CUSCI_GEN_STAGE1 256
#endif
constexpr int kChunks = CUSCI_GEN_CHUNKS;  // 32-entry chunks (128-bit loads per lane) in flight per step

template <int W> struct GenCfg {
  static constexpr int STAGE = W == 1 ? CUSCI_GEN_STAGE1 : 192;  // staged records per warp (4 CTAs/SM)
  static constexpr size_t BYTES_PER_REC = (W == 1 ? 16 : 24) + 1;
  static constexpr size_t SMEM = (size_t)kGenWarps * STAGE * BYTES_PER_REC;
};

struct GenArgs {
  const uint64_t* parents;
  uint64_t n_parents;
  int m, n_elec, K;
  uint32_t units_per_parent;
  uint32_t rows_per_parent;  // 1 (all singles) + n(n-1)/2 pair rows
  uint64_t n_units;
  const uint32_t* rowptr;
  const PairEnt* ent;
  const uint32_t* srowptr;
  const uint8_t* sa;
  const double* topp;
  const double* tsame;
  const double* h;
  double eps;
  uint64_t* keys;
  double* hij;
  uint32_t* src;
  int8_t* phase;
  uint64_t capacity;
  unsigned long long* counter;  // [0] records, [1] unit work counter, [2] first bad parent
  int count_only;
  uint32_t src_base;  // added to every src (streamed mini-batches write global parent indices)
};

// ---- bit helpers on W-word keys
__device__ __forceinline__ bool occ_bit(const KeyT<1>& k, int t) { return (k.w0 >> t) & 1ull; }
__device__ __forceinline__ bool occ_bit(const KeyT<2>& k, int t) {
  return t < 64 ? ((k.w0 >> t) & 1ull) : ((k.w1 >> (t - 64)) & 1ull);
}
__device__ __forceinline__ KeyT<1> bitk1(int t) { return KeyT<1>{1ull << t}; }
__device__ __forceinline__ KeyT<2> bitk2(int t) {
  return t < 64 ? KeyT<2>{1ull << t, 0ull} : KeyT<2>{0ull, 1ull << (t - 64)};
}
template <int W> __device__ __forceinline__ KeyT<W> bitk(int t);
template <> __device__ __forceinline__ KeyT<1> bitk<1>(int t) { return bitk1(t); }
template <> __device__ __forceinline__ KeyT<2> bitk<2>(int t) { return bitk2(t); }
__device__ __forceinline__ KeyT<1> kxor(const KeyT<1>& a, const KeyT<1>& b) { return KeyT<1>{a.w0 ^ b.w0}; }
__device__ __forceinline__ KeyT<2> kxor(const KeyT<2>& a, const KeyT<2>& b) { return KeyT<2>{a.w0 ^ b.w0, a.w1 ^ b.w1}; }
__device__ __forceinline__ bool kdisjoint(const KeyT<1>& a, const KeyT<1>& b) { return (a.w0 & b.w0) == 0; }
__device__ __forceinline__ bool kdisjoint(const KeyT<2>& a, const KeyT<2>& b) {
  return ((a.w0 & b.w0) | (a.w1 & b.w1)) == 0;
}
__device__ __forceinline__ uint32_t kparity_and(const KeyT<1>& a, const KeyT<1>& b) {
  // parity of popc(a & b) = parity of popc of the two halves xor-folded (two LOP3 + one POPC)
  const uint64_t x = a.w0 & b.w0;
  return __popc((uint32_t)x ^ (uint32_t)(x >> 32)) & 1u;
}
__device__ __forceinline__ uint32_t kparity_and(const KeyT<2>& a, const KeyT<2>& b) {
  return (__popcll(a.w0 & b.w0) ^ __popcll(a.w1 & b.w1)) & 1u;
}
// bits strictly above t
template <int W> __device__ __forceinline__ KeyT<W> abovek(int t);
template <> __device__ __forceinline__ KeyT<1> abovek<1>(int t) { return KeyT<1>{t >= 63 ? 0ull : (~0ull << (t + 1))}; }
template <> __device__ __forceinline__ KeyT<2> abovek<2>(int t) {
  if (t < 63) return KeyT<2>{~0ull << (t + 1), ~0ull};
  if (t == 63) return KeyT<2>{0ull, ~0ull};
  return KeyT<2>{0ull, t >= 127 ? 0ull : (~0ull << (t - 63))};
}
// exclusive prefix parity: bit t = parity of popc(k & bits below t)
__device__ __forceinline__ uint64_t prefix_xor_incl(uint64_t x) {
  x ^= x << 1;
  x ^= x << 2;
  x ^= x << 4;
  x ^= x << 8;
  x ^= x << 16;
  x ^= x << 32;
  return x;
}
__device__ __forceinline__ KeyT<1> prefix_parity(const KeyT<1>& k) { return KeyT<1>{prefix_xor_incl(k.w0) << 1}; }
__device__ __forceinline__ KeyT<2> prefix_parity(const KeyT<2>& k) {
  const uint64_t lo = prefix_xor_incl(k.w0);
  const uint64_t carry = (lo >> 63) ? ~0ull : 0ull;  // parity of the whole of word 0
  const uint64_t hi = prefix_xor_incl(k.w1);
  return KeyT<2>{lo << 1, (hi << 1) ^ carry};
}
// table entry -> abmask: stored (W = 1) or built from (a, b) (W = 2)
__device__ __forceinline__ void ent_mask(uint64_t x, KeyT<1>& m) { m.w0 = x; }
__device__ __forceinline__ void ent_mask(uint64_t x, KeyT<2>& m) {
  const KeyT<2> ma = bitk2((int)(x & 0xff)), mb = bitk2((int)((x >> 8) & 0xff));
  m.w0 = ma.w0 | mb.w0;
  m.w1 = ma.w1 | mb.w1;
}

template <int W>
__global__ void validate_kernel(const uint64_t* __restrict__ parents, uint64_t n, int m, int na, int nb,
                                unsigned long long* __restrict__ counter) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += stride) {
    const KeyT<W> k = load_key<W>(parents, s);
    constexpr uint64_t EVEN = 0x5555555555555555ull;
    int ca = __popcll(k.w0 & EVEN), cb = __popcll(k.w0 & ~EVEN);
    bool hi_bad;
    if constexpr (W == 2) {
      ca += __popcll(k.w1 & EVEN);
      cb += __popcll(k.w1 & ~EVEN);
      hi_bad = m <= 64 ? (k.w1 != 0 || (m < 64 && (k.w0 >> m))) : (m < 128 && (k.w1 >> (m - 64)));
    } else {
      hi_bad = m < 64 && (k.w0 >> m);
    }
    if (hi_bad || ca != na || cb != nb) atomicMin(&counter[2], (unsigned long long)s);
  }
}

// per-warp staging buffer in shared memory: kh = (key, H) interleaved (one
// 16-byte store per record at W=1), phase (only if requested).  The source
// index is not staged per record: the records of one work unit are
// contiguous in the stage, so a short list of runs (start, src) recovers it.
template <int W> struct StRec;
template <> struct __align__(16) StRec<1> {
  uint64_t k0;
  double h;
};
template <> struct __align__(8) StRec<2> {
  uint64_t k0, k1;
  double h;
};
constexpr int kRuns = 8;  // source runs per stage
template <int W>
struct Stage {
  StRec<W>* kh;
  int8_t* ph;
  uint32_t* run;  // [2 kRuns]: run start, run src
  uint32_t n;     // warp-uniform fill
  uint32_t nrun;  // warp-uniform
  uint32_t src;   // current unit's source index
};
__device__ __forceinline__ void st_put(StRec<1>& r, const KeyT<1>& k, double h) {
  *reinterpret_cast<ulonglong2*>(&r) = make_ulonglong2(k.w0, (unsigned long long)__double_as_longlong(h));
}
__device__ __forceinline__ void st_put(StRec<2>& r, const KeyT<2>& k, double h) {
  r.k0 = k.w0;
  r.k1 = k.w1;
  r.h = h;
}
__device__ __forceinline__ KeyT<1> st_key(const StRec<1>& r) { return KeyT<1>{r.k0}; }
__device__ __forceinline__ KeyT<2> st_key(const StRec<2>& r) { return KeyT<2>{r.k0, r.k1}; }

template <int W, int MODE>
__device__ __forceinline__ void stage_flush(const GenArgs& a, Stage<W>& st) {
  __syncwarp();
  if (st.n) {
    const unsigned lane = lane_id();
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&a.counter[0], (unsigned long long)st.n);
    base = __shfl_sync(kFull, base, 0);
    if (base + st.n <= a.capacity) {
      // lane pointers advanced by 32 records per step (no 64-bit index arithmetic per record)
      uint64_t* kp = a.keys + (base + lane) * W;
      double* hp = a.hij + base + lane;
      for (uint32_t i = lane; i < st.n; i += 32, kp += 32 * W, hp += 32) {
        const StRec<W> r = st.kh[i];
        store_key<W>(kp, 0, st_key(r));
        *hp = r.h;
      }
      if (a.src) {  // each source run is a contiguous range of the stage
        for (uint32_t j = 0; j < st.nrun; j++) {
          const uint32_t r0 = st.run[j], r1 = j + 1 < st.nrun ? st.run[j + 1] : st.n, sv = st.run[kRuns + j] + a.src_base;
          if (W == 1 && (reinterpret_cast<uintptr_t>(a.src) & 7u) == 0) {
            // two src per lane (8-byte stores) from an even global index; an odd
            // head / tail alone (at W = 2 the extra registers cost more than they save)
            uint32_t i0 = r0;
            if (((base + r0) & 1ull) && r0 < r1) {
              if (lane == 0) a.src[base + r0] = sv;
              i0++;
            }
            uint2* s2 = reinterpret_cast<uint2*>(a.src + base + i0);
            const uint32_t np = (r1 - i0) >> 1;
            for (uint32_t q = lane; q < np; q += 32) s2[q] = make_uint2(sv, sv);
            if (((r1 - i0) & 1u) && lane == 0) a.src[base + r1 - 1] = sv;
          } else {
            for (uint32_t i = r0 + lane; i < r1; i += 32) a.src[base + i] = sv;
          }
        }
      }
      if (MODE == 2)
        for (uint32_t i = lane; i < st.n; i += 32) a.phase[base + i] = st.ph[i];
    }
    __syncwarp();
  }
  st.n = 0;
  st.nrun = 1;  // the current unit continues as run 0
  if (lane_id() == 0) {
    st.run[0] = 0;
    st.run[kRuns] = st.src;
  }
  __syncwarp();
}

// a new work unit (source index src) starts emitting
template <int W, int MODE>
__device__ __forceinline__ void stage_unit(const GenArgs& a, Stage<W>& st, uint32_t src) {
  if (st.nrun == kRuns) stage_flush<W, MODE>(a, st);
  st.src = src;
  if (lane_id() == 0) {
    st.run[st.nrun] = st.n;
    st.run[kRuns + st.nrun] = src;
  }
  st.nrun++;
}

// append the lanes' survivors (ballot `bal`) to the stage
template <int W, int MODE>
__device__ __forceinline__ void stage_put(const GenArgs& a, Stage<W>& st, unsigned bal, bool keep, const KeyT<W>& key,
                                          double H, uint32_t par) {
  if (st.n + 32 > (uint32_t)GenCfg<W>::STAGE) stage_flush<W, MODE>(a, st);
  if (keep) {
    const uint32_t i = st.n + __popc(bal & lanemask_lt());
    st_put(st.kh[i], key, H);
    if (MODE == 2) st.ph[i] = par ? -1 : 1;
  }
  st.n += __popc(bal);
}

__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v) {
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, v, o);
    if ((int)lane_id() >= o) v += t;
  }
  return v;
}

// row 0: all singles of parent s (flattened over occupied orbitals)
template <int W, int MODE>
__device__ __forceinline__ uint32_t do_singles(const GenArgs& a, const KeyT<W>& par, const KeyT<W>& PP,
                                               const uint8_t* occ, uint32_t s, Stage<W>& st) {
  constexpr bool emit = MODE != 0;
  const unsigned lane = lane_id();
  const int n = a.n_elec;
  uint32_t total_kept = 0;
  for (int xc = 0; xc < n; xc += 32) {
    const int xl = xc + (int)lane;
    int p = 0;
    uint32_t c0 = 0, c = 0;
    if (xl < n) {
      p = occ[xl];
      c0 = __ldg(a.srowptr + p);
      c = __ldg(a.srowptr + p + 1) - c0;
    }
    const uint32_t incl = warp_incl_scan_u32(c);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    for (uint32_t f0 = 0; f0 < total; f0 += 32) {
      const uint32_t f = f0 + lane;
      // owner lane L of candidate f = number of lanes whose inclusive count <= f
      int L = 0;
#pragma unroll
      for (int b = 16; b >= 1; b >>= 1) {
        const uint32_t v = __shfl_sync(kFull, incl, L + b - 1);
        if (v <= f) L += b;
      }
      L = min(L, 31);
      const int pL = __shfl_sync(kFull, p, L);
      const uint32_t c0L = __shfl_sync(kFull, c0, L);
      const uint32_t exL = __shfl_sync(kFull, incl, L) - __shfl_sync(kFull, c, L);
      bool keep = false;
      double H = 0.0;
      uint32_t ph = 0;
      int t = pL;
      if (f < total) {
        t = __ldg(a.sa + c0L + (f - exL));
        if (!occ_bit(par, t)) {
          const int P = pL >> 1, A = t >> 1;
          double v = __ldg(a.h + P * a.K + A);
          for (int xx = 0; xx < n; xx++) {
            const int kk = occ[xx];
            if (kk == pL) continue;
            const size_t o = ((size_t)(kk >> 1) * a.K + P) * a.K + A;
            const double tv = ((kk & 1) == (pL & 1)) ? __ldg(a.tsame + o) : __ldg(a.topp + o);
            v = __dadd_rn(v, tv);
          }
          // parity = c(p) + c(a) + [a > p], c(p) = index of p in occ
          ph = (uint32_t)((xc + L) & 1) ^ (uint32_t)occ_bit(PP, t) ^ (uint32_t)(t > pL);
          H = ph ? -v : v;
          keep = fabs(H) > a.eps;
        }
      }
      const unsigned bal = __ballot_sync(kFull, keep);
      if (emit) {
        const KeyT<W> j = kxor(par, kxor(bitk<W>(pL), bitk<W>(t)));
        stage_put<W, MODE>(a, st, bal, keep, j, H, ph);
      } else {
        total_kept += __popc(bal);
      }
    }
  }
  return total_kept;
}

// Pair rows [r0, r1) (1-based over the occupied pairs x < y) of the parent,
// processed in batches of <= kRowBatch rows.  Per batch the warp first sets up
// one descriptor per row lane-parallel (table start, phase constant, target
// base and phase mask of the row, start in the batch's entry stream), so the
// serial row loop only reads one broadcast descriptor per row.
constexpr int kRowBatch = 96;  // rows per descriptor batch (N2-like parents: one batch)
template <int W> struct RowInfo;
template <> struct __align__(8) RowInfo<1> {
  uint32_t rb;   // table index of the row's first entry | phase constant << 31
  uint32_t len;  // entries in the row
  uint64_t base, M;
};
template <> struct __align__(16) RowInfo<2> {
  uint32_t rb, len;
  uint32_t pq;  // p | q << 8
  uint32_t pad;
};

// the row loop reads its descriptors through a pinned 32-bit shared address
// (an asm result cannot be rematerialised: without the pin the compiler
// recomputes the warp's descriptor base from %tid and the CTA window every row)
__device__ __forceinline__ uint32_t pin_u32(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ RowInfo<1> ld_rowinfo(uint32_t sa, const RowInfo<1>*) {
  RowInfo<1> r;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.rb), "=r"(r.len) : "r"(sa));
  asm volatile("ld.shared.u64 %0, [%1+8];" : "=l"(r.base) : "r"(sa));
  asm volatile("ld.shared.u64 %0, [%1+16];" : "=l"(r.M) : "r"(sa));
  return r;
}
__device__ __forceinline__ RowInfo<2> ld_rowinfo(uint32_t sa, const RowInfo<2>*) {
  RowInfo<2> r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.rb), "=r"(r.len), "=r"(r.pq), "=r"(r.pad) : "r"(sa));
  return r;
}

template <int W, int MODE>
__device__ __forceinline__ uint32_t do_pairs(const GenArgs& a, const KeyT<W>& par, const KeyT<W>& PP,
                                             const uint8_t* occ, RowInfo<W>* ri, uint32_t r0, uint32_t r1,
                                             Stage<W>& st) {
  const unsigned lane = lane_id();
  const int n = a.n_elec;
  uint32_t total_kept = 0;
  const ulonglong2* ent = reinterpret_cast<const ulonglong2*>(a.ent);
  for (uint32_t b0 = r0; b0 < r1; b0 += kRowBatch) {
    const uint32_t nr = min((uint32_t)kRowBatch, r1 - b0);
    // ---- row descriptors (lane-parallel)
    for (uint32_t j0 = 0; j0 < nr; j0 += 32) {
      const uint32_t j = j0 + lane;
      if (j < nr) {
        uint32_t k = b0 + j - 1;  // pair index -> (x, y), x < y
        int x = 0;
        while (k >= (uint32_t)(n - 1 - x)) {
          k -= (uint32_t)(n - 1 - x);
          x++;
        }
        const int y = x + 1 + (int)k;
        const int p = occ[x], q = occ[y];
        const uint32_t row = (uint32_t)q * (q - 1) / 2 + p;
        const uint32_t e0 = __ldg(a.rowptr + row);
        RowInfo<W> r;
        r.len = __ldg(a.rowptr + row + 1) - e0;
        r.rb = e0 | ((uint32_t)((x + y + 1) & 1) << 31);
        if constexpr (W == 1) {
          r.base = par.w0 ^ (1ull << p) ^ (1ull << q);
          r.M = PP.w0 ^ (p >= 63 ? 0ull : (~0ull << (p + 1))) ^ (q >= 63 ? 0ull : (~0ull << (q + 1)));
        } else {
          r.pq = (uint32_t)p | ((uint32_t)q << 8);
          r.pad = 0;
        }
        ri[j] = r;
      }
    }
    __syncwarp();
    // ---- rows: warp-uniform descriptor (broadcast loads), kChunks 32-entry
    // chunks (128-bit loads) in flight per step
    const uint32_t ri_sa = pin_u32((uint32_t)__cvta_generic_to_shared(ri));
    for (uint32_t j = 0; j < nr; j++) {
      const RowInfo<W> R = ld_rowinfo(ri_sa + j * (uint32_t)sizeof(RowInfo<W>), ri);
      const uint32_t len = R.len;
      const ulonglong2* rowp = ent + (R.rb & 0x7fffffffu);
      KeyT<W> base, M;
      if constexpr (W == 1) {
        base = KeyT<W>{R.base};
        M = KeyT<W>{R.M};
      } else {
        const int p = (int)(R.pq & 0xff), q = (int)(R.pq >> 8);
        base = kxor(par, kxor(bitk<W>(p), bitk<W>(q)));
        M = kxor(PP, kxor(abovek<W>(p), abovek<W>(q)));
      }
      const uint32_t rc = R.rb >> 31;
      for (uint32_t e = 0; e < len; e += 32 * kChunks) {
        ulonglong2 raw[kChunks];
#pragma unroll
        for (int u = 0; u < kChunks; u++) {
          const uint32_t i = e + 32 * u + lane;
#if CUSCI_GEN_IFLOAD
          if (i < len) raw[u] = __ldg(rowp + i);  // lanes past the row are masked out of `keep`
#else
          raw[u] = i < len ? __ldg(rowp + i) : make_ulonglong2(~0ull, 0ull);
#endif
        }
#pragma unroll
        for (int u = 0; u < kChunks; u++) {
          if (e + 32 * u >= len) break;
          KeyT<W> abm{};
          ent_mask(raw[u].x, abm);
          const bool keep = e + 32 * u + lane < len && kdisjoint(par, abm);
          const unsigned bal = __ballot_sync(kFull, keep);
          if (MODE != 0) {
            const uint32_t ph = rc ^ kparity_and(M, abm);
            // H = +-v: flip the sign bit (exact)
            const double H = __longlong_as_double((long long)(raw[u].y ^ ((unsigned long long)ph << 63)));
            stage_put<W, MODE>(a, st, bal, keep, kxor(base, abm), H, ph);
          } else {
            total_kept += __popc(bal);
          }
        }
      }
    }
    __syncwarp();
  }
  return total_kept;
}

template <int W, int MODE>
__global__ void __launch_bounds__(kGenThreads, CUSCI_GEN_MINB) gen_kernel(const GenArgs a) {
  extern __shared__ __align__(16) unsigned char gsm[];
  __shared__ uint8_t occ_s[kGenWarps][128];
  __shared__ RowInfo<W> ri_s[kGenWarps][kRowBatch];       // pair-row descriptors of the current batch
  __shared__ uint32_t run_s[kGenWarps][2 * kRuns];          // stage source runs
  __shared__ unsigned long long unit_s[kGenWarps];
  if (a.counter[2] != kNoError) return;  // invalid parent: write nothing
  const int w = threadIdx.x >> 5;
  const unsigned lane = lane_id();
  constexpr int S = GenCfg<W>::STAGE;
  constexpr bool emit = MODE != 0;
  Stage<W> st;
  st.kh = reinterpret_cast<StRec<W>*>(gsm) + (size_t)w * S;
  st.ph = reinterpret_cast<int8_t*>(gsm + (size_t)kGenWarps * S * sizeof(StRec<W>)) + (size_t)w * S;
  st.run = run_s[w];
  st.n = 0;
  st.nrun = 0;
  st.src = 0;
  uint8_t* occ = occ_s[w];
  for (;;) {
    if (lane == 0) unit_s[w] = atomicAdd(&a.counter[1], 1ull);
    __syncwarp();
    const uint64_t u = unit_s[w];
    __syncwarp();
    if (u >= a.n_units) break;
    const uint64_t s = u / a.units_per_parent;
    const uint32_t sub = (uint32_t)(u % a.units_per_parent);
    const uint32_t R = a.rows_per_parent;
    const uint32_t r0 = (uint32_t)(((uint64_t)sub * R) / a.units_per_parent);
    const uint32_t r1 = (uint32_t)(((uint64_t)(sub + 1) * R) / a.units_per_parent);
    const KeyT<W> par = load_key<W>(a.parents, s);
    // a1: occupied list (ascending) via ballots
    uint32_t nocc = 0;
#pragma unroll
    for (int c = 0; c < 2 * W; c++) {
      const int t = c * 32 + (int)lane;
      const bool b = t < a.m && occ_bit(par, t);
      const unsigned bal = __ballot_sync(kFull, b);
      if (b) occ[nocc + __popc(bal & lanemask_lt())] = (uint8_t)t;
      nocc += __popc(bal);
    }
    const KeyT<W> PP = prefix_parity(par);
    __syncwarp();
    if (emit) stage_unit<W, MODE>(a, st, (uint32_t)s);
    uint32_t cnt = 0;
    if (r0 == 0 && r1 > 0) cnt += do_singles<W, MODE>(a, par, PP, occ, (uint32_t)s, st);
    const uint32_t pr0 = r0 == 0 ? 1 : r0;
    if (r1 > pr0) cnt += do_pairs<W, MODE>(a, par, PP, occ, ri_s[w], pr0, r1, st);
    if (!emit && lane == 0 && cnt) atomicAdd(&a.counter[0], (unsigned long long)cnt);
    __syncwarp();
  }
  if (emit) stage_flush<W, MODE>(a, st);
}

int gen_impl(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
             const cusci_integrals* ints, double threshold, cusci_records* out, bool count_only, uint64_t* count_out,
             uint32_t src_base = 0) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  CUSCI_TRY(check_space(ctx, sp));
  if (!ints || !ints->h || !ints->eri) return set_error(ctx, CUSCI_E_INVALID_ARG, "integrals are NULL");
  if (ints->n_spatial * 2 != sp->m)
    return set_error(ctx, CUSCI_E_INVALID_ARG, "n_spatial=%d but m=%d", ints->n_spatial, sp->m);
  if (!(threshold >= 0.0)) return set_error(ctx, CUSCI_E_INVALID_ARG, "threshold must be >= 0 (got %g)", threshold);
  if (n_parents && !parents) return set_error(ctx, CUSCI_E_INVALID_ARG, "parents is NULL");
  if (n_parents >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "n_parents must be < 2^32");
  if (!count_only && (!out || ((!out->keys || !out->hij) && out->capacity)))
    return set_error(ctx, CUSCI_E_INVALID_ARG, "output record buffers are NULL");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  if (!count_only) out->count = 0;
  if (n_parents == 0) {
    if (count_out) *count_out = 0;
    return CUSCI_OK;
  }
  CUSCI_TRY(prep_build(ctx, sp, ints, threshold));
  const int W = sp->words;
  const int n = sp->n_alpha + sp->n_beta;
  Scratch s(ctx);
  unsigned long long* counter;
  CUSCI_TRY(s.get_t(4, &counter));
  unsigned long long init[4] = {0, 0, kNoError, 0};
  memcpy(ctx->host_pinned, init, sizeof(init));
  CUSCI_CUDA(ctx, cudaMemcpyAsync(counter, ctx->host_pinned, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
  {
    const unsigned blocks = (unsigned)std::min<uint64_t>((n_parents + 255) / 256, (uint64_t)ctx->num_sms * 8);
    if (W == 1)
      CUSCI_LAUNCH(ctx, PT_VALIDATE, validate_kernel<1><<<blocks, 256, 0, ctx->stream>>>(parents, n_parents, sp->m, sp->n_alpha, sp->n_beta, counter));
    else
      CUSCI_LAUNCH(ctx, PT_VALIDATE, validate_kernel<2><<<blocks, 256, 0, ctx->stream>>>(parents, n_parents, sp->m, sp->n_alpha, sp->n_beta, counter));
  }
  GenArgs a{};
  a.parents = parents;
  a.n_parents = n_parents;
  a.m = sp->m;
  a.n_elec = n;
  a.K = ints->n_spatial;
  a.rows_per_parent = (uint32_t)(1 + n * (n - 1) / 2);
  const uint64_t target_units = (uint64_t)ctx->num_sms * 16 * 4;
  uint64_t U = (target_units + n_parents - 1) / n_parents;
  if (U < 1) U = 1;
  if (U > a.rows_per_parent) U = a.rows_per_parent;
  a.units_per_parent = (uint32_t)U;
  a.n_units = n_parents * U;
  const Prep& pr = ctx->prep;
  a.rowptr = pr.rowptr;
  a.ent = pr.ent;
  a.srowptr = pr.srowptr;
  a.sa = pr.sa;
  a.topp = pr.topp;
  a.tsame = pr.tsame;
  a.h = ints->h;
  a.eps = threshold;
  if (!count_only) {
    a.keys = out->keys;
    a.hij = out->hij;
    a.src = out->src;
    a.phase = out->phase;
    a.capacity = out->capacity;
  }
  a.counter = counter;
  a.count_only = count_only ? 1 : 0;
  a.src_base = src_base;
  const int mode = count_only ? 0 : (out->phase ? 2 : 1);
  const size_t smem = mode == 0 ? 0 : (W == 1 ? GenCfg<1>::SMEM : GenCfg<2>::SMEM);
  void (*kern)(const GenArgs) = nullptr;
  if (W == 1) kern = mode == 0 ? gen_kernel<1, 0> : (mode == 1 ? gen_kernel<1, 1> : gen_kernel<1, 2>);
  else kern = mode == 0 ? gen_kernel<2, 0> : (mode == 1 ? gen_kernel<2, 1> : gen_kernel<2, 2>);
  int per_sm = 1;
  CUSCI_TRY(kernel_setup(ctx, (const void*)kern, kGenThreads, smem, &per_sm));
  const unsigned blocks = (unsigned)(ctx->num_sms * per_sm);
  CUSCI_LAUNCH(ctx, PT_GEN, kern<<<blocks, kGenThreads, smem, ctx->stream>>>(a));
  unsigned long long res[4];
  CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, counter, sizeof(res), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(res, ctx->host_pinned, sizeof(res));
  if (res[2] != kNoError)
    return set_error(ctx, CUSCI_E_INVALID_PARENT,
                     "parent %llu is invalid (a bit >= m=%d or spin popcounts != (%d,%d))", res[2], sp->m,
                     sp->n_alpha, sp->n_beta);
  if (count_out) *count_out = res[0];
  if (!count_only) {
    out->count = res[0];
    if (res[0] > out->capacity)
      return set_error(ctx, CUSCI_E_CAPACITY, "gen_coupled: %llu records exceed capacity %llu", res[0],
                       (unsigned long long)out->capacity);
  }
  return CUSCI_OK;
}

}  // namespace

int gen_records(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
                const cusci_integrals* ints, double threshold, cusci_records* out, uint32_t src_base) {
  return gen_impl(ctx, sp, parents, n_parents, ints, threshold, out, false, nullptr, src_base);
}
int gen_count(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
              const cusci_integrals* ints, double threshold, uint64_t* count) {
  return gen_impl(ctx, sp, parents, n_parents, ints, threshold, nullptr, true, count);
}

}  // namespace cusci

using namespace cusci;

extern "C" int gen_coupled(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
                           const cusci_integrals* ints, double threshold, cusci_records* out) {
  if (!out) return ctx ? set_error(ctx, CUSCI_E_INVALID_ARG, "out is NULL") : CUSCI_E_INVALID_ARG;
  return gen_impl(ctx, sp, parents, n_parents, ints, threshold, out, false, nullptr);
}

extern "C" int gen_coupled_count(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
                                 const cusci_integrals* ints, double threshold, uint64_t* count) {
  if (!count) return ctx ? set_error(ctx, CUSCI_E_INVALID_ARG, "count is NULL") : CUSCI_E_INVALID_ARG;
  return gen_impl(ctx, sp, parents, n_parents, ints, threshold, nullptr, true, count);
}
