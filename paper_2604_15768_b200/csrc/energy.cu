// energy_contract: Stage-3 contraction of the coupled records with amplitudes
// (SURVEY 8(f) row f1; Eq. 5 :267-270, Stage 3 :398-403, :634).
//
//   e[s] = sum over records r with src[r] = s of H[r] * psi[idx(key[r])]
//
// B200 design (reading r14):
//   reverse index  the unique set is sorted in the hash order pi (reading
//                  r13) and pi is uniform, so its (key, psi) pairs are laid
//                  out in an ORDERED direct-mapped table (element i at slot
//                  max(home_i, slot_{i-1} + 1), home = top k bits of hi,
//                  2^k >= 2 n_space; built by a max-scan, no atomics): a
//                  record probes from its home and almost always resolves in
//                  one 32-byte sector ("just in time", nothing materialised
//                  per record);
//   reduction      each product p = H * psi (IEEE fp64) is rounded half-to-even
//                  to the grid 2^-80 and accumulated EXACTLY as a 128-bit
//                  integer: a warp first sums the runs of equal src among its
//                  lanes (gen_coupled writes a parent's records in runs), then
//                  the run totals go into per-parent 4 x 32-bit limb
//                  accumulators with 64-bit atomics.  Integer addition is
//                  associative, so the result is independent of record order
//                  and of the launch configuration; e[s] = the exact sum
//                  rounded once to fp64.
#include <algorithm>
#include <climits>

#include "internal.cuh"

namespace cusci {
namespace {

constexpr int kET = 256;

template <int W>
__device__ __forceinline__ bool pi_less(const KeyT<W>& a, const KeyT<W>& b) { return pi_lt(a, b); }

// (key, psi) side by side: one random sector serves the match and the amplitude
template <int W> struct KPsi;
template <> struct __align__(16) KPsi<1> {
  uint64_t k0;
  double psi;
};
template <> struct __align__(32) KPsi<2> {
  uint64_t k0, k1;
  double psi;
  double pad;
};
template <int W> __device__ __forceinline__ bool kp_eq(const KPsi<W>& r, const KeyT<W>& k);
template <> __device__ __forceinline__ bool kp_eq<1>(const KPsi<1>& r, const KeyT<1>& k) { return r.k0 == k.w0; }
template <> __device__ __forceinline__ bool kp_eq<2>(const KPsi<2>& r, const KeyT<2>& k) {
  return r.k0 == k.w0 && r.k1 == k.w1;
}


// ---- ordered direct-mapped (key, psi) table: the space is sorted in the hash
// order, so placing element i at p_i = max(h_i, p_{i-1} + 1) (h = top k bits of
// hi, 2^k >= 2 n) keeps homes monotone: a record probes from its home and
// almost always resolves in one 32-byte sector.  p_i = i + max_{j<=i}(h_j - j):
// a max-scan, done as chunk maxima -> one-block exclusive prefix -> in-chunk scan.
constexpr uint32_t kPCh = 4096;  // elements per chunk
template <int W>
__device__ __forceinline__ long long home_minus_i(const uint64_t* space, uint64_t i, int k) {
  const uint64_t h = to_pi(load_key<W>(space, i)).w0 >> (64 - k);
  return (long long)h - (long long)i;
}
template <int W>
__global__ void __launch_bounds__(kET) chunk_max_kernel(const uint64_t* __restrict__ space, uint64_t n, int k,
                                                       long long* __restrict__ cmax) {
  __shared__ long long red[kET / 32];
  const uint64_t c0 = (uint64_t)blockIdx.x * kPCh;
  long long m = LLONG_MIN;
  for (uint64_t i = c0 + threadIdx.x; i < min(n, c0 + kPCh); i += kET) m = max(m, home_minus_i<W>(space, i, k));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(kFull, m, o));
  if (lane_id() == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kET / 32; w++) m = max(m, red[w]);
    m = max(m, red[0]);
    cmax[blockIdx.x] = m;
  }
}
// one block: cpre[c] = max(cmax[0..c-1]) (LLONG_MIN for c = 0)
__global__ void __launch_bounds__(1024) chunk_prefix_kernel(const long long* __restrict__ cmax, uint64_t nc,
                                                           long long* __restrict__ cpre) {
  __shared__ long long red[32];
  const uint64_t per = (nc + 1023) / 1024, a = threadIdx.x * per, b = min(nc, a + per);
  long long m = LLONG_MIN;
  for (uint64_t c = a; c < b; c++) m = max(m, cmax[c]);
  // exclusive max-scan of the per-thread maxima
  long long inc = m;
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(kFull, inc, o);
    if ((int)lane_id() >= o) inc = max(inc, y);
  }
  if (lane_id() == 31) red[threadIdx.x >> 5] = inc;
  __syncthreads();
  long long wpre = LLONG_MIN;
  for (int w = 0; w < (int)(threadIdx.x >> 5); w++) wpre = max(wpre, red[w]);
  long long ex = max(wpre, __shfl_up_sync(kFull, inc, 1));
  if (lane_id() == 0) ex = wpre;
  for (uint64_t c = a; c < b; c++) {
    cpre[c] = ex;
    ex = max(ex, cmax[c]);
  }
}
template <int W>
__global__ void __launch_bounds__(kET) place_kernel(const uint64_t* __restrict__ space, const double* __restrict__ psi,
                                                   uint64_t n, int k, const long long* __restrict__ cpre,
                                                   KPsi<W>* __restrict__ table, uint64_t tslots, unsigned long long* ovf) {
  __shared__ long long red[kET / 32];
  __shared__ long long carry;
  const uint64_t c0 = (uint64_t)blockIdx.x * kPCh;
  if (threadIdx.x == 0) carry = cpre[blockIdx.x];
  __syncthreads();
  for (uint64_t r0 = c0; r0 < min(n, c0 + kPCh); r0 += kET) {
    const uint64_t i = r0 + threadIdx.x;
    const long long d = i < n ? home_minus_i<W>(space, i, k) : LLONG_MIN;
    long long inc = d;  // inclusive max-scan over the block
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(kFull, inc, o);
      if ((int)lane_id() >= o) inc = max(inc, y);
    }
    if (lane_id() == 31) red[threadIdx.x >> 5] = inc;
    __syncthreads();
    long long pre = carry;
    for (int w = 0; w < (int)(threadIdx.x >> 5); w++) pre = max(pre, red[w]);
    const long long full = max(pre, inc);
    if (i < n) {
      KPsi<W> r{};
      const KeyT<W> kk = load_key<W>(space, i);
      r.k0 = kk.w0;
      if constexpr (W == 2) r.k1 = kk.w1;
      r.psi = psi ? psi[i] : __longlong_as_double((long long)i);  // no psi: the element's index
      const uint64_t slot = (uint64_t)((long long)i + full);
      if (slot < tslots) table[slot] = r;
      else *ovf = 1;  // (impossible for hash-uniform keys: displacement >> n/16)
    }
    __syncthreads();
    if (threadIdx.x == kET - 1) carry = full;  // the block's inclusive maximum so far
    __syncthreads();
  }
}
template <int W> __device__ __forceinline__ bool kp_empty(const KPsi<W>& r);
// an amplitude the owner did not have (multi-rank lookup): this NaN payload
__device__ __forceinline__ bool psi_missing(double x) {
  return (unsigned long long)__double_as_longlong(x) == 0x7FF4DEADBEEF0001ull;
}
template <> __device__ __forceinline__ bool kp_empty<1>(const KPsi<1>& r) { return r.k0 == 0; }
template <> __device__ __forceinline__ bool kp_empty<2>(const KPsi<2>& r) { return (r.k0 | r.k1) == 0; }

// p -> round_half_even(p * 2^80) for |p| < 2^20 (exact integer arithmetic)
__device__ __forceinline__ __int128 quantize80(double p) {
  if (p == 0.0) return 0;
  int E;
  const double f = frexp(p, &E);                 // p = f 2^E, 0.5 <= |f| < 1
  const long long m = (long long)ldexp(f, 53);   // exact: |m| < 2^53
  const int sh = E - 53 + 80;
  const bool neg = m < 0;
  const unsigned long long am = neg ? (unsigned long long)(-m) : (unsigned long long)m;
  unsigned __int128 q;
  if (sh >= 0) {
    q = (unsigned __int128)am << sh;
  } else {
    const int r = -sh;
    if (r > 63) {
      q = 0;  // |am| / 2^r < 2^53 / 2^64 < 1/2
    } else {
      const unsigned long long whole = am >> r, rem = am & ((1ull << r) - 1), half = 1ull << (r - 1);
      q = whole + ((rem > half || (rem == half && (whole & 1ull))) ? 1u : 0u);
    }
  }
  return neg ? -(__int128)q : (__int128)q;
}

// exact 128-bit integer -> nearest fp64 (ties to even)
__device__ __forceinline__ double int128_to_double_rn(__int128 x) {
  if (x == 0) return 0.0;
  const bool neg = x < 0;
  const unsigned __int128 u = neg ? (unsigned __int128)(-x) : (unsigned __int128)x;
  const unsigned long long hi = (unsigned long long)(u >> 64), lo = (unsigned long long)u;
  const int msb = hi ? 127 - __clzll((long long)hi) : 63 - __clzll((long long)lo);
  double r;
  if (msb < 53) {
    r = (double)lo;
  } else {
    const int sh = msb - 52;
    unsigned long long mant = (unsigned long long)(u >> sh);  // 53 bits
    const unsigned __int128 rem = u & ((((unsigned __int128)1) << sh) - 1);
    const unsigned __int128 half = ((unsigned __int128)1) << (sh - 1);
    if (rem > half || (rem == half && (mant & 1ull))) mant++;
    r = ldexp((double)mant, sh);  // mant may be 2^53: still exact in fp64
  }
  return neg ? -r : r;
}

template <int W>
__global__ void __launch_bounds__(kET, 4) contract_kernel(const uint64_t* __restrict__ keys, const double* __restrict__ hij,
                                                      const uint32_t* __restrict__ src, uint64_t n_rec,
                                                      const KPsi<W>* __restrict__ table, uint64_t tslots,
                                                      int k, uint64_t n_parents, unsigned long long* __restrict__ acc,
                                                      unsigned long long* __restrict__ flags,
                                                      const unsigned long long* __restrict__ rcnt, uint64_t rcap,
                                                      const int* __restrict__ rovf, const uint64_t* __restrict__ fkeys,
                                                      const double* __restrict__ fhij, const uint32_t* __restrict__ fsrc,
                                                      uint64_t fn, unsigned long long* __restrict__ tick) {
  // region mode (rcnt != null): the records were partitioned by rec_partition_kernel
  // into regions of rcap slots (rcap % 64 == 0), region g holding rcnt[g] records;
  // if that partition overflowed (*rovf), the flat records (f*) are contracted instead
  if (rcnt && *rovf) {
    keys = fkeys;
    hij = fhij;
    src = fsrc;
    n_rec = fn;
    rcnt = nullptr;
    tick = nullptr;
  }
  const unsigned lane = lane_id();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t missing = 0;
  bool big = false, badsrc = false;
  // warp-uniform trip count so the warp-level reduction always has all lanes;
  // kU consecutive 32-record groups per step: their lookups are in flight together
  constexpr int kU = 2;
  const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = stride >> 5;
  auto group = [&](const uint64_t w0) {
    // records of this 64-record group that exist (a group never straddles a region)
    const uint64_t lim = rcnt ? (w0 / rcap) * rcap + min((uint64_t)rcnt[w0 / rcap], rcap) : n_rec;
    uint32_t sv[kU];
    KeyT<W> kv[kU];
    uint64_t hm[kU];
    KPsi<W> ev[kU];
    double hv[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const uint64_t r = w0 + u * 32 + lane;
      sv[u] = 0xffffffffu;
      if (r < lim) {
        sv[u] = __ldcs(src + r);  // streamed once: evict-first, the table slice keeps L2
        if (sv[u] >= n_parents) {  // out-of-range parent index: flagged, never accumulated
          badsrc = true;
          sv[u] = 0xffffffffu;
        }
        hv[u] = __ldcs(hij + r);
        if constexpr (W == 1) kv[u] = KeyT<W>{__ldcs(reinterpret_cast<const unsigned long long*>(keys) + r)};
        else {
          const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(keys) + r);
          kv[u] = KeyT<W>{x.x, x.y};
        }
        // home slot of the key in the ordered (key, psi) table
        hm[u] = k ? (to_pi(kv[u]).w0 >> (64 - k)) : 0ull;
        ev[u] = table[hm[u]];
      }
    }
    __int128 qv[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      qv[u] = 0;
      const uint64_t r = w0 + u * 32 + lane;
      if (r < lim) {
        bool found = false;
        double ps = 0.0;
        KPsi<W> e = ev[u];
        for (uint64_t slot = hm[u];;) {  // probe forward until the key or an empty slot
          if (kp_eq<W>(e, kv[u])) {
            found = !psi_missing(e.psi);
            ps = e.psi;
            break;
          }
          if (kp_empty<W>(e) || ++slot >= tslots) break;
          e = table[slot];
        }
        if (found) {
          const double prod = __dmul_rn(hv[u], ps);
          if (!(fabs(prod) < 1048576.0)) big = true;
          else qv[u] = quantize80(prod);
        } else {
          missing++;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const uint32_t s = sv[u];
      const bool valid = w0 + u * 32 + lane < lim;
      // segmented inclusive sum over runs of equal src (lanes in record order)
      const uint32_t sprev = __shfl_up_sync(kFull, s, 1);
      const unsigned heads = __ballot_sync(kFull, lane == 0 || sprev != s);
      const int start = 31 - __clz(heads & ((2u << lane) - 1u));  // head of this lane's run
      __int128 acc128 = qv[u];
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long ql = __shfl_up_sync(kFull, (unsigned long long)acc128, o);
        const unsigned long long qh = __shfl_up_sync(kFull, (unsigned long long)((unsigned __int128)acc128 >> 64), o);
        if ((int)lane - o >= start) acc128 += (__int128)(((unsigned __int128)qh << 64) | ql);
      }
      // the last lane of each run adds the run total to the parent's limbs
      const uint32_t snext = __shfl_down_sync(kFull, s, 1);
      const bool tail = valid && s != 0xffffffffu && (lane == 31 || snext != s);
      if (tail && acc128 != 0) {
        const unsigned __int128 uu = (unsigned __int128)acc128;
        const long long l0 = (long long)(uint32_t)(uu), l1 = (long long)(uint32_t)(uu >> 32),
                        l2 = (long long)(uint32_t)(uu >> 64), l3 = (long long)(int32_t)(uint32_t)(uu >> 96);
        unsigned long long* a4 = acc + 4ull * s;
        atomicAdd(a4 + 0, (unsigned long long)l0);
        atomicAdd(a4 + 1, (unsigned long long)l1);
        atomicAdd(a4 + 2, (unsigned long long)l2);
        atomicAdd(a4 + 3, (unsigned long long)l3);
      }
    }
  };
  if (tick) {  // region mode: 512-record chunks in order from a ticket (the grid's chunks in flight stay
               // within one or two regions, so their table slices stay in L2)
    for (;;) {
      unsigned long long c = 0;
      if (lane == 0) c = atomicAdd(tick, 1ull);
      const uint64_t cb = __shfl_sync(kFull, c, 0) * 512ull;
      if (cb >= n_rec) break;
      for (uint64_t w0 = cb; w0 < cb + 512 && w0 < n_rec; w0 += 32 * kU) group(w0);
    }
  } else {
    for (uint64_t w0 = wid * 32 * kU; w0 < n_rec; w0 += nw * 32 * kU) group(w0);
  }
  for (int o = 16; o; o >>= 1) missing += __shfl_xor_sync(kFull, missing, o);
  if (lane == 0 && missing) atomicAdd(&flags[0], (unsigned long long)missing);
  if (__any_sync(kFull, big) && lane == 0) atomicOr(&flags[1], 1ull);
  if (__any_sync(kFull, badsrc) && lane == 0) atomicOr(&flags[1], 2ull);
}

// ---- pi-partition of the records (f1 at scale): the (key, psi) table is far
// larger than L2 and a record's probe is a random sector (ncu: ~130 DRAM bytes
// per probe).  Records are first scattered by the top 8 bits of their key's
// pi-value into 256 regions (hist-free: regions of rcap slots, runs reserved
// per (sub-round, digit) with one global atomic, as dedup's first pass); the
// contraction then sweeps the regions in order with a persistent grid, so the
// table slice the probes touch (1/256 of the table) stays in L2.  Within a
// region a sub-round's records of one digit stay together, so a parent's
// records still arrive in runs for the warp-level src reduction.
constexpr int kRPT = 512;
template <int W> struct RPCfg {
  static constexpr int SUB = W == 1 ? 4096 : 2048;  // records per sub-round
  static constexpr size_t SMEM = (size_t)SUB * (8 * W + 8 + 4 + 1);
};
template <int W>
__global__ void __launch_bounds__(kRPT, 2) rec_partition_kernel(const uint64_t* __restrict__ keys,
                                                               const double* __restrict__ hij,
                                                               const uint32_t* __restrict__ src, uint64_t n,
                                                               uint64_t rcap, unsigned long long* __restrict__ gcur,
                                                               uint64_t* __restrict__ okeys, double* __restrict__ oh,
                                                               uint32_t* __restrict__ osrc, int* __restrict__ ovf) {
  constexpr int SUB = RPCfg<W>::SUB, IT = SUB / kRPT, R = 256;
  extern __shared__ __align__(16) unsigned char rsm[];
  KeyT<W>* sk = reinterpret_cast<KeyT<W>*>(rsm);
  double* sh = reinterpret_cast<double*>(sk + SUB);
  uint32_t* ss = reinterpret_cast<uint32_t*>(sh + SUB);
  uint8_t* sd = reinterpret_cast<uint8_t*>(ss + SUB);
  __shared__ uint32_t cnt[R], lst[R];
  __shared__ unsigned long long dl[R];
  const uint32_t t = threadIdx.x;
  const uint64_t nsub = (n + SUB - 1) / SUB;
  for (uint64_t sb = blockIdx.x; sb < nsub; sb += gridDim.x) {
    for (uint32_t d = t; d < R; d += kRPT) cnt[d] = 0;
    __syncthreads();
    const uint64_t r0 = sb * SUB;
    const uint32_t m = (uint32_t)min((uint64_t)SUB, n - r0);
    KeyT<W> kv[IT];
    double hv[IT];
    uint32_t sv[IT], dr[IT];
#pragma unroll
    for (int u = 0; u < IT; u++) {
      const uint32_t i = u * kRPT + t;
      if (i < m) {
        kv[u] = load_key<W>(keys, r0 + i);
        hv[u] = hij[r0 + i];
        sv[u] = src[r0 + i];
        const uint32_t d = (uint32_t)(to_pi(kv[u]).w0 >> 56);
        dr[u] = (d << 16) | atomicAdd(&cnt[d], 1u);
      }
    }
    __syncthreads();
    if (t < 32) {  // exclusive scan of the digit counts (8 per lane)
      uint32_t c[R / 32], loc = 0;
#pragma unroll
      for (int j = 0; j < R / 32; j++) {
        c[j] = cnt[t * (R / 32) + j];
        loc += c[j];
      }
      uint32_t inc = loc;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if ((int)t >= o) inc += y;
      }
      uint32_t ex = inc - loc;
#pragma unroll
      for (int j = 0; j < R / 32; j++) {
        lst[t * (R / 32) + j] = ex;
        ex += c[j];
      }
    }
    if (t < R) {  // reserve this sub-round's run in region t
      const uint32_t c = cnt[t];
      unsigned long long b = c ? atomicAdd(&gcur[t], (unsigned long long)c) : 0ull;
      if (c && b + c > rcap) {
        *ovf = 1;
        b = ~0ull;
      }
      dl[t] = c ? (b == ~0ull ? ~0ull : (unsigned long long)t * rcap + b) : ~0ull;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IT; u++) {
      const uint32_t i = u * kRPT + t;
      if (i < m) {
        const uint32_t d = dr[u] >> 16, p = lst[d] + (dr[u] & 0xffffu);
        sk[p] = kv[u];
        sh[p] = hv[u];
        ss[p] = sv[u];
        sd[p] = (uint8_t)d;
      }
    }
    __syncthreads();
    for (uint32_t j = t; j < m; j += kRPT) {  // runs of consecutive addresses per digit
      const uint32_t d = sd[j];
      const unsigned long long b = dl[d];
      if (b != ~0ull) {
        const uint64_t o = b + (j - lst[d]);
        store_key<W>(okeys, o, sk[j]);
        oh[o] = sh[j];
        osrc[o] = ss[j];
      }
    }
    __syncthreads();
  }
}

__global__ void contract_finalize_kernel(const unsigned long long* __restrict__ acc, uint64_t n, double* __restrict__ e) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += stride) {
    const long long a0 = (long long)acc[4 * s], a1 = (long long)acc[4 * s + 1], a2 = (long long)acc[4 * s + 2],
                    a3 = (long long)acc[4 * s + 3];
    const __int128 v = (__int128)a0 + ((__int128)a1 << 32) + ((__int128)a2 << 64) + ((__int128)a3 << 96);
    e[s] = ldexp(int128_to_double_rn(v), -80);
  }
}

// owner side of the multi-rank reverse index: psi of each requested key from
// the ordered (key, psi) table of the owned shard, the missing marker if absent
template <int W>
__global__ void __launch_bounds__(kET) lookup_kernel(const uint64_t* __restrict__ req, uint64_t n,
                                                    const KPsi<W>* __restrict__ table, uint64_t tslots, int k,
                                                    double* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const KeyT<W> kv = load_key<W>(req, r);
    double ps = __longlong_as_double((long long)0x7FF4DEADBEEF0001ull);
    for (uint64_t slot = k ? (to_pi(kv).w0 >> (64 - k)) : 0ull; slot < tslots; slot++) {
      const KPsi<W> e = table[slot];
      if (kp_eq<W>(e, kv)) {
        ps = e.psi;
        break;
      }
      if (kp_empty<W>(e)) break;
    }
    out[r] = ps;
  }
}

// ordered (key, psi) table of a pi-sorted space (see place_kernel)
template <int W>
int build_table(cusci_ctx* ctx, Scratch& s, const uint64_t* space, uint64_t n_space, const double* psi, KPsi<W>** table,
                uint64_t* tslots_out, int* k_out, unsigned long long* ovf) {
  int k = 1;
  while ((1ull << k) < 2 * n_space && k < 40) k++;
  const uint64_t tslots = (1ull << k) + 4096 + n_space / 16;
  const uint64_t nc = (n_space + kPCh - 1) / kPCh;
  long long *cmax, *cpre;
  CUSCI_TRY(s.get_t(tslots, table));
  CUSCI_TRY(s.get_t(std::max<uint64_t>(nc, 1), &cmax));
  CUSCI_TRY(s.get_t(std::max<uint64_t>(nc, 1), &cpre));
  CUSCI_CUDA(ctx, cudaMemsetAsync(*table, 0, tslots * sizeof(KPsi<W>), ctx->stream));
  if (n_space) {
    CUSCI_LAUNCH(ctx, PT_ENERGY, chunk_max_kernel<W><<<(unsigned)nc, kET, 0, ctx->stream>>>(space, n_space, k, cmax));
    CUSCI_LAUNCH(ctx, PT_ENERGY, chunk_prefix_kernel<<<1, 1024, 0, ctx->stream>>>(cmax, nc, cpre));
    CUSCI_LAUNCH(ctx, PT_ENERGY, place_kernel<W><<<(unsigned)nc, kET, 0, ctx->stream>>>(space, psi, n_space, k, cpre, *table, tslots, ovf));
  }
  *tslots_out = tslots;
  *k_out = k;
  return CUSCI_OK;
}

template <int W>
int contract_begin_t(cusci_ctx* ctx, Scratch& s, const uint64_t* space, uint64_t n_space, const double* psi,
                     uint64_t n_parents, CState* st) {
  st->W = W;
  st->n_parents = n_parents;
  CUSCI_TRY(s.get_t(std::max<uint64_t>(4 * n_parents, 1), &st->acc));
  CUSCI_TRY(s.get_t(2, &st->flags));
  CUSCI_CUDA(ctx, cudaMemsetAsync(st->acc, 0, std::max<uint64_t>(4 * n_parents, 1) * 8, ctx->stream));
  CUSCI_CUDA(ctx, cudaMemsetAsync(st->flags, 0, 16, ctx->stream));
  // ordered (key, psi) table: 2^k >= 2 n_space home slots + a tail for the
  // displacements at the top end
  KPsi<W>* table;
  CUSCI_TRY(build_table<W>(ctx, s, space, n_space, psi, &table, &st->tslots, &st->k, st->flags + 1));
  st->table = table;
  return CUSCI_OK;
}

template <int W>
int contract_add_t(cusci_ctx* ctx, const CState& st, const uint64_t* keys, const double* hij, const uint32_t* src,
                   uint64_t n_rec) {
  if (!n_rec) return CUSCI_OK;
  const uint64_t tbytes = st.tslots * sizeof(KPsi<W>);
  // Measured on one N2 batch (1.94e9 records, 4.24e8-key space, 17 GB table): the
  // flat kernel reads ~150 DRAM bytes per record (a random probe pulls whole
  // lines) and takes 73 ms; partitioned, the contraction reads 38 B per record
  // (73 GB; the slices stay in L2) but becomes bound by its per-record integer
  // work (65 ms) and the partition costs 35 ms -- so automatic mode keeps the
  // flat kernel; CUSCI_OPT_CONTRACT_PARTITION = 1 selects the partitioned one.
  (void)tbytes;
  const bool part = ctx->contract_partition > 0;
  if (!part) {
    const unsigned g2 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_rec + kET - 1) / kET, (uint64_t)ctx->num_sms * 16));
    CUSCI_LAUNCH(ctx, PT_ENERGY, contract_kernel<W><<<g2, kET, 0, ctx->stream>>>(keys, hij, src, n_rec, (const KPsi<W>*)st.table, st.tslots, st.k, st.n_parents, st.acc, st.flags, nullptr, 0, nullptr, nullptr, nullptr, nullptr, 0, nullptr));
    return CUSCI_OK;
  }
  // pi-partitioned: regions of rcap slots (mean + 2% + 4 Ki, a multiple of 64)
  Scratch s(ctx);
  const uint64_t rcap = ((n_rec / 256 + n_rec / 256 / 50 + 4096) + 63) & ~63ull;
  uint64_t* pk;
  double* ph;
  uint32_t* ps;
  unsigned long long *gcur, *tick;
  int* ovf;
  CUSCI_TRY(s.get_t(256 * rcap * W, &pk));
  CUSCI_TRY(s.get_t(1, &tick));
  CUSCI_TRY(s.get_t(256 * rcap, &ph));
  CUSCI_TRY(s.get_t(256 * rcap, &ps));
  CUSCI_TRY(s.get_t(256, &gcur));
  CUSCI_TRY(s.get_t(1, &ovf));
  CUSCI_CUDA(ctx, cudaMemsetAsync(gcur, 0, 256 * sizeof(unsigned long long), ctx->stream));
  CUSCI_CUDA(ctx, cudaMemsetAsync(ovf, 0, sizeof(int), ctx->stream));
  CUSCI_CUDA(ctx, cudaMemsetAsync(tick, 0, sizeof(unsigned long long), ctx->stream));
  int pper = 1, cper = 1;
  CUSCI_TRY(kernel_setup(ctx, (const void*)rec_partition_kernel<W>, kRPT, RPCfg<W>::SMEM, &pper));
  CUSCI_TRY(kernel_setup(ctx, (const void*)contract_kernel<W>, kET, 0, &cper));
  const uint64_t nsub = (n_rec + RPCfg<W>::SUB - 1) / RPCfg<W>::SUB;
  const unsigned gp = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nsub, (uint64_t)ctx->num_sms * pper));
  CUSCI_LAUNCH(ctx, PT_ENERGY, rec_partition_kernel<W><<<gp, kRPT, RPCfg<W>::SMEM, ctx->stream>>>(keys, hij, src, n_rec, rcap, gcur, pk, ph, ps, ovf));
  // persistent grid: every warp sweeps the regions in step with the others, so
  // the probes of the whole grid stay inside one or two table slices
  const unsigned gc = (unsigned)(ctx->num_sms * std::max(1, cper));
  CUSCI_LAUNCH(ctx, PT_ENERGY, contract_kernel<W><<<gc, kET, 0, ctx->stream>>>(pk, ph, ps, 256 * rcap, (const KPsi<W>*)st.table, st.tslots, st.k, st.n_parents, st.acc, st.flags, gcur, rcap, ovf, keys, hij, src, n_rec, tick));
  return CUSCI_OK;
}

int contract_end_impl(cusci_ctx* ctx, const CState& st, double* e, uint64_t* n_missing) {
  uint64_t h[2];
  CUSCI_TRY(read_u64(ctx, reinterpret_cast<const uint64_t*>(st.flags), h, 2));
  if (h[1] & 2) return set_error(ctx, CUSCI_E_INVALID_ARG, "energy_contract: a record's src >= n_parents");
  if (h[1]) return set_error(ctx, CUSCI_E_INVALID_ARG, "energy_contract: |H psi| >= 2^20 (outside the exact-sum range) or a skewed space");
  *n_missing = h[0];
  if (st.n_parents) {
    const unsigned g3 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((st.n_parents + kET - 1) / kET, (uint64_t)ctx->num_sms * 8));
    CUSCI_LAUNCH(ctx, PT_ENERGY, contract_finalize_kernel<<<g3, kET, 0, ctx->stream>>>(st.acc, st.n_parents, e));
  }
  return CUSCI_OK;
}

template <int W>
int contract_impl(cusci_ctx* ctx, const uint64_t* keys, const double* hij, const uint32_t* src, uint64_t n_rec,
                  uint64_t n_parents, const uint64_t* space, uint64_t n_space, const double* psi, double* e,
                  uint64_t* n_missing) {
  Scratch s(ctx);
  CState st;
  CUSCI_TRY(contract_begin_t<W>(ctx, s, space, n_space, psi, n_parents, &st));
  CUSCI_TRY(contract_add_t<W>(ctx, st, keys, hij, src, n_rec));
  return contract_end_impl(ctx, st, e, n_missing);
}

// world > 1 (or a forced collective): records and psi meet at the key's owner
// (PAPER.md :634 "reverse index just-in-time"): each rank sends its records'
// locally-unique keys to their owners (the dedup_global partition + the a10
// exchange), the owner answers every request with psi from its shard (ordered
// table lookup; a marker when absent), the answers come back over the reverse
// exchange aligned with the requests, and the records are contracted locally
// against (requested keys, psi).  Two status-carrying exchanges: a failure on
// any rank before the second one is agreed by every rank.
template <int W>
int contract_collective(cusci_ctx* ctx, const uint64_t* keys, const double* hij, const uint32_t* src, uint64_t n_rec,
                        uint64_t n_parents, const uint64_t* space, uint64_t n_space, const double* psi, double* e,
                        uint64_t* n_missing, int rc) {
  const int P = ctx->world;
  Scratch s(ctx);
  uint64_t* L = nullptr;
  uint64_t send[CUSCI_MAX_WORLD] = {0}, rcounts[CUSCI_MAX_WORLD] = {0}, nl = 0;
  if (rc == CUSCI_OK) rc = s.get_t(std::max<uint64_t>(n_rec, 1) * W, &L);
  if (rc == CUSCI_OK) rc = dedup_local_bins(ctx, W, keys, n_rec, P, L, send, &nl);
  if (ctx->broken) return rc;
  uint64_t *req, nreq;
  CUSCI_TRY(exchange_bins(ctx, W, L, send, s, &req, &nreq, rc, rcounts));
  // owner: psi of every requested key
  double* ans = nullptr;
  KPsi<W>* table;
  uint64_t tslots;
  int k;
  unsigned long long* ovf = nullptr;
  rc = s.get_t(std::max<uint64_t>(nreq, 1), &ans);
  if (rc == CUSCI_OK) rc = s.get_t(1, &ovf);
  if (rc == CUSCI_OK) rc = cudaMemsetAsync(ovf, 0, 8, ctx->stream) == cudaSuccess ? CUSCI_OK : CUSCI_E_CUDA;
  if (rc == CUSCI_OK) rc = build_table<W>(ctx, s, space, n_space, psi, &table, &tslots, &k, ovf);
  if (rc == CUSCI_OK && nreq) {
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nreq + kET - 1) / kET, (uint64_t)ctx->num_sms * 16));
    lookup_kernel<W><<<g, kET, 0, ctx->stream>>>(req, nreq, table, tslots, k, ans);
    ctx->launches++;
    if (cudaGetLastError() != cudaSuccess) rc = CUSCI_E_CUDA;
  }
  if (ctx->broken) return rc;
  // answers back to the requesters (8-byte words), aligned with their requests
  uint64_t *back, nback;
  CUSCI_TRY(exchange_bins(ctx, 1, reinterpret_cast<const uint64_t*>(ans), rcounts, s, &back, &nback, rc));
  if (nback != nl) return set_error(ctx, CUSCI_E_CUDA, "energy_contract: %llu answers for %llu requests",
                                    (unsigned long long)nback, (unsigned long long)nl);
  return contract_impl<W>(ctx, keys, hij, src, n_rec, n_parents, L, nl, reinterpret_cast<const double*>(back), e,
                          n_missing);
}


// ---------------------------------------------------------------- f4: heat-bath selection
// (Sec 2.2 :310-312 "selecting a subset of
// important configurations from the newly generated candidates (e.g. top-K
// ranked by inferred amplitudes psi) and merging them into S"; the NNQS
// amplitude is replaced by the heat-bath surrogate, reading r16):
//   score_j = max over records (i -> j) of |H_ij psi_i|, packed as
//             v = bits(|p|) << 1 | [p < 0] (p the winning product: order by
//             |p|, ties by sign), for j in C \ S;
//   select   the K largest v > 0, ties in pi order (C is pi-sorted);
//   psi_j   = -p (first-order amplitude with a unit energy denominator).
template <int W>
__global__ void __launch_bounds__(kET) hb_score_kernel(const uint64_t* __restrict__ keys, const double* __restrict__ hij,
                                                      const uint32_t* __restrict__ src, uint64_t n_rec,
                                                      const double* __restrict__ psi_par,
                                                      const KPsi<W>* __restrict__ table, uint64_t tslots, int k,
                                                      unsigned long long* __restrict__ score) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rec; r += stride) {
    const KeyT<W> kv = load_key<W>(keys, r);
    const double p = __dmul_rn(hij[r], psi_par[src[r]]);
    const unsigned long long v = ((unsigned long long)__double_as_longlong(fabs(p)) << 1) | (p < 0.0 ? 1ull : 0ull);
    if (!v) continue;
    for (uint64_t slot = k ? (to_pi(kv).w0 >> (64 - k)) : 0ull; slot < tslots; slot++) {
      const KPsi<W> e = table[slot];
      if (kp_eq<W>(e, kv)) {
        atomicMax(&score[(uint64_t)__double_as_longlong(e.psi)], v);
        break;
      }
      if (kp_empty<W>(e)) break;
    }
  }
}
// candidates already in S score 0
template <int W>
__global__ void __launch_bounds__(kET) hb_exclude_kernel(const uint64_t* __restrict__ S, uint64_t nS,
                                                        const KPsi<W>* __restrict__ table, uint64_t tslots, int k,
                                                        unsigned long long* __restrict__ score) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nS; r += stride) {
    const KeyT<W> kv = load_key<W>(S, r);
    for (uint64_t slot = k ? (to_pi(kv).w0 >> (64 - k)) : 0ull; slot < tslots; slot++) {
      const KPsi<W> e = table[slot];
      if (kp_eq<W>(e, kv)) {
        score[(uint64_t)__double_as_longlong(e.psi)] = 0ull;
        break;
      }
      if (kp_empty<W>(e)) break;
    }
  }
}
// radix-select step: histogram of digit (v >> shift) & 255 over the v > 0 that
// match `prefix` on the bits of pmask
__global__ void __launch_bounds__(kET) hb_hist_kernel(const unsigned long long* __restrict__ v, uint64_t n,
                                                     unsigned long long prefix, unsigned long long pmask, int shift,
                                                     unsigned long long* __restrict__ hist) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += kET) h[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned long long x = v[i];
    if (x && (x & pmask) == prefix) atomicAdd(&h[(x >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += kET)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}
constexpr uint32_t kHB = 1024;  // elements per compaction block
// per block: elements with v > T (cnt[2b]) and v == T (cnt[2b + 1])
__global__ void __launch_bounds__(kET) hb_count_kernel(const unsigned long long* __restrict__ v, uint64_t n,
                                                      unsigned long long T, uint64_t* __restrict__ gt,
                                                      uint64_t* __restrict__ eq) {
  __shared__ uint32_t a, b;
  if (threadIdx.x == 0) a = b = 0;
  __syncthreads();
  const uint64_t i0 = (uint64_t)blockIdx.x * kHB;
  uint32_t ca = 0, cb = 0;
  for (uint64_t i = i0 + threadIdx.x; i < min(n, i0 + kHB); i += kET) {
    const unsigned long long x = v[i];
    ca += x > T;
    cb += x == T && x;
  }
  atomicAdd(&a, ca);
  atomicAdd(&b, cb);
  __syncthreads();
  if (threadIdx.x == 0) {
    gt[blockIdx.x] = a;
    eq[blockIdx.x] = b;
  }
}
// stable compaction: element x is kept iff v > T, or v == T among the first
// `need` such elements (index order = pi order); position = (kept before x)
template <int W>
__global__ void __launch_bounds__(kET) hb_compact_kernel(const unsigned long long* __restrict__ v, uint64_t n,
                                                        unsigned long long T, uint64_t need,
                                                        const uint64_t* __restrict__ gt_off,
                                                        const uint64_t* __restrict__ eq_off,
                                                        const uint64_t* __restrict__ cand, uint64_t* __restrict__ out,
                                                        double* __restrict__ psi_out) {
  __shared__ uint32_t red[33];
  const uint64_t i0 = (uint64_t)blockIdx.x * kHB;
  uint32_t gbase = 0, ebase = 0;
  for (uint32_t c = 0; c < kHB; c += kET) {
    const uint64_t i = i0 + c + threadIdx.x;
    const unsigned long long x = i < n ? v[i] : 0ull;
    const uint32_t fg = x > T, fe = x == T && x;
    uint32_t tg, te;
    const uint32_t pg = block_excl_scan_u32(fg, red, tg);
    const uint32_t pe = block_excl_scan_u32(fe, red, te);
    const uint64_t eb = eq_off[blockIdx.x] + ebase + pe;  // equal elements before x
    if (fg || (fe && eb < need)) {
      const uint64_t pos = gt_off[blockIdx.x] + gbase + pg + min(eb, need);
      store_key<W>(out, pos, load_key<W>(cand, i));
      const double a = __longlong_as_double((long long)(x >> 1));
      psi_out[pos] = (x & 1ull) ? a : -a;  // psi_j = -p
    }
    gbase += tg;
    ebase += te;
  }
}
// psi of the merged space: from S_old (binary search in pi order) or the selection
template <int W>
__device__ __forceinline__ bool pi_find(const uint64_t* keys, uint64_t n, const KeyT<W>& x, uint64_t* pos) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (hk_lt<W>(load_key<W>(keys, mid), x)) lo = mid + 1;
    else hi = mid;
  }
  *pos = lo;
  return lo < n && key_eq(load_key<W>(keys, lo), x);
}
template <int W>
__global__ void __launch_bounds__(kET) realign_kernel(const uint64_t* __restrict__ merged, uint64_t n,
                                                     const uint64_t* __restrict__ s_old, uint64_t ns,
                                                     const double* __restrict__ psi_old,
                                                     const uint64_t* __restrict__ sel, uint64_t nsel,
                                                     const double* __restrict__ psi_sel, double* __restrict__ psi_out,
                                                     unsigned long long* __restrict__ bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const KeyT<W> x = load_key<W>(merged, i);
    uint64_t p;
    if (pi_find<W>(s_old, ns, x, &p)) psi_out[i] = psi_old[p];
    else if (pi_find<W>(sel, nsel, x, &p)) psi_out[i] = psi_sel[p];
    else atomicAdd(bad, 1ull);
  }
}

template <int W>
int grow_step_t(cusci_ctx* ctx, const cusci_space* sp, cusci_pool* pool, const double* psi,
                const cusci_integrals* ints, double threshold, uint64_t K, double* psi_out, uint64_t cap,
                cusci_grow_stats* st) {
  Scratch s(ctx);
  const uint64_t nS = pool->count;
  st->space_before = nS;
  // S_t (the merge replaces the pool's buffers)
  uint64_t* Sold;
  CUSCI_TRY(s.get_t(std::max<uint64_t>(nS, 1) * W, &Sold));
  if (nS) CUSCI_CUDA(ctx, cudaMemcpyAsync(Sold, pool->buf[pool->cur], nS * W * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  // records of S_t, then the candidates C_t
  uint64_t nrec = 0;
  CUSCI_TRY(gen_count(ctx, sp, Sold, nS, ints, threshold, &nrec));
  uint64_t *rk;
  double* rh;
  uint32_t* rs;
  CUSCI_TRY(s.get_t(std::max<uint64_t>(nrec, 1) * W, &rk));
  CUSCI_TRY(s.get_t(std::max<uint64_t>(nrec, 1), &rh));
  CUSCI_TRY(s.get_t(std::max<uint64_t>(nrec, 1), &rs));
  cusci_records rec{rk, rh, rs, nullptr, nrec, 0};
  CUSCI_TRY(gen_records(ctx, sp, Sold, nS, ints, threshold, &rec, 0));
  st->records = rec.count;
  cusci_keys C{nullptr, 0};
  CUSCI_TRY(dedup_global(ctx, sp, rk, rec.count, &C));
  struct OutGuard {
    cusci_ctx* c;
    void* p;
    ~OutGuard() { out_free(c, p); }
  } cg{ctx, C.keys};
  const uint64_t nC = C.count;
  st->unique = nC;
  // index table over C_t, heat-bath scores, S_t excluded
  KPsi<W>* table;
  uint64_t tslots;
  int k;
  unsigned long long *score, *flags, *hist;
  CUSCI_TRY(s.get_t(std::max<uint64_t>(nC, 1), &score));
  CUSCI_TRY(s.get_t(2, &flags));
  CUSCI_TRY(s.get_t(256, &hist));
  CUSCI_CUDA(ctx, cudaMemsetAsync(score, 0, std::max<uint64_t>(nC, 1) * 8, ctx->stream));
  CUSCI_CUDA(ctx, cudaMemsetAsync(flags, 0, 16, ctx->stream));
  CUSCI_TRY(build_table<W>(ctx, s, C.keys, nC, nullptr, &table, &tslots, &k, flags + 1));
  const unsigned g = (unsigned)ctx->num_sms * 8;
  if (rec.count) CUSCI_LAUNCH(ctx, PT_ENERGY, hb_score_kernel<W><<<g, kET, 0, ctx->stream>>>(rk, rh, rs, rec.count, psi, table, tslots, k, score));
  if (nS) CUSCI_LAUNCH(ctx, PT_ENERGY, hb_exclude_kernel<W><<<g, kET, 0, ctx->stream>>>(Sold, nS, table, tslots, k, score));
  // radix select of the K-th largest score (8 x 8-bit digits, most significant first)
  unsigned long long prefix = 0, pmask = 0;
  uint64_t remaining = K, positive = 0;
  for (int d = 7; d >= 0 && remaining; d--) {
    CUSCI_CUDA(ctx, cudaMemsetAsync(hist, 0, 256 * 8, ctx->stream));
    CUSCI_LAUNCH(ctx, PT_ENERGY, hb_hist_kernel<<<g, kET, 0, ctx->stream>>>(score, nC, prefix, pmask, 8 * d, hist));
    uint64_t hh[256];
    CUSCI_TRY(read_u64(ctx, reinterpret_cast<const uint64_t*>(hist), hh, 256));
    uint64_t tot = 0;
    for (int x = 0; x < 256; x++) tot += hh[x];
    if (d == 7) positive = tot;
    if (tot <= remaining) {  // every matching value is taken: threshold = the smallest of them
      for (int x = 0; x < 256; x++)
        if (hh[x]) {
          prefix |= (unsigned long long)x << (8 * d);
          break;
        }
      pmask |= 0xffull << (8 * d);
      if (tot == 0) remaining = 0;
      continue;
    }
    uint64_t above = 0;
    int x = 255;
    for (; x > 0 && above + hh[x] < remaining; x--) above += hh[x];
    remaining -= above;
    prefix |= (unsigned long long)x << (8 * d);
    pmask |= 0xffull << (8 * d);
  }
  st->candidates = positive;
  uint64_t nsel = 0;
  uint64_t* sel = nullptr;
  double* psel = nullptr;
  if (K && positive) {
    unsigned long long T;
    uint64_t need;
    if (positive <= K) {  // every candidate: threshold 1, all equal-or-above taken
      T = 1ull;
      need = ~0ull;
    } else {
      T = prefix;
      need = remaining;
    }
    const uint64_t nb = (nC + kHB - 1) / kHB;
    uint64_t *gt, *eq, *gto, *eqo;
    CUSCI_TRY(s.get_t(nb + 1, &gt));
    CUSCI_TRY(s.get_t(nb + 1, &eq));
    CUSCI_TRY(s.get_t(nb + 1, &gto));
    CUSCI_TRY(s.get_t(nb + 1, &eqo));
    CUSCI_CUDA(ctx, cudaMemsetAsync(gt + nb, 0, 8, ctx->stream));
    CUSCI_CUDA(ctx, cudaMemsetAsync(eq + nb, 0, 8, ctx->stream));
    CUSCI_LAUNCH(ctx, PT_ENERGY, hb_count_kernel<<<(unsigned)nb, kET, 0, ctx->stream>>>(score, nC, T, gt, eq));
    CUSCI_TRY(scan_exclusive_u64(ctx, gt, gto, nb + 1, nullptr));
    CUSCI_TRY(scan_exclusive_u64(ctx, eq, eqo, nb + 1, nullptr));
    uint64_t tot[2];
    CUSCI_TRY(read_u64(ctx, gto + nb, &tot[0], 1));
    CUSCI_TRY(read_u64(ctx, eqo + nb, &tot[1], 1));
    nsel = tot[0] + std::min(tot[1], need);
    CUSCI_TRY(s.get_t(std::max<uint64_t>(nsel, 1) * W, &sel));
    CUSCI_TRY(s.get_t(std::max<uint64_t>(nsel, 1), &psel));
    CUSCI_LAUNCH(ctx, PT_ENERGY, hb_compact_kernel<W><<<(unsigned)nb, kET, 0, ctx->stream>>>(score, nC, T, need, gto, eqo, C.keys, sel, psel));
  }
  st->selected = nsel;
  // S <- S u selected, psi re-aligned with the new pool order
  CUSCI_TRY(merge_space(ctx, pool, sel, nsel, nullptr));
  const uint64_t nN = pool->count;
  st->space_after = nN;
  if (nN > cap) return set_error(ctx, CUSCI_E_CAPACITY, "sci_grow_step: the space grew to %llu > psi_out capacity %llu",
                                 (unsigned long long)nN, (unsigned long long)cap);
  if (nN)
    CUSCI_LAUNCH(ctx, PT_ENERGY, realign_kernel<W><<<g, kET, 0, ctx->stream>>>(pool->buf[pool->cur], nN, Sold, nS, psi, sel, nsel, psel, psi_out, flags));
  uint64_t h[2];
  CUSCI_TRY(read_u64(ctx, reinterpret_cast<const uint64_t*>(flags), h, 2));
  if (h[0] || h[1]) return set_error(ctx, CUSCI_E_CUDA, "sci_grow_step: internal inconsistency (%llu, %llu)",
                                     (unsigned long long)h[0], (unsigned long long)h[1]);
  return CUSCI_OK;
}
}  // namespace

int contract_begin(cusci_ctx* ctx, Scratch& s, int W, const uint64_t* space, uint64_t n_space, const double* psi,
                   uint64_t n_parents, CState* st) {
  return W == 1 ? contract_begin_t<1>(ctx, s, space, n_space, psi, n_parents, st)
                : contract_begin_t<2>(ctx, s, space, n_space, psi, n_parents, st);
}
int contract_add(cusci_ctx* ctx, const CState& st, const uint64_t* keys, const double* hij, const uint32_t* src,
                 uint64_t n_rec) {
  return st.W == 1 ? contract_add_t<1>(ctx, st, keys, hij, src, n_rec) : contract_add_t<2>(ctx, st, keys, hij, src, n_rec);
}
int contract_end(cusci_ctx* ctx, const CState& st, double* e, uint64_t* n_missing) {
  return contract_end_impl(ctx, st, e, n_missing);
}

}  // namespace cusci

using namespace cusci;

extern "C" int energy_contract(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* keys, const double* hij,
                               const uint32_t* src, uint64_t n_rec, uint64_t n_parents, const uint64_t* space_keys,
                               uint64_t n_space, const double* psi, double* e, uint64_t* n_missing) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  int rc = check_space(ctx, sp);
  if (rc == CUSCI_OK && !n_missing) rc = set_error(ctx, CUSCI_E_INVALID_ARG, "n_missing is NULL");
  if (rc == CUSCI_OK && n_rec && (!keys || !hij || !src)) rc = set_error(ctx, CUSCI_E_INVALID_ARG, "record arrays are NULL");
  if (rc == CUSCI_OK && n_parents && !e) rc = set_error(ctx, CUSCI_E_INVALID_ARG, "e is NULL");
  if (rc == CUSCI_OK && n_space && (!space_keys || !psi)) rc = set_error(ctx, CUSCI_E_INVALID_ARG, "space arrays are NULL");
  if (rc == CUSCI_OK && n_space >= (1ull << 32)) rc = set_error(ctx, CUSCI_E_INVALID_ARG, "n_space must be < 2^32");
  if (rc == CUSCI_OK && n_rec >= (1ull << 32)) rc = set_error(ctx, CUSCI_E_INVALID_ARG, "n_rec must be < 2^32 per call");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  if (n_missing) *n_missing = 0;
  if (collective(ctx)) {
    const int W = rc == CUSCI_OK ? sp->words : 1;
    return W == 1 ? contract_collective<1>(ctx, keys, hij, src, n_rec, n_parents, space_keys, n_space, psi, e, n_missing, rc)
                  : contract_collective<2>(ctx, keys, hij, src, n_rec, n_parents, space_keys, n_space, psi, e, n_missing, rc);
  }
  if (rc != CUSCI_OK) return rc;
  return sp->words == 1 ? contract_impl<1>(ctx, keys, hij, src, n_rec, n_parents, space_keys, n_space, psi, e, n_missing)
                        : contract_impl<2>(ctx, keys, hij, src, n_rec, n_parents, space_keys, n_space, psi, e, n_missing);
}

extern "C" int sci_grow_step(cusci_ctx* ctx, const cusci_space* sp, cusci_pool* space, const double* psi,
                             const cusci_integrals* ints, double threshold, uint64_t K, double* psi_out,
                             uint64_t psi_out_capacity, cusci_grow_stats* stats) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  CUSCI_TRY(check_space(ctx, sp));
  if (!space || space->ctx != ctx || space->sp.m != sp->m || space->sp.n_alpha != sp->n_alpha ||
      space->sp.n_beta != sp->n_beta)
    return set_error(ctx, CUSCI_E_INVALID_ARG, "sci_grow_step: pool of another context or space");
  if (!stats || (space->count && !psi) || !psi_out) return set_error(ctx, CUSCI_E_INVALID_ARG, "sci_grow_step: NULL argument");
  if (collective(ctx)) return set_error(ctx, CUSCI_E_INVALID_ARG, "sci_grow_step: one rank");
  if (space->count >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "sci_grow_step: |S| must be < 2^32");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  memset(stats, 0, sizeof(*stats));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, ctx->stream);
  const int rc = sp->words == 1 ? grow_step_t<1>(ctx, sp, space, psi, ints, threshold, K, psi_out, psi_out_capacity, stats)
                                : grow_step_t<2>(ctx, sp, space, psi, ints, threshold, K, psi_out, psi_out_capacity, stats);
  cudaEventRecord(b, ctx->stream);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  stats->ms = ms;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return rc;
}
