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

// T[b] = first index i with top_k(hi(space[i])) >= b, b in [0, 2^k]
template <int W>
__global__ void rindex_table_kernel(const uint64_t* __restrict__ space, uint64_t n, int k, uint32_t* __restrict__ T) {
  const uint64_t nb = 1ull << k;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += stride) {
    // buckets (prev, cur] start at i
    const uint64_t cur = i < n ? (k ? (to_pi(load_key<W>(space, i)).w0 >> (64 - k)) : 0ull) : nb;
    const int64_t prev = i > 0 ? (int64_t)(k ? (to_pi(load_key<W>(space, i - 1)).w0 >> (64 - k)) : 0ull) : -1;
    for (int64_t b = prev + 1; b <= (int64_t)cur; b++) T[b] = (uint32_t)i;
  }
}

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
template <int W>
__global__ void kpsi_kernel(const uint64_t* __restrict__ space, const double* __restrict__ psi, uint64_t n,
                            KPsi<W>* __restrict__ kp) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    KPsi<W> r{};
    const KeyT<W> k = load_key<W>(space, i);
    r.k0 = k.w0;
    if constexpr (W == 2) r.k1 = k.w1;
    r.psi = psi[i];
    kp[i] = r;
  }
}
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
      r.psi = psi[i];
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
                                                      unsigned long long* __restrict__ flags) {
  const unsigned lane = lane_id();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t missing = 0;
  bool big = false, badsrc = false;
  // warp-uniform trip count so the warp-level reduction always has all lanes;
  // kU consecutive 32-record groups per step: their lookups are in flight together
  constexpr int kU = 2;
  const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = stride >> 5;
  for (uint64_t w0 = wid * 32 * kU; w0 < n_rec; w0 += nw * 32 * kU) {
    uint32_t sv[kU];
    KeyT<W> kv[kU];
    uint64_t hm[kU];
    KPsi<W> ev[kU];
    double hv[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const uint64_t r = w0 + u * 32 + lane;
      sv[u] = 0xffffffffu;
      if (r < n_rec) {
        sv[u] = src[r];
        if (sv[u] >= n_parents) {  // out-of-range parent index: flagged, never accumulated
          badsrc = true;
          sv[u] = 0xffffffffu;
        }
        hv[u] = hij[r];
        kv[u] = load_key<W>(keys, r);
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
      if (r < n_rec) {
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
      const bool valid = w0 + u * 32 + lane < n_rec;
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
  }
  for (int o = 16; o; o >>= 1) missing += __shfl_xor_sync(kFull, missing, o);
  if (lane == 0 && missing) atomicAdd(&flags[0], (unsigned long long)missing);
  if (__any_sync(kFull, big) && lane == 0) atomicOr(&flags[1], 1ull);
  if (__any_sync(kFull, badsrc) && lane == 0) atomicOr(&flags[1], 2ull);
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
  const unsigned g2 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_rec + kET - 1) / kET, (uint64_t)ctx->num_sms * 16));
  CUSCI_LAUNCH(ctx, PT_ENERGY, contract_kernel<W><<<g2, kET, 0, ctx->stream>>>(keys, hij, src, n_rec, (const KPsi<W>*)st.table, st.tslots, st.k, st.n_parents, st.acc, st.flags));
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
