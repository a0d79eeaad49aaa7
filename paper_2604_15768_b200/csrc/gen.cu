// gen_coupled: excitation enumerator + Slater-Condon evaluator + screening +
// compaction (Alg. 1 :514-554, Sec 4.2.2
// :561-571; Eq. 4 :261-265).
//
// B200 design: a persistent grid of warps pulls work
// units (parent, contiguous range of excitation rows) from a global counter.
// Per unit one warp
//   a1  loads the parent (one 8/16-byte broadcast load) and builds its sorted
//       occupied list in shared memory with ballots + popc (no loops over bits
//       per lane);
//   a2  walks its rows: row r < n is the singles row of occupied orbital
//       occ[r] (targets from the singles candidate table), row r >= n is the
//       pair row of occupied pair (occ[x], occ[y]), x < y, read from the
//       prescreened CSR pair table (a0) 32 entries per step, coalesced;
//   a3  forms the target key with XORs;
//   a4  the phase from popc over masked ranges (sequential singles p->a, q->b);
//   a5  H from the table value (doubles) or the sequential sum over occ(i)\p
//       of the [K][P][A] tables (singles, same order as the definition);
//   a6  keeps |H| > eps (doubles: already folded into the table);
//   a7  counts survivors in a first sweep, reserves exactly that many output
//       slots with ONE atomicAdd per unit, then re-sweeps and writes survivors
//       compacted with ballot/popc offsets: every store instruction of the warp
//       covers consecutive records (coalesced), there are no gaps, and no
//       per-record atomics (the paper's "one atomicAdd per block").
#include <cmath>

#include "internal.cuh"

namespace cusci {
namespace {

constexpr int kGenThreads = 256;
constexpr int kGenWarps = kGenThreads / 32;
constexpr unsigned long long kNoError = ~0ull;

struct GenArgs {
  const uint64_t* parents;
  uint64_t n_parents;
  int m, n_elec, K;
  uint32_t units_per_parent;
  uint32_t rows_per_parent;
  uint64_t n_units;
  const uint32_t* rowptr;
  const uint16_t* ab;
  const double* v;
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
  unsigned long long* counter;    // [0] = records reserved, [1] = unit work counter, [2] = first bad parent
  int count_only;
};

// ---- bit helpers on W-word keys
__device__ __forceinline__ bool occ_bit(const KeyT<1>& k, int t) { return (k.w0 >> t) & 1ull; }
__device__ __forceinline__ bool occ_bit(const KeyT<2>& k, int t) {
  return t < 64 ? ((k.w0 >> t) & 1ull) : ((k.w1 >> (t - 64)) & 1ull);
}
__device__ __forceinline__ void flip2(KeyT<1>& k, int s, int t) { k.w0 ^= (1ull << s) ^ (1ull << t); }
__device__ __forceinline__ void flip2(KeyT<2>& k, int s, int t) {
  if (s < 64) k.w0 ^= 1ull << s; else k.w1 ^= 1ull << (s - 64);
  if (t < 64) k.w0 ^= 1ull << t; else k.w1 ^= 1ull << (t - 64);
}
// bits < t, t in [0, 64]
__device__ __forceinline__ uint64_t below64(int t) { return t >= 64 ? ~0ull : ((1ull << t) - 1ull); }
// parity of the occupied orbitals strictly between x and y
__device__ __forceinline__ uint32_t parity_between(const KeyT<1>& k, int x, int y) {
  const int lo = min(x, y), hi = max(x, y);
  const uint64_t mask = below64(hi) & ~below64(lo + 1);
  return __popcll(k.w0 & mask) & 1u;
}
__device__ __forceinline__ uint32_t parity_between(const KeyT<2>& k, int x, int y) {
  const int lo = min(x, y), hi = max(x, y);
  const uint64_t m0 = below64(min(hi, 64)) & ~below64(min(lo + 1, 64));
  const uint64_t m1 = below64(max(hi - 64, 0)) & ~below64(max(lo + 1 - 64, 0));
  return (__popcll(k.w0 & m0) + __popcll(k.w1 & m1)) & 1u;
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

// one warp processes the rows [r0, r1) of parent s; pass 0 counts, pass 1 emits
template <int W>
__device__ __forceinline__ uint32_t process_rows(const GenArgs& a, const KeyT<W>& par, const uint8_t* occ, uint64_t s,
                                                 uint32_t r0, uint32_t r1, bool emit, uint64_t cursor) {
  const unsigned lane = lane_id();
  const int n = a.n_elec;
  uint32_t total = 0;
  // decode the first pair row
  int x = 0, y = 1;
  if (r1 > (uint32_t)n) {
    uint32_t k = r0 > (uint32_t)n ? r0 - n : 0;
    while (k >= (uint32_t)(n - 1 - x)) {
      k -= (uint32_t)(n - 1 - x);
      x++;
    }
    y = x + 1 + (int)k;
  }
  for (uint32_t r = r0; r < r1; r++) {
    if (r < (uint32_t)n) {
      // ---------------- singles row: p = occ[r]
      const int p = occ[r];
      const int P = p >> 1;
      const uint32_t c0 = __ldg(a.srowptr + p), c1 = __ldg(a.srowptr + p + 1);
      for (uint32_t c = c0; c < c1; c += 32) {
        const uint32_t ci = c + lane;
        bool keep = false;
        int t = 0;
        double H = 0.0;
        uint32_t ph = 0;
        if (ci < c1) {
          t = __ldg(a.sa + ci);
          if (!occ_bit(par, t)) {
            const int A = t >> 1;
            double v = __ldg(a.h + P * a.K + A);
            for (int xx = 0; xx < n; xx++) {
              const int kk = occ[xx];
              if (kk == p) continue;
              const size_t o = ((size_t)(kk >> 1) * a.K + P) * a.K + A;
              const double tv = ((kk & 1) == (p & 1)) ? __ldg(a.tsame + o) : __ldg(a.topp + o);
              v = __dadd_rn(v, tv);
            }
            ph = parity_between(par, p, t);
            H = ph ? -v : v;
            keep = fabs(H) > a.eps;
          }
        }
        const unsigned bal = __ballot_sync(kFull, keep);
        if (emit && keep) {
          const uint64_t pos = cursor + total + __popc(bal & lanemask_lt());
          KeyT<W> j = par;
          flip2(j, p, t);
          store_key<W>(a.keys, pos, j);
          a.hij[pos] = H;
          if (a.src) a.src[pos] = (uint32_t)s;
          if (a.phase) a.phase[pos] = ph ? -1 : 1;
        }
        total += __popc(bal);
      }
    } else {
      // ---------------- pair row (p, q) = (occ[x], occ[y])
      const int p = occ[x], q = occ[y];
      const uint32_t row = (uint32_t)q * (q - 1) / 2 + p;
      const uint32_t e0 = __ldg(a.rowptr + row), e1 = __ldg(a.rowptr + row + 1);
      KeyT<W> base = par;
      flip2(base, p, q);
      for (uint32_t e = e0; e < e1; e += 32) {
        const uint32_t ei = e + lane;
        bool keep = false;
        int ta = 0, tb = 0;
        if (ei < e1) {
          const uint32_t abv = __ldg(a.ab + ei);
          ta = abv & 0xff;
          tb = abv >> 8;
          keep = !occ_bit(par, ta) && !occ_bit(par, tb);
        }
        const unsigned bal = __ballot_sync(kFull, keep);
        if (emit && keep) {
          const double v = __ldg(a.v + ei);
          // sequential singles p->a on i, then q->b on i' = i ^ p ^ a
          KeyT<W> i1 = par;
          flip2(i1, p, ta);
          const uint32_t ph = parity_between(par, p, ta) ^ parity_between(i1, q, tb);
          const uint64_t pos = cursor + total + __popc(bal & lanemask_lt());
          KeyT<W> j = base;
          flip2(j, ta, tb);
          store_key<W>(a.keys, pos, j);
          a.hij[pos] = ph ? -v : v;
          if (a.src) a.src[pos] = (uint32_t)s;
          if (a.phase) a.phase[pos] = ph ? -1 : 1;
        }
        total += __popc(bal);
      }
      if (++y == n) {
        x++;
        y = x + 1;
      }
    }
  }
  return total;
}

template <int W>
__global__ void __launch_bounds__(kGenThreads) gen_kernel(const GenArgs a) {
  __shared__ uint8_t occ_s[kGenWarps][128];
  __shared__ unsigned long long unit_s[kGenWarps];
  if (a.counter[2] != kNoError) return;  // invalid parent: write nothing
  const int w = threadIdx.x >> 5;
  const unsigned lane = lane_id();
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
    __syncwarp();
    const uint32_t cnt = process_rows<W>(a, par, occ, s, r0, r1, false, 0);
    if (cnt == 0 || a.count_only) {
      if (lane == 0 && cnt) atomicAdd(&a.counter[0], (unsigned long long)cnt);
      continue;
    }
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&a.counter[0], (unsigned long long)cnt);
    base = __shfl_sync(kFull, base, 0);
    if (base + cnt <= a.capacity) process_rows<W>(a, par, occ, s, r0, r1, true, base);
    __syncwarp();
  }
}

int gen_impl(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
             const cusci_integrals* ints, double threshold, cusci_records* out, bool count_only, uint64_t* count_out) {
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
  a.rows_per_parent = (uint32_t)(n + n * (n - 1) / 2);
  const uint64_t target_units = (uint64_t)ctx->num_sms * 64 * 4;
  uint64_t U = (target_units + n_parents - 1) / n_parents;
  if (U < 1) U = 1;
  if (U > a.rows_per_parent) U = a.rows_per_parent;
  if (a.rows_per_parent == 0) U = 1;
  a.units_per_parent = (uint32_t)U;
  a.n_units = n_parents * U;
  const Prep& pr = ctx->prep;
  a.rowptr = pr.rowptr;
  a.ab = pr.ab;
  a.v = pr.v;
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
  const unsigned blocks = (unsigned)ctx->num_sms * (2048 / kGenThreads);
  if (W == 1)
    CUSCI_LAUNCH(ctx, PT_GEN, gen_kernel<1><<<blocks, kGenThreads, 0, ctx->stream>>>(a));
  else
    CUSCI_LAUNCH(ctx, PT_GEN, gen_kernel<2><<<blocks, kGenThreads, 0, ctx->stream>>>(a));
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
