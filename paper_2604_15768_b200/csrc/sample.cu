// dedup_sorted: the paper's sort-based regular-sampling de-duplication
// (Sec 4.1.1 :448-462, Steps 1-3, Fig. "unique").
//
//   Step 1  each rank sorts its keys (LSD radix sort over the m significant
//           bits = the big-integer key order) and removes duplicates (reading
//           r15: local unique before sampling; the hash dedup runs
//           first so only the survivors are sorted), then takes
//           S regular samples at indices floor(k |D_i| / S), k = 0..S-1
//           (all of D_i when |D_i| < S).
//   Step 2  the samples are all-gathered (every rank computes what the
//           paper's root computes, so no broadcast: same result, reading
//           r15); the M gathered samples are sorted and the P-1 splitters are
//           sorted[floor(r M / P)], r = 1..P-1; each rank binary-searches the
//           splitters in its sorted array (lower bound): partition r =
//           [spl_r, spl_{r+1}).
//   Step 3  payload all-to-all-v over NCCL (exchange_bins, shared with
//           dedup_global), then sort + adjacent unique of the received runs:
//           the owned shard, globally sorted across ranks.
//
// The hot path (dedup_global) partitions by hash owner instead (DESIGN.md r9,
// r13); this row exists for the paper-faithful comparison (Table 1 balance
// metrics, bench.py "f2").  The building blocks are exported for the virtual-
// rank parity tests.
#include <algorithm>

#include "internal.cuh"

namespace cusci {
namespace {

template <int W> __device__ __forceinline__ bool int_lt(const KeyT<W>& a, const KeyT<W>& b);
template <> __device__ __forceinline__ bool int_lt<1>(const KeyT<1>& a, const KeyT<1>& b) { return a.w0 < b.w0; }
template <> __device__ __forceinline__ bool int_lt<2>(const KeyT<2>& a, const KeyT<2>& b) {
  return a.w1 < b.w1 || (a.w1 == b.w1 && a.w0 < b.w0);
}

// samples[k] = sorted[floor(k n / S)], k < taken (= min(S, n))
template <int W>
__global__ void regular_sample_kernel(const uint64_t* __restrict__ srt, uint64_t n, uint32_t S, uint32_t taken,
                                      uint64_t* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= taken) return;
  const uint64_t i = taken == n ? k : ((uint64_t)k * n) / S;
  store_key<W>(out, k, load_key<W>(srt, i));
}

// spl[r-1] = sorted samples[floor(r M / P)], r = 1..P-1 (zero keys if M = 0)
template <int W>
__global__ void pick_splitters_kernel(const uint64_t* __restrict__ s, uint64_t M, int P, uint64_t* __restrict__ spl) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (r >= P) return;
  KeyT<W> k{};
  if (M) k = load_key<W>(s, ((uint64_t)r * M) / P);
  store_key<W>(spl, r - 1, k);
}

// bounds[r] = lower_bound(sorted, spl_r), bounds[0] = 0, bounds[P] = n
template <int W>
__global__ void split_bounds_kernel(const uint64_t* __restrict__ srt, uint64_t n, const uint64_t* __restrict__ spl,
                                    int P, uint64_t* __restrict__ bounds) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > P) return;
  if (r == 0 || r == P) {
    bounds[r] = r == 0 ? 0 : n;
    return;
  }
  const KeyT<W> x = load_key<W>(spl, r - 1);
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (int_lt<W>(load_key<W>(srt, mid), x)) lo = mid + 1;
    else hi = mid;
  }
  bounds[r] = lo;
}

int args_ok(cusci_ctx* ctx, const cusci_space* sp) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  return check_space(ctx, sp);
}

// Step 1: out (device, >= n keys) <- sorted unique keys; *u (host) their number.
// The hash dedup runs first (SURVEY 8(a) a11 variant: only the survivors are
// sorted), then an LSD radix sort over the m significant bits -- the same set
// and order as sort + adjacent unique of the raw buffer, with ~1/redundancy of
// the sort traffic.
int sort_unique_impl(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n, uint64_t* out,
                     uint64_t* u) {
  const int W = sp->words;
  *u = 0;
  if (n == 0) return CUSCI_OK;
  Scratch s(ctx);
  uint64_t* a;
  CUSCI_TRY(s.get_t(n * W, &a));
  uint64_t nu = 0;
  CUSCI_TRY(local_dedup(ctx, W, configs, n, a, &nu));
  uint64_t* srt = a;
  if (nu) CUSCI_TRY(radix_sort_keys(ctx, W, a, out, nu, sp->m, &srt));
  if (srt != out && nu) CUSCI_CUDA(ctx, cudaMemcpyAsync(out, srt, nu * W * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *u = nu;
  return CUSCI_OK;
}

int samples_impl(cusci_ctx* ctx, int W, const uint64_t* srt, uint64_t n, uint32_t S, uint64_t* out, uint64_t* taken) {
  const uint32_t t = (uint32_t)std::min<uint64_t>(S, n);
  *taken = t;
  if (!t) return CUSCI_OK;
  if (W == 1) CUSCI_LAUNCH(ctx, PT_PREP, regular_sample_kernel<1><<<(t + 255) / 256, 256, 0, ctx->stream>>>(srt, n, S, t, out));
  else CUSCI_LAUNCH(ctx, PT_PREP, regular_sample_kernel<2><<<(t + 255) / 256, 256, 0, ctx->stream>>>(srt, n, S, t, out));
  return CUSCI_OK;
}

int splitters_impl(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* samples, uint64_t M, int P, uint64_t* spl) {
  const int W = sp->words;
  if (P < 2) return CUSCI_OK;
  Scratch s(ctx);
  const uint64_t* srt = samples;
  if (M) {
    uint64_t *a, *b;
    CUSCI_TRY(s.get_t(M * W, &a));
    CUSCI_TRY(s.get_t(M * W, &b));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(a, samples, M * W * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    uint64_t* o;
    CUSCI_TRY(radix_sort_keys(ctx, W, a, b, M, sp->m, &o));
    srt = o;
  }
  const unsigned g = (unsigned)((P - 1 + 255) / 256);
  if (W == 1) CUSCI_LAUNCH(ctx, PT_PREP, pick_splitters_kernel<1><<<g, 256, 0, ctx->stream>>>(srt, M, P, spl));
  else CUSCI_LAUNCH(ctx, PT_PREP, pick_splitters_kernel<2><<<g, 256, 0, ctx->stream>>>(srt, M, P, spl));
  // the sort buffers are released with s: finish before returning
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return CUSCI_OK;
}

int bounds_impl(cusci_ctx* ctx, int W, const uint64_t* srt, uint64_t n, const uint64_t* spl, int P, uint64_t* bounds) {
  Scratch s(ctx);
  uint64_t* d;
  CUSCI_TRY(s.get_t(P + 1, &d));
  const unsigned g = (unsigned)((P + 1 + 255) / 256);
  if (W == 1) CUSCI_LAUNCH(ctx, PT_PREP, split_bounds_kernel<1><<<g, 256, 0, ctx->stream>>>(srt, n, spl, P, d));
  else CUSCI_LAUNCH(ctx, PT_PREP, split_bounds_kernel<2><<<g, 256, 0, ctx->stream>>>(srt, n, spl, P, d));
  return read_u64(ctx, d, bounds, P + 1);
}

}  // namespace
}  // namespace cusci

using namespace cusci;

extern "C" int sort_unique(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n,
                           cusci_keys* out) {
  CUSCI_TRY(args_ok(ctx, sp));
  if (!out) return set_error(ctx, CUSCI_E_INVALID_ARG, "output is NULL");
  if (n && !configs) return set_error(ctx, CUSCI_E_INVALID_ARG, "configs is NULL");
  if (n >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "n must be < 2^32 per call");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  out->keys = nullptr;
  out->count = 0;
  void* o;
  CUSCI_TRY(out_alloc(ctx, std::max<uint64_t>(n, 1) * sp->words * 8, &o));
  uint64_t u;
  const int rc = sort_unique_impl(ctx, sp, configs, n, (uint64_t*)o, &u);
  if (rc != CUSCI_OK) {
    out_free(ctx, o);
    return rc;
  }
  out->keys = (uint64_t*)o;
  out->count = u;
  return CUSCI_OK;
}

extern "C" int regular_samples(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* sorted, uint64_t n,
                               int n_samples, uint64_t* samples, uint64_t* n_taken) {
  CUSCI_TRY(args_ok(ctx, sp));
  if (n_samples < 1 || n_samples > (1 << 16) || !samples || !n_taken || (n && !sorted))
    return set_error(ctx, CUSCI_E_INVALID_ARG, "regular_samples: bad arguments");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  CUSCI_TRY(samples_impl(ctx, sp->words, sorted, n, (uint32_t)n_samples, samples, n_taken));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return CUSCI_OK;
}

extern "C" int select_splitters(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* samples, uint64_t n_samples,
                                int n_parts, uint64_t* splitters) {
  CUSCI_TRY(args_ok(ctx, sp));
  if (n_parts < 1 || n_parts > 256 || (n_parts > 1 && !splitters) || (n_samples && !samples) || n_samples >= (1ull << 32))
    return set_error(ctx, CUSCI_E_INVALID_ARG, "select_splitters: bad arguments");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  return splitters_impl(ctx, sp, samples, n_samples, n_parts, splitters);
}

extern "C" int split_bounds(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* sorted, uint64_t n,
                            const uint64_t* splitters, int n_parts, uint64_t* bounds) {
  CUSCI_TRY(args_ok(ctx, sp));
  if (n_parts < 1 || n_parts > 256 || !bounds || (n_parts > 1 && !splitters) || (n && !sorted))
    return set_error(ctx, CUSCI_E_INVALID_ARG, "split_bounds: bad arguments");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  return bounds_impl(ctx, sp->words, sorted, n, splitters, n_parts, bounds);
}

extern "C" int dedup_sorted(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n,
                            int n_samples, cusci_keys* owned_sorted, uint64_t* splitters_host) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  int rc = args_ok(ctx, sp);
  if (rc == CUSCI_OK && (!owned_sorted || (n && !configs) || n >= (1ull << 32) || n_samples < 1 || n_samples > (1 << 16) || ctx->world > 256))
    rc = set_error(ctx, CUSCI_E_INVALID_ARG, "dedup_sorted: bad arguments");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  if (owned_sorted) {
    owned_sorted->keys = nullptr;
    owned_sorted->count = 0;
  }
  const int P = ctx->world;
  if (!collective(ctx)) {  // one rank: Steps 2-3 are the identity, the sorted unique keys
    if (rc != CUSCI_OK) return rc;
    const int W = sp->words;
    void* o;
    CUSCI_TRY(out_alloc(ctx, std::max<uint64_t>(n, 1) * W * 8, &o));
    uint64_t u;
    rc = sort_unique_impl(ctx, sp, configs, n, (uint64_t*)o, &u);
    if (rc != CUSCI_OK) {
      out_free(ctx, o);
      return rc;
    }
    owned_sorted->keys = (uint64_t*)o;
    owned_sorted->count = u;
    return CUSCI_OK;
  }
  // collective protocol; a rank that fails before data moves still takes part
  // in the status-carrying count all-gather (and the status all-reduce after
  // the gather buffer is reserved), so no peer is left blocked
  const int W = rc == CUSCI_OK ? sp->words : 1;
  const uint32_t S = rc == CUSCI_OK ? (uint32_t)n_samples : 1u;
  Scratch s(ctx);
  // Step 1: local sort + unique, regular samples
  uint64_t* D = nullptr;
  uint64_t nd = 0, taken = 0;
  uint64_t* smp_local = nullptr;
  if (rc == CUSCI_OK) rc = s.get_t(std::max<uint64_t>(n, 1) * W, &D);
  if (rc == CUSCI_OK) rc = sort_unique_impl(ctx, sp, configs, n, D, &nd);
  if (rc == CUSCI_OK) rc = s.get_t((uint64_t)S * W, &smp_local);
  if (rc == CUSCI_OK) rc = samples_impl(ctx, W, D, nd, S, smp_local, &taken);
  if (ctx->broken) return rc;
  // Step 2a: all-gather of the sample counts, each carrying its rank's status
  constexpr uint64_t kFail = 0xFA11000000000000ull;
  uint64_t* cnt = ctx->dcomm;  // [P] (persistent: cannot fail)
  uint64_t* hp = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  hp[0] = rc == CUSCI_OK ? taken : (kFail | (uint64_t)rc);
  CUSCI_CUDA(ctx, cudaMemcpyAsync(cnt + ctx->rank, hp, sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  CUSCI_TRY(nccl_ok(ctx, ncclAllGather(cnt + ctx->rank, cnt, 1, ncclUint64, ctx->comm, ctx->stream), "count allgather"));
  uint64_t hc[CUSCI_MAX_WORLD], M = 0;
  CUSCI_TRY(read_u64(ctx, cnt, hc, P));
  int agreed = rc;
  for (int r = 0; r < P; r++)
    if ((hc[r] & 0xFFFF000000000000ull) == kFail) agreed = std::max(agreed, (int)(hc[r] & 0xffff));
  if (agreed != CUSCI_OK) {
    if (rc == CUSCI_OK) set_error(ctx, agreed, "dedup_sorted failed on a peer rank (code %d)", agreed);
    return agreed;
  }
  for (int r = 0; r < P; r++) M += hc[r];
  // Step 2b: gather the samples back to back (grouped sends/recvs of each
  // rank's taken samples), splitters, bounds
  uint64_t *smp = nullptr, *spl = nullptr;
  int arc = s.get_t(std::max<uint64_t>(M, 1) * W, &smp);
  if (arc == CUSCI_OK) arc = s.get_t((uint64_t)std::max(P - 1, 1) * W, &spl);
  const int rc2 = agree_status_all(ctx, arc);
  if (rc2 != CUSCI_OK) {
    if (arc == CUSCI_OK) set_error(ctx, rc2, "dedup_sorted failed on a peer rank (code %d)", rc2);
    return rc2;
  }
  CUSCI_TRY(nccl_ok(ctx, ncclGroupStart(), "group start"));
  {
    uint64_t off = 0;
    for (int r = 0; r < P; r++) {
      if (taken) CUSCI_TRY(nccl_ok(ctx, ncclSend(smp_local, taken * W, ncclUint64, r, ctx->comm, ctx->stream), "sample send"));
      if (hc[r]) CUSCI_TRY(nccl_ok(ctx, ncclRecv(smp + off * W, hc[r] * W, ncclUint64, r, ctx->comm, ctx->stream), "sample recv"));
      off += hc[r];
    }
  }
  CUSCI_TRY(nccl_ok(ctx, ncclGroupEnd(), "group end"));
  CUSCI_TRY(splitters_impl(ctx, sp, smp, M, P, spl));
  uint64_t bounds[CUSCI_MAX_WORLD + 1], send[CUSCI_MAX_WORLD];
  CUSCI_TRY(bounds_impl(ctx, W, D, nd, spl, P, bounds));
  for (int r = 0; r < P; r++) send[r] = bounds[r + 1] - bounds[r];
  // Step 3: exchange, then sort + unique of the received runs
  uint64_t* rbuf;
  uint64_t nrecv;
  CUSCI_TRY(exchange_bins(ctx, W, D, send, s, &rbuf, &nrecv));
  void* o;
  rc = out_alloc(ctx, std::max<uint64_t>(nrecv, 1) * W * 8, &o);
  if (rc != CUSCI_OK) return rc;
  uint64_t u;
  rc = sort_unique_impl(ctx, sp, rbuf, nrecv, (uint64_t*)o, &u);
  if (rc == CUSCI_OK && splitters_host && P > 1) {
    CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, spl, (size_t)(P - 1) * W * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    memcpy(splitters_host, ctx->host_pinned, (size_t)(P - 1) * W * 8);
  }
  if (rc != CUSCI_OK) {
    out_free(ctx, o);
    return rc;
  }
  owned_sorted->keys = (uint64_t*)o;
  owned_sorted->count = u;
  return CUSCI_OK;
}
