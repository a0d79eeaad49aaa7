// dedup_global: distributed de-duplication of configuration keys
// (Sec 2.2, Sec 4.1.1 :448-462,
// Sec 3 :380-382 "local uniqueness filtering is applied immediately after
// generation").
//
// B200 design:
//   a8+a9  keys are scattered into buckets bucket(j) = owner(j) * 2^s + top s
//          bits of a bijective 64-bit mix (owner(j) = floor(mix(j) P / 2^64),
//          DESIGN.md r9), ~1024 keys per bucket (histogram + scatter with
//          L2-resident per-bucket atomics); one CTA per bucket then removes
//          duplicates with an open-addressing hash table in SHARED memory
//          (32-bit atomicCAS, linear probing): the random probes never touch
//          HBM.  Survivors of the buckets of owner r form contiguous owner
//          bin r (P = 1: one atomic append per bucket).
//   a10    counts all-to-all then one payload all-to-all-v over NCCL grouped
//          ncclSend/ncclRecv (NVLink/NVSwitch); one host sync for the sizes.
//   a11    LSD radix sort over the m significant key bits + adjacent-unique
//          compaction -> the sorted unique owned shard.
// The hash filter is a pre-filter: a rare duplicate it lets through (e.g. a
// torn 128-bit read) is removed by the sort + unique, so the result is exact.
#include <algorithm>

#include "internal.cuh"

namespace cusci {
namespace {

constexpr int kHashThreads = 256;

// ---------------------------------------------------------------- bucket dedup
// After the onesweep passes the keys are ordered by bucket(j) = the top `bits`
// bits of the owner mix (a bijective 64-bit mix), ~<= 4096 keys per bucket.
// Each CTA takes ranges of 64 Ki positions and processes the buckets that
// START in its range: it streams a bucket's keys in rounds of 256 through an
// open-addressing hash table held in SHARED memory (the keys themselves are
// the slots: 64-bit atomicCAS, or ATOMS.CAS.128 for W=2; empty = 0, key 0 is
// tracked by a flag; linear probing on the low bits of an independent mix).
// The first copy of each key is appended to `out` (one atomic per warp-round).
// If a bucket holds more distinct keys than the table can take, the table is
// flushed and restarted; the duplicates that then survive are removed by the
// final sort + unique, so the result stays exact.
template <int W> struct SDCfg {
  static constexpr int TS = W == 1 ? 8192 : 4096;  // slots (64 KB)
  static constexpr size_t SMEM = (size_t)TS * sizeof(KeyT<W>);
  static constexpr uint32_t FILL_LIMIT = (TS * 3) / 4;
  static constexpr uint64_t RANGE = 1ull << 16;
};

__device__ __forceinline__ uint64_t cas_slot(KeyT<1>* slot, const KeyT<1>& k, KeyT<1>& old) {
  old.w0 = atomicCAS(reinterpret_cast<unsigned long long*>(&slot->w0), 0ull, (unsigned long long)k.w0);
  return 0;
}
__device__ __forceinline__ uint64_t cas_slot(KeyT<2>* slot, const KeyT<2>& k, KeyT<2>& old) {
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
  return 0;
}
__device__ __forceinline__ bool key_zero(const KeyT<1>& k) { return k.w0 == 0; }
__device__ __forceinline__ bool key_zero(const KeyT<2>& k) { return (k.w0 | k.w1) == 0; }

template <int W>
__device__ __forceinline__ uint32_t bucket_id(const KeyT<W>& k, int bits) {
  return bits ? (uint32_t)(owner_mix(k) >> (64 - bits)) : 0u;
}

template <int W>
__device__ __forceinline__ bool table_insert(KeyT<W>* tab, const KeyT<W>& k, int* s_zero, uint32_t* s_fill) {
  constexpr uint32_t TS = SDCfg<W>::TS;
  if (key_zero(k)) return atomicExch(s_zero, 1) == 0;
  uint32_t h = (uint32_t)slot_hash(k) & (TS - 1);
  for (uint32_t probe = 0; probe < TS; probe++) {
    const KeyT<W> cur = tab[h];
    if (key_eq(cur, k)) return false;
    if (key_zero(cur)) {
      KeyT<W> old;
      cas_slot(&tab[h], k, old);
      if (key_zero(old)) {
        atomicAdd(s_fill, 1u);
        return true;
      }
      if (key_eq(old, k)) return false;
    }
    h = (h + 1) & (TS - 1);
  }
  return true;  // table full: pass through (removed later by sort + unique)
}

template <int W>
__global__ void __launch_bounds__(kHashThreads) sorted_dedup_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                                                   int bits, uint64_t* __restrict__ out,
                                                                   unsigned long long* __restrict__ counters) {
  extern __shared__ __align__(16) unsigned char sd_smem[];
  KeyT<W>* tab = reinterpret_cast<KeyT<W>*>(sd_smem);
  constexpr uint32_t TS = SDCfg<W>::TS;
  constexpr int IT = 8;  // keys per thread per round (all loads issued first)
  const uint32_t RND = IT * kHashThreads;
  __shared__ int s_zero;
  __shared__ uint32_t s_fill, s_first;
  const unsigned lane = lane_id();
  const uint64_t range = SDCfg<W>::RANGE;
  for (uint64_t r = blockIdx.x; r * range < n; r += gridDim.x) {
    const uint64_t lo = r * range, hi = std::min(n, lo + range);
    // first bucket start >= lo: skip the tail of the bucket that began before lo
    uint64_t pos = lo;
    if (lo > 0) {
      const uint32_t bprev = bucket_id<W>(load_key<W>(keys, lo - 1), bits);
      for (;;) {
        const uint64_t j = pos + threadIdx.x;
        const bool same = j < n && bucket_id<W>(load_key<W>(keys, j), bits) == bprev;
        const int c = __syncthreads_count(same);
        pos += c;
        if (c < (int)blockDim.x || pos >= hi) break;
      }
    }
    while (pos < hi) {
      const uint32_t b = bucket_id<W>(load_key<W>(keys, pos), bits);
      bool fresh = true;
      for (;;) {
        KeyT<W> k[IT];
        bool inb[IT];
#pragma unroll
        for (int u = 0; u < IT; u++) {
          const uint64_t j = pos + (uint64_t)u * kHashThreads + threadIdx.x;
          if (j < n) k[u] = load_key<W>(keys, j);
        }
        if (fresh) {
          for (uint32_t i = threadIdx.x; i < TS; i += blockDim.x) tab[i] = KeyT<W>{};
          if (threadIdx.x == 0) {
            s_zero = 0;
            s_fill = 0;
          }
          fresh = false;
        }
        if (threadIdx.x == 0) s_first = RND;
        __syncthreads();
#pragma unroll
        for (int u = 0; u < IT; u++) {
          const uint64_t j = pos + (uint64_t)u * kHashThreads + threadIdx.x;
          inb[u] = j < n && bucket_id<W>(k[u], bits) == b;
          if (!inb[u]) atomicMin(&s_first, (uint32_t)(u * kHashThreads + threadIdx.x));
        }
#pragma unroll
        for (int u = 0; u < IT; u++) {
          const bool keep = inb[u] && table_insert<W>(tab, k[u], &s_zero, &s_fill);
          const unsigned bal = __ballot_sync(kFull, keep);
          if (bal) {
            unsigned long long wb = 0;
            if (lane == 0) wb = atomicAdd(&counters[0], (unsigned long long)__popc(bal));
            wb = __shfl_sync(kFull, wb, 0);
            if (keep) store_key<W>(out, wb + __popc(bal & lanemask_lt()), k[u]);
          }
        }
        __syncthreads();
        const uint32_t c = s_first;
        pos += c;
        if (c < RND) break;
        if (s_fill > SDCfg<W>::FILL_LIMIT) {  // too many distinct keys: restart the table
          fresh = true;
          if (threadIdx.x == 0) atomicAdd(&counters[1], 1ull);
        }
        __syncthreads();
      }
      __syncthreads();
    }
  }
}

int nccl_check(cusci_ctx* ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return CUSCI_OK;
  ctx->broken = true;
  if (ctx->comm) ncclCommAbort(ctx->comm);
  ctx->comm = nullptr;
  return set_error(ctx, CUSCI_E_NCCL, "%s: %s", what, ncclGetErrorString(r));
}

// agree on a status code across ranks (max); returns the agreed code
int agree_status(cusci_ctx* ctx, int local) {
  if (ctx->world == 1) return local;
  Scratch s(ctx);
  int* d;
  if (s.get_t(1, &d) != CUSCI_OK) return CUSCI_E_OOM;
  *(int*)ctx->host_pinned = local;
  CUSCI_CUDA(ctx, cudaMemcpyAsync(d, ctx->host_pinned, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  CUSCI_TRY(nccl_check(ctx, ncclAllReduce(d, d, 1, ncclInt32, ncclMax, ctx->comm, ctx->stream), "status allreduce"));
  CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return *(int*)ctx->host_pinned;
}

// local unique filter (a8) + owner partition (a9): survivors of the bucket
// dedup, grouped into contiguous owner bins (P > 1: one onesweep pass with
// digit = owner over the survivors only).  bins_out holds >= n keys.
template <int W>
int partition_impl(cusci_ctx* ctx, const uint64_t* configs, uint64_t n, int P, uint64_t* bins_out,
                   uint64_t* counts /*host [P]*/, uint64_t* total) {
  Scratch s(ctx);
  for (int r = 0; r < P; r++) counts[r] = 0;
  *total = 0;
  if (n == 0) return CUSCI_OK;
  // bucket bits: <= ~capacity/2 keys per bucket even with no redundancy
  const uint64_t per_bucket = (uint64_t)SDCfg<W>::TS / 2;
  int bits = 0;
  while ((n >> bits) > per_bucket && bits < 27) bits++;
  uint64_t *b0, *b1, *surv;
  unsigned long long* ctr;
  CUSCI_TRY(s.get_t(n * W, &b0));
  CUSCI_TRY(s.get_t(n * W, &b1));
  CUSCI_TRY(s.get_t(2, &ctr));
  CUSCI_CUDA(ctx, cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), ctx->stream));
  const uint64_t* sorted = configs;
  if (bits) {
    DigitSpecs specs{};
    // LSD over the top `bits` bits of the owner mix, <= 9 bits per pass
    const int npass = (bits + 8) / 9;
    const int per = (bits + npass - 1) / npass;
    for (int q = 0, lowbit = 64 - bits; q < npass; q++) {
      const int nb = std::min(per, 64 - lowbit);
      specs.d[specs.n++] = DigitSpec{1, lowbit, nb, 0u};
      lowbit += nb;
    }
    CUSCI_TRY(onesweep_passes(ctx, W, configs, b0, b1, n, specs, &sorted, nullptr));
  }
  surv = (P == 1) ? bins_out : ((sorted == b0) ? b1 : b0);
  static bool attr_set[3] = {false, false, false};
  if (!attr_set[W]) {
    CUSCI_CUDA(ctx, cudaFuncSetAttribute(sorted_dedup_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SDCfg<W>::SMEM));
    attr_set[W] = true;
  }
  const uint64_t nranges = (n + SDCfg<W>::RANGE - 1) / SDCfg<W>::RANGE;
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(nranges, (uint64_t)ctx->num_sms * 3));
  CUSCI_LAUNCH(ctx, PT_HASH, sorted_dedup_kernel<W><<<blocks, kHashThreads, SDCfg<W>::SMEM, ctx->stream>>>(sorted, n, bits, surv, ctr));
  uint64_t hc[2];
  CUSCI_TRY(read_u64(ctx, (const uint64_t*)ctr, hc, 2));
  *total = hc[0];
  if (P == 1) {
    counts[0] = hc[0];
    return CUSCI_OK;
  }
  // owner bins: one stable pass over the survivors with digit = owner
  DigitSpecs os{};
  int obits = 1;
  while ((1 << obits) < P) obits++;
  os.d[os.n++] = DigitSpec{2, 0, obits, (uint32_t)P};
  std::vector<uint64_t> h0((size_t)1 << obits);
  const uint64_t* binned = surv;
  uint64_t* spare = (surv == b0) ? b1 : b0;
  CUSCI_TRY(onesweep_passes(ctx, W, surv, bins_out, spare, hc[0], os, &binned, h0.data()));
  if (binned != bins_out && hc[0])
    CUSCI_CUDA(ctx, cudaMemcpyAsync(bins_out, binned, hc[0] * W * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  for (int r = 0; r < P; r++) counts[r] = h0[r];
  return CUSCI_OK;
}

int finalize_impl(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* keys, uint64_t n, bool keys_are_scratch_owned,
                  uint64_t* keys_mut, cusci_keys* out) {
  const int W = sp->words;
  out->keys = nullptr;
  out->count = 0;
  Scratch s(ctx);
  uint64_t *a, *b;
  if (keys_are_scratch_owned) {
    a = keys_mut;
  } else {
    CUSCI_TRY(s.get_t(std::max<uint64_t>(n, 1) * W, &a));
    if (n) CUSCI_CUDA(ctx, cudaMemcpyAsync(a, keys, n * W * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  CUSCI_TRY(s.get_t(std::max<uint64_t>(n, 1) * W, &b));
  uint64_t* sorted = a;
  CUSCI_TRY(radix_sort_keys(ctx, W, a, b, n, sp->m, &sorted));
  void* o = nullptr;
  CUSCI_TRY(out_alloc(ctx, std::max<uint64_t>(n, 1) * W * 8, &o));
  uint64_t* cnt;
  if (s.get_t(1, &cnt) != CUSCI_OK) {
    out_free(ctx, o);
    return CUSCI_E_OOM;
  }
  int rc = unique_sorted_keys(ctx, W, sorted, n, (uint64_t*)o, cnt);
  uint64_t u = 0;
  if (rc == CUSCI_OK) rc = read_u64(ctx, cnt, &u, 1);
  if (rc != CUSCI_OK) {
    out_free(ctx, o);
    return rc;
  }
  out->keys = (uint64_t*)o;
  out->count = u;
  return CUSCI_OK;
}

int dedup_args(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n, const void* out) {
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  CUSCI_TRY(check_space(ctx, sp));
  if (!out) return set_error(ctx, CUSCI_E_INVALID_ARG, "output is NULL");
  if (n && !configs) return set_error(ctx, CUSCI_E_INVALID_ARG, "configs is NULL");
  if (n >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "n must be < 2^32 per call");
  return CUSCI_OK;
}

}  // namespace
}  // namespace cusci

using namespace cusci;

extern "C" int dedup_partition(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n,
                               int n_owners, cusci_keys* bins, uint64_t* counts) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  CUSCI_TRY(dedup_args(ctx, sp, configs, n, bins));
  if (n_owners < 1 || n_owners > 512 || !counts) return set_error(ctx, CUSCI_E_INVALID_ARG, "bad n_owners/counts");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  const int W = sp->words;
  void* o = nullptr;
  CUSCI_TRY(out_alloc(ctx, std::max<uint64_t>(n, 1) * W * 8, &o));
  uint64_t total = 0;
  int rc = W == 1 ? partition_impl<1>(ctx, configs, n, n_owners, (uint64_t*)o, counts, &total)
                  : partition_impl<2>(ctx, configs, n, n_owners, (uint64_t*)o, counts, &total);
  if (rc != CUSCI_OK) {
    out_free(ctx, o);
    return rc;
  }
  bins->keys = (uint64_t*)o;
  bins->count = total;
  return CUSCI_OK;
}

extern "C" int dedup_finalize(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* keys, uint64_t n,
                              cusci_keys* unique_sorted) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  CUSCI_TRY(dedup_args(ctx, sp, keys, n, unique_sorted));
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  return finalize_impl(ctx, sp, keys, n, false, nullptr, unique_sorted);
}

extern "C" int dedup_global(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n,
                            cusci_keys* owned_unique) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  int rc = dedup_args(ctx, sp, configs, n, owned_unique);
  if (ctx->broken) return rc;
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  rc = agree_status(ctx, rc);  // collective: failing ranks still take part
  if (rc != CUSCI_OK) {
    if (ctx->err.empty()) set_error(ctx, rc, "dedup_global: a peer rank rejected its arguments");
    return rc;
  }
  const int W = sp->words;
  const int P = ctx->world;
  Scratch s(ctx);
  uint64_t* bins;
  CUSCI_TRY(s.get_t(std::max<uint64_t>(n, 1) * W, &bins));
  uint64_t send[512], recv[512];
  uint64_t total = 0;
  CUSCI_TRY(W == 1 ? partition_impl<1>(ctx, configs, n, P, bins, send, &total)
                   : partition_impl<2>(ctx, configs, n, P, bins, send, &total));
  if (P == 1) return finalize_impl(ctx, sp, bins, total, true, bins, owned_unique);
  // ---- a10: counts exchange, then payload all-to-all-v over NCCL
  uint64_t *dsend, *drecv;
  CUSCI_TRY(s.get_t(P, &dsend));
  CUSCI_TRY(s.get_t(P, &drecv));
  memcpy(ctx->host_pinned, send, P * sizeof(uint64_t));
  CUSCI_CUDA(ctx, cudaMemcpyAsync(dsend, ctx->host_pinned, P * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  CUSCI_TRY(nccl_check(ctx, ncclGroupStart(), "group start"));
  for (int r = 0; r < P; r++) {
    CUSCI_TRY(nccl_check(ctx, ncclSend(dsend + r, 1, ncclUint64, r, ctx->comm, ctx->stream), "count send"));
    CUSCI_TRY(nccl_check(ctx, ncclRecv(drecv + r, 1, ncclUint64, r, ctx->comm, ctx->stream), "count recv"));
  }
  CUSCI_TRY(nccl_check(ctx, ncclGroupEnd(), "group end"));
  CUSCI_TRY(read_u64(ctx, drecv, recv, P));
  uint64_t nrecv = 0, soff[512], roff[512];
  {
    uint64_t a = 0;
    for (int r = 0; r < P; r++) {
      soff[r] = a;
      a += send[r];
      roff[r] = nrecv;
      nrecv += recv[r];
    }
  }
  uint64_t* rbuf;
  CUSCI_TRY(s.get_t(std::max<uint64_t>(nrecv, 1) * W, &rbuf));
  Prof pf_x(ctx, PT_NCCL);
  CUSCI_TRY(nccl_check(ctx, ncclGroupStart(), "group start"));
  for (int r = 0; r < P; r++) {
    if (r == ctx->rank) continue;
    if (send[r])
      CUSCI_TRY(nccl_check(ctx, ncclSend(bins + soff[r] * W, send[r] * W, ncclUint64, r, ctx->comm, ctx->stream), "send"));
    if (recv[r])
      CUSCI_TRY(nccl_check(ctx, ncclRecv(rbuf + roff[r] * W, recv[r] * W, ncclUint64, r, ctx->comm, ctx->stream), "recv"));
  }
  CUSCI_TRY(nccl_check(ctx, ncclGroupEnd(), "group end"));
  if (send[ctx->rank])
    CUSCI_CUDA(ctx, cudaMemcpyAsync(rbuf + roff[ctx->rank] * W, bins + soff[ctx->rank] * W, send[ctx->rank] * W * 8,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
  return finalize_impl(ctx, sp, rbuf, nrecv, true, rbuf, owned_unique);
}
