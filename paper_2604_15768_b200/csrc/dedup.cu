// dedup_global: distributed de-duplication of configuration keys
// (Sec 2.2, Sec 4.1.1 :448-462,
// Sec 3 :380-382 "local uniqueness filtering is applied immediately after
// generation").
//
// B200 design:
//   a8+a9  one kernel: open-addressing hash filter (load <= 0.5, empty slot = 0,
//          64-bit atomicCAS for W=1, 128-bit atom.cas.b128 for W=2) keeps the
//          first copy of each key; survivors are appended with one warp-
//          aggregated atomic per warp step, and per-owner counts are
//          accumulated (owner(j) = floor(mix(j) P / 2^64), DESIGN.md r9)
//          with match_any aggregation; a scatter kernel then writes the
//          survivors into P contiguous owner bins.
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

__device__ __forceinline__ void cas128(uint64_t* addr, uint64_t c0, uint64_t c1, uint64_t v0, uint64_t v1,
                                       uint64_t& o0, uint64_t& o1) {
  asm volatile(
      "{\n\t.reg .b128 c, v, o;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.global.cas.b128 o, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(o0), "=l"(o1)
      : "l"(c0), "l"(c1), "l"(v0), "l"(v1), "l"(addr)
      : "memory");
}

// returns true iff this thread inserted k (first copy)
__device__ __forceinline__ bool hash_insert(uint64_t* table, uint64_t mask, const KeyT<1>& k) {
  uint64_t slot = slot_hash(k) & mask;
  for (;;) {
    uint64_t cur = __ldcg(table + slot);
    if (cur == k.w0) return false;
    if (cur == 0) {
      const uint64_t old = atomicCAS((unsigned long long*)(table + slot), 0ull, (unsigned long long)k.w0);
      if (old == 0) return true;
      if (old == k.w0) return false;
    }
    slot = (slot + 1) & mask;
  }
}

__device__ __forceinline__ bool hash_insert(uint64_t* table, uint64_t mask, const KeyT<2>& k) {
  uint64_t slot = slot_hash(k) & mask;
  for (;;) {
    const ulonglong2 cur = __ldcg(reinterpret_cast<const ulonglong2*>(table) + slot);
    if (cur.x == k.w0 && cur.y == k.w1) return false;
    if (cur.x == 0 && cur.y == 0) {
      uint64_t o0, o1;
      cas128(table + 2 * slot, 0, 0, k.w0, k.w1, o0, o1);
      if (o0 == 0 && o1 == 0) return true;
      if (o0 == k.w0 && o1 == k.w1) return false;
    }
    slot = (slot + 1) & mask;
  }
}

template <int W>
__global__ void __launch_bounds__(kHashThreads) hash_filter_kernel(const uint64_t* __restrict__ in, uint64_t n,
                                                                  uint64_t* __restrict__ table, uint64_t mask,
                                                                  uint64_t* __restrict__ out,
                                                                  unsigned long long* __restrict__ counters,
                                                                  uint32_t n_owners) {
  // counters[0] = survivors, counters[1 + r] = survivors owned by r
  const unsigned lane = lane_id();
  const uint64_t warp_global = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = warp_global * 32; base < n; base += nwarps * 32) {
    const uint64_t idx = base + lane;
    bool keep = false;
    KeyT<W> k{};
    if (idx < n) {
      k = load_key<W>(in, idx);
      keep = hash_insert(table, mask, k);
    }
    const unsigned bal = __ballot_sync(kFull, keep);
    if (bal == 0) continue;
    unsigned long long wbase = 0;
    if (lane == 0) wbase = atomicAdd(&counters[0], (unsigned long long)__popc(bal));
    wbase = __shfl_sync(kFull, wbase, 0);
    if (keep) store_key<W>(out, wbase + __popc(bal & lanemask_lt()), k);
    if (n_owners > 1) {
      const uint32_t o = keep ? owner_of<W>(k, n_owners) : 0xffffffffu;
      const unsigned peers = __match_any_sync(kFull, o);
      if (keep && lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(&counters[1 + o], (unsigned long long)__popc(peers));
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kHashThreads) owner_scatter_kernel(const uint64_t* __restrict__ in, uint64_t n,
                                                                    uint64_t* __restrict__ bins,
                                                                    unsigned long long* __restrict__ cursor,
                                                                    uint32_t n_owners) {
  const unsigned lane = lane_id();
  const uint64_t warp_global = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t base = warp_global * 32; base < n; base += nwarps * 32) {
    const uint64_t idx = base + lane;
    const bool valid = idx < n;
    KeyT<W> k{};
    uint32_t o = 0xffffffffu;
    if (valid) {
      k = load_key<W>(in, idx);
      o = owner_of<W>(k, n_owners);
    }
    const unsigned peers = __match_any_sync(kFull, o);
    const unsigned leader = __ffs(peers) - 1;
    unsigned long long b = 0;
    if (valid && lane == leader) b = atomicAdd(&cursor[o], (unsigned long long)__popc(peers));
    b = __shfl_sync(kFull, b, leader);
    if (valid) store_key<W>(bins, b + __popc(peers & lanemask_lt()), k);
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

template <int W>
int partition_impl(cusci_ctx* ctx, const uint64_t* configs, uint64_t n, int P, uint64_t* bins_out /*[n][W] device*/,
                   uint64_t* counts /*host [P]*/, uint64_t* total) {
  Scratch s(ctx);
  uint64_t cap = 1024;
  while (cap < 2 * n) cap <<= 1;
  uint64_t* table;
  unsigned long long* ctr;
  CUSCI_TRY(s.get_t(cap * W, &table));
  CUSCI_TRY(s.get_t(1 + P, &ctr));
  {
    Prof pf(ctx, PT_MEMSET);
    CUSCI_CUDA(ctx, cudaMemsetAsync(table, 0, cap * W * sizeof(uint64_t), ctx->stream));
  }
  CUSCI_CUDA(ctx, cudaMemsetAsync(ctr, 0, (1 + P) * sizeof(unsigned long long), ctx->stream));
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + kHashThreads - 1) / kHashThreads,
                                                                             (uint64_t)ctx->num_sms * 8));
  uint64_t* surv = bins_out;
  if (P > 1) CUSCI_TRY(s.get_t(n * W, &surv));
  CUSCI_LAUNCH(ctx, PT_HASH, hash_filter_kernel<W><<<blocks, kHashThreads, 0, ctx->stream>>>(configs, n, table, cap - 1, surv, ctr, (uint32_t)P));
  uint64_t hc[1 + 512];
  CUSCI_TRY(read_u64(ctx, (const uint64_t*)ctr, hc, 1 + P));
  *total = hc[0];
  if (P == 1) {
    counts[0] = hc[0];
    return CUSCI_OK;
  }
  uint64_t off = 0;
  for (int r = 0; r < P; r++) {
    counts[r] = hc[1 + r];
    ((uint64_t*)ctx->host_pinned)[r] = off;
    off += hc[1 + r];
  }
  CUSCI_CUDA(ctx, cudaMemcpyAsync(ctr, ctx->host_pinned, P * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  const uint64_t ns = hc[0];
  if (ns) {
    const unsigned b2 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((ns + kHashThreads - 1) / kHashThreads,
                                                                           (uint64_t)ctx->num_sms * 8));
    CUSCI_LAUNCH(ctx, PT_SCATTER, owner_scatter_kernel<W><<<b2, kHashThreads, 0, ctx->stream>>>(surv, ns, bins_out, ctr, (uint32_t)P));
  }
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
