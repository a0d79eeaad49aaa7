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

}  // namespace

// a10: counts exchange, then payload all-to-all-v over NCCL grouped send/recv
// (bins back to back by destination, send[r] keys for rank r); the received
// runs land back to back by source rank in *rbuf (from s).
int exchange_bins(cusci_ctx* ctx, int W, const uint64_t* bins, const uint64_t* send, Scratch& s, uint64_t** rbuf_out,
                  uint64_t* nrecv_out) {
  const int P = ctx->world;
  uint64_t *dsend, *drecv, recv[512];
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
  *rbuf_out = rbuf;
  *nrecv_out = nrecv;
  return CUSCI_OK;
}

// collective status agreement (max over ranks)
int agree_status_all(cusci_ctx* ctx, int local) { return agree_status(ctx, local); }
int nccl_ok(cusci_ctx* ctx, ncclResult_t r, const char* what) { return nccl_check(ctx, r, what); }

namespace {

// local unique filter (a8) + owner partition (a9): the local dedup returns the
// distinct keys in the hash order, which is owner-major, so the owner bins are
// contiguous ranges (found by P binary searches).  bins_out holds >= n keys.
template <int W>
int partition_impl(cusci_ctx* ctx, const uint64_t* configs, uint64_t n, int P, uint64_t* bins_out,
                   uint64_t* counts /*host [P]*/, uint64_t* total) {
  for (int r = 0; r < P; r++) counts[r] = 0;
  *total = 0;
  CUSCI_TRY(local_dedup(ctx, W, configs, n, bins_out, total));
  if (P == 1) {
    counts[0] = *total;
    return CUSCI_OK;
  }
  return owner_counts(ctx, W, bins_out, *total, P, counts);
}

// a11 at the owner: dedup of the received runs (each locally unique) into the
// hash order; the output buffer comes from the context allocator
int finalize_impl(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* keys, uint64_t n, cusci_keys* out) {
  const int W = sp->words;
  out->keys = nullptr;
  out->count = 0;
  void* o = nullptr;
  CUSCI_TRY(out_alloc(ctx, std::max<uint64_t>(n, 1) * W * 8, &o));
  uint64_t u = 0;
  const int rc = local_dedup(ctx, W, keys, n, (uint64_t*)o, &u);
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
  return finalize_impl(ctx, sp, keys, n, unique_sorted);
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
  if (P == 1) {  // the local dedup is the whole job: write straight into the output
    return finalize_impl(ctx, sp, configs, n, owned_unique);
  }
  Scratch s(ctx);
  uint64_t* bins;
  CUSCI_TRY(s.get_t(std::max<uint64_t>(n, 1) * W, &bins));
  uint64_t send[512], recv[512];
  uint64_t total = 0;
  CUSCI_TRY(W == 1 ? partition_impl<1>(ctx, configs, n, P, bins, send, &total)
                   : partition_impl<2>(ctx, configs, n, P, bins, send, &total));
  uint64_t* rbuf;
  uint64_t nrecv;
  CUSCI_TRY(exchange_bins(ctx, W, bins, send, s, &rbuf, &nrecv));
  return finalize_impl(ctx, sp, rbuf, nrecv, owned_unique);
}
