// dedup_global: distributed de-duplication of configuration keys
// (Sec 2.2, Sec 4.1.1 :448-462,
// Sec 3 :380-382 "local uniqueness filtering is applied immediately after
// generation").
//
// B200 design (readings r9/r13):
//   a8+a9  local_dedup (bucket.cu): the keys are mapped to their hash-order
//          values pi, MSD-partitioned by the top bits of hi and de-duplicated
//          bucket by bucket in shared memory; the result is unique and sorted
//          in pi, which is owner-major (owner(j) = floor(hi P / 2^64)), so the
//          owner bins are contiguous ranges (P binary searches);
//   a10    one count exchange that also carries every rank's status (a rank
//          that failed sends a failure marker, all ranks return the agreed
//          error), then one payload all-to-all-v over NCCL grouped
//          ncclSend/ncclRecv (NVLink/NVSwitch);
//   a11    the owner de-duplicates the P received runs into pi order.
// With one rank the local dedup is the whole job (no communicator needed);
// CUSCI_OPT_FORCE_COLLECTIVE runs the full protocol on a 1-rank communicator.
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

// agree on a status code across ranks (max); returns the agreed code.  Uses
// the context's persistent device words, so it cannot fail for lack of memory.
int agree_status(cusci_ctx* ctx, int local) {
  if (!collective(ctx)) return local;
  int* d = reinterpret_cast<int*>(ctx->dcomm + 2 * CUSCI_MAX_WORLD);
  *(int*)ctx->host_pinned = local;
  CUSCI_CUDA(ctx, cudaMemcpyAsync(d, ctx->host_pinned, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  CUSCI_TRY(nccl_check(ctx, ncclAllReduce(d, d, 1, ncclInt32, ncclMax, ctx->comm, ctx->stream), "status allreduce"));
  CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return *(int*)ctx->host_pinned;
}

// a failing rank's count words: kFailMark | code
constexpr uint64_t kFailMark = 0xFA11000000000000ull;

}  // namespace

// a10: counts exchange (carrying every rank's local status), then payload
// all-to-all-v over NCCL grouped send/recv (bins back to back by destination,
// send[r] keys for rank r); the received runs land back to back by source
// rank in *rbuf (from s).  Host syncs: one for the counts (+ status), one
// tiny status all-reduce after the receive buffer is reserved (a local
// allocation failure must not leave a peer blocked in the payload exchange).
int exchange_bins(cusci_ctx* ctx, int W, const uint64_t* bins, const uint64_t* send, Scratch& s, uint64_t** rbuf_out,
                  uint64_t* nrecv_out, int local_rc, uint64_t* recv_counts) {
  const int P = ctx->world;
  *rbuf_out = nullptr;
  *nrecv_out = 0;
  if (!ctx->comm) return set_error(ctx, CUSCI_E_INVALID_ARG, "exchange without a communicator");
  uint64_t* dsend = ctx->dcomm;
  uint64_t* drecv = ctx->dcomm + CUSCI_MAX_WORLD;
  uint64_t* hp = reinterpret_cast<uint64_t*>(ctx->host_pinned);
  for (int r = 0; r < P; r++) hp[r] = local_rc == CUSCI_OK ? send[r] : (kFailMark | (uint64_t)local_rc);
  CUSCI_CUDA(ctx, cudaMemcpyAsync(dsend, hp, P * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  CUSCI_TRY(nccl_check(ctx, ncclGroupStart(), "group start"));
  for (int r = 0; r < P; r++) {
    CUSCI_TRY(nccl_check(ctx, ncclSend(dsend + r, 1, ncclUint64, r, ctx->comm, ctx->stream), "count send"));
    CUSCI_TRY(nccl_check(ctx, ncclRecv(drecv + r, 1, ncclUint64, r, ctx->comm, ctx->stream), "count recv"));
  }
  CUSCI_TRY(nccl_check(ctx, ncclGroupEnd(), "group end"));
  uint64_t recv[CUSCI_MAX_WORLD];
  CUSCI_TRY(read_u64(ctx, drecv, recv, P));
  int agreed = local_rc;
  for (int r = 0; r < P; r++)
    if ((recv[r] & 0xFFFF000000000000ull) == kFailMark) agreed = std::max(agreed, (int)(recv[r] & 0xffff));
  if (agreed != CUSCI_OK) {
    if (local_rc == CUSCI_OK) set_error(ctx, agreed, "collective call failed on a peer rank (code %d)", agreed);
    return agreed;
  }
  uint64_t nrecv = 0, soff[CUSCI_MAX_WORLD], roff[CUSCI_MAX_WORLD];
  {
    uint64_t a = 0;
    for (int r = 0; r < P; r++) {
      soff[r] = a;
      a += send[r];
      roff[r] = nrecv;
      nrecv += recv[r];
    }
  }
  uint64_t* rbuf = nullptr;
  const int arc = s.get_t(std::max<uint64_t>(nrecv, 1) * W, &rbuf);
  const int rc2 = agree_status(ctx, arc);
  if (rc2 != CUSCI_OK) {
    if (arc == CUSCI_OK) set_error(ctx, rc2, "collective call failed on a peer rank (code %d)", rc2);
    return rc2;
  }
  // the own bin: a device copy, or through NCCL (to self) when the collective
  // protocol is forced on a 1-rank communicator
  const bool self_nccl = ctx->force_collective != 0;
  {
    Prof pf_x(ctx, PT_NCCL);
    CUSCI_TRY(nccl_check(ctx, ncclGroupStart(), "group start"));
    for (int r = 0; r < P; r++) {
      if (r == ctx->rank && !self_nccl) continue;
      if (send[r])
        CUSCI_TRY(nccl_check(ctx, ncclSend(bins + soff[r] * W, send[r] * W, ncclUint64, r, ctx->comm, ctx->stream), "send"));
      if (recv[r])
        CUSCI_TRY(nccl_check(ctx, ncclRecv(rbuf + roff[r] * W, recv[r] * W, ncclUint64, r, ctx->comm, ctx->stream), "recv"));
    }
    CUSCI_TRY(nccl_check(ctx, ncclGroupEnd(), "group end"));
  }
  if (!self_nccl && send[ctx->rank])
    CUSCI_CUDA(ctx, cudaMemcpyAsync(rbuf + roff[ctx->rank] * W, bins + soff[ctx->rank] * W, send[ctx->rank] * W * 8,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
  if (recv_counts)
    for (int r = 0; r < P; r++) recv_counts[r] = recv[r];
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

}  // namespace

int dedup_local_bins(cusci_ctx* ctx, int W, const uint64_t* configs, uint64_t n, int P, uint64_t* bins,
                     uint64_t* counts, uint64_t* total) {
  return W == 1 ? partition_impl<1>(ctx, configs, n, P, bins, counts, total)
                : partition_impl<2>(ctx, configs, n, P, bins, counts, total);
}

namespace {

// a11 at the owner over P received runs (each strictly increasing in pi):
// bucket-wise unique straight from the runs (runs_dedup), no partition pass
int finalize_runs(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* rbuf, const uint64_t* counts, int P,
                  uint64_t nrecv, cusci_keys* out) {
  const int W = sp->words;
  out->keys = nullptr;
  out->count = 0;
  void* o = nullptr;
  CUSCI_TRY(out_alloc(ctx, std::max<uint64_t>(nrecv, 1) * W * 8, &o));
  uint64_t u = 0;
  const int rc = runs_dedup(ctx, W, rbuf, counts, P, (uint64_t*)o, &u);
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
  if (n_owners < 1 || n_owners > CUSCI_MAX_WORLD || !counts) return set_error(ctx, CUSCI_E_INVALID_ARG, "bad n_owners/counts");
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

extern "C" int dedup_finalize_runs(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* keys,
                                   const uint64_t* run_counts, int n_runs, cusci_keys* unique_sorted) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  if (n_runs < 1 || n_runs > CUSCI_MAX_WORLD || !run_counts)
    return set_error(ctx, CUSCI_E_INVALID_ARG, "bad n_runs/run_counts");
  uint64_t n = 0;
  for (int r = 0; r < n_runs; r++) n += run_counts[r];
  CUSCI_TRY(dedup_args(ctx, sp, keys, n, unique_sorted));
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  return finalize_runs(ctx, sp, keys, run_counts, n_runs, n, unique_sorted);
}

extern "C" int dedup_global(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n,
                            cusci_keys* owned_unique) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  int rc = dedup_args(ctx, sp, configs, n, owned_unique);
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  if (owned_unique) {
    owned_unique->keys = nullptr;
    owned_unique->count = 0;
  }
  if (!collective(ctx)) {  // one rank: the local dedup is the whole job, straight into the output
    if (rc != CUSCI_OK) return rc;
    return finalize_impl(ctx, sp, configs, n, owned_unique);
  }
  // collective protocol: a rank that fails anywhere before the payload moves
  // still takes part in the count exchange, which carries its status
  const int P = ctx->world;
  const int W = rc == CUSCI_OK ? sp->words : 1;
  Scratch s(ctx);
  uint64_t* bins = nullptr;
  uint64_t send[CUSCI_MAX_WORLD] = {0};
  uint64_t total = 0;
  if (rc == CUSCI_OK) rc = s.get_t(std::max<uint64_t>(n, 1) * W, &bins);
  if (rc == CUSCI_OK)
    rc = W == 1 ? partition_impl<1>(ctx, configs, n, P, bins, send, &total)
                : partition_impl<2>(ctx, configs, n, P, bins, send, &total);
  if (ctx->broken) return rc;  // CUDA/NCCL failure: the communicator is gone
  uint64_t* rbuf;
  uint64_t nrecv;
  uint64_t rcounts[CUSCI_MAX_WORLD];
  CUSCI_TRY(exchange_bins(ctx, W, bins, send, s, &rbuf, &nrecv, rc, rcounts));
  return finalize_runs(ctx, sp, rbuf, rcounts, P, nrecv, owned_unique);
}
