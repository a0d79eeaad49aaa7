// merge_space: S <- S u U on the GPU-resident pool shard (
// PAPER.md:311-312 Sec 2.2 "merging them into S", :404-405; abstract :167
// "GPU-side pooling").
//
// B200 design: merge path in the pool (hash) order
// (reading r13).  The merged sequence of S (sorted unique) and U (sorted
// unique), ties S-first, is cut into tiles of kTile outputs by a diagonal
// binary search per tile boundary; each CTA stages its S and U runs in shared
// memory, merges them (serial merge of ITEMS outputs per thread from one
// in-tile diagonal search), drops an element equal to its predecessor (an
// element of U already in S), validates U's order, and writes S' and
// inserted = U \ S at offsets found by decoupled look-back -- ONE sweep over
// S and U.  S' goes to the pool's second buffer (grown geometrically to the
// upper bound |S| + |U| when needed) and the buffers are swapped.
#include <algorithm>

#include "internal.cuh"

namespace cusci {
namespace {

constexpr int kMergeThreads = 256;
template <int W> struct MergeCfg {
  static constexpr int ITEMS = W == 1 ? 8 : 4;  // keeps static smem < 48 KB
  static constexpr int TILE = kMergeThreads * ITEMS;
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

// Single sweep: each CTA takes a tile ticket (predecessors are resident),
// merges its S and U runs in shared memory, drops an element equal to its
// predecessor, checks that its U run is strictly increasing in the hash order,
// publishes its (kept, inserted) counts and resolves its output offsets by
// decoupled look-back over its predecessors' published counts, then writes
// S' and inserted with block-ordered compaction.
constexpr uint64_t kMFlagA = 1ull << 62, kMFlagP = 2ull << 62, kMVal = (1ull << 62) - 1;

template <int W>
__global__ void __launch_bounds__(kMergeThreads) merge_tile_kernel(const uint64_t* __restrict__ S, uint64_t nS,
                                                                  const uint64_t* __restrict__ U, uint64_t nU,
                                                                  const uint64_t* __restrict__ split,
                                                                  unsigned long long* __restrict__ status,
                                                                  unsigned* __restrict__ tile_ctr,
                                                                  int* __restrict__ bad,
                                                                  uint64_t* __restrict__ out, uint64_t* __restrict__ ins) {
  constexpr int kMergeItems = MergeCfg<W>::ITEMS;
  constexpr int kTile = MergeCfg<W>::TILE;
  __shared__ KeyT<W> ab[kTile];     // S run then U run
  __shared__ uint64_t abh[kTile];   // their hash-order hi (computed once per element)
  __shared__ uint16_t mrg[kTile];   // merged tile as indices into ab (>= na: from U)
  __shared__ uint32_t wk[kMergeThreads / 32], wi[kMergeThreads / 32];
  __shared__ uint64_t run_k, run_i;
  __shared__ unsigned s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint64_t t = s_tile;
  const uint64_t i0 = split[t], i1 = split[t + 1];
  const uint64_t d0 = t * kTile, d1 = std::min<uint64_t>(d0 + kTile, nS + nU);
  const uint64_t j0 = d0 - i0, j1 = d1 - i1;
  // an unsorted U can make the merge-path splits inconsistent: flag it and
  // process nothing (the tile still publishes zero counts for its successors)
  const bool inval = i1 < i0 || j1 < j0 || (i1 - i0) + (j1 - j0) > (uint64_t)kTile || j1 > nU || i1 > nS;
  if (inval && threadIdx.x == 0) *bad = 1;
  const int na = inval ? 0 : (int)(i1 - i0), nb = inval ? 0 : (int)(j1 - j0), len = na + nb;
  for (int x = threadIdx.x; x < na; x += kMergeThreads) {
    const KeyT<W> k = load_key<W>(S, i0 + x);
    ab[x] = k;
    abh[x] = hk_hi(k);
  }
  for (int x = threadIdx.x; x < nb; x += kMergeThreads) {
    const KeyT<W> k = load_key<W>(U, j0 + x);
    ab[na + x] = k;
    abh[na + x] = hk_hi(k);
  }
  __syncthreads();
  // hash-order comparisons on the staged elements: hi first, lo only on a tie (W = 2)
  auto le = [&](int x, int y) -> bool {
    const uint64_t hx = abh[x], hy = abh[y];
    if (W == 1 || hx != hy) return hx <= hy;
    return hk_lo(ab[x]) <= hk_lo(ab[y]);
  };
  // input check: U strictly increasing in the hash order (tile run + left boundary)
  {
    bool badu = false;
    for (int x = threadIdx.x; x < nb; x += kMergeThreads) {
      if (x > 0) badu |= le(na + x, na + x - 1);
      else if (j0 > 0 && j0 <= nU) badu |= !hk_lt<W>(load_key<W>(U, j0 - 1), ab[na]);
    }
    if (badu) *bad = 1;
  }
  // each thread merges outputs [k0, k0 + ITEMS)
  const int k0 = threadIdx.x * kMergeItems;
  if (k0 < len) {
    int lo = k0 > nb ? k0 - nb : 0, hi = std::min(k0, na);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (le(mid, na + k0 - mid - 1)) lo = mid + 1;
      else hi = mid;
    }
    int i = lo, j = k0 - lo;
    for (int k = k0; k < std::min(k0 + kMergeItems, len); k++) {
      const bool takeA = i < na && (j >= nb || le(i, na + j));
      mrg[k] = (uint16_t)(takeA ? i++ : na + j++);
    }
  }
  // predecessor of the tile's first output: the larger of S[i0-1], U[j0-1]
  KeyT<W> prev0{};
  bool has_prev0 = false;
  if (!inval && i0 > 0) {
    prev0 = load_key<W>(S, i0 - 1);
    has_prev0 = true;
  }
  if (!inval && j0 > 0) {
    const KeyT<W> u = load_key<W>(U, j0 - 1);
    if (!has_prev0 || hk_lt<W>(prev0, u)) prev0 = u;
    has_prev0 = true;
  }
  __syncthreads();
  // tile counts
  const int w = threadIdx.x >> 5;
  uint32_t ck = 0, ci = 0;
  for (int r = 0; r < kMergeItems; r++) {
    const int k = r * kMergeThreads + threadIdx.x;
    if (k < len) {
      const bool dup = k > 0 ? key_eq(ab[mrg[k]], ab[mrg[k - 1]]) : (has_prev0 && key_eq(ab[mrg[0]], prev0));
      ck += !dup;
      ci += (!dup && mrg[k] >= na);
    }
  }
  for (int o = 16; o; o >>= 1) {
    ck += __shfl_xor_sync(kFull, ck, o);
    ci += __shfl_xor_sync(kFull, ci, o);
  }
  if (lane_id() == 0) {
    wk[w] = ck;
    wi[w] = ci;
  }
  __syncthreads();
  // publish + look-back (thread 0: kept, thread 32: inserted)
  volatile unsigned long long* st = status;
  if (threadIdx.x == 0 || threadIdx.x == 32) {
    const int which = threadIdx.x == 0 ? 0 : 1;
    uint64_t mine = 0;
    for (int x = 0; x < kMergeThreads / 32; x++) mine += which ? wi[x] : wk[x];
    st[2 * t + which] = (t == 0 ? kMFlagP : kMFlagA) | mine;
    uint64_t excl = 0;
    if (t > 0) {
      int64_t q = (int64_t)t - 1;
      while (q >= 0) {
        const uint64_t v = st[2 * q + which];
        if ((v >> 62) == 0) {
          __nanosleep(20);
          continue;
        }
        excl += v & kMVal;
        if ((v >> 62) == 2) break;
        q--;
      }
      st[2 * t + which] = kMFlagP | (excl + mine);
    }
    if (which == 0) run_k = excl;
    else run_i = excl;
  }
  __syncthreads();
  for (int r = 0; r < kMergeItems; r++) {
    const int k = r * kMergeThreads + threadIdx.x;
    bool keep = false, isins = false;
    if (k < len) {
      const bool dup = k > 0 ? key_eq(ab[mrg[k]], ab[mrg[k - 1]]) : (has_prev0 && key_eq(ab[mrg[0]], prev0));
      keep = !dup;
      isins = keep && mrg[k] >= na;
    }
    const unsigned bk = __ballot_sync(kFull, keep), bi = __ballot_sync(kFull, isins);
    if (lane_id() == 0) {
      wk[w] = __popc(bk);
      wi[w] = __popc(bi);
    }
    __syncthreads();
    uint32_t ok = 0, oi = 0, tk = 0, ti = 0;
    for (int x = 0; x < kMergeThreads / 32; x++) {
      if (x < w) {
        ok += wk[x];
        oi += wi[x];
      }
      tk += wk[x];
      ti += wi[x];
    }
    if (keep) store_key<W>(out, run_k + ok + __popc(bk & lanemask_lt()), ab[mrg[k]]);
    if (isins && ins) store_key<W>(ins, run_i + oi + __popc(bi & lanemask_lt()), ab[mrg[k]]);
    __syncthreads();
    if (threadIdx.x == 0) {
      run_k += tk;
      run_i += ti;
    }
    __syncthreads();
  }
}

template <int W>
int merge_impl(cusci_ctx* ctx, cusci_pool* pool, const uint64_t* U, uint64_t nU, cusci_keys* inserted) {
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
  unsigned* tctr;
  int* bad;
  CUSCI_TRY(s.get_t(ntiles + 1, &split));
  CUSCI_TRY(s.get_t(2 * ntiles, &status));
  CUSCI_TRY(s.get_t(1, &tctr));
  CUSCI_TRY(s.get_t(1, &bad));
  CUSCI_CUDA(ctx, cudaMemsetAsync(status, 0, 2 * ntiles * sizeof(unsigned long long), ctx->stream));
  CUSCI_CUDA(ctx, cudaMemsetAsync(tctr, 0, sizeof(unsigned), ctx->stream));
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
  CUSCI_LAUNCH(ctx, PT_MERGE_SPLIT, merge_split_kernel<W><<<(unsigned)((ntiles + 1 + 255) / 256), 256, 0, ctx->stream>>>(S, nS, U, nU, ntiles, split));
  CUSCI_LAUNCH(ctx, PT_MERGE_TILE, merge_tile_kernel<W><<<(unsigned)ntiles, kMergeThreads, 0, ctx->stream>>>(S, nS, U, nU, split, status, tctr, bad, dst, (uint64_t*)insp));
  // totals = the last tile's inclusive counts; plus the input check flag
  uint64_t h[3];
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
  return space->sp.words == 1 ? merge_impl<1>(ctx, space, new_keys, n_new, inserted)
                              : merge_impl<2>(ctx, space, new_keys, n_new, inserted);
}
