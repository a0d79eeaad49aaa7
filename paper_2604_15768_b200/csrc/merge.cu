// merge_space: S <- S u U on the GPU-resident pool shard (
// PAPER.md:311-312 Sec 2.2 "merging them into S", :404-405; abstract :167
// "GPU-side pooling").
//
// B200 design: merge path.  The merged sequence of
// S (sorted unique) and U (sorted unique), ties S-first, is cut into tiles of
// kTile outputs by a diagonal binary search per tile boundary; each CTA stages
// its S and U runs in shared memory, merges them (serial merge of ITEMS
// outputs per thread from one in-tile diagonal search), drops an element equal
// to its predecessor (an element of U already in S), and writes S' and
// inserted = U \ S with block-ordered compaction.  Two sweeps (count, write)
// with one scan of per-tile counts in between; S' is written to the pool's
// second buffer and the buffers are swapped (grown geometrically if needed).
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

template <int W>
__global__ void __launch_bounds__(kMergeThreads) merge_tile_kernel(const uint64_t* __restrict__ S, uint64_t nS,
                                                                  const uint64_t* __restrict__ U, uint64_t nU,
                                                                  const uint64_t* __restrict__ split, int write,
                                                                  uint64_t* __restrict__ cnt_keep,
                                                                  uint64_t* __restrict__ cnt_ins,
                                                                  const uint64_t* __restrict__ off_keep,
                                                                  const uint64_t* __restrict__ off_ins,
                                                                  uint64_t* __restrict__ out, uint64_t* __restrict__ ins) {
  constexpr int kMergeItems = MergeCfg<W>::ITEMS;
  constexpr int kTile = MergeCfg<W>::TILE;
  __shared__ KeyT<W> ab[kTile];     // S run then U run
  __shared__ KeyT<W> mrg[kTile];    // merged tile
  __shared__ uint8_t fromU[kTile];
  __shared__ uint32_t wk[kMergeThreads / 32], wi[kMergeThreads / 32];
  __shared__ uint64_t run_k, run_i;
  const uint64_t t = blockIdx.x;
  const uint64_t i0 = split[t], i1 = split[t + 1];
  const uint64_t d0 = t * kTile, d1 = std::min<uint64_t>(d0 + kTile, nS + nU);
  const uint64_t j0 = d0 - i0, j1 = d1 - i1;
  const int na = (int)(i1 - i0), nb = (int)(j1 - j0), len = na + nb;
  for (int x = threadIdx.x; x < na; x += kMergeThreads) ab[x] = load_key<W>(S, i0 + x);
  for (int x = threadIdx.x; x < nb; x += kMergeThreads) ab[na + x] = load_key<W>(U, j0 + x);
  __syncthreads();
  const KeyT<W>* A = ab;
  const KeyT<W>* B = ab + na;
  // each thread merges outputs [k0, k0 + ITEMS)
  const int k0 = threadIdx.x * kMergeItems;
  if (k0 < len) {
    int lo = k0 > nb ? k0 - nb : 0, hi = std::min(k0, na);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (hk_le<W>(A[mid], B[k0 - mid - 1])) lo = mid + 1;
      else hi = mid;
    }
    int i = lo, j = k0 - lo;
    for (int k = k0; k < std::min(k0 + kMergeItems, len); k++) {
      const bool takeA = i < na && (j >= nb || hk_le<W>(A[i], B[j]));
      if (takeA) {
        mrg[k] = A[i++];
        fromU[k] = 0;
      } else {
        mrg[k] = B[j++];
        fromU[k] = 1;
      }
    }
  }
  // predecessor of the tile's first output: the larger of S[i0-1], U[j0-1]
  KeyT<W> prev0{};
  bool has_prev0 = false;
  if (i0 > 0) {
    prev0 = load_key<W>(S, i0 - 1);
    has_prev0 = true;
  }
  if (j0 > 0) {
    const KeyT<W> u = load_key<W>(U, j0 - 1);
    if (!has_prev0 || hk_lt<W>(prev0, u)) prev0 = u;
    has_prev0 = true;
  }
  if (threadIdx.x == 0) {
    run_k = write ? off_keep[t] : 0;
    run_i = write ? off_ins[t] : 0;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  uint32_t ck = 0, ci = 0;
  for (int r = 0; r < kMergeItems; r++) {
    const int k = r * kMergeThreads + threadIdx.x;
    bool keep = false, isins = false;
    if (k < len) {
      const bool dup = k > 0 ? key_eq(mrg[k], mrg[k - 1]) : (has_prev0 && key_eq(mrg[0], prev0));
      keep = !dup;
      isins = keep && fromU[k];
    }
    if (!write) {
      ck += keep;
      ci += isins;
      continue;
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
    if (keep) store_key<W>(out, run_k + ok + __popc(bk & lanemask_lt()), mrg[k]);
    if (isins && ins) store_key<W>(ins, run_i + oi + __popc(bi & lanemask_lt()), mrg[k]);
    __syncthreads();
    if (threadIdx.x == 0) {
      run_k += tk;
      run_i += ti;
    }
    __syncthreads();
  }
  if (!write) {
    for (int o = 16; o; o >>= 1) {
      ck += __shfl_xor_sync(kFull, ck, o);
      ci += __shfl_xor_sync(kFull, ci, o);
    }
    if (lane_id() == 0) {
      wk[w] = ck;
      wi[w] = ci;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t a = 0, b = 0;
      for (int x = 0; x < kMergeThreads / 32; x++) {
        a += wk[x];
        b += wi[x];
      }
      cnt_keep[t] = a;
      cnt_ins[t] = b;
    }
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
  if (nU > 1) {
    int* flag;
    CUSCI_TRY(s.get_t(1, &flag));
    CUSCI_CUDA(ctx, cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    const unsigned blocks = (unsigned)std::min<uint64_t>((nU + 255) / 256, (uint64_t)ctx->num_sms * 8);
    CUSCI_LAUNCH(ctx, PT_CHECK, check_sorted_kernel<W><<<blocks, 256, 0, ctx->stream>>>(U, nU, flag));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (*(int*)ctx->host_pinned)
      return set_error(ctx, CUSCI_E_INVALID_ARG, "merge_space: new_keys must be sorted ascending and unique");
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
  uint64_t *split, *ck, *ci, *ok, *oi, *tot;
  CUSCI_TRY(s.get_t(ntiles + 1, &split));
  CUSCI_TRY(s.get_t(ntiles, &ck));
  CUSCI_TRY(s.get_t(ntiles, &ci));
  CUSCI_TRY(s.get_t(ntiles, &ok));
  CUSCI_TRY(s.get_t(ntiles, &oi));
  CUSCI_TRY(s.get_t(2, &tot));
  CUSCI_LAUNCH(ctx, PT_MERGE_SPLIT, merge_split_kernel<W><<<(unsigned)((ntiles + 1 + 255) / 256), 256, 0, ctx->stream>>>(S, nS, U, nU, ntiles, split));
  CUSCI_LAUNCH(ctx, PT_MERGE_TILE, merge_tile_kernel<W><<<(unsigned)ntiles, kMergeThreads, 0, ctx->stream>>>(S, nS, U, nU, split, 0, ck, ci, nullptr,
                                                                           nullptr, nullptr, nullptr));
  CUSCI_TRY(scan_exclusive_u64(ctx, ck, ok, ntiles, tot));
  CUSCI_TRY(scan_exclusive_u64(ctx, ci, oi, ntiles, tot + 1));
  uint64_t h[2];
  CUSCI_TRY(read_u64(ctx, tot, h, 2));
  const uint64_t n_new = h[0], n_ins = h[1];
  // destination buffer (grow geometrically)
  uint64_t* dst = pool->buf[1 - pool->cur];
  uint64_t* old_bufs[2] = {nullptr, nullptr};
  if (n_new > pool->cap) {
    uint64_t ncap = std::max<uint64_t>(pool->cap * 2, n_new + n_new / 4);
    uint64_t* nb[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; b++) {
      if (cudaMallocFromPoolAsync((void**)&nb[b], ncap * W * 8, ctx->pool, ctx->stream) != cudaSuccess) {
        cudaGetLastError();
        if (nb[0]) cudaFreeAsync(nb[0], ctx->stream);
        return set_error(ctx, CUSCI_E_OOM, "pool growth to %llu keys failed", (unsigned long long)ncap);
      }
    }
    old_bufs[0] = pool->buf[0];
    old_bufs[1] = pool->buf[1];
    pool->buf[0] = nb[0];
    pool->buf[1] = nb[1];
    pool->cap = ncap;
    pool->cur = 1;  // S still lives in the old buffer; write into buf[0]
    dst = pool->buf[0];
  }
  void* insp = nullptr;
  if (inserted) CUSCI_TRY(out_alloc(ctx, std::max<uint64_t>(n_ins, 1) * W * 8, &insp));
  CUSCI_LAUNCH(ctx, PT_MERGE_TILE, merge_tile_kernel<W><<<(unsigned)ntiles, kMergeThreads, 0, ctx->stream>>>(S, nS, U, nU, split, 1, nullptr, nullptr,
                                                                           ok, oi, dst, (uint64_t*)insp));
  for (int b = 0; b < 2; b++)
    if (old_bufs[b]) cudaFreeAsync(old_bufs[b], ctx->stream);
  pool->cur = (dst == pool->buf[0]) ? 0 : 1;
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
