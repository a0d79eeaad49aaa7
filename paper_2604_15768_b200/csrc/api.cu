// C-ABI lifecycle, errors, memory plumbing (include/cusci.h).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace cusci {

int set_error(cusci_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return code;
}

static void arena_release_all(cusci_ctx* ctx) {
  Arena& A = ctx->arena;
  for (auto& sg : A.segs) cudaFree(sg.base);
  A.segs.clear();
  A.cur = A.off = A.used = 0;
}

Scratch::Scratch(cusci_ctx* c) : ctx(c) {
  Arena& A = ctx->arena;
  if (A.depth == 0) {
    if (A.segs.size() > 1) {  // consolidate into one segment of the observed peak
      cudaStreamSynchronize(ctx->stream);
      arena_release_all(ctx);
      void* q = nullptr;
      if (cudaMalloc(&q, A.peak) == cudaSuccess) A.segs.push_back({(char*)q, A.peak});
      else cudaGetLastError();
    }
    A.cur = A.off = A.used = 0;
  }
  A.depth++;
  m_cur = A.cur;
  m_off = A.off;
  m_used = A.used;
}

Scratch::~Scratch() {
  Arena& A = ctx->arena;
  A.cur = m_cur;
  A.off = m_off;
  A.used = m_used;
  A.depth--;
}

int Scratch::get(size_t bytes, void** p) {
  Arena& A = ctx->arena;
  bytes = align256(bytes ? bytes : 256);
  while (A.cur < A.segs.size() && A.off + bytes > A.segs[A.cur].cap) {
    A.cur++;
    A.off = 0;
  }
  if (A.cur >= A.segs.size()) {
    size_t want = std::max(bytes, std::max(A.peak, (size_t)64 << 20));
    void* q = nullptr;
    if (cudaMalloc(&q, want) != cudaSuccess) {
      cudaGetLastError();
      want = bytes;
      if (cudaMalloc(&q, want) != cudaSuccess) {
        cudaGetLastError();
        return set_error(ctx, CUSCI_E_OOM, "scratch allocation of %zu bytes failed", bytes);
      }
    }
    A.segs.push_back({(char*)q, want});
    A.cur = A.segs.size() - 1;
    A.off = 0;
  }
  *p = A.segs[A.cur].base + A.off;
  A.off += bytes;
  A.used += bytes;
  if (A.used > A.peak) A.peak = A.used;
  return CUSCI_OK;
}

int out_alloc(cusci_ctx* ctx, size_t bytes, void** p) {
  if (bytes == 0) bytes = 256;
  void* q = nullptr;
  if (ctx->alloc) {
    q = ctx->alloc(bytes, (void*)ctx->stream, ctx->alloc_user);
  } else {
    cudaError_t e = cudaMallocFromPoolAsync(&q, bytes, ctx->pool, ctx->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      q = nullptr;
    }
  }
  if (!q) return set_error(ctx, CUSCI_E_OOM, "output allocation of %zu bytes failed", bytes);
  *p = q;
  return CUSCI_OK;
}

void out_free(cusci_ctx* ctx, void* p) {
  if (!p) return;
  if (ctx->free_fn) ctx->free_fn(p, ctx->alloc_user);
  else cudaFreeAsync(p, ctx->stream);
}

int check_space(cusci_ctx* ctx, const cusci_space* sp) {
  if (!sp) return set_error(ctx, CUSCI_E_INVALID_ARG, "space is NULL");
  if (sp->m < 2 || sp->m > 128 || (sp->m & 1))
    return set_error(ctx, CUSCI_E_INVALID_ARG, "m=%d not an even number in [2,128]", sp->m);
  int W = sp->m <= 64 ? 1 : 2;
  if (sp->words != W) return set_error(ctx, CUSCI_E_INVALID_ARG, "words=%d but m=%d needs %d", sp->words, sp->m, W);
  if (sp->n_alpha < 0 || sp->n_beta < 0 || sp->n_alpha > sp->m / 2 || sp->n_beta > sp->m / 2)
    return set_error(ctx, CUSCI_E_INVALID_ARG, "electron counts (%d,%d) invalid for m=%d", sp->n_alpha, sp->n_beta, sp->m);
  return CUSCI_OK;
}

int kernel_setup(cusci_ctx* ctx, const void* fn, int threads, size_t smem, int* per_sm) {
  for (const KSetup& k : ctx->ksetup)
    if (k.fn == fn && k.smem == smem && k.threads == threads) {
      *per_sm = k.per_sm;
      return CUSCI_OK;
    }
  // always opt in: static + dynamic shared memory above 48 KB needs it even
  // when the dynamic part alone is smaller
  if (smem) CUSCI_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CUSCI_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
  if (occ < 1) occ = 1;
  ctx->ksetup.push_back(KSetup{fn, smem, threads, occ});
  *per_sm = occ;
  return CUSCI_OK;
}

int read_u64(cusci_ctx* ctx, const uint64_t* dev, uint64_t* host, int count) {
  uint64_t* pinned = (uint64_t*)ctx->host_pinned;
  if (count < 0 || (size_t)count * sizeof(uint64_t) > kHostPinnedBytes)
    return set_error(ctx, CUSCI_E_INVALID_ARG, "read_u64 count too large");
  CUSCI_CUDA(ctx, cudaMemcpyAsync(pinned, dev, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  memcpy(host, pinned, sizeof(uint64_t) * count);
  return CUSCI_OK;
}

static cudaEvent_t ev_get(cusci_ctx* ctx) {
  if (!ctx->ev_free.empty()) {
    cudaEvent_t e = ctx->ev_free.back();
    ctx->ev_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

Prof::Prof(cusci_ctx* c, int t) : ctx(c), tag(t) {
  if (!ctx->profiling) return;
  a = ev_get(ctx);
  cudaEventRecord(a, ctx->stream);
}

Prof::~Prof() {
  if (!a) return;
  cudaEvent_t b = ev_get(ctx);
  cudaEventRecord(b, ctx->stream);
  ctx->prof.push_back(ProfRec{tag, a, b});
}

}  // namespace cusci

using namespace cusci;

extern "C" {

int cusci_nccl_unique_id(void* out128) {
  if (!out128) return CUSCI_E_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CUSCI_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  memcpy(out128, &id, sizeof(id));
  return CUSCI_OK;
}

int cusci_init(cusci_ctx** out, int device, int rank, int world, const void* nccl_unique_id, void* cuda_stream,
               cusci_alloc_fn alloc, cusci_free_fn free_fn, void* alloc_user) {
  if (!out) return CUSCI_E_INVALID_ARG;
  *out = nullptr;
  if (world < 1 || world > CUSCI_MAX_WORLD || rank < 0 || rank >= world) return CUSCI_E_INVALID_ARG;
  if (world > 1 && !nccl_unique_id) return CUSCI_E_INVALID_ARG;
  if ((alloc == nullptr) != (free_fn == nullptr)) return CUSCI_E_INVALID_ARG;
  cusci_ctx* ctx = new cusci_ctx;
  ctx->device = device;
  ctx->rank = rank;
  ctx->world = world;
  ctx->alloc = alloc;
  ctx->free_fn = free_fn;
  ctx->alloc_user = alloc_user;
  auto fail = [&](int code) {
    cusci_finalize(ctx);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return fail(CUSCI_E_CUDA);
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  // NULL = the legacy default stream (the one torch's current_stream() is by default);
  // every library call is ordered on this stream with the caller's own work.
  ctx->stream = (cudaStream_t)cuda_stream;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  if (cudaMemPoolCreate(&ctx->pool, &props) != cudaSuccess) return fail(CUSCI_E_CUDA);
  uint64_t thresh = UINT64_MAX;
  cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thresh);
  if (cudaMallocHost(&ctx->host_pinned, kHostPinnedBytes) != cudaSuccess) return fail(CUSCI_E_CUDA);
  if (nccl_unique_id) {  // world = 1 with an id: a 1-rank communicator (CUSCI_OPT_FORCE_COLLECTIVE)
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    if (ncclCommInitRank(&ctx->comm, world, id, rank) != ncclSuccess) {
      ctx->comm = nullptr;
      return fail(CUSCI_E_NCCL);
    }
    // persistent device words of the collective protocol (counts, status), so
    // the exchange never needs a scratch allocation that could fail on one rank
    if (cudaMalloc((void**)&ctx->dcomm, kCommWords * sizeof(uint64_t)) != cudaSuccess) return fail(CUSCI_E_CUDA);
  }
  *out = ctx;
  return CUSCI_OK;
}

static void prep_release(cusci_ctx* ctx) {
  if (ctx->prep.block) cudaFree(ctx->prep.block);
  ctx->prep = Prep{};
}

void cusci_finalize(cusci_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  prep_release(ctx);
  arena_release_all(ctx);
  if (ctx->comm) {
    if (ctx->broken) ncclCommAbort(ctx->comm);
    else ncclCommDestroy(ctx->comm);
  }
  for (auto& r : ctx->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ctx->ev_free) cudaEventDestroy(e);
  if (ctx->dcomm) cudaFree(ctx->dcomm);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
  if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* cusci_last_error(const cusci_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

int cusci_set_option(cusci_ctx* ctx, int option, int64_t value) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  switch (option) {
    case CUSCI_OPT_FORCE_COLLECTIVE:
      if (value && !ctx->comm)
        return set_error(ctx, CUSCI_E_INVALID_ARG, "CUSCI_OPT_FORCE_COLLECTIVE needs a communicator (pass an NCCL id to cusci_init)");
      ctx->force_collective = value ? 1 : 0;
      return CUSCI_OK;
    case CUSCI_OPT_CONTRACT_PARTITION:
      if (value < -1 || value > 1) return set_error(ctx, CUSCI_E_INVALID_ARG, "CUSCI_OPT_CONTRACT_PARTITION takes -1, 0 or 1");
      ctx->contract_partition = (int)value;
      return CUSCI_OK;
    default:
      return set_error(ctx, CUSCI_E_INVALID_ARG, "unknown option %d", option);
  }
}

int cusci_release_cached(cusci_ctx* ctx) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  if (ctx->arena.depth) return set_error(ctx, CUSCI_E_INVALID_ARG, "cusci_release_cached inside a library call");
  cudaSetDevice(ctx->device);
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  arena_release_all(ctx);
  ctx->arena.peak = 0;
  CUSCI_CUDA(ctx, cudaMemPoolTrimTo(ctx->pool, 0));
  return CUSCI_OK;
}

void cusci_invalidate_integrals(cusci_ctx* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  prep_release(ctx);
}

void cusci_free(cusci_ctx* ctx, void* ptr) {
  if (ctx && ptr) out_free(ctx, ptr);
}

uint64_t cusci_kernel_launches(const cusci_ctx* ctx) { return ctx ? ctx->launches : 0; }

int cusci_dedup_stats(cusci_ctx* ctx, uint64_t stats[8], int reset) {
  if (!ctx || !stats) return CUSCI_E_INVALID_ARG;
  for (int i = 0; i < 8; i++) stats[i] = ctx->dstats[i];
  if (reset)
    for (int i = 0; i < 8; i++) ctx->dstats[i] = 0;
  return CUSCI_OK;
}

void cusci_profile_enable(cusci_ctx* ctx, int on) {
  if (ctx) ctx->profiling = on != 0;
}

int cusci_profile_read(cusci_ctx* ctx, double* ms, uint64_t* launches, int n_tags) {
  if (!ctx || !ms || !launches) return CUSCI_E_INVALID_ARG;
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  for (int t = 0; t < n_tags; t++) {
    ms[t] = 0;
    launches[t] = 0;
  }
  for (const ProfRec& r : ctx->prof) {
    float e = 0;
    cudaEventElapsedTime(&e, r.a, r.b);
    if (r.tag < n_tags) {
      ms[r.tag] += e;
      launches[r.tag]++;
    }
    ctx->ev_free.push_back(r.a);
    ctx->ev_free.push_back(r.b);
  }
  ctx->prof.clear();
  return CUSCI_OK;
}

static uint64_t binom2(uint64_t n) { return n < 2 ? 0 : n * (n - 1) / 2; }

uint64_t gen_coupled_bound(const cusci_space* sp, uint64_t n_parents) {
  if (!sp) return 0;
  uint64_t K = (uint64_t)sp->m / 2;
  uint64_t na = sp->n_alpha, nb = sp->n_beta, va = K - na, vb = K - nb;
  uint64_t per = na * va + nb * vb + binom2(na) * binom2(va) + binom2(nb) * binom2(vb) + na * va * nb * vb;
  return per * n_parents;
}

// ------------------------------------------------------------------ pool
int cusci_pool_create(cusci_ctx* ctx, const cusci_space* sp, uint64_t capacity, cusci_pool** out) {
  if (!ctx || !out) return CUSCI_E_INVALID_ARG;
  CUSCI_TRY(check_space(ctx, sp));
  cusci_pool* p = new cusci_pool;
  p->ctx = ctx;
  p->sp = *sp;
  p->cap = capacity < 1024 ? 1024 : capacity;
  for (int b = 0; b < 2; b++) {
    if (cudaMallocFromPoolAsync((void**)&p->buf[b], p->cap * sp->words * 8, ctx->pool, ctx->stream) != cudaSuccess) {
      cudaGetLastError();
      cusci_pool_destroy(p);
      return set_error(ctx, CUSCI_E_OOM, "pool allocation failed");
    }
  }
  *out = p;
  return CUSCI_OK;
}

int cusci_pool_view(const cusci_pool* pool, const uint64_t** keys, uint64_t* count) {
  if (!pool || !keys || !count) return CUSCI_E_INVALID_ARG;
  *keys = pool->buf[pool->cur];
  *count = pool->count;
  return CUSCI_OK;
}

int cusci_pool_clear(cusci_pool* pool) {
  if (!pool) return CUSCI_E_INVALID_ARG;
  pool->count = 0;
  return CUSCI_OK;
}

int cusci_pool_copy(const cusci_pool* pool, uint64_t* dst, uint64_t capacity_keys) {
  if (!pool || (!dst && pool->count)) return CUSCI_E_INVALID_ARG;
  cusci_ctx* ctx = pool->ctx;
  if (capacity_keys < pool->count)
    return set_error(ctx, CUSCI_E_CAPACITY, "pool copy: %llu keys > capacity %llu", (unsigned long long)pool->count,
                     (unsigned long long)capacity_keys);
  if (pool->count)
    CUSCI_CUDA(ctx, cudaMemcpyAsync(dst, pool->buf[pool->cur], pool->count * pool->sp.words * 8,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
  return CUSCI_OK;
}

void cusci_pool_destroy(cusci_pool* pool) {
  if (!pool) return;
  for (int b = 0; b < 2; b++)
    if (pool->buf[b]) cudaFreeAsync(pool->buf[b], pool->ctx->stream);
  cudaStreamSynchronize(pool->ctx->stream);
  delete pool;
}

}  // extern "C"
