// Memory-centric streaming (Sec 4.3 :583-634,
// fig:mem_flow): the device is a scratchpad for mini-batches, three CUDA
// streams overlap host->device prefetch, compute and device->host offload.
//
//   stream_generate (Stage 1)  per parent mini-batch i:
//       H2D stream   parents of batch i+1 -> parent slot (i+1) % 2   (prefetch)
//       compute      count, gen_coupled -> record slot i % 2 (src = global parent
//                    index), dedup_global of its keys, merge_space into the
//                    GPU-resident unique pool
//       D2H stream   records of batch i -> the host "original set"  (offload)
//     A record slot is rewritten (batch i+2) only after its D2H finished; a
//     parent slot only after the gen that read it.  Host syncs inside the
//     compute calls (counts) stall only the compute stream: the copy engines
//     keep running.
//   stream_energy (Stage 3, reload)  the original set streamed back H2D in
//     record batches (double-buffered) and contracted against the unique set
//     and psi: one (key, psi) table for the whole stage, every batch
//     accumulated exactly, e written once -- bit-identical to energy_contract
//     over all records at once.
//   stream_energy_regen (Stage 3, B200 design)  the records are REGENERATED per
//     parent batch instead of reloaded: gen_coupled produces ~1e11 records/s
//     from L2-resident tables, ~50x what PCIe reloads, so on B200 the original
//     set need not be kept at all; same e, bit for bit.
// Peak device memory is accounted by the library: its stream buffers, the
// unique pool's buffers, the scratch arena's high-water mark and the transient
// dedup outputs.
#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace cusci {
namespace {

struct Streams {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev;
  ~Streams() {  // declared after the stage's buffers: joined before they are freed
    if (h2d) cudaStreamSynchronize(h2d);
    if (d2h) cudaStreamSynchronize(d2h);
    for (auto e : ev) cudaEventDestroy(e);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
  }
  cudaEvent_t make(bool timing) {
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming);
    ev.push_back(e);
    return e;
  }
};

// a device buffer of the stage (stream-ordered on the context stream)
struct DBuf {
  cusci_ctx* ctx = nullptr;
  void* p = nullptr;
  size_t bytes = 0;
  ~DBuf() {
    if (p) cudaFreeAsync(p, ctx->stream);
  }
  int ensure(cusci_ctx* c, size_t b) {
    ctx = c;
    if (b <= bytes) return CUSCI_OK;
    if (p) cudaFreeAsync(p, ctx->stream);
    p = nullptr;
    bytes = 0;
    if (cudaMallocFromPoolAsync(&p, b, ctx->pool, ctx->stream) != cudaSuccess) {
      cudaGetLastError();
      return set_error(ctx, CUSCI_E_OOM, "stream buffer of %zu bytes failed", b);
    }
    bytes = b;
    return CUSCI_OK;
  }
};

// busy time of one stream: the sum of its [a, b) event spans
struct Busy {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spans;
  double ms() const {
    double t = 0;
    for (auto& s : spans) {
      float x = 0;
      cudaEventElapsedTime(&x, s.first, s.second);
      t += x;
    }
    return t;
  }
};

// scratch-arena high-water mark over a stage
struct ArenaPeak {
  cusci_ctx* ctx;
  size_t saved;
  explicit ArenaPeak(cusci_ctx* c) : ctx(c), saved(c->arena.peak) { ctx->arena.peak = ctx->arena.used; }
  size_t peak() const { return ctx->arena.peak; }
  ~ArenaPeak() { ctx->arena.peak = std::max(saved, ctx->arena.peak); }
};

int stream_args(cusci_ctx* ctx, const cusci_space* sp, const cusci_stream_cfg* cfg, cusci_stream_stats* st) {
  if (ctx->broken) return set_error(ctx, CUSCI_E_CUDA, "context is unusable after an earlier CUDA/NCCL error");
  CUSCI_TRY(check_space(ctx, sp));
  if (!cfg || !st) return set_error(ctx, CUSCI_E_INVALID_ARG, "stream cfg/stats are NULL");
  if (cfg->host_keys && (!cfg->host_hij || !cfg->host_src))
    return set_error(ctx, CUSCI_E_INVALID_ARG, "host original set: keys, hij and src are all required");
  memset(st, 0, sizeof(*st));
  return CUSCI_OK;
}

int agree_max(cusci_ctx* ctx, uint64_t* v) {
  if (!collective(ctx)) return CUSCI_OK;
  uint64_t* d = ctx->dcomm + 2 * CUSCI_MAX_WORLD + 2;
  *(uint64_t*)ctx->host_pinned = *v;
  CUSCI_CUDA(ctx, cudaMemcpyAsync(d, ctx->host_pinned, 8, cudaMemcpyHostToDevice, ctx->stream));
  CUSCI_TRY(nccl_ok(ctx, ncclAllReduce(d, d, 1, ncclUint64, ncclMax, ctx->comm, ctx->stream), "batch-count allreduce"));
  return read_u64(ctx, d, v, 1);
}

}  // namespace
}  // namespace cusci

using namespace cusci;

extern "C" int stream_generate(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents_host, uint64_t n_parents,
                               const cusci_integrals* ints, double threshold, const cusci_stream_cfg* cfg,
                               cusci_pool* unique_pool, cusci_stream_stats* st) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  CUSCI_TRY(stream_args(ctx, sp, cfg, st));
  if (!unique_pool || unique_pool->ctx != ctx) return set_error(ctx, CUSCI_E_INVALID_ARG, "unique_pool is NULL or of another context");
  if (n_parents && !parents_host) return set_error(ctx, CUSCI_E_INVALID_ARG, "parents_host is NULL");
  if (!cfg->batch_parents) return set_error(ctx, CUSCI_E_INVALID_ARG, "batch_parents must be >= 1");
  if (n_parents >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "n_parents must be < 2^32");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  const int W = sp->words;
  const uint64_t B = cfg->batch_parents;
  uint64_t nb = (n_parents + B - 1) / B;
  CUSCI_TRY(agree_max(ctx, &nb));  // dedup_global is collective: every rank makes the same number of calls
  const bool offload = cfg->host_keys != nullptr;
  ArenaPeak ap(ctx);
  DBuf par[2], rk[2], rh[2], rs[2];
  Streams ss;
  CUSCI_CUDA(ctx, cudaStreamCreateWithFlags(&ss.h2d, cudaStreamNonBlocking));
  CUSCI_CUDA(ctx, cudaStreamCreateWithFlags(&ss.d2h, cudaStreamNonBlocking));
  std::vector<cudaEvent_t> ev_h2d(nb + 1), ev_gen(nb + 1), ev_d2h(nb + 1);
  for (uint64_t i = 0; i < nb; i++) {
    ev_h2d[i] = ss.make(false);
    ev_gen[i] = ss.make(false);
    ev_d2h[i] = ss.make(false);
  }
  Busy bh, bc, bd;
  cudaEvent_t w0 = ss.make(true), w1 = ss.make(true);
  auto span = [&](Busy& b, cudaStream_t s) -> cudaEvent_t {
    cudaEvent_t a = ss.make(true);
    cudaEventRecord(a, s);
    b.spans.push_back({a, nullptr});
    return a;
  };
  auto close = [&](Busy& b, cudaStream_t s) {
    cudaEvent_t e = ss.make(true);
    cudaEventRecord(e, s);
    b.spans.back().second = e;
  };
  auto batch = [&](uint64_t i, uint64_t* a, uint64_t* n) {
    *a = std::min(n_parents, i * B);
    *n = std::min(n_parents, (i + 1) * B) - *a;
  };
  CUSCI_TRY(par[0].ensure(ctx, std::max<uint64_t>(B, 1) * W * 8));
  CUSCI_TRY(par[1].ensure(ctx, std::max<uint64_t>(B, 1) * W * 8));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // the parent slots exist before the copy streams use them
  CUSCI_CUDA(ctx, cudaEventRecord(w0, ctx->stream));
  auto prefetch = [&](uint64_t i) -> int {
    uint64_t a, n;
    batch(i, &a, &n);
    if (i >= 2) CUSCI_CUDA(ctx, cudaStreamWaitEvent(ss.h2d, ev_gen[i - 2], 0));  // slot free: gen(i-2) read it
    span(bh, ss.h2d);
    if (n)
      CUSCI_CUDA(ctx, cudaMemcpyAsync(par[i % 2].p, parents_host + a * W, n * W * 8, cudaMemcpyHostToDevice, ss.h2d));
    close(bh, ss.h2d);
    st->h2d_bytes += n * W * 8;
    CUSCI_CUDA(ctx, cudaEventRecord(ev_h2d[i], ss.h2d));
    return CUSCI_OK;
  };
  if (nb) CUSCI_TRY(prefetch(0));
  uint64_t host_at = 0, peak = 0;
  int rc_cap = CUSCI_OK;
  for (uint64_t i = 0; i < nb; i++) {
    if (i + 1 < nb) CUSCI_TRY(prefetch(i + 1));
    uint64_t a, n;
    batch(i, &a, &n);
    const int ps = (int)(i % 2);               // parent slot
    const int sl = offload ? (int)(i % 2) : 0;  // record slot: one suffices when nothing is offloaded
    CUSCI_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ev_h2d[i], 0));
    span(bc, ctx->stream);
    if (offload && i >= 2) CUSCI_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ev_d2h[i - 2], 0));  // slot free: its offload done
    // record capacity: the caller's hint (cfg->batch_records) or an exact count;
    // a batch that exceeds the hint is counted and generated again
    uint64_t cnt = cfg->batch_records;
    if (!cnt) CUSCI_TRY(gen_count(ctx, sp, (const uint64_t*)par[ps].p, n, ints, threshold, &cnt));
    cusci_records rec{};
    for (int attempt = 0;; attempt++) {
      if (rk[sl].bytes < cnt * W * 8 && offload) CUSCI_CUDA(ctx, cudaStreamSynchronize(ss.d2h));  // (re)allocation
      CUSCI_TRY(rk[sl].ensure(ctx, std::max<uint64_t>(cnt, 1) * W * 8));
      CUSCI_TRY(rh[sl].ensure(ctx, std::max<uint64_t>(cnt, 1) * 8));
      CUSCI_TRY(rs[sl].ensure(ctx, std::max<uint64_t>(cnt, 1) * 4));
      rec = cusci_records{(uint64_t*)rk[sl].p, (double*)rh[sl].p, (uint32_t*)rs[sl].p, nullptr,
                          rk[sl].bytes / (W * 8), 0};
      const int rc = gen_records(ctx, sp, (const uint64_t*)par[ps].p, n, ints, threshold, &rec, (uint32_t)a);
      if (rc == CUSCI_E_CAPACITY && attempt == 0) {
        cnt = rec.count;
        ctx->err.clear();
        continue;
      }
      CUSCI_TRY(rc);
      break;
    }
    CUSCI_CUDA(ctx, cudaEventRecord(ev_gen[i], ctx->stream));
    st->records += rec.count;
    if (offload) {  // the original set -> host memory while the next batch computes
      const uint64_t m = host_at >= cfg->host_capacity ? 0 : std::min(rec.count, cfg->host_capacity - host_at);
      if (m < rec.count) rc_cap = CUSCI_E_CAPACITY;
      CUSCI_CUDA(ctx, cudaStreamWaitEvent(ss.d2h, ev_gen[i], 0));
      span(bd, ss.d2h);
      if (m) {
        CUSCI_CUDA(ctx, cudaMemcpyAsync(cfg->host_keys + host_at * W, rk[sl].p, m * W * 8, cudaMemcpyDeviceToHost, ss.d2h));
        CUSCI_CUDA(ctx, cudaMemcpyAsync(cfg->host_hij + host_at, rh[sl].p, m * 8, cudaMemcpyDeviceToHost, ss.d2h));
        CUSCI_CUDA(ctx, cudaMemcpyAsync(cfg->host_src + host_at, rs[sl].p, m * 4, cudaMemcpyDeviceToHost, ss.d2h));
      }
      close(bd, ss.d2h);
      st->d2h_bytes += m * (W * 8 + 12);
      host_at += m;
    }
    CUSCI_CUDA(ctx, cudaEventRecord(ev_d2h[i], offload ? ss.d2h : ctx->stream));
    cusci_keys u{nullptr, 0};
    CUSCI_TRY(dedup_global(ctx, sp, rec.keys, rec.count, &u));
    const size_t ubytes = u.count * W * 8;
    const int mrc = merge_space(ctx, unique_pool, u.keys, u.count, nullptr);
    out_free(ctx, u.keys);
    CUSCI_TRY(mrc);
    close(bc, ctx->stream);
    const uint64_t now = par[0].bytes + par[1].bytes + rk[0].bytes + rk[1].bytes + rh[0].bytes + rh[1].bytes +
                         rs[0].bytes + rs[1].bytes + 2 * unique_pool->cap * W * 8 + ubytes + ap.peak();
    peak = std::max(peak, now);
  }
  // join the copy streams, then stop the clock
  cudaEvent_t jh = ss.make(false), jd = ss.make(false);
  CUSCI_CUDA(ctx, cudaEventRecord(jh, ss.h2d));
  CUSCI_CUDA(ctx, cudaEventRecord(jd, ss.d2h));
  CUSCI_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, jh, 0));
  CUSCI_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, jd, 0));
  CUSCI_CUDA(ctx, cudaEventRecord(w1, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  float wall = 0;
  cudaEventElapsedTime(&wall, w0, w1);
  st->batches = nb;
  st->unique = unique_pool->count;
  st->ms_wall = wall;
  st->ms_h2d = bh.ms();
  st->ms_compute = bc.ms();
  st->ms_d2h = bd.ms();
  st->peak_device_bytes = peak;
  if (rc_cap != CUSCI_OK)
    return set_error(ctx, rc_cap, "stream_generate: %llu records, the host original set holds %llu",
                     (unsigned long long)st->records, (unsigned long long)cfg->host_capacity);
  return CUSCI_OK;
}

extern "C" int stream_energy(cusci_ctx* ctx, const cusci_space* sp, const cusci_stream_cfg* cfg, uint64_t n_rec,
                             uint64_t n_parents, const uint64_t* space_keys, uint64_t n_space, const double* psi,
                             double* e, uint64_t* n_missing, cusci_stream_stats* st) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  CUSCI_TRY(stream_args(ctx, sp, cfg, st));
  if (collective(ctx)) return set_error(ctx, CUSCI_E_INVALID_ARG, "stream_energy: one rank (use energy_contract per batch)");
  if (n_rec && !cfg->host_keys) return set_error(ctx, CUSCI_E_INVALID_ARG, "stream_energy: no host original set");
  if (n_rec > cfg->host_capacity) return set_error(ctx, CUSCI_E_INVALID_ARG, "n_rec > host_capacity");
  if (!cfg->batch_records) return set_error(ctx, CUSCI_E_INVALID_ARG, "batch_records must be >= 1");
  if ((n_parents && !e) || !n_missing || (n_space && (!space_keys || !psi)))
    return set_error(ctx, CUSCI_E_INVALID_ARG, "stream_energy: NULL argument");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  const int W = sp->words;
  const uint64_t R = cfg->batch_records, nb = (n_rec + R - 1) / R;
  ArenaPeak ap(ctx);
  Scratch s(ctx);
  CState cs;
  CUSCI_TRY(contract_begin(ctx, s, W, space_keys, n_space, psi, n_parents, &cs));
  DBuf rk[2], rh[2], rs[2];
  Streams ss;
  CUSCI_CUDA(ctx, cudaStreamCreateWithFlags(&ss.h2d, cudaStreamNonBlocking));
  for (int b = 0; b < 2; b++) {
    CUSCI_TRY(rk[b].ensure(ctx, std::max<uint64_t>(R, 1) * W * 8));
    CUSCI_TRY(rh[b].ensure(ctx, std::max<uint64_t>(R, 1) * 8));
    CUSCI_TRY(rs[b].ensure(ctx, std::max<uint64_t>(R, 1) * 4));
  }
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<cudaEvent_t> ev_h2d(nb + 1), ev_use(nb + 1);
  for (uint64_t j = 0; j < nb; j++) {
    ev_h2d[j] = ss.make(false);
    ev_use[j] = ss.make(false);
  }
  Busy bh, bc;
  cudaEvent_t w0 = ss.make(true), w1 = ss.make(true);
  CUSCI_CUDA(ctx, cudaEventRecord(w0, ctx->stream));
  auto load = [&](uint64_t j) -> int {
    const uint64_t a = j * R, m = std::min(n_rec, a + R) - a;
    const int sl = (int)(j % 2);
    if (j >= 2) CUSCI_CUDA(ctx, cudaStreamWaitEvent(ss.h2d, ev_use[j - 2], 0));
    cudaEvent_t x = ss.make(true), y = ss.make(true);
    CUSCI_CUDA(ctx, cudaEventRecord(x, ss.h2d));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(rk[sl].p, cfg->host_keys + a * W, m * W * 8, cudaMemcpyHostToDevice, ss.h2d));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(rh[sl].p, cfg->host_hij + a, m * 8, cudaMemcpyHostToDevice, ss.h2d));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(rs[sl].p, cfg->host_src + a, m * 4, cudaMemcpyHostToDevice, ss.h2d));
    CUSCI_CUDA(ctx, cudaEventRecord(y, ss.h2d));
    bh.spans.push_back({x, y});
    st->h2d_bytes += m * (W * 8 + 12);
    CUSCI_CUDA(ctx, cudaEventRecord(ev_h2d[j], ss.h2d));
    return CUSCI_OK;
  };
  if (nb) CUSCI_TRY(load(0));
  for (uint64_t j = 0; j < nb; j++) {
    if (j + 1 < nb) CUSCI_TRY(load(j + 1));
    const uint64_t a = j * R, m = std::min(n_rec, a + R) - a;
    const int sl = (int)(j % 2);
    CUSCI_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ev_h2d[j], 0));
    cudaEvent_t x = ss.make(true), y = ss.make(true);
    CUSCI_CUDA(ctx, cudaEventRecord(x, ctx->stream));
    CUSCI_TRY(contract_add(ctx, cs, (const uint64_t*)rk[sl].p, (const double*)rh[sl].p, (const uint32_t*)rs[sl].p, m));
    CUSCI_CUDA(ctx, cudaEventRecord(y, ctx->stream));
    bc.spans.push_back({x, y});
    CUSCI_CUDA(ctx, cudaEventRecord(ev_use[j], ctx->stream));
  }
  CUSCI_TRY(contract_end(ctx, cs, e, n_missing));
  CUSCI_CUDA(ctx, cudaEventRecord(w1, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  float wall = 0;
  cudaEventElapsedTime(&wall, w0, w1);
  st->batches = nb;
  st->records = n_rec;
  st->ms_wall = wall;
  st->ms_h2d = bh.ms();
  st->ms_compute = bc.ms();
  st->peak_device_bytes = 2 * (rk[0].bytes + rh[0].bytes + rs[0].bytes) + ap.peak();
  return CUSCI_OK;
}

extern "C" int stream_energy_regen(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents_host,
                                   uint64_t n_parents, const cusci_integrals* ints, double threshold,
                                   const cusci_stream_cfg* cfg, const uint64_t* space_keys, uint64_t n_space,
                                   const double* psi, double* e, uint64_t* n_missing, cusci_stream_stats* st) {
  if (!ctx) return CUSCI_E_INVALID_ARG;
  CUSCI_TRY(stream_args(ctx, sp, cfg, st));
  if (collective(ctx)) return set_error(ctx, CUSCI_E_INVALID_ARG, "stream_energy_regen: one rank");
  if ((n_parents && (!parents_host || !e)) || !n_missing || (n_space && (!space_keys || !psi)))
    return set_error(ctx, CUSCI_E_INVALID_ARG, "stream_energy_regen: NULL argument");
  if (!cfg->batch_parents) return set_error(ctx, CUSCI_E_INVALID_ARG, "batch_parents must be >= 1");
  if (n_parents >= (1ull << 32)) return set_error(ctx, CUSCI_E_INVALID_ARG, "n_parents must be < 2^32");
  CUSCI_CUDA(ctx, cudaSetDevice(ctx->device));
  const int W = sp->words;
  const uint64_t B = cfg->batch_parents, nb = (n_parents + B - 1) / B;
  ArenaPeak ap(ctx);
  Scratch s(ctx);
  CState cs;
  CUSCI_TRY(contract_begin(ctx, s, W, space_keys, n_space, psi, n_parents, &cs));
  DBuf par[2], rk, rh, rsb;
  Streams ss;
  CUSCI_CUDA(ctx, cudaStreamCreateWithFlags(&ss.h2d, cudaStreamNonBlocking));
  CUSCI_TRY(par[0].ensure(ctx, std::max<uint64_t>(B, 1) * W * 8));
  CUSCI_TRY(par[1].ensure(ctx, std::max<uint64_t>(B, 1) * W * 8));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<cudaEvent_t> ev_h2d(nb + 1), ev_gen(nb + 1);
  for (uint64_t i = 0; i < nb; i++) {
    ev_h2d[i] = ss.make(false);
    ev_gen[i] = ss.make(false);
  }
  Busy bh, bc;
  cudaEvent_t w0 = ss.make(true), w1 = ss.make(true);
  CUSCI_CUDA(ctx, cudaEventRecord(w0, ctx->stream));
  auto prefetch = [&](uint64_t i) -> int {
    const uint64_t a = i * B, n = std::min(n_parents, a + B) - a;
    if (i >= 2) CUSCI_CUDA(ctx, cudaStreamWaitEvent(ss.h2d, ev_gen[i - 2], 0));
    cudaEvent_t x = ss.make(true), y = ss.make(true);
    CUSCI_CUDA(ctx, cudaEventRecord(x, ss.h2d));
    CUSCI_CUDA(ctx, cudaMemcpyAsync(par[i % 2].p, parents_host + a * W, n * W * 8, cudaMemcpyHostToDevice, ss.h2d));
    CUSCI_CUDA(ctx, cudaEventRecord(y, ss.h2d));
    bh.spans.push_back({x, y});
    st->h2d_bytes += n * W * 8;
    CUSCI_CUDA(ctx, cudaEventRecord(ev_h2d[i], ss.h2d));
    return CUSCI_OK;
  };
  if (nb) CUSCI_TRY(prefetch(0));
  uint64_t peak = 0;
  for (uint64_t i = 0; i < nb; i++) {
    if (i + 1 < nb) CUSCI_TRY(prefetch(i + 1));
    const uint64_t a = i * B, n = std::min(n_parents, a + B) - a;
    CUSCI_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ev_h2d[i], 0));
    cudaEvent_t x = ss.make(true), y = ss.make(true);
    CUSCI_CUDA(ctx, cudaEventRecord(x, ctx->stream));
    uint64_t cnt = 0;
    CUSCI_TRY(gen_count(ctx, sp, (const uint64_t*)par[i % 2].p, n, ints, threshold, &cnt));
    CUSCI_TRY(rk.ensure(ctx, std::max<uint64_t>(cnt, 1) * W * 8));
    CUSCI_TRY(rh.ensure(ctx, std::max<uint64_t>(cnt, 1) * 8));
    CUSCI_TRY(rsb.ensure(ctx, std::max<uint64_t>(cnt, 1) * 4));
    cusci_records rec{(uint64_t*)rk.p, (double*)rh.p, (uint32_t*)rsb.p, nullptr, cnt, 0};
    CUSCI_TRY(gen_records(ctx, sp, (const uint64_t*)par[i % 2].p, n, ints, threshold, &rec, (uint32_t)a));
    CUSCI_CUDA(ctx, cudaEventRecord(ev_gen[i], ctx->stream));
    CUSCI_TRY(contract_add(ctx, cs, rec.keys, rec.hij, rec.src, rec.count));
    CUSCI_CUDA(ctx, cudaEventRecord(y, ctx->stream));
    bc.spans.push_back({x, y});
    st->records += rec.count;
    peak = std::max<uint64_t>(peak, par[0].bytes + par[1].bytes + rk.bytes + rh.bytes + rsb.bytes + ap.peak());
  }
  CUSCI_TRY(contract_end(ctx, cs, e, n_missing));
  CUSCI_CUDA(ctx, cudaEventRecord(w1, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  float wall = 0;
  cudaEventElapsedTime(&wall, w0, w1);
  st->batches = nb;
  st->ms_wall = wall;
  st->ms_h2d = bh.ms();
  st->ms_compute = bc.ms();
  st->peak_device_bytes = peak;
  return CUSCI_OK;
}
