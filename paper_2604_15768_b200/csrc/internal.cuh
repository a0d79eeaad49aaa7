// Internal definitions shared by the libcusci translation units (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/cusci.h"

namespace cusci {

constexpr int kWarp = 32;
constexpr size_t kHostPinnedBytes = 3 * CUSCI_MAX_WORLD * sizeof(uint64_t) + 4096;
constexpr size_t kCommWords = 2 * CUSCI_MAX_WORLD + 8;  // send counts, recv counts, status words
constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ status
struct Status {
  int code = CUSCI_OK;
};

// ------------------------------------------------------------------ scratch arena
// Scratch memory is bump-allocated from a context-owned, grow-only device
// arena (a list of cudaMalloc'd segments).  Scratch scopes nest LIFO; a scope
// releases its bytes when it ends (all work is ordered on the context stream,
// so the bytes can be reused by later launches without a sync).  When a call
// needed more than one segment, the next top-level call synchronises the
// stream and replaces the segments by one segment of the observed peak, so the
// steady state performs no device allocation at all.
struct Arena {
  struct Seg {
    char* base;
    size_t cap;
  };
  std::vector<Seg> segs;
  size_t cur = 0;    // active segment
  size_t off = 0;    // bump offset in segs[cur]
  size_t used = 0;   // bytes live across segments
  size_t peak = 0;   // high-water mark
  int depth = 0;     // live Scratch scopes
};
// pair-table entry (16 B, one 128-bit load): x = occupation mask 2^a | 2^b
// (m <= 64) or a | b << 8 (m > 64); v = <pq||ab>
struct __align__(16) PairEnt {
  uint64_t x;
  double v;
};

// Cached Hamiltonian prep: built on device from (h, eri).
struct Prep {
  const double* h = nullptr;
  const double* eri = nullptr;
  int K = 0;
  double eps = -1.0;
  bool valid = false;
  // pair rows over spin-orbital pairs p<q, row id = q(q-1)/2 + p
  uint32_t* rowptr = nullptr;   // [npq + 1]
  PairEnt* ent = nullptr;       // [nnz]  (a < b, <pq||ab> = d1-d2 | d1 | -d2), |v| > eps
  uint64_t nnz = 0;
  // singles candidates per spin orbital p: targets a (same spin, a != p) with
  // any nonzero constituent integral
  uint32_t* srowptr = nullptr;  // [m + 1]
  uint8_t* sa = nullptr;        // [snnz]
  uint64_t snnz = 0;
  double* topp = nullptr;       // [K][K][K]  (PA|KK)
  double* tsame = nullptr;      // [K][K][K]  (PA|KK) - (PK|KA)
  void* block = nullptr;        // single cudaMalloc holding all of the above
  size_t block_bytes = 0;
};

// kernel classes for the optional per-launch event profiler (cusci_profile_*)
enum ProfTag {
  PT_PREP = 0, PT_VALIDATE, PT_GEN, PT_HASH, PT_SCATTER, PT_RADIX_UP, PT_RADIX_DOWN, PT_SCAN, PT_UNIQUE,
  PT_MERGE_SPLIT, PT_MERGE_TILE, PT_CHECK, PT_NCCL, PT_MEMSET, PT_ENERGY, PT_COUNT
};
struct ProfRec {
  int tag;
  cudaEvent_t a, b;
};
// per-context launch setup of one kernel (the large-shared-memory opt-in is a
// property of the device context, so it is cached per library context, never
// in process-wide statics)
struct KSetup {
  const void* fn;
  size_t smem;
  int threads;
  int per_sm;
};

}  // namespace cusci

struct cusci_ctx {
  int device = 0;
  int rank = 0;
  int world = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  bool broken = false;
  cusci_alloc_fn alloc = nullptr;
  cusci_free_fn free_fn = nullptr;
  void* alloc_user = nullptr;
  cudaMemPool_t pool = nullptr;
  cusci::Arena arena;
  cusci::Prep prep;
  void* host_pinned = nullptr;  // small pinned staging (counts, flags), kHostPinnedBytes
  uint64_t* dcomm = nullptr;    // device [kCommWords]: collective counts / status (with a communicator)
  uint64_t launches = 0;
  int num_sms = 148;
  bool profiling = false;
  uint64_t dstats[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // cusci_dedup_stats
  std::vector<cusci::ProfRec> prof;
  std::vector<cudaEvent_t> ev_free;
  std::vector<cusci::KSetup> ksetup;  // kernel_setup cache (this context's device)
  int force_collective = 0;           // CUSCI_OPT_FORCE_COLLECTIVE
  int contract_partition = 0;         // CUSCI_OPT_CONTRACT_PARTITION: -1 off, 0 auto, 1 on
  std::string err;
};

struct cusci_pool {
  cusci_ctx* ctx = nullptr;
  cusci_space sp{};
  uint64_t* buf[2] = {nullptr, nullptr};
  uint64_t cap = 0;  // keys per buffer
  int cur = 0;
  uint64_t count = 0;
};

namespace cusci {

int set_error(cusci_ctx* ctx, int code, const char* fmt, ...);

#define CUSCI_CUDA(ctx, call)                                                              \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      (ctx)->broken = true;                                                                \
      return ::cusci::set_error((ctx), CUSCI_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, \
                                cudaGetErrorString(e_));                                   \
    }                                                                                      \
  } while (0)

#define CUSCI_TRY(expr)        \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != CUSCI_OK) return rc_; \
  } while (0)

// cudaGetLastError (not Peek): a failed launch's error is consumed here, so it
// cannot be reported again by a later, unrelated launch check
#define CUSCI_LAUNCH_CHECK(ctx)                  \
  do {                                           \
    (ctx)->launches++;                           \
    CUSCI_CUDA((ctx), cudaGetLastError());       \
  } while (0)

// launch a kernel under the profiler scope of class `tag`
#define CUSCI_LAUNCH(ctx, tag, ...)              \
  do {                                           \
    ::cusci::Prof pf_((ctx), (tag));             \
    __VA_ARGS__;                                 \
    CUSCI_LAUNCH_CHECK(ctx);                     \
  } while (0)

// Profiler scope: when ctx->profiling, records a CUDA event pair on the
// context stream around the enclosed launches (tagged by kernel class).
struct Prof {
  cusci_ctx* ctx;
  int tag;
  cudaEvent_t a = nullptr;
  Prof(cusci_ctx* c, int t);
  ~Prof();
};

// scratch (stream-ordered, from the context pool)
struct Scratch {
  cusci_ctx* ctx;
  size_t m_cur, m_off, m_used;
  explicit Scratch(cusci_ctx* c);
  ~Scratch();
  // returns CUSCI_OK or CUSCI_E_OOM (with message); zero-byte requests give a valid dummy
  int get(size_t bytes, void** p);
  template <typename T> int get_t(size_t count, T** p) { return get(count * sizeof(T), (void**)p); }
};

// output allocation through the context's allocator
int out_alloc(cusci_ctx* ctx, size_t bytes, void** p);
void out_free(cusci_ctx* ctx, void* p);

int check_space(cusci_ctx* ctx, const cusci_space* sp);
// opt a kernel into `smem` bytes of dynamic shared memory on this context's
// device (once per context) and return its resident CTAs per SM
int kernel_setup(cusci_ctx* ctx, const void* fn, int threads, size_t smem, int* per_sm);
// collective calls run their NCCL protocol (status + count exchange, payload
// exchange) when the context spans several ranks, or when a 1-rank
// communicator exists and CUSCI_OPT_FORCE_COLLECTIVE is set (tests)
inline bool collective(const cusci_ctx* ctx) { return ctx->world > 1 || (ctx->force_collective && ctx->comm); }
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// ------------------------------------------------------------------ keys
template <int W> struct KeyT;
template <> struct KeyT<1> {
  uint64_t w0;
};
template <> struct alignas(16) KeyT<2> {
  uint64_t w0, w1;
};

template <int W> __device__ __forceinline__ KeyT<W> load_key(const uint64_t* base, uint64_t i);
template <> __device__ __forceinline__ KeyT<1> load_key<1>(const uint64_t* base, uint64_t i) {
  return KeyT<1>{base[i]};
}
template <> __device__ __forceinline__ KeyT<2> load_key<2>(const uint64_t* base, uint64_t i) {
  ulonglong2 v = reinterpret_cast<const ulonglong2*>(base)[i];
  return KeyT<2>{v.x, v.y};
}
template <int W> __device__ __forceinline__ void store_key(uint64_t* base, uint64_t i, const KeyT<W>& k);
template <> __device__ __forceinline__ void store_key<1>(uint64_t* base, uint64_t i, const KeyT<1>& k) {
  base[i] = k.w0;
}
template <> __device__ __forceinline__ void store_key<2>(uint64_t* base, uint64_t i, const KeyT<2>& k) {
  reinterpret_cast<ulonglong2*>(base)[i] = make_ulonglong2(k.w0, k.w1);
}
__device__ __forceinline__ bool key_eq(const KeyT<1>& a, const KeyT<1>& b) { return a.w0 == b.w0; }
__device__ __forceinline__ bool key_eq(const KeyT<2>& a, const KeyT<2>& b) { return a.w0 == b.w0 && a.w1 == b.w1; }
__device__ __forceinline__ bool key_lt(const KeyT<1>& a, const KeyT<1>& b) { return a.w0 < b.w0; }
__device__ __forceinline__ bool key_lt(const KeyT<2>& a, const KeyT<2>& b) {
  return a.w1 < b.w1 || (a.w1 == b.w1 && a.w0 < b.w0);
}
__device__ __forceinline__ bool key_le(const KeyT<1>& a, const KeyT<1>& b) { return a.w0 <= b.w0; }
__device__ __forceinline__ bool key_le(const KeyT<2>& a, const KeyT<2>& b) { return !key_lt(b, a); }

// 8-bit digit d (bits [8d, 8d+8)) of the big integer
__device__ __forceinline__ uint32_t key_digit(const KeyT<1>& k, int shift) { return (uint32_t)(k.w0 >> shift) & 0xffu; }
__device__ __forceinline__ uint32_t key_digit(const KeyT<2>& k, int shift) {
  return (uint32_t)((shift < 64 ? (k.w0 >> shift) : (k.w1 >> (shift - 64)))) & 0xffu;
}

// bits [shift, shift+32) of the big integer (shift < 64W)
__device__ __forceinline__ uint32_t key_digit_bits(const KeyT<1>& k, int shift) { return (uint32_t)(k.w0 >> shift); }
__device__ __forceinline__ uint32_t key_digit_bits(const KeyT<2>& k, int shift) {
  if (shift >= 64) return (uint32_t)(k.w1 >> (shift - 64));
  const uint64_t lo = k.w0 >> shift;
  const uint64_t hi = shift ? (k.w1 << (64 - shift)) : 0ull;
  return (uint32_t)(lo | hi);
}

// splitmix64 finalizer
__device__ __forceinline__ uint64_t fmix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
// owner(j) = floor(mix(j) * P / 2^64)   (reading r9)
__device__ __forceinline__ uint64_t owner_mix(const KeyT<1>& k) { return fmix64(k.w0); }
__device__ __forceinline__ uint64_t owner_mix(const KeyT<2>& k) {
  return fmix64(k.w0 ^ fmix64(k.w1 ^ 0x9E3779B97F4A7C15ull));
}
template <int W> __device__ __forceinline__ uint32_t owner_of(const KeyT<W>& k, uint32_t P) {
  return (uint32_t)__umul64hi(owner_mix(k), (uint64_t)P);
}
// Hash order (reading r13): pi(j) = (hi, lo), a bijection of the
// key space; hi = owner mix (owner(j) = floor(hi P / 2^64) is monotone in pi).
//   W = 1: hi = fmix(w0), lo = 0;   W = 2: lo = fmix(w1 ^ C), hi = fmix(w0 ^ lo).
__device__ __forceinline__ uint64_t hk_hi(const KeyT<1>& k) { return fmix64(k.w0); }
__device__ __forceinline__ uint64_t hk_hi(const KeyT<2>& k) { return owner_mix(k); }
__device__ __forceinline__ uint64_t hk_lo(const KeyT<1>&) { return 0ull; }
__device__ __forceinline__ uint64_t hk_lo(const KeyT<2>& k) { return fmix64(k.w1 ^ 0x9E3779B97F4A7C15ull); }
template <int W> __device__ __forceinline__ bool hk_lt(const KeyT<W>& a, const KeyT<W>& b) {
  const uint64_t ha = hk_hi(a), hb = hk_hi(b);
  if (W == 1) return ha < hb;
  return ha < hb || (ha == hb && hk_lo(a) < hk_lo(b));
}
template <int W> __device__ __forceinline__ bool hk_le(const KeyT<W>& a, const KeyT<W>& b) { return !hk_lt<W>(b, a); }

// inverse of fmix64 (odd multipliers are invertible mod 2^64; x ^= x >> s is
// undone by x ^= x >> s ^ x >> 2s ...)
__device__ __forceinline__ uint64_t fmix64_inv(uint64_t x) {
  x ^= (x >> 31) ^ (x >> 62);
  x *= 0x319642B2D24D8EC3ull;  // (0x94D049BB133111EB)^-1 mod 2^64
  x ^= (x >> 27) ^ (x >> 54);
  x *= 0x96DE1B173F119089ull;  // (0xBF58476D1CE4E5B9)^-1 mod 2^64
  x ^= (x >> 30) ^ (x >> 60);
  return x;
}
// pi-values: the hash-order image of a key, stored in a KeyT slot.
//   W = 1: w0 = hi;   W = 2: w0 = hi, w1 = lo   (compare w0 first)
// Inside the dedup pipeline keys travel as pi-values (the mix is computed once,
// on the first read) and are mapped back with the exact inverse on output.
__device__ __forceinline__ KeyT<1> to_pi(const KeyT<1>& k) { return KeyT<1>{fmix64(k.w0)}; }
__device__ __forceinline__ KeyT<2> to_pi(const KeyT<2>& k) {
  const uint64_t lo = fmix64(k.w1 ^ 0x9E3779B97F4A7C15ull);
  return KeyT<2>{fmix64(k.w0 ^ lo), lo};
}
__device__ __forceinline__ KeyT<1> from_pi(const KeyT<1>& p) { return KeyT<1>{fmix64_inv(p.w0)}; }
__device__ __forceinline__ KeyT<2> from_pi(const KeyT<2>& p) {
  return KeyT<2>{fmix64_inv(p.w0) ^ p.w1, fmix64_inv(p.w1) ^ 0x9E3779B97F4A7C15ull};
}
__device__ __forceinline__ bool pi_lt(const KeyT<1>& a, const KeyT<1>& b) { return a.w0 < b.w0; }
__device__ __forceinline__ bool pi_lt(const KeyT<2>& a, const KeyT<2>& b) {
  return a.w0 < b.w0 || (a.w0 == b.w0 && a.w1 < b.w1);
}

// ------------------------------------------------------------------ TMA bulk copies (1-D) + mbarriers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// order earlier generic-proxy shared-memory accesses before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// one elected thread: arm `bar` for `bytes` and start global -> shared bulk copy
// (src, dst 16-byte aligned, bytes a multiple of 16)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// hash-table slot hash (independent of the owner mix)
__device__ __forceinline__ uint64_t slot_hash(const KeyT<1>& k) { return fmix64(k.w0 ^ 0xD6E8FEB86659FD93ull); }
__device__ __forceinline__ uint64_t slot_hash(const KeyT<2>& k) {
  return fmix64(k.w1 ^ fmix64(k.w0 ^ 0xD6E8FEB86659FD93ull));
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// block-wide exclusive scan of one u32 per thread (smem: >= 33 words); returns
// this thread's exclusive prefix and the block total
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t* smem, uint32_t& total) {
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if ((int)lane_id() >= o) inc += t;
  }
  if (lane_id() == 31) smem[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t sv = (int)lane_id() < nw ? smem[lane_id()] : 0u;
    uint32_t si = sv;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, si, o);
      if ((int)lane_id() >= o) si += t;
    }
    if ((int)lane_id() < nw) smem[lane_id()] = si - sv;
    if (lane_id() == 31) smem[32] = si;
  }
  __syncthreads();
  const uint32_t r = smem[w] + inc - v;
  total = smem[32];
  __syncthreads();
  return r;
}

// radix pass digit: mode 0 = key bits [shift, shift+bits), 1 = hash-order hi
// (owner-mix) bits, 2 = owner(j) among P (bits = ceil(log2 P)), 3 = hash lo bits
struct DigitSpec {
  int mode;
  int shift;
  int bits;
  uint32_t P;
};
constexpr int kMaxPasses = 8;
struct DigitSpecs {
  DigitSpec d[kMaxPasses];
  int n;
};

// ------------------------------------------------------------------ launchers (per .cu)
// gen_coupled with src written as src_base + (parent index in this call)
int gen_records(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
                const cusci_integrals* ints, double threshold, cusci_records* out, uint32_t src_base);
int gen_count(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
              const cusci_integrals* ints, double threshold, uint64_t* count);
// Stage-3 contraction in pieces (energy.cu): the (key, psi) table once, any
// number of record batches accumulated exactly, e written once
struct CState {
  int W = 1;
  void* table = nullptr;
  uint64_t tslots = 0;
  int k = 0;
  unsigned long long* acc = nullptr;    // [4 n_parents] exact limbs
  unsigned long long* flags = nullptr;  // [2] missing, errors
  uint64_t n_parents = 0;
};
int contract_begin(cusci_ctx* ctx, Scratch& s, int W, const uint64_t* space, uint64_t n_space, const double* psi,
                   uint64_t n_parents, CState* st);
int contract_add(cusci_ctx* ctx, const CState& st, const uint64_t* keys, const double* hij, const uint32_t* src,
                 uint64_t n_rec);
int contract_end(cusci_ctx* ctx, const CState& st, double* e, uint64_t* n_missing);
int prep_build(cusci_ctx* ctx, const cusci_space* sp, const cusci_integrals* ints, double eps);

// exclusive scan of n values (u32 or u64) in place-safe out; optional device total
int scan_exclusive_u32(cusci_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n);
int scan_exclusive_u64(cusci_ctx* ctx, const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* total_dev);

// Onesweep LSD passes: pass 0 reads `in` and writes buf0, then the passes
// alternate buf0 <-> buf1; *out points at the buffer holding the result (`in`
// itself if every pass was trivial).  hist0 (host, optional, [2^bits of pass 0])
// receives pass 0's digit histogram.
int onesweep_passes(cusci_ctx* ctx, int W, const uint64_t* in, uint64_t* buf0, uint64_t* buf1, uint64_t n,
                    const DigitSpecs& specs, const uint64_t** out, uint64_t* hist0);
// LSD radix sort of keys[n][W] over bits [0, nbits); the sorted keys end in
// *out_sorted, which is `keys` or `alt` (both [n][W] device buffers).
int radix_sort_keys(cusci_ctx* ctx, int W, uint64_t* keys, uint64_t* alt, uint64_t n, int nbits,
                    uint64_t** out_sorted);
// local dedup (bucket.cu): out (capacity n) receives the distinct keys of in,
// sorted in the hash order; *n_out their number (host)
int local_dedup(cusci_ctx* ctx, int W, const uint64_t* in, uint64_t n, uint64_t* out, uint64_t* n_out);
// owner-side finalize: P pi-sorted runs back to back (counts HOST [P]) -> the
// distinct keys in pi order (no partition pass)
int runs_dedup(cusci_ctx* ctx, int W, const uint64_t* in, const uint64_t* counts, int P, uint64_t* out,
               uint64_t* n_out);
// owner range sizes of a hash-ordered array (host counts[P])
int owner_counts(cusci_ctx* ctx, int W, const uint64_t* keys, uint64_t n, int P, uint64_t* counts);
// unique compaction of sorted keys into out; count written to device *n_out_dev
int unique_sorted_keys(cusci_ctx* ctx, int W, const uint64_t* in, uint64_t n, uint64_t* out,
                       uint64_t* n_out_dev);
// dedup.cu: payload all-to-all-v of bins (send[r] keys to rank r, back to back)
// into a scratch buffer *rbuf (received runs back to back by source rank)
// The counts exchange carries each rank's local status: a rank that failed
// sends ~0 to every peer and every rank returns the agreed error (no peer is
// left waiting in a send/recv).  local_rc is this rank's status so far.
int exchange_bins(cusci_ctx* ctx, int W, const uint64_t* bins, const uint64_t* send, Scratch& s, uint64_t** rbuf,
                  uint64_t* nrecv, int local_rc = CUSCI_OK, uint64_t* recv_counts = nullptr);
int agree_status_all(cusci_ctx* ctx, int local);
// a8 + a9: the distinct keys of configs in pi order, grouped into P owner
// bins (back to back; counts HOST [P]); *total = distinct keys
int dedup_local_bins(cusci_ctx* ctx, int W, const uint64_t* configs, uint64_t n, int P, uint64_t* bins,
                     uint64_t* counts, uint64_t* total);
int nccl_ok(cusci_ctx* ctx, ncclResult_t r, const char* what);
// sync the stream and read a device u64
int read_u64(cusci_ctx* ctx, const uint64_t* dev, uint64_t* host, int count = 1);

}  // namespace cusci
