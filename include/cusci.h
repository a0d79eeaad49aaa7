/* cusci.h -- C ABI of libcusci, the B200-native (sm_100a) selected-CI hot path
 * of QiankunNet-cuSCI (arXiv 2604.15768):
 *
 *     gen_coupled(parents, integrals, threshold) -> dedup_global(configs) -> merge_space(space, new)
 *
 * Citations: "P:L" = /reference PAPER.md line L, "S:L" = SPEC.md line L.
 *
 * Conventions (readings r1-r9):
 *   - A configuration (determinant) over m spin orbitals is `words` uint64
 *     words, words = 1 if m <= 64 else 2 (m <= 128).  Spin orbital t lives in
 *     word t/64 at bit t%64.  Spin orbitals are interleaved:
 *     t = 2P + sigma, sigma 0 = alpha, 1 = beta; P = t/2 is the spatial index.
 *   - Key arrays are row-major [n][words].  Two key orders are used:
 *       big-integer order: the key as one unsigned integer, word (words-1)
 *         most significant -- the order of the f2 calls (dedup_sorted,
 *         sort_unique, ...);
 *       pool hash order pi (reading r13): pi(j) = (hi, lo) compared
 *         lexicographically, with fmix = the splitmix64 finalizer and
 *           words = 1: hi = fmix(w0), lo = 0;
 *           words = 2: lo = fmix(w1 ^ 0x9E3779B97F4A7C15), hi = fmix(w0 ^ lo);
 *         pi is a bijection, and owner(j) = floor(hi * world / 2^64), so
 *         every rank's shard is a contiguous pi range.  dedup_global's
 *         output, the pool and merge_space's inputs/outputs are strictly
 *         increasing in pi.
 *   - Integrals are real fp64: h[K*K] (symmetric, row-major) and the
 *     two-electron integrals (PQ|RS) in chemist notation, 8-fold packed:
 *       ij = max(P,Q)(max(P,Q)+1)/2 + min(P,Q);  idx = max(ij,kl)(max(ij,kl)+1)/2 + min(ij,kl).
 *
 * Memory: unless stated otherwise every array pointer is a DEVICE pointer on
 * the context's device.  Every call is ordered on the context's CUDA stream;
 * calls that return a count synchronise that stream before returning.
 * Inputs are caller-owned and read-only during the call; the library never
 * frees caller memory.  Outputs of dedup_global / merge_space(inserted) are
 * allocated with the context's allocator callback (cudaMallocAsync when no
 * callback is given) and ownership passes to the caller (free with the
 * matching free callback, or cusci_free when none was given).
 *
 * Errors: every entry point returning int returns 0 on success or one of the
 * CUSCI_E_* codes below; cusci_last_error(ctx) returns a one-line message.
 * A context that returned CUSCI_E_NCCL or CUSCI_E_CUDA is unusable
 * (the communicator has been aborted); destroy it.
 */
#ifndef CUSCI_H
#define CUSCI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CUSCI_OK 0
#define CUSCI_E_INVALID_ARG 1    /* m not in [2,128]; words mismatch; n_alpha+n_beta > m; eps < 0 or NaN; NULL required pointer */
#define CUSCI_E_INVALID_PARENT 2 /* a parent with a bit >= m or spin popcounts != (n_alpha, n_beta) */
#define CUSCI_E_CAPACITY 3       /* output capacity too small: *count holds the true total; retry with a larger buffer */
#define CUSCI_E_CUDA 4           /* CUDA runtime error */
#define CUSCI_E_NCCL 5           /* NCCL error (communicator aborted; all ranks report it) */
#define CUSCI_E_OOM 6            /* device scratch allocation failed */

#define CUSCI_MAX_WORLD 512      /* ranks per communicator */

typedef struct cusci_ctx cusci_ctx;    /* device, stream, NCCL comm, allocator, workspace, cached Hamiltonian prep */
typedef struct cusci_pool cusci_pool;  /* GPU-resident owned shard of the configuration space S (sorted, unique) */

typedef struct {
  int32_t m;        /* spin orbitals, 2 <= m <= 128, m even (m = 2K) */
  int32_t n_alpha;  /* electrons on even (alpha) spin orbitals */
  int32_t n_beta;   /* electrons on odd (beta) spin orbitals */
  int32_t words;    /* must equal (m <= 64 ? 1 : 2) */
} cusci_space;

typedef struct {
  int32_t n_spatial;  /* K = m/2 */
  const double* h;    /* device, [K*K] */
  const double* eri;  /* device, packed 8-fold, [npair(npair+1)/2], npair = K(K+1)/2 */
} cusci_integrals;

typedef struct {
  uint64_t* keys;     /* device, [capacity][words]   target configuration j          (required) */
  double* hij;        /* device, [capacity]          H_ij (fp64), |H_ij| > threshold (required) */
  uint32_t* src;      /* device, [capacity]          index of the parent i in `parents` (nullable) */
  int8_t* phase;      /* device, [capacity]          fermionic phase +-1 of the excitation (nullable) */
  uint64_t capacity;  /* records the buffers hold */
  uint64_t count;     /* OUT (host): number of records produced (the true total on CUSCI_E_CAPACITY) */
} cusci_records;

typedef struct {
  uint64_t* keys;   /* device, [count][words]; allocated by the library, owned by the caller */
  uint64_t count;
} cusci_keys;

/* Allocator callbacks (e.g. backed by the torch caching allocator).  alloc must
 * return a device pointer aligned to >= 256 bytes, usable on `stream`, or NULL. */
typedef void* (*cusci_alloc_fn)(size_t bytes, void* stream, void* user);
typedef void (*cusci_free_fn)(void* ptr, void* user);

/* ---- lifecycle ------------------------------------------------------------ */

/* Writes a fresh 128-byte NCCL unique id to host memory `out128` (call on rank
 * 0, then broadcast it to all ranks, e.g. with torch.distributed). */
int cusci_nccl_unique_id(void* out128);

/* Create a context on `device` for rank `rank` of `world` (1 <= world <=
 * CUSCI_MAX_WORLD, else CUSCI_E_INVALID_ARG).
 * nccl_unique_id: host pointer to the 128-byte id (required when world > 1;
 * collective over all ranks).  With world = 1 it is optional: when given, a
 * 1-rank NCCL communicator is created, which CUSCI_OPT_FORCE_COLLECTIVE uses.  cuda_stream: the cudaStream_t on
 * `device` every call is ordered on (NULL = the legacy default stream; pass the
 * stream the caller's producers and consumers of these buffers use).  alloc/free: output
 * allocator (both NULL = cudaMallocAsync / cudaFreeAsync on the stream). */
int cusci_init(cusci_ctx** ctx, int device, int rank, int world, const void* nccl_unique_id,
               void* cuda_stream, cusci_alloc_fn alloc, cusci_free_fn free_fn, void* alloc_user);
void cusci_finalize(cusci_ctx* ctx);
const char* cusci_last_error(const cusci_ctx* ctx);
/* Context options.  CUSCI_OPT_FORCE_COLLECTIVE (value 0/1): run the
 * collective protocol of dedup_global / dedup_sorted / energy_contract --
 * status-carrying count exchange, NCCL payload exchange (the own bin too,
 * through ncclSend/ncclRecv to self), owner-side finalize -- even at
 * world = 1 (needs a communicator: pass an NCCL id to cusci_init).  This is
 * how the exchange step is exercised on one GPU; results are
 * identical to the world = 1 shortcut.  Errors: E_INVALID_ARG (unknown
 * option, or no communicator). */
#define CUSCI_OPT_FORCE_COLLECTIVE 1
/* CUSCI_OPT_CONTRACT_PARTITION (value -1 / 0 / 1): energy_contract and the
 * Stage-3 stream paths first scatter the records by the top 8 bits of their
 * key's hash-order value into 256 regions, so the reverse-index probes of a
 * region stay inside an L2-resident slice of the (key, psi) table: 1 on,
 * 0 (default) / -1 off (on one N2 batch the partition cuts the contraction's
 * DRAM reads 4x but costs more than it saves).  Results are
 * identical either way (exact sums). */
#define CUSCI_OPT_CONTRACT_PARTITION 2
int cusci_set_option(cusci_ctx* ctx, int option, int64_t value);
/* Drop the cached Hamiltonian prep (call after mutating or freeing the
 * integrals the cache was built from). */
void cusci_invalidate_integrals(cusci_ctx* ctx);
/* Return the context's cached device memory to the driver: the scratch
 * arena (it grows to the peak of the calls made so far and is kept) and the
 * freed blocks of its stream-ordered memory pool (stream-stage buffers).
 * Synchronises the context stream.  Pools and outputs stay valid.  Use
 * between phases with different memory profiles (Sec 4.3: the
 * device as a scratchpad). */
int cusci_release_cached(cusci_ctx* ctx);
/* Free a library-allocated output when the context has no free callback. */
void cusci_free(cusci_ctx* ctx, void* ptr);
/* Number of kernels this context has launched (instrumentation). */
uint64_t cusci_kernel_launches(const cusci_ctx* ctx);
/* Per-kernel-class CUDA-event profiler (instrumentation for bench.py): when
 * enabled, every library launch is bracketed by an event pair on the context
 * stream.  cusci_profile_read synchronises the stream, writes the summed
 * milliseconds and launch counts per class into ms[n_tags] / launches[n_tags]
 * (class ids: 0 prep, 1 validate, 2 gen, 3 bucket dedup, 4 pack / owner
 * bounds, 5 partition histogram, 6 partition scatter, 7 scan, 8 unique,
 * 9 merge split, 10 merge tile, 11 sorted check, 12 NCCL exchange, 13 memset)
 * and clears the log. */
void cusci_profile_enable(cusci_ctx* ctx, int on);
int cusci_profile_read(cusci_ctx* ctx, double* ms, uint64_t* launches, int n_tags);
/* Local-dedup plan statistics accumulated since the last read (instrumentation
 * for bench.py's algorithmic-byte accounting): stats[0] = dedup calls,
 * stats[1] = keys in, stats[2] = key-passes of the partition (sum over calls
 * of keys x scatter passes), stats[3] = distinct keys out, stats[4] = bucket
 * work units, stats[5] = calls that took the overflow slow path, stats[6] =
 * keys read by histogram passes, stats[7] = keys scattered by the hist-free
 * first pass.  reset != 0 clears them.  Returns CUSCI_OK (CUSCI_E_INVALID_ARG
 * for NULL arguments). */
int cusci_dedup_stats(cusci_ctx* ctx, uint64_t stats[8], int reset);

/* ---- step 1: coupled generation ------------------------------------------ */

/* Upper bound on the records gen_coupled can emit for n_parents parents: the
 * dense closed form per parent, sum_s n_s v_s + sum_s C(n_s,2) C(v_s,2)
 * + n_a v_a n_b v_b, times n_parents (SURVEY 8 "closed forms"). Host only. */
uint64_t gen_coupled_bound(const cusci_space* sp, uint64_t n_parents);

/* For every parent i (device, [n_parents][words]) emit every configuration j
 * of the coupled set C_i (Eq. 4): all spin-conserving single
 * (p->a) and double (p<q -> a<b) excitations, with the Slater-Condon element
 * (Sec 4.2.1)
 *     single: H = ph * (h_PA + sum_{k in occ(i)\p, ascending} [(PA|KK) - [s_k = s_p] (PK|KA)])
 *     double: H = ph * <pq||ab>,  <pq||ab> = d1 - d2 | d1 | -d2 with
 *             d1 = (PA|QB) [s_p=s_a, s_q=s_b], d2 = (PB|QA) [s_p=s_b, s_q=s_a]
 * and ph the fermionic phase of sequential singles p->a then q->b,
 * keeping the record iff |H| > threshold (strict; Alg. 1 line 12).
 * The diagonal is not emitted.  Records are written compactly (no gaps)
 * into `out` in an unspecified order (src identifies the parent; compare
 * record sets after sorting by (src, key)).  threshold >= 0 (NaN rejected).
 * Parents are validated on device before anything is written
 * (CUSCI_E_INVALID_PARENT, the message names the first bad index).
 * If the total exceeds out->capacity, nothing beyond capacity is written,
 * out->count = true total and CUSCI_E_CAPACITY is returned.
 * The Hamiltonian prep (pair tables) is built on first use and cached per
 * (h pointer, eri pointer, K, threshold) without re-reading the integrals:
 * after mutating the integrals in place, or freeing them while the context
 * lives (a new buffer can reuse the address), call cusci_invalidate_integrals
 * (the Python binding keeps the integrals of the cached prep alive and
 * invalidates when another integrals object is passed). */
int gen_coupled(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
                const cusci_integrals* ints, double threshold, cusci_records* out);

/* Exact record count gen_coupled would produce (no records written). */
int gen_coupled_count(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents, uint64_t n_parents,
                      const cusci_integrals* ints, double threshold, uint64_t* count);

/* ---- step 2: global de-duplication (COLLECTIVE when world > 1) ------------ */

/* Global de-duplication of the union over all ranks of `configs` (device,
 * [n][words], n < 2^32) (Sec 2.2; Sec 4.1.1): local
 * unique filter, hash-owner partition owner(j) = floor(hi(j) *
 * world / 2^64) (DESIGN.md r9), one all-to-all exchange over NCCL,
 * owner-side unique of the received runs.  On return owned_unique holds,
 * strictly increasing in the pool hash order pi, exactly the distinct keys j
 * of the global union with owner(j) == rank.  Every rank must call it with
 * the same cusci_space.  Errors are agreed across ranks: a rank whose
 * arguments or local step failed still takes part in the count exchange
 * (sending a failure marker), and every rank then returns an error (its own
 * code, or that code of a peer's failure) -- no rank is left blocked in the
 * exchange. */
int dedup_global(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n,
                 cusci_keys* owned_unique);

/* The two local halves of dedup_global, exposed for logical-rank tests and
 * custom transports:
 *   dedup_partition: local unique filter + owner partition into n_owners bins;
 *     bins->keys holds the bins back to back (bin r first at offset
 *     sum_{r'<r} counts[r']); counts (HOST, [n_owners]) receives the sizes.
 *   dedup_finalize: unique of a received buffer (device, [n][words]) into
 *     the pool hash order pi.  Its buckets are planned for keys spread over
 *     the whole hash space; on one owner's keys (1/P of the space) it is
 *     exact but may take the slow path (a full sort) -- dedup_global uses
 *     dedup_finalize_runs, which buckets over the received keys' range. */
int dedup_partition(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n,
                    int n_owners, cusci_keys* bins, uint64_t* counts);
int dedup_finalize(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* keys, uint64_t n,
                   cusci_keys* unique_sorted);
/* dedup_finalize for what dedup_global's owner receives: n_runs runs back to
 * back (device keys; run r has run_counts[r] keys, HOST array), each strictly
 * increasing in pi (a dedup_partition bin of some rank).  Same output as
 * dedup_finalize on the concatenation, without a partition pass: every
 * bucket's keys are located in each run by binary search, and the buckets
 * cover only the runs' hash range [min, max] (an owner's runs lie in 1/P of
 * the space), so they hold the planned number of keys (1 <= n_runs <=
 * CUSCI_MAX_WORLD; unsorted runs give an unspecified result). */
int dedup_finalize_runs(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* keys, const uint64_t* run_counts,
                        int n_runs, cusci_keys* unique_sorted);

/* ---- the paper's sort-based regular-sampling dedup ------
 * PAPER.md Sec 4.1.1 :448-462 ("Sort-Based Regular Sampling De-duplication",
 * Steps 1-3).  Key order here is the big-integer order of the configuration
 * bitstring (bit t of the key = orbital t; at words = 2 word 1 is the high
 * word), NOT the pool's hash order.  All arrays [count][words] uint64.
 *
 * dedup_sorted (COLLECTIVE over ctx's ranks; world <= 256): Step 1 local LSD
 *   radix sort + unique, n_samples (1..65536) regular samples at indices
 *   floor(k |D| / n_samples) (all of D if |D| < n_samples); Step 2 all-gather
 *   of the samples, sort, P-1 splitters sorted[floor(r M / P)], r = 1..P-1,
 *   lower-bound partition of the local array; Step 3 NCCL all-to-all-v and
 *   sort + unique of the received runs.  owned_sorted receives this rank's
 *   shard (allocated through the ctx allocator, caller frees): the distinct
 *   keys x of the union of all ranks' configs with spl_r <= x < spl_{r+1}
 *   (spl_0 = -inf, spl_P = +inf), ascending.  splitters_host (HOST,
 *   nullable, [(P-1)][words]) receives the splitters.  world = 1: the sorted
 *   unique keys.  Errors: E_INVALID_ARG (bad arguments on any rank: every
 *   rank returns it), E_OOM, E_CUDA / E_NCCL (context unusable).
 *
 * Building blocks (one GPU, no communication; the virtual-rank tests and the
 * bench's balance metrics compose them):
 *   sort_unique: out <- sorted unique keys of configs (DEVICE, n < 2^32).
 *   regular_samples: samples (DEVICE, >= min(n_samples, n) keys) <- the
 *     regular samples of a sorted unique array; *n_taken (HOST) their number.
 *   select_splitters: splitters (DEVICE, [n_parts-1]) <- the splitters of
 *     n_samples gathered samples (DEVICE, any order; not modified).
 *   split_bounds: bounds (HOST, [n_parts+1]) <- 0, lower_bound(sorted,
 *     spl_r) for r = 1..n_parts-1, n.  n_parts in 1..256. */
int dedup_sorted(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n, int n_samples,
                 cusci_keys* owned_sorted, uint64_t* splitters_host);
int sort_unique(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* configs, uint64_t n, cusci_keys* out);
int regular_samples(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* sorted, uint64_t n, int n_samples,
                    uint64_t* samples, uint64_t* n_taken);
int select_splitters(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* samples, uint64_t n_samples, int n_parts,
                     uint64_t* splitters);
int split_bounds(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* sorted, uint64_t n, const uint64_t* splitters,
                 int n_parts, uint64_t* bounds);

/* ---- step 3: the GPU-resident configuration pool --------------------------- */

/* Create an empty pool (capacity = initial key capacity; it grows). */
int cusci_pool_create(cusci_ctx* ctx, const cusci_space* sp, uint64_t capacity, cusci_pool** out);
/* Read-only view of the pool's keys (strictly increasing in pi); valid until
 * the next merge_space or cusci_pool_merge into this pool. */
int cusci_pool_view(const cusci_pool* pool, const uint64_t** keys, uint64_t* count);
/* Empty the pool (keeps its buffers, so a reused pool never reallocates). */
int cusci_pool_clear(cusci_pool* pool);
/* Copy the pool's keys into dst (device, capacity_keys >= count), stream-ordered. */
int cusci_pool_copy(const cusci_pool* pool, uint64_t* dst, uint64_t capacity_keys);
void cusci_pool_destroy(cusci_pool* pool);

/* S <- S u new (Sec 2.2).  new_keys (device,
 * [n_new][words]) must be strictly increasing in the pool hash order pi (as
 * returned by dedup_global on this rank; CUSCI_E_INVALID_ARG otherwise -- a
 * big-integer-sorted array such as dedup_sorted's output is rejected).  If
 * `inserted` is non-NULL it receives new \ S_old, in pi order.  Local: the pool shard and the
 * new keys share the owner function, so no communication is needed. */
int merge_space(cusci_ctx* ctx, cusci_pool* space, const uint64_t* new_keys, uint64_t n_new,
                cusci_keys* inserted);
/* S <- S u src for two pools of the same space (S <- S u C with C
 * held in a pool).  src's keys are read in place and, being a pool's, are
 * sorted and unique by construction, so they are not re-validated (the one
 * difference from merge_space(space, view(src))).  src may be space itself.
 * inserted as in merge_space.  Errors: E_INVALID_ARG (NULL, pools of another
 * context or of different spaces), E_OOM (pool growth), E_CUDA. */
int cusci_pool_merge(cusci_ctx* ctx, cusci_pool* space, const cusci_pool* src, cusci_keys* inserted);

/* ---- next row: Stage-3 contraction ----------------------- */

/* Local-energy numerators of Eq. 5 over this rank's records, with
 * the just-in-time reverse index of Stage 3 ("we construct
 * the required reverse index just-in-time by searching against the full
 * unique set"):
 *     e[s] = sum over records r with src[r] = s of  H[r] * psi[idx(key[r])]
 * idx(key) = position of key in `space_keys` ([n_space][words], device, sorted
 * strictly in the pool hash order, e.g. a pool view or a dedup_global output);
 * psi[n_space] (device, fp64) is aligned with it.  keys/hij/src are a
 * gen_coupled output (device, n_rec records, src < n_parents); e[n_parents]
 * (device, fp64) is overwritten.
 * Deterministic reduction (reading r14): each product p = H*psi is
 * the IEEE fp64 product, rounded half-to-even to the grid 2^-80 and summed
 * EXACTLY in 128-bit integers (order independent), and e[s] is that sum
 * rounded once to fp64.  Requires |p| < 2^20 (CUSCI_E_INVALID_ARG otherwise,
 * e untouched).  A record whose key is not in the space contributes 0 and is
 * counted in *n_missing (host).  src[r] >= n_parents: CUSCI_E_INVALID_ARG.
 * COLLECTIVE when world > 1 (or CUSCI_OPT_FORCE_COLLECTIVE): space_keys/psi
 * are this rank's OWNED shard (dedup_global's output on this rank), and the
 * records' keys are looked up at their owners: each rank sends its records'
 * distinct keys to the owners (the dedup_global partition + exchange), the
 * owners answer with psi over a reverse exchange, and the records are
 * contracted locally (PAPER.md :634 "just-in-time" reverse index).  Errors are
 * agreed across ranks as in dedup_global. */
int energy_contract(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* keys, const double* hij,
                    const uint32_t* src, uint64_t n_rec, uint64_t n_parents, const uint64_t* space_keys,
                    uint64_t n_space, const double* psi, double* e, uint64_t* n_missing);

/* ---- next row: memory-centric streaming -------------------
 * PAPER.md Sec 4.3 :583-634 (fig:mem_flow): mini-batches with the device as a
 * scratchpad; separate streams for host->device prefetch, compute and
 * device->host offload, double-buffered so batch i+1 loads and batch i-1
 * offloads while batch i computes (:617).  Host buffers should be pinned
 * (cudaHostAlloc / torch pin_memory) for the copies to overlap. */
typedef struct {
  uint64_t batch_parents;  /* parents per mini-batch (stream_generate, stream_energy_regen) */
  uint64_t batch_records;  /* stream_energy: records per mini-batch; stream_generate: record-slot capacity
                              hint (0 = count every batch exactly first; a batch above the hint is
                              counted and generated again) */
  uint64_t* host_keys;     /* HOST [host_capacity][words]: the "original set" (nullable: no offload) */
  double* host_hij;        /* HOST [host_capacity] */
  uint32_t* host_src;      /* HOST [host_capacity]: GLOBAL parent index (batch start + index in batch) */
  uint64_t host_capacity;  /* records the host buffers hold */
} cusci_stream_cfg;
typedef struct {
  uint64_t batches, records, unique;  /* unique: the pool's size after stream_generate */
  double ms_wall;                     /* the stage on the device clock (events) */
  double ms_h2d, ms_compute, ms_d2h;  /* busy time of each stream (sum of its spans): overlap = sum - wall */
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t peak_device_bytes;         /* library-held device memory high-water mark during the stage */
} cusci_stream_stats;

/* Stage 1 (PAPER.md :628 "cold data are immediately offloaded to host memory
 * via an asynchronous D2H stream ... global de-duplication is then performed
 * on the retained device data"): for each parent mini-batch of parents_host
 * (HOST [n_parents][words]): prefetch the next batch (H2D stream), gen_coupled
 * into one of two device record slots, dedup_global of its keys and
 * merge_space into unique_pool (compute stream), and -- if host_keys is set --
 * offload the batch's records into the host original set (D2H stream), in
 * batch order, src = global parent index (two record slots; one without
 * offload).  Peak device memory is bounded by
 * the batch, not by n_parents (plus the pool).  COLLECTIVE when world > 1
 * (dedup_global; the batch count is agreed, max over ranks).  Errors: as
 * gen_coupled / dedup_global / merge_space; E_CAPACITY when the host buffers
 * hold fewer records than generated (stats->records = the true total, the
 * first host_capacity records were written, the pool is complete). */
int stream_generate(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents_host, uint64_t n_parents,
                    const cusci_integrals* ints, double threshold, const cusci_stream_cfg* cfg,
                    cusci_pool* unique_pool, cusci_stream_stats* stats);
/* Stage 3, reload (PAPER.md :634): the original set (the cfg host buffers,
 * n_rec records) streamed back in batches of batch_records (H2D stream,
 * double-buffered prefetch) and contracted as energy_contract does against
 * (space_keys, psi) (device): one table for the stage, batches accumulated
 * exactly, so e is bit-identical to one energy_contract over all records.
 * One rank (E_INVALID_ARG when collective). */
int stream_energy(cusci_ctx* ctx, const cusci_space* sp, const cusci_stream_cfg* cfg, uint64_t n_rec,
                  uint64_t n_parents, const uint64_t* space_keys, uint64_t n_space, const double* psi, double* e,
                  uint64_t* n_missing, cusci_stream_stats* stats);
/* Stage 3, regenerate (the B200 alternative to keeping the original set):
 * the records of each parent mini-batch are generated again on the device
 * (parents prefetched H2D) and contracted; same e as stream_energy, bit for
 * bit, with no host original set at all.  One rank. */
int stream_energy_regen(cusci_ctx* ctx, const cusci_space* sp, const uint64_t* parents_host, uint64_t n_parents,
                        const cusci_integrals* ints, double threshold, const cusci_stream_cfg* cfg,
                        const uint64_t* space_keys, uint64_t n_space, const double* psi, double* e,
                        uint64_t* n_missing, cusci_stream_stats* stats);

/* ---- next row: SCI growth with a surrogate selector --------
 * One iteration of the selected-CI loop (Sec 2.2 :308-312, Fig. 2:
 * generate C from S, de-duplicate, select the top-K new configurations,
 * merge them into S), with the NNQS amplitude replaced by the heat-bath
 * surrogate (reading r16):
 *   records (i -> j, H_ij) = gen_coupled(S); C = dedup_global(records);
 *   score_j = max over records of |p|, p = fl(H_ij psi_i), ties between
 *     equal |p| by sign (negative wins), for j in C \ S (score 0 excluded);
 *   selected = the K best scores, ties in the pool hash order pi;
 *   S <- S u selected (merge_space);  psi_out = psi over the new S in pool
 *   order: psi_i kept for i in S, psi_j = -p_j (first-order amplitude with a
 *   unit energy denominator) for the new j.
 * space: the pool holding S; psi (device, [|S|]) aligned with its pi order;
 * psi_out (device, capacity psi_out_capacity >= |S| + K) receives the new
 * psi.  One rank (E_INVALID_ARG when collective).  E_CAPACITY if psi_out is
 * too small (S has been merged; stats->space_after = |S|). */
typedef struct {
  uint64_t records, unique;         /* records of S, distinct coupled configurations */
  uint64_t candidates, selected;    /* j in C \ S with a positive score; selected (<= K) */
  uint64_t space_before, space_after;
  double ms;                        /* device time of the step */
} cusci_grow_stats;
int sci_grow_step(cusci_ctx* ctx, const cusci_space* sp, cusci_pool* space, const double* psi,
                  const cusci_integrals* ints, double threshold, uint64_t K, double* psi_out,
                  uint64_t psi_out_capacity, cusci_grow_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* CUSCI_H */
