// Hamiltonian prep (Sec 4.2.1 "pre-process
// its rules into two highly compressed Excitation Tables").
//
// B200 design: instead of the paper's padded T_single /
// T_double, build UNPADDED CSR tables on device, once per (h, eri, K, eps):
//   * pair rows, one per spin-orbital pair p<q (row id q(q-1)/2 + p): the
//     entries (a<b, v) with a,b not in {p,q}, spin-allowed and |v| > eps,
//     v = <pq||ab> = d1 - d2 | d1 | -d2 (d1 = (PA|QB) [s_p=s_a,s_q=s_b],
//     d2 = (PB|QA) [s_p=s_b,s_q=s_a]); rows sorted by (b, a).  The doubles
//     threshold test |H| > eps is parent independent (|H| = |v|), so it is
//     folded in here exactly.  Point-group zeros drop out automatically.
//   * singles candidates per spin orbital p: same-spin a != p with any nonzero
//     constituent (h_PA, (PA|KK) or (PK|KA) for some K); all other singles are
//     sums of exact zeros.  The exact occupation-dependent value is summed at
//     generation time from the tables topp[K][P][A] = (PA|KK) and
//     tsame[K][P][A] = (PA|KK) - (PK|KA) (same ops, same order as the
//     definition, so the result is bit-identical).
#include <algorithm>
#include <cmath>

#include "internal.cuh"

namespace cusci {
namespace {

__device__ __forceinline__ long pidx(long a, long b) { return a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a; }
__device__ __forceinline__ double gint(const double* __restrict__ eri, int P, int Q, int R, int S) {
  return __ldg(eri + pidx(pidx(P, Q), pidx(R, S)));
}

// decode candidate index c -> (a, b), a < b, over all C(m,2) pairs in order (b, a)
__device__ __forceinline__ void decode_pair(uint32_t c, int& a, int& b) {
  int bb = (int)((1.0 + sqrt(1.0 + 8.0 * (double)c)) * 0.5);
  while ((uint32_t)bb * (bb - 1) / 2 > c) bb--;
  while ((uint32_t)(bb + 1) * bb / 2 <= c) bb++;
  b = bb;
  a = (int)(c - (uint32_t)bb * (bb - 1) / 2);
}

__device__ __forceinline__ bool pair_value(const double* __restrict__ eri, int p, int q, int a, int b, double eps,
                                           double& v) {
  if (a == p || a == q || b == p || b == q) return false;
  const int sp = p & 1, sq = q & 1, sa = a & 1, sb = b & 1;
  const bool e1 = (sp == sa) && (sq == sb);
  const bool e2 = (sp == sb) && (sq == sa);
  if (!e1 && !e2) return false;
  const int P = p >> 1, Q = q >> 1, A = a >> 1, B = b >> 1;
  double x;
  if (e1 && e2) x = __dsub_rn(gint(eri, P, A, Q, B), gint(eri, P, B, Q, A));
  else if (e1) x = gint(eri, P, A, Q, B);
  else x = -gint(eri, P, B, Q, A);
  v = x;
  return fabs(x) > eps;
}

__global__ void pair_count_kernel(const double* __restrict__ eri, int m, double eps, uint32_t* __restrict__ counts) {
  const int row = blockIdx.x;
  int q = (int)((1.0 + sqrt(1.0 + 8.0 * (double)row)) * 0.5);
  while (q * (q - 1) / 2 > row) q--;
  while ((q + 1) * q / 2 <= row) q++;
  const int p = row - q * (q - 1) / 2;
  const uint32_t ncand = (uint32_t)m * (m - 1) / 2;
  uint32_t cnt = 0;
  for (uint32_t c = threadIdx.x; c < ncand; c += blockDim.x) {
    int a, b;
    decode_pair(c, a, b);
    double v;
    cnt += pair_value(eri, p, q, a, b, eps, v) ? 1u : 0u;
  }
  __shared__ uint32_t red[32];
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
  if (lane_id() == 0) red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w];
    counts[row] = s;
  }
}

// ordered fill: the block walks candidates in chunks of blockDim, block-scans
// the keep flags and appends in candidate order (rows sorted by (b, a)).
__global__ void pair_fill_kernel(const double* __restrict__ eri, int m, double eps, const uint32_t* __restrict__ rowptr,
                                 PairEnt* __restrict__ ent) {
  const int row = blockIdx.x;
  int q = (int)((1.0 + sqrt(1.0 + 8.0 * (double)row)) * 0.5);
  while (q * (q - 1) / 2 > row) q--;
  while ((q + 1) * q / 2 <= row) q++;
  const int p = row - q * (q - 1) / 2;
  const uint32_t ncand = (uint32_t)m * (m - 1) / 2;
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t base;
  if (threadIdx.x == 0) base = rowptr[row];
  __syncthreads();
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
  for (uint32_t c0 = 0; c0 < ncand; c0 += blockDim.x) {
    const uint32_t c = c0 + threadIdx.x;
    int a = 0, b = 0;
    double v = 0;
    bool keep = false;
    if (c < ncand) {
      decode_pair(c, a, b);
      keep = pair_value(eri, p, q, a, b, eps, v);
    }
    const unsigned bal = __ballot_sync(kFull, keep);
    if (lane_id() == 0) wsum[w] = __popc(bal);
    __syncthreads();
    uint32_t off = 0, tot = 0;
    for (int i = 0; i < nw; i++) {
      if (i < w) off += wsum[i];
      tot += wsum[i];
    }
    if (keep) {
      const uint32_t pos = base + off + __popc(bal & lanemask_lt());
      PairEnt e;
      e.x = m <= 64 ? ((1ull << a) | (1ull << b)) : (uint64_t)(a | (b << 8));
      e.v = v;
      ent[pos] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
}

// singles: candidate flags per (p, a) and the [K][P][A] tables
__global__ void singles_tables_kernel(const double* __restrict__ h, const double* __restrict__ eri, int K,
                                      double* __restrict__ topp, double* __restrict__ tsame,
                                      uint8_t* __restrict__ nonzero /* [K][K] */) {
  const int P = blockIdx.x, A = blockIdx.y;
  bool nz = false;
  for (int Kk = threadIdx.x; Kk < K; Kk += blockDim.x) {
    const double j = gint(eri, P, A, Kk, Kk);
    const double x = gint(eri, P, Kk, Kk, A);
    const size_t o = ((size_t)Kk * K + P) * K + A;
    topp[o] = j;
    tsame[o] = __dsub_rn(j, x);
    nz |= (j != 0.0) || (x != 0.0);
  }
  nz = __syncthreads_or(nz);
  if (threadIdx.x == 0) nonzero[P * K + A] = (nz || h[P * K + A] != 0.0) ? 1 : 0;
}

__global__ void singles_rows_kernel(const uint8_t* __restrict__ nonzero, int K, uint32_t* __restrict__ srowptr,
                                    uint8_t* __restrict__ sa) {
  // tiny (m <= 128 rows): one thread does everything, deterministic order
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int m = 2 * K;
  uint32_t n = 0;
  for (int p = 0; p < m; p++) {
    srowptr[p] = n;
    for (int a = p & 1; a < m; a += 2) {
      if (a == p) continue;
      if (nonzero[(p >> 1) * K + (a >> 1)]) sa[n++] = (uint8_t)a;
    }
  }
  srowptr[m] = n;
}

}  // namespace

int prep_build(cusci_ctx* ctx, const cusci_space* sp, const cusci_integrals* ints, double eps) {
  Prep& pr = ctx->prep;
  const int K = ints->n_spatial, m = sp->m;
  if (pr.valid && pr.h == ints->h && pr.eri == ints->eri && pr.K == K && pr.eps == eps)
    return CUSCI_OK;
  if (pr.block) {
    CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    cudaFree(pr.block);
  }
  pr = Prep{};
  const uint32_t npq = (uint32_t)m * (m - 1) / 2;
  Scratch s(ctx);
  uint32_t* counts;
  uint8_t* nz;
  CUSCI_TRY(s.get_t(npq + 1, &counts));
  CUSCI_TRY(s.get_t((size_t)K * K, &nz));
  CUSCI_LAUNCH(ctx, PT_PREP, pair_count_kernel<<<npq, 256, 0, ctx->stream>>>(ints->eri, m, eps, counts));
  CUSCI_CUDA(ctx, cudaMemsetAsync(counts + npq, 0, sizeof(uint32_t), ctx->stream));
  // rowptr = exclusive scan of counts (npq + 1 entries -> last = nnz)
  uint32_t* rowptr_tmp;
  CUSCI_TRY(s.get_t(npq + 1, &rowptr_tmp));
  CUSCI_TRY(scan_exclusive_u32(ctx, counts, rowptr_tmp, npq + 1));
  uint32_t nnz32 = 0;
  CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, rowptr_tmp + npq, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  nnz32 = *(uint32_t*)ctx->host_pinned;
  const size_t nnz = nnz32;
  const size_t kkk = (size_t)K * K * K;
  // one block: rowptr | srowptr | ent | topp | tsame | sa
  size_t off = 0;
  auto place = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  const size_t o_rowptr = place(sizeof(uint32_t) * (npq + 1));
  const size_t o_srow = place(sizeof(uint32_t) * (m + 1));
  const size_t o_ent = place(sizeof(PairEnt) * (nnz ? nnz : 1));
  const size_t o_topp = place(sizeof(double) * kkk);
  const size_t o_tsame = place(sizeof(double) * kkk);
  const size_t o_sa = place((size_t)m * m);
  void* block = nullptr;
  if (cudaMalloc(&block, off) != cudaSuccess) {
    cudaGetLastError();
    return set_error(ctx, CUSCI_E_OOM, "prep tables (%zu bytes) allocation failed", off);
  }
  char* b8 = (char*)block;
  pr.block = block;
  pr.block_bytes = off;
  pr.rowptr = (uint32_t*)(b8 + o_rowptr);
  pr.srowptr = (uint32_t*)(b8 + o_srow);
  pr.ent = (PairEnt*)(b8 + o_ent);
  pr.topp = (double*)(b8 + o_topp);
  pr.tsame = (double*)(b8 + o_tsame);
  pr.sa = (uint8_t*)(b8 + o_sa);
  pr.nnz = nnz;
  CUSCI_CUDA(ctx, cudaMemcpyAsync(pr.rowptr, rowptr_tmp, sizeof(uint32_t) * (npq + 1), cudaMemcpyDeviceToDevice,
                                  ctx->stream));
  if (nnz) {
    CUSCI_LAUNCH(ctx, PT_PREP, pair_fill_kernel<<<npq, 256, 0, ctx->stream>>>(ints->eri, m, eps, pr.rowptr, pr.ent));
  }
  CUSCI_LAUNCH(ctx, PT_PREP, singles_tables_kernel<<<dim3(K, K), 64, 0, ctx->stream>>>(ints->h, ints->eri, K, pr.topp, pr.tsame, nz));
  CUSCI_LAUNCH(ctx, PT_PREP, singles_rows_kernel<<<1, 32, 0, ctx->stream>>>(nz, K, pr.srowptr, pr.sa));
  uint32_t sn = 0;
  CUSCI_CUDA(ctx, cudaMemcpyAsync(ctx->host_pinned, pr.srowptr + m, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUSCI_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  sn = *(uint32_t*)ctx->host_pinned;
  pr.snnz = sn;
  pr.h = ints->h;
  pr.eri = ints->eri;
  pr.K = K;
  pr.eps = eps;
  pr.valid = true;
  return CUSCI_OK;
}

}  // namespace cusci
