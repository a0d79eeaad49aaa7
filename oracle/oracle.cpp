// ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded CPU definition of what the cuSCI hot path
// computes (arXiv 2604.15768).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  It
// shares no code, header, table or constant generator with the CUDA path in
// paper_2604_15768_b200/csrc/.
//
// What it computes (each function cites the passage it follows):
//   oracle_gen      -- the coupled sets C_i of Eq. 4 (Sec 2.1)
//                      with H_ij from the Slater-Condon rules (PAPER.md:505,
//                      Sec 4.2.1; SPEC.md:147 slater_condon) and the threshold
//                      |H_ij| > eps (Alg. 1 line 12).
//   oracle_dedup    -- the global de-duplication of {C_i} (PAPER.md:301-303,
//                      Sec 2.2; Sec 4.1.1 Step 3) with std::set,
//                      restricted to the keys a given hash owner holds
//                      (reading r9).
//   oracle_merge    -- S' = S u U and inserted = U \ S (PAPER.md:311-312,
//                      Sec 2.2 "merging them into S").
//   oracle_apply_single / oracle_apply_double -- SPEC.md:56-73 (apply_single,
//                      apply_double: sequential singles p->a then q->b).
//
// Conventions (readings r1-r8): spin orbital t = 2P + sigma
// (interleaved), orbital t in word t/64 bit t%64, keys ordered as big
// integers (word 1 most significant), chemist (PQ|RS) packed 8-fold.
//
// Parity pins for every function live in tests/test_oracle_*.py; none is
// "parity unpinned".
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <map>
#include <set>
#include <vector>
#include <algorithm>
#include <iterator>

namespace {

struct Key {
  uint64_t w[2];
  bool operator<(const Key& o) const {  // big-integer order, word 1 most significant
    if (w[1] != o.w[1]) return w[1] < o.w[1];
    return w[0] < o.w[0];
  }
  bool operator==(const Key& o) const { return w[0] == o.w[0] && w[1] == o.w[1]; }
};

Key load_key(const uint64_t* p, int W) {
  Key k;
  k.w[0] = p[0];
  k.w[1] = (W == 2) ? p[1] : 0;
  return k;
}

void store_key(uint64_t* p, int W, const Key& k) {
  p[0] = k.w[0];
  if (W == 2) p[1] = k.w[1];
}

bool bit(const Key& k, int t) { return (k.w[t / 64] >> (t % 64)) & 1ull; }
void flip(Key& k, int t) { k.w[t / 64] ^= (1ull << (t % 64)); }

// number of occupied orbitals strictly between x and y, counted one by one
int occupied_between(const Key& k, int x, int y) {
  int lo = x < y ? x : y, hi = x < y ? y : x, c = 0;
  for (int t = lo + 1; t < hi; t++) c += bit(k, t);
  return c;
}

// (PQ|RS) from the 8-fold packed array (reading r4)
struct Ints {
  int K;
  const double* h;    // [K*K]
  const double* eri;  // packed
  static long pidx(long a, long b) { return a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a; }
  double g(int P, int Q, int R, int S) const { return eri[pidx(pidx(P, Q), pidx(R, S))]; }
  double hh(int P, int Q) const { return h[(long)P * K + Q]; }
};

struct Rec {
  uint32_t src;
  Key key;
  double H;
  int8_t phase;
};

struct GenResult {
  std::vector<Rec> recs;
};

struct KeysResult {
  std::vector<Key> keys;
  std::vector<Key> extra;  // merge: inserted
};

// owner(j) = floor(mix(j) * P / 2^64), mix = splitmix64 finalizer
// (reading r9).  Written out here independently.
uint64_t fmix(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
uint32_t owner_of(const Key& k, int W, uint32_t P) {
  uint64_t mix = (W == 1) ? fmix(k.w[0]) : fmix(k.w[0] ^ fmix(k.w[1] ^ 0x9E3779B97F4A7C15ull));
  unsigned __int128 prod = (unsigned __int128)mix * P;
  return (uint32_t)(prod >> 64);
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------------------
// parent validation: popcount(even bits) = n_alpha,
// popcount(odd bits) = n_beta, no bit >= m.  Returns the first bad index or -1.
long long oracle_validate(int m, int n_alpha, int n_beta, int W, const uint64_t* parents, long long n) {
  for (long long s = 0; s < n; s++) {
    Key k = load_key(parents + s * W, W);
    int na = 0, nb = 0, bad = 0;
    for (int t = 0; t < 64 * W; t++) {
      if (!bit(k, t)) continue;
      if (t >= m) bad = 1;
      else if (t % 2 == 0) na++;
      else nb++;
    }
    if (bad || na != n_alpha || nb != n_beta) return s;
  }
  return -1;
}

// ---------------------------------------------------------------------------
// SPEC.md:56-62 apply_single: result = c xor p xor a, parity =
// (-1)^(occupied orbitals strictly between p and a).  Returns 0 ok, -1 invalid.
int oracle_apply_single(int W, const uint64_t* c, int p, int a, uint64_t* out, int* parity) {
  Key k = load_key(c, W);
  if (!bit(k, p) || bit(k, a) || p == a) return -1;
  *parity = (occupied_between(k, p, a) % 2) ? -1 : 1;
  flip(k, p);
  flip(k, a);
  store_key(out, W, k);
  return 0;
}

// SPEC.md:63-73 apply_double: p<q occupied, a<b unoccupied; single p->a on c,
// then q->b on the intermediate; parity = product.
int oracle_apply_double(int W, const uint64_t* c, int p, int q, int a, int b, uint64_t* out, int* parity) {
  Key k = load_key(c, W);
  if (!(p < q) || !(a < b) || !bit(k, p) || !bit(k, q) || bit(k, a) || bit(k, b)) return -1;
  int s1 = occupied_between(k, p, a) % 2;
  flip(k, p);
  flip(k, a);
  int s2 = occupied_between(k, q, b) % 2;
  flip(k, q);
  flip(k, b);
  *parity = ((s1 + s2) % 2) ? -1 : 1;
  store_key(out, W, k);
  return 0;
}

// ---------------------------------------------------------------------------
// Coupled-set generation, Eq. 4: "record the indices of all
// 1s in the bitstring of i and enumerate all configurations obtained by moving
// one or two of these occupied positions"; keep j iff |H_ij| > eps
// (PAPER.md:542).  H_ij by the Slater-Condon rules:
//   single p->a:  H = parity * ( h_PA + sum_{k in occ(i)\p, ascending}
//                                 [ (PA|KK) - [sigma_k = sigma_p] (PK|KA) ] )
//   double pq->ab (p<q, a<b): H = parity * <pq||ab>, with
//       d1 = (PA|QB) if sigma_p = sigma_a and sigma_q = sigma_b
//       d2 = (PB|QA) if sigma_p = sigma_b and sigma_q = sigma_a
//       <pq||ab> = d1 - d2 (both), d1 (only d1), -d2 (only d2), 0 (neither).
// Capital letters are spatial indices t/2.  The diagonal is not emitted
// (reading r7).  Records are returned in canonical order (src, key).
void* oracle_gen(int m, int n_alpha, int n_beta, int W, const uint64_t* parents, long long n_parents,
                 int K, const double* h, const double* eri, double eps) {
  (void)n_alpha;
  (void)n_beta;
  Ints I{K, h, eri};
  GenResult* R = new GenResult;
  for (long long s = 0; s < n_parents; s++) {
    const Key i = load_key(parents + s * W, W);
    std::vector<int> occ, vir;
    for (int t = 0; t < m; t++) (bit(i, t) ? occ : vir).push_back(t);
    std::map<Key, std::pair<double, int>> Ci;
    // singles
    for (int p : occ) {
      for (int a : vir) {
        if (p % 2 != a % 2) continue;  // spin-forbidden: element is identically zero
        int P = p / 2, A = a / 2;
        double v = I.hh(P, A);
        for (int k : occ) {
          if (k == p) continue;
          int Kk = k / 2;
          double t = I.g(P, A, Kk, Kk);
          if (k % 2 == p % 2) t = t - I.g(P, Kk, Kk, A);
          v = v + t;
        }
        Key j = i;
        flip(j, p);
        flip(j, a);
        int ph = (occupied_between(i, p, a) % 2) ? -1 : 1;
        double H = ph * v;
        if (std::fabs(H) > eps) Ci[j] = {H, ph};
      }
    }
    // doubles
    for (size_t x = 0; x < occ.size(); x++)
      for (size_t y = x + 1; y < occ.size(); y++)
        for (size_t u = 0; u < vir.size(); u++)
          for (size_t w = u + 1; w < vir.size(); w++) {
            int p = occ[x], q = occ[y], a = vir[u], b = vir[w];
            int P = p / 2, Q = q / 2, A = a / 2, B = b / 2;
            bool e1 = (p % 2 == a % 2) && (q % 2 == b % 2);
            bool e2 = (p % 2 == b % 2) && (q % 2 == a % 2);
            double v = 0.0;
            if (e1 && e2) v = I.g(P, A, Q, B) - I.g(P, B, Q, A);
            else if (e1) v = I.g(P, A, Q, B);
            else if (e2) v = -I.g(P, B, Q, A);
            Key i1 = i;
            int s1 = occupied_between(i1, p, a) % 2;
            flip(i1, p);
            flip(i1, a);
            int s2 = occupied_between(i1, q, b) % 2;
            Key j = i1;
            flip(j, q);
            flip(j, b);
            int ph = ((s1 + s2) % 2) ? -1 : 1;
            double H = ph * v;
            if (std::fabs(H) > eps) Ci[j] = {H, ph};
          }
    for (auto& kv : Ci) R->recs.push_back(Rec{(uint32_t)s, kv.first, kv.second.first, (int8_t)kv.second.second});
  }
  return R;
}

long long oracle_gen_count(void* r) { return (long long)((GenResult*)r)->recs.size(); }

void oracle_gen_copy(void* r, int W, uint64_t* keys, double* H, uint32_t* src, int8_t* phase) {
  GenResult* R = (GenResult*)r;
  for (size_t x = 0; x < R->recs.size(); x++) {
    const Rec& e = R->recs[x];
    if (keys) store_key(keys + x * W, W, e.key);
    if (H) H[x] = e.H;
    if (src) src[x] = e.src;
    if (phase) phase[x] = e.phase;
  }
}

void oracle_gen_free(void* r) { delete (GenResult*)r; }

// ---------------------------------------------------------------------------
// Global de-duplication (Sec 4.1.1 Step 3):
// U = the set of all keys, as a std::set (big-integer order); the shard of
// owner `rank` among P owners is { j in U : owner(j) = rank }.
void* oracle_dedup(int W, const uint64_t* keys, long long n, int P, int rank) {
  std::set<Key> U;
  for (long long x = 0; x < n; x++) U.insert(load_key(keys + x * W, W));
  KeysResult* R = new KeysResult;
  for (const Key& k : U)
    if (P <= 1 || owner_of(k, W, (uint32_t)P) == (uint32_t)rank) R->keys.push_back(k);
  return R;
}

// owner of each key (for tests of the partition rule)
void oracle_owner(int W, const uint64_t* keys, long long n, int P, uint32_t* out) {
  for (long long x = 0; x < n; x++) out[x] = owner_of(load_key(keys + x * W, W), W, (uint32_t)P);
}

// ---------------------------------------------------------------------------
// merge_space ("merging them into S"): S' = S u U
// (std::set_union), inserted = U \ S (std::set_difference).  S and U are
// sets (duplicates in the input collapse).
void* oracle_merge(int W, const uint64_t* S, long long nS, const uint64_t* U, long long nU) {
  std::set<Key> s, u;
  for (long long x = 0; x < nS; x++) s.insert(load_key(S + x * W, W));
  for (long long x = 0; x < nU; x++) u.insert(load_key(U + x * W, W));
  KeysResult* R = new KeysResult;
  std::set_union(s.begin(), s.end(), u.begin(), u.end(), std::back_inserter(R->keys));
  std::set_difference(u.begin(), u.end(), s.begin(), s.end(), std::back_inserter(R->extra));
  return R;
}

long long oracle_keys_count(void* r, int which) {
  KeysResult* R = (KeysResult*)r;
  return (long long)(which ? R->extra.size() : R->keys.size());
}

void oracle_keys_copy(void* r, int which, int W, uint64_t* out) {
  KeysResult* R = (KeysResult*)r;
  const std::vector<Key>& v = which ? R->extra : R->keys;
  for (size_t x = 0; x < v.size(); x++) store_key(out + x * W, W, v[x]);
}

void oracle_keys_free(void* r) { delete (KeysResult*)r; }

}  // extern "C"
