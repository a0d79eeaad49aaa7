/* HF-ball parent sampler (input generator only; holds none of the method's
 * arithmetic).  Recipe: SURVEY.md 8(d) / DESIGN.md "Input recipe".
 *
 * Draw loop (counter-based splitmix64 RNG, so the stream is identical on every
 * machine):
 *   L ~ level_weights; La ~ Binomial(L, 1/2); Lb = L - La; reject the draw if
 *   La or Lb exceeds min(n_sigma, K - n_sigma) (clipping would change L);
 *   per spin: La holes among the HF-occupied spatial orbitals P < n_sigma,
 *   drawn without replacement with weight exp((P - n_sigma)/tau), and La
 *   particles among A >= n_sigma with weight exp(-(A - n_sigma)/tau);
 *   if g > 1 keep only determinants whose XOR of occupied irreps (P mod g,
 *   both spins) is 0; keep the first n_parents distinct determinants.
 *   If, over a window of 2^20 draws, fewer than 10% of draws are new, tau is
 *   widened by 1.25x (the ball is too small for the requested count).
 * Output: uint64 [n_parents][W] in draw order (the caller sorts).  Returns the
 * number written (< n_parents only if max_draws was exhausted).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t smix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
typedef struct { uint64_t seed, ctr; } rng_t;
static inline uint64_t rnext(rng_t* r) { r->ctr++; return smix(r->seed + r->ctr * 0x9E3779B97F4A7C15ull); }
static inline double runif(rng_t* r) { return (double)(rnext(r) >> 11) * 0x1.0p-53; }

static int pick(rng_t* r, const double* cdf, int n) {
  double u = runif(r) * cdf[n - 1];
  int lo = 0, hi = n - 1;
  while (lo < hi) { int mid = (lo + hi) / 2; if (cdf[mid] > u) hi = mid; else lo = mid + 1; }
  return lo;
}

/* choose k distinct of n with weights (cdf), mark in sel[] */
static void choose(rng_t* r, const double* cdf, int n, int k, uint8_t* sel) {
  memset(sel, 0, (size_t)n);
  for (int got = 0; got < k;) {
    int c = pick(r, cdf, n);
    if (!sel[c]) { sel[c] = 1; got++; }
  }
}

static uint64_t hkey(const uint64_t* k, int W) {
  uint64_t h = smix(k[0] ^ 0x1234567ull);
  if (W == 2) h = smix(h ^ k[1]);
  return h;
}

long long synth_hf_ball(int K, int na, int nb, int g, long long n_parents, uint64_t seed,
                        double tau, const double* level_w, int n_levels, long long max_draws,
                        uint64_t* out) {
  const int m = 2 * K, W = m <= 64 ? 1 : 2;
  rng_t r = {seed, 0};
  double lcdf[16];
  double acc = 0;
  for (int i = 0; i < n_levels; i++) { acc += level_w[i]; lcdf[i] = acc; }
  /* open-addressing set of found keys */
  uint64_t cap = 1;
  while (cap < (uint64_t)n_parents * 2 + 16) cap <<= 1;
  uint64_t* tab = (uint64_t*)calloc(cap * W, sizeof(uint64_t));
  uint8_t* used = (uint8_t*)calloc(cap, 1);
  double *hc[2], *pc[2];
  uint8_t sel_h[128], sel_p[128];
  int ns[2] = {na, nb};
  long long found = 0, window = 0, window_new = 0;
  for (int s = 0; s < 2; s++) { hc[s] = malloc(sizeof(double) * (K + 1)); pc[s] = malloc(sizeof(double) * (K + 1)); }
  for (;;) {
    for (int s = 0; s < 2; s++) {
      double a = 0;
      for (int P = 0; P < ns[s]; P++) { a += exp((P - ns[s]) / tau); hc[s][P] = a; }
      a = 0;
      for (int A = ns[s]; A < K; A++) { a += exp(-(A - ns[s]) / tau); pc[s][A - ns[s]] = a; }
    }
    int widen = 0;
    while (!widen) {
      if (max_draws-- <= 0 || found >= n_parents) goto done;
      int L = pick(&r, lcdf, n_levels);
      int La = 0;
      for (int i = 0; i < L; i++) La += (int)(rnext(&r) >> 63);
      int Lb = L - La;
      int mxa = na < K - na ? na : K - na, mxb = nb < K - nb ? nb : K - nb;
      window++;
      if (La > mxa || Lb > mxb) goto tally;
      {
        uint64_t key[2] = {0, 0};
        int sym = 0;
        int Ls[2] = {La, Lb};
        for (int s = 0; s < 2; s++) {
          choose(&r, hc[s], ns[s], Ls[s], sel_h);
          choose(&r, pc[s], K - ns[s], Ls[s], sel_p);
          for (int P = 0; P < K; P++) {
            int occ = P < ns[s] ? !sel_h[P] : sel_p[P - ns[s]];
            if (occ) {
              int t = 2 * P + s;
              key[t >> 6] |= 1ull << (t & 63);
              sym ^= P % g;
            }
          }
        }
        if (g > 1 && sym != 0) goto tally;
        uint64_t h = hkey(key, W) & (cap - 1);
        for (;;) {
          if (!used[h]) {
            used[h] = 1;
            memcpy(tab + h * W, key, sizeof(uint64_t) * W);
            memcpy(out + found * W, key, sizeof(uint64_t) * W);
            found++;
            window_new++;
            break;
          }
          if (memcmp(tab + h * W, key, sizeof(uint64_t) * W) == 0) break;
          h = (h + 1) & (cap - 1);
        }
      }
    tally:
      if (window == (1 << 20)) {
        if (window_new * 10 < window) { tau *= 1.25; widen = 1; }
        window = window_new = 0;
      }
    }
  }
done:
  free(tab); free(used);
  for (int s = 0; s < 2; s++) { free(hc[s]); free(pc[s]); }
  return found;
}
