/* TEST INFRASTRUCTURE ONLY -- CPU RNS-CKKS restatement (plain C11).
 *
 * This file is the written specification the CUDA engine must match bit for
 * bit.  See ckks_oracle.h for the parity status ("parity unpinned" against
 * the reference for RNS-level values: the reference has no CKKS arithmetic,
 * SURVEY.md section 0 item 1-2; pinned instead by the known-answer tests in
 * tests/test_oracle_kat.py and at the decrypted level by oracle/_ref).
 *
 * Where the reference defines semantics, this file follows it:
 *   rotation direction  out[j] = in[(j + t) mod S]     kernels.hpp:26, backend.cpp:165-182
 *   level rules         mult_plain level-1, mult_cipher min-1, add min
 *                                                    backend.hpp:10-16, backend.cpp:184-231
 *   depth exhaustion    multiplication at level 0 fails  backend.cpp:27-32
 * The CKKS realisation (RNS, hybrid key switching with dnum digits, FLEXIBLEAUTO-
 * style scale targets) follows the published algorithms the paper cites
 * (OpenFHE v1.2.4): Cheon-Kim-Kim-Song encoding via the
 * special FFT, Han-Ki hybrid key switching, Harvey/Shoup NTT conventions.
 */
#include "ckks_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

#define MAXP 80

struct ock_ctx {
  int logN, L, K, dnum, alpha, S;
  int dig[MAXP + 1]; /* key-switching digit boundaries: D_j = [dig[j], dig[j+1]) */
  int ndig;
  size_t N;
  u64 seed;
  u64 q[MAXP];
  u64 psi[MAXP];
  u64 ninv[MAXP];
  u64* tw[MAXP];  /* psi^{brv(i)}   */
  u64* itw[MAXP]; /* psi^{-brv(i)}  */
  double T[MAXP];
  u64* rotgroup;  /* 5^j mod 2N, j < S */
  double* ksi_re; /* cos(2 pi k / 2N), k <= 2N */
  double* ksi_im;
  int h;          /* secret Hamming weight (0 = uniform ternary) */
  int8_t* s;      /* secret, coefficient domain */
  u64* s_ntt;     /* [L+K][N] */
  u64* sb_ntt;    /* ephemeral sparse bootstrapping secret (sparse-secret encapsulation), or NULL */
};

/* ------------------------------------------------------------ arithmetic */
static inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static inline u64 addmod(u64 a, u64 b, u64 q) { u64 r = a + b; return r >= q ? r - q : r; }
static inline u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
static u64 powmod(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod(r, a, q);
    a = mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
static inline u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }
static inline u64 reduce_signed(int64_t v, u64 q) {
  if (v >= 0) return (u64)v % q;
  u64 r = (u64)(-(v + 1)) % q; /* -(v+1) >= 0 avoids INT64_MIN overflow */
  return q - 1 - r;
}

static int is_prime(u64 n) {
  static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; i++) {
    if (n % bases[i] == 0) return n == bases[i];
  }
  u64 d = n - 1;
  int r = 0;
  while ((d & 1) == 0) { d >>= 1; r++; }
  for (int i = 0; i < 12; i++) {
    u64 x = powmod(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int ok = 0;
    for (int j = 1; j < r; j++) {
      x = mulmod(x, x, n);
      if (x == n - 1) { ok = 1; break; }
    }
    if (!ok) return 0;
  }
  return 1;
}

static unsigned brv(unsigned x, int bits) {
  unsigned r = 0;
  for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

/* ------------------------------------------------------------------ PRNG
 * Counter-based: value = F(seed, stream, index).  Shared spec with the engine
 * (paper_2510_03996_b200/csrc/prng.hpp). */
static inline u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline u64 prng(u64 seed, u64 stream, u64 idx) {
  u64 h = mix64(seed + 0x9E3779B97F4A7C15ULL * (stream + 1));
  return mix64(h ^ (idx * 0xD1B54A32D192ED03ULL + 0x8CB92BA72F3D8DD7ULL));
}
static inline int cbd21(u64 r) {
  return __builtin_popcountll(r & 0x1FFFFFULL) - __builtin_popcountll((r >> 21) & 0x1FFFFFULL);
}
static inline u64 uniform_mod(u64 r, u64 q) { return (u64)(((u128)r * q) >> 64); }

#define STREAM_SECRET 1ULL
static inline u64 stream_key(u64 key_id, int digit, int kind) {
  return (key_id << 16) | ((u64)digit << 4) | (u64)kind; /* kind 2 = a, 3 = e */
}
static inline u64 stream_enc(u64 counter, int kind) {
  return (1ULL << 60) | (counter << 4) | (u64)kind; /* kind 4 = a, 5 = e */
}

/* ------------------------------------------------------------ parameters */
static int used(const ock_ctx* c, int n, u64 x) {
  for (int i = 0; i < n; i++) if (c->q[i] == x) return 1;
  return 0;
}

static ock_ctx* alloc_ctx(int logN, int L, int K, int dnum, u64 seed) {
  ock_ctx* c = (ock_ctx*)calloc(1, sizeof(ock_ctx));
  c->logN = logN;
  c->N = (size_t)1 << logN;
  c->S = (int)(c->N / 2);
  c->L = L;
  c->K = K;
  c->dnum = dnum;
  c->alpha = (L + dnum - 1) / dnum;
  c->ndig = 0;
  for (int j = 0; j * c->alpha < L; j++) c->dig[c->ndig++] = j * c->alpha;
  c->dig[c->ndig] = L;
  c->seed = seed;
  return c;
}

/* roots, twiddles (psi^brv by one running power per limb), encoder tables, secret */
static ock_ctx* finish_ctx(ock_ctx* c) {
  const int logN = c->logN, L = c->L, K = c->K;
  const u64 M = 2 * (u64)c->N;
  /* roots and twiddles */
#pragma omp parallel for schedule(dynamic)
  for (int i = 0; i < L + K; i++) {
    const u64 q = c->q[i];
    u64 psi = 0;
    for (u64 g = 2;; g++) {
      psi = powmod(g, (q - 1) / M, q);
      if (powmod(psi, c->N, q) == q - 1) break;
    }
    c->psi[i] = psi;
    const u64 ipsi = invmod(psi, q);
    c->tw[i] = (u64*)malloc(c->N * sizeof(u64));
    c->itw[i] = (u64*)malloc(c->N * sizeof(u64));
    u64 pw = 1, ipw = 1; /* psi^e, psi^-e for e = 0, 1, ... */
    for (size_t e = 0; e < c->N; e++) {
      const unsigned k = brv((unsigned)e, logN);
      c->tw[i][k] = pw;
      c->itw[i][k] = ipw;
      pw = mulmod(pw, psi, q);
      ipw = mulmod(ipw, ipsi, q);
    }
    c->ninv[i] = invmod((u64)(c->N % q), q);
  }
  /* encoder tables */
  c->rotgroup = (u64*)malloc(c->S * sizeof(u64));
  {
    u64 g = 1;
    for (int j = 0; j < c->S; j++) { c->rotgroup[j] = g; g = (g * 5) % M; }
  }
  c->ksi_re = (double*)malloc((M + 1) * sizeof(double));
  c->ksi_im = (double*)malloc((M + 1) * sizeof(double));
  for (u64 k = 0; k <= M; k++) {
    const double ang = 2.0 * 3.14159265358979323846 * (double)k / (double)M;
    c->ksi_re[k] = cos(ang);
    c->ksi_im[k] = sin(ang);
  }
  /* secret */
  c->s = (int8_t*)malloc(c->N);
  ock_secret(c, c->s);
  c->s_ntt = (u64*)malloc((size_t)(L + K) * c->N * sizeof(u64));
#pragma omp parallel for
  for (int i = 0; i < L + K; i++) {
    u64* d = c->s_ntt + (size_t)i * c->N;
    for (size_t k = 0; k < c->N; k++) d[k] = reduce_signed(c->s[k], c->q[i]);
    ock_ntt_fwd(c, i, d);
  }
  return c;
}


ock_ctx* ock_create(int logN, int L, int K, int dnum, int first_bits,
                    int scale_bits, int special_bits, u64 seed) {
  if (logN < 3 || logN > 17 || L < 1 || K < 1 || L + K > MAXP || dnum < 1 ||
      first_bits > 61 || scale_bits > 61 || special_bits > 61)
    return NULL;
  ock_ctx* c = alloc_ctx(logN, L, K, dnum, seed);
  const u64 M = 2 * (u64)c->N;
  int np = 0;
  /* q_0: largest prime = 1 mod 2N below 2^first_bits */
  {
    u64 x = (((1ULL << first_bits) - 1) / M) * M + 1;
    if (x >= (1ULL << first_bits)) x -= M;
    while (!is_prime(x)) x -= M;
    c->q[np++] = x;
  }
  /* scaling primes, top-down, each the unused prime = 1 mod 2N closest to
   * T_lv^2 / 2^scale_bits; T_{lv-1} = T_lv^2 / q_lv (FLEXIBLEAUTO targets) */
  {
    double T = ldexp(1.0, scale_bits);
    c->T[L - 1] = T;
    u64 chosen[MAXP];
    for (int lv = L - 1; lv >= 1; lv--) {
      const double target = (T * T) / ldexp(1.0, scale_bits);
      const u64 tgt = (u64)target;
      const u64 base = ((tgt - 1) / M) * M + 1;
      u64 pick = 0;
      for (u64 k = 0; !pick; k++) {
        const u64 down = base - k * M, up = base + (k + 1) * M;
        const u64 first = (tgt - down <= up - tgt) ? down : up;
        const u64 second = (first == down) ? up : down;
        const u64 cand[2] = {first, second};
        for (int ci = 0; ci < 2 && !pick; ci++) {
          const u64 x = cand[ci];
          int ok = is_prime(x) && !used(c, np, x);
          for (int i = L - 1; ok && i > lv; i--) if (chosen[i] == x) ok = 0;
          if (ok) pick = x;
        }
      }
      chosen[lv] = pick;
      T = (T * T) / (double)pick;
      c->T[lv - 1] = T;
    }
    for (int lv = 1; lv < L; lv++) c->q[np++] = chosen[lv];
  }
  /* special primes: largest primes = 1 mod 2N below 2^special_bits */
  {
    u64 x = (((1ULL << special_bits) - 1) / M) * M + 1;
    if (x >= (1ULL << special_bits)) x -= M;
    for (int k = 0; k < K; k++) {
      while (!is_prime(x) || used(c, np, x)) x -= M;
      c->q[np++] = x;
      x -= M;
    }
  }
  return finish_ctx(c);
}

/* Context over an explicit chain (the engine's own primes and per-level scale
 * targets, e.g. the model runtime's bootstrapping chains with mixed 55/40-bit
 * levels): q_0..q_{L-1}, p_0..p_{K-1} in primes[L+K], T[L]; every prime must be
 * = 1 mod 2N.  Everything after prime selection is shared with ock_create. */
ock_ctx* ock_create_chain(int logN, int L, int K, int dnum, const u64* primes,
                          const double* T, u64 seed) {
  if (logN < 3 || logN > 17 || L < 1 || K < 1 || L + K > MAXP || dnum < 1) return NULL;
  const u64 M = (u64)2 << logN;
  for (int i = 0; i < L + K; i++)
    if (primes[i] % M != 1 || !is_prime(primes[i]) || primes[i] >> 61) return NULL;
  ock_ctx* c = alloc_ctx(logN, L, K, dnum, seed);
  for (int i = 0; i < L + K; i++) c->q[i] = primes[i];
  for (int i = 0; i < L; i++) c->T[i] = T[i];
  return finish_ctx(c);
}

void ock_destroy(ock_ctx* c) {
  if (!c) return;
  for (int i = 0; i < c->L + c->K; i++) { free(c->tw[i]); free(c->itw[i]); }
  free(c->rotgroup); free(c->ksi_re); free(c->ksi_im); free(c->s); free(c->s_ntt); free(c->sb_ntt);
  free(c);
}

void ock_info(const ock_ctx* c, u64* primes, u64* psi, double* T) {
  for (int i = 0; i < c->L + c->K; i++) {
    if (primes) primes[i] = c->q[i];
    if (psi) psi[i] = c->psi[i];
  }
  if (T) for (int i = 0; i < c->L; i++) T[i] = c->T[i];
}

/* ------------------------------------------------------------------- NTT
 * Forward: Cooley-Tukey, natural order in, bit-reversed order out; output
 * index i holds a(psi^{2 brv(i) + 1}).  Inverse: Gentleman-Sande, bit-reversed
 * in, natural out, scaled by N^{-1}. */
void ock_ntt_fwd(const ock_ctx* c, int pi, u64* a) {
  const u64 q = c->q[pi];
  const u64* tw = c->tw[pi];
  const size_t N = c->N;
  size_t t = N;
  for (size_t m = 1; m < N; m <<= 1) {
    t >>= 1;
    for (size_t i = 0; i < m; i++) {
      const size_t j1 = 2 * i * t;
      const u64 S = tw[m + i];
      for (size_t j = j1; j < j1 + t; j++) {
        const u64 U = a[j], V = mulmod(a[j + t], S, q);
        a[j] = addmod(U, V, q);
        a[j + t] = submod(U, V, q);
      }
    }
  }
}

void ock_ntt_inv(const ock_ctx* c, int pi, u64* a) {
  const u64 q = c->q[pi];
  const u64* itw = c->itw[pi];
  const size_t N = c->N;
  size_t t = 1;
  for (size_t m = N >> 1; m >= 1; m >>= 1) {
    for (size_t i = 0; i < m; i++) {
      const size_t j1 = 2 * i * t;
      const u64 S = itw[m + i];
      for (size_t j = j1; j < j1 + t; j++) {
        const u64 U = a[j], V = a[j + t];
        a[j] = addmod(U, V, q);
        a[j + t] = mulmod(submod(U, V, q), S, q);
      }
    }
    t <<= 1;
  }
  for (size_t j = 0; j < N; j++) a[j] = mulmod(a[j], c->ninv[pi], q);
}

void ock_ntt_naive(const ock_ctx* c, int pi, const u64* a, u64* out) {
  const u64 q = c->q[pi];
  for (size_t i = 0; i < c->N; i++) {
    const u64 e = 2 * (u64)brv((unsigned)i, c->logN) + 1;
    const u64 x = powmod(c->psi[pi], e, q);
    u64 acc = 0, xp = 1;
    for (size_t k = 0; k < c->N; k++) {
      acc = addmod(acc, mulmod(a[k], xp, q), q);
      xp = mulmod(xp, x, q);
    }
    out[i] = acc;
  }
}

void ock_negacyclic_mul_naive(const ock_ctx* c, int pi, const u64* a,
                              const u64* b, u64* out) {
  const u64 q = c->q[pi];
  const size_t N = c->N;
  memset(out, 0, N * sizeof(u64));
  for (size_t i = 0; i < N; i++)
    for (size_t j = 0; j < N; j++) {
      const u64 p = mulmod(a[i], b[j], q);
      const size_t k = i + j;
      if (k < N) out[k] = addmod(out[k], p, q);
      else out[k - N] = submod(out[k - N], p, q);
    }
}

static inline int limb_prime(const int* map, int i) { return map ? map[i] : i; }

void ock_ntt_fwd_limbs(const ock_ctx* c, u64* a, int nlimbs, const int* limb_map) {
#pragma omp parallel for
  for (int i = 0; i < nlimbs; i++) ock_ntt_fwd(c, limb_prime(limb_map, i), a + (size_t)i * c->N);
}
void ock_ntt_inv_limbs(const ock_ctx* c, u64* a, int nlimbs, const int* limb_map) {
#pragma omp parallel for
  for (int i = 0; i < nlimbs; i++) ock_ntt_inv(c, limb_prime(limb_map, i), a + (size_t)i * c->N);
}

/* ----------------------------------------------------------- automorphism */
uint64_t ock_galois_elt(const ock_ctx* c, long t) {
  const long S = c->S;
  long r = t % S;
  if (r < 0) r += S;
  return powmod(5, (u64)r, 2 * (u64)c->N);
}

/* NTT domain: out[i] = in[j], evaluation exponent e_j = e_i * g mod 2N */
static inline size_t auto_index(const ock_ctx* c, size_t i, u64 g) {
  const u64 M = 2 * (u64)c->N;
  const u64 e = 2 * (u64)brv((unsigned)i, c->logN) + 1;
  const u64 eg = (e * g) % M;
  return brv((unsigned)((eg - 1) / 2), c->logN);
}

void ock_automorph_ntt(const ock_ctx* c, u64 g, const u64* in, u64* out, int nlimbs) {
  const size_t N = c->N;
  size_t* idx = (size_t*)malloc(N * sizeof(size_t));
  for (size_t i = 0; i < N; i++) idx[i] = auto_index(c, i, g);
#pragma omp parallel for
  for (int l = 0; l < nlimbs; l++)
    for (size_t i = 0; i < N; i++) out[(size_t)l * N + i] = in[(size_t)l * N + idx[i]];
  free(idx);
}

/* coefficient domain: X^k -> X^{kg mod 2N}, negated when kg mod 2N >= N */
void ock_automorph_coeff(const ock_ctx* c, u64 g, const u64* in, u64* out,
                         int nlimbs, const int* limb_map) {
  const size_t N = c->N;
  const u64 M = 2 * (u64)N;
  for (int l = 0; l < nlimbs; l++) {
    const u64 q = c->q[limb_prime(limb_map, l)];
    for (size_t k = 0; k < N; k++) {
      const u64 kg = ((u64)k * g) % M;
      const u64 v = in[(size_t)l * N + k];
      if (kg < N) out[(size_t)l * N + kg] = v;
      else out[(size_t)l * N + (kg - N)] = v ? q - v : 0;
    }
  }
}

/* ---------------------------------------------------------------- encoder
 * Canonical embedding with full packing: slot j <-> root zeta^{5^j},
 * zeta = exp(2 pi i / 2N).  Special FFT in the Cheon et al. formulation. */
static void bitrev_complex(double* re, double* im, int n) {
  for (int i = 1, j = 0; i < n; i++) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double t = re[i]; re[i] = re[j]; re[j] = t;
      t = im[i]; im[i] = im[j]; im[j] = t;
    }
  }
}

static void fft_special_inv(const ock_ctx* c, double* re, double* im) {
  const int S = c->S;
  const u64 M = 2 * (u64)c->N;
  for (int len = S; len >= 1; len >>= 1) {
    const int lenh = len >> 1;
    const u64 lenq = (u64)len << 2;
    for (int i = 0; i < S; i += len) {
      for (int j = 0; j < lenh; j++) {
        const u64 idx = (lenq - (c->rotgroup[j] % lenq)) * (M / lenq);
        const double ur = re[i + j] + re[i + j + lenh];
        const double ui = im[i + j] + im[i + j + lenh];
        const double vr0 = re[i + j] - re[i + j + lenh];
        const double vi0 = im[i + j] - im[i + j + lenh];
        const double wr = c->ksi_re[idx], wi = c->ksi_im[idx];
        re[i + j] = ur;
        im[i + j] = ui;
        re[i + j + lenh] = vr0 * wr - vi0 * wi;
        im[i + j + lenh] = vr0 * wi + vi0 * wr;
      }
    }
  }
  bitrev_complex(re, im, S);
  for (int i = 0; i < S; i++) { re[i] /= (double)S; im[i] /= (double)S; }
}

static void fft_special(const ock_ctx* c, double* re, double* im) {
  const int S = c->S;
  const u64 M = 2 * (u64)c->N;
  bitrev_complex(re, im, S);
  for (int len = 2; len <= S; len <<= 1) {
    const int lenh = len >> 1;
    const u64 lenq = (u64)len << 2;
    for (int i = 0; i < S; i += len) {
      for (int j = 0; j < lenh; j++) {
        const u64 idx = (c->rotgroup[j] % lenq) * (M / lenq);
        const double wr = c->ksi_re[idx], wi = c->ksi_im[idx];
        const double ur = re[i + j], ui = im[i + j];
        const double xr = re[i + j + lenh], xi = im[i + j + lenh];
        const double vr = xr * wr - xi * wi;
        const double vi = xr * wi + xi * wr;
        re[i + j] = ur + vr;
        im[i + j] = ui + vi;
        re[i + j + lenh] = ur - vr;
        im[i + j + lenh] = ui - vi;
      }
    }
  }
}

int ock_encode_coeffs(const ock_ctx* c, const double* vals, size_t n,
                      double scale, int64_t* coeffs) {
  const int S = c->S;
  if (n > (size_t)S) return -1;
  double* re = (double*)calloc(S, sizeof(double));
  double* im = (double*)calloc(S, sizeof(double));
  for (size_t i = 0; i < n; i++) re[i] = vals[i];
  fft_special_inv(c, re, im);
  int rc = 0;
  const double lim = 4611686018427387904.0; /* 2^62 */
  for (int i = 0; i < S; i++) {
    const double a = re[i] * scale, b = im[i] * scale;
    if (!(fabs(a) < lim) || !(fabs(b) < lim)) { rc = -2; break; }
    coeffs[i] = llround(a);
    coeffs[i + S] = llround(b);
  }
  free(re);
  free(im);
  return rc;
}

static int is_constant(const double* vals, size_t n, int S, double* cval) {
  if (n == 0) { *cval = 0.0; return 1; }
  const double v = vals[0];
  for (size_t i = 1; i < n; i++) if (vals[i] != v) return 0;
  if (n < (size_t)S && v != 0.0) return 0;
  *cval = v;
  return 1;
}

int ock_encode(const ock_ctx* c, const double* vals, size_t n, int limbs,
               double scale, u64* out) {
  const size_t N = c->N;
  double cv;
  if (is_constant(vals, n, c->S, &cv)) {
    const double x = cv * scale;
    if (!(fabs(x) < 4611686018427387904.0)) return -2;
    const int64_t k = llround(x);
    for (int l = 0; l < limbs; l++) {
      const u64 r = reduce_signed(k, c->q[l]);
      for (size_t i = 0; i < N; i++) out[(size_t)l * N + i] = r;
    }
    return 0;
  }
  int64_t* m = (int64_t*)malloc(N * sizeof(int64_t));
  const int rc = ock_encode_coeffs(c, vals, n, scale, m);
  if (rc) { free(m); return rc; }
#pragma omp parallel for
  for (int l = 0; l < limbs; l++) {
    u64* d = out + (size_t)l * N;
    for (size_t i = 0; i < N; i++) d[i] = reduce_signed(m[i], c->q[l]);
    ock_ntt_fwd(c, l, d);
  }
  free(m);
  return 0;
}

void ock_decode_coeffs(const ock_ctx* c, const double* coeffs, double scale, double* out) {
  const int S = c->S;
  double* re = (double*)malloc(S * sizeof(double));
  double* im = (double*)malloc(S * sizeof(double));
  for (int i = 0; i < S; i++) { re[i] = coeffs[i] / scale; im[i] = coeffs[i + S] / scale; }
  fft_special(c, re, im);
  for (int i = 0; i < S; i++) out[i] = re[i];
  free(re);
  free(im);
}

/* ------------------------------------------------------- keys / encryption */
/* secret: uniform ternary (h = 0) or exactly h nonzero +-1 coefficients
 * (sparse, for bootstrapping): candidate j picks position prng(seed, 6, j) % N,
 * accepted when unused, sign from bit 0 of prng(seed, 7, j). */
static void sparse_secret(const ock_ctx* c, int8_t* s, int h, u64 pos_stream) {
  memset(s, 0, c->N);
  int got = 0;
  for (u64 j = 0; got < h; j++) {
    const size_t pos = (size_t)(prng(c->seed, pos_stream, j) % c->N);
    if (s[pos]) continue;
    s[pos] = (prng(c->seed, pos_stream + 1, j) & 1) ? 1 : -1;
    got++;
  }
}

void ock_secret(const ock_ctx* c, int8_t* s) {
  if (c->h <= 0) {
    for (size_t k = 0; k < c->N; k++) s[k] = (int8_t)((int)(prng(c->seed, STREAM_SECRET, k) % 3) - 1);
    return;
  }
  sparse_secret(c, s, c->h, 6);
}

/* Sparse-secret encapsulation (engine Context::sse, evaluator.cpp mod_raise): the
 * ephemeral sparse bootstrapping secret s_b with h_b nonzero coefficients from
 * streams 8 (positions) / 9 (signs) -- the main secret's recipe on other streams. */
void ock_set_boot_secret(ock_ctx* c, int hb) {
  int8_t* sb = (int8_t*)malloc(c->N);
  sparse_secret(c, sb, hb, 8);
  if (!c->sb_ntt) c->sb_ntt = (u64*)malloc((size_t)(c->L + c->K) * c->N * sizeof(u64));
#pragma omp parallel for
  for (int i = 0; i < c->L + c->K; i++) {
    u64* d = c->sb_ntt + (size_t)i * c->N;
    for (size_t k = 0; k < c->N; k++) d[k] = reduce_signed(sb[k], c->q[i]);
    ock_ntt_fwd(c, i, d);
  }
  free(sb);
}

void ock_set_hamming_weight(ock_ctx* c, int h) {
  c->h = h;
  ock_secret(c, c->s);
#pragma omp parallel for
  for (int i = 0; i < c->L + c->K; i++) {
    u64* d = c->s_ntt + (size_t)i * c->N;
    for (size_t k = 0; k < c->N; k++) d[k] = reduce_signed(c->s[k], c->q[i]);
    ock_ntt_fwd(c, i, d);
  }
}

/* error polynomial (CBD, eta = 21) reduced into prime pi and NTT'd */
static void error_ntt(const ock_ctx* c, u64 stream, int pi, u64* d) {
  for (size_t k = 0; k < c->N; k++) d[k] = reduce_signed(cbd21(prng(c->seed, stream, k)), c->q[pi]);
  ock_ntt_fwd(c, pi, d);
}

int ock_keygen(const ock_ctx* c, u64 key_id, u64* key) {
  const int L = c->L, K = c->K, LK = L + K;
  const size_t N = c->N;
  /* s' : s^2 (relinearisation, key_id 0), sigma_g(s) (rotation, key_id g odd), or the
   * sparse-secret encapsulation keys: 2 = s -> s_b (b = -a s_b + e + P s, on digit 0's
   * q_0 and the special primes only: every other limb and digit is zero), 4 = s_b -> s */
  u64* sp = (u64*)malloc((size_t)LK * N * sizeof(u64));
  const u64* s_to = c->s_ntt;
  const int to_sparse = key_id == 2, sse = key_id == 2 || key_id == 4;
  if (sse && !c->sb_ntt) { free(sp); return -1; }
  if (sse) {
    memcpy(sp, to_sparse ? c->s_ntt : c->sb_ntt, (size_t)LK * N * sizeof(u64));
    if (to_sparse) s_to = c->sb_ntt;
    memset(key, 0, (size_t)c->dnum * 2 * LK * N * sizeof(u64));
  } else if (key_id == 0) {
    for (int i = 0; i < LK; i++)
      for (size_t k = 0; k < N; k++) {
        const u64 v = c->s_ntt[(size_t)i * N + k];
        sp[(size_t)i * N + k] = mulmod(v, v, c->q[i]);
      }
  } else {
    if ((key_id & 1) == 0) { free(sp); return -1; }
    ock_automorph_ntt(c, key_id, c->s_ntt, sp, LK);
  }
  for (int j = 0; j < (to_sparse ? 1 : c->dnum); j++) { /* digits past ndig stay empty */
    const int lo = j < c->ndig ? c->dig[j] : L, hi = j < c->ndig ? c->dig[j + 1] : L;
    u64* b = key + ((size_t)j * 2 + 0) * LK * N;
    u64* a = key + ((size_t)j * 2 + 1) * LK * N;
#pragma omp parallel for
    for (int i = 0; i < LK; i++) {
      if (to_sparse && i >= 1 && i < L) continue;
      const u64 q = c->q[i];
      u64 Pmod = 1;
      for (int k = 0; k < K; k++) Pmod = mulmod(Pmod, c->q[L + k] % q, q);
      u64* bi = b + (size_t)i * N;
      u64* ai = a + (size_t)i * N;
      error_ntt(c, stream_key(key_id, j, 3), i, bi);
      for (size_t k = 0; k < N; k++) {
        ai[k] = uniform_mod(prng(c->seed, stream_key(key_id, j, 2), (u64)i * N + k), q);
        u64 v = submod(bi[k], mulmod(ai[k], s_to[(size_t)i * N + k], q), q);
        if (i >= lo && i < hi) v = addmod(v, mulmod(Pmod, sp[(size_t)i * N + k], q), q);
        bi[k] = v;
      }
    }
  }
  free(sp);
  return 0;
}

int ock_encrypt(const ock_ctx* c, const double* vals, size_t n, u64 counter, u64* ct) {
  const int L = c->L;
  const size_t N = c->N;
  u64* c0 = ct;
  u64* c1 = ct + (size_t)L * N;
  const int rc = ock_encode(c, vals, n, L, c->T[L - 1], c0);
  if (rc) return rc;
#pragma omp parallel for
  for (int i = 0; i < L; i++) {
    const u64 q = c->q[i];
    u64* e = (u64*)malloc(N * sizeof(u64));
    error_ntt(c, stream_enc(counter, 5), i, e);
    for (size_t k = 0; k < N; k++) {
      const u64 a = uniform_mod(prng(c->seed, stream_enc(counter, 4), (u64)i * N + k), q);
      c1[(size_t)i * N + k] = a;
      u64 v = submod(e[k], mulmod(a, c->s_ntt[(size_t)i * N + k], q), q);
      c0[(size_t)i * N + k] = addmod(c0[(size_t)i * N + k], v, q);
    }
    free(e);
  }
  return 0;
}

int ock_decrypt(const ock_ctx* c, const u64* ct, int limbs, double scale, double* out) {
  const size_t N = c->N;
  const int use = limbs >= 2 ? 2 : 1;
  u64* m = (u64*)malloc((size_t)use * N * sizeof(u64));
  for (int i = 0; i < use; i++) {
    const u64 q = c->q[i];
    for (size_t k = 0; k < N; k++)
      m[(size_t)i * N + k] = addmod(ct[(size_t)i * N + k],
                                    mulmod(ct[((size_t)limbs + i) * N + k], c->s_ntt[(size_t)i * N + k], q), q);
    ock_ntt_inv(c, i, m + (size_t)i * N);
  }
  double* coeffs = (double*)malloc(N * sizeof(double));
  if (use == 1) {
    const u64 q = c->q[0];
    for (size_t k = 0; k < N; k++) {
      const u64 v = m[k];
      coeffs[k] = (v > q / 2) ? -(double)(q - v) : (double)v;
    }
  } else {
    const u64 q0 = c->q[0], q1 = c->q[1];
    const u64 q0inv = invmod(q0 % q1, q1);
    const u128 Q = (u128)q0 * q1;
    for (size_t k = 0; k < N; k++) {
      const u64 x0 = m[k], x1 = m[N + k];
      const u64 t = mulmod(submod(x1, x0 % q1, q1), q0inv, q1);
      const u128 X = (u128)x0 + (u128)q0 * t;
      coeffs[k] = (X > Q / 2) ? -(double)(Q - X) : (double)X;
    }
  }
  ock_decode_coeffs(c, coeffs, scale, out);
  free(coeffs);
  free(m);
  return 0;
}

/* --------------------------------------------------------- key switching */
/* digits with an active limb at `limbs` limbs */
static int digit_count(const ock_ctx* c, int limbs) {
  int k = 0;
  while (k < c->ndig && c->dig[k] < limbs) k++;
  return k;
}

/* Contiguous digits balanced by bit size (engine params.cpp balanced_digits):
 * bisection on the widest digit's bit sum, greedy packing under it, <= 15 limbs
 * per digit, at most dnum digits. */
static int split_digits(const double* bits, int L, int dnum, double cap, int* d) {
  int n = 0, size = 0;
  double acc = 0.0;
  d[n++] = 0;
  for (int i = 0; i < L; i++) {
    if (bits[i] > cap) return -1;
    if (size == 15 || acc + bits[i] > cap) {
      d[n++] = i;
      acc = 0.0;
      size = 0;
    }
    acc += bits[i];
    size++;
  }
  d[n] = L;
  return n > dnum ? -1 : n;
}

int ock_set_digit_split(ock_ctx* c, int balanced) {
  if (!balanced) {
    c->ndig = 0;
    for (int j = 0; j * c->alpha < c->L; j++) c->dig[c->ndig++] = j * c->alpha;
    c->dig[c->ndig] = c->L;
    return 0;
  }
  double bits[MAXP];
  double lo = 0.0, hi = 0.0;
  for (int i = 0; i < c->L; i++) {
    bits[i] = log2((double)c->q[i]);
    hi += bits[i];
  }
  int best[MAXP + 1], tmp[MAXP + 1];
  int nb = split_digits(bits, c->L, c->dnum, hi + 1.0, best);
  if (nb < 0) return -1;
  for (int it = 0; it < 60; it++) {
    const double mid = 0.5 * (lo + hi);
    const int n = split_digits(bits, c->L, c->dnum, mid, tmp);
    if (n >= 0) {
      hi = mid;
      nb = n;
      memcpy(best, tmp, sizeof(int) * (size_t)(n + 1));
    } else {
      lo = mid;
    }
  }
  c->ndig = nb;
  memcpy(c->dig, best, sizeof(int) * (size_t)(nb + 1));
  return 0;
}

static inline int ext_prime(const ock_ctx* c, int limbs, int t) {
  return t < limbs ? t : c->L + (t - limbs);
}

/* out: [beta][limbs+K][N] in NTT domain */
int ock_modup(const ock_ctx* c, const u64* d, int limbs, u64* out) {
  const int K = c->K, E = limbs + K;
  const size_t N = c->N;
  const int beta = digit_count(c, limbs);
  u64* x = (u64*)malloc((size_t)limbs * N * sizeof(u64));
  memcpy(x, d, (size_t)limbs * N * sizeof(u64));
  ock_ntt_inv_limbs(c, x, limbs, NULL);
  for (int j = 0; j < beta; j++) {
    const int lo = c->dig[j], hi = c->dig[j + 1] < limbs ? c->dig[j + 1] : limbs;
    const int a = hi - lo;
    u64* y = (u64*)malloc((size_t)a * N * sizeof(u64));
    for (int i = lo; i < hi; i++) {
      const u64 qi = c->q[i];
      u64 hat = 1;
      for (int i2 = lo; i2 < hi; i2++) if (i2 != i) hat = mulmod(hat, c->q[i2] % qi, qi);
      const u64 hinv = invmod(hat, qi);
      for (size_t k = 0; k < N; k++) y[(size_t)(i - lo) * N + k] = mulmod(x[(size_t)i * N + k], hinv, qi);
    }
    u64* o = out + (size_t)j * E * N;
#pragma omp parallel for
    for (int t = 0; t < E; t++) {
      if (t >= lo && t < hi) {
        memcpy(o + (size_t)t * N, d + (size_t)t * N, N * sizeof(u64));
        continue;
      }
      const int pt = ext_prime(c, limbs, t);
      const u64 m = c->q[pt];
      u64 hm[MAXP];
      for (int i = lo; i < hi; i++) {
        u64 h = 1;
        for (int i2 = lo; i2 < hi; i2++) if (i2 != i) h = mulmod(h, c->q[i2] % m, m);
        hm[i - lo] = h;
      }
      u64* ot = o + (size_t)t * N;
      for (size_t k = 0; k < N; k++) {
        u128 acc = 0;
        for (int i = 0; i < a; i++) acc += (u128)y[(size_t)i * N + k] * hm[i];
        ot[k] = (u64)(acc % m);
      }
      ock_ntt_fwd(c, pt, ot);
    }
    free(y);
  }
  free(x);
  return 0;
}

/* (P - 1) / 2 mod m, P = prod of the special primes */
static u64 half_P_mod(const ock_ctx* c, u64 m) {
  /* (P-1)/2 = (P mod 2m - 1)/2 computed exactly: P odd, so use P*inv2 - inv2 */
  u64 Pm = 1;
  for (int k = 0; k < c->K; k++) Pm = mulmod(Pm, c->q[c->L + k] % m, m);
  const u64 inv2 = (m + 1) / 2;
  return mulmod(submod(Pm, 1 % m, m), inv2, m);
}

/* acc: [limbs+K][N] NTT domain -> out [limbs][N] NTT domain.
 * out = round(acc / P): the P-part is replaced by its centred residue
 * [acc + h]_P - h, h = (P-1)/2, whose exact value is recovered from the
 * fast basis conversion with the FP64 overflow estimate
 * u = floor(sum_k y_k / p_k) (each term fl(y_k * fl(1/p_k)), summed in k order,
 * no FMA contraction). */
int ock_moddown(const ock_ctx* c, const u64* acc, int limbs, u64* out) {
  const int L = c->L, K = c->K;
  const size_t N = c->N;
  u64* z = (u64*)malloc((size_t)K * N * sizeof(u64));
  uint32_t* u = (uint32_t*)malloc(N * sizeof(uint32_t));
  memcpy(z, acc + (size_t)limbs * N, (size_t)K * N * sizeof(u64));
  for (int k = 0; k < K; k++) {
    const u64 pk = c->q[L + k];
    ock_ntt_inv(c, L + k, z + (size_t)k * N);
    u64 hat = 1;
    for (int k2 = 0; k2 < K; k2++) if (k2 != k) hat = mulmod(hat, c->q[L + k2] % pk, pk);
    const u64 hinv = invmod(hat, pk);
    const u64 hk = half_P_mod(c, pk);
    for (size_t n = 0; n < N; n++)
      z[(size_t)k * N + n] = mulmod(addmod(z[(size_t)k * N + n], hk, pk), hinv, pk);
  }
  for (size_t n = 0; n < N; n++) {
    double v = 0.0;
    for (int k = 0; k < K; k++) {
      const double pinv = 1.0 / (double)c->q[L + k];
      const double term = (double)z[(size_t)k * N + n] * pinv;
      v = v + term;
    }
    u[n] = (uint32_t)v;
  }
#pragma omp parallel for
  for (int i = 0; i < limbs; i++) {
    const u64 qi = c->q[i];
    u64 hm[MAXP];
    u64 Pmod = 1;
    for (int k = 0; k < K; k++) {
      u64 h = 1;
      for (int k2 = 0; k2 < K; k2++) if (k2 != k) h = mulmod(h, c->q[L + k2] % qi, qi);
      hm[k] = h;
      Pmod = mulmod(Pmod, c->q[L + k] % qi, qi);
    }
    const u64 Pinv = invmod(Pmod, qi);
    const u64 hq = half_P_mod(c, qi);
    u64* conv = (u64*)malloc(N * sizeof(u64));
    for (size_t n = 0; n < N; n++) {
      u128 s = 0;
      for (int k = 0; k < K; k++) s += (u128)z[(size_t)k * N + n] * hm[k];
      u64 x = (u64)(s % qi);
      x = submod(x, mulmod((u64)u[n], Pmod, qi), qi);
      conv[n] = submod(x, hq, qi);
    }
    ock_ntt_fwd(c, i, conv);
    for (size_t n = 0; n < N; n++)
      out[(size_t)i * N + n] = mulmod(submod(acc[(size_t)i * N + n], conv[n], qi), Pinv, qi);
    free(conv);
  }
  free(z);
  free(u);
  return 0;
}

/* ModDown by P' = P q_l, l = limbs - 1 (the fused relinearisation + rescale):
 * z: [limbs+K][N] NTT domain over Q_limbs u P -> out [l][N] = round(z / P').
 * Special limbs in this order: s = 0 is q_l, s = 1..K is p_{s-1}; the centred
 * residue [z + h']_{P'} - h' (h' = (P'-1)/2) comes from the fast basis
 * conversion with the FP64 overflow estimate summed in s order. */
int ock_moddown_fused(const ock_ctx* c, const u64* z, int limbs, u64* out) {
  const int L = c->L, K = c->K, l = limbs - 1, S = K + 1;
  const size_t N = c->N;
  if (l < 1) return -1;
  int sp[MAXP];
  sp[0] = l;
  for (int k = 0; k < K; k++) sp[1 + k] = L + k;
  u64* y = (u64*)malloc((size_t)S * N * sizeof(u64));
  uint32_t* u = (uint32_t*)malloc(N * sizeof(uint32_t));
  for (int s = 0; s < S; s++) {
    const u64 m = c->q[sp[s]];
    const size_t src = (s == 0) ? (size_t)l : (size_t)limbs + (size_t)(s - 1);
    memcpy(y + (size_t)s * N, z + src * N, N * sizeof(u64));
    ock_ntt_inv(c, sp[s], y + (size_t)s * N);
    u64 hat = 1, Pp = 1;
    for (int s2 = 0; s2 < S; s2++) {
      Pp = mulmod(Pp, c->q[sp[s2]] % m, m);
      if (s2 != s) hat = mulmod(hat, c->q[sp[s2]] % m, m);
    }
    const u64 hinv = invmod(hat, m);
    const u64 hh = mulmod(submod(Pp, 1 % m, m), (m + 1) / 2, m);
    for (size_t n = 0; n < N; n++)
      y[(size_t)s * N + n] = mulmod(addmod(y[(size_t)s * N + n], hh, m), hinv, m);
  }
  for (size_t n = 0; n < N; n++) {
    double v = 0.0;
    for (int s = 0; s < S; s++) {
      const double pinv = 1.0 / (double)c->q[sp[s]];
      const double term = (double)y[(size_t)s * N + n] * pinv;
      v = v + term;
    }
    u[n] = (uint32_t)v;
  }
#pragma omp parallel for
  for (int i = 0; i < l; i++) {
    const u64 qi = c->q[i];
    u64 hm[MAXP];
    u64 Pp = 1;
    for (int s = 0; s < S; s++) {
      u64 h = 1;
      for (int s2 = 0; s2 < S; s2++) if (s2 != s) h = mulmod(h, c->q[sp[s2]] % qi, qi);
      hm[s] = h;
      Pp = mulmod(Pp, c->q[sp[s]] % qi, qi);
    }
    const u64 Ppinv = invmod(Pp, qi);
    const u64 hq = mulmod(submod(Pp, 1 % qi, qi), (qi + 1) / 2, qi);
    u64* conv = (u64*)malloc(N * sizeof(u64));
    for (size_t n = 0; n < N; n++) {
      u128 acc = 0;
      for (int s = 0; s < S; s++) acc += (u128)y[(size_t)s * N + n] * hm[s];
      u64 x = (u64)(acc % qi);
      x = submod(x, mulmod((u64)u[n], Pp, qi), qi);
      conv[n] = submod(x, hq, qi);
    }
    ock_ntt_fwd(c, i, conv);
    for (size_t n = 0; n < N; n++)
      out[(size_t)i * N + n] = mulmod(submod(z[(size_t)i * N + n], conv[n], qi), Ppinv, qi);
    free(conv);
  }
  free(y);
  free(u);
  return 0;
}

/* key inner product of a key switch before its ModDown: acc_p over Q_limbs u P */
static void ks_acc(const ock_ctx* c, const u64* d, int limbs, const u64* key, u64 g, u64* acc0, u64* acc1) {
  const int K = c->K, E = limbs + K, LK = c->L + K;
  const size_t N = c->N;
  const int beta = digit_count(c, limbs);
  u64* up = (u64*)malloc((size_t)beta * E * N * sizeof(u64));
  ock_modup(c, d, limbs, up);
  size_t* idx = (size_t*)malloc(N * sizeof(size_t));
  for (size_t n = 0; n < N; n++) idx[n] = (g == 1) ? n : auto_index(c, n, g);
#pragma omp parallel for
  for (int t = 0; t < E; t++) {
    const int pt = ext_prime(c, limbs, t);
    const u64 m = c->q[pt];
    for (size_t n = 0; n < N; n++) {
      u128 s0 = 0, s1 = 0;
      for (int j = 0; j < beta; j++) {
        const u64 dv = up[((size_t)j * E + t) * N + idx[n]];
        s0 += (u128)dv * key[(((size_t)j * 2 + 0) * LK + pt) * N + n];
        s1 += (u128)dv * key[(((size_t)j * 2 + 1) * LK + pt) * N + n];
      }
      acc0[(size_t)t * N + n] = (u64)(s0 % m);
      acc1[(size_t)t * N + n] = (u64)(s1 % m);
    }
  }
  free(up);
  free(idx);
}

int ock_keyswitch(const ock_ctx* c, const u64* d, int limbs, const u64* key,
                  u64 g, u64* ks0, u64* ks1) {
  const int L = c->L, K = c->K, E = limbs + K, LK = L + K;
  const size_t N = c->N;
  const int beta = digit_count(c, limbs);
  u64* up = (u64*)malloc((size_t)beta * E * N * sizeof(u64));
  ock_modup(c, d, limbs, up);
  size_t* idx = (size_t*)malloc(N * sizeof(size_t));
  for (size_t n = 0; n < N; n++) idx[n] = (g == 1) ? n : auto_index(c, n, g);
  u64* acc0 = (u64*)malloc((size_t)E * N * sizeof(u64));
  u64* acc1 = (u64*)malloc((size_t)E * N * sizeof(u64));
#pragma omp parallel for
  for (int t = 0; t < E; t++) {
    const int pt = ext_prime(c, limbs, t);
    const u64 m = c->q[pt];
    for (size_t n = 0; n < N; n++) {
      u128 s0 = 0, s1 = 0;
      for (int j = 0; j < beta; j++) {
        const u64 dv = up[((size_t)j * E + t) * N + idx[n]];
        s0 += (u128)dv * key[(((size_t)j * 2 + 0) * LK + pt) * N + n];
        s1 += (u128)dv * key[(((size_t)j * 2 + 1) * LK + pt) * N + n];
      }
      acc0[(size_t)t * N + n] = (u64)(s0 % m);
      acc1[(size_t)t * N + n] = (u64)(s1 % m);
    }
  }
  ock_moddown(c, acc0, limbs, ks0);
  ock_moddown(c, acc1, limbs, ks1);
  free(up); free(idx); free(acc0); free(acc1);
  return 0;
}

/* Rotate-and-sum with ONE ModDown (the engine's rotate_sum_many):
 *   acc_p = sum_j [ sum_digit sigma_{g_j}(ModUp(c1_j))_digit * evk_{g_j, digit, p}
 *                   + (p == 0 ? P * sigma_{g_j}(c0_j) on the Q limbs : 0) ]
 *   out_p = ModDown(acc_p)
 * P * c0 is 0 mod every special prime, so ModDown returns sum_j sigma(c0_j) +
 * round(sum_j ks_j / P) exactly: one rounding instead of one per term. */
int ock_rotate_sum(const ock_ctx* c, const u64* const* cts, const long* ts, int n, int limbs,
                   const u64* const* keys, u64* out) {
  const int L = c->L, K = c->K, E = limbs + K, LK = L + K;
  const size_t N = c->N;
  const int beta = digit_count(c, limbs);
  u64* acc0 = (u64*)calloc((size_t)E * N, sizeof(u64));
  u64* acc1 = (u64*)calloc((size_t)E * N, sizeof(u64));
  u64* up = (u64*)malloc((size_t)beta * E * N * sizeof(u64));
  size_t* idx = (size_t*)malloc(N * sizeof(size_t));
  for (int j = 0; j < n; j++) {
    const u64 g = ock_galois_elt(c, ts[j]);
    const u64* ct = cts[j];
    const u64* key = keys[j];
    ock_modup(c, ct + (size_t)limbs * N, limbs, up);
    for (size_t k = 0; k < N; k++) idx[k] = (g == 1) ? k : auto_index(c, k, g);
#pragma omp parallel for
    for (int t = 0; t < E; t++) {
      const int pt = ext_prime(c, limbs, t);
      const u64 m = c->q[pt];
      u64 Pm = 1;
      for (int k = 0; k < K; k++) Pm = mulmod(Pm, c->q[L + k] % m, m);
      for (size_t k = 0; k < N; k++) {
        u128 s0 = 0, s1 = 0;
        for (int d = 0; d < beta; d++) {
          const u64 dv = up[((size_t)d * E + t) * N + idx[k]];
          s0 += (u128)dv * key[(((size_t)d * 2 + 0) * LK + pt) * N + k];
          s1 += (u128)dv * key[(((size_t)d * 2 + 1) * LK + pt) * N + k];
        }
        if (t < limbs) s0 += (u128)ct[(size_t)t * N + idx[k]] * (t < limbs ? Pm : 0);
        acc0[(size_t)t * N + k] = addmod(acc0[(size_t)t * N + k], (u64)(s0 % m), m);
        acc1[(size_t)t * N + k] = addmod(acc1[(size_t)t * N + k], (u64)(s1 % m), m);
      }
    }
  }
  ock_moddown(c, acc0, limbs, out);
  ock_moddown(c, acc1, limbs, out + (size_t)limbs * N);
  free(acc0); free(acc1); free(up); free(idx);
  return 0;
}

/* -------------------------------------------------------------- evaluator */
int ock_rotate(const ock_ctx* c, const u64* ct, int limbs, long t, const u64* key, u64* out) {
  const size_t N = c->N;
  const u64 g = ock_galois_elt(c, t);
  u64* ks0 = (u64*)malloc((size_t)limbs * N * sizeof(u64));
  ock_keyswitch(c, ct + (size_t)limbs * N, limbs, key, g, ks0, out + (size_t)limbs * N);
  ock_automorph_ntt(c, g, ct, out, limbs);
  for (int i = 0; i < limbs; i++)
    for (size_t n = 0; n < N; n++)
      out[(size_t)i * N + n] = addmod(out[(size_t)i * N + n], ks0[(size_t)i * N + n], c->q[i]);
  free(ks0);
  return 0;
}

int ock_rescale_poly(const ock_ctx* c, const u64* a, int limbs, u64* out) {
  if (limbs < 2) return -1;
  const size_t N = c->N;
  const int l = limbs - 1;
  const u64 ql = c->q[l];
  u64* last = (u64*)malloc(N * sizeof(u64));
  memcpy(last, a + (size_t)l * N, N * sizeof(u64));
  ock_ntt_inv(c, l, last);
#pragma omp parallel for
  for (int i = 0; i < l; i++) {
    const u64 qi = c->q[i];
    const u64 qlmod = ql % qi;
    const u64 qlinv = invmod(qlmod, qi);
    u64* r = (u64*)malloc(N * sizeof(u64));
    for (size_t n = 0; n < N; n++) {
      const u64 v = last[n];
      u64 x = v % qi;
      if (v > ql / 2) x = submod(x, qlmod, qi); /* centred lift v - ql */
      r[n] = x;
    }
    ock_ntt_fwd(c, i, r);
    for (size_t n = 0; n < N; n++)
      out[(size_t)i * N + n] = mulmod(submod(a[(size_t)i * N + n], r[n], qi), qlinv, qi);
    free(r);
  }
  free(last);
  return 0;
}

int ock_rescale(const ock_ctx* c, const u64* ct, int limbs, u64* out) {
  const size_t N = c->N;
  if (ock_rescale_poly(c, ct, limbs, out)) return -1;
  return ock_rescale_poly(c, ct + (size_t)limbs * N, limbs, out + (size_t)(limbs - 1) * N);
}

void ock_add(const ock_ctx* c, const u64* a, const u64* b, int npolys, int limbs, u64* out) {
  const size_t N = c->N;
  for (int p = 0; p < npolys; p++)
    for (int i = 0; i < limbs; i++)
      for (size_t n = 0; n < N; n++) {
        const size_t o = ((size_t)p * limbs + i) * N + n;
        out[o] = addmod(a[o], b[o], c->q[i]);
      }
}
void ock_sub(const ock_ctx* c, const u64* a, const u64* b, int npolys, int limbs, u64* out) {
  const size_t N = c->N;
  for (int p = 0; p < npolys; p++)
    for (int i = 0; i < limbs; i++)
      for (size_t n = 0; n < N; n++) {
        const size_t o = ((size_t)p * limbs + i) * N + n;
        out[o] = submod(a[o], b[o], c->q[i]);
      }
}
void ock_mul_pt(const ock_ctx* c, const u64* a, const u64* pt, int npolys, int limbs, u64* out) {
  const size_t N = c->N;
  for (int p = 0; p < npolys; p++)
    for (int i = 0; i < limbs; i++)
      for (size_t n = 0; n < N; n++) {
        const size_t o = ((size_t)p * limbs + i) * N + n;
        out[o] = mulmod(a[o], pt[(size_t)i * N + n], c->q[i]);
      }
}

int ock_mult_plain(const ock_ctx* c, const u64* ct, int limbs, double ct_scale,
                   const double* vals, size_t n, u64* out, double* out_scale) {
  if (limbs < 2) return -3; /* depth exhausted */
  const size_t N = c->N;
  const int lv = limbs - 1;
  const double pt_scale = c->T[lv - 1] * (double)c->q[lv] / ct_scale;
  u64* pt = (u64*)malloc((size_t)limbs * N * sizeof(u64));
  int rc = ock_encode(c, vals, n, limbs, pt_scale, pt);
  if (rc) { free(pt); return rc; }
  u64* prod = (u64*)malloc((size_t)2 * limbs * N * sizeof(u64));
  ock_mul_pt(c, ct, pt, 2, limbs, prod);
  rc = ock_rescale(c, prod, limbs, out);
  if (out_scale) *out_scale = c->T[lv - 1];
  free(pt);
  free(prod);
  return rc;
}

/* mult_cipher: tensor (d0, d1, d2), then the relinearisation and the rescale as
 * ONE ModDown by P q_l: z_p = <ModUp(d2), rlk_p> + P d_p over Q u P, out_p =
 * round(z_p / (P q_l)) on the remaining limbs (ock_moddown_fused). */
int ock_mult_cipher(const ock_ctx* c, const u64* a, const u64* b, int limbs,
                    const u64* rk, u64* out) {
  if (limbs < 2) return -3;
  const int L = c->L, K = c->K, E = limbs + K;
  const size_t N = c->N;
  const size_t P = (size_t)limbs * N;
  u64* d = (u64*)malloc(3 * P * sizeof(u64));
  for (int i = 0; i < limbs; i++) {
    const u64 q = c->q[i];
    for (size_t n = 0; n < N; n++) {
      const size_t o = (size_t)i * N + n;
      d[o] = mulmod(a[o], b[o], q);
      d[P + o] = addmod(mulmod(a[o], b[P + o], q), mulmod(a[P + o], b[o], q), q);
      d[2 * P + o] = mulmod(a[P + o], b[P + o], q);
    }
  }
  u64* z0 = (u64*)malloc((size_t)E * N * sizeof(u64));
  u64* z1 = (u64*)malloc((size_t)E * N * sizeof(u64));
  ks_acc(c, d + 2 * P, limbs, rk, 1, z0, z1);
  for (int i = 0; i < limbs; i++) {
    const u64 q = c->q[i];
    u64 Pm = 1;
    for (int k = 0; k < K; k++) Pm = mulmod(Pm, c->q[L + k] % q, q);
    for (size_t n = 0; n < N; n++) {
      const size_t o = (size_t)i * N + n;
      z0[o] = addmod(z0[o], mulmod(d[o], Pm, q), q);
      z1[o] = addmod(z1[o], mulmod(d[P + o], Pm, q), q);
    }
  }
  int rc = ock_moddown_fused(c, z0, limbs, out);
  if (!rc) rc = ock_moddown_fused(c, z1, limbs, out + (size_t)(limbs - 1) * N);
  free(d);
  free(z0);
  free(z1);
  return rc;
}

int ock_level_down(const ock_ctx* c, const u64* ct, int limbs, double scale,
                   int target_limbs, u64* out, double* out_scale) {
  const size_t N = c->N;
  if (target_limbs > limbs || target_limbs < 1) return -1;
  if (target_limbs == limbs) {
    memcpy(out, ct, (size_t)2 * limbs * N * sizeof(u64));
    if (out_scale) *out_scale = scale;
    return 0;
  }
  const int keep = target_limbs + 1; /* drop to target+1 limbs, then rescale */
  u64* tmp = (u64*)malloc((size_t)2 * keep * N * sizeof(u64));
  const double cst = c->T[target_limbs - 1] * (double)c->q[target_limbs] / scale;
  const int64_t k = llround(cst);
  for (int p = 0; p < 2; p++)
    for (int i = 0; i < keep; i++) {
      const u64 q = c->q[i];
      const u64 kr = reduce_signed(k, q);
      for (size_t n = 0; n < N; n++)
        tmp[((size_t)p * keep + i) * N + n] = mulmod(ct[((size_t)p * limbs + i) * N + n], kr, q);
    }
  const int rc = ock_rescale(c, tmp, keep, out);
  if (out_scale) *out_scale = c->T[target_limbs - 1];
  free(tmp);
  return rc;
}

/* ------------------------------------------------------------ packed wire format
 * (the engine's fheon_ct_upload_packed / fheon_ct_download_packed, include/fheon_b200.h):
 * [2][limbs] bitstreams, limb i = N canonical words of b_i = bit_length(q_i) bits each,
 * coefficient k at stream bits [k b_i, (k+1) b_i), bit j of the stream = bit (j mod 64)
 * of word j / 64.  Restated bit by bit (the device packs whole words). */
static int bitlen64(u64 q) {
  int b = 0;
  while (b < 64 && (q >> b) != 0) ++b;
  return b;
}

size_t ock_packed_words(const ock_ctx* c, int limbs) {
  size_t w = 0;
  for (int i = 0; i < limbs; ++i) w += c->N * (size_t)bitlen64(c->q[i]) / 64;
  return 2 * w;
}

void ock_pack(const ock_ctx* c, const uint64_t* ct, int limbs, uint64_t* out) {
  const size_t N = c->N;
  memset(out, 0, ock_packed_words(c, limbs) * sizeof(u64));
  size_t base = 0; /* bit position of the current limb's stream */
  for (int p = 0; p < 2; ++p)
    for (int i = 0; i < limbs; ++i) {
      const int b = bitlen64(c->q[i]);
      const u64* src = ct + ((size_t)p * limbs + i) * N;
      for (size_t k = 0; k < N; ++k)
        for (int j = 0; j < b; ++j)
          if ((src[k] >> j) & 1u) {
            const size_t bit = base + k * (size_t)b + (size_t)j;
            out[bit / 64] |= (u64)1 << (bit % 64);
          }
      base += N * (size_t)b;
    }
}

void ock_unpack(const ock_ctx* c, const uint64_t* in, int limbs, uint64_t* ct) {
  const size_t N = c->N;
  size_t base = 0;
  for (int p = 0; p < 2; ++p)
    for (int i = 0; i < limbs; ++i) {
      const int b = bitlen64(c->q[i]);
      u64* dst = ct + ((size_t)p * limbs + i) * N;
      for (size_t k = 0; k < N; ++k) {
        u64 v = 0;
        for (int j = 0; j < b; ++j) {
          const size_t bit = base + k * (size_t)b + (size_t)j;
          v |= ((in[bit / 64] >> (bit % 64)) & 1u) << j;
        }
        dst[k] = v;
      }
      base += N * (size_t)b;
    }
}
