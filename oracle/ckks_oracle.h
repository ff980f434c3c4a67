/* TEST INFRASTRUCTURE ONLY -- the CPU RNS-CKKS restatement used as the
 * bit-exact checker for the CUDA engine.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity status: the reference (slotcnn, SURVEY.md
 * section 0) contains NO RNS-CKKS arithmetic -- its backend is a cleartext
 * slot simulator (proj/src/backend.cpp:165-249) and the real FHEON depended
 * on OpenFHE v1.2.4, which is absent.  The RNS-level
 * primitives here are therefore "parity unpinned" against the reference; they
 * are pinned by known-answer tests against definitions (naive O(N^2)
 * negacyclic products and evaluations, direct coefficient automorphisms,
 * CRT-exact rescaling, encoder round trips) in tests/test_oracle_kat.py.
 * What the reference DOES pin is the decrypted-level semantics of every op
 * (rotation direction kernels.hpp:26, level rules backend.hpp:10-16), checked
 * in tests/test_oracle_vs_reference.py against oracle/_ref.
 *
 * All polynomials are arrays of uint64 words, limb-major: poly[limb][N];
 * a ciphertext is [2][limbs][N]; an evaluation key is [dnum][2][L+K][N].
 * Limb index i < L is prime q_i, index L+k is special prime p_k.
 */
#ifndef FHEON_CKKS_ORACLE_H
#define FHEON_CKKS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ock_ctx ock_ctx;

ock_ctx* ock_create(int logN, int L, int K, int dnum, int first_bits,
                    int scale_bits, int special_bits, uint64_t seed);
/* the same context over an explicit chain: primes[L+K] (q_0..q_{L-1}, p_0..p_{K-1},
 * each = 1 mod 2N), T[L] per-level scale targets -- e.g. the engine's own chain */
ock_ctx* ock_create_chain(int logN, int L, int K, int dnum, const uint64_t* primes,
                          const double* T, uint64_t seed);
void ock_destroy(ock_ctx* c);
/* primes[L+K], psi[L+K], T[L] (scale target per level, level = limbs-1) */
void ock_info(const ock_ctx* c, uint64_t* primes, uint64_t* psi, double* T);

/* ---- NTT (prime index pi in [0, L+K)) ---- */
void ock_ntt_fwd(const ock_ctx* c, int pi, uint64_t* a);
void ock_ntt_inv(const ock_ctx* c, int pi, uint64_t* a);
/* definitions for known-answer tests */
void ock_ntt_naive(const ock_ctx* c, int pi, const uint64_t* a, uint64_t* out);
void ock_negacyclic_mul_naive(const ock_ctx* c, int pi, const uint64_t* a,
                              const uint64_t* b, uint64_t* out);
/* batched over limbs 0..nlimbs-1 with prime index = limb_map[i] (NULL: i) */
void ock_ntt_fwd_limbs(const ock_ctx* c, uint64_t* a, int nlimbs, const int* limb_map);
void ock_ntt_inv_limbs(const ock_ctx* c, uint64_t* a, int nlimbs, const int* limb_map);

/* ---- automorphism X -> X^g (g odd) ---- */
void ock_automorph_ntt(const ock_ctx* c, uint64_t g, const uint64_t* in,
                       uint64_t* out, int nlimbs);
void ock_automorph_coeff(const ock_ctx* c, uint64_t g, const uint64_t* in,
                         uint64_t* out, int nlimbs, const int* limb_map);
uint64_t ock_galois_elt(const ock_ctx* c, long t); /* 5^t mod 2N, t in (-S, S) */

/* ---- encoder (canonical embedding, full packing S = N/2) ---- */
int ock_encode(const ock_ctx* c, const double* vals, size_t n, int limbs,
               double scale, uint64_t* out_ntt);
int ock_encode_coeffs(const ock_ctx* c, const double* vals, size_t n,
                      double scale, int64_t* coeffs);
void ock_decode_coeffs(const ock_ctx* c, const double* coeffs, double scale,
                       double* out);

/* ---- keys / encryption ---- */
void ock_secret(const ock_ctx* c, int8_t* s);
/* switch to a sparse secret with exactly h nonzero coefficients (0 = uniform ternary) */
void ock_set_hamming_weight(ock_ctx* c, int h);
/* ephemeral sparse bootstrapping secret s_b (h_b nonzero) of the sparse-secret encapsulation;
 * enables key ids 2 (s -> s_b, digit 0 on q_0 and P only) and 4 (s_b -> s) in ock_keygen */
void ock_set_boot_secret(ock_ctx* c, int hb);
int ock_keygen(const ock_ctx* c, uint64_t key_id, uint64_t* key);
int ock_encrypt(const ock_ctx* c, const double* vals, size_t n,
                uint64_t counter, uint64_t* ct);
int ock_decrypt(const ock_ctx* c, const uint64_t* ct, int limbs, double scale,
                double* out);

/* ---- key switching pieces ---- */
int ock_modup(const ock_ctx* c, const uint64_t* d, int limbs, uint64_t* out);
/* 1: key-switching digits balanced by bit size (engine Params::digit_split), 0: uniform */
int ock_set_digit_split(ock_ctx* c, int balanced);
/* sum_j rotate(cts[j], ts[j]) with one ModDown (engine rotate_sum_many); cts[j] [2][limbs][N] */
int ock_rotate_sum(const ock_ctx* c, const uint64_t* const* cts, const long* ts, int n, int limbs,
                   const uint64_t* const* keys, uint64_t* out);
int ock_moddown(const ock_ctx* c, const uint64_t* acc, int limbs, uint64_t* out);
int ock_keyswitch(const ock_ctx* c, const uint64_t* d, int limbs,
                  const uint64_t* key, uint64_t g, uint64_t* ks0, uint64_t* ks1);

/* ---- evaluator (ciphertexts [2][limbs][N]) ---- */
int ock_rotate(const ock_ctx* c, const uint64_t* ct, int limbs, long t,
               const uint64_t* key, uint64_t* out);
int ock_rescale(const ock_ctx* c, const uint64_t* ct, int limbs, uint64_t* out);
int ock_rescale_poly(const ock_ctx* c, const uint64_t* a, int limbs, uint64_t* out);
void ock_add(const ock_ctx* c, const uint64_t* a, const uint64_t* b, int npolys,
             int limbs, uint64_t* out);
void ock_sub(const ock_ctx* c, const uint64_t* a, const uint64_t* b, int npolys,
             int limbs, uint64_t* out);
/* out[p][i] = a[p][i] (*) pt[i] over npolys polys, no rescale */
void ock_mul_pt(const ock_ctx* c, const uint64_t* a, const uint64_t* pt,
                int npolys, int limbs, uint64_t* out);
int ock_mult_plain(const ock_ctx* c, const uint64_t* ct, int limbs,
                   double ct_scale, const double* vals, size_t n, uint64_t* out,
                   double* out_scale);
int ock_mult_cipher(const ock_ctx* c, const uint64_t* a, const uint64_t* b,
                    int limbs, const uint64_t* relin_key, uint64_t* out);
int ock_level_down(const ock_ctx* c, const uint64_t* ct, int limbs,
                   double scale, int target_limbs, uint64_t* out,
                   double* out_scale);

/* packed wire format of a [2][limbs][N] ciphertext (engine: fheon_ct_*_packed) */
size_t ock_packed_words(const ock_ctx* c, int limbs);
void ock_pack(const ock_ctx* c, const uint64_t* ct, int limbs, uint64_t* out);
void ock_unpack(const ock_ctx* c, const uint64_t* in, int limbs, uint64_t* ct);

#ifdef __cplusplus
}
#endif
#endif
