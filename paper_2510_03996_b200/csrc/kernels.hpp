// Host-callable launchers for the sm_100a kernels.  Plain pointers, explicit
// stream; no torch types.  Every launcher enqueues asynchronously.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "device.cuh"

namespace fheon {

// Throws fheon::Error on a launch-configuration error (no device sync);
// also counts launches (OpStats::launches).
void launch_check(const char* what);

// Live per-kernel-class timing with CUDA events on the launching stream
// (bench.py roofline).  Classes: 1 key-switch inner product, 2 NTT/iNTT
// (both phases), 3 ModUp basis conversion, 4 ModDown conversion.
struct KernelTimer;
enum KernelClass { kKsInner = 1, kNtt = 2, kModUp = 3, kModDown = 4 };

// Device-resident constant tables of one context (built in engine.cpp).
struct DevTables {
  int logN = 0, n1 = 0, n2 = 0;
  std::size_t N = 0;
  int L = 0, K = 0, dnum = 0, alpha = 0;
  DigitTable dig{};  // key-switching digit boundaries
  unsigned char* digit_owner = nullptr;  // [L]: digit of each Q limb
  PrimeConst* pc = nullptr;   // [L+K]
  u64* tw = nullptr;          // [L+K][4][N]: tw, tw', itw, itw'
  // ModUp, indexed by tab = (limbs-1)*dnum + digit
  u64* modup_qhinv = nullptr;     // [L*dnum][kMaxAlpha][2] (value, shoup) mod q_i
  u64* modup_qhat = nullptr;      // [L*dnum][L+K][kMaxAlpha] Montgomery form mod target
  // ModDown
  u64* md_pk = nullptr;           // [K][4]: (P/p_k)^{-1} mod p_k (value, shoup), (P-1)/2 mod p_k, 0
  double* md_pinv = nullptr;      // [K] fl(1/p_k)
  u64* md_phat = nullptr;         // [L][kMaxK] (P/p_k) mod q_i, Montgomery form
  u64* md_q = nullptr;            // [L][4]: P mod q_i (Montgomery), (P-1)/2 mod q_i, P^{-1} mod q_i, shoup
  // Fused relinearisation + rescale: ModDown by P' = P q_l (l = limbs - 1), special
  // limbs s = 0: q_l, s = 1..K: p_{s-1}; same layouts as md_* per dropped limb l
  u64* md2_pk = nullptr;          // [L][kMaxK][4]
  double* md2_pinv = nullptr;     // [L][kMaxK]
  u64* md2_phat = nullptr;        // [L][L][kMaxK]
  u64* md2_q = nullptr;           // [L][L][4]
  // Rescale: [l][i][4]: q_l^{-1} mod q_i, shoup, q_l mod q_i, 0
  u64* rs = nullptr;
  // secret key, NTT domain standard form [L+K][N]
  u64* s_ntt = nullptr;
  u64* sb_ntt = nullptr;  // ephemeral sparse bootstrapping secret (sparse-secret encapsulation), NTT over L+K
  // encoder (special FFT on the device, encode.cu): 5^j mod 2N (j < S), e^{2 pi i k / 2N} (k <= 2N)
  u64* rotgroup = nullptr;
  double* ksi_re = nullptr;
  double* ksi_im = nullptr;
  // optional live kernel timer (owned by the Context)
  KernelTimer* timer = nullptr;
};

// RAII scope: records a start/stop event pair around the enclosed launches
// when the context's timer is armed for class `cls`.
struct TimedScope {
  const DevTables& t;
  int cls;
  cudaStream_t st;
  TimedScope(const DevTables& t_, int c, cudaStream_t s);
  ~TimedScope();
};

constexpr int kMaxAlpha = 16;
constexpr int kMaxK = 16;
constexpr int kMaxPolys = 64;

// A list of polynomials (each [limbs][N], limb i uses prime p0 + i), optional
// per-poly Galois element used by kernels that read a permuted operand.
struct PolyList {
  u64* p[kMaxPolys];
  u64 g[kMaxPolys];
  int n;
};

// ---- NTT (batched over every limb-polynomial of the set)
// `src` (optional, same shape and primes): out-of-place -- the first phase reads
// src and writes `set`, the second phase runs in place on `set`.
void ntt_forward(const DevTables& t, const LimbSet& set, cudaStream_t st, const LimbSet* src = nullptr);
// Forward NTT whose store writes, instead of v = NTT(set) for limb-poly p, limb t:
//   out[p][t] = (src[p][t] - v) * c_t + sigma_{add_g[p]}(add[p])[t]      (add[p] may be null)
// with c_t = cst[t * cst_stride] (value, Shoup at +1): ModDown's (acc - conv) P^-1 + sigma(c0)
// and rescale's (a - lift) q_l^-1 without a separate pass over the limbs.
struct NttEpilogue {
  u64* out[kMaxPolys];
  const u64* src[kMaxPolys];
  const u64* add[kMaxPolys];
  u64 add_g[kMaxPolys];
  const u64* cst;
  int cst_stride;
  const u64* acst = nullptr;  // optional multiplier (value, Shoup) of `add` per limb
  int acst_stride = 0;
};
void ntt_forward_epilogue(const DevTables& t, const LimbSet& set, const NttEpilogue& epi, cudaStream_t st);
void ntt_inverse(const DevTables& t, const LimbSet& set, cudaStream_t st, const LimbSet* src = nullptr);

// ---- elementwise over the polys of a list, `limbs` limbs each, primes 0..limbs-1
void ew_add(const DevTables& t, const PolyList& out, const PolyList& a, const PolyList& b, int limbs, cudaStream_t st);
void ew_sub(const DevTables& t, const PolyList& out, const PolyList& a, const PolyList& b, int limbs, cudaStream_t st);
void ew_neg(const DevTables& t, const PolyList& out, const PolyList& a, int limbs, cudaStream_t st);
// out = a (*) pt (pt standard form, [limbs][N]); out may alias a
void ew_mul_pt(const DevTables& t, const PolyList& out, const PolyList& a, const u64* pt, int limbs, cudaStream_t st);
// per-limb constants (standard form value + shoup), out = a * c
struct LimbConsts {
  u64 c[64];
  u64 sh[64];
};
void ew_mul_const(const DevTables& t, const PolyList& out, const PolyList& a, const LimbConsts& c, int limbs,
                  cudaStream_t st);
void ew_add_const(const DevTables& t, const PolyList& out, const PolyList& a, const LimbConsts& c, int limbs,
                  cudaStream_t st);
// out = sum_i k_i (*) x_i over `limbs` limbs of both polys (x_i may hold more
// limbs: the tail is ignored).  kc = [n][limbs][2] (k_i mod q_t, Shoup) on the device.
constexpr int kMaxLincomb = 64;
struct LincombTerms {
  const u64* c0[kMaxLincomb];
  long long c1_off[kMaxLincomb];  // c1 - c0 in words
  int n;
};
void lincomb_const(const DevTables& t, u64* out0, u64* out1, const LincombTerms& terms, const u64* kc, int limbs,
                   cudaStream_t st);
// (d0, d1, d2) = (a0 b0, a0 b1 + a1 b0, a1 b1)
void ew_tensor(const DevTables& t, u64* d0, u64* d1, u64* d2, const u64* a0, const u64* a1, const u64* b0,
               const u64* b1, int limbs, cudaStream_t st);
// d = 2 (a (x) b) - k (s0, s1, 0): the Chebyshev step 2 T_a T_b - T_{a-b} before its
// relinearise-and-rescale (s0 = nullptr: doubling only)
void ew_tensor_cheb(const DevTables& t, u64* d0, u64* d1, u64* d2, const u64* a0, const u64* a1, const u64* b0,
                    const u64* b1, const u64* s0, const u64* s1, const LimbConsts& kc, int limbs, cudaStream_t st);
// out[p] = sigma_{g[p]}(in[p]) in the NTT domain
void automorph(const DevTables& t, const PolyList& out, const PolyList& in, int limbs, cudaStream_t st);

// ---- key switching
// ModUp basis conversion. x[b]: coefficient-domain input [limbs][N];
// ext[b]: [beta][limbs+K][N], written for every limb outside the digit's own range.
void modup_bconv(const DevTables& t, const PolyList& ext, const PolyList& x, int limbs, cudaStream_t st);
// tensor-core basis conversions (bconv_tc.cu): ModUp of digit j, ModDown conversion
void modup_bconv_tc(const DevTables& t, const PolyList& ext, const PolyList& x, int limbs, int j, cudaStream_t st);
// every digit of the ModUp in one launch; false when the shape needs the per-digit launches
bool modup_bconv_tc_all(const DevTables& t, const PolyList& ext, const PolyList& x, int limbs, cudaStream_t st);
void moddown_conv_tc(const DevTables& t, const PolyList& conv, const PolyList& z, int limbs, cudaStream_t st);
// ModDown conversion by P' = P q_l for the fused relinearisation + rescale: z points at
// limb l of each accumulator (q_l then the K special limbs, coefficient domain),
// conv gets l = limbs - 1 limbs
void moddown_fused_conv_tc(const DevTables& t, const PolyList& conv, const PolyList& z, int limbs, cudaStream_t st);
// acc[n] += x[n] * c (c Montgomery) on one limb (prime index `prime`) of every poly
void ew_axpy_limb(const DevTables& t, const PolyList& acc, const PolyList& x, u64 c_mont, int prime, cudaStream_t st);
bool bconv_tc_enabled();
// Inner product with automorphism. For each job r: acc[r] ([2][limbs+K][N]) =
//   sum_j sigma_g(D_j) (x) key_j   where D_j = d (own limbs, NTT c1) | ext (other limbs)
struct KsJobs {
  const u64* key[kMaxBases];  // [dnum][2][L+K][N] Montgomery
  const u64* ext[kMaxBases];  // [beta][limbs+K][N]
  const u64* d[kMaxBases];    // [limbs][N]
  u64* acc[kMaxBases];
  u64 g[kMaxBases];
  int n;
};
void ks_inner_product(const DevTables& t, const KsJobs& jobs, int limbs, cudaStream_t st);
// Rotate-and-sum inner product: group r accumulates its jobs [begin[r], begin[r+1])
//   acc_r = sum_j ( sum_digit sigma_{g_j}(ext_j) * key_j  +  P * sigma_{g_j}(c0_j) [Q limbs, poly 0] )
// so that ONE ModDown of acc_r yields sum_j rot(x_j): the c0 terms ride through
// the division by P exactly (P * c0 is 0 mod every p_k).
constexpr int kMaxSumJobs = 64;
constexpr int kMaxSumGroups = 64;  // (a batch's babies x images in one launch: every key read once)
struct KsSumJobs {
  const u64* key[kMaxSumJobs];
  const u64* ext[kMaxSumJobs];
  const u64* d[kMaxSumJobs];   // c1 of the input: the digit's own limbs pass through
  const u64* c0[kMaxSumJobs];  // c0 of the input
  u64 g[kMaxSumJobs];
  int begin[kMaxSumGroups + 1];
  u64* acc[kMaxSumGroups];  // [2][limbs+K][N]
  int ngroups;
  // c0_qp: c0[j] is a Q u P polynomial ([limbs+K][N], already P-scaled: the c0 half of an
  // un-ModDown'd accumulator) added as sigma_g(c0) on every limb instead of P sigma_g(c0) on Q.
  // direct[j] (c0_qp only): no key switch -- c0[j] and d[j] ([limbs+K][N] each) are added as they are.
  int c0_qp;
  unsigned char direct[kMaxSumJobs];
};
void ks_inner_sum(const DevTables& t, const KsSumJobs& jobs, int limbs, cudaStream_t st);
// Hoisted rotate-and-sum over many inputs sharing ONE key list (channel sums, FC
// folds): acc_r = sum_j sigma_{g_j}(ext_r) key_j (+ P sigma_{g_j}(c0_r)); CTAs of
// all groups walk the same keys together (grid: groups fastest), so each key
// slice is read from HBM once per launch instead of once per group.
constexpr int kMaxSharedKeys = 16;
constexpr int kMaxSharedGroups = 40;
struct KsSharedJobs {
  const u64* key[kMaxSharedKeys];
  u64 g[kMaxSharedKeys];
  int nkeys;
  const u64* ext[kMaxSharedGroups];
  const u64* d[kMaxSharedGroups];
  const u64* c0[kMaxSharedGroups];
  u64* acc[kMaxSharedGroups];
  int ngroups;
};
void ks_inner_shared(const DevTables& t, const KsSharedJobs& jobs, int limbs, cudaStream_t st);
// ModDown front half: z[p] = coefficient-domain P limbs ([K][N], prime L+k);
// conv[p] ([limbs][N]) = centred P-residue lifted to q_0..q_{limbs-1}
void moddown_conv(const DevTables& t, const PolyList& conv, const PolyList& z, int limbs, cudaStream_t st);
// (ModDown's back half (acc - conv) P^{-1} + sigma(add) runs in ntt_forward_epilogue.)
// Rescale: last[p] coefficient-domain limb (limbs-1); r[p] ([limbs-1][N]) centred lift;
// the back half (a - r) q_{limbs-1}^{-1} runs in ntt_forward_epilogue
void rescale_lift(const DevTables& t, const PolyList& r, const PolyList& last, int limbs, cudaStream_t st);

// ---- fused layer kernels
// Multiply-accumulate of plaintext diagonals: for each output o,
//   out[o] = sum_{j < nterm[o]} ct[o][j] (*) pt[o][j]     (2 polys, `limbs` limbs)
// with one 128-bit accumulation and a single reduction (no per-term rescale).
constexpr int kMacMaxOut = 8;
constexpr int kMacMaxTerms = 32;
struct MacJobs {
  const u64* ct[kMacMaxOut][kMacMaxTerms];  // c0 pointer; c1 = c0 + c1_off[o][j]
  long long c1_off[kMacMaxOut][kMacMaxTerms];
  const u64* pt[kMacMaxOut][kMacMaxTerms];  // [limbs][N] standard form
  u64* out0[kMacMaxOut];
  u64* out1[kMacMaxOut];
  int nterm[kMacMaxOut];
  int nout;
};
// The inner sums of a double-hoisted transform over a batch of inputs in ONE launch:
// output (g, i) = sum_j pt[g][j] (*) baby(i, bidx[g][j]) over Q u P, baby(i, b) =
// babies[i] + b * baby_stride (b >= 0) or ident[i] (b < 0); grid x = g * nin + i (fastest), so
// the CTAs running together read each diagonal once per batch and each baby once per giant set.
constexpr int kBsgsMaxGiants = 16;
constexpr int kBsgsMaxIn = 16;
struct BsgsMacJobs {
  const u64* pt[kBsgsMaxGiants][kMacMaxTerms];  // [E][N] standard form
  short bidx[kBsgsMaxGiants][kMacMaxTerms];
  int nterm[kBsgsMaxGiants];
  const u64* babies[kBsgsMaxIn];  // [nb][2][E][N]
  const u64* ident[kBsgsMaxIn];   // [2][E][N] or null
  u64* out[kBsgsMaxIn];           // [ngiants][2][E][N]: giant g at out[i] + g * out_stride
  long long baby_stride, out_stride, c1_off;
  int ngiants, nin;
};
void mac_bsgs(const DevTables& t, const BsgsMacJobs& jobs, int E, cudaStream_t st, int ell);
// ell >= 0: Q u P operands ([limbs][N], limbs ell.. on the special primes)
void mac_pt(const DevTables& t, const MacJobs& jobs, int limbs, cudaStream_t st, int ell = -1);
// Plaintext as a linear combination of cached real-coefficient basis vectors
// (block-indicator encodings): coeff[k] = rint(scale * sum_b w_b basis_b[k]),
// written as RNS limbs (coefficient domain, then forward NTT by the caller).
constexpr int kMaxBasis = 128;  // LinComb is a kernel parameter: 128 x 16 B + count (< 4 KiB)
struct LinComb {
  const double* basis[kMaxBasis];
  double w[kMaxBasis];
  int nb;
};
void encode_lincomb(const DevTables& t, u64* out, const LinComb& lc, double scale, int limbs, cudaStream_t st);

// ---- packed wire format: every limb's N canonical words as a contiguous
// bitstream of b_i = bit_length(q_i) bits per coefficient (N b_i / 64 words,
// coefficient k at bits [k b_i, (k+1) b_i), little-endian within and across words)
struct PackLayout {
  int bits[64];             // b_i per limb
  long long off[64 + 1];    // word offset of limb i within one packed poly; off[limbs] = poly words
  int limbs;
};
// src polys ([limbs][N] each) -> dst ([npolys][off[limbs]] words)
void pack_limbs(const DevTables& t, u64* dst, const PolyList& src, const PackLayout& lay, cudaStream_t st);
void unpack_limbs(const DevTables& t, const PolyList& dst, const u64* src, const PackLayout& lay, cudaStream_t st);

// ---- bootstrapping helpers
// ModRaise: in[p] = coefficient-domain limb 0 (mod q_0); out[p] ([L][N]) = centred lift to q_0..q_{L-1}
void modraise(const DevTables& t, const PolyList& out, const PolyList& in, int L, cudaStream_t st);
// multiply by the monomial X^{N/2} (slot-wise multiplication by i) in the NTT domain:
// out = a * (+-i_q) with i_q = psi^{N/2} (sign - on the upper half of NTT indices)
void mul_monomial_half(const DevTables& t, const PolyList& out, const PolyList& a, const LimbConsts& iq, int limbs,
                       cudaStream_t st);

// ---- encode / encrypt / keygen / decrypt
// signed coefficients -> RNS coefficient domain [limbs][N]
void coeffs_to_rns(const DevTables& t, u64* out, const long long* coeffs, int limbs, cudaStream_t st, int p0 = 0);
// canonical-embedding encode on the device: work = [re S][im S] slot values (zero-padded),
// overwritten; coeffs [N] = llround(scale * special_fft_inv / S), bit-identical to the host
void encode_fft_device(const DevTables& t, long long* coeffs, double* work, double scale, cudaStream_t st);
// CBD21 error polynomial for `stream_key` into limbs 0..nlimbs-1 (prime rule: i < ell ? i : L + i - ell)
void sample_error(const DevTables& t, u64* out, u64 stream_key, int nlimbs, int ell, cudaStream_t st);
// c1 = uniform(stream); c0 = m + e - c1 s (m, e NTT domain) over q_0..q_{limbs-1}
void encrypt_combine(const DevTables& t, u64* c0, u64* c1, const u64* m, const u64* e, u64 stream_a, int limbs,
                     cudaStream_t st);
// one key digit over all L+K limbs: a uniform, b = e - a s + [i in digit] (P mod q_i) sp; stored Montgomery
void keygen_digit(const DevTables& t, u64* b, u64* a, const u64* e, const u64* sp, const u64* s_to, u64 stream_a,
                  int lo, int hi, const u64* pmod, cudaStream_t st);
// out = s^2 over all L+K limbs
void secret_square(const DevTables& t, u64* out, cudaStream_t st);
// m_i = c0_i + c1_i s_i, i < limbs
void decrypt_core(const DevTables& t, u64* m, const u64* c0, const u64* c1, int limbs, cudaStream_t st);
// Montgomery <-> standard for nlimbs limbs with the ell prime rule
void convert_mont(const DevTables& t, u64* out, const u64* in, int nlimbs, int ell, bool to_mont, cudaStream_t st);

}  // namespace fheon
