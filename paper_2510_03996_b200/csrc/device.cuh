// Device-side 64-bit modular arithmetic for sm_100a, built from the 32-bit
// IMAD datapath (nvcc lowers mul.lo/mul.hi.u64 to IMAD.WIDE.U32 chains).
//
//  * Shoup multiplication by a precomputed constant w (w' = floor(w 2^64 / q))
//    for NTT twiddles and per-limb scalars.
//  * Montgomery REDC (R = 2^64) for variable x variable products and 128-bit
//    lazy accumulations (basis conversion, key inner product): any sum
//    x < q * 2^64 reduces with one REDC.  Keys and multiplicand plaintexts are
//    held in Montgomery form so REDC(sum a_i * (b_i R)) = sum a_i b_i mod q.
//  * All ciphertext words are canonical in [0, q) between kernels, so every
//    kernel output is directly comparable word-for-word with the oracle.
#pragma once

#include <cstdint>
#ifdef FHEON_DEVICE_CHECKS
#include <cstdio>
#endif

namespace fheon {

using u64 = std::uint64_t;

struct PrimeConst {
  u64 q;
  u64 qinv_neg;  // -q^{-1} mod 2^64
  u64 r2;        // R^2 mod q
  u64 mu64;      // floor(2^64 / q)
  u64 ninv, ninv_sh;
  u64 rmod;      // R mod q
  u64 pad;
};

constexpr int kMaxBases = 32;
constexpr int kMaxDigits = 16;

// Key-switching digits D_j = [b[j], b[j+1]) (contiguous, b[0] = 0, b[n] = L);
// at `limbs` active limbs digit j holds [b[j], min(b[j+1], limbs)).
struct DigitTable {
  int b[kMaxDigits + 1];
  int n;
  __host__ __device__ int lo(int j) const { return b[j]; }
  __host__ __device__ int hi(int j, int limbs) const { return b[j + 1] < limbs ? b[j + 1] : limbs; }
  __host__ __device__ int beta(int limbs) const {  // digits with an active limb
    int k = 0;
    while (k < n && b[k] < limbs) ++k;
    return k;
  }
  __host__ __device__ int digit_of(int t) const {  // digit holding Q limb t
    int k = 0;
    while (k + 1 < n && b[k + 1] <= t) ++k;
    return k;
  }
};

// Key-switch inner-product launch facts: beta active digits (host-resolved) and
// the device table owner[t] = digit of Q limb t (a broadcast load per CTA; a
// dynamically indexed kernel-parameter array would spill to local memory).
struct DigitOwner {
  const unsigned char* owner;
  int beta;
};

// A set of limb-polynomials addressed as base[b] + blk * block_stride + t * N
// with blk < blocks_per_base and t < E; prime of limb t is p0 + t (t < ell) or
// L + (t - ell) (special primes).  skip_digits = beta > 0 skips t in digit
// j = blk mod beta's own range [dig.b[j], min(dig.b[j+1], ell)) (ModUp outputs of
// several inputs, beta digits each: the digit's own limbs pass through).
struct LimbSet {
  u64* base[kMaxBases];
  int nbase;
  int blocks_per_base;
  long long block_stride;
  int E;
  int ell;
  int L;
  int skip_digits;
  DigitTable dig;
  int p0;  // prime index of limb t = 0 (q limbs)
  int count() const { return nbase * blocks_per_base * E; }
};

#ifdef __CUDACC__

// Device bounds checks (the checked build, make CHECKS=1 -> FHEON_DEVICE_CHECKS): an
// index outside its buffer prints the kernel's file:line and traps the launch, so
// the host call fails loudly instead of reading or corrupting neighbouring words.
// compute-sanitizer is closed on this GPU pool; this is what stands in.
#ifdef FHEON_DEVICE_CHECKS
#define FHEON_DCHECK(cond)                                                                                 \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("FHEON_DCHECK failed: %s at %s:%d (block %d,%d,%d thread %d)\n", #cond, __FILE__, __LINE__,   \
             (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z, (int)threadIdx.x);                           \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define FHEON_DCHECK(cond) \
  do {                     \
  } while (0)
#endif

__device__ __forceinline__ u64 mulhi(u64 a, u64 b) { return __umul64hi(a, b); }

__device__ __forceinline__ u64 csub(u64 x, u64 q) { return x >= q ? x - q : x; }
__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// a * w mod q for canonical-or-lazy a < 2^64 and constant w < q.
__device__ __forceinline__ u64 shoup_mul(u64 a, u64 w, u64 wsh, u64 q) {
  const u64 h = mulhi(a, wsh);
  return csub(a * w - h * q, q);
}

// x = hi:lo < q * 2^64  ->  x * 2^-64 mod q (canonical).
__device__ __forceinline__ u64 redc(u64 hi, u64 lo, u64 q, u64 qneg) {
  const u64 m = lo * qneg;
  const u64 t = hi + mulhi(m, q) + (lo != 0 ? 1ULL : 0ULL);
  return csub(t, q);
}

struct Acc128 {
  u64 lo = 0, hi = 0;
  __device__ __forceinline__ void mac(u64 a, u64 b) {
    const u64 l = a * b;
    const u64 h = mulhi(a, b);
    lo += l;
    hi += h + (lo < l ? 1ULL : 0ULL);
  }
};

__device__ __forceinline__ u64 mont_mul(u64 a, u64 b_mont, const PrimeConst& p) {
  return redc(mulhi(a, b_mont), a * b_mont, p.q, p.qinv_neg);
}
// standard-form product of two canonical values
__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, const PrimeConst& p) {
  const u64 t = redc(mulhi(a, b), a * b, p.q, p.qinv_neg);
  return redc(mulhi(t, p.r2), t * p.r2, p.q, p.qinv_neg);
}
__device__ __forceinline__ u64 to_mont_d(u64 a, const PrimeConst& p) {
  return redc(mulhi(a, p.r2), a * p.r2, p.q, p.qinv_neg);
}
// x mod q for any 64-bit x
__device__ __forceinline__ u64 reduce64(u64 x, const PrimeConst& p) {
  return csub(x - mulhi(x, p.mu64) * p.q, p.q);
}
__device__ __forceinline__ u64 reduce_signed(long long v, const PrimeConst& p) {
  if (v >= 0) return reduce64((u64)v, p);
  const u64 r = reduce64((u64)(-(v + 1)), p);
  return p.q - 1 - r;
}

__device__ __forceinline__ bool limbset_get(const LimbSet& s, int idx, std::size_t N,
                                            u64*& ptr, int& prime) {
  const int per_base = s.blocks_per_base * s.E;
  const int b = idx / per_base;
  const int r = idx - b * per_base;
  const int blk = r / s.E;
  const int t = r - blk * s.E;
  if (s.skip_digits > 0) {
    const int j = blk % s.skip_digits;
    if (t >= s.dig.lo(j) && t < s.dig.hi(j, s.ell)) return false;
  }
  FHEON_DCHECK(b >= 0 && b < s.nbase && b < kMaxBases && blk < s.blocks_per_base && t < s.E);
  ptr = s.base[b] + (long long)blk * s.block_stride + (long long)t * (long long)N;
  prime = t < s.ell ? s.p0 + t : s.L + (t - s.ell);
  FHEON_DCHECK(ptr != nullptr && prime >= 0 && prime < 64 + 16);
  return true;
}

// ---- counter-based PRNG (spec: DESIGN.md section 3; mirrored by the oracle)
__device__ __forceinline__ u64 mix64_d(u64 z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ u64 prng_d(u64 stream_key, u64 idx) {
  return mix64_d(stream_key ^ (idx * 0xD1B54A32D192ED03ULL + 0x8CB92BA72F3D8DD7ULL));
}
__device__ __forceinline__ int cbd21_d(u64 r) {
  return __popcll(r & 0x1FFFFFULL) - __popcll((r >> 21) & 0x1FFFFFULL);
}

__device__ __forceinline__ unsigned brev_bits(unsigned x, int bits) {
  return __brev(x) >> (32 - bits);
}

// NTT-domain automorphism source index: out[i] = in[auto_src(i)]
__device__ __forceinline__ unsigned auto_src(unsigned i, u64 g, int logN) {
  const u64 M = 2ULL << logN;
  const u64 e = 2ULL * brev_bits(i, logN) + 1ULL;
  const u64 eg = (e * g) & (M - 1);
  FHEON_DCHECK((g & 1) == 1 && i < (1u << logN));  // Galois elements are odd
  return brev_bits((unsigned)((eg - 1) >> 1), logN);
}

#endif  // __CUDACC__

}  // namespace fheon
