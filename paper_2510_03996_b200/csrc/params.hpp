// Host-side RNS-CKKS parameter generation and precomputed constant tables.
//
// The reference carries crypto parameters as metadata only
// (proj/include/slotcnn/backend.hpp:32-49, CryptoMetadata{first_modulus_bits,
// rescale_bits, key_switch_digits}); this engine interprets them.  The prime
// chain, roots, FLEXIBLEAUTO scale targets and PRNG streams follow the spec
// written out in DESIGN.md section 3 (mirrored by oracle/ckks_oracle.c, the
// test-only checker -- no code is shared between the two).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace fheon {

using u64 = std::uint64_t;
using u128 = unsigned __int128;

constexpr int kMaxPrimes = 80;

struct Params {
  int logN = 14;
  int L = 11;       // Q limbs (levels 0..L-1)
  int K = 4;        // special P limbs
  int dnum = 3;     // key-switching digits
  int first_bits = 50;
  int scale_bits = 40;
  int special_bits = 60;
  u64 seed = 1;
  int depth_budget = -1;  // simulator-facing level budget (<= L-1); -1 = L-1
  int hamming_weight = 0; // secret: 0 = uniform ternary, h > 0 = exactly h nonzero (+-1)
  int bootstrap = 0;      // 1: build the bootstrapping pipeline (needs a sparse secret)
  int boot_scale_bits = 0;  // scale of the bootstrapping levels (0 = scale_bits)
  // bootstrapping shape (see bootstrap.hpp)
  int boot_k_range = 16;
  int boot_double_angles = 3;
  int boot_cts_levels = 3;
  int boot_stc_levels = 3;
  // sparse-slot bootstrapping variants over n = S/2, S/4, ..., S/2^boot_sparse slots
  // (bootstrap_active picks the smallest that holds the active slots; 0 = none)
  int boot_sparse = 0;
  // key-switching digits: 0 = uniform alpha = ceil(L / dnum) limbs each; 1 = contiguous
  // digits balanced by bit size (the widest digit decides how many special primes
  // P needs, so a chain of mixed 40/55-bit primes wants unequal limb counts)
  int digit_split = 0;
  // Sparse-secret encapsulation (bootstrapping with a DENSE main secret, hamming_weight = 0):
  // the level-0 ciphertext is switched to an ephemeral sparse secret s_b with this many
  // nonzero coefficients, ModRaised (|I| stays inside boot_k_range), and switched back to
  // the dense secret at the top of the chain.  The s -> s_b key lives only on q_0 and the
  // special primes.
  int boot_hamming_weight = 64;
  // HE-standard security (he_standard_max_logqp): context creation refuses a chain whose
  // log2(QP) exceeds the bound for N at min_security bits unless allow_insecure is set
  int min_security = 128;
  int allow_insecure = 0;
  // 1: a server context holding NO secret key -- evaluation keys must be uploaded
  // (fheon_key_upload*), encrypt / decrypt / key generation are refused
  int no_secret = 0;
};

// HE-standard (homomorphicencryption.org, 2018) maximum log2(QP) for a uniform
// ternary secret at N = 2^logN and `bits` of classical security (128, 192, 256);
// 0 when the table has no entry
double he_standard_max_logqp(int logN, int bits);
// security level (256/192/128) the chain meets under the table, 0 when below 128;
// -1 when the main secret is sparse (not covered by the table)
int he_standard_security(int logN, double log_qp, int hamming_weight);

// key ids of the sparse-secret encapsulation keys (even: never a Galois element)
constexpr std::uint64_t kKeyToSparse = 2;    // s -> s_b, on q_0 and P only
constexpr std::uint64_t kKeyFromSparse = 4;  // s_b -> s, whole chain
// sigma_g(s_b) -> s, whole chain: the encapsulation's switch back merged into the sparse-slot
// bootstrapping trace (id = g << 4 | 6, g an odd Galois element)
constexpr std::uint64_t kKeyFromSparseRotTag = 6;
constexpr std::uint64_t key_from_sparse_rot(std::uint64_t g) { return (g << 4) | kKeyFromSparseRotTag; }
constexpr bool is_key_from_sparse_rot(std::uint64_t id) { return (id & 15) == kKeyFromSparseRotTag && id > 15; }

// contiguous split of per-limb bit sizes into at most `dnum` digits minimising the
// widest digit's bit sum (each digit <= max_size limbs); returns boundaries 0 = d_0 < ... < d_n = L
std::vector<int> balanced_digits(const std::vector<double>& bits, int dnum, int max_size);

// levels consumed by bootstrapping for these parameters (bootstrap.cpp)
int bootstrap_depth(const Params& p);

// Everything derived from Params on the host.
struct HostTables {
  Params p;
  std::size_t N = 0;
  int S = 0, alpha = 0, nprimes = 0;  // alpha = widest digit (limbs)
  std::vector<int> dig;                 // digit boundaries d_0 = 0 < ... < d_ndig = L
  int ndig = 0;
  std::vector<u64> q;        // [L+K]: q_0..q_{L-1}, p_0..p_{K-1}
  std::vector<u64> psi;      // primitive 2N-th roots
  std::vector<double> T;     // scale target per level (level = limbs-1)
  std::vector<u64> rotgroup; // 5^j mod 2N
  std::vector<double> ksi_re, ksi_im;  // e^{2 pi i k / 2N}, k in [0, 2N]
};

HostTables make_tables(const Params& p);

// ---- modular helpers (host)
inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
inline u64 addmod(u64 a, u64 b, u64 q) { u64 r = a + b; return r >= q ? r - q : r; }
inline u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
u64 powmod(u64 a, u64 e, u64 q);
inline u64 invmod(u64 a, u64 q) { return powmod(a % q, q - 2, q); }
inline u64 shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
inline u64 to_mont(u64 a, u64 q) { return (u64)(((u128)(a % q) << 64) % q); }
bool is_prime(u64 n);
unsigned bitrev(unsigned x, int bits);

// ---- counter-based PRNG (spec shared with the oracle)
inline u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline u64 prng_stream_key(u64 seed, u64 stream) {
  return mix64(seed + 0x9E3779B97F4A7C15ULL * (stream + 1));
}
constexpr u64 kStreamSecret = 1;
inline u64 stream_key(u64 key_id, int digit, int kind) {  // kind 2 = a, 3 = e
  return (key_id << 16) | ((u64)digit << 4) | (u64)kind;
}
inline u64 stream_enc(u64 counter, int kind) {  // kind 4 = a, 5 = e
  return (1ULL << 60) | (counter << 4) | (u64)kind;
}

}  // namespace fheon
