// Host-side parameter generation; see params.hpp and DESIGN.md section 3.
#include "params.hpp"

#include <cmath>
#include <stdexcept>

namespace fheon {

u64 powmod(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod(r, a, q);
    a = mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}

bool is_prime(u64 n) {
  static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (u64 b : bases)
    if (n % b == 0) return n == b;
  u64 d = n - 1;
  int r = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++r;
  }
  for (u64 b : bases) {
    u64 x = powmod(b, d, n);
    if (x == 1 || x == n - 1) continue;
    bool composite = true;
    for (int j = 1; j < r; ++j) {
      x = mulmod(x, x, n);
      if (x == n - 1) {
        composite = false;
        break;
      }
    }
    if (composite) return false;
  }
  return true;
}

unsigned bitrev(unsigned x, int bits) {
  unsigned r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1u);
    x >>= 1;
  }
  return r;
}

namespace {

bool contains(const std::vector<u64>& v, u64 x) {
  for (u64 y : v)
    if (y == x) return true;
  return false;
}

// Largest value = 1 mod M strictly below 2^bits.
u64 top_candidate(int bits, u64 M) {
  u64 x = (((1ULL << bits) - 1) / M) * M + 1;
  if (x >= (1ULL << bits)) x -= M;
  return x;
}

}  // namespace

std::vector<int> balanced_digits(const std::vector<double>& bits, int dnum, int max_size) {
  const int L = (int)bits.size();
  auto split = [&](double cap, std::vector<int>* out) {  // greedy: fewest digits under cap
    std::vector<int> d{0};
    double acc = 0.0;
    int size = 0;
    for (int i = 0; i < L; ++i) {
      if (bits[i] > cap) return false;
      if (size == max_size || acc + bits[i] > cap) {
        d.push_back(i);
        acc = 0.0;
        size = 0;
      }
      acc += bits[i];
      ++size;
    }
    d.push_back(L);
    if ((int)d.size() - 1 > dnum) return false;
    if (out) *out = d;
    return true;
  };
  double lo = 0.0, hi = 0.0;
  for (double b : bits) hi += b;
  std::vector<int> best;
  if (!split(hi + 1.0, &best)) throw std::invalid_argument("digit split: too many limbs for dnum digits");
  for (int it = 0; it < 60; ++it) {  // bisection on the widest digit's bits
    const double mid = 0.5 * (lo + hi);
    std::vector<int> d;
    if (split(mid, &d)) {
      hi = mid;
      best = d;
    } else {
      lo = mid;
    }
  }
  return best;
}

// HE standard (Albrecht et al., "Homomorphic Encryption Security Standard",
// homomorphicencryption.org 2018, Table 1, uniform ternary secret, classical
// attacks): max log2(q) for N = 2^10 .. 2^15.  The standard stops at 2^15; the
// 2^16 row is the extension libraries ship beside it (OpenFHE's HEStd tables).
double he_standard_max_logqp(int logN, int bits) {
  static const double tab[7][3] = {{27, 19, 14},    {54, 37, 29},    {109, 75, 58},   {218, 152, 118},
                                   {438, 305, 237}, {881, 611, 476}, {1747, 1224, 956}};
  if (logN < 10 || logN > 16) return 0.0;
  const int col = bits <= 128 ? 0 : bits <= 192 ? 1 : 2;
  return tab[logN - 10][col];
}

int he_standard_security(int logN, double log_qp, int hamming_weight) {
  if (hamming_weight > 0) return -1;
  for (int bits : {256, 192, 128})
    if (log_qp <= he_standard_max_logqp(logN, bits)) return bits;
  return 0;
}

HostTables make_tables(const Params& p) {
  if (p.logN < 10 || p.logN > 16) throw std::invalid_argument("logN must be in [10, 16]");
  if (p.L < 1 || p.K < 1 || p.L + p.K > kMaxPrimes || p.dnum < 1)
    throw std::invalid_argument("bad limb counts");
  if (p.first_bits > 60 || p.scale_bits > 60 || p.special_bits > 60 || p.scale_bits < 20)
    throw std::invalid_argument("prime bit sizes must be in [20, 60]");
  HostTables t;
  t.p = p;
  t.N = std::size_t{1} << p.logN;
  t.S = static_cast<int>(t.N / 2);
  t.alpha = (p.L + p.dnum - 1) / p.dnum;
  t.nprimes = p.L + p.K;
  const u64 M = 2 * static_cast<u64>(t.N);

  std::vector<u64> q;
  {  // q_0
    u64 x = top_candidate(p.first_bits, M);
    while (!is_prime(x)) x -= M;
    q.push_back(x);
  }
  // Scaling primes, chosen top-down so the FLEXIBLEAUTO targets
  // T_{lv-1} = T_lv^2 / q_lv follow the per-level schedule tbits[] (no
  // compounding drift).  Without bootstrapping every level targets
  // 2^scale_bits.  With bootstrapping the top levels (CoeffsToSlots, EvalMod)
  // target 2^boot_scale_bits and the SlotsToCoeffs levels step linearly down
  // to 2^scale_bits, so the raised ciphertext's linear transforms and the
  // modular-reduction polynomial run at full precision.
  std::vector<double> tbits(p.L, (double)p.scale_bits);
  // "free" levels: the SlotsToCoeffs rescales when the bootstrapping levels are wider
  // than 55 bits.  Those levels only ever multiply by plaintexts (encoded at
  // T_{lv-1} q_lv / T_lv, bootstrap.cpp plan), so their primes need not follow
  // T_lv^2 / T_{lv-1} -- which would exceed 2^61 on a steep 60 -> 40-bit ramp:
  // q_lv is the prime nearest 4 T_{lv-1} and T_{lv-1} is the exact ramp target.
  std::vector<char> free_level(p.L, 0);
  if (p.bootstrap && p.boot_scale_bits > p.scale_bits) {
    const int D = bootstrap_depth(p);
    const int lv_in = p.L - 1 - (D - p.boot_stc_levels);  // SlotsToCoeffs input level
    for (int lv = 0; lv < p.L; ++lv) {
      if (lv >= lv_in) tbits[lv] = p.boot_scale_bits;
      else if (lv >= lv_in - p.boot_stc_levels) {
        const int k = lv_in - lv;  // 1..stc
        tbits[lv] = p.boot_scale_bits - (double)(p.boot_scale_bits - p.scale_bits) * k / p.boot_stc_levels;
      }
      if (p.boot_scale_bits > 55 && lv <= lv_in && lv > lv_in - p.boot_stc_levels) free_level[lv] = 1;
    }
  }
  t.T.assign(p.L, 0.0);
  std::vector<u64> chosen(p.L, 0);
  {
    double T = std::ldexp(1.0, (int)std::lround(tbits[p.L - 1]));
    t.T[p.L - 1] = T;
    for (int lv = p.L - 1; lv >= 1; --lv) {
      const double target = free_level[lv] ? std::exp2(tbits[lv - 1] + 2.0)
                                            : (T * T) / std::ldexp(1.0, (int)std::lround(tbits[lv - 1]));
      if (!(target < std::ldexp(1.0, 61)) || !(target > std::ldexp(1.0, 20)))
        throw std::invalid_argument("scale schedule needs a prime outside [2^20, 2^61)");
      const u64 tgt = static_cast<u64>(target);
      const u64 base = ((tgt - 1) / M) * M + 1;
      u64 pick = 0;
      auto ok = [&](u64 x) {
        if (!is_prime(x) || contains(q, x)) return false;
        for (int i = p.L - 1; i > lv; --i)
          if (chosen[i] == x) return false;
        return true;
      };
      for (u64 k = 0; pick == 0; ++k) {
        const u64 down = base - k * M, up = base + (k + 1) * M;
        const u64 first = (tgt - down <= up - tgt) ? down : up;
        const u64 second = (first == down) ? up : down;
        if (ok(first)) pick = first;
        else if (ok(second)) pick = second;
      }
      chosen[lv] = pick;
      T = free_level[lv] ? std::exp2(tbits[lv - 1]) : (T * T) / static_cast<double>(pick);
      t.T[lv - 1] = T;
    }
    for (int lv = 1; lv < p.L; ++lv) q.push_back(chosen[lv]);
  }
  {  // special primes
    u64 x = top_candidate(p.special_bits, M);
    for (int k = 0; k < p.K; ++k) {
      while (!is_prime(x) || contains(q, x)) x -= M;
      q.push_back(x);
      x -= M;
    }
  }
  t.q = q;
  if (p.digit_split) {
    std::vector<double> bits(p.L);
    for (int i = 0; i < p.L; ++i) bits[i] = std::log2((double)q[i]);
    t.dig = balanced_digits(bits, p.dnum, 15);
  } else {
    for (int j = 0; j * t.alpha < p.L; ++j) t.dig.push_back(j * t.alpha);
    t.dig.push_back(p.L);
  }
  t.ndig = (int)t.dig.size() - 1;
  t.alpha = 0;
  for (int j = 0; j < t.ndig; ++j) t.alpha = std::max(t.alpha, t.dig[j + 1] - t.dig[j]);
  t.psi.resize(q.size());
  for (std::size_t i = 0; i < q.size(); ++i) {
    const u64 qi = q[i];
    for (u64 g = 2;; ++g) {
      const u64 psi = powmod(g, (qi - 1) / M, qi);
      if (powmod(psi, t.N, qi) == qi - 1) {
        t.psi[i] = psi;
        break;
      }
    }
  }
  t.rotgroup.resize(t.S);
  u64 g = 1;
  for (int j = 0; j < t.S; ++j) {
    t.rotgroup[j] = g;
    g = (g * 5) % M;
  }
  t.ksi_re.resize(M + 1);
  t.ksi_im.resize(M + 1);
  for (u64 k = 0; k <= M; ++k) {
    const double ang = 2.0 * 3.14159265358979323846 * static_cast<double>(k) / static_cast<double>(M);
    t.ksi_re[k] = std::cos(ang);
    t.ksi_im[k] = std::sin(ang);
  }
  return t;
}

}  // namespace fheon
