// Full-slot CKKS bootstrapping (see bootstrap.hpp).
#include "bootstrap.hpp"

#include <algorithm>
#include <chrono>
#include <cuda_profiler_api.h>
#include <string>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <set>

#include "layers.hpp"

namespace fheon {

namespace {
constexpr double kPi = 3.14159265358979323846;

long ilog2(long v) {
  long l = 0;
  while ((1L << l) < v) ++l;
  return l;
}

// signed representative of a slot offset in (-S/2, S/2]
long signed_off(long d, long S) {
  d %= S;
  if (d < 0) d += S;
  return d > S / 2 ? d - S : d;
}
}  // namespace

// One special-FFT stage as a 3-diagonal slot matrix: M x = sum_d diag_d (*) rot(x, d).
// Forward (decode, Context::decode_coeffs): for p = k mod len < len/2:
//   out[k] = x[k] + w_p x[k+len/2];  p >= len/2: out[k] = x[k-len/2] - w x[k]
// Inverse (encode, fft_special_inv) with the 1/2 of U^{-1} = (1/S) ... per stage.
Bootstrapper::Mat Bootstrapper::stage(int len, bool inverse) const {
  const HostTables& h = ctx_.host();
  const long S = S_, M = 2 * (long)h.N;
  const int lenh = len / 2;
  const long lenq = (long)len * 4;
  Mat m;
  Diag d0(S), dp(S), dm(S);
  for (long k = 0; k < S; ++k) {
    const long p = k % len;
    const long j = p < lenh ? p : p - lenh;
    long idx;
    if (!inverse) idx = (long)(h.rotgroup[j] % lenq) * (M / lenq);
    else idx = (lenq - (long)(h.rotgroup[j] % lenq)) * (M / lenq);
    const std::complex<double> w(h.ksi_re[idx], h.ksi_im[idx]);
    if (!inverse) {
      if (p < lenh) {
        d0[k] = 1.0;
        dp[k] = w;
      } else {
        d0[k] = -w;
        dm[k] = 1.0;
      }
    } else {
      if (p < lenh) {
        d0[k] = 0.5;
        dp[k] = 0.5;
      } else {
        d0[k] = -0.5 * w;
        dm[k] = 0.5 * w;
      }
    }
  }
  // +len/2 and -len/2 coincide when len = S (disjoint supports): accumulate
  for (const auto& [off, d] : {std::pair<long, const Diag*>{0, &d0}, {signed_off(lenh, S), &dp},
                               {signed_off(-lenh, S), &dm}}) {
    Diag& dst = m[off];
    if (dst.empty()) dst.assign(S, 0.0);
    for (long k = 0; k < S; ++k) dst[k] += (*d)[k];
  }
  return m;
}

// (A B) x = sum_{a,b} (A_a (*) rot(B_b, a)) (*) rot(x, a + b)
Bootstrapper::Mat Bootstrapper::mul(const Mat& A, const Mat& B) const {
  const long S = S_;
  Mat out;
  for (const auto& [a, da] : A)
    for (const auto& [b, db] : B) {
      const long o = signed_off(a + b, S);
      Diag& dst = out[o];
      if (dst.empty()) dst.assign(S, 0.0);
      for (long k = 0; k < S; ++k) dst[k] += da[k] * db[(k + a % S + S) % S];
    }
  // drop all-zero diagonals
  for (auto it = out.begin(); it != out.end();) {
    bool nz = false;
    for (const auto& v : it->second) nz = nz || std::abs(v) > 1e-300;
    it = nz ? std::next(it) : out.erase(it);
  }
  return out;
}

Bootstrapper::Mat Bootstrapper::reduce_period(const Mat& M, long period) const {
  if (period >= S_) return M;
  Mat out;
  for (const auto& [d, v] : M) {
    long r = ((d % period) + period) % period;
    if (r > period / 2) r -= period;
    Diag& dst = out[r];
    if (dst.empty()) dst.assign(S_, 0.0);
    for (long k = 0; k < S_; ++k) dst[k] += v[k];
  }
  for (auto it = out.begin(); it != out.end();) {
    bool nz = false;
    for (const auto& v : it->second) nz = nz || std::abs(v) > 1e-300;
    it = nz ? std::next(it) : out.erase(it);
  }
  return out;
}

std::vector<Bootstrapper::Level> Bootstrapper::plan(const std::vector<Mat>& groups, int limbs_in, double scale_in,
                                                   const std::vector<long>& periods) {
  const HostTables& h = ctx_.host();
  const long S = S_;
  std::vector<Level> out;
  int limbs = limbs_in;
  double scale = scale_in;
  for (std::size_t gi_ = 0; gi_ < groups.size(); ++gi_) {
    const Mat& M = groups[gi_];
    const long period = gi_ < periods.size() ? periods[gi_] : S;
    // offset representations: signed (-S/2, S/2]; for a period-periodic input also
    // [0, period) -- the diagonals then fit under fewer giants (rot(x, d) = rot(x, d - period))
    std::vector<int> reps = {0};
    if (period < S) reps.push_back(1);
    auto rep_of = [&](long d, int rep) {
      if (rep == 0) return d;
      return ((d % period) + period) % period;
    };
    // baby-step size: minimise the key-switch cost.  Single hoisting: every baby
    // and giant is a full key switch (cost 1 each).  Double hoisting: a baby is one
    // key inner product (1), a giant its inner sum's ModDown + a ModUp + an inner
    // product (8.5, measured best of 5 / 6.7 / 8.5 / 12 / 20 on the 128-bit chain), the
    // unrotated giant its ModDown only; at most 32 MAC terms per giant
    const bool dh = bp_.double_hoist;
    static const double gcost = [] {
      const char* e = std::getenv("FHEON_DH_GCOST");
      return e ? std::atof(e) : 8.5;
    }();
    static const double g0cost = [] {
      const char* e = std::getenv("FHEON_DH_G0COST");
      return e ? std::atof(e) : 2.4;
    }();
    long best_n1 = 1, best_u = 1;
    int best_rep = 0;
    double best_cost = 1e300;
    for (int rep : reps) {
      long u = S;
      for (const auto& [d0, v] : M) {
        const long d = rep_of(d0, rep);
        if (d != 0) u = std::min(u, std::labs(d) & -std::labs(d));  // lowest set bit
      }
      if (u == S) u = 1;
      std::vector<long> ks;
      for (const auto& [d0, v] : M) ks.push_back(rep_of(d0, rep) / u);
      for (long n1 = 1; n1 <= 64; n1 *= 2) {
        std::set<long> bs, gs;
        std::map<long, int> per_giant;
        for (long k : ks) {
          const long g = (long)std::floor((double)k / (double)n1);
          bs.insert(k - g * n1);
          gs.insert(g);
          per_giant[g]++;
        }
        int maxterms = 0;
        for (const auto& [g, c] : per_giant) maxterms = std::max(maxterms, c);
        if (dh && maxterms > kMacMaxTerms) continue;
        const double nb = (double)(bs.size() - (bs.count(0) ? 1 : 0)), ng = (double)gs.size();
        const double g0 = gs.count(0) ? 1.0 : 0.0;
        const double cost = dh ? nb + gcost * (ng - g0) + g0cost * g0 : nb + ng - g0;
        if (cost < best_cost - 1e-9) {
          best_cost = cost;
          best_n1 = n1;
          best_u = u;
          best_rep = rep;
        }
      }
    }
    const long n1 = best_n1, u = best_u;
    const int lv = limbs - 1;
    const double pt_scale = h.T[lv - 1] * (double)h.q[lv] / scale;
    Level L;
    std::map<long, Giant> giants;
    std::set<long> babies;
    for (const auto& [d0, diag] : M) {
      const long k = rep_of(d0, best_rep) / u;
      const long g = (long)std::floor((double)k / (double)n1);
      const long b = k - g * n1;
      const long G = g * n1 * u;
      // pre-rotate: p = rot(diag, -G)
      std::vector<double> re(S), im(S);
      for (long j = 0; j < S; ++j) {
        const auto v = diag[((j - G) % S + S) % S];
        re[j] = v.real();
        im[j] = v.imag();
      }
      BufPtr pt = ctx_.encode_complex(re.data(), im.data(), (std::size_t)S, limbs, pt_scale, dh ? h.p.K : 0);
      Giant& gi = giants[g];
      gi.rot = signed_off(G, S);
      gi.terms.push_back({signed_off(b * u, S), pt});
      if (b != 0) babies.insert(signed_off(b * u, S));
    }
    L.babies.assign(babies.begin(), babies.end());
    for (auto& [g, gi] : giants) L.giants.push_back(gi);
    L.qp = dh;
    out.push_back(L);
    limbs -= 1;
    scale = h.T[limbs - 1];
  }
  return out;
}

namespace {
// EvalMod cosine: cos(2 pi ((K+1) u - 1/4) / 2^r) on u in [-1, 1]
std::function<double(double)> evalmod_fn(int k_range, int r) {
  const double K1 = k_range + 1.0;
  return [K1, r](double u) { return std::cos(2.0 * kPi * (K1 * u - 0.25) / std::ldexp(1.0, r)); };
}
int evalmod_degree(int k_range, int r) {
  const std::vector<double> c = cheb_coefficients(evalmod_fn(k_range, r), 127);
  int deg = 1;
  for (int d = 1; d < (int)c.size(); ++d)
    if (std::fabs(c[d]) > 1e-13) deg = d;
  return deg;
}
}  // namespace

int bootstrap_depth(const Params& p) {
  return p.boot_cts_levels + cheb_eval_depth(evalmod_degree(p.boot_k_range, p.boot_double_angles)) +
         p.boot_double_angles + p.boot_stc_levels;
}

BootParams boot_params_of(const Params& p) {
  BootParams b;
  b.k_range = p.boot_k_range;
  b.double_angles = p.boot_double_angles;
  b.cts_levels = p.boot_cts_levels;
  b.stc_levels = p.boot_stc_levels;
  if (const char* e = std::getenv("FHEON_BOOT_DH")) b.double_hoist = std::atoi(e) != 0;
  return b;
}

Bootstrapper::Bootstrapper(Context& ctx, const BootParams& bp) : ctx_(ctx), bp_(bp) {
  const HostTables& h = ctx.host();
  S_ = h.S;
  n_ = bp.log_slots > 0 ? (1L << bp.log_slots) : (long)S_;
  if (n_ > S_ || n_ < 4) throw Error(ErrKind::shape, "bootstrapping: sparse slot count must lie in [4, S]");
  const int L = h.p.L;
  const long logS = ilog2(n_);
  const double K1 = bp.k_range + 1.0;
  const int r = bp.double_angles;
  const int deg = bp.cos_degree > 0 ? bp.cos_degree : evalmod_degree(bp.k_range, r);
  cos_coeffs_ = cheb_coefficients(evalmod_fn(bp.k_range, r), deg);
  depth_ = bp.cts_levels + cheb_eval_depth(deg) + r + bp.stc_levels;
  if (depth_ > L - 2)
    throw Error(ErrKind::shape, "bootstrapping needs " + std::to_string(depth_) + " levels; the chain has " +
                                    std::to_string(L - 1));
  if (bp.cts_levels < 1 || bp.stc_levels < 1 || bp.cts_levels > logS || bp.stc_levels > logS)
    throw Error(ErrKind::shape, "bootstrapping: bad linear-transform level split");
  auto split = [&](int levels) {
    std::vector<int> sizes(levels, (int)(logS / levels));
    for (int i = 0; i < (int)(logS % levels); ++i) sizes[i]++;
    return sizes;
  };
  // CoeffsToSlots: inverse stages len = n .. 2 (first applied first).  Sparse: the
  // smaller group first (fewer diagonals on the top level, and the lower groups
  // then hold the same stages as the full pipeline's)
  const long g = S_ / n_;
  {
    std::vector<int> sizes = split(bp.cts_levels);
    if (sparse()) std::reverse(sizes.begin(), sizes.end());
    std::vector<Mat> groups;
    // 1 / (2 (K + 1)) spread evenly over the levels -- or, when the first level's
    // plaintexts (scale T_{L-2} q_{L-1} / q_0, about 2^65 on 60-bit bootstrapping
    // levels) would overflow the encoder's 2^62, all on the first level.  Sparse:
    // the trace's factor g is divided out on the first level too
    const double first_pt_scale = h.T[L - 2] * (double)h.q[L - 1] / (double)h.q[0];
    const double c_even = std::pow(1.0 / (2.0 * K1), 1.0 / bp.cts_levels);
    const bool front = first_pt_scale * c_even > std::ldexp(1.0, 60);
    long len = n_;
    for (int gsz : sizes) {
      Mat M = stage((int)len, true);
      len /= 2;
      for (int i = 1; i < gsz; ++i, len /= 2) M = mul(stage((int)len, true), M);
      double c = front ? (groups.empty() ? 1.0 / (2.0 * K1) : 1.0) : c_even;
      if (groups.empty()) c /= (double)g;
      for (auto& [d, v] : M)
        for (auto& x : v) x *= c;
      groups.push_back(M);
    }
    if (sparse()) {  // pack: slots k mod 2n < n keep z, the others take -i z (v + conj v = [2 Re | 2 Im])
      Diag dv(S_);
      for (long k = 0; k < S_; ++k) dv[k] = (k % (2 * n_)) < n_ ? std::complex<double>(1.0, 0.0)
                                                                : std::complex<double>(0.0, -1.0);
      groups.back() = mul(Mat{{0, dv}}, groups.back());
      // every CtS input is n-periodic (the trace's output and the stages' images)
      for (Mat& M : groups) M = reduce_period(M, n_);
    }
    cts_ = plan(groups, L, (double)h.q[0], std::vector<long>(groups.size(), n_));
  }
  // SlotsToCoeffs: forward stages len = 2 .. n, scaled by q0 / (2 pi Delta_0)
  {
    std::vector<int> sizes = split(bp.stc_levels);
    // sparse: the smaller groups first as well -- StC's first factor also carries the
    // unpacking P (twice the diagonals) and runs on StC's highest level
    static const bool stc_small_first = [] {
      const char* e = std::getenv("FHEON_STC_SMALL_FIRST");
      return !(e && e[0] == '0');
    }();
    if (sparse() && stc_small_first) std::reverse(sizes.begin(), sizes.end());
    std::vector<Mat> groups;
    const double c = std::pow((double)h.q[0] / (2.0 * kPi * h.T[0]), 1.0 / bp.stc_levels);
    long len = 2;
    for (int gsz : sizes) {
      Mat M = stage((int)len, false);
      len *= 2;
      for (int i = 1; i < gsz; ++i, len *= 2) M = mul(stage((int)len, false), M);
      for (auto& [d, v] : M)
        for (auto& x : v) x *= c;
      groups.push_back(M);
    }
    if (sparse()) {
      // unpack: z_k = w_k + i w_{k+n} (k mod 2n < n), w_{k-n} + i w_k (otherwise)
      Diag da(S_), db(S_);
      for (long k = 0; k < S_; ++k) {
        const bool lo = (k % (2 * n_)) < n_;
        da[k] = lo ? std::complex<double>(1.0, 0.0) : std::complex<double>(0.0, 1.0);
        db[k] = lo ? std::complex<double>(0.0, 1.0) : std::complex<double>(1.0, 0.0);
      }
      groups.front() = mul(groups.front(), Mat{{0, da}, {signed_off(n_, S_), db}});
      Diag mask(S_);
      for (long k = 0; k < S_; ++k) mask[k] = k < n_ ? 1.0 : 0.0;
      groups.back() = mul(Mat{{0, mask}}, groups.back());
      // the first factor reads the 2n-periodic EvalMod output, the others n-periodic images
      for (std::size_t i = 0; i < groups.size(); ++i) groups[i] = reduce_period(groups[i], i == 0 ? 2 * n_ : n_);
    }
    const int stc_limbs = L - bp.cts_levels - cheb_eval_depth(deg) - r;
    stc_limbs_ = stc_limbs;
    std::vector<long> periods(groups.size(), n_);
    periods[0] = std::min<long>(2 * n_, S_);  // the EvalMod output is 2n-periodic
    stc_ = plan(groups, stc_limbs, h.T[stc_limbs - 1], periods);
  }
  if (sparse())
    for (long j = 1; j < g; ++j) sub_steps_.push_back(j * n_);
  if (std::getenv("FHEON_BOOT_TIMING")) {
    for (const auto* v : {&cts_, &stc_}) {
      std::fprintf(stderr, "[boot n=%ld] %s:", n_, v == &cts_ ? "CtS" : "StC");
      for (const Level& lv : *v) {
        std::size_t terms = 0;
        for (const Giant& gi : lv.giants) terms += gi.terms.size();
        std::fprintf(stderr, " (%zu babies, %zu giants, %zu diagonals)", lv.babies.size(), lv.giants.size(), terms);
      }
      std::fprintf(stderr, "\n");
    }
  }
  for (long s : rotation_steps()) {  // a server context (no secret) receives them by upload
    if (ctx.has_secret() && !ctx.inheriting_keys) ctx.gen_key(ctx.galois(s));
    ctx.pin_key(ctx.galois(s));
  }
  if (sparse()) {  // conj o rot_G for the last CtS level's giant steps
    const u64 twoN = 2 * (u64)h.N;
    for (const Giant& gi : cts_.back().giants) {
      const u64 gc = (ctx.galois(gi.rot) * (twoN - 1)) % twoN;
      if (ctx.has_secret() && !ctx.inheriting_keys) ctx.gen_key(gc);
      ctx.pin_key(gc);
    }
  }
  if (ctx.has_secret() && !ctx.inheriting_keys) {
    ctx.gen_key(2 * (u64)h.N - 1);  // conjugation
    ctx.gen_key(0);                 // relinearisation
  }
  ctx.pin_key(2 * (u64)h.N - 1);
  ctx.pin_key(0);
  if (ctx.sse()) {  // sparse-secret encapsulation keys
    std::vector<u64> ids = {kKeyToSparse, kKeyFromSparse};
    for (long t : sub_steps_) ids.push_back(key_from_sparse_rot(ctx.galois(t)));  // trace + switch back
    for (u64 id : ids) {
      if (ctx.has_secret() && !ctx.inheriting_keys) ctx.gen_key(id);
      ctx.pin_key(id);
    }
  }
}

Bootstrapper::Bootstrapper(Context& ctx, const Bootstrapper& o)
    : ctx_(ctx), bp_(o.bp_), S_(o.S_), n_(o.n_), sub_steps_(o.sub_steps_), depth_(o.depth_), stc_limbs_(o.stc_limbs_),
      cts_(o.cts_), stc_(o.stc_), cos_coeffs_(o.cos_coeffs_) {}

std::vector<long> Bootstrapper::rotation_steps() const {
  std::set<long> s;
  for (long t : sub_steps_) s.insert(t);
  for (const auto* v : {&cts_, &stc_})
    for (const Level& lv : *v) {
      for (long b : lv.babies) s.insert(b);
      for (const Giant& g : lv.giants)
        if (g.rot != 0) s.insert(g.rot);
    }
  return std::vector<long>(s.begin(), s.end());
}

std::vector<Ciphertext> Bootstrapper::apply_many(const std::vector<Ciphertext>& xs, const Level& lv, bool with_conj) {
  if (!lv.qp) {
    std::vector<Ciphertext> out;
    for (const Ciphertext& x : xs) out.push_back(apply(x, lv, with_conj));
    return out;
  }
  std::map<long, int> idx;
  for (std::size_t i = 0; i < lv.babies.size(); ++i) idx[lv.babies[i]] = (int)i;
  std::vector<DhGiant> gs;
  for (const Giant& g : lv.giants) {
    DhGiant d;
    d.rot = g.rot;
    for (const auto& [b, pt] : g.terms) d.terms.push_back({b == 0 ? -1 : idx.at(b), pt});
    gs.push_back(std::move(d));
  }
  return bsgs_double_hoisted_many(ctx_, xs, lv.babies, gs, with_conj);
}

Ciphertext Bootstrapper::apply(const Ciphertext& x, const Level& lv, bool with_conj) {
  if (lv.qp) return apply_many({x}, lv, with_conj)[0];
  std::vector<Ciphertext> rot = rotate_hoisted(ctx_, x, lv.babies);
  std::map<long, Ciphertext> by_b;
  by_b[0] = x;
  for (std::size_t i = 0; i < lv.babies.size(); ++i) by_b[lv.babies[i]] = rot[i];
  std::vector<std::vector<Ciphertext>> terms;
  std::vector<std::vector<BufPtr>> pts;
  for (const Giant& g : lv.giants) {
    std::vector<Ciphertext> t;
    std::vector<BufPtr> p;
    for (const auto& [b, pt] : g.terms) {
      t.push_back(by_b.at(b));
      p.push_back(pt);
    }
    terms.push_back(t);
    pts.push_back(p);
  }
  // giant steps: rotate-and-sum of the unrescaled inner sums -- one ModDown and one
  // rescale for the whole level
  std::vector<Ciphertext> inner = mac_plain_many_unrescaled(ctx_, terms, pts);
  std::vector<std::pair<Ciphertext, long>> g;
  for (std::size_t i = 0; i < lv.giants.size(); ++i) g.push_back({inner[i], lv.giants[i].rot});
  return rotate_sum_to_target(ctx_, {g}, true, with_conj)[0];
}

Ciphertext Bootstrapper::debug_stage(const Ciphertext& x0, int what) {
  const HostTables& h = ctx_.host();
  Ciphertext y = x0;
  if (what == 1) {
    y.scale = (double)h.q[0];
    for (const Level& lv : cts_) y = apply(y, lv);
    return y;
  }
  if (what == 2) {
    std::vector<Ciphertext> ys = cheb_eval_many(ctx_, {y}, cos_coeffs_, true);
    for (int i = 0; i < bp_.double_angles; ++i) {
      std::vector<Ciphertext> sq = mult_cipher_many(ctx_, ys, ys);
      ys = add_many(ctx_, sq, sq);
      for (Ciphertext& c : ys) c = add_const(ctx_, c, -1.0);
    }
    return ys[0];
  }
  if (what == 3) {
    if (y.limbs > stc_limbs_) y = level_down(ctx_, y, stc_limbs_);
    for (const Level& lv : stc_) y = apply(y, lv);
    return y;
  }
  if (what == 4) return mod_raise(ctx_, x0.limbs > 1 ? level_down(ctx_, x0, 1) : x0);
  throw Error(ErrKind::internal, "debug_stage: unknown stage");
}

std::vector<Ciphertext> Bootstrapper::subsum_many(const std::vector<Ciphertext>& xs) {
  if (sub_steps_.empty()) return xs;
  std::vector<std::vector<std::pair<Ciphertext, long>>> groups;
  for (const Ciphertext& x : xs) {
    std::vector<std::pair<Ciphertext, long>> terms = {{x, 0}};
    for (long t : sub_steps_) terms.push_back({x, t});
    groups.push_back(std::move(terms));
  }
  return rotate_sum_many(ctx_, groups);
}

Ciphertext Bootstrapper::run(const Ciphertext& x0, bool clean) {
  if (sparse()) return run_many({x0}, clean)[0];
  return run_full(x0);
}

// Sparse-slot pipeline on several ciphertexts of one level in lockstep (the images of a
// batched inference): every stage is one batched call, so keys and encoded diagonals are
// read once per batch and the NTT / basis-conversion launches carry B times the limbs.
// Per input the operations are those of the single-input pipeline (bit-identical outputs).
std::vector<Ciphertext> Bootstrapper::run_many(const std::vector<Ciphertext>& xs0, bool clean) {
  if (xs0.empty()) return {};
  if (!sparse()) {
    std::vector<Ciphertext> out;
    for (const Ciphertext& x : xs0) out.push_back(run_full(x));
    return out;
  }
  for (const Ciphertext& x : xs0)
    if (x.limbs != xs0[0].limbs) throw Error(ErrKind::internal, "bootstrap_many: inputs at different levels");
  const bool tracing = ctx_.tracing();
  ctx_.set_tracing(false);
  try {
    const HostTables& h = ctx_.host();
    const std::size_t B = xs0.size();
    if (xs0[0].limbs < 2 && !clean)
      throw Error(ErrKind::internal, "sparse-slot bootstrapping needs an input above level 0 (the mask)");
    // mask to [0, n) on the last level, replicate n-periodically, raise, trace
    static const bool timing = std::getenv("FHEON_BOOT_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!timing) return;
      FHEON_CUDA(cudaStreamSynchronize(ctx_.stream()));
      const auto t = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[boot n=%ld x%zu] %-10s %8.3f ms\n", n_, B, what,
                   std::chrono::duration<double, std::milli>(t - t_last).count());
      t_last = t;
    };
    lap("start");
    static const char* prof_env = std::getenv("FHEON_BOOT_PROFILE");  // ncu range: "all" | "cos"
    const bool prof_all = prof_env && std::string(prof_env) == "all";
    if (prof_all) FHEON_CUDA(cudaProfilerStart());
    std::vector<Ciphertext> xs(B);
    if (clean) {  // slots [n, S) already zero: no mask
      for (std::size_t i = 0; i < B; ++i) xs[i] = xs0[i].limbs > 1 ? level_down(ctx_, xs0[i], 1) : xs0[i];
    } else {
      const long n = n_, S = S_;
      std::vector<std::vector<Ciphertext>> terms;
      std::vector<std::vector<BufPtr>> pts;
      for (std::size_t i = 0; i < B; ++i) {
        const Ciphertext x = xs0[i].limbs > 2 ? level_down(ctx_, xs0[i], 2) : xs0[i];
        BufPtr mask = ctx_.encode_named("boot_mask_" + std::to_string(n),
                                        [n, S] {
                                          std::vector<double> m((std::size_t)S, 0.0);
                                          std::fill(m.begin(), m.begin() + n, 1.0);
                                          return m;
                                        },
                                        x.limbs, pt_scale_for(ctx_, x));
        terms.push_back({x});
        pts.push_back({mask});
      }
      xs = mac_plain_many(ctx_, terms, pts);
    }
    xs = subsum_many(xs);
    lap("mask+rep");
    std::vector<double> corr(B);
    for (std::size_t i = 0; i < B; ++i) corr[i] = xs[i].scale / h.T[0];
    std::vector<Ciphertext> ys = mod_raise_trace_many(ctx_, xs, n_);
    lap("modraise+trace");
    // the last CtS level returns y + conj(y) directly: its giant steps enter twice, as
    // rot_G and conj o rot_G, in one ModDown (no separate conjugation key switch)
    for (std::size_t i = 0; i < cts_.size(); ++i) {
      ys = apply_many(ys, cts_[i], i + 1 == cts_.size());
      lap("cts");
    }
    const bool prof_cos = prof_env && std::string(prof_env) == "cos";
    if (prof_cos) FHEON_CUDA(cudaProfilerStart());
    ys = cheb_eval_many(ctx_, ys, cos_coeffs_, true);
    if (prof_cos) FHEON_CUDA(cudaProfilerStop());
    lap("cos");
    for (int i = 0; i < bp_.double_angles; ++i) {  // y <- 2 y^2 - 1
      ys = mult_cipher_cheb_many(ctx_, ys, ys, std::vector<Ciphertext>(ys.size()));
      for (Ciphertext& c : ys) c = add_const(ctx_, c, -1.0);
    }
    lap("dbl-angle");
    for (const Level& lv : stc_) {
      ys = apply_many(ys, lv);
      lap("stc");
    }
    if (prof_all) FHEON_CUDA(cudaProfilerStop());
    ctx_.set_tracing(tracing);
    for (std::size_t i = 0; i < B; ++i) {
      Ciphertext& z = ys[i];
      z.scale *= corr[i];
      if (z.level() > ctx_.depth_budget()) z = level_down(ctx_, z, ctx_.depth_budget() + 1);
      ctx_.record(3, z.level());
      ctx_.stats.bootstraps++;
    }
    return ys;
  } catch (...) {
    ctx_.set_tracing(tracing);
    throw;
  }
}

Ciphertext Bootstrapper::run_full(const Ciphertext& x0) {
  const bool tracing = ctx_.tracing();
  ctx_.set_tracing(false);
  try {
    const HostTables& h = ctx_.host();
    Ciphertext x = x0.limbs > 1 ? level_down(ctx_, x0, 1) : x0;
    const double corr = x.scale / h.T[0];
    static const bool dbg = std::getenv("FHEON_BOOT_DEBUG") != nullptr;
    const std::size_t S = (std::size_t)h.S;
    std::vector<double> are(S), aim(S), bre(S), bim(S), cre(S), cim(S);
    auto maxdiff = [&](const std::vector<double>& a, const std::vector<double>& b) {
      double m = 0.0;
      for (std::size_t i = 0; i < S; ++i) m = std::max(m, std::fabs(a[i] - b[i]));
      return m;
    };
    Ciphertext y = mod_raise(ctx_, x);
    for (const Level& lv : cts_) y = apply(y, lv);
    const Ciphertext yc = conjugate_many(ctx_, {y})[0];
    std::vector<Ciphertext> ys = {add(ctx_, y, yc), mul_by_i(ctx_, sub(ctx_, yc, y))};
    std::vector<double> in0, in1;
    if (dbg) {
      decrypt(ctx_, y, are.data(), aim.data());
      decrypt(ctx_, ys[0], bre.data(), bim.data());
      decrypt(ctx_, ys[1], cre.data(), cim.data());
      std::vector<double> t0(S), t1(S), z0(S, 0.0);
      double mx = 0.0;
      for (std::size_t i = 0; i < S; ++i) {
        t0[i] = 2 * are[i];
        t1[i] = 2 * aim[i];
        mx = std::max(mx, std::fabs(are[i]) + std::fabs(aim[i]));
      }
      std::fprintf(stderr, "[boot] CtS out max|u| %.3e limbs %d scale 2^%.2f; split re err %.3e im-part %.3e; "
                           "split im err %.3e im-part %.3e\n", mx, y.limbs, std::log2(y.scale), maxdiff(bre, t0),
                   maxdiff(bim, z0), maxdiff(cre, t1), maxdiff(cim, z0));
      in0 = bre;
      in1 = cre;
    }
    ys = cheb_eval_many(ctx_, ys, cos_coeffs_, true);
    if (dbg) {
      decrypt(ctx_, ys[0], bre.data(), bim.data());
      std::vector<double> w(S);
      const double K1 = bp_.k_range + 1.0;
      for (std::size_t i = 0; i < S; ++i) w[i] = std::cos(2.0 * kPi * (K1 * in0[i] / 2.0 - 0.25) / std::ldexp(1.0, bp_.double_angles));
      std::fprintf(stderr, "[boot] cos poly out limbs %d scale 2^%.2f err %.3e\n", ys[0].limbs, std::log2(ys[0].scale),
                   maxdiff(bre, w));
    }
    for (int i = 0; i < bp_.double_angles; ++i) {  // y <- 2 y^2 - 1
      ys = mult_cipher_cheb_many(ctx_, ys, ys, std::vector<Ciphertext>(ys.size()));
      for (Ciphertext& c : ys) c = add_const(ctx_, c, -1.0);
    }
    if (dbg) {
      decrypt(ctx_, ys[0], bre.data(), bim.data());
      decrypt(ctx_, ys[1], cre.data(), cim.data());
      std::vector<double> w0(S), w1(S);
      const double K1 = bp_.k_range + 1.0;
      for (std::size_t i = 0; i < S; ++i) {
        w0[i] = std::sin(2.0 * kPi * K1 * in0[i] / 2.0);
        w1[i] = std::sin(2.0 * kPi * K1 * in1[i] / 2.0);
      }
      double mo = 0.0;
      for (std::size_t i = 0; i < S; ++i) mo = std::max(mo, std::fabs(w0[i]));
      std::fprintf(stderr, "[boot] EvalMod out limbs %d scale 2^%.2f err re %.3e im %.3e (max|sin| %.3e)\n",
                   ys[0].limbs, std::log2(ys[0].scale), maxdiff(bre, w0), maxdiff(cre, w1), mo);
    }
    Ciphertext z = add(ctx_, ys[0], mul_by_i(ctx_, ys[1]));
    std::vector<double> zre(S), zim(S);
    if (dbg) decrypt(ctx_, z, zre.data(), zim.data());
    for (const Level& lv : stc_) z = apply(z, lv);
    if (dbg) {
      // expected StC output: the slots whose coefficients are (Re, Im) of z in bit-reversed
      // order times q0 / (2 pi T_0)
      const int logS = (int)std::lround(std::log2((double)S));
      std::vector<double> co(2 * S), ore(S), oim(S), wre(S), wim(S);
      const double c = (double)h.q[0] / (2.0 * kPi * h.T[0]);
      for (std::size_t k = 0; k < S; ++k) {
        const std::size_t b = bitrev((unsigned)k, logS);
        co[k] = zre[b] * c;
        co[k + S] = zim[b] * c;
      }
      ctx_.decode_coeffs(co.data(), 1.0, wre.data(), wim.data());
      decrypt(ctx_, z, ore.data(), oim.data());
      double zm = 0.0;
      for (std::size_t i = 0; i < S; ++i) zm = std::max(zm, std::fabs(zre[i]) + std::fabs(zim[i]));
      std::fprintf(stderr, "[boot] StC in max|z| %.3e; StC out limbs %d scale 2^%.2f err re %.3e im %.3e\n", zm,
                   z.limbs, std::log2(z.scale), maxdiff(ore, wre), maxdiff(oim, wim));
    }
    z.scale *= corr;
    if (z.level() > ctx_.depth_budget()) z = level_down(ctx_, z, ctx_.depth_budget() + 1);
    ctx_.set_tracing(tracing);
    ctx_.record(3, z.level());
    ctx_.stats.bootstraps++;
    return z;
  } catch (...) {
    ctx_.set_tracing(tracing);
    throw;
  }
}

}  // namespace fheon
