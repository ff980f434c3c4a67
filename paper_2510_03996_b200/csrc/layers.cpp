// Layer algorithms over device ciphertexts.  Each function follows the
// reference's algorithm (cited per function): the same rotation indices, mask
// values, level consumption, and the same multiset of trace events.  The GPU
// realisation batches what the reference does one op at a time:
//   * rotations that share a source are hoisted (one ModUp), independent
//     rotations across output channels / rows run as one key-switch batch;
//   * a sum of plaintext products at one level ("rotate-and-MAC") is one fused
//     MAC kernel and ONE rescale instead of one rescale per term;
//   * block-constant plaintexts (kernel vectors, masked kernel vectors, biases)
//     are built on the GPU as linear combinations of cached block-indicator
//     encodings -- no host FFT per plaintext;
//   * the Chebyshev T_d tree is evaluated band by band (all d in
//     (2^{g-1}, 2^g] together) with batched relinearisation.
// Event ORDER differs from the reference where independent ops are batched;
// the event multiset (what keyplan/ledger consume) is identical.
//
// That is the reference schedule (Context::kScheduleReference).  The default
// fast schedule (Context::kScheduleFast) computes the same slot values at the
// same levels with far fewer key switches: rotation chains sum_i rot(x, i*s)
// become doubling trees, chains of rotations of one value become hoisted sets,
// Horner placement chains become one batched key switch, and stride
// extraction becomes a baby-step giant-step transform (stride_bsgs_many).
#include "layers.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>

namespace fheon {

namespace {

bool is_pow2(std::size_t v) { return v != 0 && (v & (v - 1)) == 0; }
std::size_t log2_exact(std::size_t v) {
  std::size_t l = 0;
  while ((std::size_t{1} << l) < v) ++l;
  return l;
}

Error shape_error(const std::string& m) { return Error(ErrKind::shape, m); }
Error capacity_error(const std::string& m) { return Error(ErrKind::capacity, m); }

// PlainVector::from_values(S, v) (backend.cpp:114-125): zero-filled to S
std::vector<double> plain(const Context& ctx, const std::vector<double>& v) {
  if (v.size() > (std::size_t)ctx.S())
    throw capacity_error("plain vector payload of " + std::to_string(v.size()) + " values does not fit in " +
                         std::to_string(ctx.S()) + " slots");
  std::vector<double> out(ctx.S(), 0.0);
  std::copy(v.begin(), v.end(), out.begin());
  return out;
}

// range_mask (layers_conv.cpp:39-44, layers_misc.cpp:21-26)
std::vector<double> range_mask(const Context& ctx, std::size_t begin, std::size_t count, double value = 1.0) {
  std::vector<double> v(begin + count, 0.0);
  std::fill(v.begin() + (long)begin, v.end(), value);
  return plain(ctx, v);
}

// plaintext for `like` from slot values (content-cached host encode)
BufPtr pt_of(Context& ctx, const Ciphertext& like, const std::vector<double>& full) {
  return ctx.encode_cached(full, like.limbs, pt_scale_for(ctx, like));
}

// mult_plain by a slot vector through the content-keyed plaintext cache (masks repeat
// across layers and inferences: encoded once); one mult_plain event, one rescale
Ciphertext mp(Context& ctx, const Ciphertext& x, const std::vector<double>& full) {
  if (x.level() < 1)
    throw Error(ErrKind::depth_exhausted, "mult_plain: no multiplicative depth left (level " +
                                              std::to_string(x.level()) + ")");
  return mac_plain_many(ctx, {{x}}, {{pt_of(ctx, x, full)}})[0];
}

// 128-bit content key of a weight tensor (keys the resident weight plaintexts): FNV-1a
// and an independent multiply-xorshift chain over the bit patterns, plus the shape --
// a hit on another layer's plaintexts would need both 64-bit hashes to collide
std::string weight_key(const char* tag, const KernelTensor& w, std::size_t W) {
  u64 h = 1469598103934665603ULL, g = 0x9E3779B97F4A7C15ULL;
  for (double v : w.weights) {
    u64 b;
    std::memcpy(&b, &v, 8);
    h = (h ^ b) * 1099511628211ULL;
    g = mix64(g ^ (b + 0x632BE59BD9B4E019ULL));
  }
  return std::string(tag) + ":" + std::to_string(h) + ":" + std::to_string(g) + ":" + std::to_string(w.out_channels) + "x" +
         std::to_string(w.in_channels) + "x" + std::to_string(w.kernel) + ":" + std::to_string(W);
}

// indicator of block c (size m) as a cached device basis vector
const double* block_basis(Context& ctx, std::size_t m, std::size_t c) {
  std::vector<double> v((c + 1) * m, 0.0);
  std::fill(v.begin() + (long)(c * m), v.end(), 1.0);
  return ctx.basis("blk:" + std::to_string(m) + ":" + std::to_string(c), v);
}

// plaintext sum_c w[c] * 1_{block c} at `like`'s level and pt scale (GPU-built)
BufPtr pt_blocks(Context& ctx, const Ciphertext& like, const std::vector<double>& w, std::size_t m, double scale) {
  LinComb lc{};
  for (std::size_t c = 0; c < w.size(); ++c) {
    if (w[c] == 0.0) continue;
    if (lc.nb == kMaxBasis) throw Error(ErrKind::capacity, "too many plaintext blocks");
    lc.basis[lc.nb] = block_basis(ctx, m, c);
    lc.w[lc.nb] = w[c];
    ++lc.nb;
  }
  return ctx.encode_lincomb(lc, like.limbs, scale);
}

// single-term MAC over a batch: out[i] = rescale(xs[i] (*) pts[i]); with `defer`
// the rescale is left to the caller (rescale_to_target after a rotate-and-sum:
// one rescale for the sum instead of one per term)
std::vector<Ciphertext> mp_many(Context& ctx, const std::vector<Ciphertext>& xs, const std::vector<BufPtr>& pts,
                                bool defer = false) {
  std::vector<std::vector<Ciphertext>> t(xs.size());
  std::vector<std::vector<BufPtr>> p(xs.size());
  for (std::size_t i = 0; i < xs.size(); ++i) {
    t[i] = {xs[i]};
    p[i] = {pts[i]};
  }
  return defer ? mac_plain_many_unrescaled(ctx, t, p) : mac_plain_many(ctx, t, p);
}

Ciphertext rescale_one(Context& ctx, const Ciphertext& c) { return rescale_to_target(ctx, {c})[0]; }

void check_stride_geometry(const Context& ctx, const Ciphertext& a, std::size_t W, std::size_t S, std::size_t W_out) {
  if (!a.valid()) throw Error(ErrKind::internal, "striding: operand is not initialized");
  if (W == 0 || S == 0 || W_out == 0) throw shape_error("striding: width, stride and output edge must be positive");
  if ((W_out - 1) * S + 1 > W)
    throw shape_error("striding: output edge " + std::to_string(W_out) + " at stride " + std::to_string(S) +
                      " overruns input edge " + std::to_string(W));
  if (W * W > (std::size_t)ctx.S())
    throw capacity_error("striding: block of edge " + std::to_string(W) + " exceeds the slot count");
}

// bias_vector (layers_conv.cpp:77-85) added as a plaintext at the operand's level
Ciphertext add_bias(Context& ctx, const Ciphertext& out, const std::vector<double>& bias, std::size_t block) {
  if (bias.size() * block > (std::size_t)ctx.S()) throw capacity_error("bias does not fit in the slot count");
  bool any = false;
  for (double b : bias) any = any || b != 0.0;
  if (!any) return add_const(ctx, out, 0.0);  // exact zero plaintext
  if (bias.size() > (std::size_t)kMaxBasis) {
    std::vector<double> v(bias.size() * block);
    for (std::size_t f = 0; f < bias.size(); ++f)
      std::fill(v.begin() + (long)(f * block), v.begin() + (long)((f + 1) * block), bias[f]);
    return add_plain(ctx, out, v.data(), v.size());
  }
  return add_plain_pt(ctx, out, pt_blocks(ctx, out, bias, block, out.scale));
}

// tap_rotations (layers_conv.cpp:102-113): one hoisted ModUp for all k^2-1 taps
std::vector<Ciphertext> tap_rotations(Context& ctx, const Ciphertext& x, std::size_t k, std::size_t W) {
  std::vector<long> ts;
  for (std::size_t i = 0; i < k; ++i)
    for (std::size_t j = 0; j < k; ++j)
      if (i * W + j != 0) ts.push_back((long)(i * W + j));
  std::vector<Ciphertext> r = rotate_hoisted(ctx, x, ts);
  std::vector<Ciphertext> taps;
  taps.reserve(k * k);
  taps.push_back(x);
  for (Ciphertext& c : r) taps.push_back(c);
  return taps;
}

using RotTerms = std::vector<std::pair<Ciphertext, long>>;

bool same_level_and_scale(const RotTerms& g) {
  for (const auto& [x, t] : g)
    if (x.limbs != g[0].first.limbs || std::fabs(x.scale / g[0].first.scale - 1.0) > 1e-9) return false;
  return true;
}

// out[r] = sum_k rot(x_rk, t_rk) for every group: rotate-and-sum key switches
// (one ModDown per output) when a group's terms share level and scale, else
// rotations + aligned additions.  Terms with t = 0 are plain additions (no
// rotation event, as in the reference's loops).
std::vector<Ciphertext> sum_rotations(Context& ctx, const std::vector<RotTerms>& groups) {
  bool uniform = true;
  for (const RotTerms& g : groups) uniform = uniform && same_level_and_scale(g);
  if (uniform) {
    std::vector<RotTerms> rot;
    std::vector<std::size_t> who;
    for (std::size_t r = 0; r < groups.size(); ++r) {
      RotTerms g;
      for (const auto& term : groups[r])
        if (term.second != 0) g.push_back(term);
      if (!g.empty()) {
        rot.push_back(std::move(g));
        who.push_back(r);
      }
    }
    const std::vector<Ciphertext> rs = rot.empty() ? std::vector<Ciphertext>{} : rotate_sum_many(ctx, rot);
    std::vector<Ciphertext> outs(groups.size());
    for (std::size_t k = 0; k < who.size(); ++k) outs[who[k]] = rs[k];
    for (std::size_t r = 0; r < groups.size(); ++r)
      for (const auto& [x, t] : groups[r])
        if (t == 0) outs[r] = outs[r].valid() ? add(ctx, outs[r], x) : x;
    return outs;
  }
  std::vector<Ciphertext> outs;
  for (const RotTerms& g : groups) {
    std::vector<Ciphertext> xs;
    std::vector<long> ts;
    Ciphertext acc;
    for (const auto& [x, t] : g) {
      if (t == 0) {
        acc = acc.valid() ? add(ctx, acc, x) : x;
        continue;
      }
      xs.push_back(x);
      ts.push_back(t);
    }
    for (const Ciphertext& r : rotate_many(ctx, xs, ts)) acc = acc.valid() ? add(ctx, acc, r) : r;
    outs.push_back(acc);
  }
  return outs;
}

// rescale_to_target(sum_rotations(groups)) with the rescale folded into the ModDowns
// when every group is uniform (rotate_sum_to_target); the same events
std::vector<Ciphertext> sum_rotations_to_target(Context& ctx, const std::vector<RotTerms>& groups) {
  bool uniform = !groups.empty();
  for (const RotTerms& g : groups) uniform = uniform && !g.empty() && same_level_and_scale(g);
  for (const RotTerms& g : groups) uniform = uniform && g[0].first.limbs == groups[0][0].first.limbs;
  if (uniform) return rotate_sum_to_target(ctx, groups, false);
  return rescale_to_target(ctx, sum_rotations(ctx, groups));
}

// out = sum_f rot(r_f, -f * block): placement rotations share one ModDown
Ciphertext place_and_sum(Context& ctx, const std::vector<Ciphertext>& r, std::size_t block) {
  // Up to 64 placements: one rotate-and-sum with one key per placement (the
  // reference's multiset).  More (FC layers of 1024 outputs) under the fast
  // schedule: baby-step giant-step, sum_G rot(sum_b rot(r_{G nb + b}, -b block),
  // -G nb block) -- about 2 sqrt(n) keys instead of n (each key is 100-200 MB at
  // N = 2^16), the same terms, one more ModDown per giant.
  constexpr std::size_t kMaxPlacementKeys = 64;
  const std::size_t n = r.size();
  if (n <= kMaxPlacementKeys || !ctx.fast_schedule()) {
    RotTerms g;
    for (std::size_t f = 0; f < n; ++f) g.push_back({r[f], -(long)(f * block)});
    return sum_rotations(ctx, {g})[0];
  }
  std::size_t nb = 1;
  while (nb * nb < n) nb <<= 1;
  std::vector<RotTerms> babies((n + nb - 1) / nb);
  for (std::size_t f = 0; f < n; ++f) babies[f / nb].push_back({r[f], -(long)((f % nb) * block)});
  const std::vector<Ciphertext> inner = sum_rotations(ctx, babies);
  RotTerms giants;
  for (std::size_t G = 0; G < inner.size(); ++G) giants.push_back({inner[G], -(long)(G * nb * block)});
  return sum_rotations(ctx, {giants})[0];
}

// sum_{i < span} rot(x, i * stride) for every x (fast schedule): a doubling
// tree (x + rot(x, p*stride) for p = 1, 2, 4, ...) plus one batched round for
// the binary tail of span -- floor(log2 span) + popcount(span) - 1 rotations
// per input instead of a span-1 chain.  Same value: rotations are linear.
std::vector<Ciphertext> strided_sum_many(Context& ctx, const std::vector<Ciphertext>& xs, std::size_t span,
                                         std::size_t stride) {
  if (span <= 1 || xs.empty()) return xs;
  const std::size_t B = xs.size();
  // Hoisted stages: sum_{i < n1 n2} rot(x, i s) = sum_{g < n2} rot(sum_{b < n1} rot(x, b s), g n1 s);
  // each stage is ONE rotate-and-sum per input (one ModUp, one ModDown, n-1 inner
  // products) instead of log2(n) full key switches.  Fan-in <= 8 per stage.
  constexpr std::size_t kFan = 8;
  std::vector<std::size_t> stages;
  for (std::size_t rest = span; rest > 1;) {
    std::size_t f = std::min(rest, kFan);
    while (rest % f != 0) --f;
    if (f == 1) break;  // no factor <= 8 (prime > 8): doubling tree below
    stages.push_back(f);
    rest /= f;
  }
  std::size_t covered = 1;
  for (std::size_t f : stages) covered *= f;
  if (covered == span) {
    std::vector<Ciphertext> cur = xs;
    std::size_t step = stride;
    for (std::size_t f : stages) {
      std::vector<RotTerms> groups(B);
      for (std::size_t i = 0; i < B; ++i)
        for (std::size_t b = 0; b < f; ++b) groups[i].push_back({cur[i], (long)(b * step)});
      cur = sum_rotations(ctx, groups);
      step *= f;
    }
    return cur;
  }
  std::vector<std::vector<Ciphertext>> pw{xs};  // pw[k] = sum_{i < 2^k} rot(x, i * stride)
  std::size_t p = 1;
  while (p * 2 <= span) {
    pw.push_back(add_many(ctx, pw.back(), rotate_many(ctx, pw.back(), std::vector<long>(B, (long)(p * stride)))));
    p *= 2;
  }
  if (p == span) return pw.back();
  std::vector<RotTerms> groups(B);
  for (std::size_t i = 0; i < B; ++i) groups[i].push_back({pw.back()[i], 0});
  std::size_t off = p;
  for (std::size_t bit = pw.size() - 1; bit-- > 0;)
    if ((span >> bit) & 1u) {
      for (std::size_t i = 0; i < B; ++i) groups[i].push_back({pw[bit][i], (long)(off * stride)});
      off += std::size_t{1} << bit;
    }
  return sum_rotations(ctx, groups);
}

// Channel accumulation chains (layers_conv.cpp:155-161), all output channels
// advanced together: C-1 batched rotations by m (reference schedule), or the
// log-depth strided sum (fast schedule).
std::vector<Ciphertext> channel_accumulate_many(Context& ctx, std::vector<Ciphertext> sums, std::size_t C,
                                                std::size_t m) {
  if (C <= 1) return sums;
  if (ctx.fast_schedule()) return strided_sum_many(ctx, sums, C, m);
  std::vector<Ciphertext> cur = sums;
  for (std::size_t c = 1; c < C; ++c) {
    cur = rotate_many(ctx, cur, std::vector<long>(cur.size(), (long)m));
    sums = add_many(ctx, sums, cur);
  }
  return sums;
}

// out = sum_f rotate(r_f, -f * block): placement rotations batched
// cur[c] = rot(x, c*m), c < C: a chain (reference) or one hoisted set (fast)
std::vector<Ciphertext> channel_cursors(Context& ctx, const Ciphertext& x, std::size_t C, std::size_t m) {
  std::vector<Ciphertext> cur{x};
  if (ctx.fast_schedule()) {
    std::vector<long> ts;
    for (std::size_t c = 1; c < C; ++c) ts.push_back((long)(c * m));
    const std::vector<Ciphertext> r = rotate_hoisted(ctx, x, ts);
    cur.insert(cur.end(), r.begin(), r.end());
    return cur;
  }
  for (std::size_t c = 1; c < C; ++c) cur.push_back(rotate(ctx, cur.back(), (long)m));
  return cur;
}

std::vector<Ciphertext> stride_many(Context& ctx, const std::vector<Ciphertext>& a, std::size_t W, std::size_t S,
                                    std::size_t W_out, int variant);

// One masked permutation of slots inside every block (nblk blocks of size blk):
// out[c blk + dest] = x[c blk + src] for every move, zero elsewhere, as
//   out = sum_g rot( sum_h M_{g,h} (*) rot(x, h), g ),   src - dest = g + h,
// M_{g,h} = 1 where the moves with that (g, h) sit after the baby rotation
// (c blk + src - h).  Babies one hoisted set, products one unrescaled MAC,
// giants one rotate-and-sum, one rescale: one plaintext level.
struct SlotMove {
  std::size_t dest, src;
  long g, h;
};

Ciphertext bsgs_moves(Context& ctx, const Ciphertext& x, const std::vector<SlotMove>& moves, std::size_t blk,
                      std::size_t nblk, const std::string& key, double value = 1.0) {
  std::vector<long> hs, gs;
  for (const SlotMove& mv : moves) {
    hs.push_back(mv.h);
    gs.push_back(mv.g);
  }
  std::sort(hs.begin(), hs.end());
  hs.erase(std::unique(hs.begin(), hs.end()), hs.end());
  std::sort(gs.begin(), gs.end());
  gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
  std::vector<long> nz;
  for (long h : hs)
    if (h != 0) nz.push_back(h);
  const std::vector<Ciphertext> r = nz.empty() ? std::vector<Ciphertext>{} : rotate_hoisted(ctx, x, nz);
  std::map<long, Ciphertext> baby;
  {
    std::size_t k = 0;
    for (long h : hs) baby[h] = h == 0 ? x : r[k++];
  }
  const long Sl = ctx.S();
  const double ps = pt_scale_for(ctx, x);
  std::map<std::pair<long, long>, std::vector<std::size_t>> cls;  // (g, h) -> move indices
  for (std::size_t i = 0; i < moves.size(); ++i) cls[{moves[i].g, moves[i].h}].push_back(i);
  std::vector<std::vector<Ciphertext>> terms(gs.size());
  std::vector<std::vector<BufPtr>> pts(gs.size());
  for (const auto& [gh, idx] : cls) {
    const std::size_t gi = (std::size_t)(std::lower_bound(gs.begin(), gs.end(), gh.first) - gs.begin());
    terms[gi].push_back(baby[gh.second]);
    pts[gi].push_back(ctx.encode_named(key + ":" + std::to_string(gh.first) + ":" + std::to_string(gh.second), [&] {
      std::vector<double> v((std::size_t)Sl, 0.0);
      for (std::size_t i : idx)
        for (std::size_t c = 0; c < nblk; ++c) {
          const long p = (((long)(c * blk + moves[i].src) - gh.second) % Sl + Sl) % Sl;
          v[(std::size_t)p] = value;
        }
      return v;
    }, x.limbs, ps));
  }
  const std::vector<Ciphertext> rows = mac_plain_many_unrescaled(ctx, terms, pts);
  RotTerms giants;
  for (std::size_t i = 0; i < rows.size(); ++i) giants.push_back({rows[i], gs[i]});
  return sum_rotations_to_target(ctx, {giants})[0];
}

// out[f mb + p] = sum_{q < nq} wfn(f, q) z[q mb + p] for f < F, with z periodic
// (period nq mb over all S slots): diagonals d = (q - f) mod nq as a baby-step
// giant-step sum, d = d1 + D d2, babies rot(z, d1 mb), giants rot(., D d2 mb);
// plaintext Q(d2, d1) holds wfn(f, (f + d) mod nq) on block f + D d2.
Ciphertext diag_mix(Context& ctx, const Ciphertext& z, std::size_t nq, std::size_t F, std::size_t mb,
                    const std::function<double(std::size_t, std::size_t)>& wfn, const std::string& key) {
  const std::size_t nblk = (std::size_t)ctx.S() / mb;
  std::size_t D = 1;
  double best = 1e300;
  for (std::size_t d = 1; d <= std::min<std::size_t>(nq, 32); ++d) {
    const double G = (double)((nq + d - 1) / d);
    const double cost = 3.3 * G + 2.4 * (double)d + ((double)d - 1.0 + G - 1.0);
    if (cost < best) {
      best = cost;
      D = d;
    }
  }
  const std::size_t G = (nq + D - 1) / D;
  std::vector<long> offs;
  for (std::size_t d1 = 1; d1 < D; ++d1) offs.push_back((long)(d1 * mb));
  std::vector<Ciphertext> baby{z};
  if (!offs.empty()) {
    const std::vector<Ciphertext> r = rotate_hoisted(ctx, z, offs);
    baby.insert(baby.end(), r.begin(), r.end());
  }
  const double ps = pt_scale_for(ctx, z);
  std::vector<std::vector<Ciphertext>> terms;
  std::vector<std::vector<BufPtr>> pts;
  std::vector<long> gsh;
  for (std::size_t d2 = 0; d2 < G; ++d2) {
    std::vector<Ciphertext> t;
    std::vector<BufPtr> p;
    for (std::size_t d1 = 0; d1 < D; ++d1) {
      const std::size_t d = d1 + D * d2;
      if (d >= nq) continue;
      bool any = false;
      for (std::size_t f = 0; f < F && !any; ++f) any = wfn(f, (f + d) % nq) != 0.0;
      if (!any) continue;
      t.push_back(baby[d1]);
      p.push_back(ctx.weight_pt(key + ":" + std::to_string(d), z.limbs, ps, [&] {
        LinComb lc{};
        for (std::size_t f = 0; f < F; ++f) {
          const double wv = wfn(f, (f + d) % nq);
          if (wv == 0.0) continue;
          lc.basis[lc.nb] = block_basis(ctx, mb, (f + D * d2) % nblk);
          lc.w[lc.nb] = wv;
          ++lc.nb;
        }
        return ctx.encode_lincomb(lc, z.limbs, ps);
      }));
    }
    if (t.empty()) continue;
    terms.push_back(std::move(t));
    pts.push_back(std::move(p));
    gsh.push_back((long)(D * d2 * mb));
  }
  const std::vector<Ciphertext> rows = mac_plain_many_unrescaled(ctx, terms, pts);
  RotTerms giants;
  for (std::size_t i = 0; i < rows.size(); ++i) giants.push_back({rows[i], gsh[i]});
  return sum_rotations_to_target(ctx, {giants})[0];
}

std::size_t best_divisor_split(std::size_t n, std::size_t giants_per_unit) {
  // babies B | n minimising (B - 1) baby key switches + (giants_per_unit n / B - 1) giant ones
  std::size_t best = 1;
  double bc = 1e300;
  for (std::size_t b = 1; b <= n; ++b) {
    if (n % b) continue;
    const double c = 3.4 * (double)(b - 1) + 4.3 * (double)(giants_per_unit * n / b - 1);
    if (c < bc) {
      bc = c;
      best = b;
    }
  }
  return best;
}

// Fast-schedule 2x2 / stride-2 convolution (ResNet-20's downsampling convs) via
// the polyphase decomposition: out[f][a][b] = sum_{c,i,j} w[f,c,i,j] x_ij[c][a][b]
// with x_ij[c][a][b] = x[c][2a+i][2b+j].  Two masked permutations turn every
// W x W channel block into its four W/2 x W/2 phase blocks (columns, then rows
// and phases), the input is replicated to fill all slots, and the conv is a 1x1
// channel mixing over the 4C phase blocks (diag_mix).  Three plaintext levels,
// as the reference's MAC + cleanup + stride; a few dozen key switches instead of
// a per-output-channel stride extraction.
bool conv2x2s2_polyphase_applies(const Context& ctx, std::size_t C, std::size_t F, std::size_t W, std::size_t k,
                                 std::size_t S) {
  const std::size_t Sl = (std::size_t)ctx.S();
  return ctx.fast_schedule() && k == 2 && S == 2 && W >= 4 && W % 2 == 0 && C * W * W <= Sl &&
         Sl % (C * W * W) == 0 && F <= (std::size_t)kMaxBasis && F * (W / 2) * (W / 2) <= Sl && 4 * C >= 2;
}

PackedTensor conv_2x2s2_polyphase(Context& ctx, const PackedTensor& x, const KernelTensor& w) {
  const std::size_t W = x.width, C = x.channels, F = w.out_channels;
  const std::size_t Wo = W / 2, m = W * W, mo = Wo * Wo;
  const std::size_t Sl = (std::size_t)ctx.S();
  const std::string geo = std::to_string(W) + ":" + std::to_string(C);
  // A: column de-interleave inside every row, s = 2b + j -> j Wo + b
  std::vector<SlotMove> mA;
  const std::size_t BA = best_divisor_split(Wo, 2);
  for (std::size_t r = 0; r < W; ++r)
    for (std::size_t j = 0; j < 2; ++j)
      for (std::size_t b = 0; b < Wo; ++b) {
        const long t = (long)b + (long)j * (1 - (long)Wo);
        const long h = (long)(b % BA);
        mA.push_back({r * W + j * Wo + b, r * W + 2 * b + j, t - h, h});
      }
  const Ciphertext za = bsgs_moves(ctx, x.data, mA, m, C, "pp-A:" + geo);
  // B: rows and phases, row 2a + i, half j -> phase block 2i + j, row a
  std::vector<SlotMove> mB;
  const std::size_t BB = best_divisor_split(Wo, 4);
  const long gstep = (long)(2 * W - Wo);
  for (std::size_t a = 0; a < Wo; ++a)
    for (std::size_t i = 0; i < 2; ++i)
      for (std::size_t j = 0; j < 2; ++j)
        for (std::size_t b = 0; b < Wo; ++b) {
          const std::size_t src = (2 * a + i) * W + j * Wo + b, dest = (2 * i + j) * mo + a * Wo + b;
          const long t = (long)src - (long)dest;
          const long h = (long)(a % BB) * gstep;
          mB.push_back({dest, src, t - h, h});
        }
  Ciphertext z = bsgs_moves(ctx, za, mB, m, C, "pp-B:" + geo);
  // periodic over all slots (period C m): phase block q = 4c + 2i + j
  for (std::size_t span = C * m; span < Sl; span *= 2) z = add(ctx, z, rotate(ctx, z, -(long)span));
  Ciphertext out = diag_mix(ctx, z, 4 * C, F, mo,
                            [&](std::size_t f, std::size_t q) { return w.at(f, q / 4, (q % 4) / 2, q % 2); },
                            weight_key("pp", w, W));
  out = add_bias(ctx, out, w.bias, mo);
  return {out, F, Wo};
}

// conv_core_generic (layers_conv.cpp:117-180)
PackedTensor conv_core_generic(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  const std::size_t W = x.width, C = x.channels;
  const std::size_t F = cfg.out_channels, k = cfg.kernel, S = cfg.stride;
  if (cfg.in_channels != C)
    throw shape_error("convolution expects " + std::to_string(cfg.in_channels) + " input channels, tensor has " +
                      std::to_string(C));
  if (w.in_channels != C || w.out_channels != F || w.kernel != k)
    throw shape_error("kernel tensor shape does not match the layer config");
  const std::size_t W_out = conv_output_width(W, k, S, 0);
  const std::size_t m = W * W;
  if (F * W_out * W_out > (std::size_t)ctx.S())
    throw capacity_error("convolution output needs " + std::to_string(F * W_out * W_out) +
                         " slots but the context provides " + std::to_string(ctx.S()));
  if (C > (std::size_t)kMaxBasis) throw capacity_error("too many input channels for one plaintext combination");
  if (conv2x2s2_polyphase_applies(ctx, C, F, W, k, S)) return conv_2x2s2_polyphase(ctx, x, w);
  const std::vector<Ciphertext> taps = tap_rotations(ctx, x.data, k, W);
  const double ps = pt_scale_for(ctx, taps[0]);
  // fused rotate-and-MAC: sum_f = sum_taps tap (*) repeated_kernel_vector(f, tap)
  std::vector<std::vector<Ciphertext>> terms(F, taps);
  std::vector<std::vector<BufPtr>> pts(F);
  const std::string wk = weight_key("g", w, W);
  for (std::size_t f = 0; f < F; ++f)
    for (std::size_t i = 0; i < k; ++i)
      for (std::size_t j = 0; j < k; ++j) {
        std::vector<double> wc(C);
        for (std::size_t c = 0; c < C; ++c) wc[c] = w.at(f, c, i, j);
        const std::string key = wk + ":" + std::to_string(f) + ":" + std::to_string(i * k + j);
        pts[f].push_back(ctx.weight_pt(key, taps[0].limbs, ps, [&] { return pt_blocks(ctx, taps[0], wc, m, ps); }));
      }
  std::vector<Ciphertext> sums = mac_plain_many(ctx, terms, pts);
  sums = channel_accumulate_many(ctx, sums, C, m);
  const BufPtr cleanup = pt_of(ctx, sums[0], plain(ctx, extraction_mask(W, C)));
  const bool strided = !(S == 1 && W_out == W);
  const bool defer = ctx.fast_schedule() && !strided;  // the placement sum rescales once
  std::vector<Ciphertext> a_star = mp_many(ctx, sums, std::vector<BufPtr>(F, cleanup), defer);
  std::vector<Ciphertext> r = strided ? stride_many(ctx, a_star, W, S, W_out, cfg.stride_variant) : a_star;
  Ciphertext out = place_and_sum(ctx, r, W_out * W_out);
  if (defer) out = rescale_one(ctx, out);
  out = add_bias(ctx, out, w.bias, W_out * W_out);
  return {out, F, W_out};
}

// conv_grouped_fallback (layers_conv.cpp:184-216)
PackedTensor conv_grouped_fallback(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w,
                                   std::size_t W_out) {
  const std::size_t W = x.width, g = x.channels;
  const std::size_t F = cfg.out_channels, k = cfg.kernel, S = cfg.stride;
  const std::size_t m = W * W;
  const std::vector<Ciphertext> taps = tap_rotations(ctx, x.data, k, W);
  const double ps = pt_scale_for(ctx, taps[0]);
  std::vector<std::vector<Ciphertext>> terms(F, taps);
  std::vector<std::vector<BufPtr>> pts(F);
  for (std::size_t f = 0; f < F; ++f)
    for (std::size_t i = 0; i < k; ++i)
      for (std::size_t j = 0; j < k; ++j) {
        std::vector<double> wc(f % g + 1, 0.0);
        wc[f % g] = w.at(f, 0, i, j);
        pts[f].push_back(pt_blocks(ctx, taps[0], wc, m, ps));
      }
  std::vector<Ciphertext> sums = mac_plain_many(ctx, terms, pts);
  // bring member c's block to the front (c > 0): batched
  std::vector<Ciphertext> xs;
  std::vector<long> ts;
  std::vector<std::size_t> who;
  for (std::size_t f = 0; f < F; ++f)
    if (f % g > 0) {
      xs.push_back(sums[f]);
      ts.push_back((long)((f % g) * m));
      who.push_back(f);
    }
  std::vector<Ciphertext> moved = rotate_many(ctx, xs, ts);
  for (std::size_t i = 0; i < who.size(); ++i) sums[who[i]] = moved[i];
  std::vector<Ciphertext> r = stride_many(ctx, sums, W, S, W_out, 0);
  Ciphertext out = place_and_sum(ctx, r, W_out * W_out);
  out = add_bias(ctx, out, w.bias, W_out * W_out);
  return {out, F, W_out};
}

}  // namespace

KernelTensor KernelTensor::from(const ConvConfig& cfg, const double* w, const double* bias) {
  KernelTensor k;
  k.out_channels = cfg.out_channels;
  k.in_channels = cfg.mode == 2 ? 1 : cfg.in_channels;
  k.kernel = cfg.kernel;
  const std::size_t nw = k.out_channels * k.in_channels * k.kernel * k.kernel;
  if (!w && nw) throw Error(ErrKind::internal, "kernel weights are null");
  k.weights.assign(w, w + nw);
  k.bias.assign(k.out_channels, 0.0);
  if (bias) std::copy(bias, bias + k.out_channels, k.bias.begin());
  return k;
}

// ------------------------------------------------------------- packing
std::vector<double> repeated_kernel_vector(const KernelTensor& w, std::size_t f, std::size_t ti, std::size_t tj,
                                           std::size_t C, std::size_t W) {
  if (f >= w.out_channels || ti >= w.kernel || tj >= w.kernel) throw shape_error("kernel tap index out of range");
  if (C > w.in_channels) throw shape_error("requested more channel blocks than the kernel has input channels");
  const std::size_t block = W * W;
  std::vector<double> out(C * block, 0.0);
  for (std::size_t c = 0; c < C; ++c) {
    const double v = w.at(f, c, ti, tj);
    std::fill(out.begin() + (long)(c * block), out.begin() + (long)((c + 1) * block), v);
  }
  return out;
}

std::vector<double> build_mask(std::size_t sp, std::size_t ep, std::size_t w, std::size_t m, std::size_t t) {
  if (ep > m) throw shape_error("mask end padding exceeds the pattern length");
  std::vector<double> pattern;
  pattern.reserve(m + w + 1);
  pattern.insert(pattern.end(), sp, 0.0);
  while (pattern.size() < m - ep) {
    pattern.insert(pattern.end(), w, 1.0);
    pattern.push_back(0.0);
  }
  if (pattern.size() > m) pattern.resize(m);
  while (pattern.size() < m) pattern.push_back(0.0);
  for (std::size_t i = m - ep; i < m; ++i) pattern[i] = 0.0;
  std::vector<double> mask;
  mask.reserve(m * t);
  for (std::size_t r = 0; r < t; ++r) mask.insert(mask.end(), pattern.begin(), pattern.end());
  return mask;
}

std::array<std::vector<double>, 9> build_all_masks(std::size_t m, std::size_t C, std::size_t W) {
  return {build_mask(W + 1, 0, W - 1, m, C), build_mask(W, 0, m, m, C),         build_mask(W, 0, W - 1, m, C),
          build_mask(1, 0, W - 1, m, C),     build_mask(0, 0, m, m, C),         build_mask(0, 1, W - 1, m, C),
          build_mask(1, W - 1, W - 1, m, C), build_mask(0, W, m, m, C),         build_mask(0, W + 1, W - 1, m, C)};
}

std::vector<double> extraction_mask(std::size_t W, std::size_t C) {
  std::vector<double> v(C * W * W, 0.0);
  std::fill(v.begin(), v.begin() + (long)(W * W), 1.0);
  return v;
}

// ------------------------------------------------------------- geometry
std::size_t conv_output_width(std::size_t W, std::size_t k, std::size_t S, std::size_t P) {
  if (k == 0 || S == 0) throw shape_error("kernel and stride must be positive");
  const std::size_t Wp = W + 2 * P;
  if (k > Wp) throw shape_error("kernel edge " + std::to_string(k) + " exceeds padded input edge " + std::to_string(Wp));
  if ((Wp - k) % S != 0)
    throw shape_error("geometry is not divisible: (" + std::to_string(Wp) + " - " + std::to_string(k) +
                      ") is not a multiple of stride " + std::to_string(S));
  return (Wp - k) / S + 1;
}

// pad_input (layers_conv.cpp:238-283)
PackedTensor pad_input(Context& ctx, const PackedTensor& x, std::size_t padding) {
  if (padding == 0) return x;
  const std::size_t W = x.width, C = x.channels, P = padding;
  const std::size_t Wp = W + 2 * P, mp_ = Wp * Wp;
  if (C * mp_ > (std::size_t)ctx.S())
    throw capacity_error("padded tensor needs " + std::to_string(C * mp_) + " slots but the context provides " +
                         std::to_string(ctx.S()));
  const std::vector<double> rowmask = range_mask(ctx, 0, W);
  // channel cursor chain, then every channel's row cursor chain advanced together
  std::vector<Ciphertext> chans{x.data};
  for (std::size_t c = 1; c < C; ++c) chans.push_back(rotate(ctx, chans.back(), (long)(W * W)));
  std::vector<std::vector<Ciphertext>> rowcur(W);
  rowcur[0] = chans;
  for (std::size_t r = 1; r < W; ++r) rowcur[r] = rotate_many(ctx, rowcur[r - 1], std::vector<long>(C, (long)W));
  const BufPtr rm = pt_of(ctx, x.data, rowmask);
  std::vector<Ciphertext> flat;
  for (std::size_t r = 0; r < W; ++r) flat.insert(flat.end(), rowcur[r].begin(), rowcur[r].end());
  std::vector<Ciphertext> rows_flat = mp_many(ctx, flat, std::vector<BufPtr>(flat.size(), rm));
  // re-space rows back to front (dependent chain per channel, channels batched)
  std::vector<Ciphertext> racc(rows_flat.begin() + (long)((W - 1) * C), rows_flat.begin() + (long)(W * C));
  for (std::size_t r = W - 1; r-- > 0;) {
    std::vector<Ciphertext> rot = rotate_many(ctx, racc, std::vector<long>(C, -(long)Wp));
    std::vector<Ciphertext> rows_r(rows_flat.begin() + (long)(r * C), rows_flat.begin() + (long)((r + 1) * C));
    racc = add_many(ctx, rot, rows_r);
  }
  Ciphertext out = place_and_sum(ctx, racc, mp_);
  out = rotate(ctx, out, -(long)(P * (Wp + 1)));
  return {out, C, Wp};
}

namespace {
// stride_extract_v1's map as one baby-step giant-step linear transform (fast
// schedule).  v1 computes out[a*W_out + b] = in[a*S*W + S*b] (a, b < W_out),
// zero elsewhere, for one level.  Write the source offset as
//   t(a, b) = g_a + h_b,  g_a = a*(S*W - W_out),  h_b = b*(S-1):
//   out = sum_a rot( sum_b M_ab (*) rot(in, h_b), g_a ),  M_ab = 1 at slot a*S*W + b.
// Baby steps are hoisted per input (one ModUp), each row is one fused MAC, the
// giant steps one batched key switch: 2(W_out-1) rotations per input instead
// of W_out^2 + W_out - 2, same level cost (one plaintext product).
std::vector<Ciphertext> stride_bsgs_many(Context& ctx, const std::vector<Ciphertext>& as, std::size_t W,
                                         std::size_t S, std::size_t W_out) {
  const std::size_t B = as.size();
  const std::size_t nb = S > 1 ? W_out : 1;  // distinct baby steps (S = 1: h_b = 0 for all b)
  std::vector<std::vector<Ciphertext>> baby(B, std::vector<Ciphertext>(nb));
  {
    std::vector<Ciphertext> xs;
    std::vector<long> ts;
    for (std::size_t i = 0; i < B; ++i) {
      baby[i][0] = as[i];
      for (std::size_t b = 1; b < nb; ++b) {
        xs.push_back(as[i]);
        ts.push_back((long)(b * (S - 1)));
      }
    }
    const std::vector<Ciphertext> r = rotate_many(ctx, xs, ts);
    std::size_t k = 0;
    for (std::size_t i = 0; i < B; ++i)
      for (std::size_t b = 1; b < nb; ++b) baby[i][b] = r[k++];
  }
  const int limbs = as[0].limbs;
  const double ps = pt_scale_for(ctx, as[0]);
  const std::size_t Sl = (std::size_t)ctx.S();
  std::vector<std::vector<Ciphertext>> terms(B * W_out);
  std::vector<std::vector<BufPtr>> pts(B * W_out);
  for (std::size_t a = 0; a < W_out; ++a) {
    std::vector<BufPtr> masks(nb);
    for (std::size_t b = 0; b < nb; ++b) {
      const std::string name = "bsgs-stride:" + std::to_string(W) + ":" + std::to_string(S) + ":" +
                               std::to_string(W_out) + ":" + std::to_string(a) + ":" + std::to_string(b);
      masks[b] = ctx.encode_named(name, [&] {
        std::vector<double> v(Sl, 0.0);
        if (S > 1) v[a * S * W + b] = 1.0;
        else std::fill(v.begin() + (long)(a * W), v.begin() + (long)(a * W + W_out), 1.0);
        return v;
      }, limbs, ps);
    }
    for (std::size_t i = 0; i < B; ++i)
      for (std::size_t b = 0; b < nb; ++b) {
        terms[i * W_out + a].push_back(baby[i][b]);
        pts[i * W_out + a].push_back(masks[b]);
      }
  }
  // rows stay unrescaled through the giant-step rotate-and-sum: one rescale per input
  const std::vector<Ciphertext> rows = mac_plain_many_unrescaled(ctx, terms, pts);
  std::vector<RotTerms> giants(B);
  for (std::size_t i = 0; i < B; ++i)
    for (std::size_t a = 0; a < W_out; ++a) giants[i].push_back({rows[i * W_out + a], (long)(a * (S * W - W_out))});
  return sum_rotations_to_target(ctx, giants);
}
}  // namespace

// stride_extract_v1 (layers_conv.cpp:289-317), batched over several inputs
std::vector<Ciphertext> stride_v1_many(Context& ctx, const std::vector<Ciphertext>& as, std::size_t W, std::size_t S,
                                       std::size_t W_out) {
  for (const Ciphertext& a : as) check_stride_geometry(ctx, a, W, S, W_out);
  if (ctx.fast_schedule()) return stride_bsgs_many(ctx, as, W, S, W_out);
  const std::size_t B = as.size();
  std::vector<Ciphertext> vcur = as;
  std::vector<std::vector<Ciphertext>> rows(W_out);
  for (std::size_t a = 0; a < W_out; ++a) {
    if (a > 0) vcur = rotate_many(ctx, vcur, std::vector<long>(B, (long)(S * W)));
    if (S == 1) {
      rows[a] = mp_many(ctx, vcur, std::vector<BufPtr>(B, pt_of(ctx, vcur[0], range_mask(ctx, 0, W_out))));
    } else {
      // gather kept columns: hcur_b = rot^b(vcur, S-1); row = sum_b hcur_b (*) e_b (fused MAC)
      std::vector<std::vector<Ciphertext>> terms(B);
      std::vector<std::vector<BufPtr>> pts(B);
      std::vector<Ciphertext> hcur = vcur;
      for (std::size_t b = 0; b < W_out; ++b) {
        if (b > 0) hcur = rotate_many(ctx, hcur, std::vector<long>(B, (long)(S - 1)));
        const BufPtr e = pt_of(ctx, vcur[0], range_mask(ctx, b, 1));
        for (std::size_t i = 0; i < B; ++i) {
          terms[i].push_back(hcur[i]);
          pts[i].push_back(e);
        }
      }
      rows[a] = mac_plain_many(ctx, terms, pts);
    }
  }
  // row placements: all (a, input) pairs in one batch
  std::vector<Ciphertext> xs;
  std::vector<long> ts;
  for (std::size_t a = 1; a < W_out; ++a)
    for (std::size_t i = 0; i < B; ++i) {
      xs.push_back(rows[a][i]);
      ts.push_back(-(long)(a * W_out));
    }
  std::vector<Ciphertext> placed = rotate_many(ctx, xs, ts);
  std::vector<Ciphertext> out = rows[0];
  for (std::size_t a = 1; a < W_out; ++a) {
    std::vector<Ciphertext> pa(placed.begin() + (long)((a - 1) * B), placed.begin() + (long)(a * B));
    out = add_many(ctx, out, pa);
  }
  return out;
}

Ciphertext stride_extract_v1(Context& ctx, const Ciphertext& a_star, std::size_t W, std::size_t S, std::size_t W_out) {
  return stride_v1_many(ctx, {a_star}, W, S, W_out)[0];
}

namespace detail {
std::vector<Ciphertext> stride_mask_compact_many(Context& ctx, const std::vector<Ciphertext>& ys, std::size_t W,
                                                 std::size_t S, std::size_t W_out, std::size_t blocks);
}

// stride_extract_v2 (layers_conv.cpp:323-334)
Ciphertext stride_extract_v2(Context& ctx, const Ciphertext& a_star, std::size_t W, std::size_t S, std::size_t W_out) {
  check_stride_geometry(ctx, a_star, W, S, W_out);
  if (!detail::masked_stride_applicable(W_out)) {
    ctx.record(4, 0, "striding: masked flavor needs a power-of-two output edge >= 2; using the extraction flavor");
    return stride_extract_v1(ctx, a_star, W, S, W_out);
  }
  return detail::stride_mask_compact(ctx, a_star, W, S, W_out, 1);
}

namespace {
std::vector<Ciphertext> stride_many(Context& ctx, const std::vector<Ciphertext>& a, std::size_t W, std::size_t S,
                                    std::size_t W_out, int variant) {
  if (variant == 1) {
    for (const Ciphertext& c : a) check_stride_geometry(ctx, c, W, S, W_out);
    if (detail::masked_stride_applicable(W_out)) return detail::stride_mask_compact_many(ctx, a, W, S, W_out, 1);
    ctx.record(4, 0, "striding: masked flavor needs a power-of-two output edge >= 2; using the extraction flavor");
  }
  return stride_v1_many(ctx, a, W, S, W_out);
}
}  // namespace

namespace detail {

bool masked_stride_applicable(std::size_t W_out) { return W_out >= 2 && is_pow2(W_out); }

int stride_mask_compact_depth(std::size_t S, std::size_t W_out) {
  return S >= 2 ? (int)log2_exact(W_out) + 1 : 2;
}

// stride_mask_compact (layers_conv.cpp:349-421), batched over several inputs
std::vector<Ciphertext> stride_mask_compact_many(Context& ctx, const std::vector<Ciphertext>& ys, std::size_t W,
                                                 std::size_t S, std::size_t W_out, std::size_t blocks) {
  for (const Ciphertext& y : ys) check_stride_geometry(ctx, y, W, S, W_out);
  if (!masked_stride_applicable(W_out))
    throw Error(ErrKind::internal, "masked compaction requires a power-of-two output edge");
  const std::size_t m = W * W;
  if (blocks * m > (std::size_t)ctx.S() || blocks * W_out * W_out > (std::size_t)ctx.S())
    throw capacity_error("masked compaction does not fit in the slot count");
  const std::size_t B = ys.size();
  std::vector<double> sel(blocks * m, 0.0);
  for (std::size_t c = 0; c < blocks; ++c)
    for (std::size_t a = 0; a < W_out; ++a)
      for (std::size_t b = 0; b < W_out; ++b) sel[c * m + (S * a) * W + S * b] = 1.0;
  std::vector<Ciphertext> cur = mp_many(ctx, ys, std::vector<BufPtr>(B, pt_of(ctx, ys[0], plain(ctx, sel))));
  if (S >= 2) {
    const std::size_t l = log2_exact(W_out);
    for (std::size_t s = 1; s < l; ++s) {
      const long amount = (long)((S - 1) << (s - 1));
      std::vector<Ciphertext> merged = add_many(ctx, cur, rotate_many(ctx, cur, std::vector<long>(B, amount)));
      std::vector<double> keep(blocks * m, 0.0);
      const std::size_t period = S << s;
      const std::size_t run = std::size_t{1} << s;
      for (std::size_t c = 0; c < blocks; ++c)
        for (std::size_t a = 0; a < W_out; ++a)
          for (std::size_t j = 0; j < W; ++j)
            if (j % period < run) keep[c * m + (S * a) * W + j] = 1.0;
      cur = mp_many(ctx, merged, std::vector<BufPtr>(B, pt_of(ctx, merged[0], plain(ctx, keep))));
    }
    cur = add_many(ctx, cur, rotate_many(ctx, cur, std::vector<long>(B, (long)((S - 1) << (l - 1)))));
  }
  // gather rows/blocks with one cumulative cursor; all masks apply to rotations
  // of the same value (one level) -> one fused MAC per input
  const std::size_t step_row = S * W - W_out;
  const std::size_t step_chan = W * W - S * W * (W_out - 1) - W_out;
  std::vector<std::vector<Ciphertext>> terms(B);
  std::vector<std::vector<BufPtr>> pts(B);
  std::vector<Ciphertext> cursor = cur;
  for (std::size_t c = 0; c < blocks; ++c)
    for (std::size_t a = 0; a < W_out; ++a) {
      if (c != 0 || a != 0) {
        const std::size_t step = (a == 0) ? step_chan : step_row;
        if (step != 0) cursor = rotate_many(ctx, cursor, std::vector<long>(B, (long)step));
      }
      const BufPtr e = pt_of(ctx, cur[0], range_mask(ctx, (c * W_out + a) * W_out, W_out));
      for (std::size_t i = 0; i < B; ++i) {
        terms[i].push_back(cursor[i]);
        pts[i].push_back(e);
      }
    }
  return mac_plain_many(ctx, terms, pts);
}

Ciphertext stride_mask_compact(Context& ctx, const Ciphertext& y, std::size_t W, std::size_t S, std::size_t W_out,
                               std::size_t blocks) {
  return stride_mask_compact_many(ctx, {y}, W, S, W_out, blocks)[0];
}

std::vector<long> block_sum_rotations(std::size_t span) {
  std::vector<long> amounts;
  std::size_t p = 1;
  while (p * 2 <= span) {
    amounts.push_back((long)p);
    p *= 2;
  }
  std::size_t off = 0;
  for (std::size_t bit = std::bit_width(span); bit-- > 0;)
    if ((span >> bit) & 1u) {
      if (off != 0) amounts.push_back((long)off);
      off += std::size_t{1} << bit;
    }
  std::sort(amounts.begin(), amounts.end());
  amounts.erase(std::unique(amounts.begin(), amounts.end()), amounts.end());
  return amounts;
}

// block_sum (layers_misc.cpp:66-95)
Ciphertext block_sum(Context& ctx, const Ciphertext& v, std::size_t span) {
  if (span == 0) throw shape_error("block sum requires a positive span");
  if (span > (std::size_t)ctx.S()) throw capacity_error("block sum span exceeds the slot count");
  if (span == 1) return v;
  std::vector<Ciphertext> sums{v};
  std::size_t p = 1;
  while (p * 2 <= span) {
    sums.push_back(add(ctx, sums.back(), rotate(ctx, sums.back(), (long)p)));
    p *= 2;
  }
  // the tail combination rotates distinct partial sums: one batch
  std::vector<Ciphertext> parts;
  std::vector<long> offs;
  std::size_t off = 0;
  for (std::size_t bit = std::bit_width(span); bit-- > 0;) {
    if (((span >> bit) & 1u) == 0) continue;
    parts.push_back(sums[bit]);
    offs.push_back((long)off);
    off += std::size_t{1} << bit;
  }
  std::vector<Ciphertext> xs(parts.begin() + 1, parts.end());
  std::vector<long> ts(offs.begin() + 1, offs.end());
  std::vector<Ciphertext> rot = rotate_many(ctx, xs, ts);
  Ciphertext acc = parts[0];
  for (const Ciphertext& r : rot) acc = add(ctx, acc, r);
  return acc;
}

}  // namespace detail

// ------------------------------------------------------------- conv paths
PackedTensor conv_generic(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  if (cfg.stride != 1 || cfg.padding != 0)
    throw shape_error("the generic convolution path handles stride 1 without padding");
  return conv_core_generic(ctx, x, cfg, w);
}

namespace {
// Fast-schedule special 3x3 convolution with C == F channels and 2 C m <= S:
// the channel mixing as a diagonal (channel-rotation) transform instead of one
// channel-sum rotate-and-sum per output channel.
//   x_rep = clean(x) + rot(clean(x), -C m)       (level 1: the block mask the
//                                                  reference spends on its cleanup)
//   out[f m + p] = sum_{d < C, tap} w(f, (f+d) mod C, tap) mask_tap[p] x_rep[(f+d) m + p + o_tap]
// With d = d1 + D d2, b(tap, d1) = rot(x_rep, o_tap + d1 m) (one hoisted set) and
//   out = sum_d2 rot( sum_{tap,d1} Q(d2,tap,d1) (*) b(tap,d1), D d2 m )      (level 2)
// where Q(d2,tap,d1) holds w(f, (f+d) mod C, tap) mask_tap at block f + D d2.
// The giants are one rotate-and-sum (one ModDown) and the products one
// unrescaled MAC + one rescale.  Same slot values and levels as the reference's
// algorithm (taps, channel sums, cleanup, placement); C/D + 9D rotations instead of
// 8 + F (2 log-stages + placement) -- e.g. 51 vs 968 inner products at C = 64.
// baby range D: minimise a key-switch cost model (ModUp 3.3, ModDown 2.4, inner
// product 1 -- measured ratios at N = 2^16): babies 9D-1 inner + ModDowns, giants
// ceil(C/D)-1 ModUps + inner, plus the replication rotation and the hoisted ModUp
std::size_t diag_baby_range(std::size_t C) {
  std::size_t best = 1;
  double best_cost = 1e300;
  for (std::size_t D = 1; D <= std::min<std::size_t>(8, C); ++D) {
    const double G = (double)((C + D - 1) / D);
    const double cost = 3.3 * (1.0 + G) + 2.4 * (1.0 + 9.0 * D) + (9.0 * D + G - 1.0);
    if (cost < best_cost) {
      best_cost = cost;
      best = D;
    }
  }
  return best;
}

bool special3x3_diag_applies(const Context& ctx, std::size_t C, std::size_t F, std::size_t m) {
  return ctx.fast_schedule() && C == F && C >= 8 && 2 * C * m <= (std::size_t)ctx.S() &&
         C <= (std::size_t)kMaxBasis;
}

PackedTensor conv_special_3x3_diag(Context& ctx, const PackedTensor& x, const KernelTensor& w) {
  const std::size_t W = x.width, C = x.channels, m = W * W;
  const std::size_t D = diag_baby_range(C);
  const std::size_t G = (C + D - 1) / D;  // giants d2 < G
  // level 1: clean the input outside its C blocks, replicate it after itself
  const BufPtr keep = pt_of(ctx, x.data, range_mask(ctx, 0, C * m));
  const Ciphertext xc = mp_many(ctx, {x.data}, {keep})[0];
  const Ciphertext xr = add(ctx, xc, rotate(ctx, xc, -(long)(C * m)));
  // babies b(tap, d1) = rot(x_rep, o_tap + d1 m): one hoisted set
  std::vector<long> offs;
  for (std::size_t d1 = 0; d1 < D; ++d1)
    for (std::size_t tap = 0; tap < 9; ++tap) {
      const long o = ((long)(tap / 3) - 1) * (long)W + ((long)(tap % 3) - 1) + (long)(d1 * m);
      if (o != 0) offs.push_back(o);
    }
  const std::vector<Ciphertext> rot = rotate_hoisted(ctx, xr, offs);
  std::vector<Ciphertext> baby;  // index d1 * 9 + tap
  {
    std::size_t k = 0;
    for (std::size_t d1 = 0; d1 < D; ++d1)
      for (std::size_t tap = 0; tap < 9; ++tap) {
        const long o = ((long)(tap / 3) - 1) * (long)W + ((long)(tap % 3) - 1) + (long)(d1 * m);
        baby.push_back(o == 0 ? xr : rot[k++]);
      }
  }
  const std::array<std::vector<double>, 9> masks = build_all_masks(m, 1, W);
  // mask_tap restricted to block blk < 2C (same cache keys as the reference-schedule path)
  std::vector<const double*> bases(9 * 2 * C);
  for (std::size_t tap = 0; tap < 9; ++tap)
    for (std::size_t blk = 0; blk < 2 * C; ++blk)
      bases[tap * 2 * C + blk] =
          ctx.basis("m3:" + std::to_string(W) + ":" + std::to_string(tap) + ":" + std::to_string(blk), [&] {
            std::vector<double> v((blk + 1) * m, 0.0);
            for (std::size_t i = 0; i < m; ++i) v[blk * m + i] = masks[tap][i];
            return v;
          });
  const double ps = pt_scale_for(ctx, xr);
  const std::string wk = weight_key("s3d", w, W);
  std::vector<std::vector<Ciphertext>> terms(G);
  std::vector<std::vector<BufPtr>> pts(G);
  for (std::size_t d2 = 0; d2 < G; ++d2)
    for (std::size_t d1 = 0; d1 < D; ++d1) {
      const std::size_t d = d1 + D * d2;
      if (d >= C) continue;
      for (std::size_t tap = 0; tap < 9; ++tap) {
        bool any = false;
        for (std::size_t f = 0; f < C && !any; ++f) any = w.at(f, (f + d) % C, tap / 3, tap % 3) != 0.0;
        if (!any) continue;
        terms[d2].push_back(baby[d1 * 9 + tap]);
        pts[d2].push_back(ctx.weight_pt(wk + ":" + std::to_string(d) + ":" + std::to_string(tap), xr.limbs, ps, [&] {
          LinComb lc{};
          for (std::size_t f = 0; f < C; ++f) {
            const double wv = w.at(f, (f + d) % C, tap / 3, tap % 3);
            if (wv == 0.0) continue;
            lc.basis[lc.nb] = bases[tap * 2 * C + f + D * d2];
            lc.w[lc.nb] = wv;
            ++lc.nb;
          }
          return ctx.encode_lincomb(lc, xr.limbs, ps);
        }));
      }
    }
  // giants: one rotate-and-sum over d2 (rows unrescaled), one rescale
  std::vector<std::vector<Ciphertext>> nz_terms;
  std::vector<std::vector<BufPtr>> nz_pts;
  std::vector<std::size_t> nz_d2;
  for (std::size_t d2 = 0; d2 < G; ++d2)
    if (!terms[d2].empty()) {
      nz_terms.push_back(terms[d2]);
      nz_pts.push_back(pts[d2]);
      nz_d2.push_back(d2);
    }
  const std::vector<Ciphertext> rows = mac_plain_many_unrescaled(ctx, nz_terms, nz_pts);
  RotTerms giants;
  for (std::size_t i = 0; i < rows.size(); ++i) giants.push_back({rows[i], (long)(D * nz_d2[i] * m)});
  Ciphertext out = sum_rotations_to_target(ctx, {giants})[0];
  out = add_bias(ctx, out, w.bias, m);
  return {out, C, W};
}
}  // namespace

// conv_special_3x3 (layers_conv.cpp:435-502)
PackedTensor conv_special_3x3(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  if (cfg.kernel != 3 || cfg.stride != 1 || cfg.padding != 1)
    throw shape_error("the shape-preserving path requires kernel 3, stride 1, padding 1");
  const std::size_t W = x.width, C = x.channels, F = cfg.out_channels;
  if (W < 2) throw shape_error("the shape-preserving path requires input edge >= 2");
  if (cfg.in_channels != C || w.in_channels != C || w.out_channels != F || w.kernel != 3)
    throw shape_error("kernel tensor shape does not match the layer config");
  const std::size_t m = W * W;
  if (F * m > (std::size_t)ctx.S()) throw capacity_error("convolution output does not fit in the slot count");
  if (C > (std::size_t)kMaxBasis) throw capacity_error("too many input channels for one plaintext combination");
  if (special3x3_diag_applies(ctx, C, F, m)) return conv_special_3x3_diag(ctx, x, w);
  const std::vector<Ciphertext> ud = rotate_hoisted(ctx, x.data, {-(long)W, (long)W});
  // the six +-1 shifts of up / x / down: one batched key switch (three hoisted pairs)
  const std::vector<Ciphertext> sh = rotate_many(ctx, {ud[0], ud[0], x.data, x.data, ud[1], ud[1]}, {-1, 1, -1, 1, -1, 1});
  const std::vector<Ciphertext> taps = {sh[0], ud[0], sh[1], sh[2], x.data, sh[3], sh[4], ud[1], sh[5]};
  const std::array<std::vector<double>, 9> masks = build_all_masks(m, C, W);
  const double ps = pt_scale_for(ctx, taps[4]);
  // basis: mask_tap restricted to block c (masks folded into the kernel companions)
  std::vector<std::vector<const double*>> bases(9, std::vector<const double*>(C));
  for (std::size_t tap = 0; tap < 9; ++tap)
    for (std::size_t c = 0; c < C; ++c) {
      std::vector<double> v((c + 1) * m, 0.0);
      for (std::size_t i = 0; i < m; ++i) v[c * m + i] = masks[tap][c * m + i];
      bases[tap][c] = ctx.basis("m3:" + std::to_string(W) + ":" + std::to_string(tap) + ":" + std::to_string(c), v);
    }
  std::vector<std::vector<Ciphertext>> terms(F, taps);
  std::vector<std::vector<BufPtr>> pts(F);
  const std::string wk = weight_key("s3", w, W);
  for (std::size_t f = 0; f < F; ++f)
    for (std::size_t tap = 0; tap < 9; ++tap) {
      LinComb lc{};
      for (std::size_t c = 0; c < C; ++c) {
        const double wv = w.at(f, c, tap / 3, tap % 3);
        if (wv == 0.0) continue;
        lc.basis[lc.nb] = bases[tap][c];
        lc.w[lc.nb] = wv;
        ++lc.nb;
      }
      pts[f].push_back(ctx.weight_pt(wk + ":" + std::to_string(f) + ":" + std::to_string(tap), taps[4].limbs, ps,
                                     [&] { return ctx.encode_lincomb(lc, taps[4].limbs, ps); }));
    }
  std::vector<Ciphertext> sums = mac_plain_many(ctx, terms, pts);
  sums = channel_accumulate_many(ctx, sums, C, m);
  const BufPtr cleanup = pt_of(ctx, sums[0], plain(ctx, extraction_mask(W, C)));
  const bool defer = ctx.fast_schedule();
  std::vector<Ciphertext> cleaned = mp_many(ctx, sums, std::vector<BufPtr>(F, cleanup), defer);
  Ciphertext out = place_and_sum(ctx, cleaned, m);
  if (defer) out = rescale_one(ctx, out);
  out = add_bias(ctx, out, w.bias, m);
  return {out, F, W};
}

// conv_grouped_stride (layers_conv.cpp:504-575)
PackedTensor conv_grouped_stride(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  const std::size_t g = cfg.in_channels, F = cfg.out_channels;
  if (g < 2) throw shape_error("grouped convolution with one group degenerates to the generic path");
  if (x.channels != g) throw shape_error("grouped convolution input channel mismatch");
  if (F % g != 0) throw shape_error("grouped convolution requires out_channels divisible by groups");
  if (w.out_channels != F || w.in_channels != 1 || w.kernel != cfg.kernel)
    throw shape_error("grouped kernel tensor must be (out_channels, 1, k, k) matching the layer config");
  const PackedTensor xp = cfg.padding > 0 ? pad_input(ctx, x, cfg.padding) : x;
  const std::size_t W = xp.width, k = cfg.kernel, S = cfg.stride;
  const std::size_t W_out = conv_output_width(W, k, S, 0);
  if (F * W_out * W_out > (std::size_t)ctx.S()) throw capacity_error("convolution output does not fit in the slot count");
  if (!detail::masked_stride_applicable(W_out)) {
    ctx.record(4, 0, "grouped striding needs a power-of-two output edge >= 2; using per-member extraction");
    return conv_grouped_fallback(ctx, xp, cfg, w, W_out);
  }
  const std::size_t m = W * W;
  const std::vector<Ciphertext> taps = tap_rotations(ctx, xp.data, k, W);
  const double ps = pt_scale_for(ctx, taps[0]);
  const std::size_t groups = F / g;
  // joint_u = sum_{c, tap} tap (*) member_kernel_vector(u*g + c, tap, c): one MAC per group
  std::vector<std::vector<Ciphertext>> terms(groups);
  std::vector<std::vector<BufPtr>> pts(groups);
  for (std::size_t u = 0; u < groups; ++u)
    for (std::size_t c = 0; c < g; ++c)
      for (std::size_t i = 0; i < k; ++i)
        for (std::size_t j = 0; j < k; ++j) {
          std::vector<double> wc(c + 1, 0.0);
          wc[c] = w.at(u * g + c, 0, i, j);
          terms[u].push_back(taps[i * k + j]);
          pts[u].push_back(pt_blocks(ctx, taps[0], wc, m, ps));
        }
  std::vector<Ciphertext> joint = mac_plain_many(ctx, terms, pts);
  std::vector<Ciphertext> packed = detail::stride_mask_compact_many(ctx, joint, W, S, W_out, g);
  Ciphertext out = packed[groups - 1];
  for (std::size_t u = groups - 1; u-- > 0;) out = add(ctx, rotate(ctx, out, -(long)(g * W_out * W_out)), packed[u]);
  out = add_bias(ctx, out, w.bias, W_out * W_out);
  return {out, F, W_out};
}

// convolution dispatcher (layers_conv.cpp:577-594)
PackedTensor convolution(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  if (cfg.mode == 1) return conv_special_3x3(ctx, x, cfg, w);
  if (cfg.mode == 2 && cfg.in_channels != 1) return conv_grouped_stride(ctx, x, cfg, w);
  const PackedTensor xp = cfg.padding > 0 ? pad_input(ctx, x, cfg.padding) : x;
  ConvConfig inner = cfg;
  inner.padding = 0;
  return conv_core_generic(ctx, xp, inner, w);
}

// ------------------------------------------------------------- pooling
// avg_pool (layers_misc.cpp:99-144)
PackedTensor avg_pool(Context& ctx, const PackedTensor& x, std::size_t k, std::size_t S, int variant) {
  const std::size_t W = x.width, C = x.channels;
  const std::size_t W_out = conv_output_width(W, k, S, 0);
  const std::size_t m = W * W;
  if (C * W_out * W_out > (std::size_t)ctx.S()) throw capacity_error("pooling output does not fit in the slot count");
  std::vector<long> ts;
  for (std::size_t i = 0; i < k; ++i)
    for (std::size_t j = 0; j < k; ++j)
      if (i != 0 || j != 0) ts.push_back((long)(i * W + j));
  Ciphertext T = x.data;
  if (!ts.empty()) {  // hoisted window taps summed under one ModDown
    RotTerms g{{x.data, 0}};
    for (long t : ts) g.push_back({x.data, t});
    T = sum_rotations(ctx, {g})[0];
  }
  const Ciphertext T2 = mp(ctx, T, range_mask(ctx, 0, C * m, 1.0 / (double)(k * k)));
  if (S == 1 && W_out == W) return {T2, C, W};
  std::vector<Ciphertext> chans = channel_cursors(ctx, T2, C, m);
  std::vector<Ciphertext> r = stride_many(ctx, chans, W, S, W_out, variant);
  Ciphertext out = place_and_sum(ctx, r, W_out * W_out);
  return {out, C, W_out};
}

namespace {
// merge_channel_slots (layers_misc.cpp:31-37): Horner chain by -1 (reference
// schedule) or sum_c rot(piece_c, -c) as one batched key switch (fast)
// Fast-schedule pooled-channel gather: out[c] = value * sums[c m] for c < C (zero
// elsewhere), the head mask, channel cursors and -c placements of the reference
// (layers_misc.cpp:159-165) as ONE masked slot permutation: shift c (m - 1)
// split as baby (c mod B)(m - 1) + giant (c - c mod B)(m - 1) -- B - 1 hoisted
// babies and ceil(C / B) - 1 giants instead of 2 (C - 1) rotations; one level.
Ciphertext gather_block_heads(Context& ctx, const Ciphertext& sums, std::size_t C, std::size_t m, double value) {
  std::size_t B = 1;
  while (B * B < C) ++B;
  std::vector<SlotMove> moves;
  for (std::size_t c = 0; c < C; ++c) {
    const long t = (long)(c * (m - 1));
    const long h = (long)((c % B) * (m - 1));
    moves.push_back({c, c * m, t - h, h});
  }
  char vk[32];
  std::snprintf(vk, sizeof vk, "%.17g", value);
  return bsgs_moves(ctx, sums, moves, (std::size_t)ctx.S(), 1,
                    "heads:" + std::to_string(C) + ":" + std::to_string(m) + ":" + vk, value);
}

Ciphertext merge_channel_slots(Context& ctx, const std::vector<Ciphertext>& pieces) {
  if (ctx.fast_schedule()) return place_and_sum(ctx, pieces, 1);
  Ciphertext out = pieces.back();
  for (std::size_t c = pieces.size() - 1; c-- > 0;) out = add(ctx, rotate(ctx, out, -1), pieces[c]);
  return out;
}
}  // namespace

// global_avg_pool (layers_misc.cpp:146-166)
Ciphertext global_avg_pool(Context& ctx, const PackedTensor& x) {
  const std::size_t W = x.width, C = x.channels, m = W * W;
  const Ciphertext sums = detail::block_sum(ctx, x.data, m);
  if (ctx.fast_schedule() && C > 1) return gather_block_heads(ctx, sums, C, m, 1.0 / (double)m);
  const std::vector<Ciphertext> cur = channel_cursors(ctx, sums, C, m);
  const BufPtr head = pt_of(ctx, sums, range_mask(ctx, 0, 1, 1.0 / (double)m));
  const bool defer = ctx.fast_schedule();
  const Ciphertext out = merge_channel_slots(ctx, mp_many(ctx, cur, std::vector<BufPtr>(C, head), defer));
  return defer ? rescale_one(ctx, out) : out;
}

// whole_channel_pool (layers_misc.cpp:168-195)
Ciphertext whole_channel_pool(Context& ctx, const PackedTensor& x, std::size_t k) {
  if (k != x.width) throw shape_error("whole-channel pooling requires the window to span the full channel edge");
  const std::size_t W = x.width, C = x.channels, m = W * W;
  const Ciphertext v = mp(ctx, x.data, range_mask(ctx, 0, C * m, 1.0 / (double)(k * k)));
  const Ciphertext sums = detail::block_sum(ctx, v, m);
  if (ctx.fast_schedule() && C > 1) return gather_block_heads(ctx, sums, C, m, 1.0);
  const std::vector<Ciphertext> cur = channel_cursors(ctx, sums, C, m);
  const BufPtr head = pt_of(ctx, sums, range_mask(ctx, 0, 1));
  const bool defer = ctx.fast_schedule();
  const Ciphertext out = merge_channel_slots(ctx, mp_many(ctx, cur, std::vector<BufPtr>(C, head), defer));
  return defer ? rescale_one(ctx, out) : out;
}

// ------------------------------------------------------------- FC
// fully_connected (layers_misc.cpp:197-255): neurons batched
namespace {
// y = W x (m x n, row-major) as a baby-step giant-step sum of GENERALISED diagonals (fast
// schedule): y_i = sum_{k < n + m - 1} diag_k[i] x[i + k - (m - 1)] with diag_k[i] =
// W[i][i + k - (m - 1)] where i < m and the column lies in [0, n), 0 elsewhere.  The zero
// entries make every product ignore the slots of x outside [0, n) (post-ReLU p(0), say)
// and leave [m, S) exactly zero -- the reference FC's output layout -- in ONE level.
// Babies rot(x, k0 + b) (one hoisted set), giants g: rot(sum_b diag'_{g n1 + b} (*) baby_b,
// g n1) with the diagonals pre-rotated by -g n1, one fused MAC per giant, one
// rotate-and-sum, one rescale.  n1 = 32 (the MAC's terms per output): a 1024 x 1024 layer
// is 32 + 64 key switches and 2047 plaintext products instead of 1024 neurons x log2(1024)
// folds.  The diagonals are resident weight plaintexts.
Ciphertext fc_diagonal(Context& ctx, const Ciphertext& x, std::size_t n, std::size_t m, const double* w) {
  const long S = ctx.S();
  const std::size_t D = n + m - 1;
  const long k0 = -(long)(m - 1);
  const std::size_t n1 = std::min<std::size_t>((std::size_t)kMacMaxTerms, D);
  const std::size_t G = (D + n1 - 1) / n1;
  auto norm = [S](long t) {
    long r = t % S;
    return r < 0 ? r + S : r;
  };
  std::vector<long> offs;
  for (std::size_t b = 0; b < n1; ++b)
    if (norm(k0 + (long)b) != 0) offs.push_back(k0 + (long)b);
  const std::vector<Ciphertext> rot = rotate_hoisted(ctx, x, offs);
  std::vector<Ciphertext> baby;
  {
    std::size_t r = 0;
    for (std::size_t b = 0; b < n1; ++b) baby.push_back(norm(k0 + (long)b) == 0 ? x : rot[r++]);
  }
  // 128-bit content key of the weight matrix (as weight_key for kernel tensors)
  u64 h = 1469598103934665603ULL, g2 = 0x9E3779B97F4A7C15ULL;
  for (std::size_t i = 0; i < m * n; ++i) {
    u64 bits;
    std::memcpy(&bits, w + i, 8);
    h = (h ^ bits) * 1099511628211ULL;
    g2 = mix64(g2 ^ (bits + 0x632BE59BD9B4E019ULL));
  }
  const std::string wk = "fcd:" + std::to_string(h) + ":" + std::to_string(g2) + ":" + std::to_string(m) + "x" +
                         std::to_string(n);
  const double ps = pt_scale_for(ctx, x);
  std::vector<std::vector<Ciphertext>> terms;
  std::vector<std::vector<BufPtr>> pts;
  std::vector<long> gofs;
  for (std::size_t g = 0; g < G; ++g) {
    std::vector<Ciphertext> tg;
    std::vector<BufPtr> pg;
    for (std::size_t b = 0; b < n1 && g * n1 + b < D; ++b) {
      const std::size_t k = g * n1 + b;
      tg.push_back(baby[b]);
      pg.push_back(ctx.weight_pt(wk + ":" + std::to_string(k), x.limbs, ps, [&] {
        std::vector<double> v((std::size_t)S, 0.0);
        for (std::size_t i = 0; i < m; ++i) {
          const long c = (long)i + k0 + (long)k;
          if (c >= 0 && c < (long)n) v[(std::size_t)norm((long)i + (long)(g * n1))] = w[i * n + (std::size_t)c];
        }
        return ctx.encode(v.data(), v.size(), x.limbs, ps);
      }));
    }
    terms.push_back(tg);
    pts.push_back(pg);
    gofs.push_back((long)(g * n1));
  }
  const std::vector<Ciphertext> rows = mac_plain_many_unrescaled(ctx, terms, pts);
  RotTerms giants;
  for (std::size_t g = 0; g < rows.size(); ++g) giants.push_back({rows[g], gofs[g]});
  return sum_rotations_to_target(ctx, {giants})[0];
}
}  // namespace

Ciphertext fully_connected(Context& ctx, const Ciphertext& x, std::size_t n, std::size_t m, std::size_t B,
                           const double* w, const double* bias) {
  if (n == 0 || m == 0) throw shape_error("fully-connected layer needs positive input/output sizes");
  if (n > (std::size_t)ctx.S() || m > (std::size_t)ctx.S())
    throw capacity_error("fully-connected layer does not fit in the slot count");
  if (B == 0) throw shape_error("merge budget must be >= 1");
  if (ctx.fast_schedule() && m >= 64 && n + m - 1 <= (std::size_t)ctx.S() && x.limbs >= 3) {
    Ciphertext y = fc_diagonal(ctx, x, n, m, w);
    // the reference's FC consumes two levels (row product + head mask); the diagonal
    // form needs one, the second is an exact level drop so the ledger is unchanged
    y = level_down(ctx, y, y.limbs - 1);
    std::vector<double> b(m, 0.0);
    if (bias) std::copy(bias, bias + m, b.begin());
    return add_plain(ctx, y, b.data(), b.size());
  }
  const std::size_t p2 = std::bit_ceil(n);
  std::vector<BufPtr> rows;
  rows.reserve(m);
  for (std::size_t i = 0; i < m; ++i) rows.push_back(pt_of(ctx, x, plain(ctx, std::vector<double>(w + i * n, w + (i + 1) * n))));
  std::vector<Ciphertext> y = mp_many(ctx, std::vector<Ciphertext>(m, x), rows);
  if (ctx.fast_schedule()) {
    y = strided_sum_many(ctx, y, p2, 1);  // hoisted rotate-and-sum stages
  } else {
    for (std::size_t off = 1; off < p2; off <<= 1)
      y = add_many(ctx, y, rotate_many(ctx, y, std::vector<long>(m, (long)off)));
  }
  const BufPtr head = pt_of(ctx, y[0], range_mask(ctx, 0, 1));
  const bool defer = ctx.fast_schedule();
  std::vector<Ciphertext> neurons = mp_many(ctx, y, std::vector<BufPtr>(m, head), defer);
  const std::size_t r = (m <= B + 1) ? m : B;
  const std::size_t T = (m + r - 1) / r;
  // in-group placements are independent: one rotate-and-sum batch
  std::vector<RotTerms> gterms(T);
  for (std::size_t t = 0; t < T; ++t) {
    const std::size_t sz = std::min(r, m - t * r);
    for (std::size_t u = 0; u < sz; ++u) gterms[t].push_back({neurons[t * r + u], -(long)u});
  }
  std::vector<Ciphertext> groups = sum_rotations(ctx, gterms);
  Ciphertext out = groups[T - 1];
  if (ctx.fast_schedule()) out = place_and_sum(ctx, groups, r);
  else
    for (std::size_t t = T - 1; t-- > 0;) out = add(ctx, rotate(ctx, out, -(long)r), groups[t]);
  if (defer) out = rescale_one(ctx, out);
  std::vector<double> b(m, 0.0);
  if (bias) std::copy(bias, bias + m, b.begin());
  return add_plain(ctx, out, b.data(), b.size());
}

// ------------------------------------------------------------- ReLU
std::vector<double> cheb_coefficients(const std::function<double(double)>& f, int degree) {
  if (degree < 0) throw shape_error("polynomial degree must be non-negative");
  const double pi = 3.14159265358979323846;
  const int n = degree + 1;
  std::vector<double> nodes(n), fx(n), coeffs(n, 0.0);
  for (int j = 0; j < n; ++j) nodes[j] = std::cos(pi * (2.0 * j + 1.0) / (2.0 * n));
  for (int j = 0; j < n; ++j) fx[j] = f(nodes[j]);
  for (int d = 0; d < n; ++d) {
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc += fx[j] * std::cos(d * pi * (2.0 * j + 1.0) / (2.0 * n));
    coeffs[d] = (d == 0 ? 1.0 : 2.0) * acc / n;
  }
  return coeffs;
}

int cheb_eval_depth(int degree) {
  if (degree <= 0) return 0;
  if (degree == 1) return 1;
  return (int)std::bit_width((unsigned)(degree - 1)) + 1;
}

// cheb_eval (chebyshev.cpp:62-104).  T_d = 2 T_a T_b - T_{a-b} with a = ceil(d/2),
// b = floor(d/2); every d in (2^{g-1}, 2^g] depends only on smaller degrees, so
// each band is one batched relinearisation.  Event order matches the reference.
Ciphertext cheb_eval(Context& ctx, const Ciphertext& x, const std::vector<double>& coeffs) {
  return cheb_eval_many(ctx, {x}, coeffs)[0];
}

namespace {
// ---- Paterson-Stockmeyer in the Chebyshev basis (fast schedule).
// Babies T_1..T_k (k = 2^lk), giants G_j = T_{k 2^j}; p is split recursively by
// Chebyshev division p = q T_g + r (T_i = 2 T_g T_{i-g} - T_{2g-i}, g < i <= 2g)
// down to leaves of degree < k, each a constant linear combination of babies
// (one rescale).  Degree 59 takes 16 ciphertext products instead of the
// T_d tree's 58, at the same depth.
struct PsNode {
  std::vector<double> c;  // leaf coefficients (degree < k) when leaf
  int j = 0;              // giant index of the split (G_{j-1} = T_{k 2^{j-1}})
  bool leaf = true;
  std::unique_ptr<PsNode> q, r;
};

void cheb_divide(const std::vector<double>& c, int g, std::vector<double>& q, std::vector<double>& r) {
  const int n = (int)c.size();
  r.assign(c.begin(), c.begin() + std::min(n, g));
  q.assign(std::max(0, n - g), 0.0);
  for (int i = g; i < n; ++i) {
    if (i == g) {
      q[0] += c[i];
      continue;
    }
    q[i - g] += 2.0 * c[i];
    r[2 * g - i] -= c[i];
  }
}

std::unique_ptr<PsNode> ps_build(const std::vector<double>& c, int j, int k) {
  auto nd = std::make_unique<PsNode>();
  const int g = j > 0 ? k << (j - 1) : 0;
  if (j == 0 || (int)c.size() <= g) {
    if (j == 0) {
      nd->c = c;
      return nd;
    }
    return ps_build(c, j - 1, k);
  }
  std::vector<double> q, r;
  cheb_divide(c, g, q, r);
  nd->leaf = false;
  nd->j = j;
  nd->q = ps_build(q, j - 1, k);
  nd->r = ps_build(r, j - 1, k);
  return nd;
}

bool nonconst(const std::vector<double>& c) {
  for (std::size_t i = 1; i < c.size(); ++i)
    if (c[i] != 0.0) return true;
  return false;
}

int tdepth(int d) { return d <= 1 ? 0 : (int)std::bit_width((unsigned)(d - 1)); }

// (depth, ciphertext products, max |coefficient|) of a tree; depth -1 = constant
struct PsCost {
  int depth = -1, mults = 0;
  double cmax = 0.0;
};
PsCost ps_cost(const PsNode& nd, int lk) {
  PsCost out;
  if (nd.leaf) {
    for (std::size_t i = 0; i < nd.c.size(); ++i) {
      out.cmax = std::max(out.cmax, std::fabs(nd.c[i]));
      if (i >= 1 && nd.c[i] != 0.0) out.depth = std::max(out.depth, tdepth((int)i) + 1);
    }
    return out;
  }
  const PsCost q = ps_cost(*nd.q, lk), r = ps_cost(*nd.r, lk);
  const int gd = lk + nd.j - 1;  // depth of G_{j-1}
  out.mults = q.mults + r.mults + (q.depth >= 0 ? 1 : 0);
  out.depth = std::max(std::max(q.depth, gd) + 1, r.depth);
  out.cmax = std::max(q.cmax, r.cmax);
  return out;
}

struct PsVal {
  Ciphertext ct;   // invalid: constant
  double c = 0.0;  // constant part when ct is invalid
};

// Evaluate the tree for every input so that each node lands EXACTLY on (tl[i]
// limbs, scale ts[i]) -- no level alignment anywhere in the tree.  A split node
// p = q G + r multiplies q, evaluated at (tl + 1, ts q_tl / scale(G)), by G
// viewed at tl + 1 limbs (a zero-copy limb drop keeps G's scale), so the fused
// relinearise-and-rescale lands on ts; r is evaluated at (tl, ts) directly and
// the leaves are constant linear combinations of babies with per-term
// constants c_d ts' q / scale(T_d) (one rescale).  Feasible whenever the node's
// PS depth fits: the target level of a node of depth d is at most
// level(x) - d (ps_cost).  T[i][d] babies, G[i][j] giants.
//
// Targets are assigned top-down first; the products then run bottom-up, ALL
// nodes of one height (and every input) in one batched relinearisation, so the
// serial key-switch chain is the tree's height, not its node count.
struct PsTask {
  const PsNode* nd = nullptr;
  std::vector<int> tl;
  std::vector<double> ts;
  std::vector<Ciphertext> gv;  // G_{j-1} viewed at tl + 1 limbs
  int height = 0;
  int q = -1, r = -1;          // child tasks
  std::vector<PsVal> val;
};

int ps_plan(Context& ctx, const PsNode& nd, std::vector<std::vector<Ciphertext>>& G, const std::vector<int>& tl,
            const std::vector<double>& ts, std::vector<PsTask>& tasks) {
  const int id = (int)tasks.size();
  tasks.emplace_back();
  tasks[id].nd = &nd;
  tasks[id].tl = tl;
  tasks[id].ts = ts;
  if (nd.leaf) return id;
  const HostTables& h = ctx.host();
  const std::size_t B = tl.size();
  std::vector<int> tq(B);
  std::vector<double> sq(B);
  std::vector<Ciphertext> gv(B);
  for (std::size_t i = 0; i < B; ++i) {
    gv[i] = G[i][nd.j - 1];
    if (gv[i].limbs < tl[i] + 1) throw Error(ErrKind::internal, "Paterson-Stockmeyer: giant below its node");
    gv[i].limbs = tl[i] + 1;  // zero-copy limb drop, scale kept
    tq[i] = tl[i] + 1;
    sq[i] = ts[i] * (double)h.q[tl[i]] / gv[i].scale;
  }
  const int q = ps_plan(ctx, *nd.q, G, tq, sq, tasks);
  const int r = ps_plan(ctx, *nd.r, G, tl, ts, tasks);
  tasks[id].gv = std::move(gv);
  tasks[id].q = q;
  tasks[id].r = r;
  tasks[id].height = std::max(tasks[q].height, tasks[r].height) + 1;
  return id;
}

std::vector<PsVal> ps_eval(Context& ctx, const PsNode& root, std::vector<std::vector<Ciphertext>>& T,
                           std::vector<std::vector<Ciphertext>>& G, const std::vector<int>& tl,
                           const std::vector<double>& ts) {
  const std::size_t B = T.size();
  std::vector<PsTask> tasks;
  ps_plan(ctx, root, G, tl, ts, tasks);
  int H = 0;
  // every leaf (constant linear combination of babies) at once: one rescale per level
  std::vector<LincombItem> items;
  std::vector<std::pair<std::size_t, std::size_t>> where;  // (task, input)
  for (std::size_t k = 0; k < tasks.size(); ++k) {
    PsTask& t = tasks[k];
    H = std::max(H, t.height);
    if (!t.nd->leaf) continue;
    t.val.resize(B);
    for (std::size_t i = 0; i < B; ++i) {
      if (!nonconst(t.nd->c)) {
        t.val[i].c = t.nd->c.empty() ? 0.0 : t.nd->c[0];
        continue;
      }
      LincombItem it;
      for (std::size_t d = 1; d < t.nd->c.size(); ++d)
        if (t.nd->c[d] != 0.0) {
          it.xs.push_back(T[i][d]);
          it.cs.push_back(t.nd->c[d]);
        }
      it.c0 = t.nd->c[0];
      it.out_limbs = t.tl[i];
      it.out_scale = t.ts[i];
      items.push_back(std::move(it));
      where.push_back({k, i});
    }
  }
  const std::vector<Ciphertext> leaves = lincomb_const_to_many(ctx, items);
  for (std::size_t m = 0; m < leaves.size(); ++m) tasks[where[m].first].val[where[m].second].ct = leaves[m];
  for (int ht = 1; ht <= H; ++ht) {
    std::vector<Ciphertext> as, bs;
    for (const PsTask& t : tasks)
      if (t.height == ht)
        for (std::size_t i = 0; i < B; ++i)
          if (tasks[t.q].val[i].ct.valid()) {
            as.push_back(tasks[t.q].val[i].ct);
            bs.push_back(t.gv[i]);
          }
    const std::vector<Ciphertext> prods = mult_cipher_many(ctx, as, bs);
    std::size_t k = 0;
    for (PsTask& t : tasks) {
      if (t.height != ht) continue;
      const int j = t.nd->j;
      t.val.resize(B);
      for (std::size_t i = 0; i < B; ++i) {
        const PsVal& q = tasks[t.q].val[i];
        const PsVal& r = tasks[t.r].val[i];
        Ciphertext p = q.ct.valid() ? prods[k++] : lincomb_const_to(ctx, {G[i][j - 1]}, {q.c}, 0.0, t.tl[i], t.ts[i]);
        p.scale = t.ts[i];  // exact up to floating-point rounding of the scale bookkeeping
        t.val[i].ct = r.ct.valid() ? add(ctx, p, r.ct) : add_const(ctx, p, r.c);
      }
    }
  }
  return tasks[0].val;
}
}  // namespace

// Paterson-Stockmeyer evaluation of sum_d c_d T_d(x) for every input; empty
// result when no baby size meets the T_d tree's depth (the caller falls back).
// The output is brought to exactly the tree's level (input level - depth).
std::vector<Ciphertext> cheb_eval_ps_many(Context& ctx, const std::vector<Ciphertext>& xs,
                                          const std::vector<double>& coeffs) {
  const int D = (int)coeffs.size() - 1;
  if (D < 2 || xs.empty()) return {};
  const int want = cheb_eval_depth(D);
  for (const Ciphertext& x : xs)
    if (x.level() < want)  // the T_d tree would exhaust the chain mid-way (chebyshev.cpp:62-104)
      throw Error(ErrKind::depth_exhausted, "cheb_eval: degree " + std::to_string(D) + " needs " +
                                                std::to_string(want) + " levels, operand is at level " +
                                                std::to_string(x.level()));
  int best_lk = -1, best_m = 0, best_mults = 1 << 30;
  std::unique_ptr<PsNode> best;
  for (int lk = 1; lk <= 5; ++lk) {
    const int k = 1 << lk;
    int m = 0;
    while ((k << m) < D + 1) ++m;
    std::unique_ptr<PsNode> root = ps_build(coeffs, m, k);
    const PsCost c = ps_cost(*root, lk);
    const int mults = c.mults + (std::min(k, D) - 1) + std::max(0, m - 1);
    if (c.depth > want || c.cmax > 1e12) continue;
    if (mults < best_mults) {
      best_mults = mults;
      best_lk = lk;
      best_m = m;
      best = std::move(root);
    }
  }
  if (best_lk < 0) return {};
  const int k = 1 << best_lk;
  const std::size_t B = xs.size();
  const int nb = std::min(k, D);  // babies T_1..T_nb
  std::vector<std::vector<Ciphertext>> T(B, std::vector<Ciphertext>(nb + 1));
  for (std::size_t i = 0; i < B; ++i) T[i][1] = xs[i];
  std::map<std::tuple<std::size_t, int, int>, Ciphertext> lowered;
  auto at = [&](std::size_t i, int d, int limbs) -> Ciphertext {
    if (T[i][d].limbs <= limbs) return T[i][d];
    auto key = std::make_tuple(i, d, limbs);
    auto it = lowered.find(key);
    if (it != lowered.end()) return it->second;
    return lowered[key] = level_down(ctx, T[i][d], limbs);
  };
  for (int lo = 2; lo <= nb; lo = lo * 2 - 1) {
    const int hi = std::min(nb, 2 * lo - 2 > lo ? 2 * lo - 2 : lo);
    // T_d = 2 T_a T_b - T_{a-b}: T_1 (odd d) is subtracted inside the product's
    // relinearise-and-rescale (mult_cipher_cheb_many), T_0 = 1 (even d) afterwards
    std::vector<Ciphertext> as, bs, subs;
    for (std::size_t i = 0; i < B; ++i)
      for (int d = lo; d <= hi; ++d) {
        const int a = (d + 1) / 2, b = d / 2;
        const int l = std::min(T[i][a].limbs, T[i][b].limbs);
        as.push_back(at(i, a, l));
        bs.push_back(at(i, b, l));
        subs.push_back(d % 2 == 0 ? Ciphertext{} : T[i][1]);
      }
    std::vector<Ciphertext> prods = mult_cipher_cheb_many(ctx, as, bs, subs);
    std::size_t j = 0;
    for (std::size_t i = 0; i < B; ++i)
      for (int d = lo; d <= hi; ++d, ++j) T[i][d] = (d % 2 == 0) ? add_const(ctx, prods[j], -1.0) : prods[j];
    if (hi == nb) break;
  }
  // giants G_0 = T_k, G_j = 2 G_{j-1}^2 - 1
  std::vector<std::vector<Ciphertext>> G(B);
  if (best_m >= 1)
    for (std::size_t i = 0; i < B; ++i) G[i].push_back(T[i][k]);
  for (int j = 1; j < best_m; ++j) {
    std::vector<Ciphertext> g;
    for (std::size_t i = 0; i < B; ++i) g.push_back(G[i].back());
    std::vector<Ciphertext> dbl = mult_cipher_cheb_many(ctx, g, g, std::vector<Ciphertext>(g.size()));
    for (std::size_t i = 0; i < B; ++i) G[i].push_back(add_const(ctx, dbl[i], -1.0));
  }
  std::vector<int> tl(B);
  std::vector<double> ts(B);
  for (std::size_t i = 0; i < B; ++i) {
    tl[i] = xs[i].limbs - want;
    ts[i] = ctx.host().T[tl[i] - 1];
  }
  const std::vector<PsVal> v = ps_eval(ctx, *best, T, G, tl, ts);
  std::vector<Ciphertext> out(B);
  for (std::size_t i = 0; i < B; ++i) {
    out[i] = v[i].ct.valid() ? v[i].ct : add_const(ctx, sub(ctx, xs[i], xs[i]), v[i].c);
    if (out[i].limbs > tl[i]) out[i] = level_down(ctx, out[i], tl[i]);
  }
  return out;
}

// Several inputs through the same series: every band's products for all
// inputs go through one batched relinearisation.
std::vector<Ciphertext> cheb_eval_many(Context& ctx, const std::vector<Ciphertext>& xs,
                                       const std::vector<double>& coeffs) {
  return cheb_eval_many(ctx, xs, coeffs, ctx.fast_schedule());
}

std::vector<Ciphertext> cheb_eval_many(Context& ctx, const std::vector<Ciphertext>& xs,
                                       const std::vector<double>& coeffs, bool fused_sum) {
  if (fused_sum) {
    std::vector<Ciphertext> ps = cheb_eval_ps_many(ctx, xs, coeffs);
    if (!ps.empty()) return ps;
  }
  for (const Ciphertext& x : xs)
    if (!x.valid()) throw Error(ErrKind::internal, "cheb_eval: operand is not initialized");
  if (coeffs.empty()) throw shape_error("cheb_eval: empty coefficient list");
  const int D = (int)coeffs.size() - 1;
  const std::size_t B = xs.size();
  std::vector<Ciphertext> out(B);
  if (D == 0) {
    for (std::size_t i = 0; i < B; ++i) out[i] = add_const(ctx, sub(ctx, xs[i], xs[i]), coeffs[0]);
    return out;
  }
  std::vector<std::vector<Ciphertext>> T(B, std::vector<Ciphertext>(D + 1));
  for (std::size_t i = 0; i < B; ++i) T[i][1] = xs[i];
  // T_k brought down to a lower level once and reused (the operand alignment
  // of mult_cipher / sub would otherwise repeat the same level_down per use)
  std::map<std::tuple<std::size_t, int, int>, Ciphertext> lowered;
  auto at = [&](std::size_t i, int k, int limbs) -> Ciphertext {
    if (T[i][k].limbs <= limbs) return T[i][k];
    auto key = std::make_tuple(i, k, limbs);
    auto it = lowered.find(key);
    if (it != lowered.end()) return it->second;
    return lowered[key] = level_down(ctx, T[i][k], limbs);
  };
  for (int lo = 2; lo <= D; lo = lo * 2 - 1) {
    const int hi = std::min(D, 2 * lo - 2 > lo ? 2 * lo - 2 : lo);
    std::vector<Ciphertext> as, bs;
    for (std::size_t i = 0; i < B; ++i)
      for (int d = lo; d <= hi; ++d) {
        const int a = (d + 1) / 2, b = d / 2;
        const int l = std::min(T[i][a].limbs, T[i][b].limbs);
        as.push_back(at(i, a, l));
        bs.push_back(at(i, b, l));
      }
    std::vector<Ciphertext> prods = mult_cipher_many(ctx, as, bs);
    std::vector<Ciphertext> doubled = add_many(ctx, prods, prods);
    std::size_t k = 0;
    for (std::size_t i = 0; i < B; ++i)
      for (int d = lo; d <= hi; ++d, ++k)
        T[i][d] = (d % 2 == 0) ? add_const(ctx, doubled[k], -1.0) : sub(ctx, doubled[k], at(i, 1, doubled[k].limbs));
    if (hi == D) break;
  }
  if (fused_sum) {  // sum_d c_d T_d: one fused constant MAC and one rescale per input
    for (std::size_t i = 0; i < B; ++i)
      out[i] = lincomb_const(ctx, std::vector<Ciphertext>(T[i].begin() + 1, T[i].end()),
                             std::vector<double>(coeffs.begin() + 1, coeffs.end()), coeffs[0]);
    return out;
  }
  std::vector<Ciphertext> ts;
  std::vector<double> cs;
  for (std::size_t i = 0; i < B; ++i)
    for (int d = 1; d <= D; ++d) {
      ts.push_back(T[i][d]);
      cs.push_back(coeffs[d]);
    }
  std::vector<Ciphertext> terms = mult_const_many(ctx, ts, cs);
  for (std::size_t i = 0; i < B; ++i) {
    Ciphertext acc = terms[i * D];
    for (int d = 1; d < D; ++d) acc = add(ctx, acc, terms[i * D + d]);
    out[i] = add_const(ctx, acc, coeffs[0]);
  }
  return out;
}

// secure_relu (layers_misc.cpp:268-295)
Ciphertext secure_relu(Context& ctx, const Ciphertext& x, double scale, int degree, std::size_t active_slots) {
  return secure_relu_many(ctx, {x}, scale, degree, active_slots)[0];
}

// The same activation on several ciphertexts (the images of a batched inference): one
// polynomial evaluation whose relinearisations, rescales and constant combinations carry
// every input (cheb_eval_many).  Per input bit-identical to secure_relu.
std::vector<Ciphertext> secure_relu_many(Context& ctx, const std::vector<Ciphertext>& xs, double scale, int degree,
                                         std::size_t active_slots) {
  if (degree < 0) throw shape_error("activation degree must be >= 0");
  const bool scaled = scale > 1.0;
  const double beta = scaled ? scale : 1.0;
  std::vector<Ciphertext> vs = xs;
  if (scaled) {
    if (active_slots == 0) throw shape_error("scaled activation requires the active slot count");
    if (active_slots > (std::size_t)ctx.S()) throw capacity_error("active slot count exceeds the context");
    for (Ciphertext& v : vs) v = mp(ctx, v, range_mask(ctx, 0, active_slots, 1.0 / beta));
  }
  const auto f = [beta](double z) { return z < 0.0 ? 0.0 : beta * z; };
  return cheb_eval_many(ctx, vs, cheb_coefficients(f, degree));
}

// ------------------------------------------------------------- depth costs
int pad_depth_cost(std::size_t padding) { return padding > 0 ? 1 : 0; }

int stride_depth_cost(int variant, std::size_t W, std::size_t S, std::size_t W_out) {
  (void)W;
  if (variant == 1 && detail::masked_stride_applicable(W_out)) return detail::stride_mask_compact_depth(S, W_out);
  return 1;
}

int conv_depth_cost(const ConvConfig& cfg, std::size_t W_in) {
  if (cfg.mode == 1) return 2;
  const std::size_t Wp = W_in + 2 * cfg.padding;
  const std::size_t W_out = conv_output_width(W_in, cfg.kernel, cfg.stride, cfg.padding);
  const int pad = pad_depth_cost(cfg.padding);
  if (cfg.mode == 2 && cfg.in_channels > 1) {
    if (detail::masked_stride_applicable(W_out)) return pad + 1 + detail::stride_mask_compact_depth(cfg.stride, W_out);
    return pad + 2;
  }
  const int sc = (cfg.stride == 1 && W_out == Wp) ? 0 : stride_depth_cost(cfg.stride_variant, Wp, cfg.stride, W_out);
  return pad + 2 + sc;
}

int pool_depth_cost(int kind, std::size_t k, std::size_t S, int variant, std::size_t W_in) {
  if (kind == 1) return 1;
  if (kind == 2) return 2;
  const std::size_t W_out = conv_output_width(W_in, k, S, 0);
  const int sc = (S == 1 && W_out == W_in) ? 0 : stride_depth_cost(variant, W_in, S, W_out);
  return 1 + sc;
}

int fc_depth_cost() { return 2; }

int relu_depth_cost(double scale, int degree) { return (scale > 1.0 ? 1 : 0) + cheb_eval_depth(degree); }

}  // namespace fheon
