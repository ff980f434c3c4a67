// Evaluator ops over device ciphertexts (see engine.hpp for the mapping to
// proj/src/backend.cpp).  Every op enqueues on the context stream; nothing
// here synchronises except decrypt/download.
#include <cmath>
#include <cstring>
#include <map>

#include "engine.hpp"

#include "bootstrap.hpp"

namespace fheon {

namespace {

LimbSet limbset(u64* base, int blocks, std::size_t stride, int E, int ell, int L, int p0 = 0,
                const DigitTable* skip = nullptr) {
  LimbSet s{};
  s.base[0] = base;
  s.nbase = 1;
  s.blocks_per_base = blocks;
  s.block_stride = (long long)stride;
  s.E = E;
  s.ell = ell;
  s.L = L;
  s.p0 = p0;
  s.skip_digits = skip != nullptr ? skip->beta(ell) : 0;
  if (skip) s.dig = *skip;
  return s;
}

PolyList plist(std::initializer_list<u64*> ps) {
  PolyList l{};
  l.n = 0;
  for (u64* p : ps) {
    l.p[l.n] = p;
    l.g[l.n] = 1;
    ++l.n;
  }
  return l;
}

u64 signed_mod(long long k, u64 q) { return k >= 0 ? (u64)k % q : (q - 1 - (u64)(-(k + 1)) % q); }

// round(x) mod q for |x| < 2^100 (constants past 2^62 are split at 2^32)
u64 round_mod(double x, u64 q) {
  if (std::fabs(x) < 4611686018427387904.0) return signed_mod(std::llround(x), q);
  if (!(std::fabs(x) < 1.2676506002282294e30)) throw Error(ErrKind::capacity, "constant exceeds 2^100");
  const double hi = std::floor(x / 4294967296.0);
  const long long lo = std::llround(x - hi * 4294967296.0);
  const u64 two32 = ((u64)1 << 32) % q;
  const u64 h = mulmod(signed_mod((long long)hi, q), two32, q);
  return addmod(h, signed_mod(lo, q), q);
}

void require_valid(const Ciphertext& c, const char* op) {
  if (!c.valid()) throw Error(ErrKind::internal, std::string(op) + ": operand is not initialized");
}

void require_depth(const Ciphertext& c, const char* op) {
  if (c.level() < 1)
    throw Error(ErrKind::depth_exhausted,
                std::string(op) + ": no multiplicative depth left (level " + std::to_string(c.level()) + ")");
}

void check_scales(const Ciphertext& a, const Ciphertext& b, const char* op) {
  const double r = a.scale / b.scale;
  if (!(std::fabs(r - 1.0) < 1e-6))
    throw Error(ErrKind::internal, std::string(op) + ": operand scales differ (" + std::to_string(a.scale) + " vs " +
                                       std::to_string(b.scale) + ")");
}

// ModDown's finish (acc - conv) P^-1 + sigma(add) fused into the conv's forward NTT
NttEpilogue moddown_epilogue(const DevTables& t, const PolyList& out, const PolyList& acc, const PolyList& add) {
  NttEpilogue e{};
  for (int i = 0; i < out.n; ++i) {
    e.out[i] = out.p[i];
    e.src[i] = acc.p[i];
    e.add[i] = add.p[i];
    e.add_g[i] = add.g[i];
  }
  e.cst = t.md_q + 2;  // md_q[i * 4 + 2] = P^-1 mod q_i, + 3 Shoup
  e.cst_stride = 4;
  return e;
}

// rescale's finish (a - lift) q_l^-1 fused into the lift's forward NTT
NttEpilogue rescale_epilogue(const DevTables& t, const PolyList& out, const PolyList& a, int limbs) {
  NttEpilogue e{};
  for (int i = 0; i < out.n; ++i) {
    e.out[i] = out.p[i];
    e.src[i] = a.p[i];
    e.add[i] = nullptr;
    e.add_g[i] = 1;
  }
  e.cst = t.rs + (std::size_t)(limbs - 1) * t.L * 4;  // rs[(l * L + i) * 4] = q_l^-1 mod q_i, + 1 Shoup
  e.cst_stride = 4;
  return e;
}

// ModUp of every input, batched (one pipeline of launches per 32 inputs):
// [nin][beta][limbs+K][N] extended digits in the NTT domain
BufPtr modup_all(Context& ctx, const std::vector<const u64*>& inputs, int limbs) {
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  const int L = ctx.L(), E = limbs + ctx.K();
  const int beta = t.dig.beta(limbs);
  const int nin = (int)inputs.size();
  const std::size_t ext_words = (std::size_t)beta * E * N;
  BufPtr xc = ctx.alloc((std::size_t)std::min(nin, kMaxBases) * limbs * N);
  BufPtr ext = ctx.alloc((std::size_t)nin * ext_words);
  for (int i0 = 0; i0 < nin; i0 += kMaxBases) {
    const int ni = std::min(kMaxBases, nin - i0);
    LimbSet dst = limbset(xc->ptr, ni, (std::size_t)limbs * N, limbs, limbs, L);
    LimbSet src = dst;
    src.nbase = ni;
    src.blocks_per_base = 1;
    for (int i = 0; i < ni; ++i) src.base[i] = const_cast<u64*>(inputs[i0 + i]);
    ntt_inverse(t, dst, st, &src);
    PolyList xl{}, el{};
    xl.n = el.n = ni;
    for (int i = 0; i < ni; ++i) {
      xl.p[i] = xc->ptr + (std::size_t)i * limbs * N;
      el.p[i] = ext->ptr + (std::size_t)(i0 + i) * ext_words;
    }
    modup_bconv(t, el, xl, limbs, st);
    ntt_forward(t, limbset(ext->ptr + (std::size_t)i0 * ext_words, ni * beta, (std::size_t)E * N, E, limbs, L, 0,
                           &t.dig),
                st);
  }
  std::size_t own = 0;  // limbs the digits pass through un-NTT'd
  for (int j = 0; j < beta; ++j) own += (std::size_t)(t.dig.hi(j, limbs) - t.dig.lo(j));
  ctx.stats.ntt_limbs += (std::size_t)nin * ((std::size_t)limbs + (std::size_t)beta * E - own);
  return ext;
}

// Hybrid key switch of several NTT-domain inputs d_i ([limbs][N] each).  Job r
// switches input `in` under key `key_id` with automorphism g (hoisting: jobs
// sharing an input share its ModUp).  Output r:
//   c0 = ModDown(acc0) + sigma_{add0_g}(add0)   (add0 may be null)
//   c1 = ModDown(acc1) + add1                   (add1 may be null)
struct KsJob {
  u64 key_id;
  u64 g;
  const u64* add0;
  u64 add0_g;
  const u64* add1;
  int in = 0;
};

std::vector<Ciphertext> keyswitch(Context& ctx, const std::vector<const u64*>& inputs, int limbs,
                                  const std::vector<KsJob>& jobs) {
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  const int L = ctx.L(), K = ctx.K(), E = limbs + K;
  const int beta = t.dig.beta(limbs);
  ctx.stats.keyswitches += jobs.size();

  const std::size_t ext_words = (std::size_t)beta * E * N;
  BufPtr ext = modup_all(ctx, inputs, limbs);

  std::vector<const u64*> keys(jobs.size());
  for (std::size_t r = 0; r < jobs.size(); ++r) keys[r] = ctx.key(jobs[r].key_id);

  std::vector<Ciphertext> outs;
  outs.reserve(jobs.size());
  constexpr int kChunk = kMaxPolys / 2;
  for (std::size_t r0 = 0; r0 < jobs.size(); r0 += kChunk) {
    const int R = (int)std::min<std::size_t>(kChunk, jobs.size() - r0);
    BufPtr acc = ctx.alloc((std::size_t)R * 2 * E * N);
    KsJobs kj{};
    kj.n = R;
    for (int r = 0; r < R; ++r) {
      const int in = jobs[r0 + r].in;
      kj.key[r] = keys[r0 + r];
      kj.ext[r] = ext->ptr + (std::size_t)in * ext_words;
      kj.d[r] = inputs[in];
      kj.acc[r] = acc->ptr + (std::size_t)r * 2 * E * N;
      kj.g[r] = jobs[r0 + r].g;
    }
    ks_inner_product(t, kj, limbs, st);
    // ModDown of both accumulator polys of every job
    LimbSet zs{};
    zs.nbase = R;
    for (int r = 0; r < R; ++r) zs.base[r] = kj.acc[r] + (std::size_t)limbs * N;
    zs.blocks_per_base = 2;
    zs.block_stride = (long long)E * N;
    zs.E = K;
    zs.ell = 0;
    zs.L = L;
    ntt_inverse(t, zs, st);
    BufPtr conv = ctx.alloc((std::size_t)R * 2 * limbs * N);
    PolyList cl{}, zl{}, al{}, ol{}, addl{};
    cl.n = zl.n = al.n = ol.n = addl.n = 2 * R;
    for (int r = 0; r < R; ++r) {
      Ciphertext o = ctx.new_ct(limbs);
      for (int p = 0; p < 2; ++p) {
        const int i = 2 * r + p;
        cl.p[i] = conv->ptr + (std::size_t)i * limbs * N;
        zl.p[i] = kj.acc[r] + (std::size_t)p * E * N + (std::size_t)limbs * N;
        al.p[i] = kj.acc[r] + (std::size_t)p * E * N;
        ol.p[i] = p == 0 ? o.c0 : o.c1;
        const KsJob& jb = jobs[r0 + r];
        addl.p[i] = const_cast<u64*>(p == 0 ? jb.add0 : jb.add1);
        addl.g[i] = p == 0 ? jb.add0_g : 1;
      }
      outs.push_back(o);
    }
    moddown_conv(t, cl, zl, limbs, st);
    ntt_forward_epilogue(t, limbset(conv->ptr, 2 * R, (std::size_t)limbs * N, limbs, limbs, L),
                         moddown_epilogue(t, ol, al, addl), st);
    ctx.stats.ntt_limbs += (std::size_t)R * 2 * (K + limbs);
  }
  return outs;
}

// Relinearisation fused with the rescale: for every job the
// key inner product acc = <ModUp(d2), rlk> over Q u P, then z = acc + P (d0, d1)
// is divided by P' = P q_l (l = limbs - 1) in ONE ModDown: the special limbs are
// q_l and the K p's (z's q_l limb gets + P d_l, then the K + 1 limbs go to the
// coefficient domain), the basis conversion runs over K + 1 inputs, and the
// forward NTT's store computes (acc_i - conv_i) P'^-1 + d_i q_l^-1 = round(z / P')
// on the l remaining limbs.  One rounding instead of ModDown + rescale, and no
// rescale NTTs.  Mirrored by oracle/ckks_oracle.c ock_mult_cipher.
std::vector<Ciphertext> keyswitch_relin_rescale(Context& ctx, const std::vector<const u64*>& inputs, int limbs,
                                                const std::vector<KsJob>& jobs) {
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  const int L = ctx.L(), K = ctx.K(), E = limbs + K;
  const int l = limbs - 1;
  const int beta = t.dig.beta(limbs);
  ctx.stats.keyswitches += jobs.size();
  const std::size_t ext_words = (std::size_t)beta * E * N;
  BufPtr ext = modup_all(ctx, inputs, limbs);
  std::vector<Ciphertext> outs;
  outs.reserve(jobs.size());
  constexpr int kChunk = kMaxPolys / 2;
  for (std::size_t r0 = 0; r0 < jobs.size(); r0 += kChunk) {
    const int R = (int)std::min<std::size_t>(kChunk, jobs.size() - r0);
    BufPtr acc = ctx.alloc((std::size_t)R * 2 * E * N);
    KsJobs kj{};
    kj.n = R;
    for (int r = 0; r < R; ++r) {
      const int in = jobs[r0 + r].in;
      kj.key[r] = ctx.key(jobs[r0 + r].key_id);
      kj.ext[r] = ext->ptr + (std::size_t)in * ext_words;
      kj.d[r] = inputs[in];
      kj.acc[r] = acc->ptr + (std::size_t)r * 2 * E * N;
      kj.g[r] = jobs[r0 + r].g;
    }
    ks_inner_product(t, kj, limbs, st);
    // z_l = acc_l + P d_l on the dropped limb
    PolyList za{}, dl{};
    za.n = dl.n = 2 * R;
    for (int r = 0; r < R; ++r)
      for (int p = 0; p < 2; ++p) {
        za.p[2 * r + p] = kj.acc[r] + (std::size_t)p * E * N + (std::size_t)l * N;
        const KsJob& jb = jobs[r0 + r];
        dl.p[2 * r + p] = const_cast<u64*>(p == 0 ? jb.add0 : jb.add1) + (std::size_t)l * N;
      }
    const HostTables& h = ctx.host();
    u64 pm_l = 1;  // P mod q_l, Montgomery form
    for (int k = 0; k < K; ++k) pm_l = mulmod(pm_l, h.q[L + k] % h.q[l], h.q[l]);
    ew_axpy_limb(t, za, dl, to_mont(pm_l, h.q[l]), l, st);
    // the K + 1 special limbs (q_l, p_0..p_K-1) to the coefficient domain
    LimbSet zs{};
    zs.nbase = R;
    for (int r = 0; r < R; ++r) zs.base[r] = kj.acc[r] + (std::size_t)l * N;
    zs.blocks_per_base = 2;
    zs.block_stride = (long long)E * N;
    zs.E = K + 1;
    zs.ell = 1;
    zs.p0 = l;
    zs.L = L;
    ntt_inverse(t, zs, st);
    BufPtr conv = ctx.alloc((std::size_t)R * 2 * l * N);
    PolyList cl{}, zl{}, al{}, ol{}, addl{};
    cl.n = zl.n = al.n = ol.n = addl.n = 2 * R;
    for (int r = 0; r < R; ++r) {
      Ciphertext o = ctx.new_ct(l);
      for (int p = 0; p < 2; ++p) {
        const int i = 2 * r + p;
        cl.p[i] = conv->ptr + (std::size_t)i * l * N;
        zl.p[i] = kj.acc[r] + (std::size_t)p * E * N + (std::size_t)l * N;
        al.p[i] = kj.acc[r] + (std::size_t)p * E * N;
        ol.p[i] = p == 0 ? o.c0 : o.c1;
        const KsJob& jb = jobs[r0 + r];
        addl.p[i] = const_cast<u64*>(p == 0 ? jb.add0 : jb.add1);
        addl.g[i] = 1;
      }
      outs.push_back(o);
    }
    moddown_fused_conv_tc(t, cl, zl, limbs, st);
    NttEpilogue e{};
    for (int i = 0; i < 2 * R; ++i) {
      e.out[i] = ol.p[i];
      e.src[i] = al.p[i];
      e.add[i] = addl.p[i];
      e.add_g[i] = 1;
    }
    e.cst = t.md2_q + (std::size_t)l * L * 4 + 2;  // P'^-1 mod q_i, Shoup
    e.cst_stride = 4;
    e.acst = t.rs + (std::size_t)l * L * 4;  // q_l^-1 mod q_i, Shoup
    e.acst_stride = 4;
    ntt_forward_epilogue(t, limbset(conv->ptr, 2 * R, (std::size_t)l * N, l, l, L), e, st);
    ctx.stats.ntt_limbs += (std::size_t)R * 2 * (K + 1 + l);
    ctx.stats.rescales += (std::size_t)R;
  }
  return outs;
}

// Rotate-and-sum: output r = sum over jobs of group r of rot(input, g), with
// ONE ModDown per output (kernels.hpp KsSumJobs).  jobs[k].in indexes `inputs`
// (c1 pointers, ModUp shared by repeated inputs), c0s[in] is that input's c0.
struct SumJob {
  u64 g;
  int in;
  int group;
  u64 key_id = kNoKeyOverride;  // the key to read when it is not the Galois element's own
  // Q u P mode (every job of a call or none): c0qp = the job's c0 as a [limbs+K][N] polynomial
  // over Q u P, added as sigma_g(c0qp) on every limb (the c0 half of an accumulator that was
  // never ModDown'd); direct_c1 != null: no key switch at all, (c0qp, direct_c1) join as they are
  const u64* c0qp = nullptr;
  const u64* direct_c1 = nullptr;
  static constexpr u64 kNoKeyOverride = ~0ULL;
  u64 key() const { return key_id == kNoKeyOverride ? g : key_id; }
};
// Q u P accumulators of every group, [ngroups][2][limbs+K][N] (canonical, standard form):
// acc_r = sum_{jobs of r} <sigma_g(ModUp(d)), key_g> + P sigma_g(c0) on the Q limbs
BufPtr keyswitch_sum_accs(Context& ctx, const std::vector<const u64*>& inputs, const std::vector<const u64*>& c0s,
                          int limbs, const std::vector<SumJob>& jobs, int ngroups) {
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  const int K = ctx.K(), E = limbs + K;
  const int beta = t.dig.beta(limbs);
  const std::size_t ext_words = (std::size_t)beta * E * N;
  ctx.stats.keyswitches += jobs.size();
  BufPtr ext = modup_all(ctx, inputs, limbs);
  std::vector<std::vector<const SumJob*>> by_group(ngroups);
  for (const SumJob& j : jobs) by_group[j.group].push_back(&j);
  // every group = one input under the same key list (a hoisted stage)?
  const bool qp = !jobs.empty() && jobs[0].c0qp != nullptr;
  for (const SumJob& j : jobs)
    if ((j.c0qp != nullptr) != qp) throw Error(ErrKind::internal, "rotate_sum: mixed Q and Q u P c0 terms");
  bool shared = !qp && ngroups > 1 && !by_group[0].empty() && (int)by_group[0].size() <= kMaxSharedKeys;
  for (const SumJob& j : jobs) shared = shared && j.key_id == SumJob::kNoKeyOverride;
  for (int r = 0; r < ngroups && shared; ++r) {
    shared = by_group[r].size() == by_group[0].size();
    for (std::size_t k = 0; k < by_group[r].size() && shared; ++k)
      shared = by_group[r][k]->g == by_group[0][k]->g && by_group[r][k]->in == by_group[r][0]->in;
  }
  // accumulators of all groups, [2][limbs+K][N] each
  BufPtr accs = ctx.alloc((std::size_t)ngroups * 2 * E * N);
  auto acc_of = [&](int r) { return accs->ptr + (std::size_t)r * 2 * E * N; };
  if (shared) {
    for (int r0 = 0; r0 < ngroups; r0 += kMaxSharedGroups) {
      KsSharedJobs kj{};
      kj.nkeys = (int)by_group[0].size();
      for (int k = 0; k < kj.nkeys; ++k) {
        kj.key[k] = ctx.key(by_group[0][k]->g);
        kj.g[k] = by_group[0][k]->g;
      }
      kj.ngroups = std::min(kMaxSharedGroups, ngroups - r0);
      for (int r = 0; r < kj.ngroups; ++r) {
        const int in = by_group[r0 + r][0]->in;
        kj.ext[r] = ext->ptr + (std::size_t)in * ext_words;
        kj.d[r] = inputs[in];
        kj.c0[r] = c0s[in];
        kj.acc[r] = acc_of(r0 + r);
      }
      ks_inner_shared(t, kj, limbs, st);
    }
  } else {
    int r0 = 0;
    while (r0 < ngroups) {
      // pack whole groups into one launch (<= kMaxSumGroups groups, <= kMaxSumJobs jobs)
      KsSumJobs kj{};
      int nj = 0, R = 0;
      while (r0 + R < ngroups && R < kMaxSumGroups) {
        const int gsz = (int)by_group[r0 + R].size();
        if (gsz > kMaxSumJobs) throw Error(ErrKind::internal, "rotate_sum: group larger than one launch");
        if (nj + gsz > kMaxSumJobs) break;
        kj.begin[R] = nj;
        for (const SumJob* j : by_group[r0 + R]) {
          if (j->direct_c1) {
            kj.direct[nj] = 1;
            kj.d[nj] = j->direct_c1;
          } else {
            kj.key[nj] = ctx.key(j->key());
            kj.ext[nj] = ext->ptr + (std::size_t)j->in * ext_words;
            kj.d[nj] = inputs[j->in];
          }
          kj.c0[nj] = qp ? j->c0qp : c0s[j->in];
          kj.g[nj] = j->g;
          ++nj;
        }
        ++R;
      }
      kj.begin[R] = nj;
      kj.ngroups = R;
      kj.c0_qp = qp ? 1 : 0;
      for (int r = 0; r < R; ++r) kj.acc[r] = acc_of(r0 + r);
      ks_inner_sum(t, kj, limbs, st);
      r0 += R;
    }
  }
  return accs;
}

// ModDown of Q u P accumulators ([2][limbs+K][N] each): round(acc / P) over the
// Q limbs, 32 accumulators (64 polys) per pipeline
std::vector<Ciphertext> moddown_accs(Context& ctx, const std::vector<u64*>& accp, int limbs) {
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  const int L = ctx.L(), K = ctx.K(), E = limbs + K;
  const int ngroups = (int)accp.size();
  std::vector<Ciphertext> outs;
  outs.reserve(ngroups);
  for (int r0 = 0; r0 < ngroups; r0 += kMaxPolys / 2) {
    const int R = std::min(kMaxPolys / 2, ngroups - r0);
    struct {
      u64* acc[kMaxPolys / 2];
    } kj{};
    for (int r = 0; r < R; ++r) kj.acc[r] = accp[r0 + r];
    LimbSet zs{};
    zs.nbase = R;
    for (int r = 0; r < R; ++r) zs.base[r] = kj.acc[r] + (std::size_t)limbs * N;
    zs.blocks_per_base = 2;
    zs.block_stride = (long long)E * N;
    zs.E = K;
    zs.ell = 0;
    zs.L = L;
    ntt_inverse(t, zs, st);
    BufPtr conv = ctx.alloc((std::size_t)R * 2 * limbs * N);
    PolyList cl{}, zl{}, al{}, ol{}, addl{};
    cl.n = zl.n = al.n = ol.n = addl.n = 2 * R;
    for (int r = 0; r < R; ++r) {
      Ciphertext o = ctx.new_ct(limbs);
      for (int p = 0; p < 2; ++p) {
        const int i = 2 * r + p;
        cl.p[i] = conv->ptr + (std::size_t)i * limbs * N;
        zl.p[i] = kj.acc[r] + (std::size_t)p * E * N + (std::size_t)limbs * N;
        al.p[i] = kj.acc[r] + (std::size_t)p * E * N;
        ol.p[i] = p == 0 ? o.c0 : o.c1;
        addl.p[i] = nullptr;
        addl.g[i] = 1;
      }
      outs.push_back(o);
    }
    moddown_conv(t, cl, zl, limbs, st);
    ntt_forward_epilogue(t, limbset(conv->ptr, 2 * R, (std::size_t)limbs * N, limbs, limbs, L),
                         moddown_epilogue(t, ol, al, addl), st);
    ctx.stats.ntt_limbs += (std::size_t)R * 2 * (K + limbs);
  }
  return outs;
}

// ModDown of Q u P accumulators with the rescale folded in (as keyswitch_relin_rescale):
// z = acc + P add (add: the group's unrotated terms, or none) divided by P' = P q_l,
// l = limbs - 1, in ONE rounding -- round(z / P') on the l remaining limbs, no
// rescale NTTs.  Outputs [2][l][N], scale left to the caller.
std::vector<Ciphertext> moddown_rescale_accs(Context& ctx, const std::vector<u64*>& accp,
                                             const std::vector<Ciphertext>& adds, int limbs) {
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  const int L = ctx.L(), K = ctx.K(), E = limbs + K;
  const int l = limbs - 1;
  const HostTables& h = ctx.host();
  u64 pm_l = 1;  // P mod q_l
  for (int k = 0; k < K; ++k) pm_l = mulmod(pm_l, h.q[L + k] % h.q[l], h.q[l]);
  const u64 pm_mont = to_mont(pm_l, h.q[l]);
  const int ngroups = (int)accp.size();
  std::vector<Ciphertext> outs;
  outs.reserve(ngroups);
  constexpr int kChunk = kMaxPolys / 2;
  for (int r0 = 0; r0 < ngroups; r0 += kChunk) {
    const int R = std::min(kChunk, ngroups - r0);
    // z_l = acc_l + P add_l on the dropped limb
    PolyList za{}, dl{};
    for (int r = 0; r < R; ++r) {
      const Ciphertext& a = adds[r0 + r];
      if (!a.valid()) continue;
      for (int p = 0; p < 2; ++p) {
        za.p[za.n++] = accp[r0 + r] + (std::size_t)p * E * N + (std::size_t)l * N;
        dl.p[dl.n++] = (p == 0 ? a.c0 : a.c1) + (std::size_t)l * N;
      }
    }
    if (za.n) ew_axpy_limb(t, za, dl, pm_mont, l, st);
    // the K + 1 special limbs (q_l, p_0..p_K-1) to the coefficient domain
    LimbSet zs{};
    zs.nbase = R;
    for (int r = 0; r < R; ++r) zs.base[r] = accp[r0 + r] + (std::size_t)l * N;
    zs.blocks_per_base = 2;
    zs.block_stride = (long long)E * N;
    zs.E = K + 1;
    zs.ell = 1;
    zs.p0 = l;
    zs.L = L;
    ntt_inverse(t, zs, st);
    BufPtr conv = ctx.alloc((std::size_t)R * 2 * l * N);
    PolyList cl{}, zl{};
    cl.n = zl.n = 2 * R;
    NttEpilogue e{};
    for (int r = 0; r < R; ++r) {
      Ciphertext o = ctx.new_ct(l);
      const Ciphertext& a = adds[r0 + r];
      for (int p = 0; p < 2; ++p) {
        const int i = 2 * r + p;
        cl.p[i] = conv->ptr + (std::size_t)i * l * N;
        zl.p[i] = accp[r0 + r] + (std::size_t)p * E * N + (std::size_t)l * N;
        e.out[i] = p == 0 ? o.c0 : o.c1;
        e.src[i] = accp[r0 + r] + (std::size_t)p * E * N;
        e.add[i] = a.valid() ? (p == 0 ? a.c0 : a.c1) : nullptr;
        e.add_g[i] = 1;
      }
      outs.push_back(o);
    }
    moddown_fused_conv_tc(t, cl, zl, limbs, st);
    e.cst = t.md2_q + (std::size_t)l * L * 4 + 2;  // P'^-1 mod q_i, Shoup
    e.cst_stride = 4;
    e.acst = t.rs + (std::size_t)l * L * 4;  // q_l^-1 mod q_i, Shoup
    e.acst_stride = 4;
    ntt_forward_epilogue(t, limbset(conv->ptr, 2 * R, (std::size_t)l * N, l, l, L), e, st);
    ctx.stats.ntt_limbs += (std::size_t)R * 2 * (K + 1 + l);
    ctx.stats.rescales += (std::size_t)R;
  }
  return outs;
}

std::vector<Ciphertext> keyswitch_sum(Context& ctx, const std::vector<const u64*>& inputs,
                                      const std::vector<const u64*>& c0s, int limbs, const std::vector<SumJob>& jobs,
                                      int ngroups) {
  BufPtr accs = keyswitch_sum_accs(ctx, inputs, c0s, limbs, jobs, ngroups);
  const std::size_t stride = (std::size_t)2 * (limbs + ctx.K()) * ctx.N();
  std::vector<u64*> accp(ngroups);
  for (int r = 0; r < ngroups; ++r) accp[r] = accs->ptr + (std::size_t)r * stride;
  return moddown_accs(ctx, accp, limbs);
}

}  // namespace

namespace {
// ModDown of the c1 half alone of Q u P accumulators ([2][limbs+K][N] each): [n][limbs][N]
BufPtr moddown_c1(Context& ctx, const std::vector<u64*>& accp, int limbs) {
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  const int L = ctx.L(), K = ctx.K(), E = limbs + K;
  const int n = (int)accp.size();
  BufPtr out = ctx.alloc((std::size_t)n * limbs * N);
  for (int r0 = 0; r0 < n; r0 += kMaxBases) {
    const int R = std::min(kMaxBases, n - r0);
    // the special limbs go to the coefficient domain OUT of place: the accumulator stays whole
    // (an unrotated giant that also enters conjugated is added as it is afterwards)
    BufPtr z = ctx.alloc((std::size_t)R * K * N);
    LimbSet zs = limbset(z->ptr, R, (std::size_t)K * N, K, 0, L);
    LimbSet src = zs;
    src.nbase = R;
    src.blocks_per_base = 1;
    for (int r = 0; r < R; ++r) src.base[r] = accp[r0 + r] + (std::size_t)E * N + (std::size_t)limbs * N;
    ntt_inverse(t, zs, st, &src);
    BufPtr conv = ctx.alloc((std::size_t)R * limbs * N);
    PolyList cl{}, zl{}, al{}, ol{}, addl{};
    cl.n = zl.n = al.n = ol.n = addl.n = R;
    for (int r = 0; r < R; ++r) {
      cl.p[r] = conv->ptr + (std::size_t)r * limbs * N;
      zl.p[r] = z->ptr + (std::size_t)r * K * N;
      al.p[r] = accp[r0 + r] + (std::size_t)E * N;
      ol.p[r] = out->ptr + (std::size_t)(r0 + r) * limbs * N;
      addl.p[r] = nullptr;
      addl.g[r] = 1;
    }
    moddown_conv(t, cl, zl, limbs, st);
    ntt_forward_epilogue(t, limbset(conv->ptr, R, (std::size_t)limbs * N, limbs, limbs, L),
                         moddown_epilogue(t, ol, al, addl), st);
    ctx.stats.ntt_limbs += (std::size_t)R * (K + limbs);
  }
  return out;
}

bool dh_c0qp_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FHEON_DH_C0QP");
    return e ? std::atoi(e) != 0 : true;  // FHEON_DH_C0QP=0: the two-ModDown form, for A/B runs
  }();
  return on;
}
}  // namespace

// Double-hoisted baby-step giant-step transform:
//   out = rescale( sum_g rot( ModDown( sum_t pt_{g,t} (*) B_{b(g,t)} ), G_g ) )
// B_b = (P sigma_b(c0) + ks0_b, ks1_b) over Q u P is baby rotation b WITHOUT its
// ModDown (one shared ModUp, one key inner product each); the identity baby is
// (P c0, P c1) on Q and 0 on P.  The plaintexts live over Q u P, so each giant's
// inner sum needs ONE ModDown instead of one per baby; the giant rotations are a
// rotate-and-sum (one more ModDown) and the sum is rescaled once.
Ciphertext bsgs_double_hoisted(Context& ctx, const Ciphertext& x, const std::vector<long>& babies,
                               const std::vector<DhGiant>& giants, bool with_conj) {
  return bsgs_double_hoisted_many(ctx, {x}, babies, giants, with_conj)[0];
}

// The same transform on several ciphertexts of one level and scale (lockstep images of a
// batched inference): accumulator groups are ordered baby-major / giant-major with the
// inputs innermost, so the CTAs that run side by side (grid x = group / output) read the
// same key slice or plaintext diagonal and every key and diagonal leaves HBM once per
// batch instead of once per input.  Per input the operations and their order are those of
// the single-input transform: outputs are bit-identical.
std::vector<Ciphertext> bsgs_double_hoisted_many(Context& ctx, const std::vector<Ciphertext>& xs,
                                                 const std::vector<long>& babies, const std::vector<DhGiant>& giants,
                                                 bool with_conj) {
  if (xs.empty()) return {};
  const int B = (int)xs.size();
  for (const Ciphertext& x : xs) {
    require_valid(x, "linear transform");
    require_depth(x, "linear transform");
    if (x.limbs != xs[0].limbs) throw Error(ErrKind::internal, "linear transform: inputs at different levels");
    check_scales(x, xs[0], "linear transform");
  }
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  const int limbs = xs[0].limbs, K = ctx.K(), E = limbs + K, lv = limbs - 1;
  const std::size_t accw = (std::size_t)2 * E * N;
  const HostTables& h = ctx.host();
  const int nb = (int)babies.size(), ng = (int)giants.size();
  // baby accumulators: group k * B + i = baby k of input i
  std::vector<SumJob> jobs;
  for (int k = 0; k < nb; ++k) {
    const u64 g = ctx.galois(babies[k]);
    if (g == 1) throw Error(ErrKind::internal, "double-hoisted transform: identity baby must be index -1");
    for (int i = 0; i < B; ++i) {
      ctx.record(0, babies[k]);
      ctx.stats.rotations++;
      jobs.push_back({g, i, k * B + i});
    }
  }
  std::vector<const u64*> c1s, c0s;
  for (const Ciphertext& x : xs) {
    c1s.push_back(x.c1);
    c0s.push_back(x.c0);
  }
  BufPtr accs = babies.empty() ? nullptr : keyswitch_sum_accs(ctx, c1s, c0s, limbs, jobs, nb * B);
  BufPtr ident;
  bool need_ident = false;
  for (const DhGiant& gi : giants)
    for (const auto& [b, pt] : gi.terms) need_ident = need_ident || b < 0;
  if (need_ident) {
    ident = ctx.alloc((std::size_t)B * accw);
    LimbConsts pc{};
    for (int i = 0; i < limbs; ++i) {
      u64 pm = 1 % h.q[i];
      for (int k = 0; k < K; ++k) pm = mulmod(pm, h.q[ctx.L() + k] % h.q[i], h.q[i]);
      pc.c[i] = pm;
      pc.sh[i] = shoup(pm, h.q[i]);
    }
    for (int i = 0; i < B; ++i) {
      u64* id = ident->ptr + (std::size_t)i * accw;
      ew_mul_const(t, plist({id, id + (std::size_t)E * N}), plist({xs[i].c0, xs[i].c1}), pc, limbs, st);
      for (int p = 0; p < 2; ++p)
        FHEON_CUDA(cudaMemsetAsync(id + (std::size_t)p * E * N + (std::size_t)limbs * N, 0,
                                   (std::size_t)K * N * sizeof(u64), st));
    }
  }
  // inner sums over Q u P, one output accumulator per (giant, input): output g * B + i; every
  // giant set x input chunk in one launch (each diagonal read once per batch, each baby once
  // per giant set)
  const std::size_t nout = (std::size_t)ng * B;
  BufPtr inner = ctx.alloc(nout * accw);
  for (int g0 = 0; g0 < ng; g0 += kBsgsMaxGiants)
    for (int i0 = 0; i0 < B; i0 += kBsgsMaxIn) {
      BsgsMacJobs jb{};
      jb.ngiants = std::min(kBsgsMaxGiants, ng - g0);
      jb.nin = std::min(kBsgsMaxIn, B - i0);
      jb.baby_stride = (long long)B * (long long)accw;
      jb.out_stride = (long long)B * (long long)accw;
      jb.c1_off = (long long)E * (long long)N;
      for (int z = 0; z < jb.ngiants; ++z) {
        const DhGiant& gi = giants[g0 + z];
        if (gi.terms.empty() || gi.terms.size() > (std::size_t)kMacMaxTerms)
          throw Error(ErrKind::internal, "double-hoisted transform: 1..32 terms per giant");
        for (std::size_t j = 0; j < gi.terms.size(); ++j) {
          jb.pt[z][j] = gi.terms[j].second->ptr;
          jb.bidx[z][j] = (short)gi.terms[j].first;
        }
        jb.nterm[z] = (int)gi.terms.size();
      }
      for (int i = 0; i < jb.nin; ++i) {
        jb.babies[i] = accs ? accs->ptr + (std::size_t)(i0 + i) * accw : nullptr;
        jb.ident[i] = ident ? ident->ptr + (std::size_t)(i0 + i) * accw : nullptr;
        jb.out[i] = inner->ptr + ((std::size_t)g0 * B + i0 + i) * accw;
      }
      mac_bsgs(t, jb, E, st, limbs);
    }
  std::vector<u64*> accp(nout);
  for (std::size_t o = 0; o < nout; ++o) accp[o] = inner->ptr + o * accw;
  const bool fused_tail = limbs >= 2 && bconv_tc_enabled() && K + 1 + 2 <= 16;
  if (dh_c0qp_enabled() && fused_tail && (with_conj ? 2 : 1) * ng <= kMaxSumJobs) {
    // Giant steps on the un-ModDown'd inner sums: only the c1 half of a giant is brought down to Q
    // (the key switch decomposes it); its c0 half stays over Q u P and joins the rotate-and-sum
    // accumulator as sigma_G(c0) on every limb, and the unrotated giant joins whole, with no key
    // switch and no ModDown of its own.  Half the giants' ModDown work, and one rounding fewer
    // on c0 (the result differs from the two-ModDown form by rounding only).
    const u64 conj = 2 * (u64)ctx.N() - 1, twoN = 2 * (u64)ctx.N();
    std::vector<int> slot_of(nout, -1);  // (g, i) -> c1 input index
    std::vector<u64*> need;
    for (int g = 0; g < ng; ++g) {
      const bool ident_g = ctx.galois(giants[g].rot) == 1;
      for (int i = 0; i < B; ++i)
        if (!ident_g || with_conj) {
          slot_of[(std::size_t)g * B + i] = (int)need.size();
          need.push_back(accp[(std::size_t)g * B + i]);
        }
    }
    BufPtr c1q = need.empty() ? nullptr : moddown_c1(ctx, need, limbs);
    std::vector<const u64*> inputs, c0s;
    for (std::size_t k = 0; k < need.size(); ++k) {
      inputs.push_back(c1q->ptr + k * (std::size_t)limbs * N);
      c0s.push_back(nullptr);
    }
    std::vector<SumJob> sj;
    for (int i = 0; i < B; ++i)
      for (int g = 0; g < ng; ++g) {
        const u64 ge = ctx.galois(giants[g].rot);
        const u64* acc = accp[(std::size_t)g * B + i];
        const int in = slot_of[(std::size_t)g * B + i];
        ctx.record(0, giants[g].rot);
        ctx.stats.rotations++;
        for (std::size_t j = 0; j < giants[g].terms.size(); ++j) {
          ctx.stats.mult_plain++;
          ctx.record(1, lv - 1);
        }
        SumJob a{ge, in, i};
        a.c0qp = acc;
        if (ge == 1) a.direct_c1 = acc + (std::size_t)E * N;
        sj.push_back(a);
        if (with_conj) {
          SumJob c{(ge * conj) % twoN, in, i};
          c.c0qp = acc;
          sj.push_back(c);
        }
      }
    BufPtr accs2 = keyswitch_sum_accs(ctx, inputs, c0s, limbs, sj, B);
    std::vector<u64*> ap(B);
    for (int i = 0; i < B; ++i) ap[i] = accs2->ptr + (std::size_t)i * accw;
    std::vector<Ciphertext> outs = moddown_rescale_accs(ctx, ap, std::vector<Ciphertext>(B), limbs);
    for (Ciphertext& o : outs) o.scale = h.T[lv - 1];
    return outs;
  }
  std::vector<Ciphertext> rows = moddown_accs(ctx, accp, limbs);
  const double sc = h.T[lv - 1] * (double)h.q[lv];  // plaintexts encoded at T_{lv-1} q_lv / scale(x)
  std::vector<std::vector<std::pair<Ciphertext, long>>> terms(B);
  for (int i = 0; i < B; ++i)
    for (int g = 0; g < ng; ++g) {
      Ciphertext& row = rows[(std::size_t)g * B + i];
      row.scale = sc;
      terms[i].push_back({row, giants[g].rot});
      for (std::size_t j = 0; j < giants[g].terms.size(); ++j) {
        ctx.stats.mult_plain++;
        ctx.record(1, lv - 1);
      }
    }
  return rotate_sum_to_target(ctx, terms, true, with_conj);
}

// out[r] = sum_k rot(groups[r][k].first, groups[r][k].second): every group's
// rotations share one ModDown; repeated inputs share one ModUp.  All terms of
// a group must share level and scale.  Records one rotation event per term.
std::vector<Ciphertext> rotate_sum_many(Context& ctx, const std::vector<std::vector<std::pair<Ciphertext, long>>>& groups) {
  const long S = ctx.S();
  std::vector<Ciphertext> outs(groups.size());
  std::vector<std::vector<Ciphertext>> direct(groups.size());  // identity terms
  std::map<int, std::vector<std::size_t>> by_level;              // groups with key-switched terms
  for (std::size_t r = 0; r < groups.size(); ++r) {
    if (groups[r].empty()) throw Error(ErrKind::internal, "rotate_sum: empty group");
    const Ciphertext& x0 = groups[r][0].first;
    bool ks = false;
    for (const auto& [x, tt] : groups[r]) {
      require_valid(x, "rotate");
      if (tt <= -S || tt >= S)
        throw Error(ErrKind::invalid_rotation,
                    "rotation amount " + std::to_string(tt) + " out of range for " + std::to_string(S) + " slots");
      if (x.limbs != x0.limbs) throw Error(ErrKind::internal, "rotate_sum: terms at different levels");
      check_scales(x, x0, "rotate_sum");
      ctx.record(0, tt);
      ctx.stats.rotations++;
      if (ctx.galois(tt) == 1) direct[r].push_back(x);
      else ks = true;
    }
    if (ks) by_level[x0.limbs].push_back(r);
  }
  for (auto& [limbs, rs] : by_level) {
    std::vector<const u64*> inputs, c0s;
    std::map<const u64*, int> slot;
    std::vector<SumJob> jobs;
    std::vector<std::size_t> owner;  // sub-group -> group (groups larger than one launch are split)
    for (std::size_t gi = 0; gi < rs.size(); ++gi) {
      int in_sub = kMaxSumJobs;
      for (const auto& [x, tt] : groups[rs[gi]]) {
        const u64 g = ctx.galois(tt);
        if (g == 1) continue;
        auto it = slot.find(x.c1);
        int in;
        if (it == slot.end()) {
          in = (int)inputs.size();
          slot[x.c1] = in;
          inputs.push_back(x.c1);
          c0s.push_back(x.c0);
        } else {
          in = it->second;
        }
        if (in_sub == kMaxSumJobs) {
          owner.push_back(rs[gi]);
          in_sub = 0;
        }
        jobs.push_back({g, in, (int)owner.size() - 1});
        ++in_sub;
      }
    }
    std::vector<Ciphertext> r = keyswitch_sum(ctx, inputs, c0s, limbs, jobs, (int)owner.size());
    for (std::size_t sg = 0; sg < owner.size(); ++sg) {
      r[sg].scale = groups[owner[sg]][0].first.scale;
      Ciphertext& o = outs[owner[sg]];
      o = o.valid() ? add(ctx, o, r[sg]) : r[sg];
    }
  }
  for (std::size_t r = 0; r < groups.size(); ++r)
    for (const Ciphertext& d : direct[r]) outs[r] = outs[r].valid() ? add(ctx, outs[r], d) : d;
  return outs;
}

// rescale_to_target(rotate_sum_many(groups)) with the rescale folded into each group's
// ModDown (moddown_rescale_accs): one rounding by P q_l, no rescale NTTs.  Every term
// of a group shares level and scale (the unrescaled MAC outputs of a layer or a
// linear transform); outputs land on T_{l-1}.  Records one rotation event per term.
std::vector<Ciphertext> rotate_sum_to_target(Context& ctx,
                                             const std::vector<std::vector<std::pair<Ciphertext, long>>>& groups,
                                             bool record_identity, bool with_conj) {
  if (groups.empty()) return {};
  const long S = ctx.S();
  const int limbs = groups[0].at(0).first.limbs;
  bool fused = limbs >= 2 && bconv_tc_enabled() && ctx.K() + 1 + 2 <= 16;
  for (const auto& g : groups) {
    if (g.empty()) throw Error(ErrKind::internal, "rotate_sum: empty group");
    for (const auto& [x, tt] : g) fused = fused && x.limbs == limbs;
  }
  const u64 conj = 2 * (u64)ctx.N() - 1;
  const u64 twoN = 2 * (u64)ctx.N();
  if (!fused && with_conj) {  // out + conj(out) the plain way
    std::vector<Ciphertext> o = rescale_to_target(ctx, rotate_sum_many(ctx, groups));
    std::vector<Ciphertext> c = conjugate_many(ctx, o);
    return add_many(ctx, o, c);
  }
  if (!fused) return rescale_to_target(ctx, rotate_sum_many(ctx, groups));
  std::vector<const u64*> inputs, c0s;
  std::map<const u64*, int> slot;
  std::vector<SumJob> jobs;
  std::vector<int> gidx(groups.size(), -1);  // group -> accumulator
  std::vector<Ciphertext> direct(groups.size());
  int nacc = 0;
  for (std::size_t r = 0; r < groups.size(); ++r) {
    const Ciphertext& x0 = groups[r][0].first;
    int in_group = 0;
    for (const auto& [x, tt] : groups[r]) {
      require_valid(x, "rotate");
      if (tt <= -S || tt >= S)
        throw Error(ErrKind::invalid_rotation,
                    "rotation amount " + std::to_string(tt) + " out of range for " + std::to_string(S) + " slots");
      check_scales(x, x0, "rotate_sum");
      const u64 g = ctx.galois(tt);
      if (g != 1 || record_identity) {
        ctx.record(0, tt);
        ctx.stats.rotations++;
      }
      if (with_conj) ++in_group;  // the conjugated term is always key-switched
      if (g == 1) {
        direct[r] = direct[r].valid() ? add(ctx, direct[r], x) : x;
        continue;
      }
      ++in_group;
    }
    if (in_group > kMaxSumJobs) {
      if (with_conj) {
        std::vector<Ciphertext> o = rescale_to_target(ctx, rotate_sum_many(ctx, groups));
        return add_many(ctx, o, conjugate_many(ctx, o));
      }
      return rescale_to_target(ctx, rotate_sum_many(ctx, groups));
    }
    if (in_group == 0) continue;
    gidx[r] = nacc++;
    for (const auto& [x, tt] : groups[r]) {
      const u64 g = ctx.galois(tt);
      if (g == 1 && !with_conj) continue;
      auto it = slot.find(x.c1);
      int in;
      if (it == slot.end()) {
        in = (int)inputs.size();
        slot[x.c1] = in;
        inputs.push_back(x.c1);
        c0s.push_back(x.c0);
      } else {
        in = it->second;
      }
      if (g != 1) jobs.push_back({g, in, gidx[r]});
      if (with_conj) jobs.push_back({(g * conj) % twoN, in, gidx[r]});  // conj o rot_t
    }
  }
  const int lv = limbs - 1;
  std::vector<Ciphertext> outs(groups.size());
  if (nacc > 0) {
    BufPtr accs = keyswitch_sum_accs(ctx, inputs, c0s, limbs, jobs, nacc);
    const std::size_t stride = (std::size_t)2 * (limbs + ctx.K()) * ctx.N();
    std::vector<u64*> accp(nacc);
    std::vector<Ciphertext> adds(nacc);
    for (std::size_t r = 0; r < groups.size(); ++r)
      if (gidx[r] >= 0) {
        accp[gidx[r]] = accs->ptr + (std::size_t)gidx[r] * stride;
        adds[gidx[r]] = direct[r];
      }
    std::vector<Ciphertext> rs = moddown_rescale_accs(ctx, accp, adds, limbs);
    for (std::size_t r = 0; r < groups.size(); ++r)
      if (gidx[r] >= 0) outs[r] = rs[gidx[r]];
  }
  for (std::size_t r = 0; r < groups.size(); ++r)
    if (gidx[r] < 0) outs[r] = rescale_many(ctx, {direct[r]})[0];
  for (Ciphertext& o : outs) o.scale = ctx.host().T[lv - 1];
  return outs;
}

// ---------------------------------------------------------------- rescale
Ciphertext rescale(Context& ctx, const Ciphertext& a) {
  require_valid(a, "rescale");
  if (a.limbs < 2) throw Error(ErrKind::depth_exhausted, "rescale: no limb left to drop");
  return rescale_many(ctx, {a})[0];
}

// -------------------------------------------------------------- level down
Ciphertext level_down(Context& ctx, const Ciphertext& a, int target) {
  require_valid(a, "level_down");
  if (target == a.limbs) return a;
  if (target > a.limbs || target < 1) throw Error(ErrKind::internal, "level_down: bad target");
  const int keep = target + 1;
  const HostTables& h = ctx.host();
  const double c = h.T[target - 1] * (double)h.q[target] / a.scale;
  // the integer constant k carries the scale change; below 2^30 its rounding would move
  // the result off T_{target-1} by more than 2^-31 relative (an unrescaled product
  // reaching add/sub, say), above 2^62 it does not fit a signed word -- both are bugs
  // of the caller, not something to absorb silently
  if (!(c >= 1073741824.0) || !(c < 4.6e18))
    throw Error(ErrKind::internal, "level_down: scale 2^" + std::to_string(std::log2(a.scale)) + " at " +
                                       std::to_string(a.limbs) + " limbs cannot be brought to the target scale of " +
                                       std::to_string(target) + " limbs with an integer constant (rescale first)");
  const long long k = std::llround(c);
  LimbConsts lc{};
  for (int i = 0; i < keep; ++i) {
    lc.c[i] = signed_mod(k, h.q[i]);
    lc.sh[i] = shoup(lc.c[i], h.q[i]);
  }
  Ciphertext tmp = ctx.new_ct(keep);
  ew_mul_const(ctx.dev(), plist({tmp.c0, tmp.c1}), plist({a.c0, a.c1}), lc, keep, ctx.stream());
  Ciphertext out = rescale(ctx, tmp);
  out.scale = h.T[target - 1];
  return out;
}

namespace {
void align(Context& ctx, Ciphertext& a, Ciphertext& b) {
  if (a.limbs > b.limbs) a = level_down(ctx, a, b.limbs);
  else if (b.limbs > a.limbs) b = level_down(ctx, b, a.limbs);
}
}  // namespace

// --------------------------------------------------------------- encrypt
Ciphertext encrypt_top(Context& ctx, const double* vals, std::size_t n) { return encrypt_at(ctx, vals, n, ctx.L()); }

// secret-key encryption over the first L limbs at the level's scale target (the same
// randomness streams as a top-level encryption restricted to those limbs)
Ciphertext encrypt_at(Context& ctx, const double* vals, std::size_t n, int L) {
  ctx.require_secret("encrypt");
  if (L < 1 || L > ctx.L()) throw Error(ErrKind::internal, "encrypt: bad limb count");
  const std::size_t N = ctx.N();
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const u64 counter = ctx.enc_counter++;
  BufPtr m = ctx.encode(vals, n, L, ctx.host().T[L - 1]);
  BufPtr e = ctx.alloc((std::size_t)L * N);
  const u64 seed = ctx.host().p.seed;
  sample_error(t, e->ptr, prng_stream_key(seed, stream_enc(counter, 5)), L, L, st);
  ntt_forward(t, limbset(e->ptr, 1, 0, L, L, L), st);
  Ciphertext ct = ctx.new_ct(L);
  encrypt_combine(t, ct.c0, ct.c1, m->ptr, e->ptr, prng_stream_key(seed, stream_enc(counter, 4)), L, st);
  ct.scale = ctx.host().T[L - 1];
  return ct;
}

Ciphertext encrypt(Context& ctx, const double* vals, std::size_t n) {
  if (n > (std::size_t)ctx.S())
    throw Error(ErrKind::capacity, "payload of " + std::to_string(n) + " values does not fit in " +
                                       std::to_string(ctx.S()) + " slots");
  // directly at the depth budget: a top-level encryption brought down by level_down
  // would carry its scale change in a small integer constant (2^22 on 60-bit
  // bootstrapping chains) and lose precision
  return encrypt_at(ctx, vals, n, ctx.depth_budget() + 1);
}

void decrypt(Context& ctx, const Ciphertext& ct, double* out, double* out_im) {
  require_valid(ct, "decrypt");
  ctx.require_secret("decrypt");
  const std::size_t N = ctx.N();
  const int use = ct.limbs >= 2 ? 2 : 1;
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  BufPtr m = ctx.alloc((std::size_t)use * N);
  decrypt_core(t, m->ptr, ct.c0, ct.c1, use, st);
  ntt_inverse(t, limbset(m->ptr, 1, 0, use, use, ctx.L()), st);
  std::vector<u64> h((std::size_t)use * N);
  FHEON_CUDA(cudaMemcpyAsync(h.data(), m->ptr, h.size() * sizeof(u64), cudaMemcpyDeviceToHost, st));
  FHEON_CUDA(cudaStreamSynchronize(st));
  std::vector<double> coeffs(N);
  const std::vector<u64>& q = ctx.host().q;
  if (use == 1) {
    for (std::size_t k = 0; k < N; ++k) coeffs[k] = h[k] > q[0] / 2 ? -(double)(q[0] - h[k]) : (double)h[k];
  } else {
    const u64 q0 = q[0], q1 = q[1];
    const u64 q0inv = invmod(q0 % q1, q1);
    const u128 Q = (u128)q0 * q1;
    for (std::size_t k = 0; k < N; ++k) {
      const u64 x0 = h[k], x1 = h[N + k];
      const u64 tt = mulmod(submod(x1, x0 % q1, q1), q0inv, q1);
      const u128 X = (u128)x0 + (u128)q0 * tt;
      coeffs[k] = X > Q / 2 ? -(double)(Q - X) : (double)X;
    }
  }
  ctx.decode_coeffs(coeffs.data(), ct.scale, out, out_im);
}

// ---------------------------------------------------------------- rotate
Ciphertext rotate(Context& ctx, const Ciphertext& x, long t) {
  return rotate_hoisted(ctx, x, std::vector<long>{t})[0];
}

// Rotation i: xs[i] by ts[i].  Distinct inputs are key-switched in one batched
// pipeline; repeated inputs share their ModUp (hoisting).  Trace events are
// recorded in call order, exactly as sequential rotate() calls would.
std::vector<Ciphertext> rotate_many(Context& ctx, const std::vector<Ciphertext>& xs, const std::vector<long>& ts) {
  if (xs.size() != ts.size()) throw Error(ErrKind::internal, "rotate_many: size mismatch");
  const long S = ctx.S();
  for (std::size_t i = 0; i < ts.size(); ++i) {
    require_valid(xs[i], "rotate");
    if (ts[i] <= -S || ts[i] >= S)
      throw Error(ErrKind::invalid_rotation,
                  "rotation amount " + std::to_string(ts[i]) + " out of range for " + std::to_string(S) + " slots");
  }
  std::vector<Ciphertext> outs(ts.size());
  // group by level; within a level, dedupe inputs by their c1 pointer
  std::map<int, std::vector<std::size_t>> by_level;
  for (std::size_t i = 0; i < ts.size(); ++i) {
    ctx.record(0, ts[i]);
    ctx.stats.rotations++;
    if (ctx.galois(ts[i]) == 1) {
      outs[i] = xs[i];
      outs[i].id = ctx.next_id();
      continue;
    }
    by_level[xs[i].limbs].push_back(i);
  }
  for (auto& [limbs, idx] : by_level) {
    std::vector<const u64*> inputs;
    std::map<const u64*, int> slot;
    std::vector<KsJob> jobs;
    for (std::size_t i : idx) {
      const Ciphertext& x = xs[i];
      auto it = slot.find(x.c1);
      int in;
      if (it == slot.end()) {
        in = (int)inputs.size();
        slot[x.c1] = in;
        inputs.push_back(x.c1);
      } else {
        in = it->second;
      }
      const u64 g = ctx.galois(ts[i]);
      KsJob jb{g, g, x.c0, g, nullptr};
      jb.in = in;
      jobs.push_back(jb);
    }
    std::vector<Ciphertext> r = keyswitch(ctx, inputs, limbs, jobs);
    for (std::size_t k = 0; k < r.size(); ++k) {
      r[k].scale = xs[idx[k]].scale;
      outs[idx[k]] = r[k];
    }
  }
  return outs;
}

std::vector<Ciphertext> rotate_hoisted(Context& ctx, const Ciphertext& x, const std::vector<long>& ts) {
  return rotate_many(ctx, std::vector<Ciphertext>(ts.size(), x), ts);
}

// complex conjugation of the slots: automorphism X -> X^{2N-1} + key switch
std::vector<Ciphertext> conjugate_many(Context& ctx, const std::vector<Ciphertext>& xs) {
  const u64 g = 2 * (u64)ctx.N() - 1;
  std::vector<Ciphertext> outs(xs.size());
  std::map<int, std::vector<std::size_t>> by_level;
  for (std::size_t i = 0; i < xs.size(); ++i) by_level[xs[i].limbs].push_back(i);
  for (auto& [limbs, idx] : by_level) {
    std::vector<const u64*> inputs;
    std::vector<KsJob> jobs;
    for (std::size_t k = 0; k < idx.size(); ++k) {
      inputs.push_back(xs[idx[k]].c1);
      KsJob jb{g, g, xs[idx[k]].c0, g, nullptr};
      jb.in = (int)k;
      jobs.push_back(jb);
    }
    std::vector<Ciphertext> r = keyswitch(ctx, inputs, limbs, jobs);
    for (std::size_t k = 0; k < idx.size(); ++k) {
      r[k].scale = xs[idx[k]].scale;
      outs[idx[k]] = r[k];
    }
  }
  return outs;
}

// slot-wise multiplication by i: exact monomial X^{N/2} product, no level used
Ciphertext mul_by_i(Context& ctx, const Ciphertext& x) {
  const HostTables& h = ctx.host();
  LimbConsts iq{};
  for (int i = 0; i < x.limbs; ++i) {
    iq.c[i] = powmod(h.psi[i], ctx.N() / 2, h.q[i]);
    iq.sh[i] = shoup(iq.c[i], h.q[i]);
  }
  Ciphertext out = ctx.new_ct(x.limbs);
  mul_monomial_half(ctx.dev(), plist({out.c0, out.c1}), plist({x.c0, x.c1}), iq, x.limbs, ctx.stream());
  out.scale = x.scale;
  return out;
}

namespace {
// key switch of every x to the secret a key encapsulates: (c0 + ks0, ks1), automorphism-free
std::vector<Ciphertext> switch_secret_many(Context& ctx, const std::vector<Ciphertext>& xs, u64 key_id) {
  std::vector<const u64*> inputs;
  std::vector<KsJob> jobs;
  for (std::size_t i = 0; i < xs.size(); ++i) {
    inputs.push_back(xs[i].c1);
    KsJob jb{key_id, 1, xs[i].c0, 1, nullptr};
    jb.in = (int)i;
    jobs.push_back(jb);
  }
  std::vector<Ciphertext> ys = keyswitch(ctx, inputs, xs[0].limbs, jobs);
  for (std::size_t i = 0; i < xs.size(); ++i) ys[i].scale = xs[i].scale;
  return ys;
}
Ciphertext switch_secret(Context& ctx, const Ciphertext& x, u64 key_id) {
  return switch_secret_many(ctx, {x}, key_id)[0];
}
Ciphertext mod_raise_raw(Context& ctx, const Ciphertext& x);
std::vector<Ciphertext> mod_raise_raw_many(Context& ctx, const std::vector<Ciphertext>& xs);
}  // namespace

// ModRaise followed by the trace sum_{j < S/n} rot(., j n) of sparse-slot bootstrapping.
// Under the encapsulation (dense main secret) the raised ciphertext is under s_b; each
// trace term is key-switched from sigma_{5^{jn}}(s_b) straight to s (j = 0: the plain
// switch back), so the switch back costs no key switch of its own: one ModUp, S/n key
// inner products, one ModDown.
Ciphertext mod_raise_trace(Context& ctx, const Ciphertext& x, long n) {
  return mod_raise_trace_many(ctx, {x}, n)[0];
}

// several level-0 ciphertexts in lockstep (one group per input under the same key list)
std::vector<Ciphertext> mod_raise_trace_many(Context& ctx, const std::vector<Ciphertext>& xs, long n) {
  const long S = ctx.S();
  if (xs.empty()) return {};
  for (const Ciphertext& x : xs)
    if (x.limbs != 1) throw Error(ErrKind::internal, "mod_raise expects a level-0 ciphertext");
  if (n <= 0 || S % n != 0) throw Error(ErrKind::internal, "mod_raise_trace: n must divide the slot count");
  const int B = (int)xs.size();
  if (!ctx.sse()) {
    std::vector<Ciphertext> ys = mod_raise_raw_many(ctx, xs);
    if (n == S) return ys;
    std::vector<std::vector<std::pair<Ciphertext, long>>> groups(B);
    for (int i = 0; i < B; ++i)
      for (long j = 0; j < S / n; ++j) groups[i].push_back({ys[i], j * n});
    return rotate_sum_many(ctx, groups);
  }
  std::vector<Ciphertext> ys = mod_raise_raw_many(ctx, switch_secret_many(ctx, xs, kKeyToSparse));
  std::vector<SumJob> jobs;
  std::vector<const u64*> c1s, c0s;
  for (int i = 0; i < B; ++i) {
    c1s.push_back(ys[i].c1);
    c0s.push_back(ys[i].c0);
    for (long j = 0; j < S / n; ++j) {
      const u64 g = ctx.galois(j * n);
      SumJob jb{g, i, i};
      jb.key_id = j == 0 ? kKeyFromSparse : key_from_sparse_rot(g);
      jobs.push_back(jb);
      if (j > 0) ctx.stats.rotations++;
    }
  }
  std::vector<Ciphertext> outs = keyswitch_sum(ctx, c1s, c0s, ys[0].limbs, jobs, B);
  for (int i = 0; i < B; ++i) outs[i].scale = ys[i].scale;
  return outs;
}

// ModRaise of a level-0 ciphertext to all L limbs (decrypts to m + q_0 I).  With a
// dense main secret (sparse-secret encapsulation, Bossuat et al. 2022) the level-0
// ciphertext is first switched to the sparse bootstrapping secret s_b -- on q_0 only,
// so |I| stays within the EvalMod range -- raised under s_b, and switched back to
// the dense secret over the whole chain.
Ciphertext mod_raise(Context& ctx, const Ciphertext& x) {
  if (x.limbs != 1) throw Error(ErrKind::internal, "mod_raise expects a level-0 ciphertext");
  if (!ctx.sse()) return mod_raise_raw(ctx, x);
  Ciphertext y = mod_raise_raw(ctx, switch_secret(ctx, x, kKeyToSparse));
  return switch_secret(ctx, y, kKeyFromSparse);
}

namespace {
Ciphertext mod_raise_raw(Context& ctx, const Ciphertext& x) { return mod_raise_raw_many(ctx, {x})[0]; }

std::vector<Ciphertext> mod_raise_raw_many(Context& ctx, const std::vector<Ciphertext>& xs) {
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  const int L = ctx.L();
  std::vector<Ciphertext> outs;
  for (std::size_t i0 = 0; i0 < xs.size(); i0 += kMaxBases) {
    const int B = (int)std::min<std::size_t>(kMaxBases, xs.size() - i0);
    BufPtr coef = ctx.alloc((std::size_t)B * 2 * N);
    LimbSet dst = limbset(coef->ptr, 2 * B, N, 1, 1, L);
    LimbSet src = dst;
    src.nbase = B;
    src.blocks_per_base = 2;
    const long long cstride = (long long)(xs[i0].c1 - xs[i0].c0);
    src.block_stride = cstride;
    for (int i = 0; i < B; ++i) {
      const Ciphertext& x = xs[i0 + i];
      if ((long long)(x.c1 - x.c0) != cstride) throw Error(ErrKind::internal, "mod_raise: mixed ciphertext strides");
      src.base[i] = x.c0;
    }
    ntt_inverse(t, dst, st, &src);
    LimbSet fw{};
    long long ostride = 0;
    for (int i = 0; i < B; ++i) {
      Ciphertext out = ctx.new_ct(L);
      modraise(t, plist({out.c0, out.c1}),
               plist({coef->ptr + (std::size_t)(2 * i) * N, coef->ptr + (std::size_t)(2 * i + 1) * N}), L, st);
      if (i == 0) {
        ostride = (long long)(out.c1 - out.c0);
        fw = limbset(out.c0, 2, (std::size_t)ostride, L, L, L);
      } else if ((long long)(out.c1 - out.c0) != ostride) {
        throw Error(ErrKind::internal, "mod_raise: mixed ciphertext strides");
      }
      fw.base[i] = out.c0;
      out.scale = (double)ctx.host().q[0];
      outs.push_back(out);
    }
    fw.nbase = B;
    ntt_forward(t, fw, st);
  }
  return outs;
}
}  // namespace

Ciphertext keyswitch_raw(Context& ctx, const Ciphertext& d, u64 key_id, u64 g) {
  std::vector<Ciphertext> r = keyswitch(ctx, {d.c1}, d.limbs, {{key_id, g, nullptr, 1, nullptr}});
  r[0].scale = d.scale;
  return r[0];
}

// ---------------------------------------------------------------- add/sub
Ciphertext add(Context& ctx, const Ciphertext& a0, const Ciphertext& b0) {
  require_valid(a0, "add");
  require_valid(b0, "add");
  Ciphertext a = a0, b = b0;
  align(ctx, a, b);
  check_scales(a, b, "add");
  Ciphertext out = ctx.new_ct(a.limbs);
  ew_add(ctx.dev(), plist({out.c0, out.c1}), plist({a.c0, a.c1}), plist({b.c0, b.c1}), a.limbs, ctx.stream());
  out.scale = a.scale;
  ctx.stats.adds++;
  return out;
}

Ciphertext sub(Context& ctx, const Ciphertext& a0, const Ciphertext& b0) {
  require_valid(a0, "sub");
  require_valid(b0, "sub");
  Ciphertext a = a0, b = b0;
  align(ctx, a, b);
  check_scales(a, b, "sub");
  Ciphertext out = ctx.new_ct(a.limbs);
  ew_sub(ctx.dev(), plist({out.c0, out.c1}), plist({a.c0, a.c1}), plist({b.c0, b.c1}), a.limbs, ctx.stream());
  out.scale = a.scale;
  ctx.stats.adds++;
  return out;
}

Ciphertext add_plain(Context& ctx, const Ciphertext& a, const double* vals, std::size_t n) {
  require_valid(a, "add_plain");
  BufPtr pt = ctx.encode(vals, n, a.limbs, a.scale);
  Ciphertext out = ctx.new_ct(a.limbs);
  ew_add(ctx.dev(), plist({out.c0}), plist({a.c0}), plist({pt->ptr}), a.limbs, ctx.stream());
  FHEON_CUDA(cudaMemcpyAsync(out.c1, a.c1, (std::size_t)a.limbs * ctx.N() * sizeof(u64), cudaMemcpyDeviceToDevice,
                             ctx.stream()));
  out.scale = a.scale;
  return out;
}

Ciphertext add_const(Context& ctx, const Ciphertext& a, double c) {
  require_valid(a, "add_const");
  const long long k = std::llround(c * a.scale);
  LimbConsts lc{};
  for (int i = 0; i < a.limbs; ++i) lc.c[i] = signed_mod(k, ctx.host().q[i]);
  Ciphertext out = ctx.new_ct(a.limbs);
  ew_add_const(ctx.dev(), plist({out.c0}), plist({a.c0}), lc, a.limbs, ctx.stream());
  FHEON_CUDA(cudaMemcpyAsync(out.c1, a.c1, (std::size_t)a.limbs * ctx.N() * sizeof(u64), cudaMemcpyDeviceToDevice,
                             ctx.stream()));
  out.scale = a.scale;
  return out;
}

// ------------------------------------------------------------- multiply
Ciphertext mult_const(Context& ctx, const Ciphertext& a, double c) {
  require_valid(a, "mult_plain");
  require_depth(a, "mult_plain");
  const HostTables& h = ctx.host();
  const int lv = a.level();
  const double pt_scale = h.T[lv - 1] * (double)h.q[lv] / a.scale;
  const double x = c * pt_scale;
  if (!(std::fabs(x) < 4611686018427387904.0)) throw Error(ErrKind::capacity, "constant exceeds 2^62");
  const long long k = std::llround(x);
  LimbConsts lc{};
  for (int i = 0; i < a.limbs; ++i) {
    lc.c[i] = signed_mod(k, h.q[i]);
    lc.sh[i] = shoup(lc.c[i], h.q[i]);
  }
  Ciphertext prod = ctx.new_ct(a.limbs);
  ew_mul_const(ctx.dev(), plist({prod.c0, prod.c1}), plist({a.c0, a.c1}), lc, a.limbs, ctx.stream());
  Ciphertext out = rescale(ctx, prod);
  out.scale = h.T[lv - 1];
  ctx.stats.mult_plain++;
  ctx.record(1, lv - 1);
  return out;
}

Ciphertext mult_plain(Context& ctx, const Ciphertext& a, const double* vals, std::size_t n) {
  require_valid(a, "mult_plain");
  if (n != (std::size_t)ctx.S())
    throw Error(ErrKind::shape, "mult_plain: plaintext length " + std::to_string(n) + " does not match slot count " +
                                    std::to_string(ctx.S()));
  require_depth(a, "mult_plain");
  bool constant = true;
  for (std::size_t i = 1; i < n && constant; ++i) constant = vals[i] == vals[0];
  if (constant) return mult_const(ctx, a, vals[0]);
  const HostTables& h = ctx.host();
  const int lv = a.level();
  const double pt_scale = h.T[lv - 1] * (double)h.q[lv] / a.scale;
  BufPtr pt = ctx.encode(vals, n, a.limbs, pt_scale);
  Ciphertext prod = ctx.new_ct(a.limbs);
  ew_mul_pt(ctx.dev(), plist({prod.c0, prod.c1}), plist({a.c0, a.c1}), pt->ptr, a.limbs, ctx.stream());
  Ciphertext out = rescale(ctx, prod);
  out.scale = h.T[lv - 1];
  ctx.stats.mult_plain++;
  ctx.record(1, lv - 1);
  return out;
}

Ciphertext mult_cipher(Context& ctx, const Ciphertext& a0, const Ciphertext& b0) {
  require_valid(a0, "mult_cipher");
  require_valid(b0, "mult_cipher");
  require_depth(a0, "mult_cipher");
  require_depth(b0, "mult_cipher");
  Ciphertext a = a0, b = b0;
  align(ctx, a, b);
  const int l = a.limbs;
  const std::size_t N = ctx.N();
  BufPtr d = ctx.alloc(3 * (std::size_t)l * N);
  u64* d0 = d->ptr;
  u64* d1 = d0 + (std::size_t)l * N;
  u64* d2 = d1 + (std::size_t)l * N;
  ew_tensor(ctx.dev(), d0, d1, d2, a.c0, a.c1, b.c0, b.c1, l, ctx.stream());
  std::vector<Ciphertext> r = keyswitch(ctx, {d2}, l, {{0, 1, d0, 1, d1}});
  Ciphertext out = rescale(ctx, r[0]);
  out.scale = a.scale * b.scale / (double)ctx.host().q[l - 1];
  ctx.stats.mult_cipher++;
  ctx.record(2, out.level());
  return out;
}

// ------------------------------------------------------------- batched ops
double pt_scale_for(const Context& ctx, const Ciphertext& a) {
  const HostTables& h = ctx.host();
  const int lv = a.level();
  return h.T[lv - 1] * (double)h.q[lv] / a.scale;
}

std::vector<Ciphertext> rescale_many(Context& ctx, const std::vector<Ciphertext>& as) {
  std::vector<Ciphertext> outs;
  outs.reserve(as.size());
  if (as.empty()) return outs;
  const int l = as[0].limbs;
  for (const Ciphertext& a : as) {
    require_valid(a, "rescale");
    if (a.limbs != l) throw Error(ErrKind::internal, "rescale_many: mixed levels");
  }
  if (l < 2) throw Error(ErrKind::depth_exhausted, "rescale: no limb left to drop");
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  constexpr int kChunk = kMaxBases;  // 32 ciphertexts = 64 polys per launch group
  for (std::size_t c0 = 0; c0 < as.size(); c0 += kChunk) {
    const int R = (int)std::min<std::size_t>(kChunk, as.size() - c0);
    BufPtr last = ctx.alloc((std::size_t)2 * R * N);
    // out-of-place iNTT of each poly's last limb straight from the ciphertexts
    LimbSet dst = limbset(last->ptr, 2 * R, N, 1, 1, ctx.L(), l - 1);
    LimbSet src = dst;
    src.nbase = R;
    src.blocks_per_base = 2;
    for (int r = 0; r < R; ++r) src.base[r] = as[c0 + r].c0 + (std::size_t)(l - 1) * N;
    src.block_stride = 0;
    bool uniform = true;
    for (int r = 0; r < R; ++r)
      uniform = uniform && (as[c0 + r].c1 - as[c0 + r].c0) == (as[c0].c1 - as[c0].c0);
    if (uniform) {
      src.block_stride = (long long)(as[c0].c1 - as[c0].c0);
      ntt_inverse(t, dst, st, &src);
    } else {
      for (int r = 0; r < R; ++r) {
        LimbSet d1 = limbset(last->ptr + (std::size_t)2 * r * N, 2, N, 1, 1, ctx.L(), l - 1);
        LimbSet s1 = d1;
        s1.base[0] = as[c0 + r].c0 + (std::size_t)(l - 1) * N;
        s1.block_stride = (long long)(as[c0 + r].c1 - as[c0 + r].c0);
        ntt_inverse(t, d1, st, &s1);
      }
    }
    BufPtr rb = ctx.alloc((std::size_t)2 * R * (l - 1) * N);
    PolyList rl{}, ll{}, ol{}, al{};
    rl.n = ll.n = ol.n = al.n = 2 * R;
    for (int r = 0; r < R; ++r) {
      Ciphertext o = ctx.new_ct(l - 1);
      o.scale = as[c0 + r].scale;
      for (int p = 0; p < 2; ++p) {
        const int i = 2 * r + p;
        rl.p[i] = rb->ptr + (std::size_t)i * (l - 1) * N;
        ll.p[i] = last->ptr + (std::size_t)i * N;
        ol.p[i] = p ? o.c1 : o.c0;
        al.p[i] = const_cast<u64*>(p ? as[c0 + r].c1 : as[c0 + r].c0);
        rl.g[i] = ll.g[i] = ol.g[i] = al.g[i] = 1;
      }
      outs.push_back(o);
    }
    rescale_lift(t, rl, ll, l, st);
    ntt_forward_epilogue(t, limbset(rb->ptr, 2 * R, (std::size_t)(l - 1) * N, l - 1, l - 1, ctx.L()),
                         rescale_epilogue(t, ol, al, l), st);
    ctx.stats.rescales += R;
    ctx.stats.ntt_limbs += (std::size_t)R * 2 * l;
  }
  return outs;
}

std::vector<Ciphertext> mac_plain_many(Context& ctx, const std::vector<std::vector<Ciphertext>>& terms,
                                       const std::vector<std::vector<BufPtr>>& pts) {
  std::vector<Ciphertext> prods = mac_plain_many_unrescaled(ctx, terms, pts);
  return rescale_to_target(ctx, prods);
}

std::vector<Ciphertext> rescale_to_target(Context& ctx, const std::vector<Ciphertext>& prods) {
  if (prods.empty()) return {};
  const int lv = prods[0].limbs - 1;
  std::vector<Ciphertext> outs = rescale_many(ctx, prods);
  for (Ciphertext& o : outs) o.scale = ctx.host().T[lv - 1];
  return outs;
}

std::vector<Ciphertext> mac_plain_many_unrescaled(Context& ctx, const std::vector<std::vector<Ciphertext>>& terms,
                                                  const std::vector<std::vector<BufPtr>>& pts) {
  if (terms.size() != pts.size()) throw Error(ErrKind::internal, "mac_plain_many: size mismatch");
  std::vector<Ciphertext> prods;
  prods.reserve(terms.size());
  if (terms.empty()) return prods;
  const Ciphertext& ref = terms[0].at(0);
  const int l = ref.limbs;
  for (std::size_t o = 0; o < terms.size(); ++o) {
    if (terms[o].empty() || terms[o].size() != pts[o].size())
      throw Error(ErrKind::internal, "mac_plain_many: term/plaintext count mismatch");
    for (const Ciphertext& c : terms[o]) {
      require_valid(c, "mult_plain");
      require_depth(c, "mult_plain");
      if (c.limbs != l) throw Error(ErrKind::internal, "mac_plain_many: terms at different levels");
      check_scales(c, ref, "mac_plain_many");
    }
  }
  const HostTables& h = ctx.host();
  const int lv = l - 1;
  for (std::size_t o0 = 0; o0 < terms.size(); o0 += kMacMaxOut) {
    MacJobs jobs{};
    jobs.nout = (int)std::min<std::size_t>(kMacMaxOut, terms.size() - o0);
    for (int z = 0; z < jobs.nout; ++z) prods.push_back(ctx.new_ct(l));
    // split long sums into kMacMaxTerms-term partial products accumulated in place
    std::size_t maxt = 0;
    for (int z = 0; z < jobs.nout; ++z) maxt = std::max(maxt, terms[o0 + z].size());
    for (std::size_t j0 = 0; j0 < maxt; j0 += kMacMaxTerms) {
      MacJobs jb{};
      int nz = 0;
      std::vector<Ciphertext> partial;
      for (int z = 0; z < jobs.nout; ++z) {
        const auto& tz = terms[o0 + z];
        if (j0 >= tz.size()) continue;
        const int nt = (int)std::min<std::size_t>(kMacMaxTerms, tz.size() - j0);
        Ciphertext& dst = prods[o0 + z];
        Ciphertext tmp = j0 == 0 ? dst : ctx.new_ct(l);
        for (int j = 0; j < nt; ++j) {
          jb.ct[nz][j] = tz[j0 + j].c0;
          jb.c1_off[nz][j] = (long long)(tz[j0 + j].c1 - tz[j0 + j].c0);
          jb.pt[nz][j] = pts[o0 + z][j0 + j]->ptr;
        }
        jb.nterm[nz] = nt;
        jb.out0[nz] = tmp.c0;
        jb.out1[nz] = tmp.c1;
        if (j0 > 0) partial.push_back(tmp);
        ++nz;
      }
      jb.nout = nz;
      mac_pt(ctx.dev(), jb, l, ctx.stream());
      if (j0 > 0) {  // fold the partial sums into the outputs
        int k = 0;
        for (int z = 0; z < jobs.nout; ++z) {
          if (j0 >= terms[o0 + z].size()) continue;
          Ciphertext& dst = prods[o0 + z];
          ew_add(ctx.dev(), plist({dst.c0, dst.c1}), plist({dst.c0, dst.c1}), plist({partial[k].c0, partial[k].c1}),
                 l, ctx.stream());
          ++k;
        }
      }
    }
  }
  // plaintexts were encoded at T_{lv-1} q_lv / scale: the products sit at T_{lv-1} q_lv
  for (Ciphertext& p : prods) p.scale = h.T[lv - 1] * (double)h.q[lv];
  for (std::size_t o = 0; o < prods.size(); ++o)
    for (std::size_t j = 0; j < terms[o].size(); ++j) {
      ctx.stats.mult_plain++;
      ctx.record(1, lv - 1);
    }
  return prods;
}

Ciphertext add_plain_pt(Context& ctx, const Ciphertext& a, const BufPtr& pt) {
  require_valid(a, "add_plain");
  Ciphertext out = ctx.new_ct(a.limbs);
  ew_add(ctx.dev(), plist({out.c0}), plist({a.c0}), plist({pt->ptr}), a.limbs, ctx.stream());
  FHEON_CUDA(cudaMemcpyAsync(out.c1, a.c1, (std::size_t)a.limbs * ctx.N() * sizeof(u64), cudaMemcpyDeviceToDevice,
                             ctx.stream()));
  out.scale = a.scale;
  return out;
}

// pairs (a_i, b_i) multiplied with one batched relinearisation key switch and
// one batched rescale; records one mult_cipher event per pair, in order.
std::vector<Ciphertext> mult_cipher_many(Context& ctx, const std::vector<Ciphertext>& as,
                                         const std::vector<Ciphertext>& bs) {
  if (as.size() != bs.size()) throw Error(ErrKind::internal, "mult_cipher_many: size mismatch");
  std::vector<Ciphertext> outs(as.size());
  if (as.empty()) return outs;
  std::vector<Ciphertext> A(as.size()), B(bs.size());
  for (std::size_t i = 0; i < as.size(); ++i) {
    require_valid(as[i], "mult_cipher");
    require_valid(bs[i], "mult_cipher");
    require_depth(as[i], "mult_cipher");
    require_depth(bs[i], "mult_cipher");
    A[i] = as[i];
    B[i] = bs[i];
    align(ctx, A[i], B[i]);
  }
  std::map<int, std::vector<std::size_t>> by_level;
  for (std::size_t i = 0; i < A.size(); ++i) by_level[A[i].limbs].push_back(i);
  const std::size_t N = ctx.N();
  for (auto& [l, idx] : by_level) {
    const std::size_t P = (std::size_t)l * N;
    BufPtr d = ctx.alloc(3 * P * idx.size());
    std::vector<const u64*> inputs;
    std::vector<KsJob> jobs;
    for (std::size_t k = 0; k < idx.size(); ++k) {
      const std::size_t i = idx[k];
      u64* d0 = d->ptr + 3 * P * k;
      ew_tensor(ctx.dev(), d0, d0 + P, d0 + 2 * P, A[i].c0, A[i].c1, B[i].c0, B[i].c1, l, ctx.stream());
      inputs.push_back(d0 + 2 * P);
      KsJob jb{0, 1, d0, 1, d0 + P};
      jb.in = (int)k;
      jobs.push_back(jb);
    }
    std::vector<Ciphertext> rs = keyswitch_relin_rescale(ctx, inputs, l, jobs);
    for (std::size_t k = 0; k < idx.size(); ++k) {
      const std::size_t i = idx[k];
      rs[k].scale = A[i].scale * B[i].scale / (double)ctx.host().q[l - 1];
      outs[i] = rs[k];
      ctx.stats.mult_cipher++;
    }
  }
  for (const Ciphertext& o : outs) ctx.record(2, o.level());
  return outs;
}

// 2 a_i b_i - s_i (s_i invalid: 2 a_i b_i) with the subtraction and the doubling folded
// into the tensor product, ahead of ONE relinearise-and-rescale: the Chebyshev
// recurrence step T_{a+b} = 2 T_a T_b - T_{a-b} without bringing T_{a-b} down a level
// (no level_down rescale).  s_i is read at the product's limbs (zero-copy drop) and
// multiplied by the integer k = round(scale(a) scale(b) / scale(s)) (>= 2^30 -- the
// same rounding level_down applies).  Same trace events as mult_cipher_many.
std::vector<Ciphertext> mult_cipher_cheb_many(Context& ctx, const std::vector<Ciphertext>& as,
                                              const std::vector<Ciphertext>& bs, const std::vector<Ciphertext>& subs) {
  if (as.size() != bs.size() || as.size() != subs.size())
    throw Error(ErrKind::internal, "mult_cipher_cheb_many: size mismatch");
  std::vector<Ciphertext> outs(as.size());
  if (as.empty()) return outs;
  std::vector<Ciphertext> A(as.size()), B(bs.size());
  for (std::size_t i = 0; i < as.size(); ++i) {
    require_valid(as[i], "mult_cipher");
    require_valid(bs[i], "mult_cipher");
    require_depth(as[i], "mult_cipher");
    require_depth(bs[i], "mult_cipher");
    A[i] = as[i];
    B[i] = bs[i];
    align(ctx, A[i], B[i]);
  }
  std::map<int, std::vector<std::size_t>> by_level;
  for (std::size_t i = 0; i < A.size(); ++i) by_level[A[i].limbs].push_back(i);
  const std::size_t N = ctx.N();
  const HostTables& h = ctx.host();
  for (auto& [l, idx] : by_level) {
    const std::size_t P = (std::size_t)l * N;
    BufPtr d = ctx.alloc(3 * P * idx.size());
    std::vector<const u64*> inputs;
    std::vector<KsJob> jobs;
    for (std::size_t k = 0; k < idx.size(); ++k) {
      const std::size_t i = idx[k];
      u64* d0 = d->ptr + 3 * P * k;
      const Ciphertext& s = subs[i];
      LimbConsts kc{};
      const u64 *s0 = nullptr, *s1 = nullptr;
      if (s.valid()) {
        if (s.limbs < l) throw Error(ErrKind::internal, "mult_cipher_cheb: subtrahend below the product");
        const double c = A[i].scale * B[i].scale / s.scale;
        if (!(c >= 1073741824.0) || !(c < 4.6e18))
          throw Error(ErrKind::internal, "mult_cipher_cheb: subtrahend scale out of range");
        const long long kk = std::llround(c);
        for (int q = 0; q < l; ++q) {
          kc.c[q] = signed_mod(kk, h.q[q]);
          kc.sh[q] = shoup(kc.c[q], h.q[q]);
        }
        s0 = s.c0;
        s1 = s.c1;
      }
      ew_tensor_cheb(ctx.dev(), d0, d0 + P, d0 + 2 * P, A[i].c0, A[i].c1, B[i].c0, B[i].c1, s0, s1, kc, l,
                     ctx.stream());
      inputs.push_back(d0 + 2 * P);
      KsJob jb{0, 1, d0, 1, d0 + P};
      jb.in = (int)k;
      jobs.push_back(jb);
    }
    std::vector<Ciphertext> rs = keyswitch_relin_rescale(ctx, inputs, l, jobs);
    for (std::size_t k = 0; k < idx.size(); ++k) {
      const std::size_t i = idx[k];
      rs[k].scale = A[i].scale * B[i].scale / (double)h.q[l - 1];
      outs[i] = rs[k];
      ctx.stats.mult_cipher++;
    }
  }
  for (const Ciphertext& o : outs) ctx.record(2, o.level());
  return outs;
}

// a_i * c_i (constant vectors) with one batched rescale per level
std::vector<Ciphertext> mult_const_many(Context& ctx, const std::vector<Ciphertext>& as, const std::vector<double>& cs) {
  std::vector<Ciphertext> outs(as.size());
  std::map<int, std::vector<std::size_t>> by_level;
  for (std::size_t i = 0; i < as.size(); ++i) {
    require_valid(as[i], "mult_plain");
    require_depth(as[i], "mult_plain");
    by_level[as[i].limbs].push_back(i);
  }
  const HostTables& h = ctx.host();
  for (auto& [l, idx] : by_level) {
    std::vector<Ciphertext> prods;
    for (std::size_t i : idx) {
      const double x = cs[i] * pt_scale_for(ctx, as[i]);
      if (!(std::fabs(x) < 4611686018427387904.0)) throw Error(ErrKind::capacity, "constant exceeds 2^62");
      const long long k = std::llround(x);
      LimbConsts lc{};
      for (int j = 0; j < l; ++j) {
        lc.c[j] = signed_mod(k, h.q[j]);
        lc.sh[j] = shoup(lc.c[j], h.q[j]);
      }
      Ciphertext p = ctx.new_ct(l);
      ew_mul_const(ctx.dev(), plist({p.c0, p.c1}), plist({as[i].c0, as[i].c1}), lc, l, ctx.stream());
      p.scale = as[i].scale;
      prods.push_back(p);
    }
    std::vector<Ciphertext> rs = rescale_many(ctx, prods);
    for (std::size_t k = 0; k < idx.size(); ++k) {
      rs[k].scale = h.T[l - 2];
      outs[idx[k]] = rs[k];
      ctx.stats.mult_plain++;
    }
  }
  for (const Ciphertext& o : outs) ctx.record(1, o.level());
  return outs;
}

// out = sum_i cs[i] * xs[i] + c0 with ONE rescale: every term is read at the
// lowest input level (limb drop, zero copy) and multiplied by the integer
// k_i = round(c_i * T_out * q_top / scale_i), so the rescaled sum lands on the
// target scale T_out of level (min level - 1) -- the level the reference's
// per-term const-mults + aligned adds reach.  Records one mult_plain event per term.
Ciphertext lincomb_const(Context& ctx, const std::vector<Ciphertext>& xs, const std::vector<double>& cs, double c0) {
  if (xs.empty() || xs.size() != cs.size()) throw Error(ErrKind::internal, "lincomb_const: bad term list");
  int l = xs[0].limbs;
  for (const Ciphertext& x : xs) {
    require_valid(x, "mult_plain");
    require_depth(x, "mult_plain");
    l = std::min(l, x.limbs);
  }
  return lincomb_const_to(ctx, xs, cs, c0, l - 1, ctx.host().T[l - 2]);
}

// The sum is formed at out_limbs + 1 limbs (terms' tails ignored), each constant
// scaled by out_scale q_{out_limbs} / scale(x_i) and rounded, then ONE rescale:
// the result lands exactly on (out_limbs, out_scale).
namespace {
// sum_i k_i x_i at out_limbs + 1 limbs with k_i = round(c_i out_scale q_{out_limbs} / scale(x_i)):
// the unrescaled part of lincomb_const_to
Ciphertext lincomb_const_sum(Context& ctx, const std::vector<Ciphertext>& xs, const std::vector<double>& cs,
                             int out_limbs, double out_scale) {
  if (xs.empty() || xs.size() != cs.size()) throw Error(ErrKind::internal, "lincomb_const: bad term list");
  const int l = out_limbs + 1;
  for (const Ciphertext& x : xs) {
    require_valid(x, "mult_plain");
    require_depth(x, "mult_plain");
    if (x.limbs < l) throw Error(ErrKind::internal, "lincomb_const: term below the target level");
  }
  const HostTables& h = ctx.host();
  const double t_out = out_scale;
  const std::size_t n = xs.size();
  std::vector<u64> kc(n * (std::size_t)l * 2);
  for (std::size_t i = 0; i < n; ++i) {
    const double x = cs[i] * t_out * (double)h.q[l - 1] / xs[i].scale;
    for (int t = 0; t < l; ++t) {
      const u64 v = round_mod(x, h.q[t]);
      kc[(i * l + t) * 2] = v;
      kc[(i * l + t) * 2 + 1] = shoup(v, h.q[t]);
    }
  }
  // through a pinned staging slot: a pageable copy would serialise host and stream
  if (kc.size() * sizeof(u64) > ctx.N() * sizeof(long long))
    throw Error(ErrKind::capacity, "lincomb_const: constant table exceeds a staging slot");
  BufPtr kd = ctx.alloc(kc.size());
  {
    cudaEvent_t* ev = nullptr;
    long long* stage = ctx.staging_slot(&ev);
    std::memcpy(stage, kc.data(), kc.size() * sizeof(u64));
    FHEON_CUDA(cudaMemcpyAsync(kd->ptr, stage, kc.size() * sizeof(u64), cudaMemcpyHostToDevice, ctx.stream()));
    FHEON_CUDA(cudaEventRecord(*ev, ctx.stream()));
  }
  Ciphertext sum = ctx.new_ct(l);
  sum.scale = t_out * (double)h.q[l - 1];
  for (std::size_t i0 = 0; i0 < n; i0 += kMaxLincomb) {
    LincombTerms lt{};
    lt.n = (int)std::min<std::size_t>(kMaxLincomb, n - i0);
    for (int j = 0; j < lt.n; ++j) {
      lt.c0[j] = xs[i0 + j].c0;
      lt.c1_off[j] = (long long)(xs[i0 + j].c1 - xs[i0 + j].c0);
    }
    if (i0 == 0) {
      lincomb_const(ctx.dev(), sum.c0, sum.c1, lt, kd->ptr, l, ctx.stream());
    } else {
      Ciphertext part = ctx.new_ct(l);
      lincomb_const(ctx.dev(), part.c0, part.c1, lt, kd->ptr + i0 * l * 2, l, ctx.stream());
      ew_add(ctx.dev(), plist({sum.c0, sum.c1}), plist({sum.c0, sum.c1}), plist({part.c0, part.c1}), l,
             ctx.stream());
    }
  }
  return sum;
}

Ciphertext lincomb_finish(Context& ctx, Ciphertext out, std::size_t nterms, double c0, double out_scale) {
  out.scale = out_scale;
  ctx.stats.mult_plain += nterms;
  for (std::size_t i = 0; i < nterms; ++i) ctx.record(1, out.level());
  return c0 != 0.0 ? add_const(ctx, out, c0) : out;
}
}  // namespace

Ciphertext lincomb_const_to(Context& ctx, const std::vector<Ciphertext>& xs, const std::vector<double>& cs, double c0,
                            int out_limbs, double out_scale) {
  Ciphertext sum = lincomb_const_sum(ctx, xs, cs, out_limbs, out_scale);
  return lincomb_finish(ctx, rescale(ctx, sum), xs.size(), c0, out_scale);
}

std::vector<Ciphertext> lincomb_const_to_many(Context& ctx, const std::vector<LincombItem>& items) {
  std::vector<Ciphertext> sums(items.size()), outs(items.size());
  std::map<int, std::vector<std::size_t>> by_level;
  for (std::size_t i = 0; i < items.size(); ++i) {
    sums[i] = lincomb_const_sum(ctx, items[i].xs, items[i].cs, items[i].out_limbs, items[i].out_scale);
    by_level[sums[i].limbs].push_back(i);
  }
  for (auto& [l, idx] : by_level) {  // one batched rescale per level
    std::vector<Ciphertext> in;
    for (std::size_t i : idx) in.push_back(sums[i]);
    std::vector<Ciphertext> r = rescale_many(ctx, in);
    for (std::size_t k = 0; k < idx.size(); ++k) {
      const LincombItem& it = items[idx[k]];
      outs[idx[k]] = lincomb_finish(ctx, r[k], it.xs.size(), it.c0, it.out_scale);
    }
  }
  return outs;
}

std::vector<Ciphertext> add_many(Context& ctx, const std::vector<Ciphertext>& a, const std::vector<Ciphertext>& b) {
  if (a.size() != b.size()) throw Error(ErrKind::internal, "add_many: size mismatch");
  std::vector<Ciphertext> outs(a.size());
  // same-level pairs in one launch (up to 32 pairs), others one by one
  std::vector<std::size_t> batch;
  for (std::size_t i = 0; i < a.size(); ++i) {
    if (a[i].limbs == b[i].limbs && a[i].limbs == a[0].limbs) batch.push_back(i);
    else outs[i] = add(ctx, a[i], b[i]);
  }
  for (std::size_t k0 = 0; k0 < batch.size(); k0 += kMaxPolys / 2) {
    const int R = (int)std::min<std::size_t>(kMaxPolys / 2, batch.size() - k0);
    PolyList ol{}, al{}, bl{};
    ol.n = al.n = bl.n = 2 * R;
    for (int r = 0; r < R; ++r) {
      const std::size_t i = batch[k0 + r];
      check_scales(a[i], b[i], "add");
      outs[i] = ctx.new_ct(a[i].limbs);
      outs[i].scale = a[i].scale;
      ol.p[2 * r] = outs[i].c0;
      ol.p[2 * r + 1] = outs[i].c1;
      al.p[2 * r] = a[i].c0;
      al.p[2 * r + 1] = a[i].c1;
      bl.p[2 * r] = b[i].c0;
      bl.p[2 * r + 1] = b[i].c1;
    }
    ew_add(ctx.dev(), ol, al, bl, a[batch[k0]].limbs, ctx.stream());
    ctx.stats.adds += R;
  }
  return outs;
}

// bootstrap (backend.cpp:233-249): same slots, level := depth budget
Ciphertext bootstrap(Context& ctx, const Ciphertext& a) {
  require_valid(a, "bootstrap");
  if (!ctx.boot)
    throw Error(ErrKind::not_implemented,
                "bootstrap: this context was created without bootstrapping (set bootstrap = 1 and a sparse "
                "secret, hamming_weight > 0)");
  return ctx.boot->run(a);
}

Ciphertext bootstrap_active(Context& ctx, const Ciphertext& a, std::size_t active, bool clean) {
  require_valid(a, "bootstrap");
  if (!ctx.boot) return bootstrap(ctx, a);
  if (active == 0 || active > (std::size_t)ctx.S())
    throw Error(ErrKind::shape, "bootstrap: active slot count " + std::to_string(active) + " outside [1, " +
                                    std::to_string(ctx.S()) + "]");
  Bootstrapper* best = nullptr;
  if (a.limbs >= 2 || clean)
    for (auto& b : ctx.boot_sparse)
      if ((std::size_t)b->slots() >= active && (!best || b->slots() < best->slots())) best = b.get();
  return best ? best->run(a, clean) : ctx.boot->run(a);
}

// bootstrap_active on several ciphertexts (the images of a batched inference) in lockstep:
// inputs of one level take the sparse-slot variant together (Bootstrapper::run_many),
// anything else runs one after the other.  Outputs bit-identical to bootstrap_active.
std::vector<Ciphertext> bootstrap_active_many(Context& ctx, const std::vector<Ciphertext>& as, std::size_t active,
                                              bool clean) {
  for (const Ciphertext& a : as) require_valid(a, "bootstrap");
  std::vector<Ciphertext> outs;
  bool same = !as.empty() && ctx.boot != nullptr;
  for (const Ciphertext& a : as) same = same && a.limbs == as[0].limbs;
  if (!same) {
    for (const Ciphertext& a : as) outs.push_back(bootstrap_active(ctx, a, active, clean));
    return outs;
  }
  if (active == 0 || active > (std::size_t)ctx.S())
    throw Error(ErrKind::shape, "bootstrap: active slot count " + std::to_string(active) + " outside [1, " +
                                    std::to_string(ctx.S()) + "]");
  Bootstrapper* best = nullptr;
  if (as[0].limbs >= 2 || clean)
    for (auto& b : ctx.boot_sparse)
      if ((std::size_t)b->slots() >= active && (!best || b->slots() < best->slots())) best = b.get();
  return best ? best->run_many(as, clean) : ctx.boot->run_many(as);
}

// -------------------------------------------------------------- raw access
Ciphertext upload_ct(Context& ctx, const u64* host, int limbs, double scale) {
  Ciphertext ct = ctx.new_ct(limbs);
  FHEON_CUDA(cudaMemcpyAsync(ct.c0, host, 2 * (std::size_t)limbs * ctx.N() * sizeof(u64), cudaMemcpyHostToDevice,
                             ctx.stream()));
  FHEON_CUDA(cudaStreamSynchronize(ctx.stream()));
  ct.scale = scale;
  return ct;
}

Ciphertext upload_ct_async(Context& ctx, const u64* host, int limbs, double scale) {
  const std::size_t words = 2 * (std::size_t)limbs * ctx.N();
  Ciphertext ct;
  ct.buf = std::make_shared<DevBuffer>(&ctx, words, ctx.h2d_stream());
  ct.c0 = ct.buf->ptr;
  ct.c1 = ct.buf->ptr + (std::size_t)limbs * ctx.N();
  ct.limbs = limbs;
  ct.id = ctx.next_id();
  ct.scale = scale;
  FHEON_CUDA(cudaMemcpyAsync(ct.c0, host, words * sizeof(u64), cudaMemcpyHostToDevice, ctx.h2d_stream()));
  cudaEvent_t up = ctx.take_event();
  FHEON_CUDA(cudaEventRecord(up, ctx.h2d_stream()));
  FHEON_CUDA(cudaStreamWaitEvent(ctx.stream(), up, 0));  // compute on it after the copy lands
  ctx.give_event(up);  // safe: a recorded event may be re-recorded once waited on
  return ct;
}

void download_ct_async(Context& ctx, const Ciphertext& ct, u64* host) {
  const std::size_t LN = (std::size_t)ct.limbs * ctx.N();
  cudaEvent_t ready = ctx.take_event();
  FHEON_CUDA(cudaEventRecord(ready, ctx.stream()));
  FHEON_CUDA(cudaStreamWaitEvent(ctx.d2h_stream(), ready, 0));
  ctx.give_event(ready);
  FHEON_CUDA(cudaMemcpyAsync(host, ct.c0, LN * sizeof(u64), cudaMemcpyDeviceToHost, ctx.d2h_stream()));
  FHEON_CUDA(cudaMemcpyAsync(host + LN, ct.c1, LN * sizeof(u64), cudaMemcpyDeviceToHost, ctx.d2h_stream()));
  cudaEvent_t done = ctx.take_event();
  FHEON_CUDA(cudaEventRecord(done, ctx.d2h_stream()));
  ctx.hold_until(done, ct.buf);  // the buffer outlives the copy
}

// ---- packed wire format (kernels.hpp PackLayout)
PackLayout pack_layout(const Context& ctx, int limbs) {
  if (limbs < 1 || limbs > 64) throw Error(ErrKind::shape, "packed transfer: bad limb count");
  PackLayout lay{};
  lay.limbs = limbs;
  lay.off[0] = 0;
  for (int i = 0; i < limbs; ++i) {
    lay.bits[i] = 64 - __builtin_clzll(ctx.host().q[i]);
    lay.off[i + 1] = lay.off[i] + (long long)(ctx.N() * (std::size_t)lay.bits[i] / 64);
  }
  return lay;
}

std::size_t packed_words(const Context& ctx, int limbs) { return 2 * (std::size_t)pack_layout(ctx, limbs).off[limbs]; }

Ciphertext upload_ct_packed_async(Context& ctx, const u64* host, int limbs, double scale) {
  const PackLayout lay = pack_layout(ctx, limbs);
  const std::size_t pw = 2 * (std::size_t)lay.off[limbs];
  const std::size_t words = 2 * (std::size_t)limbs * ctx.N();
  Ciphertext ct;
  ct.buf = std::make_shared<DevBuffer>(&ctx, words, ctx.h2d_stream());
  ct.c0 = ct.buf->ptr;
  ct.c1 = ct.buf->ptr + (std::size_t)limbs * ctx.N();
  ct.limbs = limbs;
  ct.id = ctx.next_id();
  ct.scale = scale;
  BufPtr stage = std::make_shared<DevBuffer>(&ctx, pw, ctx.h2d_stream());
  FHEON_CUDA(cudaMemcpyAsync(stage->ptr, host, pw * sizeof(u64), cudaMemcpyHostToDevice, ctx.h2d_stream()));
  cudaEvent_t landed = ctx.take_event();
  FHEON_CUDA(cudaEventRecord(landed, ctx.h2d_stream()));
  FHEON_CUDA(cudaStreamWaitEvent(ctx.unpack_stream(), landed, 0));
  ctx.give_event(landed);
  unpack_limbs(ctx.dev(), plist({ct.c0, ct.c1}), stage->ptr, lay, ctx.unpack_stream());
  cudaEvent_t up = ctx.take_event();
  FHEON_CUDA(cudaEventRecord(up, ctx.unpack_stream()));
  FHEON_CUDA(cudaStreamWaitEvent(ctx.stream(), up, 0));  // the staging buffer is freed after this point
  ctx.give_event(up);
  return ct;
}

std::size_t key_packed_words(const Context& ctx) {
  const int NP = ctx.L() + ctx.K();
  return (std::size_t)ctx.host().p.dnum * 2 * (std::size_t)pack_layout(ctx, NP).off[NP];
}

void download_key_packed(Context& ctx, u64 key_id, u64* host) {
  const int NP = ctx.L() + ctx.K();
  const std::size_t LN = (std::size_t)NP * ctx.N();
  const std::size_t nblk = (std::size_t)ctx.host().p.dnum * 2;
  const u64* k = ctx.key(key_id);
  BufPtr std_form = ctx.alloc(nblk * LN);
  for (std::size_t b = 0; b < nblk; ++b)
    convert_mont(ctx.dev(), std_form->ptr + b * LN, k + b * LN, NP, NP, false, ctx.stream());
  const PackLayout lay = pack_layout(ctx, NP);
  BufPtr stage = ctx.alloc(key_packed_words(ctx));
  PolyList src{};
  for (std::size_t b0 = 0; b0 < nblk; b0 += kMaxPolys) {
    src.n = (int)std::min<std::size_t>(kMaxPolys, nblk - b0);
    for (int i = 0; i < src.n; ++i) src.p[i] = std_form->ptr + (b0 + i) * LN;
    pack_limbs(ctx.dev(), stage->ptr + b0 * lay.off[NP], src, lay, ctx.stream());
  }
  FHEON_CUDA(cudaMemcpyAsync(host, stage->ptr, key_packed_words(ctx) * sizeof(u64), cudaMemcpyDeviceToHost,
                             ctx.stream()));
  FHEON_CUDA(cudaStreamSynchronize(ctx.stream()));
}

void upload_key_async(Context& ctx, u64 key_id, const u64* host, bool packed) {
  if (key_id != 0 && (key_id & 1) == 0 && key_id != kKeyToSparse && key_id != kKeyFromSparse &&
      !is_key_from_sparse_rot(key_id))
    throw Error(ErrKind::internal, "key upload: key id " + std::to_string(key_id) +
                                       " is neither 0 (relinearisation), a Galois element nor an encapsulation key");
  const int NP = ctx.L() + ctx.K();
  const std::size_t LN = (std::size_t)NP * ctx.N();
  const std::size_t nblk = (std::size_t)ctx.host().p.dnum * 2;
  const std::size_t words = packed ? key_packed_words(ctx) : nblk * LN;
  BufPtr kb = std::make_shared<DevBuffer>(&ctx, nblk * LN, ctx.h2d_stream());
  BufPtr stage = packed ? std::make_shared<DevBuffer>(&ctx, words, ctx.h2d_stream()) : kb;
  FHEON_CUDA(cudaMemcpyAsync(stage->ptr, host, words * sizeof(u64), cudaMemcpyHostToDevice, ctx.h2d_stream()));
  cudaEvent_t landed = ctx.take_event();
  FHEON_CUDA(cudaEventRecord(landed, ctx.h2d_stream()));
  FHEON_CUDA(cudaStreamWaitEvent(ctx.unpack_stream(), landed, 0));
  ctx.give_event(landed);
  if (packed) {
    const PackLayout lay = pack_layout(ctx, NP);
    PolyList dst{};
    for (std::size_t b0 = 0; b0 < nblk; b0 += kMaxPolys) {
      dst.n = (int)std::min<std::size_t>(kMaxPolys, nblk - b0);
      for (int i = 0; i < dst.n; ++i) dst.p[i] = kb->ptr + (b0 + i) * LN;
      unpack_limbs(ctx.dev(), dst, stage->ptr + b0 * lay.off[NP], lay, ctx.unpack_stream());
    }
  }
  for (std::size_t b = 0; b < nblk; ++b)  // standard -> Montgomery form, in place
    convert_mont(ctx.dev(), kb->ptr + b * LN, kb->ptr + b * LN, NP, NP, true, ctx.unpack_stream());
  cudaEvent_t ready = ctx.take_event();
  FHEON_CUDA(cudaEventRecord(ready, ctx.unpack_stream()));
  FHEON_CUDA(cudaStreamWaitEvent(ctx.stream(), ready, 0));  // later uses (and the frees) follow on the compute stream
  ctx.give_event(ready);
  ctx.put_key(key_id, kb);
  ctx.stats.key_uploads++;
  ctx.stats.key_upload_bytes += words * sizeof(u64);
}

void download_ct_packed_async(Context& ctx, const Ciphertext& ct, u64* host) {
  const PackLayout lay = pack_layout(ctx, ct.limbs);
  const std::size_t pw = 2 * (std::size_t)lay.off[ct.limbs];
  cudaEvent_t ready = ctx.take_event();
  FHEON_CUDA(cudaEventRecord(ready, ctx.stream()));
  FHEON_CUDA(cudaStreamWaitEvent(ctx.pack_stream(), ready, 0));
  ctx.give_event(ready);
  BufPtr stage = std::make_shared<DevBuffer>(&ctx, pw, ctx.pack_stream());
  pack_limbs(ctx.dev(), stage->ptr, plist({ct.c0, ct.c1}), lay, ctx.pack_stream());
  cudaEvent_t packed = ctx.take_event();
  FHEON_CUDA(cudaEventRecord(packed, ctx.pack_stream()));
  FHEON_CUDA(cudaStreamWaitEvent(ctx.d2h_stream(), packed, 0));
  ctx.give_event(packed);
  FHEON_CUDA(cudaMemcpyAsync(host, stage->ptr, pw * sizeof(u64), cudaMemcpyDeviceToHost, ctx.d2h_stream()));
  // one event per held buffer: reaping returns each event to the pool once
  for (BufPtr held : {ct.buf, stage}) {
    cudaEvent_t done = ctx.take_event();
    FHEON_CUDA(cudaEventRecord(done, ctx.d2h_stream()));
    ctx.hold_until(done, std::move(held));
  }
}

void wait_transfers(Context& ctx) {
  FHEON_CUDA(cudaStreamSynchronize(ctx.unpack_stream()));
  FHEON_CUDA(cudaStreamSynchronize(ctx.pack_stream()));
  FHEON_CUDA(cudaStreamSynchronize(ctx.h2d_stream()));
  FHEON_CUDA(cudaStreamSynchronize(ctx.d2h_stream()));
  ctx.reap_transfers(true);
}

void download_ct(Context& ctx, const Ciphertext& ct, u64* host) {
  const std::size_t LN = (std::size_t)ct.limbs * ctx.N();
  FHEON_CUDA(cudaMemcpyAsync(host, ct.c0, LN * sizeof(u64), cudaMemcpyDeviceToHost, ctx.stream()));
  FHEON_CUDA(cudaMemcpyAsync(host + LN, ct.c1, LN * sizeof(u64), cudaMemcpyDeviceToHost, ctx.stream()));
  FHEON_CUDA(cudaStreamSynchronize(ctx.stream()));
}

}  // namespace fheon
