// Evaluator ops over device ciphertexts (see engine.hpp for the mapping to
// proj/src/backend.cpp).  Every op enqueues on the context stream; nothing
// here synchronises except decrypt/download.
#include <cmath>
#include <cstring>
#include <map>

#include "engine.hpp"

namespace fheon {

namespace {

LimbSet limbset(u64* base, int blocks, std::size_t stride, int E, int ell, int L, int p0 = 0, int skip_alpha = 0) {
  LimbSet s{};
  s.base[0] = base;
  s.nbase = 1;
  s.blocks_per_base = blocks;
  s.block_stride = (long long)stride;
  s.E = E;
  s.ell = ell;
  s.L = L;
  s.p0 = p0;
  s.skip_alpha = skip_alpha;
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
  const int beta = (limbs + t.alpha - 1) / t.alpha;
  const int nin = (int)inputs.size();
  ctx.stats.keyswitches += jobs.size();

  // ModUp of every input, batched (one pipeline of launches per 32 inputs)
  const std::size_t ext_words = (std::size_t)beta * E * N;
  BufPtr xc = ctx.alloc((std::size_t)nin * limbs * N);
  BufPtr ext = ctx.alloc((std::size_t)nin * ext_words);
  for (int i0 = 0; i0 < nin; i0 += kMaxBases) {
    const int ni = std::min(kMaxBases, nin - i0);
    LimbSet dst = limbset(xc->ptr + (std::size_t)i0 * limbs * N, ni, (std::size_t)limbs * N, limbs, limbs, L);
    LimbSet src = dst;
    src.nbase = ni;
    src.blocks_per_base = 1;
    for (int i = 0; i < ni; ++i) src.base[i] = const_cast<u64*>(inputs[i0 + i]);
    ntt_inverse(t, dst, st, &src);  // out of place: c1 stays untouched
    PolyList xl{}, el{};
    xl.n = el.n = ni;
    for (int i = 0; i < ni; ++i) {
      xl.p[i] = xc->ptr + (std::size_t)(i0 + i) * limbs * N;
      el.p[i] = ext->ptr + (std::size_t)(i0 + i) * ext_words;
    }
    modup_bconv(t, el, xl, limbs, st);
    ntt_forward(t, limbset(ext->ptr + (std::size_t)i0 * ext_words, ni * beta, (std::size_t)E * N, E, limbs, L, 0,
                           t.alpha),
                st);
  }
  ctx.stats.ntt_limbs += (std::size_t)nin * ((std::size_t)limbs + (std::size_t)beta * (E - t.alpha));

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
    ntt_forward(t, limbset(conv->ptr, 2 * R, (std::size_t)limbs * N, limbs, limbs, L), st);
    moddown_finish(t, ol, al, cl, addl, limbs, st);
    ctx.stats.ntt_limbs += (std::size_t)R * 2 * (K + limbs);
  }
  return outs;
}

}  // namespace

// ---------------------------------------------------------------- rescale
Ciphertext rescale(Context& ctx, const Ciphertext& a) {
  require_valid(a, "rescale");
  const int l = a.limbs;
  if (l < 2) throw Error(ErrKind::depth_exhausted, "rescale: no limb left to drop");
  const DevTables& t = ctx.dev();
  cudaStream_t st = ctx.stream();
  const std::size_t N = ctx.N();
  BufPtr last = ctx.alloc(2 * N);
  FHEON_CUDA(cudaMemcpyAsync(last->ptr, a.c0 + (std::size_t)(l - 1) * N, N * sizeof(u64), cudaMemcpyDeviceToDevice, st));
  FHEON_CUDA(cudaMemcpyAsync(last->ptr + N, a.c1 + (std::size_t)(l - 1) * N, N * sizeof(u64),
                             cudaMemcpyDeviceToDevice, st));
  ntt_inverse(t, limbset(last->ptr, 2, N, 1, 1, ctx.L(), l - 1), st);
  BufPtr r = ctx.alloc(2 * (std::size_t)(l - 1) * N);
  u64* r0 = r->ptr;
  u64* r1 = r->ptr + (std::size_t)(l - 1) * N;
  rescale_lift(t, plist({r0, r1}), plist({last->ptr, last->ptr + N}), l, st);
  ntt_forward(t, limbset(r->ptr, 2, (std::size_t)(l - 1) * N, l - 1, l - 1, ctx.L()), st);
  Ciphertext out = ctx.new_ct(l - 1);
  rescale_finish(t, plist({out.c0, out.c1}), plist({a.c0, a.c1}), plist({r0, r1}), l, st);
  out.scale = a.scale;
  ctx.stats.rescales++;
  ctx.stats.ntt_limbs += 2 + 2 * (std::size_t)(l - 1);
  return out;
}

// -------------------------------------------------------------- level down
Ciphertext level_down(Context& ctx, const Ciphertext& a, int target) {
  require_valid(a, "level_down");
  if (target == a.limbs) return a;
  if (target > a.limbs || target < 1) throw Error(ErrKind::internal, "level_down: bad target");
  const int keep = target + 1;
  const HostTables& h = ctx.host();
  const double c = h.T[target - 1] * (double)h.q[target] / a.scale;
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
Ciphertext encrypt_top(Context& ctx, const double* vals, std::size_t n) {
  const int L = ctx.L();
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
  Ciphertext ct = encrypt_top(ctx, vals, n);
  return level_down(ctx, ct, ctx.depth_budget() + 1);
}

void decrypt(Context& ctx, const Ciphertext& ct, double* out) {
  require_valid(ct, "decrypt");
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
  ctx.decode_coeffs(coeffs.data(), ct.scale, out);
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

std::vector<Ciphertext> rotate_same(Context& ctx, const std::vector<Ciphertext>& xs, long t) {
  return rotate_many(ctx, xs, std::vector<long>(xs.size(), t));
}

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

Ciphertext bootstrap(Context& ctx, const Ciphertext& a) {
  require_valid(a, "bootstrap");
  (void)ctx;
  throw Error(ErrKind::not_implemented,
              "bootstrap: CKKS bootstrapping is not available in this build; size the modulus chain for the "
              "network depth");
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

void download_ct(Context& ctx, const Ciphertext& ct, u64* host) {
  const std::size_t LN = (std::size_t)ct.limbs * ctx.N();
  FHEON_CUDA(cudaMemcpyAsync(host, ct.c0, LN * sizeof(u64), cudaMemcpyDeviceToHost, ctx.stream()));
  FHEON_CUDA(cudaMemcpyAsync(host + LN, ct.c1, LN * sizeof(u64), cudaMemcpyDeviceToHost, ctx.stream()));
  FHEON_CUDA(cudaStreamSynchronize(ctx.stream()));
}

}  // namespace fheon
