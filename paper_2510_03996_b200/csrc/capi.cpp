// extern "C" boundary (include/fheon_b200.h): opaque handles, int status,
// thread-local error message.  Exceptions never cross this boundary.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../include/fheon_b200.h"
#include "engine.hpp"
#include "layers.hpp"
#include "bootstrap.hpp"

struct fheon_ctx {
  fheon::Context* impl;
};
struct fheon_ct {
  fheon::Ciphertext ct;
};

namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const fheon::Error& e) {
    g_err = e.what();
    g_kind = static_cast<int>(e.kind);
    return fheon::category_of(e.kind);
  } catch (const std::exception& e) {
    g_err = e.what();
    g_kind = static_cast<int>(fheon::ErrKind::internal);
    return 3;
  }
}

fheon_ct* wrap(const fheon::Ciphertext& c) { return new fheon_ct{c}; }

void need(const void* p, const char* what) {
  if (!p) throw fheon::Error(fheon::ErrKind::internal, std::string(what) + " is null");
}

}  // namespace

extern "C" {

const char* fheon_last_error(void) { return g_err.c_str(); }
int fheon_last_error_kind(void) { return g_kind; }
int fheon_version(void) { return 1; }

static fheon::Params to_params(const fheon_params* p) {
  fheon::Params prm;
  prm.logN = p->log_n;
  prm.L = p->limbs;
  prm.K = p->special_limbs;
  prm.dnum = p->dnum;
  prm.first_bits = p->first_mod_bits;
  prm.scale_bits = p->scale_bits;
  prm.special_bits = p->special_bits;
  prm.depth_budget = p->depth_budget;
  prm.seed = p->seed;
  prm.hamming_weight = p->hamming_weight;
  prm.bootstrap = p->bootstrap;
  prm.boot_scale_bits = p->boot_scale_bits;
  prm.digit_split = p->digit_split;
  if (p->boot_hamming_weight > 0) prm.boot_hamming_weight = p->boot_hamming_weight;
  if (p->min_security > 0) prm.min_security = p->min_security;
  prm.allow_insecure = p->allow_insecure;
  prm.no_secret = p->no_secret;
  if (p->boot_k_range > 0) prm.boot_k_range = p->boot_k_range;
  if (p->boot_cts_levels > 0) prm.boot_cts_levels = p->boot_cts_levels;
  if (p->boot_stc_levels > 0) prm.boot_stc_levels = p->boot_stc_levels;
  prm.boot_sparse = p->boot_sparse > 0 ? p->boot_sparse : 0;
  return prm;
}

int fheon_host_bootstrap_depth(const fheon_params* p, int* depth) {
  return guard([&] {
    need(p, "params");
    need(depth, "depth");
    *depth = fheon::bootstrap_depth(to_params(p));
  });
}

int fheon_host_security(const fheon_params* p, double* log_qp, int* level, double* bound) {
  return guard([&] {
    need(p, "params");
    fheon::HostTables h;
    try {
      h = fheon::make_tables(to_params(p));
    } catch (const std::invalid_argument& e) {
      throw fheon::Error(fheon::ErrKind::shape, e.what());
    }
    double b = 0.0;
    for (std::size_t i = 0; i < h.q.size(); ++i) b += std::log2((double)h.q[i]);
    if (log_qp) *log_qp = b;
    if (level) *level = fheon::he_standard_security(h.p.logN, b, h.p.hamming_weight);
    if (bound) *bound = fheon::he_standard_max_logqp(h.p.logN, h.p.min_security);
  });
}

int fheon_host_primes(const fheon_params* p, uint64_t* primes, double* scales) {
  return guard([&] {
    need(p, "params");
    fheon::HostTables h;
    try {
      h = fheon::make_tables(to_params(p));
    } catch (const std::invalid_argument& e) {
      throw fheon::Error(fheon::ErrKind::shape, e.what());
    }
    if (primes)
      for (std::size_t i = 0; i < h.q.size(); ++i) primes[i] = h.q[i];
    if (scales)
      for (std::size_t i = 0; i < h.T.size(); ++i) scales[i] = h.T[i];
  });
}

int fheon_host_encode(const fheon_params* p, const double* values, size_t n, double scale, int64_t* coeffs) {
  return guard([&] {
    need(p, "params");
    fheon::HostTables h;
    try {
      h = fheon::make_tables(to_params(p));
    } catch (const std::invalid_argument& e) {
      throw fheon::Error(fheon::ErrKind::shape, e.what());
    }
    fheon::encode_coeffs_host(h, values, n, scale, reinterpret_cast<long long*>(coeffs));
  });
}

int fheon_cheb_relu_coefficients(double beta, int degree, double* coeffs) {
  return guard([&] {
    const auto f = [beta](double z) { return z < 0.0 ? 0.0 : beta * z; };
    const std::vector<double> c = fheon::cheb_coefficients(f, degree);
    std::copy(c.begin(), c.end(), coeffs);
  });
}

int fheon_ctx_create(const fheon_params* p, fheon_ctx** out) {
  return guard([&] {
    need(p, "params");
    need(out, "out");
    const fheon::Params prm = to_params(p);
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      throw fheon::Error(fheon::ErrKind::cuda, "no CUDA device visible: the B200 engine has no CPU fallback");
    try {
      *out = new fheon_ctx{new fheon::Context(prm)};
    } catch (const std::invalid_argument& e) {
      throw fheon::Error(fheon::ErrKind::shape, e.what());
    }
  });
}

void fheon_ctx_destroy(fheon_ctx* ctx) {
  if (!ctx) return;
  delete ctx->impl;
  delete ctx;
}

int fheon_ctx_clone(fheon_ctx* parent, fheon_ctx** out) {
  return guard([&] {
    need(parent, "parent");
    need(out, "out");
    *out = new fheon_ctx{new fheon::Context(parent->impl->host().p, *parent->impl)};
    (*out)->impl->schedule = parent->impl->schedule;
    // the keys are shared, the resident weight plaintexts are not: split the parent's
    // budget so the two caches together stay within what the parent alone was given
    const std::size_t half = parent->impl->weight_cache_budget / 2;
    parent->impl->weight_cache_budget = half;
    (*out)->impl->weight_cache_budget = half;
  });
}

int fheon_release_memory(void) {
  return guard([&] {
    int dev = 0;
    FHEON_CUDA(cudaGetDevice(&dev));
    FHEON_CUDA(cudaDeviceSynchronize());
    cudaMemPool_t pool;
    FHEON_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    FHEON_CUDA(cudaMemPoolTrimTo(pool, 0));
  });
}

int fheon_ctx_security(const fheon_ctx* ctx, double* log_qp, int* level) {
  return guard([&] {
    need(ctx, "ctx");
    if (log_qp) *log_qp = ctx->impl->log_qp();
    if (level) *level = ctx->impl->security();
  });
}

int fheon_ctx_info(const fheon_ctx* ctx, uint64_t* primes, double* scales, int* slots) {
  return guard([&] {
    need(ctx, "ctx");
    const fheon::HostTables& h = ctx->impl->host();
    if (primes)
      for (std::size_t i = 0; i < h.q.size(); ++i) primes[i] = h.q[i];
    if (scales)
      for (std::size_t i = 0; i < h.T.size(); ++i) scales[i] = h.T[i];
    if (slots) *slots = h.S;
  });
}

void* fheon_ctx_stream(fheon_ctx* ctx) { return ctx ? static_cast<void*>(ctx->impl->stream()) : nullptr; }

int fheon_ctx_sync(fheon_ctx* ctx) {
  return guard([&] {
    FHEON_CUDA(cudaStreamSynchronize(ctx->impl->stream()));
    fheon::wait_transfers(*ctx->impl);
  });
}

int fheon_ctx_stats(const fheon_ctx* ctx, uint64_t* o) {
  return guard([&] {
    const fheon::OpStats& s = ctx->impl->stats;
    o[0] = s.rotations;
    o[1] = s.keyswitches;
    o[2] = s.mult_plain;
    o[3] = s.mult_cipher;
    o[4] = s.rescales;
    o[5] = s.ntt_limbs;
    o[6] = s.encodes;
    o[7] = s.adds;
    o[8] = fheon::g_kernel_launches.load() - s.launches;  // kernels launched since the last reset
  });
}
int fheon_ctx_reset_stats(fheon_ctx* ctx) {
  return guard([&] {
    ctx->impl->stats = fheon::OpStats{};
    ctx->impl->stats.launches = fheon::g_kernel_launches.load();  // baseline
  });
}
int fheon_timer_arm(fheon_ctx* ctx, int kernel_class) {
  return guard([&] {
    ctx->impl->timer.cls = kernel_class;
    ctx->impl->timer.reset();
  });
}
int fheon_timer_read(fheon_ctx* ctx, double* total_ms, int* count) {
  return guard([&] { *total_ms = ctx->impl->timer.total_ms(count); });
}

int fheon_set_tracing(fheon_ctx* ctx, int on) {
  return guard([&] { ctx->impl->set_tracing(on != 0); });
}
int fheon_trace(fheon_ctx* ctx, long* ev, size_t cap, size_t* n) {
  return guard([&] {
    std::size_t k = 0;
    for (const fheon::TraceEvent& e : ctx->impl->trace_snapshot()) {
      if (e.kind > 3) continue;
      if (ev && k < cap) {
        ev[2 * k] = e.kind;
        ev[2 * k + 1] = e.value;
      }
      ++k;
    }
    if (n) *n = k;
  });
}
int fheon_trace_clear(fheon_ctx* ctx) {
  return guard([&] { ctx->impl->clear_trace(); });
}

uint64_t fheon_galois_elt(const fheon_ctx* ctx, long t) { return ctx->impl->galois(t); }

int fheon_keygen_rotations(fheon_ctx* ctx, const long* steps, size_t n) {
  return guard([&] {
    for (size_t i = 0; i < n; ++i) {
      const fheon::u64 g = ctx->impl->galois(steps[i]);
      if (g != 1) ctx->impl->gen_key(g);
    }
    FHEON_CUDA(cudaStreamSynchronize(ctx->impl->stream()));
  });
}
int fheon_keygen_relin(fheon_ctx* ctx) {
  return guard([&] { ctx->impl->gen_key(0); });
}
int fheon_set_strict_keys(fheon_ctx* ctx, int strict) {
  return guard([&] { ctx->impl->strict_keys = strict != 0; });
}
size_t fheon_key_count(const fheon_ctx* ctx) { return ctx->impl->num_keys(); }
int fheon_key_events(const fheon_ctx* ctx, uint64_t* gens, uint64_t* drops) {
  return guard([&] {
    need(ctx, "ctx");
    if (gens) *gens = ctx->impl->stats.key_gens;
    if (drops) *drops = ctx->impl->stats.key_drops;
  });
}
uint64_t fheon_key_bytes(const fheon_ctx* ctx) {
  return (uint64_t)ctx->impl->num_keys() * ctx->impl->key_words() * sizeof(uint64_t);
}
int fheon_prefetch_rotation_keys(fheon_ctx* ctx, const long* steps, size_t n) {
  return guard([&] {
    for (size_t i = 0; i < n; ++i) {
      const fheon::u64 g = ctx->impl->galois(steps[i]);
      if (g != 1) ctx->impl->gen_key(g);  // stream-ordered, no host sync
    }
  });
}
int fheon_drop_rotation_keys(fheon_ctx* ctx, const long* steps, size_t n) {
  return guard([&] {
    for (size_t i = 0; i < n; ++i) {
      const fheon::u64 g = ctx->impl->galois(steps[i]);
      if (g != 1) ctx->impl->drop_key(g);  // freed in stream order after its last use
    }
  });
}

size_t fheon_key_packed_words(const fheon_ctx* ctx) {
  try {
    return fheon::key_packed_words(*ctx->impl);
  } catch (...) {
    return 0;
  }
}
int fheon_key_download_packed(fheon_ctx* ctx, uint64_t key_id, uint64_t* packed) {
  return guard([&] {
    need(ctx, "ctx");
    need(packed, "packed");
    fheon::download_key_packed(*ctx->impl, key_id, packed);
  });
}
int fheon_key_upload(fheon_ctx* ctx, uint64_t key_id, const uint64_t* words) {
  return guard([&] {
    need(ctx, "ctx");
    need(words, "words");
    fheon::upload_key_async(*ctx->impl, key_id, words, false);
    fheon::wait_transfers(*ctx->impl);
  });
}
int fheon_key_upload_packed_async(fheon_ctx* ctx, uint64_t key_id, const uint64_t* packed) {
  return guard([&] {
    need(ctx, "ctx");
    need(packed, "packed");
    fheon::upload_key_async(*ctx->impl, key_id, packed, true);
  });
}
int fheon_key_upload_packed(fheon_ctx* ctx, uint64_t key_id, const uint64_t* packed) {
  const int rc = fheon_key_upload_packed_async(ctx, key_id, packed);
  if (rc) return rc;
  return guard([&] { fheon::wait_transfers(*ctx->impl); });
}
int fheon_required_key_ids(const fheon_ctx* ctx, uint64_t* ids, size_t cap, size_t* n) {
  return guard([&] {
    need(ctx, "ctx");
    const std::vector<fheon::u64> v = ctx->impl->pinned_keys();
    if (n) *n = v.size();
    for (size_t i = 0; i < v.size() && i < cap && ids; ++i) ids[i] = v[i];
  });
}
int fheon_key_uploads(const fheon_ctx* ctx, uint64_t* count, uint64_t* bytes) {
  return guard([&] {
    need(ctx, "ctx");
    if (count) *count = ctx->impl->stats.key_uploads;
    if (bytes) *bytes = ctx->impl->stats.key_upload_bytes;
  });
}

int fheon_key_download(fheon_ctx* ctx, uint64_t key_id, uint64_t* out) {
  return guard([&] {
    fheon::Context& c = *ctx->impl;
    const fheon::u64* k = c.key(key_id);
    const std::size_t words = c.key_words();
    fheon::BufPtr tmp = c.alloc(words);
    const int NP = c.L() + c.K();
    const std::size_t LN = (std::size_t)NP * c.N();
    for (std::size_t blk = 0; blk < words / LN; ++blk)
      fheon::convert_mont(c.dev(), tmp->ptr + blk * LN, k + blk * LN, NP, NP, false, c.stream());
    FHEON_CUDA(cudaMemcpyAsync(out, tmp->ptr, words * sizeof(uint64_t), cudaMemcpyDeviceToHost, c.stream()));
    FHEON_CUDA(cudaStreamSynchronize(c.stream()));
  });
}

void fheon_ct_free(fheon_ct* ct) { delete ct; }
int fheon_ct_level(const fheon_ct* ct) { return ct ? ct->ct.level() : -1; }
int fheon_ct_limbs(const fheon_ct* ct) { return ct ? ct->ct.limbs : 0; }
double fheon_ct_scale(const fheon_ct* ct) { return ct ? ct->ct.scale : 0.0; }

int fheon_encrypt(fheon_ctx* ctx, const double* v, size_t n, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::encrypt(*ctx->impl, v, n)); });
}
int fheon_encrypt_top(fheon_ctx* ctx, const double* v, size_t n, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::encrypt_top(*ctx->impl, v, n)); });
}
int fheon_decrypt(fheon_ctx* ctx, const fheon_ct* ct, double* out, size_t n) {
  return guard([&] {
    need(ct, "ciphertext");
    if (n < (size_t)ctx->impl->S()) throw fheon::Error(fheon::ErrKind::capacity, "output buffer smaller than S");
    fheon::decrypt(*ctx->impl, ct->ct, out);
  });
}
int fheon_decrypt_complex(fheon_ctx* ctx, const fheon_ct* ct, double* re, double* im, size_t n) {
  return guard([&] {
    need(ct, "ciphertext");
    if (n < (size_t)ctx->impl->S()) throw fheon::Error(fheon::ErrKind::capacity, "output buffer smaller than S");
    fheon::decrypt(*ctx->impl, ct->ct, re, im);
  });
}
int fheon_ctx_depth_budget(const fheon_ctx* ctx) { return ctx ? ctx->impl->depth_budget() : -1; }

int fheon_ctx_set_schedule(fheon_ctx* ctx, int schedule) {
  return guard([&] {
    if (schedule != fheon::Context::kScheduleFast && schedule != fheon::Context::kScheduleReference)
      throw fheon::Error(fheon::ErrKind::shape, "schedule must be 0 (fast) or 1 (reference)");
    ctx->impl->schedule = schedule;
  });
}

int fheon_ctx_schedule(const fheon_ctx* ctx) { return ctx ? ctx->impl->schedule : -1; }

int fheon_ctx_set_weight_cache(fheon_ctx* ctx, uint64_t bytes) {
  return guard([&] { ctx->impl->weight_cache_budget = (std::size_t)bytes; });
}
int fheon_ct_upload(fheon_ctx* ctx, const uint64_t* w, int limbs, double scale, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::upload_ct(*ctx->impl, w, limbs, scale)); });
}
int fheon_ct_download(fheon_ctx* ctx, const fheon_ct* ct, uint64_t* w) {
  return guard([&] { fheon::download_ct(*ctx->impl, ct->ct, w); });
}
int fheon_ct_upload_async(fheon_ctx* ctx, const uint64_t* w, int limbs, double scale, fheon_ct** out) {
  return guard([&] {
    if (limbs < 1 || limbs > ctx->impl->L()) throw fheon::Error(fheon::ErrKind::shape, "upload: bad limb count");
    *out = wrap(fheon::upload_ct_async(*ctx->impl, w, limbs, scale));
  });
}
int fheon_ct_download_async(fheon_ctx* ctx, const fheon_ct* ct, uint64_t* w) {
  return guard([&] {
    need(ct, "ciphertext");
    fheon::download_ct_async(*ctx->impl, ct->ct, w);
  });
}
size_t fheon_ct_packed_words(const fheon_ctx* ctx, int limbs) {
  try {
    return fheon::packed_words(*ctx->impl, limbs);
  } catch (...) {
    return 0;
  }
}
int fheon_ct_upload_packed_async(fheon_ctx* ctx, const uint64_t* packed, int limbs, double scale, fheon_ct** out) {
  return guard([&] {
    if (limbs < 1 || limbs > ctx->impl->L()) throw fheon::Error(fheon::ErrKind::shape, "upload: bad limb count");
    *out = wrap(fheon::upload_ct_packed_async(*ctx->impl, packed, limbs, scale));
  });
}
int fheon_ct_download_packed_async(fheon_ctx* ctx, const fheon_ct* ct, uint64_t* packed) {
  return guard([&] {
    need(ct, "ciphertext");
    fheon::download_ct_packed_async(*ctx->impl, ct->ct, packed);
  });
}
int fheon_ct_upload_packed(fheon_ctx* ctx, const uint64_t* packed, int limbs, double scale, fheon_ct** out) {
  const int rc = fheon_ct_upload_packed_async(ctx, packed, limbs, scale, out);
  return rc != 0 ? rc : fheon_ctx_wait_transfers(ctx);
}
int fheon_ct_download_packed(fheon_ctx* ctx, const fheon_ct* ct, uint64_t* packed) {
  const int rc = fheon_ct_download_packed_async(ctx, ct, packed);
  return rc != 0 ? rc : fheon_ctx_wait_transfers(ctx);
}
int fheon_ctx_wait_transfers(fheon_ctx* ctx) {
  return guard([&] { fheon::wait_transfers(*ctx->impl); });
}

int fheon_rotate(fheon_ctx* ctx, const fheon_ct* x, long t, fheon_ct** out) {
  return guard([&] {
    need(x, "ciphertext");
    *out = wrap(fheon::rotate(*ctx->impl, x->ct, t));
  });
}
int fheon_rotate_hoisted(fheon_ctx* ctx, const fheon_ct* x, const long* ts, size_t n, fheon_ct** outs) {
  return guard([&] {
    need(x, "ciphertext");
    std::vector<long> v(ts, ts + n);
    std::vector<fheon::Ciphertext> r = fheon::rotate_hoisted(*ctx->impl, x->ct, v);
    for (size_t i = 0; i < n; ++i) outs[i] = wrap(r[i]);
  });
}
int fheon_rotate_many(fheon_ctx* ctx, const fheon_ct* const* xs, const long* ts, size_t n, fheon_ct** outs) {
  return guard([&] {
    std::vector<fheon::Ciphertext> in;
    in.reserve(n);
    for (size_t i = 0; i < n; ++i) {
      need(xs[i], "ciphertext");
      in.push_back(xs[i]->ct);
    }
    std::vector<fheon::Ciphertext> r = fheon::rotate_many(*ctx->impl, in, std::vector<long>(ts, ts + n));
    for (size_t i = 0; i < n; ++i) outs[i] = wrap(r[i]);
  });
}
int fheon_rotate_sum(fheon_ctx* ctx, const fheon_ct* const* xs, const long* ts, size_t n, fheon_ct** out) {
  return guard([&] {
    if (n == 0) throw fheon::Error(fheon::ErrKind::shape, "rotate_sum needs at least one term");
    std::vector<std::pair<fheon::Ciphertext, long>> g;
    g.reserve(n);
    for (size_t i = 0; i < n; ++i) {
      need(xs[i], "ciphertext");
      g.push_back({xs[i]->ct, ts[i]});
    }
    *out = wrap(fheon::rotate_sum_many(*ctx->impl, {g})[0]);
  });
}
int fheon_rotate_sum_many(fheon_ctx* ctx, const fheon_ct* const* xs, const long* ts, const size_t* sizes,
                          size_t ngroups, fheon_ct** outs) {
  return guard([&] {
    std::vector<std::vector<std::pair<fheon::Ciphertext, long>>> groups(ngroups);
    size_t k = 0;
    for (size_t r = 0; r < ngroups; ++r) {
      if (sizes[r] == 0) throw fheon::Error(fheon::ErrKind::shape, "rotate_sum needs at least one term per group");
      for (size_t i = 0; i < sizes[r]; ++i, ++k) {
        need(xs[k], "ciphertext");
        groups[r].push_back({xs[k]->ct, ts[k]});
      }
    }
    std::vector<fheon::Ciphertext> r = fheon::rotate_sum_many(*ctx->impl, groups);
    for (size_t i = 0; i < ngroups; ++i) outs[i] = wrap(r[i]);
  });
}
int fheon_add(fheon_ctx* ctx, const fheon_ct* a, const fheon_ct* b, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::add(*ctx->impl, a->ct, b->ct)); });
}
int fheon_sub(fheon_ctx* ctx, const fheon_ct* a, const fheon_ct* b, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::sub(*ctx->impl, a->ct, b->ct)); });
}
int fheon_add_plain(fheon_ctx* ctx, const fheon_ct* a, const double* v, size_t n, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::add_plain(*ctx->impl, a->ct, v, n)); });
}
int fheon_mult_plain(fheon_ctx* ctx, const fheon_ct* a, const double* v, size_t n, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::mult_plain(*ctx->impl, a->ct, v, n)); });
}
int fheon_mult_cipher(fheon_ctx* ctx, const fheon_ct* a, const fheon_ct* b, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::mult_cipher(*ctx->impl, a->ct, b->ct)); });
}
int fheon_bootstrap(fheon_ctx* ctx, const fheon_ct* a, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::bootstrap(*ctx->impl, a->ct)); });
}
int fheon_bootstrap_active(fheon_ctx* ctx, const fheon_ct* a, size_t active_slots, int flags, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::bootstrap_active(*ctx->impl, a->ct, active_slots, (flags & 1) != 0)); });
}
int fheon_bootstrap_active_many(fheon_ctx* ctx, const fheon_ct* const* as, size_t n, size_t active_slots, int flags,
                                fheon_ct** outs) {
  return guard([&] {
    std::vector<fheon::Ciphertext> in;
    in.reserve(n);
    for (size_t i = 0; i < n; ++i) {
      need(as[i], "ciphertext");
      in.push_back(as[i]->ct);
    }
    std::vector<fheon::Ciphertext> r = fheon::bootstrap_active_many(*ctx->impl, in, active_slots, (flags & 1) != 0);
    for (size_t i = 0; i < n; ++i) outs[i] = wrap(r[i]);
  });
}
int fheon_bootstrap_stage(fheon_ctx* ctx, const fheon_ct* a, int stage, fheon_ct** out) {
  return guard([&] {
    if (!ctx->impl->boot) throw fheon::Error(fheon::ErrKind::not_implemented, "context has no bootstrapper");
    *out = wrap(ctx->impl->boot->debug_stage(a->ct, stage));
  });
}
int fheon_bootstrap_info(fheon_ctx* ctx, int* info4, double* coeffs, size_t cap, size_t* n) {
  return guard([&] {
    if (!ctx->impl->boot) throw fheon::Error(fheon::ErrKind::not_implemented, "context has no bootstrapper");
    const fheon::Bootstrapper& b = *ctx->impl->boot;
    if (info4) {
      info4[0] = b.depth();
      info4[1] = 16;
      info4[2] = 3;
      info4[3] = b.stc_input_limbs();
    }
    const std::vector<double>& c = b.cos_coeffs();
    if (n) *n = c.size();
    if (coeffs)
      for (size_t i = 0; i < c.size() && i < cap; ++i) coeffs[i] = c[i];
  });
}
int fheon_rescale(fheon_ctx* ctx, const fheon_ct* a, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::rescale(*ctx->impl, a->ct)); });
}
int fheon_level_down(fheon_ctx* ctx, const fheon_ct* a, int limbs, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::level_down(*ctx->impl, a->ct, limbs)); });
}
int fheon_keyswitch_raw(fheon_ctx* ctx, const fheon_ct* a, uint64_t key_id, uint64_t g, fheon_ct** out) {
  return guard([&] { *out = wrap(fheon::keyswitch_raw(*ctx->impl, a->ct, key_id, g)); });
}

int fheon_ntt_host(fheon_ctx* ctx, uint64_t* w, int npolys, int nlimbs, int inverse) {
  return guard([&] {
    fheon::Context& c = *ctx->impl;
    const std::size_t words = (std::size_t)npolys * nlimbs * c.N();
    fheon::BufPtr b = c.alloc(words);
    FHEON_CUDA(cudaMemcpyAsync(b->ptr, w, words * sizeof(uint64_t), cudaMemcpyHostToDevice, c.stream()));
    fheon::LimbSet s{};
    s.base[0] = b->ptr;
    s.nbase = 1;
    s.blocks_per_base = npolys;
    s.block_stride = (long long)nlimbs * c.N();
    s.E = nlimbs;
    s.ell = nlimbs;
    s.L = c.L();
    if (inverse) fheon::ntt_inverse(c.dev(), s, c.stream());
    else fheon::ntt_forward(c.dev(), s, c.stream());
    FHEON_CUDA(cudaMemcpyAsync(w, b->ptr, words * sizeof(uint64_t), cudaMemcpyDeviceToHost, c.stream()));
    FHEON_CUDA(cudaStreamSynchronize(c.stream()));
  });
}

int fheon_automorph_host(fheon_ctx* ctx, uint64_t* w, int npolys, int nlimbs, uint64_t g) {
  return guard([&] {
    fheon::Context& c = *ctx->impl;
    const std::size_t words = (std::size_t)npolys * nlimbs * c.N();
    fheon::BufPtr in = c.alloc(words), out = c.alloc(words);
    FHEON_CUDA(cudaMemcpyAsync(in->ptr, w, words * sizeof(uint64_t), cudaMemcpyHostToDevice, c.stream()));
    fheon::PolyList o{}, i{};
    for (int p = 0; p < npolys; ++p) {
      o.p[p] = out->ptr + (std::size_t)p * nlimbs * c.N();
      o.g[p] = g;
      i.p[p] = in->ptr + (std::size_t)p * nlimbs * c.N();
    }
    o.n = i.n = npolys;
    fheon::automorph(c.dev(), o, i, nlimbs, c.stream());
    FHEON_CUDA(cudaMemcpyAsync(w, out->ptr, words * sizeof(uint64_t), cudaMemcpyDeviceToHost, c.stream()));
    FHEON_CUDA(cudaStreamSynchronize(c.stream()));
  });
}

int fheon_microbench(fheon_ctx* ctx, int kind, int batch, int limbs, int n_rot, int iters, double* ms) {
  return guard([&] { *ms = fheon::microbench(*ctx->impl, kind, batch, limbs, n_rot, iters); });
}

// ---------------------------------------------------------------- layers
int fheon_convolution(fheon_ctx* ctx, const fheon_ct* x, size_t C, size_t W, const fheon_conv_cfg* cfg,
                      const double* w, const double* bias, fheon_ct** out, size_t* oc, size_t* ow) {
  return guard([&] {
    need(x, "ciphertext");
    need(cfg, "config");
    fheon::ConvConfig c{cfg->in_channels, cfg->out_channels, cfg->kernel, cfg->stride, cfg->padding, cfg->mode,
                        cfg->stride_variant};
    fheon::PackedTensor in{x->ct, C, W};
    fheon::KernelTensor kt = fheon::KernelTensor::from(c, w, bias);
    fheon::PackedTensor r = fheon::convolution(*ctx->impl, in, c, kt);
    *out = wrap(r.data);
    if (oc) *oc = r.channels;
    if (ow) *ow = r.width;
  });
}

int fheon_pool(fheon_ctx* ctx, const fheon_ct* x, size_t C, size_t W, int kind, size_t k, size_t stride,
               int variant, fheon_ct** out, size_t* oc, size_t* ow) {
  return guard([&] {
    need(x, "ciphertext");
    fheon::PackedTensor in{x->ct, C, W};
    if (kind == 0) {
      fheon::PackedTensor r = fheon::avg_pool(*ctx->impl, in, k, stride, variant);
      *out = wrap(r.data);
      if (oc) *oc = r.channels;
      if (ow) *ow = r.width;
    } else {
      fheon::Ciphertext r = kind == 1 ? fheon::global_avg_pool(*ctx->impl, in)
                                      : fheon::whole_channel_pool(*ctx->impl, in, k);
      *out = wrap(r);
      if (oc) *oc = C;
      if (ow) *ow = 1;
    }
  });
}

int fheon_fully_connected(fheon_ctx* ctx, const fheon_ct* x, size_t n, size_t m, size_t merge_budget,
                          const double* w, const double* bias, fheon_ct** out) {
  return guard([&] {
    need(x, "ciphertext");
    *out = wrap(fheon::fully_connected(*ctx->impl, x->ct, n, m, merge_budget, w, bias));
  });
}

int fheon_secure_relu(fheon_ctx* ctx, const fheon_ct* x, double scale, int degree, size_t active, fheon_ct** out) {
  return guard([&] {
    need(x, "ciphertext");
    *out = wrap(fheon::secure_relu(*ctx->impl, x->ct, scale, degree, active));
  });
}

int fheon_secure_relu_many(fheon_ctx* ctx, const fheon_ct* const* xs, size_t n, double scale, int degree,
                           size_t active, fheon_ct** outs) {
  return guard([&] {
    std::vector<fheon::Ciphertext> in;
    in.reserve(n);
    for (size_t i = 0; i < n; ++i) {
      need(xs[i], "ciphertext");
      in.push_back(xs[i]->ct);
    }
    std::vector<fheon::Ciphertext> r = fheon::secure_relu_many(*ctx->impl, in, scale, degree, active);
    for (size_t i = 0; i < n; ++i) outs[i] = wrap(r[i]);
  });
}

int fheon_stride(fheon_ctx* ctx, const fheon_ct* x, size_t W, size_t S, size_t w_out, int variant, fheon_ct** out) {
  return guard([&] {
    need(x, "ciphertext");
    const size_t wo = w_out ? w_out : (W + S - 1) / S;
    *out = wrap(variant == 1 ? fheon::stride_extract_v2(*ctx->impl, x->ct, W, S, wo)
                             : fheon::stride_extract_v1(*ctx->impl, x->ct, W, S, wo));
  });
}

int fheon_pad_input(fheon_ctx* ctx, const fheon_ct* x, size_t C, size_t W, size_t P, fheon_ct** out) {
  return guard([&] {
    need(x, "ciphertext");
    fheon::PackedTensor r = fheon::pad_input(*ctx->impl, fheon::PackedTensor{x->ct, C, W}, P);
    *out = wrap(r.data);
  });
}

int fheon_conv_depth_cost(const fheon_conv_cfg* cfg, size_t w_in, int* cost) {
  return guard([&] {
    fheon::ConvConfig c{cfg->in_channels, cfg->out_channels, cfg->kernel, cfg->stride, cfg->padding, cfg->mode,
                        cfg->stride_variant};
    *cost = fheon::conv_depth_cost(c, w_in);
  });
}

}  // extern "C"
