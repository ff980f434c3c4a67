// backend_b200.cpp -- the reference's backend (slotcnn backend.hpp:134-153,
// backend.cpp:38-251) implemented on the B200 RNS-CKKS engine through its C ABI
// (include/fheon_b200.h) only.  Linked in place of the reference's
// backend.cpp, it lets the reference's own layers, model runtime and acceptance
// harness run encrypted on the GPU unchanged (integration/Makefile,
// tests/test_gpu_integration.py).
//
// Semantics kept from the reference: level accounting (rotate keeps, add/sub
// min, mult_plain -1, mult_cipher min-1, bootstrap -> depth budget), the error
// classes and their triggering conditions, trace events (rotation index /
// level_after), bootstrap's optional N(0, sigma^2) perturbation from the
// context's seeded RNG.  What changes: values are ciphertexts in HBM, slots()
// decrypts.
#include <cmath>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "fheon_b200.h"
#include "slotcnn/backend.hpp"

namespace slotcnn {

namespace {

// engine status -> the reference's exception classes (fheon_last_error_kind)
[[noreturn]] void raise_engine_error() {
  const std::string msg = fheon_last_error();
  switch (fheon_last_error_kind()) {
    case 1: throw InvalidRotationError(msg);
    case 2: throw DepthExhaustedError(msg);
    case 3: throw ShapeError(msg);
    case 4: throw CapacityError(msg);
    case 5: throw ModelError(msg);
    default: throw InternalError("B200 engine: " + msg);
  }
}

void check(int rc) {
  if (rc != 0) raise_engine_error();
}

bool power_of_two(std::size_t n) { return n != 0 && (n & (n - 1)) == 0; }

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

// Widest digit (bits) of the balanced contiguous split into <= dnum digits of
// <= 15 limbs -- the engine's digit_split = 1 rule (params.cpp balanced_digits).
double widest_digit_bits(const std::vector<double>& bits, int dnum) {
  auto fits = [&](double cap) {
    int n = 1, size = 0;
    double acc = 0.0;
    for (double b : bits) {
      if (b > cap) return false;
      if (size == 15 || acc + b > cap) {
        ++n;
        acc = 0.0;
        size = 0;
      }
      acc += b;
      ++size;
    }
    return n <= dnum;
  };
  double lo = 0.0, hi = 0.0;
  for (double b : bits) hi += b;
  if (!fits(hi)) throw ShapeError("B200 backend: key_switch_digits too small for a chain of " +
                                  std::to_string(bits.size()) + " limbs (15 limbs per digit at most)");
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    (fits(mid) ? hi : lo) = mid;
  }
  return hi;
}

// RNS chain for a reference ContextConfig.  The reference only carries
// CryptoMetadata; its simulator has no modulus.  Here: full packing (S = N/2),
// the depth budget as application levels at 2^FHEON_SHIM_SCALE_BITS (default
// 45) over a 60-bit q_0, plus 16 bootstrapping levels at 55 bits (sparse h = 64
// secret) so bootstrap() works at every depth, dnum = key_switch_digits with
// digits balanced by bit size, and the fewest 60-bit special primes above the
// widest digit.  The reference's presets (depth 25 at N = 2^14 / 2^15) cannot
// meet 128-bit security, so the chain is created with allow_insecure.
fheon_params chain_for(const ContextConfig& c) {
  if (c.slot_count * 2 != c.ring_dimension)
    throw ShapeError("B200 backend: slot count " + std::to_string(c.slot_count) +
                     " must be half the ring dimension " + std::to_string(c.ring_dimension) +
                     " (the engine packs fully)");
  fheon_params p{};
  p.log_n = 0;
  while ((std::size_t{1} << p.log_n) < c.ring_dimension) ++p.log_n;
  const bool boot = p.log_n >= 11 && env_int("FHEON_SHIM_BOOTSTRAP", 1) != 0;
  p.limbs = c.depth_budget + 1 + (boot ? 16 : 0);
  p.dnum = c.crypto.key_switch_digits > 0 ? c.crypto.key_switch_digits : 4;
  p.first_mod_bits = env_int("FHEON_SHIM_FIRST_BITS", 60);
  p.scale_bits = env_int("FHEON_SHIM_SCALE_BITS", 45);
  p.special_bits = 60;
  p.depth_budget = boot ? -1 : c.depth_budget;
  p.seed = 1;
  p.hamming_weight = boot ? 64 : 0;
  p.bootstrap = boot ? 1 : 0;
  p.boot_scale_bits = boot ? 55 : 0;
  p.digit_split = 1;
  p.allow_insecure = 1;
  p.special_limbs = 1;
  std::vector<std::uint64_t> primes(p.limbs + 16);
  std::vector<double> scales(p.limbs);
  check(fheon_host_primes(&p, primes.data(), scales.data()));
  std::vector<double> qbits(p.limbs);
  for (int i = 0; i < p.limbs; ++i) qbits[i] = std::log2((double)primes[i]);
  const double widest = widest_digit_bits(qbits, p.dnum);
  for (p.special_limbs = 1; p.special_limbs < 16; ++p.special_limbs) {
    check(fheon_host_primes(&p, primes.data(), scales.data()));
    double pbits = 0.0;
    for (int k = 0; k < p.special_limbs; ++k) pbits += std::log2((double)primes[p.limbs + k]);
    if (pbits > widest + 1.0) return p;
  }
  throw ShapeError("B200 backend: no special modulus covers the widest key-switching digit; raise "
                   "key_switch_digits");
}

void require_valid(const SlotVector& v, const char* op) {
  if (!v.valid()) throw InternalError(std::string(op) + ": operand is not initialized");
}

void require_same_context(const SlotVector& a, const SlotVector& b, const char* op) {
  if (!a.valid() || !b.valid()) throw InternalError(std::string(op) + ": operand is not initialized");
  if (a.context() != b.context()) throw InternalError(std::string(op) + ": operands belong to different contexts");
}

void require_depth(const SlotVector& v, const char* op) {
  if (v.level() < 1)
    throw DepthExhaustedError(std::string(op) + ": no multiplicative depth left (level " +
                              std::to_string(v.level()) + ")");
}

}  // namespace

// ------------------------------------------------------------- ContextConfig

void ContextConfig::validate() const {
  if (!power_of_two(slot_count))
    throw ShapeError("slot count must be a power of two, got " + std::to_string(slot_count));
  if (!power_of_two(ring_dimension))
    throw ShapeError("ring dimension must be a power of two, got " + std::to_string(ring_dimension));
  if (slot_count * 2 > ring_dimension)
    throw ShapeError("slot count " + std::to_string(slot_count) + " exceeds half the ring dimension " +
                     std::to_string(ring_dimension));
  if (depth_budget < 1) throw ShapeError("depth budget must be positive, got " + std::to_string(depth_budget));
  if (noise_sigma < 0.0) throw ShapeError("noise sigma must be non-negative");
}

ContextConfig ContextConfig::preset(const std::string& name) {
  ContextConfig cfg;
  if (name == "lenet5") {
    cfg.ring_dimension = 16384;
    cfg.slot_count = 8192;
  } else if (name == "large") {
    cfg.ring_dimension = 32768;
    cfg.slot_count = 16384;
  } else {
    throw ModelError("unknown context preset \"" + name + "\" (expected \"lenet5\" or \"large\")");
  }
  cfg.depth_budget = 25;
  return cfg;
}

bool ContextConfig::is_preset(const std::string& name) { return name == "lenet5" || name == "large"; }

// --------------------------------------------------------------- SlotContext

SlotContext::SlotContext(ContextConfig config)
    : config_(std::move(config)),
      noise_rng_(config_.noise_seed),
      noise_dist_(0.0, config_.noise_sigma > 0.0 ? config_.noise_sigma : 1.0) {
  const fheon_params p = chain_for(config_);
  check(fheon_ctx_create(&p, &engine_));
  if (fheon_ctx_depth_budget(engine_) != config_.depth_budget) {
    fheon_ctx_destroy(engine_);
    engine_ = nullptr;
    throw InternalError("B200 backend: engine depth budget differs from the context's");
  }
}

SlotContext::~SlotContext() {
  if (engine_) fheon_ctx_destroy(engine_);
}

SlotContextPtr SlotContext::create(ContextConfig config) {
  config.validate();
  return SlotContextPtr(new SlotContext(std::move(config)));
}

std::shared_ptr<TraceRecorder> SlotContext::attach_recorder() {
  recorder_ = std::make_shared<TraceRecorder>();
  return recorder_;
}

void SlotContext::attach_recorder(std::shared_ptr<TraceRecorder> recorder) { recorder_ = std::move(recorder); }

void SlotContext::detach_recorder() { recorder_.reset(); }

double SlotContext::sample_noise() { return config_.noise_sigma > 0.0 ? noise_dist_(noise_rng_) : 0.0; }

// --------------------------------------------------------------- PlainVector

PlainVector PlainVector::from_values(std::size_t n, const std::vector<double>& values) {
  if (values.size() > n)
    throw CapacityError("plain vector payload of " + std::to_string(values.size()) + " values does not fit in " +
                        std::to_string(n) + " slots");
  PlainVector p = zeros(n);
  for (std::size_t i = 0; i < values.size(); ++i) p.slots[i] = values[i];
  return p;
}

// ---------------------------------------------------------------- SlotVector

SlotVector::SlotVector(SlotContextPtr ctx, std::vector<double> slots, int level) : ctx_(std::move(ctx)) {
  if (!ctx_) throw InternalError("SlotVector requires a context");
  if (slots.size() != ctx_->slots())
    throw ShapeError("slot payload length " + std::to_string(slots.size()) + " does not match context slot count " +
                     std::to_string(ctx_->slots()));
  if (level < 0 || level > ctx_->depth_budget())
    throw InternalError("SlotVector level " + std::to_string(level) + " outside [0, depth budget]");
  fheon_ct* top = nullptr;
  check(fheon_encrypt(ctx_->engine(), slots.data(), slots.size(), &top));
  fheon_ct* h = top;
  if (level < ctx_->depth_budget()) {
    const int rc = fheon_level_down(ctx_->engine(), top, level + 1, &h);
    fheon_ct_free(top);
    check(rc);
  }
  ct_ = std::shared_ptr<fheon_ct>(h, fheon_ct_free);
  level_ = fheon_ct_level(h);
  id_ = ctx_->next_id();
}

SlotVector::SlotVector(SlotContextPtr ctx, fheon_ct* handle) : ctx_(std::move(ctx)) {
  if (!ctx_ || !handle) throw InternalError("SlotVector requires a context and a ciphertext");
  ct_ = std::shared_ptr<fheon_ct>(handle, fheon_ct_free);
  level_ = fheon_ct_level(handle);
  id_ = ctx_->next_id();
}

SlotVector SlotVector::encode(const SlotContextPtr& ctx, const std::vector<double>& values) {
  if (!ctx) throw InternalError("encode requires a context");
  if (values.size() > ctx->slots())
    throw CapacityError("payload of " + std::to_string(values.size()) + " values does not fit in " +
                        std::to_string(ctx->slots()) + " slots");
  std::vector<double> slots(ctx->slots(), 0.0);
  for (std::size_t i = 0; i < values.size(); ++i) slots[i] = values[i];
  return SlotVector(ctx, std::move(slots), ctx->depth_budget());
}

const std::vector<double>& SlotVector::slots() const {
  if (!slots_) {
    if (!valid()) throw InternalError("slots: value is not initialized");
    auto v = std::make_shared<std::vector<double>>(ctx_->slots());
    check(fheon_decrypt(ctx_->engine(), ct_.get(), v->data(), v->size()));
    slots_ = std::move(v);
  }
  return *slots_;
}

// ----------------------------------------------------------------------- ops

SlotVector rotate(const SlotVector& v, long t) {
  require_valid(v, "rotate");
  const long n = static_cast<long>(v.size());
  if (t <= -n || t >= n)
    throw InvalidRotationError("rotation amount " + std::to_string(t) + " out of range for " + std::to_string(n) +
                               " slots");
  fheon_ct* out = nullptr;
  check(fheon_rotate(v.context()->engine(), v.handle(), t, &out));
  if (TraceRecorder* rec = v.context()->recorder()) rec->record_rotation(t);
  return SlotVector(v.context(), out);
}

SlotVector add(const SlotVector& a, const SlotVector& b) {
  require_same_context(a, b, "add");
  fheon_ct* out = nullptr;
  check(fheon_add(a.context()->engine(), a.handle(), b.handle(), &out));
  return SlotVector(a.context(), out);
}

SlotVector sub(const SlotVector& a, const SlotVector& b) {
  require_same_context(a, b, "sub");
  fheon_ct* out = nullptr;
  check(fheon_sub(a.context()->engine(), a.handle(), b.handle(), &out));
  return SlotVector(a.context(), out);
}

SlotVector mult_plain(const SlotVector& v, const PlainVector& p) {
  require_valid(v, "mult_plain");
  if (p.slots.size() != v.size())
    throw ShapeError("mult_plain: plaintext length " + std::to_string(p.slots.size()) +
                     " does not match slot count " + std::to_string(v.size()));
  require_depth(v, "mult_plain");
  fheon_ct* out = nullptr;
  check(fheon_mult_plain(v.context()->engine(), v.handle(), p.slots.data(), p.slots.size(), &out));
  SlotVector r(v.context(), out);
  if (r.level() != v.level() - 1) throw InternalError("mult_plain: engine level accounting differs");
  if (TraceRecorder* rec = v.context()->recorder()) rec->record_mult_plain(r.level());
  return r;
}

SlotVector mult_cipher(const SlotVector& a, const SlotVector& b) {
  require_same_context(a, b, "mult_cipher");
  require_depth(a, "mult_cipher");
  require_depth(b, "mult_cipher");
  fheon_ct* out = nullptr;
  check(fheon_mult_cipher(a.context()->engine(), a.handle(), b.handle(), &out));
  SlotVector r(a.context(), out);
  if (TraceRecorder* rec = a.context()->recorder()) rec->record_mult_cipher(r.level());
  return r;
}

SlotVector bootstrap(const SlotVector& v) {
  require_valid(v, "bootstrap");
  SlotContext& ctx = *v.context();
  fheon_ct* out = nullptr;
  check(fheon_bootstrap(ctx.engine(), v.handle(), &out));
  if (ctx.config().noise_sigma > 0.0) {
    std::vector<double> noise(ctx.slots());
    for (double& s : noise) s = ctx.sample_noise();
    fheon_ct* noisy = nullptr;
    const int rc = fheon_add_plain(ctx.engine(), out, noise.data(), noise.size(), &noisy);
    fheon_ct_free(out);
    check(rc);
    out = noisy;
  }
  SlotVector r(v.context(), out);
  if (r.level() != ctx.depth_budget()) throw InternalError("bootstrap: engine did not restore the depth budget");
  if (TraceRecorder* rec = ctx.recorder()) rec->record_bootstrap(r.level());
  return r;
}

}  // namespace slotcnn
