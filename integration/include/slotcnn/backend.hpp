// slotcnn/backend.hpp -- the B200 drop-in replacement of the reference's
// backend header (/root/reference/proj/include/slotcnn/backend.hpp:1-155).
//
// Same namespace, types, member functions and free functions as the reference,
// so its layers (layers_conv.cpp, layers_misc.cpp), Chebyshev evaluator,
// packing helpers, model builder / runtime and its tests compile UNCHANGED
// against this header (integration/Makefile puts integration/include ahead of
// the reference's include directory).  The only delta is the representation:
//
//   reference  SlotVector = shared_ptr<const vector<double>> of S cleartext
//              slots + level (a simulator, backend.cpp:165-249)
//   here       SlotVector = shared handle to an RNS-CKKS ciphertext resident in
//              HBM (fheon_ct, include/fheon_b200.h); level() is the
//              ciphertext's level; slots() decrypts on first use and caches
//
// and SlotContext owns an engine context (fheon_ctx) created from the
// ContextConfig.  Every op is implemented in integration/backend_b200.cpp on
// top of the C ABI only.  See INTEGRATION.md.
#pragma once

#include <cstdint>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "slotcnn/errors.hpp"
#include "slotcnn/trace.hpp"

struct fheon_ctx;
struct fheon_ct;

namespace slotcnn {

/// CKKS metadata (backend.hpp:34-39 in the reference, where it is carried only):
/// the B200 backend reads key_switch_digits as dnum; see backend_b200.cpp
/// chain_for() for how the RNS chain is derived.
struct CryptoMetadata {
  int first_modulus_bits = 50;
  int rescale_bits = 46;
  int key_switch_digits = 4;
  std::string rescaling_strategy = "flexibleauto";
};

struct ContextConfig {
  std::size_t ring_dimension = 16384;
  std::size_t slot_count = 8192;
  int depth_budget = 25;
  CryptoMetadata crypto{};
  /// bootstrap() adds N(0, noise_sigma^2) per slot after refreshing, as the
  /// reference's simulator does (0 keeps the refresh noise-free beyond CKKS's own)
  double noise_sigma = 0.0;
  std::uint64_t noise_seed = 1;

  void validate() const;
  static ContextConfig preset(const std::string& name);
  static bool is_preset(const std::string& name);
};

class SlotContext;
using SlotContextPtr = std::shared_ptr<SlotContext>;

/// Owns the GPU engine context (keys resident in HBM, one CUDA stream) plus the
/// reference's trace recorder and bootstrap-noise source.
class SlotContext : public std::enable_shared_from_this<SlotContext> {
 public:
  static SlotContextPtr create(ContextConfig config);
  ~SlotContext();
  SlotContext(const SlotContext&) = delete;
  SlotContext& operator=(const SlotContext&) = delete;

  const ContextConfig& config() const { return config_; }
  std::size_t slots() const { return config_.slot_count; }
  int depth_budget() const { return config_.depth_budget; }

  std::shared_ptr<TraceRecorder> attach_recorder();
  void attach_recorder(std::shared_ptr<TraceRecorder> recorder);
  void detach_recorder();
  TraceRecorder* recorder() const { return recorder_.get(); }

  double sample_noise();
  std::uint64_t next_id() { return ++id_counter_; }

  /// the engine context behind this SlotContext (C ABI handle)
  fheon_ctx* engine() const { return engine_; }

 private:
  explicit SlotContext(ContextConfig config);

  ContextConfig config_;
  fheon_ctx* engine_ = nullptr;
  std::shared_ptr<TraceRecorder> recorder_;
  std::mt19937_64 noise_rng_;
  std::normal_distribution<double> noise_dist_;
  std::uint64_t id_counter_ = 0;
};

/// A plaintext operand (S slot values); encoded on the device at the
/// consumer's level and scale by mult_plain.
struct PlainVector {
  std::vector<double> slots;

  static PlainVector zeros(std::size_t n) { return {std::vector<double>(n, 0.0)}; }
  static PlainVector from_values(std::size_t n, const std::vector<double>& values);
};

/// A packed ciphertext handle: immutable, cheap to copy (shared handle).
class SlotVector {
 public:
  SlotVector() = default;

  /// Encrypts `slots` (S values) at `level` -- the reference's constructor of a
  /// fresh value (used for constants, chebyshev.cpp:75,84).
  SlotVector(SlotContextPtr ctx, std::vector<double> slots, int level);
  /// Wraps an engine ciphertext the caller owns (ownership moves in).
  SlotVector(SlotContextPtr ctx, fheon_ct* handle);

  static SlotVector encode(const SlotContextPtr& ctx, const std::vector<double>& values);

  bool valid() const { return static_cast<bool>(ctx_) && static_cast<bool>(ct_); }
  const SlotContextPtr& context() const { return ctx_; }
  /// decrypted slot values (decrypted once per handle, then cached)
  const std::vector<double>& slots() const;
  std::size_t size() const { return ctx_ ? ctx_->slots() : 0; }
  double at(std::size_t i) const { return slots()[i]; }
  int level() const { return level_; }
  std::uint64_t id() const { return id_; }

  /// the engine ciphertext (valid while this value lives)
  const fheon_ct* handle() const { return ct_.get(); }

 private:
  SlotContextPtr ctx_;
  std::shared_ptr<fheon_ct> ct_;
  mutable std::shared_ptr<const std::vector<double>> slots_;
  int level_ = 0;
  std::uint64_t id_ = 0;
};

SlotVector rotate(const SlotVector& v, long t);
SlotVector add(const SlotVector& a, const SlotVector& b);
SlotVector sub(const SlotVector& a, const SlotVector& b);
SlotVector mult_plain(const SlotVector& v, const PlainVector& p);
SlotVector mult_cipher(const SlotVector& a, const SlotVector& b);
SlotVector bootstrap(const SlotVector& v);

}  // namespace slotcnn
