// B200 RNS-CKKS engine: context (device tables, keys, stream, allocator),
// device ciphertext handles and the evaluator ops that replace the
// reference's slot-vector backend (proj/include/slotcnn/backend.hpp:134-153):
//
//   reference op (backend.cpp)      engine realisation
//   rotate      :165-182            Galois automorphism + hybrid key switch
//   add / sub   :184-198            level/scale alignment + limb-wise mod add
//   mult_plain  :200-217            encode at the operand's scale, Hadamard, rescale
//   mult_cipher :219-231            tensor, relinearise (key switch), rescale
//   bootstrap   :233-249            not yet available (throws)
//   SlotVector::encode :148-161     encode + encrypt at the depth budget
//
// Level semantics follow the reference exactly: level = limbs - 1, add/sub
// give min(level), mult_plain level-1, mult_cipher min-1, multiplication at
// level 0 throws DepthExhaustedError (backend.cpp:27-32).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "kernels.hpp"
#include "params.hpp"

namespace fheon {

// ---- errors (mirrors proj/include/slotcnn/errors.hpp:18-80)
enum class ErrKind : int {
  generic = 0,
  invalid_rotation = 1,  // data
  depth_exhausted = 2,   // internal
  shape = 3,             // data
  capacity = 4,          // data
  model = 5,             // data
  internal = 6,          // internal
  cuda = 7,              // internal
  not_implemented = 8,   // usage
};
int category_of(ErrKind k);  // usage 1, data 2, internal 3

struct Error : std::runtime_error {
  ErrKind kind;
  Error(ErrKind k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

void cuda_check(cudaError_t e, const char* what);
extern std::atomic<std::uint64_t> g_kernel_launches;
#define FHEON_CUDA(x) ::fheon::cuda_check((x), #x)

class Context;
class Bootstrapper;

struct DevBuffer {
  // stream-ordered free while the owning context lives; a synchronous free if
  // a handle outlives its context
  std::shared_ptr<std::atomic<bool>> alive;
  cudaStream_t stream = nullptr;
  u64* ptr = nullptr;
  std::size_t words = 0;
  DevBuffer(Context* c, std::size_t w);
  // allocated in `alloc_stream`'s order (e.g. the upload stream), freed in the context stream's
  DevBuffer(Context* c, std::size_t w, cudaStream_t alloc_stream);
  ~DevBuffer();
  DevBuffer(const DevBuffer&) = delete;
  DevBuffer& operator=(const DevBuffer&) = delete;
};
using BufPtr = std::shared_ptr<DevBuffer>;

// Immutable ciphertext handle: (c0, c1) in the NTT domain, `limbs` active
// limbs (q_0..q_{limbs-1}); copies share the device buffer.  Dropping limbs
// is a zero-copy view (the tail limbs stay allocated).
struct Ciphertext {
  BufPtr buf;
  u64* c0 = nullptr;
  u64* c1 = nullptr;
  int limbs = 0;
  double scale = 0.0;
  std::uint64_t id = 0;
  bool valid() const { return static_cast<bool>(buf); }
  int level() const { return limbs - 1; }
};

struct TraceEvent {
  int kind;    // 0 rotation, 1 mult_plain, 2 mult_cipher, 3 bootstrap, 4 marker
  long value;  // rotation index or level_after
  std::string label;
};

struct OpStats {
  std::uint64_t rotations = 0, keyswitches = 0, mult_plain = 0, mult_cipher = 0, rescales = 0, ntt_limbs = 0,
                encodes = 0, adds = 0, launches = 0, bootstraps = 0;
  std::uint64_t key_gens = 0, key_drops = 0;  // key residency (keyplan block mode)
  std::uint64_t key_uploads = 0, key_upload_bytes = 0;  // keys received over PCIe (fheon_key_upload*)
};

struct KernelTimer {
  int cls = 0;  // armed class (0 = off)
  std::vector<cudaEvent_t> ev;
  std::size_t used = 0;
  int depth = 0;
  ~KernelTimer();
  void begin(cudaStream_t st);
  void end(cudaStream_t st);
  // total milliseconds and number of timed scopes since the last reset (synchronises)
  double total_ms(int* count);
  void reset() { used = 0; depth = 0; }
};

class Context {
 public:
  explicit Context(const Params& p);
  // (delegation target of both public constructors)
  Context(const Params& p, const Context* share_keys_from);
  // a second context over the same parameters and secret that SHARES the parent's
  // resident evaluation keys (read-only device buffers) instead of generating its
  // own: its own stream, pools' streams, caches and counters, so two images can be
  // in flight on one GPU without doubling the key memory
  Context(const Params& p, const Context& share_keys_from);
  ~Context();
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  const HostTables& host() const { return ht_; }
  const DevTables& dev() const { return dt_; }
  cudaStream_t stream() const { return stream_; }
  // this context's own stream-ordered pool (null: the device's default pool)
  cudaMemPool_t mem_pool() const { return pool_; }
  std::size_t N() const { return ht_.N; }
  int S() const { return ht_.S; }
  int L() const { return ht_.p.L; }
  int K() const { return ht_.p.K; }
  int depth_budget() const { return depth_budget_; }
  // security disclosure: log2(QP) of the whole chain and the HE-standard level it meets
  // (he_standard_security: 128/192/256, 0 below 128, -1 sparse main secret)
  double log_qp() const { return log_qp_; }
  int security() const { return security_; }
  // bootstrapping through the sparse-secret encapsulation (dense main secret)
  bool sse() const { return ht_.p.bootstrap && ht_.p.hamming_weight <= 0; }

  BufPtr alloc(std::size_t words);
  Ciphertext new_ct(int limbs);
  std::uint64_t next_id() { return ++id_counter_; }

  // ---- keys: [dnum][2][L+K][N] Montgomery form on the device
  u64 galois(long t) const;
  const u64* key(u64 key_id);  // generates on demand unless strict_keys
  void gen_key(u64 key_id);
  bool has_key(u64 key_id) const { return keys_.count(key_id) != 0; }
  void drop_keys() { keys_.clear(); }
  // pinned keys (relinearisation, conjugation, bootstrapping rotations) are never dropped
  void pin_key(u64 key_id) { pinned_keys_.insert(key_id); }
  // the pinned set: relinearisation, conjugation, bootstrapping rotations, encapsulation keys
  std::vector<u64> pinned_keys() const { return {pinned_keys_.begin(), pinned_keys_.end()}; }
  void drop_key(u64 key_id) {
    if (!pinned_keys_.count(key_id) && keys_.erase(key_id)) ++stats.key_drops;
  }
  std::size_t key_words() const;
  std::size_t num_keys() const { return keys_.size(); }
  // make an uploaded key (Montgomery form, [dnum][2][L+K][N]) resident under key_id
  void put_key(u64 key_id, BufPtr kb) { keys_[key_id] = std::move(kb); }
  // a server context (Params::no_secret) cannot generate keys, encrypt or decrypt
  bool has_secret() const { return dt_.s_ntt != nullptr; }
  // true while a key-sharing clone is being built (its keys come from the parent)
  bool inheriting_keys = false;
  void require_secret(const char* what) const;
  bool strict_keys = false;

  // ---- encoder (host special FFT)
  void encode_coeffs(const double* vals, std::size_t n, double scale, long long* coeffs) const;
  void decode_coeffs(const double* coeffs, double scale, double* out, double* out_im = nullptr) const;
  // encode `vals` at `scale` over `limbs` limbs into a device [limbs][N] NTT-domain buffer
  BufPtr encode(const double* vals, std::size_t n, int limbs, double scale);
  // the N signed coefficients of round(scale * canonical-embedding preimage), computed on the device
  BufPtr encode_device(const double* re, const double* im, std::size_t n, double scale);
  // complex slot values (re + i im), host special FFT
  // special > 0: also the first `special` special primes (limbs + special rows, Q u P operands)
  BufPtr encode_complex(const double* re, const double* im, std::size_t n, int limbs, double scale, int special = 0);
  // content-addressed cache over encode() (masks reused across a layer)
  BufPtr encode_cached(const std::vector<double>& vals, int limbs, double scale);
  // same cache keyed by a caller-chosen name (the slot values are built only on a miss)
  BufPtr encode_named(const std::string& name, const std::function<std::vector<double>()>& make, int limbs,
                      double scale);
  // weight plaintexts (conv kernel vectors) kept resident across calls, the
  // reference's weight_mode "preload" (model.hpp:46-48): built once by `make`
  // under `key`, then reused; past the budget new entries are built but not kept
  BufPtr weight_pt(const std::string& key, int limbs, double scale, const std::function<BufPtr()>& make);
  std::size_t weight_cache_budget = (std::size_t)96 << 30;  // bytes (<= free HBM / 2 at creation); 0 disables
  // drop the resident plaintext caches (weights, masks, diagonals); buffers still in
  // use stay alive through their handles.  Called when a device allocation fails
  // (HBM shared with the lazily generated keys), before the allocation is retried.
  std::size_t release_caches();
  // device real-coefficient (unscaled, unrounded) encoding of a slot vector,
  // cached under `key` (block indicators of a layer geometry)
  const double* basis(const std::string& key, const std::vector<double>& slot_values);
  // same, building the slot values only on a cache miss
  const double* basis(const std::string& key, const std::function<std::vector<double>()>& make);
  // plaintext = round(scale * sum_b w_b basis_b), NTT domain over `limbs` limbs
  BufPtr encode_lincomb(const LinComb& lc, int limbs, double scale);

  // ---- trace (mirrors slotcnn TraceRecorder, trace.hpp:22-103)
  void set_tracing(bool on) { tracing_ = on; }
  bool tracing() const { return tracing_; }
  void record(int kind, long value, const std::string& label = {});
  std::vector<TraceEvent> trace_snapshot() const;
  void clear_trace();

  // rotation schedule of the layer algorithms: kScheduleFast hoists rotation
  // chains into log-depth trees / baby-step giant-step sets (same outputs and
  // levels, far fewer key switches); kScheduleReference replays the
  // reference's exact rotation sequence (identical trace multiset)
  static constexpr int kScheduleFast = 0, kScheduleReference = 1;
  int schedule = kScheduleFast;
  bool fast_schedule() const { return schedule == kScheduleFast; }

  OpStats stats;
  KernelTimer timer;
  std::uint64_t enc_counter = 0;
  std::unique_ptr<Bootstrapper> boot;  // present when Params::bootstrap
  // sparse-slot variants: boot_sparse[k - 1] carries n = S >> k slots (Params::boot_sparse)
  std::vector<std::unique_ptr<Bootstrapper>> boot_sparse;

  // staging for host -> device copies of encoded coefficients
  long long* staging_slot(cudaEvent_t** ev);

  // ---- asynchronous ciphertext transfers on dedicated copy streams (the
  // host -> device copy of the next batch, the compute of this one and the
  // device -> host copy of the previous one overlap)
  cudaStream_t h2d_stream() const { return h2d_; }
  cudaStream_t d2h_stream() const { return d2h_; }
  // (un)pack kernels of the packed transfers: off the copy streams, so the copy
  // engines stream back to back while the previous ciphertext is (un)packed
  cudaStream_t unpack_stream() const { return unpack_; }
  cudaStream_t pack_stream() const { return pack_; }
  cudaEvent_t take_event();
  void give_event(cudaEvent_t e);
  // keep `buf` alive until `done` has completed (a device -> host copy in flight)
  void hold_until(cudaEvent_t done, BufPtr buf);
  void reap_transfers(bool wait);  // release finished (or, with wait, all) held buffers

 private:
  void build_device_tables();

  HostTables ht_;
  DevTables dt_{};
  cudaStream_t stream_ = nullptr;
  cudaMemPool_t pool_ = nullptr;
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr, unpack_ = nullptr, pack_ = nullptr;
  std::vector<cudaEvent_t> event_pool_;
  std::vector<std::pair<cudaEvent_t, BufPtr>> held_;
  int depth_budget_ = 0;
  double log_qp_ = 0.0;
  int security_ = 0;
  std::uint64_t id_counter_ = 0;
  std::vector<void*> dev_allocs_;  // table allocations
 public:
  std::shared_ptr<std::atomic<bool>> alive = std::make_shared<std::atomic<bool>>(true);

 private:
  std::map<u64, BufPtr> keys_;
  std::set<u64> pinned_keys_;
  std::map<std::string, BufPtr> basis_;
  struct PtEntry {
    std::vector<double> vals;
    BufPtr buf;
  };
  std::map<std::tuple<u64, int, double>, std::vector<PtEntry>> ptcache_;
  std::map<std::tuple<std::string, int, double>, BufPtr> namedcache_;
  std::map<std::tuple<std::string, int, double>, BufPtr> weightcache_;
  std::size_t weightcache_bytes_ = 0;
  std::size_t ptcache_words_ = 0;
  void ptcache_reserve(std::size_t words);
  mutable std::mutex trace_mu_;
  bool tracing_ = false;
  std::vector<TraceEvent> trace_;
  static constexpr int kStaging = 16;
  long long* staging_[kStaging] = {};
  cudaEvent_t staging_ev_[kStaging] = {};
  int staging_next_ = 0;
};

// canonical-embedding encode on the host (special FFT)
void encode_coeffs_host(const HostTables& h, const double* vals, std::size_t n, double scale, long long* coeffs);
// unscaled real coefficients (N doubles: re[0..S), im[0..S)) before rounding
void encode_real_host(const HostTables& h, const double* vals, std::size_t n, double* out);

// ---- batched evaluator ops (layer kernels)
// plaintext scale that lands a mult_plain on the next level's target scale
double pt_scale_for(const Context& ctx, const Ciphertext& a);
std::vector<Ciphertext> rescale_many(Context& ctx, const std::vector<Ciphertext>& as);
// out[o] = rescale( sum_j terms[o][j] (*) pts[o][j] ): one fused MAC, one rescale.
// All terms share level and scale; pts are encoded at pt_scale_for(term).  Records
// one mult_plain trace event per term (level_after = level - 1), o-major.
std::vector<Ciphertext> mac_plain_many(Context& ctx, const std::vector<std::vector<Ciphertext>>& terms,
                                       const std::vector<std::vector<BufPtr>>& pts);
// the same fused MAC without the rescale: outputs stay at `limbs` with scale
// T_{lv-1} q_lv (rotations commute with the deferred rescale, so a rotate-and-sum
// over such outputs needs one rescale instead of one per term); trace as above
std::vector<Ciphertext> mac_plain_many_unrescaled(Context& ctx, const std::vector<std::vector<Ciphertext>>& terms,
                                                  const std::vector<std::vector<BufPtr>>& pts);
// rescale_to_target(rotate_sum_many(groups)) with each group's rescale folded into its
// ModDown (one rounding by P q_l); identity terms join before the division
// (record_identity: trace the t = 0 terms as rotations, as rotate_sum_many does)
// with_conj: every term also enters conjugated (Galois element -5^t: the sum becomes
// out + conj(out) in the same ModDown; keys for conj o rot_t must be resident)
std::vector<Ciphertext> rotate_sum_to_target(Context& ctx,
                                             const std::vector<std::vector<std::pair<Ciphertext, long>>>& groups,
                                             bool record_identity = true, bool with_conj = false);
// rescale unrescaled MAC outputs onto the next level's target scale
std::vector<Ciphertext> rescale_to_target(Context& ctx, const std::vector<Ciphertext>& prods);
std::vector<Ciphertext> add_many(Context& ctx, const std::vector<Ciphertext>& a, const std::vector<Ciphertext>& b);
std::vector<Ciphertext> conjugate_many(Context& ctx, const std::vector<Ciphertext>& xs);
Ciphertext mul_by_i(Context& ctx, const Ciphertext& x);
Ciphertext mod_raise(Context& ctx, const Ciphertext& x);
// ModRaise + the sparse-slot trace sum_{j < S/n} rot(., j n), the encapsulation's switch back
// folded into the trace's key switches (keys key_from_sparse_rot)
Ciphertext mod_raise_trace(Context& ctx, const Ciphertext& x, long n);
std::vector<Ciphertext> mod_raise_trace_many(Context& ctx, const std::vector<Ciphertext>& xs, long n);
Ciphertext encrypt_at(Context& ctx, const double* vals, std::size_t n, int limbs);
// add an encoded plaintext (encoded at a's level and scale)
Ciphertext add_plain_pt(Context& ctx, const Ciphertext& a, const BufPtr& pt);
std::vector<Ciphertext> mult_cipher_many(Context& ctx, const std::vector<Ciphertext>& as,
                                         const std::vector<Ciphertext>& bs);
// 2 a_i b_i - subs_i (subs_i may be invalid: 2 a_i b_i), the Chebyshev recurrence step,
// in one relinearise-and-rescale (the subtrahend joins before the rescale)
std::vector<Ciphertext> mult_cipher_cheb_many(Context& ctx, const std::vector<Ciphertext>& as,
                                              const std::vector<Ciphertext>& bs, const std::vector<Ciphertext>& subs);
std::vector<Ciphertext> mult_const_many(Context& ctx, const std::vector<Ciphertext>& as, const std::vector<double>& cs);
// sum_i cs[i] * xs[i] + c0 with one rescale (terms may sit at different levels)
Ciphertext lincomb_const(Context& ctx, const std::vector<Ciphertext>& xs, const std::vector<double>& cs, double c0);
// the same landing exactly on (out_limbs, out_scale); every term needs >= out_limbs + 1 limbs
struct LincombItem {
  std::vector<Ciphertext> xs;
  std::vector<double> cs;
  double c0 = 0.0;
  int out_limbs = 0;
  double out_scale = 0.0;
};
// several lincomb_const_to at once: the rescales of one level batched
std::vector<Ciphertext> lincomb_const_to_many(Context& ctx, const std::vector<LincombItem>& items);
Ciphertext lincomb_const_to(Context& ctx, const std::vector<Ciphertext>& xs, const std::vector<double>& cs, double c0,
                            int out_limbs, double out_scale);

// ---------------------------------------------------------------- ops
Ciphertext encrypt(Context& ctx, const double* vals, std::size_t n);            // at the depth budget
Ciphertext encrypt_top(Context& ctx, const double* vals, std::size_t n);        // at L-1 (all limbs)
void decrypt(Context& ctx, const Ciphertext& ct, double* out, double* out_im = nullptr);  // S slots
Ciphertext rotate(Context& ctx, const Ciphertext& x, long t);
std::vector<Ciphertext> rotate_hoisted(Context& ctx, const Ciphertext& x, const std::vector<long>& ts);
// xs[i] rotated by ts[i]: one batched key-switch pipeline, shared ModUp for repeated inputs
std::vector<Ciphertext> rotate_many(Context& ctx, const std::vector<Ciphertext>& xs, const std::vector<long>& ts);
// out[r] = sum_k rot(x_rk, t_rk): rotate-and-sum, one ModDown per output (the
// rotated c0 terms are folded into the key-switch accumulator as P * c0)
std::vector<Ciphertext> rotate_sum_many(Context& ctx,
                                        const std::vector<std::vector<std::pair<Ciphertext, long>>>& groups);
// Double-hoisted baby-step giant-step linear transform (evaluator.cpp):
// out = rescale(sum_g rot(sum_t pt_t (*) rot(x, babies[b_t]), rot_g)); a term's baby
// index -1 is the identity; plaintexts are [limbs+K][N] over Q u P, encoded at
// pt_scale_for(x) (at most 32 terms per giant)
struct DhGiant {
  long rot = 0;
  std::vector<std::pair<int, BufPtr>> terms;
};
Ciphertext bsgs_double_hoisted(Context& ctx, const Ciphertext& x, const std::vector<long>& babies,
                               const std::vector<DhGiant>& giants, bool with_conj = false);
// the same transform on several ciphertexts of one level and scale in lockstep (keys and
// plaintext diagonals read once per batch); outputs bit-identical to the single-input call
std::vector<Ciphertext> bsgs_double_hoisted_many(Context& ctx, const std::vector<Ciphertext>& xs,
                                                 const std::vector<long>& babies, const std::vector<DhGiant>& giants,
                                                 bool with_conj = false);
Ciphertext add(Context& ctx, const Ciphertext& a, const Ciphertext& b);
Ciphertext sub(Context& ctx, const Ciphertext& a, const Ciphertext& b);
Ciphertext add_plain(Context& ctx, const Ciphertext& a, const double* vals, std::size_t n);
Ciphertext add_const(Context& ctx, const Ciphertext& a, double c);
Ciphertext mult_plain(Context& ctx, const Ciphertext& a, const double* vals, std::size_t n);
Ciphertext mult_const(Context& ctx, const Ciphertext& a, double c);
Ciphertext mult_cipher(Context& ctx, const Ciphertext& a, const Ciphertext& b);
Ciphertext level_down(Context& ctx, const Ciphertext& a, int target_limbs);
Ciphertext rescale(Context& ctx, const Ciphertext& a);
Ciphertext bootstrap(Context& ctx, const Ciphertext& a);
// bootstrap when only slots [0, active) matter: the smallest sparse-slot variant
// holding them (input above level 0), else the full pipeline.  Output slots
// [0, active) = input (the rest 0 for a sparse variant, the input's for the full one)
// clean: the caller knows slots [active, S) of a are zero (a convolution's output) -- no
// mask, so a level-0 input can take a sparse variant too
Ciphertext bootstrap_active(Context& ctx, const Ciphertext& a, std::size_t active, bool clean = false);
std::vector<Ciphertext> bootstrap_active_many(Context& ctx, const std::vector<Ciphertext>& as, std::size_t active,
                                              bool clean = false);
// raw key switch of one polynomial d ([limbs][N], NTT) for parity tests:
// returns (ks0, ks1) as a 2-poly ciphertext without scale meaning
Ciphertext keyswitch_raw(Context& ctx, const Ciphertext& d_as_c1, u64 key_id, u64 g);

// device <-> host for parity tests
Ciphertext upload_ct(Context& ctx, const u64* host, int limbs, double scale);
void download_ct(Context& ctx, const Ciphertext& ct, u64* host);
// non-blocking variants (host buffers must stay valid -- and should be pinned --
// until wait_transfers): the upload runs on the H2D stream and the context stream
// waits for it; the download waits for the context stream and runs on the D2H stream
Ciphertext upload_ct_async(Context& ctx, const u64* host, int limbs, double scale);
void download_ct_async(Context& ctx, const Ciphertext& ct, u64* host);
void wait_transfers(Context& ctx);
// packed wire format (kernels.hpp PackLayout): [2][limbs][N b_i / 64] words, b_i = bit_length(q_i)
PackLayout pack_layout(const Context& ctx, int limbs);
std::size_t packed_words(const Context& ctx, int limbs);
Ciphertext upload_ct_packed_async(Context& ctx, const u64* host, int limbs, double scale);
// evaluation-key transfer (client -> server, keyplan streaming): standard-form words
// [dnum][2][L+K][N], raw or in the packed wire format (every limb b_i = bit_length of
// its prime, the ciphertext layout applied to the 2 dnum polys of L+K limbs)
std::size_t key_packed_words(const Context& ctx);
void download_key_packed(Context& ctx, u64 key_id, u64* host);
// upload on the context's upload stream; the compute stream waits for it, the host
// buffer must stay valid (and should be pinned) until the copy completes
// (fheon_ctx_wait_transfers); replaces a resident key of the same id
void upload_key_async(Context& ctx, u64 key_id, const u64* host, bool packed);
void download_ct_packed_async(Context& ctx, const Ciphertext& ct, u64* host);

}  // namespace fheon
