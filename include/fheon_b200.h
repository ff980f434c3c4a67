/* fheon_b200.h -- C ABI of the B200-native RNS-CKKS engine for FHEON's
 * encrypted-CNN hot path (arXiv 2510.03996).
 *
 * The reference (slotcnn, /root/reference/proj) is a C++ library with no FFI:
 * its "plug point" is the backend free functions of
 * proj/include/slotcnn/backend.hpp:134-153 and the layer API of
 * proj/include/slotcnn/layers.hpp:83-158, replaced at link time
 * (SURVEY.md section 8(b)).  Each entry point below names the reference
 * interface it replaces.  INTEGRATION.md shows the C++ shim a maintainer
 * links into slotcnn (and the ctypes stub used by this repo's tests).
 *
 * Conventions
 *   - every function returns 0 on success, else the reference ErrorCategory
 *     (errors.hpp:18-22): 1 usage, 2 data, 3 internal; fheon_last_error()
 *     returns the message (thread-local), fheon_last_error_kind() the
 *     exception class (1 InvalidRotationError, 2 DepthExhaustedError,
 *     3 ShapeError, 4 CapacityError, 5 ModelError, 6 InternalError, 7 CUDA,
 *     8 not implemented).
 *   - ciphertext handles are immutable values (backend.hpp:106-131); every op
 *     returns a fresh handle the caller releases with fheon_ct_free().
 *   - all work is enqueued on the context's CUDA stream (fheon_ctx_stream);
 *     calls that return host data synchronise it.
 *   - levels follow the reference: level = limbs - 1; add/sub -> min level,
 *     mult_plain -> level - 1, mult_cipher -> min - 1 (backend.hpp:10-16).
 */
#ifndef FHEON_B200_H
#define FHEON_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fheon_ctx fheon_ctx;
typedef struct fheon_ct fheon_ct;

/* Replaces ContextConfig + CryptoMetadata (backend.hpp:34-59), which the
 * reference only carries as metadata; here they define the RNS chain. */
typedef struct {
  int log_n;          /* ring degree N = 2^log_n (10..16); slots S = N/2 */
  int limbs;          /* L: Q-chain limbs (levels 0..L-1) */
  int special_limbs;  /* K: special primes for hybrid key switching */
  int dnum;           /* key-switching digits */
  int first_mod_bits; /* bits of q_0 (CryptoMetadata::first_modulus_bits) */
  int scale_bits;     /* scaling-prime bits (CryptoMetadata::rescale_bits) */
  int special_bits;   /* special-prime bits */
  int depth_budget;   /* ContextConfig::depth_budget; -1 = limbs - 1 */
  uint64_t seed;      /* key / encryption randomness seed */
  int hamming_weight; /* secret: 0 uniform ternary, h > 0 sparse with h nonzero coefficients */
  int bootstrap;      /* 1: enable CKKS bootstrapping (bootstrap() refreshes to depth_budget) */
  int boot_scale_bits;/* scale of the bootstrapping levels (0 = scale_bits) */
  int digit_split;    /* key-switching digits: 0 uniform ceil(limbs/dnum), 1 balanced by bit size */
  /* bootstrapping with a dense secret (hamming_weight 0) runs the sparse-secret encapsulation:
   * the level-0 ciphertext is switched to an ephemeral sparse secret of this Hamming weight
   * (0 = 64) on q_0 and the special primes only, ModRaised, and switched back */
  int boot_hamming_weight;
  /* security: context creation refuses a chain whose log2(QP) exceeds the HE-standard bound
   * (uniform ternary secret, classical) for N at min_security bits (0 = 128), or whose main
   * secret is sparse, unless allow_insecure = 1 (the reference's presets need it) */
  int min_security;
  int allow_insecure;
  /* 1: a SERVER context holding no secret key.  Evaluation keys (rotation, relinearisation,
   * the bootstrapping set listed by fheon_required_key_ids) arrive by fheon_key_upload*;
   * encrypt / decrypt / key generation fail.  The client creates a context with the same
   * parameters (and seed) and generates / downloads the keys. */
  int no_secret;
  /* EvalMod range K of bootstrapping: |I| <= K for the ModRaise overflow (0 = 16).  With the
   * encapsulation secret at h_b = 32 (sigma(I) = 1.66) K = 12 is a 7-sigma margin and lowers
   * the cosine's degree -- one bootstrapping level less */
  int boot_k_range;
  /* levels of the bootstrapping linear transforms (0 = 3 each): CoeffsToSlots, SlotsToCoeffs */
  int boot_cts_levels;
  int boot_stc_levels;
  /* sparse-slot bootstrapping variants over n = S/2, S/4, ..., S/2^boot_sparse slots, built at
   * context creation (their rotation keys join the pinned set); fheon_bootstrap_active picks one */
  int boot_sparse;
} fheon_params;

/* ---- errors / version */
const char* fheon_last_error(void);
int fheon_last_error_kind(void);
int fheon_version(void);

/* ---- host-only helpers (no device needed) */
/* prime chain q_0..q_{L-1}, p_0..p_{K-1} and the per-level scale targets */
int fheon_host_primes(const fheon_params* p, uint64_t* primes, double* scales);
/* canonical-embedding encode of n <= N/2 slot values at `scale` -> N signed coefficients */
int fheon_host_encode(const fheon_params* p, const double* values, size_t n, double scale, int64_t* coeffs);
/* security disclosure of a parameter set: log2(QP) over the whole chain, the HE-standard level it
 * meets (256/192/128; 0 below 128; -1 sparse main secret, not covered by the table) and the
 * table's log2(QP) bound at min_security (homomorphicencryption.org 2018 Table 1, ternary) */
int fheon_host_security(const fheon_params* p, double* log_qp, int* level, double* bound);
/* levels bootstrapping consumes for these parameters (CtS + EvalMod + StC) */
int fheon_host_bootstrap_depth(const fheon_params* p, int* depth);
/* Chebyshev interpolant coefficients of max(0, beta z) on [-1, 1] (chebyshev.cpp:33-50) */
int fheon_cheb_relu_coefficients(double beta, int degree, double* coeffs);

/* ---- context (SlotContext::create, backend.hpp:69) */
int fheon_ctx_create(const fheon_params* p, fheon_ctx** out);
void fheon_ctx_destroy(fheon_ctx* ctx);
/* a second context over the same parameters and secret that SHARES the parent's resident
 * evaluation keys (read-only device buffers; keys made later are per-context): its own CUDA
 * stream, pools and caches, so several images are in flight on one GPU (one host thread per
 * context) without duplicating the tens of GB of keys.  Ciphertexts are bit-compatible. */
int fheon_ctx_clone(fheon_ctx* parent, fheon_ctx** out);
/* synchronise the device and return the stream-ordered pool's unused memory to the system
 * (between workloads: contexts destroyed, their buffers released) */
int fheon_release_memory(void);
/* the context's log2(QP) and HE-standard security level (as fheon_host_security) */
int fheon_ctx_security(const fheon_ctx* ctx, double* log_qp, int* level);
/* primes[L+K], scales[L] (scale target per level), slots */
int fheon_ctx_info(const fheon_ctx* ctx, uint64_t* primes, double* scales, int* slots);
void* fheon_ctx_stream(fheon_ctx* ctx); /* cudaStream_t */
int fheon_ctx_sync(fheon_ctx* ctx);
/* op counters: rotations, keyswitches, mult_plain, mult_cipher, rescales, ntt_limbs, encodes, adds,
 * kernel launches (all contexts of the process) since this context's last reset */
int fheon_ctx_stats(const fheon_ctx* ctx, uint64_t* out9);
int fheon_ctx_reset_stats(fheon_ctx* ctx);
/* live kernel timing with CUDA events on the context stream: arm a class
 * (1 key-switch inner product, 2 NTT, 3 ModUp conversion, 4 ModDown
 * conversion, 0 off), run work, read the summed milliseconds + scope count. */
int fheon_timer_arm(fheon_ctx* ctx, int kernel_class);
int fheon_timer_read(fheon_ctx* ctx, double* total_ms, int* count);

/* ---- trace (TraceRecorder, trace.hpp:37-103; SlotContext::attach_recorder)
 * events: pairs (kind, value); kind 0 rotation (index), 1 mult_plain
 * (level_after), 2 mult_cipher (level_after), 3 bootstrap (level_after). */
int fheon_set_tracing(fheon_ctx* ctx, int on);
int fheon_trace(fheon_ctx* ctx, long* events, size_t cap, size_t* n);
int fheon_trace_clear(fheon_ctx* ctx);

/* ---- keys (keyplan.hpp KeySet: rotation keys resident in HBM) */
uint64_t fheon_galois_elt(const fheon_ctx* ctx, long t); /* 5^t mod 2N */
int fheon_keygen_rotations(fheon_ctx* ctx, const long* steps, size_t n);
int fheon_keygen_relin(fheon_ctx* ctx);
int fheon_set_strict_keys(fheon_ctx* ctx, int strict); /* 1: missing key is an error */
/* key_id: 0 = relinearisation, else Galois element; out [dnum][2][L+K][N] standard form */
int fheon_key_download(fheon_ctx* ctx, uint64_t key_id, uint64_t* out);
size_t fheon_key_count(const fheon_ctx* ctx);
/* evaluation-key serialization (PAPER.md:541-566 describes serialized keys; the reference has
 * none): the packed wire format of the ciphertexts applied to the key's 2 dnum polys of L+K
 * limbs, standard form.  Upload makes the key resident under key_id (replacing one of the same
 * id); the _async variant copies on the context's upload stream and converts on the device,
 * the compute stream waits for it, the pinned host buffer must stay valid until
 * fheon_ctx_wait_transfers.  fheon_key_upload takes raw [dnum][2][L+K][N] standard-form words. */
size_t fheon_key_packed_words(const fheon_ctx* ctx);
int fheon_key_download_packed(fheon_ctx* ctx, uint64_t key_id, uint64_t* packed);
int fheon_key_upload(fheon_ctx* ctx, uint64_t key_id, const uint64_t* words);
int fheon_key_upload_packed(fheon_ctx* ctx, uint64_t key_id, const uint64_t* packed);
int fheon_key_upload_packed_async(fheon_ctx* ctx, uint64_t key_id, const uint64_t* packed);
/* ids of the keys the context needs beyond rotation keys: relinearisation (0), conjugation,
 * the bootstrapping rotations and the encapsulation keys (2, 4) -- what a client uploads to a
 * no_secret server context before the first bootstrap */
int fheon_required_key_ids(const fheon_ctx* ctx, uint64_t* ids, size_t cap, size_t* n);
/* keys received by upload (count, bytes) since the last fheon_ctx_reset_stats */
int fheon_key_uploads(const fheon_ctx* ctx, uint64_t* count, uint64_t* bytes);
/* key residency for keyplan block mode (keyplan.hpp:69-112 BlockPlan; model_run.cpp:150 key_mode):
 * resident evaluation-key bytes; generate a block's rotation keys ahead of it (stream-ordered,
 * no host sync); drop keys the next block does not use (freed after their last enqueued use,
 * regenerated bit-identically on demand); counters of generations / drops since the last
 * fheon_ctx_reset_stats */
uint64_t fheon_key_bytes(const fheon_ctx* ctx);
int fheon_prefetch_rotation_keys(fheon_ctx* ctx, const long* steps, size_t n);
int fheon_drop_rotation_keys(fheon_ctx* ctx, const long* steps, size_t n);
int fheon_key_events(const fheon_ctx* ctx, uint64_t* gens, uint64_t* drops);

/* ---- ciphertexts (SlotVector, backend.hpp:108-132) */
void fheon_ct_free(fheon_ct* ct);
int fheon_ct_level(const fheon_ct* ct);
int fheon_ct_limbs(const fheon_ct* ct);
double fheon_ct_scale(const fheon_ct* ct);
/* SlotVector::encode (backend.cpp:148-161): encode + encrypt at the depth budget */
int fheon_encrypt(fheon_ctx* ctx, const double* values, size_t n, fheon_ct** out);
/* encode + encrypt at the top of the chain (L limbs) */
int fheon_encrypt_top(fheon_ctx* ctx, const double* values, size_t n, fheon_ct** out);
/* decrypt + decode all S slots into out[n >= S] */
int fheon_decrypt(fheon_ctx* ctx, const fheon_ct* ct, double* out, size_t n);
/* decrypt + decode complex slots (real and imaginary parts, n >= S each) */
int fheon_decrypt_complex(fheon_ctx* ctx, const fheon_ct* ct, double* re, double* im, size_t n);
/* effective depth budget (levels of fresh encryptions and bootstrap outputs) */
int fheon_ctx_depth_budget(const fheon_ctx* ctx);
/* rotation schedule of the layer functions: 0 = fast (hoisted sets, log-depth
 * trees, baby-step giant-step striding; same values and levels), 1 = the
 * reference's exact rotation sequence (layers_conv.cpp / layers_misc.cpp) */
int fheon_ctx_set_schedule(fheon_ctx* ctx, int schedule);
int fheon_ctx_schedule(const fheon_ctx* ctx);
/* HBM budget (bytes) of the resident weight-plaintext cache (conv kernel vectors encoded once at
 * their consumer level): the reference's weight_mode "preload" (model.hpp:46-48); 0 = "lazy",
 * re-encode per call.  Default 64 GiB. */
int fheon_ctx_set_weight_cache(fheon_ctx* ctx, uint64_t bytes);
/* raw RNS words, layout [2][limbs][N] */
int fheon_ct_upload(fheon_ctx* ctx, const uint64_t* words, int limbs, double scale, fheon_ct** out);
int fheon_ct_download(fheon_ctx* ctx, const fheon_ct* ct, uint64_t* words);
/* non-blocking transfers on the context's copy streams (host buffers pinned and kept
 * valid until fheon_ctx_wait_transfers): uploads of the next batch, compute of this
 * one and downloads of the previous one overlap */
int fheon_ct_upload_async(fheon_ctx* ctx, const uint64_t* words, int limbs, double scale, fheon_ct** out);
int fheon_ct_download_async(fheon_ctx* ctx, const fheon_ct* ct, uint64_t* words);
int fheon_ctx_wait_transfers(fheon_ctx* ctx);
/* packed wire format (ciphertext serialization; the reference has none -- SURVEY 8(f) item 4,
 * PAPER.md:541-566 describes the paper's serialized keys/ciphertexts): layout [2][limbs][N b_i / 64]
 * uint64 words, limb i a little-endian bitstream of N canonical words of b_i = bit_length(q_i)
 * bits.  At N = 2^16 with 60 + 23 x 50-bit limbs: 0.79 of the raw [2][limbs][N] words.  The
 * (un)packing runs on the device, on the copy streams (async variants as above). */
size_t fheon_ct_packed_words(const fheon_ctx* ctx, int limbs); /* 0 on a bad limb count */
int fheon_ct_upload_packed(fheon_ctx* ctx, const uint64_t* packed, int limbs, double scale, fheon_ct** out);
int fheon_ct_download_packed(fheon_ctx* ctx, const fheon_ct* ct, uint64_t* packed);
int fheon_ct_upload_packed_async(fheon_ctx* ctx, const uint64_t* packed, int limbs, double scale, fheon_ct** out);
int fheon_ct_download_packed_async(fheon_ctx* ctx, const fheon_ct* ct, uint64_t* packed);

/* ---- backend ops (backend.hpp:134-153) */
int fheon_rotate(fheon_ctx* ctx, const fheon_ct* x, long t, fheon_ct** out);
/* hoisted rotation set sharing one ModUp of x (layers_conv.cpp:102-113 tap_rotations) */
int fheon_rotate_hoisted(fheon_ctx* ctx, const fheon_ct* x, const long* ts, size_t n, fheon_ct** outs);
/* batch: xs[i] rotated by ts[i] in one key-switch pipeline (distinct inputs batched,
 * repeated inputs hoisted); trace events in call order */
int fheon_rotate_many(fheon_ctx* ctx, const fheon_ct* const* xs, const long* ts, size_t n, fheon_ct** outs);
/* rotate-and-sum: *out = sum_i rotate(xs[i], ts[i]) with ONE ModDown (the rotated
 * c0 parts ride in the key-switch accumulator as P * c0); same level/scale terms.
 * Replaces the reference's rotate + add accumulation loops (layers_conv.cpp:155-177,
 * layers_misc.cpp:132-142); one rotation trace event per term */
int fheon_rotate_sum(fheon_ctx* ctx, const fheon_ct* const* xs, const long* ts, size_t n, fheon_ct** out);
/* several rotate-and-sum groups in one pipeline (terms flattened group by group, sizes[r] terms in
 * group r); groups that rotate one input each under the same key list run as one hoisted stage
 * (every key slice read once per launch) */
int fheon_rotate_sum_many(fheon_ctx* ctx, const fheon_ct* const* xs, const long* ts, const size_t* sizes,
                          size_t ngroups, fheon_ct** outs);
int fheon_add(fheon_ctx* ctx, const fheon_ct* a, const fheon_ct* b, fheon_ct** out);
int fheon_sub(fheon_ctx* ctx, const fheon_ct* a, const fheon_ct* b, fheon_ct** out);
int fheon_add_plain(fheon_ctx* ctx, const fheon_ct* a, const double* values, size_t n, fheon_ct** out);
int fheon_mult_plain(fheon_ctx* ctx, const fheon_ct* a, const double* values, size_t n, fheon_ct** out);
int fheon_mult_cipher(fheon_ctx* ctx, const fheon_ct* a, const fheon_ct* b, fheon_ct** out);
int fheon_bootstrap(fheon_ctx* ctx, const fheon_ct* a, fheon_ct** out);
/* bootstrap() when only slots [0, active_slots) matter (a packed tensor's active region): runs the
 * smallest sparse-slot variant (fheon_params.boot_sparse) holding them -- the input must sit above
 * level 0, its last level takes the mask -- else the full pipeline.  Same level accounting and
 * trace event as fheon_bootstrap; output slots [0, active_slots) = input, the rest 0 (sparse).
 * flags bit 0 (FHEON_BOOT_CLEAN): the caller asserts slots [active_slots, S) of the input are
 * zero (a convolution's output): no mask, so a level-0 input takes a sparse variant too */
#define FHEON_BOOT_CLEAN 1
int fheon_bootstrap_active(fheon_ctx* ctx, const fheon_ct* a, size_t active_slots, int flags, fheon_ct** out);
/* fheon_bootstrap_active on n ciphertexts in lockstep (the images of a batched inference,
 * model_run.cpp:100-159 run once per image): inputs on one level go through the sparse-slot
 * pipeline together, so each evaluation key and encoded diagonal is read from HBM once per batch
 * and every NTT / basis-conversion launch carries n times the limbs.  outs[i] is bit-identical
 * to fheon_bootstrap_active(as[i]); one bootstrap trace event per input. */
int fheon_bootstrap_active_many(fheon_ctx* ctx, const fheon_ct* const* as, size_t n, size_t active_slots, int flags,
                                fheon_ct** outs);
/* bootstrapping stage probes (tests): 1 CoeffsToSlots, 2 EvalMod, 3 SlotsToCoeffs, 4 ModRaise;
 * info (may be NULL): [depth, k_range, double_angles, stc_input_limbs] */
int fheon_bootstrap_stage(fheon_ctx* ctx, const fheon_ct* a, int stage, fheon_ct** out);
int fheon_bootstrap_info(fheon_ctx* ctx, int* info4, double* cos_coeffs, size_t cap, size_t* ncoeffs);
int fheon_rescale(fheon_ctx* ctx, const fheon_ct* a, fheon_ct** out);
int fheon_level_down(fheon_ctx* ctx, const fheon_ct* a, int limbs, fheon_ct** out);
/* key switch of a's c1 (as d) with key key_id under automorphism g (1 = none); out = (ks0, ks1) */
int fheon_keyswitch_raw(fheon_ctx* ctx, const fheon_ct* a, uint64_t key_id, uint64_t g, fheon_ct** out);

/* ---- RNS primitives on host buffers (parity checking / microbench).
 * words [npolys][nlimbs][N]; limb i uses prime i. */
int fheon_ntt_host(fheon_ctx* ctx, uint64_t* words, int npolys, int nlimbs, int inverse);
int fheon_automorph_host(fheon_ctx* ctx, uint64_t* words, int npolys, int nlimbs, uint64_t g);

/* ---- device-resident microbench (config 2): times `iters` launches of a
 * primitive with CUDA events on the context stream; returns mean ms.
 * kind: 0 NTT fwd, 1 iNTT, 2 automorphism, 3 rotation (single key switch),
 * 4 hoisted rotations (n_rot), 5 pt x ct MAC term, 6 rescale, 7 add,
 * 8 batch of `batch` (<= 64) ciphertexts rotated by the same step (one key),
 * 9 fused MAC of k = n_rot terms sum_j pt_j (*) ct_j + rescale,
 * 10 automorphism cycling through every step t in [1, S) one per launch */
int fheon_microbench(fheon_ctx* ctx, int kind, int batch, int limbs, int n_rot, int iters, double* ms);

/* ---- layers (layers.hpp:83-158).  Tensors are packed channel-major
 * (slot c*W^2 + i*W + j, packing.hpp:8-10). */
typedef struct {
  size_t in_channels, out_channels, kernel, stride, padding;
  int mode;           /* 0 generic, 1 special3x3, 2 grouped (ConvMode) */
  int stride_variant; /* 0 extract, 1 masked (StrideVariant) */
} fheon_conv_cfg;

/* convolution (layers_conv.cpp:577-594); weights (F, C or 1, k, k), bias F (may be NULL) */
int fheon_convolution(fheon_ctx* ctx, const fheon_ct* x, size_t channels, size_t width, const fheon_conv_cfg* cfg,
                      const double* weights, const double* bias, fheon_ct** out, size_t* out_channels,
                      size_t* out_width);
/* avg_pool (layers_misc.cpp:99-144): kind 0 average(k, stride, variant), 1 global, 2 whole-channel(k) */
int fheon_pool(fheon_ctx* ctx, const fheon_ct* x, size_t channels, size_t width, int kind, size_t kernel,
               size_t stride, int stride_variant, fheon_ct** out, size_t* out_channels, size_t* out_width);
/* fully_connected (layers_misc.cpp:197-255); weights (m, n) row-major, bias m (may be NULL) */
int fheon_fully_connected(fheon_ctx* ctx, const fheon_ct* x, size_t inputs, size_t outputs, size_t merge_budget,
                          const double* weights, const double* bias, fheon_ct** out);
/* secure_relu (layers_misc.cpp:268-295): Chebyshev interpolant of max(0, scale*z), degree */
int fheon_secure_relu(fheon_ctx* ctx, const fheon_ct* x, double scale, int degree, size_t active_slots,
                      fheon_ct** out);
/* secure_relu (layers_misc.cpp:268-295) on n ciphertexts in lockstep (the images of a batched
 * inference, model_run.cpp:100-159 once per image): one polynomial
 * evaluation whose relinearisations and rescales carry every input; outs[i] bit-identical to
 * fheon_secure_relu(xs[i]) */
int fheon_secure_relu_many(fheon_ctx* ctx, const fheon_ct* const* xs, size_t n, double scale, int degree,
                           size_t active_slots, fheon_ct** outs);
/* stride stage (layers_conv.cpp:285-421): variant 0 extract (v1), 1 masked (v2); w_out 0 = default */
int fheon_stride(fheon_ctx* ctx, const fheon_ct* x, size_t width, size_t stride, size_t w_out, int variant,
                 fheon_ct** out);
/* pad_input (layers_conv.cpp:238-283) */
int fheon_pad_input(fheon_ctx* ctx, const fheon_ct* x, size_t channels, size_t width, size_t padding,
                    fheon_ct** out);
/* declared depth costs (layers_conv.cpp:596-628, layers_misc.cpp:297-322) */
int fheon_conv_depth_cost(const fheon_conv_cfg* cfg, size_t w_in, int* cost);

#ifdef __cplusplus
}
#endif
#endif /* FHEON_B200_H */
