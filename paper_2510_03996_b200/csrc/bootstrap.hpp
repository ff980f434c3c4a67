// Full-slot CKKS bootstrapping: the realisation of the reference's
// bootstrap() (proj/src/backend.cpp:233-249: identity on the slots, level :=
// depth budget).  Pipeline (Cheon-Han-Kim-Kim-Song 2018; BSGS linear
// transforms and double-angle EvalMod as in Han-Ki 2020 / Bossuat et al. 2021):
//
//   ModRaise   level-0 ct -> all L limbs; decrypts to m + q0 I (|I| <= K)
//   CoeffsToSlots  B U^{-1}: the special-FFT stages of the encoder, grouped
//              into `cts_levels` sparse matrices (2^{r+1}-1 diagonals each),
//              each evaluated as a baby-step/giant-step sum with hoisted baby
//              rotations and one fused MAC per giant step; the bit reversal B
//              is never applied (EvalMod is slot-wise, SlotsToCoeffs consumes
//              the bit-reversed order)
//   split      re = y + conj(y), im = -i (y - conj(y))  (1/2 folded into CtS)
//   EvalMod    sin(2 pi t) = cos(2 pi (t - 1/4)): Chebyshev interpolant of
//              cos(2 pi ((K+1) u - 1/4) / 2^r) on u in [-1, 1] (u = t/(K+1),
//              folded into CtS), then r double-angle steps y <- 2 y^2 - 1
//   SlotsToCoeffs  U (stages F_2 .. F_S), with q0 / (2 pi Delta_0) folded in
//
// The output lands on the context's depth budget with the input's slot values.
//
// Sparse-slot variant (BootParams::log_slots = log2 n, n < S): for inputs whose
// slots [n, S) carry nothing the caller needs (a packed tensor's inactive
// region).  The input is masked to [0, n) on its last level and replicated
// n-periodically (one hoisted rotate-and-sum at one limb), so its plaintext
// lies in the subring Z[X^{S/n}]; after ModRaise the same rotate-and-sum over
// the raised ciphertext (the trace to the subring, divided by g = S/n inside
// CtS) projects q0 I there as well.  CtS and StC then run the n-point special
// FFT (stages n..2 / 2..n: fewer diagonals), the real and imaginary halves of
// the 2n coefficients are packed into ONE real ciphertext (D = [1 | -i] folded
// into CtS's last factor, one conjugation), so EvalMod runs once instead of
// twice, and StC's first factor unpacks them (P = [1 | i] + [i | 1] rot_n) while
// its last factor masks the output to [0, n).  Same levels as the full
// pipeline; output slots [0, n) = input, [n, S) = 0.
#pragma once

#include <complex>
#include <map>
#include <vector>

#include "engine.hpp"

namespace fheon {

struct BootParams {
  int k_range = 16;       // EvalMod input range |t| <= k_range + 1/2
  int double_angles = 3;  // r
  int cts_levels = 3;
  int stc_levels = 3;
  int cos_degree = 0;     // 0: chosen automatically
  // linear transforms double-hoisted (babies kept over Q u P, one ModDown per
  // giant); env FHEON_BOOT_DH=0 selects the single-hoisted schedule for A/B runs
  bool double_hoist = true;
  int log_slots = 0;      // sparse-slot variant over n = 2^log_slots < S slots (0: full)
};

BootParams boot_params_of(const Params& p);

class Bootstrapper {
 public:
  Bootstrapper(Context& ctx, const BootParams& bp = {});
  // a key-sharing clone's bootstrapper: the parent's plan and encoded diagonals
  // (read-only device buffers) shared, operations issued on `ctx`
  Bootstrapper(Context& ctx, const Bootstrapper& parent);
  // levels consumed between ModRaise (top) and the output
  int depth() const { return depth_; }
  // full: any level; sparse: x must hold >= 2 limbs (the mask takes one level) unless
  // `clean` (slots [n, S) of x are already zero: no mask, any level)
  Ciphertext run(const Ciphertext& x, bool clean = false);
  // several ciphertexts of one level in lockstep (sparse variants: every stage batched, keys
  // and diagonals read once per batch; full variant: one after the other); bit-identical to run
  std::vector<Ciphertext> run_many(const std::vector<Ciphertext>& xs, bool clean = false);
  long slots() const { return n_; }
  bool sparse() const { return n_ < S_; }
  // stage probes for tests: 1 CoeffsToSlots on x (scale reinterpreted as q0),
  // 2 EvalMod of x (slots u -> sin(2 pi (K+1) u)), 3 SlotsToCoeffs on x,
  // 4 ModRaise of x
  Ciphertext debug_stage(const Ciphertext& x, int what);
  const std::vector<double>& cos_coeffs() const { return cos_coeffs_; }
  int stc_input_limbs() const { return stc_limbs_; }
  // rotation steps whose keys the pipeline uses (plus conjugation)
  std::vector<long> rotation_steps() const;

 private:
  struct Giant {
    long rot = 0;                            // giant-step rotation (slots)
    std::vector<std::pair<long, BufPtr>> terms;  // (baby rotation, plaintext)
  };
  struct Level {
    std::vector<long> babies;  // nonzero baby rotations
    std::vector<Giant> giants;
    bool qp = false;           // plaintexts over Q u P (double-hoisted)
  };
  using Diag = std::vector<std::complex<double>>;
  using Mat = std::map<long, Diag>;

  Mat stage(int len, bool inverse) const;
  Mat mul(const Mat& A, const Mat& B) const;
  // offsets taken mod `period` (the input is period-periodic): coinciding diagonals merge
  Mat reduce_period(const Mat& M, long period) const;
  // periods[i]: group i's input is periods[i]-periodic (S: no structure)
  std::vector<Level> plan(const std::vector<Mat>& groups, int limbs_in, double scale_in,
                          const std::vector<long>& periods);
  // with_conj: returns T x + conj(T x) (the conjugated giant steps join the same ModDown)
  Ciphertext apply(const Ciphertext& x, const Level& lv, bool with_conj = false);
  std::vector<Ciphertext> apply_many(const std::vector<Ciphertext>& xs, const Level& lv, bool with_conj = false);
  // sum_{j < S/n} rot(x, j n): one hoisted rotate-and-sum (all inputs in one pipeline)
  std::vector<Ciphertext> subsum_many(const std::vector<Ciphertext>& xs);
  Ciphertext run_full(const Ciphertext& x);

  Context& ctx_;
  BootParams bp_;
  int S_ = 0;
  long n_ = 0;  // slots the pipeline carries (S_ for the full variant)
  std::vector<long> sub_steps_;  // sparse: the trace rotations j n, 0 < j < S / n
  int depth_ = 0;
  int stc_limbs_ = 0;
  std::vector<Level> cts_, stc_;
  std::vector<double> cos_coeffs_;
};

}  // namespace fheon
