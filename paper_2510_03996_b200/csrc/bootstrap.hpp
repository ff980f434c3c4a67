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
};

BootParams boot_params_of(const Params& p);

class Bootstrapper {
 public:
  Bootstrapper(Context& ctx, const BootParams& bp = {});
  // levels consumed between ModRaise (top) and the output
  int depth() const { return depth_; }
  Ciphertext run(const Ciphertext& x);
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
  std::vector<Level> plan(const std::vector<Mat>& groups, int limbs_in, double scale_in);
  Ciphertext apply(const Ciphertext& x, const Level& lv);

  Context& ctx_;
  BootParams bp_;
  int S_ = 0;
  int depth_ = 0;
  int stc_limbs_ = 0;
  std::vector<Level> cts_, stc_;
  std::vector<double> cos_coeffs_;
};

}  // namespace fheon
