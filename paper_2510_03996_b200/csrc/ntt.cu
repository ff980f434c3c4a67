// Batched negacyclic NTT / inverse NTT over every limb-polynomial of a
// LimbSet, for N = 2^10 .. 2^16 and 64-bit words (primes < 2^60).
//
// Definition (oracle/ckks_oracle.c ock_ntt_fwd): forward
// Cooley-Tukey with psi^{brv(i)} twiddles, natural order in, bit-reversed out;
// inverse Gentleman-Sande, bit-reversed in, natural out, times N^{-1}.
// Outputs are canonical in [0, q).
//
// Decomposition N = N1 x N2 (N1 = 2^n1 columns of length N1, rows of N2):
//   forward: phase COL runs the first n1 stages on each of the N2 columns
//            (stride-N2 elements), phase ROW runs the last n2 stages on each
//            contiguous row of N2 elements;
//   inverse: ROW (first n2 GS stages) then COL (last n1 stages, scale N^{-1}).
// Each thread owns E = 8 elements of one line (sub-NTT of M <= 256 points,
// M/8 threads per line) and runs up to 3 radix-2 stages per register pass.
// The first pass's layout (elements tp + e*M/8 for forward, 8 tp + e for
// inverse) and the last pass's are read / written straight from / to global
// memory, coalesced: in COL tiles the lanes of a warp span 16 adjacent
// columns, in ROW tiles a line's threads are consecutive.  Only the
// re-layouts between passes go through shared memory (line-major, one pad
// word per 8 so both tile shapes are bank-conflict free); a line never spans
// warps in ROW tiles (__syncwarp), it does in COL tiles (__syncthreads).
//
// Arithmetic: Harvey lazy butterflies.  Forward values live in [0, 4q)
// (CT: X <- X mod 2q; T = Shoup(Y, W) in [0, 2q); X+T, X-T+2q), inverse
// values in [0, 2q) (GS).  The intermediate between the two phases stays
// lazy; the second phase reduces to canonical on store.  Twiddles are read as
// 16-byte (value, Shoup) pairs, once per stage per thread.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace fheon {

namespace {

#ifndef FHEON_NTT_COL_LINES
#define FHEON_NTT_COL_LINES 16
#endif
#ifndef FHEON_NTT_ROW_THREADS
#define FHEON_NTT_ROW_THREADS 256
#endif
#ifndef FHEON_NTT_RB
#define FHEON_NTT_RB 3  // radix-2 stages per register pass (E = 2^RB elements per thread)
#endif
#ifndef FHEON_NTT_SMALL_CTAS
#define FHEON_NTT_SMALL_CTAS 600
#endif

__device__ __forceinline__ int pad8(int k) { return k + (k >> 3); }

// r = a * w mod q in [0, 2q) for any a < 2^64 (Shoup, no final correction)
__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 wsh, u64 q) { return a * w - mulhi(a, wsh) * q; }

// SMALL: a quarter of the lines per CTA (4x the CTAs) for batches too small
// to fill the GPU with the default tiles
template <int LOGM, bool COL, bool SMALL>
struct Geometry {
  static constexpr int M = 1 << LOGM;
  static constexpr int E = 1 << FHEON_NTT_RB;  // elements per thread
  static constexpr int T = M / E;    // threads per line
  static constexpr int ROW_THREADS = SMALL ? FHEON_NTT_ROW_THREADS / 4 : FHEON_NTT_ROW_THREADS;
  static constexpr int ROWL = (ROW_THREADS / T) < 1 ? 1 : ((ROW_THREADS / T) < 32 ? (ROW_THREADS / T) : 32);
  static constexpr int LPC = COL ? (SMALL ? FHEON_NTT_COL_LINES / 4 : FHEON_NTT_COL_LINES) : ROWL;  // lines per CTA
  static constexpr int THREADS = LPC * T;
  static constexpr int LS = M + M / 8 + 1;  // padded line stride (words)
  static constexpr int NG = (LOGM + FHEON_NTT_RB - 1) / FHEON_NTT_RB;  // register passes
};

// element positions of pass gi: idx(e) = base | (e << b)
template <int LOGM, bool INV>
__device__ __forceinline__ void pass_shape(int gi, int tp, int& b, int& nst, int& hb0, int& base) {
  if (!INV) {
    constexpr int RB = FHEON_NTT_RB;
    const int top = LOGM - 1 - RB * gi;
    nst = top + 1 < RB ? top + 1 : RB;
    b = top - (RB - 1) > 0 ? top - (RB - 1) : 0;
    hb0 = top;
  } else {
    constexpr int RB = FHEON_NTT_RB;
    const int low = RB * gi;
    nst = LOGM - low < RB ? LOGM - low : RB;
    b = low < LOGM - RB ? low : LOGM - RB;
    hb0 = low;
  }
  base = ((tp >> b) << (b + FHEON_NTT_RB)) | (tp & ((1 << b) - 1));
}

// All register passes of one phase on E elements per thread: x holds pass 0's
// layout on entry and the last pass's on exit (b, base describe it); re-layouts
// go through the thread's line in shared memory (`lsm`).  SYNC: 1 = the line's
// threads are one warp (__syncwarp), 2 = they span warps (__syncthreads).
// row = -1 for column lines (twiddles independent of the line), else the row.
template <int LOGM, bool INV, int SYNC>
__device__ __forceinline__ void run_passes(u64 (&x)[1 << FHEON_NTT_RB], int tp, int row, u64* lsm,
                                           const ulonglong2* __restrict__ twp, u64 q, int n1, int& b, int& nst,
                                           int& hb0, int& base) {
  constexpr int E = 1 << FHEON_NTT_RB;
  constexpr int NG = (LOGM + FHEON_NTT_RB - 1) / FHEON_NTT_RB;
  const u64 q2 = 2 * q;
  pass_shape<LOGM, INV>(0, tp, b, nst, hb0, base);
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    if (gi > 0) {  // re-layout through shared memory
      int pb, pn, ph, pbase;
      pass_shape<LOGM, INV>(gi - 1, tp, pb, pn, ph, pbase);
#pragma unroll
      for (int e = 0; e < E; ++e) lsm[pad8(pbase | (e << pb))] = x[e];
      if (SYNC == 2) __syncthreads();
      else __syncwarp();
      pass_shape<LOGM, INV>(gi, tp, b, nst, hb0, base);
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = lsm[pad8(base | (e << b))];
    }
#pragma unroll
    for (int st = 0; st < FHEON_NTT_RB; ++st) {
      if (st < nst) {
        const int hb = INV ? hb0 + st : hb0 - st;
        const int eb = hb - b;
        const int s = LOGM - 1 - hb;
#pragma unroll
        for (int j = 0; j < E / 2; ++j) {
          if (j < (E >> (eb + 1))) {
            // twiddle of the butterflies whose e-bits above eb equal j
            const int idx = base | ((j << (eb + 1)) << b);
            const int sj = idx >> (hb + 1);
            const ulonglong2 wv = __ldg(twp + (row < 0 ? (1 << s) + sj : (1 << (n1 + s)) + (row << s) + sj));
#pragma unroll
            for (int lo = 0; lo < (1 << eb); ++lo) {
              const int e = (j << (eb + 1)) | lo;
              const int e2 = e | (1 << eb);
              if (!INV) {
                u64 X = x[e];
                X = X >= q2 ? X - q2 : X;
                const u64 Tv = shoup_lazy(x[e2], wv.x, wv.y, q);
                x[e] = X + Tv;
                x[e2] = X - Tv + q2;
              } else {
                const u64 X = x[e], Y = x[e2];
                const u64 sm2 = X + Y;
                x[e] = sm2 >= q2 ? sm2 - q2 : sm2;
                x[e2] = shoup_lazy(X - Y + q2, wv.x, wv.y, q);
              }
            }
          }
        }
      }
    }
  }
}

struct NoEpilogue {};
template <bool EPI>
struct EpiArg {
  using type = NoEpilogue;
};
template <>
struct EpiArg<true> {
  using type = NttEpilogue;
};

#ifndef FHEON_NTT_OCC
#define FHEON_NTT_OCC 1024  // resident threads per SM the register budget is sized for
#endif
template <int LOGM, bool INV, bool COL, bool SMALL, bool EPI = false>
__global__ void __launch_bounds__(Geometry<LOGM, COL, SMALL>::THREADS,
                                  FHEON_NTT_OCC / Geometry<LOGM, COL, SMALL>::THREADS)
    ntt_phase_kernel(LimbSet set, LimbSet src, bool has_src, const PrimeConst* __restrict__ pc,
                     const u64* __restrict__ tw, int logN, int n1, int n2, typename EpiArg<EPI>::type epi) {
  using G = Geometry<LOGM, COL, SMALL>;
  constexpr int E = G::E, T = G::T, LPC = G::LPC, LS = G::LS, NG = G::NG;
  // the phase that runs first (forward COL / inverse ROW) reads canonical input and
  // leaves lazy values; the second phase reduces to canonical.
  constexpr bool FIRST = (COL != INV);
  extern __shared__ u64 sm[];

  u64* data;
  int prime;
  if (!limbset_get(set, blockIdx.y, (std::size_t)1 << logN, data, prime)) return;
  const u64* in = data;  // out-of-place first phase: read the source set
  if (has_src) {
    u64* sp;
    int sprime;
    limbset_get(src, blockIdx.y, (std::size_t)1 << logN, sp, sprime);
    in = sp;
  }
  const std::size_t N = (std::size_t)1 << logN;
  const PrimeConst P = pc[prime];
  const u64 q = P.q;
  const u64 q2 = 2 * q;
  const ulonglong2* twp = reinterpret_cast<const ulonglong2*>(tw + (std::size_t)prime * 4 * N + (INV ? 2 * N : 0));
  const int N2 = 1 << n2;
  const int line0 = blockIdx.x * LPC;
  // COL: lanes span the tile's 16 columns; ROW: a line's T threads are consecutive
  const int li = COL ? (int)(threadIdx.x % LPC) : (int)(threadIdx.x / T);
  const int tp = COL ? (int)(threadIdx.x / LPC) : (int)(threadIdx.x % T);
  u64* lsm = sm + li * LS;
  auto gaddr = [&](int k) -> std::size_t {
    const std::size_t a = COL ? (std::size_t)k * N2 + line0 + li : (std::size_t)(line0 + li) * N2 + k;
    FHEON_DCHECK(a < N && k < G::M && li < LPC);
    return a;
  };

  u64 x[E];
  int b, nst, hb0, base;
  pass_shape<LOGM, INV>(0, tp, b, nst, hb0, base);
  if (!COL && b == 0) {  // 8 consecutive words per thread: 16-byte loads
    const ulonglong2* srcv = reinterpret_cast<const ulonglong2*>(in + gaddr(base));
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      const ulonglong2 v = srcv[e / 2];
      x[e] = v.x;
      x[e + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = in[gaddr(base | (e << b))];
  }

  run_passes<LOGM, INV, COL ? 2 : 1>(x, tp, COL ? -1 : line0 + li, lsm, twp, q, n1, b, nst, hb0, base);

  // ---- store the last pass's layout straight to global memory
#pragma unroll
  for (int e = 0; e < E; ++e) {
    u64 v = x[e];
    if (!FIRST) {
      if (INV) {
        v = csub(shoup_lazy(v, P.ninv, P.ninv_sh, q), q);  // [0, 2q) -> canonical
      } else {
        v = v >= q2 ? v - q2 : v;  // [0, 4q) -> canonical
        v = csub(v, q);
      }
    }
    x[e] = v;
  }
  if constexpr (EPI) {  // forward ROW phase: fused ModDown / rescale finish
    const int per_base = set.blocks_per_base * set.E;
    const int bb = blockIdx.y / per_base;
    const int rr = blockIdx.y - bb * per_base;
    const int blk = rr / set.E;
    const int tl = rr - blk * set.E;  // Q limb
    const int pi = bb * set.blocks_per_base + blk;
    const std::size_t off = (std::size_t)tl << logN;
    const u64* srcp = epi.src[pi] + off;
    const u64* addp = epi.add[pi] ? epi.add[pi] + off : nullptr;
    const u64 g = epi.add_g[pi];
    const u64 c = __ldg(epi.cst + (std::size_t)tl * epi.cst_stride);
    const u64 csh = __ldg(epi.cst + (std::size_t)tl * epi.cst_stride + 1);
    const bool amul = epi.acst != nullptr;
    const u64 ac = amul ? __ldg(epi.acst + (std::size_t)tl * epi.acst_stride) : 0;
    const u64 acsh = amul ? __ldg(epi.acst + (std::size_t)tl * epi.acst_stride + 1) : 0;
    u64* outp = epi.out[pi] + off;
    if (!COL && b == 0) {  // the thread's E elements are consecutive: 16-byte accesses
      const int k0 = (int)gaddr(base);
#pragma unroll
      for (int e = 0; e < E; e += 2) {
        const ulonglong2 sv = *reinterpret_cast<const ulonglong2*>(srcp + k0 + e);
        u64 v0 = shoup_mul(sub_mod(sv.x, x[e], q), c, csh, q);
        u64 v1 = shoup_mul(sub_mod(sv.y, x[e + 1], q), c, csh, q);
        if (addp) {
          u64 a0, a1;
          if (g == 1) {
            const ulonglong2 av = *reinterpret_cast<const ulonglong2*>(addp + k0 + e);
            a0 = av.x;
            a1 = av.y;
          } else {
            a0 = addp[auto_src((unsigned)(k0 + e), g, logN)];
            a1 = addp[auto_src((unsigned)(k0 + e + 1), g, logN)];
          }
          if (amul) {
            a0 = shoup_mul(a0, ac, acsh, q);
            a1 = shoup_mul(a1, ac, acsh, q);
          }
          v0 = add_mod(v0, a0, q);
          v1 = add_mod(v1, a1, q);
        }
        *reinterpret_cast<ulonglong2*>(outp + k0 + e) = make_ulonglong2(v0, v1);
      }
      return;
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = (int)gaddr(base | (e << b));  // element index within the limb-poly
      u64 v = shoup_mul(sub_mod(srcp[k], x[e], q), c, csh, q);
      if (addp) {
        u64 av = addp[(g == 1) ? (unsigned)k : auto_src((unsigned)k, g, logN)];
        if (amul) av = shoup_mul(av, ac, acsh, q);
        v = add_mod(v, av, q);
      }
      outp[k] = v;
    }
    return;
  }
  if (!COL && b == 0) {  // 8 consecutive words per thread: 16-byte stores
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(data + gaddr(base));
#pragma unroll
    for (int e = 0; e < E; e += 2) dst[e / 2] = make_ulonglong2(x[e], x[e + 1]);
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) data[gaddr(base | (e << b))] = x[e];
  }
}

template <int LOGM, bool INV, bool COL, bool SMALL, bool EPI = false>
void launch_phase_g(const DevTables& t, const LimbSet& set, const LimbSet* src, cudaStream_t st,
                    const typename EpiArg<EPI>::type& epi = {}) {
  using G = Geometry<LOGM, COL, SMALL>;
  const std::size_t smem = (std::size_t)G::LPC * G::LS * sizeof(u64);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(ntt_phase_kernel<LOGM, INV, COL, SMALL, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr_set = true;
  }
  const int lines = COL ? (1 << t.n2) : (1 << t.n1);
  dim3 grid(lines / G::LPC, set.count());
  ntt_phase_kernel<LOGM, INV, COL, SMALL, EPI><<<grid, G::THREADS, smem, st>>>(
      set, src ? *src : set, src != nullptr, t.pc, t.tw, t.logN, t.n1, t.n2, epi);
  launch_check("ntt_phase_kernel");
}

// Tile size: the small tiles (4 columns / 2 rows of 256 per CTA) measured faster at every
// batch size (0.88 vs 0.91 us per 2^16 limb-poly at 768, 1.46 vs 1.54 at 16); the large
// ones stay selectable for A/B runs: FHEON_NTT_SMALL = 0 large, 1 small (default),
// 2 small below FHEON_NTT_SMALL_CTAS large-tile CTAs
int small_mode() {
  static int m = [] {
    const char* e = std::getenv("FHEON_NTT_SMALL");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}

template <int LOGM, bool INV, bool COL>
void launch_phase(const DevTables& t, const LimbSet& set, const LimbSet* src, cudaStream_t st) {
  using G = Geometry<LOGM, COL, false>;
  const int lines = COL ? (1 << t.n2) : (1 << t.n1);
  const long ctas = (long)(lines / G::LPC) * set.count();
  const int mode = small_mode();
  const bool small = mode == 1 || (mode == 2 && ctas < FHEON_NTT_SMALL_CTAS);
  if (small) launch_phase_g<LOGM, INV, COL, true>(t, set, src, st);
  else launch_phase_g<LOGM, INV, COL, false>(t, set, src, st);
}

template <bool INV, bool COL>
void dispatch(const DevTables& t, const LimbSet& set, const LimbSet* src, cudaStream_t st) {
  const int logm = COL ? t.n1 : t.n2;
  switch (logm) {
    case 5: launch_phase<5, INV, COL>(t, set, src, st); break;
    case 6: launch_phase<6, INV, COL>(t, set, src, st); break;
    case 7: launch_phase<7, INV, COL>(t, set, src, st); break;
    case 8: launch_phase<8, INV, COL>(t, set, src, st); break;
    default: throw std::runtime_error("unsupported NTT split " + std::to_string(logm));
  }
}

}  // namespace

void ntt_forward(const DevTables& t, const LimbSet& set, cudaStream_t st, const LimbSet* src) {
  if (set.count() == 0) return;
  TimedScope ts(t, kNtt, st);
  dispatch<false, true>(t, set, src, st);
  dispatch<false, false>(t, set, nullptr, st);
}

void ntt_forward_epilogue(const DevTables& t, const LimbSet& set, const NttEpilogue& epi, cudaStream_t st) {
  if (set.count() == 0) return;
  TimedScope ts(t, kNtt, st);
  dispatch<false, true>(t, set, nullptr, st);
  switch (t.n2) {  // ROW phase with the fused store (small tiles)
    case 5: launch_phase_g<5, false, false, true, true>(t, set, nullptr, st, epi); break;
    case 6: launch_phase_g<6, false, false, true, true>(t, set, nullptr, st, epi); break;
    case 7: launch_phase_g<7, false, false, true, true>(t, set, nullptr, st, epi); break;
    case 8: launch_phase_g<8, false, false, true, true>(t, set, nullptr, st, epi); break;
    default: throw std::runtime_error("unsupported NTT split " + std::to_string(t.n2));
  }
}

void ntt_inverse(const DevTables& t, const LimbSet& set, cudaStream_t st, const LimbSet* src) {
  if (set.count() == 0) return;
  TimedScope ts(t, kNtt, st);
  dispatch<true, false>(t, set, src, st);
  dispatch<true, true>(t, set, nullptr, st);
}

}  // namespace fheon
