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
// Each CTA stages a tile of lines (16 columns, or a block of rows) in shared
// memory; each line (sub-NTT of M <= 256 points) is owned by M/E threads that
// hold E = 2^RB elements in registers and run RB radix-2 stages per register
// pass (one smem exchange per RB stages, __syncwarp only: a line never spans
// warps).  Shared-memory rows are padded by one word per 8 so the strided
// register passes and the transposed column loads hit distinct banks.
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

__device__ __forceinline__ int pad8(int k) { return k + (k >> 3); }

// r = a * w mod q in [0, 2q) for any a < 2^64 (Shoup, no final correction)
__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 wsh, u64 q) { return a * w - mulhi(a, wsh) * q; }

template <int LOGM, bool COL, int RB>
struct Geometry {
  static constexpr int M = 1 << LOGM;
  static constexpr int E = 1 << RB;  // elements per thread
  static constexpr int T = M / E;    // threads per line
  // columns: 16 per CTA (128-byte row segments); rows: ~256 threads per CTA
  static constexpr int ROWL = (256 / T) < 32 ? (256 / T) : 32;
  static constexpr int LPC = COL ? 16 : (ROWL < 1 ? 1 : ROWL);
  static constexpr int THREADS = LPC * T;
  static constexpr int LS = M + M / 8 + 1;  // padded line stride (words)
};

template <int LOGM, bool INV, bool COL, int RB>
__global__ void __launch_bounds__(Geometry<LOGM, COL, RB>::THREADS)
    ntt_phase_kernel(LimbSet set, LimbSet src, bool has_src, const PrimeConst* __restrict__ pc,
                     const u64* __restrict__ tw, int logN, int n1, int n2) {
  using G = Geometry<LOGM, COL, RB>;
  constexpr int M = G::M, E = G::E, T = G::T, LPC = G::LPC, LS = G::LS;
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

  // ---- load tile (16-byte vector loads: two adjacent columns / elements)
  for (int x = threadIdx.x; x < LPC * M / 2; x += blockDim.x) {
    int line, k;
    std::size_t g;
    if (COL) {
      k = x / (LPC / 2);
      line = 2 * (x - k * (LPC / 2));
      g = (std::size_t)k * N2 + line0 + line;
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(in + g);
      sm[line * LS + pad8(k)] = v.x;
      sm[(line + 1) * LS + pad8(k)] = v.y;
    } else {
      line = x / (M / 2);
      k = 2 * (x - line * (M / 2));
      g = (std::size_t)(line0 + line) * N2 + k;
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(in + g);
      sm[line * LS + pad8(k)] = v.x;
      sm[line * LS + pad8(k + 1)] = v.y;
    }
  }
  __syncthreads();

  const int li = threadIdx.x / T;
  const int t = threadIdx.x - li * T;
  u64* lsm = sm + li * LS;

  u64 x[E];
  constexpr int NG = (LOGM + RB - 1) / RB;
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    int b, nst, hb0;
    if (!INV) {
      const int top = LOGM - 1 - RB * gi;
      nst = top + 1 < RB ? top + 1 : RB;
      b = top - (RB - 1) > 0 ? top - (RB - 1) : 0;
      hb0 = top;
    } else {
      const int low = RB * gi;
      nst = LOGM - low < RB ? LOGM - low : RB;
      b = low < LOGM - RB ? low : LOGM - RB;
      hb0 = low;
    }
    const int lowmask = (1 << b) - 1;
    const int baseidx = ((t >> b) << (b + RB)) | (t & lowmask);
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = lsm[pad8(baseidx | (e << b))];
#pragma unroll
    for (int st = 0; st < RB; ++st) {
      if (st < nst) {
        const int hb = INV ? hb0 + st : hb0 - st;
        const int eb = hb - b;
        const int s = LOGM - 1 - hb;
#pragma unroll
        for (int j = 0; j < E / 2; ++j) {
          if (j < (E >> (eb + 1))) {
            // twiddle of the butterflies whose e-bits above eb equal j
            const int idx = baseidx | ((j << (eb + 1)) << b);
            const int sj = idx >> (hb + 1);
            const ulonglong2 wv =
                __ldg(twp + (COL ? (1 << s) + sj : (1 << (n1 + s)) + ((line0 + li) << s) + sj));
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
#pragma unroll
    for (int e = 0; e < E; ++e) lsm[pad8(baseidx | (e << b))] = x[e];
    __syncwarp();
  }
  __syncthreads();

  // ---- store tile
  for (int xi = threadIdx.x; xi < LPC * M / 2; xi += blockDim.x) {
    int line, k;
    std::size_t g;
    u64 v0, v1;
    if (COL) {
      k = xi / (LPC / 2);
      line = 2 * (xi - k * (LPC / 2));
      g = (std::size_t)k * N2 + line0 + line;
      v0 = sm[line * LS + pad8(k)];
      v1 = sm[(line + 1) * LS + pad8(k)];
    } else {
      line = xi / (M / 2);
      k = 2 * (xi - line * (M / 2));
      g = (std::size_t)(line0 + line) * N2 + k;
      v0 = sm[line * LS + pad8(k)];
      v1 = sm[line * LS + pad8(k + 1)];
    }
    if (!FIRST) {
      if (INV) {
        v0 = csub(shoup_lazy(v0, P.ninv, P.ninv_sh, q), q);  // [0, 2q) -> canonical
        v1 = csub(shoup_lazy(v1, P.ninv, P.ninv_sh, q), q);
      } else {
        v0 = v0 >= q2 ? v0 - q2 : v0;  // [0, 4q) -> canonical
        v1 = v1 >= q2 ? v1 - q2 : v1;
        v0 = csub(v0, q);
        v1 = csub(v1, q);
      }
    }
    *reinterpret_cast<ulonglong2*>(data + g) = make_ulonglong2(v0, v1);
  }
}

template <int LOGM, bool INV, bool COL, int RB>
void launch_phase_t(const DevTables& t, const LimbSet& set, const LimbSet* src, cudaStream_t st) {
  using G = Geometry<LOGM, COL, RB>;
  const std::size_t smem = (std::size_t)G::LPC * G::LS * sizeof(u64);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(ntt_phase_kernel<LOGM, INV, COL, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr_set = true;
  }
  const int lines = COL ? (1 << t.n2) : (1 << t.n1);
  dim3 grid(lines / G::LPC, set.count());
  ntt_phase_kernel<LOGM, INV, COL, RB><<<grid, G::THREADS, smem, st>>>(set, src ? *src : set, src != nullptr, t.pc,
                                                                       t.tw, t.logN, t.n1, t.n2);
  launch_check("ntt_phase_kernel");
}

int radix_bits() {
  static int rb = [] {
    const char* e = std::getenv("FHEON_NTT_RB");
    const int v = e ? std::atoi(e) : 3;
    return (v == 4) ? 4 : 3;
  }();
  return rb;
}

template <int LOGM, bool INV, bool COL>
void launch_phase(const DevTables& t, const LimbSet& set, const LimbSet* src, cudaStream_t st) {
  if (radix_bits() == 4 && LOGM >= 6) launch_phase_t<LOGM, INV, COL, 4>(t, set, src, st);
  else launch_phase_t<LOGM, INV, COL, 3>(t, set, src, st);
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

void ntt_inverse(const DevTables& t, const LimbSet& set, cudaStream_t st, const LimbSet* src) {
  if (set.count() == 0) return;
  TimedScope ts(t, kNtt, st);
  dispatch<true, false>(t, set, src, st);
  dispatch<true, true>(t, set, nullptr, st);
}

}  // namespace fheon
