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
// Each CTA stages a tile of lines (16 columns, or 2048/M rows) in shared
// memory; each line (sub-NTT of M <= 256 points) is owned by M/8 threads that
// hold 8 elements in registers and run 3 radix-2 stages per register pass
// (one smem exchange per 3 stages, __syncwarp only: a line never spans warps).
// Shared memory rows are padded by one word per 8 so the strided register
// passes and the transposed column loads hit distinct banks.
//
// Arithmetic: Harvey lazy butterflies.  Forward values live in [0, 4q)
// (CT: X <- X mod 2q; T = Shoup(Y, W) in [0, 2q); X+T, X-T+2q), inverse
// values in [0, 2q) (GS).  The intermediate between the two phases stays
// lazy; the second phase reduces to canonical on store.  Twiddles are read as
// 16-byte (value, Shoup) pairs, once per register pass (1 + 2 + 4 per thread).
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

template <int LOGM, bool INV, bool COL, bool TWS>
__global__ void __launch_bounds__(512) ntt_phase_kernel(LimbSet set, LimbSet src, bool has_src,
                                                        const PrimeConst* __restrict__ pc,
                                                        const u64* __restrict__ tw, int logN, int n1, int n2) {
  constexpr int M = 1 << LOGM;
  constexpr int T = M / 8;                                   // threads per line
  constexpr int LPC = COL ? 16 : (M >= 64 ? 2048 / M : 32);  // lines per CTA
  constexpr int LS = M + M / 8 + 1;                          // padded line stride (words)
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

  // ---- stage this CTA's twiddles in smem (after the data tile).  Stage s of
  // this phase (s = LOGM-1-hb) uses global index (1<<s) + j (COL, shared by
  // every column) or (1<<(n1+s)) + (row<<s) + j (ROW; forward and inverse
  // tables have the same shape), so each stage's range is contiguous.
  ulonglong2* sw = reinterpret_cast<ulonglong2*>(sm + LPC * LS + (LPC * LS) % 2);
  if (!TWS) {
  } else if (COL) {
    for (int k = threadIdx.x; k < M; k += blockDim.x) sw[k] = __ldg(twp + k);
  } else {
#pragma unroll
    for (int s = 0; s < LOGM; ++s) {
      const int cnt = LPC << s;
      const int gbase = (1 << (n1 + s)) + (line0 << s);
      for (int k = threadIdx.x; k < cnt; k += blockDim.x) sw[LPC * ((1 << s) - 1) + k] = __ldg(twp + gbase + k);
    }
  }

  // ---- load tile
  for (int x = threadIdx.x; x < LPC * M; x += blockDim.x) {
    int line, k;
    std::size_t g;
    if (COL) {
      k = x / LPC;
      line = x - k * LPC;
      g = (std::size_t)k * N2 + line0 + line;
    } else {
      line = x / M;
      k = x - line * M;
      g = (std::size_t)(line0 + line) * N2 + k;
    }
    sm[line * LS + pad8(k)] = in[g];
  }
  __syncthreads();

  const int li = threadIdx.x / T;
  const int t = threadIdx.x - li * T;
  u64* lsm = sm + li * LS;

  u64 x[8];
  constexpr int NG = (LOGM + 2) / 3;
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    int b, nst, hb0;
    if (!INV) {
      const int top = LOGM - 1 - 3 * gi;
      nst = top + 1 < 3 ? top + 1 : 3;
      b = top - 2 > 0 ? top - 2 : 0;
      hb0 = top;
    } else {
      const int low = 3 * gi;
      nst = LOGM - low < 3 ? LOGM - low : 3;
      b = low < LOGM - 3 ? low : LOGM - 3;
      hb0 = low;
    }
    const int lowmask = (1 << b) - 1;
    const int baseidx = ((t >> b) << (b + 3)) | (t & lowmask);
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = lsm[pad8(baseidx | (e << b))];
#pragma unroll
    for (int st = 0; st < 3; ++st) {
      if (st < nst) {
        const int hb = INV ? hb0 + st : hb0 - st;
        const int eb = hb - b;
        // distinct twiddles of this stage: indexed by the e-bits above eb
        constexpr int MAXW = 4;
        ulonglong2 w[MAXW];
        const int nw = 8 >> (eb + 1);
#pragma unroll
        for (int j = 0; j < MAXW; ++j) {
          if (j < nw) {
            const int idx = baseidx | ((j << (eb + 1)) << b);
            const int s = LOGM - 1 - hb;
            const int sj = idx >> (hb + 1);
            if (TWS) {
              w[j] = COL ? sw[(1 << s) + sj] : sw[LPC * ((1 << s) - 1) + (li << s) + sj];
            } else {
              w[j] = __ldg(twp + (COL ? (1 << s) + sj : (1 << (n1 + s)) + ((line0 + li) << s) + sj));
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (((e >> eb) & 1) == 0) {
            const int e2 = e | (1 << eb);
            const ulonglong2 wv = w[e >> (eb + 1)];
            if (!INV) {
              u64 X = x[e];
              X = X >= q2 ? X - q2 : X;
              const u64 Tv = shoup_lazy(x[e2], wv.x, wv.y, q);
              x[e] = X + Tv;
              x[e2] = X - Tv + q2;
            } else {
              const u64 X = x[e], Y = x[e2];
              const u64 s = X + Y;
              x[e] = s >= q2 ? s - q2 : s;
              x[e2] = shoup_lazy(X - Y + q2, wv.x, wv.y, q);
            }
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) lsm[pad8(baseidx | (e << b))] = x[e];
    __syncwarp();
  }
  __syncthreads();

  // ---- store tile
  for (int xi = threadIdx.x; xi < LPC * M; xi += blockDim.x) {
    int line, k;
    std::size_t g;
    if (COL) {
      k = xi / LPC;
      line = xi - k * LPC;
      g = (std::size_t)k * N2 + line0 + line;
    } else {
      line = xi / M;
      k = xi - line * M;
      g = (std::size_t)(line0 + line) * N2 + k;
    }
    u64 v = sm[line * LS + pad8(k)];
    if (!FIRST) {
      if (INV) {
        v = csub(shoup_lazy(v, P.ninv, P.ninv_sh, q), q);  // [0, 2q) -> canonical
      } else {
        v = v >= q2 ? v - q2 : v;  // [0, 4q) -> canonical
        v = csub(v, q);
      }
    }
    data[g] = v;
  }
}

template <int LOGM, bool INV, bool COL, bool TWS>
void launch_phase_t(const DevTables& t, const LimbSet& set, const LimbSet* src, cudaStream_t st) {
  constexpr int M = 1 << LOGM;
  constexpr int LPC = COL ? 16 : (M >= 64 ? 2048 / M : 32);
  constexpr int threads = LPC * (M / 8);
  constexpr int LS = M + M / 8 + 1;
  constexpr int TWN = !TWS ? 0 : COL ? M : LPC * (M - 1);  // staged twiddles (16 B each)
  const std::size_t smem = ((std::size_t)LPC * LS + (LPC * LS) % 2) * sizeof(u64) + (std::size_t)TWN * 16;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(ntt_phase_kernel<LOGM, INV, COL, TWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  const int lines = COL ? (1 << t.n2) : (1 << t.n1);
  dim3 grid(lines / LPC, set.count());
  ntt_phase_kernel<LOGM, INV, COL, TWS><<<grid, threads, smem, st>>>(set, src ? *src : set, src != nullptr, t.pc, t.tw,
                                                                 t.logN, t.n1, t.n2);
  launch_check("ntt_phase_kernel");
}

int twiddle_mode() {
  static int mode = [] {
    const char* e = std::getenv("FHEON_NTT_TWSMEM");
    return e ? std::atoi(e) : 0;
  }();
  return mode;
}

template <int LOGM, bool INV, bool COL>
void launch_phase(const DevTables& t, const LimbSet& set, const LimbSet* src, cudaStream_t st) {
  if (twiddle_mode()) launch_phase_t<LOGM, INV, COL, true>(t, set, src, st);
  else launch_phase_t<LOGM, INV, COL, false>(t, set, src, st);
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
