// Batched negacyclic NTT / inverse NTT over every limb-polynomial of a
// LimbSet, for N = 2^10 .. 2^16 and 64-bit words (primes < 2^60).
//
// Definition (oracle/ckks_oracle.c ock_ntt_fwd): forward
// Cooley-Tukey with psi^{brv(i)} twiddles, natural order in, bit-reversed out;
// inverse Gentleman-Sande, bit-reversed in, natural out, times N^{-1}.
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
#include <cstdio>
#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace fheon {

namespace {

__device__ __forceinline__ int pad8(int k) { return k + (k >> 3); }

template <int LOGM, bool INV, bool COL>
__global__ void __launch_bounds__(512) ntt_phase_kernel(LimbSet set, const PrimeConst* __restrict__ pc,
                                                        const u64* __restrict__ tw, int logN, int n1, int n2) {
  constexpr int M = 1 << LOGM;
  constexpr int T = M / 8;                    // threads per line
  constexpr int LPC = COL ? 16 : (M >= 64 ? 2048 / M : 32);  // lines per CTA
  constexpr int LS = M + M / 8 + 1;           // padded line stride (words)
  extern __shared__ u64 sm[];

  u64* data;
  int prime;
  if (!limbset_get(set, blockIdx.y, (std::size_t)1 << logN, data, prime)) return;
  const std::size_t N = (std::size_t)1 << logN;
  const PrimeConst P = pc[prime];
  const u64 q = P.q;
  const u64* twv = tw + (std::size_t)prime * 4 * N + (INV ? 2 * N : 0);
  const u64* tws = twv + N;
  const int N2 = 1 << n2;
  const int line0 = blockIdx.x * LPC;

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
    sm[line * LS + pad8(k)] = data[g];
  }
  __syncthreads();

  const int li = threadIdx.x / T;
  const int t = threadIdx.x - li * T;
  u64* lsm = sm + li * LS;
  const int row = line0 + li;  // row index (ROW phases)

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
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (((e >> eb) & 1) == 0) {
            const int e2 = e | (1 << eb);
            const int idx = baseidx | (e << b);
            int twi;
            if (!INV) {
              const int s = LOGM - 1 - hb;
              if (COL) twi = (1 << s) + (idx >> (hb + 1));
              else twi = (1 << (n1 + s)) + (row << s) + (idx >> (hb + 1));
            } else {
              if (COL) twi = ((1 << n1) >> (hb + 1)) + (idx >> (hb + 1));
              else twi = (int)(N >> (hb + 1)) + (row << (LOGM - hb - 1)) + (idx >> (hb + 1));
            }
            const u64 w = __ldg(twv + twi), ws = __ldg(tws + twi);
            if (!INV) {
              const u64 U = x[e];
              const u64 V = shoup_mul(x[e2], w, ws, q);
              x[e] = add_mod(U, V, q);
              x[e2] = sub_mod(U, V, q);
            } else {
              const u64 U = x[e], V = x[e2];
              x[e] = add_mod(U, V, q);
              x[e2] = shoup_mul(sub_mod(U, V, q), w, ws, q);
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
    if (INV && COL) v = shoup_mul(v, P.ninv, P.ninv_sh, q);
    data[g] = v;
  }
}

template <int LOGM, bool INV, bool COL>
void launch_phase(const DevTables& t, const LimbSet& set, cudaStream_t st) {
  constexpr int M = 1 << LOGM;
  constexpr int LPC = COL ? 16 : (M >= 64 ? 2048 / M : 32);
  constexpr int threads = LPC * (M / 8);
  constexpr int LS = M + M / 8 + 1;
  const std::size_t smem = (std::size_t)LPC * LS * sizeof(u64);
  const int lines = COL ? (1 << t.n2) : (1 << t.n1);
  dim3 grid(lines / LPC, set.count());
  ntt_phase_kernel<LOGM, INV, COL><<<grid, threads, smem, st>>>(set, t.pc, t.tw, t.logN, t.n1, t.n2);
  launch_check("ntt_phase_kernel");
}

template <bool INV, bool COL>
void dispatch(const DevTables& t, const LimbSet& set, cudaStream_t st) {
  const int logm = COL ? t.n1 : t.n2;
  switch (logm) {
    case 5: launch_phase<5, INV, COL>(t, set, st); break;
    case 6: launch_phase<6, INV, COL>(t, set, st); break;
    case 7: launch_phase<7, INV, COL>(t, set, st); break;
    case 8: launch_phase<8, INV, COL>(t, set, st); break;
    default: throw std::runtime_error("unsupported NTT split " + std::to_string(logm));
  }
}

}  // namespace

void ntt_forward(const DevTables& t, const LimbSet& set, cudaStream_t st) {
  if (set.count() == 0) return;
  TimedScope ts(t, kNtt, st);
  dispatch<false, true>(t, set, st);
  dispatch<false, false>(t, set, st);
}

void ntt_inverse(const DevTables& t, const LimbSet& set, cudaStream_t st) {
  if (set.count() == 0) return;
  TimedScope ts(t, kNtt, st);
  dispatch<true, false>(t, set, st);
  dispatch<true, true>(t, set, st);
}

}  // namespace fheon
