// Plaintext encoding on the device: the special inverse FFT of the canonical
// embedding ("Encoding"), scaled and rounded to the N
// signed coefficients, then RNS / NTT by the existing kernels.
//
// Same arithmetic, in the same order, as the host restatement
// (engine.cpp fft_special_inv_host + encode_coeffs_host, itself mirrored by
// oracle/ckks_oracle.c ock_encode_coeffs): stages len = S, S/2, .., 2 of
//   u = x[j] + x[j + len/2],  v = (x[j] - x[j + len/2]) * ksi[(4 len - 5^j mod 4 len) (2N / 4 len)]
// then the bit reversal, /S, *scale, llround.  Every double operation is an
// explicitly rounded __dadd_rn / __dsub_rn / __dmul_rn (no FMA contraction,
// matching the host's -ffp-contract=off), so the coefficients are bit-identical.
//
// The last stages (len <= 2^LOG_SMEM) run in one kernel per 2^LOG_SMEM-point block
// staged in shared memory; the earlier, longer-stride stages one launch each.
#include "kernels.hpp"

namespace fheon {

namespace {

constexpr int kFftLogSmem = 11;  // 2048 complex points per CTA in shared memory (32 KiB)
constexpr int kFftThreads = 256;

__device__ __forceinline__ void fft_bfly(double& xr, double& xi, double& yr, double& yi, double wr, double wi) {
  const double ur = __dadd_rn(xr, yr), ui = __dadd_rn(xi, yi);
  const double vr = __dsub_rn(xr, yr), vi = __dsub_rn(xi, yi);
  xr = ur;
  xi = ui;
  yr = __dsub_rn(__dmul_rn(vr, wr), __dmul_rn(vi, wi));
  yi = __dadd_rn(__dmul_rn(vr, wi), __dmul_rn(vi, wr));
}

__device__ __forceinline__ u64 fft_root_index(const u64* rotgroup, int j, int len, u64 M) {
  const u64 lenq = (u64)len << 2;
  return (lenq - (rotgroup[j] % lenq)) * (M / lenq);
}

// one stage over all S/2 butterflies (len > 2^kFftLogSmem)
__global__ void k_fft_stage(double* re, double* im, int S, int len, const u64* __restrict__ rotgroup,
                            const double* __restrict__ ksi_re, const double* __restrict__ ksi_im, u64 M) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S / 2) return;
  const int lenh = len >> 1;
  const int blk = t / lenh, j = t - blk * lenh;
  const int a = blk * len + j, b = a + lenh;
  const u64 idx = fft_root_index(rotgroup, j, len, M);
  double xr = re[a], xi = im[a], yr = re[b], yi = im[b];
  fft_bfly(xr, xi, yr, yi, __ldg(ksi_re + idx), __ldg(ksi_im + idx));
  re[a] = xr;
  im[a] = xi;
  re[b] = yr;
  im[b] = yi;
}

// the remaining stages len = min(S, 2^kFftLogSmem) .. 2 on one 2^kFftLogSmem-point block per CTA
__global__ void k_fft_tail(double* re, double* im, int S, int len0, const u64* __restrict__ rotgroup,
                           const double* __restrict__ ksi_re, const double* __restrict__ ksi_im, u64 M) {
  __shared__ double sr[1 << kFftLogSmem], si[1 << kFftLogSmem];
  const int B = len0;  // block size = the first len handled here
  const int base = blockIdx.x * B;
  for (int k = threadIdx.x; k < B; k += blockDim.x) {
    sr[k] = re[base + k];
    si[k] = im[base + k];
  }
  __syncthreads();
  for (int len = B; len >= 2; len >>= 1) {
    const int lenh = len >> 1;
    for (int t = threadIdx.x; t < B / 2; t += blockDim.x) {
      const int blk = t / lenh, j = t - blk * lenh;
      const int a = blk * len + j, b = a + lenh;
      const u64 idx = fft_root_index(rotgroup, j, len, M);
      fft_bfly(sr[a], si[a], sr[b], si[b], __ldg(ksi_re + idx), __ldg(ksi_im + idx));
    }
    __syncthreads();
  }
  for (int k = threadIdx.x; k < B; k += blockDim.x) {
    re[base + k] = sr[k];
    im[base + k] = si[k];
  }
}

// bit reversal, / S, * scale, llround: coefficient i (real part) and i + S (imaginary)
__global__ void k_fft_finish(const double* __restrict__ re, const double* __restrict__ im, long long* coeffs, int S,
                             int logS, double scale) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S) return;
  const int r = (int)(__brev((unsigned)i) >> (32 - logS));
  const double a = __dmul_rn(__ddiv_rn(re[r], (double)S), scale);
  const double b = __dmul_rn(__ddiv_rn(im[r], (double)S), scale);
  coeffs[i] = llround(a);
  coeffs[i + S] = llround(b);
}

}  // namespace

void encode_fft_device(const DevTables& t, long long* coeffs, double* work, double scale, cudaStream_t st) {
  const int S = (int)(t.N / 2);
  const int logS = t.logN - 1;
  const u64 M = 2 * (u64)t.N;
  double* re = work;
  double* im = work + S;
  int len = S;
  const int tail = S < (1 << kFftLogSmem) ? S : (1 << kFftLogSmem);
  for (; len > tail; len >>= 1) {
    k_fft_stage<<<(S / 2 + kFftThreads - 1) / kFftThreads, kFftThreads, 0, st>>>(re, im, S, len, t.rotgroup,
                                                                               t.ksi_re, t.ksi_im, M);
    launch_check("k_fft_stage");
  }
  if (S >= 2) {
    k_fft_tail<<<S / tail, kFftThreads, 0, st>>>(re, im, S, tail, t.rotgroup, t.ksi_re, t.ksi_im, M);
    launch_check("k_fft_tail");
  }
  k_fft_finish<<<(S + kFftThreads - 1) / kFftThreads, kFftThreads, 0, st>>>(re, im, coeffs, S, logS, scale);
  launch_check("k_fft_finish");
}

}  // namespace fheon
