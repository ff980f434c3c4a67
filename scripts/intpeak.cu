// Integer-pipe peak microbenchmark for the NTT roofline:
// dependency-free IMAD (32-bit), IMAD.WIDE.U32 (32x32->64) and the full lazy
// Shoup butterfly used by the NTT (64-bit words, q < 2^60), all SMs busy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o intpeak intpeak.cu
#include <cstdint>
#include <cstdio>

typedef unsigned long long u64;

__global__ void k_imad(unsigned* out, unsigned seed, int iters) {
  unsigned a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed + threadIdx.x * 16 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = a[i] * a[i] + 0x7F4A7C15u;  // nonlinear: no closed form
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imad_wide(u64* out, unsigned seed, int iters) {
  u64 a[16];
  unsigned m[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = seed + threadIdx.x * 16 + i;
    m[i] = 0x9E3779B1u + i;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const unsigned lo = (unsigned)a[i];
      a[i] = (u64)lo * lo + m[i];  // one IMAD.WIDE.U32 per step (nonlinear)
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imad_hi(unsigned* out, unsigned seed, int iters) {
  unsigned a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed + threadIdx.x * 16 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = __umulhi(a[i], a[i] | 0x80000001u) ^ (unsigned)i;
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 wsh, u64 q) { return a * w - __umul64hi(a, wsh) * q; }

__global__ void k_butterfly(u64* out, u64 q, u64 w, u64 wsh, int iters) {
  u64 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x * 8 + i) % q;
  const u64 q2 = 2 * q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {  // 4 independent lazy CT butterflies
      u64 X = x[i];
      X = X >= q2 ? X - q2 : X;
      const u64 T = shoup_lazy(x[i + 1], w, wsh, q);
      x[i] = X + T;
      x[i + 1] = X - T + q2;
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// approximate Shoup quotient: floor(Y W' / 2^64) - {0, 1}; drops the lo x lo partial product
__device__ __forceinline__ u64 mulhi_approx(u64 y, u64 w) {
  const unsigned yl = (unsigned)y, yh = (unsigned)(y >> 32), wl = (unsigned)w, wh = (unsigned)(w >> 32);
  const u64 hh = (u64)yh * wh, hl = (u64)yh * wl, lh = (u64)yl * wh;
  const u64 mid = (hl >> 32) + (lh >> 32) + (((u64)(unsigned)hl + (unsigned)lh) >> 32);
  return hh + mid;
}

__global__ void k_butterfly_approx(u64* out, u64 q, u64 w, u64 wsh, int iters) {
  u64 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x * 8 + i) % q;
  const u64 q2 = 2 * q, q3 = 3 * q, q4 = 4 * q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {  // values in [0, 6q)
      u64 X = x[i];
      X = X >= q4 ? X - q4 : X;
      X = X >= q2 ? X - q2 : X;
      const u64 T = x[i + 1] * w - mulhi_approx(x[i + 1], wsh) * q;  // [0, 3q)
      x[i] = X + T;
      x[i + 1] = X - T + q3;
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3-product high word (drops lo x lo: result in {hi - 1, hi}), PTX carry chains
__device__ __forceinline__ u64 mulhi3(u64 a, u64 b) {
  const unsigned alo = (unsigned)a, ahi = (unsigned)(a >> 32), blo = (unsigned)b, bhi = (unsigned)(b >> 32);
  unsigned rlo, rhi;
  asm("{\n\t"
      ".reg .u32 m0, m1, c;\n\t"
      "mul.lo.u32 m0, %2, %5;\n\t"
      "mul.hi.u32 m1, %2, %5;\n\t"
      "mad.lo.cc.u32 m0, %3, %4, m0;\n\t"
      "madc.hi.cc.u32 m1, %3, %4, m1;\n\t"
      "addc.u32 c, 0, 0;\n\t"
      "mad.lo.cc.u32 %0, %3, %5, m1;\n\t"
      "madc.hi.u32 %1, %3, %5, c;\n\t"
      "}"
      : "=r"(rlo), "=r"(rhi)
      : "r"(alo), "r"(ahi), "r"(blo), "r"(bhi));
  return ((u64)rhi << 32) | rlo;
}

// lazy CT butterfly on [0, 8q) with the 3-product quotient (T in [0, 3q))
__global__ void k_butterfly3(u64* out, u64 q, u64 w, u64 wsh, int iters) {
  u64 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x * 8 + i) % q;
  const u64 q3 = 3 * q, q4 = 4 * q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      u64 X = x[i];
      X = X >= q4 ? X - q4 : X;
      const u64 T = x[i + 1] * w - mulhi3(x[i + 1], wsh) * q;
      x[i] = X + T;
      x[i + 1] = X - T + q3;
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, double seed, int iters) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed + threadIdx.x * 16 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], 0.999999, 1e-7);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FP64 lazy CT butterfly for q < 2^50: values are exact integers in doubles,
// a*w mod q via hi = fl(a w), lo = fma(a, w, -hi) (exact), quotient = rint(hi / q)
// (magic-number rounding), r = fma(-quot, q, hi) + lo in (-q, q)
__global__ void k_butterfly_f64(double* out, double q, double w, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (double)((threadIdx.x * 8 + i) % 1000003);
  const double qinv = 1.0 / q, magic = 6755399441055744.0, q2 = 2 * q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      double X = x[i];
      X = X >= q2 ? X - q2 : X;
      const double y = x[i + 1];
      const double hi = y * w;
      const double lo = fma(y, w, -hi);
      const double qt = fma(hi, qinv, magic) - magic;
      double T = fma(-qt, q, hi) + lo;
      T = T < 0 ? T + q : T;
      x[i] = X + T;
      x[i + 1] = X - T + q;
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  u64* out;
  cudaMalloc(&out, (size_t)blocks * threads * sizeof(u64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  const double thr = (double)blocks * threads;
  // warm
  k_imad<<<blocks, threads>>>((unsigned*)out, 1, 16);
  k_imad_wide<<<blocks, threads>>>(out, 1, 16);
  k_butterfly<<<blocks, threads>>>(out, 1152921504606846883ULL, 12345, 678, 16);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k_imad<<<blocks, threads>>>((unsigned*)out, 1, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double imad = thr * iters * 16 / (ms * 1e-3);
  cudaEventRecord(e0);
  k_imad_wide<<<blocks, threads>>>(out, 1, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double wide = thr * iters * 16 / (ms * 1e-3);
  k_imad_hi<<<blocks, threads>>>((unsigned*)out, 1, 16);
  cudaEventRecord(e0);
  k_imad_hi<<<blocks, threads>>>((unsigned*)out, 1, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double hi = thr * iters * 16 / (ms * 1e-3);
  printf("{\"imad_hi_per_s\": %.4e, \"imad_hi_per_clk_per_sm\": %.2f}\n", hi, hi / sms / (clk * 1e3));
  cudaEventRecord(e0);
  k_butterfly<<<blocks, threads>>>(out, 1152921504606846883ULL, 0x123456789ULL, 0xABCDEF12345ULL, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double bf = thr * iters * 4 / (ms * 1e-3);
  k_butterfly_approx<<<blocks, threads>>>(out, 1152921504606846883ULL, 0x123456789ULL, 0xABCDEF12345ULL, 16);
  cudaEventRecord(e0);
  k_butterfly_approx<<<blocks, threads>>>(out, 1152921504606846883ULL, 0x123456789ULL, 0xABCDEF12345ULL, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double bfa = thr * iters * 4 / (ms * 1e-3);
  printf("{\"approx_butterflies_per_s\": %.4e, \"approx_butterflies_per_clk_per_sm\": %.3f}\n", bfa,
         bfa / sms / (clk * 1e3));
  k_butterfly3<<<blocks, threads>>>(out, 1152921504606846883ULL, 0x123456789ULL, 0xABCDEF12345ULL, 16);
  cudaEventRecord(e0);
  k_butterfly3<<<blocks, threads>>>(out, 1152921504606846883ULL, 0x123456789ULL, 0xABCDEF12345ULL, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double bf3 = thr * iters * 4 / (ms * 1e-3);
  k_dfma<<<blocks, threads>>>((double*)out, 1.0, 16);
  cudaEventRecord(e0);
  k_dfma<<<blocks, threads>>>((double*)out, 1.0, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma = thr * iters * 16 / (ms * 1e-3);
  k_butterfly_f64<<<blocks, threads>>>((double*)out, 1099511627689.0, 123456789.0, 16);
  cudaEventRecord(e0);
  k_butterfly_f64<<<blocks, threads>>>((double*)out, 1099511627689.0, 123456789.0, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double bff = thr * iters * 4 / (ms * 1e-3);
  printf("{\"dfma_per_clk_per_sm\": %.2f, \"f64_butterflies_per_s\": %.4e, \"f64_butterflies_per_clk_per_sm\": %.3f}\n",
         dfma / sms / (clk * 1e3), bff, bff / sms / (clk * 1e3));
  printf("{\"ptx3_butterflies_per_s\": %.4e, \"ptx3_butterflies_per_clk_per_sm\": %.3f}\n", bf3,
         bf3 / sms / (clk * 1e3));
  printf("{\"sms\": %d, \"clock_khz\": %d, \"imad_per_s\": %.4e, \"imad_wide_u32_per_s\": %.4e, "
         "\"shoup_ct_butterflies_per_s\": %.4e, \"imad_per_clk_per_sm\": %.2f, \"imad_wide_per_clk_per_sm\": %.2f, "
         "\"butterflies_per_clk_per_sm\": %.3f}\n",
         sms, clk, imad, wide, bf, imad / sms / (clk * 1e3), wide / sms / (clk * 1e3), bf / sms / (clk * 1e3));
  return 0;
}
