// Prototype: exact 64x64-bit RNS basis-conversion sums on the int8 tensor cores
// (tcgen05.mma kind::i8).  S[n][t] = sum_k y_k[n] * c[t][k] (< 2^124) computed as
// sum_s 2^(8s) D[n][(t,s)], D = A(bytes of y) x B(shifted bytes of c), then REDC.
// Checks the (hi, lo) sums and the REDC'd outputs against a CPU __int128
// reference and times the kernel against the CUDA-core Acc128 kernel.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a scripts/tcbconv_proto.cu -o scripts/bin/tcbconv
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <cuda_runtime.h>

typedef unsigned long long u64;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ u64 mulhi(u64 a, u64 b) { return __umul64hi(a, b); }
__device__ __forceinline__ u64 csub(u64 a, u64 q) { return a >= q ? a - q : a; }
__device__ __forceinline__ u64 redc(u64 hi, u64 lo, u64 q, u64 qneg) {
  const u64 m = lo * qneg;
  const u64 t = hi + mulhi(m, q) + (lo != 0 ? 1ULL : 0ULL);
  return csub(t, q);
}
struct Acc128 {
  u64 lo = 0, hi = 0;
  __device__ __forceinline__ void mac(u64 a, u64 b) {
    const u64 l = a * b, h = mulhi(a, b);
    lo += l;
    hi += h + (lo < l ? 1ULL : 0ULL);
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ u64 sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (u64)((saddr >> 4) & 0x3FFF) | ((u64)((lbo >> 4) & 0x3FFF) << 16) | ((u64)((sbo >> 4) & 0x3FFF) << 32) |
         ((u64)1 << 46);
}

constexpr int kTch = 8;  // targets per MMA (N = 16 * kTch = 128 columns)

// KIN inputs (padded to KINP, multiple of 4), T targets.  256 threads: warp w
// reads TMEM lanes 32*(w%4).. and handles the targets of parity w/4; two TMEM
// buffers of 128 columns so chunk i+1's MMAs run under chunk i's epilogue.
template <int KINP>
__global__ void __launch_bounds__(256) k_tc(const u64* __restrict__ y, const u64* __restrict__ c,
                                            const u64* __restrict__ q, const u64* __restrict__ qn,
                                            u64* __restrict__ out, u64* __restrict__ shi, u64* __restrict__ slo,
                                            int N, int KIN, int T) {
  constexpr int KC = KINP / 2;       // 16-byte chunks per row
  constexpr int SBO = KC * 16 * 8;   // bytes per 8-row group
  constexpr int KSTEPS = KINP / 4;   // 32-byte MMA K steps
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) u64 mbar[2];
  const int Tp = (T + kTch - 1) / kTch * kTch;
  unsigned char* A = sm;
  unsigned char* B = sm + 128 * KC * 16;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = (warp & 3) * 32 + (tid & 31);
  const int par = warp >> 2;
  for (int idx = tid; idx < Tp * KINP; idx += 256) {
    const int t = idx / KINP, k = idx % KINP;
    const u64 cv = (t < T && k < KIN) ? c[(size_t)t * KIN + k] : 0;
    const u64 r = ((u64)__byte_perm((uint32_t)cv, 0, 0x0123) << 32) | __byte_perm((uint32_t)(cv >> 32), 0, 0x0123);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const u64 v = s <= 7 ? (r >> (8 * (7 - s))) : (s < 15 ? (r << (8 * (s - 7))) : 0);
      const int br = t * 16 + s;
      *(u64*)(B + (br >> 3) * SBO + (k >> 1) * 128 + (br & 7) * 16 + (k & 1) * 8) = v;
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(16 * kTch >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  uint32_t phase[2] = {0, 0};
  const int tiles = N / 128;
  const int nch = (T + kTch - 1) / kTch;
  auto issue = [&](int ch) {
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int j = 0; j < KSTEPS; ++j) {
        const u64 ad = sdesc(smem_u32(A) + j * 256, 128, SBO);
        const u64 bd = sdesc(smem_u32(B) + (ch * kTch * 16 / 8) * SBO + j * 256, 128, SBO);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + (ch & 1) * 128),
            "l"(ad), "l"(bd), "r"(idesc), "r"(j));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&mbar[ch & 1]))
                   : "memory");
    }
  };
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    if (tid < 128) {
      const int n = tile * 128 + tid;
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) {
        const int k0 = 2 * cc, k1 = 2 * cc + 1;
        const u64 v0 = k0 < KIN ? y[(size_t)k0 * N + n] : 0;
        const u64 v1 = k1 < KIN ? y[(size_t)k1 * N + n] : 0;
        unsigned char* p = A + (tid >> 3) * SBO + cc * 128 + (tid & 7) * 16;
        *(ulonglong2*)p = make_ulonglong2(v0, v1);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    issue(0);
    const int n = tile * 128 + row;
    for (int ch = 0; ch < nch; ++ch) {
      const uint32_t mb = smem_u32(&mbar[ch & 1]);
      asm volatile(
          "{\n.reg .pred P1;\nWAIT_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(mb),
          "r"(phase[ch & 1])
          : "memory");
      phase[ch & 1] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (ch + 1 < nch) issue(ch + 1);
      const int t0 = ch * kTch;
      const int nt = min(kTch, T - t0);
      for (int tt = par; tt < nt; tt += 2) {
        uint32_t d[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
              "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
            : "r"(tm + (ch & 1) * 128 + ((uint32_t)((warp & 3) * 32) << 16) + tt * 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const u64 x0 = (u64)d[0] + ((u64)d[1] << 8) + ((u64)d[2] << 16) + ((u64)d[3] << 24) + ((u64)d[4] << 32) +
                       ((u64)d[5] << 40);
        const u64 x1 = (u64)d[6] + ((u64)d[7] << 8) + ((u64)d[8] << 16) + ((u64)d[9] << 24) + ((u64)d[10] << 32) +
                       ((u64)d[11] << 40);
        const u64 x2 = (u64)d[12] + ((u64)d[13] << 8) + ((u64)d[14] << 16);
        const u64 lo = x0 + (x1 << 48);
        const u64 hi = (x1 >> 16) + (x2 << 32) + (lo < x0 ? 1ULL : 0ULL);
        const int t = t0 + tt;
        out[(size_t)t * N + n] = redc(hi, lo, q[t], qn[t]);
        if (shi) {
          shi[(size_t)t * N + n] = hi;
          slo[(size_t)t * N + n] = lo;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
    }
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(mb),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t mb) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t a, uint32_t* d) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
        "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
      : "r"(a));
}
__device__ __forceinline__ u64 madw(uint32_t a, uint32_t b, u64 c) {
  u64 d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
// S = sum_s d[s] 2^(8s), d[s] < 2^23, S < 2^124 (so hi is exact mod 2^64)
__device__ __forceinline__ void combine(const uint32_t* d, u64& hi, u64& lo) {
  u64 x0 = madw(d[3], 1u << 24, madw(d[2], 1u << 16, madw(d[1], 1u << 8, d[0])));
  x0 += (u64)(d[5] * 256u + d[4]) << 32;
  u64 x1 = madw(d[9], 1u << 24, madw(d[8], 1u << 16, madw(d[7], 1u << 8, d[6])));
  x1 += (u64)(d[11] * 256u + d[10]) << 32;
  const u64 x2 = madw(d[14], 1u << 16, madw(d[13], 1u << 8, d[12]));
  lo = x0 + (x1 << 48);
  hi = (x1 >> 16) + (x2 << 32) + (lo < x0 ? 1ULL : 0ULL);
}

// Warp-specialised: warps 0-7 epilogue (warp w: TMEM lanes 32*(w%4), targets of
// parity w/4), warp 8 loads A (double-buffered) and issues the MMAs; two TMEM
// buffers of 128 columns with full/empty mbarriers.
template <int KINP>
__global__ void __launch_bounds__(320) k_tc2(const u64* __restrict__ y, const u64* __restrict__ c,
                                             const u64* __restrict__ q, const u64* __restrict__ qn,
                                             u64* __restrict__ out, int N, int KIN, int T) {
  constexpr int KC = KINP / 2;
  constexpr int SBO = KC * 16 * 8;
  constexpr int KSTEPS = KINP / 4;
  constexpr int ABYTES = 128 * KC * 16;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) u64 full[2], empty[2], afree[2], afull[2];
  __shared__ u64 sq[64][2];
  const int Tp = (T + kTch - 1) / kTch * kTch;
  unsigned char* A = sm;                 // [2][ABYTES]
  unsigned char* B = sm + 2 * ABYTES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // constants staged in smem first (one global load per thread, all in flight)
  __shared__ u64 cst[64 * 16];
  for (int z = tid; z < T * KIN; z += blockDim.x) cst[z] = __ldg(c + z);
  __syncthreads();
  // B slots in smem order (conflict-free): slot z = ((rowgroup*KC + chunk)*8 + r)*2 + kb
  for (int z = tid; z < Tp * 16 * KINP; z += blockDim.x) {
    const int kb = z & 1, r = (z >> 1) & 7, chunk = (z >> 4) % KC, rg = (z >> 4) / KC;
    const int br = rg * 8 + r, t = br >> 4, s = br & 15, k = chunk * 2 + kb;
    const u64 cv = (t < T && k < KIN) ? cst[t * KIN + k] : 0;
    const u64 rv = ((u64)__byte_perm((uint32_t)cv, 0, 0x0123) << 32) | __byte_perm((uint32_t)(cv >> 32), 0, 0x0123);
    ((u64*)B)[z] = s <= 7 ? (rv >> (8 * (7 - s))) : (s < 15 ? (rv << (8 * (s - 7))) : 0);
  }
  for (int t = tid; t < T; t += blockDim.x) {
    sq[t][0] = q[t];
    sq[t][1] = qn[t];
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&empty[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&afree[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&afull[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(16 * kTch >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int tiles = N / 128;
  const int nch = (T + kTch - 1) / kTch;
  if (warp == 8) {  // A loader, one tile ahead
    int tl = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tl) {
      const int ab = tl & 1;
      mbar_wait(smem_u32(&afree[ab]), ((tl >> 1) & 1) ^ 1);
      unsigned char* Ab = A + ab * ABYTES;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = lane + 32 * i;
        const int n = tile * 128 + r;
#pragma unroll
        for (int cc = 0; cc < KC; ++cc) {
          const int k0 = 2 * cc, k1 = 2 * cc + 1;
          const u64 v0 = k0 < KIN ? y[(size_t)k0 * N + n] : 0;
          const u64 v1 = k1 < KIN ? y[(size_t)k1 * N + n] : 0;
          *(ulonglong2*)(Ab + (r >> 3) * SBO + cc * 128 + (r & 7) * 16) = make_ulonglong2(v0, v1);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&afull[ab])) : "memory");
    }
  } else if (warp == 9) {  // MMA issuer
    int use = 0, tl = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tl) {
      const int ab = tl & 1;
      unsigned char* Ab = A + ab * ABYTES;
      if (lane == 0) {
        mbar_wait(smem_u32(&afull[ab]), (tl >> 1) & 1);
        for (int ch = 0; ch < nch; ++ch, ++use) {
          const int b = use & 1;
          mbar_wait(smem_u32(&empty[b]), ((use >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
          for (int j = 0; j < KSTEPS; ++j) {
            const u64 ad = sdesc(smem_u32(Ab) + j * 256, 128, SBO);
            const u64 bd = sdesc(smem_u32(B) + (ch * kTch * 16 / 8) * SBO + j * 256, 128, SBO);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + b * 128),
                "l"(ad), "l"(bd), "r"(idesc), "r"(j));
          }
          mma_commit(smem_u32(&full[b]));
        }
        mma_commit(smem_u32(&afree[ab]));
      }
      __syncwarp();
    }
  } else {
    const int par = warp >> 2;
    const uint32_t lanebase = (uint32_t)((warp & 3) * 32) << 16;
    int use = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const int n = tile * 128 + (warp & 3) * 32 + lane;
      for (int ch = 0; ch < nch; ++ch, ++use) {
        const int b = use & 1;
        mbar_wait(smem_u32(&full[b]), (use >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int t0 = ch * kTch;
        const int nt = min(kTch, T - t0);
        uint32_t d[4][16];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (par + 2 * i < nt) tmem_ld16(tm + b * 128 + lanebase + (par + 2 * i) * 16, d[i]);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[b])) : "memory");
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int tt = par + 2 * i;
          if (tt < nt) {
            u64 hi, lo;
            combine(d[i], hi, lo);
            const int t = t0 + tt;
            out[(size_t)t * N + n] = redc(hi, lo, sq[t][0], sq[t][1]);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

// CUDA-core reference kernel (the engine's current scheme): 8 targets per CTA
template <int KIN>
__global__ void __launch_bounds__(256) k_cc(const u64* __restrict__ y, const u64* __restrict__ c,
                                            const u64* __restrict__ q, const u64* __restrict__ qn,
                                            u64* __restrict__ out, int N, int T) {
  __shared__ u64 cs[8][KIN];
  const int n = blockIdx.x * 256 + threadIdx.x;
  const int t0 = blockIdx.y * 8;
  if (threadIdx.x < 8 * KIN) {
    const int cc = threadIdx.x / KIN, k = threadIdx.x % KIN;
    cs[cc][k] = t0 + cc < T ? c[(size_t)(t0 + cc) * KIN + k] : 0;
  }
  __syncthreads();
  u64 yy[KIN];
#pragma unroll
  for (int k = 0; k < KIN; ++k) yy[k] = y[(size_t)k * N + n];
  const int nt = min(8, T - t0);
  for (int cc = 0; cc < nt; ++cc) {
    Acc128 a;
#pragma unroll
    for (int k = 0; k < KIN; ++k) a.mac(yy[k], cs[cc][k]);
    out[(size_t)(t0 + cc) * N + n] = redc(a.hi, a.lo, q[t0 + cc], qn[t0 + cc]);
  }
}

static u64 inv_neg(u64 q) {  // -q^-1 mod 2^64
  u64 x = 1;
  for (int i = 0; i < 7; ++i) x *= 2 - q * x;
  return (u64)0 - x;
}

int main(int argc, char** argv) {
  const int N = 1 << (argc > 4 ? atoi(argv[4]) : 16), KIN = argc > 1 ? atoi(argv[1]) : 12, T = argc > 2 ? atoi(argv[2]) : 30;
  const int reps = 20;
  std::mt19937_64 rng(7);
  std::vector<u64> y((size_t)KIN * N), c((size_t)T * KIN), q(T), qn(T);
  for (auto& v : y) v = rng() >> 4;
  for (int t = 0; t < T; ++t) {
    q[t] = ((rng() >> 4) | 1ULL) | (1ULL << 59);
    qn[t] = inv_neg(q[t]);
  }
  for (auto& v : c) v = rng() >> 4;
  u64 *dy, *dc, *dq, *dqn, *dout, *dout2, *dhi, *dlo;
  CK(cudaMalloc(&dy, y.size() * 8));
  CK(cudaMalloc(&dc, c.size() * 8));
  CK(cudaMalloc(&dq, T * 8));
  CK(cudaMalloc(&dqn, T * 8));
  CK(cudaMalloc(&dout, (size_t)T * N * 8));
  CK(cudaMalloc(&dout2, (size_t)T * N * 8));
  CK(cudaMalloc(&dhi, (size_t)T * N * 8));
  CK(cudaMalloc(&dlo, (size_t)T * N * 8));
  CK(cudaMemcpy(dy, y.data(), y.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dc, c.data(), c.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dq, q.data(), T * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dqn, qn.data(), T * 8, cudaMemcpyHostToDevice));
  const int KINP = (KIN + 3) / 4 * 4;
  const int Tp = (T + kTch - 1) / kTch * kTch;
  const size_t smem = (size_t)128 * KINP * 8 + (size_t)Tp * 16 * KINP * 8;
  auto tc = KINP == 12 ? k_tc<12> : KINP == 16 ? k_tc<16> : KINP == 8 ? k_tc<8> : k_tc<4>;
  auto cc = KIN == 12 ? k_cc<12> : KIN == 15 ? k_cc<15> : KIN == 4 ? k_cc<4> : k_cc<8>;
  CK(cudaFuncSetAttribute(tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev_sms = 148;
  const int grid = argc > 3 ? atoi(argv[3]) : 148 * 2;
  printf("KIN %d T %d smem %zu grid %d\n", KIN, T, smem, grid);
  tc<<<grid, 256, smem>>>(dy, dc, dq, dqn, dout, dhi, dlo, N, KIN, T);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<u64> hi((size_t)T * N), lo((size_t)T * N), o1((size_t)T * N), o2((size_t)T * N);
  CK(cudaMemcpy(hi.data(), dhi, hi.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(lo.data(), dlo, lo.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(o1.data(), dout, o1.size() * 8, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (int t = 0; t < T; ++t)
    for (int n = 0; n < N; n += (n < 1024 ? 1 : 37)) {
      unsigned __int128 s = 0;
      for (int k = 0; k < KIN; ++k) s += (unsigned __int128)y[(size_t)k * N + n] * c[(size_t)t * KIN + k];
      if ((u64)s != lo[(size_t)t * N + n] || (u64)(s >> 64) != hi[(size_t)t * N + n]) {
        if (bad < 5) printf("mismatch t %d n %d: got %llx:%llx want %llx:%llx\n", t, n, hi[(size_t)t * N + n],
                            lo[(size_t)t * N + n], (u64)(s >> 64), (u64)s);
        ++bad;
      }
    }
  cc<<<dim3(N / 256, (T + 7) / 8), 256>>>(dy, dc, dq, dqn, dout2, N, T);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(o2.data(), dout2, o2.size() * 8, cudaMemcpyDeviceToHost));
  size_t bad2 = 0;
  for (size_t i = 0; i < o1.size(); ++i) bad2 += o1[i] != o2[i];
  printf("exact-sum mismatches %zu, redc mismatches vs cuda-core %zu\n", bad, bad2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int g : {148, 296, 444, 592, 1024}) {
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) tc<<<g, 256, smem>>>(dy, dc, dq, dqn, dout, nullptr, nullptr, N, KIN, T);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("tc grid %4d: %.2f us\n", g, 1000 * ms / reps);
  }
  {
    auto tc2 = KINP == 12 ? k_tc2<12> : KINP == 16 ? k_tc2<16> : KINP == 8 ? k_tc2<8> : k_tc2<4>;
    const size_t smem2 = (size_t)2 * 128 * KINP * 8 + (size_t)Tp * 16 * KINP * 8;
    CK(cudaFuncSetAttribute(tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    CK(cudaMemset(dout, 0, (size_t)T * N * 8));
    tc2<<<296, 320, smem2>>>(dy, dc, dq, dqn, dout, N, KIN, T);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(o1.data(), dout, o1.size() * 8, cudaMemcpyDeviceToHost));
    size_t b3 = 0;
    for (size_t i = 0; i < o1.size(); ++i) b3 += o1[i] != o2[i];
    printf("tc2 smem %zu: redc mismatches vs cuda-core %zu\n", smem2, b3);
    for (int g : {148, 296, 444, 592}) {
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) tc2<<<g, 320, smem2>>>(dy, dc, dq, dqn, dout, N, KIN, T);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("tc2 grid %4d: %.2f us\n", g, 1000 * ms / reps);
    }
  }
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) cc<<<dim3(N / 256, (T + 7) / 8), 256>>>(dy, dc, dq, dqn, dout2, N, T);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cuda-core: %.2f us\n", 1000 * ms / reps);
  return 0;
}
