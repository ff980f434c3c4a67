// RNS basis conversion on the int8 tensor cores (tcgen05.mma kind::i8).
//
// ModUp and ModDown both need, per coefficient n and target limb t, the exact
// 128-bit sum S[n][t] = sum_k y_k[n] * c[t][k] of KIN (<= 16) products of
// 60-bit words (S < 2^124), followed by one REDC mod q_t.  On the CUDA cores
// every product costs 4 IMAD.WIDE on the half-rate pipe.  Here the products run
// on the tensor cores, exactly:
//
//   y_k = sum_a 2^(8a) y_k[a]   (bytes a = 0..7),   c = sum_b 2^(8b) c[b]
//   S   = sum_s 2^(8s) D[s],    D[s] = sum_k sum_{a+b=s} y_k[a] c[t][k][b]
//
// D is an int8 GEMM: A[n][(k,a)] = y_k[a] (each A row is just the y_k words,
// little-endian), B[(t,s)][(k,a)] = c[t][k][s-a] (0 outside 0..7), 16 columns
// s per target (s = 15 is zero padding), u8 x u8 -> s32 with D[s] < 8 * 16 *
// 255^2 < 2^23.  The epilogue recombines the 15 partial sums into (hi, lo)
// with mad.wide and runs the same REDC as the CUDA-core kernels, so results are
// bit-identical to them (and to oracle/ckks_oracle.c).
//
// One CTA = 13 warps, persistent over 128-coefficient tiles of every poly:
//   warps 8-11 (loaders, one row per lane): y_k of the tile's 128 rows (mode-specific: Shoup product
//     for ModUp, + the FP64 overflow estimate for ModDown) -> A[tile & 1] in
//     the canonical no-swizzle K-major layout; mbarrier afull.
//   warp 12 (MMA): per chunk of 8 targets, KINP/4 tcgen05.mma (M=128, N=128,
//     K=32) into one of two 128-column TMEM buffers; commit -> full[b].
//   warps 0-7 (epilogue): tcgen05.ld 32 lanes x 16 columns per target, warp w
//     reading lanes 32*(w%4).. and the targets of parity w/4; recombine, REDC,
//     mode-specific finish, coalesced store; arrive empty[b].
// B (all targets, byte-expanded) is built once per CTA in shared memory.
#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "kernels.hpp"

namespace fheon {

namespace {

constexpr int kTcTargets = 8;       // targets per MMA chunk (N = 128 columns)
constexpr int kTcThreads = 416;     // 8 epilogue warps + 4 loader warps + MMA warp
constexpr int kTcMmaWarp = 12;
constexpr int kTcMaxT = 64;         // max targets per launch (larger sets are split)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// shared-memory matrix descriptor, no swizzle (K-major: LBO = K-chunk stride,
// SBO = 8-row-group stride), Blackwell descriptor version 1
__device__ __forceinline__ u64 tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (u64)((saddr >> 4) & 0x3FFF) | ((u64)((lbo >> 4) & 0x3FFF) << 16) | ((u64)((sbo >> 4) & 0x3FFF) << 32) |
         ((u64)1 << 46);
}
__device__ __forceinline__ void mbar_init(u64* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(u64* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mma_commit(u64* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
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
// S = sum_s d[s] 2^(8s) with d[s] < 2^23, d[15] = 0 and S < 2^124:
//   e_j = d_2j + 2^8 d_2j+1 < 2^32 (one IMAD), f_i = e_2i + 2^16 e_2i+1 < 2^49 (one
//   IMAD.WIDE; m16 = 2^16 arrives as a kernel argument so ptxas keeps the
//   multiply), S = f0 + 2^32 f1 + 2^64 f2 + 2^96 f3 (one carry chain).
__device__ __forceinline__ void recombine(const uint32_t* d, uint32_t m16, u64& hi, u64& lo) {
  uint32_t e[8];
#pragma unroll
  for (int j = 0; j < 7; ++j) e[j] = d[2 * j + 1] * 256u + d[2 * j];
  e[7] = d[14];
  u64 f[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) f[i] = madw(e[2 * i + 1], m16, e[2 * i]);
  uint32_t w1, w2, w3;
  asm("add.cc.u32 %0, %3, %4;\n\taddc.cc.u32 %1, %5, %6;\n\taddc.u32 %2, %7, %8;"
      : "=r"(w1), "=r"(w2), "=r"(w3)
      : "r"((uint32_t)(f[0] >> 32)), "r"((uint32_t)f[1]), "r"((uint32_t)(f[1] >> 32)), "r"((uint32_t)f[2]),
        "r"((uint32_t)(f[2] >> 32)), "r"((uint32_t)f[3]));
  lo = ((u64)w1 << 32) | (uint32_t)f[0];
  hi = ((u64)w3 << 32) | w2;
}

struct TcBconvArgs {
  PolyList in, out;
  const PrimeConst* pc;
  const u64* qhinv;    // ModUp: [tab][kMaxAlpha][2]
  const u64* qhat;     // ModUp: [tab][L+K][kMaxAlpha]
  const u64* md_pk;    // ModDown
  const double* md_pinv;
  const u64* md_phat;
  const u64* md_q;
  int logN, limbs, L, K;
  int kin, T, tb;      // GEMM inputs, targets of this launch, first target
  int nin;             // inputs read from memory (ModDown folded: kin = nin + 2)
  int lo, j, tab;      // ModUp digit
  // ModUp, every digit in one launch (ndig > 0): CTAs [cta0[d], cta0[d+1]) convert digit d
  int ndig;
  int dlo[kMaxDigits], dkin[kMaxDigits], dT[kMaxDigits], dj[kMaxDigits], dtab[kMaxDigits];
  int cta0[kMaxDigits + 1];
  int s_ell, sp0;      // ModDown inputs: s < s_ell are Q limbs sp0 + s, the rest p_{s - s_ell}
  uint32_t m16;        // 2^16 (opaque to ptxas, see recombine)
};

// MODE 0 = ModUp digit j.  MODE 1 = ModDown with the finish folded into the
// GEMM: two extra inputs (the last two K columns) y = u (overflow estimate) and 1, constants
// [-P]_q and [-(P-1)/2]_q R (Montgomery), so REDC(S') = REDC(S) - u P R^-1 -
// (P-1)/2 mod q, the same canonical residue as the explicit finish; needs
// K + 2 <= 16 and (K 2^60 + 17) q < 2^64 q.  MODE 2 = ModDown, explicit finish.
template <int KINP, int MODE>
__global__ void __launch_bounds__(kTcThreads, 2) k_bconv_tc(TcBconvArgs a) {
  constexpr int KC = KINP / 2;       // 16-byte K chunks per row
  constexpr int SBO = KC * 128;      // bytes per 8-row group
  constexpr int ABYTES = 128 * KC * 16;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) u64 full[2], empty[2], afree[2], afull[2], ufree[2];
  __shared__ u64 cst[kTcMaxT * 16];  // c[t][k]
  __shared__ u64 tq[kTcMaxT][4];     // q, qinv_neg, mode consts
  __shared__ u64 toff[kTcMaxT];      // destination limb offset (limb * N) of each target
  __shared__ u64 yin[16][4];         // per-input (w, w', q, add)
  __shared__ double ypinv[16];
  __shared__ u64 urow[2][128];       // ModDown overflow estimate per row
  unsigned char* A = smem;           // [2][ABYTES]
  unsigned char* B = smem + 2 * ABYTES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int KIN = a.kin, T = a.T, nin = a.nin, lo = a.lo, jd = a.j, tab = a.tab, tb = a.tb;
  int bx = blockIdx.x, gx = gridDim.x;
  if (MODE == 0 && a.ndig > 0) {  // this CTA's digit
    int d = 0;
    while (d + 1 < a.ndig && (int)blockIdx.x >= a.cta0[d + 1]) ++d;
    lo = a.dlo[d];
    KIN = nin = a.dkin[d];
    T = a.dT[d];
    jd = a.dj[d];
    tab = a.dtab[d];
    tb = 0;
    bx = (int)blockIdx.x - a.cta0[d];
    gx = a.cta0[d + 1] - a.cta0[d];
  }
  FHEON_DCHECK(T >= 1 && T <= kTcMaxT && KIN >= 1 && KIN <= KINP && nin <= KIN && (MODE != 0 || a.ndig <= kMaxDigits) &&
               bx >= 0 && gx >= 1);
  const int Tp = (T + kTcTargets - 1) / kTcTargets * kTcTargets;
  const std::size_t N = (std::size_t)1 << a.logN;
  const int E = a.limbs + a.K;

  // ---- per-launch tables
  for (int z = tid; z < T * KIN; z += blockDim.x) {
    const int t = tb + z / KIN, k = z % KIN;
    if (MODE == 0) {
      const int tt = t < lo ? t : t + KIN;
      const int pt = tt < a.limbs ? tt : a.L + (tt - a.limbs);
      cst[z] = a.qhat[((std::size_t)tab * (a.L + a.K) + pt) * kMaxAlpha + k];
    } else if (MODE == 2 || k < nin) {
      cst[z] = a.md_phat[(std::size_t)t * kMaxK + k];
    } else if (k >= KIN - 2) {  // folded finish in the last two columns
      const PrimeConst P = a.pc[t];
      const u64 v = a.md_q[(std::size_t)t * 4 + (k == KIN - 2 ? 0 : 1)];
      const u64 neg = v ? P.q - v : 0;
      cst[z] = k == KIN - 2 ? neg : to_mont_d(neg, P);
    } else {
      cst[z] = 0;
    }
  }
  for (int i = tid; i < T; i += blockDim.x) {
    const int t = tb + i;
    if (MODE == 0) {
      const int tt = t < lo ? t : t + KIN;
      const int pt = tt < a.limbs ? tt : a.L + (tt - a.limbs);
      tq[i][0] = a.pc[pt].q;
      tq[i][1] = a.pc[pt].qinv_neg;
      toff[i] = (u64)tt << a.logN;
    } else {
      tq[i][0] = a.pc[t].q;
      tq[i][1] = a.pc[t].qinv_neg;
      tq[i][2] = a.md_q[(std::size_t)t * 4];
      tq[i][3] = a.md_q[(std::size_t)t * 4 + 1];
      toff[i] = (u64)t << a.logN;
    }
  }
  if (tid < nin) {
    if (MODE == 0) {
      const u64* h = a.qhinv + ((std::size_t)tab * kMaxAlpha + tid) * 2;
      yin[tid][0] = h[0];
      yin[tid][1] = h[1];
      yin[tid][2] = a.pc[lo + tid].q;
      yin[tid][3] = 0;
    } else {
      const u64* c = a.md_pk + (std::size_t)tid * 4;
      yin[tid][0] = c[0];
      yin[tid][1] = c[1];
      yin[tid][2] = a.pc[tid < a.s_ell ? a.sp0 + tid : a.L + (tid - a.s_ell)].q;
      yin[tid][3] = c[2];
      ypinv[tid] = a.md_pinv[tid];
    }
  }
  __syncthreads();
  // byte-expanded B, written in smem order (conflict-free):
  // slot z = ((rowgroup * KC + chunk) * 8 + r) * 2 + kb, row = (t, s), k = 2 chunk + kb
  for (int z = tid; z < Tp * 16 * KINP; z += blockDim.x) {
    const int kb = z & 1, r = (z >> 1) & 7, chunk = (z >> 4) % KC, rg = (z >> 4) / KC;
    const int br = rg * 8 + r, t = br >> 4, s = br & 15, k = chunk * 2 + kb;
    const u64 cv = (t < T && k < KIN) ? cst[t * KIN + k] : 0;  // t local here
    const u64 rv = ((u64)__byte_perm((uint32_t)cv, 0, 0x0123) << 32) | __byte_perm((uint32_t)(cv >> 32), 0, 0x0123);
    ((u64*)B)[z] = s <= 7 ? (rv >> (8 * (7 - s))) : (s < 15 ? (rv << (8 * (s - 7))) : 0);
  }
  if (warp == kTcMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], 8);
      mbar_init(&afree[b], 1);
      mbar_init(&afull[b], 4);
      mbar_init(&ufree[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(16 * kTcTargets >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int tiles_per_poly = (int)(N / 128);
  const int tiles = tiles_per_poly * a.in.n;
  const int nch = (T + kTcTargets - 1) / kTcTargets;

  if (warp >= 8 && warp < kTcMmaWarp) {
    // ---- loaders: warp 8 + i fills rows 32 i .. 32 i + 31, one row per lane;
    // lane k < nin prefetches its limb's 256-byte slice of the tile two ahead into L2
    const int r = (warp - 8) * 32 + lane;
    const int xoff = MODE == 0 ? lo : 0;
    auto slice = [&](int g, int k) {
      return a.in.p[g / tiles_per_poly] + (std::size_t)(xoff + k) * N + (std::size_t)(g % tiles_per_poly) * 128 +
             (warp - 8) * 32;
    };
    if (lane < nin)
      for (int d = 0; d < 2; ++d) {
        const int g = bx + d * gx;
        if (g < tiles) asm volatile("cp.async.bulk.prefetch.L2.global [%0], 256;" ::"l"(slice(g, lane)) : "memory");
      }
    int tl = 0;
    for (int g = bx; g < tiles; g += gx, ++tl) {
      const int ab = tl & 1;
      const int gp = g + 2 * gx;
      if (lane < nin && gp < tiles)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], 256;" ::"l"(slice(gp, lane)) : "memory");
      u64 xr[KINP];
      {
        const u64* x = slice(g, 0) + lane;
#pragma unroll
        for (int k = 0; k < KINP; ++k) xr[k] = k < nin ? x[(std::size_t)k * N] : 0;
      }
      double v = 0.0;  // y_k computed in place of the inputs
#pragma unroll
      for (int k = 0; k < KINP; ++k) {
        if (k < nin) {
          const u64 q = yin[k][2];
          if (MODE == 0) {
            xr[k] = shoup_mul(xr[k], yin[k][0], yin[k][1], q);
          } else {
            xr[k] = shoup_mul(add_mod(xr[k], yin[k][3], q), yin[k][0], yin[k][1], q);
            v = __dadd_rn(v, __dmul_rn(__ull2double_rn(xr[k]), ypinv[k]));
          }
        } else if (MODE == 1 && k == KINP - 2) {
          xr[k] = (u64)v;  // every input precedes it, so v is complete
        } else {
          xr[k] = (MODE == 1 && k == KINP - 1) ? 1 : 0;
        }
      }
      mbar_wait(&afree[ab], ((tl >> 1) & 1) ^ 1);
      if (MODE == 2) {
        mbar_wait(&ufree[ab], ((tl >> 1) & 1) ^ 1);
        urow[ab][r] = (u64)v;
      }
      unsigned char* Ab = A + ab * ABYTES;
#pragma unroll
      for (int cc = 0; cc < KC; ++cc)
        *(ulonglong2*)(Ab + (r >> 3) * SBO + cc * 128 + (r & 7) * 16) = make_ulonglong2(xr[2 * cc], xr[2 * cc + 1]);
      asm volatile("fence.proxy.async.shared::cta;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ab]);
    }
  } else if (warp == kTcMmaWarp) {
    // ---- MMA issuer
    int use = 0, tl = 0;
    for (int g = bx; g < tiles; g += gx, ++tl) {
      const int ab = tl & 1;
      const uint32_t abase = smem_u32(A + ab * ABYTES);
      if (lane == 0) {
        mbar_wait(&afull[ab], (tl >> 1) & 1);
        for (int ch = 0; ch < nch; ++ch, ++use) {
          const int b = use & 1;
          mbar_wait(&empty[b], ((use >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
          for (int j = 0; j < KINP / 4; ++j) {
            const u64 ad = tc_desc(abase + j * 256, 128, SBO);
            const u64 bd = tc_desc(smem_u32(B) + (ch * kTcTargets * 2) * SBO + j * 256, 128, SBO);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + b * 128),
                "l"(ad), "l"(bd), "r"(idesc), "r"(j));
          }
          mma_commit(&full[b]);
        }
        mma_commit(&afree[ab]);
      }
      __syncwarp();
    }
  } else {
    // ---- epilogue
    const int par = warp >> 2;
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lanebase = (uint32_t)((warp & 3) * 32) << 16;
    int use = 0, tl = 0;
    for (int g = bx; g < tiles; g += gx, ++tl) {
      const int z = g / tiles_per_poly;
      const std::size_t n = (std::size_t)(g % tiles_per_poly) * 128 + row;
      u64* out = a.out.p[z] + (MODE == 0 ? (std::size_t)jd * E * N : 0);
      u64 u = 0;
      if (MODE == 2) {  // the tile's overflow estimates: read, then release the slot
        mbar_wait(&afull[tl & 1], (tl >> 1) & 1);
        u = urow[tl & 1][row];
        __syncwarp();
        if (lane == 0) mbar_arrive(&ufree[tl & 1]);
      }
      for (int ch = 0; ch < nch; ++ch, ++use) {
        const int b = use & 1;
        mbar_wait(&full[b], (use >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int t0 = ch * kTcTargets;
        const int nt = min(kTcTargets, T - t0);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t d[2][16];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int tt = par + 2 * (2 * h + i);
            if (tt < nt) tmem_ld16(tm + b * 128 + lanebase + tt * 16, d[i]);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          if (h == 1) {
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[b]);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int tt = par + 2 * (2 * h + i);
            if (tt < nt) {
              const int t = t0 + tt;
              u64 hi, lo;
              recombine(d[i], a.m16, hi, lo);
              const u64 q = tq[t][0], qn = tq[t][1];
              u64 r = redc(hi, lo, q, qn);
              if (MODE == 2) {
                r = sub_mod(r, redc(mulhi(u, tq[t][2]), u * tq[t][2], q, qn), q);
                r = sub_mod(r, tq[t][3], q);
              }
              out[toff[t] + n] = r;
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kTcMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

template <int KINP, int MODE>
void launch_tc(const TcBconvArgs& a, std::size_t N, cudaStream_t st, int grid_override = 0) {
  const int Tp = (a.T + kTcTargets - 1) / kTcTargets * kTcTargets;
  const std::size_t smem = (std::size_t)2 * 128 * KINP * 8 + (std::size_t)Tp * 16 * KINP * 8;
  static int configured = 0;
  if (!configured) {
    cudaFuncSetAttribute(k_bconv_tc<KINP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = 1;
  }
  const int tiles = (int)(N / 128) * a.in.n;
  const int grid = grid_override > 0 ? grid_override : std::min(tiles, 2 * sm_count());
  k_bconv_tc<KINP, MODE><<<grid, kTcThreads, smem, st>>>(a);
}

template <int MODE>
void dispatch_tc(TcBconvArgs a, std::size_t N, cudaStream_t st) {
  if (a.kin > 16 || a.kin < 1) throw std::runtime_error("bconv_tc: digit size out of range");
  const int total = a.T;
  for (int tb = 0; tb < total; tb += kTcMaxT) {
    a.tb = tb;
    a.T = std::min(kTcMaxT, total - tb);
    if (a.kin <= 4) launch_tc<4, MODE>(a, N, st);
    else if (a.kin <= 8) launch_tc<8, MODE>(a, N, st);
    else if (a.kin <= 12) launch_tc<12, MODE>(a, N, st);
    else launch_tc<16, MODE>(a, N, st);
  }
}

}  // namespace

bool bconv_tc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FHEON_BCONV_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool modup_bconv_tc_all(const DevTables& t, const PolyList& ext, const PolyList& x, int limbs, cudaStream_t st) {
  const int beta = t.dig.beta(limbs);
  if (beta < 2) return false;
  TcBconvArgs a{};
  a.m16 = 1u << 16;
  a.in = x;
  a.out = ext;
  a.pc = t.pc;
  a.qhinv = t.modup_qhinv;
  a.qhat = t.modup_qhat;
  a.logN = t.logN;
  a.limbs = limbs;
  a.L = t.L;
  a.K = t.K;
  a.ndig = beta;
  int kmax = 0, tmax = 0;
  for (int j = 0; j < beta; ++j) {
    a.dlo[j] = t.dig.lo(j);
    a.dkin[j] = t.dig.hi(j, limbs) - a.dlo[j];
    a.dT[j] = limbs + t.K - a.dkin[j];
    a.dj[j] = j;
    a.dtab[j] = (limbs - 1) * t.dnum + j;
    kmax = std::max(kmax, a.dkin[j]);
    tmax = std::max(tmax, a.dT[j]);
  }
  if (tmax > kTcMaxT || kmax > 16) return false;
  // the widest digit's targets size the shared B (the others use a prefix)
  a.kin = a.nin = kmax;
  a.T = tmax;
  const int tiles = (int)(t.N / 128) * x.n;
  const int per = std::max(1, std::min(tiles, 2 * sm_count() / beta));
  for (int j = 0; j <= beta; ++j) a.cta0[j] = j * per;
  const std::size_t N = t.N;
  if (kmax <= 4) launch_tc<4, 0>(a, N, st, beta * per);
  else if (kmax <= 8) launch_tc<8, 0>(a, N, st, beta * per);
  else if (kmax <= 12) launch_tc<12, 0>(a, N, st, beta * per);
  else launch_tc<16, 0>(a, N, st, beta * per);
  return true;
}

void modup_bconv_tc(const DevTables& t, const PolyList& ext, const PolyList& x, int limbs, int j, cudaStream_t st) {
  TcBconvArgs a{};
  a.m16 = 1u << 16;
  a.in = x;
  a.out = ext;
  a.pc = t.pc;
  a.qhinv = t.modup_qhinv;
  a.qhat = t.modup_qhat;
  a.logN = t.logN;
  a.limbs = limbs;
  a.L = t.L;
  a.K = t.K;
  a.lo = t.dig.lo(j);
  a.kin = a.nin = t.dig.hi(j, limbs) - a.lo;
  a.T = limbs + t.K - a.kin;
  a.j = j;
  a.tab = (limbs - 1) * t.dnum + j;
  dispatch_tc<0>(a, t.N, st);
}

void moddown_fused_conv_tc(const DevTables& t, const PolyList& conv, const PolyList& z, int limbs, cudaStream_t st) {
  const int l = limbs - 1;
  TcBconvArgs a{};
  a.m16 = 1u << 16;
  a.in = z;
  a.out = conv;
  a.pc = t.pc;
  a.md_pk = t.md2_pk + (std::size_t)l * kMaxK * 4;
  a.md_pinv = t.md2_pinv + (std::size_t)l * kMaxK;
  a.md_phat = t.md2_phat + (std::size_t)l * t.L * kMaxK;
  a.md_q = t.md2_q + (std::size_t)l * t.L * 4;
  a.logN = t.logN;
  a.limbs = l;
  a.L = t.L;
  a.K = t.K;
  a.nin = t.K + 1;
  a.T = l;
  a.s_ell = 1;
  a.sp0 = l;
  if (a.nin + 2 <= 16) {
    a.kin = (a.nin + 2 + 3) / 4 * 4;
    dispatch_tc<1>(a, t.N, st);
  } else {
    a.kin = a.nin;
    dispatch_tc<2>(a, t.N, st);
  }
}

void moddown_conv_tc(const DevTables& t, const PolyList& conv, const PolyList& z, int limbs, cudaStream_t st) {
  TcBconvArgs a{};
  a.m16 = 1u << 16;
  a.in = z;
  a.out = conv;
  a.pc = t.pc;
  a.md_pk = t.md_pk;
  a.md_pinv = t.md_pinv;
  a.md_phat = t.md_phat;
  a.md_q = t.md_q;
  a.logN = t.logN;
  a.limbs = limbs;
  a.L = t.L;
  a.K = t.K;
  a.nin = t.K;
  a.T = limbs;
  if (t.K + 2 <= 16) {
    a.kin = (t.K + 2 + 3) / 4 * 4;  // = KINP: u and 1 sit in the last two columns
    dispatch_tc<1>(a, t.N, st);
  } else {
    a.kin = t.K;
    dispatch_tc<2>(a, t.N, st);
  }
}

}  // namespace fheon
