// Elementwise RNS kernels, automorphism, hybrid key-switching pieces
// (ModUp basis conversion, key inner product, ModDown), rescale, and the
// encrypt / keygen / decrypt helpers.  Definitions: DESIGN.md section 3
// (mirrored by oracle/ckks_oracle.c, which these must match bit for bit).
#include <algorithm>
#include <stdexcept>

#include "kernels.hpp"

namespace fheon {

namespace {

constexpr int kThreads = 256;

inline dim3 grid_for(std::size_t N, int y, int z = 1) {
  return dim3((unsigned)(N / kThreads), (unsigned)y, (unsigned)z);
}

// ------------------------------------------------------------ elementwise
__global__ void k_add(PolyList out, PolyList a, PolyList b, const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const u64 q = pc[blockIdx.y].q;
  out.p[blockIdx.z][o] = add_mod(a.p[blockIdx.z][o], b.p[blockIdx.z][o], q);
}
__global__ void k_sub(PolyList out, PolyList a, PolyList b, const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const u64 q = pc[blockIdx.y].q;
  out.p[blockIdx.z][o] = sub_mod(a.p[blockIdx.z][o], b.p[blockIdx.z][o], q);
}
__global__ void k_neg(PolyList out, PolyList a, const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const u64 q = pc[blockIdx.y].q;
  const u64 v = a.p[blockIdx.z][o];
  out.p[blockIdx.z][o] = v ? q - v : 0;
}
__global__ void k_mul_pt(PolyList out, PolyList a, const u64* __restrict__ pt, const PrimeConst* __restrict__ pc,
                         int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst P = pc[blockIdx.y];
  out.p[blockIdx.z][o] = mul_mod(a.p[blockIdx.z][o], pt[o], P);
}
__global__ void k_mul_const(PolyList out, PolyList a, LimbConsts c, const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const u64 q = pc[blockIdx.y].q;
  out.p[blockIdx.z][o] = shoup_mul(a.p[blockIdx.z][o], c.c[blockIdx.y], c.sh[blockIdx.y], q);
}
__global__ void k_add_const(PolyList out, PolyList a, LimbConsts c, const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const u64 q = pc[blockIdx.y].q;
  out.p[blockIdx.z][o] = add_mod(a.p[blockIdx.z][o], c.c[blockIdx.y], q);
}
// Two-coefficient (16-byte) variants of the elementwise kernels, used when every
// pointer of the launch is 16-byte aligned (always, for ciphertext and key
// buffers; checked per launch): grid (N/512, limbs, npolys)
template <int OP>  // 0 add, 1 sub, 2 add_const, 3 mul_const
__global__ void k_ew2(PolyList out, PolyList a, PolyList b, LimbConsts c, const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const u64 q = pc[blockIdx.y].q;
  const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(a.p[blockIdx.z] + o);
  ulonglong2 r;
  if constexpr (OP == 0 || OP == 1) {
    const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(b.p[blockIdx.z] + o);
    r = OP == 0 ? make_ulonglong2(add_mod(x.x, y.x, q), add_mod(x.y, y.y, q))
                : make_ulonglong2(sub_mod(x.x, y.x, q), sub_mod(x.y, y.y, q));
  } else if constexpr (OP == 2) {
    const u64 k = c.c[blockIdx.y];
    r = make_ulonglong2(add_mod(x.x, k, q), add_mod(x.y, k, q));
  } else {
    const u64 k = c.c[blockIdx.y], ks = c.sh[blockIdx.y];
    r = make_ulonglong2(shoup_mul(x.x, k, ks, q), shoup_mul(x.y, k, ks, q));
  }
  *reinterpret_cast<ulonglong2*>(out.p[blockIdx.z] + o) = r;
}
bool aligned16(const PolyList& l) {
  for (int i = 0; i < l.n; ++i)
    if (reinterpret_cast<std::uintptr_t>(l.p[i]) & 15u) return false;
  return true;
}

// grid (N/256, limbs, 2 polys)
__global__ void k_lincomb_const(u64* out0, u64* out1, LincombTerms terms, const u64* __restrict__ kc,
                                const PrimeConst* __restrict__ pc, int logN, int limbs) {
  // two adjacent coefficients per thread (16-byte loads / stores)
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int t = blockIdx.y;
  const u64 q = pc[t].q;
  u64 s0 = 0, s1 = 0;
  for (int i = 0; i < terms.n; ++i) {
    const u64* x = terms.c0[i] + (blockIdx.z ? terms.c1_off[i] : 0);
    const u64* k = kc + ((std::size_t)i * limbs + t) * 2;
    const u64 kv = k[0], ksh = k[1];
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(x + o);
    s0 = add_mod(s0, shoup_mul(v.x, kv, ksh, q), q);
    s1 = add_mod(s1, shoup_mul(v.y, kv, ksh, q), q);
  }
  *reinterpret_cast<ulonglong2*>((blockIdx.z ? out1 : out0) + o) = make_ulonglong2(s0, s1);
}

// grid (N/256, npolys): acc[n] += x[n] * c (Montgomery constant) on one limb
__global__ void k_axpy_limb(PolyList acc, PolyList x, u64 c, const PrimeConst* __restrict__ pc, int prime) {
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst P = pc[prime];
  u64* a = acc.p[blockIdx.y];
  a[n] = add_mod(a[n], mont_mul(x.p[blockIdx.y][n], c, P), P.q);
}

__global__ void k_tensor(u64* d0, u64* d1, u64* d2, const u64* a0, const u64* a1, const u64* b0, const u64* b1,
                         const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst P = pc[blockIdx.y];
  const u64 x0 = a0[o], x1 = a1[o], y0 = b0[o], y1 = b1[o];
  d0[o] = mul_mod(x0, y0, P);
  // the cross term's two products (< 2 q^2 < q 2^64) share one REDC + conversion
  Acc128 c;
  c.mac(x0, y1);
  c.mac(x1, y0);
  const u64 tm = redc(c.hi, c.lo, P.q, P.qinv_neg);
  d1[o] = redc(mulhi(tm, P.r2), tm * P.r2, P.q, P.qinv_neg);
  d2[o] = mul_mod(x1, y1, P);
}
// Chebyshev step 2 a (x) b - k s before the relinearise-and-rescale: d = 2 (a (x) b)
// on all three parts, minus k s on d0 / d1 (s: the step's subtrahend T_{a-b} viewed
// at these limbs, k ~ scale(a) scale(b) / scale(s) so it lands on the product's scale)
__global__ void k_tensor_cheb(u64* d0, u64* d1, u64* d2, const u64* a0, const u64* a1, const u64* b0, const u64* b1,
                              const u64* s0, const u64* s1, LimbConsts kc, const PrimeConst* __restrict__ pc,
                              int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst P = pc[blockIdx.y];
  const u64 x0 = a0[o], x1 = a1[o], y0 = b0[o], y1 = b1[o];
  u64 t0 = mul_mod(x0, y0, P);
  Acc128 c;
  c.mac(x0, y1);
  c.mac(x1, y0);
  const u64 tm = redc(c.hi, c.lo, P.q, P.qinv_neg);
  u64 t1 = redc(mulhi(tm, P.r2), tm * P.r2, P.q, P.qinv_neg);
  const u64 t2 = mul_mod(x1, y1, P);
  t0 = add_mod(t0, t0, P.q);
  t1 = add_mod(t1, t1, P.q);
  if (s0 != nullptr) {
    const u64 k = kc.c[blockIdx.y], ksh = kc.sh[blockIdx.y];
    t0 = sub_mod(t0, shoup_mul(s0[o], k, ksh, P.q), P.q);
    t1 = sub_mod(t1, shoup_mul(s1[o], k, ksh, P.q), P.q);
  }
  d0[o] = t0;
  d1[o] = t1;
  d2[o] = add_mod(t2, t2, P.q);
}
__global__ void k_automorph(PolyList out, PolyList in, int logN) {
  const unsigned n = blockIdx.x * blockDim.x + threadIdx.x;
  const std::size_t base = (std::size_t)blockIdx.y << logN;
  const u64 g = out.g[blockIdx.z];
  out.p[blockIdx.z][base + n] = in.p[blockIdx.z][base + auto_src(n, g, logN)];
}

// ------------------------------------------------------------ key switching
// ModUp basis conversion for one digit j with A = |D_j| limbs (compile time).
// grid (N/256, ceil((E - A) / kTC), npolys): each CTA converts a chunk of kTC
// target limbs; the chunk's constants [Q_j/q_i]_t (Montgomery) sit in smem.
constexpr int kTC = 8;
template <int A>
__global__ void __launch_bounds__(256) k_modup_bconv(PolyList ext, PolyList x, const PrimeConst* __restrict__ pc,
                                                     const u64* __restrict__ qhinv, const u64* __restrict__ qhat,
                                                     int logN, int limbs, int L, int K, int dnum, int lo, int j) {
  __shared__ u64 cs[kTC][A];
  __shared__ u64 tq[kTC][2];
  __shared__ int tdst[kTC];
  const std::size_t N = (std::size_t)1 << logN;
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const int E = limbs + K;
  const int tab = (limbs - 1) * dnum + j;
  const int nt = min(kTC, E - A - (int)blockIdx.y * kTC);
  if (threadIdx.x < kTC * A) {
    const int c = threadIdx.x / A, i = threadIdx.x % A;
    if (c < nt) {
      const int tt = blockIdx.y * kTC + c;
      const int t = tt < lo ? tt : tt + A;
      const int pt = t < limbs ? t : L + (t - limbs);
      cs[c][i] = qhat[((std::size_t)tab * (L + K) + pt) * kMaxAlpha + i];
      if (i == 0) {
        tq[c][0] = pc[pt].q;
        tq[c][1] = pc[pt].qinv_neg;
        tdst[c] = t;
      }
    }
  }
  __syncthreads();
  const u64* xin = x.p[blockIdx.z];
  u64* out = ext.p[blockIdx.z] + (std::size_t)j * E * N;
  u64 y[A];
#pragma unroll
  for (int i = 0; i < A; ++i) {
    const u64* h = qhinv + ((std::size_t)tab * kMaxAlpha + i) * 2;
    y[i] = shoup_mul(xin[(std::size_t)(lo + i) * N + n], __ldg(h), __ldg(h + 1), pc[lo + i].q);
  }
  for (int c = 0; c < nt; ++c) {
    Acc128 acc;
#pragma unroll
    for (int i = 0; i < A; ++i) acc.mac(y[i], cs[c][i]);
    out[(std::size_t)tdst[c] * N + n] = redc(acc.hi, acc.lo, tq[c][0], tq[c][1]);
  }
}

// grid (jobs, N/256, E): the job index varies fastest, so CTAs of jobs that share
// a key (same-key batches) run together and reuse its slices from L2
__global__ void k_ks_inner(KsJobs jobs, const PrimeConst* __restrict__ pc, int logN, int limbs, int L, int K,
                           DigitOwner dig) {
  // two adjacent coefficients per thread: 16-byte key and accumulator accesses,
  // per-CTA setup amortised (as k_ks_inner_sum); same products per coefficient
  const std::size_t N = (std::size_t)1 << logN;
  const unsigned n = 2 * (blockIdx.y * blockDim.x + threadIdx.x);
  const int t = blockIdx.z;
  const int r = blockIdx.x;
  const int E = limbs + K;
  const int pt = t < limbs ? t : L + (t - limbs);
  const PrimeConst P = pc[pt];
  const u64 g = jobs.g[r];
  const unsigned src0 = (g == 1) ? n : auto_src(n, g, logN);
  const unsigned src1 = (g == 1) ? n + 1 : auto_src(n + 1, g, logN);
  const int beta = dig.beta;
  const int jown = t < limbs ? (int)__ldg(dig.owner + t) : -1;  // CTA-uniform: limb t's own digit passes d through
  FHEON_DCHECK(r < jobs.n && t < E && beta >= 1 && beta <= kMaxDigits && jown < beta && n + 1 < N);
  const u64* key = jobs.key[r];
  const u64* ext = jobs.ext[r];
  const u64* d = jobs.d[r];
  const std::size_t LKN = (std::size_t)(L + K) * N;
  Acc128 a0[2], a1[2];
  for (int j = 0; j < beta; ++j) {
    const u64* vb = j == jown ? d + (std::size_t)t * N : ext + ((std::size_t)j * E + t) * N;
    const u64* kj = key + ((std::size_t)(j * 2) * (L + K) + pt) * N;
    const ulonglong2 kb = *reinterpret_cast<const ulonglong2*>(kj + n);
    const ulonglong2 ka = *reinterpret_cast<const ulonglong2*>(kj + LKN + n);
    const u64 v0 = vb[src0], v1 = vb[src1];
    a0[0].mac(v0, kb.x);
    a1[0].mac(v0, ka.x);
    a0[1].mac(v1, kb.y);
    a1[1].mac(v1, ka.y);
  }
  u64* acc = jobs.acc[r];
  *reinterpret_cast<ulonglong2*>(acc + (std::size_t)t * N + n) =
      make_ulonglong2(redc(a0[0].hi, a0[0].lo, P.q, P.qinv_neg), redc(a0[1].hi, a0[1].lo, P.q, P.qinv_neg));
  *reinterpret_cast<ulonglong2*>(acc + ((std::size_t)E + t) * N + n) =
      make_ulonglong2(redc(a1[0].hi, a1[0].lo, P.q, P.qinv_neg), redc(a1[1].hi, a1[1].lo, P.q, P.qinv_neg));
}

// Lazy reduction across jobs: every product is < q^2 (canonical digit x
// Montgomery key), so up to 32 of them stay below 32 q^2 < 2^125; REDC of
// such a sum is < S / 2^64 + q < 3q (q < 2^60) and two conditional
// subtractions make it canonical -- the same residue as one REDC per job.
__device__ __forceinline__ int lazy_chunk(int beta) { return max(1, 32 / (beta + 1)); }
__device__ __forceinline__ void lazy_flush(u64& s0, u64& s1, Acc128& a0, Acc128& a1, const PrimeConst& P) {
  const u64 m0 = a0.lo * P.qinv_neg, m1 = a1.lo * P.qinv_neg;
  const u64 t0 = a0.hi + mulhi(m0, P.q) + (a0.lo != 0 ? 1ULL : 0ULL);
  const u64 t1 = a1.hi + mulhi(m1, P.q) + (a1.lo != 0 ? 1ULL : 0ULL);
  s0 = add_mod(s0, csub(csub(t0, P.q), P.q), P.q);
  s1 = add_mod(s1, csub(csub(t1, P.q), P.q), P.q);
  a0 = Acc128{};
  a1 = Acc128{};
}

// grid (N/256, E, groups): rotate-and-sum accumulation (kernels.hpp KsSumJobs).
// Each job's digit sum (<= beta + 1 products < q^2) is REDC'd on its own so the
// 128-bit accumulator never exceeds q * 2^64; job results add mod q.
__global__ void k_ks_inner_sum(KsSumJobs jobs, const PrimeConst* __restrict__ pc, const u64* __restrict__ md_q,
                               int logN, int limbs, int L, int K, DigitOwner dig) {
  // grid (groups, N/512, E): groups vary fastest -- the groups of a hoisted stage
  // use the same key list, so their CTAs share each key slice through L2.  Two
  // adjacent coefficients per thread: the per-job and per-CTA setup (constants,
  // job pointers, digit owner) is amortised over both, key words and the
  // accumulator move as 16-byte pairs; same products, same order per coefficient.
  const std::size_t N = (std::size_t)1 << logN;
  const unsigned n = 2 * (blockIdx.y * blockDim.x + threadIdx.x);
  const int t = blockIdx.z;
  const int r = blockIdx.x;
  const int E = limbs + K;
  const int pt = t < limbs ? t : L + (t - limbs);
  const PrimeConst P = pc[pt];
  const int beta = dig.beta;
  const int jown = t < limbs ? (int)__ldg(dig.owner + t) : -1;
  const u64 pm = t < limbs ? md_q[(std::size_t)t * 4] : 0;  // P mod q_t, Montgomery form
  const std::size_t LKN = (std::size_t)(L + K) * N;
  FHEON_DCHECK(r < jobs.ngroups && r < kMaxSumGroups && t < E && beta >= 1 && beta <= kMaxDigits && jown < beta &&
               n + 1 < N && jobs.begin[r] >= 0 && jobs.begin[r + 1] <= kMaxSumJobs &&
               jobs.begin[r] <= jobs.begin[r + 1]);
  u64 s0[2] = {0, 0}, s1[2] = {0, 0};
  const int chunk = lazy_chunk(beta);
  Acc128 a0[2], a1[2];
  int cnt = 0;
  for (int jb = jobs.begin[r]; jb < jobs.begin[r + 1]; ++jb) {
    const u64 g = jobs.g[jb];
    unsigned src[2];
    src[0] = (g == 1) ? n : auto_src(n, g, logN);
    src[1] = (g == 1) ? n + 1 : auto_src(n + 1, g, logN);
    const u64* key = jobs.key[jb];
    const u64* ext = jobs.ext[jb];
    const u64* d = jobs.d[jb];
    if (jobs.c0_qp) {  // CTA-uniform
      const u64* c0 = jobs.c0[jb] + (std::size_t)t * N;
      s0[0] = add_mod(s0[0], c0[src[0]], P.q);
      s0[1] = add_mod(s0[1], c0[src[1]], P.q);
      if (jobs.direct[jb]) {
        const u64* c1 = d + (std::size_t)t * N;
        s1[0] = add_mod(s1[0], c1[src[0]], P.q);
        s1[1] = add_mod(s1[1], c1[src[1]], P.q);
        continue;
      }
    }
    for (int j = 0; j < beta; ++j) {
      const u64* vb = j == jown ? d + (std::size_t)t * N : ext + ((std::size_t)j * E + t) * N;
      const u64* kj = key + ((std::size_t)(j * 2) * (L + K) + pt) * N;
      const ulonglong2 kb = *reinterpret_cast<const ulonglong2*>(kj + n);
      const ulonglong2 ka = *reinterpret_cast<const ulonglong2*>(kj + LKN + n);
      const u64 v0 = vb[src[0]], v1 = vb[src[1]];
      a0[0].mac(v0, kb.x);
      a1[0].mac(v0, ka.x);
      a0[1].mac(v1, kb.y);
      a1[1].mac(v1, ka.y);
    }
    if (t < limbs && !jobs.c0_qp) {
      const u64* c0 = jobs.c0[jb] + (std::size_t)t * N;
      a0[0].mac(c0[src[0]], pm);
      a0[1].mac(c0[src[1]], pm);
    }
    if (++cnt == chunk) {
      lazy_flush(s0[0], s1[0], a0[0], a1[0], P);
      lazy_flush(s0[1], s1[1], a0[1], a1[1], P);
      cnt = 0;
    }
  }
  if (cnt) {
    lazy_flush(s0[0], s1[0], a0[0], a1[0], P);
    lazy_flush(s0[1], s1[1], a0[1], a1[1], P);
  }
  u64* acc = jobs.acc[r];
  *reinterpret_cast<ulonglong2*>(acc + (std::size_t)t * N + n) = make_ulonglong2(s0[0], s0[1]);
  *reinterpret_cast<ulonglong2*>(acc + ((std::size_t)E + t) * N + n) = make_ulonglong2(s1[0], s1[1]);
}

// grid (groups, N/256, E): groups fastest (every group uses the same keys)
__global__ void k_ks_inner_shared(KsSharedJobs jobs, const PrimeConst* __restrict__ pc,
                                  const u64* __restrict__ md_q, int logN, int limbs, int L, int K, DigitOwner dig) {
  // two adjacent coefficients per thread (as k_ks_inner_sum)
  const std::size_t N = (std::size_t)1 << logN;
  const unsigned n = 2 * (blockIdx.y * blockDim.x + threadIdx.x);
  const int t = blockIdx.z;
  const int r = blockIdx.x;
  const int E = limbs + K;
  const int pt = t < limbs ? t : L + (t - limbs);
  const PrimeConst P = pc[pt];
  const int beta = dig.beta;
  const int jown = t < limbs ? (int)__ldg(dig.owner + t) : -1;
  const u64 pm = t < limbs ? md_q[(std::size_t)t * 4] : 0;
  const u64* ext = jobs.ext[r];
  const u64* d = jobs.d[r];
  const u64* c0 = jobs.c0[r] + (std::size_t)t * N;
  const std::size_t LKN = (std::size_t)(L + K) * N;
  u64 s0[2] = {0, 0}, s1[2] = {0, 0};
  const int chunk = lazy_chunk(beta);
  Acc128 a0[2], a1[2];
  int cnt = 0;
  for (int jb = 0; jb < jobs.nkeys; ++jb) {
    const u64 g = jobs.g[jb];
    const unsigned src0 = (g == 1) ? n : auto_src(n, g, logN);
    const unsigned src1 = (g == 1) ? n + 1 : auto_src(n + 1, g, logN);
    const u64* key = jobs.key[jb];
    for (int j = 0; j < beta; ++j) {
      const u64* vb = j == jown ? d + (std::size_t)t * N : ext + ((std::size_t)j * E + t) * N;
      const u64* kj = key + ((std::size_t)(j * 2) * (L + K) + pt) * N;
      const ulonglong2 kb = *reinterpret_cast<const ulonglong2*>(kj + n);
      const ulonglong2 ka = *reinterpret_cast<const ulonglong2*>(kj + LKN + n);
      const u64 v0 = vb[src0], v1 = vb[src1];
      a0[0].mac(v0, kb.x);
      a1[0].mac(v0, ka.x);
      a0[1].mac(v1, kb.y);
      a1[1].mac(v1, ka.y);
    }
    if (t < limbs) {
      a0[0].mac(c0[src0], pm);
      a0[1].mac(c0[src1], pm);
    }
    if (++cnt == chunk) {
      lazy_flush(s0[0], s1[0], a0[0], a1[0], P);
      lazy_flush(s0[1], s1[1], a0[1], a1[1], P);
      cnt = 0;
    }
  }
  if (cnt) {
    lazy_flush(s0[0], s1[0], a0[0], a1[0], P);
    lazy_flush(s0[1], s1[1], a0[1], a1[1], P);
  }
  u64* acc = jobs.acc[r];
  *reinterpret_cast<ulonglong2*>(acc + (std::size_t)t * N + n) = make_ulonglong2(s0[0], s0[1]);
  *reinterpret_cast<ulonglong2*>(acc + ((std::size_t)E + t) * N + n) = make_ulonglong2(s1[0], s1[1]);
}

// ModDown conversion with KK = K special limbs (compile time).
// grid (N/256, ceil(limbs / kTC), npolys); the chunk's constants sit in smem.
template <int KK>
__global__ void __launch_bounds__(256) k_moddown_conv(PolyList conv, PolyList z, const PrimeConst* __restrict__ pc,
                                                      const u64* __restrict__ md_pk, const double* __restrict__ md_pinv,
                                                      const u64* __restrict__ md_phat, const u64* __restrict__ md_q,
                                                      int logN, int limbs, int L) {
  __shared__ u64 cs[kTC][KK];
  __shared__ u64 tq[kTC][4];  // q, qinv_neg, P mod q (Montgomery), (P-1)/2 mod q
  const std::size_t N = (std::size_t)1 << logN;
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const int i0 = blockIdx.y * kTC;
  const int nt = min(kTC, limbs - i0);
  if (threadIdx.x < kTC * KK) {
    const int c = threadIdx.x / KK, k = threadIdx.x % KK;
    if (c < nt) {
      cs[c][k] = md_phat[(std::size_t)(i0 + c) * kMaxK + k];
      if (k == 0) {
        tq[c][0] = pc[i0 + c].q;
        tq[c][1] = pc[i0 + c].qinv_neg;
        tq[c][2] = md_q[(std::size_t)(i0 + c) * 4];
        tq[c][3] = md_q[(std::size_t)(i0 + c) * 4 + 1];
      }
    }
  }
  __syncthreads();
  const u64* zp = z.p[blockIdx.z];
  u64 y[KK];
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < KK; ++k) {
    const u64 pk = pc[L + k].q;
    const u64* c = md_pk + (std::size_t)k * 4;
    y[k] = shoup_mul(add_mod(zp[(std::size_t)k * N + n], __ldg(c + 2), pk), __ldg(c), __ldg(c + 1), pk);
    v = __dadd_rn(v, __dmul_rn(__ull2double_rn(y[k]), md_pinv[k]));
  }
  const u64 u = (u64)v;
  u64* out = conv.p[blockIdx.z];
  for (int c = 0; c < nt; ++c) {
    const u64 q = tq[c][0], qn = tq[c][1];
    Acc128 acc;
#pragma unroll
    for (int k = 0; k < KK; ++k) acc.mac(y[k], cs[c][k]);
    u64 x = redc(acc.hi, acc.lo, q, qn);
    x = sub_mod(x, redc(mulhi(u, tq[c][2]), u * tq[c][2], q, qn), q);
    out[(std::size_t)(i0 + c) * N + n] = sub_mod(x, tq[c][3], q);
  }
}

// grid (N/256, npolys)
__global__ void k_rescale_lift(PolyList r, PolyList last, const PrimeConst* __restrict__ pc,
                               const u64* __restrict__ rs, int logN, int limbs, int L) {
  const std::size_t N = (std::size_t)1 << logN;
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = limbs - 1;
  const u64 ql = pc[l].q;
  const u64 v = last.p[blockIdx.z][n];
  const bool neg = v > ql / 2;
  u64* out = r.p[blockIdx.z];
  for (int i = 0; i < l; ++i) {
    const PrimeConst P = pc[i];
    u64 x = reduce64(v, P);
    if (neg) x = sub_mod(x, rs[((std::size_t)l * L + i) * 4 + 2], P.q);
    out[(std::size_t)i * N + n] = x;
  }
}

// ------------------------------------------------------------ fused layer kernels
// grid (N/256, limbs, nout).  Accumulates up to 32 products in 128 bits, folds
// with one REDC into an R^-1-domain sum, and converts back with a final REDC
// by R^2: out = sum_j ct_j (*) pt_j mod q exactly.
// grid (nout, N/256, limbs): outputs fastest, so the CTAs of outputs that share
// their terms (a conv's taps, a BSGS level's baby steps) read each term tile
// from L2 instead of HBM
// limb t < ell uses q_t, limb t >= ell the special prime p_{t - ell} (Q u P operands)
__global__ void k_mac(MacJobs jobs, const PrimeConst* __restrict__ pc, int logN, int ell, int L) {
  // two adjacent coefficients per thread, 16-byte loads and stores
  const std::size_t o = ((std::size_t)blockIdx.z << logN) + 2 * (blockIdx.y * blockDim.x + threadIdx.x);
  const int z = blockIdx.x;
  const int t = (int)blockIdx.z;
  const PrimeConst P = pc[t < ell ? t : L + (t - ell)];
  const int nt = jobs.nterm[z];
  FHEON_DCHECK(z < jobs.nout && z < kMacMaxOut && nt >= 1 && nt <= kMacMaxTerms);
  u64 s0[2] = {0, 0}, s1[2] = {0, 0};
  Acc128 a0[2], a1[2];
  for (int j = 0; j < nt; ++j) {  // nt <= kMacMaxTerms = 32 products < 32 q^2: one lazy flush
    const u64* c = jobs.ct[z][j];
    const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(jobs.pt[z][j] + o);
    const ulonglong2 x0 = *reinterpret_cast<const ulonglong2*>(c + o);
    const ulonglong2 x1 = *reinterpret_cast<const ulonglong2*>(c + jobs.c1_off[z][j] + o);
    a0[0].mac(x0.x, p.x);
    a1[0].mac(x1.x, p.x);
    a0[1].mac(x0.y, p.y);
    a1[1].mac(x1.y, p.y);
    if ((j & 31) == 31 || j == nt - 1) {
      lazy_flush(s0[0], s1[0], a0[0], a1[0], P);
      lazy_flush(s0[1], s1[1], a0[1], a1[1], P);
    }
  }
  *reinterpret_cast<ulonglong2*>(jobs.out0[z] + o) =
      make_ulonglong2(redc(mulhi(s0[0], P.r2), s0[0] * P.r2, P.q, P.qinv_neg),
                      redc(mulhi(s0[1], P.r2), s0[1] * P.r2, P.q, P.qinv_neg));
  *reinterpret_cast<ulonglong2*>(jobs.out1[z] + o) =
      make_ulonglong2(redc(mulhi(s1[0], P.r2), s1[0] * P.r2, P.q, P.qinv_neg),
                      redc(mulhi(s1[1], P.r2), s1[1] * P.r2, P.q, P.qinv_neg));
}

// grid (ngiants * nin, N/512, E): kernels.hpp BsgsMacJobs.  Per output the products and
// their order are k_mac's (bit-identical sums).
__global__ void k_mac_bsgs(BsgsMacJobs jobs, const PrimeConst* __restrict__ pc, int logN, int ell, int L) {
  const std::size_t o = ((std::size_t)blockIdx.z << logN) + 2 * (blockIdx.y * blockDim.x + threadIdx.x);
  const int g = blockIdx.x / jobs.nin;
  const int i = blockIdx.x - g * jobs.nin;
  const int t = (int)blockIdx.z;
  const PrimeConst P = pc[t < ell ? t : L + (t - ell)];
  const int nt = jobs.nterm[g];
  FHEON_DCHECK(g < jobs.ngiants && g < kBsgsMaxGiants && i < kBsgsMaxIn && nt >= 1 && nt <= kMacMaxTerms);
  const u64* babies = jobs.babies[i];
  const u64* ident = jobs.ident[i];
  u64 s0[2] = {0, 0}, s1[2] = {0, 0};
  Acc128 a0[2], a1[2];
  for (int j = 0; j < nt; ++j) {  // nt <= kMacMaxTerms = 32 products < 32 q^2: one lazy flush
    const int b = jobs.bidx[g][j];
    const u64* c = b < 0 ? ident : babies + (long long)b * jobs.baby_stride;
    const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(jobs.pt[g][j] + o);
    const ulonglong2 x0 = *reinterpret_cast<const ulonglong2*>(c + o);
    const ulonglong2 x1 = *reinterpret_cast<const ulonglong2*>(c + jobs.c1_off + o);
    a0[0].mac(x0.x, p.x);
    a1[0].mac(x1.x, p.x);
    a0[1].mac(x0.y, p.y);
    a1[1].mac(x1.y, p.y);
  }
  lazy_flush(s0[0], s1[0], a0[0], a1[0], P);
  lazy_flush(s0[1], s1[1], a0[1], a1[1], P);
  u64* out = jobs.out[i] + (long long)g * jobs.out_stride;
  *reinterpret_cast<ulonglong2*>(out + o) =
      make_ulonglong2(redc(mulhi(s0[0], P.r2), s0[0] * P.r2, P.q, P.qinv_neg),
                      redc(mulhi(s0[1], P.r2), s0[1] * P.r2, P.q, P.qinv_neg));
  *reinterpret_cast<ulonglong2*>(out + jobs.c1_off + o) =
      make_ulonglong2(redc(mulhi(s1[0], P.r2), s1[0] * P.r2, P.q, P.qinv_neg),
                      redc(mulhi(s1[1], P.r2), s1[1] * P.r2, P.q, P.qinv_neg));
}

// grid (N/256, 1)
__global__ void k_encode_lincomb(u64* out, LinComb lc, double scale, const PrimeConst* __restrict__ pc, int logN,
                                 int limbs) {
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  for (int b = 0; b < lc.nb; ++b) v = __dadd_rn(v, __dmul_rn(lc.w[b], lc.basis[b][n]));
  const long long c = __double2ll_rn(__dmul_rn(v, scale));
  for (int i = 0; i < limbs; ++i) out[((std::size_t)i << logN) + n] = reduce_signed(c, pc[i]);
}

// ------------------------------------------------------------ packed wire format
// grid (words/256, limbs, npolys): one packed output word per thread
__global__ void k_pack(u64* __restrict__ dst, PolyList src, PackLayout lay, int logN) {
  const int i = blockIdx.y;
  const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nw = lay.off[i + 1] - lay.off[i];
  if (w >= nw) return;
  const int b = lay.bits[i];
  const u64* s = src.p[blockIdx.z] + ((std::size_t)i << logN);
  const long long bit0 = w * 64;
  long long k = bit0 / b;
  const int o = (int)(bit0 - k * b);  // bits of coefficient k already in the previous word
  u64 v = s[k] >> o;
  int filled = b - o;
  for (++k; filled < 64 && k < ((long long)1 << logN); ++k) {
    v |= s[k] << filled;
    filled += b;
  }
  dst[(std::size_t)blockIdx.z * lay.off[lay.limbs] + lay.off[i] + w] = v;
}
// grid (N/256, limbs, npolys): one coefficient per thread
__global__ void k_unpack(PolyList dst, const u64* __restrict__ src, PackLayout lay, int logN) {
  const int i = blockIdx.y;
  const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = lay.bits[i];
  const u64* s = src + (std::size_t)blockIdx.z * lay.off[lay.limbs] + lay.off[i];
  const long long bit = (long long)k * b;
  const long long w = bit >> 6;
  const int o = (int)(bit & 63);
  u64 v = s[w] >> o;
  if (o + b > 64) v |= s[w + 1] << (64 - o);
  if (b < 64) v &= (1ULL << b) - 1;
  dst.p[blockIdx.z][((std::size_t)i << logN) + k] = v;
}

// ------------------------------------------------------------ bootstrapping
// grid (N/256, npolys)
__global__ void k_modraise(PolyList out, PolyList in, const PrimeConst* __restrict__ pc, int logN, int L) {
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const u64 q0 = pc[0].q;
  const u64 v = in.p[blockIdx.z][n];
  const bool neg = v > q0 / 2;
  u64* o = out.p[blockIdx.z];
  for (int i = 0; i < L; ++i) {
    const PrimeConst P = pc[i];
    u64 x = reduce64(v, P);
    if (neg) x = sub_mod(x, reduce64(q0, P), P.q);
    o[((std::size_t)i << logN) + n] = x;
  }
}
// grid (N/256, limbs, npolys)
__global__ void k_mul_monomial_half(PolyList out, PolyList a, LimbConsts iq, const PrimeConst* __restrict__ pc,
                                    int logN) {
  const unsigned n = blockIdx.x * blockDim.x + threadIdx.x;
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + n;
  const u64 q = pc[blockIdx.y].q;
  u64 v = shoup_mul(a.p[blockIdx.z][o], iq.c[blockIdx.y], iq.sh[blockIdx.y], q);
  if ((n >> (logN - 1)) & 1u) v = v ? q - v : 0;
  out.p[blockIdx.z][o] = v;
}

// ------------------------------------------------------------ encode etc.
__global__ void k_coeffs_to_rns(u64* out, const long long* __restrict__ coeffs, const PrimeConst* __restrict__ pc,
                                int logN) {
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  out[((std::size_t)blockIdx.y << logN) + n] = reduce_signed(coeffs[n], pc[blockIdx.y]);  // pc offset by the launcher
}
__global__ void k_sample_error(u64* out, u64 key, const PrimeConst* __restrict__ pc, int logN, int ell, int L) {
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const int prime = i < ell ? i : L + (i - ell);
  out[((std::size_t)i << logN) + n] = reduce_signed(cbd21_d(prng_d(key, n)), pc[prime]);
}
__global__ void k_encrypt_combine(u64* c0, u64* c1, const u64* m, const u64* e, const u64* s, u64 stream_a,
                                  const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const std::size_t o = ((std::size_t)i << logN) + n;
  const PrimeConst P = pc[i];
  const u64 a = mulhi(prng_d(stream_a, (u64)o), P.q);
  c1[o] = a;
  c0[o] = sub_mod(add_mod(m[o], e[o], P.q), mul_mod(a, s[o], P), P.q);
}
__global__ void k_keygen_digit(u64* b, u64* a, const u64* e, const u64* s, const u64* sp, u64 stream_a, int lo,
                               int hi, const u64* __restrict__ pmod, const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t n = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const std::size_t o = ((std::size_t)i << logN) + n;
  const PrimeConst P = pc[i];
  const u64 av = mulhi(prng_d(stream_a, (u64)o), P.q);
  u64 bv = sub_mod(e[o], mul_mod(av, s[o], P), P.q);
  if (i >= lo && i < hi) bv = add_mod(bv, mul_mod(pmod[i], sp[o], P), P.q);
  b[o] = to_mont_d(bv, P);
  a[o] = to_mont_d(av, P);
}
__global__ void k_secret_square(u64* out, const u64* s, const PrimeConst* __restrict__ pc, int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  out[o] = mul_mod(s[o], s[o], pc[blockIdx.y]);
}
__global__ void k_decrypt_core(u64* m, const u64* c0, const u64* c1, const u64* s, const PrimeConst* __restrict__ pc,
                               int logN) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst P = pc[blockIdx.y];
  m[o] = add_mod(c0[o], mul_mod(c1[o], s[o], P), P.q);
}
__global__ void k_convert_mont(u64* out, const u64* in, const PrimeConst* __restrict__ pc, int logN, int ell, int L,
                               bool to) {
  const std::size_t o = ((std::size_t)blockIdx.y << logN) + blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  const PrimeConst P = pc[i < ell ? i : L + (i - ell)];
  out[o] = to ? to_mont_d(in[o], P) : redc(0, in[o], P.q, P.qinv_neg);
}

}  // namespace

void ew_add(const DevTables& t, const PolyList& out, const PolyList& a, const PolyList& b, int limbs, cudaStream_t st) {
  if (out.n == 0 || limbs == 0) return;
  if (aligned16(out) && aligned16(a) && aligned16(b)) {
    k_ew2<0><<<grid_for(t.N / 2, limbs, out.n), kThreads, 0, st>>>(out, a, b, LimbConsts{}, t.pc, t.logN);
    launch_check("k_add");
    return;
  }
  k_add<<<grid_for(t.N, limbs, out.n), kThreads, 0, st>>>(out, a, b, t.pc, t.logN);
  launch_check("k_add");
}
void ew_sub(const DevTables& t, const PolyList& out, const PolyList& a, const PolyList& b, int limbs, cudaStream_t st) {
  if (out.n == 0 || limbs == 0) return;
  if (aligned16(out) && aligned16(a) && aligned16(b)) {
    k_ew2<1><<<grid_for(t.N / 2, limbs, out.n), kThreads, 0, st>>>(out, a, b, LimbConsts{}, t.pc, t.logN);
    launch_check("k_sub");
    return;
  }
  k_sub<<<grid_for(t.N, limbs, out.n), kThreads, 0, st>>>(out, a, b, t.pc, t.logN);
  launch_check("k_sub");
}
void ew_neg(const DevTables& t, const PolyList& out, const PolyList& a, int limbs, cudaStream_t st) {
  if (out.n == 0 || limbs == 0) return;
  k_neg<<<grid_for(t.N, limbs, out.n), kThreads, 0, st>>>(out, a, t.pc, t.logN);
  launch_check("k_neg");
}
void ew_mul_pt(const DevTables& t, const PolyList& out, const PolyList& a, const u64* pt, int limbs, cudaStream_t st) {
  if (out.n == 0 || limbs == 0) return;
  k_mul_pt<<<grid_for(t.N, limbs, out.n), kThreads, 0, st>>>(out, a, pt, t.pc, t.logN);
  launch_check("k_mul_pt");
}
void ew_mul_const(const DevTables& t, const PolyList& out, const PolyList& a, const LimbConsts& c, int limbs,
                  cudaStream_t st) {
  if (out.n == 0 || limbs == 0) return;
  if (aligned16(out) && aligned16(a)) {
    k_ew2<3><<<grid_for(t.N / 2, limbs, out.n), kThreads, 0, st>>>(out, a, a, c, t.pc, t.logN);
    launch_check("k_mul_const");
    return;
  }
  k_mul_const<<<grid_for(t.N, limbs, out.n), kThreads, 0, st>>>(out, a, c, t.pc, t.logN);
  launch_check("k_mul_const");
}
void ew_add_const(const DevTables& t, const PolyList& out, const PolyList& a, const LimbConsts& c, int limbs,
                  cudaStream_t st) {
  if (out.n == 0 || limbs == 0) return;
  if (aligned16(out) && aligned16(a)) {
    k_ew2<2><<<grid_for(t.N / 2, limbs, out.n), kThreads, 0, st>>>(out, a, a, c, t.pc, t.logN);
    launch_check("k_add_const");
    return;
  }
  k_add_const<<<grid_for(t.N, limbs, out.n), kThreads, 0, st>>>(out, a, c, t.pc, t.logN);
  launch_check("k_add_const");
}
void lincomb_const(const DevTables& t, u64* out0, u64* out1, const LincombTerms& terms, const u64* kc, int limbs,
                   cudaStream_t st) {
  if (terms.n == 0 || limbs == 0) return;
  k_lincomb_const<<<grid_for(t.N / 2, limbs, 2), kThreads, 0, st>>>(out0, out1, terms, kc, t.pc, t.logN, limbs);
  launch_check("k_lincomb_const");
}
void ew_axpy_limb(const DevTables& t, const PolyList& acc, const PolyList& x, u64 c_mont, int prime, cudaStream_t st) {
  if (acc.n == 0) return;
  k_axpy_limb<<<dim3((unsigned)(t.N / kThreads), (unsigned)acc.n), kThreads, 0, st>>>(acc, x, c_mont, t.pc, prime);
  launch_check("k_axpy_limb");
}
void ew_tensor(const DevTables& t, u64* d0, u64* d1, u64* d2, const u64* a0, const u64* a1, const u64* b0,
               const u64* b1, int limbs, cudaStream_t st) {
  k_tensor<<<grid_for(t.N, limbs), kThreads, 0, st>>>(d0, d1, d2, a0, a1, b0, b1, t.pc, t.logN);
  launch_check("k_tensor");
}
void ew_tensor_cheb(const DevTables& t, u64* d0, u64* d1, u64* d2, const u64* a0, const u64* a1, const u64* b0,
                    const u64* b1, const u64* s0, const u64* s1, const LimbConsts& kc, int limbs, cudaStream_t st) {
  k_tensor_cheb<<<grid_for(t.N, limbs), kThreads, 0, st>>>(d0, d1, d2, a0, a1, b0, b1, s0, s1, kc, t.pc, t.logN);
  launch_check("k_tensor_cheb");
}
void automorph(const DevTables& t, const PolyList& out, const PolyList& in, int limbs, cudaStream_t st) {
  if (out.n == 0 || limbs == 0) return;
  k_automorph<<<grid_for(t.N, limbs, out.n), kThreads, 0, st>>>(out, in, t.logN);
  launch_check("k_automorph");
}

void modup_bconv(const DevTables& t, const PolyList& ext, const PolyList& x, int limbs, cudaStream_t st) {
  const int beta = t.dig.beta(limbs);
  TimedScope ts(t, kModUp, st);
  const int E = limbs + t.K;
  if (bconv_tc_enabled() && modup_bconv_tc_all(t, ext, x, limbs, st)) {  // every digit in one launch
    launch_check("k_bconv_tc<modup>");
    return;
  }
  for (int j = 0; j < beta; ++j) {
    if (bconv_tc_enabled()) {
      modup_bconv_tc(t, ext, x, limbs, j, st);
      launch_check("k_bconv_tc<modup>");
      continue;
    }
    const int lo = t.dig.lo(j);
    const int a = t.dig.hi(j, limbs) - lo;
    const dim3 grid = grid_for(t.N, (E - a + kTC - 1) / kTC, x.n);
#define FHEON_BCONV(AA)                                                                                        \
  case AA:                                                                                                     \
    k_modup_bconv<AA><<<grid, kThreads, 0, st>>>(ext, x, t.pc, t.modup_qhinv, t.modup_qhat, t.logN, limbs, t.L, \
                                                 t.K, t.dnum, lo, j);                                          \
    break;
    switch (a) {
      FHEON_BCONV(1) FHEON_BCONV(2) FHEON_BCONV(3) FHEON_BCONV(4) FHEON_BCONV(5) FHEON_BCONV(6) FHEON_BCONV(7)
      FHEON_BCONV(8) FHEON_BCONV(9) FHEON_BCONV(10) FHEON_BCONV(11) FHEON_BCONV(12) FHEON_BCONV(13)
      FHEON_BCONV(14) FHEON_BCONV(15)
      default: throw std::runtime_error("digit size out of range");
    }
#undef FHEON_BCONV
    launch_check("k_modup_bconv");
  }
}
void ks_inner_product(const DevTables& t, const KsJobs& jobs, int limbs, cudaStream_t st) {
  if (jobs.n == 0) return;
  TimedScope ts(t, kKsInner, st);
  const dim3 grid(jobs.n, (unsigned)(t.N / (2 * kThreads)), limbs + t.K);
  k_ks_inner<<<grid, kThreads, 0, st>>>(jobs, t.pc, t.logN, limbs, t.L, t.K,
                                                                       DigitOwner{t.digit_owner, t.dig.beta(limbs)});
  launch_check("k_ks_inner");
}
void ks_inner_sum(const DevTables& t, const KsSumJobs& jobs, int limbs, cudaStream_t st) {
  if (jobs.ngroups == 0) return;
  TimedScope ts(t, kKsInner, st);
  const dim3 grid(jobs.ngroups, (unsigned)(t.N / (2 * kThreads)), limbs + t.K);
  k_ks_inner_sum<<<grid, kThreads, 0, st>>>(jobs, t.pc, t.md_q, t.logN, limbs,
                                                                                 t.L, t.K, DigitOwner{t.digit_owner, t.dig.beta(limbs)});
  launch_check("k_ks_inner_sum");
}
void ks_inner_shared(const DevTables& t, const KsSharedJobs& jobs, int limbs, cudaStream_t st) {
  if (jobs.ngroups == 0) return;
  TimedScope ts(t, kKsInner, st);
  const dim3 grid(jobs.ngroups, (unsigned)(t.N / (2 * kThreads)), limbs + t.K);
  k_ks_inner_shared<<<grid, kThreads, 0, st>>>(jobs, t.pc, t.md_q, t.logN, limbs, t.L, t.K,
                                               DigitOwner{t.digit_owner, t.dig.beta(limbs)});
  launch_check("k_ks_inner_shared");
}
void moddown_conv(const DevTables& t, const PolyList& conv, const PolyList& z, int limbs, cudaStream_t st) {
  if (conv.n == 0) return;
  TimedScope ts(t, kModDown, st);
  if (bconv_tc_enabled()) {
    moddown_conv_tc(t, conv, z, limbs, st);
    launch_check("k_bconv_tc<moddown>");
    return;
  }
  const dim3 grid = grid_for(t.N, (limbs + kTC - 1) / kTC, conv.n);
#define FHEON_MDC(KK)                                                                                             \
  case KK:                                                                                                        \
    k_moddown_conv<KK><<<grid, kThreads, 0, st>>>(conv, z, t.pc, t.md_pk, t.md_pinv, t.md_phat, t.md_q, t.logN, \
                                                  limbs, t.L);                                                    \
    break;
  switch (t.K) {
    FHEON_MDC(1) FHEON_MDC(2) FHEON_MDC(3) FHEON_MDC(4) FHEON_MDC(5) FHEON_MDC(6) FHEON_MDC(7) FHEON_MDC(8)
    FHEON_MDC(9) FHEON_MDC(10) FHEON_MDC(11) FHEON_MDC(12) FHEON_MDC(13) FHEON_MDC(14) FHEON_MDC(15)
    default: throw std::runtime_error("K out of range");
  }
#undef FHEON_MDC
  launch_check("k_moddown_conv");
}
void rescale_lift(const DevTables& t, const PolyList& r, const PolyList& last, int limbs, cudaStream_t st) {
  if (r.n == 0) return;
  k_rescale_lift<<<grid_for(t.N, 1, r.n), kThreads, 0, st>>>(r, last, t.pc, t.rs, t.logN, limbs, t.L);
  launch_check("k_rescale_lift");
}

void pack_limbs(const DevTables& t, u64* dst, const PolyList& src, const PackLayout& lay, cudaStream_t st) {
  if (src.n == 0 || lay.limbs == 0) return;
  long long maxw = 0;
  for (int i = 0; i < lay.limbs; ++i) maxw = std::max(maxw, lay.off[i + 1] - lay.off[i]);
  const dim3 grid((unsigned)((maxw + kThreads - 1) / kThreads), lay.limbs, src.n);
  k_pack<<<grid, kThreads, 0, st>>>(dst, src, lay, t.logN);
  launch_check("k_pack");
}
void unpack_limbs(const DevTables& t, const PolyList& dst, const u64* src, const PackLayout& lay, cudaStream_t st) {
  if (dst.n == 0 || lay.limbs == 0) return;
  k_unpack<<<grid_for(t.N, lay.limbs, dst.n), kThreads, 0, st>>>(dst, src, lay, t.logN);
  launch_check("k_unpack");
}
void modraise(const DevTables& t, const PolyList& out, const PolyList& in, int L, cudaStream_t st) {
  if (out.n == 0) return;
  k_modraise<<<grid_for(t.N, 1, out.n), kThreads, 0, st>>>(out, in, t.pc, t.logN, L);
  launch_check("k_modraise");
}
void mul_monomial_half(const DevTables& t, const PolyList& out, const PolyList& a, const LimbConsts& iq, int limbs,
                       cudaStream_t st) {
  if (out.n == 0) return;
  k_mul_monomial_half<<<grid_for(t.N, limbs, out.n), kThreads, 0, st>>>(out, a, iq, t.pc, t.logN);
  launch_check("k_mul_monomial_half");
}
void mac_pt(const DevTables& t, const MacJobs& jobs, int limbs, cudaStream_t st, int ell) {
  if (jobs.nout == 0) return;
  const dim3 grid(jobs.nout, (unsigned)(t.N / (2 * kThreads)), limbs);
  k_mac<<<grid, kThreads, 0, st>>>(jobs, t.pc, t.logN, ell < 0 ? limbs : ell, t.L);
  launch_check("k_mac");
}
void mac_bsgs(const DevTables& t, const BsgsMacJobs& jobs, int E, cudaStream_t st, int ell) {
  if (jobs.ngiants == 0 || jobs.nin == 0) return;
  const dim3 grid(jobs.ngiants * jobs.nin, (unsigned)(t.N / (2 * kThreads)), E);
  k_mac_bsgs<<<grid, kThreads, 0, st>>>(jobs, t.pc, t.logN, ell, t.L);
  launch_check("k_mac_bsgs");
}
void encode_lincomb(const DevTables& t, u64* out, const LinComb& lc, double scale, int limbs, cudaStream_t st) {
  k_encode_lincomb<<<grid_for(t.N, 1), kThreads, 0, st>>>(out, lc, scale, t.pc, t.logN, limbs);
  launch_check("k_encode_lincomb");
}
void coeffs_to_rns(const DevTables& t, u64* out, const long long* coeffs, int limbs, cudaStream_t st, int p0) {
  k_coeffs_to_rns<<<grid_for(t.N, limbs), kThreads, 0, st>>>(out, coeffs, t.pc + p0, t.logN);
  launch_check("k_coeffs_to_rns");
}
void sample_error(const DevTables& t, u64* out, u64 stream_key, int nlimbs, int ell, cudaStream_t st) {
  k_sample_error<<<grid_for(t.N, nlimbs), kThreads, 0, st>>>(out, stream_key, t.pc, t.logN, ell, t.L);
  launch_check("k_sample_error");
}
void encrypt_combine(const DevTables& t, u64* c0, u64* c1, const u64* m, const u64* e, u64 stream_a, int limbs,
                     cudaStream_t st) {
  k_encrypt_combine<<<grid_for(t.N, limbs), kThreads, 0, st>>>(c0, c1, m, e, t.s_ntt, stream_a, t.pc, t.logN);
  launch_check("k_encrypt_combine");
}
void keygen_digit(const DevTables& t, u64* b, u64* a, const u64* e, const u64* sp, const u64* s_to, u64 stream_a,
                  int lo, int hi, const u64* pmod, cudaStream_t st) {
  k_keygen_digit<<<grid_for(t.N, t.L + t.K), kThreads, 0, st>>>(b, a, e, s_to, sp, stream_a, lo, hi, pmod, t.pc,
                                                                 t.logN);
}
void secret_square(const DevTables& t, u64* out, cudaStream_t st) {
  k_secret_square<<<grid_for(t.N, t.L + t.K), kThreads, 0, st>>>(out, t.s_ntt, t.pc, t.logN);
  launch_check("k_secret_square");
}
void decrypt_core(const DevTables& t, u64* m, const u64* c0, const u64* c1, int limbs, cudaStream_t st) {
  k_decrypt_core<<<grid_for(t.N, limbs), kThreads, 0, st>>>(m, c0, c1, t.s_ntt, t.pc, t.logN);
  launch_check("k_decrypt_core");
}
void convert_mont(const DevTables& t, u64* out, const u64* in, int nlimbs, int ell, bool to_mont, cudaStream_t st) {
  k_convert_mont<<<grid_for(t.N, nlimbs), kThreads, 0, st>>>(out, in, t.pc, t.logN, ell, t.L, to_mont);
  launch_check("k_convert_mont");
}

}  // namespace fheon
