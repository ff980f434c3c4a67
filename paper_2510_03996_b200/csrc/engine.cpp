// Context construction (device constant tables), allocator, keys, encoder,
// trace.  See engine.hpp.
#include "engine.hpp"

#include "bootstrap.hpp"

#include <atomic>
#include <cmath>
#include <cstring>

namespace fheon {

int category_of(ErrKind k) {
  switch (k) {
    case ErrKind::invalid_rotation:
    case ErrKind::shape:
    case ErrKind::capacity:
    case ErrKind::model:
      return 2;
    case ErrKind::not_implemented:
      return 1;
    default:
      return 3;
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(ErrKind::cuda, std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what);
  }
}

std::atomic<std::uint64_t> g_kernel_launches{0};

void launch_check(const char* what) {
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(ErrKind::cuda, std::string("kernel launch failed: ") + what + ": " + cudaGetErrorString(e));
  }
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
}

// ------------------------------------------------------------- kernel timer
KernelTimer::~KernelTimer() {
  for (cudaEvent_t e : ev) cudaEventDestroy(e);
}
void KernelTimer::begin(cudaStream_t st) {
  if (depth++ > 0) return;
  if (used + 2 > ev.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      FHEON_CUDA(cudaEventCreate(&e));
      ev.push_back(e);
    }
  }
  FHEON_CUDA(cudaEventRecord(ev[used], st));
}
void KernelTimer::end(cudaStream_t st) {
  if (--depth > 0) return;
  FHEON_CUDA(cudaEventRecord(ev[used + 1], st));
  used += 2;
}
double KernelTimer::total_ms(int* count) {
  double tot = 0.0;
  for (std::size_t i = 0; i + 1 < used; i += 2) {
    FHEON_CUDA(cudaEventSynchronize(ev[i + 1]));
    float ms = 0.f;
    FHEON_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
    tot += ms;
  }
  if (count) *count = (int)(used / 2);
  return tot;
}

TimedScope::TimedScope(const DevTables& t_, int c, cudaStream_t s) : t(t_), cls(c), st(s) {
  if (t.timer && t.timer->cls == cls) t.timer->begin(st);
}
TimedScope::~TimedScope() {
  if (t.timer && t.timer->cls == cls) t.timer->end(st);
}

// ------------------------------------------------------------- buffers
namespace {
// stream-ordered allocation; on out-of-memory the context's plaintext caches are
// released (their buffers return to the pool once the compute stream passes their
// last use) and the allocation is retried once
cudaError_t pool_alloc(Context* c, void** p, std::size_t bytes, cudaStream_t st) {
  return c->mem_pool() ? cudaMallocFromPoolAsync(p, bytes, c->mem_pool(), st) : cudaMallocAsync(p, bytes, st);
}
u64* device_alloc(Context* c, std::size_t words, cudaStream_t st) {
  void* p = nullptr;
  cudaError_t e = pool_alloc(c, &p, words * sizeof(u64), st);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    static const bool dbg = std::getenv("FHEON_ALLOC_DEBUG") != nullptr;
    if (dbg) std::fprintf(stderr, "[fheon] allocation of %zu bytes failed: releasing plaintext caches\n", words * 8);
    if (c->release_caches() > 0) {
      FHEON_CUDA(cudaStreamSynchronize(c->stream()));
      e = pool_alloc(c, &p, words * sizeof(u64), st);
    }
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(ErrKind::cuda, std::string("CUDA error: ") + cudaGetErrorString(e) + " allocating " +
                                   std::to_string(words * sizeof(u64)) + " bytes (resident keys and caches exceed HBM)");
  }
  return static_cast<u64*>(p);
}
}  // namespace

std::size_t Context::release_caches() {
  std::size_t bytes = weightcache_bytes_ + ptcache_words_ * sizeof(u64);
  // the resident set did not fit beside the keys: keep at most half of it from now on
  if (weightcache_bytes_ > 0) weight_cache_budget = std::min(weight_cache_budget, weightcache_bytes_ / 2);
  weightcache_.clear();
  weightcache_bytes_ = 0;
  ptcache_.clear();
  namedcache_.clear();
  ptcache_words_ = 0;
  return bytes;
}

DevBuffer::DevBuffer(Context* c, std::size_t w) : alive(c->alive), stream(c->stream()), words(w) {
  if (w == 0) return;
  ptr = device_alloc(c, w, stream);
}
DevBuffer::~DevBuffer() {
  if (!ptr) return;
  if (alive && alive->load()) cudaFreeAsync(ptr, stream);
  else cudaFree(ptr);
}

DevBuffer::DevBuffer(Context* c, std::size_t w, cudaStream_t alloc_stream)
    : alive(c->alive), stream(c->stream()), words(w) {
  if (w == 0) return;
  ptr = device_alloc(c, w, alloc_stream);
}

BufPtr Context::alloc(std::size_t words) { return std::make_shared<DevBuffer>(this, words); }

cudaEvent_t Context::take_event() {
  if (!event_pool_.empty()) {
    cudaEvent_t e = event_pool_.back();
    event_pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  FHEON_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return e;
}

void Context::give_event(cudaEvent_t e) { event_pool_.push_back(e); }

void Context::hold_until(cudaEvent_t done, BufPtr buf) {
  reap_transfers(false);
  held_.emplace_back(done, std::move(buf));
}

void Context::reap_transfers(bool wait) {
  std::size_t k = 0;
  for (auto& [e, b] : held_) {
    if (wait) FHEON_CUDA(cudaEventSynchronize(e));
    if (wait || cudaEventQuery(e) == cudaSuccess) {
      give_event(e);
      b.reset();
    } else {
      held_[k++] = {e, std::move(b)};
    }
  }
  held_.resize(k);
  cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error
}

Ciphertext Context::new_ct(int limbs) {
  Ciphertext c;
  c.buf = alloc(2 * static_cast<std::size_t>(limbs) * N());
  c.c0 = c.buf->ptr;
  c.c1 = c.buf->ptr + static_cast<std::size_t>(limbs) * N();
  c.limbs = limbs;
  c.id = next_id();
  return c;
}

// ------------------------------------------------------------- context
namespace {

u64 neg_inv64(u64 q) {
  u64 inv = q;  // q * q = 1 mod 8 for odd q
  for (int i = 0; i < 6; ++i) inv *= 2 - q * inv;
  return ~inv + 1;  // -q^{-1}
}

template <class T>
T* upload(std::vector<void*>& track, const std::vector<T>& v, cudaStream_t st) {
  T* d = nullptr;
  FHEON_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), std::max<std::size_t>(1, v.size()) * sizeof(T)));
  track.push_back(d);
  if (!v.empty()) FHEON_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return d;
}

u64 prod_mod(const std::vector<u64>& primes, int lo, int hi, int skip, u64 m) {
  u64 r = 1 % m;
  for (int i = lo; i < hi; ++i)
    if (i != skip) r = mulmod(r, primes[i] % m, m);
  return r;
}

}  // namespace

Context::Context(const Params& p, const Context* parent) : ht_(make_tables(p)) {
  if (parent) {
    const Params& pp = parent->host().p;
    if (pp.logN != p.logN || pp.L != p.L || pp.K != p.K || pp.dnum != p.dnum || pp.seed != p.seed ||
        pp.hamming_weight != p.hamming_weight || parent->host().q != ht_.q)
      throw Error(ErrKind::internal, "key-sharing context: parameters differ from the parent's");
    inheriting_keys = true;  // the bootstrapper pins the parent's keys instead of generating
  }
  if (ht_.alpha > kMaxAlpha - 1) throw Error(ErrKind::shape, "a key-switching digit must hold < 16 limbs");
  if (ht_.ndig > kMaxDigits) throw Error(ErrKind::shape, "at most 16 key-switching digits");
  if (p.K > kMaxK - 1) throw Error(ErrKind::shape, "K must be < 16");
  if (p.L > 64) throw Error(ErrKind::shape, "L must be <= 64");
  {
    // Hybrid key switching needs P = prod(p_k) to dominate every digit
    // modulus Q_j, otherwise the key-switch noise Q_j * e / P swamps the scale.
    double logP = 0.0;
    for (int k = 0; k < p.K; ++k) logP += std::log2((double)ht_.q[p.L + k]);
    for (int j = 0; j < ht_.ndig; ++j) {
      double logQ = 0.0;
      for (int i = ht_.dig[j]; i < ht_.dig[j + 1]; ++i) logQ += std::log2((double)ht_.q[i]);
      if (logQ > logP)
        throw Error(ErrKind::shape, "special modulus P (" + std::to_string((int)logP) +
                                        " bits) must exceed every key-switching digit modulus (digit " +
                                        std::to_string(j) + ": " + std::to_string((int)logQ) +
                                        " bits); raise special_limbs or dnum");
    }
  }
  depth_budget_ = p.depth_budget < 0 ? p.L - 1 : p.depth_budget;
  if (depth_budget_ < 1 || depth_budget_ > p.L - 1)
    throw Error(ErrKind::shape, "depth budget must lie in [1, L-1]");
  if (p.bootstrap && p.hamming_weight <= 0 && p.boot_hamming_weight <= 0)
    throw Error(ErrKind::shape, "bootstrapping with a dense secret needs boot_hamming_weight > 0 (sparse-secret "
                                "encapsulation)");
  {
    double logqp = 0.0;
    for (int i = 0; i < p.L + p.K; ++i) logqp += std::log2((double)ht_.q[i]);
    log_qp_ = logqp;
    security_ = he_standard_security(p.logN, logqp, p.hamming_weight);
    const int want = p.min_security > 0 ? p.min_security : 128;
    if (!p.allow_insecure && security_ < want) {
      const double bound = he_standard_max_logqp(p.logN, want);
      std::string why = p.hamming_weight > 0
                            ? "a sparse main secret (hamming_weight " + std::to_string(p.hamming_weight) +
                                  ") is not covered by the HE-standard table; use a dense secret (bootstrapping "
                                  "then runs the sparse-secret encapsulation)"
                            : "log2(QP) = " + std::to_string((int)std::ceil(logqp)) + " bits exceeds the HE-standard "
                                  "bound of " + std::to_string((int)bound) + " bits for N = 2^" +
                                  std::to_string(p.logN) + " at " + std::to_string(want) + "-bit security";
      throw Error(ErrKind::shape, "insecure parameters: " + why + " (set allow_insecure to run them anyway)");
    }
  }
  int dev = 0;
  FHEON_CUDA(cudaGetDevice(&dev));
  FHEON_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  // copy streams at the highest priority: their (un)pack kernels are scheduled ahead of
  // the compute stream's grids, so the copy engines are not left waiting behind them
  int prio_least = 0, prio_greatest = 0;
  FHEON_CUDA(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
  FHEON_CUDA(cudaStreamCreateWithPriority(&h2d_, cudaStreamNonBlocking, prio_greatest));
  FHEON_CUDA(cudaStreamCreateWithPriority(&d2h_, cudaStreamNonBlocking, prio_greatest));
  FHEON_CUDA(cudaStreamCreateWithPriority(&unpack_, cudaStreamNonBlocking, prio_greatest));
  FHEON_CUDA(cudaStreamCreateWithPriority(&pack_, cudaStreamNonBlocking, prio_greatest));
  {
    // One stream-ordered pool PER CONTEXT: contexts in flight (key-sharing clones, one stream and
    // host thread each) must not recycle each other's blocks -- a block freed on one stream and
    // handed to another makes the allocator either insert a dependency between the streams (they
    // serialise at random points) or map new memory mid-run; both showed as a bimodal 0.31-0.38
    // s/image with batches in flight.  FHEON_PRIVATE_POOL=0: the device's default pool (A/B).
    cudaMemPool_t pool;
    const char* pp = std::getenv("FHEON_PRIVATE_POOL");
    if (pp && std::atoi(pp) == 0) {
      FHEON_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    } else {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      FHEON_CUDA(cudaMemPoolCreate(&pool_, &props));
      pool = pool_;
    }
    std::uint64_t thr = UINT64_MAX;
    FHEON_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // Pre-grow the stream-ordered pool so steady-state key switching never
    // maps new physical memory mid-pipeline: reserve ~64 ciphertexts' worth
    // of scratch (capped at 1/4 of free HBM).
    std::size_t free_b = 0, total_b = 0;
    FHEON_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const std::size_t ct_bytes = 2 * (std::size_t)(p.L + p.K) * ((std::size_t)1 << p.logN) * sizeof(u64);
    std::size_t want = std::min<std::size_t>(free_b / 4, 64 * ct_bytes * 3);
    // resident weight plaintexts: up to half of the free HBM (96 GiB cap); the keys
    // (~40 GB for ResNet-20 at depth 25), the mask/diagonal cache (24 GiB) and the
    // key-switch scratch pool need the rest
    weight_cache_budget = std::min<std::size_t>(weight_cache_budget, free_b / 2);
    void* r = nullptr;
    if (want > 0 && pool_alloc(this, &r, want, stream_) == cudaSuccess) cudaFreeAsync(r, stream_);
    cudaGetLastError();
  }
  for (int i = 0; i < kStaging; ++i) {
    FHEON_CUDA(cudaMallocHost(reinterpret_cast<void**>(&staging_[i]), ht_.N * sizeof(long long)));
    FHEON_CUDA(cudaEventCreateWithFlags(&staging_ev_[i], cudaEventDisableTiming));
  }
  build_device_tables();
  if (p.bootstrap && parent && parent->boot) {
    // a clone shares the parent's bootstrapping plans and encoded diagonals (read-only);
    // the parent's stream has finished writing them before this context reads them
    FHEON_CUDA(cudaStreamSynchronize(parent->stream()));
    boot = std::make_unique<Bootstrapper>(*this, *parent->boot);
    for (const auto& b : parent->boot_sparse) boot_sparse.push_back(std::make_unique<Bootstrapper>(*this, *b));
    depth_budget_ = parent->depth_budget();
  } else if (p.bootstrap) {
    boot = std::make_unique<Bootstrapper>(*this, boot_params_of(p));
    const int after = p.L - 1 - boot->depth();
    if (p.depth_budget < 0) depth_budget_ = after;
    else if (p.depth_budget > after)
      throw Error(ErrKind::shape, "depth budget " + std::to_string(p.depth_budget) +
                                      " exceeds the levels left after bootstrapping (" + std::to_string(after) + ")");
    for (int k = 1; k <= p.boot_sparse && (ht_.S >> k) >= 4; ++k) {
      BootParams bp = boot_params_of(p);
      int ls = 0;
      while ((1L << ls) < (long)(ht_.S >> k)) ++ls;
      bp.log_slots = ls;
      boot_sparse.push_back(std::make_unique<Bootstrapper>(*this, bp));
    }
  }
  if (parent) {
    keys_ = parent->keys_;  // shared read-only device buffers
    for (u64 id : parent->pinned_keys_) pinned_keys_.insert(id);
    inheriting_keys = false;
  }
}

Context::Context(const Params& p) : Context(p, nullptr) {}
Context::Context(const Params& p, const Context& parent) : Context(p, &parent) {}

Context::~Context() {
  boot.reset();
  boot_sparse.clear();
  keys_.clear();
  basis_.clear();
  ptcache_.clear();
  namedcache_.clear();
  weightcache_.clear();
  if (stream_) cudaStreamSynchronize(stream_);
  alive->store(false);
  for (void* d : dev_allocs_) cudaFree(d);
  for (int i = 0; i < kStaging; ++i) {
    if (staging_[i]) cudaFreeHost(staging_[i]);
    if (staging_ev_[i]) cudaEventDestroy(staging_ev_[i]);
  }
  if (h2d_) cudaStreamSynchronize(h2d_);
  if (d2h_) cudaStreamSynchronize(d2h_);
  if (unpack_) cudaStreamSynchronize(unpack_);
  if (pack_) cudaStreamSynchronize(pack_);
  for (auto& [e, b] : held_) cudaEventDestroy(e);
  held_.clear();
  for (cudaEvent_t e : event_pool_) cudaEventDestroy(e);
  if (h2d_) cudaStreamDestroy(h2d_);
  if (d2h_) cudaStreamDestroy(d2h_);
  if (unpack_) cudaStreamDestroy(unpack_);
  if (pack_) cudaStreamDestroy(pack_);
  if (stream_) cudaStreamDestroy(stream_);
  // released once the last outstanding allocation (a handle that outlives the context) is freed
  if (pool_) {
    cudaMemPoolTrimTo(pool_, 0);
    cudaMemPoolDestroy(pool_);
  }
}

void Context::build_device_tables() {
  const Params& p = ht_.p;
  const int L = p.L, K = p.K, NP = L + K, dnum = p.dnum;
  const std::size_t N = ht_.N;
  const std::vector<u64>& q = ht_.q;
  DevTables& t = dt_;
  t.logN = p.logN;
  t.n1 = p.logN / 2;
  t.n2 = p.logN - t.n1;
  t.N = N;
  t.L = L;
  t.K = K;
  t.dnum = dnum;
  t.alpha = ht_.alpha;
  t.dig.n = ht_.ndig;
  for (int j = 0; j <= ht_.ndig; ++j) t.dig.b[j] = ht_.dig[j];
  {
    std::vector<unsigned char> own(L);
    for (int i = 0; i < L; ++i) own[i] = (unsigned char)t.dig.digit_of(i);
    t.digit_owner = upload(dev_allocs_, own, stream_);
  }
  t.timer = &timer;

  std::vector<PrimeConst> pcs(NP);
  for (int i = 0; i < NP; ++i) {
    PrimeConst& c = pcs[i];
    c.q = q[i];
    c.qinv_neg = neg_inv64(q[i]);
    const u64 rmod = (u64)(((u128)1 << 64) % q[i]);
    c.rmod = rmod;
    c.r2 = mulmod(rmod, rmod, q[i]);
    c.mu64 = (u64)(((u128)1 << 64) / q[i]);
    c.ninv = invmod(N % q[i], q[i]);
    c.ninv_sh = shoup(c.ninv, q[i]);
    c.pad = 0;
  }
  t.pc = upload(dev_allocs_, pcs, stream_);
  t.rotgroup = upload(dev_allocs_, ht_.rotgroup, stream_);
  t.ksi_re = upload(dev_allocs_, ht_.ksi_re, stream_);
  t.ksi_im = upload(dev_allocs_, ht_.ksi_im, stream_);

  // twiddles [NP][4][N]
  std::vector<u64> tw((std::size_t)NP * 4 * N);
#pragma omp parallel for
  for (int i = 0; i < NP; ++i) {
    const u64 qi = q[i];
    const u64 psi = ht_.psi[i], ipsi = invmod(psi, qi);
    std::vector<u64> pw(N), ipw(N);
    pw[0] = ipw[0] = 1;
    for (std::size_t e = 1; e < N; ++e) {
      pw[e] = mulmod(pw[e - 1], psi, qi);
      ipw[e] = mulmod(ipw[e - 1], ipsi, qi);
    }
    u64* base = tw.data() + (std::size_t)i * 4 * N;
    for (std::size_t k = 0; k < N; ++k) {
      const unsigned e = bitrev((unsigned)k, p.logN);
      base[2 * k] = pw[e];  // (value, Shoup) pairs: one 16-byte load per twiddle
      base[2 * k + 1] = shoup(pw[e], qi);
      base[2 * N + 2 * k] = ipw[e];
      base[2 * N + 2 * k + 1] = shoup(ipw[e], qi);
    }
  }
  t.tw = upload(dev_allocs_, tw, stream_);

  // ModUp tables
  std::vector<u64> qhinv((std::size_t)L * dnum * kMaxAlpha * 2, 0);
  std::vector<u64> qhat((std::size_t)L * dnum * NP * kMaxAlpha, 0);
  for (int limbs = 1; limbs <= L; ++limbs) {
    for (int j = 0; j < ht_.ndig; ++j) {
      const int lo = ht_.dig[j], hi = std::min(ht_.dig[j + 1], limbs);
      if (lo >= hi) continue;
      const int tab = (limbs - 1) * dnum + j;
      for (int i = lo; i < hi; ++i) {
        const u64 h = prod_mod(q, lo, hi, i, q[i]);
        const u64 hi_inv = invmod(h, q[i]);
        qhinv[((std::size_t)tab * kMaxAlpha + (i - lo)) * 2] = hi_inv;
        qhinv[((std::size_t)tab * kMaxAlpha + (i - lo)) * 2 + 1] = shoup(hi_inv, q[i]);
        for (int pt = 0; pt < NP; ++pt) {
          const u64 m = q[pt];
          qhat[((std::size_t)tab * NP + pt) * kMaxAlpha + (i - lo)] = to_mont(prod_mod(q, lo, hi, i, m), m);
        }
      }
    }
  }
  t.modup_qhinv = upload(dev_allocs_, qhinv, stream_);
  t.modup_qhat = upload(dev_allocs_, qhat, stream_);

  // ModDown tables
  std::vector<u64> pk((std::size_t)K * 4, 0);
  std::vector<double> pinv(K);
  std::vector<u64> phat((std::size_t)L * kMaxK, 0);
  std::vector<u64> mq((std::size_t)L * 4, 0);
  auto half_P = [&](u64 m) {
    const u64 Pm = prod_mod(q, L, L + K, -1, m);
    return mulmod(submod(Pm, 1 % m, m), (m + 1) / 2, m);
  };
  for (int k = 0; k < K; ++k) {
    const u64 pkv = q[L + k];
    const u64 h = prod_mod(q, L, L + K, L + k, pkv);
    const u64 hinv = invmod(h, pkv);
    pk[k * 4] = hinv;
    pk[k * 4 + 1] = shoup(hinv, pkv);
    pk[k * 4 + 2] = half_P(pkv);
    pinv[k] = 1.0 / (double)pkv;
  }
  for (int i = 0; i < L; ++i) {
    for (int k = 0; k < K; ++k) phat[(std::size_t)i * kMaxK + k] = to_mont(prod_mod(q, L, L + K, L + k, q[i]), q[i]);
    const u64 Pm = prod_mod(q, L, L + K, -1, q[i]);
    const u64 Pinv = invmod(Pm, q[i]);
    mq[i * 4] = to_mont(Pm, q[i]);
    mq[i * 4 + 1] = half_P(q[i]);
    mq[i * 4 + 2] = Pinv;
    mq[i * 4 + 3] = shoup(Pinv, q[i]);
  }
  t.md_pk = upload(dev_allocs_, pk, stream_);
  t.md_pinv = upload(dev_allocs_, pinv, stream_);
  t.md_phat = upload(dev_allocs_, phat, stream_);
  t.md_q = upload(dev_allocs_, mq, stream_);

  // Fused relinearisation + rescale tables: P' = P q_l, special s = 0: q_l, s >= 1: p_{s-1}
  {
    std::vector<u64> pk2((std::size_t)L * kMaxK * 4, 0);
    std::vector<double> pinv2((std::size_t)L * kMaxK, 0.0);
    std::vector<u64> phat2((std::size_t)L * L * kMaxK, 0);
    std::vector<u64> mq2((std::size_t)L * L * 4, 0);
    for (int l = 1; l < L && K + 1 <= kMaxK; ++l) {
      auto sprime = [&](int sidx) { return sidx == 0 ? q[l] : q[L + sidx - 1]; };
      auto Pp_mod = [&](u64 m) { return mulmod(prod_mod(q, L, L + K, -1, m), q[l] % m, m); };
      auto half2 = [&](u64 m) { return mulmod(submod(Pp_mod(m), 1 % m, m), (m + 1) / 2, m); };
      // P'/s mod m
      auto hat = [&](int sidx, u64 m) {
        return sidx == 0 ? prod_mod(q, L, L + K, -1, m) : mulmod(prod_mod(q, L, L + K, L + sidx - 1, m), q[l] % m, m);
      };
      for (int sidx = 0; sidx <= K; ++sidx) {
        const u64 sv = sprime(sidx);
        const u64 hinv = invmod(hat(sidx, sv), sv);
        u64* c = pk2.data() + ((std::size_t)l * kMaxK + sidx) * 4;
        c[0] = hinv;
        c[1] = shoup(hinv, sv);
        c[2] = half2(sv);
        pinv2[(std::size_t)l * kMaxK + sidx] = 1.0 / (double)sv;
      }
      for (int i = 0; i < l; ++i) {
        for (int sidx = 0; sidx <= K; ++sidx)
          phat2[((std::size_t)l * L + i) * kMaxK + sidx] = to_mont(hat(sidx, q[i]), q[i]);
        const u64 Pm = Pp_mod(q[i]);
        const u64 Pinv = invmod(Pm, q[i]);
        u64* c = mq2.data() + ((std::size_t)l * L + i) * 4;
        c[0] = to_mont(Pm, q[i]);
        c[1] = half2(q[i]);
        c[2] = Pinv;
        c[3] = shoup(Pinv, q[i]);
      }
    }
    t.md2_pk = upload(dev_allocs_, pk2, stream_);
    t.md2_pinv = upload(dev_allocs_, pinv2, stream_);
    t.md2_phat = upload(dev_allocs_, phat2, stream_);
    t.md2_q = upload(dev_allocs_, mq2, stream_);
  }

  // Rescale tables
  std::vector<u64> rs((std::size_t)L * L * 4, 0);
  for (int l = 1; l < L; ++l)
    for (int i = 0; i < l; ++i) {
      const u64 qlm = q[l] % q[i];
      const u64 inv = invmod(qlm, q[i]);
      u64* c = rs.data() + ((std::size_t)l * L + i) * 4;
      c[0] = inv;
      c[1] = shoup(inv, q[i]);
      c[2] = qlm;
    }
  t.rs = upload(dev_allocs_, rs, stream_);

  // secret key: ternary from the counter PRNG, NTT domain over all L+K primes
  if (!p.no_secret) {
    std::vector<long long> s(N, 0);
    auto prng_h = [&](u64 stream, u64 idx) {
      return mix64(prng_stream_key(p.seed, stream) ^ (idx * 0xD1B54A32D192ED03ULL + 0x8CB92BA72F3D8DD7ULL));
    };
    // sparse: candidate j -> position prng(pos_stream, j) % N if unused, sign bit 0 of
    // prng(pos_stream + 1, j); main secret streams 6/7, bootstrapping secret 8/9
    auto sparse = [&](std::vector<long long>& v, int h, u64 pos_stream) {
      int got = 0;
      for (u64 j = 0; got < h; ++j) {
        const std::size_t pos = (std::size_t)(prng_h(pos_stream, j) % N);
        if (v[pos]) continue;
        v[pos] = (prng_h(pos_stream + 1, j) & 1) ? 1 : -1;
        ++got;
      }
    };
    if (p.hamming_weight <= 0) {
      for (std::size_t k = 0; k < N; ++k) s[k] = (long long)(prng_h(kStreamSecret, k) % 3) - 1;
    } else {
      sparse(s, p.hamming_weight, 6);
    }
    auto to_ntt = [&](const std::vector<long long>& v) {
      long long* dcoef = upload(dev_allocs_, v, stream_);
      u64* sntt = nullptr;
      FHEON_CUDA(cudaMalloc(reinterpret_cast<void**>(&sntt), (std::size_t)NP * N * sizeof(u64)));
      dev_allocs_.push_back(sntt);
      coeffs_to_rns(dt_, sntt, dcoef, NP, stream_);
      LimbSet ls{};
      ls.base[0] = sntt;
      ls.nbase = 1;
      ls.blocks_per_base = 1;
      ls.block_stride = 0;
      ls.E = NP;
      ls.ell = NP;
      ls.L = L;
      ntt_forward(dt_, ls, stream_);
      return sntt;
    };
    t.s_ntt = to_ntt(s);
    if (p.bootstrap && p.hamming_weight <= 0) {
      std::vector<long long> sb(N, 0);
      sparse(sb, p.boot_hamming_weight, 8);
      t.sb_ntt = to_ntt(sb);
    }
  }
  FHEON_CUDA(cudaStreamSynchronize(stream_));
}

// ------------------------------------------------------------- keys
u64 Context::galois(long t) const {
  const long S = ht_.S;
  long r = t % S;
  if (r < 0) r += S;
  return powmod(5, (u64)r, 2 * (u64)ht_.N);
}

std::size_t Context::key_words() const {
  return (std::size_t)ht_.p.dnum * 2 * (ht_.p.L + ht_.p.K) * ht_.N;
}

const u64* Context::key(u64 key_id) {
  auto it = keys_.find(key_id);
  if (it != keys_.end()) return it->second->ptr;
  if (strict_keys) throw Error(ErrKind::internal, "evaluation key " + std::to_string(key_id) + " not resident");
  gen_key(key_id);
  return keys_.at(key_id)->ptr;
}

void Context::require_secret(const char* what) const {
  if (!has_secret())
    throw Error(ErrKind::internal, std::string(what) + ": this context holds no secret key (no_secret); upload "
                                                      "the evaluation keys (fheon_key_upload*) and encrypt / "
                                                      "decrypt on the client");
}

void Context::gen_key(u64 key_id) {
  if (keys_.count(key_id)) return;
  if (!has_secret())
    throw Error(ErrKind::internal, "evaluation key " + std::to_string(key_id) +
                                       " is not resident and this context holds no secret to generate it: upload "
                                       "it (fheon_key_upload*)");
  ++stats.key_gens;
  const Params& p = ht_.p;
  const int L = p.L, K = p.K, NP = L + K;
  const std::size_t N = ht_.N, LN = (std::size_t)NP * N;
  BufPtr kb = alloc(key_words());
  BufPtr sp = alloc(LN);
  // evk_j = (-a_j s_to + e_j + [i in D_j] P s_from, a_j): s_from = s^2 (relinearisation),
  // sigma_g(s) (rotation), s (-> sparse) or s_b (<- sparse); s_to = s except for the
  // switch to the sparse bootstrapping secret
  const u64* s_to = dt_.s_ntt;
  const bool sse_key = key_id == kKeyToSparse || key_id == kKeyFromSparse || is_key_from_sparse_rot(key_id);
  if (sse_key && !dt_.sb_ntt) throw Error(ErrKind::internal, "no sparse bootstrapping secret in this context");
  if (key_id == 0) {
    secret_square(dt_, sp->ptr, stream_);
  } else if (key_id == kKeyToSparse) {
    FHEON_CUDA(cudaMemcpyAsync(sp->ptr, dt_.s_ntt, LN * sizeof(u64), cudaMemcpyDeviceToDevice, stream_));
    s_to = dt_.sb_ntt;
  } else if (key_id == kKeyFromSparse) {
    FHEON_CUDA(cudaMemcpyAsync(sp->ptr, dt_.sb_ntt, LN * sizeof(u64), cudaMemcpyDeviceToDevice, stream_));
  } else if (is_key_from_sparse_rot(key_id)) {  // sigma_g(s_b) -> s
    PolyList o{}, in{};
    o.p[0] = sp->ptr;
    o.g[0] = key_id >> 4;
    o.n = 1;
    in.p[0] = dt_.sb_ntt;
    in.n = 1;
    automorph(dt_, o, in, NP, stream_);
  } else {
    if ((key_id & 1) == 0) throw Error(ErrKind::internal, "Galois element must be odd");
    PolyList o{}, in{};
    o.p[0] = sp->ptr;
    o.g[0] = key_id;
    o.n = 1;
    in.p[0] = dt_.s_ntt;
    in.n = 1;
    automorph(dt_, o, in, NP, stream_);
  }
  std::vector<u64> pmod(NP, 0);
  for (int i = 0; i < NP; ++i) pmod[i] = prod_mod(ht_.q, L, L + K, -1, ht_.q[i]);
  BufPtr dpm = alloc(NP);
  FHEON_CUDA(cudaMemcpyAsync(dpm->ptr, pmod.data(), NP * sizeof(u64), cudaMemcpyHostToDevice, stream_));
  BufPtr e = alloc(LN);
  LimbSet ls{};
  ls.base[0] = e->ptr;
  ls.nbase = 1;
  ls.blocks_per_base = 1;
  ls.E = NP;
  ls.ell = NP;
  ls.L = L;
  if (key_id == kKeyToSparse)  // only digit 0's q_0 and P limbs are ever read (level 0)
    FHEON_CUDA(cudaMemsetAsync(kb->ptr, 0, key_words() * sizeof(u64), stream_));
  for (int j = 0; j < (key_id == kKeyToSparse ? 1 : p.dnum); ++j) {  // digits past ndig stay empty (lo = hi = L)
    const int lo = j < ht_.ndig ? ht_.dig[j] : L, hi = j < ht_.ndig ? ht_.dig[j + 1] : L;
    sample_error(dt_, e->ptr, prng_stream_key(p.seed, stream_key(key_id, j, 3)), NP, NP, stream_);
    ntt_forward(dt_, ls, stream_);
    u64* b = kb->ptr + (std::size_t)(j * 2) * LN;
    u64* a = b + LN;
    keygen_digit(dt_, b, a, e->ptr, sp->ptr, s_to, prng_stream_key(p.seed, stream_key(key_id, j, 2)), lo, hi,
                 dpm->ptr, stream_);
    if (key_id == kKeyToSparse) {  // the sparse-secret sample exists on q_0 and P only
      FHEON_CUDA(cudaMemsetAsync(b + N, 0, (std::size_t)(L - 1) * N * sizeof(u64), stream_));
      FHEON_CUDA(cudaMemsetAsync(a + N, 0, (std::size_t)(L - 1) * N * sizeof(u64), stream_));
    }
  }
  FHEON_CUDA(cudaStreamSynchronize(stream_));  // pmod host vector goes out of scope
  keys_[key_id] = kb;
}

// ------------------------------------------------------------- encoder
void Context::encode_coeffs(const double* vals, std::size_t n, double scale, long long* coeffs) const {
  encode_coeffs_host(ht_, vals, n, scale, coeffs);
}

namespace {
// special inverse FFT of the zero-filled slot vector (imaginary parts optional)
void fft_special_inv_host(const HostTables& ht_, const double* vals, std::size_t n, std::vector<double>& re,
                          std::vector<double>& im, const double* ivals = nullptr);
}  // namespace

void encode_complex_coeffs_host(const HostTables& ht_, const double* re_in, const double* im_in, std::size_t n,
                                double scale, long long* coeffs) {
  std::vector<double> re, im;
  fft_special_inv_host(ht_, re_in, n, re, im, im_in);
  const int S = ht_.S;
  const double lim = 4611686018427387904.0;
  for (int i = 0; i < S; ++i) {
    const double a = (re[i] / (double)S) * scale, b = (im[i] / (double)S) * scale;
    if (!(std::fabs(a) < lim) || !(std::fabs(b) < lim))
      throw Error(ErrKind::capacity, "encoded value exceeds the 2^62 coefficient range");
    coeffs[i] = std::llround(a);
    coeffs[i + S] = std::llround(b);
  }
}

BufPtr Context::encode_complex(const double* re, const double* im, std::size_t n, int limbs, double scale,
                               int special) {
  const std::size_t N = ht_.N;
  BufPtr out = alloc((std::size_t)(limbs + special) * N);
  ++stats.encodes;
  BufPtr dcoef = encode_device(re, im, n, scale);
  coeffs_to_rns(dt_, out->ptr, reinterpret_cast<const long long*>(dcoef->ptr), limbs, stream_);
  if (special > 0)
    coeffs_to_rns(dt_, out->ptr + (std::size_t)limbs * N, reinterpret_cast<const long long*>(dcoef->ptr), special,
                  stream_, ht_.p.L);
  LimbSet ls{};
  ls.base[0] = out->ptr;
  ls.nbase = 1;
  ls.blocks_per_base = 1;
  ls.E = limbs + special;
  ls.ell = limbs;
  ls.L = ht_.p.L;
  ntt_forward(dt_, ls, stream_);
  return out;
}

void encode_real_host(const HostTables& ht_, const double* vals, std::size_t n, double* out) {
  std::vector<double> re, im;
  fft_special_inv_host(ht_, vals, n, re, im);
  const int S = ht_.S;
  for (int i = 0; i < S; ++i) {
    out[i] = re[i] / (double)S;
    out[i + S] = im[i] / (double)S;
  }
}

namespace {
void fft_special_inv_host(const HostTables& ht_, const double* vals, std::size_t n, std::vector<double>& re,
                          std::vector<double>& im, const double* ivals) {
  const int S = ht_.S;
  if (n > (std::size_t)S) throw Error(ErrKind::capacity, "payload exceeds the slot count");
  const u64 M = 2 * (u64)ht_.N;
  re.assign(S, 0.0);
  im.assign(S, 0.0);
  for (std::size_t i = 0; i < n; ++i) re[i] = vals[i];
  if (ivals)
    for (std::size_t i = 0; i < n; ++i) im[i] = ivals[i];
  for (int len = S; len >= 1; len >>= 1) {
    const int lenh = len >> 1;
    const u64 lenq = (u64)len << 2;
    for (int i = 0; i < S; i += len) {
      for (int j = 0; j < lenh; ++j) {
        const u64 idx = (lenq - (ht_.rotgroup[j] % lenq)) * (M / lenq);
        const double ur = re[i + j] + re[i + j + lenh];
        const double ui = im[i + j] + im[i + j + lenh];
        const double vr0 = re[i + j] - re[i + j + lenh];
        const double vi0 = im[i + j] - im[i + j + lenh];
        const double wr = ht_.ksi_re[idx], wi = ht_.ksi_im[idx];
        re[i + j] = ur;
        im[i + j] = ui;
        re[i + j + lenh] = vr0 * wr - vi0 * wi;
        im[i + j + lenh] = vr0 * wi + vi0 * wr;
      }
    }
  }
  for (int i = 1, j = 0; i < S; ++i) {
    int bit = S >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      std::swap(re[i], re[j]);
      std::swap(im[i], im[j]);
    }
  }
}
}  // namespace

void encode_coeffs_host(const HostTables& ht_, const double* vals, std::size_t n, double scale, long long* coeffs) {
  const int S = ht_.S;
  if (n > (std::size_t)S) throw Error(ErrKind::capacity, "payload exceeds the slot count");
  const u64 M = 2 * (u64)ht_.N;
  std::vector<double> re(S, 0.0), im(S, 0.0);
  for (std::size_t i = 0; i < n; ++i) re[i] = vals[i];
  for (int len = S; len >= 1; len >>= 1) {
    const int lenh = len >> 1;
    const u64 lenq = (u64)len << 2;
    for (int i = 0; i < S; i += len) {
      for (int j = 0; j < lenh; ++j) {
        const u64 idx = (lenq - (ht_.rotgroup[j] % lenq)) * (M / lenq);
        const double ur = re[i + j] + re[i + j + lenh];
        const double ui = im[i + j] + im[i + j + lenh];
        const double vr0 = re[i + j] - re[i + j + lenh];
        const double vi0 = im[i + j] - im[i + j + lenh];
        const double wr = ht_.ksi_re[idx], wi = ht_.ksi_im[idx];
        re[i + j] = ur;
        im[i + j] = ui;
        re[i + j + lenh] = vr0 * wr - vi0 * wi;
        im[i + j + lenh] = vr0 * wi + vi0 * wr;
      }
    }
  }
  // bit reversal
  for (int i = 1, j = 0; i < S; ++i) {
    int bit = S >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      std::swap(re[i], re[j]);
      std::swap(im[i], im[j]);
    }
  }
  const double lim = 4611686018427387904.0;  // 2^62
  for (int i = 0; i < S; ++i) {
    const double a = (re[i] / (double)S) * scale, b = (im[i] / (double)S) * scale;
    if (!(std::fabs(a) < lim) || !(std::fabs(b) < lim))
      throw Error(ErrKind::capacity, "encoded value exceeds the 2^62 coefficient range");
    coeffs[i] = std::llround(a);
    coeffs[i + S] = std::llround(b);
  }
}

void Context::decode_coeffs(const double* coeffs, double scale, double* out, double* out_im) const {
  const int S = ht_.S;
  const u64 M = 2 * (u64)ht_.N;
  std::vector<double> re(S), im(S);
  for (int i = 0; i < S; ++i) {
    re[i] = coeffs[i] / scale;
    im[i] = coeffs[i + S] / scale;
  }
  for (int i = 1, j = 0; i < S; ++i) {
    int bit = S >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      std::swap(re[i], re[j]);
      std::swap(im[i], im[j]);
    }
  }
  for (int len = 2; len <= S; len <<= 1) {
    const int lenh = len >> 1;
    const u64 lenq = (u64)len << 2;
    for (int i = 0; i < S; i += len) {
      for (int j = 0; j < lenh; ++j) {
        const u64 idx = (ht_.rotgroup[j] % lenq) * (M / lenq);
        const double wr = ht_.ksi_re[idx], wi = ht_.ksi_im[idx];
        const double ur = re[i + j], ui = im[i + j];
        const double xr = re[i + j + lenh], xi = im[i + j + lenh];
        const double vr = xr * wr - xi * wi;
        const double vi = xr * wi + xi * wr;
        re[i + j] = ur + vr;
        im[i + j] = ui + vi;
        re[i + j + lenh] = ur - vr;
        im[i + j + lenh] = ui - vi;
      }
    }
  }
  for (int i = 0; i < S; ++i) out[i] = re[i];
  if (out_im)
    for (int i = 0; i < S; ++i) out_im[i] = im[i];
}

const double* Context::basis(const std::string& key, const std::vector<double>& slot_values) {
  auto it = basis_.find(key);
  if (it != basis_.end()) return reinterpret_cast<const double*>(it->second->ptr);
  std::vector<double> real(ht_.N);
  encode_real_host(ht_, slot_values.data(), slot_values.size(), real.data());
  BufPtr b = alloc(ht_.N);
  FHEON_CUDA(cudaMemcpyAsync(b->ptr, real.data(), ht_.N * sizeof(double), cudaMemcpyHostToDevice, stream_));
  FHEON_CUDA(cudaStreamSynchronize(stream_));  // `real` is pageable and local
  basis_[key] = b;
  return reinterpret_cast<const double*>(b->ptr);
}

const double* Context::basis(const std::string& key, const std::function<std::vector<double>()>& make) {
  auto it = basis_.find(key);
  if (it != basis_.end()) return reinterpret_cast<const double*>(it->second->ptr);
  return basis(key, make());
}

BufPtr Context::encode_lincomb(const LinComb& lc, int limbs, double scale) {
  BufPtr out = alloc((std::size_t)limbs * ht_.N);
  ++stats.encodes;
  fheon::encode_lincomb(dt_, out->ptr, lc, scale, limbs, stream_);
  LimbSet ls{};
  ls.base[0] = out->ptr;
  ls.nbase = 1;
  ls.blocks_per_base = 1;
  ls.E = limbs;
  ls.ell = limbs;
  ls.L = ht_.p.L;
  ntt_forward(dt_, ls, stream_);
  return out;
}

BufPtr Context::encode_cached(const std::vector<double>& vals, int limbs, double scale) {
  u64 h = 1469598103934665603ULL;  // FNV-1a over the bit patterns
  for (double v : vals) {
    u64 b;
    std::memcpy(&b, &v, 8);
    h = (h ^ b) * 1099511628211ULL;
  }
  auto key = std::make_tuple(h, limbs, scale);
  auto& bucket = ptcache_[key];
  for (const PtEntry& e : bucket)
    if (e.vals == vals) return e.buf;
  BufPtr b = encode(vals.data(), vals.size(), limbs, scale);
  ptcache_reserve((std::size_t)limbs * ht_.N);
  ptcache_[key].push_back({vals, b});
  return b;
}

BufPtr Context::encode_named(const std::string& name, const std::function<std::vector<double>()>& make, int limbs,
                             double scale) {
  auto key = std::make_tuple(name, limbs, scale);
  auto it = namedcache_.find(key);
  if (it != namedcache_.end()) return it->second;
  const std::vector<double> vals = make();
  BufPtr b = encode(vals.data(), vals.size(), limbs, scale);
  ptcache_reserve((std::size_t)limbs * ht_.N);
  namedcache_[key] = b;
  return b;
}

BufPtr Context::weight_pt(const std::string& key, int limbs, double scale, const std::function<BufPtr()>& make) {
  if (weight_cache_budget == 0) return make();
  auto k = std::make_tuple(key, limbs, scale);
  auto it = weightcache_.find(k);
  if (it != weightcache_.end()) return it->second;
  BufPtr b = make();
  const std::size_t bytes = (std::size_t)limbs * ht_.N * sizeof(u64);
  if (weightcache_bytes_ + bytes <= weight_cache_budget) {
    weightcache_[k] = b;
    weightcache_bytes_ += bytes;
  }
  return b;
}

// cached plaintexts stay resident up to 24 GiB of HBM (mask sets of the
// baby-step giant-step schedules run to a few GiB at N = 2^16); past that the
// caches start over
void Context::ptcache_reserve(std::size_t words) {
  const std::size_t budget = (std::size_t)3 << 30;
  if (ptcache_words_ + words > budget) {
    ptcache_.clear();
    namedcache_.clear();
    ptcache_words_ = 0;
  }
  ptcache_words_ += words;
}

long long* Context::staging_slot(cudaEvent_t** ev) {
  const int i = staging_next_;
  staging_next_ = (staging_next_ + 1) % kStaging;
  FHEON_CUDA(cudaEventSynchronize(staging_ev_[i]));
  *ev = &staging_ev_[i];
  return staging_[i];
}

namespace {
bool constant_value(const double* vals, std::size_t n, int S, double* c) {
  if (n == 0) {
    *c = 0.0;
    return true;
  }
  for (std::size_t i = 1; i < n; ++i)
    if (vals[i] != vals[0]) return false;
  if (n < (std::size_t)S && vals[0] != 0.0) return false;
  *c = vals[0];
  return true;
}
}  // namespace

// slot values -> N signed coefficients on the device (encode.cu): the values ride the
// pinned staging ring to the device, the special FFT runs there
BufPtr Context::encode_device(const double* re, const double* im, std::size_t n, double scale) {
  const std::size_t N = ht_.N, S = (std::size_t)ht_.S;
  if (n > S) throw Error(ErrKind::capacity, "payload exceeds the slot count");
  // every coefficient is an average of the slot values times unit roots: |c| <= max|v| * scale
  double mx = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    mx = std::max(mx, std::fabs(re[i]));
    if (im) mx = std::max(mx, std::fabs(im[i]));
  }
  if (!(mx * std::fabs(scale) < 4611686018427387904.0))
    throw Error(ErrKind::capacity, "encoded value exceeds the 2^62 coefficient range");
  BufPtr work = alloc(N);  // [re S][im S] doubles
  FHEON_CUDA(cudaMemsetAsync(work->ptr, 0, N * sizeof(u64), stream_));
  cudaEvent_t* ev = nullptr;
  long long* h = staging_slot(&ev);
  double* hd = reinterpret_cast<double*>(h);
  std::memcpy(hd, re, n * sizeof(double));
  if (im) std::memcpy(hd + S, im, n * sizeof(double));
  FHEON_CUDA(cudaMemcpyAsync(work->ptr, hd, n * sizeof(double), cudaMemcpyHostToDevice, stream_));
  if (im)
    FHEON_CUDA(cudaMemcpyAsync(work->ptr + S, hd + S, n * sizeof(double), cudaMemcpyHostToDevice, stream_));
  FHEON_CUDA(cudaEventRecord(*ev, stream_));
  BufPtr dcoef = alloc(N);
  encode_fft_device(dt_, reinterpret_cast<long long*>(dcoef->ptr), reinterpret_cast<double*>(work->ptr), scale,
                    stream_);
  return dcoef;
}

BufPtr Context::encode(const double* vals, std::size_t n, int limbs, double scale) {
  const std::size_t N = ht_.N;
  BufPtr out = alloc((std::size_t)limbs * N);
  ++stats.encodes;
  double cv;
  if (constant_value(vals, n, ht_.S, &cv)) {
    const double x = cv * scale;
    if (!(std::fabs(x) < 4611686018427387904.0)) throw Error(ErrKind::capacity, "constant exceeds 2^62");
    const long long k = std::llround(x);
    FHEON_CUDA(cudaMemsetAsync(out->ptr, 0, (std::size_t)limbs * N * sizeof(u64), stream_));
    LimbConsts lc{};
    for (int i = 0; i < limbs; ++i) {
      const u64 q = ht_.q[i];
      lc.c[i] = k >= 0 ? (u64)k % q : (q - 1 - (u64)(-(k + 1)) % q);
    }
    PolyList o{};
    o.p[0] = out->ptr;
    o.n = 1;
    ew_add_const(dt_, o, o, lc, limbs, stream_);
    return out;
  }
  BufPtr dcoef = encode_device(vals, nullptr, n, scale);
  coeffs_to_rns(dt_, out->ptr, reinterpret_cast<const long long*>(dcoef->ptr), limbs, stream_);
  LimbSet ls{};
  ls.base[0] = out->ptr;
  ls.nbase = 1;
  ls.blocks_per_base = 1;
  ls.E = limbs;
  ls.ell = limbs;
  ls.L = ht_.p.L;
  ntt_forward(dt_, ls, stream_);
  return out;
}

// ------------------------------------------------------------- trace
void Context::record(int kind, long value, const std::string& label) {
  if (!tracing_) return;
  std::lock_guard<std::mutex> g(trace_mu_);
  trace_.push_back({kind, value, label});
}
std::vector<TraceEvent> Context::trace_snapshot() const {
  std::lock_guard<std::mutex> g(trace_mu_);
  return trace_;
}
void Context::clear_trace() {
  std::lock_guard<std::mutex> g(trace_mu_);
  trace_.clear();
}

}  // namespace fheon
