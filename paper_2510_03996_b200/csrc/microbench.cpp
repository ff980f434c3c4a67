// Config-2 primitive microbench (BASELINE.json configs[1]): times batched
// launches of each RNS primitive on the context stream with CUDA events.
#include <cuda_runtime.h>

#include <random>

#include "layers.hpp"

namespace fheon {

double microbench(Context& ctx, int kind, int batch, int limbs, int n_rot, int iters) {
  if (limbs < 2 || limbs > ctx.L()) throw Error(ErrKind::shape, "microbench: limbs out of range");
  if (batch < 1 || batch > (kind == 8 ? 64 : kMaxBases)) throw Error(ErrKind::shape, "microbench: batch out of range");
  cudaStream_t st = ctx.stream();
  const DevTables& t = ctx.dev();
  const std::size_t N = ctx.N();
  std::vector<double> vals(ctx.S());
  std::mt19937_64 rng(2001);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (double& v : vals) v = u(rng);
  std::vector<Ciphertext> cts;
  const int ncts = kind == 9 ? std::max(batch, n_rot) : batch;  // MAC: k distinct terms
  for (int b = 0; b < ncts; ++b) cts.push_back(encrypt_at(ctx, vals.data(), vals.size(), limbs));
  BufPtr pt = ctx.encode(vals.data(), vals.size(), limbs, ctx.host().T[limbs - 1]);
  std::vector<long> steps;
  for (int r = 0; r < std::max(1, n_rot); ++r) steps.push_back(1L << (r % 15));
  if (kind == 3 || kind == 4 || kind == 8)
    for (long s : steps) ctx.gen_key(ctx.galois(s));
  // kind 9: the fused MAC sum_j pt_j (*) ct_j over k = n_rot terms (distinct plaintexts)
  std::vector<BufPtr> mac_pts;
  if (kind == 9)
    for (int j = 0; j < std::max(1, n_rot); ++j) {
      for (double& v : vals) v = u(rng);
      mac_pts.push_back(ctx.encode(vals.data(), vals.size(), limbs, pt_scale_for(ctx, cts[0])));
    }
  // kind 10: the automorphism for every rotation step t in [1, S) (keyless permutation)
  long auto_t = 1;
  std::vector<Ciphertext> keep;
  auto run = [&]() {
    keep.clear();
    switch (kind) {
      case 0:
      case 1: {
        LimbSet s{};
        s.nbase = batch;
        for (int b = 0; b < batch; ++b) s.base[b] = cts[b].c0;
        s.blocks_per_base = 2;
        s.block_stride = (long long)(cts[0].c1 - cts[0].c0);
        s.E = limbs;
        s.ell = limbs;
        s.L = ctx.L();
        if (kind == 0) ntt_forward(t, s, st);
        else ntt_inverse(t, s, st);
        break;
      }
      case 2: {
        PolyList o{}, in{};
        std::vector<BufPtr> outs;
        for (int b = 0; b < batch; ++b) {
          outs.push_back(ctx.alloc(2 * (std::size_t)limbs * N));
          for (int p = 0; p < 2; ++p) {
            in.p[2 * b + p] = p ? cts[b].c1 : cts[b].c0;
            o.p[2 * b + p] = outs.back()->ptr + (std::size_t)p * limbs * N;
            o.g[2 * b + p] = ctx.galois(5);
          }
        }
        o.n = in.n = 2 * batch;
        automorph(t, o, in, limbs, st);
        break;
      }
      case 3:
        for (int b = 0; b < batch; ++b) keep.push_back(rotate(ctx, cts[b], steps[0]));
        break;
      case 4:
        for (int b = 0; b < batch; ++b) {
          std::vector<Ciphertext> r = rotate_hoisted(ctx, cts[b], steps);
          keep.insert(keep.end(), r.begin(), r.end());
        }
        break;
      case 5: {
        PolyList o{}, a{};
        std::vector<Ciphertext> outs;
        for (int b = 0; b < batch; ++b) {
          outs.push_back(ctx.new_ct(limbs));
          o.p[2 * b] = outs.back().c0;
          o.p[2 * b + 1] = outs.back().c1;
          a.p[2 * b] = cts[b].c0;
          a.p[2 * b + 1] = cts[b].c1;
        }
        o.n = a.n = 2 * batch;
        ew_mul_pt(t, o, a, pt->ptr, limbs, st);
        keep = outs;
        break;
      }
      case 6:
        for (int b = 0; b < batch; ++b) keep.push_back(rescale(ctx, cts[b]));
        break;
      case 7:
        for (int b = 0; b < batch; ++b) keep.push_back(add(ctx, cts[b], cts[(b + 1) % batch]));
        break;
      case 8:  // batch of `batch` distinct ciphertexts rotated by the SAME step: one key read per launch
        keep = rotate_many(ctx, cts, std::vector<long>(batch, steps[0]));
        break;
      case 9: {
        std::vector<Ciphertext> terms(cts.begin(), cts.begin() + std::max(1, n_rot));
        keep = mac_plain_many(ctx, {terms}, {mac_pts});
        break;
      }
      case 10: {
        PolyList o{}, in{};
        BufPtr out = ctx.alloc(2 * (std::size_t)limbs * N);
        for (int p = 0; p < 2; ++p) {
          in.p[p] = p ? cts[0].c1 : cts[0].c0;
          o.p[p] = out->ptr + (std::size_t)p * limbs * N;
          o.g[p] = ctx.galois(auto_t);
        }
        o.n = in.n = 2;
        automorph(t, o, in, limbs, st);
        auto_t = auto_t % (ctx.S() - 1) + 1;
        break;
      }
      default:
        throw Error(ErrKind::shape, "microbench: unknown kind");
    }
  };
  run();
  FHEON_CUDA(cudaStreamSynchronize(st));
  cudaEvent_t e0, e1;
  FHEON_CUDA(cudaEventCreate(&e0));
  FHEON_CUDA(cudaEventCreate(&e1));
  FHEON_CUDA(cudaEventRecord(e0, st));
  for (int i = 0; i < iters; ++i) run();
  FHEON_CUDA(cudaEventRecord(e1, st));
  FHEON_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  FHEON_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (double)ms / iters;
}

}  // namespace fheon
