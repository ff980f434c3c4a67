// Layer algorithms over device ciphertexts.  Each function follows the
// reference's algorithm op for op (cited per function) so rotation indices,
// mask values, level consumption and trace events are identical; the GPU
// realisation hoists rotation sets that share a source ciphertext.
#include "layers.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <string>

namespace fheon {

namespace {

bool is_pow2(std::size_t v) { return v != 0 && (v & (v - 1)) == 0; }
std::size_t log2_exact(std::size_t v) {
  std::size_t l = 0;
  while ((std::size_t{1} << l) < v) ++l;
  return l;
}

Error shape_error(const std::string& m) { return Error(ErrKind::shape, m); }
Error capacity_error(const std::string& m) { return Error(ErrKind::capacity, m); }

// PlainVector::from_values(S, v) (backend.cpp:114-125): zero-filled to S
std::vector<double> plain(const Context& ctx, const std::vector<double>& v) {
  if (v.size() > (std::size_t)ctx.S())
    throw capacity_error("plain vector payload of " + std::to_string(v.size()) + " values does not fit in " +
                         std::to_string(ctx.S()) + " slots");
  std::vector<double> out(ctx.S(), 0.0);
  std::copy(v.begin(), v.end(), out.begin());
  return out;
}

// range_mask (layers_conv.cpp:39-44, layers_misc.cpp:21-26)
std::vector<double> range_mask(const Context& ctx, std::size_t begin, std::size_t count, double value = 1.0) {
  std::vector<double> v(begin + count, 0.0);
  std::fill(v.begin() + (long)begin, v.end(), value);
  return plain(ctx, v);
}

Ciphertext mp(Context& ctx, const Ciphertext& x, const std::vector<double>& full) {
  return mult_plain(ctx, x, full.data(), full.size());
}

void check_stride_geometry(const Context& ctx, const Ciphertext& a, std::size_t W, std::size_t S, std::size_t W_out) {
  if (!a.valid()) throw Error(ErrKind::internal, "striding: operand is not initialized");
  if (W == 0 || S == 0 || W_out == 0) throw shape_error("striding: width, stride and output edge must be positive");
  if ((W_out - 1) * S + 1 > W)
    throw shape_error("striding: output edge " + std::to_string(W_out) + " at stride " + std::to_string(S) +
                      " overruns input edge " + std::to_string(W));
  if (W * W > (std::size_t)ctx.S())
    throw capacity_error("striding: block of edge " + std::to_string(W) + " exceeds the slot count");
}

// bias_vector (layers_conv.cpp:77-85) added as a plaintext at the operand's level
Ciphertext add_bias(Context& ctx, const Ciphertext& out, const std::vector<double>& bias, std::size_t block) {
  std::vector<double> v(bias.size() * block);
  for (std::size_t f = 0; f < bias.size(); ++f)
    std::fill(v.begin() + (long)(f * block), v.begin() + (long)((f + 1) * block), bias[f]);
  if (v.size() > (std::size_t)ctx.S()) throw capacity_error("bias does not fit in the slot count");
  return add_plain(ctx, out, v.data(), v.size());
}

std::vector<double> member_kernel_vector(const KernelTensor& w, std::size_t f, std::size_t ti, std::size_t tj,
                                         std::size_t c, std::size_t C, std::size_t W) {
  const std::size_t block = W * W;
  std::vector<double> out(C * block, 0.0);
  const double v = w.at(f, 0, ti, tj);
  std::fill(out.begin() + (long)(c * block), out.begin() + (long)((c + 1) * block), v);
  return out;
}

// tap_rotations (layers_conv.cpp:102-113): one hoisted ModUp for all k^2-1 taps
std::vector<Ciphertext> tap_rotations(Context& ctx, const Ciphertext& x, std::size_t k, std::size_t W) {
  std::vector<long> ts;
  for (std::size_t i = 0; i < k; ++i)
    for (std::size_t j = 0; j < k; ++j)
      if (i * W + j != 0) ts.push_back((long)(i * W + j));
  std::vector<Ciphertext> r = rotate_hoisted(ctx, x, ts);
  std::vector<Ciphertext> taps;
  taps.reserve(k * k);
  taps.push_back(x);
  for (Ciphertext& c : r) taps.push_back(c);
  return taps;
}

// Channel accumulation chain (layers_conv.cpp:155-161): C-1 rotations by m
Ciphertext channel_accumulate(Context& ctx, Ciphertext sum, std::size_t C, std::size_t m) {
  if (C > 1) {
    Ciphertext cur = sum;
    for (std::size_t c = 1; c < C; ++c) {
      cur = rotate(ctx, cur, (long)m);
      sum = add(ctx, sum, cur);
    }
  }
  return sum;
}

// conv_core_generic (layers_conv.cpp:117-180)
PackedTensor conv_core_generic(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  const std::size_t W = x.width, C = x.channels;
  const std::size_t F = cfg.out_channels, k = cfg.kernel, S = cfg.stride;
  if (cfg.in_channels != C)
    throw shape_error("convolution expects " + std::to_string(cfg.in_channels) + " input channels, tensor has " +
                      std::to_string(C));
  if (w.in_channels != C || w.out_channels != F || w.kernel != k)
    throw shape_error("kernel tensor shape does not match the layer config");
  const std::size_t W_out = conv_output_width(W, k, S, 0);
  const std::size_t m = W * W;
  if (F * W_out * W_out > (std::size_t)ctx.S())
    throw capacity_error("convolution output needs " + std::to_string(F * W_out * W_out) +
                         " slots but the context provides " + std::to_string(ctx.S()));
  const std::vector<Ciphertext> taps = tap_rotations(ctx, x.data, k, W);
  const std::vector<double> cleanup = plain(ctx, extraction_mask(W, C));
  Ciphertext out;
  for (std::size_t f = 0; f < F; ++f) {
    Ciphertext sum;
    for (std::size_t i = 0; i < k; ++i)
      for (std::size_t j = 0; j < k; ++j) {
        const Ciphertext term = mp(ctx, taps[i * k + j], plain(ctx, repeated_kernel_vector(w, f, i, j, C, W)));
        sum = (i == 0 && j == 0) ? term : add(ctx, sum, term);
      }
    sum = channel_accumulate(ctx, sum, C, m);
    const Ciphertext a_star = mp(ctx, sum, cleanup);
    Ciphertext r_f;
    if (S == 1 && W_out == W) r_f = a_star;
    else if (cfg.stride_variant == 1) r_f = stride_extract_v2(ctx, a_star, W, S, W_out);
    else r_f = stride_extract_v1(ctx, a_star, W, S, W_out);
    out = (f == 0) ? r_f : add(ctx, out, rotate(ctx, r_f, -(long)(f * W_out * W_out)));
  }
  out = add_bias(ctx, out, w.bias, W_out * W_out);
  return {out, F, W_out};
}

// conv_grouped_fallback (layers_conv.cpp:184-216)
PackedTensor conv_grouped_fallback(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w,
                                   std::size_t W_out) {
  const std::size_t W = x.width, g = x.channels;
  const std::size_t F = cfg.out_channels, k = cfg.kernel, S = cfg.stride;
  const std::size_t m = W * W;
  const std::vector<Ciphertext> taps = tap_rotations(ctx, x.data, k, W);
  Ciphertext out;
  for (std::size_t f = 0; f < F; ++f) {
    const std::size_t c = f % g;
    Ciphertext sum;
    for (std::size_t i = 0; i < k; ++i)
      for (std::size_t j = 0; j < k; ++j) {
        const Ciphertext term = mp(ctx, taps[i * k + j], plain(ctx, member_kernel_vector(w, f, i, j, c, g, W)));
        sum = (i == 0 && j == 0) ? term : add(ctx, sum, term);
      }
    if (c > 0) sum = rotate(ctx, sum, (long)(c * m));
    const Ciphertext r_f = stride_extract_v1(ctx, sum, W, S, W_out);
    out = (f == 0) ? r_f : add(ctx, out, rotate(ctx, r_f, -(long)(f * W_out * W_out)));
  }
  out = add_bias(ctx, out, w.bias, W_out * W_out);
  return {out, F, W_out};
}

}  // namespace

KernelTensor KernelTensor::from(const ConvConfig& cfg, const double* w, const double* bias) {
  KernelTensor k;
  k.out_channels = cfg.out_channels;
  k.in_channels = cfg.mode == 2 ? 1 : cfg.in_channels;
  k.kernel = cfg.kernel;
  const std::size_t nw = k.out_channels * k.in_channels * k.kernel * k.kernel;
  if (!w && nw) throw Error(ErrKind::internal, "kernel weights are null");
  k.weights.assign(w, w + nw);
  k.bias.assign(k.out_channels, 0.0);
  if (bias) std::copy(bias, bias + k.out_channels, k.bias.begin());
  return k;
}

// ------------------------------------------------------------- packing
std::vector<double> repeated_kernel_vector(const KernelTensor& w, std::size_t f, std::size_t ti, std::size_t tj,
                                           std::size_t C, std::size_t W) {
  if (f >= w.out_channels || ti >= w.kernel || tj >= w.kernel) throw shape_error("kernel tap index out of range");
  if (C > w.in_channels) throw shape_error("requested more channel blocks than the kernel has input channels");
  const std::size_t block = W * W;
  std::vector<double> out(C * block, 0.0);
  for (std::size_t c = 0; c < C; ++c) {
    const double v = w.at(f, c, ti, tj);
    std::fill(out.begin() + (long)(c * block), out.begin() + (long)((c + 1) * block), v);
  }
  return out;
}

std::vector<double> build_mask(std::size_t sp, std::size_t ep, std::size_t w, std::size_t m, std::size_t t) {
  if (ep > m) throw shape_error("mask end padding exceeds the pattern length");
  std::vector<double> pattern;
  pattern.reserve(m + w + 1);
  pattern.insert(pattern.end(), sp, 0.0);
  while (pattern.size() < m - ep) {
    pattern.insert(pattern.end(), w, 1.0);
    pattern.push_back(0.0);
  }
  if (pattern.size() > m) pattern.resize(m);
  while (pattern.size() < m) pattern.push_back(0.0);
  for (std::size_t i = m - ep; i < m; ++i) pattern[i] = 0.0;
  std::vector<double> mask;
  mask.reserve(m * t);
  for (std::size_t r = 0; r < t; ++r) mask.insert(mask.end(), pattern.begin(), pattern.end());
  return mask;
}

std::array<std::vector<double>, 9> build_all_masks(std::size_t m, std::size_t C, std::size_t W) {
  return {build_mask(W + 1, 0, W - 1, m, C), build_mask(W, 0, m, m, C),         build_mask(W, 0, W - 1, m, C),
          build_mask(1, 0, W - 1, m, C),     build_mask(0, 0, m, m, C),         build_mask(0, 1, W - 1, m, C),
          build_mask(1, W - 1, W - 1, m, C), build_mask(0, W, m, m, C),         build_mask(0, W + 1, W - 1, m, C)};
}

std::vector<double> extraction_mask(std::size_t W, std::size_t C) {
  std::vector<double> v(C * W * W, 0.0);
  std::fill(v.begin(), v.begin() + (long)(W * W), 1.0);
  return v;
}

// ------------------------------------------------------------- geometry
std::size_t conv_output_width(std::size_t W, std::size_t k, std::size_t S, std::size_t P) {
  if (k == 0 || S == 0) throw shape_error("kernel and stride must be positive");
  const std::size_t Wp = W + 2 * P;
  if (k > Wp) throw shape_error("kernel edge " + std::to_string(k) + " exceeds padded input edge " + std::to_string(Wp));
  if ((Wp - k) % S != 0)
    throw shape_error("geometry is not divisible: (" + std::to_string(Wp) + " - " + std::to_string(k) +
                      ") is not a multiple of stride " + std::to_string(S));
  return (Wp - k) / S + 1;
}

// pad_input (layers_conv.cpp:238-283)
PackedTensor pad_input(Context& ctx, const PackedTensor& x, std::size_t padding) {
  if (padding == 0) return x;
  const std::size_t W = x.width, C = x.channels, P = padding;
  const std::size_t Wp = W + 2 * P, mp_ = Wp * Wp;
  if (C * mp_ > (std::size_t)ctx.S())
    throw capacity_error("padded tensor needs " + std::to_string(C * mp_) + " slots but the context provides " +
                         std::to_string(ctx.S()));
  const std::vector<double> rowmask = range_mask(ctx, 0, W);
  Ciphertext out, chancur;
  for (std::size_t c = 0; c < C; ++c) {
    chancur = (c == 0) ? x.data : rotate(ctx, chancur, (long)(W * W));
    std::vector<Ciphertext> rows;
    rows.reserve(W);
    Ciphertext rowcur = chancur;
    for (std::size_t r = 0; r < W; ++r) {
      if (r > 0) rowcur = rotate(ctx, rowcur, (long)W);
      rows.push_back(mp(ctx, rowcur, rowmask));
    }
    Ciphertext racc = rows[W - 1];
    for (std::size_t r = W - 1; r-- > 0;) racc = add(ctx, rotate(ctx, racc, -(long)Wp), rows[r]);
    out = (c == 0) ? racc : add(ctx, out, rotate(ctx, racc, -(long)(c * mp_)));
  }
  out = rotate(ctx, out, -(long)(P * (Wp + 1)));
  return {out, C, Wp};
}

// stride_extract_v1 (layers_conv.cpp:289-317)
Ciphertext stride_extract_v1(Context& ctx, const Ciphertext& a_star, std::size_t W, std::size_t S, std::size_t W_out) {
  check_stride_geometry(ctx, a_star, W, S, W_out);
  Ciphertext out, vcur = a_star;
  for (std::size_t a = 0; a < W_out; ++a) {
    if (a > 0) vcur = rotate(ctx, vcur, (long)(S * W));
    Ciphertext row;
    if (S == 1) {
      row = mp(ctx, vcur, range_mask(ctx, 0, W_out));
    } else {
      row = mp(ctx, vcur, range_mask(ctx, 0, 1));
      Ciphertext hcur = vcur;
      for (std::size_t b = 1; b < W_out; ++b) {
        hcur = rotate(ctx, hcur, (long)(S - 1));
        row = add(ctx, row, mp(ctx, hcur, range_mask(ctx, b, 1)));
      }
    }
    out = (a == 0) ? row : add(ctx, out, rotate(ctx, row, -(long)(a * W_out)));
  }
  return out;
}

// stride_extract_v2 (layers_conv.cpp:323-334)
Ciphertext stride_extract_v2(Context& ctx, const Ciphertext& a_star, std::size_t W, std::size_t S, std::size_t W_out) {
  check_stride_geometry(ctx, a_star, W, S, W_out);
  if (!detail::masked_stride_applicable(W_out)) {
    ctx.record(4, 0, "striding: masked flavor needs a power-of-two output edge >= 2; using the extraction flavor");
    return stride_extract_v1(ctx, a_star, W, S, W_out);
  }
  return detail::stride_mask_compact(ctx, a_star, W, S, W_out, 1);
}

namespace detail {

bool masked_stride_applicable(std::size_t W_out) { return W_out >= 2 && is_pow2(W_out); }

int stride_mask_compact_depth(std::size_t S, std::size_t W_out) {
  return S >= 2 ? (int)log2_exact(W_out) + 1 : 2;
}

// stride_mask_compact (layers_conv.cpp:349-421)
Ciphertext stride_mask_compact(Context& ctx, const Ciphertext& y, std::size_t W, std::size_t S, std::size_t W_out,
                               std::size_t blocks) {
  check_stride_geometry(ctx, y, W, S, W_out);
  if (!masked_stride_applicable(W_out))
    throw Error(ErrKind::internal, "masked compaction requires a power-of-two output edge");
  const std::size_t m = W * W;
  if (blocks * m > (std::size_t)ctx.S() || blocks * W_out * W_out > (std::size_t)ctx.S())
    throw capacity_error("masked compaction does not fit in the slot count");
  std::vector<double> sel(blocks * m, 0.0);
  for (std::size_t c = 0; c < blocks; ++c)
    for (std::size_t a = 0; a < W_out; ++a)
      for (std::size_t b = 0; b < W_out; ++b) sel[c * m + (S * a) * W + S * b] = 1.0;
  Ciphertext cur = mp(ctx, y, plain(ctx, sel));
  if (S >= 2) {
    const std::size_t l = log2_exact(W_out);
    for (std::size_t s = 1; s < l; ++s) {
      const long amount = (long)((S - 1) << (s - 1));
      const Ciphertext merged = add(ctx, cur, rotate(ctx, cur, amount));
      std::vector<double> keep(blocks * m, 0.0);
      const std::size_t period = S << s;
      const std::size_t run = std::size_t{1} << s;
      for (std::size_t c = 0; c < blocks; ++c)
        for (std::size_t a = 0; a < W_out; ++a)
          for (std::size_t j = 0; j < W; ++j)
            if (j % period < run) keep[c * m + (S * a) * W + j] = 1.0;
      cur = mp(ctx, merged, plain(ctx, keep));
    }
    cur = add(ctx, cur, rotate(ctx, cur, (long)((S - 1) << (l - 1))));
  }
  const std::size_t step_row = S * W - W_out;
  const std::size_t step_chan = W * W - S * W * (W_out - 1) - W_out;
  Ciphertext acc, cursor = cur;
  for (std::size_t c = 0; c < blocks; ++c)
    for (std::size_t a = 0; a < W_out; ++a) {
      if (c != 0 || a != 0) {
        const std::size_t step = (a == 0) ? step_chan : step_row;
        if (step != 0) cursor = rotate(ctx, cursor, (long)step);
      }
      const std::size_t dst = (c * W_out + a) * W_out;
      const Ciphertext piece = mp(ctx, cursor, range_mask(ctx, dst, W_out));
      acc = (c == 0 && a == 0) ? piece : add(ctx, acc, piece);
    }
  return acc;
}

std::vector<long> block_sum_rotations(std::size_t span) {
  std::vector<long> amounts;
  std::size_t p = 1;
  while (p * 2 <= span) {
    amounts.push_back((long)p);
    p *= 2;
  }
  std::size_t off = 0;
  for (std::size_t bit = std::bit_width(span); bit-- > 0;)
    if ((span >> bit) & 1u) {
      if (off != 0) amounts.push_back((long)off);
      off += std::size_t{1} << bit;
    }
  std::sort(amounts.begin(), amounts.end());
  amounts.erase(std::unique(amounts.begin(), amounts.end()), amounts.end());
  return amounts;
}

// block_sum (layers_misc.cpp:66-95)
Ciphertext block_sum(Context& ctx, const Ciphertext& v, std::size_t span) {
  if (span == 0) throw shape_error("block sum requires a positive span");
  if (span > (std::size_t)ctx.S()) throw capacity_error("block sum span exceeds the slot count");
  if (span == 1) return v;
  std::vector<Ciphertext> sums{v};
  std::size_t p = 1;
  while (p * 2 <= span) {
    sums.push_back(add(ctx, sums.back(), rotate(ctx, sums.back(), (long)p)));
    p *= 2;
  }
  Ciphertext acc;
  std::size_t off = 0;
  for (std::size_t bit = std::bit_width(span); bit-- > 0;) {
    if (((span >> bit) & 1u) == 0) continue;
    const Ciphertext& part = sums[bit];
    acc = (off == 0) ? part : add(ctx, acc, rotate(ctx, part, (long)off));
    off += std::size_t{1} << bit;
  }
  return acc;
}

}  // namespace detail

// ------------------------------------------------------------- conv paths
PackedTensor conv_generic(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  if (cfg.stride != 1 || cfg.padding != 0)
    throw shape_error("the generic convolution path handles stride 1 without padding");
  return conv_core_generic(ctx, x, cfg, w);
}

// conv_special_3x3 (layers_conv.cpp:435-502)
PackedTensor conv_special_3x3(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  if (cfg.kernel != 3 || cfg.stride != 1 || cfg.padding != 1)
    throw shape_error("the shape-preserving path requires kernel 3, stride 1, padding 1");
  const std::size_t W = x.width, C = x.channels, F = cfg.out_channels;
  if (W < 2) throw shape_error("the shape-preserving path requires input edge >= 2");
  if (cfg.in_channels != C || w.in_channels != C || w.out_channels != F || w.kernel != 3)
    throw shape_error("kernel tensor shape does not match the layer config");
  const std::size_t m = W * W;
  if (F * m > (std::size_t)ctx.S()) throw capacity_error("convolution output does not fit in the slot count");
  const std::vector<Ciphertext> ud = rotate_hoisted(ctx, x.data, {-(long)W, (long)W});
  const Ciphertext& up = ud[0];
  const Ciphertext& down = ud[1];
  std::vector<Ciphertext> taps(9);
  {
    std::vector<Ciphertext> r = rotate_hoisted(ctx, up, {-1, 1});
    taps[0] = r[0];
    taps[2] = r[1];
  }
  taps[1] = up;
  {
    std::vector<Ciphertext> r = rotate_hoisted(ctx, x.data, {-1, 1});
    taps[3] = r[0];
    taps[5] = r[1];
  }
  taps[4] = x.data;
  {
    std::vector<Ciphertext> r = rotate_hoisted(ctx, down, {-1, 1});
    taps[6] = r[0];
    taps[8] = r[1];
  }
  taps[7] = down;
  const std::array<std::vector<double>, 9> masks = build_all_masks(m, C, W);
  const std::vector<double> cleanup = plain(ctx, extraction_mask(W, C));
  Ciphertext out;
  for (std::size_t f = 0; f < F; ++f) {
    Ciphertext sum;
    for (std::size_t tap = 0; tap < 9; ++tap) {
      std::vector<double> kv = repeated_kernel_vector(w, f, tap / 3, tap % 3, C, W);
      for (std::size_t i = 0; i < kv.size(); ++i) kv[i] *= masks[tap][i];
      const Ciphertext term = mp(ctx, taps[tap], plain(ctx, kv));
      sum = (tap == 0) ? term : add(ctx, sum, term);
    }
    sum = channel_accumulate(ctx, sum, C, m);
    const Ciphertext cleaned = mp(ctx, sum, cleanup);
    out = (f == 0) ? cleaned : add(ctx, out, rotate(ctx, cleaned, -(long)(f * m)));
  }
  out = add_bias(ctx, out, w.bias, m);
  return {out, F, W};
}

// conv_grouped_stride (layers_conv.cpp:504-575)
PackedTensor conv_grouped_stride(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  const std::size_t g = cfg.in_channels, F = cfg.out_channels;
  if (g < 2) throw shape_error("grouped convolution with one group degenerates to the generic path");
  if (x.channels != g) throw shape_error("grouped convolution input channel mismatch");
  if (F % g != 0) throw shape_error("grouped convolution requires out_channels divisible by groups");
  if (w.out_channels != F || w.in_channels != 1 || w.kernel != cfg.kernel)
    throw shape_error("grouped kernel tensor must be (out_channels, 1, k, k) matching the layer config");
  const PackedTensor xp = cfg.padding > 0 ? pad_input(ctx, x, cfg.padding) : x;
  const std::size_t W = xp.width, k = cfg.kernel, S = cfg.stride;
  const std::size_t W_out = conv_output_width(W, k, S, 0);
  if (F * W_out * W_out > (std::size_t)ctx.S()) throw capacity_error("convolution output does not fit in the slot count");
  if (!detail::masked_stride_applicable(W_out)) {
    ctx.record(4, 0, "grouped striding needs a power-of-two output edge >= 2; using per-member extraction");
    return conv_grouped_fallback(ctx, xp, cfg, w, W_out);
  }
  const std::vector<Ciphertext> taps = tap_rotations(ctx, xp.data, k, W);
  const std::size_t groups = F / g;
  std::vector<Ciphertext> packed;
  packed.reserve(groups);
  for (std::size_t u = 0; u < groups; ++u) {
    Ciphertext joint;
    for (std::size_t c = 0; c < g; ++c) {
      const std::size_t f = u * g + c;
      for (std::size_t i = 0; i < k; ++i)
        for (std::size_t j = 0; j < k; ++j) {
          const Ciphertext term = mp(ctx, taps[i * k + j], plain(ctx, member_kernel_vector(w, f, i, j, c, g, W)));
          joint = (c == 0 && i == 0 && j == 0) ? term : add(ctx, joint, term);
        }
    }
    packed.push_back(detail::stride_mask_compact(ctx, joint, W, S, W_out, g));
  }
  Ciphertext out = packed[groups - 1];
  for (std::size_t u = groups - 1; u-- > 0;) out = add(ctx, rotate(ctx, out, -(long)(g * W_out * W_out)), packed[u]);
  out = add_bias(ctx, out, w.bias, W_out * W_out);
  return {out, F, W_out};
}

// convolution dispatcher (layers_conv.cpp:577-594)
PackedTensor convolution(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w) {
  if (cfg.mode == 1) return conv_special_3x3(ctx, x, cfg, w);
  if (cfg.mode == 2 && cfg.in_channels != 1) return conv_grouped_stride(ctx, x, cfg, w);
  const PackedTensor xp = cfg.padding > 0 ? pad_input(ctx, x, cfg.padding) : x;
  ConvConfig inner = cfg;
  inner.padding = 0;
  return conv_core_generic(ctx, xp, inner, w);
}

// ------------------------------------------------------------- pooling
// avg_pool (layers_misc.cpp:99-144)
PackedTensor avg_pool(Context& ctx, const PackedTensor& x, std::size_t k, std::size_t S, int variant) {
  const std::size_t W = x.width, C = x.channels;
  const std::size_t W_out = conv_output_width(W, k, S, 0);
  const std::size_t m = W * W;
  if (C * W_out * W_out > (std::size_t)ctx.S()) throw capacity_error("pooling output does not fit in the slot count");
  std::vector<long> ts;
  for (std::size_t i = 0; i < k; ++i)
    for (std::size_t j = 0; j < k; ++j)
      if (i != 0 || j != 0) ts.push_back((long)(i * W + j));
  Ciphertext T = x.data;
  if (!ts.empty()) {
    const std::vector<Ciphertext> r = rotate_hoisted(ctx, x.data, ts);
    for (const Ciphertext& c : r) T = add(ctx, T, c);
  }
  const Ciphertext T2 = mp(ctx, T, range_mask(ctx, 0, C * m, 1.0 / (double)(k * k)));
  if (S == 1 && W_out == W) return {T2, C, W};
  Ciphertext out, ccur = T2;
  for (std::size_t c = 0; c < C; ++c) {
    if (c > 0) ccur = rotate(ctx, ccur, (long)m);
    const Ciphertext r_c =
        variant == 1 ? stride_extract_v2(ctx, ccur, W, S, W_out) : stride_extract_v1(ctx, ccur, W, S, W_out);
    out = (c == 0) ? r_c : add(ctx, out, rotate(ctx, r_c, -(long)(c * W_out * W_out)));
  }
  return {out, C, W_out};
}

namespace {
// merge_channel_slots (layers_misc.cpp:31-37)
Ciphertext merge_channel_slots(Context& ctx, const std::vector<Ciphertext>& pieces) {
  Ciphertext out = pieces.back();
  for (std::size_t c = pieces.size() - 1; c-- > 0;) out = add(ctx, rotate(ctx, out, -1), pieces[c]);
  return out;
}
}  // namespace

// global_avg_pool (layers_misc.cpp:146-166)
Ciphertext global_avg_pool(Context& ctx, const PackedTensor& x) {
  const std::size_t W = x.width, C = x.channels, m = W * W;
  const Ciphertext sums = detail::block_sum(ctx, x.data, m);
  const std::vector<double> head = range_mask(ctx, 0, 1, 1.0 / (double)m);
  std::vector<Ciphertext> pieces;
  Ciphertext ccur = sums;
  for (std::size_t c = 0; c < C; ++c) {
    if (c > 0) ccur = rotate(ctx, ccur, (long)m);
    pieces.push_back(mp(ctx, ccur, head));
  }
  return merge_channel_slots(ctx, pieces);
}

// whole_channel_pool (layers_misc.cpp:168-195)
Ciphertext whole_channel_pool(Context& ctx, const PackedTensor& x, std::size_t k) {
  if (k != x.width) throw shape_error("whole-channel pooling requires the window to span the full channel edge");
  const std::size_t W = x.width, C = x.channels, m = W * W;
  const Ciphertext v = mp(ctx, x.data, range_mask(ctx, 0, C * m, 1.0 / (double)(k * k)));
  const Ciphertext sums = detail::block_sum(ctx, v, m);
  const std::vector<double> head = range_mask(ctx, 0, 1);
  std::vector<Ciphertext> pieces;
  Ciphertext ccur = sums;
  for (std::size_t c = 0; c < C; ++c) {
    if (c > 0) ccur = rotate(ctx, ccur, (long)m);
    pieces.push_back(mp(ctx, ccur, head));
  }
  return merge_channel_slots(ctx, pieces);
}

// ------------------------------------------------------------- FC
// fully_connected (layers_misc.cpp:197-255)
Ciphertext fully_connected(Context& ctx, const Ciphertext& x, std::size_t n, std::size_t m, std::size_t B,
                           const double* w, const double* bias) {
  if (n == 0 || m == 0) throw shape_error("fully-connected layer needs positive input/output sizes");
  if (n > (std::size_t)ctx.S() || m > (std::size_t)ctx.S())
    throw capacity_error("fully-connected layer does not fit in the slot count");
  if (B == 0) throw shape_error("merge budget must be >= 1");
  const std::size_t p2 = std::bit_ceil(n);
  const std::vector<double> head = range_mask(ctx, 0, 1);
  std::vector<Ciphertext> neurons;
  neurons.reserve(m);
  for (std::size_t i = 0; i < m; ++i) {
    std::vector<double> row(w + i * n, w + (i + 1) * n);
    Ciphertext y = mp(ctx, x, plain(ctx, row));
    for (std::size_t off = 1; off < p2; off <<= 1) y = add(ctx, y, rotate(ctx, y, (long)off));
    neurons.push_back(mp(ctx, y, head));
  }
  const std::size_t r = (m <= B + 1) ? m : B;
  const std::size_t T = (m + r - 1) / r;
  std::vector<Ciphertext> groups;
  for (std::size_t t = 0; t < T; ++t) {
    const std::size_t sz = std::min(r, m - t * r);
    Ciphertext g = neurons[t * r];
    for (std::size_t u = 1; u < sz; ++u) g = add(ctx, g, rotate(ctx, neurons[t * r + u], -(long)u));
    groups.push_back(g);
  }
  Ciphertext out = groups[T - 1];
  for (std::size_t t = T - 1; t-- > 0;) out = add(ctx, rotate(ctx, out, -(long)r), groups[t]);
  std::vector<double> b(m, 0.0);
  if (bias) std::copy(bias, bias + m, b.begin());
  return add_plain(ctx, out, b.data(), b.size());
}

// ------------------------------------------------------------- ReLU
std::vector<double> cheb_coefficients(const std::function<double(double)>& f, int degree) {
  if (degree < 0) throw shape_error("polynomial degree must be non-negative");
  const double pi = 3.14159265358979323846;
  const int n = degree + 1;
  std::vector<double> nodes(n), fx(n), coeffs(n, 0.0);
  for (int j = 0; j < n; ++j) nodes[j] = std::cos(pi * (2.0 * j + 1.0) / (2.0 * n));
  for (int j = 0; j < n; ++j) fx[j] = f(nodes[j]);
  for (int d = 0; d < n; ++d) {
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc += fx[j] * std::cos(d * pi * (2.0 * j + 1.0) / (2.0 * n));
    coeffs[d] = (d == 0 ? 1.0 : 2.0) * acc / n;
  }
  return coeffs;
}

int cheb_eval_depth(int degree) {
  if (degree <= 0) return 0;
  if (degree == 1) return 1;
  return (int)std::bit_width((unsigned)(degree - 1)) + 1;
}

// cheb_eval (chebyshev.cpp:62-104): balanced T_d tree, then constant MACs
Ciphertext cheb_eval(Context& ctx, const Ciphertext& x, const std::vector<double>& coeffs) {
  if (!x.valid()) throw Error(ErrKind::internal, "cheb_eval: operand is not initialized");
  if (coeffs.empty()) throw shape_error("cheb_eval: empty coefficient list");
  const int D = (int)coeffs.size() - 1;
  if (D == 0) {
    // constant series: c0 in every slot, no depth consumed
    return add_const(ctx, sub(ctx, x, x), coeffs[0]);
  }
  std::vector<Ciphertext> T(D + 1);
  T[1] = x;
  for (int d = 2; d <= D; ++d) {
    const int a = (d + 1) / 2, b = d / 2;
    const Ciphertext prod = mult_cipher(ctx, T[a], T[b]);
    const Ciphertext doubled = add(ctx, prod, prod);
    T[d] = (d % 2 == 0) ? add_const(ctx, doubled, -1.0) : sub(ctx, doubled, T[1]);
  }
  Ciphertext acc;
  for (int d = 1; d <= D; ++d) {
    const Ciphertext term = mult_const(ctx, T[d], coeffs[d]);
    acc = (d == 1) ? term : add(ctx, acc, term);
  }
  return add_const(ctx, acc, coeffs[0]);
}

// secure_relu (layers_misc.cpp:268-295)
Ciphertext secure_relu(Context& ctx, const Ciphertext& x, double scale, int degree, std::size_t active_slots) {
  if (degree < 0) throw shape_error("activation degree must be >= 0");
  const bool scaled = scale > 1.0;
  const double beta = scaled ? scale : 1.0;
  Ciphertext v = x;
  if (scaled) {
    if (active_slots == 0) throw shape_error("scaled activation requires the active slot count");
    if (active_slots > (std::size_t)ctx.S()) throw capacity_error("active slot count exceeds the context");
    v = mp(ctx, x, range_mask(ctx, 0, active_slots, 1.0 / beta));
  }
  const auto f = [beta](double z) { return z < 0.0 ? 0.0 : beta * z; };
  return cheb_eval(ctx, v, cheb_coefficients(f, degree));
}

// ------------------------------------------------------------- depth costs
int pad_depth_cost(std::size_t padding) { return padding > 0 ? 1 : 0; }

int stride_depth_cost(int variant, std::size_t W, std::size_t S, std::size_t W_out) {
  (void)W;
  if (variant == 1 && detail::masked_stride_applicable(W_out)) return detail::stride_mask_compact_depth(S, W_out);
  return 1;
}

int conv_depth_cost(const ConvConfig& cfg, std::size_t W_in) {
  if (cfg.mode == 1) return 2;
  const std::size_t Wp = W_in + 2 * cfg.padding;
  const std::size_t W_out = conv_output_width(W_in, cfg.kernel, cfg.stride, cfg.padding);
  const int pad = pad_depth_cost(cfg.padding);
  if (cfg.mode == 2 && cfg.in_channels > 1) {
    if (detail::masked_stride_applicable(W_out)) return pad + 1 + detail::stride_mask_compact_depth(cfg.stride, W_out);
    return pad + 2;
  }
  const int sc = (cfg.stride == 1 && W_out == Wp) ? 0 : stride_depth_cost(cfg.stride_variant, Wp, cfg.stride, W_out);
  return pad + 2 + sc;
}

int pool_depth_cost(int kind, std::size_t k, std::size_t S, int variant, std::size_t W_in) {
  if (kind == 1) return 1;
  if (kind == 2) return 2;
  const std::size_t W_out = conv_output_width(W_in, k, S, 0);
  const int sc = (S == 1 && W_out == W_in) ? 0 : stride_depth_cost(variant, W_in, S, W_out);
  return 1 + sc;
}

int fc_depth_cost() { return 2; }

int relu_depth_cost(double scale, int degree) { return (scale > 1.0 ? 1 : 0) + cheb_eval_depth(degree); }

}  // namespace fheon
