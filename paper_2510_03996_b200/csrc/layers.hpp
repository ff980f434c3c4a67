// Layer API over device ciphertexts: the drop-in for
// proj/include/slotcnn/layers.hpp:83-158 (convolution family, pooling,
// fully connected, polynomial ReLU) plus the packing helpers of
// proj/include/slotcnn/packing.hpp.  Same slot layout (c*W^2 + i*W + j),
// rotation indices, masks, declared depth costs and trace events as the
// reference; the realisation batches rotations (hoisting) on the GPU.
#pragma once

#include <array>
#include <cstddef>
#include <functional>
#include <vector>

#include "engine.hpp"

namespace fheon {

struct ConvConfig {
  std::size_t in_channels = 1, out_channels = 1, kernel = 1, stride = 1, padding = 0;
  int mode = 0;            // 0 generic, 1 special3x3, 2 grouped
  int stride_variant = 0;  // 0 extract, 1 masked
};

struct KernelTensor {
  std::size_t out_channels = 0, in_channels = 0, kernel = 0;
  std::vector<double> weights;  // f*C*k*k + c*k*k + i*k + j
  std::vector<double> bias;
  double at(std::size_t f, std::size_t c, std::size_t i, std::size_t j) const {
    return weights[((f * in_channels + c) * kernel + i) * kernel + j];
  }
  static KernelTensor from(const ConvConfig& cfg, const double* w, const double* bias);
};

struct PackedTensor {
  Ciphertext data;
  std::size_t channels = 0, width = 0;
  std::size_t used_slots() const { return channels * width * width; }
};

// ---- packing helpers (packing.cpp)
std::vector<double> repeated_kernel_vector(const KernelTensor& w, std::size_t f, std::size_t ti, std::size_t tj,
                                           std::size_t C, std::size_t W);
std::vector<double> build_mask(std::size_t sp, std::size_t ep, std::size_t w, std::size_t m, std::size_t t);
std::array<std::vector<double>, 9> build_all_masks(std::size_t m, std::size_t C, std::size_t W);
std::vector<double> extraction_mask(std::size_t W, std::size_t C);

// ---- layers
std::size_t conv_output_width(std::size_t W, std::size_t k, std::size_t S, std::size_t P);
PackedTensor convolution(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w);
PackedTensor conv_generic(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w);
PackedTensor conv_special_3x3(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w);
PackedTensor conv_grouped_stride(Context& ctx, const PackedTensor& x, const ConvConfig& cfg, const KernelTensor& w);
PackedTensor pad_input(Context& ctx, const PackedTensor& x, std::size_t padding);
Ciphertext stride_extract_v1(Context& ctx, const Ciphertext& a, std::size_t W, std::size_t S, std::size_t W_out);
Ciphertext stride_extract_v2(Context& ctx, const Ciphertext& a, std::size_t W, std::size_t S, std::size_t W_out);
PackedTensor avg_pool(Context& ctx, const PackedTensor& x, std::size_t k, std::size_t S, int variant);
Ciphertext global_avg_pool(Context& ctx, const PackedTensor& x);
Ciphertext whole_channel_pool(Context& ctx, const PackedTensor& x, std::size_t k);
Ciphertext fully_connected(Context& ctx, const Ciphertext& x, std::size_t n, std::size_t m, std::size_t merge_budget,
                           const double* w, const double* bias);
Ciphertext secure_relu(Context& ctx, const Ciphertext& x, double scale, int degree, std::size_t active_slots);
std::vector<Ciphertext> secure_relu_many(Context& ctx, const std::vector<Ciphertext>& xs, double scale, int degree,
                                         std::size_t active_slots);

// ---- Chebyshev (chebyshev.cpp)
std::vector<double> cheb_coefficients(const std::function<double(double)>& f, int degree);
Ciphertext cheb_eval(Context& ctx, const Ciphertext& x, const std::vector<double>& coeffs);
std::vector<Ciphertext> cheb_eval_many(Context& ctx, const std::vector<Ciphertext>& xs,
                                       const std::vector<double>& coeffs);
// fused_sum: the final sum_d c_d T_d as one constant MAC + one rescale
std::vector<Ciphertext> cheb_eval_many(Context& ctx, const std::vector<Ciphertext>& xs,
                                       const std::vector<double>& coeffs, bool fused_sum);
int cheb_eval_depth(int degree);

// ---- declared depth costs
int pad_depth_cost(std::size_t padding);
int stride_depth_cost(int variant, std::size_t W, std::size_t S, std::size_t W_out);
int conv_depth_cost(const ConvConfig& cfg, std::size_t W_in);
int pool_depth_cost(int kind, std::size_t k, std::size_t S, int variant, std::size_t W_in);
int fc_depth_cost();
int relu_depth_cost(double scale, int degree);

namespace detail {
std::vector<long> block_sum_rotations(std::size_t span);
Ciphertext block_sum(Context& ctx, const Ciphertext& v, std::size_t span);
bool masked_stride_applicable(std::size_t W_out);
Ciphertext stride_mask_compact(Context& ctx, const Ciphertext& y, std::size_t W, std::size_t S, std::size_t W_out,
                               std::size_t blocks);
int stride_mask_compact_depth(std::size_t S, std::size_t W_out);
}  // namespace detail

// config-2 primitive microbench (bench.py); returns mean ms per launch group
double microbench(Context& ctx, int kind, int batch, int limbs, int n_rot, int iters);

}  // namespace fheon
