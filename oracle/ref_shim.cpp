// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference slotcnn library
// (/root/reference/proj, compiled in place by oracle/Makefile into
// oracle/_ref/libslotcnn_ref.so).  It exposes the reference's layer API
// (layers.hpp:83-158) and backend ops (backend.hpp:134-153) on flat double
// arrays so that the pytest suite and bench.py's reference arm can call the
// reference directly through ctypes.  Every entry point returns 0 on success
// or the reference's ErrorCategory (errors.hpp:18-22: usage 1, data 2,
// internal 3) with the message available from sref_last_error().
//
// Trace events are returned as (kind, value) pairs:
//   kind 0 rotation (value = index), 1 mult_plain (value = level_after),
//   2 mult_cipher (level_after), 3 bootstrap (level_after); markers dropped.

#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "slotcnn/backend.hpp"
#include "slotcnn/chebyshev.hpp"
#include "slotcnn/keyplan.hpp"
#include "slotcnn/layers.hpp"
#include "slotcnn/model.hpp"
#include "slotcnn/packing.hpp"

using namespace slotcnn;

namespace {

thread_local std::string g_err;

struct Session {
  SlotContextPtr ctx;
  std::shared_ptr<TraceRecorder> rec;
};

Session make_session(std::size_t ring, std::size_t slots, int depth) {
  ContextConfig cfg;
  cfg.ring_dimension = ring;
  cfg.slot_count = slots;
  cfg.depth_budget = depth;
  Session s;
  s.ctx = SlotContext::create(cfg);
  s.rec = s.ctx->attach_recorder();
  return s;
}

SlotVector make_vec(const Session& s, const double* x, int level) {
  std::vector<double> v(x, x + s.ctx->slots());
  return SlotVector(s.ctx, std::move(v), level);
}

void put_events(const Session& s, long* ev, std::size_t cap, std::size_t* n) {
  if (!n) return;
  std::size_t k = 0;
  for (const TraceEvent& e : s.rec->snapshot()) {
    long kind = -1, value = 0;
    switch (e.kind) {
      case TraceEvent::Kind::rotation: kind = 0; value = e.rotation_index; break;
      case TraceEvent::Kind::mult_plain: kind = 1; value = e.level_after; break;
      case TraceEvent::Kind::mult_cipher: kind = 2; value = e.level_after; break;
      case TraceEvent::Kind::bootstrap: kind = 3; value = e.level_after; break;
      case TraceEvent::Kind::marker: break;
    }
    if (kind < 0) continue;
    if (ev && k < cap) {
      ev[2 * k] = kind;
      ev[2 * k + 1] = value;
    }
    ++k;
  }
  *n = k;
}

void put_vec(const SlotVector& v, double* out, int* level) {
  if (out) std::memcpy(out, v.slots().data(), v.size() * sizeof(double));
  if (level) *level = v.level();
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return e.exit_code();
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

KernelTensor make_kernel(std::size_t F, std::size_t C, std::size_t k,
                         const double* w, const double* b) {
  KernelTensor kt(F, C, k);
  std::memcpy(kt.weights.data(), w, kt.weights.size() * sizeof(double));
  if (b) std::memcpy(kt.bias.data(), b, F * sizeof(double));
  return kt;
}

ConvConfig make_conv_cfg(std::size_t C, std::size_t F, std::size_t k,
                         std::size_t stride, std::size_t pad, int mode,
                         int variant) {
  ConvConfig cfg;
  cfg.in_channels = C;
  cfg.out_channels = F;
  cfg.kernel = k;
  cfg.stride = stride;
  cfg.padding = pad;
  cfg.mode = mode == 1 ? ConvMode::special3x3
                       : (mode == 2 ? ConvMode::grouped : ConvMode::generic);
  cfg.stride_variant =
      variant == 1 ? StrideVariant::masked : StrideVariant::extract;
  return cfg;
}

}  // namespace

extern "C" {

const char* sref_last_error() { return g_err.c_str(); }

// --------------------------------------------------------------- backend ops
// op: 0 rotate(a, t), 1 add(a,b), 2 sub(a,b), 3 mult_plain(a, b-as-plain),
//     4 mult_cipher(a,b), 5 bootstrap(a)
int sref_backend_op(std::size_t ring, std::size_t slots, int depth, int op,
                    const double* a, int level_a, const double* b, int level_b,
                    long t, double* out, int* out_level, long* ev,
                    std::size_t ev_cap, std::size_t* n_ev) {
  return guard([&] {
    Session s = make_session(ring, slots, depth);
    const SlotVector va = make_vec(s, a, level_a);
    SlotVector r;
    switch (op) {
      case 0: r = rotate(va, t); break;
      case 1: r = add(va, make_vec(s, b, level_b)); break;
      case 2: r = sub(va, make_vec(s, b, level_b)); break;
      case 3: r = mult_plain(va, PlainVector{std::vector<double>(b, b + slots)}); break;
      case 4: r = mult_cipher(va, make_vec(s, b, level_b)); break;
      case 5: r = bootstrap(va); break;
      default: throw InternalError("unknown op");
    }
    put_vec(r, out, out_level);
    put_events(s, ev, ev_cap, n_ev);
  });
}

// -------------------------------------------------------------------- layers
int sref_convolution(std::size_t ring, std::size_t slots, int depth,
                     const double* x, int level, std::size_t C, std::size_t W,
                     std::size_t F, std::size_t k, std::size_t stride,
                     std::size_t pad, int mode, int variant, const double* w,
                     const double* bias, double* out, int* out_level,
                     std::size_t* out_C, std::size_t* out_W, long* ev,
                     std::size_t ev_cap, std::size_t* n_ev) {
  return guard([&] {
    Session s = make_session(ring, slots, depth);
    PackedTensor px{make_vec(s, x, level), C, W};
    const std::size_t wc = (mode == 2) ? 1 : C;
    const KernelTensor kt = make_kernel(F, wc, k, w, bias);
    const PackedTensor r =
        convolution(px, make_conv_cfg(C, F, k, stride, pad, mode, variant), kt);
    put_vec(r.data, out, out_level);
    if (out_C) *out_C = r.channels;
    if (out_W) *out_W = r.width;
    put_events(s, ev, ev_cap, n_ev);
  });
}

// Average pooling kinds: 0 average(k, stride, variant), 1 global, 2 whole-channel(k)
int sref_pool(std::size_t ring, std::size_t slots, int depth, const double* x,
              int level, std::size_t C, std::size_t W, int kind, std::size_t k,
              std::size_t stride, int variant, double* out, int* out_level,
              std::size_t* out_C, std::size_t* out_W, long* ev,
              std::size_t ev_cap, std::size_t* n_ev) {
  return guard([&] {
    Session s = make_session(ring, slots, depth);
    PackedTensor px{make_vec(s, x, level), C, W};
    if (kind == 0) {
      PoolConfig cfg;
      cfg.kind = PoolKind::average;
      cfg.kernel = k;
      cfg.stride = stride;
      cfg.stride_variant =
          variant == 1 ? StrideVariant::masked : StrideVariant::extract;
      const PackedTensor r = avg_pool(px, cfg);
      put_vec(r.data, out, out_level);
      if (out_C) *out_C = r.channels;
      if (out_W) *out_W = r.width;
    } else {
      const SlotVector r =
          kind == 1 ? global_avg_pool(px) : whole_channel_pool(px, k);
      put_vec(r, out, out_level);
      if (out_C) *out_C = C;
      if (out_W) *out_W = 1;
    }
    put_events(s, ev, ev_cap, n_ev);
  });
}

int sref_fully_connected(std::size_t ring, std::size_t slots, int depth,
                         const double* x, int level, std::size_t n,
                         std::size_t m, std::size_t merge_budget,
                         const double* w, const double* bias, double* out,
                         int* out_level, long* ev, std::size_t ev_cap,
                         std::size_t* n_ev) {
  return guard([&] {
    Session s = make_session(ring, slots, depth);
    FcConfig cfg;
    cfg.inputs = n;
    cfg.outputs = m;
    cfg.merge_budget = merge_budget;
    FcWeights fw(m, n);
    std::memcpy(fw.weights.data(), w, m * n * sizeof(double));
    if (bias) std::memcpy(fw.bias.data(), bias, m * sizeof(double));
    const SlotVector r = fully_connected(make_vec(s, x, level), cfg, fw);
    put_vec(r, out, out_level);
    put_events(s, ev, ev_cap, n_ev);
  });
}

int sref_secure_relu(std::size_t ring, std::size_t slots, int depth,
                     const double* x, int level, double scale, int degree,
                     std::size_t active_slots, double* out, int* out_level,
                     long* ev, std::size_t ev_cap, std::size_t* n_ev) {
  return guard([&] {
    Session s = make_session(ring, slots, depth);
    ReluConfig cfg;
    cfg.scale = scale;
    cfg.degree = degree;
    cfg.active_slots = active_slots;
    const SlotVector r = secure_relu(make_vec(s, x, level), cfg);
    put_vec(r, out, out_level);
    put_events(s, ev, ev_cap, n_ev);
  });
}

// variant 0 extract (v1), 1 masked (v2); W_out 0 = default edge
int sref_stride(std::size_t ring, std::size_t slots, int depth, const double* x,
                int level, std::size_t W, std::size_t S, std::size_t W_out,
                int variant, double* out, int* out_level, long* ev,
                std::size_t ev_cap, std::size_t* n_ev) {
  return guard([&] {
    Session s = make_session(ring, slots, depth);
    const SlotVector v = make_vec(s, x, level);
    SlotVector r;
    if (variant == 1) {
      r = W_out ? stride_extract_v2(v, W, S, W_out) : stride_extract_v2(v, W, S);
    } else {
      r = W_out ? stride_extract_v1(v, W, S, W_out) : stride_extract_v1(v, W, S);
    }
    put_vec(r, out, out_level);
    put_events(s, ev, ev_cap, n_ev);
  });
}

int sref_pad_input(std::size_t ring, std::size_t slots, int depth,
                   const double* x, int level, std::size_t C, std::size_t W,
                   std::size_t P, double* out, int* out_level, long* ev,
                   std::size_t ev_cap, std::size_t* n_ev) {
  return guard([&] {
    Session s = make_session(ring, slots, depth);
    PackedTensor px{make_vec(s, x, level), C, W};
    const PackedTensor r = pad_input(px, P);
    put_vec(r.data, out, out_level);
    put_events(s, ev, ev_cap, n_ev);
  });
}

// Chebyshev helpers (chebyshev.cpp:21-117)
int sref_cheb_relu_coefficients(double beta, int degree, double* coeffs) {
  return guard([&] {
    const auto f = [beta](double z) { return z < 0.0 ? 0.0 : beta * z; };
    const std::vector<double> c = cheb_coefficients(f, degree);
    std::memcpy(coeffs, c.data(), c.size() * sizeof(double));
  });
}

double sref_cheb_eval_scalar(double x, const double* coeffs, int n) {
  return cheb_eval_scalar(x, std::vector<double>(coeffs, coeffs + n));
}

int sref_depth_costs(std::size_t C, std::size_t F, std::size_t k,
                     std::size_t stride, std::size_t pad, int mode, int variant,
                     std::size_t W_in, int* conv_cost) {
  return guard([&] {
    *conv_cost = conv_depth_cost(make_conv_cfg(C, F, k, stride, pad, mode, variant), W_in);
  });
}

// ----------------------------------------------------------------- models
// build_model (model_spec.cpp:864) + infer (model_run.cpp:100) on a spec JSON
// with CSV weights next to it.  ledger: 3 ints per executed layer
// (level_in, level_out, is_bootstrap); names: '\n'-separated layer names.
int sref_infer(const char* spec_path, const double* input, std::size_t n_in,
               double* logits, std::size_t cap, std::size_t* n_logits,
               double* wall_ms, int* ledger, std::size_t ledger_cap,
               std::size_t* n_layers, char* names, std::size_t names_cap,
               long* ev, std::size_t ev_cap, std::size_t* n_ev) {
  return guard([&] {
    const ModelSpec spec = ModelSpec::from_json_file(spec_path);
    const BuiltModel model = build_model(spec);
    HostTensor x(model.input_shape.channels, model.input_shape.width,
                 model.input_shape.width);
    if (x.values.size() != n_in) throw ShapeError("input size mismatch");
    std::copy(input, input + n_in, x.values.begin());
    const InferResult r = infer(model, x);
    if (n_logits) *n_logits = r.logits.size();
    for (std::size_t i = 0; i < r.logits.size() && i < cap; ++i) logits[i] = r.logits[i];
    if (wall_ms) *wall_ms = r.wall_ms;
    std::string all;
    std::size_t k = 0;
    for (const auto& e : r.ledger) {
      if (ledger && k < ledger_cap) {
        ledger[3 * k] = e.level_in;
        ledger[3 * k + 1] = e.level_out;
        ledger[3 * k + 2] = e.bootstrap ? 1 : 0;
      }
      all += e.name + "\n";
      ++k;
    }
    if (n_layers) *n_layers = k;
    if (names && names_cap) {
      std::strncpy(names, all.c_str(), names_cap - 1);
      names[names_cap - 1] = 0;
    }
    if (n_ev) {
      std::size_t m = 0;
      for (const TraceEvent& e : r.trace->snapshot()) {
        long kind = -1, value = 0;
        switch (e.kind) {
          case TraceEvent::Kind::rotation: kind = 0; value = e.rotation_index; break;
          case TraceEvent::Kind::mult_plain: kind = 1; value = e.level_after; break;
          case TraceEvent::Kind::mult_cipher: kind = 2; value = e.level_after; break;
          case TraceEvent::Kind::bootstrap: kind = 3; value = e.level_after; break;
          case TraceEvent::Kind::marker: break;
        }
        if (kind < 0) continue;
        if (ev && m < ev_cap) {
          ev[2 * m] = kind;
          ev[2 * m + 1] = value;
        }
        ++m;
      }
      *n_ev = m;
    }
  });
}

// ----------------------------------------------------------------- keyplan
// BuiltModel::layer_keys (model_spec.cpp:944-950) of a spec: entries (layer, index,
// count) flattened, ends_block per layer.
int sref_layer_keys(const char* spec_path, long* entries, std::size_t cap, std::size_t* n_entries,
                    int* ends, std::size_t layer_cap, std::size_t* n_layers) {
  return guard([&] {
    const BuiltModel model = build_model(ModelSpec::from_json_file(spec_path));
    const std::vector<LayerKeys> lk = model.layer_keys();
    std::size_t m = 0;
    for (std::size_t i = 0; i < lk.size(); ++i) {
      if (i < layer_cap) ends[i] = lk[i].ends_block ? 1 : 0;
      for (const auto& [idx, cnt] : lk[i].keys.usage) {
        if (m < cap) {
          entries[3 * m] = (long)i;
          entries[3 * m + 1] = idx;
          entries[3 * m + 2] = cnt;
        }
        ++m;
      }
    }
    *n_entries = m;
    *n_layers = lk.size();
  });
}

// plan_single_block (mode 0) / plan_blocks (1) / plan_blocks with ranges (2)
// (keyplan.cpp:319-368) over layers given as entries (layer, index, count), then
// verify_trace (keyplan.cpp:370-421) of events (kind 0 rotation / 4 marker
// "layer:<value>:x" / other, value).  blocks: 3 longs (first, last, keys) each;
// out: union size, peak resident, violations, unused keys, rotations checked.
int sref_plan(int mode, std::size_t n_layers, const long* entries, std::size_t n_entries, const int* ends,
              const long* ranges, std::size_t n_ranges, const long* ev, std::size_t n_ev, long* blocks,
              std::size_t block_cap, std::size_t* n_blocks, long* out) {
  return guard([&] {
    std::vector<LayerKeys> lk(n_layers);
    for (std::size_t i = 0; i < n_layers; ++i) {
      lk[i].name = "L" + std::to_string(i);
      lk[i].ends_block = ends[i] != 0;
    }
    for (std::size_t m = 0; m < n_entries; ++m) lk[(std::size_t)entries[3 * m]].keys.add(entries[3 * m + 1], entries[3 * m + 2]);
    BlockPlan plan;
    if (mode == 0) {
      plan = plan_single_block(lk);
    } else if (mode == 1) {
      plan = plan_blocks(lk);
    } else {
      std::vector<std::pair<std::size_t, std::size_t>> r;
      for (std::size_t k = 0; k < n_ranges; ++k) r.push_back({(std::size_t)ranges[2 * k], (std::size_t)ranges[2 * k + 1]});
      plan = plan_blocks(lk, r);
    }
    std::vector<TraceEvent> events;
    for (std::size_t k = 0; k < n_ev; ++k) {
      TraceEvent e{};
      if (ev[2 * k] == 0) {
        e.kind = TraceEvent::Kind::rotation;
        e.rotation_index = ev[2 * k + 1];
      } else if (ev[2 * k] == 4) {
        e.kind = TraceEvent::Kind::marker;
        e.label = "layer:" + std::to_string(ev[2 * k + 1]) + ":x";
      } else {
        e.kind = TraceEvent::Kind::mult_plain;
        e.level_after = (int)ev[2 * k + 1];
      }
      events.push_back(e);
    }
    const TraceCheck tc = verify_trace(plan, events);
    for (std::size_t b = 0; b < plan.blocks.size() && b < block_cap; ++b) {
      blocks[3 * b] = (long)plan.blocks[b].first_layer;
      blocks[3 * b + 1] = (long)plan.blocks[b].last_layer;
      blocks[3 * b + 2] = (long)plan.blocks[b].keys.size();
    }
    *n_blocks = plan.blocks.size();
    out[0] = (long)plan.union_keys.size();
    out[1] = (long)plan.peak_resident_keys;
    out[2] = (long)tc.violations.size();
    out[3] = (long)tc.unused_keys.size();
    out[4] = (long)tc.rotations_checked;
  });
}

// ----------------------------------------------------------------- timing
// Mean wall seconds per convolution() call over `iters` calls (fresh input
// SlotVector each call, as the reference's infer() would see).
int sref_time_convolution(std::size_t ring, std::size_t slots, int depth,
                          const double* x, std::size_t C, std::size_t W,
                          std::size_t F, std::size_t k, std::size_t stride,
                          std::size_t pad, int mode, int variant,
                          const double* w, const double* bias, int iters,
                          double* seconds) {
  return guard([&] {
    ContextConfig cfg;
    cfg.ring_dimension = ring;
    cfg.slot_count = slots;
    cfg.depth_budget = depth;
    SlotContextPtr ctx = SlotContext::create(cfg);
    const std::size_t wc = (mode == 2) ? 1 : C;
    const KernelTensor kt = make_kernel(F, wc, k, w, bias);
    const ConvConfig cc = make_conv_cfg(C, F, k, stride, pad, mode, variant);
    std::vector<double> xin(x, x + C * W * W);
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) {
      PackedTensor px{SlotVector::encode(ctx, xin), C, W};
      const PackedTensor r = convolution(px, cc, kt);
      (void)r;
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / iters;
  });
}

// Mean wall seconds per rotate() at the given slot count.
int sref_time_rotate(std::size_t ring, std::size_t slots, int depth, long t,
                     int iters, double* seconds) {
  return guard([&] {
    ContextConfig cfg;
    cfg.ring_dimension = ring;
    cfg.slot_count = slots;
    cfg.depth_budget = depth;
    SlotContextPtr ctx = SlotContext::create(cfg);
    std::vector<double> v(slots);
    for (std::size_t i = 0; i < slots; ++i) v[i] = static_cast<double>(i % 97) / 97.0;
    SlotVector x = SlotVector::encode(ctx, v);
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) x = rotate(x, t);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / iters;
  });
}

}  // extern "C"
