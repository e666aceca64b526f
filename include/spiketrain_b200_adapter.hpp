// spiketrain_b200_adapter.hpp -- the reference-side drop-in.
//
// A maintainer of the reference (spiketrain, C++20 header-only) adds this header
// next to spiketrain/optimize.hpp.  It keeps the reference's own TrainState<float>
// (NetworkParams, OptimizerState, TrainConfig) and routes the training step
// train_step(st, packed_x, original_t, targets) (optimize.hpp:152-156) through the
// B200 engine's C ABI (include/snn_engine.h).  Two ways to use it:
//
//   1. explicit: construct spiketrain::B200Step gpu(st, batch, T) and call
//      gpu(bx, by) where train() calls train_step (optimize.hpp:284), then
//      gpu.sync_to(st) before using st.params / st.opt (e.g. write_checkpoint);
//   2. swap in the reference's OWN train() unchanged: in exactly one translation
//      unit, before any use of train<float>, write
//          SPIKETRAIN_B200_SWAP_TRAIN_STEP()
//      which declares the explicit specialization train_step<float> that the
//      reference's train() then calls; call spiketrain::b200::sync_all() from the
//      epoch callback (or after train() returns) to copy parameters and optimizer
//      state back into the TrainState.  (Do not include commands.hpp in that TU
//      before the macro: cmd_train instantiates train<float>.)
//
// Types crossing the boundary are plain pointers and sizes (snn_engine.h); the
// parameter order is the reference's entry order (network.hpp:210-226).
#pragma once

#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "snn_engine.h"
#include "spiketrain/optimize.hpp"

namespace spiketrain {

namespace b200_detail {

inline int activation_id(const std::string& n) {
  if (n == "custom") return SNN_ACT_CUSTOM;
  if (n == "superspike") return SNN_ACT_SUPERSPIKE;
  if (n == "triangular") return SNN_ACT_TRIANGULAR;
  if (n == "arctan") return SNN_ACT_ARCTAN;
  if (n == "boxcar") return SNN_ACT_BOXCAR;
  throw ArgumentError("unknown activation: " + n);
}

// snn_status -> the reference's exception classes (errors.hpp:9-64)
[[noreturn]] inline void raise(int rc, const char* msg) {
  const std::string m = msg ? msg : "snn_engine error";
  switch (rc) {
    case SNN_ERR_SHAPE: throw ShapeError(m);
    case SNN_ERR_ARGUMENT: throw ArgumentError(m);
    case SNN_ERR_CONTRACT: throw ContractError(m);
    case SNN_ERR_STATE: throw StateError(m);
    case SNN_ERR_FORMAT: throw FormatError(m);
    case SNN_ERR_IO: throw IoError(m);
    case SNN_ERR_SPEC: throw SpecError(m);
    case SNN_ERR_CONFIG: throw ConfigError(m);
    case SNN_ERR_UNSUPPORTED: throw UnsupportedError(m);
    default: throw Error(m);
  }
}
inline void check(int rc, const snn_engine* e) {
  if (rc != SNN_OK) raise(rc, snn_last_error(e));
}

}  // namespace b200_detail

// The reference NetworkSpec as the engine's POD descriptor: the feed-forward
// family [Linear, LIF, (Monitor)]*k, Linear, LI of normalize() (network.hpp:125-157).
inline snn_network_desc b200_desc(const NetworkSpec& spec) {
  if (spec.input_shape.empty()) throw SpecError("network: input shape not declared");
  std::vector<Layer> ls;
  std::vector<int> monitor;
  for (std::size_t i = 0; i < spec.layers.size(); ++i) {
    if (std::holds_alternative<MonitorLayer>(spec.layers[i])) {
      if (i == 0 || !std::holds_alternative<LIFLayer>(spec.layers[i - 1]))
        throw SpecError("layer " + std::to_string(i) + ": monitor must follow a lif layer");
      monitor.push_back(int(ls.size() / 2) - 1);
      continue;
    }
    ls.push_back(spec.layers[i]);
  }
  if (ls.size() < 4 || ls.size() % 2) throw UnsupportedError("engine supports [Linear, LIF]*k + Linear + LI");
  snn_network_desc d{};
  std::size_t in = 1;
  for (auto v : spec.input_shape) in *= v;
  d.input = int32_t(in);
  d.n_hidden = int32_t(ls.size() / 2 - 1);
  if (d.n_hidden > SNN_MAX_HIDDEN) throw UnsupportedError("too many hidden layers");
  for (int i = 0; i < d.n_hidden; ++i) {
    const auto* lin = std::get_if<LinearLayer>(&ls[2 * i]);
    const auto* lif = std::get_if<LIFLayer>(&ls[2 * i + 1]);
    if (!lin || !lif) throw UnsupportedError("expected Linear + LIF pairs");
    d.hidden[i] = int32_t(lin->out);
    d.bias = lin->bias;
    d.threshold = float(lif->threshold);
    d.activation = b200_detail::activation_id(lif->activation.name);
    d.slope = float(lif->activation.slope);
    d.aux = float(lif->activation.aux);
    d.beta_mode[i] = int32_t(lif->beta_mode);
    d.fixed_beta[i] = float(lif->fixed_beta);
  }
  const auto* lin = std::get_if<LinearLayer>(&ls[ls.size() - 2]);
  if (!lin) throw UnsupportedError("readout must be Linear + LI or Linear + LIF");
  d.classes = int32_t(lin->out);
  if (const auto* ro = std::get_if<LIFLayer>(&ls.back())) {  // spikes are the trace (network.hpp:396)
    if (float(ro->threshold) != d.threshold || b200_detail::activation_id(ro->activation.name) != d.activation)
      throw UnsupportedError("a LIF readout shares the hidden layers' threshold and surrogate");
    d.readout_lif = 1;
    d.beta_mode[d.n_hidden] = int32_t(ro->beta_mode);
    d.fixed_beta[d.n_hidden] = float(ro->fixed_beta);
  } else if (const auto* li = std::get_if<LILayer>(&ls.back())) {
    d.beta_mode[d.n_hidden] = int32_t(li->beta_mode);
    d.fixed_beta[d.n_hidden] = float(li->fixed_beta);
  } else {
    throw UnsupportedError("readout must be Linear + LI or Linear + LIF");
  }
  for (int m : monitor) d.monitor[m] = 1;
  return d;
}

inline snn_train_config b200_config(const TrainConfig& cfg, std::size_t batch, std::size_t original_t) {
  snn_train_config c{};
  c.batch_size = int32_t(batch);
  c.time_steps = int32_t(original_t);
  c.lr = float(cfg.lr);
  c.beta1 = 0.9f;  // adam_update's constants (optimize.hpp:119)
  c.beta2 = 0.999f;
  c.eps = 1e-8f;
  c.seed = cfg.seed;
  c.unroll = int32_t(cfg.unroll);
  c.optimizer = cfg.optimizer == OptimizerKind::Sgd ? 1 : 0;
  c.momentum = float(cfg.momentum);
  c.loss = cfg.loss == LossKind::SpikeRateMse ? 1 : 0;
  c.rate_hi = float(cfg.rate_hi);
  c.rate_lo = float(cfg.rate_lo);
  // max_shift stays 0: the reference loop applies shift_augment to each batch
  // itself (optimize.hpp:276-278) before train_step sees it
  c.f_min = float(cfg.f_min);
  c.f_max = float(cfg.f_max);
  c.lambda_low = float(cfg.lambda_low);
  c.lambda_high = float(cfg.lambda_high);
  c.gemm_planes = 3;  // the fp32 path
  return c;
}

// One engine per TrainState: parameters and optimizer state uploaded from the
// reference's structures once, then every step runs on the GPU.
class B200Step {
 public:
  B200Step(const TrainState<float>& st, std::size_t batch, std::size_t original_t, int device = 0)
      : batch_(batch), t_(original_t) {
    const snn_network_desc d = b200_desc(st.spec);
    const snn_train_config c = b200_config(st.cfg, batch, original_t);
    snn_engine* e = nullptr;
    b200_detail::check(snn_engine_create(&d, &c, device, &e), nullptr);
    e_.reset(e);
    b200_detail::check(snn_param_count(e, &n_), e);
    std::size_t total = 0;
    for (const auto& en : st.params.entries) total += en.tensor.size();
    if (total != n_) throw ContractError("b200: parameter count differs from the reference spec");
    std::vector<float> flat(n_), m(n_, 0.0f), v(n_, 0.0f);
    std::size_t off = 0, ti = 0;
    for (const auto& en : st.params.entries) {
      std::memcpy(flat.data() + off, en.tensor.data(), en.tensor.size() * sizeof(float));
      if (en.trainable) {  // OptimizerState m / v hold trainable entries only (optimize.hpp:37-48)
        if (ti < st.opt.m.size()) std::memcpy(m.data() + off, st.opt.m[ti].data(), en.tensor.size() * 4);
        if (ti < st.opt.v.size()) std::memcpy(v.data() + off, st.opt.v[ti].data(), en.tensor.size() * 4);
        ++ti;
      }
      off += en.tensor.size();
    }
    b200_detail::check(snn_set_params(e, flat.data(), n_), e);
    b200_detail::check(snn_set_opt_state(e, m.data(), v.data(), uint64_t(st.opt.step), n_), e);
  }

  // train_step(st, packed_x, original_t, targets) on the GPU (host batch in the
  // reference layout [B, ceil(T/8), features...]).
  StepResult<float> operator()(const Tensor<std::uint8_t>& packed_x, std::size_t original_t,
                               const std::vector<std::int64_t>& targets) {
    if (original_t != t_)
      throw FormatError("unpack_time: packed extent inconsistent with T=" + std::to_string(original_t));
    if (targets.size() != batch_ || packed_x.shape().empty() || packed_x.shape()[0] != batch_)
      throw ArgumentError("b200: batch of " + std::to_string(targets.size()) + " for an engine of " +
                          std::to_string(batch_));
    StepResult<float> r;
    b200_detail::check(snn_train_step_packed(e_.get(), packed_x.data(), targets.data(), &r.loss, &r.accuracy),
                       e_.get());
    return r;
  }

  // Parameters and optimizer state back into the reference's TrainState.
  void sync_to(TrainState<float>& st) const {
    std::vector<float> flat(n_), m(n_), v(n_);
    uint64_t step = 0;
    b200_detail::check(snn_get_params(e_.get(), flat.data(), n_), e_.get());
    b200_detail::check(snn_get_opt_state(e_.get(), m.data(), v.data(), &step, n_), e_.get());
    std::size_t off = 0, ti = 0;
    for (auto& en : st.params.entries) {
      std::memcpy(en.tensor.data(), flat.data() + off, en.tensor.size() * sizeof(float));
      if (en.trainable) {
        if (ti < st.opt.m.size()) std::memcpy(st.opt.m[ti].data(), m.data() + off, en.tensor.size() * 4);
        if (ti < st.opt.v.size()) std::memcpy(st.opt.v[ti].data(), v.data() + off, en.tensor.size() * 4);
        ++ti;
      }
      off += en.tensor.size();
    }
    st.opt.step = std::size_t(step);
  }

 private:
  struct Destroy {
    void operator()(snn_engine* e) const { snn_engine_destroy(e); }
  };
  std::unique_ptr<snn_engine, Destroy> e_;
  std::size_t n_ = 0, batch_ = 0, t_ = 0;
};

namespace b200 {
// Engines created by the swapped-in train_step, one per TrainState.
struct Registry {
  std::map<TrainState<float>*, std::unique_ptr<B200Step>> engines;
  int device = 0;
};
inline Registry& registry() {
  static Registry r;
  return r;
}
inline StepResult<float> step(TrainState<float>& st, const Tensor<std::uint8_t>& packed_x,
                              std::size_t original_t, const std::vector<std::int64_t>& targets) {
  auto& slot = registry().engines[&st];
  if (!slot) slot.reset(new B200Step(st, targets.size(), original_t, registry().device));
  return (*slot)(packed_x, original_t, targets);
}
// Copy every engine's parameters and optimizer state back into its TrainState.
inline void sync_all() {
  for (auto& kv : registry().engines) kv.second->sync_to(*kv.first);
}
inline void release(TrainState<float>& st) { registry().engines.erase(&st); }
}  // namespace b200

}  // namespace spiketrain

// The reference's own train() (optimize.hpp:260-299) then runs every step on the
// GPU: an explicit specialization of train_step<float> (optimize.hpp:152-156).
#define SPIKETRAIN_B200_SWAP_TRAIN_STEP()                                                        \
  namespace spiketrain {                                                                         \
  template <>                                                                                    \
  inline StepResult<float> train_step<float>(TrainState<float> & st,                             \
                                             const Tensor<std::uint8_t>& packed_x,               \
                                             std::size_t original_t,                             \
                                             const std::vector<std::int64_t>& targets) {         \
    return b200::step(st, packed_x, original_t, targets);                                        \
  }                                                                                              \
  }
