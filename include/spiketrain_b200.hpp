// spiketrain_b200.hpp -- header-only C++ mirror of the reference's training API
// (spiketrain: network.hpp, optimize.hpp, surrogate.hpp, errors.hpp, data.hpp)
// implemented over the engine's C ABI (snn_engine.h).  Code written against
// spiketrain::train_step / train can switch namespaces and link
// libsnn_b200.so; the numerics run on the B200, never on the CPU.
//
// Mirrored (reference file:line):
//   errors        errors.hpp:9-64         exception classes <- snn_status
//   ActivationDesc surrogate.hpp:134-157   name/slope/aux + default_activation_desc
//   LinearLayer / LIFLayer / LILayer / NetworkSpec   network.hpp:23-65
//   TrainConfig   optimize.hpp:116-133
//   TrainState    optimize.hpp:135-141   (params live on the device)
//   StepResult    optimize.hpp:143-147
//   train_step    optimize.hpp:152-214
//   train         optimize.hpp:237-299   (same key schedule; callback may stop)
#pragma once

#include <chrono>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "snn_engine.h"

namespace spiketrain_b200 {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : Error { using Error::Error; };
struct ArgumentError : Error { using Error::Error; };
struct ContractError : Error { using Error::Error; };
struct StateError : Error { using Error::Error; };
struct FormatError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct SpecError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct UnsupportedError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

inline void check(snn_status st, const snn_engine* e) {
  if (st == SNN_OK) return;
  const std::string msg = snn_last_error(e);
  switch (st) {
    case SNN_ERR_SHAPE: throw ShapeError(msg);
    case SNN_ERR_ARGUMENT: throw ArgumentError(msg);
    case SNN_ERR_CONTRACT: throw ContractError(msg);
    case SNN_ERR_STATE: throw StateError(msg);
    case SNN_ERR_FORMAT: throw FormatError(msg);
    case SNN_ERR_IO: throw IoError(msg);
    case SNN_ERR_SPEC: throw SpecError(msg);
    case SNN_ERR_CONFIG: throw ConfigError(msg);
    case SNN_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    default: throw DeviceError(msg);
  }
}

// -------------------------------------------------------------- spec types
struct ActivationDesc {
  std::string name = "superspike";
  double slope = 25.0;
  double aux = 0.0;
};

inline ActivationDesc default_activation_desc(const std::string& name) {
  if (name == "custom") return {"custom", 0.0, 0.0};
  if (name == "superspike") return {"superspike", 25.0, 0.0};
  if (name == "triangular") return {"triangular", 0.5, 0.0};
  if (name == "arctan") return {"arctan", 2.0, 0.0};
  if (name == "boxcar") return {"boxcar", 2.0, 0.5};
  throw ArgumentError("unknown activation: " + name);
}

struct LinearLayer {
  std::size_t out = 0;
  bool bias = true;
};
enum class BetaMode { PerNeuron, LearnableScalar, Fixed };  // neuron.hpp:24

// B200 extension (not in the reference): the DECLARED adaptive-threshold and
// recurrent cells of BASELINE configs 2 and 4 (snn_engine.h snn_cell; checker
// oracle/spiketrain_oracle.h).  The default keeps the reference's LIF.
enum class CellKind { LIF = SNN_CELL_LIF, ALIF = SNN_CELL_ALIF, RLIF = SNN_CELL_RLIF };

struct LIFLayer {
  std::vector<std::size_t> shape;
  ActivationDesc activation = {"superspike", 25.0, 0.0};
  BetaMode beta_mode = BetaMode::PerNeuron;
  double fixed_beta = 0.5;
  double threshold = 1.0;
  CellKind cell = CellKind::LIF;  // extension field, last so reference aggregate inits still work
};
struct LILayer {
  std::vector<std::size_t> shape;
  BetaMode beta_mode = BetaMode::PerNeuron;
  double fixed_beta = 0.5;
};
struct MonitorLayer {};  // network.hpp:57: spike counts of the LIF before it
using Layer = std::variant<LinearLayer, LIFLayer, LILayer, MonitorLayer>;

struct NetworkSpec {
  std::vector<std::size_t> input_shape;
  std::vector<Layer> layers;
};

enum class OptimizerKind { Adam, Sgd };                       // optimize.hpp:22
enum class LossKind { IntegralCrossentropy, SpikeRateMse };  // optimize.hpp:23

// optimize.hpp:116-133 (the fields the training step consumes)
struct TrainConfig {
  std::size_t epochs = 100;
  std::size_t batch_size = 64;
  double lr = 1e-3;
  OptimizerKind optimizer = OptimizerKind::Adam;
  double momentum = 0.9;  // SGD only
  LossKind loss = LossKind::IntegralCrossentropy;
  double rate_hi = 0.9;  // rate-MSE targets
  double rate_lo = 0.1;
  double f_min = 0.0;  // activity regularizer; zero lambdas disable it
  double f_max = 1.0;
  double lambda_low = 0.0;
  double lambda_high = 0.0;
  int gemm_planes = 3;            // engine option: 3 fp32 path, 2 fast (bf16x2), 1 bf16
  std::int64_t max_shift = 0;     // shift augmentation on packed batches
  std::vector<long> shift_axes;   // feature axis only (2 or -1)
  std::uint64_t seed = 0;
  std::size_t unroll = 32;
};

struct PackedDataset {
  std::vector<std::uint8_t> x;  // [N, ceil(T/8), input...] MSB-first
  std::size_t n = 0;
  std::size_t original_t = 0;
  std::vector<std::int64_t> y;
};

struct StepResult {
  float loss = 0;
  double accuracy = 0;
};

struct EpochMetrics {
  std::size_t epoch = 0;
  double loss = 0;
  double accuracy = 0;
  double wall_ms = 0;
};
using EpochCallback = std::function<bool(const EpochMetrics&)>;

namespace detail {

inline int activation_id(const std::string& n) {
  if (n == "custom") return SNN_ACT_CUSTOM;
  if (n == "superspike") return SNN_ACT_SUPERSPIKE;
  if (n == "triangular") return SNN_ACT_TRIANGULAR;
  if (n == "arctan") return SNN_ACT_ARCTAN;
  if (n == "boxcar") return SNN_ACT_BOXCAR;
  if (n == "sigmoid") return SNN_ACT_SIGMOID;  // declared (snn_engine.h)
  throw ArgumentError("unknown activation: " + n);
}

// normalize() subset (network.hpp:125-157): [Linear, LIF, (Monitor)]*k, Linear, LI
inline snn_network_desc describe(const NetworkSpec& spec) {
  if (spec.input_shape.empty()) throw SpecError("network: input shape not declared");
  if (spec.layers.empty()) throw SpecError("network: no layers");
  if (!std::holds_alternative<LIFLayer>(spec.layers.back()) &&
      !std::holds_alternative<LILayer>(spec.layers.back()))
    throw SpecError("network must end in a lif or li readout");
  // monitors: must follow a LIF (network.hpp:139-144); recorded per hidden block
  NetworkSpec s;
  s.input_shape = spec.input_shape;
  std::vector<int> monitor;
  for (std::size_t i = 0; i < spec.layers.size(); ++i) {
    if (std::holds_alternative<MonitorLayer>(spec.layers[i])) {
      if (i == 0 || !std::holds_alternative<LIFLayer>(spec.layers[i - 1]))
        throw SpecError("layer " + std::to_string(i) + ": monitor must follow a lif layer");
      monitor.push_back(int(s.layers.size() / 2) - 1);
      continue;
    }
    s.layers.push_back(spec.layers[i]);
  }
  if (s.layers.size() < 4 || s.layers.size() % 2)
    throw UnsupportedError("engine supports [Linear, LIF]*k + Linear + LI");
  snn_network_desc d{};
  std::size_t in = 1;
  for (auto v : s.input_shape) in *= v;
  d.input = int32_t(in);
  d.n_hidden = int32_t(s.layers.size() / 2 - 1);
  if (d.n_hidden > SNN_MAX_HIDDEN) throw UnsupportedError("too many hidden layers");
  for (int i = 0; i < d.n_hidden; ++i) {
    const auto* lin = std::get_if<LinearLayer>(&s.layers[2 * i]);
    const auto* lif = std::get_if<LIFLayer>(&s.layers[2 * i + 1]);
    if (!lin || !lif) throw UnsupportedError("expected Linear + LIF pairs");
    d.hidden[i] = int32_t(lin->out);
    d.bias = lin->bias;
    d.threshold = float(lif->threshold);
    d.activation = activation_id(lif->activation.name);
    d.slope = float(lif->activation.slope);
    d.aux = float(lif->activation.aux);
    d.beta_mode[i] = int32_t(lif->beta_mode);
    d.fixed_beta[i] = float(lif->fixed_beta);
    d.cell[i] = int32_t(lif->cell);
  }
  const auto* lin = std::get_if<LinearLayer>(&s.layers[s.layers.size() - 2]);
  if (!lin) throw UnsupportedError("readout must be Linear + LI or Linear + LIF");
  d.classes = int32_t(lin->out);
  if (const auto* ro = std::get_if<LIFLayer>(&s.layers.back())) {
    // a LIF readout: its spikes are the trace (network.hpp:396)
    if (ro->cell != CellKind::LIF || float(ro->threshold) != d.threshold ||
        activation_id(ro->activation.name) != d.activation || float(ro->activation.slope) != d.slope)
      throw UnsupportedError("a LIF readout shares the hidden layers' cell, threshold and surrogate");
    d.readout_lif = 1;
    d.beta_mode[d.n_hidden] = int32_t(ro->beta_mode);
    d.fixed_beta[d.n_hidden] = float(ro->fixed_beta);
  } else {
    const auto& li = std::get<LILayer>(s.layers.back());
    d.beta_mode[d.n_hidden] = int32_t(li.beta_mode);
    d.fixed_beta[d.n_hidden] = float(li.fixed_beta);
  }
  for (int m : monitor) d.monitor[m] = 1;
  return d;
}

}  // namespace detail

// TrainState: NetworkSpec + TrainConfig + device-resident params/optimizer state.
class TrainState {
 public:
  TrainState(const NetworkSpec& spec, const TrainConfig& cfg, std::size_t original_t,
             int device = 0)
      : spec_(spec), cfg_(cfg), t_(original_t) {
    const snn_network_desc d = detail::describe(spec);
    snn_train_config c{};
    c.batch_size = int32_t(cfg.batch_size);
    c.time_steps = int32_t(original_t);
    c.lr = float(cfg.lr);
    c.beta1 = 0.9f;
    c.beta2 = 0.999f;
    c.eps = 1e-8f;
    c.seed = cfg.seed;
    c.unroll = int32_t(cfg.unroll);
    c.optimizer = cfg.optimizer == OptimizerKind::Sgd ? 1 : 0;
    c.momentum = float(cfg.momentum);
    c.loss = cfg.loss == LossKind::SpikeRateMse ? 1 : 0;
    c.rate_hi = float(cfg.rate_hi);
    c.rate_lo = float(cfg.rate_lo);
    if (cfg.shift_axes.size() > 4) throw ArgumentError("train: at most 4 shift axes");
    c.max_shift = int32_t(cfg.max_shift);
    c.n_shift_axes = int32_t(cfg.shift_axes.size());
    for (std::size_t i = 0; i < cfg.shift_axes.size(); ++i) c.shift_axes[i] = int32_t(cfg.shift_axes[i]);
    c.f_min = float(cfg.f_min);
    c.f_max = float(cfg.f_max);
    c.lambda_low = float(cfg.lambda_low);
    c.lambda_high = float(cfg.lambda_high);
    c.gemm_planes = int32_t(cfg.gemm_planes);
    snn_engine* e = nullptr;
    check(snn_engine_create(&d, &c, device, &e), nullptr);
    eng_.reset(e);
    check(snn_param_count(e, &n_params_), e);
  }

  snn_engine* engine() const { return eng_.get(); }
  const NetworkSpec& spec() const { return spec_; }
  const TrainConfig& cfg() const { return cfg_; }
  std::size_t original_t() const { return t_; }
  std::size_t scalar_count() const { return n_params_; }

  // NetworkParams flat view (entry order of network.hpp:210-226)
  std::vector<float> params() const {
    std::vector<float> p(n_params_);
    check(snn_get_params(eng_.get(), p.data(), p.size()), eng_.get());
    return p;
  }
  void set_params(const std::vector<float>& p) {
    check(snn_set_params(eng_.get(), p.data(), p.size()), eng_.get());
  }
  std::uint64_t optimizer_step() const {
    std::uint64_t s = 0;
    check(snn_get_opt_state(eng_.get(), nullptr, nullptr, &s, n_params_), eng_.get());
    return s;
  }

 private:
  struct Deleter {
    void operator()(snn_engine* e) const { snn_engine_destroy(e); }
  };
  NetworkSpec spec_;
  TrainConfig cfg_;
  std::size_t t_;
  std::size_t n_params_ = 0;
  std::unique_ptr<snn_engine, Deleter> eng_;
};

// optimize.hpp:152-156: one fused step on a packed host batch.
inline StepResult train_step(TrainState& st, const std::vector<std::uint8_t>& packed_x,
                             std::size_t original_t, const std::vector<std::int64_t>& targets) {
  if (original_t != st.original_t())
    throw FormatError("unpack_time: packed extent inconsistent with T=" + std::to_string(original_t));
  if (targets.size() != st.cfg().batch_size)
    throw ArgumentError("targets: " + std::to_string(targets.size()) + " labels for batch " +
                        std::to_string(st.cfg().batch_size));
  StepResult r;
  check(snn_train_step_packed(st.engine(), packed_x.data(), targets.data(), &r.loss, &r.accuracy),
        st.engine());
  return r;
}

// cmd_eval (commands.hpp:144-169) on the dataset staged in the engine (train() /
// snn_stage_dataset): integral accuracy over all `n_rows` rows, walked in batches
// of the engine batch size, forward only.
inline double evaluate(TrainState& st, std::size_t n_rows) {
  std::vector<std::uint32_t> rows(n_rows);
  for (std::size_t i = 0; i < n_rows; ++i) rows[i] = std::uint32_t(i);
  double acc = 0.0;
  check(snn_evaluate(st.engine(), rows.data(), rows.size(), &acc, nullptr), st.engine());
  return acc;
}

// apply (network.hpp:435-448) for one batch of staged rows: readout trace [B][T][C].
inline std::vector<float> apply(TrainState& st, const std::vector<std::uint32_t>& rows,
                                std::size_t classes) {
  std::vector<float> trace(st.cfg().batch_size * st.original_t() * classes);
  check(snn_apply(st.engine(), rows.data(), trace.data(), trace.size()), st.engine());
  return trace;
}

// read_container / write_container (data.hpp:229-341) straight into / out of the
// engine's HBM-resident dataset; returns the number of examples staged.
inline std::size_t load_container(TrainState& st, const std::string& path) {
  std::size_t n = 0;
  check(snn_load_container(st.engine(), path.c_str(), &n), st.engine());
  return n;
}
inline void save_container(TrainState& st, const std::string& path) {
  check(snn_save_container(st.engine(), path.c_str()), st.engine());
}

// ApplyResult.monitors entry of the monitor after hidden LIF `layer`: spike counts
// [B][H] of the last forward (apply / step / evaluation batch).
inline std::vector<float> monitor_counts(TrainState& st, int layer, std::size_t hidden) {
  std::vector<float> c(st.cfg().batch_size * hidden);
  check(snn_monitor_counts(st.engine(), int32_t(layer), c.data(), c.size()), st.engine());
  return c;
}

// write_checkpoint / read_checkpoint (optimize.hpp:334-436) of the engine state in
// the reference .spkc format (bit-exact); read returns the stored config text.
inline void write_checkpoint(TrainState& st, const std::string& path, const std::string& config_text) {
  check(snn_save_checkpoint(st.engine(), path.c_str(), config_text.data(), config_text.size()),
        st.engine());
}
inline std::string read_checkpoint(TrainState& st, const std::string& path) {
  std::string cfg((1u << 20) + 1, '\0');
  std::size_t n = 0;
  check(snn_load_checkpoint(st.engine(), path.c_str(), cfg.data(), cfg.size(), &n), st.engine());
  cfg.resize(n);
  return cfg;
}

struct TrainResult {
  std::vector<float> params;
  std::vector<EpochMetrics> metrics;
  std::uint64_t step = 0;
};

// optimize.hpp:260-299: epoch loop over the dataset staged once in HBM.
inline TrainResult train(TrainState& st, const PackedDataset& data,
                         const EpochCallback& on_epoch = nullptr) {
  check(snn_stage_dataset(st.engine(), data.x.data(), data.n, data.y.data()), st.engine());
  TrainResult out;
  for (std::size_t e = 0; e < st.cfg().epochs; ++e) {
    const auto t0 = std::chrono::steady_clock::now();
    double m[2];
    // one epoch with the reference's epoch key (the engine keeps the epoch index)
    check(snn_train_epochs_from(st.engine(), e, 1, m), st.engine());
    EpochMetrics em;
    em.epoch = e;
    em.loss = m[0];
    em.accuracy = m[1];
    em.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    out.metrics.push_back(em);
    if (on_epoch && on_epoch(em)) break;
  }
  out.params = st.params();
  out.step = st.optimizer_step();
  return out;
}

// optimize.hpp:237-256: fresh state (init from master.child(0)) + epoch loop.
inline TrainResult train(const NetworkSpec& spec, const TrainConfig& cfg, const PackedDataset& data,
                         const EpochCallback& on_epoch = nullptr, int device = 0) {
  if (cfg.batch_size == 0) throw ArgumentError("train: batch size 0");
  TrainState st(spec, cfg, data.original_t, device);
  return train(st, data, on_epoch);
}

}  // namespace spiketrain_b200
