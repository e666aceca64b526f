// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (see spiketrain_oracle.h).
//
// extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/spiketrain, included read-only via -I by
// oracle/Makefile).  It exports the orc_* interface under the ref_* prefix so
// the tests can compare the plain-C restatement with the reference itself,
// and so bench.py can time the reference's own CPU train_step.  Output goes
// to oracle/_ref/ only.
#include <cstring>
#include <vector>

#include "spiketrain/data.hpp"
#include "spiketrain/network.hpp"
#include "spiketrain/objective.hpp"
#include "spiketrain/optimize.hpp"
#include "spiketrain/commands.hpp"

#include "spiketrain_oracle.h"

using namespace spiketrain;

namespace {

ActivationDesc act_desc(const orc_net* n) {
  static const char* names[] = {"custom", "superspike", "triangular", "arctan",
                                "boxcar"};
  // sigmoid is not in make_activation's catalogue (surrogate.hpp:140-148): the
  // reference reaches it only through custom() (ref_surrogate_vjp below)
  if (n->act < 0 || n->act > 4) throw std::invalid_argument("surrogate outside the reference catalogue");
  ActivationDesc d;
  d.name = names[n->act];
  d.slope = double(n->slope);
  d.aux = double(n->aux);
  return d;
}

BetaMode beta_mode(const orc_net* n, int l) {
  return n->beta_mode[l] == 1 ? BetaMode::LearnableScalar
                              : n->beta_mode[l] == 2 ? BetaMode::Fixed : BetaMode::PerNeuron;
}

NetworkSpec make_spec(const orc_net* n) {
  NetworkSpec s;
  s.input_shape = {std::size_t(n->in)};
  for (int l = 0; l < n->n_hidden; ++l) {
    // the reference has LIF / LI cells only: no ALIF to drive
    if (n->cell[l] != 0) throw std::invalid_argument("ALIF cells are not part of the reference");
    s.layers.push_back(LinearLayer{std::size_t(n->hidden[l]), n->bias != 0});
    LIFLayer lif;
    lif.activation = act_desc(n);
    lif.threshold = double(n->threshold);
    lif.beta_mode = beta_mode(n, l);
    lif.fixed_beta = double(n->fixed_beta[l]);
    s.layers.push_back(lif);
    if (n->monitor[l]) s.layers.push_back(MonitorLayer{});
  }
  s.layers.push_back(LinearLayer{std::size_t(n->classes), n->bias != 0});
  if (n->readout_lif) {  // a LIF readout: its spikes are the trace (network.hpp:396)
    LIFLayer ro;
    ro.activation = act_desc(n);
    ro.threshold = double(n->threshold);
    ro.beta_mode = beta_mode(n, n->n_hidden);
    ro.fixed_beta = double(n->fixed_beta[n->n_hidden]);
    s.layers.push_back(ro);
    return s;
  }
  LILayer li;
  li.beta_mode = beta_mode(n, n->n_hidden);
  li.fixed_beta = double(n->fixed_beta[n->n_hidden]);
  s.layers.push_back(li);
  return s;
}

NetworkParams<float> params_from_flat(const NetworkParams<float>& shape_src,
                                      const float* flat) {
  NetworkParams<float> p;
  std::size_t off = 0;
  for (const auto& e : shape_src.entries) {
    Tensor<float> t(e.tensor.shape());
    std::memcpy(t.data(), flat + off, t.size() * sizeof(float));
    off += t.size();
    p.entries.push_back({e.name, t, e.trainable});
  }
  return p;
}

void params_to_flat(const NetworkParams<float>& p, float* flat) {
  std::size_t off = 0;
  for (const auto& e : p.entries) {
    std::memcpy(flat + off, e.tensor.data(), e.tensor.size() * sizeof(float));
    off += e.tensor.size();
  }
}

NetworkParams<float> skeleton(const orc_net* n) {
  return init<float>(make_spec(n), RngKey::from_seed(0),
                     Tensor<float>::zeros({1, 1, std::size_t(n->in)}));
}

}  // namespace

extern "C" {

int ref_entry_count(const orc_net* n) {
  return int(skeleton(n).entries.size());
}

size_t ref_param_count(const orc_net* n) { return skeleton(n).scalar_count(); }

void ref_entry_layout(const orc_net* n, size_t* offsets, size_t* sizes,
                      char (*names)[16]) {
  std::size_t off = 0;
  int i = 0;
  for (const auto& e : skeleton(n).entries) {
    if (offsets) offsets[i] = off;
    if (sizes) sizes[i] = e.tensor.size();
    if (names) std::snprintf(names[i], 16, "%s", e.name.c_str());
    off += e.tensor.size();
    ++i;
  }
}

uint64_t ref_key_from_seed(uint64_t seed) {
  return RngKey::from_seed(seed).word;
}
uint64_t ref_key_child(uint64_t key, uint64_t index) {
  return RngKey{key}.child(index).word;
}
uint64_t ref_key_bits(uint64_t key, uint64_t counter) {
  return RngKey{key}.bits(counter);
}
double ref_uniform01(uint64_t key, uint64_t counter) {
  return uniform01(RngKey{key}, counter);
}
void ref_permutation(uint64_t key, size_t n, uint64_t* out) {
  const auto p = permutation(RngKey{key}, n);
  for (size_t i = 0; i < n; ++i) out[i] = p[i];
}
void ref_truncated_normal(uint64_t key, size_t n, float mean, float sd,
                          float* out) {
  const auto t = rng_truncated_normal<float>(RngKey{key}, Shape{n}, mean, sd);
  std::memcpy(out, t.data(), n * sizeof(float));
}

void ref_synth_raster(size_t classes, size_t n, size_t t, size_t f,
                      uint64_t seed, uint8_t* x, int64_t* y) {
  const RasterDataset d = synth_raster(classes, n, t, Shape{f}, seed);
  std::memcpy(x, d.x.data(), d.x.size());
  for (size_t i = 0; i < n; ++i) y[i] = d.y[i];
}

void ref_pack_time(const uint8_t* x, size_t n, size_t t, size_t f,
                   uint8_t* out) {
  Tensor<std::uint8_t> xt(Shape{n, t, f});
  std::memcpy(xt.data(), x, n * t * f);
  const auto p = pack_time(xt, 1);
  std::memcpy(out, p.data(), p.size());
}

void ref_unpack_time(const uint8_t* packed, size_t n, size_t t, size_t f,
                     uint8_t* out) {
  Tensor<std::uint8_t> pt(Shape{n, (t + 7) / 8, f});
  std::memcpy(pt.data(), packed, pt.size());
  const auto u = unpack_time<std::uint8_t>(pt, t, 1);
  std::memcpy(out, u.data(), u.size());
}

void ref_init(const orc_net* n, uint64_t key, float* params) {
  const auto p = init<float>(make_spec(n), RngKey{key},
                             Tensor<float>::zeros({1, 1, std::size_t(n->in)}));
  params_to_flat(p, params);
}

int ref_forward_backward_ex(const orc_net* n, const orc_train_opts* opts,
                            const float* params, const uint8_t* packed, size_t batch,
                            size_t t_steps, const int64_t* targets, float* loss,
                            double* acc, float* grads, uint8_t* spikes, float* vtrace,
                            float* trace);

int ref_forward_backward(const orc_net* n, const float* params,
                         const uint8_t* packed, size_t batch, size_t t_steps,
                         const int64_t* targets, float* loss, double* acc,
                         float* grads, uint8_t* spikes, float* vtrace,
                         float* trace) {
  return ref_forward_backward_ex(n, nullptr, params, packed, batch, t_steps, targets,
                                 loss, acc, grads, spikes, vtrace, trace);
}

int ref_forward_backward_ex(const orc_net* n, const orc_train_opts* opts,
                            const float* params, const uint8_t* packed, size_t batch,
                            size_t t_steps, const int64_t* targets, float* loss,
                            double* acc, float* grads, uint8_t* spikes, float* vtrace,
                            float* trace) {
  (void)vtrace;
  try {
    const NetworkSpec spec = make_spec(n);
    const NetworkParams<float> p = params_from_flat(skeleton(n), params);
    Tensor<std::uint8_t> px(Shape{batch, (t_steps + 7) / 8, std::size_t(n->in)});
    std::memcpy(px.data(), packed, px.size());
    const std::vector<std::int64_t> y(targets, targets + batch);
    // train_step without the update, mirroring optimize.hpp:157-203.
    Tensor<float> x = unpack_time<float>(px, t_steps, 1);
    Tape<float> tape;
    std::vector<Tape<float>::Id> ids;
    for (const auto& e : p.entries)
      ids.push_back(e.trainable ? tape.leaf(e.tensor) : tape.constant(e.tensor));
    auto fwd = forward_taped(tape, spec, ids, tape.constant(std::move(x)),
                             std::size_t(n->unroll));
    auto l = (opts && opts->loss == 1)
                 ? spike_rate_mse_taped(tape, fwd.trace, y, opts->rate_hi, opts->rate_lo)
                 : integral_crossentropy_taped(tape, fwd.trace, y);
    if (opts && (opts->lambda_low != 0.0f || opts->lambda_high != 0.0f))  // optimize.hpp:185-191
      for (auto& [name, counts] : fwd.monitors)
        l = tape.add(l, activity_regularizer_taped(tape, counts, t_steps, opts->f_min, opts->f_max,
                                                   opts->lambda_low, opts->lambda_high));
    *loss = tape.value(l)[0];
    *acc = integral_accuracy(tape.value(fwd.trace), y);
    if (trace)
      std::memcpy(trace, tape.value(fwd.trace).data(),
                  tape.value(fwd.trace).size() * sizeof(float));
    if (grads) {
      tape.backward(l);
      std::size_t off = 0;
      for (std::size_t i = 0; i < ids.size(); ++i) {
        const std::size_t sz = p.entries[i].tensor.size();
        if (p.entries[i].trainable) {
          const Tensor<float> g = tape.grad(ids[i]);
          std::memcpy(grads + off, g.data(), sz * sizeof(float));
        } else {
          std::memset(grads + off, 0, sz * sizeof(float));  // constant: no gradient
        }
        off += sz;
      }
    }
    if (spikes) {
      // Hidden rasters via the prefix-network trick (network_test.cpp:180-185):
      // the prefix ending at LIF l reuses the identical entries, so its
      // readout trace is that cell's spike train.
      std::size_t off = 0;
      const int per = n->bias ? 3 : 2;
      std::size_t end = 0;  // one past LIF h in spec.layers (monitors take slots too)
      for (int h = 0; h < n->n_hidden; ++h) {
        end += 2 + ((h > 0 && n->monitor[h - 1]) ? 1 : 0);
        NetworkSpec prefix;
        prefix.input_shape = spec.input_shape;
        prefix.layers.assign(spec.layers.begin(), spec.layers.begin() + std::ptrdiff_t(end));
        NetworkParams<float> pp;
        pp.entries.assign(p.entries.begin(),
                          p.entries.begin() + per * (h + 1));
        Tensor<float> xin = unpack_time<float>(px, t_steps, 1);
        const auto r = apply(prefix, pp, xin, std::size_t(n->unroll));
        for (std::size_t i = 0; i < r.trace.size(); ++i)
          spikes[off + i] = r.trace[i] != 0.0f;
        off += r.trace.size();
      }
    }
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

void ref_adam(float* p, const float* g, float* m, float* v, size_t n,
              uint64_t* step, float lr, float beta1, float beta2, float eps) {
  NetworkParams<float> holder;
  Tensor<float> pt(Shape{n});
  std::memcpy(pt.data(), p, n * sizeof(float));
  holder.entries.push_back({"p", pt, true});
  auto st = init_optimizer(OptimizerKind::Adam, holder);
  std::memcpy(st.m[0].data(), m, n * sizeof(float));
  std::memcpy(st.v[0].data(), v, n * sizeof(float));
  st.step = *step;
  Tensor<float> gt(Shape{n});
  std::memcpy(gt.data(), g, n * sizeof(float));
  std::vector<Tensor<float>*> ps = {&holder.entries[0].tensor};
  adam_update(ps, {gt}, st, lr, beta1, beta2, eps);
  std::memcpy(p, holder.entries[0].tensor.data(), n * sizeof(float));
  std::memcpy(m, st.m[0].data(), n * sizeof(float));
  std::memcpy(v, st.v[0].data(), n * sizeof(float));
  *step = st.step;
}

namespace {

TrainState<float> make_state(const orc_net* n, const float* params,
                             const float* m, const float* v, uint64_t step,
                             float lr, const orc_train_opts* opts = nullptr) {
  TrainState<float> st;
  st.spec = make_spec(n);
  st.cfg.unroll = std::size_t(n->unroll);
  st.cfg.lr = double(lr);
  const OptimizerKind kind =
      (opts && opts->optimizer == 1) ? OptimizerKind::Sgd : OptimizerKind::Adam;
  if (opts) {
    st.cfg.optimizer = kind;
    st.cfg.momentum = double(opts->momentum);
    st.cfg.loss = opts->loss == 1 ? LossKind::SpikeRateMse : LossKind::IntegralCrossentropy;
    st.cfg.rate_hi = double(opts->rate_hi);
    st.cfg.rate_lo = double(opts->rate_lo);
    st.cfg.f_min = double(opts->f_min);
    st.cfg.f_max = double(opts->f_max);
    st.cfg.lambda_low = double(opts->lambda_low);
    st.cfg.lambda_high = double(opts->lambda_high);
  }
  st.params = params_from_flat(skeleton(n), params);
  st.opt = init_optimizer(kind, st.params);
  // flat m/v span every entry (zeros for constants); the state holds trainable ones
  std::size_t off = 0, ti = 0;
  for (const auto& e : st.params.entries) {
    if (e.trainable) {
      std::memcpy(st.opt.m[ti].data(), m + off, e.tensor.size() * sizeof(float));
      if (ti < st.opt.v.size())
        std::memcpy(st.opt.v[ti].data(), v + off, e.tensor.size() * sizeof(float));
      ++ti;
    }
    off += e.tensor.size();
  }
  st.opt.step = step;
  return st;
}

void unload_state(const TrainState<float>& st, float* params, float* m,
                  float* v, uint64_t* step) {
  params_to_flat(st.params, params);
  std::size_t off = 0, ti = 0;
  for (const auto& e : st.params.entries) {
    if (e.trainable) {
      std::memcpy(m + off, st.opt.m[ti].data(), e.tensor.size() * sizeof(float));
      if (ti < st.opt.v.size())
        std::memcpy(v + off, st.opt.v[ti].data(), e.tensor.size() * sizeof(float));
      ++ti;
    }
    off += e.tensor.size();
  }
  *step = st.opt.step;
}

}  // namespace

int ref_train_step_ex(const orc_net* n, const orc_train_opts* opts, float* params,
                      float* m, float* v, uint64_t* step, const uint8_t* packed,
                      size_t batch, size_t t_steps, const int64_t* targets, float lr,
                      float* loss, double* acc);

int ref_train_step(const orc_net* n, float* params, float* m, float* v,
                   uint64_t* step, const uint8_t* packed, size_t batch,
                   size_t t_steps, const int64_t* targets, float lr,
                   float* loss, double* acc) {
  return ref_train_step_ex(n, nullptr, params, m, v, step, packed, batch, t_steps,
                           targets, lr, loss, acc);
}

int ref_train_step_ex(const orc_net* n, const orc_train_opts* opts, float* params,
                      float* m, float* v, uint64_t* step, const uint8_t* packed,
                      size_t batch, size_t t_steps, const int64_t* targets, float lr,
                      float* loss, double* acc) {
  try {
    TrainState<float> st = make_state(n, params, m, v, *step, lr, opts);
    Tensor<std::uint8_t> px(Shape{batch, (t_steps + 7) / 8, std::size_t(n->in)});
    std::memcpy(px.data(), packed, px.size());
    const std::vector<std::int64_t> y(targets, targets + batch);
    const StepResult<float> r = train_step(st, px, t_steps, y);
    *loss = r.loss;
    *acc = r.accuracy;
    unload_state(st, params, m, v, step);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

int ref_train_epochs_ex(const orc_net* n, const orc_train_opts* opts, float* params,
                        float* m, float* v, uint64_t* step, const uint8_t* packed,
                        const int64_t* y, size_t count, size_t t_steps, size_t batch,
                        size_t epochs, uint64_t seed, float lr, double* metrics);

int ref_train_epochs(const orc_net* n, float* params, float* m, float* v,
                     uint64_t* step, const uint8_t* packed, const int64_t* y,
                     size_t count, size_t t_steps, size_t batch, size_t epochs,
                     uint64_t seed, float lr, double* metrics) {
  return ref_train_epochs_ex(n, nullptr, params, m, v, step, packed, y, count, t_steps, batch,
                             epochs, seed, lr, metrics);
}

int ref_train_epochs_ex(const orc_net* n, const orc_train_opts* opts, float* params,
                        float* m, float* v, uint64_t* step, const uint8_t* packed,
                        const int64_t* y, size_t count, size_t t_steps, size_t batch,
                        size_t epochs, uint64_t seed, float lr, double* metrics) {
  try {
    TrainState<float> st = make_state(n, params, m, v, *step, lr, opts);
    if (opts) {
      // train(spec, cfg, data)'s axis check (optimize.hpp:241-245); the resume
      // overload train(st, data) called below does not repeat it
      for (int i = 0; i < opts->n_shift_axes; ++i)
        if (opts->shift_axes[i] == 0 || opts->shift_axes[i] == 1) return 4;
      st.cfg.max_shift = opts->max_shift;
      for (int i = 0; i < opts->n_shift_axes; ++i) st.cfg.shift_axes.push_back(opts->shift_axes[i]);
    }
    st.cfg.batch_size = batch;
    st.cfg.epochs = epochs;
    st.cfg.seed = seed;
    PackedDataset d;
    d.x = Tensor<std::uint8_t>(Shape{count, (t_steps + 7) / 8, std::size_t(n->in)});
    std::memcpy(d.x.data(), packed, d.x.size());
    d.original_t = t_steps;
    d.y.assign(y, y + count);
    const auto r = train(st, d);
    for (std::size_t e = 0; e < r.metrics.size(); ++e) {
      metrics[2 * e] = r.metrics[e].loss;
      metrics[2 * e + 1] = r.metrics[e].accuracy;
    }
    unload_state(st, params, m, v, step);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// write_checkpoint (optimize.hpp:334-366) of a flat parameter / optimizer state:
// optimizer 0 = Adam (m and v), 1 = SGD (m only).  Golden .spkc fixtures.
int ref_write_checkpoint(const orc_net* n, const float* params, const float* m,
                         const float* v, uint64_t step, int optimizer,
                         const char* config_text, const char* path) {
  try {
    const NetworkParams<float> p = params_from_flat(skeleton(n), params);
    OptimizerState<float> st =
        init_optimizer(optimizer == 1 ? OptimizerKind::Sgd : OptimizerKind::Adam, p);
    std::size_t off = 0, ti = 0;
    for (const auto& e : p.entries) {
      if (e.trainable) {
        std::memcpy(st.m[ti].data(), m + off, e.tensor.size() * sizeof(float));
        if (ti < st.v.size()) std::memcpy(st.v[ti].data(), v + off, e.tensor.size() * sizeof(float));
        ++ti;
      }
      off += e.tensor.size();
    }
    st.step = step;
    write_checkpoint(path, p, st, std::string(config_text));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// write_container / read_container (data.hpp:229-341): golden .spkd fixtures.
// shape = the packed tensor's [N, ceil(T/8), features...] (ndim entries).
int ref_write_container(const char* path, const uint8_t* packed, const uint64_t* shape, int ndim,
                        uint32_t original_t, const int64_t* labels) {
  try {
    PackedDataset d;
    Shape s(shape, shape + ndim);
    d.x = Tensor<std::uint8_t>(s);
    std::memcpy(d.x.data(), packed, d.x.size());
    d.y.assign(labels, labels + shape[0]);
    d.original_t = original_t;
    write_container(path, d);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

int ref_read_container(const char* path, uint8_t* packed, size_t cap, int64_t* labels,
                       size_t label_cap, uint32_t* original_t, uint64_t* n) {
  try {
    const PackedDataset d = read_container(path);
    if (d.x.size() > cap || d.y.size() > label_cap) return 2;
    std::memcpy(packed, d.x.data(), d.x.size());
    std::copy(d.y.begin(), d.y.end(), labels);
    *original_t = uint32_t(d.original_t);
    *n = d.y.size();
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// The declared sigmoid surrogate (ORC_ACT_SIGMOID, spiketrain_oracle.h) as a
// caller would add it to the reference: custom(heaviside, bwd) with bwd the
// derivative of sigmoid(kx) (surrogate.hpp:45-57).
static SpikingActivation<float> sigmoid_activation(float k) {
  return custom<float>(nullptr, [k](const Tensor<float>& x) {
    Tensor<float> out(x.shape());
    for (std::size_t i = 0; i < x.size(); ++i) {
      const float e = std::exp(-(k * std::fabs(x[i])));
      out[i] = (k * e) / ((1.0f + e) * (1.0f + e));
    }
    return out;
  });
}

// g(x) through the reference's own tape: leaf x -> spike(tape, x, act)
// (surrogate.hpp:124-129, register_custom autodiff.hpp:389-413) -> sum, so the
// leaf gradient is 1 * g(x) exactly.  act 0..4 via make_activation, 5 =
// sigmoid through custom().
void ref_surrogate(int act, float slope, float aux, const float* x, size_t n, float* out) {
  static const char* names[] = {"custom", "superspike", "triangular", "arctan", "boxcar"};
  SpikingActivation<float> a;
  if (act == 5) {
    a = sigmoid_activation(slope);
  } else {
    ActivationDesc d;
    d.name = names[act];
    d.slope = double(slope);
    d.aux = double(aux);
    a = make_activation<float>(d);
  }
  Tape<float> tape;
  Tensor<float> xt(Shape{n});
  std::memcpy(xt.data(), x, n * sizeof(float));
  auto xi = tape.leaf(xt);
  auto y = spike(tape, xi, a);
  auto l = tape.sum(y);
  tape.backward(l);
  Tensor<float> g = tape.grad(xi);
  std::memcpy(out, g.data(), n * sizeof(float));
}

void ref_set_threads(int) {}  // the reference is single-threaded (ops.hpp:12-14)

}  // extern "C"
