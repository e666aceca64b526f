// C++ parity/behaviour tests of the spiketrain_b200 shim, written like the
// reference's optimize_test.cpp (Catch2 is not in this image: tiny harness).
// Built and run by tests/test_cpp_shim.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "spiketrain_b200.hpp"
#include "../../paper_2402_18994_b200/csrc/host_rng.hpp"

namespace st = spiketrain_b200;
namespace rng = snn::hostrng;

static int failures = 0;
#define CHECK(c)                                                            \
  do {                                                                      \
    if (!(c)) {                                                             \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);              \
      ++failures;                                                           \
    }                                                                       \
  } while (0)

// optimize_test.cpp:39-56: separable two-class rasters, 8 features
static st::PackedDataset toy_data(std::size_t n, std::size_t t, std::uint64_t key) {
  st::PackedDataset d;
  d.n = n;
  d.original_t = t;
  const std::size_t tp = (t + 7) / 8;
  d.x.assign(n * tp * 8, 0);
  d.y.resize(n);
  for (std::size_t i = 0; i < n; ++i) {
    const std::size_t cls = i % 2;
    d.y[i] = std::int64_t(cls);
    const std::uint64_t ek = rng::child(key, i);
    std::size_t draw = 0;
    for (std::size_t s = 0; s < t; ++s)
      for (std::size_t j = 0; j < 8; ++j) {
        const bool in_block = j / 4 == cls;
        const double rate = in_block ? 0.8 : 0.05;
        if (rng::uniform01(ek, draw++) < rate)
          d.x[(i * tp + s / 8) * 8 + j] |= std::uint8_t(1u << (7 - s % 8));
      }
  }
  return d;
}

static st::NetworkSpec toy_spec() {
  st::NetworkSpec s;
  s.input_shape = {8};
  s.layers = {st::LinearLayer{8}, st::LIFLayer{}, st::LinearLayer{2}, st::LILayer{}};
  return s;
}

int main() {
  // "loss falls on a separable toy problem" (optimize_test.cpp:193-207)
  {
    const auto data = toy_data(16, 16, rng::from_seed(703));
    st::TrainConfig cfg;
    cfg.epochs = 30;
    cfg.batch_size = 8;
    cfg.lr = 5e-3;
    cfg.seed = 1;
    cfg.unroll = 8;
    const auto r = st::train(toy_spec(), cfg, data);
    CHECK(r.metrics.size() == 30);
    CHECK(r.metrics.back().loss < r.metrics.front().loss);
    CHECK(r.metrics.back().accuracy >= 0.75);
    CHECK(r.step == 30 * 2);
    std::printf("toy: loss %.4f -> %.4f, acc %.3f, steps %llu\n", r.metrics.front().loss,
                r.metrics.back().loss, r.metrics.back().accuracy, (unsigned long long)r.step);
  }
  // the declared ALIF / RLIF cells (B200 extension) train the same toy problem
  for (auto kind : {st::CellKind::ALIF, st::CellKind::RLIF}) {
    const auto data = toy_data(16, 16, rng::from_seed(703));
    st::TrainConfig cfg;
    cfg.epochs = 30;
    cfg.batch_size = 8;
    cfg.lr = 5e-3;
    cfg.seed = 1;
    auto spec = toy_spec();
    st::LIFLayer cell;
    cell.cell = kind;
    spec.layers[1] = cell;
    const auto r = st::train(spec, cfg, data);
    CHECK(r.metrics.back().loss < r.metrics.front().loss);
    CHECK(r.metrics.back().accuracy >= 0.75);
    std::printf("toy %s: loss %.4f -> %.4f, acc %.3f\n", kind == st::CellKind::ALIF ? "alif" : "rlif",
                r.metrics.front().loss, r.metrics.back().loss, r.metrics.back().accuracy);
  }
  // cmd_eval after training (commands.hpp:144-169): the trained toy separates its
  // own data; evaluation is forward only (no optimizer step)
  {
    const auto data = toy_data(16, 16, rng::from_seed(703));
    st::TrainConfig cfg;
    cfg.epochs = 30;
    cfg.batch_size = 8;
    cfg.lr = 5e-3;
    cfg.seed = 1;
    cfg.unroll = 8;
    st::TrainState state(toy_spec(), cfg, data.original_t);
    st::train(state, data);
    const auto step = state.optimizer_step();
    const double acc = st::evaluate(state, data.n);
    CHECK(acc >= 0.75 && acc <= 1.0);
    CHECK(state.optimizer_step() == step);
    CHECK(st::evaluate(state, data.n) == acc);
    std::printf("toy eval accuracy %.3f\n", acc);
  }
  // "training is deterministic in the seed" (optimize_test.cpp:170-191)
  {
    const auto data = toy_data(8, 16, rng::from_seed(702));
    st::TrainConfig cfg;
    cfg.epochs = 3;
    cfg.batch_size = 4;
    cfg.seed = 9;
    cfg.unroll = 4;
    const auto a = st::train(toy_spec(), cfg, data);
    const auto b = st::train(toy_spec(), cfg, data);
    CHECK(a.params == b.params);
    CHECK(a.metrics.size() == 3 && a.metrics[2].loss == b.metrics[2].loss);
    cfg.seed = 10;
    const auto c = st::train(toy_spec(), cfg, data);
    CHECK(!(a.params == c.params));
  }
  // "zero epochs returns the untouched initialization" (optimize_test.cpp:149-168)
  {
    const auto data = toy_data(8, 16, rng::from_seed(701));
    st::TrainConfig cfg;
    cfg.epochs = 0;
    cfg.batch_size = 4;
    cfg.seed = 42;
    const auto r = st::train(toy_spec(), cfg, data);
    CHECK(r.metrics.empty());
    CHECK(r.step == 0);
    // init(spec, from_seed(42).child(0)): l0.w ~ TN(child(0).child(0), sd 1/sqrt(8))
    std::vector<float> w(64);
    const std::uint64_t key = rng::child(rng::from_seed(42), 0);
    rng::truncated_normal(rng::child(rng::child(key, 0), 0), 64, 0.0f, 1.0f / std::sqrt(8.0f), w.data());
    bool same = true;
    for (int i = 0; i < 64; ++i) same = same && (w[i] == r.params[i]);
    CHECK(same);
  }
  // errors map onto the reference's exception classes
  {
    bool threw = false;
    try {
      st::NetworkSpec bad;
      bad.layers = {st::LinearLayer{4}, st::LILayer{}};
      st::TrainState s(bad, st::TrainConfig{}, 16);
    } catch (const st::SpecError&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      st::TrainConfig cfg;
      cfg.batch_size = 4;
      st::TrainState s(toy_spec(), cfg, 16);
      std::vector<std::uint8_t> x(4 * 2 * 8, 0);
      st::train_step(s, x, 16, {0, 1});
    } catch (const st::ArgumentError&) {
      threw = true;
    }
    CHECK(threw);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
