// The drop-in proof: the reference's OWN train()
// (optimize.hpp:237-299, unmodified headers from /root/reference) with its
// train_step<float> swapped for the B200 engine by the adapter's explicit
// specialization.  Test infrastructure: built by tests/dropin/Makefile into
// tests/dropin/_build/ (the headers exist only in the build container), run by
// tests/test_dropin.py on the GPU box, which compares the epoch metrics and final
// parameters with the pure reference (oracle/_ref) on the same container file.
//
//   train_swap <data.spkd> <hidden> <act> <epochs> <batch> <seed> <out.bin>
// out.bin: f64 [epochs][2] (loss, accuracy), then f32 params (entry order),
// then u64 optimizer step.
#include <cstdio>
#include <cstdlib>
#include <fstream>

#include "spiketrain/data.hpp"
#include "spiketrain_b200_adapter.hpp"

SPIKETRAIN_B200_SWAP_TRAIN_STEP()

int main(int argc, char** argv) {
  using namespace spiketrain;
  if (argc != 8) {
    std::fprintf(stderr, "usage: train_swap data.spkd hidden act epochs batch seed out.bin\n");
    return 2;
  }
  try {
    const PackedDataset data = read_container(argv[1]);
    const std::size_t hidden = std::strtoul(argv[2], nullptr, 10);
    const std::string act = argv[3];
    NetworkSpec spec;
    spec.input_shape = Shape{data.x.shape()[2]};
    LIFLayer lif;
    lif.activation = default_activation_desc(act);
    spec.layers = {LinearLayer{hidden, false}, lif, LinearLayer{hidden, false}, lif,
                   LinearLayer{20, false}, LILayer{}};
    TrainConfig cfg;
    cfg.epochs = std::strtoul(argv[4], nullptr, 10);
    cfg.batch_size = std::strtoul(argv[5], nullptr, 10);
    cfg.seed = std::strtoull(argv[6], nullptr, 10);
    // the reference's own epoch loop; every train_step<float> runs on the GPU, and the
    // epoch callback copies the engine's state back into the TrainState that train()
    // returns
    const TrainResult<float> r = train<float>(spec, cfg, data, [](const EpochMetrics&) {
      b200::sync_all();
      return false;
    });
    std::ofstream o(argv[7], std::ios::binary);
    for (const auto& m : r.metrics) {
      o.write(reinterpret_cast<const char*>(&m.loss), 8);
      o.write(reinterpret_cast<const char*>(&m.accuracy), 8);
    }
    for (const auto& e : r.params.entries)
      o.write(reinterpret_cast<const char*>(e.tensor.data()), std::streamsize(e.tensor.size() * 4));
    const uint64_t step = r.opt.step;
    o.write(reinterpret_cast<const char*>(&step), 8);
    std::printf("train_swap: %zu epochs, last loss %.6f acc %.4f, step %llu\n", r.metrics.size(),
                r.metrics.back().loss, r.metrics.back().accuracy, (unsigned long long)step);
    return 0;
  } catch (const std::exception& ex) {
    std::fprintf(stderr, "train_swap: %s\n", ex.what());
    return 1;
  }
}
