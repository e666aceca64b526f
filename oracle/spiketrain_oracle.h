/*
 * spiketrain_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference training step (spiketrain, header-only
 * C++20 under /root/reference/proj/include/spiketrain).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker or the timed CPU baseline.
 * The product path (paper_2402_18994_b200) never links or calls it.
 *
 * Two implementations export this interface:
 *   orc_*  -- oracle/spiketrain_oracle.c, an independent plain-C restatement
 *             (fp32, same operation order as the reference, so results are
 *             bit-identical to it on the same libm);
 *   ref_*  -- oracle/ref_driver.cpp, a thin extern "C" driver that calls the
 *             reference headers themselves; compiled into oracle/_ref/.
 * The CPU test-suite pins orc_* against ref_* bit for bit and against the
 * committed golden vectors in tests/golden/.
 */
#ifndef SPIKETRAIN_ORACLE_H
#define SPIKETRAIN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_HIDDEN 8

/* Surrogate catalogue (surrogate.hpp:134-157). */
enum orc_act {
  ORC_ACT_CUSTOM = 0,     /* straight-through: g = 1          (surrogate.hpp:45-57) */
  ORC_ACT_SUPERSPIKE = 1, /* 1/(1+k|x|)^2                     (surrogate.hpp:59-73) */
  ORC_ACT_TRIANGULAR = 2, /* max(0, 1-|kx|)                   (surrogate.hpp:75-88) */
  ORC_ACT_ARCTAN = 3,     /* 1/(1+(pi k x/2)^2)               (surrogate.hpp:90-104) */
  ORC_ACT_BOXCAR = 4,     /* h on |x|<=w/2                    (surrogate.hpp:106-120) */
  /* DECLARED, not in the reference catalogue (SPEC.md:283 lists sigmoid as
   * "addable via custom()"; config.hpp:487-490 rejects the name): the
   * backward a caller passes to custom(fwd = heaviside, bwd), surrogate.hpp:45-57,
   *   e = exp(-(k |x|)) ;  g = (k e) / ((1 + e) (1 + e))   (k = slope, default 25)
   * i.e. d/dx sigmoid(kx) = k s (1 - s) (the snnTorch / Zenke & Vogels form),
   * written in the cancellation-free form: k s (1 - s) with s -> 1 loses every
   * digit of 1 - s, so two fp32 implementations would disagree in the tails.  Pinned at the
   * op level against the reference's own custom() + register_custom tape
   * closure (ref_surrogate_vjp, tests/test_oracle.py); the network path is the
   * reference-pinned surrogate plumbing with this g.                          */
  ORC_ACT_SIGMOID = 5
};

/* Host threads for the big-shape parity tests (default 1).  Results are
 * bit-identical for every thread count: threads split output elements only. */
void orc_set_threads(int n);

/* g(x) of a surrogate, elementwise (act = enum orc_act). */
void orc_surrogate(int act, float slope, float aux, const float* x, size_t n, float* out);

/*
 * Feed-forward SNN of the shape every BASELINE config uses:
 *   Linear(in->h0) -> LIF -> Linear(h0->h1) -> LIF ... -> Linear(->classes) -> LI
 * (network.hpp:23-60, normalised layer ids 0..2*n_hidden+1).  beta is per
 * neuron (BetaMode::PerNeuron, neuron.hpp:22).
 */
typedef struct orc_net {
  int in;                      /* per-timestep input features            */
  int n_hidden;                /* number of Linear+LIF blocks            */
  int hidden[ORC_MAX_HIDDEN];  /* LIF widths                             */
  int classes;                 /* readout width (Linear + LI)            */
  int bias;                    /* Linear layers carry a bias entry       */
  float threshold;             /* LIF threshold theta (network.hpp:47)   */
  int act;                     /* enum orc_act                           */
  float slope;                 /* ActivationDesc.slope                   */
  float aux;                   /* ActivationDesc.aux (boxcar height)     */
  int unroll;                  /* TrainConfig.unroll (optimize.hpp:130)  */
  /* BetaMode per cell (neuron.hpp:24, network.hpp:45-53): index l < n_hidden =
   * LIF layer l, index n_hidden = the LI readout.  0 PerNeuron (entry [H]),
   * 1 LearnableScalar (entry [] = 1 value), 2 Fixed (entry [] = fixed_beta,
   * not trainable).  Zero-initialised = PerNeuron everywhere.             */
  int beta_mode[ORC_MAX_HIDDEN + 1];
  float fixed_beta[ORC_MAX_HIDDEN + 1];
  /* MonitorLayer after LIF layer l (network.hpp:57, :139-144): spike counts
   * over time (neuron.hpp:106-114) that feed the activity regularizer.  A
   * monitor takes a normalised layer id, so every later layer's id -- its
   * init key child(id) and entry names -- moves up by one.                 */
  int monitor[ORC_MAX_HIDDEN];
  /* Cell kind of hidden layer l: 0 LIF (neuron.hpp:127-136), 1 ALIF, 2 RLIF.
   *
   * ALIF is NOT in the reference: this is a
   * DECLARED restatement -- parity unpinned against the reference.  It follows
   * the adaptive-threshold LIF of Spyx (the paper's library; the
   * LSNN form of Bellec et al. 2018) written in the reference's LIF op order:
   *   th = theta + a ;  pre = v - th ;  s = [pre >= 0]
   *   v' = ((v * bc) + I) - s * th        (bc = clip01(beta))
   *   a' = (a * gc) + (1 - gc) * s        (gc = clip01(gamma), a_0 = 0)
   * The cell carries a second per-neuron entry "l{id}.gamma" after "l{id}.beta",
   * initialised TN(0.5, 0.25, +-2 sigma) from child(cell_key, 3) (beta uses
   * child 2).  The backward is the exact reverse of these ops (surrogate on pre,
   * reset and threshold paths differentiated); tests/test_alif_oracle.py pins it
   * against torch autograd of the same forward.
   *
   * RLIF is likewise NOT in the reference (feed-forward only, network.hpp:16,
   * SPEC.md:382, :456): a DECLARED restatement of Spyx's recurrent LIF in the
   * reference's LIF op order -- parity unpinned against the reference:
   *   pre = v - theta ; s = [pre >= 0] ; fb_j = sum_i s_i rec[i][j]
   *   v' = (((v * bc) + I) + fb) - s * theta
   * fb sums the rows of the spiking neurons in ascending i (the zero-skip
   * matmul order, ops.hpp:163-172).  Entry "l{id}.rec" [H][H] (row = source
   * neuron) after "l{id}.beta", init TN(0, 1/sqrt(H), +-2 sigma) from
   * child(cell_key, 4).  Pinned against torch autograd like ALIF.          */
  int cell[ORC_MAX_HIDDEN];
  /* Readout cell (network.hpp:153-155: a network ends in a LIF or LI readout):
   * 0 LI (neuron.hpp:139-144, the trace is the membrane), 1 LIF (the trace is the
   * readout's spikes, network.hpp:396; its threshold / surrogate are the hidden
   * layers' theta / act).  The readout beta entry and init are the same for both
   * (init_lif, network.hpp:266-279).                                          */
  int readout_lif;
} orc_net;

/* Parameter entries in NetworkParams order (network.hpp:231-286). */
int orc_entry_count(const orc_net* net);
/* offsets/sizes in floats into the flat parameter vector; names "l{i}.w" ... */
void orc_entry_layout(const orc_net* net, size_t* offsets, size_t* sizes,
                      char (*names)[16]);
size_t orc_param_count(const orc_net* net);

/* SplitMix64 key algebra (rng.hpp:20-48). Keys are the 64-bit `word`. */
uint64_t orc_key_from_seed(uint64_t seed);
uint64_t orc_key_child(uint64_t key, uint64_t index);
uint64_t orc_key_bits(uint64_t key, uint64_t counter);
double orc_uniform01(uint64_t key, uint64_t counter);
void orc_permutation(uint64_t key, size_t n, uint64_t* out);
void orc_truncated_normal(uint64_t key, size_t n, float mean, float stddev,
                          float* out);

/* synth_raster (commands.hpp:50-86): x [n, t, f] u8, y [n]. */
void orc_synth_raster(size_t classes, size_t n, size_t t, size_t f,
                      uint64_t seed, uint8_t* x, int64_t* y);
/* pack_time / unpack_time along axis 1 (data.hpp:105-149). */
void orc_pack_time(const uint8_t* x, size_t n, size_t t, size_t f,
                   uint8_t* out);
void orc_unpack_time(const uint8_t* packed, size_t n, size_t t, size_t f,
                     uint8_t* out);

/* init(spec, key, sample) (network.hpp:231-286); key = master.child(0). */
void orc_init(const orc_net* net, uint64_t key, float* params);

/*
 * One taped forward + loss + accuracy + reverse sweep (optimize.hpp:152-203),
 * without the optimizer update.  packed: [B, ceil(T/8), in] MSB-first.
 * Outputs (all optional except loss/acc):
 *   grads   [param_count]                 tape.grad of every entry
 *   spikes  [sum_l B*T*hidden[l]]  u8     hidden spike rasters, layer-major
 *   vtrace  [sum_l B*T*hidden[l]]  f32    membrane entering each step
 *   trace   [B*T*classes]          f32    LI readout trace
 * Returns 0 on success, nonzero on a shape/argument error.
 */
int orc_forward_backward(const orc_net* net, const float* params,
                         const uint8_t* packed, size_t batch, size_t t_steps,
                         const int64_t* targets, float* loss, double* acc,
                         float* grads, uint8_t* spikes, float* vtrace,
                         float* trace);

/* TrainConfig options on the same path (optimize.hpp:113-131), all off by default. */
typedef struct orc_train_opts {
  int optimizer;   /* 0 Adam (optimize.hpp:86-111), 1 SGD + momentum (:69-84)       */
  float momentum;  /* SGD momentum (TrainConfig.momentum, default 0.9)              */
  int loss;        /* 0 integral CE (objective.hpp:88-114), 1 spike-rate MSE (:139-183) */
  float rate_hi;   /* rate-MSE target on the true class (default 0.9)               */
  float rate_lo;   /* rate-MSE target elsewhere (default 0.1)                       */
  /* shift_augment in the epoch loop (data.hpp:216-227, optimize.hpp:278-280):
   * per batch b and listed axis i a roll by randint(epoch_key.child(1+b), i,
   * -max_shift, max_shift); axes must name the feature axis (2 or -1).      */
  int max_shift;
  int n_shift_axes;
  int shift_axes[4];
  /* activity regularizer on every monitor (objective.hpp:186-227, optimize.hpp:185-191);
   * both lambdas zero = off (defaults f_min 0, f_max 1)                    */
  float f_min, f_max, lambda_low, lambda_high;
} orc_train_opts;

/* forward_backward / train_step with TrainConfig options (NULL = defaults). */
int orc_forward_backward_ex(const orc_net* net, const orc_train_opts* opts,
                            const float* params, const uint8_t* packed,
                            size_t batch, size_t t_steps, const int64_t* targets,
                            float* loss, double* acc, float* grads,
                            uint8_t* spikes, float* vtrace, float* trace);
int orc_train_step_ex(const orc_net* net, const orc_train_opts* opts,
                      float* params, float* m, float* v, uint64_t* step,
                      const uint8_t* packed, size_t batch, size_t t_steps,
                      const int64_t* targets, float lr, float* loss, double* acc);
/* train() epoch loop with TrainConfig options, shift augmentation included. */
int orc_train_epochs_ex(const orc_net* net, const orc_train_opts* opts, float* params,
                        float* m, float* v, uint64_t* step, const uint8_t* packed,
                        const int64_t* y, size_t n, size_t t_steps, size_t batch,
                        size_t epochs, uint64_t seed, float lr, double* metrics);
/* Teacher-forced forward_backward (TEST-ONLY diagnostic): identical to
 * orc_forward_backward_ex except that every hidden cell's spike s_t is taken
 * from `forced` (layer-major u8 rasters [sum_l B*T*hidden[l]], the layout of
 * spikes_out) instead of [v - th >= 0]; membranes, resets, surrogates and all
 * gradients then follow those spikes.  Fed the GPU's own rasters it isolates
 * the gradient error of the kernels from the legitimate effect of a spike
 * that flipped on an fp32 near-tie.                                           */
int orc_forward_backward_forced(const orc_net* net, const orc_train_opts* opts,
                                const float* params, const uint8_t* packed, size_t batch,
                                size_t t_steps, const int64_t* targets, const uint8_t* forced,
                                float* loss, double* acc, float* grads,
                                uint8_t* spikes, float* vtrace, float* trace);

/* sgd_update over a flat buffer (optimize.hpp:69-84): m doubles as momentum. */
void orc_sgd(float* p, const float* g, float* m, size_t n, uint64_t* step,
             float lr, float momentum);

/* adam_update over a flat buffer (optimize.hpp:86-111); *step is the
 * optimizer step counter, incremented here before the bias correction. */
void orc_adam(float* p, const float* g, float* m, float* v, size_t n,
              uint64_t* step, float lr, float beta1, float beta2, float eps);

/* Full train_step: forward_backward + Adam over trainable entries. */
int orc_train_step(const orc_net* net, float* params, float* m, float* v,
                   uint64_t* step, const uint8_t* packed, size_t batch,
                   size_t t_steps, const int64_t* targets, float lr,
                   float* loss, double* acc);

/*
 * train(TrainState&, data) epoch loop (optimize.hpp:260-299): per epoch e the
 * permutation key master.child(1+e).child(0), drop-remainder batches, one
 * train_step each.  metrics: [epochs][2] = {mean loss, mean accuracy}.
 */
int orc_train_epochs(const orc_net* net, float* params, float* m, float* v,
                     uint64_t* step, const uint8_t* packed, const int64_t* y,
                     size_t n, size_t t_steps, size_t batch, size_t epochs,
                     uint64_t seed, float lr, double* metrics);

#ifdef __cplusplus
}
#endif

#endif
