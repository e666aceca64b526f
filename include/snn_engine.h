/*
 * snn_engine.h -- C ABI of the B200-native SNN training engine.
 *
 * Drop-in boundary for the reference's training step.  Each entry point cites
 * the reference interface it replaces (paths relative to
 * /root/reference/proj/include/spiketrain/).  Plain pointers and sizes only:
 * no torch, no C++ types.  All compute runs on the GPU through hand-written
 * sm_100a kernels; there is no CPU fallback -- without a usable B200 every
 * call that needs the device returns SNN_ERR_CUDA.
 *
 * Threading: an engine handle is not thread-safe (the reference Tape is
 * single-threaded and single-use, autodiff.hpp:12-16).  Distinct handles may
 * be driven from distinct threads.
 */
#ifndef SNN_ENGINE_H
#define SNN_ENGINE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNN_ABI_VERSION 8
#define SNN_MAX_HIDDEN 8

/* Error taxonomy, 1:1 with spiketrain's exception classes (errors.hpp:9-64). */
typedef enum snn_status {
  SNN_OK = 0,
  SNN_ERR_SHAPE = 1,       /* ShapeError       */
  SNN_ERR_ARGUMENT = 2,    /* ArgumentError    */
  SNN_ERR_CONTRACT = 3,    /* ContractError    */
  SNN_ERR_STATE = 4,       /* StateError       */
  SNN_ERR_FORMAT = 5,      /* FormatError      */
  SNN_ERR_IO = 6,          /* IoError          */
  SNN_ERR_SPEC = 7,        /* SpecError        */
  SNN_ERR_CONFIG = 8,      /* ConfigError      */
  SNN_ERR_UNSUPPORTED = 9, /* UnsupportedError */
  SNN_ERR_CUDA = 10        /* device failure or no B200: nothing ran on the CPU */
} snn_status;

/* Surrogate catalogue (surrogate.hpp:134-157 make_activation). */
typedef enum snn_activation {
  SNN_ACT_CUSTOM = 0,
  SNN_ACT_SUPERSPIKE = 1,
  SNN_ACT_TRIANGULAR = 2,
  SNN_ACT_ARCTAN = 3,
  SNN_ACT_BOXCAR = 4,
  /* DECLARED, not in the reference catalogue ("addable via
   * custom()"; config.hpp:487-490 rejects the name): custom(heaviside, bwd)
   * with bwd = d/dx sigmoid(kx) = k e / (1 + e)^2, e = exp(-k |x|) (the
   * cancellation-free form of k s (1 - s)); slope k default 25.              */
  SNN_ACT_SIGMOID = 5
} snn_activation;

/*
 * NetworkSpec for the supported family (network.hpp:62-65):
 *   input_shape {input}; layers = [Linear(hidden[i], bias), LIF]*n_hidden,
 *                                  Linear(classes, bias), LI
 * LIF: LIFLayer{activation, PerNeuron beta, threshold} (network.hpp:42-48);
 * LI : LILayer{PerNeuron} (network.hpp:50-54).
 */
typedef struct snn_network_desc {
  int32_t input;
  int32_t n_hidden;
  int32_t hidden[SNN_MAX_HIDDEN];
  int32_t classes;
  int32_t bias;         /* LinearLayer.bias (network.hpp:25) */
  float threshold;      /* LIFLayer.threshold, must be > 0  */
  int32_t activation;   /* snn_activation                   */
  float slope;          /* ActivationDesc.slope             */
  float aux;            /* ActivationDesc.aux               */
  /* BetaMode per cell (neuron.hpp:24; LIFLayer/LILayer.beta_mode): index l <
   * n_hidden = LIF layer l, index n_hidden = the LI readout.  0 PerNeuron (entry
   * [H]), 1 LearnableScalar (entry [], one value), 2 Fixed (entry [] = fixed_beta,
   * not trainable).  Zero = PerNeuron everywhere. */
  int32_t beta_mode[SNN_MAX_HIDDEN + 1];
  float fixed_beta[SNN_MAX_HIDDEN + 1];
  /* MonitorLayer after hidden LIF l (network.hpp:57, :139-144): its spike counts
   * feed the activity regularizer and are readable with snn_monitor_counts.  A
   * monitor takes a normalised layer id, so the entry names and init keys of
   * every later layer move up by one (network.hpp:231-286). */
  int32_t monitor[SNN_MAX_HIDDEN];
  /* Cell kind of hidden layer l (snn_cell).  SNN_CELL_ALIF is a DECLARED cell that
   * the reference does not have: threshold theta + a, reset by
   * it, a' = a*clip01(gamma) + (1 - clip01(gamma))*s, with a second per-neuron entry
   * "l{id}.gamma" after "l{id}.beta" (init TN(0.5, 0.25) from child(cell_key, 3)).
   * Its checker is the restatement in oracle/spiketrain_oracle.h.  Zero = LIF. */
  int32_t cell[SNN_MAX_HIDDEN];
  /* readout cell (network.hpp:153-155): 0 LILayer (the trace is its membrane),
   * 1 LIFLayer (the trace is its spikes, network.hpp:396; same threshold and
   * surrogate as the hidden LIF layers, beta entry and init as for LI) */
  int32_t readout_lif;
} snn_network_desc;

/* SNN_CELL_RLIF is likewise DECLARED (the reference is feed-forward only, network.hpp:16,
 * SPEC.md:382): pre = v - theta, s = [pre >= 0], fb_j = sum_i s_i rec[i][j] (spiking i
 * ascending), v' = (((v*clip01(beta)) + I) + fb) - s*theta, with an entry "l{id}.rec"
 * [H][H] after "l{id}.beta" (init TN(0, 1/sqrt(H)) from child(cell_key, 4)); H <= 1024. */
typedef enum snn_cell { SNN_CELL_LIF = 0, SNN_CELL_ALIF = 1, SNN_CELL_RLIF = 2 } snn_cell;

/* TrainConfig subset that reaches the step (optimize.hpp:116-133). */
typedef struct snn_train_config {
  int32_t batch_size;   /* examples per step on THIS rank (global = batch_size * world) */
  int32_t time_steps;   /* original T of the packed data (PackedDataset.original_t) */
  float lr;             /* TrainConfig.lr, Adam (optimize.hpp:86-111) */
  float beta1, beta2, eps;
  uint64_t seed;        /* TrainConfig.seed: init key child(0), epoch keys child(1+e) */
  int32_t unroll;       /* accepted for API parity; scheduling only (network.hpp:352) */
  /* TrainConfig options on the step (optimize.hpp:113-131); zero = Adam + integral CE */
  int32_t optimizer;    /* 0 Adam, 1 SGD with momentum (optimize.hpp:69-84) */
  float momentum;       /* SGD momentum (TrainConfig default 0.9) */
  int32_t loss;         /* 0 integral CE (objective.hpp:88-114), 1 spike-rate MSE (:139-183) */
  float rate_hi, rate_lo; /* rate-MSE targets on / off the true class (defaults 0.9 / 0.1) */
  /* shift_augment in the epoch loop (optimize.hpp:131-132, 276-278, data.hpp:216-227):
   * when max_shift > 0 every batch of snn_train_epochs is rolled along the feature
   * axis by sum_i randint(child(epoch_key, 1 + b), i, -max_shift, max_shift).
   * Axes 0 / 1 are rejected like train() does; with max_shift > 0 only the feature
   * axis (2 or -1) is supported. */
  int32_t max_shift;
  int32_t n_shift_axes; /* 0..4 */
  int32_t shift_axes[4];
  /* activity regularizer on every monitor (objective.hpp:186-227, optimize.hpp:185-191):
   * squared hinge on the rates count/T outside [f_min, f_max]; both lambdas 0 = off
   * (then the band is not checked, like the reference). */
  float f_min, f_max, lambda_low, lambda_high;
  /* GEMM precision mode (not a reference option): bf16 operand planes per real
   * operand on the tensor cores.  0 or 3 = the fp32 path (x = hi + mid + lo, 2^-24:
   * the north_star parity bar); 2 = fast mode (hi + mid, <= 2^-16 relative per
   * operand; dS uses hi*hi + hi*mid + mid*hi); 1 = bf16 (hi only).  The sparse
   * readout projection and every scan stay fp32 in all modes.  Fast modes are
   * reported separately with their own measured tolerance. */
  int32_t gemm_planes;
} snn_train_config;

typedef struct snn_engine snn_engine;

/* Last error message of a handle (or of the last failed create when NULL). */
const char* snn_last_error(const snn_engine* e);
int snn_abi_version(void);

/* Construct: validates the spec like normalize() (network.hpp:125-157),
 * allocates all device state, initialises parameters exactly like
 * train(spec, cfg, data) does (init(spec, master.child(0)), optimize.hpp:246-254). */
snn_status snn_engine_create(const snn_network_desc* net, const snn_train_config* cfg,
                             int device, snn_engine** out);
void snn_engine_destroy(snn_engine* e);

/* NetworkParams as one flat f32 vector in entry order l{i}.w, l{i}.b, l{i}.beta
 * (network.hpp:164-226).  Entry i: name, offset, size, trainable. */
snn_status snn_param_count(const snn_engine* e, size_t* n);
snn_status snn_entry_count(const snn_engine* e, int32_t* n);
snn_status snn_entry_info(const snn_engine* e, int32_t i, char name[16], size_t* offset,
                          size_t* size, int32_t* trainable);
snn_status snn_set_params(snn_engine* e, const float* host, size_t n);
snn_status snn_get_params(snn_engine* e, float* host, size_t n);
/* Reference init (network.hpp:231-286) from an explicit key word. */
snn_status snn_init_params(snn_engine* e, uint64_t key_word);
/* OptimizerState m, v, step (optimize.hpp:28-48), trainable entries in order. */
/* Checkpoints in the reference .spkc format (optimize.hpp:300-436), bit-exact:
 * parameters, optimizer kind / step / m (/ v for Adam) and the caller's config
 * text with its FNV-1a hash.  Load checks the entries against the network and
 * copies the stored config text into config_out (NUL-terminated, truncated to
 * config_cap) and its full length into *config_len (either may be NULL). */
snn_status snn_save_checkpoint(snn_engine* e, const char* path, const char* config_text,
                               size_t config_len);
snn_status snn_load_checkpoint(snn_engine* e, const char* path, char* config_out,
                               size_t config_cap, size_t* config_len);
snn_status snn_get_opt_state(snn_engine* e, float* m, float* v, uint64_t* step, size_t n);
snn_status snn_set_opt_state(snn_engine* e, const float* m, const float* v, uint64_t step,
                             size_t n);
/* Gradients of the last step (tape.grad of every entry, before the update). */
snn_status snn_get_grads(snn_engine* e, float* host, size_t n);

/* PackedDataset staged once in HBM (data.hpp:159-163): packed u8
 * [n][ceil(T/8)][input] MSB-first, labels in [0, classes). */
snn_status snn_stage_dataset(snn_engine* e, const uint8_t* packed, size_t n,
                             const int64_t* labels);

/* synth_raster(classes, n, T, {input}, seed) + pack_time generated on the GPU
 * straight into the staged HBM dataset, bit-identical to the reference
 * (commands.hpp:50-86, data.hpp:105-126, rng.hpp:20-64). */
snn_status snn_synth_dataset(snn_engine* e, size_t n, uint64_t seed);

/* Copy rows [start, start+n) of the staged dataset back to the host in the
 * reference's packed layout [n][ceil(T/8)][input] + labels. */
snn_status snn_read_dataset(snn_engine* e, size_t start, size_t n, uint8_t* packed,
                            int64_t* labels);

/* .spkd container I/O (data.hpp:229-341): snn_load_container reads the
 * reference's read_container format with its checks and error classes
 * (FormatError with byte offsets, IoError) and stages it like
 * snn_stage_dataset; the container's T must be the engine's and its per-step
 * feature dims must flatten to the network input.  snn_save_container writes
 * the staged dataset as [N, ceil(T/8), input] byte-for-byte like
 * write_container. */
snn_status snn_load_container(snn_engine* e, const char* path, size_t* n);
snn_status snn_save_container(snn_engine* e, const char* path);

/* permutation(master.child(1+epoch).child(0), n): the epoch shuffle of
 * train() (optimize.hpp:266-268, data.hpp:181-208, rng.hpp:78-87). */
snn_status snn_epoch_permutation(snn_engine* e, size_t epoch, uint32_t* out, size_t n);

/* train_step on rows of the staged dataset (optimize.hpp:152-214).  rows: host
 * array of batch_size dataset indices.  Updates params + optimizer state in
 * place and returns StepResult{loss, accuracy} (global over ranks). */
snn_status snn_train_step(snn_engine* e, const uint32_t* rows, float* loss, double* accuracy);

/* Reference-shaped compatibility entry: train_step(st, packed_x, T, targets)
 * with a HOST packed batch [batch_size][ceil(T/8)][input] and int64 targets. */
snn_status snn_train_step_packed(snn_engine* e, const uint8_t* packed_batch,
                                 const int64_t* targets, float* loss, double* accuracy);
/* The reference's train() loop over host batches (optimize.hpp:260-299, one train_step
 * per batch) with the uploads pipelined: n_steps packed batches back to back in host
 * memory ([n_steps][B][ceil(T/8)][input], pinned for overlap) and their targets
 * [n_steps][B].  Batch k+1 is DMA'd and re-laid out on a copy stream while step k runs;
 * every step's StepResult is read back (losses / accuracies [n_steps], may be NULL).
 * Same results as n_steps calls of snn_train_step_packed. */
snn_status snn_train_steps_packed(snn_engine* e, const uint8_t* packed, const int64_t* targets,
                                  size_t n_steps, float* losses, double* accuracies);

/* Forward + loss + reverse sweep without the optimizer update (gradients are
 * then readable with snn_get_grads). */
snn_status snn_forward_backward(snn_engine* e, const uint32_t* rows, float* loss,
                                double* accuracy);

/* train(TrainState&, data) epoch loop over the staged dataset
 * (optimize.hpp:260-299): epoch e shuffles with master.child(1+e).child(0),
 * drop-remainder batches.  metrics: [epochs][2] mean loss, mean accuracy. */
snn_status snn_train_epochs(snn_engine* e, size_t epochs, double* metrics);
/* Same loop for epochs [first_epoch, first_epoch + epochs) of the key schedule. */
snn_status snn_train_epochs_from(snn_engine* e, size_t first_epoch, size_t epochs,
                                 double* metrics);

/* Asynchronous stepping for throughput measurement: enqueue one full step
 * (captured CUDA graph) on the engine stream with batch rows taken from slot
 * `slot` of the uploaded device-resident schedule; no host sync.  The slot is
 * a device counter the step advances, so consecutive slots need no host->device
 * traffic.  snn_enqueue_steps enqueues slots [first_slot, first_slot + n_steps)
 * as multi-step graphs (8 steps per graph launch). */
snn_status snn_upload_schedule(snn_engine* e, const uint32_t* rows, size_t n_steps);
snn_status snn_enqueue_step(snn_engine* e, size_t slot);
snn_status snn_enqueue_steps(snn_engine* e, size_t first_slot, size_t n_steps);
/* Forward launches of one step: launch i runs hidden layers [first, first + count)
 * (narrow layers are fused into one launch).  Returns count, or 0 when i is out of
 * range; *first may be NULL. */
int32_t snn_forward_launch_layers(const snn_engine* e, int32_t i, int32_t* first);
/* Evaluation.  snn_evaluate mirrors cmd_eval
 * (commands.hpp:144-169): integral accuracy over `n` dataset rows walked in
 * batches of the engine batch size (last batch short), forward only; mean_loss
 * (optional) is the mean integral-CE loss over the rows.  snn_apply mirrors
 * apply (network.hpp:435-448) for one batch of B rows: the readout trace
 * [B][T][classes] (n = B*T*classes floats). */
snn_status snn_evaluate(snn_engine* e, const uint32_t* rows, size_t n, double* accuracy,
                        double* mean_loss);
snn_status snn_apply(snn_engine* e, const uint32_t* rows, float* trace, size_t n);
/* ApplyResult.monitors (network.hpp:435-448, neuron.hpp:106-114): spike counts
 * [B][hidden[layer]] of the monitor after hidden LIF `layer`, from the last
 * forward (snn_apply, a step, or an evaluation batch). */
snn_status snn_monitor_counts(snn_engine* e, int32_t layer, float* counts, size_t n);
snn_status snn_sync(snn_engine* e);
snn_status snn_read_result(snn_engine* e, float* loss, double* accuracy);
/* cudaStream_t of the engine, for CUDA-event timing by the caller. */
void* snn_stream(snn_engine* e);
/* Number of kernel launches one step issues. */
int32_t snn_launches_per_step(const snn_engine* e);
/* Device time of every launch of a step, averaged over `steps` steps (a
 * captured graph with event-record nodes between kernels). */
snn_status snn_profile_steps(snn_engine* e, int32_t steps, double* ms, int32_t max_launches,
                             int32_t* n_launches);
const char* snn_launch_name(const snn_engine* e, int32_t i);

/* Data-parallel training: one engine per GPU/process.  Every rank passes the
 * same 128-byte ncclUniqueId (rank 0 creates it with snn_nccl_unique_id).
 * After this call each step allreduces the flat gradient (sum) and uses the
 * global batch in the loss mean. */
snn_status snn_nccl_unique_id(uint8_t id[128]);
snn_status snn_comm_init(snn_engine* e, const uint8_t id[128], int32_t rank, int32_t world);

/* Data-parallel training over peer memory (the B200-native tail; replaces the
 * NCCL allreduce + update): each rank exports its exchange buffer with
 * snn_peer_handle (a 64-byte cudaIpcMemHandle_t), the caller all-gathers the
 * handles (bench.py: torch.distributed.all_gather_object) and every rank calls
 * snn_peer_open with all of them in rank order.  A step then ends, owner-computes,
 * with k_reduce (local gradient + loss into the exchange buffer, release flag A
 * to every rank), k_peer_owner (rank r waits for all A flags, sums ITS parameter
 * slice [r n/W, (r+1) n/W) over the ranks' buffers by peer loads in rank order,
 * Adam/SGD on that slice -- m, v sharded with the owner -- result into its own
 * buffer, release flag B to every rank) and k_peer_gather (wait for all B flags,
 * copy every slice from its owner, planes, StepResult): ~2 n (W-1)/W floats read
 * per rank per step, bit-identical replicas, no NCCL.  snn_get_opt_state and
 * checkpoints pull the other owners' m / v slices back first.  A peer that never
 * publishes (SNN_PEER_TIMEOUT_S, default 20 s) raises SNN_ERR_CUDA on the next
 * result read instead of hanging.  world <= 8, one node (IPC handles). */
snn_status snn_peer_handle(snn_engine* e, uint8_t handle[64]);
snn_status snn_peer_open(snn_engine* e, int32_t rank, int32_t world, const uint8_t* handles);
/* Test hooks for the peer tail with fewer GPUs than ranks (B200_PROFILING: ranks
 * whose kernels wait on one another must not run as separate launches on one
 * GPU): attach `world` engines of ONE device as ranks 0..world-1 through plain
 * device pointers, and split a step at its cross-rank waits (part 0: forward ..
 * k_reduce; part 1: k_peer_owner; part 2: k_peer_gather -> StepResult).  Running
 * each part on every rank before any rank's next part means no kernel ever waits
 * on a rank that has not run. */
snn_status snn_peer_attach_local(snn_engine* const* engines, int32_t world);
snn_status snn_train_step_split(snn_engine* e, const uint32_t* rows, int32_t part, float* loss,
                                double* accuracy);

/* Diagnostics: raw intermediate tensors of the last forward_backward when
 * enabled (costs extra HBM writes; off by default).  snn_debug_enable(e, 1):
 * tensors + per-CTA clock stamps; (e, 2): clock stamps only (the kernels keep
 * their production code paths); (e, 0): off.
 *   which 0: projection I of hidden layer `layer`   [B][T][H]
 *         1: membrane V (entering step t)           [B][T][H]
 *         2: spikes (0/1 as u8)                     [B][T][H]
 *         3: readout trace                          [B][T][C]
 *         4: dS (grad of spikes) of hidden `layer`  [B][T][H]
 *         5: per-kernel phase clocks (tests/clk_probe.py)
 *         6: ALIF adaptation a (entering step t)    [B][T][H]
 *         7: dI of Linear `layer` (0..L, L = readout; hi + (mid + lo) of
 *            its three bf16 planes)                 [B][T][H or C]  */
snn_status snn_debug_enable(snn_engine* e, int32_t on);
/* With SNN_GUARD=1 in the environment when buffers are allocated, every device
 * buffer of the process carries 4 KB of a known byte pattern past its end;
 * this checks them all (SNN_ERR_CONTRACT names the first overwritten one) and
 * returns how many buffers were checked (0 when guards are off). */
snn_status snn_debug_check_guards(snn_engine* e, int32_t* checked);
snn_status snn_debug_fetch(snn_engine* e, int32_t which, int32_t layer, void* host, size_t bytes);

#ifdef __cplusplus
}
#endif

#endif /* SNN_ENGINE_H */
