// engine.cu -- host side of the B200 SNN training engine and its C ABI
// (include/snn_engine.h).  One engine = one GPU = one data-parallel rank.
//
// Step schedule (all on one stream, captured once into a CUDA graph):
//   k_lif_fwd x L          GEMM (tcgen05, TMEM) + LIF scan per (sample, 128 neurons)
//   k_readout              readout projection + LI + integral CE + LI reverse scan
//   k_lif_bwd              dS = dI_next W_next^T on tcgen05 + LIF reverse scan (TMEM epilogue)
//   k_wgrad x (L+1)        dW = A^T dI on tcgen05, split-K partials
//   k_reduce (+loss, step), [ncclAllReduce], k_adam (+StepResult)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <memory>
#include <string>
#include <vector>

#include "../../include/snn_engine.h"
#include "host_rng.hpp"
#include "kernels.cuh"

using namespace snn;

namespace {

thread_local std::string g_create_error;

struct SnnError {
  snn_status code;
  std::string msg;
};

[[noreturn]] void fail(snn_status code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  throw SnnError{code, buf};
}

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t err__ = (x);                                                           \
    if (err__ != cudaSuccess)                                                          \
      fail(SNN_ERR_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(err__), __FILE__, \
           __LINE__);                                                                  \
  } while (0)

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  using comm_t = void*;
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(comm_t*, int, void* /*by value 128B*/, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, comm_t, cudaStream_t) = nullptr;
  int (*CommDestroy)(comm_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
};

struct UniqueId {
  char internal[128];
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* env = std::getenv("SNN_NCCL_LIB");
    void* h = nullptr;
    if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
      api.AllReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*,
                                               cudaStream_t)>(dlsym(h, "ncclAllReduce"));
      api.CommDestroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
      api.GetErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
      api.CommInitRank = reinterpret_cast<int (*)(void**, int, void*, int)>(
          dlsym(h, "ncclCommInitRank"));
      api.ok = api.GetUniqueId && api.AllReduce && api.CommDestroy && api.CommInitRank;
    }
  }
  return api;
}

// ncclCommInitRank takes ncclUniqueId by value (128 bytes): call through a
// correctly typed pointer.
using InitRankFn = int (*)(void**, int, UniqueId, int);

// -------------------------------------------------------------- tensor maps
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 tensor [rows][cols] (cols contiguous), box {64 cols, box_rows}, 128B swizzle.
CUtensorMap make_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return m;
}

// 2-D f32 tensor [rows][cols], box {32 cols, 128 rows}, 128B swizzle (wgrad partials).
CUtensorMap make_map_f32(const void* base, uint64_t rows, uint64_t cols) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (%d)", int(r));
  return m;
}

// Out-of-bounds write guards (SNN_GUARD=1, diagnostics): every device buffer gets
// kGuardBytes of a known pattern past its end, checked by snn_debug_check_guards.
// Stands in for compute-sanitizer, which this GPU pool does not allow.
namespace guards {
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kPattern = 0xA5;
inline bool enabled() {
  static const bool on = [] {
    const char* v = std::getenv("SNN_GUARD");
    return v && *v == '1';
  }();
  return on;
}
inline std::mutex& mu() {
  static std::mutex m;
  return m;
}
inline std::map<const void*, size_t>& live() {  // base pointer -> data bytes
  static std::map<const void*, size_t> m;
  return m;
}
}  // namespace guards

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count, bool zero = true) {
    free();
    n = count;
    if (count == 0) return;
    const size_t bytes = count * sizeof(T), extra = guards::enabled() ? guards::kGuardBytes : 0;
    CK(cudaMalloc(&p, bytes + extra));
    if (extra) {
      CK(cudaMemset(reinterpret_cast<unsigned char*>(p) + bytes, guards::kPattern, extra));
      CK(cudaDeviceSynchronize());
      std::lock_guard<std::mutex> lk(guards::mu());
      guards::live()[p] = bytes;
    }
    if (zero) {
      // the legacy stream is not ordered with the engine's non-blocking stream:
      // finish the fill before any engine work can touch the buffer
      CK(cudaMemsetAsync(p, 0, count * sizeof(T), cudaStreamLegacy));
      CK(cudaStreamSynchronize(cudaStreamLegacy));
    }
  }
  void free() {
    if (p) {
      if (guards::enabled()) {
        std::lock_guard<std::mutex> lk(guards::mu());
        guards::live().erase(p);
      }
      cudaFree(p);
    }
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { free(); }
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

inline int rup(int x, int m) { return (x + m - 1) / m * m; }

struct EntryHost {
  std::string name;
  int kind, layer, rows, cols;
  size_t offset, size;
  int beta_mode = 0;  // beta entries: 0 per neuron [H], 1 scalar [], 2 fixed [] (constant)
  bool trainable() const { return !(kind == kEntryBeta && beta_mode == 2); }
  int ndim() const { return kind == kEntryW ? 2 : (kind == kEntryBeta && beta_mode != 0 ? 0 : 1); }
};

struct Dataset {
  DevBuf<uint8_t> x;       // [n][T_pad/8][row]
  DevBuf<int32_t> labels;  // [n]
  size_t n = 0;
  int row = 0;             // bytes per packed time row: IN_pad (staged), or IN for a host
                           // batch kept in the reference layout (Engine::raw_layout_ok); 0 = IN_pad
};

// Host memcpy split over a few persistent worker threads (the caller takes part).
// A host batch (e.g. 2.87 MB at C1) is copied into pinned memory at several times
// one core's memcpy rate; the engine pipelines the chunks with their DMA.  Workers
// spin on an atomic job counter for ~2 ms after each job (steps arrive every few
// hundred us while training) and sleep on a condition variable otherwise.
class CopyPool {
 public:
  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(void* dst, const void* src, size_t bytes) {
    dst_ = static_cast<uint8_t*>(dst);
    src_ = static_cast<const uint8_t*>(src);
    bytes_ = bytes;
    pending_.store(int(th_.size()), std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu_);  // orders the job fields before the counter
      gen_.fetch_add(1, std::memory_order_release);
    }
    if (sleepers_.load() > 0) cv_.notify_all();
    part(0);
    while (pending_.load(std::memory_order_acquire) > 0) cpu_relax();
  }

 private:
  static void cpu_relax() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  void part(int i) {
    const size_t parts = th_.size() + 1;
    const size_t per = ((bytes_ + parts - 1) / parts + 63) & ~size_t(63);
    const size_t lo = std::min(bytes_, per * size_t(i)), hi = std::min(bytes_, lo + per);
    if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void run(int i) {
    uint64_t seen = 0;
    for (;;) {
      // spin ~2 ms for the next job, then sleep
      const auto t0 = std::chrono::steady_clock::now();
      for (int k = 0; gen_.load(std::memory_order_acquire) == seen && !stop_.load(); ++k) {
        cpu_relax();
        if ((k & 1023) == 1023 && std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(2)) {
          std::unique_lock<std::mutex> lk(mu_);
          sleepers_.fetch_add(1);
          cv_.wait(lk, [&] { return stop_.load() || gen_.load() != seen; });
          sleepers_.fetch_sub(1);
          break;
        }
      }
      if (stop_.load()) return;
      seen = gen_.load(std::memory_order_acquire);
      part(i + 1);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_;
  uint8_t* dst_ = nullptr;
  const uint8_t* src_ = nullptr;
  size_t bytes_ = 0;
  std::atomic<int> pending_{0}, sleepers_{0};
  std::atomic<uint64_t> gen_{0};
  std::atomic<bool> stop_{false};
};

}  // namespace

struct snn_engine {
  snn_network_desc net{};
  snn_train_config cfg{};
  int planes = 3;  // bf16 operand planes per real GEMM operand (cfg.gemm_planes)
  int device = 0;
  std::string err;

  // dimensions
  int B = 0, T = 0, TT = 0, NT = 0, T_pad = 0, IN = 0, IN_pad = 0, L = 0, C = 0;
  int H[SNN_MAX_HIDDEN]{}, H_pad[SNN_MAX_HIDDEN]{};
  int K[kMaxLayers]{}, N[kMaxLayers]{}, K_pad[kMaxLayers]{}, N_pad[kMaxLayers]{};
  int M_pad_w[kMaxLayers]{}, n_tile_w[kMaxLayers]{}, splits_w[kMaxLayers]{}, mg_w[kMaxLayers]{};
  int wg_stages_l[kMaxLayers]{};
  int wg_mg_max = 1;
  std::vector<EntryHost> entries;
  size_t n_params = 0;

  cudaStream_t stream = nullptr;
  // parameters / optimizer
  DevBuf<float> params, m, v, comm;  // comm = grads [n_params] + loss_sum + hits
  DevBuf<float> bc;
  size_t bc_steps = 0;
  DevBuf<int64_t> step;
  int64_t host_step = 0;               // host mirror of *step (advanced per update launch)
  DevBuf<int64_t> sched_slot;          // schedule mode: slot of the next step (device counter)
  DevBuf<unsigned int> tail_done;      // completion counter of k_reduce_adam
  DevBuf<unsigned int> wg_tile_cnt;    // fused tail: per output tile arrival counters
  DevBuf<unsigned int> wg_done;        // fused tail: k_wgrad completion counter
  int wg_blocks = 0, wg_tiles = 0, sm_count = 148;
  size_t slot_expected = ~size_t(0);   // host mirror of *sched_slot
  // bf16 operand planes of every Linear W [3][K_pad][N_pad] (hi/mid/lo split of the
  // f32 master): MN-major A of the forward GEMM, K-major A of the backward dS GEMM
  DevBuf<__nv_bfloat16> wb[kMaxLayers];
  // activations
  DevBuf<float> V[SNN_MAX_HIDDEN];
  DevBuf<float> Aad[SNN_MAX_HIDDEN], dgamma[SNN_MAX_HIDDEN];  // ALIF adaptation trace, d gamma partials
  // RLIF: projection I, dS, and the f32 transpose of rec per layer; the rec weight
  // gradient is an extra wgrad layer j = rec_j[l] in [L+1, NJ) (rec_l[j] = l)
  DevBuf<float> Ibuf[SNN_MAX_HIDDEN], dsbuf[SNN_MAX_HIDDEN], rec_t[SNN_MAX_HIDDEN];
  int NJ = 0, rec_j[SNN_MAX_HIDDEN]{}, rec_l[kMaxLayers]{};
  DevBuf<uint32_t> s_np[SNN_MAX_HIDDEN], s_tp[SNN_MAX_HIDDEN];
  DevBuf<__nv_bfloat16> di[kMaxLayers];  // per Linear j: dI of its output
  DevBuf<float> dbeta[kMaxLayers], dbias[kMaxLayers];
  DevBuf<float> loss_b;
  DevBuf<float> loss_terms;  // rate-MSE: [B][C] squared rate gaps
  DevBuf<unsigned int> hist;  // activity regularizer: [n_mon][T+1] spike-count histograms
  DevBuf<float> mon_counts;   // snn_monitor_counts output staging [B][H]
  std::vector<int> mon_layers;  // monitored hidden layers feeding the regularizer, in order
  DevBuf<int32_t> correct_b;
  DevBuf<float> partial[kMaxLayers];
  DevBuf<int32_t> vec_index;
  int n_vec = 0;
  DevBuf<float> result_loss;
  DevBuf<double> result_acc;
  // StepResult ring in mapped pinned memory, written by the one-rank fused tail at
  // entry (step & (kRing - 1)): host-batch calls read it after their sync
  static constexpr int64_t kRing = 4096;
  float* ring_loss_h = nullptr;
  double* ring_acc_h = nullptr;
  float* ring_loss_d = nullptr;
  double* ring_acc_d = nullptr;
  bool ring_on() const { return tail_mode == 0 && fused_tail(); }
  float* h_loss = nullptr;
  double* h_acc = nullptr;
  uint32_t* h_rows = nullptr;
  // data
  Dataset data, scratch;
  DevBuf<uint32_t> rows_cur, sched;
  DevBuf<int32_t> xshift;  // shift_augment roll of the current batch (0 = none)
  int32_t xshift_host = 0;
  size_t sched_steps = 0;
  // tensor maps
  CUtensorMap tm_wt[kMaxLayers], tm_wb[kMaxLayers], tm_di_k[kMaxLayers], tm_di_w[kMaxLayers];
  CUtensorMap tm_di_out[kMaxLayers];  // hidden dI planes, 128-row boxes (K3 TMA stores)
  WgradMaps wg_maps;
  // debug
  bool debug = false;   // capture intermediate tensors (+ clock stamps)
  bool clocks = false;  // clock stamps
  DevBuf<float> dbg_i[SNN_MAX_HIDDEN], dbg_ds[SNN_MAX_HIDDEN], dbg_trace;
  // evaluation graphs (update flag): kEval = forward + readout, kEvalTrace = + the
  // readout trace [B][T][C] into eval_trace (apply, network.hpp:435-448)
  static constexpr int kEval = 2, kEvalTrace = 3;
  DevBuf<float> eval_trace;
  DevBuf<long long> dbg_clk;
  // graphs keyed by (dataset ptr, update flag, mode): mode 0 = rows_cur, mode g >= 1 =
  // g consecutive schedule steps (rows from sched[*sched_slot])
  std::map<std::tuple<const void*, int, int>, cudaGraphExec_t> graphs;
  // multi-GPU: tail 0 = one rank (k_reduce_adam), 1 = NCCL (k_reduce, ncclAllReduce,
  // k_adam), 2 = peer memory, owner-computes (k_reduce publishing into IPC-mapped
  // exchange buffers, k_peer_owner updating this rank's slice, k_peer_gather)
  void* comm_handle = nullptr;
  int rank = 0, world = 1;
  int tail_mode = 0;
  DevBuf<uint8_t> peer_mem;          // [2][n_comm] f32 exchange buffers, then kMaxRanks u64 flags
  int64_t n_comm = 0;
  float* peer_xchg[kMaxRanks] = {};  // every rank's exchange buffer (mapped; own = local)
  unsigned long long* peer_flags[kMaxRanks] = {};    // every rank's A flags (k_reduce published)
  unsigned long long* peer_flags_b[kMaxRanks] = {};  // every rank's B flags (owner phase done)
  void* peer_ipc[kMaxRanks] = {};    // opened IPC mappings (closed on destroy)
  DevBuf<int64_t> peer_seq;
  DevBuf<unsigned int> peer_done;    // completion counters: [0] k_reduce, [1] k_peer_owner, [2] k_peer_gather
  DevBuf<unsigned int> peer_timeout; // set by a peer wait that gave up (checked on every result read)
  int split_part = -1;               // test hook: enqueue only part 0 (body + k_reduce), 1 (owner
                                     // phase) or 2 (gather) of a peer-tail step
  bool planes_dirty = true;
  // pipeline depths (smem per CTA decides how many CTAs share an SM)
  int fwd_stages = std::min(kFwdStagesMax, env_int("SNN_FWD_STAGES", 2));
  int fwd_spb_env = env_int("SNN_FWD_SPB", 2);
  int fwd_fuse = env_int("SNN_FWD_FUSE", 2) - 1;  // 1: one launch per hidden layer
  int copy_chunks = env_int("SNN_COPY_CHUNKS", 4);  // host batch: copy / DMA pipeline depth
  // samples per forward CTA: N = spb * TT <= 256 and TMEM (doubled for NT > 1) <= 512
  int fwd_spb(int tt) const { return std::max(1, std::min(fwd_spb_env, std::min(kFwdSpbMax, 256 / tt))); }
  int bwd_stages = env_int("SNN_BWD_STAGES", 1);
  int exp_mode = env_int("SNN_EXP_MODE", 1) - 1;  // default 0 = fp64-rounded exp/log
  int wg_stages_cap = env_int("SNN_WG_STAGES", kWgStagesMax);
  int pdl = env_int("SNN_PDL", 2) - 1;  // programmatic dependent launch: same device step, +3 % e2e (r02)
  static int env_int(const char* k, int d) {
    const char* v = std::getenv(k);
    return (v && *v) ? std::max(1, std::atoi(v)) : d;
  }
  static double env_double(const char* k, double d) {
    const char* v = std::getenv(k);
    return (v && *v && std::atof(v) > 0.0) ? std::atof(v) : d;
  }

  ~snn_engine() {
    if (device >= 0) cudaSetDevice(device);
    for (auto& g : graphs) cudaGraphExecDestroy(g.second);
    if (comm_handle && nccl().ok) nccl().CommDestroy(comm_handle);
    for (void* p : peer_ipc)
      if (p) cudaIpcCloseMemHandle(p);
    if (h_loss) cudaFreeHost(h_loss);
    if (h_acc) cudaFreeHost(h_acc);
    if (h_rows) cudaFreeHost(h_rows);
    if (pinned) cudaFreeHost(pinned);
    if (plab_host) cudaFreeHost(plab_host);
    if (pres_loss) cudaFreeHost(pres_loss);
    if (pres_acc) cudaFreeHost(pres_acc);
    if (ring_loss_h) cudaFreeHost(ring_loss_h);
    if (ring_acc_h) cudaFreeHost(ring_acc_h);
    for (int s = 0; s < 2; ++s) {
      if (ev_ready[s]) cudaEventDestroy(ev_ready[s]);
      if (ev_used[s]) cudaEventDestroy(ev_used[s]);
    }
    if (cstream) cudaStreamDestroy(cstream);
    for (auto& g : prof_graphs) cudaGraphExecDestroy(g.second);
    for (auto& ev : prof_ev) cudaEventDestroy(ev);
    if (stream) cudaStreamDestroy(stream);
  }

  void clear_graphs() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.second);
    graphs.clear();
    for (auto& g : prof_graphs) cudaGraphExecDestroy(g.second);
    prof_graphs.clear();
  }

  int B_global() const { return B * world; }
  // debug clock stamps: one region per kernel of the step, kClkStride per CTA
  // clock-stamp rows per kernel slot: every CTA of the widest launch (backward grids are
  // B x H_pad/128); tests/wg_probe.py etc. read it through snn_debug_fetch(5)
  size_t clk_region() const {
    int tiles = 4;
    for (int l = 0; l < L; ++l) tiles = std::max(tiles, H_pad[l] / 128);
    return size_t(std::max(4096, B * tiles)) * kClkStride;
  }

  // ---------------------------------------------------------------- setup
  void validate_and_size() {
    const snn_network_desc& n = net;
    if (n.input <= 0) fail(SNN_ERR_SPEC, "network: input shape not declared");
    if (n.n_hidden < 1 || n.n_hidden > SNN_MAX_HIDDEN)
      fail(SNN_ERR_UNSUPPORTED, "n_hidden=%d outside [1,%d]", n.n_hidden, SNN_MAX_HIDDEN);
    if (n.readout_lif != 0 && n.readout_lif != 1) fail(SNN_ERR_ARGUMENT, "readout_lif must be 0 or 1");
    if (n.classes < 1 || n.classes > kMaxClasses)
      fail(SNN_ERR_UNSUPPORTED, "classes=%d outside [1,%d]", n.classes, kMaxClasses);
    for (int l = 0; l < n.n_hidden; ++l)
      if (n.hidden[l] < 1) fail(SNN_ERR_SPEC, "layer %d: zero width", 2 * l);
    if (!(n.threshold > 0.0f)) fail(SNN_ERR_UNSUPPORTED, "LIF threshold must be > 0");
    if (n.activation < 0 || n.activation > 5) fail(SNN_ERR_ARGUMENT, "unknown activation");
    if (n.activation != SNN_ACT_CUSTOM && !(n.slope > 0.0f))
      fail(SNN_ERR_ARGUMENT, "activation slope must be positive");
    for (int l = 0; l <= n.n_hidden; ++l)
      if (n.beta_mode[l] < 0 || n.beta_mode[l] > 2) fail(SNN_ERR_ARGUMENT, "unknown beta mode");
    for (int l = 0; l < SNN_MAX_HIDDEN; ++l)
      if (n.cell[l] != SNN_CELL_LIF &&
          ((n.cell[l] != SNN_CELL_ALIF && n.cell[l] != SNN_CELL_RLIF) || l >= n.n_hidden))
        fail(SNN_ERR_SPEC, "hidden layer %d: unknown cell kind %d", l, n.cell[l]);
    if (n.activation == SNN_ACT_BOXCAR && !(n.aux > 0.0f))
      fail(SNN_ERR_ARGUMENT, "boxcar: width and height must be positive");
    if (cfg.batch_size < 1) fail(SNN_ERR_ARGUMENT, "train: batch size 0");
    if (cfg.batch_size > 65535)  // one grid dimension carries the samples
      fail(SNN_ERR_UNSUPPORTED, "batch size per rank above 65535 (split it over ranks or steps)");
    if (cfg.time_steps < 1) fail(SNN_ERR_ARGUMENT, "apply: zero timesteps");
    if (cfg.unroll < 1) fail(SNN_ERR_ARGUMENT, "apply: unroll must be >= 1");
    if (cfg.optimizer != 0 && cfg.optimizer != 1) fail(SNN_ERR_ARGUMENT, "train_step: unknown optimizer");
    if (cfg.loss != 0 && cfg.loss != 1) fail(SNN_ERR_ARGUMENT, "train_step: unknown loss kind");
    if (cfg.loss == 1 && !(cfg.rate_hi >= 0.0f && cfg.rate_hi <= 1.0f && cfg.rate_lo >= 0.0f &&
                           cfg.rate_lo <= 1.0f))
      fail(SNN_ERR_ARGUMENT, "spike_rate_mse: rates must lie in [0,1]");
    for (int l = 0; l < SNN_MAX_HIDDEN; ++l)
      if (n.monitor[l] != 0 && (n.monitor[l] != 1 || l >= n.n_hidden))
        fail(SNN_ERR_SPEC, "monitor must follow a lif layer");
    {
      bool mon = false;
      for (int l = 0; l < n.n_hidden; ++l) mon = mon || n.monitor[l] != 0;
      if (mon && (cfg.lambda_low != 0.0f || cfg.lambda_high != 0.0f) &&
          !(cfg.f_min <= cfg.f_max && cfg.f_min >= 0.0f && cfg.f_max <= 1.0f))
        fail(SNN_ERR_ARGUMENT, "activity_regularizer: need 0 <= f_min <= f_max <= 1");
    }
    // train()'s axis check (optimize.hpp:241-245); max_shift <= 0 never shifts (:276)
    if (cfg.n_shift_axes < 0 || cfg.n_shift_axes > 4) fail(SNN_ERR_ARGUMENT, "train: 0..4 shift axes");
    for (int i = 0; i < cfg.n_shift_axes; ++i) {
      const int ax = cfg.shift_axes[i];
      if (ax == 0 || ax == 1)
        fail(SNN_ERR_ARGUMENT, "train: shift axes must name feature axes (>= 2); axis %d is the "
             "batch/packed-time axis", ax);
      if (cfg.max_shift > 0 && ax != 2 && ax != -1)
        fail(SNN_ERR_UNSUPPORTED, "shift axis %d: only the (flat) feature axis 2 / -1 is supported", ax);
    }
    if (cfg.gemm_planes < 0 || cfg.gemm_planes > 3)
      fail(SNN_ERR_ARGUMENT, "gemm_planes %d: 1, 2 or 3 (0 = default 3)", cfg.gemm_planes);
    planes = cfg.gemm_planes == 0 ? 3 : cfg.gemm_planes;
    B = cfg.batch_size;
    T = cfg.time_steps;
    TT = T <= 64 ? 64 : 128;
    NT = (T + TT - 1) / TT;
    T_pad = NT * TT;
    IN = n.input;
    IN_pad = rup(IN, 64);
    L = n.n_hidden;
    C = n.classes;
    for (int l = 0; l < L; ++l) {
      H[l] = n.hidden[l];
      H_pad[l] = rup(H[l], 128);
    }
    for (int j = 0; j <= L; ++j) {
      K[j] = j == 0 ? IN : H[j - 1];
      K_pad[j] = j == 0 ? IN_pad : H_pad[j - 1];
      N[j] = j < L ? H[j] : C;
      N_pad[j] = j < L ? H_pad[j] : 64;
      M_pad_w[j] = rup(K[j], 128);
      n_tile_w[j] = j < L ? 128 : 64;
    }
    // declared RLIF cells: d rec = S_l^T dI_l is one more weight-gradient layer
    NJ = L + 1;
    for (int l = 0; l < L; ++l) {
      rec_j[l] = -1;
      if (!rlif(l)) continue;
      if (NJ >= kMaxLayers) fail(SNN_ERR_UNSUPPORTED, "too many RLIF layers for %d hidden", L);
      if (H_pad[l] > 1024) fail(SNN_ERR_UNSUPPORTED, "RLIF layer %d: width %d > 1024", l, H[l]);
      const int j = NJ++;
      rec_j[l] = j;
      rec_l[j] = l;
      K[j] = N[j] = H[l];
      K_pad[j] = N_pad[j] = H_pad[l];
      M_pad_w[j] = rup(H[l], 128);
      n_tile_w[j] = 128;
    }
    const size_t ro_smem = readout_smem_bytes(H[L - 1], H_pad[L - 1], T, C);
    if (ro_smem > 200 * 1024) fail(SNN_ERR_UNSUPPORTED, "readout working set too large");
    if (size_t(T) * C * 4 > 200 * 1024) fail(SNN_ERR_UNSUPPORTED, "T * classes too large");
    // weight-gradient work split: each CTA owns mg M-tiles (shared dI stages, TMEM
    // mg*n_tile <= 512 columns) of one n-tile and a contiguous range of samples.
    // Pipeline depth per layer = what fits the smem budget (small stages -> more
    // stages in flight).  Splits minimise the modelled finish time of the slowest
    // CTA, fixed + iterations x per-iteration cycles, calibrated on B200 phase
    // clocks (tests/clk_probe.py): fixed = prologue + first stage (~8K) + epilogue
    // (f32 partial bytes at ~22 B/clk); per iteration = 600 + max(MMA issue,
    // 600 per A tile decoded).  Binary search on the finish time tau.
    {
      int sms = 148;
      int dev_sms = 0;
      if (cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess &&
          dev_sms > 0)
        sms = dev_sms;
      sm_count = sms;
      const double budget = double(kWgBarrierOffset);
      const double xrun = double(wg_xrun_bytes(IN_pad));
      // mg cap: 2 stages of (mg A tiles + 3 B planes + dataset run) must fit
      wg_mg_max = std::max(1, std::min(kWgMgMax, int((budget / 2 - 3 * 128 * 128 - xrun) / kPlaneTile)));
      wg_mg_max = std::min(wg_mg_max, env_int("SNN_WG_MG", kWgMgMax));  // M-tiles per CTA cap
      double fixed[kMaxLayers], per_unit[kMaxLayers], units[kMaxLayers];
      const double iters = double(B) * (T_pad / 64);
      for (int j = 0; j < NJ; ++j) {
        const int m_tiles = M_pad_w[j] / 128, n_tiles = N_pad[j] / n_tile_w[j];
        // mg: TMEM columns (mg * n_tile <= 512), the 2-stage smem cap, and the epilogue
        // staging of mg f32 tiles (mg * 128 padded rows) within the budget
        const int mg_epi = int(budget / (128.0 * wg_epi_row_stride(n_tile_w[j])));
        const int mg_cap = std::max(1, std::min(std::min(wg_mg_max, mg_epi),
                                                std::min(m_tiles, 512 / n_tile_w[j])));
        const int groups = (m_tiles + mg_cap - 1) / mg_cap;
        mg_w[j] = (m_tiles + groups - 1) / groups;  // balanced groups (6 tiles -> 3 + 3)
        const double stage = double(wg_stage_bytes(n_tile_w[j], mg_w[j])) + (j == 0 ? xrun : 0.0);
        wg_stages_l[j] = std::max(1, std::min(std::min(kWgStagesMax, wg_stages_cap), int(budget / stage)));
        const int m_groups = (m_tiles + mg_w[j] - 1) / mg_w[j];
        units[j] = double(m_groups) * n_tiles;
        const double mma = 12.0 * mg_w[j] * (n_tile_w[j] / 2.0);  // tcgen05 issue cycles
        const double per_it = 600.0 + std::max(mma, 600.0 * mg_w[j]);
        fixed[j] = 8000.0 + mg_w[j] * n_tile_w[j] * 512.0 / 22.0;
        per_unit[j] = iters * per_it;  // all samples through one CTA
      }
      auto splits_for = [&](double tau, int j) {
        const double room = tau - fixed[j];
        if (room <= 0) return B;
        return std::max(1, std::min(B, int(std::ceil(per_unit[j] / room))));
      };
      double lo = 0, hi = 1e12;
      for (int j = 0; j < NJ; ++j) lo = std::max(lo, fixed[j]);
      for (int rep = 0; rep < 100; ++rep) {
        const double mid = 0.5 * (lo + hi);
        double ctas = 0;
        for (int j = 0; j < NJ; ++j) ctas += units[j] * splits_for(mid, j);
        if (ctas <= sms) hi = mid; else lo = mid;
      }
      for (int j = 0; j < NJ; ++j) splits_w[j] = splits_for(hi, j);
      if (const char* v = std::getenv("SNN_WG_SPLIT_SAMPLES"))
        for (int j = 0; j < NJ; ++j) splits_w[j] = std::max(1, B / std::max(1, std::atoi(v)));
      if (std::getenv("SNN_PRINT_PLAN"))  // diagnostics: the weight-gradient split plan
        for (int j = 0; j < NJ; ++j)
          std::fprintf(stderr, "wgrad layer %d: m_tiles %d mg %d n_tiles %d splits %d stages %d\n", j,
                       M_pad_w[j] / 128, mg_w[j], N_pad[j] / n_tile_w[j], splits_w[j], wg_stages_l[j]);
    }
    // parameter entries (network.hpp:210-226 order)
    entries.clear();
    size_t off = 0;
    for (int j = 0; j <= L; ++j) {
      const int lin = lin_id(j), cell = lin + 1;
      entries.push_back({"l" + std::to_string(lin) + ".w", kEntryW, j, K[j], N[j], off,
                         size_t(K[j]) * N[j]});
      off += size_t(K[j]) * N[j];
      if (n.bias) {
        entries.push_back({"l" + std::to_string(lin) + ".b", kEntryB, j, 1, N[j], off, size_t(N[j])});
        off += N[j];
      }
      // BetaMode (neuron.hpp:56-76): per-neuron [N] or one value (scalar / fixed)
      const int bm = n.beta_mode[j];
      const size_t bsz = bm == 0 ? size_t(N[j]) : 1;
      entries.push_back({"l" + std::to_string(cell) + ".beta", kEntryBeta, j, 1, N[j], off, bsz, bm});
      off += bsz;
      if (alif(j)) {  // declared ALIF cell: adaptation decay after beta (oracle/spiketrain_oracle.h)
        entries.push_back({"l" + std::to_string(cell) + ".gamma", kEntryGamma, j, 1, N[j], off, size_t(N[j])});
        off += N[j];
      }
      if (rlif(j)) {  // declared RLIF cell: recurrent weight [H][H] after beta (a W of layer rec_j)
        entries.push_back({"l" + std::to_string(cell) + ".rec", kEntryW, rec_j[j], N[j], N[j], off,
                           size_t(N[j]) * N[j]});
        off += size_t(N[j]) * N[j];
      }
    }
    n_params = off;
  }

  void allocate() {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    params.alloc(n_params);
    m.alloc(n_params);
    v.alloc(n_params);
    comm.alloc(n_params + 2 + L);  // grads, loss sum, hits, one regularizer value per monitor
    step.alloc(1);
    sched_slot.alloc(1);
    tail_done.alloc(1);
    {
      wg_blocks = 0;
      wg_tiles = 0;
      for (int j = 0; j < NJ; ++j) {
        const int units = (M_pad_w[j] / 128 + mg_w[j] - 1) / mg_w[j] * (N_pad[j] / n_tile_w[j]);
        wg_tiles += units;
        wg_blocks += units * splits_w[j];
      }
      wg_tile_cnt.alloc(size_t(wg_tiles));
      wg_done.alloc(1);
    }
    grow_bc(1 << 20);
    for (int j = 0; j < L; ++j) {
    }
    for (int j = 0; j <= L; ++j) wb[j].alloc(size_t(3) * K_pad[j] * N_pad[j]);
    const size_t rows = size_t(B) * T_pad;
    for (int l = 0; l < L; ++l) {
      V[l].alloc(rows * H_pad[l], false);
      if (alif(l)) {
        Aad[l].alloc(rows * H_pad[l], false);
        dgamma[l].alloc(size_t(B) * H[l]);
      }
      if (rlif(l)) {
        Ibuf[l].alloc(rows * H_pad[l], false);
        dsbuf[l].alloc(rows * H_pad[l], false);
        rec_t[l].alloc(size_t(H[l]) * H_pad[l]);
      }
      s_np[l].alloc(rows * (H_pad[l] / 32));
      s_tp[l].alloc(size_t(H_pad[l]) * (rows / 32));
    }
    for (int j = 0; j <= L; ++j) {
      di[j].alloc(size_t(3) * rows * N_pad[j]);  // zero: padded rows/cols stay zero
      dbeta[j].alloc(size_t(B) * N[j]);
      if (net.bias) dbias[j].alloc(size_t(B) * N[j]);
      partial[j].alloc(size_t(splits_w[j]) * M_pad_w[j] * N_pad[j], false);
    }
    loss_b.alloc(B);
    if (cfg.loss == 1) loss_terms.alloc(size_t(B) * C);
    mon_layers.clear();
    if (reg_on())
      for (int l = 0; l < L; ++l)
        if (net.monitor[l]) mon_layers.push_back(l);
    if (!mon_layers.empty()) hist.alloc(mon_layers.size() * size_t(T + 1));
    correct_b.alloc(B);
    result_loss.alloc(1);
    result_acc.alloc(1);
    if (!ring_loss_h) {
      CK(cudaHostAlloc(reinterpret_cast<void**>(&ring_loss_h), sizeof(float) * kRing, cudaHostAllocMapped));
      CK(cudaHostAlloc(reinterpret_cast<void**>(&ring_acc_h), sizeof(double) * kRing, cudaHostAllocMapped));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ring_loss_d), ring_loss_h, 0));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ring_acc_d), ring_acc_h, 0));
    }
    rows_cur.alloc(B);
    xshift.alloc(1);
    CK(cudaMallocHost(&h_loss, sizeof(float)));
    CK(cudaMallocHost(&h_acc, sizeof(double)));
    CK(cudaMallocHost(&h_rows, sizeof(uint32_t) * B));
    // tensor maps
    for (int j = 0; j < L; ++j) {
      tm_wt[j] = make_map(wb[j].p, uint64_t(3) * K_pad[j], N_pad[j], 64);  // 64x64 MN-major boxes
    }
    for (int j = 1; j <= L; ++j) tm_wb[j] = make_map(wb[j].p, uint64_t(3) * K_pad[j], N_pad[j], 128);
    // dI planes [3][N_pad][B*T_pad]: MN-major boxes for the backward GEMM, K-major
    // boxes (rows = output neurons) for the weight-gradient GEMM
    for (int j = 0; j <= L; ++j) {
      tm_di_k[j] = make_map(di[j].p, uint64_t(3) * N_pad[j], rows, 64);
      tm_di_w[j] = make_map(di[j].p, uint64_t(3) * N_pad[j], rows, uint32_t(n_tile_w[j]));
      if (j < L) tm_di_out[j] = make_map(di[j].p, uint64_t(3) * N_pad[j], rows, 128);
      wg_maps.m[j] = tm_di_w[j];
    }
    for (int j = L + 1; j < NJ; ++j) {
      partial[j].alloc(size_t(splits_w[j]) * M_pad_w[j] * N_pad[j], false);
      wg_maps.m[j] = tm_di_w[rec_l[j]];  // d rec: the RLIF layer's own dI planes
    }
    for (int j = 0; j < NJ; ++j)  // fused tail: TMA tensor stores of the f32 partials
      wg_maps.pm[j] = make_map_f32(partial[j].p, uint64_t(splits_w[j]) * M_pad_w[j], uint64_t(N_pad[j]));
    for (auto fn : {k_lif_fwd<false>, k_lif_fwd<true>, k_lif_fwd<false, true>, k_lif_fwd<true, true>,
                    k_lif_fwd<false, false, true>, k_lif_fwd<true, false, true>})
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              227 * 1024));
    for (auto fn : {k_lif_bwd<0>, k_lif_bwd<1>, k_lif_bwd<2>, k_lif_bwd<3>, k_lif_bwd<4>, k_lif_bwd<5>,
                    k_lif_bwd<0, false, false, false, 2>, k_lif_bwd<1, false, false, false, 2>,
                    k_lif_bwd<2, false, false, false, 2>, k_lif_bwd<3, false, false, false, 2>,
                    k_lif_bwd<4, false, false, false, 2>, k_lif_bwd<5, false, false, false, 2>,
                    k_lif_bwd<0, true>, k_lif_bwd<1, true>, k_lif_bwd<2, true>, k_lif_bwd<3, true>,
                    k_lif_bwd<4, true>, k_lif_bwd<5, true>})
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              int(bwd_smem_bytes(TT, 2))));
    {
      for (auto fn : {k_rlif_fwd_cl<1>, k_rlif_fwd_cl<2>})
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kRlSmemMax));
      for (auto fn : {k_rlif_bwd_cl<0>, k_rlif_bwd_cl<1>, k_rlif_bwd_cl<2>, k_rlif_bwd_cl<3>, k_rlif_bwd_cl<4>,
                      k_rlif_bwd_cl<5>})
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kRlSmemMax));
      for (auto fn : {k_rlif_bwd_tc<0>, k_rlif_bwd_tc<1>, k_rlif_bwd_tc<2>, k_rlif_bwd_tc<3>, k_rlif_bwd_tc<4>,
                      k_rlif_bwd_tc<5>})
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rlif_bwd_tc_smem())));
      for (int l = 0; l < L; ++l)
        if (rlif(l) && rlif_cluster(l)) {
          rl_sb_fwd[l] = rlif_pick_sb(l, true);
          rl_sb_bwd[l] = rlif_pick_sb(l, false);
        }
    }
    for (auto fn : {k_lif_bwd<0, false, false, true>, k_lif_bwd<0, true, false, true>})
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              int(bwd_smem_bytes(TT, 2))));
    for (auto fn : {k_lif_bwd<0, false, true>, k_lif_bwd<1, false, true>, k_lif_bwd<2, false, true>,
                    k_lif_bwd<3, false, true>, k_lif_bwd<4, false, true>, k_lif_bwd<5, false, true>,
                    k_lif_bwd<0, true, true>, k_lif_bwd<1, true, true>, k_lif_bwd<2, true, true>,
                    k_lif_bwd<3, true, true>, k_lif_bwd<4, true, true>, k_lif_bwd<5, true, true>})
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              int(bwd_smem_bytes(TT, 2, true))));
    CK(cudaFuncSetAttribute(k_wgrad<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(kWgSmemLaunch)));
    CK(cudaFuncSetAttribute(k_wgrad<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(kWgSmemLaunch)));
    for (auto fn : {k_readout<1>, k_readout<2>, k_readout<3>, k_readout<4>})
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(200 * 1024)));
    {
      std::vector<int32_t> vi;
      for (const auto& en : entries)
        if (en.kind != kEntryW)
          for (size_t q = 0; q < en.size; ++q) vi.push_back(int32_t(en.offset + q));
      vec_index.alloc(vi.size(), false);
      CK(cudaMemcpy(vec_index.p, vi.data(), vi.size() * 4, cudaMemcpyHostToDevice));
      n_vec = int(vi.size());
    }
  }

  void grow_bc(size_t steps) {
    if (steps <= bc_steps) return;
    if (stream) CK(cudaStreamSynchronize(stream));  // graphs in flight hold the old table
    std::vector<float> h(2 * steps);
    const float b1 = cfg.beta1, b2 = cfg.beta2;
    for (size_t s = 0; s < steps; ++s) {
      // optimize.hpp:96-97: bc = T(1) - std::pow(beta, T(step)) in float
      h[2 * s] = 1.0f - std::pow(b1, float(s + 1));
      h[2 * s + 1] = 1.0f - std::pow(b2, float(s + 1));
    }
    DevBuf<float> nb;
    nb.alloc(2 * steps, false);
    CK(cudaMemcpy(nb.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
    std::swap(bc.p, nb.p);
    std::swap(bc.n, nb.n);
    bc_steps = steps;
    clear_graphs();
  }

  // bias-correction table must cover the next `more` update steps
  void ensure_bc_capacity(size_t more = 1) {
    const size_t need = size_t(host_step) + more + 1;
    if (need > bc_steps) grow_bc(std::max(bc_steps * 2, need));
  }

  // ---------------------------------------------------------- parameters
  // normalised layer id of Linear j (network.hpp:125-157): its cell follows, and
  // a monitor after LIF i < j takes one more id
  int lin_id(int j) const {
    int id = 2 * j;
    for (int i = 0; i < j && i < L; ++i) id += net.monitor[i] ? 1 : 0;
    return id;
  }
  bool alif(int l) const { return l < L && net.cell[l] == SNN_CELL_ALIF; }
  bool rlif(int l) const { return l < L && net.cell[l] == SNN_CELL_RLIF; }
  bool reg_on() const {
    if (cfg.lambda_low == 0.0f && cfg.lambda_high == 0.0f) return false;
    for (int l = 0; l < L; ++l)
      if (net.monitor[l]) return true;
    return false;
  }

  void init_params_host(uint64_t key) {
    // network.hpp:231-286: layer i key rng.child(i); W ~ TN(child(0)); beta ~ TN(child(2))
    std::vector<float> h(n_params, 0.0f);
    for (const auto& e : entries) {
      if (e.kind == kEntryW && e.layer > L) {  // declared RLIF rec ~ TN(0, 1/sqrt(H)) from child 4
        const uint64_t lk = hostrng::child(key, uint64_t(lin_id(rec_l[e.layer]) + 1));
        const float sd = 1.0f / std::sqrt(float(e.rows));
        hostrng::truncated_normal(hostrng::child(lk, 4), e.size, 0.0f, sd, h.data() + e.offset);
      } else if (e.kind == kEntryW) {
        const uint64_t lk = hostrng::child(key, uint64_t(lin_id(e.layer)));
        const float sd = 1.0f / std::sqrt(float(e.rows));
        hostrng::truncated_normal(hostrng::child(lk, 0), e.size, 0.0f, sd, h.data() + e.offset);
      } else if (e.kind == kEntryBeta) {
        const uint64_t lk = hostrng::child(key, uint64_t(lin_id(e.layer) + 1));
        if (e.beta_mode == 2)
          h[e.offset] = net.fixed_beta[e.layer];  // Tensor::scalar(fixed_beta)
        else  // per-neuron [H] or LearnableScalar [] from the same key
          hostrng::truncated_normal(hostrng::child(lk, 2), e.size, 0.5f, 0.25f, h.data() + e.offset);
      } else if (e.kind == kEntryGamma) {  // declared ALIF: gamma ~ TN(0.5, 0.25) from child 3
        const uint64_t lk = hostrng::child(key, uint64_t(lin_id(e.layer) + 1));
        hostrng::truncated_normal(hostrng::child(lk, 3), e.size, 0.5f, 0.25f, h.data() + e.offset);
      }
    }
    upload_params(h.data());
  }

  void upload_params(const float* h) {
    CK(cudaMemcpyAsync(params.p, h, n_params * sizeof(float), cudaMemcpyHostToDevice, stream));
    refresh_planes();
  }

  void fill_entries(Entry* out, int* n_out) const {
    int i = 0;
    for (const auto& e : entries) {
      out[i].kind = e.kind;
      out[i].layer = e.layer;
      out[i].rows = e.rows;
      out[i].cols = e.cols;
      out[i].beta_mode = e.beta_mode;
      out[i].offset = int64_t(e.offset);
      ++i;
    }
    *n_out = i;
  }

  AdamArgs adam_args(int update) {
    AdamArgs a{};
    fill_entries(a.entries, &a.n_entries);
    a.n_params = int64_t(n_params);
    for (int j = 0; j <= L; ++j) {
      a.planes[j].wb = wb[j].p;
      a.planes[j].K_pad = K_pad[j];
      a.planes[j].N_pad = N_pad[j];
    }
    for (int j = L + 1; j < NJ; ++j) {  // RLIF rec: f32 transpose for k_rlif_bwd
      a.planes[j].wt = rec_t[rec_l[j]].p;
      a.planes[j].wt_ld = H_pad[rec_l[j]];
    }
    a.params = params.p;
    a.m = m.p;
    a.v = v.p;
    a.grads = comm.p;
    a.bc = bc.p;
    a.step = step.p;
    a.lr = cfg.lr;
    a.b1 = cfg.beta1;
    a.b2 = cfg.beta2;
    a.eps = cfg.eps;
    a.omb1 = 1.0f - cfg.beta1;
    a.omb2 = 1.0f - cfg.beta2;
    a.update = update;
    a.B_global = B_global();
    // StepResult.loss = numerator / (B) for CE, / T(b * c) for rate-MSE (objective.hpp:158)
    a.loss_denom = cfg.loss == 1 ? float(int64_t(B_global()) * C) : float(B_global());
    a.opt_kind = cfg.optimizer;
    a.momentum = cfg.momentum;
    a.n_mon = int(mon_layers.size());
    a.loss_out = result_loss.p;
    a.acc_out = result_acc.p;
    a.ring_loss = ring_loss_d;
    a.ring_acc = ring_acc_d;
    a.ring_mask = kRing - 1;
    return a;
  }

  void refresh_planes() {
    AdamArgs a = adam_args(0);
    const int threads = 256;
    k_adam<<<unsigned((n_params + threads - 1) / threads), threads, 0, stream>>>(a);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(stream));
  }

  // ---------------------------------------------------------------- data
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  bool sync_after_stage = true;

  void stage(Dataset& ds, const uint8_t* packed, size_t n, const int64_t* labels) {
    const int tp8 = (T + 7) / 8;
    const int tp8_pad = T_pad / 8;
    for (size_t i = 0; i < n; ++i)
      if (labels[i] < 0 || labels[i] >= C)
        fail(SNN_ERR_ARGUMENT, "target %lld outside [0,%d)", (long long)labels[i], C);
    const size_t bytes = n * size_t(tp8_pad) * IN_pad;
    // pinned staging area: the H2D copy of every step's input runs at full PCIe rate
    if (pinned_bytes < bytes + n * sizeof(int32_t)) {
      if (pinned) cudaFreeHost(pinned);
      pinned = nullptr;
      pinned_bytes = 0;
      CK(cudaMallocHost(&pinned, bytes + n * sizeof(int32_t)));
      pinned_bytes = bytes + n * sizeof(int32_t);
    }
    uint8_t* h = static_cast<uint8_t*>(pinned);
    std::memset(h, 0, bytes);
    for (size_t i = 0; i < n; ++i)
      for (int g = 0; g < tp8; ++g)
        std::memcpy(h + (i * tp8_pad + g) * IN_pad, packed + (i * tp8 + g) * size_t(IN), IN);
    int32_t* lab = reinterpret_cast<int32_t*>(h + bytes);
    for (size_t i = 0; i < n; ++i) lab[i] = int32_t(labels[i]);
    if (ds.n != n) {
      ds.x.alloc(bytes, false);
      ds.labels.alloc(n, false);
      ds.n = n;
      clear_graphs();
    }
    CK(cudaMemcpyAsync(ds.x.p, h, bytes, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(ds.labels.p, lab, n * sizeof(int32_t), cudaMemcpyHostToDevice, stream));
    if (sync_after_stage) CK(cudaStreamSynchronize(stream));
  }

  // A host batch in the reference layout [n][ceil(T/8)][IN] (train_step_packed):
  // copied verbatim into pinned memory by the copy pool in chunks whose DMA
  // overlaps the next chunk's copy, then re-laid into [n][T_pad/8][IN_pad] on the
  // device (k_relayout) -- no host memset or per-row copies.
  std::unique_ptr<CopyPool> copy_pool;
  DevBuf<uint8_t> raw_in;
  void stage_batch(Dataset& ds, const uint8_t* packed, size_t n, const int64_t* labels) {
    const int tp8 = (T + 7) / 8, tp8_pad = T_pad / 8;
    for (size_t i = 0; i < n; ++i)
      if (labels[i] < 0 || labels[i] >= C)
        fail(SNN_ERR_ARGUMENT, "target %lld outside [0,%d)", (long long)labels[i], C);
    const size_t raw = n * size_t(tp8) * IN, lab_off = (raw + 15) & ~size_t(15);
    if (pinned_bytes < lab_off + n * sizeof(int32_t)) {
      if (pinned) cudaFreeHost(pinned);
      pinned = nullptr;
      pinned_bytes = 0;
      CK(cudaMallocHost(&pinned, lab_off + n * sizeof(int32_t)));
      pinned_bytes = lab_off + n * sizeof(int32_t);
    }
    const bool in_place = raw_layout_ok();
    if (!in_place && raw_in.n < raw) raw_in.alloc(raw, false);
    if (ds.n != n) {
      ds.x.alloc(n * size_t(tp8_pad) * IN_pad, false);
      ds.labels.alloc(n, false);
      ds.n = n;
      clear_graphs();
    }
    ds.row = in_place ? IN : IN_pad;
    uint8_t* dst = in_place ? ds.x.p : raw_in.p;
    uint8_t* h = static_cast<uint8_t*>(pinned);
    // a caller batch that already lives in pinned (page-locked) memory is DMA'd as is
    cudaPointerAttributes pa{};
    const bool caller_pinned = cudaPointerGetAttributes(&pa, packed) == cudaSuccess &&
                               pa.type == cudaMemoryTypeHost;
    if (!caller_pinned) cudaGetLastError();  // clear a pageable-pointer query error
    if (caller_pinned) {
      CK(cudaMemcpyAsync(dst, packed, raw, cudaMemcpyHostToDevice, stream));
    } else {
      if (!copy_pool) {  // created on the first pageable batch
        const unsigned hc = std::thread::hardware_concurrency();
        const int dflt = int(std::min(7u, hc > 2 ? hc / 2 - 1 : 0u));
        const char* ev = std::getenv("SNN_COPY_THREADS");  // extra copy threads
        copy_pool.reset(new CopyPool(ev && *ev ? std::max(0, std::atoi(ev)) : dflt));
      }
      const size_t chunks = raw >= (size_t(1) << 20) ? size_t(copy_chunks) : 1;
      const size_t per = ((raw + chunks - 1) / chunks + 15) & ~size_t(15);
      for (size_t off = 0; off < raw; off += per) {
        const size_t len = std::min(per, raw - off);
        copy_pool->copy(h + off, packed + off, len);
        CK(cudaMemcpyAsync(dst + off, h + off, len, cudaMemcpyHostToDevice, stream));
      }
    }
    int32_t* lab = reinterpret_cast<int32_t*>(h + lab_off);
    for (size_t i = 0; i < n; ++i) lab[i] = int32_t(labels[i]);
    CK(cudaMemcpyAsync(ds.labels.p, lab, n * sizeof(int32_t), cudaMemcpyHostToDevice, stream));
    if (!in_place) {
      const size_t out = n * size_t(tp8_pad) * IN_pad;
      k_relayout<<<unsigned((out / 4 + 255) / 256), 256, 0, stream>>>(raw_in.p, ds.x.p, int64_t(n), tp8,
                                                                     tp8_pad, IN, IN_pad);
      CK(cudaGetLastError());
    }
  }

  // A host batch in the reference layout [n][ceil(T/8)][IN] is used in place (no
  // k_relayout) when it already has the device's time extent and its rows suit the
  // kernels' bulk copies / 4-byte decoder loads; features >= IN of the last 64-k
  // block are masked in the decoders.
  bool raw_layout_ok() const { return (T + 7) / 8 == T_pad / 8 && IN % 4 == 0; }
  int row_of(const Dataset& ds) const { return ds.row > 0 ? ds.row : IN_pad; }

  // Pipelined host batches (snn_train_steps_packed): two device slots; a copy stream
  // DMAs batch k+1 (pinned caller memory) and re-lays it out while the step graph of
  // batch k runs; per-step loss / accuracy are read back into pinned memory.
  cudaStream_t cstream = nullptr;
  Dataset pslot[2];
  DevBuf<uint8_t> praw[2];
  cudaEvent_t ev_ready[2] = {}, ev_used[2] = {};
  int32_t* plab_host = nullptr;     // pinned [steps][B] labels of the call
  size_t plab_cap = 0;
  float* pres_loss = nullptr;       // pinned per-step results
  double* pres_acc = nullptr;
  size_t pres_cap = 0;
  void pipe_init(size_t steps) {
    const int tp8 = (T + 7) / 8, tp8_pad = T_pad / 8;
    if (!cstream) {
      CK(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
      for (int s = 0; s < 2; ++s) {
        CK(cudaEventCreateWithFlags(&ev_ready[s], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_used[s], cudaEventDisableTiming));
        if (!raw_layout_ok()) praw[s].alloc(size_t(B) * tp8 * IN, false);
        pslot[s].x.alloc(size_t(B) * tp8_pad * IN_pad, false);
        pslot[s].row = raw_layout_ok() ? IN : IN_pad;
        pslot[s].labels.alloc(size_t(B), false);
        pslot[s].n = size_t(B);
        CK(cudaEventRecord(ev_used[s], stream));
      }
    }
    if (steps > plab_cap) {
      if (plab_host) cudaFreeHost(plab_host);
      plab_host = nullptr;
      CK(cudaMallocHost(&plab_host, sizeof(int32_t) * B * steps));
      plab_cap = steps;
    }
    if (steps > pres_cap) {
      if (pres_loss) cudaFreeHost(pres_loss);
      if (pres_acc) cudaFreeHost(pres_acc);
      pres_loss = nullptr;
      pres_acc = nullptr;
      // mapped: the step's k_result_out writes straight into it
      CK(cudaHostAlloc(reinterpret_cast<void**>(&pres_loss), sizeof(float) * steps, cudaHostAllocMapped));
      CK(cudaHostAlloc(reinterpret_cast<void**>(&pres_acc), sizeof(double) * steps, cudaHostAllocMapped));
      pres_cap = steps;
    }
  }
  // batch k into slot k & 1 on the copy stream (after the graph that last read the slot)
  void pipe_stage(size_t k, const uint8_t* packed, const int64_t* labels) {
    const int tp8 = (T + 7) / 8, tp8_pad = T_pad / 8;
    const int sl = int(k & 1);
    const size_t raw = size_t(B) * tp8 * IN;
    CK(cudaStreamWaitEvent(cstream, ev_used[sl], 0));
    // the batch in 4 DMA pieces (measured ~5 % faster end to end than one copy)
    static const int pipe_exp = env_int("SNN_PIPE_EXP", 1) - 1;  // timing experiment: 1 = no batch H2D
    const bool in_place = raw_layout_ok();  // the DMA lands in the slot itself
    uint8_t* dst = in_place ? pslot[sl].x.p : praw[sl].p;
    if (pipe_exp != 1) {
      const size_t per = ((raw + 3) / 4 + 15) & ~size_t(15);
      for (size_t off = 0; off < raw; off += per)
        CK(cudaMemcpyAsync(dst + off, packed + k * raw + off, std::min(per, raw - off),
                           cudaMemcpyHostToDevice, cstream));
    }
    // labels from the call's pinned copy (filled and checked up front): no host wait
    CK(cudaMemcpyAsync(pslot[sl].labels.p, plab_host + k * size_t(B), sizeof(int32_t) * B,
                       cudaMemcpyHostToDevice, cstream));
    // otherwise re-laid out on the copy stream too: it overlaps the previous step's graph
    if (!in_place) {
      const size_t out = size_t(B) * tp8_pad * IN_pad;
      k_relayout<<<unsigned((out / 4 + 255) / 256), 256, 0, cstream>>>(praw[sl].p, pslot[sl].x.p, int64_t(B),
                                                                       tp8, tp8_pad, IN, IN_pad);
      CK(cudaGetLastError());
    }
    CK(cudaEventRecord(ev_ready[sl], cstream));
  }

  // Roll of the next batches along the features (read by the layer-0 forward and
  // the input wgrad from device memory, so captured graphs stay valid).
  void set_shift(int32_t s) {
    if (s == xshift_host) return;
    CK(cudaMemcpyAsync(xshift.p, &s, sizeof(s), cudaMemcpyHostToDevice, stream));  // pageable: staged before return
    xshift_host = s;
  }

  void synth(size_t n, uint64_t seed) {
    if (n == 0) fail(SNN_ERR_ARGUMENT, "synth: classes, examples, and steps must be >= 1");
    Dataset& ds = data;
    const size_t bytes = n * size_t(T_pad / 8) * IN_pad;
    if (ds.n != n) {
      ds.x.alloc(bytes, false);
      ds.labels.alloc(n, false);
      ds.n = n;
      clear_graphs();
    }
    SynthArgs a{};
    a.x = ds.x.p;
    a.labels = ds.labels.p;
    a.master = hostrng::from_seed(seed);
    a.n = int64_t(n);
    a.T = T; a.T_pad = T_pad; a.f = IN; a.f_pad = IN_pad; a.classes = C;
    const int64_t total = int64_t(bytes);
    k_synth<<<unsigned((total + 255) / 256), 256, 0, stream>>>(a);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(stream));
  }

  // Every step kernel is launched with programmatic stream serialization (PDL):
  // its prologue overlaps the previous kernel; griddepcontrol.wait orders data.
  template <typename... KArgs, typename... Args>
  void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  }

  // kernel launch on a cluster of cx CTAs along x (the RLIF cluster scans)
  template <typename... KArgs, typename... Args>
  void launch_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, int cx, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = unsigned(cx);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  }
  // samples per cluster of the RLIF cluster scans: the smallest that keeps every
  // cluster of the grid co-resident (one wave; cudaOccupancyMaxActiveClusters)
  static constexpr int kRlSmemMax = 220 * 1024;
  int rl_sb_fwd[SNN_MAX_HIDDEN]{}, rl_sb_bwd[SNN_MAX_HIDDEN]{};
  int rlif_pick_sb(int l, bool fwd) {
    const int NS = H_pad[l] / kRlCl;
    int best = 0;
    for (int sb = kRlSPT; sb <= kRlSBMax; sb += kRlSPT) {
      const size_t smem = fwd ? rlif_fwd_cl_smem(H[l], H_pad[l], sb) : rlif_bwd_cl_smem(H[l], H_pad[l], sb);
      const int threads = fwd ? 32 * sb / kRlFPT : NS * sb / kRlSPT;
      if (smem > size_t(kRlSmemMax) || threads > (fwd ? 1024 : 512)) break;
      const int clusters = (B + sb - 1) / sb;
      cudaLaunchConfig_t c{};
      c.gridDim = dim3(kRlCl, unsigned(clusters));
      c.blockDim = dim3(unsigned(threads));
      c.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kRlCl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      c.attrs = at;
      c.numAttrs = 1;
      int active = 0;
      if (fwd) CK(cudaOccupancyMaxActiveClusters(&active, NS == 64 ? k_rlif_fwd_cl<2> : k_rlif_fwd_cl<1>, &c));
      else CK(cudaOccupancyMaxActiveClusters(&active, k_rlif_bwd_cl<0>, &c));
      best = sb;
      if (clusters <= active) break;
    }
    if (best == 0) fail(SNN_ERR_UNSUPPORTED, "RLIF layer %d: no cluster configuration fits", l);
    return best;
  }
  // RLIF scans on a cluster (rec slice in smem) when the slices are whole warps
  // and fit: H_pad 256 or 512 (SNN_RLIF_CL=1 forces the single-CTA kernels)
  // the reverse scan's recurrent product on tcgen05 (SNN_RLIF_TC=1 keeps the FP32 form)
  bool rlif_tc(int l) const { return env_int("SNN_RLIF_TC", 2) == 2 && H_pad[l] == 512; }
  bool rlif_cluster(int l) const {
    return env_int("SNN_RLIF_CL", 2) == 2 && (H_pad[l] == 256 || H_pad[l] == 512);
  }
  // samples per k_rlif_bwd CTA: rec^T is re-read from L2 once per step per CTA, so
  // CTAs share it across kSB samples while the grid still covers the SMs
  int rlif_sb() const { return B >= 4 * 148 ? 4 : B >= 2 * 148 ? 2 : 1; }
  template <int kAct>
  void launch_rlif_bwd_sb(int sb, const RlifBwdArgs& ra, int hp) {
    const size_t smem = size_t(2) * sb * hp * sizeof(float);
    if (sb == 4) launch(k_rlif_bwd<kAct, 4>, dim3((B + 3) / 4), dim3(hp), smem, ra);
    else if (sb == 2) launch(k_rlif_bwd<kAct, 2>, dim3((B + 1) / 2), dim3(hp), smem, ra);
    else launch(k_rlif_bwd<kAct, 1>, dim3(B), dim3(hp), smem, ra);
  }
  void launch_rlif_bwd(int l) {
    RlifBwdArgs ra{};
    ra.ds = dsbuf[l].p;
    ra.v_in = V[l].p;
    ra.beta = params.p + entry_of(kEntryBeta, l).offset;
    ra.beta_stride = net.beta_mode[l] == 0 ? 1 : 0;
    ra.rec_t = rec_t[l].p;
    ra.rec = params.p + entry_of(kEntryW, rec_j[l]).offset;
    ra.di_planes = di[l].p;
    ra.dbeta_part = dbeta[l].p;
    ra.dbias_part = net.bias ? dbias[l].p : nullptr;
    ra.B = B; ra.T = T; ra.T_pad = T_pad; ra.H = H[l]; ra.H_pad = H_pad[l];
    ra.theta = net.threshold; ra.slope = net.slope; ra.aux = net.aux;
    if (rlif_tc(l)) {  // tcgen05 recurrent product (H_pad = 512)
      const dim3 grid(kRlCl, unsigned((B + kRtN - 1) / kRtN));
      switch (net.activation) {
        case 1: launch_cluster(k_rlif_bwd_tc<1>, grid, dim3(kRtThreads), rlif_bwd_tc_smem(), kRlCl, ra); break;
        case 2: launch_cluster(k_rlif_bwd_tc<2>, grid, dim3(kRtThreads), rlif_bwd_tc_smem(), kRlCl, ra); break;
        case 3: launch_cluster(k_rlif_bwd_tc<3>, grid, dim3(kRtThreads), rlif_bwd_tc_smem(), kRlCl, ra); break;
        case 4: launch_cluster(k_rlif_bwd_tc<4>, grid, dim3(kRtThreads), rlif_bwd_tc_smem(), kRlCl, ra); break;
        case 5: launch_cluster(k_rlif_bwd_tc<5>, grid, dim3(kRtThreads), rlif_bwd_tc_smem(), kRlCl, ra); break;
        default: launch_cluster(k_rlif_bwd_tc<0>, grid, dim3(kRtThreads), rlif_bwd_tc_smem(), kRlCl, ra); break;
      }
      return;
    }
    if (rlif_cluster(l)) {
      const int sb = rl_sb_bwd[l];
      ra.sb = sb;
      const dim3 grid(kRlCl, unsigned((B + sb - 1) / sb));
      const dim3 block(unsigned(H_pad[l] / kRlCl * (sb / kRlSPT)));
      const size_t smem = rlif_bwd_cl_smem(H[l], H_pad[l], sb);
      switch (net.activation) {
        case 1: launch_cluster(k_rlif_bwd_cl<1>, grid, block, smem, kRlCl, ra); break;
        case 2: launch_cluster(k_rlif_bwd_cl<2>, grid, block, smem, kRlCl, ra); break;
        case 3: launch_cluster(k_rlif_bwd_cl<3>, grid, block, smem, kRlCl, ra); break;
        case 4: launch_cluster(k_rlif_bwd_cl<4>, grid, block, smem, kRlCl, ra); break;
        case 5: launch_cluster(k_rlif_bwd_cl<5>, grid, block, smem, kRlCl, ra); break;
        default: launch_cluster(k_rlif_bwd_cl<0>, grid, block, smem, kRlCl, ra); break;
      }
      return;
    }
    const int sb = rlif_sb();
    switch (net.activation) {
      case 1: launch_rlif_bwd_sb<1>(sb, ra, H_pad[l]); break;
      case 2: launch_rlif_bwd_sb<2>(sb, ra, H_pad[l]); break;
      case 3: launch_rlif_bwd_sb<3>(sb, ra, H_pad[l]); break;
      case 4: launch_rlif_bwd_sb<4>(sb, ra, H_pad[l]); break;
      case 5: launch_rlif_bwd_sb<5>(sb, ra, H_pad[l]); break;
      default: launch_rlif_bwd_sb<0>(sb, ra, H_pad[l]); break;
    }
  }
  template <bool kAlif>
  void launch_bwd_alif(int act, dim3 grid, size_t smem, const CUtensorMap& tw, const CUtensorMap& td,
                       const CUtensorMap& to, const BwdArgs& bw) {
    const bool reg = bw.hist != nullptr;
    switch (act) {
      case 1: launch(reg ? k_lif_bwd<1, true, kAlif> : k_lif_bwd<1, false, kAlif>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      case 2: launch(reg ? k_lif_bwd<2, true, kAlif> : k_lif_bwd<2, false, kAlif>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      case 3: launch(reg ? k_lif_bwd<3, true, kAlif> : k_lif_bwd<3, false, kAlif>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      case 4: launch(reg ? k_lif_bwd<4, true, kAlif> : k_lif_bwd<4, false, kAlif>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      case 5: launch(reg ? k_lif_bwd<5, true, kAlif> : k_lif_bwd<5, false, kAlif>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      default: launch(reg ? k_lif_bwd<0, true, kAlif> : k_lif_bwd<0, false, kAlif>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
    }
  }
  void launch_bwd(int act, dim3 grid, size_t smem, const CUtensorMap& tw, const CUtensorMap& td,
                  const CUtensorMap& to, const BwdArgs& bw) {
    if (bw.gamma != nullptr) {  // declared ALIF cell
      launch_bwd_alif<true>(act, grid, smem, tw, td, to, bw);
      return;
    }
    if (bw.hist != nullptr) {  // monitored layer with the activity regularizer on
      switch (act) {
        case 1: launch(k_lif_bwd<1, true>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
        case 2: launch(k_lif_bwd<2, true>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
        case 3: launch(k_lif_bwd<3, true>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
        case 4: launch(k_lif_bwd<4, true>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
        case 5: launch(k_lif_bwd<5, true>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
        default: launch(k_lif_bwd<0, true>, grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      }
      return;
    }
    // plain LIF: several t-tiles take the 32-byte sector-store kernel
    const bool one = bw.NT == 1;
#define SNN_BWD_PLAIN(A) (one ? k_lif_bwd<A> : k_lif_bwd<A, false, false, false, 2>)
    switch (act) {
      case 1: launch(SNN_BWD_PLAIN(1), grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      case 2: launch(SNN_BWD_PLAIN(2), grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      case 3: launch(SNN_BWD_PLAIN(3), grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      case 4: launch(SNN_BWD_PLAIN(4), grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      case 5: launch(SNN_BWD_PLAIN(5), grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
      default: launch(SNN_BWD_PLAIN(0), grid, dim3(kBwdThreads), smem, tw, td, to, bw); break;
    }
#undef SNN_BWD_PLAIN
  }

  // ---------------------------------------------------------------- step
  // Forward launch groups (first layer, layer count): consecutive hidden layers run
  // in one launch when each fits one 128-neuron tile and the step one t-tile --
  // the next layer's GEMM then consumes the spikes straight from shared memory.
  std::vector<std::pair<int, int>> fwd_groups() const {
    std::vector<std::pair<int, int>> g;
    for (int l = 0; l < L;) {
      int nl = 1;
      // RLIF layers run their recurrent scan in a separate kernel: never fused
      if (fwd_fuse && NT == 1 && H_pad[l] == 128 && K_pad[l] >= 128 && fwd_stages >= 2 && !rlif(l))
        while (l + nl < L && nl < kFwdFuseMax && H_pad[l + nl] == 128 && K_pad[l + nl] == 128 &&
               !rlif(l + nl))
          ++nl;
      g.emplace_back(l, nl);
      l += nl;
    }
    return g;
  }
  // forward groups + readout + L bwd + wgrad + tail (fused reduce+Adam without a
  // communicator; reduce, adam with one -- the allreduce between them is NCCL's)
  int n_rlif() const {
    int c = 0;
    for (int l = 0; l < L; ++l) c += rlif(l) ? 1 : 0;
    return c;
  }
  // + the RLIF recurrent scans (one forward, one backward per RLIF layer)
  // one rank: the step tail runs inside k_wgrad when its grid fits one wave (the
  // tile waits need every CTA co-resident), else k_reduce_adam
  bool fused_tail() const { return tail_mode == 0 && wg_blocks <= sm_count; }
  int launches_per_step() const {
    return int(fwd_groups().size()) + L + (tail_mode == 0 ? (fused_tail() ? 2 : 3) : tail_mode == 1 ? 4 : 5) +
           2 * n_rlif();
  }

  // exchange buffers + flags of the peer tail (cudaMalloc'd: IPC-exportable)
  void ensure_peer_mem() {
    if (peer_mem.p) return;
    n_comm = (int64_t(n_params) + 2 + L + 63) / 64 * 64;
    // [2] grad regions | [2] result regions | m mirror | v mirror (f32, n_comm each),
    // then the A and B flag arrays (kMaxRanks u64 each); see k_peer_owner
    peer_mem.alloc(size_t(6 * n_comm) * 4 + 2 * kMaxRanks * 8);
    peer_seq.alloc(1);
    peer_done.alloc(3);
    peer_timeout.alloc(1);
  }
  unsigned long long* flags_of(uint8_t* base) const {
    return reinterpret_cast<unsigned long long*>(base + size_t(6 * n_comm) * 4);
  }
  void set_peers(int r, int w, uint8_t* const* bases) {
    for (int q = 0; q < w; ++q) {
      peer_xchg[q] = reinterpret_cast<float*>(bases[q]);
      peer_flags[q] = flags_of(bases[q]);
      peer_flags_b[q] = flags_of(bases[q]) + kMaxRanks;
    }
    rank = r;
    world = w;
    tail_mode = 2;
    clear_graphs();
  }

  std::vector<std::string> launch_names;
  std::vector<cudaEvent_t> prof_ev;
  std::map<std::pair<const void*, int>, cudaGraphExec_t> prof_graphs;

  // Records an event after each kernel when profiling (graph event nodes).
  void mark(std::vector<cudaEvent_t>* evs, const char* name, int layer) {
    CK(cudaGetLastError());
    launch_names.push_back(std::string(name) + (layer >= 0 ? "[" + std::to_string(layer) + "]" : ""));
    if (evs) {
      if (evs->size() < launch_names.size() + 1) fail(SNN_ERR_STATE, "profiling events exhausted");
      CK(cudaEventRecordWithFlags((*evs)[launch_names.size()], stream, cudaEventRecordExternal));
    }
  }

  // One step.  sched_mode: rows = sched[*sched_slot] (advanced by the step tail).
  // Peer tail: cross-rank gradient sum over mapped peer memory + the update.
  void enqueue_peer_tail(int update, std::vector<cudaEvent_t>* evs, bool sched_mode) {
    PeerArgs pa{};
    for (int q = 0; q < world; ++q) {
      pa.xchg[q] = peer_xchg[q];
      pa.peer_flags_b[q] = peer_flags_b[q];
    }
    pa.flags_a = peer_flags[rank];
    pa.flags_b = peer_flags_b[rank];
    pa.n_comm = n_comm;
    pa.seq = peer_seq.p;
    pa.done = peer_done.p + 1;
    pa.timeout = peer_timeout.p;
    pa.grads_out = comm.p;
    pa.rows_slot = sched_mode ? sched_slot.p : nullptr;
    pa.step = step.p;
    pa.rank = rank;
    pa.world = world;
    pa.spin_ns = (long long)(1e9 * env_double("SNN_PEER_TIMEOUT_S", 20.0));
    AdamArgs a = adam_args(update);
    const int64_t slice = peer_slice_lo(int64_t(n_params), rank + 1, world) -
                          peer_slice_lo(int64_t(n_params), rank, world);
    if (split_part != 2) {
      launch(k_peer_owner, dim3(unsigned(std::max<int64_t>(1, (slice + 255) / 256))), dim3(256), 0, pa, a);
      mark(evs, "peer_owner", -1);
    }
    if (split_part != 1) {
      launch(k_peer_gather, dim3(unsigned((n_params + 255) / 256)), dim3(256), 0, pa, a);
      mark(evs, "peer_gather", -1);
    }
  }
  // the owner phase keeps m / v of this rank's slice only (ZeRO-1 style) and mirrors
  // them into the exchange buffer: pull every other owner's slice back in
  void sync_opt_from_owners() {
    if (tail_mode != 2) return;
    for (int q = 0; q < world; ++q) {
      if (q == rank) continue;
      const int64_t lo = peer_slice_lo(int64_t(n_params), q, world);
      const int64_t hi = peer_slice_lo(int64_t(n_params), q + 1, world);
      if (hi <= lo) continue;
      CK(cudaMemcpyAsync(m.p + lo, peer_xchg[q] + peer_m_off(n_comm) + lo, size_t(hi - lo) * 4,
                         cudaMemcpyDeviceToDevice, stream));
      CK(cudaMemcpyAsync(v.p + lo, peer_xchg[q] + peer_v_off(n_comm) + lo, size_t(hi - lo) * 4,
                         cudaMemcpyDeviceToDevice, stream));
    }
  }
  void check_peer_timeout() {
    if (tail_mode != 2 || !peer_timeout.p) return;
    unsigned int t = 0;
    CK(cudaMemcpy(&t, peer_timeout.p, 4, cudaMemcpyDeviceToHost));
    if (t) fail(SNN_ERR_CUDA, "peer tail: a rank did not publish within SNN_PEER_TIMEOUT_S");
  }

  void enqueue_body(const Dataset& ds, int update, std::vector<cudaEvent_t>* evs = nullptr,
                    bool sched_mode = false) {
    launch_names.clear();
    if (tail_mode == 2 && split_part >= 1) {  // test hook: only a tail part of a split step
      if (evs) CK(cudaEventRecordWithFlags((*evs)[0], stream, cudaEventRecordExternal));
      enqueue_peer_tail(update, evs, sched_mode);
      return;
    }
    const uint32_t* rows_p = sched_mode ? sched.p : rows_cur.p;
    const int64_t* slot_p = sched_mode ? sched_slot.p : nullptr;
    if (evs) CK(cudaEventRecordWithFlags((*evs)[0], stream, cudaEventRecordExternal));
    // readout arguments (K4)
    ReadoutArgs ro_args{};
    {
      ReadoutArgs& r = ro_args;
      r.s_in = s_np[L - 1].p;
      r.rows = rows_p;
      r.rows_slot = slot_p;
      r.labels = ds.labels.p;
      r.w = params.p + entry_of(kEntryW, L).offset;
      r.bias = net.bias ? params.p + entry_of(kEntryB, L).offset : nullptr;
      r.beta = params.p + entry_of(kEntryBeta, L).offset;
    r.beta_stride = net.beta_mode[L] == 0 ? 1 : 0;
      r.d3_planes = di[L].p;
      r.loss_b = loss_b.p;
      r.correct_b = correct_b.p;
      r.dbeta_part = dbeta[L].p;
      r.dbias_part = net.bias ? dbias[L].p : nullptr;
      r.dbg_trace = update == kEvalTrace ? eval_trace.p : (debug ? dbg_trace.p : nullptr);
      r.dbg_clk = clocks ? dbg_clk.p : nullptr;
      r.exp_mode = exp_mode;
      r.B = B; r.T = T; r.T_pad = T_pad; r.HL = H[L - 1]; r.HL_pad = H_pad[L - 1]; r.C = C;
      r.inv_b = 1.0f / float(B_global());
      r.loss_kind = cfg.loss;
      r.rate_hi = cfg.rate_hi;
      r.rate_lo = cfg.rate_lo;
      // gs = g * T(2) / (T(b * c) * T(t)) with g = 1 (objective.hpp:172), in float
      r.mse_gs = 1.0f * 2.0f / (float(int64_t(B_global()) * C) * float(T));
      r.readout_lif = net.readout_lif;
      r.act = net.activation;
      r.theta = net.threshold;
      r.slope = net.slope;
      r.aux = net.aux;
      r.loss_terms = cfg.loss == 1 ? loss_terms.p : nullptr;
    }
    // forward: one launch per group of consecutive hidden layers (fwd_groups)
    for (const auto& grp : fwd_groups()) {
      const int l = grp.first, nl = grp.second;
      FwdArgs f{};
      f.planes = planes;
      FwdMaps fm{};
      f.x = ds.x.p;
      f.x_row = row_of(ds);
      f.rows = rows_p;
      f.rows_slot = slot_p;
      f.s_in = l > 0 ? s_np[l - 1].p : nullptr;
      for (int i = 0; i < nl; ++i) {
        FwdLayer& ly = f.lay[i];
        ly.beta = params.p + entry_of(kEntryBeta, l + i).offset;
        ly.beta_stride = net.beta_mode[l + i] == 0 ? 1 : 0;
        ly.bias = net.bias ? params.p + entry_of(kEntryB, l + i).offset : nullptr;
        ly.v_out = V[l + i].p;
        ly.s_np = s_np[l + i].p;
        ly.s_tp = s_tp[l + i].p;
        ly.dbg_i = debug ? dbg_i[l + i].p : nullptr;
        ly.gamma = alif(l + i) ? params.p + entry_of(kEntryGamma, l + i).offset : nullptr;
        ly.a_out = alif(l + i) ? Aad[l + i].p : nullptr;
        ly.i_out = rlif(l + i) ? Ibuf[l + i].p : nullptr;
        ly.K_pad = K_pad[l + i]; ly.H = H[l + i]; ly.H_pad = H_pad[l + i];
        fm.m[i] = tm_wt[l + i];
      }
      f.n_layers = nl;
      f.dbg_clk = clocks ? dbg_clk.p + size_t(1 + l) * clk_region() : nullptr;
      f.B = B; f.T = T; f.T_pad = T_pad; f.TT = TT; f.NT = NT;
      f.in_kind = l == 0 ? 0 : 1;
      f.xshift = l == 0 ? xshift.p : nullptr;
      f.in_features = IN;
      f.theta = net.threshold;
      f.stages = std::min(fwd_stages, NT * (K_pad[l] / 64));
      f.spb = fwd_spb(TT);
      const bool shifting = l == 0 && cfg.max_shift > 0 && cfg.n_shift_axes > 0;
      bool any_alif = false;
      for (int i = 0; i < nl; ++i) any_alif = any_alif || alif(l + i);
      auto kfn = rlif(l) ? (shifting ? k_lif_fwd<true, false, true> : k_lif_fwd<false, false, true>)
                 : any_alif ? (shifting ? k_lif_fwd<true, true> : k_lif_fwd<false, true>)
                            : (shifting ? k_lif_fwd<true> : k_lif_fwd<false>);
      launch(kfn, dim3(H_pad[l] / 128, (B + f.spb - 1) / f.spb),
             dim3(kFwdThreads),
             fwd_smem_bytes(TT, f.spb, f.stages, l == 0 ? K_pad[0] : 0, planes), fm, f);
      mark(evs, "lif_fwd", l);
      if (nl == 1 && rlif(l)) {  // declared RLIF: the recurrent scan over the projection
        RlifFwdArgs ra{};
        ra.i_in = Ibuf[l].p;
        ra.beta = params.p + entry_of(kEntryBeta, l).offset;
        ra.beta_stride = net.beta_mode[l] == 0 ? 1 : 0;
        ra.rec = params.p + entry_of(kEntryW, rec_j[l]).offset;
        ra.v_out = V[l].p;
        ra.s_np = s_np[l].p;
        ra.s_tp = s_tp[l].p;
        ra.B = B; ra.T = T; ra.T_pad = T_pad; ra.H = H[l]; ra.H_pad = H_pad[l];
        ra.theta = net.threshold;
        if (rlif_cluster(l)) {
          const int sb = rl_sb_fwd[l];
          ra.sb = sb;
          launch_cluster(H_pad[l] == 512 ? k_rlif_fwd_cl<2> : k_rlif_fwd_cl<1>,
                         dim3(kRlCl, unsigned((B + sb - 1) / sb)), dim3(unsigned(32 * sb / kRlFPT)),
                         rlif_fwd_cl_smem(H[l], H_pad[l], sb), kRlCl, ra);
        } else
          launch(k_rlif_fwd, dim3(B), dim3(H_pad[l]), 0, ra);
        mark(evs, "rlif_fwd", l);
      }
    }
    // readout + loss + LI backward
    {
      const ReadoutArgs r = ro_args;
      const size_t smem = readout_smem_bytes(H[L - 1], H_pad[L - 1], T, C);
      const int ng = readout_groups(C);
      launch(ng == 1 ? k_readout<1> : ng == 2 ? k_readout<2> : ng == 3 ? k_readout<3> : k_readout<4>,
             dim3(B), dim3(kRoThreads), smem, r);
      mark(evs, "readout", -1);
    }
    if (update >= kEval) return;  // evaluation: forward + readout only (apply, cmd_eval)
    // hidden backward, top-down: dS on tcgen05 (readout-fed layer: K = classes)
    for (int l = L - 1; l >= 0; --l) {
      BwdArgs bw{};
      bw.planes = planes;
      bw.v_in = V[l].p;
      bw.beta = params.p + entry_of(kEntryBeta, l).offset;
      bw.beta_stride = net.beta_mode[l] == 0 ? 1 : 0;
      bw.di_planes = di[l].p;
      bw.dbeta_part = dbeta[l].p;
      bw.dbias_part = net.bias ? dbias[l].p : nullptr;
      bw.dbg_ds = debug ? dbg_ds[l].p : nullptr;
      if (alif(l)) {
        bw.a_in = Aad[l].p;
        bw.gamma = params.p + entry_of(kEntryGamma, l).offset;
        bw.dgamma_part = dgamma[l].p;
      }
      bw.dbg_clk = clocks ? dbg_clk.p + size_t(1 + L + l) * clk_region() : nullptr;
      bw.B = B; bw.T = T; bw.T_pad = T_pad; bw.TT = TT; bw.NT = NT;
      bw.K_pad = N_pad[l + 1]; bw.K = N[l + 1]; bw.H = H[l]; bw.H_pad = H_pad[l]; bw.act = net.activation;
      bw.stages = std::min(bwd_stages, NT * (N_pad[l + 1] / 64));
      bw.theta = net.threshold; bw.slope = net.slope; bw.aux = net.aux;
      for (size_t m = 0; m < mon_layers.size(); ++m)
        if (mon_layers[m] == l) {  // activity_regularizer_taped backward (objective.hpp:208-227)
          bw.s_tp = s_tp[l].p;
          bw.hist = hist.p + m * size_t(T + 1);
          bw.reg_gs = 1.0f * 2.0f / (float(int64_t(B_global()) * H[l]) * float(T));
          bw.f_min = cfg.f_min; bw.f_max = cfg.f_max;
          bw.lambda_low = cfg.lambda_low; bw.lambda_high = cfg.lambda_high;
        }
      if (rlif(l)) {  // declared RLIF: dS on tcgen05, then the recurrent reverse scan
        bw.ds_out = dsbuf[l].p;
        launch(bw.hist != nullptr ? k_lif_bwd<0, true, false, true> : k_lif_bwd<0, false, false, true>,
               dim3(H_pad[l] / 128, B), dim3(kBwdThreads), bwd_smem_bytes(TT, bw.stages), tm_wb[l + 1],
               tm_di_k[l + 1], tm_di_out[l], bw);
        mark(evs, "ds", l);
        launch_rlif_bwd(l);
        mark(evs, "rlif_bwd", l);
        continue;
      }
      launch_bwd(net.activation, dim3(H_pad[l] / 128, B), bwd_smem_bytes(TT, bw.stages, alif(l)),
                 tm_wb[l + 1], tm_di_k[l + 1], tm_di_out[l], bw);
      mark(evs, "lif_bwd", l);
    }
    // gradient assembly (+ loss sum, hits, step counter)
    {
      ReduceArgs r{};
      fill_entries(r.entries, &r.n_entries);
      r.n_params = int64_t(n_params);
      for (int j = L + 1; j < NJ; ++j) {
        r.partial[j] = partial[j].p;
        r.M_pad[j] = M_pad_w[j];
        r.N_pad[j] = N_pad[j];
        r.splits[j] = splits_w[j];
      }
      for (int j = 0; j <= L; ++j) {
        r.partial[j] = partial[j].p;
        r.M_pad[j] = M_pad_w[j];
        r.N_pad[j] = N_pad[j];
        r.splits[j] = splits_w[j];
        r.dbeta_part[j] = dbeta[j].p;
        r.dbias_part[j] = net.bias ? dbias[j].p : nullptr;
        r.dgamma_part[j] = alif(j) ? dgamma[j].p : nullptr;
      }
      r.vec_index = vec_index.p;
      r.n_vec = n_vec;
      r.params = params.p;
      r.grads = comm.p;
      r.loss_b = loss_b.p;
      r.correct_b = correct_b.p;
      r.step = step.p;
      r.update = update;
      r.B = B;
      r.loss_terms = cfg.loss == 1 ? loss_terms.p : nullptr;
      r.n_loss_terms = cfg.loss == 1 ? B * C : B;
      r.w_blocks = int((n_params + kRedElemsPerBlock - 1) / kRedElemsPerBlock);
      r.hist = hist.p;
      r.n_mon = int(mon_layers.size());
      r.hist_stride = T + 1;
      r.reg_T = T;
      for (size_t m = 0; m < mon_layers.size(); ++m)
        r.mon_n[m] = float(int64_t(B_global()) * H[mon_layers[m]]);
      r.f_min = cfg.f_min; r.f_max = cfg.f_max;
      r.lambda_low = cfg.lambda_low; r.lambda_high = cfg.lambda_high;
      const int blocks = r.w_blocks + (n_vec + 7) / 8 + 1;
      const bool fused = update && fused_tail();
      if (tail_mode == 2) {
        r.xchg = reinterpret_cast<float*>(peer_mem.p);
        r.n_comm = n_comm;
        r.seq = peer_seq.p;
        for (int q = 0; q < world; ++q) r.peer_flags[q] = peer_flags[q];
        r.rank = rank;
        r.world = world;
        r.done = peer_done.p;
      }
      // weight gradients: one launch over every Linear layer (split-K partials); with
      // the fused tail it also reduces them, updates and writes the StepResult
      {
        WgradArgs w{};
        w.planes = planes;
        w.x = ds.x.p;
        w.rows = rows_p;
        w.rows_slot = slot_p;
        w.B = B; w.T_pad = T_pad; w.x_row_stride = row_of(ds);
        w.xshift = xshift.p;
        w.in_features = IN;
        w.dbg_clk = clocks ? dbg_clk.p + size_t(1 + 2 * L) * clk_region() : nullptr;
        int blocks = 0;
        w.n_layers = NJ;  // + one d rec layer per RLIF cell (A = its own spikes)
        for (int j = 0; j < NJ; ++j) {
          WgradLayer& g = w.layer[j];
          g.s_tp = j > L ? s_tp[rec_l[j]].p : j > 0 ? s_tp[j - 1].p : nullptr;
          g.partial = partial[j].p;
          g.kind = j == 0 ? 0 : 1;
          g.M_pad = M_pad_w[j]; g.N_pad = N_pad[j]; g.n_tile = n_tile_w[j]; g.splits = splits_w[j];
          g.m_tiles = M_pad_w[j] / 128; g.n_tiles = N_pad[j] / n_tile_w[j];
          g.mg = mg_w[j]; g.m_groups = (g.m_tiles + g.mg - 1) / g.mg;
          g.stages = wg_stages_l[j];
          g.block_start = blocks;
          blocks += g.m_groups * g.n_tiles * g.splits;
        }
        if (fused) {
          WgradTail tl{};
          tl.tile_cnt = wg_tile_cnt.p;
          tl.done = wg_done.p;
          tl.rows_slot = sched_mode ? sched_slot.p : nullptr;
          tl.n_tiles_total = wg_tiles;
          int tb = 0;
          for (int j = 0; j < NJ; ++j) {
            const EntryHost* we = nullptr;
            for (const auto& en : entries)
              if (en.kind == kEntryW && en.layer == j) we = &en;
            tl.w_off[j] = int64_t(we->offset);
            tl.rows[j] = we->rows;
            tl.cols[j] = we->cols;
            tl.tile_base[j] = tb;
            tb += w.layer[j].m_groups * w.layer[j].n_tiles;
          }
          launch(k_wgrad<true>, dim3(blocks), dim3(kWgThreads), kWgSmemLaunch, wg_maps, w, r, adam_args(1), tl);
          mark(evs, "wgrad", -1);
          return;
        }
        launch(k_wgrad<false>, dim3(blocks), dim3(kWgThreads), kWgSmemLaunch, wg_maps, w, r, AdamArgs{},
               WgradTail{});
        mark(evs, "wgrad", -1);
      }
      if (update && tail_mode == 0) {
        // no communicator: no allreduce between reduction and update -> one kernel
        AdamArgs a = adam_args(1);
        long long* tclk = clocks && size_t(blocks) * kClkStride <= clk_region()
                              ? dbg_clk.p + size_t(2 + 2 * L) * clk_region() : nullptr;
        launch(k_reduce_adam, dim3(blocks), dim3(256), 0, r, a, tail_done.p,
               sched_mode ? sched_slot.p : (int64_t*)nullptr, tclk);
        mark(evs, "reduce_adam", -1);
        return;
      }
      if (split_part < 1) {
        launch(k_reduce, dim3(blocks), dim3(256), 0, r);
        mark(evs, "reduce", -1);
      }
    }
    if (tail_mode == 2) {
      if (split_part != 0) enqueue_peer_tail(update, evs, sched_mode);
      return;
    }
    if (comm_handle != nullptr) {
      const int rc = nccl().AllReduce(comm.p, comm.p, n_params + 2 + mon_layers.size(), /*ncclFloat32*/ 7,
                                      /*ncclSum*/ 0, comm_handle, stream);
      if (rc != 0) fail(SNN_ERR_CUDA, "ncclAllReduce failed (%d)", rc);
      mark(evs, "nccl_allreduce", -1);
    }
    if (update) {
      AdamArgs a = adam_args(1);
      a.rows_slot = sched_mode ? sched_slot.p : nullptr;
      launch(k_adam, dim3(unsigned((n_params + 255) / 256)), dim3(256), 0, a);
      mark(evs, "adam", -1);
    } else {
      launch(k_result, dim3(1), dim3(32), 0, (const float*)(comm.p + n_params), B_global(),
             cfg.loss == 1 ? float(int64_t(B_global()) * C) : float(B_global()), step.p,
             0, result_loss.p, result_acc.p, int(mon_layers.size()));
      mark(evs, "result", -1);
    }
  }

  // Per-launch device times of `steps` full steps (graph with event nodes).
  std::vector<double> profile(int steps) {
    const int max_ev = 64;
    if (prof_ev.empty()) {
      prof_ev.resize(max_ev);
      for (auto& ev : prof_ev) CK(cudaEventCreate(&ev));
    }
    const Dataset& ds = data;
    if (ds.n == 0) fail(SNN_ERR_STATE, "no dataset staged");
    auto key = std::make_pair(static_cast<const void*>(ds.x.p), 1);
    cudaGraphExec_t ex = nullptr;
    ensure_bc_capacity(64 + 4 * size_t(steps));
    auto it = prof_graphs.find(key);
    if (it == prof_graphs.end()) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue_body(ds, 1, &prof_ev);
      } catch (...) {
        cudaStreamEndCapture(stream, &g);
        throw;
      }
      CK(cudaStreamEndCapture(stream, &g));
      CK(cudaGraphInstantiate(&ex, g, 0));
      CK(cudaGraphDestroy(g));
      prof_graphs[key] = ex;
    } else {
      ex = it->second;
    }
    const size_t nl = launch_names.size();
    std::vector<double> acc(nl, 0.0);
    // keep the GPU busy (boost clocks) around every profiled step: the event
    // graph runs between plain step graphs, one sync per 4 steps
    cudaGraphExec_t plain = graph_for(ds, 1);
    for (int w = 0; w < 64; ++w) CK(cudaGraphLaunch(plain, stream));
    host_step += 64;
    for (int s = 0; s < steps; ++s) {
      CK(cudaGraphLaunch(ex, stream));
      for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(plain, stream));
      host_step += 4;
      CK(cudaStreamSynchronize(stream));
      for (size_t i = 0; i < nl; ++i) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, prof_ev[i], prof_ev[i + 1]));
        acc[i] += ms;
      }
    }
    for (auto& a : acc) a /= std::max(1, steps);
    return acc;
  }

  const EntryHost& entry_of(int kind, int layer) const {
    for (const auto& e : entries)
      if (e.kind == kind && e.layer == layer) return e;
    fail(SNN_ERR_ARGUMENT, "no entry kind %d layer %d", kind, layer);
  }

  // mode 0: one step on rows_cur; mode g >= 1: g schedule steps back to back
  cudaGraphExec_t graph_for(const Dataset& ds, int update, int mode = 0) {
    auto key = std::make_tuple(static_cast<const void*>(ds.x.p), update, mode);
    auto it = graphs.find(key);
    if (it != graphs.end()) return it->second;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    try {
      if (mode == 0) enqueue_body(ds, update);
      for (int i = 0; i < mode; ++i) enqueue_body(ds, update, nullptr, true);
    } catch (...) {
      cudaStreamEndCapture(stream, &g);
      throw;
    }
    CK(cudaStreamEndCapture(stream, &g));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    CK(cudaGraphDestroy(g));
    // upload now: a first launch would otherwise upload inside the caller's (timed) stream work
    CK(cudaGraphUpload(ex, stream));
    graphs[key] = ex;
    return ex;
  }

  void launch(const Dataset& ds, int update) {
    if (ds.n == 0) fail(SNN_ERR_STATE, "no dataset staged");
    if (update) ensure_bc_capacity();
    CK(cudaGraphLaunch(graph_for(ds, update), stream));
    if (update) ++host_step;
  }

  // `n` schedule steps starting at `slot`: graphs of kSchedGraphSteps steps, then singles
  static constexpr int kSchedGraphSteps = 8;
  void launch_sched(size_t slot, size_t n) {
    if (data.n == 0) fail(SNN_ERR_STATE, "no dataset staged");
    if (slot + n > sched_steps) fail(SNN_ERR_ARGUMENT, "schedule slots [%zu, %zu) out of range", slot, slot + n);
    ensure_bc_capacity(n);
    if (slot != slot_expected) {
      const int64_t s = int64_t(slot);  // pageable source: staged before the call returns
      CK(cudaMemcpyAsync(sched_slot.p, &s, sizeof(s), cudaMemcpyHostToDevice, stream));
    }
    size_t done = 0;
    for (; done + kSchedGraphSteps <= n; done += kSchedGraphSteps)
      CK(cudaGraphLaunch(graph_for(data, 1, kSchedGraphSteps), stream));
    for (; done < n; ++done) CK(cudaGraphLaunch(graph_for(data, 1, 1), stream));
    slot_expected = slot + n;
    host_step += int64_t(n);
  }

  void set_rows_host(const uint32_t* rows, const Dataset& ds) {
    for (int i = 0; i < B; ++i) {
      if (rows[i] >= ds.n) fail(SNN_ERR_ARGUMENT, "row %u outside dataset of %zu", rows[i], ds.n);
      h_rows[i] = rows[i];
    }
    CK(cudaMemcpyAsync(rows_cur.p, h_rows, sizeof(uint32_t) * B, cudaMemcpyHostToDevice, stream));
  }

  void read_result(float* loss, double* acc) {
    CK(cudaMemcpyAsync(h_loss, result_loss.p, sizeof(float), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(h_acc, result_acc.p, sizeof(double), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    check_peer_timeout();
    if (loss) *loss = *h_loss;
    if (acc) *acc = *h_acc;
  }
  // after an update launch: the fused tail already wrote the StepResult into the
  // mapped ring, so only the sync remains (no D2H copies)
  void read_step_result(float* loss, double* acc) {
    if (!ring_on()) return read_result(loss, acc);
    CK(cudaStreamSynchronize(stream));
    const int64_t r = (host_step - 1) & (kRing - 1);
    if (loss) *loss = ring_loss_h[r];
    if (acc) *acc = ring_acc_h[r];
  }

  void step_rows(const uint32_t* rows, const Dataset& ds, int update, float* loss, double* acc) {
    set_rows_host(rows, ds);
    launch(ds, update);
    if (update) read_step_result(loss, acc);
    else read_result(loss, acc);
  }

  // level 0 off, 1 tensors + clock stamps, 2 clock stamps only (kernels run their
  // production code paths: no capture stores)
  void set_debug(int level) {
    const bool on = level == 1;
    debug = on;
    clocks = level != 0;
    const size_t rows = size_t(B) * T_pad;
    for (int l = 0; l < L; ++l) {
      if (on) {
        dbg_i[l].alloc(rows * H_pad[l]);
        dbg_ds[l].alloc(rows * H_pad[l]);
      } else {
        dbg_i[l].free();
        dbg_ds[l].free();
      }
    }
    if (on) dbg_trace.alloc(size_t(B) * T * C); else dbg_trace.free();
    // clock stamps: slot 0 readout [B][8], slots 1..L fwd, L+1..2L bwd ([B*8 ctas][8] each)
    if (clocks) dbg_clk.alloc(size_t(3 + 2 * L) * clk_region()); else dbg_clk.free();
    clear_graphs();
  }
};

// =================================================================== C ABI
namespace {

template <typename F>
snn_status guard(snn_engine* e, F&& f) {
  try {
    if (e) CK(cudaSetDevice(e->device));
    f();
    return SNN_OK;
  } catch (const SnnError& err) {
    if (e) e->err = err.msg; else g_create_error = err.msg;
    return err.code;
  } catch (const std::exception& ex) {
    if (e) e->err = ex.what(); else g_create_error = ex.what();
    return SNN_ERR_CUDA;
  }
}

void check_n(const snn_engine* e, size_t n) {
  if (n != e->n_params)
    fail(SNN_ERR_SHAPE, "expected %zu parameter scalars, got %zu", e->n_params, n);
}

}  // namespace

extern "C" {

int snn_abi_version(void) { return SNN_ABI_VERSION; }

const char* snn_last_error(const snn_engine* e) {
  return e ? e->err.c_str() : g_create_error.c_str();
}

snn_status snn_engine_create(const snn_network_desc* net, const snn_train_config* cfg, int device,
                             snn_engine** out) {
  if (!net || !cfg || !out) {
    g_create_error = "null argument";
    return SNN_ERR_ARGUMENT;
  }
  *out = nullptr;
  auto e = std::make_unique<snn_engine>();
  e->net = *net;
  e->cfg = *cfg;
  e->device = device;
  const snn_status st = guard(nullptr, [&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device)
      fail(SNN_ERR_CUDA, "no CUDA device %d (this engine has no CPU fallback)", device);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(SNN_ERR_CUDA, "device %d is sm_%d%d; this engine is built for sm_100a only", device,
           prop.major, prop.minor);
    e->validate_and_size();
    e->allocate();
    // train(spec, cfg, data): params from master.child(0) (optimize.hpp:246-254)
    e->init_params_host(hostrng::child(hostrng::from_seed(cfg->seed), 0));
  });
  if (st != SNN_OK) return st;
  *out = e.release();
  return SNN_OK;
}

void snn_engine_destroy(snn_engine* e) { delete e; }

snn_status snn_param_count(const snn_engine* e, size_t* n) {
  if (!e || !n) return SNN_ERR_ARGUMENT;
  *n = e->n_params;
  return SNN_OK;
}

snn_status snn_entry_count(const snn_engine* e, int32_t* n) {
  if (!e || !n) return SNN_ERR_ARGUMENT;
  *n = int32_t(e->entries.size());
  return SNN_OK;
}

snn_status snn_entry_info(const snn_engine* e, int32_t i, char name[16], size_t* offset,
                          size_t* size, int32_t* trainable) {
  if (!e || i < 0 || size_t(i) >= e->entries.size()) return SNN_ERR_ARGUMENT;
  const auto& en = e->entries[size_t(i)];
  if (name) std::snprintf(name, 16, "%s", en.name.c_str());
  if (offset) *offset = en.offset;
  if (size) *size = en.size;
  if (trainable) *trainable = 1;
  return SNN_OK;
}

snn_status snn_set_params(snn_engine* e, const float* host, size_t n) {
  if (!e || !host) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    check_n(e, n);
    e->upload_params(host);
  });
}

snn_status snn_get_params(snn_engine* e, float* host, size_t n) {
  if (!e || !host) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    check_n(e, n);
    CK(cudaMemcpyAsync(host, e->params.p, n * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
  });
}

snn_status snn_init_params(snn_engine* e, uint64_t key_word) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] { e->init_params_host(key_word); });
}

// ------------------------------------------------------------- checkpoints
// .spkc (optimize.hpp:300-436): "SPKC", u32 version 1, u64 fnv1a(config), u64
// config length, config bytes, u8 scalar width, u32 entry count, entries (u16
// name length, name, u8 trainable, u32 ndim, u64 dims, payload), u8 optimizer
// kind, u64 step, m payloads, v payloads (Adam only).  Little-endian, bit-exact.
namespace {
uint64_t fnv1a(const char* s, size_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= static_cast<unsigned char>(s[i]);
    h *= 0x100000001B3ull;
  }
  return h;
}
struct Reader {
  const std::vector<uint8_t>& b;
  size_t off = 0;
  void take(void* dst, size_t n) {
    if (off + n > b.size()) fail(SNN_ERR_IO, "short read at byte offset %zu", off);
    std::memcpy(dst, b.data() + off, n);
    off += n;
  }
  uint8_t u8() { uint8_t v; take(&v, 1); return v; }
  uint16_t u16() { uint16_t v; take(&v, 2); return v; }
  uint32_t u32() { uint32_t v; take(&v, 4); return v; }
  uint64_t u64() { uint64_t v; take(&v, 8); return v; }
};
void put_bytes(std::vector<uint8_t>& o, const void* p, size_t n) {
  const uint8_t* c = static_cast<const uint8_t*>(p);
  o.insert(o.end(), c, c + n);
}
void put_u8(std::vector<uint8_t>& o, uint8_t v) { put_bytes(o, &v, 1); }
void put_u16(std::vector<uint8_t>& o, uint16_t v) { put_bytes(o, &v, 2); }
void put_u32(std::vector<uint8_t>& o, uint32_t v) { put_bytes(o, &v, 4); }
void put_u64(std::vector<uint8_t>& o, uint64_t v) { put_bytes(o, &v, 8); }
}  // namespace

snn_status snn_save_checkpoint(snn_engine* e, const char* path, const char* config_text,
                               size_t config_len) {
  if (!e || !path || (!config_text && config_len)) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    const size_t n = e->n_params;
    std::vector<float> p(n), m(n), v(n);
    int64_t step = 0;
    e->sync_opt_from_owners();
    CK(cudaMemcpyAsync(p.data(), e->params.p, n * 4, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemcpyAsync(m.data(), e->m.p, n * 4, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemcpyAsync(v.data(), e->v.p, n * 4, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemcpyAsync(&step, e->step.p, 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    std::vector<uint8_t> o;
    put_bytes(o, "SPKC", 4);
    put_u32(o, 1);
    put_u64(o, fnv1a(config_text, config_len));
    put_u64(o, config_len);
    put_bytes(o, config_text, config_len);
    put_u8(o, 4);
    put_u32(o, uint32_t(e->entries.size()));
    for (const auto& en : e->entries) {
      put_u16(o, uint16_t(en.name.size()));
      put_bytes(o, en.name.data(), en.name.size());
      put_u8(o, en.trainable() ? 1 : 0);  // Fixed beta is not trainable (neuron.hpp:32)
      put_u32(o, uint32_t(en.ndim()));
      if (en.ndim() == 2) {
        put_u64(o, uint64_t(en.rows));
        put_u64(o, uint64_t(en.cols));
      } else if (en.ndim() == 1) {
        put_u64(o, uint64_t(en.cols));
      }
      put_bytes(o, p.data() + en.offset, en.size * 4);
    }
    put_u8(o, e->cfg.optimizer == 1 ? 1 : 0);
    put_u64(o, uint64_t(step));
    // optimizer state covers the trainable entries only (init_optimizer, optimize.hpp:37-48)
    for (const auto& en : e->entries)
      if (en.trainable()) put_bytes(o, m.data() + en.offset, en.size * 4);
    if (e->cfg.optimizer != 1)
      for (const auto& en : e->entries)
        if (en.trainable()) put_bytes(o, v.data() + en.offset, en.size * 4);
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(SNN_ERR_IO, "cannot open for writing: %s", path);
    const size_t w = std::fwrite(o.data(), 1, o.size(), f);
    const int rc = std::fclose(f);
    if (w != o.size() || rc != 0) fail(SNN_ERR_IO, "short write: %s", path);
  });
}

snn_status snn_load_checkpoint(snn_engine* e, const char* path, char* config_out,
                               size_t config_cap, size_t* config_len) {
  if (!e || !path) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(SNN_ERR_IO, "cannot open for reading: %s", path);
    std::vector<uint8_t> b;
    uint8_t buf[1 << 16];
    for (size_t r; (r = std::fread(buf, 1, sizeof(buf), f)) > 0;) b.insert(b.end(), buf, buf + r);
    std::fclose(f);
    Reader rd{b};
    char magic[4];
    rd.take(magic, 4);
    if (std::memcmp(magic, "SPKC", 4) != 0) fail(SNN_ERR_FORMAT, "bad magic at byte offset 0");
    const uint32_t version = rd.u32();
    if (version != 1) fail(SNN_ERR_FORMAT, "unsupported checkpoint version %u at byte offset 4", version);
    const uint64_t hash = rd.u64();
    const uint64_t clen = rd.u64();
    if (clen > (1u << 20)) fail(SNN_ERR_FORMAT, "implausible config length at byte offset 16");
    std::string cfg(clen, '\0');
    rd.take(cfg.data(), clen);
    if (fnv1a(cfg.data(), cfg.size()) != hash)
      fail(SNN_ERR_FORMAT, "config hash mismatch (stored %llu)", (unsigned long long)hash);
    const uint8_t width = rd.u8();
    if (width != 4) fail(SNN_ERR_FORMAT, "checkpoint scalar width %u, expected 4", unsigned(width));
    const uint32_t ne = rd.u32();
    if (ne != e->entries.size())
      fail(SNN_ERR_SHAPE, "checkpoint holds %u entries, the network %zu", ne, e->entries.size());
    const size_t n = e->n_params;
    std::vector<float> p(n), m(n, 0.0f), v(n, 0.0f);
    for (const auto& en : e->entries) {
      const uint16_t nl = rd.u16();
      std::string name(nl, '\0');
      rd.take(name.data(), nl);
      const uint8_t trainable = rd.u8();
      const uint32_t nd = rd.u32();
      if (nd > 16) fail(SNN_ERR_FORMAT, "implausible tensor rank at byte offset %zu", rd.off - 4);
      std::vector<uint64_t> dims(nd);
      for (auto& d : dims) d = rd.u64();
      const bool shape_ok = int(nd) == en.ndim() &&
                            (nd == 0 || (nd == 1 && dims[0] == uint64_t(en.cols)) ||
                             (nd == 2 && dims[0] == uint64_t(en.rows) && dims[1] == uint64_t(en.cols)));
      if (name != en.name || !shape_ok || trainable != (en.trainable() ? 1 : 0))
        fail(SNN_ERR_SHAPE, "checkpoint entry %s does not match network entry %s", name.c_str(),
             en.name.c_str());
      rd.take(p.data() + en.offset, en.size * 4);
    }
    const uint8_t kind = rd.u8();
    if (int(kind) != (e->cfg.optimizer == 1 ? 1 : 0))
      fail(SNN_ERR_ARGUMENT, "checkpoint optimizer kind %u differs from the engine's", unsigned(kind));
    const int64_t step = int64_t(rd.u64());
    for (const auto& en : e->entries)
      if (en.trainable()) rd.take(m.data() + en.offset, en.size * 4);
    if (kind == 0)
      for (const auto& en : e->entries)
        if (en.trainable()) rd.take(v.data() + en.offset, en.size * 4);
    e->upload_params(p.data());
    CK(cudaMemcpyAsync(e->m.p, m.data(), n * 4, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(e->v.p, v.data(), n * 4, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(e->step.p, &step, 8, cudaMemcpyHostToDevice, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    e->host_step = step;
    e->ensure_bc_capacity();
    if (config_len) *config_len = cfg.size();
    if (config_out && config_cap) {
      const size_t c = std::min(config_cap - 1, cfg.size());
      std::memcpy(config_out, cfg.data(), c);
      config_out[c] = '\0';
    }
  });
}

snn_status snn_get_opt_state(snn_engine* e, float* m, float* v, uint64_t* step, size_t n) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    check_n(e, n);
    e->sync_opt_from_owners();
    if (m) CK(cudaMemcpyAsync(m, e->m.p, n * 4, cudaMemcpyDeviceToHost, e->stream));
    if (v) CK(cudaMemcpyAsync(v, e->v.p, n * 4, cudaMemcpyDeviceToHost, e->stream));
    int64_t s = 0;
    CK(cudaMemcpyAsync(&s, e->step.p, 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    e->host_step = s;
    if (step) *step = uint64_t(s);
  });
}

snn_status snn_set_opt_state(snn_engine* e, const float* m, const float* v, uint64_t step,
                             size_t n) {
  if (!e || !m || !v) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    check_n(e, n);
    const int64_t s = int64_t(step);
    CK(cudaMemcpyAsync(e->m.p, m, n * 4, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(e->v.p, v, n * 4, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(e->step.p, &s, 8, cudaMemcpyHostToDevice, e->stream));
    if (e->tail_mode == 2) {  // the mirrors other ranks pull from (sync_opt_from_owners)
      float* x = e->peer_xchg[e->rank];
      CK(cudaMemcpyAsync(x + peer_m_off(e->n_comm), m, n * 4, cudaMemcpyHostToDevice, e->stream));
      CK(cudaMemcpyAsync(x + peer_v_off(e->n_comm), v, n * 4, cudaMemcpyHostToDevice, e->stream));
    }
    CK(cudaStreamSynchronize(e->stream));
    e->host_step = s;
    e->ensure_bc_capacity();
  });
}

snn_status snn_get_grads(snn_engine* e, float* host, size_t n) {
  if (!e || !host) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    check_n(e, n);
    CK(cudaMemcpyAsync(host, e->comm.p, n * 4, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
  });
}

snn_status snn_stage_dataset(snn_engine* e, const uint8_t* packed, size_t n,
                             const int64_t* labels) {
  if (!e || !packed || !labels || n == 0) return SNN_ERR_ARGUMENT;
  return guard(e, [&] { e->stage(e->data, packed, n, labels); });
}

snn_status snn_train_step(snn_engine* e, const uint32_t* rows, float* loss, double* accuracy) {
  if (!e || !rows) return SNN_ERR_ARGUMENT;
  return guard(e, [&] { e->step_rows(rows, e->data, 1, loss, accuracy); });
}

snn_status snn_forward_backward(snn_engine* e, const uint32_t* rows, float* loss,
                                double* accuracy) {
  if (!e || !rows) return SNN_ERR_ARGUMENT;
  return guard(e, [&] { e->step_rows(rows, e->data, 0, loss, accuracy); });
}

snn_status snn_train_step_packed(snn_engine* e, const uint8_t* packed_batch,
                                 const int64_t* targets, float* loss, double* accuracy) {
  if (!e || !packed_batch || !targets) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    static const bool trace = std::getenv("SNN_E2E_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    e->stage_batch(e->scratch, packed_batch, size_t(e->B), targets);
    const auto t1 = std::chrono::steady_clock::now();
    std::vector<uint32_t> rows(size_t(e->B));
    for (int i = 0; i < e->B; ++i) rows[size_t(i)] = uint32_t(i);
    e->set_rows_host(rows.data(), e->scratch);
    e->launch(e->scratch, 1);
    const auto t2 = std::chrono::steady_clock::now();
    e->read_step_result(loss, accuracy);
    const auto t3 = std::chrono::steady_clock::now();
    if (trace) {  // host-side phase times of the e2e call (diagnostics)
      static double acc[3];
      static int calls;
      acc[0] += std::chrono::duration<double, std::micro>(t1 - t0).count();
      acc[1] += std::chrono::duration<double, std::micro>(t2 - t1).count();
      acc[2] += std::chrono::duration<double, std::micro>(t3 - t2).count();
      if (++calls % 200 == 0)
        std::fprintf(stderr, "e2e host us/step: stage %.1f  launch %.1f  wait+result %.1f\n", acc[0] / calls,
                     acc[1] / calls, acc[2] / calls);
    }
  });
}

snn_status snn_train_steps_packed(snn_engine* e, const uint8_t* packed, const int64_t* targets,
                                  size_t n_steps, float* losses, double* accuracies) {
  if (!e || !packed || !targets) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    if (n_steps == 0) return;
    e->pipe_init(n_steps);
    e->ensure_bc_capacity(n_steps);
    std::vector<uint32_t> rows(size_t(e->B));
    for (int i = 0; i < e->B; ++i) rows[size_t(i)] = uint32_t(i);
    e->set_rows_host(rows.data(), e->pslot[0]);
    CK(cudaStreamSynchronize(e->stream));  // the pinned label / result arrays are free
    for (size_t i = 0; i < n_steps * size_t(e->B); ++i) {
      if (targets[i] < 0 || targets[i] >= e->C)
        fail(SNN_ERR_ARGUMENT, "target %lld outside [0,%d)", (long long)targets[i], e->C);
      e->plab_host[i] = int32_t(targets[i]);
    }
    // StepResults: the fused tail writes them into the mapped ring (read after a sync
    // at least every kRing steps); other tails copy each one out with k_result_out
    const bool ring = e->ring_on();
    const int64_t s0 = e->host_step;
    size_t read = 0;
    auto drain = [&](size_t upto) {
      CK(cudaStreamSynchronize(e->stream));
      for (; read < upto; ++read) {
        const int64_t r = (s0 + int64_t(read)) & (snn_engine::kRing - 1);
        if (losses) losses[read] = ring ? e->ring_loss_h[r] : e->pres_loss[read];
        if (accuracies) accuracies[read] = ring ? e->ring_acc_h[r] : e->pres_acc[read];
      }
    };
    e->pipe_stage(0, packed, targets);
    for (size_t k = 0; k < n_steps; ++k) {
      const int sl = int(k & 1);
      if (ring && k + 1 - read > size_t(snn_engine::kRing)) drain(k);  // step k reuses an unread entry
      CK(cudaStreamWaitEvent(e->stream, e->ev_ready[sl], 0));
      e->launch(e->pslot[sl], 1);
      CK(cudaEventRecord(e->ev_used[sl], e->stream));
      if (k + 1 < n_steps) e->pipe_stage(k + 1, packed, targets);  // runs while step k does
      if (ring) continue;
      float* hl = nullptr;
      double* ha = nullptr;
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hl), e->pres_loss + k, 0));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ha), e->pres_acc + k, 0));
      k_result_out<<<1, 1, 0, e->stream>>>(e->result_loss.p, e->result_acc.p, hl, ha);
      CK(cudaGetLastError());
    }
    drain(n_steps);
  });
}

snn_status snn_train_epochs_from(snn_engine* e, size_t first_epoch, size_t epochs,
                                 double* metrics) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    const size_t n = e->data.n;
    if (n == 0) fail(SNN_ERR_STATE, "no dataset staged");
    const size_t gb = size_t(e->B_global());
    if (gb > n) fail(SNN_ERR_ARGUMENT, "shuffle: batch size %zu for %zu examples", gb, n);
    const uint64_t master = hostrng::from_seed(e->cfg.seed);
    const size_t nb = n / gb;
    struct ShiftReset {  // an interrupted epoch must not leave later steps rolled
      snn_engine* e;
      ~ShiftReset() {
        try { e->set_shift(0); } catch (...) {}
      }
    } shift_reset{e};
    for (size_t k = 0; k < epochs; ++k) {
      const size_t ep = first_epoch + k;
      const uint64_t ek = hostrng::child(master, 1 + ep);
      const std::vector<uint32_t> perm = hostrng::permutation(hostrng::child(ek, 0), n);
      double ls = 0, as = 0;
      for (size_t bi = 0; bi < nb; ++bi) {
        float l;
        double a;
        e->set_shift(hostrng::batch_roll(ek, bi, e->cfg.max_shift, e->cfg.n_shift_axes, e->IN));
        e->step_rows(perm.data() + bi * gb + size_t(e->rank) * e->B, e->data, 1, &l, &a);
        ls += double(l);
        as += a;
      }
      e->set_shift(0);
      if (metrics) {
        metrics[2 * k] = ls / double(nb ? nb : 1);
        metrics[2 * k + 1] = as / double(nb ? nb : 1);
      }
    }
  });
}

snn_status snn_train_epochs(snn_engine* e, size_t epochs, double* metrics) {
  return snn_train_epochs_from(e, 0, epochs, metrics);
}

snn_status snn_upload_schedule(snn_engine* e, const uint32_t* rows, size_t n_steps) {
  if (!e || !rows || n_steps == 0) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    for (size_t i = 0; i < n_steps * size_t(e->B); ++i)
      if (rows[i] >= e->data.n) fail(SNN_ERR_ARGUMENT, "schedule row outside dataset");
    CK(cudaStreamSynchronize(e->stream));
    e->sched.alloc(n_steps * size_t(e->B), false);
    e->sched_steps = n_steps;
    e->slot_expected = ~size_t(0);
    CK(cudaMemcpy(e->sched.p, rows, n_steps * e->B * sizeof(uint32_t), cudaMemcpyHostToDevice));
    e->clear_graphs();  // schedule-mode graphs bake the schedule pointer
    if (e->data.n > 0) {  // capture both schedule graphs now, outside any timed region
      e->graph_for(e->data, 1, 1);
      e->graph_for(e->data, 1, snn_engine::kSchedGraphSteps);
    }
  });
}

snn_status snn_enqueue_step(snn_engine* e, size_t slot) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    e->launch_sched(slot, 1);
  });
}

snn_status snn_enqueue_steps(snn_engine* e, size_t first_slot, size_t n_steps) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] { e->launch_sched(first_slot, n_steps); });
}

// cmd_eval (commands.hpp:144-169): accuracy over `n` dataset rows in batches of the
// engine batch size B, the last batch short (its padding rows are not counted);
// per batch integral_accuracy = hits / nb (objective.hpp:118-134), accumulated as
// correct += acc * nb and divided by n, in the reference's double arithmetic.
snn_status snn_evaluate(snn_engine* e, const uint32_t* rows, size_t n, double* accuracy,
                        double* mean_loss) {
  if (!e || !rows || n == 0) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    if (e->data.n == 0) fail(SNN_ERR_STATE, "no dataset staged");
    for (size_t i = 0; i < n; ++i)
      if (rows[i] >= e->data.n) fail(SNN_ERR_ARGUMENT, "row %u outside dataset of %zu", rows[i], e->data.n);
    const size_t B = size_t(e->B), nb = (n + B - 1) / B;
    uint32_t* h_rows = nullptr;
    int32_t* h_hit = nullptr;
    float* h_loss = nullptr;
    CK(cudaMallocHost(&h_rows, nb * B * sizeof(uint32_t)));
    CK(cudaMallocHost(&h_hit, nb * B * sizeof(int32_t)));
    CK(cudaMallocHost(&h_loss, nb * B * sizeof(float)));
    struct Free {
      void* p[3];
      ~Free() { for (void* q : p) if (q) cudaFreeHost(q); }
    } fr{{h_rows, h_hit, h_loss}};
    for (size_t i = 0; i < nb * B; ++i) h_rows[i] = i < n ? rows[i] : rows[0];
    cudaGraphExec_t g = e->graph_for(e->data, snn_engine::kEval);
    for (size_t i = 0; i < nb; ++i) {
      CK(cudaMemcpyAsync(e->rows_cur.p, h_rows + i * B, B * sizeof(uint32_t), cudaMemcpyHostToDevice, e->stream));
      CK(cudaGraphLaunch(g, e->stream));
      CK(cudaMemcpyAsync(h_hit + i * B, e->correct_b.p, B * sizeof(int32_t), cudaMemcpyDeviceToHost, e->stream));
      CK(cudaMemcpyAsync(h_loss + i * B, e->loss_b.p, B * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    }
    CK(cudaStreamSynchronize(e->stream));
    double correct = 0.0, loss = 0.0;
    for (size_t i = 0; i < nb; ++i) {
      const size_t cnt = std::min(B, n - i * B);
      size_t hits = 0;
      for (size_t j = 0; j < cnt; ++j) {
        hits += h_hit[i * B + j] != 0;
        loss += double(h_loss[i * B + j]);
      }
      correct += double(hits) / double(cnt) * double(cnt);
    }
    if (accuracy) *accuracy = correct / double(n);
    if (mean_loss) *mean_loss = loss / double(n);
  });
}

// apply (network.hpp:435-448) on one batch of B dataset rows: the readout (LI)
// trace [B][T][C], forward only.
snn_status snn_apply(snn_engine* e, const uint32_t* rows, float* trace, size_t n) {
  if (!e || !rows || !trace) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    if (e->data.n == 0) fail(SNN_ERR_STATE, "no dataset staged");
    const size_t need = size_t(e->B) * e->T * e->C;
    if (n != need) fail(SNN_ERR_SHAPE, "trace holds %zu floats, need %zu", n, need);
    if (e->eval_trace.n != need) {
      e->eval_trace.alloc(need);
      e->clear_graphs();
    }
    e->set_rows_host(rows, e->data);
    CK(cudaGraphLaunch(e->graph_for(e->data, snn_engine::kEvalTrace), e->stream));
    CK(cudaMemcpyAsync(trace, e->eval_trace.p, need * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
  });
}

snn_status snn_monitor_counts(snn_engine* e, int32_t layer, float* counts, size_t n) {
  if (!e || !counts) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    if (layer < 0 || layer >= e->L || !e->net.monitor[layer])
      fail(SNN_ERR_ARGUMENT, "hidden layer %d has no monitor", int(layer));
    const size_t need = size_t(e->B) * e->H[layer];
    if (n != need) fail(SNN_ERR_SHAPE, "counts holds %zu floats, need %zu", n, need);
    if (e->mon_counts.n < need) e->mon_counts.alloc(need, false);
    k_spike_counts<<<unsigned((need + 255) / 256), 256, 0, e->stream>>>(e->s_tp[layer].p, e->B, e->T_pad,
                                                                         e->H[layer], e->mon_counts.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(counts, e->mon_counts.p, need * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
  });
}

snn_status snn_sync(snn_engine* e) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] { CK(cudaStreamSynchronize(e->stream)); });
}

snn_status snn_read_result(snn_engine* e, float* loss, double* accuracy) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] { e->read_result(loss, accuracy); });
}

snn_status snn_synth_dataset(snn_engine* e, size_t n, uint64_t seed) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] { e->synth(n, seed); });
}

snn_status snn_read_dataset(snn_engine* e, size_t start, size_t n, uint8_t* packed,
                            int64_t* labels) {
  if (!e || !packed || !labels) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    if (start + n > e->data.n) fail(SNN_ERR_ARGUMENT, "rows [%zu,%zu) outside dataset", start, start + n);
    const int tp8 = (e->T + 7) / 8, tp8_pad = e->T_pad / 8;
    std::vector<uint8_t> h(n * size_t(tp8_pad) * e->IN_pad);
    std::vector<int32_t> lab(n);
    CK(cudaMemcpy(h.data(), e->data.x.p + start * size_t(tp8_pad) * e->IN_pad, h.size(),
                  cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(lab.data(), e->data.labels.p + start, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) {
      labels[i] = lab[i];
      for (int g = 0; g < tp8; ++g)
        std::memcpy(packed + (i * tp8 + g) * size_t(e->IN), h.data() + (i * tp8_pad + g) * e->IN_pad,
                    size_t(e->IN));
    }
  });
}

// .spkd container (data.hpp:229-341): little-endian header, i32 labels, packed payload.
snn_status snn_load_container(snn_engine* e, const char* path, size_t* n_out) {
  if (!e || !path) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(SNN_ERR_IO, "cannot open for reading: %s", path);
    std::unique_ptr<FILE, int (*)(FILE*)> hold(f, std::fclose);
    size_t off = 0;
    auto take = [&](void* p, size_t n) {  // io_read (data.hpp:255-263)
      const size_t got = std::fread(p, 1, n, f);
      if (got != n) fail(SNN_ERR_FORMAT, "container truncated at byte offset %zu", off + got);
      off += n;
    };
    char magic[4];
    take(magic, 4);
    if (std::memcmp(magic, "SPKD", 4) != 0) fail(SNN_ERR_FORMAT, "bad magic at byte offset 0");
    uint32_t version;
    take(&version, 4);
    if (version != 1) fail(SNN_ERR_FORMAT, "unsupported container version %u at byte offset 4", version);
    uint8_t dtype, order;
    take(&dtype, 1);
    if (dtype != 0) fail(SNN_ERR_FORMAT, "unknown dtype %u at byte offset 8", unsigned(dtype));
    take(&order, 1);
    if (order != 0) fail(SNN_ERR_FORMAT, "unknown bit order %u at byte offset 9", unsigned(order));
    uint16_t reserved;
    take(&reserved, 2);
    uint32_t original_t, ndim;
    take(&original_t, 4);
    take(&ndim, 4);
    if (ndim < 2 || ndim > 16) fail(SNN_ERR_FORMAT, "implausible ndim %u at byte offset 16", ndim);
    std::vector<uint64_t> shape(ndim);
    for (auto& d : shape) take(&d, 8);
    if (shape[1] != (uint64_t(original_t) + 7) / 8)
      fail(SNN_ERR_FORMAT, "packed time extent %llu inconsistent with T=%u", (unsigned long long)shape[1],
           original_t);
    uint64_t n_labels;
    take(&n_labels, 8);
    if (n_labels != shape[0])
      fail(SNN_ERR_FORMAT, "label count %llu does not match N=%llu", (unsigned long long)n_labels,
           (unsigned long long)shape[0]);
    // the engine's shape: T and the flattened per-step features (a Linear flattens, network.hpp:133-138)
    uint64_t feat = 1;
    for (uint32_t i = 2; i < ndim; ++i) feat *= shape[i];
    if (int64_t(original_t) != e->T)
      fail(SNN_ERR_FORMAT, "unpack_time: container T=%u, engine T=%d", original_t, e->T);
    if (feat != uint64_t(e->IN))
      fail(SNN_ERR_SHAPE, "container has %llu features per step, network input %d", (unsigned long long)feat,
           e->IN);
    if (n_labels == 0) fail(SNN_ERR_ARGUMENT, "empty container");
    std::vector<int32_t> lab32(n_labels);
    take(lab32.data(), n_labels * 4);
    std::vector<int64_t> lab(lab32.begin(), lab32.end());
    std::vector<uint8_t> x(size_t(n_labels) * shape[1] * feat);
    take(x.data(), x.size());
    e->stage(e->data, x.data(), size_t(n_labels), lab.data());
    if (n_out) *n_out = size_t(n_labels);
  });
}

snn_status snn_save_container(snn_engine* e, const char* path) {
  if (!e || !path) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    const size_t n = e->data.n;
    if (n == 0) fail(SNN_ERR_STATE, "no dataset staged");
    const int tp8 = (e->T + 7) / 8;
    std::vector<uint8_t> x(n * size_t(tp8) * e->IN);
    std::vector<int64_t> lab(n);
    const snn_status st = snn_read_dataset(e, 0, n, x.data(), lab.data());
    if (st != SNN_OK) fail(st, "%s", e->err.c_str());
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(SNN_ERR_IO, "cannot open for writing: %s", path);
    std::unique_ptr<FILE, int (*)(FILE*)> hold(f, std::fclose);
    bool ok = true;
    auto put = [&](const void* p, size_t b) { ok = ok && std::fwrite(p, 1, b, f) == b; };
    const uint32_t version = 1, T = uint32_t(e->T), ndim = 3;
    const uint8_t zero8 = 0;
    const uint16_t zero16 = 0;
    put("SPKD", 4);
    put(&version, 4);
    put(&zero8, 1);   // dtype u8
    put(&zero8, 1);   // MSB-first
    put(&zero16, 2);  // reserved
    put(&T, 4);
    put(&ndim, 4);
    const uint64_t shape[3] = {uint64_t(n), uint64_t(tp8), uint64_t(e->IN)};
    put(shape, sizeof(shape));
    const uint64_t nl = n;
    put(&nl, 8);
    for (int64_t l : lab) {
      const int32_t v = int32_t(l);
      put(&v, 4);
    }
    put(x.data(), x.size());
    if (!ok) fail(SNN_ERR_IO, "short write: %s", path);
  });
}

snn_status snn_epoch_permutation(snn_engine* e, size_t epoch, uint32_t* out, size_t n) {
  if (!e || !out) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    const uint64_t ek = hostrng::child(hostrng::from_seed(e->cfg.seed), 1 + epoch);
    const std::vector<uint32_t> p = hostrng::permutation(hostrng::child(ek, 0), n);
    std::memcpy(out, p.data(), n * sizeof(uint32_t));
  });
}

snn_status snn_profile_steps(snn_engine* e, int32_t steps, double* ms, int32_t max_launches,
                             int32_t* n_launches) {
  if (!e || !ms || !n_launches || steps < 1) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    const std::vector<double> t = e->profile(steps);
    *n_launches = int32_t(t.size());
    for (size_t i = 0; i < t.size() && int32_t(i) < max_launches; ++i) ms[i] = t[i];
  });
}

const char* snn_launch_name(const snn_engine* e, int32_t i) {
  if (!e || i < 0 || size_t(i) >= e->launch_names.size()) return "";
  return e->launch_names[size_t(i)].c_str();
}

void* snn_stream(snn_engine* e) { return e ? static_cast<void*>(e->stream) : nullptr; }

int32_t snn_launches_per_step(const snn_engine* e) { return e ? e->launches_per_step() : 0; }

int32_t snn_forward_launch_layers(const snn_engine* e, int32_t i, int32_t* first) {
  if (!e || i < 0) return 0;
  const auto g = e->fwd_groups();
  if (size_t(i) >= g.size()) return 0;
  if (first) *first = g[size_t(i)].first;
  return g[size_t(i)].second;
}

snn_status snn_nccl_unique_id(uint8_t id[128]) {
  if (!id) return SNN_ERR_ARGUMENT;
  NcclApi& api = nccl();
  if (!api.ok) {
    g_create_error = "libnccl.so.2 not loadable";
    return SNN_ERR_CUDA;
  }
  UniqueId u;
  const int rc = api.GetUniqueId(&u);
  if (rc != 0) {
    g_create_error = "ncclGetUniqueId failed";
    return SNN_ERR_CUDA;
  }
  std::memcpy(id, u.internal, 128);
  return SNN_OK;
}

snn_status snn_comm_init(snn_engine* e, const uint8_t id[128], int32_t rank, int32_t world) {
  if (!e || !id || world < 1 || rank < 0 || rank >= world) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    // world == 1 still creates a (single-rank) communicator: the step then runs the
    // multi-rank tail (k_reduce -> ncclAllReduce -> k_adam), testable on one GPU
    if (e->tail_mode == 2) fail(SNN_ERR_STATE, "engine already runs the peer-memory tail");
    NcclApi& api = nccl();
    if (!api.ok) fail(SNN_ERR_CUDA, "libnccl.so.2 not loadable");
    UniqueId u;
    std::memcpy(u.internal, id, 128);
    void* comm = nullptr;
    const int rc = reinterpret_cast<InitRankFn>(api.CommInitRank)(&comm, world, u, rank);
    if (rc != 0) fail(SNN_ERR_CUDA, "ncclCommInitRank failed (%d)", rc);
    e->comm_handle = comm;
    e->rank = rank;
    e->world = world;
    e->tail_mode = 1;
    e->clear_graphs();
  });
}

snn_status snn_peer_handle(snn_engine* e, uint8_t handle[64]) {
  if (!e || !handle) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    e->ensure_peer_mem();
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, e->peer_mem.p));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, 64);
  });
}

snn_status snn_peer_open(snn_engine* e, int32_t rank, int32_t world, const uint8_t* handles) {
  if (!e || !handles || world < 1 || world > kMaxRanks || rank < 0 || rank >= world) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    if (e->comm_handle) fail(SNN_ERR_STATE, "engine already has an NCCL communicator");
    e->ensure_peer_mem();
    uint8_t* bases[kMaxRanks] = {};
    for (int q = 0; q < world; ++q) {
      if (q == rank) {
        bases[q] = e->peer_mem.p;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + size_t(q) * 64, 64);
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      e->peer_ipc[q] = p;
      bases[q] = static_cast<uint8_t*>(p);
    }
    e->set_peers(rank, world, bases);
  });
}

snn_status snn_peer_attach_local(snn_engine* const* engines, int32_t world) {
  if (!engines || world < 1 || world > kMaxRanks) return SNN_ERR_ARGUMENT;
  for (int q = 0; q < world; ++q)
    if (!engines[q]) return SNN_ERR_ARGUMENT;
  snn_status st = SNN_OK;
  uint8_t* bases[kMaxRanks] = {};
  for (int q = 0; q < world && st == SNN_OK; ++q)
    st = guard(engines[q], [&] {
      if (engines[q]->device != engines[0]->device) fail(SNN_ERR_ARGUMENT, "ranks on different devices");
      if (engines[q]->n_params != engines[0]->n_params) fail(SNN_ERR_ARGUMENT, "ranks differ in network");
      engines[q]->ensure_peer_mem();
      bases[q] = engines[q]->peer_mem.p;
    });
  for (int q = 0; q < world && st == SNN_OK; ++q)
    st = guard(engines[q], [&] { engines[q]->set_peers(q, world, bases); });
  return st;
}

snn_status snn_train_step_split(snn_engine* e, const uint32_t* rows, int32_t part, float* loss,
                                double* accuracy) {
  if (!e || part < 0 || part > 2 || (part == 0 && !rows)) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    if (e->tail_mode != 2) fail(SNN_ERR_STATE, "split steps need the peer tail");
    if (e->data.n == 0) fail(SNN_ERR_STATE, "no dataset staged");
    struct Reset {
      snn_engine* e;
      ~Reset() { e->split_part = -1; }
    } reset{e};
    e->split_part = part;
    if (part == 0) {
      e->set_rows_host(rows, e->data);
      e->ensure_bc_capacity();
      e->enqueue_body(e->data, 1);
      CK(cudaStreamSynchronize(e->stream));
    } else if (part == 1) {
      e->enqueue_body(e->data, 1);
      CK(cudaStreamSynchronize(e->stream));
    } else {
      e->enqueue_body(e->data, 1);
      e->host_step += 1;
      e->read_result(loss, accuracy);
    }
  });
}

snn_status snn_debug_check_guards(snn_engine* e, int32_t* checked) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    CK(cudaDeviceSynchronize());
    std::vector<std::pair<const void*, size_t>> bufs;
    {
      std::lock_guard<std::mutex> lk(guards::mu());
      bufs.assign(guards::live().begin(), guards::live().end());
    }
    std::vector<unsigned char> h(guards::kGuardBytes);
    for (const auto& b : bufs) {
      CK(cudaMemcpy(h.data(), static_cast<const unsigned char*>(b.first) + b.second, h.size(),
                    cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < h.size(); ++i)
        if (h[i] != guards::kPattern)
          fail(SNN_ERR_CONTRACT, "out-of-bounds write: byte %zu past the end of a %zu-byte buffer", i,
               b.second);
    }
    if (checked) *checked = int32_t(bufs.size());
  });
}

snn_status snn_debug_enable(snn_engine* e, int32_t on) {
  if (!e) return SNN_ERR_ARGUMENT;
  return guard(e, [&] { e->set_debug(on == 2 ? 2 : on != 0 ? 1 : 0); });
}

snn_status snn_debug_fetch(snn_engine* e, int32_t which, int32_t layer, void* host, size_t bytes) {
  if (!e || !host) return SNN_ERR_ARGUMENT;
  return guard(e, [&] {
    if (which == 5 ? !e->clocks : !e->debug) fail(SNN_ERR_STATE, "debug capture not enabled");
    const int B = e->B, T = e->T, T_pad = e->T_pad;
    if (which == 5) {
      const size_t need = size_t(3 + 2 * e->L) * e->clk_region() * sizeof(long long);
      if (bytes != need) fail(SNN_ERR_SHAPE, "need %zu bytes", need);
      CK(cudaMemcpy(host, e->dbg_clk.p, need, cudaMemcpyDeviceToHost));
      return;
    }
    if (which == 3) {
      const size_t need = size_t(B) * T * e->C * sizeof(float);
      if (bytes != need) fail(SNN_ERR_SHAPE, "need %zu bytes", need);
      CK(cudaMemcpy(host, e->dbg_trace.p, need, cudaMemcpyDeviceToHost));
      return;
    }
    if (which == 7) {  // dI of Linear `layer` (0..L; L = readout), from its three bf16 planes
      if (layer < 0 || layer > e->L) fail(SNN_ERR_ARGUMENT, "layer %d", layer);
      const int W = layer < e->L ? e->H[layer] : e->C, Np = e->N_pad[layer];
      const size_t need = size_t(B) * T * W * sizeof(float);
      if (bytes != need) fail(SNN_ERR_SHAPE, "need %zu bytes", need);
      const size_t rows = size_t(B) * T_pad;
      std::vector<uint16_t> buf(size_t(3) * Np * rows);
      CK(cudaMemcpy(buf.data(), e->di[layer].p, buf.size() * 2, cudaMemcpyDeviceToHost));
      auto f = [](uint16_t h) { uint32_t u = uint32_t(h) << 16; float x; std::memcpy(&x, &u, 4); return x; };
      float* out = static_cast<float*>(host);
      for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
          for (int n = 0; n < W; ++n) {
            const size_t r = size_t(b) * T_pad + t;
            const float hi = f(buf[size_t(n) * rows + r]), mi = f(buf[(size_t(Np) + n) * rows + r]),
                        lo = f(buf[(size_t(2) * Np + n) * rows + r]);
            out[(size_t(b) * T + t) * W + n] = hi + (mi + lo);
          }
      return;
    }
    if (layer < 0 || layer >= e->L) fail(SNN_ERR_ARGUMENT, "layer %d", layer);
    const int H = e->H[layer], Hp = e->H_pad[layer];
    const size_t elem = which == 2 ? 1 : 4;
    const size_t need = size_t(B) * T * H * elem;
    if (bytes != need) fail(SNN_ERR_SHAPE, "need %zu bytes", need);
    const size_t rows = size_t(B) * T_pad;
    if (which == 6 && !e->alif(layer)) fail(SNN_ERR_ARGUMENT, "layer %d is not an ALIF cell", layer);
    if (which == 0 || which == 1 || which == 4 || which == 6) {
      std::vector<float> buf(rows * Hp);
      const bool rl = e->rlif(layer);  // RLIF: the projection / dS buffers of the step itself
      const float* src = which == 0 ? (rl ? e->Ibuf[layer].p : e->dbg_i[layer].p)
                         : which == 1 ? e->V[layer].p
                         : which == 6 ? e->Aad[layer].p : (rl ? e->dsbuf[layer].p : e->dbg_ds[layer].p);
      CK(cudaMemcpy(buf.data(), src, buf.size() * 4, cudaMemcpyDeviceToHost));
      float* out = static_cast<float*>(host);
      for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
          std::memcpy(out + (size_t(b) * T + t) * H, buf.data() + (size_t(b) * T_pad + t) * Hp,
                      size_t(H) * 4);
    } else if (which == 2) {
      const int hw = Hp / 32;
      std::vector<uint32_t> buf(rows * hw);
      CK(cudaMemcpy(buf.data(), e->s_np[layer].p, buf.size() * 4, cudaMemcpyDeviceToHost));
      uint8_t* out = static_cast<uint8_t*>(host);
      for (int b = 0; b < B; ++b)
        for (int t = 0; t < T; ++t)
          for (int n = 0; n < H; ++n)
            out[(size_t(b) * T + t) * H + n] =
                (buf[(size_t(b) * T_pad + t) * hw + n / 32] >> (n % 32)) & 1u;
    } else {
      fail(SNN_ERR_ARGUMENT, "unknown debug tensor %d", which);
    }
  });
}

}  // extern "C"
