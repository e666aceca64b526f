// kernels.cuh -- sm_100a kernels of one SNN training step.
//
// Reference semantics (all paths relative to /root/reference/proj/include/spiketrain):
//   forward LIF   neuron.hpp:127-136 (lif_step_taped), network.hpp:384-398
//   readout LI    neuron.hpp:139-144, network.hpp:399-414
//   loss          objective.hpp:40-73, :88-114 (integral CE), :118-134 (accuracy)
//   backward      autodiff.hpp:52-78 reverse sweep; closed recurrences SURVEY.md App. A.2/A.3
//   Adam          optimize.hpp:86-111
//
// Layout conventions (one rank, B local samples, time padded to T_pad):
//   dataset      u8  [N][T_pad/8][IN_pad]        MSB-first time bits (data.hpp:83-126)
//   V_l          f32 [B][T_pad][H_pad]           membrane entering step t
//   S_np_l       u32 [B][T_pad][H_pad/32]        spikes, neuron-packed (bit i = neuron 32w+i)
//   S_tp_l       u32 [H_pad][B*T_pad/32]         spikes, time-packed  (bit e = step 32w+e)
//   dI_l planes  bf16[3][B*T_pad][H_pad]         dL/dI split hi/mid/lo (sum == f32 value)
//   Wt_j planes  bf16[3][N_pad][K_pad]           W_j^T split (forward A operand, K-major)
//   Wb_j planes  bf16[3][K_pad][N_pad]           W_j   split (backward A operand, K-major)
// Tensor-core GEMMs put NEURONS on TMEM lanes and TIME on TMEM columns, so the
// scan epilogue reads its own neuron's time series with tcgen05.ld 32x32b and
// needs no transpose.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

#include "sm100.cuh"

namespace snn {

using namespace sm100;

constexpr int kMaxClasses = 32;

// ------------------------------------------------------------ small helpers
// clip(beta,0,1) = std::min(1, std::max(0, beta)) exactly (ops.hpp clip).
__device__ __forceinline__ float clip01(float b) {
  const float lo = 0.0f < b ? b : 0.0f;
  return lo < 1.0f ? lo : 1.0f;
}

// Surrogate derivative g(x) in float, operation order of surrogate.hpp:59-120.
__device__ __forceinline__ float surrogate(int act, float k, float aux, float x) {
  switch (act) {
    case 1: {  // superspike
      const float d = __fadd_rn(1.0f, __fmul_rn(k, fabsf(x)));
      return __fdiv_rn(1.0f, __fmul_rn(d, d));
    }
    case 2: {  // triangular
      const float r = __fsub_rn(1.0f, fabsf(__fmul_rn(k, x)));
      return 0.0f < r ? r : 0.0f;
    }
    case 3: {  // arctan: u = pi*k*x/2
      const float u = __fdiv_rn(__fmul_rn(__fmul_rn(3.14159265358979f, k), x), 2.0f);
      return __fdiv_rn(1.0f, __fadd_rn(1.0f, __fmul_rn(u, u)));
    }
    case 4:  // boxcar (width = k, height = aux)
      return fabsf(x) <= __fdiv_rn(k, 2.0f) ? aux : 0.0f;
    default:  // custom straight-through
      return 1.0f;
  }
}

// 8 bytes each 0/1 (byte e = element e) -> 8 bf16 {0,1} packed into 4 u32.
__device__ __forceinline__ uint4 expand_bytes01(uint64_t m) {
  uint4 r;
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    w[i] = (uint32_t((m >> (16 * i)) & 1u) * 0x3F80u) |
           (uint32_t((m >> (16 * i + 8)) & 1u) * 0x3F800000u);
  r.x = w[0]; r.y = w[1]; r.z = w[2]; r.w = w[3];
  return r;
}
// 8 bits (bit e = element e) -> 8 bf16.
__device__ __forceinline__ uint4 expand_bits_lsb(uint32_t byte) {
  uint4 r;
  r.x = ((byte >> 0) & 1u) * 0x3F80u | ((byte >> 1) & 1u) * 0x3F800000u;
  r.y = ((byte >> 2) & 1u) * 0x3F80u | ((byte >> 3) & 1u) * 0x3F800000u;
  r.z = ((byte >> 4) & 1u) * 0x3F80u | ((byte >> 5) & 1u) * 0x3F800000u;
  r.w = ((byte >> 6) & 1u) * 0x3F80u | ((byte >> 7) & 1u) * 0x3F800000u;
  return r;
}
// 8 bits MSB-first (bit 7-e = element e) -> 8 bf16 (dataset time bits).
__device__ __forceinline__ uint4 expand_bits_msb(uint32_t byte) {
  return expand_bits_lsb(__brev(byte) >> 24);
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// Split an f32 into three bf16 planes whose exact sum reproduces it (to ~2^-24 rel).
__device__ __forceinline__ void split3(float x, __nv_bfloat16& h, __nv_bfloat16& m,
                                       __nv_bfloat16& l) {
  h = __float2bfloat16_rn(x);
  const float r1 = __fsub_rn(x, __bfloat162float(h));
  m = __float2bfloat16_rn(r1);
  const float r2 = __fsub_rn(r1, __bfloat162float(m));
  l = __float2bfloat16_rn(r2);
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ============================================================================
// K1  k_lif_fwd: I^T[n][t] = sum_k Wt[n][k] * A[t][k] on tcgen05 (3 bf16 planes
// of W, binary A exact in bf16), then the LIF scan epilogue straight from TMEM.
// grid (B, H_pad/128); block 320: w0-3 scan, w4-7 B-operand decode, w8 TMA, w9 MMA.
// ============================================================================
struct FwdArgs {
  const uint8_t* x;       // staged dataset (layer 0)
  const uint32_t* rows;   // [B] dataset row per sample (layer 0)
  const uint32_t* s_in;   // neuron-packed spikes of the previous layer (layer > 0)
  const float* beta;      // [H]
  const float* bias;      // [H] or nullptr
  float* v_out;           // [B][T_pad][H_pad]
  uint32_t* s_np;         // [B][T_pad][H_pad/32]
  uint32_t* s_tp;         // [H_pad][B*T_pad/32]
  float* dbg_i;           // optional [B][T_pad][H_pad] raw projection
  int B, T, T_pad, TT, NT, K_pad, H, H_pad, in_kind;
  float theta;
};

constexpr int kFwdStages = 3;
constexpr int kFwdThreads = 320;
constexpr uint32_t kPlaneTile = 128 * 128;  // 128 rows x 64 bf16 = 16 KB

__host__ __device__ constexpr uint32_t fwd_stage_bytes(int TT) {
  return 3 * kPlaneTile + uint32_t(TT) * 128u;
}
__host__ __device__ constexpr uint32_t fwd_smem_bytes(int TT) {
  return kFwdStages * fwd_stage_bytes(TT) + 1024 + 256;
}

__global__ void __launch_bounds__(kFwdThreads, 1)
    k_lif_fwd(const __grid_constant__ CUtensorMap tm_w, FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const uint32_t stage_bytes = fwd_stage_bytes(a.TT);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kFwdStages * stage_bytes);
  uint64_t* empty = full + kFwdStages;
  uint64_t* acc_full = empty + kFwdStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x, nt = blockIdx.y;
  const int KB = a.K_pad / 64;
  const int total = a.NT * KB;
  const uint32_t tmem_cols = (a.TT >= 128) ? 256u : 128u;  // 2 accumulator buffers

  if (threadIdx.x == 0) {
    for (int s = 0; s < kFwdStages; ++s) {
      mbar_init(&full[s], 1 + 128);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 0) {
    if (tmem_cols == 256) tmem_alloc<256>(tmem_slot); else tmem_alloc<128>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ---------------- TMA producer: the three W^T planes of each k-block
    if (elect_one()) {
      tma_prefetch(&tm_w);
      for (int it = 0; it < total; ++it) {
        const int s = it % kFwdStages, ph = (it / kFwdStages) & 1, kb = it % KB;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], 3 * kPlaneTile);
        uint8_t* A = smem + s * stage_bytes;
        for (int p = 0; p < 3; ++p)
          tma_load_2d(A + p * kPlaneTile, &tm_w, &full[s], kb * 64, p * a.H_pad + nt * 128);
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    // ---------------- MMA issuer (one thread)
    const uint32_t idesc = idesc_bf16(128, a.TT, false, false);
    if (elect_one()) {
      for (int it = 0; it < total; ++it) {
        const int s = it % kFwdStages, ph = (it / kFwdStages) & 1;
        const int tt = it / KB, kb = it % KB, buf = tt & 1;
        if (kb == 0 && tt >= 2) {
          mbar_wait(&acc_empty[buf], ((tt - 2) >> 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t A = smem_u32(smem + s * stage_bytes);
        const uint32_t Bt = A + 3 * kPlaneTile;
        const uint32_t d = tmem + buf * a.TT;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t bd = sdesc_sw128(Bt + ks * 32, 16, 1024);
#pragma unroll
          for (int p = 2; p >= 0; --p) {
            const uint64_t ad = sdesc_sw128(A + p * kPlaneTile + ks * 32, 16, 1024);
            umma_bf16(d, ad, bd, idesc, (kb | ks | (2 - p)) != 0);
          }
        }
        umma_commit(&empty[s]);
        if (kb == KB - 1) umma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------- B-operand producers: activations -> bf16 {0,1} rows t, cols k
    const int tid = threadIdx.x - 128;
    const size_t kwords = size_t(a.K_pad) / 32;
    for (int it = 0; it < total; ++it) {
      const int s = it % kFwdStages, ph = (it / kFwdStages) & 1;
      const int tt = it / KB, kb = it % KB;
      mbar_wait(&empty[s], ph ^ 1);
      const uint32_t Bt = smem_u32(smem + s * stage_bytes + 3 * kPlaneTile);
      if (a.in_kind == 0) {
        // dataset bytes: [row][t/8][k], bit 7-(t%8); one u64 = 8 k of one t-group
        const size_t row = a.rows[b];
        const int groups = a.TT / 8;
        for (int u = tid; u < groups * 8; u += 128) {
          const int g = u >> 3, q = u & 7;
          const uint64_t w = *reinterpret_cast<const uint64_t*>(
              a.x + (row * (a.T_pad / 8) + tt * (a.TT / 8) + g) * size_t(a.K_pad) + kb * 64 + q * 8);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_shared_v4(Bt + sw128_off(8 * g + j, q),
                         expand_bytes01((w >> (7 - j)) & 0x0101010101010101ull));
        }
      } else {
        // neuron-packed spike words: row t, 2 words = 64 k
        for (int u = tid; u < a.TT * 8; u += 128) {
          const int r = u >> 3, q = u & 7;
          const uint32_t* src =
              a.s_in + (size_t(b) * a.T_pad + tt * a.TT + r) * kwords + kb * 2;
          const uint32_t word = src[q >> 2];
          st_shared_v4(Bt + sw128_off(r, q), expand_bits_lsb((word >> (8 * (q & 3))) & 0xFFu));
        }
      }
      fence_async_smem();
      mbar_arrive(&full[s]);
    }
  } else {
    // ---------------- LIF scan epilogue: thread = neuron (TMEM lane)
    const int n = nt * 128 + warp * 32 + lane;
    const float vb = clip01(n < a.H ? a.beta[n] : 0.0f);
    const float bn = (a.bias != nullptr && n < a.H) ? a.bias[n] : 0.0f;
    const float theta = a.theta, ntheta = -a.theta;
    const size_t hw = size_t(a.H_pad) / 32;
    const size_t tp_words = size_t(a.B) * a.T_pad / 32;
    float v = 0.0f;
    for (int tt = 0; tt < a.NT; ++tt) {
      const int buf = tt & 1;
      mbar_wait(&acc_full[buf], (tt >> 1) & 1);
      tc_fence_after();
      for (int c = 0; c < a.TT / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + buf * a.TT + c * 32, r);
        tmem_ld_wait();
        const int t0 = tt * a.TT + c * 32;
        uint32_t myword = 0, tmask = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int t = t0 + j;
          const bool valid = t < a.T;
          float I = __uint_as_float(r[j]);
          if (a.bias != nullptr) I = __fadd_rn(I, bn);
          const size_t vi = (size_t(b) * a.T_pad + t) * a.H_pad + n;
          if (valid) {
            a.v_out[vi] = v;
            if (a.dbg_i != nullptr) a.dbg_i[vi] = I;
          }
          const float pre = __fadd_rn(v, ntheta);
          const bool sp = valid && (pre >= 0.0f);
          const float m = __fmul_rn(v, vb);
          const float ai = __fadd_rn(m, I);
          const float rr = __fmul_rn(sp ? 1.0f : 0.0f, theta);
          v = __fsub_rn(ai, rr);
          const uint32_t bal = __ballot_sync(0xffffffffu, sp);
          if (lane == j) myword = bal;
          tmask |= uint32_t(sp) << j;
        }
        a.s_np[(size_t(b) * a.T_pad + t0 + lane) * hw + nt * 4 + warp] = myword;
        a.s_tp[size_t(n) * tp_words + size_t(b) * (a.T_pad / 32) + t0 / 32] = tmask;
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
  }

  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (tmem_cols == 256) tmem_dealloc<256>(tmem); else tmem_dealloc<128>(tmem);
  }
}

// ============================================================================
// K4  k_readout: readout projection (exact sparse gather in the reference's
// ascending-k order, ops.hpp:163-172), LI scan, integral CE + accuracy, CE
// backward and the closed-form LI reverse scan (App. A.3).  grid B, block 128.
// ============================================================================
struct ReadoutArgs {
  const uint32_t* s_in;     // neuron-packed spikes of the last hidden layer
  const uint32_t* rows;     // [B]
  const int32_t* labels;    // dataset labels [N]
  const float* w;           // readout W [HL][C] f32 (master)
  const float* bias;        // [C] or nullptr
  const float* beta;        // [C]
  float* d3;                // dL/dI3 f32 [B][T_pad][C]
  __nv_bfloat16* d3_planes; // [3][B*T_pad][64]
  float* loss_b;            // [B] lse - logit_y
  int32_t* correct_b;       // [B]
  float* dbeta_part;        // [B][C]
  float* dbias_part;        // [B][C] or nullptr
  float* dbg_trace;         // optional [B][T][C]
  int B, T, T_pad, HL, HL_pad, C;
  float inv_b;              // 1/B_global (objective.hpp:104)
};

__device__ __forceinline__ float exp_cr(float x) { return float(exp(double(x))); }
__device__ __forceinline__ float log_cr(float x) { return float(log(double(x))); }

__global__ void __launch_bounds__(128) k_readout(ReadoutArgs a) {
  extern __shared__ float rsm[];
  float* w = rsm;                        // [HL][C]
  float* buf = w + size_t(a.HL) * a.C;   // [T][C]: I3 -> V3 (entering state) -> dI3
  __shared__ float logits[kMaxClasses];
  const int b = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = a.C;
  for (int i = tid; i < a.HL * C; i += 128) w[i] = a.w[i];
  __syncthreads();
  const size_t hw = size_t(a.HL_pad) / 32;
  // projection: warp w handles t = w, w+4, ...; lane c accumulates class c
  for (int t = warp; t < a.T; t += 4) {
    const uint32_t* srow = a.s_in + (size_t(b) * a.T_pad + t) * hw;
    float acc = 0.0f;
    for (size_t wi = 0; wi < hw; ++wi) {
      uint32_t bits = srow[wi];
      while (bits) {
        const int i = __ffs(bits) - 1;
        bits &= bits - 1;
        const int k = int(wi) * 32 + i;
        if (lane < C) acc = __fadd_rn(acc, w[k * C + lane]);
      }
    }
    if (lane < C) {
      if (a.bias != nullptr) acc = __fadd_rn(acc, a.bias[lane]);
      buf[t * C + lane] = acc;
    }
  }
  __syncthreads();
  if (warp == 0) {
    const bool on = lane < C;
    const float vb = on ? clip01(a.beta[lane]) : 0.0f;
    float v = 0.0f, logit = 0.0f;
    for (int t = 0; t < a.T; ++t) {
      float I = on ? buf[t * C + lane] : 0.0f;
      if (on) buf[t * C + lane] = v;  // keep V3 (entering state) for dbeta
      v = __fadd_rn(__fmul_rn(v, vb), I);
      logit = __fadd_rn(logit, v);
      if (on && a.dbg_trace != nullptr) a.dbg_trace[(size_t(b) * a.T + t) * C + lane] = v;
    }
    if (on) logits[lane] = logit;
    __syncwarp();
    // softmax CE in the reference's sequential order (objective.hpp:53-73)
    float mx = logits[0];
    for (int j = 1; j < C; ++j) mx = (mx < logits[j]) ? logits[j] : mx;
    float z = 0.0f;
    for (int j = 0; j < C; ++j) z = __fadd_rn(z, exp_cr(__fsub_rn(logits[j], mx)));
    const int y = a.labels[a.rows[b]];
    if (lane == 0) {
      const float lse = __fadd_rn(mx, log_cr(z));
      a.loss_b[b] = __fsub_rn(lse, logits[y]);
      int best = 0;
      for (int j = 1; j < C; ++j)
        if (logits[j] > logits[best]) best = j;
      a.correct_b[b] = (best == y) ? 1 : 0;
    }
    float delta = 0.0f;
    if (on) {
      float d = __fdiv_rn(exp_cr(__fsub_rn(logit, mx)), z);
      if (lane == y) d = __fsub_rn(d, 1.0f);
      delta = __fmul_rn(d, a.inv_b);
    }
    // LI reverse scan: G_t = delta + G_{t+1} * bc ; dI3_t = G_t ; dbeta += G_t * V3_t
    float G = 0.0f, db = 0.0f, dbias = 0.0f;
    for (int t = a.T - 1; t >= 0; --t) {
      G = (t == a.T - 1) ? delta : __fadd_rn(delta, __fmul_rn(G, vb));
      if (on) {
        db = __fadd_rn(db, __fmul_rn(G, buf[t * C + lane]));
        dbias = __fadd_rn(dbias, G);
        const size_t row = size_t(b) * a.T_pad + t;
        a.d3[row * C + lane] = G;
        __nv_bfloat16 h, m, l;
        split3(G, h, m, l);
        const size_t plane = size_t(a.B) * a.T_pad * 64;
        a.d3_planes[row * 64 + lane] = h;
        a.d3_planes[plane + row * 64 + lane] = m;
        a.d3_planes[2 * plane + row * 64 + lane] = l;
      }
    }
    if (on) {
      a.dbeta_part[size_t(b) * C + lane] = db;
      if (a.dbias_part != nullptr) a.dbias_part[size_t(b) * C + lane] = dbias;
    }
  }
}

// ============================================================================
// K3  LIF reverse scan (App. A.2):
//   dI_t = G ; ds = dS_t - theta*G ; G = bc*G + g(V_t - theta)*ds ; dbeta += G_{t+1} V_t
// Variant "ro": dS comes from the readout, dS_t[n] = sum_c dI3[t][c] W3[n][c]
// computed here in the reference's order (matmul_nt, ops.hpp:178-199).
// Variant "gemm": dS^T[n][t] = sum_k W[n][k] dI_next[t][k] on tcgen05 (6 plane
// products), scan epilogue from TMEM.
// ============================================================================
struct BwdArgs {
  const float* v_in;           // V_l [B][T_pad][H_pad]
  const float* beta;           // [H]
  const float* d3;             // ro: dI3 [B][T_pad][C]
  const float* w3;             // ro: W3 [H][C]
  __nv_bfloat16* di_planes;    // out: dI_l planes [3][B*T_pad][H_pad]
  float* dbeta_part;           // [B][H]
  float* dbias_part;           // [B][H] or nullptr
  float* dbg_ds;               // optional [B][T_pad][H_pad]
  int B, T, T_pad, TT, NT, K_pad, H, H_pad, C, act;
  float theta, slope, aux;
};

struct ScanState {
  float G, db, dbias;
};

__device__ __forceinline__ void bwd_step(const BwdArgs& a, ScanState& st, float vb, int b, int n,
                                         int t, float dS) {
  const size_t vi = (size_t(b) * a.T_pad + t) * a.H_pad + n;
  const float V = a.v_in[vi];
  if (a.dbg_ds != nullptr) a.dbg_ds[vi] = dS;
  const float G = st.G;
  // dI_t = G (grad of the step-t input); three bf16 planes
  __nv_bfloat16 h, m, l;
  split3(G, h, m, l);
  const size_t plane = size_t(a.B) * a.T_pad * a.H_pad;
  a.di_planes[vi] = h;
  a.di_planes[plane + vi] = m;
  a.di_planes[2 * plane + vi] = l;
  st.dbias = __fadd_rn(st.dbias, G);
  st.db = __fadd_rn(st.db, __fmul_rn(G, V));
  const float rg = -G;
  const float gs = __fadd_rn(dS, __fmul_rn(rg, a.theta));
  const float pre = __fadd_rn(V, -a.theta);
  const float gpre = __fmul_rn(gs, surrogate(a.act, a.slope, a.aux, pre));
  st.G = __fadd_rn(__fmul_rn(G, vb), gpre);
}

__global__ void __launch_bounds__(128) k_lif_bwd_ro(BwdArgs a) {
  const int b = blockIdx.x, n = blockIdx.y * 128 + threadIdx.x;
  const float vb = clip01(n < a.H ? a.beta[n] : 0.0f);
  float w[kMaxClasses];
#pragma unroll
  for (int c = 0; c < kMaxClasses; ++c) w[c] = (n < a.H && c < a.C) ? a.w3[n * a.C + c] : 0.0f;
  ScanState st{0.0f, 0.0f, 0.0f};
  for (int t = a.T - 1; t >= 0; --t) {
    const float* g = a.d3 + (size_t(b) * a.T_pad + t) * a.C;
    float dS = 0.0f;
#pragma unroll
    for (int c = 0; c < kMaxClasses; ++c)
      if (c < a.C) dS = __fadd_rn(dS, __fmul_rn(g[c], w[c]));
    bwd_step(a, st, vb, b, n, t, dS);
  }
  if (n < a.H) {
    a.dbeta_part[size_t(b) * a.H + n] = st.db;
    if (a.dbias_part != nullptr) a.dbias_part[size_t(b) * a.H + n] = st.dbias;
  }
}

constexpr int kBwdStages = 2;
constexpr int kBwdThreads = 192;  // w0-3 scan, w4 TMA, w5 MMA
__host__ __device__ constexpr uint32_t bwd_stage_bytes(int TT) {
  return 3 * kPlaneTile + 3 * uint32_t(TT) * 128u;
}
__host__ __device__ constexpr uint32_t bwd_smem_bytes(int TT) {
  return kBwdStages * bwd_stage_bytes(TT) + 1024 + 256;
}

__global__ void __launch_bounds__(kBwdThreads, 1)
    k_lif_bwd_gemm(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_di,
                   BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const uint32_t stage_bytes = bwd_stage_bytes(a.TT);
  const uint32_t btile = uint32_t(a.TT) * 128u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBwdStages * stage_bytes);
  uint64_t* empty = full + kBwdStages;
  uint64_t* acc_full = empty + kBwdStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x, nt = blockIdx.y;
  const int KB = a.K_pad / 64;
  const int total = a.NT * KB;
  const uint32_t tmem_cols = (a.TT >= 128) ? 256u : 128u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kBwdStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 0) {
    if (tmem_cols == 256) tmem_alloc<256>(tmem_slot); else tmem_alloc<128>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int rows_total = a.B * a.T_pad;

  if (warp == 4) {
    if (elect_one()) {
      tma_prefetch(&tm_w);
      tma_prefetch(&tm_di);
      for (int it = 0; it < total; ++it) {
        const int s = it % kBwdStages, ph = (it / kBwdStages) & 1;
        const int tt = a.NT - 1 - it / KB, kb = it % KB;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], 3 * kPlaneTile + 3 * btile);
        uint8_t* A = smem + s * stage_bytes;
        uint8_t* Bt = A + 3 * kPlaneTile;
        for (int p = 0; p < 3; ++p) {
          tma_load_2d(A + p * kPlaneTile, &tm_w, &full[s], kb * 64, p * a.H_pad + nt * 128);
          tma_load_2d(Bt + p * btile, &tm_di, &full[s], kb * 64,
                      p * rows_total + b * a.T_pad + tt * a.TT);
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    const uint32_t idesc = idesc_bf16(128, a.TT, false, false);
    if (elect_one()) {
      for (int it = 0; it < total; ++it) {
        const int s = it % kBwdStages, ph = (it / kBwdStages) & 1;
        const int j = it / KB, kb = it % KB, buf = j & 1;
        if (kb == 0 && j >= 2) {
          mbar_wait(&acc_empty[buf], ((j - 2) >> 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t A = smem_u32(smem + s * stage_bytes);
        const uint32_t Bt = A + 3 * kPlaneTile;
        const uint32_t d = tmem + buf * a.TT;
        // (pa, pb) plane products with pa + pb <= 2, smallest terms first
        const int pa[6] = {2, 1, 0, 1, 0, 0};
        const int pb[6] = {0, 1, 2, 0, 1, 0};
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const uint64_t ad = sdesc_sw128(A + pa[q] * kPlaneTile + ks * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(Bt + pb[q] * btile + ks * 32, 16, 1024);
            umma_bf16(d, ad, bd, idesc, (kb | ks | q) != 0);
          }
        }
        umma_commit(&empty[s]);
        if (kb == KB - 1) umma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    const int n = nt * 128 + warp * 32 + lane;
    const float vb = clip01(n < a.H ? a.beta[n] : 0.0f);
    ScanState st{0.0f, 0.0f, 0.0f};
    for (int j = 0; j < a.NT; ++j) {
      const int tt = a.NT - 1 - j, buf = j & 1;
      mbar_wait(&acc_full[buf], (j >> 1) & 1);
      tc_fence_after();
      for (int c = a.TT / 32 - 1; c >= 0; --c) {
        uint32_t r[32];
        tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + buf * a.TT + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 31; e >= 0; --e) {
          const int t = tt * a.TT + c * 32 + e;
          if (t < a.T) bwd_step(a, st, vb, b, n, t, __uint_as_float(r[e]));
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
    if (n < a.H) {
      a.dbeta_part[size_t(b) * a.H + n] = st.db;
      if (a.dbias_part != nullptr) a.dbias_part[size_t(b) * a.H + n] = st.dbias;
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (tmem_cols == 256) tmem_dealloc<256>(tmem); else tmem_dealloc<128>(tmem);
  }
}

// ============================================================================
// K5  k_wgrad: partial[s][k][n] = sum_{rows in split s} A[k][row] * dI[row][n]
// A binary (dataset time bits or time-packed spikes), exact in bf16 (K-major,
// decoded by warps 0-3); dI as 3 bf16 planes via TMA (MN-major).  Epilogue
// writes f32 partials; k_reduce sums them in fixed order (deterministic).
// grid (M_pad/128, N_pad/N_TILE, splits); block 192.
// ============================================================================
struct WgradArgs {
  const uint8_t* x;        // kind 0: staged dataset
  const uint32_t* rows;    // kind 0: [B]
  const uint32_t* s_tp;    // kind 1: time-packed spikes [K_pad][B*T_pad/32]
  float* partial;          // [splits][M_pad][N_pad]
  int kind, B, T_pad, M_pad, N_pad, n_tile, splits, x_row_stride;
};

constexpr int kWgStages = 3;
constexpr int kWgThreads = 192;
__host__ __device__ constexpr uint32_t wg_stage_bytes(int n_tile) {
  return kPlaneTile + 3 * uint32_t(n_tile) * 128u;  // A 16 KB + 3 planes x (n/64 boxes x 8 KB)
}
__host__ __device__ constexpr uint32_t wg_smem_bytes(int n_tile) {
  return kWgStages * wg_stage_bytes(n_tile) + 1024 + 256;
}

__global__ void __launch_bounds__(kWgThreads, 1)
    k_wgrad(const __grid_constant__ CUtensorMap tm_di, WgradArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const uint32_t stage_bytes = wg_stage_bytes(a.n_tile);
  const uint32_t ptile = uint32_t(a.n_tile) * 128u;  // one plane: 64 rows x n_tile cols
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kWgStages * stage_bytes);
  uint64_t* empty = full + kWgStages;
  uint64_t* acc_full = empty + kWgStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, ntile = blockIdx.y, split = blockIdx.z;
  const int tq_per_b = a.T_pad / 64;
  const int b0 = int((long long)a.B * split / a.splits);
  const int b1 = int((long long)a.B * (split + 1) / a.splits);
  const int total = (b1 - b0) * tq_per_b;
  const uint32_t tmem_cols = a.n_tile <= 32 ? 32u : (a.n_tile <= 64 ? 64u : (a.n_tile <= 128 ? 128u : 256u));

  if (threadIdx.x == 0) {
    for (int s = 0; s < kWgStages; ++s) {
      mbar_init(&full[s], 1 + 128);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&acc_full[0], 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    switch (tmem_cols) {
      case 32: tmem_alloc<32>(tmem_slot); break;
      case 64: tmem_alloc<64>(tmem_slot); break;
      case 128: tmem_alloc<128>(tmem_slot); break;
      default: tmem_alloc<256>(tmem_slot); break;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int rows_total = a.B * a.T_pad;

  if (warp == 4) {
    if (elect_one()) {
      tma_prefetch(&tm_di);
      for (int it = 0; it < total; ++it) {
        const int s = it % kWgStages, ph = (it / kWgStages) & 1;
        const int bb = b0 + it / tq_per_b, tq = it % tq_per_b;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], 3 * ptile);
        uint8_t* Bp = smem + s * stage_bytes + kPlaneTile;
        for (int p = 0; p < 3; ++p)
          for (int h = 0; h < a.n_tile / 64; ++h)
            tma_load_2d(Bp + p * ptile + h * 8192, &tm_di, &full[s], ntile * a.n_tile + h * 64,
                        p * rows_total + bb * a.T_pad + tq * 64);
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    const uint32_t idesc = idesc_bf16(128, a.n_tile, false, true);
    if (elect_one()) {
      for (int it = 0; it < total; ++it) {
        const int s = it % kWgStages, ph = (it / kWgStages) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t A = smem_u32(smem + s * stage_bytes);
        const uint32_t Bp = A + kPlaneTile;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t ad = sdesc_sw128(A + ks * 32, 16, 1024);
#pragma unroll
          for (int p = 2; p >= 0; --p) {
            const uint64_t bd = sdesc_sw128(Bp + p * ptile + ks * 2048, 8192, 1024);
            umma_bf16(tmem, ad, bd, idesc, (it | ks | (2 - p)) != 0);
          }
        }
        umma_commit(&empty[s]);
      }
      umma_commit(&acc_full[0]);
    }
    __syncwarp();
  } else if (warp < 4) {
    // A producers: tile [128 k-rows][64 time cols], K-major SW128
    const int tid = threadIdx.x;
    const int k = mt * 128 + tid;  // this thread's A row
    for (int it = 0; it < total; ++it) {
      const int s = it % kWgStages, ph = (it / kWgStages) & 1;
      const int bb = b0 + it / tq_per_b, tq = it % tq_per_b;
      mbar_wait(&empty[s], ph ^ 1);
      const uint32_t A = smem_u32(smem + s * stage_bytes);
      if (a.kind == 0) {
        const uint8_t* src = a.x + (size_t(a.rows[bb]) * (a.T_pad / 8) + tq * 8) * a.x_row_stride + k;
        const bool in_row = k < a.x_row_stride;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          st_shared_v4(A + sw128_off(tid, j),
                       expand_bits_msb(in_row ? src[size_t(j) * a.x_row_stride] : 0u));
      } else {
        const uint64_t w = *reinterpret_cast<const uint64_t*>(
            a.s_tp + size_t(k) * (size_t(a.B) * a.T_pad / 32) + size_t(bb) * (a.T_pad / 32) + tq * 2);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          st_shared_v4(A + sw128_off(tid, j), expand_bits_lsb(uint32_t(w >> (8 * j)) & 0xFFu));
      }
      fence_async_smem();
      mbar_arrive(&full[s]);
    }
    // epilogue: thread = output row k, n_tile columns
    mbar_wait(&acc_full[0], 0);
    tc_fence_after();
    float* dst = a.partial + (size_t(split) * a.M_pad + k) * a.N_pad + ntile * a.n_tile;
    for (int c = 0; c < a.n_tile / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + c * 32, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 v4 = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        if (total == 0) v4 = make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(dst + c * 32 + j) = v4;
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    switch (tmem_cols) {
      case 32: tmem_dealloc<32>(tmem); break;
      case 64: tmem_dealloc<64>(tmem); break;
      case 128: tmem_dealloc<128>(tmem); break;
      default: tmem_dealloc<256>(tmem); break;
    }
  }
}

// ============================================================================
// K6  gradient assembly, Adam and operand-plane refresh.
// One thread per flat parameter in NetworkParams order (network.hpp:164-226).
// ============================================================================
enum EntryKind : int32_t { kEntryW = 0, kEntryB = 1, kEntryBeta = 2 };

struct Entry {
  int32_t kind, layer;    // layer = Linear index j (W, b) or cell index (beta)
  int32_t rows, cols;     // W: [K][N]; b/beta: [1][N]
  int64_t offset;         // into the flat vector
};

constexpr int kMaxEntries = 3 * 9;
constexpr int kMaxLayers = 9;

struct ReduceArgs {
  Entry entries[kMaxEntries];
  int n_entries;
  int64_t n_params;
  const float* partial[kMaxLayers];     // wgrad partials per Linear j
  int M_pad[kMaxLayers], N_pad[kMaxLayers], splits[kMaxLayers];
  const float* dbeta_part[kMaxLayers];  // per cell j: [B][N]
  const float* dbias_part[kMaxLayers];  // per Linear j: [B][N]
  const float* params;                  // for the clip mask
  float* grads;
  int B;
};

__global__ void k_reduce(ReduceArgs a) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= a.n_params) return;
  int e = 0;
  while (e + 1 < a.n_entries && a.entries[e + 1].offset <= i) ++e;
  const Entry en = a.entries[e];
  const int64_t li = i - en.offset;
  const int j = en.layer;
  float g = 0.0f;
  if (en.kind == kEntryW) {
    const int64_t k = li / en.cols, n = li % en.cols;
    const float* p = a.partial[j] + k * a.N_pad[j] + n;
    const int64_t sstride = int64_t(a.M_pad[j]) * a.N_pad[j];
    for (int s = 0; s < a.splits[j]; ++s) g = __fadd_rn(g, p[s * sstride]);
  } else if (en.kind == kEntryB) {
    for (int b = 0; b < a.B; ++b) g = __fadd_rn(g, a.dbias_part[j][int64_t(b) * en.cols + li]);
  } else {
    for (int b = 0; b < a.B; ++b) g = __fadd_rn(g, a.dbeta_part[j][int64_t(b) * en.cols + li]);
    const float beta = a.params[i];
    if (!(beta > 0.0f && beta < 1.0f)) g = 0.0f;  // clip01 gradient (autodiff.hpp:353-355)
  }
  a.grads[i] = g;
}

struct PlaneTarget {
  __nv_bfloat16* wt;  // forward A planes [3][N_pad][K_pad] or nullptr
  __nv_bfloat16* wb;  // backward A planes [3][K_pad][N_pad] or nullptr
  int K_pad, N_pad;
};

struct AdamArgs {
  Entry entries[kMaxEntries];
  int n_entries;
  int64_t n_params;
  PlaneTarget planes[kMaxLayers];  // per Linear j
  float* params;
  float* m;
  float* v;
  const float* grads;
  const float* bc;           // [2 * max_steps]: bc1, bc2 per step (host powf)
  const int64_t* step;       // device step counter (before this update)
  float lr, b1, b2, eps, omb1, omb2;
  int update;                // 0: only refresh planes (after set_params)
};

__global__ void k_adam(AdamArgs a) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= a.n_params) return;
  float p = a.params[i];
  if (a.update) {
    const int64_t s = *a.step;  // steps done so far; this update is s+1
    const float bc1 = a.bc[2 * s], bc2 = a.bc[2 * s + 1];
    const float g = a.grads[i];
    const float m = __fadd_rn(__fmul_rn(a.b1, a.m[i]), __fmul_rn(a.omb1, g));
    const float v = __fadd_rn(__fmul_rn(a.b2, a.v[i]), __fmul_rn(__fmul_rn(a.omb2, g), g));
    const float mhat = __fdiv_rn(m, bc1);
    const float vhat = __fdiv_rn(v, bc2);
    p = __fsub_rn(p, __fdiv_rn(__fmul_rn(a.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), a.eps)));
    a.m[i] = m;
    a.v[i] = v;
    a.params[i] = p;
  }
  int e = 0;
  while (e + 1 < a.n_entries && a.entries[e + 1].offset <= i) ++e;
  const Entry en = a.entries[e];
  if (en.kind != kEntryW) return;
  const PlaneTarget pt = a.planes[en.layer];
  if (pt.wt == nullptr && pt.wb == nullptr) return;
  const int64_t li = i - en.offset;
  const int64_t k = li / en.cols, n = li % en.cols;
  __nv_bfloat16 h, mi, lo;
  split3(p, h, mi, lo);
  if (pt.wt != nullptr) {
    const int64_t plane = int64_t(pt.N_pad) * pt.K_pad, idx = n * pt.K_pad + k;
    pt.wt[idx] = h;
    pt.wt[plane + idx] = mi;
    pt.wt[2 * plane + idx] = lo;
  }
  if (pt.wb != nullptr) {
    const int64_t plane = int64_t(pt.K_pad) * pt.N_pad, idx = k * pt.N_pad + n;
    pt.wb[idx] = h;
    pt.wb[plane + idx] = mi;
    pt.wb[2 * plane + idx] = lo;
  }
}

// ============================================================================
// K0  k_synth: synth_raster(classes, n, T, {f}, seed) + pack_time, generated
// directly into the staged HBM layout (commands.hpp:50-86, data.hpp:105-126).
// SplitMix64 counter draws (rng.hpp:20-64) in integer + fp64 math -> bit-exact.
// One thread per (example, t-group, feature) byte.
// ============================================================================
__device__ __forceinline__ uint64_t d_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct SynthArgs {
  uint8_t* x;        // [n][T_pad/8][f_pad]
  int32_t* labels;   // [n]
  uint64_t master;   // RngKey::from_seed(seed).word
  int64_t n;
  int T, T_pad, f, f_pad, classes;
};

__global__ void k_synth(SynthArgs a) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int groups = a.T_pad / 8;
  const int64_t total = a.n * groups * a.f_pad;
  if (gid >= total) return;
  const int j = int(gid % a.f_pad);
  const int g = int((gid / a.f_pad) % groups);
  const int64_t i = gid / (int64_t(a.f_pad) * groups);
  const int label = int(i % a.classes);
  if (j == 0 && g == 0) a.labels[i] = label;
  uint8_t byte = 0;
  if (j < a.f) {
    const int block = a.f / a.classes > 1 ? a.f / a.classes : 1;
    const int lo = label * block, hi = lo + block < a.f ? lo + block : a.f;
    const double rate = (j >= lo && j < hi) ? 0.4 : 0.05;
    const uint64_t ek = d_mix64(a.master ^ d_mix64(uint64_t(i) + 0xC2B2AE3D27D4EB4Full));
    for (int e = 0; e < 8; ++e) {
      const int s = g * 8 + e;
      if (s >= a.T) break;
      const uint64_t ctr = uint64_t(s) * uint64_t(a.f) + uint64_t(j);
      const uint64_t bits = d_mix64(ek ^ d_mix64(ctr + 0x165667B19E3779F9ull));
      const double u = double(bits >> 11) * 0x1.0p-53;
      if (u < rate) byte |= uint8_t(1u << (7 - e));
    }
  }
  a.x[gid] = byte;
}

// Local loss sum in batch order (objective.hpp:57-72: loss += lse - row[y]) and
// hit count, appended to the gradient buffer so one allreduce carries both.
__global__ void k_loss_partial(const float* loss_b, const int32_t* correct_b, int B,
                               float* tail) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  float loss = 0.0f;
  int hits = 0;
  for (int b = 0; b < B; ++b) {
    loss = __fadd_rn(loss, loss_b[b]);
    hits += correct_b[b];
  }
  tail[0] = loss;
  tail[1] = float(hits);
}

// StepResult{loss / B_global, hits / B_global}; advances the step counter.
__global__ void k_result(const float* tail, int B_global, int64_t* step, int do_step,
                         float* loss_out, double* acc_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  *loss_out = __fdiv_rn(tail[0], float(B_global));
  *acc_out = double(tail[1]) / double(B_global);
  if (do_step) *step += 1;
}

}  // namespace snn
