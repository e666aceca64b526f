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
constexpr int kMaxLayers = 9;  // Linear layers (hidden + readout)
constexpr int kMaxRanks = 8;   // data-parallel ranks of the peer-memory tail (one NVSwitch box)
// debug phase-timestamp record per CTA; [14]/[15] = globaltimer start/end
constexpr int kClkStride = 48;  // [16, 48): per-k-block stamps (forward MMA thread)

// The step's dataset rows: a fixed [B] buffer, or (schedule mode) slot *slot of
// a device-resident schedule [steps][B] whose slot counter the step tail advances.
__device__ __forceinline__ const uint32_t* batch_rows(const uint32_t* rows, const int64_t* slot, int B) {
  return slot != nullptr ? rows + size_t(*slot) * size_t(B) : rows;
}

// ------------------------------------------------------------ small helpers
// clip(beta,0,1) = std::min(1, std::max(0, beta)) exactly (ops.hpp clip).
__device__ __forceinline__ float clip01(float b) {
  const float lo = 0.0f < b ? b : 0.0f;
  return lo < 1.0f ? lo : 1.0f;
}

// 8 bytes each 0/1 (byte e = element e) -> 8 bf16 {0,1} packed into 4 u32.
__device__ __forceinline__ uint4 expand_bytes01(uint64_t m) {
  // bytes are 0/1: x0xFF -> 0x00/0xFF masks (no carries), PRMT duplicates each
  // mask byte into a bf16 half, AND applies 1.0 = 0x3F80
  const uint32_t ml = uint32_t(m) * 0xFFu, mh = uint32_t(m >> 32) * 0xFFu;
  uint4 r;
  r.x = __byte_perm(ml, 0u, 0x1100u) & 0x3F803F80u;
  r.y = __byte_perm(ml, 0u, 0x3322u) & 0x3F803F80u;
  r.z = __byte_perm(mh, 0u, 0x1100u) & 0x3F803F80u;
  r.w = __byte_perm(mh, 0u, 0x3322u) & 0x3F803F80u;
  return r;
}
// 8 bits (bit e = element e) -> 8 bf16 (0 or 1.0).  The multiply spreads bit i
// of a nibble to bit 8i (the four shifted copies do not overlap, so no carries),
// x0xFF turns each byte into a 0x00/0xFF mask, PRMT duplicates mask bytes into
// bf16 halves, AND applies the 1.0 pattern 0x3F80.
__device__ __forceinline__ uint4 expand_bits_lsb(uint32_t byte) {
  const uint32_t ml = (((byte & 0xFu) * 0x00204081u) & 0x01010101u) * 0xFFu;
  const uint32_t mh = ((((byte >> 4) & 0xFu) * 0x00204081u) & 0x01010101u) * 0xFFu;
  uint4 r;
  r.x = __byte_perm(ml, 0u, 0x1100u) & 0x3F803F80u;
  r.y = __byte_perm(ml, 0u, 0x3322u) & 0x3F803F80u;
  r.z = __byte_perm(mh, 0u, 0x1100u) & 0x3F803F80u;
  r.w = __byte_perm(mh, 0u, 0x3322u) & 0x3F803F80u;
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

// Split an f32 into three bf16 planes x = hi + mid + lo + r, |r| <= 2^-23 |x|:
// each plane is the truncated top 16 bits of the running residual, and the
// residual subtractions are exact (same exponent range), so no rounding
// instructions are needed.  *_bits return the raw upper halves.
__device__ __forceinline__ void split3_bits(float x, uint32_t& h, uint32_t& m, uint32_t& l) {
  const uint32_t xb = __float_as_uint(x);
  const float hf = __uint_as_float(xb & 0xFFFF0000u);
  const float r1 = __fsub_rn(x, hf);
  const uint32_t rb = __float_as_uint(r1);
  const float mf = __uint_as_float(rb & 0xFFFF0000u);
  const float r2 = __fsub_rn(r1, mf);
  h = xb >> 16;
  m = rb >> 16;
  l = __float_as_uint(r2) >> 16;
}
__device__ __forceinline__ void split3(float x, __nv_bfloat16& h, __nv_bfloat16& m,
                                       __nv_bfloat16& l) {
  uint32_t hb, mb, lb;
  split3_bits(x, hb, mb, lb);
  h = __ushort_as_bfloat16(uint16_t(hb));
  m = __ushort_as_bfloat16(uint16_t(mb));
  l = __ushort_as_bfloat16(uint16_t(lb));
}
// pack two values' planes: low half = element e, high half = element e+1
__device__ __forceinline__ void split3_pack(float x0, float x1, uint32_t& h, uint32_t& m,
                                            uint32_t& l) {
  uint32_t h0, m0, l0, h1, m1, l1;
  split3_bits(x0, h0, m0, l0);
  split3_bits(x1, h1, m1, l1);
  h = h0 | (h1 << 16);
  m = m0 | (m1 << 16);
  l = l0 | (l1 << 16);
}
__device__ __forceinline__ float rcp_approx(float y) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
  return r;
}

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Surrogate for the backward sweep (surrogate.hpp:59-120), compile-time kind so
// the unrolled step bodies stay branch-free; divisions evaluated as approximate
// reciprocals (<= 1 ulp; the backward is checked to the 1e-4 gradient bound,
// the bit-exact parts are the forward scans).
template <int kAct>
__device__ __forceinline__ float surrogate_t(float k, float aux, float x) {
  if constexpr (kAct == 1) {  // superspike 1/(1+k|x|)^2
    const float d = __fadd_rn(1.0f, __fmul_rn(k, fabsf(x)));
    return rcp_approx(__fmul_rn(d, d));
  } else if constexpr (kAct == 2) {  // triangular max(0, 1-|kx|)
    const float r = __fsub_rn(1.0f, fabsf(__fmul_rn(k, x)));
    return 0.0f < r ? r : 0.0f;
  } else if constexpr (kAct == 3) {  // arctan 1/(1+(pi k x/2)^2)
    const float u = __fmul_rn(k * 1.57079632679489662f, x);
    return rcp_approx(__fadd_rn(1.0f, __fmul_rn(u, u)));
  } else if constexpr (kAct == 4) {  // boxcar
    return fabsf(x) <= __fmul_rn(k, 0.5f) ? aux : 0.0f;
  } else if constexpr (kAct == 5) {
    // sigmoid, DECLARED (not in the reference catalogue): the
    // backward a caller hands to custom(heaviside, bwd), surrogate.hpp:45-57,
    // g = k s (1 - s) = (k e) / ((1 + e)(1 + e)), e = exp(-k |x|): the
    // cancellation-free form of oracle/spiketrain_oracle.h (accurate expf)
    const float e = expf(-__fmul_rn(k, fabsf(x)));
    const float d = __fadd_rn(1.0f, e);
    return __fdiv_rn(__fmul_rn(k, e), __fmul_rn(d, d));
  } else {  // custom straight-through
    return 1.0f;
  }
}

// the surrogate with a runtime kind (the readout's few steps per lane)
__device__ __forceinline__ float surrogate_rt(int act, float k, float aux, float x) {
  switch (act) {
    case 1: return surrogate_t<1>(k, aux, x);
    case 2: return surrogate_t<2>(k, aux, x);
    case 3: return surrogate_t<3>(k, aux, x);
    case 4: return surrogate_t<4>(k, aux, x);
    case 5: return surrogate_t<5>(k, aux, x);
    default: return 1.0f;
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
  const int64_t* rows_slot; // schedule mode: rows += *rows_slot * B (else nullptr)
  const int32_t* labels;    // dataset labels [N]
  const float* w;           // readout W [HL][C] f32 (master)
  const float* bias;        // [C] or nullptr
  const float* beta;        // [C] (or one value: beta_stride 0)
  int beta_stride;
  __nv_bfloat16* d3_planes; // [3][64][B*T_pad] (class rows, (b,t) contiguous)
  float* loss_b;            // [B] lse - logit_y
  int32_t* correct_b;       // [B]
  float* dbeta_part;        // [B][C]
  float* dbias_part;        // [B][C] or nullptr
  float* dbg_trace;         // optional [B][T][C]
  long long* dbg_clk;       // optional [B][8] phase timestamps (clock64)
  int exp_mode;             // 0: exp/log evaluated in fp64 then rounded; 1: expf/logf
  int B, T, T_pad, HL, HL_pad, C;
  float inv_b;              // 1/B_global (objective.hpp:104)
  int loss_kind;            // 0 integral CE, 1 spike-rate MSE (objective.hpp:139-183)
  float rate_hi, rate_lo;   // rate-MSE targets
  float mse_gs;             // 2 / (float(B_global*C) * float(T)) (objective.hpp:172)
  float* loss_terms;        // rate-MSE: [B][C] squared rate gaps (summed in order by the tail)
  // LIF readout (network.hpp:153-155, :396): the trace is the readout's spikes; its
  // threshold and surrogate are the hidden layers' (readout_lif 0: LI readout)
  int readout_lif, act;
  float theta, slope, aux;
};

__device__ __forceinline__ float exp_cr(float x) { return float(exp(double(x))); }
__device__ __forceinline__ float log_cr(float x) { return float(log(double(x))); }

// readout scratch: W [HL][C] | spike words [T][HL_pad/32] | per-(t, class) column
// buffer [T][33] (one column per lane; stride 33 keeps both the per-step rows
// written by the projection and the per-class columns read by the scans free
// of bank conflicts)
constexpr int kRoThreads = 256;  // projection: 2 lanes per time step (class groups split)
// per-(t, class) column buffer row stride: odd (conflict-free for both the projection's
// rows and the scans' columns) and > C, so column C is a scratch column the scan lanes
// >= C share
__host__ __device__ constexpr int readout_row_stride(int C) { return (C + 1) | 1; }
// 4-class groups per lane of the projection's lane pair (template parameter of k_readout)
__host__ __device__ constexpr int readout_groups(int C) { return (C + 7) / 8; }
// W [HL][Cp] (Cp = 8 * groups: rows zero-padded so every lane adds whole float4 groups)
// | [T][row stride] column buffer (the spike words are read from L2)
__host__ __device__ inline size_t readout_smem_bytes(int HL, int HL_pad, int T, int C) {
  return (size_t(HL) * 8 * readout_groups(C) + size_t(T) * readout_row_stride(C)) * 4;
}

// (Running the readout in the tail of the fused forward launch, one group of warps
// per sample, was measured slower: the forward's 448-thread register budget slowed
// every readout phase 1.2-8x.)
// kNG = readout_groups(C): each lane of a pair owns kNG 4-class groups
template <int kNG>
__global__ void __launch_bounds__(kRoThreads) k_readout(ReadoutArgs a) {
  extern __shared__ float rsm[];
  const int C = a.C, T = a.T;
  const int hw = a.HL_pad / 32;
  constexpr int Cp = 8 * kNG;
  const int rs = readout_row_stride(C);
  float* w = rsm;                       // [HL][Cp]
  float* buf = w + size_t(a.HL) * Cp;   // [T][rs]
  // the spike words of this sample (written by the forward kernel; read from L2)
  const uint32_t* spk = a.s_in + size_t(blockIdx.x) * a.T_pad * hw;
  const int b = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int G = kRoThreads;
#define RO_CLK(k) if (a.dbg_clk != nullptr && tid == 0) a.dbg_clk[b * kClkStride + (k)] = clock64();
  // W [HL][C] is a parameter (written by the previous step's update, long complete):
  // staged before the dependency wait, overlapping the forward kernel's tail
  {
    const int nw = a.HL * C;
    if (Cp == C && (reinterpret_cast<uintptr_t>(a.w) & 15) == 0) {
      const float4* __restrict__ src = reinterpret_cast<const float4*>(a.w);
      for (int i = tid; i < nw / 4; i += G) reinterpret_cast<float4*>(w)[i] = __ldg(src + i);
    } else {
      for (int i = tid; i < a.HL * Cp; i += G) {
        const int k = i / Cp, c = i % Cp;
        w[i] = c < C ? __ldg(a.w + k * C + c) : 0.0f;
      }
    }
  }
  const float beta_l = lane < C ? a.beta[lane * a.beta_stride] : 0.0f;
  pdl_wait();
  RO_CLK(0)
  if (a.dbg_clk != nullptr && tid == 0) a.dbg_clk[b * kClkStride + 14] = globaltimer();
  // the first spike-word chunk of this thread's first step, in flight across the label
  // load (hw = HL_pad / 32 is a multiple of 4: whole 16-byte chunks)
  const uint4 pre = (tid >> 1) < T ? __ldg(reinterpret_cast<const uint4*>(spk + (tid >> 1) * hw))
                                   : make_uint4(0u, 0u, 0u, 0u);
  __shared__ int s_label[1];
  if (tid == 0) *s_label = a.labels[batch_rows(a.rows, a.rows_slot, a.B)[b]];
  __syncthreads();
  RO_CLK(1)
  // projection (ops.hpp:163-172 order: ascending k, zero skip): a lane pair per
  // time step, lane h of the pair owning the 4-class groups j = 2jj + h (acc in
  // registers; the pair walks the same spike bits).  W rows live in smem zero-padded
  // to Cp = 8 kNG floats, so every lane adds whole groups with no per-class
  // predicates (the padded classes' sums are never stored); the row of the next
  // spike is loaded while the current one is added (two rows per trip, no register
  // moves), so a burst of spikes costs the add chain, not one smem round trip each.
  constexpr int kGroups = kNG;
  const int h = tid & 1;
  for (int t = tid >> 1; t < T; t += G / 2) {
    float acc[kGroups][4];
#pragma unroll
    for (int jj = 0; jj < kGroups; ++jj) acc[jj][0] = acc[jj][1] = acc[jj][2] = acc[jj][3] = 0.0f;
    // the step's spike words in 16-byte chunks, the next chunk in flight while the
    // current one is walked: one L2 round trip per step, not one per word
    const uint4* words = reinterpret_cast<const uint4*>(spk + t * hw);
    const int nq = hw >> 2;
    uint4 cw = t == (tid >> 1) ? pre : __ldg(words);
    const float4* wbase = reinterpret_cast<const float4*>(w) + h;
    auto load_row = [&](int k, float4 (&r)[kGroups]) {
      const float4* wr = wbase + k * (Cp / 4);
#pragma unroll
      for (int jj = 0; jj < kGroups; ++jj) r[jj] = wr[2 * jj];
    };
    auto add_row = [&](const float4 (&r)[kGroups]) {
#pragma unroll
      for (int jj = 0; jj < kGroups; ++jj) {
        acc[jj][0] = __fadd_rn(acc[jj][0], r[jj].x);
        acc[jj][1] = __fadd_rn(acc[jj][1], r[jj].y);
        acc[jj][2] = __fadd_rn(acc[jj][2], r[jj].z);
        acc[jj][3] = __fadd_rn(acc[jj][3], r[jj].w);
      }
    };
    // ascending k: 16-byte chunks of 4 words (the next chunk in flight), each word's
    // set bits lowest first -- a fixed loop over the words and a plain bit loop per
    // word (a single "next spike" walker across words measured ~200 cycles a spike)
    float4 ra[kGroups];
    for (int q4 = 0; q4 < nq; ++q4) {
      const uint4 nw = q4 + 1 < nq ? __ldg(words + q4 + 1) : make_uint4(0u, 0u, 0u, 0u);
      const uint32_t wv[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        uint32_t bits = wv[s4];
        const int kbase = (q4 * 4 + s4) * 32;
        while (bits != 0u) {
          const int k = kbase + __ffs(bits) - 1;
          bits &= bits - 1u;
          load_row(k, ra);
          add_row(ra);
        }
      }
      cw = nw;
    }
#pragma unroll
    for (int jj = 0; jj < kGroups; ++jj)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = 4 * (2 * jj + h) + e;
        float vout = 0.0f;  // (classes >= C: padded W columns, sums discarded)
        if (c < C) vout = a.bias != nullptr ? __fadd_rn(acc[jj][e], a.bias[c]) : acc[jj][e];
        if (c < rs) buf[t * rs + c] = vout;  // classes >= C (the scratch column) are zero
      }
  }
  if (a.dbg_clk != nullptr && lane == 0) a.dbg_clk[b * kClkStride + 16 + warp] = clock64();  // per warp
  __syncthreads();
  RO_CLK(2)
  if (warp == 0) {
    float* col = buf + (lane < C ? lane : C);  // lanes >= C share the scratch column
    const float vb = lane < C ? clip01(beta_l) : 0.0f;
    // LI scan (neuron.hpp:139-144) + time_sum (objective.hpp:40-50); col[t] <- V3_t
    float v = 0.0f, logit = 0.0f;
    int t = 0;
    if (a.readout_lif) {
      // LIF readout (neuron.hpp:127-136): s_t = [v - theta >= 0] is the trace, the
      // logits its time sums (network.hpp:396, objective.hpp:40-50)
      const float ntheta = -a.theta;
      for (; t < T; ++t) {
        const float I = col[t * rs];
        col[t * rs] = v;
        const bool sp = __fadd_rn(v, ntheta) >= 0.0f;
        v = __fsub_rn(__fadd_rn(__fmul_rn(v, vb), I), sp ? a.theta : 0.0f);
        logit = __fadd_rn(logit, sp ? 1.0f : 0.0f);
      }
    }
    for (; t + 8 <= T; t += 8) {
      float I[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) I[e] = col[(t + e) * rs];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        col[(t + e) * rs] = v;
        v = __fadd_rn(__fmul_rn(v, vb), I[e]);
        logit = __fadd_rn(logit, v);
      }
    }
    for (; t < T; ++t) {
      const float I = col[t * rs];
      col[t * rs] = v;
      v = __fadd_rn(__fmul_rn(v, vb), I);
      logit = __fadd_rn(logit, v);
    }
    const float v_final = v;
    RO_CLK(3)
    // softmax CE, sequential order of objective.hpp:53-73.  The class values are
    // gathered with independent shuffles first; only the max / sum chains are serial.
    float lg[kMaxClasses];
#pragma unroll
    for (int j = 0; j < kMaxClasses; ++j) lg[j] = __shfl_sync(0xffffffffu, logit, j);
    float mx = lg[0];
#pragma unroll
    for (int j = 1; j < kMaxClasses; ++j)
      if (j < C) mx = (mx < lg[j]) ? lg[j] : mx;
    const float xd = __fsub_rn(logit, mx);
    const float ex = (lane < C && a.loss_kind == 0) ? (a.exp_mode ? expf(xd) : exp_cr(xd)) : 0.0f;
#pragma unroll
    for (int j = 0; j < kMaxClasses; ++j) lg[j] = __shfl_sync(0xffffffffu, ex, j);
    float z = 0.0f;
#pragma unroll
    for (int j = 0; j < kMaxClasses; ++j)
      if (j < C) z = __fadd_rn(z, lg[j]);
    const int y = *s_label;
    const float logit_y = __shfl_sync(0xffffffffu, logit, y);
    // argmax, ties to the lowest index (objective.hpp:126-131)
    float bv = lane < C ? logit : -INFINITY;
    int bi = lane < C ? lane : 1 << 30;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      if (a.loss_kind == 0)
        a.loss_b[b] = __fsub_rn(__fadd_rn(mx, a.exp_mode ? logf(z) : log_cr(z)), logit_y);
      a.correct_b[b] = (bi == y) ? 1 : 0;
    }
    float delta = 0.0f;
    if (lane < C) {
      if (a.loss_kind == 1) {
        // spike_rate_mse (objective.hpp:139-183): r = counts / T, d = r - target;
        // the loss term d*d and the cotangent gs*d on every step
        const float r = __fdiv_rn(logit, float(T));
        const float d = __fsub_rn(r, lane == y ? a.rate_hi : a.rate_lo);
        a.loss_terms[size_t(b) * C + lane] = __fmul_rn(d, d);
        delta = __fmul_rn(a.mse_gs, d);
      } else {
        float d = __fdiv_rn(ex, z);
        if (lane == y) d = __fsub_rn(d, 1.0f);
        delta = __fmul_rn(d, a.inv_b);
      }
    }
    if (a.dbg_trace != nullptr && lane < C) {
      for (int s = 0; s < T; ++s)
        a.dbg_trace[(size_t(b) * T + s) * C + lane] =
            a.readout_lif ? (__fadd_rn(col[s * rs], -a.theta) >= 0.0f ? 1.0f : 0.0f)
                          : s + 1 < T ? col[(s + 1) * rs] : v_final;
    }
    RO_CLK(4)
    float G = delta, db = 0.0f, dbias = 0.0f;
    if (a.readout_lif) {
      // LIF reverse (the hidden layers' closure order, App. A.2) with dS_t = delta on
      // every step: dI3_t = G ; G = G bc + (delta + (-G) theta) g(V3_t - theta)
      G = 0.0f;
      for (t = T - 1; t >= 0; --t) {
        const float V3 = col[t * rs];
        const float gi = G;
        const float gs = __fadd_rn(delta, __fmul_rn(-gi, a.theta));
        const float g = surrogate_rt(a.act, a.slope, a.aux, __fadd_rn(V3, -a.theta));
        G = __fadd_rn(__fmul_rn(gi, vb), __fmul_rn(gs, g));
        db = __fadd_rn(db, __fmul_rn(gi, V3));
        dbias = __fadd_rn(dbias, gi);
        col[t * rs] = gi;
      }
    } else {
    // LI reverse scan: G_t = delta + G_{t+1} bc ; dI3_t = G_t ; dbeta += G_t V3_t
    t = T - 1;
    {
      const float V3 = col[t * rs];
      db = __fmul_rn(G, V3);
      dbias = G;
      col[t * rs] = G;
    }
    --t;
    for (; t >= 7; t -= 8) {
      float V3[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) V3[e] = col[(t - e) * rs];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        G = __fadd_rn(delta, __fmul_rn(G, vb));
        db = __fadd_rn(db, __fmul_rn(G, V3[e]));
        dbias = __fadd_rn(dbias, G);
        col[(t - e) * rs] = G;
      }
    }
    for (; t >= 0; --t) {
      const float V3 = col[t * rs];
      G = __fadd_rn(delta, __fmul_rn(G, vb));
      db = __fadd_rn(db, __fmul_rn(G, V3));
      dbias = __fadd_rn(dbias, G);
      col[t * rs] = G;
    }
    }
    if (lane < C) {
      a.dbeta_part[size_t(b) * C + lane] = db;
      if (a.dbias_part != nullptr) a.dbias_part[size_t(b) * C + lane] = dbias;
    }
    RO_CLK(5)
  }
  pdl_launch_dependents();
  __syncthreads();
  RO_CLK(6)
  // dI3 as three bf16 planes [3][64][B*T_pad] (class rows, (b,t) contiguous)
  const int chunks = (T + 7) / 8;
  const size_t cols = size_t(a.B) * a.T_pad;
  const size_t plane = size_t(64) * cols;
  for (int u = tid; u < C * chunks; u += G) {
    const int c = u / chunks, t0 = (u % chunks) * 8;
    uint32_t hp[4], mp[4], lp[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float g0 = t0 + e < T ? buf[(t0 + e) * rs + c] : 0.0f;
      const float g1 = t0 + e + 1 < T ? buf[(t0 + e + 1) * rs + c] : 0.0f;
      split3_pack(g0, g1, hp[e / 2], mp[e / 2], lp[e / 2]);
    }
    const size_t off = size_t(c) * cols + size_t(b) * a.T_pad + t0;
    *reinterpret_cast<uint4*>(a.d3_planes + off) = make_uint4(hp[0], hp[1], hp[2], hp[3]);
    *reinterpret_cast<uint4*>(a.d3_planes + plane + off) = make_uint4(mp[0], mp[1], mp[2], mp[3]);
    *reinterpret_cast<uint4*>(a.d3_planes + 2 * plane + off) = make_uint4(lp[0], lp[1], lp[2], lp[3]);
  }
  __syncthreads();
  RO_CLK(7)
  if (a.dbg_clk != nullptr && tid == 0) a.dbg_clk[b * kClkStride + 15] = globaltimer();
#undef RO_CLK
}

// ============================================================================
// K1  k_lif_fwd: I^T[n][t] = sum_k Wt[n][k] * A[t][k] on tcgen05 (3 bf16 planes
// of W, binary A exact in bf16), then the LIF scan epilogue straight from TMEM.
// One CTA = 128 neurons x SPB samples: the samples' activation rows are stacked
// into one N = SPB*TT MMA, so each W-plane tile streamed from L2 feeds SPB samples.
// grid (ceil(B/SPB), H_pad/128); block 448: w0-7 scan (sample w/4, TMEM quadrant
// w%4), w8-11 B-operand decode, w12 TMA, w13 MMA.
// ============================================================================
// One hidden LIF layer of a forward launch.
struct FwdLayer {
  const float* beta;      // [H], or one value (beta_stride 0: scalar / fixed BetaMode)
  int beta_stride;
  const float* bias;      // [H] or nullptr
  float* v_out;           // [B][T_pad][H_pad]
  uint32_t* s_np;         // [B][T_pad][H_pad/32]
  uint32_t* s_tp;         // [H_pad][B*T_pad/32]
  float* dbg_i;           // optional [B][T_pad][H_pad] raw projection
  const float* gamma;     // ALIF (declared cell): adaptation decay [H]; nullptr = LIF
  float* a_out;           // ALIF: adaptation entering step t [B][T_pad][H_pad]
  float* i_out;           // RLIF: projection only -- I (+ bias) [B][T_pad][H_pad] for
                          // k_rlif_fwd (no scan, no spikes); nullptr otherwise
  int K_pad, H, H_pad;
};
// A launch runs n_layers consecutive hidden layers.  n_layers > 1 (fused) needs
// one t-tile, one 128-neuron tile per layer and K_pad = 128 for layers >= 1: the
// scan warps write each next layer's binary B operand straight into the idle
// stages and the next GEMM runs in the same CTA.
constexpr int kFwdFuseMax = SNN_MAX_HIDDEN;
struct FwdMaps {
  CUtensorMap m[kFwdFuseMax];  // W planes of each layer (MN-major 64x64 boxes)
};
struct FwdArgs {
  const uint8_t* x;       // staged dataset (first layer = layer 0)
  const uint32_t* rows;   // [B] dataset row per sample (layer 0)
  const int64_t* rows_slot;  // schedule mode: rows += *rows_slot * B (else nullptr)
  const uint32_t* s_in;   // neuron-packed spikes of the previous layer (first layer > 0)
  FwdLayer lay[kFwdFuseMax];
  int n_layers;
  long long* dbg_clk;     // optional [gridDim.x*gridDim.y][kClkStride] phase timestamps
  const int32_t* xshift;  // layer 0: batch roll along the features, [0, in_features) (shift_augment)
  int B, T, T_pad, TT, NT, in_kind, stages, spb, in_features;
  int x_row;              // layer 0: bytes per packed time row of the dataset (K_pad of the
                          // staged layout, or in_features for a batch in the reference layout)
  int planes;  // bf16 W planes multiplied (3: the fp32 path; 2 / 1: fast modes)
  float theta;
};

constexpr int kFwdStagesMax = 4;
#ifndef SNN_FWD_EXP
#define SNN_FWD_EXP 0  // timing experiments only (A/B builds): 1 decoders skip their stores, 2 no MMAs, 3 no W loads
#endif
constexpr int kFwdSpbMax = 2;
constexpr int kFwdScanWarps = 4 * kFwdSpbMax;
constexpr int kFwdThreads = 32 * (kFwdScanWarps + 4 + 2);

constexpr uint32_t kPlaneTile = 128 * 128;  // 128 rows x 64 bf16 = 16 KB

__host__ __device__ constexpr uint32_t fwd_stage_bytes(int TT, int spb, int planes = 3) {
  return uint32_t(planes) * kPlaneTile + uint32_t(spb * TT) * 128u;
}
// dataset run of one sample for one t-tile: TT/8 rows of K_pad bytes (layer 0)
__host__ __device__ constexpr uint32_t fwd_xrun_bytes(int TT, int K_pad) {
  return uint32_t(TT / 8) * uint32_t(K_pad);
}
__host__ __device__ constexpr uint32_t fwd_smem_bytes(int TT, int spb, int stages, int x_kpad,
                                                      int planes = 3) {
  // stages | dataset runs | barriers (256) | per-scan-warp ballot rows (kFwdScanWarps x 32 words)
  return uint32_t(stages) * fwd_stage_bytes(TT, spb, planes) +
         2u * ((uint32_t(spb) * fwd_xrun_bytes(TT, x_kpad) + 1023) & ~1023u) + 1024 + 256 +
         uint32_t(kFwdScanWarps) * 128u;
}
// TMEM columns for N-wide accumulators, doubled when several t-tiles pipeline.
__host__ __device__ constexpr uint32_t tmem_cols_for(int N, int NT) {
  const int need = NT > 1 ? 2 * N : N;
  return need <= 32 ? 32u : need <= 64 ? 64u : need <= 128 ? 128u : need <= 256 ? 256u : 512u;
}
__host__ __device__ constexpr uint32_t acc_cols(int TT, int NT) { return tmem_cols_for(TT, NT); }

__device__ __forceinline__ void tmem_alloc_any(uint32_t cols, uint32_t* slot) {
  switch (cols) {
    case 32: tmem_alloc<32>(slot); break;
    case 64: tmem_alloc<64>(slot); break;
    case 128: tmem_alloc<128>(slot); break;
    case 256: tmem_alloc<256>(slot); break;
    default: tmem_alloc<512>(slot); break;
  }
}
__device__ __forceinline__ void tmem_dealloc_any(uint32_t cols, uint32_t taddr) {
  switch (cols) {
    case 32: tmem_dealloc<32>(taddr); break;
    case 64: tmem_dealloc<64>(taddr); break;
    case 128: tmem_dealloc<128>(taddr); break;
    case 256: tmem_dealloc<256>(taddr); break;
    default: tmem_dealloc<512>(taddr); break;
  }
}

// 32 LIF steps of one neuron (neuron.hpp:127-136 op order, bit-exact):
//   pre = v - theta ; s = pre >= 0 ; v = ((v * bc) + I) - s * theta
// kGeneral adds bias, a debug copy of I and a valid-step count (< 32 only in the
// last chunk).  V is stored before each step (membrane entering step t).
// The step's ballot (the 32 neurons' spikes of step j) goes to the warp's row of
// shared words sbal (lane 0 stores it) and lane j reads word j back after the chunk:
// one store per step instead of a per-step lane == j select.  kHpad > 0: the V row
// stride as a constant (immediate store offsets); 0: runtime hpad.
template <bool kGeneral, int kHpad = 0>
__device__ __forceinline__ void lif_chunk(const uint32_t (&r)[32], float* vp, float* dp, int hpad_rt,
                                          int nvalid, float vb, float bn, float theta, int lane,
                                          uint32_t* sbal, float& v, uint32_t& myword, uint32_t& tmask) {
  const int hpad = kHpad > 0 ? kHpad : hpad_rt;
  const float ntheta = -theta;
  const uint32_t sb = smem_u32(sbal);
  tmask = 0u;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    float I = __uint_as_float(r[j]);
    if (kGeneral) {
      I = __fadd_rn(I, bn);
      if (dp != nullptr && j < nvalid) dp[j * hpad] = I;
    }
    vp[j * hpad] = v;
    const float pre = __fadd_rn(v, ntheta);
    const bool sp = kGeneral ? (pre >= 0.0f && j < nvalid) : (pre >= 0.0f);
    const float m = __fmul_rn(v, vb);
    const float ai = __fadd_rn(m, I);
    v = __fsub_rn(ai, sp ? theta : 0.0f);
    const uint32_t bal = __ballot_sync(0xffffffffu, sp);
    if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(sb + 4u * j), "r"(bal) : "memory");
    if (sp) tmask |= 1u << j;
  }
  __syncwarp();
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(myword) : "r"(sb + 4u * lane) : "memory");
  __syncwarp();  // the row is rewritten by the next chunk
}

// 32 steps of the DECLARED ALIF cell (not in the reference; oracle/spiketrain_oracle.h
// states it, op order bit-identical to the oracle):
//   th = theta + a ; pre = v - th ; s = pre >= 0 ; v = ((v * bc) + I) - s * th ;
//   a = (a * gc) + (1 - gc) * s
// V and the adaptation a are stored before each step (state entering step t).
template <int kHpad = 0>
__device__ __forceinline__ void alif_chunk(const uint32_t (&r)[32], float* vp, float* ap, float* dp,
                                           int hpad_rt, int nvalid, float vb, float gc, float bn,
                                           bool has_bias, float theta, int lane, uint32_t* sbal, float& v,
                                           float& ad, uint32_t& myword, uint32_t& tmask) {
  const int hpad = kHpad > 0 ? kHpad : hpad_rt;
  const float omg = __fsub_rn(1.0f, gc);
  const uint32_t sb = smem_u32(sbal);
  tmask = 0u;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    float I = __uint_as_float(r[j]);
    if (has_bias) I = __fadd_rn(I, bn);
    if (dp != nullptr && j < nvalid) dp[j * hpad] = I;
    vp[j * hpad] = v;
    ap[j * hpad] = ad;
    const float th = __fadd_rn(theta, ad);
    const float pre = __fsub_rn(v, th);
    const bool sp = pre >= 0.0f && j < nvalid;
    const float m = __fmul_rn(v, vb);
    const float ai = __fadd_rn(m, I);
    v = __fsub_rn(ai, sp ? th : 0.0f);
    ad = __fadd_rn(__fmul_rn(ad, gc), sp ? omg : 0.0f);
    const uint32_t bal = __ballot_sync(0xffffffffu, sp);
    if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(sb + 4u * j), "r"(bal) : "memory");
    if (sp) tmask |= 1u << j;
  }
  __syncwarp();  // ballots of the chunk -> lane j takes step j's word (as lif_chunk)
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(myword) : "r"(sb + 4u * lane) : "memory");
  __syncwarp();
}

// kShift: layer-0 launches of an epoch loop with shift_augment (reads a.xshift);
// the default instantiation has no roll code in the decode loop.
// kAlif: the launch's hidden layers are declared ALIF cells (FwdLayer.gamma set);
// the LIF instantiation carries no adaptation code.
// kProj: a single RLIF layer -- the epilogue only stores the projection (FwdLayer.i_out).
template <bool kShift, bool kAlif = false, bool kProj = false>
__global__ void __launch_bounds__(kFwdThreads, 1)
    k_lif_fwd(const __grid_constant__ FwdMaps maps, FwdArgs a) {
  const CUtensorMap& tm_w = maps.m[0];
  const int K_pad0 = a.lay[0].K_pad;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int SPB = a.spb;
  const int NTOT = SPB * a.TT;  // MMA N (stacked samples)
  const uint32_t stage_bytes = fwd_stage_bytes(a.TT, SPB, a.planes);
  const int S = a.stages;
  // layer 0: each sample's dataset run for the current t-tile (TT/8 rows of x_row
  // bytes, contiguous) is bulk-copied into xbuf[tt % 2] (double-buffered across t-tiles)
  const uint32_t xrun = a.in_kind == 0 ? uint32_t(a.TT / 8) * uint32_t(a.x_row) : 0u;
  const uint32_t xbuf_bytes =
      a.in_kind == 0 ? (uint32_t(SPB) * fwd_xrun_bytes(a.TT, K_pad0) + 1023) & ~1023u : 0u;
  uint8_t* xbuf = smem + S * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(xbuf + 2 * xbuf_bytes);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* xfull = acc_empty + 2;
  uint64_t* xempty = xfull + 2;
  uint64_t* lfull = xempty + 2;  // fused layers: W planes of k-block 0 / 1 landed
  uint64_t* bready = lfull + 2;  // fused layers: next layer's B tiles written by the scan
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bready + 1);
  uint32_t* sbal_all = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(full) + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid (H_pad / 128, sample groups): a sample group's neuron tiles run together
  const int sg = blockIdx.y, b0 = sg * SPB, nt = blockIdx.x;
  const int nsamp = min(SPB, a.B - b0);
  long long* clk = a.dbg_clk != nullptr ? a.dbg_clk + (size_t(nt) * gridDim.y + sg) * kClkStride : nullptr;
  if (clk != nullptr && threadIdx.x == 0) {
    clk[0] = clock64();
    clk[6] = globaltimer();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    clk[4] = smid;
  }
  const int KB = K_pad0 / 64;
  const int total = a.NT * KB;
  // k-block order rotated per CTA: concurrent CTAs stream different W tiles
  const int rot = sg % KB;
  const uint32_t tmem_cols = tmem_cols_for(NTOT, a.NT);
  const int nbuf = a.NT > 1 ? 2 : 1;
  const int scan_threads = 128 * nsamp;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1 + 128);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], scan_threads);
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], 128);
      mbar_init(&lfull[i], 1);
    }
    mbar_init(bready, scan_threads);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_any(tmem_cols, tmem_slot);
  if (threadIdx.x == 32 * (kFwdScanWarps + 4)) tma_prefetch(&tm_w);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // activations / planes of the previous kernels are visible from here
  if (clk != nullptr && threadIdx.x == 0) clk[14] = globaltimer();  // span start: past the dependency wait
  const uint32_t tmem = *tmem_slot;
  const int dec_warp0 = kFwdScanWarps, tma_warp = kFwdScanWarps + 4, mma_warp = tma_warp + 1;

  if (warp == tma_warp) {
    // ---------------- TMA producer: the three W planes of each k-block
    if (elect_one()) {
      tma_prefetch(&tm_w);
      const uint32_t* rows = batch_rows(a.rows, a.rows_slot, a.B);
      for (int it = 0; it < total; ++it) {
        const int s = it % S, ph = (it / S) & 1, kb = (it % KB + rot) % KB;
        if (a.in_kind == 0 && it % KB == 0) {
          const int tt = it / KB, xb = tt & 1;
          if (tt >= 2) mbar_wait(&xempty[xb], ((tt - 2) >> 1) & 1);
          mbar_arrive_expect_tx(&xfull[xb], uint32_t(nsamp) * xrun);
          for (int sm = 0; sm < nsamp; ++sm)
            bulk_load(xbuf + xb * xbuf_bytes + sm * xrun,
                      a.x + (size_t(rows[b0 + sm]) * (a.T_pad / 8) + tt * (a.TT / 8)) * size_t(a.x_row),
                      xrun, &xfull[xb]);
        }
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], SNN_FWD_EXP == 3 ? 0u : uint32_t(a.planes) * kPlaneTile);
        uint8_t* A = smem + s * stage_bytes;
        // W planes [3][K_pad][H_pad] read MN-major: per plane two 64-neuron x 64-k boxes
        for (int p = 0; p < (SNN_FWD_EXP == 3 ? 0 : a.planes); ++p)
          for (int h = 0; h < 2; ++h)
            tma_load_2d(A + p * kPlaneTile + h * 8192, &tm_w, &full[s], nt * 128 + h * 64,
                        p * K_pad0 + kb * 64);

      }
      // fused layers: once the previous GEMM is complete the stages are idle; the
      // next layer's W planes land in stage kb's A part while the scan runs
      for (int li = 1; li < a.n_layers; ++li) {
        mbar_wait(&acc_full[0], (li - 1) & 1);
        const int KBl = a.lay[li].K_pad / 64;
        for (int kb = 0; kb < KBl; ++kb) {
          mbar_arrive_expect_tx(&lfull[kb], uint32_t(a.planes) * kPlaneTile);
          for (int p = 0; p < a.planes; ++p)
            for (int h = 0; h < 2; ++h)
              tma_load_2d(smem + kb * stage_bytes + p * kPlaneTile + h * 8192, &maps.m[li], &lfull[kb],
                          nt * 128 + h * 64, p * a.lay[li].K_pad + kb * 64);
        }
      }
    }
    __syncwarp();
  } else if (warp == mma_warp) {
    // ---------------- MMA issuer (one thread), N = SPB*TT stacked sample rows;
    // A (W^T) MN-major: LBO = 8 KB between the 64-neuron halves, 16 k-rows per step
    const uint32_t idesc = idesc_bf16(128, NTOT, true, false);
    if (elect_one()) {
      for (int it = 0; it < total; ++it) {
        const int s = it % S, ph = (it / S) & 1;
        const int tt = it / KB, kb = it % KB, buf = tt % nbuf;  // kb: position in the tile
        if (kb == 0 && tt >= nbuf) {
          mbar_wait(&acc_empty[buf], ((tt - nbuf) / nbuf) & 1);
          tc_fence_after();
        }
        mbar_wait(&full[s], ph);
        if (clk != nullptr && it < 32) clk[16 + it] = clock64();
        tc_fence_after();
        const uint32_t A = smem_u32(smem + s * stage_bytes);
        const uint32_t Bt = A + a.planes * kPlaneTile;
        const uint32_t d = tmem + buf * NTOT;
        if (a.planes == 3) {  // the fp32 path, fully unrolled
#pragma unroll
          for (int ks = 0; ks < (SNN_FWD_EXP == 2 ? 0 : 4); ++ks) {
            const uint64_t bd = sdesc_sw128(Bt + ks * 32, 16, 1024);
#pragma unroll
            for (int p = 2; p >= 0; --p) {
              const uint64_t ad = sdesc_sw128(A + p * kPlaneTile + ks * 2048, 8192, 1024);
              umma_bf16(d, ad, bd, idesc, (kb | ks | (2 - p)) != 0);
            }
          }
        } else {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bd = sdesc_sw128(Bt + ks * 32, 16, 1024);
            for (int p = a.planes - 1; p >= 0; --p) {
              const uint64_t ad = sdesc_sw128(A + p * kPlaneTile + ks * 2048, 8192, 1024);
              umma_bf16(d, ad, bd, idesc, (kb | ks | (a.planes - 1 - p)) != 0);
            }
          }
        }
        umma_commit(&empty[s]);
        if (kb == KB - 1) umma_commit(&acc_full[buf]);
      }
      // fused layers: A = W planes in stage kb, B = spikes the scan wrote (one t-tile)
      for (int li = 1; li < a.n_layers; ++li) {
        mbar_wait(bready, (li - 1) & 1);
        tc_fence_after();
        const int KBl = a.lay[li].K_pad / 64;
        for (int kb = 0; kb < KBl; ++kb) {
          mbar_wait(&lfull[kb], (li - 1) & 1);
          tc_fence_after();
          const uint32_t A = smem_u32(smem + kb * stage_bytes);
          const uint32_t Bt = A + a.planes * kPlaneTile;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bd = sdesc_sw128(Bt + ks * 32, 16, 1024);
            for (int p = a.planes - 1; p >= 0; --p) {
              const uint64_t ad = sdesc_sw128(A + p * kPlaneTile + ks * 2048, 8192, 1024);
              umma_bf16(tmem, ad, bd, idesc, (kb | ks | (a.planes - 1 - p)) != 0);
            }
          }
        }
        umma_commit(&acc_full[0]);
      }
    }
    __syncwarp();
  } else if (warp >= dec_warp0) {
    // ---------------- B-operand producers: activations -> bf16 {0,1} rows t, cols k,
    // sample s's rows at [s*TT, (s+1)*TT).  Loads of stage it+1 issue before the wait.
    const int tid = threadIdx.x - dec_warp0 * 32;
    const size_t kwords = size_t(K_pad0) / 32;
    // shift_augment (data.hpp:216-227): feature k of the rolled batch is feature
    // (k - xsh) mod in of the staged one; padding features stay zero
    const int xsh = kShift ? *a.xshift : 0;
    const int units = SPB * a.TT;  // kind 0: (sample, t-group, 8-feature chunk); kind 1: row
    auto fetch = [&](int it, int u) -> uint64_t {
      if (a.in_kind == 0 || u >= units || it >= total) return 0;
      const int tt = it / KB, kb = (it % KB + rot) % KB;
      const int sm = u / a.TT, r = u % a.TT;
      if (sm >= nsamp) return 0;
      return __ldg(reinterpret_cast<const unsigned long long*>(
          a.s_in + (size_t(b0 + sm) * a.T_pad + tt * a.TT + r) * kwords + kb * 2));
    };
    uint64_t cur0 = fetch(0, tid), cur1 = fetch(0, tid + 128);
    for (int it = 0; it < total; ++it) {
      const int s = it % S, ph = (it / S) & 1;
      const int tt = it / KB, kb = (it % KB + rot) % KB;
      if (a.in_kind == 0 && it % KB == 0) mbar_wait(&xfull[tt & 1], (tt >> 1) & 1);
      mbar_wait(&empty[s], ph ^ 1);
      const uint32_t Bt = smem_u32(smem + s * stage_bytes + a.planes * kPlaneTile);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = tid + 128 * h;
        if (u >= units) continue;
        const int sm = u / a.TT, r = u % a.TT;
        if (a.in_kind == 0) {
          // dataset bytes [t/8][k] (bulk-copied), bit 7-(t%8): 8 k of one t-group -> 8 rows
          const int g = r >> 3, q = r & 7;
          const uint8_t* xr = xbuf + (tt & 1) * xbuf_bytes + sm * xrun + g * a.x_row;
          uint64_t cur = 0ull;
          if (sm < nsamp) {
            if (!kShift || xsh == 0) {
              // rows of the reference layout are only 4-byte aligned; features >= in
              // of the last block belong to the next row there and are masked
              const uint32_t* xw = reinterpret_cast<const uint32_t*>(xr + kb * 64 + q * 8);
              cur = uint64_t(xw[0]) | (uint64_t(xw[1]) << 32);
              const int nb = a.in_features - (kb * 64 + q * 8);
              if (nb < 8) cur = nb <= 0 ? 0ull : cur & ((1ull << (8 * nb)) - 1ull);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int k = kb * 64 + q * 8 + i;
                if (k < a.in_features)
                  cur |= uint64_t(xr[k >= xsh ? k - xsh : k - xsh + a.in_features]) << (8 * i);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < (SNN_FWD_EXP == 1 ? 0 : 8); ++j)
            st_shared_v4(Bt + sw128_off(sm * a.TT + 8 * g + j, q),
                         expand_bytes01((cur >> (7 - j)) & 0x0101010101010101ull));
        } else {
          // neuron-packed spike words: row t, 2 words = 64 k
          const uint64_t cur = h == 0 ? cur0 : cur1;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            st_shared_v4(Bt + sw128_off(sm * a.TT + r, q), expand_bits_lsb(uint32_t(cur >> (8 * q)) & 0xFFu));
        }
      }
      if (a.in_kind == 0 && it % KB == KB - 1) mbar_arrive(&xempty[tt & 1]);
      fence_async_smem();
      mbar_arrive(&full[s]);
      // next stage's spike words after the proxy fence (it would wait for them)
      cur0 = fetch(it + 1, tid);
      cur1 = fetch(it + 1, tid + 128);
    }
  } else if (warp / 4 < nsamp) {
    // ---------------- LIF scan epilogue: thread = neuron (TMEM lane) of sample warp/4
    const int sm = warp >> 2, q = warp & 3;
    const int b = b0 + sm;
    const int n = nt * 128 + q * 32 + lane;
    const size_t tp_words = size_t(a.B) * a.T_pad / 32;
    for (int li = 0; li < a.n_layers; ++li) {
      const FwdLayer& ly = a.lay[li];
      const float vb = clip01(n < ly.H ? ly.beta[n * ly.beta_stride] : 0.0f);
      const float bn = (ly.bias != nullptr && n < ly.H) ? ly.bias[n] : 0.0f;
      const size_t hw = size_t(ly.H_pad) / 32;
      const bool alif = kAlif && ly.gamma != nullptr;
      const float gc = (alif && n < ly.H) ? clip01(ly.gamma[n]) : 0.0f;
      float ad = 0.0f;  // ALIF adaptation state
      // fused: lane j writes the next layer's B row t0+j (its quadrant's 32 spikes
      // of that step, from the ballot word) into stage q/2's B part
      const bool feed = li + 1 < a.n_layers;
      const uint32_t feed_b = smem_u32(smem + (q >> 1) * stage_bytes + a.planes * kPlaneTile);
      float v = 0.0f;
      for (int tt = 0; tt < a.NT; ++tt) {
        const int g = li * a.NT + tt;  // accumulator use (fused: one per layer)
        const int buf = g % nbuf;
        mbar_wait(&acc_full[buf], (g / nbuf) & 1);
        __syncwarp();  // reconverge after the per-thread spin: the scan's ballots then
                       // compile to plain VOTEs (no WARPSYNC.COLLECTIVE emulation)
        tc_fence_after();
        if (clk != nullptr && threadIdx.x == 0 && tt == 0 && li == 0) clk[1] = clock64();
        if (clk != nullptr && threadIdx.x == 0 && tt == 0 && li < 4) clk[8 + 2 * li] = clock64();
        for (int c = 0; c < a.TT / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tmem + (uint32_t(q * 32) << 16) + buf * NTOT + sm * a.TT + c * 32, r);
          tmem_ld_wait();
          const int t0 = tt * a.TT + c * 32;
          if (kProj) {  // RLIF layer: the recurrent scan runs in k_rlif_fwd
            float* ip = ly.i_out + (size_t(b) * a.T_pad + t0) * ly.H_pad + n;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float I = __uint_as_float(r[j]);
              ip[size_t(j) * ly.H_pad] = ly.bias != nullptr ? __fadd_rn(I, bn) : I;
            }
            continue;
          }
          uint32_t myword = 0u, tmask = 0u;
          if (t0 < a.T) {
            float* vp = ly.v_out + (size_t(b) * a.T_pad + t0) * ly.H_pad + n;
            if (kAlif && alif && ly.H_pad == 128)
              alif_chunk<128>(r, vp, ly.a_out + (vp - ly.v_out),
                              ly.dbg_i != nullptr ? ly.dbg_i + (vp - ly.v_out) : nullptr, 128,
                              min(32, a.T - t0), vb, gc, bn, ly.bias != nullptr, a.theta, lane,
                              sbal_all + warp * 32, v, ad, myword, tmask);
            else if (kAlif && alif)
              alif_chunk(r, vp, ly.a_out + (vp - ly.v_out),
                         ly.dbg_i != nullptr ? ly.dbg_i + (vp - ly.v_out) : nullptr, ly.H_pad,
                         min(32, a.T - t0), vb, gc, bn, ly.bias != nullptr, a.theta, lane,
                         sbal_all + warp * 32, v, ad, myword, tmask);
            else if (ly.bias != nullptr || ly.dbg_i != nullptr || t0 + 32 > a.T)
              lif_chunk<true>(r, vp, ly.dbg_i != nullptr ? ly.dbg_i + (vp - ly.v_out) : nullptr, ly.H_pad,
                              a.T - t0, vb, bn, a.theta, lane, sbal_all + warp * 32, v, myword, tmask);
            else if (ly.H_pad == 128)
              lif_chunk<false, 128>(r, vp, nullptr, 128, 32, vb, 0.0f, a.theta, lane, sbal_all + warp * 32, v,
                                    myword, tmask);
            else
              lif_chunk<false>(r, vp, nullptr, ly.H_pad, 32, vb, 0.0f, a.theta, lane, sbal_all + warp * 32, v,
                               myword, tmask);
          }
          // padded steps (t >= T): no spikes; V rows beyond T are never read
          ly.s_np[(size_t(b) * a.T_pad + t0 + lane) * hw + nt * 4 + q] = myword;
          ly.s_tp[size_t(n) * tp_words + size_t(b) * (a.T_pad / 32) + t0 / 32] = tmask;
          if (feed) {
            const uint32_t row = uint32_t(sm * a.TT + c * 32 + lane);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              st_shared_v4(feed_b + sw128_off(row, uint32_t((q & 1) * 4 + i)),
                           expand_bits_lsb((myword >> (8 * i)) & 0xFFu));
          }
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
      }
      if (clk != nullptr && threadIdx.x == 0 && li < 4) clk[9 + 2 * li] = clock64();
      if (feed) {
        fence_async_smem();  // B tiles -> visible to the tensor core
        tc_fence_before();   // TMEM reads of this layer done before the next MMA
        mbar_arrive(bready);
      }
    }
    if (clk != nullptr && threadIdx.x == 0) clk[2] = clock64();
  }

  pdl_launch_dependents();
  __syncthreads();
  if (clk != nullptr && threadIdx.x == 0) {
    clk[3] = clock64();
    clk[7] = globaltimer();
    clk[15] = clk[7];
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_any(tmem_cols, tmem);
  }
}

// ============================================================================
// K3  k_lif_bwd: LIF reverse scan (App. A.2) with dS from the tensor core.
//   dS^T[n][t] = sum_k Wb[n][k] dI_next^T[k][t]  (tcgen05, 6 bf16 plane products
//   ~ fp32), for the readout-fed layer k = classes (dI3 planes from k_readout).
//   Then per neuron (TMEM lane), t descending:
//     dI_t = G ; ds = dS_t - theta*G ; G = bc*G + g(V_t - theta)*ds ; dbeta += G V_t
// The scan runs in 32-step chunks split into three phases: surrogates (independent),
// the recurrence (short dependent chain), plane split + 64-byte vector stores.
// grid (B, H_pad/128); block 192: w0-3 scan, w4 TMA, w5 MMA.
// ============================================================================
struct BwdArgs {
  const float* v_in;           // V_l [B][T_pad][H_pad]
  const float* beta;           // [H] (or one value: beta_stride 0)
  int beta_stride;
  __nv_bfloat16* di_planes;    // out: dI_l planes [3][H_pad][B*T_pad]
  float* dbeta_part;           // [B][H]
  float* dbias_part;           // [B][H] or nullptr
  float* dbg_ds;               // optional [B][T_pad][H_pad]
  long long* dbg_clk;          // optional [gridDim.x*gridDim.y][8] phase timestamps
  int B, T, T_pad, TT, NT, K_pad, H, H_pad, act, stages;
  int K;                       // unpadded contraction width (next layer's neurons / classes):
                               // 16-k MMA steps past it in the last k-block are skipped
  int planes;                  // bf16 planes per real operand (3: fp32 path)
  float theta, slope, aux;
  // activity regularizer on a monitored layer (kReg launches only)
  const uint32_t* s_tp;        // this layer's spikes, time-packed [H_pad][B*T_pad/32]
  unsigned int* hist;          // [T+1] (sample, neuron) count histogram for the loss value
  float reg_gs, f_min, f_max, lambda_low, lambda_high;  // reg_gs = 2 / (B_global*H * T)
  // ALIF (kAlif launches only; declared cell, oracle/spiketrain_oracle.h)
  const float* a_in;           // adaptation entering step t [B][T_pad][H_pad]
  const float* gamma;          // [H]
  float* dgamma_part;          // [B][H]
  // RLIF (kDsOnly launches): dS of this layer [B][T_pad][H_pad] for k_rlif_bwd
  float* ds_out;
};

// d loss / d count of one (sample, neuron) (objective.hpp:208-227): with g = 1,
// gs (lambda_high dh - lambda_low dl), r = count / T -- the same float ops.
__device__ __forceinline__ float activity_dcount(const BwdArgs& a, int count) {
  const float r = __fdiv_rn(float(count), float(a.T));
  const float xl = __fsub_rn(a.f_min, r), xh = __fsub_rn(r, a.f_max);
  const float dl = xl > 0.0f ? xl : 0.0f, dh = xh > 0.0f ? xh : 0.0f;
  return __fmul_rn(a.reg_gs, __fsub_rn(__fmul_rn(a.lambda_high, dh), __fmul_rn(a.lambda_low, dl)));
}

// Monitored layer with the activity regularizer (kReg launches): the spike count
// of (sample b, neuron n) over the window (monitor_activity, neuron.hpp:106-114)
// from the time-packed raster, its d loss / d count, and -- segment 0 only -- one
// histogram entry per (sample, neuron), warp-aggregated, for the loss value.
__device__ __forceinline__ float monitor_term(const BwdArgs& a, int b, int n, int sg, int lane) {
  int count = -1;
  float rterm = 0.0f;
  if (n < a.H) {
    const int wpb = a.T_pad / 32;
    const uint32_t* w = a.s_tp + size_t(n) * (size_t(a.B) * wpb) + size_t(b) * wpb;
    count = 0;
    for (int i = 0; i < wpb; ++i) count += __popc(__ldg(w + i));
    rterm = activity_dcount(a, count);
  }
  if (sg == 0) {
    const unsigned peers = __match_any_sync(0xffffffffu, count);
    if (count >= 0 && lane == __ffs(peers) - 1) atomicAdd(a.hist + count, unsigned(__popc(peers)));
  }
  return rterm;
}

__device__ __forceinline__ void load_v_chunk(const BwdArgs& a, int b, int n, int c,
                                             float (&v)[32]) {
  const float* __restrict__ src = a.v_in + (size_t(b) * a.T_pad + c * 32) * a.H_pad + n;
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = (c * 32 + e < a.T) ? __ldg(src + size_t(e) * a.H_pad) : 0.0f;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void load_v16(const float* __restrict__ p, int hpad, int nval,
                                         float (&v)[16]) {
  if (hpad == 128 && nval >= 16) {  // 128-wide layers, whole chunk: immediate offsets
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = __ldg(p + e * 128);
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = e < nval ? __ldg(p + size_t(e) * hpad) : 0.0f;
  }
}
// affine map of 16 reverse steps: G' = (bc - theta g) G + g dS
template <int kAct, bool kTail>
__device__ __forceinline__ void bwd_compose(const uint32_t (&r)[16], const float (&vr)[16], int nval,
                                            float vb, float theta, const BwdArgs& a, float& A,
                                            float& Bc, float (&gout)[16]) {
#pragma unroll
  for (int e = 15; e >= 0; --e) {
    if (kTail && e >= nval) {
      gout[e] = 0.0f;
      continue;
    }
    const float g = surrogate_t<kAct>(a.slope, a.aux, __fsub_rn(vr[e], theta));
    gout[e] = g;
    const float at = vb - theta * g;
    Bc = at * Bc + g * __uint_as_float(r[e]);
    A = at * A;
  }
}
// 16 reverse steps in the reference order with the surrogates the compose pass
// computed (bit-identical values, read back from TMEM): dI_t = G ; gs = dS + (-G) theta ;
// G = G bc + gs g ; dbeta += G V ; dbias += G
template <bool kTail>
__device__ __forceinline__ void bwd_replay_g(const uint32_t (&r)[16], const float (&vr)[16],
                                             const uint32_t (&gr)[16], int nval, float vb, float theta,
                                             float& G, float& db, float& dbias, float (&x)[16]) {
#pragma unroll
  for (int e = 15; e >= 0; --e) {
    if (kTail && e >= nval) {
      x[e] = 0.0f;
      continue;
    }
    const float g = __uint_as_float(gr[e]);
    const float gi = G;
    const float gs = __fadd_rn(__uint_as_float(r[e]), __fmul_rn(-gi, theta));
    G = __fadd_rn(__fmul_rn(gi, vb), __fmul_rn(gs, g));
    x[e] = gi;
    db = __fadd_rn(db, __fmul_rn(gi, vr[e]));
    dbias = __fadd_rn(dbias, gi);
  }
}
// 16 reverse steps in the reference order: dI_t = G ; gs = dS + (-G) theta ;
// G = G bc + gs g ; dbeta += G V ; dbias += G
template <int kAct, bool kTail>
__device__ __forceinline__ void bwd_replay(const uint32_t (&r)[16], const float (&vr)[16], int nval,
                                           float vb, float theta, const BwdArgs& a, float& G,
                                           float& db, float& dbias, float (&x)[16]) {
#pragma unroll
  for (int e = 15; e >= 0; --e) {
    if (kTail && e >= nval) {
      x[e] = 0.0f;
      continue;
    }
    const float g = surrogate_t<kAct>(a.slope, a.aux, __fsub_rn(vr[e], theta));
    const float gi = G;
    const float gs = __fadd_rn(__uint_as_float(r[e]), __fmul_rn(-gi, theta));
    G = __fadd_rn(__fmul_rn(gi, vb), __fmul_rn(gs, g));
    x[e] = gi;
    db = __fadd_rn(db, __fmul_rn(gi, vr[e]));
    dbias = __fadd_rn(dbias, gi);
  }
}

// ALIF reverse step (declared cell; the exact reverse of alif_chunk's ops, same
// statement order as the oracle): with gv = d/dv_{t+1}, ga = d/da_{t+1}
//   th = theta + a ; s = (v - th) >= 0 ; g = g(v - th)
//   gs = (dS + (-gv) th) + ga (1 - gc) ; gp = gs g
//   gv' = gv bc + gp ; ga' = ((ga gc) - gp) - s gv
// Linear in (gv, ga): the compose pass builds the 2x2 affine map of 16 steps,
//   [gv'; ga'] = [[bc - th g, (1-gc) g], [th g - s, gc - (1-gc) g]] [gv; ga] + g dS [1; -1]
template <int kAct, bool kTail>
__device__ __forceinline__ void bwd_compose_alif(const uint32_t (&r)[16], const float (&vr)[16],
                                                 const float (&ar)[16], int nval, float vb, float gc,
                                                 float omg, float theta, const BwdArgs& a,
                                                 float (&P)[4], float (&q)[2]) {
#pragma unroll
  for (int e = 15; e >= 0; --e) {
    if (kTail && e >= nval) continue;
    const float th = __fadd_rn(theta, ar[e]);
    const float pre = __fsub_rn(vr[e], th);
    const float sp = pre >= 0.0f ? 1.0f : 0.0f;
    const float g = surrogate_t<kAct>(a.slope, a.aux, pre);
    const float tg = th * g, og = omg * g;
    const float m00 = vb - tg, m01 = og, m10 = tg - sp, m11 = gc - og;
    const float c = g * __uint_as_float(r[e]);
    const float p00 = m00 * P[0] + m01 * P[2], p01 = m00 * P[1] + m01 * P[3];
    const float p10 = m10 * P[0] + m11 * P[2], p11 = m10 * P[1] + m11 * P[3];
    const float q0 = m00 * q[0] + m01 * q[1] + c, q1 = m10 * q[0] + m11 * q[1] - c;
    P[0] = p00; P[1] = p01; P[2] = p10; P[3] = p11;
    q[0] = q0; q[1] = q1;
  }
}
template <int kAct, bool kTail>
__device__ __forceinline__ void bwd_replay_alif(const uint32_t (&r)[16], const float (&vr)[16],
                                                const float (&ar)[16], int nval, float vb, float gc,
                                                float omg, float theta, const BwdArgs& a, float& gv,
                                                float& ga, float& db, float& dbias, float& dgam,
                                                float (&x)[16]) {
#pragma unroll
  for (int e = 15; e >= 0; --e) {
    if (kTail && e >= nval) {
      x[e] = 0.0f;
      continue;
    }
    const float th = __fadd_rn(theta, ar[e]);
    const float pre = __fsub_rn(vr[e], th);
    const float sp = pre >= 0.0f ? 1.0f : 0.0f;
    const float g = surrogate_t<kAct>(a.slope, a.aux, pre);
    const float gs = __fadd_rn(__fadd_rn(__uint_as_float(r[e]), __fmul_rn(-gv, th)), __fmul_rn(ga, omg));
    const float gp = __fmul_rn(gs, g);
    x[e] = gv;
    db = __fadd_rn(db, __fmul_rn(gv, vr[e]));
    dbias = __fadd_rn(dbias, gv);
    dgam = __fadd_rn(dgam, __fmul_rn(ga, __fsub_rn(ar[e], sp)));
    const float ngv = __fadd_rn(__fmul_rn(gv, vb), gp);
    ga = __fsub_rn(__fsub_rn(__fmul_rn(ga, gc), gp), __fmul_rn(sp, gv));
    gv = ngv;
  }
}

// dS of 16 steps + the monitor's per-(sample, neuron) term (two gradient
// contributions to the stacked spikes: commutative, so the reference's order
// does not matter)
__device__ __forceinline__ void add_dcount(uint32_t (&r)[16], float term) {
#pragma unroll
  for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__fadd_rn(__uint_as_float(r[e]), term));
}

// dI of 16 steps as 3 bf16 planes: staged in smem (one t-tile, SW128 layout of
// tm_out; tl = step within the tile) or stored straight to the planes (drow = the
// neuron's row at the chunk's first step, plane = plane stride in elements).
// one 32-byte store (a whole L2 sector): 16 bf16 of one plane row
__device__ __forceinline__ void st_global_v8(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void bwd_store_di16(const float (&x)[16], bool stage_out, uint8_t* smem,
                                               int tl, int q, int lane, int TT,
                                               __nv_bfloat16* drow, size_t plane) {
  uint32_t ph_[8], pm_[8], pl_[8];
#pragma unroll
  for (int e = 0; e < 16; e += 2) split3_pack(x[e], x[e + 1], ph_[e / 2], pm_[e / 2], pl_[e / 2]);
  if (stage_out) {
    const uint32_t row = uint32_t(q * 32 + lane);
    const uint32_t base = smem_u32(smem) + uint32_t(tl >> 6) * 16384u + row * 128u;
    const uint32_t j0 = uint32_t(tl & 63) >> 3;
    const uint32_t o0 = ((j0 ^ (row & 7u)) << 4), o1 = (((j0 + 1u) ^ (row & 7u)) << 4);
    const uint32_t pstride = uint32_t(TT / 64) * 16384u;
    st_shared_v4(base + o0, make_uint4(ph_[0], ph_[1], ph_[2], ph_[3]));
    st_shared_v4(base + o1, make_uint4(ph_[4], ph_[5], ph_[6], ph_[7]));
    st_shared_v4(base + pstride + o0, make_uint4(pm_[0], pm_[1], pm_[2], pm_[3]));
    st_shared_v4(base + pstride + o1, make_uint4(pm_[4], pm_[5], pm_[6], pm_[7]));
    st_shared_v4(base + 2 * pstride + o0, make_uint4(pl_[0], pl_[1], pl_[2], pl_[3]));
    st_shared_v4(base + 2 * pstride + o1, make_uint4(pl_[4], pl_[5], pl_[6], pl_[7]));
  } else {
    uint4* dh = reinterpret_cast<uint4*>(drow);
    uint4* dm = reinterpret_cast<uint4*>(drow + plane);
    uint4* dl = reinterpret_cast<uint4*>(drow + 2 * plane);
    dh[0] = make_uint4(ph_[0], ph_[1], ph_[2], ph_[3]);
    dh[1] = make_uint4(ph_[4], ph_[5], ph_[6], ph_[7]);
    dm[0] = make_uint4(pm_[0], pm_[1], pm_[2], pm_[3]);
    dm[1] = make_uint4(pm_[4], pm_[5], pm_[6], pm_[7]);
    dl[0] = make_uint4(pl_[0], pl_[1], pl_[2], pl_[3]);
    dl[1] = make_uint4(pl_[4], pl_[5], pl_[6], pl_[7]);
  }
}

#ifndef SNN_BWD_EXP
#define SNN_BWD_EXP 0  // timing experiments only (tests/clk_probe.py): 1 = skip the dI plane stores
#endif
constexpr int kBwdSeg = 2;                        // time segments per t-tile
constexpr int kBwdScanThreads = 128 * kBwdSeg;
constexpr int kBwdThreads = kBwdScanThreads + 32;  // + control warp (lane 0 TMA, lane 1 MMA)
__host__ __device__ constexpr uint32_t bwd_stage_bytes(int TT) {
  return 3 * kPlaneTile + 3 * uint32_t(TT) * 128u;
}
// segment exchange floats per scan thread: LIF (A, Bc, G); ALIF (P 2x2, q 2, G 2)
__host__ __device__ constexpr uint32_t bwd_smem_bytes(int TT, int stages, bool alif = false) {
  return uint32_t(stages) * bwd_stage_bytes(TT) + 1024 + 256 + (alif ? 8 : 3) * 4 * kBwdScanThreads;
}

// kReg: the layer feeds a monitor and the activity regularizer is on -- every
// step's dS gains d loss / d count of its (sample, neuron) (sum_axis1 backward).
// kAlif: the layer is the declared ALIF cell (two-state reverse scan, 2x2 maps).
// kDsOnly: the layer is the declared RLIF cell -- only dS (+ the monitor term) is
// written (a.ds_out); its recurrent reverse scan is k_rlif_bwd.
// kStage: 0 = dI planes staged for TMA stores when the CTA has one t-tile (NT == 1), else
// 16-byte stores; 2 = several t-tiles (plain LIF layers), whole 32-byte sector stores (the
// 16-byte halves of a sector are partial writes: C3 / C5 reverse scans 10-25 % faster).
// One-t-tile launches keep kStage 0 as is (the reverse kernel's timing follows its code
// shape: a specialised one-t-tile variant measured slower).
template <int kAct, bool kReg = false, bool kAlif = false, bool kDsOnly = false, int kStage = 0>
__global__ void __launch_bounds__(kBwdThreads, 2)
    k_lif_bwd(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_di,
              const __grid_constant__ CUtensorMap tm_out, BwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = a.stages;
  const uint32_t stage_bytes = bwd_stage_bytes(a.TT);
  const uint32_t btile = uint32_t(a.TT) * 128u;  // one plane: 64 k-rows x TT t (MN-major)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // segment exchange: affine maps (A, Bc) and segment-start G per (segment, neuron)
  float* xA = reinterpret_cast<float*>(smem + S * stage_bytes + 256);
  float* xB = xA + kBwdScanThreads;
  float* xG = xB + kBwdScanThreads;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid (H_pad / 128, B): the neuron tiles of one sample are adjacent in launch
  // order, so the sample's dI planes come from HBM once and from L2 for the others
  const int b = blockIdx.y, nt = blockIdx.x;
  long long* clk = a.dbg_clk != nullptr ? a.dbg_clk + (size_t(nt) * a.B + b) * kClkStride : nullptr;
  if (clk != nullptr && threadIdx.x == 0) clk[0] = clock64();
  const int KB = a.K_pad / 64;
  const int total = a.NT * KB;
  // one t-tile: TT more columns cache the membranes V between the two scan passes
  const bool vcache = a.NT == 1 && !kDsOnly;
  const uint32_t tmem_cols = vcache ? acc_cols(2 * a.TT, 1) : acc_cols(a.TT, a.NT);
  const int nbuf = a.NT > 1 ? 2 : 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kBwdScanThreads);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_any(tmem_cols, tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int ctl_warp = kBwdScanThreads / 32;
  // the first stage's W planes are parameters (last written by the previous step's
  // update, complete before this step's forward passed its own wait): their TMA goes
  // out before the dependency wait, overlapping the previous kernel's tail
  if (warp == ctl_warp && lane == 0 && total > 0) {
    mbar_arrive_expect_tx(&full[0], uint32_t(a.planes) * (kPlaneTile + btile));
    for (int p = 0; p < a.planes; ++p)
      tma_load_2d(smem + p * kPlaneTile, &tm_w, &full[0], 0, p * a.H_pad + nt * 128);
  }
  pdl_wait();
  if (clk != nullptr && threadIdx.x == 0) clk[14] = globaltimer();  // span start: past the dependency wait
  const uint32_t tmem = *tmem_slot;
  const int cols_total = a.B * a.T_pad;

  if (warp == ctl_warp) {
    if (lane == 0) {
      tma_prefetch(&tm_w);
      tma_prefetch(&tm_di);
      for (int it = 0; it < total; ++it) {
        const int s = it % S, ph = (it / S) & 1;
        const int tt = a.NT - 1 - it / KB, kb = it % KB;
        mbar_wait(&empty[s], ph ^ 1);
        if (it > 0) mbar_arrive_expect_tx(&full[s], uint32_t(a.planes) * (kPlaneTile + btile));
        uint8_t* A = smem + s * stage_bytes;
        uint8_t* Bt = A + 3 * kPlaneTile;
        for (int p = 0; p < a.planes; ++p) {
          if (it > 0) tma_load_2d(A + p * kPlaneTile, &tm_w, &full[s], kb * 64, p * a.H_pad + nt * 128);
          for (int h = 0; h < a.TT / 64; ++h)
            tma_load_2d(Bt + p * btile + h * 8192, &tm_di, &full[s],
                        b * a.T_pad + tt * a.TT + h * 64, p * a.K_pad + kb * 64);
        }
      }
    } else if (lane == 1) {
    // A: K-major W planes; B: MN-major dI planes (t contiguous), LBO = 64-t block
    const uint32_t idesc = idesc_bf16(128, a.TT, false, true);
      for (int it = 0; it < total; ++it) {
        const int s = it % S, ph = (it / S) & 1;
        const int j = it / KB, kb = it % KB, buf = j % nbuf;
        if (kb == 0 && j >= nbuf) {
          mbar_wait(&acc_empty[buf], ((j - nbuf) / nbuf) & 1);
          tc_fence_after();
        }
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t A = smem_u32(smem + s * stage_bytes);
        const uint32_t Bt = A + 3 * kPlaneTile;
        const uint32_t d = tmem + buf * a.TT;
        // 16-k steps that hold data (the readout-fed layer: 20 classes of a 64-wide block)
        const int ksn = kb == KB - 1 ? min(4, (a.K - kb * 64 + 15) / 16) : 4;
        // (pa, pb) plane products with pa + pb <= planes - 1, smallest terms first:
        // 6 for the fp32 path, 3 (hi.hi + hi.mid + mid.hi) for planes = 2, 1 for bf16
        const int pa[10] = {2, 1, 0, 1, 0, 0, 1, 0, 0, 0};
        const int pb[10] = {0, 1, 2, 0, 1, 0, 0, 1, 0, 0};
        if (a.planes == 3) {  // the fp32 path, fully unrolled
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            if (ks >= ksn) break;
#pragma unroll
            for (int q = 0; q < 6; ++q) {
              const uint64_t ad = sdesc_sw128(A + pa[q] * kPlaneTile + ks * 32, 16, 1024);
              const uint64_t bd = sdesc_sw128(Bt + pb[q] * btile + ks * 2048, 8192, 1024);
              umma_bf16(d, ad, bd, idesc, (kb | ks | q) != 0);
            }
          }
        } else {
          const int q0 = a.planes == 2 ? 6 : 9, q1 = a.planes == 2 ? 9 : 10;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            for (int q = q0; q < q1; ++q) {
              const uint64_t ad = sdesc_sw128(A + pa[q] * kPlaneTile + ks * 32, 16, 1024);
              const uint64_t bd = sdesc_sw128(Bt + pb[q] * btile + ks * 2048, 8192, 1024);
              umma_bf16(d, ad, bd, idesc, (kb | ks | (q - q0)) != 0);
            }
          }
        }
        umma_commit(&empty[s]);
        if (kb == KB - 1) umma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else if constexpr (kDsOnly) {
    const int q = warp & 3, sg = warp >> 2;
    const int n = nt * 128 + q * 32 + lane;
    const int seg_len = a.TT / kBwdSeg;
    const float rterm = kReg ? monitor_term(a, b, n, sg, lane) : 0.0f;
    for (int j = 0; j < a.NT; ++j) {
      const int tt = a.NT - 1 - j, buf = j % nbuf;
      const int t_lo = tt * a.TT + sg * seg_len;
      const uint32_t tcol = tmem + (uint32_t(q * 32) << 16) + buf * a.TT + sg * seg_len;
      mbar_wait(&acc_full[buf], (j / nbuf) & 1);
      tc_fence_after();
      for (int c0 = 0; c0 < seg_len; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tcol + c0, r);
        tmem_ld_wait();
        if constexpr (kReg) add_dcount(r, rterm);
        float* dp = a.ds_out + (size_t(b) * a.T_pad + t_lo + c0) * a.H_pad + n;
#pragma unroll
        for (int e = 0; e < 16; ++e) dp[size_t(e) * a.H_pad] = __uint_as_float(r[e]);
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
  } else if constexpr (kAlif) {
    // ALIF scan warps (declared cell): the same segment structure as the LIF path
    // below with the two-state reverse step -- each segment composes its 2x2 affine
    // map (bwd_compose_alif), the maps are chained through smem, then every segment
    // replays its steps in the oracle's statement order (bwd_replay_alif).  V and
    // the adaptation a are read from HBM / L2 in both passes (no TMEM cache).
    const int q = warp & 3, sg = warp >> 2;
    const int sidx = sg * 128 + q * 32 + lane;
    const int n = nt * 128 + q * 32 + lane;
    const float vb = clip01(n < a.H ? a.beta[n * a.beta_stride] : 0.0f);
    const float gc = n < a.H ? clip01(a.gamma[n]) : 0.0f;
    const float omg = __fsub_rn(1.0f, gc);
    const float theta = a.theta;
    const size_t plane = size_t(a.H_pad) * cols_total;
    __nv_bfloat16* __restrict__ drow = a.di_planes + size_t(n) * cols_total + size_t(b) * a.T_pad;
    const float* __restrict__ vrow = a.v_in + size_t(b) * a.T_pad * a.H_pad + n;
    const float* __restrict__ arow = a.a_in + size_t(b) * a.T_pad * a.H_pad + n;
    const int seg_len = a.TT / kBwdSeg;
    const bool stage_out = a.NT == 1;
    float* xP = reinterpret_cast<float*>(smem + S * stage_bytes + 256);  // [4][256]
    float* xQ = xP + 4 * kBwdScanThreads;                                 // [2][256]
    float* xG = xQ + 2 * kBwdScanThreads;                                 // [2][256]
    const int last = (kBwdSeg - 1) * 128 + q * 32 + lane;
    float cv = 0.0f, ca = 0.0f;  // (gv, ga) entering the t-tile from above
    float db = 0.0f, dbias = 0.0f, dgam = 0.0f;
    const float rterm = kReg ? monitor_term(a, b, n, sg, lane) : 0.0f;
    for (int j = 0; j < a.NT; ++j) {
      const int tt = a.NT - 1 - j, buf = j % nbuf;
      const int t_lo = tt * a.TT + sg * seg_len;
      const int t_hi = min(t_lo + seg_len, a.T);
      const uint32_t tcol = tmem + (uint32_t(q * 32) << 16) + buf * a.TT + sg * seg_len;
      mbar_wait(&acc_full[buf], (j / nbuf) & 1);
      tc_fence_after();
      const float* vseg = vrow + size_t(t_lo) * a.H_pad;
      const float* aseg = arow + size_t(t_lo) * a.H_pad;
      const int top = seg_len - 16;
      float P[4] = {1.0f, 0.0f, 0.0f, 1.0f}, Q[2] = {0.0f, 0.0f};
      // one t-tile: the membranes are cached in TMEM columns TT.. between the passes
      const uint32_t vcol = tmem + (uint32_t(q * 32) << 16) + a.TT + sg * seg_len;
      for (int c0 = top; c0 >= 0; c0 -= 16) {
        const int nval = t_hi - (t_lo + c0);
        if (nval <= 0) continue;
        float vr[16], ar[16];
        load_v16(vseg + size_t(c0) * a.H_pad, a.H_pad, nval, vr);
        load_v16(aseg + size_t(c0) * a.H_pad, a.H_pad, nval, ar);
        if (vcache) tmem_st16(vcol + c0, vr);
        uint32_t r[16];
        tmem_ld16(tcol + c0, r);
        tmem_ld_wait();
        if constexpr (kReg) add_dcount(r, rterm);
        if (nval >= 16) bwd_compose_alif<kAct, false>(r, vr, ar, 16, vb, gc, omg, theta, a, P, Q);
        else bwd_compose_alif<kAct, true>(r, vr, ar, nval, vb, gc, omg, theta, a, P, Q);
      }
      if (vcache) tmem_st_wait();
#pragma unroll
      for (int i = 0; i < 4; ++i) xP[i * kBwdScanThreads + sidx] = P[i];
      xQ[sidx] = Q[0];
      xQ[kBwdScanThreads + sidx] = Q[1];
      if (sg == kBwdSeg - 1) {
        xG[sidx] = cv;
        xG[kBwdScanThreads + sidx] = ca;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kBwdScanThreads));
      float gv = xG[last], ga = xG[kBwdScanThreads + last];
      for (int s2 = kBwdSeg - 1; s2 > sg; --s2) {
        const int o = s2 * 128 + q * 32 + lane;
        const float ngv = xP[o] * gv + xP[kBwdScanThreads + o] * ga + xQ[o];
        ga = xP[2 * kBwdScanThreads + o] * gv + xP[3 * kBwdScanThreads + o] * ga + xQ[kBwdScanThreads + o];
        gv = ngv;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kBwdScanThreads));
      for (int c0 = top; c0 >= 0; c0 -= 16) {
        const int nval = t_hi - (t_lo + c0);
        if (nval <= 0) continue;
        float vr[16], ar[16];
        load_v16(aseg + size_t(c0) * a.H_pad, a.H_pad, nval, ar);
        uint32_t r[16];
        if (vcache) {
          uint32_t vv[16];
          tmem_ld16(vcol + c0, vv);
          tmem_ld16(tcol + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) vr[e] = __uint_as_float(vv[e]);
        } else {
          load_v16(vseg + size_t(c0) * a.H_pad, a.H_pad, nval, vr);
          tmem_ld16(tcol + c0, r);
          tmem_ld_wait();
        }
        if constexpr (kReg) add_dcount(r, rterm);
        if (a.dbg_ds != nullptr) {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (e < nval)
              a.dbg_ds[(size_t(b) * a.T_pad + t_lo + c0 + e) * a.H_pad + n] = __uint_as_float(r[e]);
        }
        float x[16];
        if (nval >= 16) bwd_replay_alif<kAct, false>(r, vr, ar, 16, vb, gc, omg, theta, a, gv, ga, db, dbias, dgam, x);
        else bwd_replay_alif<kAct, true>(r, vr, ar, nval, vb, gc, omg, theta, a, gv, ga, db, dbias, dgam, x);
        bwd_store_di16(x, stage_out, smem, sg * seg_len + c0, q, lane, a.TT, drow + t_lo + c0, plane);
      }
      if (sg == 0) {
        xG[last] = gv;
        xG[kBwdScanThreads + last] = ga;
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
      if (stage_out) fence_async_smem();
      asm volatile("bar.sync 1, %0;" ::"r"(kBwdScanThreads));
      cv = xG[last];
      ca = xG[kBwdScanThreads + last];
      if (stage_out && threadIdx.x == 0) {
        for (int p = 0; p < a.planes; ++p)  // consumers read the first `planes` planes
          for (int h = 0; h < a.TT / 64; ++h)
            tma_store_2d(&tm_out, smem + (p * (a.TT / 64) + h) * 16384, b * a.T_pad + h * 64,
                         p * a.H_pad + nt * 128);
        bulk_commit();
      }
    }
    // per-segment beta / bias / gamma partials combined in a fixed order
    if (sg > 0) {
      xP[sidx] = db;
      xP[kBwdScanThreads + sidx] = dbias;
      xP[2 * kBwdScanThreads + sidx] = dgam;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kBwdScanThreads));
    if (sg == 0) {
      for (int s2 = 1; s2 < kBwdSeg; ++s2) {
        const int o = s2 * 128 + q * 32 + lane;
        db = __fadd_rn(db, xP[o]);
        dbias = __fadd_rn(dbias, xP[kBwdScanThreads + o]);
        dgam = __fadd_rn(dgam, xP[2 * kBwdScanThreads + o]);
      }
      if (n < a.H) {
        a.dbeta_part[size_t(b) * a.H + n] = db;
        a.dgamma_part[size_t(b) * a.H + n] = dgam;
        if (a.dbias_part != nullptr) a.dbias_part[size_t(b) * a.H + n] = dbias;
      }
    }
  } else {
    // Scan warps: quadrant q (TMEM lanes 32q..32q+31 = neurons), time segment sg
    // of each t-tile.  G' = (bc - theta g) G + g dS is linear in G, so each
    // segment first composes its affine map, the maps are chained through smem,
    // then every segment replays its steps in the reference operation order.
    const int q = warp & 3, sg = warp >> 2;
    const int sidx = sg * 128 + q * 32 + lane;
    const int n = nt * 128 + q * 32 + lane;
    const float vb = clip01(n < a.H ? a.beta[n * a.beta_stride] : 0.0f);
    const float theta = a.theta, ntheta = -a.theta;
    const size_t plane = size_t(a.H_pad) * cols_total;
    __nv_bfloat16* __restrict__ drow = a.di_planes + size_t(n) * cols_total + size_t(b) * a.T_pad;
    const float* __restrict__ vrow = a.v_in + size_t(b) * a.T_pad * a.H_pad + n;
    const int seg_len = a.TT / kBwdSeg;  // multiple of 16
    // one t-tile: dI planes are staged in the (then idle) operand stages in the
    // SW128 layout of tm_out -- [plane][64-step half][128 rows][128 B] -- and
    // written by 6 TMA stores (long rows instead of 32-byte pieces of 128 rows)
    const bool stage_out = kStage == 0 && a.NT == 1;
    float Gcarry = 0.0f, db = 0.0f, dbias = 0.0f;
    float rterm = 0.0f;
    if constexpr (kReg) {
      // spike count over the window (monitor_activity, neuron.hpp:106-114)
      int count = -1;
      if (n < a.H) {
        const int wpb = a.T_pad / 32;
        const uint32_t* w = a.s_tp + size_t(n) * (size_t(a.B) * wpb) + size_t(b) * wpb;
        count = 0;
        for (int i = 0; i < wpb; ++i) count += __popc(__ldg(w + i));
        rterm = activity_dcount(a, count);
      }
      if (sg == 0) {  // one histogram entry per (sample, neuron), warp-aggregated
        const unsigned peers = __match_any_sync(0xffffffffu, count);
        if (count >= 0 && lane == __ffs(peers) - 1) atomicAdd(a.hist + count, unsigned(__popc(peers)));
      }
    }
    for (int j = 0; j < a.NT; ++j) {
      const int tt = a.NT - 1 - j, buf = j % nbuf;
      const int t_lo = tt * a.TT + sg * seg_len;               // first step of my segment
      const int t_hi = min(t_lo + seg_len, a.T);                // one past the last valid
      const uint32_t tcol = tmem + (uint32_t(q * 32) << 16) + buf * a.TT + sg * seg_len;
      // the membranes of the segment's top sub-chunk do not depend on the GEMM: their
      // loads are in flight across the accumulator wait
      const float* vseg = vrow + size_t(t_lo) * a.H_pad;
      const int top = seg_len - 16;
      float vr[16], vn[16];
      load_v16(vseg + size_t(top) * a.H_pad, a.H_pad, t_hi - (t_lo + top), vn);
      mbar_wait(&acc_full[buf], (j / nbuf) & 1);
      tc_fence_after();
      if (clk != nullptr && threadIdx.x == 0 && j == 0) clk[1] = clock64();
      // ---- pass 1: compose the segment's affine map, t descending.  The membranes
      // of the next 16-step sub-chunk are loaded while this one is processed.
      float A = 1.0f, Bc = 0.0f;
      // one t-tile: the surrogates of pass 1 are kept in spare TMEM columns for pass 3
      // (which re-reads V from L2 for the dbeta sum only)
      const uint32_t gcol = tmem + (uint32_t(q * 32) << 16) + a.TT + sg * seg_len;
      for (int c0 = top; c0 >= 0; c0 -= 16) {
        const int nval = t_hi - (t_lo + c0);
#pragma unroll
        for (int e = 0; e < 16; ++e) vr[e] = vn[e];
        // next: c0 - 16, or (end of pass 1) the top sub-chunk for pass 3
        const int cn = c0 >= 16 ? c0 - 16 : top;
        load_v16(vseg + size_t(cn) * a.H_pad, a.H_pad, t_hi - (t_lo + cn), vn);
        if (nval <= 0) continue;
        uint32_t r[16];
        tmem_ld16(tcol + c0, r);
        tmem_ld_wait();
        if constexpr (kReg) add_dcount(r, rterm);
        float gk[16];
        if (nval >= 16) bwd_compose<kAct, false>(r, vr, 16, vb, theta, a, A, Bc, gk);
        else bwd_compose<kAct, true>(r, vr, nval, vb, theta, a, A, Bc, gk);
        if (vcache) tmem_st16(gcol + c0, gk);
      }
      if (vcache) tmem_st_wait();
      xA[sidx] = A;
      xB[sidx] = Bc;
      if (sg == kBwdSeg - 1) xG[sidx] = Gcarry;
      asm volatile("bar.sync 1, %0;" ::"r"(kBwdScanThreads));
      if (clk != nullptr && threadIdx.x == 0 && j == 0) clk[2] = clock64();
      // chain the maps: segment s starts from the G leaving segment s+1
      float G = xG[(kBwdSeg - 1) * 128 + q * 32 + lane];
      for (int s2 = kBwdSeg - 1; s2 > sg; --s2) G = xA[s2 * 128 + q * 32 + lane] * G + xB[s2 * 128 + q * 32 + lane];
      asm volatile("bar.sync 1, %0;" ::"r"(kBwdScanThreads));
      if (clk != nullptr && threadIdx.x == 0 && j == 0) clk[3] = clock64();
      // ---- pass 3: exact-order replay of my segment
      for (int c0 = top; c0 >= 0; c0 -= 16) {
        const int nval = t_hi - (t_lo + c0);
        uint32_t r[16], gv[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) vr[e] = vn[e];
        if (c0 >= 16) load_v16(vseg + size_t(c0 - 16) * a.H_pad, a.H_pad, t_hi - (t_lo + c0 - 16), vn);
        if (nval <= 0) continue;
        if (vcache) tmem_ld16(gcol + c0, gv);
        tmem_ld16(tcol + c0, r);
        tmem_ld_wait();
        if constexpr (kReg) add_dcount(r, rterm);
        if (a.dbg_ds != nullptr) {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (e < nval)
              a.dbg_ds[(size_t(b) * a.T_pad + t_lo + c0 + e) * a.H_pad + n] = __uint_as_float(r[e]);
        }
        float x[16];
        if (vcache) {
          if (nval >= 16) bwd_replay_g<false>(r, vr, gv, 16, vb, theta, G, db, dbias, x);
          else bwd_replay_g<true>(r, vr, gv, nval, vb, theta, G, db, dbias, x);
        } else {
          if (nval >= 16) bwd_replay<kAct, false>(r, vr, 16, vb, theta, a, G, db, dbias, x);
          else bwd_replay<kAct, true>(r, vr, nval, vb, theta, a, G, db, dbias, x);
        }
        uint32_t ph_[8], pm_[8], pl_[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) split3_pack(x[e], x[e + 1], ph_[e / 2], pm_[e / 2], pl_[e / 2]);
#if SNN_BWD_EXP == 1
        if (ph_[0] == 0x12345u && pm_[1] == 0x777u) {  // timing experiment: stores never taken
#else
        if (stage_out) {
          const int tl = sg * seg_len + c0;  // step within the tile (multiple of 16)
          const uint32_t row = uint32_t(q * 32 + lane);
          const uint32_t base = smem_u32(smem) + uint32_t(tl >> 6) * 16384u + row * 128u;
          const uint32_t j0 = uint32_t(tl & 63) >> 3;
          const uint32_t o0 = ((j0 ^ (row & 7u)) << 4), o1 = (((j0 + 1u) ^ (row & 7u)) << 4);
          const uint32_t pstride = uint32_t(a.TT / 64) * 16384u;
          st_shared_v4(base + o0, make_uint4(ph_[0], ph_[1], ph_[2], ph_[3]));
          st_shared_v4(base + o1, make_uint4(ph_[4], ph_[5], ph_[6], ph_[7]));
          st_shared_v4(base + pstride + o0, make_uint4(pm_[0], pm_[1], pm_[2], pm_[3]));
          st_shared_v4(base + pstride + o1, make_uint4(pm_[4], pm_[5], pm_[6], pm_[7]));
          st_shared_v4(base + 2 * pstride + o0, make_uint4(pl_[0], pl_[1], pl_[2], pl_[3]));
          st_shared_v4(base + 2 * pstride + o1, make_uint4(pl_[4], pl_[5], pl_[6], pl_[7]));
        } else {
#endif
        if constexpr (kStage == 2) {
          // whole 32-byte sectors (two 16-byte halves would each be a partial write)
          st_global_v8(drow + t_lo + c0, ph_);
          st_global_v8(drow + plane + t_lo + c0, pm_);
          st_global_v8(drow + 2 * plane + t_lo + c0, pl_);
        } else {
          uint4* dh = reinterpret_cast<uint4*>(drow + t_lo + c0);
          uint4* dm = reinterpret_cast<uint4*>(drow + plane + t_lo + c0);
          uint4* dl = reinterpret_cast<uint4*>(drow + 2 * plane + t_lo + c0);
          dh[0] = make_uint4(ph_[0], ph_[1], ph_[2], ph_[3]);
          dh[1] = make_uint4(ph_[4], ph_[5], ph_[6], ph_[7]);
          dm[0] = make_uint4(pm_[0], pm_[1], pm_[2], pm_[3]);
          dm[1] = make_uint4(pm_[4], pm_[5], pm_[6], pm_[7]);
          dl[0] = make_uint4(pl_[0], pl_[1], pl_[2], pl_[3]);
          dl[1] = make_uint4(pl_[4], pl_[5], pl_[6], pl_[7]);
        }
        }
      }
      if (clk != nullptr && threadIdx.x == 0 && j == 0) clk[4] = clock64();
      // the earliest segment's final G carries into the previous t-tile
      if (sg == 0) xG[(kBwdSeg - 1) * 128 + q * 32 + lane] = G;
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
      if (stage_out) fence_async_smem();  // staged planes -> visible to the TMA stores
      asm volatile("bar.sync 1, %0;" ::"r"(kBwdScanThreads));
      Gcarry = xG[(kBwdSeg - 1) * 128 + q * 32 + lane];
      if (stage_out && threadIdx.x == 0) {
        for (int p = 0; p < a.planes; ++p)  // consumers read the first `planes` planes
          for (int h = 0; h < a.TT / 64; ++h)
            tma_store_2d(&tm_out, smem + (p * (a.TT / 64) + h) * 16384, b * a.T_pad + h * 64,
                         p * a.H_pad + nt * 128);
        bulk_commit();
      }
    }
    if (clk != nullptr && threadIdx.x == 0) clk[5] = clock64();
    // combine the per-segment dbeta / dbias partials in a fixed order
    if (sg > 0) {
      xA[sidx] = db;
      xB[sidx] = dbias;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kBwdScanThreads));
    if (sg == 0) {
      for (int s2 = 1; s2 < kBwdSeg; ++s2) {
        db = __fadd_rn(db, xA[s2 * 128 + q * 32 + lane]);
        dbias = __fadd_rn(dbias, xB[s2 * 128 + q * 32 + lane]);
      }
      if (n < a.H) {
        a.dbeta_part[size_t(b) * a.H + n] = db;
        if (a.dbias_part != nullptr) a.dbias_part[size_t(b) * a.H + n] = dbias;
      }
    }
  }
  pdl_launch_dependents();
  if (threadIdx.x == 0) bulk_wait_read_all();  // staged planes read before smem is released
  __syncthreads();
  if (clk != nullptr && threadIdx.x == 0) {
    clk[6] = clock64();
    clk[15] = globaltimer();
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_any(tmem_cols, tmem);
  }
}

// ============================================================================
// K2r / K3r  the DECLARED RLIF cell (not in the reference; oracle/spiketrain_oracle.h).
// The input projection I = A W runs on tcgen05 in k_lif_fwd (FwdLayer.i_out: no
// scan); the recurrence couples every neuron of a sample at every step, so the
// scan is its own kernel: one CTA per sample, one thread per neuron.
//   forward : s_t from the incoming v; fb_j = sum over spiking i ascending of
//             rec[i][j] (exact: the oracle's zero-skip row order); the spiking set
//             of a step is the block's warp ballots (smem, double-buffered, one
//             barrier per step); v' = (((v bc) + I) + fb) - s theta.
//   backward: dS from k_lif_bwd<., ., false, true> (dS only); per step t
//             descending rc_i = sum_j rec[i][j] G_j over the CTA's kSB samples
//             (rec^T rows coalesced over i, G broadcast from smem),
//             gs = (dS + (-G) theta) + rc ; G' = G bc + gs g(v - theta);
//             dI = G as bf16 planes, beta / bias partials per sample.
// d rec = S^T dI of the layer with itself runs in k_wgrad as an extra layer.
// ============================================================================
struct RlifFwdArgs {
  const float* i_in;      // [B][T_pad][H_pad] projection (+ bias)
  const float* beta;      // [H] or one value (beta_stride 0)
  int beta_stride;
  const float* rec;       // [H][H] (row = source neuron), the parameter itself
  float* v_out;           // [B][T_pad][H_pad]
  uint32_t* s_np;         // [B][T_pad][H_pad/32]
  uint32_t* s_tp;         // [H_pad][B*T_pad/32]
  int B, T, T_pad, H, H_pad;
  int sb;                 // cluster form: samples per cluster
  float theta;
};

__global__ void __launch_bounds__(1024) k_rlif_fwd(RlifFwdArgs a) {
  __shared__ uint32_t words[2][32];
  pdl_wait();
  const int b = blockIdx.x, n = threadIdx.x, lane = n & 31, w = n >> 5;
  const int nw = a.H_pad / 32;
  const float vb = clip01(n < a.H ? a.beta[n * a.beta_stride] : 0.0f);
  const float theta = a.theta, ntheta = -a.theta;
  const float* __restrict__ ip = a.i_in + size_t(b) * a.T_pad * a.H_pad + n;
  float* __restrict__ vp = a.v_out + size_t(b) * a.T_pad * a.H_pad + n;
  const size_t tp_words = size_t(a.B) * a.T_pad / 32;
  const float* __restrict__ recn = a.rec + (n < a.H ? n : 0);  // column n
  float v = 0.0f;
  uint32_t tmask = 0u;
  float I = __ldg(ip);
  for (int t = 0; t < a.T_pad; ++t) {
    const float In = t + 1 < a.T_pad ? __ldg(ip + size_t(t + 1) * a.H_pad) : 0.0f;
    vp[size_t(t) * a.H_pad] = v;
    const bool sp = __fadd_rn(v, ntheta) >= 0.0f && n < a.H && t < a.T;
    const uint32_t bal = __ballot_sync(0xffffffffu, sp);
    if (lane == 0) {
      words[t & 1][w] = bal;
      a.s_np[(size_t(b) * a.T_pad + t) * nw + w] = bal;
    }
    tmask |= uint32_t(sp) << (t & 31);
    if ((t & 31) == 31) {
      a.s_tp[size_t(n) * tp_words + size_t(b) * (a.T_pad / 32) + t / 32] = tmask;
      tmask = 0u;
    }
    __syncthreads();
    float fb = 0.0f;
    if (n < a.H) {
      for (int q = 0; q < nw; ++q) {
        uint32_t m = words[t & 1][q];
        while (m != 0u) {
          // up to 8 sources per round: the loads issue before the ordered adds
          float xs[8];
          int k = 0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (m != 0u) {
              const int i = q * 32 + __ffs(m) - 1;
              m &= m - 1u;
              xs[u] = __ldg(recn + size_t(i) * a.H);
              k = u + 1;
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (u < k) fb = __fadd_rn(fb, xs[u]);
        }
      }
    }
    const float ai = __fadd_rn(__fmul_rn(v, vb), I);
    v = __fsub_rn(__fadd_rn(ai, fb), sp ? theta : 0.0f);
    I = In;
  }
  pdl_launch_dependents();
}

struct RlifBwdArgs {
  const float* ds;             // [B][T_pad][H_pad] dS of this layer
  const float* v_in;           // [B][T_pad][H_pad]
  const float* beta;
  int beta_stride;
  const float* rec_t;          // [H][H_pad]: rec_t[j][i] = rec[i][j] (refreshed by Adam)
  const float* rec;            // [H][H] the parameter (k_rlif_bwd_tc builds its bf16 planes)
  __nv_bfloat16* di_planes;    // out: dI planes [3][H_pad][B*T_pad]
  float* dbeta_part;           // [B][H]
  float* dbias_part;           // [B][H] or nullptr
  int B, T, T_pad, H, H_pad;
  int sb;                      // cluster form: samples per cluster
  float theta, slope, aux;
};

template <int kAct, int kSB>
__global__ void __launch_bounds__(1024) k_rlif_bwd(RlifBwdArgs a) {
  extern __shared__ float gsm[];  // [2][kSB][H_pad]: G of every neuron, this step
  pdl_wait();
  const int b0 = blockIdx.x * kSB, i = threadIdx.x;
  const bool live = i < a.H;
  const float vb = clip01(live ? a.beta[i * a.beta_stride] : 0.0f);
  const float theta = a.theta;
  const size_t cols_total = size_t(a.B) * a.T_pad;
  const size_t plane = size_t(a.H_pad) * cols_total;
  const float* __restrict__ rt = a.rec_t + i;
  float G[kSB], db[kSB], dbias[kSB];
#pragma unroll
  for (int s = 0; s < kSB; ++s) G[s] = db[s] = dbias[s] = 0.0f;
  int par = 0;
  for (int c0 = a.T_pad - 16; c0 >= 0; c0 -= 16) {
    float x[kSB][16];
#pragma unroll
    for (int e = 15; e >= 0; --e) {
      const int t = c0 + e;
#pragma unroll
      for (int s = 0; s < kSB; ++s) {
        gsm[(par * kSB + s) * a.H_pad + i] = G[s];
        x[s][e] = G[s];
      }
      if (t >= a.T) {  // padded steps: G stays 0, dI 0
        par ^= 1;
        continue;
      }
      float dS[kSB], V[kSB];
#pragma unroll
      for (int s = 0; s < kSB; ++s) {
        const size_t idx = (size_t(b0 + s) * a.T_pad + t) * a.H_pad + i;
        dS[s] = b0 + s < a.B ? __ldg(a.ds + idx) : 0.0f;
        V[s] = b0 + s < a.B ? __ldg(a.v_in + idx) : 0.0f;
      }
      __syncthreads();
      float rc[kSB];
#pragma unroll
      for (int s = 0; s < kSB; ++s) rc[s] = 0.0f;
      if (live) {
        const float* gp = gsm + par * kSB * a.H_pad;
#pragma unroll 4
        for (int j = 0; j < a.H; ++j) {
          const float r = __ldg(rt + size_t(j) * a.H_pad);
#pragma unroll
          for (int s = 0; s < kSB; ++s) rc[s] = __fadd_rn(rc[s], __fmul_rn(r, gp[s * a.H_pad + j]));
        }
      }
#pragma unroll
      for (int s = 0; s < kSB; ++s) {
        const float gi = G[s];
        const float gs = __fadd_rn(__fadd_rn(dS[s], __fmul_rn(-gi, theta)), rc[s]);
        const float g = surrogate_t<kAct>(a.slope, a.aux, __fadd_rn(V[s], -theta));
        db[s] = __fadd_rn(db[s], __fmul_rn(gi, V[s]));
        dbias[s] = __fadd_rn(dbias[s], gi);
        G[s] = live ? __fadd_rn(__fmul_rn(gi, vb), __fmul_rn(gs, g)) : 0.0f;
      }
      par ^= 1;
    }
#pragma unroll
    for (int s = 0; s < kSB; ++s)
      if (b0 + s < a.B)
        bwd_store_di16(x[s], false, nullptr, 0, 0, 0, 0,
                       a.di_planes + size_t(i) * cols_total + size_t(b0 + s) * a.T_pad + c0, plane);
  }
  if (live) {
#pragma unroll
    for (int s = 0; s < kSB; ++s)
      if (b0 + s < a.B) {
        a.dbeta_part[size_t(b0 + s) * a.H + i] = db[s];
        if (a.dbias_part != nullptr) a.dbias_part[size_t(b0 + s) * a.H + i] = dbias[s];
      }
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// Cluster forms of the RLIF scans (256 <= H_pad <= 512): the H neurons of a
// sample group are split over a cluster of kRlCl CTAs, each keeping its slice of
// rec in shared memory (128 KB at H = 512) instead of re-reading it from L2 every
// step; the per-step exchange (spike words forward, G backward) goes to every
// CTA of the cluster through DSMEM stores, then one cluster barrier per step
// (it also retires the double-buffered exchange slot of the step before).
constexpr int kRlCl = 8;      // CTAs per cluster = neuron slices
constexpr int kRlSBMax = 32;  // samples per cluster (runtime a.sb <= this, multiple of 4)
constexpr int kRlSPT = 4;     // backward: samples per thread
constexpr int kRlFPT = 2;     // forward: samples per thread
__host__ __device__ constexpr size_t rlif_fwd_cl_smem(int H, int H_pad, int sb) {
  // rec slice + double-buffered spike words + 2 mbarriers + per-warp source lists
  return size_t(H) * (H_pad / kRlCl) * 4 + size_t(2) * sb * (H_pad / 32) * 4 + 16 +
         size_t(sb / kRlFPT) * kRlFPT * H_pad * 2;
}
__host__ __device__ constexpr size_t rlif_bwd_cl_smem(int H, int H_pad, int sb) {
  return size_t(H) * (H_pad / kRlCl) * 4 + size_t(2) * H_pad * sb * 4;
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// remote shared store that completes 4 tx bytes on the receiver's mbarrier
__device__ __forceinline__ void st_async_u32(uint32_t raddr, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr), "r"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAITW:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, 10000000;\n\t"
      "@P1 bra DONEW;\n\t"
      "bra LAB_WAITW;\n\t"
      "DONEW:\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float x, float y, float z, float w) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(x), "f"(y), "f"(z),
               "f"(w)
               : "memory");
}

#ifndef SNN_RT_EXP
#define SNN_RT_EXP 0  // timing experiments only (RLIF scans): 1 no MMA, 2 no cross-CTA wait /
                      // copies, 3 no reverse step, 4 / 5 backward / forward phase clocks
#endif
// Forward: CTA c of the cluster owns output neurons [c NS, (c+1) NS) of a.sb
// samples.  Lane l of a warp owns neurons l + 32 h (h < kNPT = NS / 32) of one
// sample group (kRlFPT samples s, s + sb/kRlFPT, ...); its smem holds rec[:, slice]
// as recs[i][kNPT l + h], so one vector load per spiking source feeds all its
// neurons.  Same statements and ascending source order as k_rlif_fwd: bit-identical.
template <int kNPT>
__global__ void __launch_bounds__(1024) k_rlif_fwd_cl(RlifFwdArgs a) {
  extern __shared__ __align__(16) float rsm[];
  constexpr int NS = 32 * kNPT;
  const int nw = a.H_pad / 32, SB = a.sb, SBT = a.sb / kRlFPT;
  float* recs = rsm;                                                     // [H][NS] permuted
  uint32_t* words = reinterpret_cast<uint32_t*>(rsm + size_t(a.H) * NS);  // [2][SB][nw]
  uint64_t* wfull = reinterpret_cast<uint64_t*>(words + 2 * SB * nw);     // [2] words of a step landed
  const uint32_t crank = cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, s0 = tid >> 5;
  // this warp's ascending spiking-source lists, one per sample it owns
  uint16_t* slist = reinterpret_cast<uint16_t*>(wfull + 2) + size_t(s0) * kRlFPT * a.H_pad;
  if (tid == 0) {
    mbar_init(&wfull[0], 1);
    mbar_init(&wfull[1], 1);
    fence_barrier_init();
  }
  pdl_wait();
  for (int idx = tid; idx < a.H * NS; idx += blockDim.x) {
    const int i = idx / NS, q = idx % NS;                    // q = kNPT l + h
    const int c = int(crank) * NS + (q / kNPT) + 32 * (q % kNPT);
    recs[idx] = c < a.H ? a.rec[size_t(i) * a.H + c] : 0.0f;
  }
  const float theta = a.theta, ntheta = -a.theta;
  const size_t tp_words = size_t(a.B) * a.T_pad / 32;
  int j[kNPT];
  float vb[kNPT];
#pragma unroll
  for (int h = 0; h < kNPT; ++h) {
    j[h] = int(crank) * NS + lane + 32 * h;
    vb[h] = clip01(j[h] < a.H ? a.beta[j[h] * a.beta_stride] : 0.0f);
  }
  const int wi0 = int(crank) * kNPT;  // the slice's first spike word
  int b[kRlFPT];
  bool bl[kRlFPT];
  size_t base[kRlFPT];
  float v[kRlFPT][kNPT], I[kRlFPT][kNPT];
  uint32_t tmask[kRlFPT][kNPT];
#pragma unroll
  for (int u = 0; u < kRlFPT; ++u) {
    b[u] = blockIdx.y * SB + s0 + u * SBT;
    bl[u] = b[u] < a.B;
    base[u] = (size_t(bl[u] ? b[u] : 0) * a.T_pad) * a.H_pad;
#pragma unroll
    for (int h = 0; h < kNPT; ++h) {
      v[u][h] = 0.0f;
      tmask[u][h] = 0u;
      I[u][h] = bl[u] ? __ldg(a.i_in + base[u] + j[h]) : 0.0f;
    }
  }
  cluster_sync_all();  // every CTA's barriers initialised before any remote store
  // per step the spike words go to every CTA with st.async completing the receiver's
  // mbarrier (SB * nw words per step) -- no cluster barrier, no fence over the
  // step's global stores.  Slot reuse two steps later is safe: a CTA sends step t+2
  // only after receiving every CTA's step t+1 words, each sent after its step t gather.
  const uint32_t step_bytes = uint32_t(SB * nw) * 4u;
  const uint32_t wbar0 = smem_u32(wfull);
#if SNN_RT_EXP == 5
  __shared__ long long fclk[24][4];
  const bool fprobe = blockIdx.x == 0 && blockIdx.y == 0 && tid == 0;
#define RF_CLK(k) if (fprobe && t < 24) fclk[t][k] = globaltimer();
#else
#define RF_CLK(k)
#endif
  for (int t = 0; t < a.T_pad; ++t) {
    const int par = t & 1;
    RF_CLK(0)
    if (tid == 0) mbar_arrive_expect_tx(&wfull[par], step_bytes);
    bool sp[kRlFPT][kNPT];
    float In[kRlFPT][kNPT];
#pragma unroll
    for (int u = 0; u < kRlFPT; ++u)
#pragma unroll
      for (int h = 0; h < kNPT; ++h) {
        const size_t o = base[u] + size_t(t) * a.H_pad + j[h];
        In[u][h] = (bl[u] && t + 1 < a.T_pad) ? __ldg(a.i_in + o + a.H_pad) : 0.0f;
        if (bl[u]) a.v_out[o] = v[u][h];
        sp[u][h] = __fadd_rn(v[u][h], ntheta) >= 0.0f && j[h] < a.H && t < a.T && bl[u];
        const uint32_t bal = __ballot_sync(0xffffffffu, sp[u][h]);
        const uint32_t slot = smem_u32(words + (par * SB + s0 + u * SBT) * nw + wi0 + h);
        if (lane < kRlCl)  // lane r -> rank r
          st_async_u32(map_rank(slot, uint32_t(lane)), bal, map_rank(wbar0 + 8u * uint32_t(par), uint32_t(lane)));
        if (lane == 0 && bl[u]) a.s_np[(size_t(b[u]) * a.T_pad + t) * nw + wi0 + h] = bal;
        tmask[u][h] |= uint32_t(sp[u][h]) << (t & 31);
        if ((t & 31) == 31) {
          if (bl[u]) a.s_tp[size_t(j[h]) * tp_words + size_t(b[u]) * (a.T_pad / 32) + t / 32] = tmask[u][h];
          tmask[u][h] = 0u;
        }
      }
    RF_CLK(1)
    mbar_wait_acq_cluster(&wfull[par], uint32_t(t >> 1) & 1u);
    RF_CLK(2)
#pragma unroll
    for (int u = 0; u < kRlFPT; ++u) {
      float fb[kNPT];
#pragma unroll
      for (int h = 0; h < kNPT; ++h) fb[h] = 0.0f;
      // the warp turns the sample's words into an ascending source list once (lane q
      // expands word q at its exclusive prefix), then every lane walks the list
      const uint32_t* wp = words + (par * SB + s0 + u * SBT) * nw;
      uint16_t* li = slist + u * a.H_pad;
      const uint32_t wq = lane < nw ? wp[lane] : 0u;
      const int cq = __popc(wq);
      int pre = cq;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, pre, d);
        if (lane >= d) pre += y;
      }
      const int total = __shfl_sync(0xffffffffu, pre, 31);
      pre -= cq;
      for (uint32_t m = wq; m != 0u; m &= m - 1u) li[pre++] = uint16_t(lane * 32 + __ffs(m) - 1);
      __syncwarp();
      int k = 0;
      for (; k + 4 <= total; k += 4) {
        const uint2 q4 = *reinterpret_cast<const uint2*>(li + k);  // 4 indices, broadcast
        const int i4[4] = {int(q4.x & 0xFFFFu), int(q4.x >> 16), int(q4.y & 0xFFFFu), int(q4.y >> 16)};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if constexpr (kNPT == 2) {
            const float2 r2 = *reinterpret_cast<const float2*>(recs + i4[e] * NS + 2 * lane);
            fb[0] = __fadd_rn(fb[0], r2.x);
            fb[1] = __fadd_rn(fb[1], r2.y);
          } else {
            fb[0] = __fadd_rn(fb[0], recs[i4[e] * NS + lane]);
          }
        }
      }
      for (; k < total; ++k) {
        const int i = li[k];
        if constexpr (kNPT == 2) {
          const float2 r2 = *reinterpret_cast<const float2*>(recs + i * NS + 2 * lane);
          fb[0] = __fadd_rn(fb[0], r2.x);
          fb[1] = __fadd_rn(fb[1], r2.y);
        } else {
          fb[0] = __fadd_rn(fb[0], recs[i * NS + lane]);
        }
      }
      __syncwarp();  // the list is rebuilt next step
#pragma unroll
      for (int h = 0; h < kNPT; ++h) {
        const float ai = __fadd_rn(__fmul_rn(v[u][h], vb[h]), I[u][h]);
        v[u][h] = __fsub_rn(__fadd_rn(ai, fb[h]), sp[u][h] ? theta : 0.0f);
        I[u][h] = In[u][h];
      }
    }
    RF_CLK(3)
  }
#if SNN_RT_EXP == 5
  if (fprobe)
    for (int k = 1; k < 24; ++k)
      printf("fwd step %d: send %lld wait %lld gather %lld | step %lld\n", k, fclk[k][1] - fclk[k][0],
             fclk[k][2] - fclk[k][1], fclk[k][3] - fclk[k][2], fclk[k][0] - fclk[k - 1][0]);
#endif
  pdl_launch_dependents();
  cluster_sync_all();  // no CTA leaves while a peer may still address its smem
}

// Backward: CTA c owns source neurons i in [c NS, (c+1) NS) -- rec[slice, :] in smem
// as recs[j][il] (conflict-free over il) -- and thread = (neuron, kRlSPT samples).
// Per step: rc over every j from the exchanged G of this step (smem, broadcast;
// fused multiply-adds: the backward is held to the 1e-4 bar, not bit-exactness),
// the reverse LIF step, then G' of its neuron to every CTA's exchange slot.
// The next step's dS / V are loaded while this step's rc sum runs.
template <int kAct>
__global__ void __launch_bounds__(512) k_rlif_bwd_cl(RlifBwdArgs a) {
  extern __shared__ __align__(16) float rsm[];
  const int NS = a.H_pad / kRlCl, SB = a.sb;
  float* recs = rsm;                             // [H][NS]
  float* gbuf = rsm + size_t(a.H) * NS;          // [2][H_pad][SB]
  const uint32_t crank = cluster_ctarank();
  const int tid = threadIdx.x;
  const int il = tid % NS, sg = tid / NS;
  const int i = int(crank) * NS + il;
  const bool live = i < a.H;
  const int b0 = blockIdx.y * SB + sg * kRlSPT;
  pdl_wait();
  for (int idx = tid; idx < a.H * NS; idx += blockDim.x) {
    const int jj = idx / NS, c = int(crank) * NS + idx % NS;
    recs[idx] = a.rec_t[size_t(jj) * a.H_pad + c];  // rec[c][jj] (0 for padded c)
  }
  for (int idx = tid; idx < 2 * a.H_pad * SB; idx += blockDim.x) gbuf[idx] = 0.0f;
  const float vb = clip01(live ? a.beta[i * a.beta_stride] : 0.0f);
  const float theta = a.theta;
  const size_t cols_total = size_t(a.B) * a.T_pad;
  const size_t plane = size_t(a.H_pad) * cols_total;
  const uint32_t gslot = smem_u32(gbuf + size_t(i) * SB + sg * kRlSPT);
  // sample s of the thread: element (t) at base + s * sstride + t * H_pad (s < nok)
  const int nok = max(0, min(kRlSPT, a.B - b0));
  const size_t sstride = size_t(a.T_pad) * a.H_pad;
  const size_t rbase = size_t(nok > 0 ? b0 : 0) * sstride + i;
  cluster_sync_all();
  float G[kRlSPT], db[kRlSPT], dbias[kRlSPT], dSn[kRlSPT], Vn[kRlSPT];
#pragma unroll
  for (int s = 0; s < kRlSPT; ++s) {
    G[s] = db[s] = dbias[s] = 0.0f;
    const size_t o = rbase + s * sstride + size_t(a.T - 1) * a.H_pad;
    dSn[s] = s < nok ? __ldg(a.ds + o) : 0.0f;
    Vn[s] = s < nok ? __ldg(a.v_in + o) : 0.0f;
  }
  int par = 0;
  for (int c0 = a.T_pad - 8; c0 >= 0; c0 -= 8) {
    float x[kRlSPT][8];
#pragma unroll
    for (int e = 7; e >= 0; --e) {
      const int t = c0 + e;
#pragma unroll
      for (int s = 0; s < kRlSPT; ++s) x[s][e] = G[s];
      if (t >= a.T) continue;  // padded steps: G stays 0 (uniform over the cluster)
      float dS[kRlSPT], V[kRlSPT];
#pragma unroll
      for (int s = 0; s < kRlSPT; ++s) {
        dS[s] = dSn[s];
        V[s] = Vn[s];
        const size_t o = rbase + s * sstride + size_t(t - 1) * a.H_pad;
        dSn[s] = (s < nok && t > 0) ? __ldg(a.ds + o) : 0.0f;
        Vn[s] = (s < nok && t > 0) ? __ldg(a.v_in + o) : 0.0f;
      }
      float rc0 = 0.0f, rc1 = 0.0f, rc2 = 0.0f, rc3 = 0.0f;
      const float* gp = gbuf + size_t(par) * a.H_pad * SB + sg * kRlSPT;
#pragma unroll 8
      for (int jj = 0; jj < a.H; ++jj) {
        const float r = recs[jj * NS + il];
        const float4 g4 = *reinterpret_cast<const float4*>(gp + jj * SB);
        rc0 = __fmaf_rn(r, g4.x, rc0);
        rc1 = __fmaf_rn(r, g4.y, rc1);
        rc2 = __fmaf_rn(r, g4.z, rc2);
        rc3 = __fmaf_rn(r, g4.w, rc3);
      }
      const float rc[kRlSPT] = {rc0, rc1, rc2, rc3};
#pragma unroll
      for (int s = 0; s < kRlSPT; ++s) {
        const float gi = G[s];
        const float gs = __fadd_rn(__fadd_rn(dS[s], __fmul_rn(-gi, theta)), rc[s]);
        const float g = surrogate_t<kAct>(a.slope, a.aux, __fadd_rn(V[s], -theta));
        db[s] = __fadd_rn(db[s], __fmul_rn(gi, V[s]));
        dbias[s] = __fadd_rn(dbias[s], gi);
        G[s] = live ? __fadd_rn(__fmul_rn(gi, vb), __fmul_rn(gs, g)) : 0.0f;
      }
      const uint32_t dst = gslot + uint32_t((par ^ 1) * a.H_pad * SB) * 4u;
#pragma unroll
      for (int r = 0; r < kRlCl; ++r) st_cluster_v4(map_rank(dst, uint32_t(r)), G[0], G[1], G[2], G[3]);
      cluster_sync_all();
      par ^= 1;
    }
    if (live) {
#pragma unroll
      for (int s = 0; s < kRlSPT; ++s)
        if (s < nok) {  // 8 steps of dI as 3 bf16 planes: one 16-byte store per plane
          uint32_t h[4], m[4], lo[4];
#pragma unroll
          for (int e = 0; e < 8; e += 2) split3_pack(x[s][e], x[s][e + 1], h[e / 2], m[e / 2], lo[e / 2]);
          uint4* d = reinterpret_cast<uint4*>(a.di_planes + size_t(i) * cols_total + size_t(b0 + s) * a.T_pad + c0);
          d[0] = make_uint4(h[0], h[1], h[2], h[3]);
          d[plane / 8] = make_uint4(m[0], m[1], m[2], m[3]);
          d[plane / 4] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
    }
  }
  if (live) {
#pragma unroll
    for (int s = 0; s < kRlSPT; ++s)
      if (s < nok) {
        a.dbeta_part[size_t(b0 + s) * a.H + i] = db[s];
        if (a.dbias_part != nullptr) a.dbias_part[size_t(b0 + s) * a.H + i] = dbias[s];
      }
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// K3t  k_rlif_bwd_tc: the RLIF reverse scan with the per-step recurrent product on
// tcgen05 (H_pad = 512).  Cluster of 8 CTAs x kRtN samples; CTA c owns the 64
// source neurons of slice c.  Per step t (descending):
//   rc[i][s] = sum_j rec[i][j] G_j(t+1)[s] as ONE M=128 x N=2 kRtN x K=512 chain:
//   A = [rec_hi; rec_lo] of the slice stacked along M (bf16, K-major SW128, resident
//   in smem), B = [G_hi; G_lo] of every neuron stacked along N, so
//     D[il][s] + D[il][kRtN + s] + D[64 + il][s] = hi.hi + hi.lo + lo.hi
//   (~2^-16 relative per product; the backward is held to the 1e-4 gradient bar;
//   lo.lo in D[64 + il][kRtN + s] is added too).  Warps 0-1 read the hi rows (TMEM
//   lanes 0-63), warps 2-3 the lo rows; they swap the partial sums of the other
//   half's samples through smem, then thread (neuron, half) runs the reverse LIF step
//   for kRtN/2 samples and writes G(t) as hi / lo bf16 into a local staging copy of
//   its k-block of B (the slice is exactly k-block c, same SW128 layout).  One
//   thread pushes the 4 KB k-block to every CTA with bulk shared->shared copies
//   (TMA engine) completing the receiver's mbarrier transaction count -- no cluster
//   barrier per step.  B is double-buffered: a CTA can only produce G(t) after every
//   CTA's G(t+1) arrived, i.e. after every CTA finished the MMA that read the
//   buffer it overwrites (and so did every copy out of a staging parity).
// ---------------------------------------------------------------------------
constexpr int kRtN = 24;                          // samples per cluster (11 clusters at B=256: one wave)
constexpr int kRtH = kRtN / 4;                    // samples per epilogue thread
constexpr int kRtEpiWarps = 8;                    // warps 0-7 epilogue (0-3 also read TMEM)
constexpr int kRtMmaWarp = kRtEpiWarps;           // warp 8: MMA issue + copies
constexpr int kRtThreads = 32 * (kRtEpiWarps + 1);
constexpr uint32_t kRtSlice = 2u * kRtN * 128u;   // one k-block of B: [G_hi; G_lo] rows x 128 B
constexpr uint32_t kRtBBuf = 8u * kRtSlice;       // 8 k-blocks
constexpr uint32_t kRtACol = 256;                 // A = [rec_hi; rec_lo] in TMEM columns 256..511
__host__ __device__ constexpr size_t rlif_bwd_tc_smem() {
  return 1024 + 2 * size_t(kRtBBuf) + 2 * size_t(kRtSlice) + 2 * 64 * kRtN * 4 + 256;
}
// D[tmem] (+)= A[tmem] * B[smem]^T (A-in-TMEM form: row m on lane m, K pairs per column)
__device__ __forceinline__ void umma_bf16_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
// local shared -> remote shared bulk copy (TMA engine), completing tx bytes on the
// receiver's mbarrier
__device__ __forceinline__ void bulk_s2s(uint32_t rdst, uint32_t src, uint32_t bytes, uint32_t rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   rdst),
               "r"(src), "r"(bytes), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAITC:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, 10000000;\n\t"
      "@P1 bra DONEC;\n\t"
      "bra LAB_WAITC;\n\t"
      "DONEC:\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

template <int kAct>
__global__ void __launch_bounds__(kRtThreads, 1) k_rlif_bwd_tc(RlifBwdArgs a) {
  extern __shared__ uint8_t rt_raw[];
  uint8_t* sm = align1024(rt_raw);
  uint8_t* Bp = sm;                                    // [2 bufs][8 kb][2 kRtN rows][128 B]
  uint8_t* gst = Bp + 2 * kRtBBuf;                     // [2 parities][2 kRtN rows][128 B]
  float* xsum = reinterpret_cast<float*>(gst + 2 * kRtSlice);  // [2: hi, lo rows][64 neurons][kRtN]
  uint64_t* full = reinterpret_cast<uint64_t*>(xsum + 2 * 64 * kRtN);  // [2] B buffer landed
  uint64_t* dfull = full + 2;                          // MMA chain of the step done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dfull + 1);
  const uint32_t crank = cluster_ctarank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b0 = blockIdx.y * kRtN;
  const int nok = max(0, min(kRtN, a.B - b0));
  constexpr uint32_t kBytesPerStep = 8u * kRtSlice;  // every CTA's k-block
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(dfull, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tslot);
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // A into TMEM: lane r of warps 0-3 = row r; r < 64 hi of neuron crank*64 + r, r >= 64
  // its lo (hi = bf16(x), lo = bf16(x - hi): ~16 significant bits together); K = source
  // j as bf16 pairs, column kRtACol + j / 2
  if (warp < 4) {
    const int r = 32 * warp + lane, il = r & 63;
    const int i = int(crank) * 64 + il;
    const float* __restrict__ row = a.rec + size_t(i < a.H ? i : 0) * a.H;
    for (int c = 0; c < 8; ++c) {
      uint32_t v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int j = c * 64 + 2 * e;
        const float x0 = (i < a.H && j < a.H) ? __ldg(row + j) : 0.0f;
        const float x1 = (i < a.H && j + 1 < a.H) ? __ldg(row + j + 1) : 0.0f;
        __nv_bfloat16 y0 = __float2bfloat16_rn(x0), y1 = __float2bfloat16_rn(x1);
        if (r >= 64) {
          y0 = __float2bfloat16_rn(x0 - __bfloat162float(y0));
          y1 = __float2bfloat16_rn(x1 - __bfloat162float(y1));
        }
        v[e] = (uint32_t(__bfloat16_as_ushort(y1)) << 16) | __bfloat16_as_ushort(y0);
      }
      tmem_st32(*tslot + (uint32_t(32 * warp) << 16) + kRtACol + uint32_t(c) * 32u, v);
    }
    tmem_st_wait();
  }
  for (int idx = tid; idx < int(2 * kRtBBuf / 16); idx += kRtThreads)
    st_shared_v4(smem_u32(Bp) + uint32_t(idx) * 16u, make_uint4(0u, 0u, 0u, 0u));
  fence_async_smem();
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and B zeroed in every CTA before any copy
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // epilogue: warp w < 4 reads TMEM lanes 32 w .. 32 w + 31 (rows 0-63 hi, 64-127 lo) and
  // publishes the row sums of all samples; then warp w < 8 runs neuron il = 32 (w & 1) +
  // lane for samples hs*kRtH .. (hs = w >> 1, a quarter of the cluster's samples)
  const bool epi = warp < kRtEpiWarps;
  const int il = 32 * (warp & 1) + lane, hs = warp >> 1;
  const int i = int(crank) * 64 + il;
  const bool live = epi && i < a.H;
  const float vb = clip01(live ? a.beta[i * a.beta_stride] : 0.0f);
  const float theta = a.theta;
  const size_t cols_total = size_t(a.B) * a.T_pad;
  const size_t plane = size_t(a.H_pad) * cols_total;
  const size_t sstride = size_t(a.T_pad) * a.H_pad;
  const int sb0 = hs * kRtH;  // first sample of this thread
  const int nmine = max(0, min(kRtH, nok - sb0));
  const size_t rbase = size_t(b0 + sb0) * sstride + (live ? i : 0);
  float G[kRtH], db[kRtH], dbias[kRtH], dSn[kRtH], Vn[kRtH];
#pragma unroll
  for (int s = 0; s < kRtH; ++s) {
    G[s] = db[s] = dbias[s] = 0.0f;
    const size_t o = rbase + s * sstride + size_t(a.T - 1) * a.H_pad;
    dSn[s] = (live && s < nmine) ? __ldg(a.ds + o) : 0.0f;
    Vn[s] = (live && s < nmine) ? __ldg(a.v_in + o) : 0.0f;
  }
  const uint32_t stg_col = uint32_t(il & 7) * 2u;
  const uint32_t idesc = idesc_bf16(128, 2 * kRtN, false, false);
  uint32_t fph[2] = {0u, 0u}, dph = 0u;
  int p = 0;
  bool first = true;
#if SNN_RT_EXP == 4
  __shared__ long long tclk[16][8];
  int nstep = 0;
  const bool probe = blockIdx.x == 0 && blockIdx.y == 0;
#define RT_CLK(k) if (probe && nstep < 16) tclk[nstep][k] = globaltimer();
#else
#define RT_CLK(k)
#endif
  // dI of a 4-step chunk as 3 bf16 planes (one 8-byte store per plane); the previous
  // chunk's samples are flushed one or two per step of the next chunk, so no step
  // carries every store (each step's exchange waits on the slowest CTA)
  auto flush = [&](const float (&xs)[4], int s, int cb) {
    uint32_t h[2], m[2], lo[2];
    split3_pack(xs[0], xs[1], h[0], m[0], lo[0]);
    split3_pack(xs[2], xs[3], h[1], m[1], lo[1]);
    uint2* d = reinterpret_cast<uint2*>(a.di_planes + size_t(i) * cols_total + size_t(b0 + sb0 + s) * a.T_pad + cb);
    d[0] = make_uint2(h[0], h[1]);
    d[plane / 4] = make_uint2(m[0], m[1]);
    d[plane / 2] = make_uint2(lo[0], lo[1]);
  };
  float xp[kRtH][4];
  int cprev = -1;
  for (int c0 = a.T_pad - 4; c0 >= 0; c0 -= 4) {
    float x[kRtH][4];
#pragma unroll
    for (int e = 3; e >= 0; --e) {
      const int t = c0 + e;
#pragma unroll
      for (int s = 0; s < kRtH; ++s) x[s][e] = G[s];
      if (live && cprev >= 0) {
#pragma unroll
        for (int s = 0; s < kRtH; ++s)
          if (s % 4 == 3 - e && s < nmine) flush(xp[s], s, cprev);
      }
      if (t >= a.T) continue;  // padded steps: uniform over the cluster
      if (warp == kRtMmaWarp) {
        if (elect_one()) {
          RT_CLK(0)
          if (!first && SNN_RT_EXP != 2) {
            mbar_wait_cluster(&full[p], fph[p]);
            fph[p] ^= 1u;
          }
          RT_CLK(1)
          // B arrived by bulk copies (async proxy) and A was fenced once: no proxy fence here
          tc_fence_after();
          if (t > 0 && SNN_RT_EXP != 2) mbar_arrive_expect_tx(&full[p ^ 1], kBytesPerStep);
          // B descriptor advances by (byte offset >> 4); A (TMEM) by 8 columns per K=16
          const uint64_t bd0 = sdesc_sw128(smem_u32(Bp) + uint32_t(p) * kRtBBuf, 16, 1024);
#pragma unroll
          for (int kb = 0; kb < (SNN_RT_EXP == 1 ? 0 : 8); ++kb) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              umma_bf16_ta(tmem, tmem + kRtACol + uint32_t((kb * 4 + ks) * 8),
                           bd0 + uint64_t((kb * int(kRtSlice) + ks * 32) >> 4), idesc, (kb | ks) != 0);
          }
          umma_commit(dfull);
          RT_CLK(2)
        }
        __syncwarp();
      }
      first = false;
      mbar_wait(dfull, dph);
      if (tid == 0) { RT_CLK(3) }
      dph ^= 1u;
      tc_fence_after();
      if (epi) {
        if (warp < 4) {  // row sums D[row][s] + D[row][kRtN + s] of every sample -> smem
          uint32_t r[2 * kRtN];
          {
            uint32_t r0[32], r1[16];
            tmem_ld32(tmem + (uint32_t(warp * 32) << 16), r0);
            tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + 32u, r1);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = r0[e];
#pragma unroll
            for (int e = 0; e < 16; ++e) r[32 + e] = r1[e];
          }
          float* xs = xsum + (warp >> 1) * (64 * kRtN) + il * kRtN;
#pragma unroll
          for (int s = 0; s < kRtN; s += 4)
            *reinterpret_cast<float4*>(xs + s) =
                make_float4(__uint_as_float(r[s]) + __uint_as_float(r[kRtN + s]),
                            __uint_as_float(r[s + 1]) + __uint_as_float(r[kRtN + s + 1]),
                            __uint_as_float(r[s + 2]) + __uint_as_float(r[kRtN + s + 2]),
                            __uint_as_float(r[s + 3]) + __uint_as_float(r[kRtN + s + 3]));
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kRtEpiWarps) : "memory");
        if (tid == 0) { RT_CLK(4) }
        if (SNN_RT_EXP != 3) {
          float hsum[kRtH], lsum[kRtH];
#pragma unroll
          for (int s2 = 0; s2 < kRtH; s2 += 2) {
            const float2 h2 = *reinterpret_cast<const float2*>(xsum + il * kRtN + sb0 + s2);
            const float2 l2 = *reinterpret_cast<const float2*>(xsum + 64 * kRtN + il * kRtN + sb0 + s2);
            hsum[s2] = h2.x; hsum[s2 + 1] = h2.y;
            lsum[s2] = l2.x; lsum[s2 + 1] = l2.y;
          }
#pragma unroll
          for (int s = 0; s < kRtH; ++s) {
            const float rc = hsum[s] + lsum[s];
            const float dS = dSn[s], V = Vn[s];
            const size_t o = rbase + s * sstride + size_t(t - 1) * a.H_pad;
            dSn[s] = (live && s < nmine && t > 0) ? __ldg(a.ds + o) : 0.0f;
            Vn[s] = (live && s < nmine && t > 0) ? __ldg(a.v_in + o) : 0.0f;
            const float gi = G[s];
            const float gs = __fadd_rn(__fadd_rn(dS, __fmul_rn(-gi, theta)), rc);
            const float g = surrogate_t<kAct>(a.slope, a.aux, __fadd_rn(V, -theta));
            db[s] = __fadd_rn(db[s], __fmul_rn(gi, V));
            dbias[s] = __fadd_rn(dbias[s], gi);
            G[s] = live ? __fadd_rn(__fmul_rn(gi, vb), __fmul_rn(gs, g)) : 0.0f;
            if (t > 0) {  // G(t) as hi / lo bf16 into staging parity p ^ 1: rows s / kRtN + s
              const __nv_bfloat16 h = __float2bfloat16_rn(G[s]);
              const __nv_bfloat16 lo = __float2bfloat16_rn(G[s] - __bfloat162float(h));
              const uint32_t base = uint32_t(p ^ 1) * kRtSlice + stg_col;
              const uint32_t c = uint32_t(il >> 3);
              *reinterpret_cast<__nv_bfloat16*>(gst + base + sw128_off(uint32_t(sb0 + s), c)) = h;
              *reinterpret_cast<__nv_bfloat16*>(gst + base + sw128_off(uint32_t(kRtN + sb0 + s), c)) = lo;
            }
          }
        }
        fence_async_smem();  // staging -> visible to the bulk copies
        if (tid == 0) { RT_CLK(5) }
      }
      tc_fence_before();
      __syncthreads();  // G(t) staged; D read before the next MMA chain; xsum reusable
      if (tid == 0) { RT_CLK(6) }
      if (warp == kRtMmaWarp && t > 0 && SNN_RT_EXP != 2 && lane < kRlCl) {
        // G(t) of this slice (k-block crank) to every CTA's B buffer p ^ 1: lane r -> rank r
        const uint32_t src = smem_u32(gst) + uint32_t(p ^ 1) * kRtSlice;
        const uint32_t dst = smem_u32(Bp) + uint32_t(p ^ 1) * kRtBBuf + crank * kRtSlice;
        const uint32_t bar = smem_u32(full) + 8u * uint32_t(p ^ 1);
        bulk_s2s(map_rank(dst, uint32_t(lane)), src, kRtSlice, map_rank(bar, uint32_t(lane)));
        if (lane == 0) { RT_CLK(7) }
      }
      p ^= 1;
#if SNN_RT_EXP == 4
      ++nstep;
#endif
    }
#pragma unroll
    for (int s = 0; s < kRtH; ++s)
#pragma unroll
      for (int e = 0; e < 4; ++e) xp[s][e] = x[s][e];
    cprev = c0;
  }
  if (live && cprev >= 0) {
#pragma unroll
    for (int s = 0; s < kRtH; ++s)
      if (s < nmine) flush(xp[s], s, cprev);
  }
  if (live) {
#pragma unroll
    for (int s = 0; s < kRtH; ++s)
      if (s < nmine) {
        a.dbeta_part[size_t(b0 + sb0 + s) * a.H + i] = db[s];
        if (a.dbias_part != nullptr) a.dbias_part[size_t(b0 + sb0 + s) * a.H + i] = dbias[s];
      }
  }
#if SNN_RT_EXP == 4
  if (probe && tid == 0)
    for (int k = 1; k < 16; ++k)
      printf("step %d: wait_full %lld mma %lld dfull %lld ld+swap %lld compute %lld sync %lld copies %lld | step %lld\n", k,
             tclk[k][1] - tclk[k][0], tclk[k][2] - tclk[k][1], tclk[k][3] - tclk[k][2], tclk[k][4] - tclk[k][3],
             tclk[k][5] - tclk[k][4], tclk[k][6] - tclk[k][5], tclk[k][7] - tclk[k][6], tclk[k][0] - tclk[k - 1][0]);
#endif
  pdl_launch_dependents();
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while a peer may still address its smem
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================================
// K6  gradient assembly, Adam and operand-plane refresh.
// One thread per flat parameter in NetworkParams order (network.hpp:164-226).
// ============================================================================
// kEntryGamma: the declared ALIF cell's adaptation decay [H] (layer = hidden index)
enum EntryKind : int32_t { kEntryW = 0, kEntryB = 1, kEntryBeta = 2, kEntryGamma = 3 };

struct Entry {
  int32_t kind, layer;    // layer = Linear index j (W, b) or cell index (beta)
  int32_t rows, cols;     // W: [K][N]; b/beta: [1][N] (beta: N = cell width, also when scalar)
  int32_t beta_mode;      // beta: 0 per neuron, 1 learnable scalar, 2 fixed (no gradient)
  int64_t offset;         // into the flat vector
};

constexpr int kMaxEntries = 4 * 9;

struct ReduceArgs {
  Entry entries[kMaxEntries];
  int n_entries;
  int64_t n_params;
  const float* partial[kMaxLayers];     // wgrad partials per Linear j
  int M_pad[kMaxLayers], N_pad[kMaxLayers], splits[kMaxLayers];
  const float* dbeta_part[kMaxLayers];  // per cell j: [B][N]
  const float* dbias_part[kMaxLayers];  // per Linear j: [B][N]
  const float* dgamma_part[kMaxLayers]; // per ALIF cell j: [B][N]
  const int32_t* vec_index;             // flat indices of the beta / bias entries
  int n_vec;
  const float* params;                  // for the clip mask
  float* grads;                         // [n_params] then loss sum, hits
  const float* loss_b;                  // [B] (integral CE: one term per sample)
  const int32_t* correct_b;             // [B]
  const float* loss_terms;              // rate-MSE: [B][C] terms, else nullptr
  int n_loss_terms;                     // B (CE) or B*C (rate-MSE), summed in order
  int64_t* step;
  int update;
  int B;
  int w_blocks;                         // blocks [0, w_blocks) handle W entries
  // activity regularizer: one count histogram [T+1] per monitor (k_lif_bwd<., true>)
  unsigned int* hist;                   // [n_mon][hist_stride], zeroed after reading
  int n_mon, hist_stride, reg_T;
  float mon_n[kMaxLayers];              // float(B_global * H) of each monitor
  float f_min, f_max, lambda_low, lambda_high;
  // peer tail (ranks exchange gradients through IPC-mapped device memory): xchg is
  // this rank's exchange buffer [2][n_comm] (nullptr otherwise), seq the exchange
  // sequence number, peer_flags every rank's flag array [kMaxRanks] (mapped)
  float* xchg;
  int64_t n_comm;
  const int64_t* seq;
  unsigned long long* peer_flags[kMaxRanks];
  int rank, world;
  unsigned int* done;
};

// 8 KB of static shared scratch shared by the tail's block-wide helpers
__device__ __forceinline__ uint32_t* tail_scratch() {
  __shared__ __align__(16) uint32_t buf[2048];
  return buf;
}

// Regularizer value of monitor m (objective.hpp:189-205) from its count histogram:
// lambda_low * (low / n) + lambda_high * (high / n), low / high summed per count
// value in double with a fixed-shape tree (deterministic; the reference's running
// float sum over (b, n) differs by rounding only), then the histogram is zeroed
// for the next step.  Whole block calls; thread 0 holds the value.
// scratch: >= 4 KB of shared memory; nthr: the calling threads (ids 0..nthr-1, a
// power of two, synchronised with named barrier 1)
__device__ __forceinline__ void bar1(int nthr) { asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory"); }
__device__ __forceinline__ float activity_value(const ReduceArgs& r, int m, uint32_t* scratch, int nthr) {
  double* s_lo = reinterpret_cast<double*>(scratch);
  double* s_hi = s_lo + nthr;
  const int tid = threadIdx.x;
  bar1(nthr);  // the scratch may still be read by the previous helper
  unsigned int* h = r.hist + size_t(m) * r.hist_stride;
  double lo = 0.0, hi = 0.0;
  for (int c = tid; c <= r.reg_T; c += nthr) {
    const unsigned k = h[c];
    if (k == 0u) continue;
    const float rate = __fdiv_rn(float(c), float(r.reg_T));
    const float xl = __fsub_rn(r.f_min, rate), xh = __fsub_rn(rate, r.f_max);
    const float dl = xl > 0.0f ? xl : 0.0f, dh = xh > 0.0f ? xh : 0.0f;
    lo += double(k) * double(__fmul_rn(dl, dl));
    hi += double(k) * double(__fmul_rn(dh, dh));
  }
  s_lo[tid] = lo;
  s_hi[tid] = hi;
  bar1(nthr);
  for (int w = nthr / 2; w > 0; w >>= 1) {
    if (tid < w) {
      s_lo[tid] += s_lo[tid + w];
      s_hi[tid] += s_hi[tid + w];
    }
    bar1(nthr);
  }
  const float n = r.mon_n[m];
  const float v = __fadd_rn(__fmul_rn(r.lambda_low, __fdiv_rn(float(s_lo[0]), n)),
                            __fmul_rn(r.lambda_high, __fdiv_rn(float(s_hi[0]), n)));
  bar1(nthr);
  for (int c = tid; c <= r.reg_T; c += nthr) h[c] = 0u;
  return v;
}

__device__ __forceinline__ int find_entry(const Entry* en, int n, int64_t i) {
  int e = 0;
  while (e + 1 < n && en[e + 1].offset <= i) ++e;
  return e;
}

// W gradient element of the split-K partials, summed by a pair of lanes: lane q
// sums splits [q*S/2, (q+1)*S/2) in order, then q0 + q1 -- a fixed order
// (deterministic), twice the loads in flight of one thread per element while
// the grid still fits one wave.  Both lanes of the pair must call it (they share
// the element and every branch before the call); both return the total.
__device__ __forceinline__ float sum_partials_pair(const ReduceArgs& r, const Entry& en, int64_t li,
                                                   int q) {
  const int j = en.layer;
  const int64_t k = li / en.cols, n = li % en.cols;
  const float* __restrict__ p = r.partial[j] + k * r.N_pad[j] + n;
  const int64_t sstride = int64_t(r.M_pad[j]) * r.N_pad[j];
  const int S = r.splits[j];
  const int s0 = q * S / 2, s1 = (q + 1) * S / 2;
  float g = 0.0f;
  int s = s0;
  for (; s + 16 <= s1; s += 16) {
    float x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = __ldg(p + (s + u) * sstride);
#pragma unroll
    for (int u = 0; u < 16; ++u) g = __fadd_rn(g, x[u]);
  }
  if (s + 8 <= s1) {
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldg(p + (s + u) * sstride);
#pragma unroll
    for (int u = 0; u < 8; ++u) g = __fadd_rn(g, x[u]);
    s += 8;
  }
  for (; s < s1; ++s) g = __fadd_rn(g, __ldg(p + s * sstride));
  const unsigned pair = 0x3u << (threadIdx.x & 30);
  const float g0 = __shfl_sync(pair, g, 0, 2);
  const float g1 = __shfl_sync(pair, g, 1, 2);
  return __fadd_rn(g0, g1);
}
constexpr int kRedElemsPerBlock = 128;  // W elements per 256-thread block (lane pairs)

// Loss numerator in the reference order -- one running float sum over the
// per-sample CE terms (objective.hpp:57-72) or the per-(sample, class) rate-MSE
// terms (objective.hpp:150-157) -- and the hit count.  Whole block calls; thread
// 0 holds the results.
__device__ __forceinline__ void loss_and_hits(const ReduceArgs& r, float& loss, int& hits,
                                              uint32_t* scratch, int nthr) {
  float* sl = reinterpret_cast<float*>(scratch);
  int* sc = reinterpret_cast<int*>(scratch + 1024);
  const int tid = threadIdx.x;
  const float* terms = r.loss_terms != nullptr ? r.loss_terms : r.loss_b;
  loss = 0.0f;
  hits = 0;
  for (int b0 = 0; b0 < r.n_loss_terms; b0 += 1024) {
    const int nb = min(1024, r.n_loss_terms - b0);
    bar1(nthr);
    for (int i = tid; i < nb; i += nthr) sl[i] = terms[b0 + i];
    bar1(nthr);
    if (tid == 0)
      for (int i = 0; i < nb; ++i) loss = __fadd_rn(loss, sl[i]);
  }
  for (int b0 = 0; b0 < r.B; b0 += 1024) {
    const int nb = min(1024, r.B - b0);
    bar1(nthr);
    for (int i = tid; i < nb; i += nthr) sc[i] = r.correct_b[b0 + i];
    bar1(nthr);
    if (tid == 0)
      for (int i = 0; i < nb; ++i) hits += sc[i];
  }
}

// Blocks [0, w_blocks): one pair of lanes per flat index, W entries only --
// fixed-order sum of the split-K partials (sum_partials_pair).  Next blocks: one warp per beta/bias element --
// lanes take strided samples, then a fixed-shape tree (deterministic).  Last
// block: loss sum in batch order (objective.hpp:57-72) + hits, step counter.
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(256) k_reduce(ReduceArgs a) {
  pdl_wait();
  const int tid = threadIdx.x;
  // peer tail: this step's gradient goes to the exchange buffer of parity seq & 1
  const int64_t seq = a.xchg != nullptr ? *reinterpret_cast<volatile const int64_t*>(a.seq) : 0;
  float* __restrict__ gout = a.xchg != nullptr ? a.xchg + (seq & 1) * a.n_comm : a.grads;
  const int vb_blocks = (a.n_vec + 7) / 8;
  if (int(blockIdx.x) < a.w_blocks) {
    // pairs stay converged: out-of-range / non-W pairs skip as a whole
    const int64_t i = int64_t(blockIdx.x) * kRedElemsPerBlock + (tid >> 1);
    if (i < a.n_params) {
      const Entry en = a.entries[find_entry(a.entries, a.n_entries, i)];
      if (en.kind == kEntryW) {
        const float g = sum_partials_pair(a, en, i - en.offset, tid & 1);
        if ((tid & 1) == 0) gout[i] = g;
      }
    }
  } else if (int(blockIdx.x) < a.w_blocks + vb_blocks) {
    const int warp = tid >> 5, lane = tid & 31;
    const int v = (int(blockIdx.x) - a.w_blocks) * 8 + warp;
    if (v < a.n_vec) {
      const int64_t i = a.vec_index[v];
      const Entry en = a.entries[find_entry(a.entries, a.n_entries, i)];
      const int64_t li = i - en.offset;
      const float* __restrict__ src =
          (en.kind == kEntryB ? a.dbias_part[en.layer]
                              : en.kind == kEntryGamma ? a.dgamma_part[en.layer] : a.dbeta_part[en.layer]) + li;
      float g = 0.0f;
      if (en.kind == kEntryBeta && en.beta_mode != 0) {
        // scalar beta: every (b, n) partial; fixed beta: no gradient
        if (en.beta_mode == 1)
          for (int q = lane; q < a.B * en.cols; q += 32) g = __fadd_rn(g, __ldg(src + q));
      } else {
        for (int b = lane; b < a.B; b += 32) g = __fadd_rn(g, __ldg(src + int64_t(b) * en.cols));
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) g = __fadd_rn(g, __shfl_xor_sync(0xffffffffu, g, off));
      if (lane == 0) {
        if (en.kind == kEntryBeta || en.kind == kEntryGamma) {
          const float beta = a.params[i];
          if (!(beta > 0.0f && beta < 1.0f)) g = 0.0f;  // clip01 gradient (autodiff.hpp:353-355)
        }
        gout[i] = g;
      }
    }
  } else {
    // loss / hits / step; activity regularizer values after them (summed over ranks
    // by the allreduce or the peer tail, added to the loss by k_adam / k_result /
    // k_peer_gather)
    float loss;
    int hits;
    loss_and_hits(a, loss, hits, tail_scratch(), 256);
    if (tid == 0) {
      gout[a.n_params] = loss;
      gout[a.n_params + 1] = float(hits);
      if (a.update && a.xchg == nullptr) *a.step += 1;  // peer tail: k_peer_gather advances it
    }
    for (int m = 0; m < a.n_mon; ++m) {
      const float v = activity_value(a, m, tail_scratch(), 256);
      if (tid == 0) gout[a.n_params + 2 + m] = v;
    }
  }
  if (a.xchg == nullptr) return;
  // peer tail: once every block's stores are visible system-wide, the last block
  // publishes seq + 1 into slot [rank] of every rank's flag array
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    if (atomicAdd(a.done, 1u) == gridDim.x - 1) {
      *a.done = 0u;
      __threadfence_system();
      for (int q = 0; q < a.world; ++q) st_release_sys(a.peer_flags[q] + a.rank, (unsigned long long)(seq + 1));
    }
  }
}

struct PlaneTarget {
  __nv_bfloat16* wb;  // operand planes [3][K_pad][N_pad] (forward MN-major A, backward K-major A)
  int K_pad, N_pad;
  float* wt;          // RLIF rec: f32 transpose [N][wt_ld] for k_rlif_bwd (else nullptr)
  int wt_ld;
};

struct AdamArgs {
  Entry entries[kMaxEntries];
  int n_entries;
  int64_t n_params;
  PlaneTarget planes[kMaxLayers];  // per Linear j
  float* params;
  float* m;
  float* v;
  const float* grads;        // [n_params] + loss sum + hits (after the allreduce)
  const float* bc;           // [2 * max_steps]: bc1, bc2 per step (host powf)
  const int64_t* step;       // device step counter (already advanced by k_reduce)
  float lr, b1, b2, eps, omb1, omb2;
  int update;                // 0: only refresh planes (after set_params)
  int B_global;
  float* loss_out;
  double* acc_out;
  int64_t* rows_slot;        // schedule mode: advanced once per update (else nullptr)
  float loss_denom;          // float(B_global) (CE) or float(B_global * C) (rate-MSE)
  int opt_kind;              // 0 Adam, 1 SGD + momentum (optimize.hpp:69-84)
  float momentum;
  int n_mon;                 // activity regularizer values at grads[n_params + 2 + m]
  // one-rank fused tail: every step's StepResult also goes to entry (step & ring_mask)
  // of a host-mapped ring (host batches read it after their one sync: no per-step
  // result kernel or copy); nullptr = off
  float* ring_loss;
  double* ring_acc;
  int64_t ring_mask;
};

// Adam on one flat parameter (optimize.hpp:88-110); bias corrections of step s+1.
// p0 / m0 / v0: the current parameter and moments (loaded by the caller, early).
__device__ __forceinline__ float adam_apply(const AdamArgs& a, int64_t i, float g, float p0, float m0,
                                            float v0, float bc1, float bc2) {
  if (a.opt_kind == 1) {
    // sgd_update (optimize.hpp:69-84): m doubles as the momentum buffer
    const float m = __fadd_rn(__fmul_rn(a.momentum, m0), g);
    const float p = __fsub_rn(p0, __fmul_rn(a.lr, m));
    a.m[i] = m;
    a.params[i] = p;
    return p;
  }
  float p = p0;
  const float m = __fadd_rn(__fmul_rn(a.b1, m0), __fmul_rn(a.omb1, g));
  const float v = __fadd_rn(__fmul_rn(a.b2, v0), __fmul_rn(__fmul_rn(a.omb2, g), g));
  const float mhat = __fdiv_rn(m, bc1);
  const float vhat = __fdiv_rn(v, bc2);
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(a.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), a.eps)));
  a.m[i] = m;
  a.v[i] = v;
  a.params[i] = p;
  return p;
}
__device__ __forceinline__ float adam_one(const AdamArgs& a, int64_t i, float g, float bc1, float bc2) {
  return adam_apply(a, i, g, a.params[i], a.m[i], a.v[i], bc1, bc2);
}

// Four consecutive elements i0..i0+3 of a W entry of Linear `layer` at (k, n0..n0+3)
// (i0 and n0 multiples of 4, no f32 transpose target): the same float ops as
// adam_apply / refresh_planes, with 16-byte parameter / moment / gradient stores and
// 8-byte plane stores.
__device__ __forceinline__ void adam4_planes(const AdamArgs& a, float* grads, int layer, int64_t i0, int64_t k,
                                             int64_t n0, const float (&g)[4], const float (&p0)[4],
                                             const float (&m0)[4], const float (&v0)[4], float bc1, float bc2) {
  float p[4], m[4], v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (a.opt_kind == 1) {  // sgd_update (optimize.hpp:69-84)
      m[e] = __fadd_rn(__fmul_rn(a.momentum, m0[e]), g[e]);
      p[e] = __fsub_rn(p0[e], __fmul_rn(a.lr, m[e]));
      v[e] = v0[e];
    } else {
      m[e] = __fadd_rn(__fmul_rn(a.b1, m0[e]), __fmul_rn(a.omb1, g[e]));
      v[e] = __fadd_rn(__fmul_rn(a.b2, v0[e]), __fmul_rn(__fmul_rn(a.omb2, g[e]), g[e]));
      const float mhat = __fdiv_rn(m[e], bc1);
      const float vhat = __fdiv_rn(v[e], bc2);
      p[e] = __fsub_rn(p0[e], __fdiv_rn(__fmul_rn(a.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), a.eps)));
    }
  }
  *reinterpret_cast<float4*>(a.params + i0) = make_float4(p[0], p[1], p[2], p[3]);
  *reinterpret_cast<float4*>(a.m + i0) = make_float4(m[0], m[1], m[2], m[3]);
  if (a.opt_kind != 1) *reinterpret_cast<float4*>(a.v + i0) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(grads + i0) = make_float4(g[0], g[1], g[2], g[3]);
  const PlaneTarget pt = a.planes[layer];
  if (pt.wb == nullptr) return;
  uint32_t h[4], mi[4], lo[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) split3_bits(p[e], h[e], mi[e], lo[e]);
  const int64_t plane = int64_t(pt.K_pad) * pt.N_pad, idx = k * pt.N_pad + n0;
  *reinterpret_cast<uint2*>(pt.wb + idx) = make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
  *reinterpret_cast<uint2*>(pt.wb + plane + idx) = make_uint2(mi[0] | (mi[1] << 16), mi[2] | (mi[3] << 16));
  *reinterpret_cast<uint2*>(pt.wb + 2 * plane + idx) = make_uint2(lo[0] | (lo[1] << 16), lo[2] | (lo[3] << 16));
}

// bf16 operand planes of W element (k, n) of Linear `layer` from its f32 master
// (consecutive n -> consecutive addresses: coalesced).
__device__ __forceinline__ void refresh_planes(const AdamArgs& a, int layer, int64_t k, int64_t n, float p) {
  const PlaneTarget pt = a.planes[layer];
  if (pt.wt != nullptr) pt.wt[n * pt.wt_ld + k] = p;
  if (pt.wb == nullptr) return;
  __nv_bfloat16 h, mi, lo;
  split3(p, h, mi, lo);
  const int64_t plane = int64_t(pt.K_pad) * pt.N_pad, idx = k * pt.N_pad + n;
  pt.wb[idx] = h;
  pt.wb[plane + idx] = mi;
  pt.wb[2 * plane + idx] = lo;
}

__global__ void __launch_bounds__(256) k_adam(AdamArgs a) {
  pdl_wait();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a.update && i == 0) {
    // StepResult{loss, accuracy} (optimize.hpp:143-147, :193-196)
    float l = __fdiv_rn(a.grads[a.n_params], a.loss_denom);
    for (int m = 0; m < a.n_mon; ++m) l = __fadd_rn(l, a.grads[a.n_params + 2 + m]);  // optimize.hpp:185-191
    *a.loss_out = l;
    *a.acc_out = double(a.grads[a.n_params + 1]) / double(a.B_global);
    if (a.rows_slot != nullptr) *a.rows_slot += 1;
  }
  if (i >= a.n_params) return;
  float p = a.params[i];
  if (a.update) {
    const int64_t s = *a.step - 1;  // bias correction of step s+1 (optimize.hpp:95-97)
    p = adam_one(a, i, a.grads[i], a.bc[2 * s], a.bc[2 * s + 1]);
  }
  const Entry en = a.entries[find_entry(a.entries, a.n_entries, i)];
  if (en.kind != kEntryW) return;
  const int64_t li = i - en.offset;
  refresh_planes(a, en.layer, li / en.cols, li % en.cols, p);
}

// Multi-rank step tail over peer memory, OWNER-COMPUTES (replaces ncclAllReduce +
// k_adam).  Every rank's k_reduce wrote its local gradient, loss numerator, hits
// and regularizer values into its exchange buffer (grad region, parity seq & 1)
// and published seq + 1 into flag array A of every rank.  Rank r owns the flat
// parameter slice [r n / W, (r + 1) n / W):
//   k_peer_owner  waits for every rank's A flag, sums its slice over the ranks'
//                 grad regions in ascending rank order (deterministic), runs Adam /
//                 SGD on it (m, v are owner-sharded, ZeRO-1 style), writes the new
//                 parameters (and m, v) into its own result region and the summed
//                 gradient back over its own grad slice, then publishes seq + 1 into
//                 flag array B of every rank;
//   k_peer_gather waits for every rank's B flag and copies each parameter from its
//                 owner's result region (local or mapped peer memory), refreshes the
//                 bf16 operand planes and the summed gradient.
// Each rank reads ~2 (W-1)/W n floats over NVLink per step: O(n), not O(W n), and
// every rank holds the same bits (each element is computed by exactly one owner).
// Reuse of a parity is race-free: a rank rewrites grad region p two steps later,
// after its own gather of the next step, i.e. after every owner published that
// step's B flag (so every owner has finished reading region p); it rewrites
// result region p after its owner phase two steps later, which waits for every
// rank's A flag of that step, i.e. for every rank's gather of the step before.
struct PeerArgs {
  float* xchg[kMaxRanks];          // every rank's exchange buffer (mapped; own = local)
  unsigned long long* flags_a;     // this rank's A flags (slot q written by rank q's k_reduce)
  unsigned long long* flags_b;     // this rank's B flags (slot q written by rank q's owner phase)
  unsigned long long* peer_flags_b[kMaxRanks];  // every rank's B flag array
  int64_t n_comm;
  int64_t* seq;                    // exchange sequence number (advanced by k_peer_gather)
  unsigned int* done;              // completion counters: [0] owner phase, [1] gather
  unsigned int* timeout;           // set to 1 (not a trap) when a peer never published
  float* grads_out;                // summed gradient, loss sum, hits (snn_get_grads)
  int64_t* rows_slot;              // schedule mode: advanced once per update
  int64_t* step;                   // the step counter (advanced once per update)
  int rank, world;
  long long spin_ns;               // peer wait limit (SNN_PEER_TIMEOUT_S)
};
// region offsets (floats) inside one rank's exchange buffer
__host__ __device__ inline int64_t peer_grad_off(int64_t n_comm, int par) { return par * n_comm; }
__host__ __device__ inline int64_t peer_res_off(int64_t n_comm, int par) { return (2 + par) * n_comm; }
__host__ __device__ inline int64_t peer_m_off(int64_t n_comm) { return 4 * n_comm; }
__host__ __device__ inline int64_t peer_v_off(int64_t n_comm) { return 5 * n_comm; }
__host__ __device__ inline int64_t peer_slice_lo(int64_t n, int r, int w) { return n * r / w; }
__device__ __forceinline__ int peer_owner(int64_t i, int64_t n, int w) {
  int q = int((i * w) / n);  // first guess; fix the floor-division edge
  while (q + 1 < w && peer_slice_lo(n, q + 1, w) <= i) ++q;
  while (q > 0 && peer_slice_lo(n, q, w) > i) --q;
  return q;
}
// thread 0 of the block spins until every rank's flag reached `target`; on a
// timeout it raises the device error flag (the host reports it) instead of
// trapping, and the block proceeds (the step's results are then invalid)
__device__ __forceinline__ void peer_wait_all(const PeerArgs& p, const unsigned long long* flags,
                                              unsigned long long target) {
  if (threadIdx.x == 0) {
    for (int q = 0; q < p.world; ++q) {
      const long long t0 = globaltimer();
      while (ld_acquire_sys(flags + q) < target) {
        if (globaltimer() - t0 > p.spin_ns) {
          atomicExch(p.timeout, 1u);
          break;
        }
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_peer_owner(const __grid_constant__ PeerArgs p, AdamArgs a) {
  pdl_wait();
  const int tid = threadIdx.x;
  const int64_t seq = *reinterpret_cast<volatile const int64_t*>(p.seq);
  const int64_t s = *reinterpret_cast<volatile const int64_t*>(a.step);  // bias corrections of step s+1
  const int par = int(seq & 1);
  peer_wait_all(p, p.flags_a, (unsigned long long)(seq + 1));
  const int64_t lo = peer_slice_lo(a.n_params, p.rank, p.world);
  const int64_t hi = peer_slice_lo(a.n_params, p.rank + 1, p.world);
  const int64_t i = lo + int64_t(blockIdx.x) * blockDim.x + tid;
  float* own = p.xchg[p.rank];
  if (i < hi) {
    float g = 0.0f;
    for (int q = 0; q < p.world; ++q) g = __fadd_rn(g, __ldcv(p.xchg[q] + peer_grad_off(p.n_comm, par) + i));
    float pv = a.params[i];
    if (a.update) pv = adam_one(a, i, g, a.bc[2 * s], a.bc[2 * s + 1]);
    own[peer_grad_off(p.n_comm, par) + i] = g;  // only this rank reads its own slice
    own[peer_res_off(p.n_comm, par) + i] = pv;
    own[peer_m_off(p.n_comm) + i] = a.m[i];
    own[peer_v_off(p.n_comm) + i] = a.v[i];
  }
  // publish: once every block's stores are visible system-wide, the last block
  // writes seq + 1 into slot [rank] of every rank's B flags
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    if (atomicAdd(p.done, 1u) == gridDim.x - 1) {
      *p.done = 0u;
      __threadfence_system();
      for (int q = 0; q < p.world; ++q) st_release_sys(p.peer_flags_b[q] + p.rank, (unsigned long long)(seq + 1));
    }
  }
}

__global__ void __launch_bounds__(256) k_peer_gather(const __grid_constant__ PeerArgs p, AdamArgs a) {
  pdl_wait();
  const int tid = threadIdx.x;
  const int64_t seq = *reinterpret_cast<volatile const int64_t*>(p.seq);
  const int64_t s = *reinterpret_cast<volatile const int64_t*>(a.step);
  const int par = int(seq & 1);
  peer_wait_all(p, p.flags_b, (unsigned long long)(seq + 1));
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + tid;
  if (i < a.n_params) {
    const int q = peer_owner(i, a.n_params, p.world);
    const float* src = p.xchg[q];
    const float pv = __ldcv(src + peer_res_off(p.n_comm, par) + i);
    p.grads_out[i] = __ldcv(src + peer_grad_off(p.n_comm, par) + i);
    if (q != p.rank) a.params[i] = pv;
    const Entry en = a.entries[find_entry(a.entries, a.n_entries, i)];
    if (en.kind == kEntryW && a.update) {
      const int64_t li = i - en.offset;
      refresh_planes(a, en.layer, li / en.cols, li % en.cols, pv);
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    // StepResult (optimize.hpp:143-147, :193-196) from the rank sums, same order
    const int64_t g0 = peer_grad_off(p.n_comm, par) + a.n_params;
    float ls = 0.0f, hs = 0.0f;
    for (int q = 0; q < p.world; ++q) {
      ls = __fadd_rn(ls, __ldcv(p.xchg[q] + g0));
      hs = __fadd_rn(hs, __ldcv(p.xchg[q] + g0 + 1));
    }
    p.grads_out[a.n_params] = ls;
    p.grads_out[a.n_params + 1] = hs;
    float l = __fdiv_rn(ls, a.loss_denom);
    for (int m = 0; m < a.n_mon; ++m) {
      float v = 0.0f;
      for (int q = 0; q < p.world; ++q) v = __fadd_rn(v, __ldcv(p.xchg[q] + g0 + 2 + m));
      l = __fadd_rn(l, v);  // optimize.hpp:185-191
    }
    *a.loss_out = l;
    *a.acc_out = double(hs) / double(a.B_global);
  }
  // completion: the last block advances the exchange sequence and the step counters
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(p.done + 1, 1u) == gridDim.x - 1) {
      p.done[1] = 0u;
      *p.seq = seq + 1;
      if (a.update) {
        *p.step = s + 1;
        if (p.rows_slot != nullptr) *p.rows_slot += 1;
      }
      __threadfence();
    }
  }
}

// ============================================================================
// K5  k_wgrad: partial[s][k][n] = sum_{rows in split s} A[k][row] * dI[row][n]
// A binary (dataset time bits or time-packed spikes), exact in bf16 (K-major,
// decoded by warps 0-3); dI as 3 bf16 planes via TMA (MN-major).  Epilogue
// writes f32 partials; k_reduce sums them in fixed order (deterministic).
// grid (M_pad/128, N_pad/N_TILE, splits); block 192.
// ============================================================================
struct WgradLayer {
  const uint32_t* s_tp;    // kind 1: time-packed spikes [K_pad][B*T_pad/32]
  float* partial;          // [splits][M_pad][N_pad]
  int kind, M_pad, N_pad, n_tile, splits, m_tiles, n_tiles, block_start;
  int mg, m_groups;        // m-tiles per CTA (share every dI stage), groups
  int stages;              // pipeline depth for this layer's stage size
};
// B operand: dI planes [3][N_pad][B*T_pad] (K-major rows = output neurons)
struct WgradArgs {
  WgradLayer layer[kMaxLayers];
  int n_layers;
  const uint8_t* x;        // kind 0: staged dataset
  const uint32_t* rows;    // kind 0: [B]
  const int64_t* rows_slot;  // schedule mode: rows += *rows_slot * B (else nullptr)
  long long* dbg_clk;      // optional [blocks][kClkStride] phase timestamps
  const int32_t* xshift;   // kind 0: batch roll along the features (shift_augment)
  int B, T_pad, x_row_stride, in_features;
  int planes;                // dI planes multiplied (3: fp32 path)
};
struct WgradMaps {
  CUtensorMap m[kMaxLayers];   // dI planes (B operand)
  CUtensorMap pm[kMaxLayers];  // fused tail: f32 partials [splits*M_pad][N_pad], box 32 x 128, SW128
};

constexpr int kWgStagesMax = 6;
constexpr int kWgMgMax = 4;
#ifndef SNN_WG_EXP
#define SNN_WG_EXP 0  // timing experiments (tests/clk_probe.py only): 1 no decode, 2 one dI plane, 3 no MMA
#endif
// A-operand producers: kWgProdWarps warps; thread p decodes row p % 128 of every
// M-tile, time half p / 128 (64 steps per stage = 2 halves of 32)
constexpr int kWgProdWarps = 8;
constexpr int kWgProd = 32 * kWgProdWarps;
constexpr int kWgThreads = kWgProd + 64;  // + TMA warp + MMA warp
__host__ __device__ constexpr uint32_t wg_stage_bytes(int n_tile, int mg) {
  return uint32_t(mg) * kPlaneTile + 3 * uint32_t(n_tile) * 128u;  // mg A tiles + 3 B planes
}
__host__ __device__ constexpr uint32_t wg_xrun_bytes(int x_row_stride) {
  return (8u * uint32_t(x_row_stride) + 1023) & ~1023u;
}
__host__ __device__ constexpr uint32_t wg_smem_bytes(int n_tile, int mg, int stages, int x_row_stride) {
  return uint32_t(stages) * (wg_stage_bytes(n_tile, mg) + wg_xrun_bytes(x_row_stride)) + 1024 + 256;
}
// epilogue staging row stride (f32 row of n_tile + 16 bytes of bank padding)
__host__ __device__ constexpr uint32_t wg_epi_row_stride(int n_tile) { return uint32_t(n_tile) * 4u + 16u; }
// the launch always requests the full carve-out: barriers at kWgBarrierOffset
constexpr uint32_t kWgSmemLaunch = 227 * 1024;

// barriers at a fixed offset past the largest per-layer stage footprint
constexpr uint32_t kWgBarrierOffset = 227 * 1024 - 2048;
constexpr uint32_t kWgRedBarOffset = kWgBarrierOffset + 1024;  // fused tail: partial-load barrier

// Fused step tail (one rank, training step): after its partial is written, every
// CTA of an output tile waits on the tile's arrival counter (all of the launch's
// CTAs are co-resident: the split model keeps the grid within one wave), then the
// tile's S CTAs each take 1/S of its elements, sum the S partials in ascending
// split order (deterministic, L2-resident), run Adam / SGD and refresh the bf16
// planes; the beta / bias / gamma entries are spread over the CTAs (one warp per
// element), block 0 sums the loss / hits / regularizer (StepResult), and the last
// CTA to finish advances the step and schedule counters and re-arms the tile
// counters.  Replaces k_reduce_adam and its launch.
struct WgradTail {
  unsigned int* tile_cnt;     // per output tile (zeroed; re-armed by the last CTA)
  unsigned int* done;         // CTA completion counter
  int64_t* rows_slot;         // schedule mode: advanced once per step (else nullptr)
  int n_tiles_total;
  int64_t w_off[kMaxLayers];  // flat offset of each layer's W entry
  int rows[kMaxLayers], cols[kMaxLayers];  // K[j], N[j] (unpadded)
  int tile_base[kMaxLayers];  // first tile id of each layer
};

__device__ __forceinline__ unsigned int ld_acquire_gpu_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Producer threads (kWgProd, named barrier 1) of one CTA after its accumulator is
// staged in smem (rows m*128 + r, padded row stride): write the partial, wait for
// the tile, reduce 1/S of it + Adam, the CTA's share of the vector entries, and
// (block 0) the loss / hits / StepResult.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// the fused tail's batch reductions that need no weight gradient: beta / bias /
// gamma entries (one warp per element, spread over the CTAs)
__device__ __forceinline__ void wgrad_vec(const ReduceArgs& rd, const AdamArgs& ad, float bc1, float bc2,
                                          long long* clk) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (clk != nullptr && tid == 0) clk[10] = clock64();
  // 4. beta / bias / gamma entries: one warp per element, spread over the CTAs
  for (int v = int(blockIdx.x) * kWgProdWarps + warp; v < rd.n_vec; v += int(gridDim.x) * kWgProdWarps) {
    const int64_t i = rd.vec_index[v];
    const Entry en = rd.entries[find_entry(rd.entries, rd.n_entries, i)];
    const int64_t li = i - en.offset;
    const float* __restrict__ src =
        (en.kind == kEntryB ? rd.dbias_part[en.layer]
                            : en.kind == kEntryGamma ? rd.dgamma_part[en.layer] : rd.dbeta_part[en.layer]) + li;
    float gs = 0.0f;
    // lane-strided partials, 8 loads in flight per lane, summed in the same order
    // as k_reduce_adam's loop (lane's samples ascending), then the warp tree
    const int cnt = (en.kind == kEntryBeta && en.beta_mode != 0) ? (en.beta_mode == 1 ? rd.B * en.cols : 0)
                                                                 : rd.B;
    const int64_t stride = (en.kind == kEntryBeta && en.beta_mode != 0) ? 1 : en.cols;
    for (int q0 = lane; q0 < cnt; q0 += 32 * 8) {
      float x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = q0 + 32 * u < cnt ? __ldcg(src + int64_t(q0 + 32 * u) * stride) : 0.0f;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q0 + 32 * u < cnt) gs = __fadd_rn(gs, x[u]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) gs = __fadd_rn(gs, __shfl_xor_sync(0xffffffffu, gs, off));
    if (lane == 0) {
      if (en.kind == kEntryBeta || en.kind == kEntryGamma) {
        const float beta = rd.params[i];
        if (!(beta > 0.0f && beta < 1.0f)) gs = 0.0f;  // clip01 gradient (autodiff.hpp:353-355)
      }
      rd.grads[i] = gs;
      adam_one(ad, i, gs, bc1, bc2);
    }
  }
  if (clk != nullptr && tid == 0) clk[11] = clock64();
}

// block 0: loss sum in batch order (objective.hpp:57-72) + hits + regularizer ->
// StepResult; scratch: 8 KB of free shared memory
__device__ __forceinline__ void wgrad_loss(const ReduceArgs& rd, const AdamArgs& ad, uint8_t* scratch_smem,
                                           int64_t step0) {
  const int tid = threadIdx.x;
  if (blockIdx.x == 0) {
    uint32_t* scratch = reinterpret_cast<uint32_t*>(scratch_smem);
    bar1(kWgProd);
    float loss;
    int hits;
    loss_and_hits(rd, loss, hits, scratch, kWgProd);
    float l = __fdiv_rn(loss, ad.loss_denom);
    for (int m = 0; m < rd.n_mon; ++m) {  // optimize.hpp:185-191
      const float v = activity_value(rd, m, scratch, kWgProd);
      if (tid == 0) {
        rd.grads[rd.n_params + 2 + m] = v;
        l = __fadd_rn(l, v);
      }
    }
    if (tid == 0) {
      rd.grads[rd.n_params] = loss;
      rd.grads[rd.n_params + 1] = float(hits);
      *ad.loss_out = l;
      *ad.acc_out = double(hits) / double(ad.B_global);
      if (ad.ring_loss != nullptr) {
        ad.ring_loss[step0 & ad.ring_mask] = l;
        ad.ring_acc[step0 & ad.ring_mask] = double(hits) / double(ad.B_global);
      }
    }
  }
}

__device__ __forceinline__ void wgrad_fused_epilogue(const WgradLayer& a, int j, const CUtensorMap* pmap,
                                                  int split, int mt0, int nm, int ntile, uint8_t* smem,
                                                  const ReduceArgs& rd, const AdamArgs& ad,
                                                  const WgradTail& tl, int64_t s, long long* clk) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt4 = a.n_tile / 4, ncg = a.n_tile / 32;
  const int S = a.splits;
  const int unit = mt0 / a.mg + (a.m_tiles + a.mg - 1) / a.mg * ntile;
  const int tile = tl.tile_base[j] + unit;
  // 2. this CTA's rows [r0, r1) of the tile, in chunks of cr rows: every split's
  //    rows are bulk-loaded into smem [split][row][n_tile], summed in the order of
  //    k_reduce's sum_partials_pair (splits [0, S/2) and [S/2, S) ascending, then
  //    the halves added: forward_backward and a train step see the same bits),
  //    then Adam / SGD and the bf16 plane refresh per element
  const int R = nm * 128;
  const int r0 = R * split / S, r1 = R * (split + 1) / S;
  const uint32_t rowb = uint32_t(a.n_tile) * 4u;
  const int cr = max(1, min(r1 - r0, int((kWgBarrierOffset - 1024) / (uint32_t(S) * rowb))));
  // Adam's operands of this thread's first element group (the first chunk) do not
  // depend on the partials: loaded before the tile wait so their latency hides in it
  const int nr_first = min(cr, r1 - r0);
  float pf_p[4] = {0.f, 0.f, 0.f, 0.f}, pf_m[4] = {0.f, 0.f, 0.f, 0.f}, pf_v[4] = {0.f, 0.f, 0.f, 0.f};
  if (tid < nr_first * nt4) {
    const int k = mt0 * 128 + r0 + tid / nt4, n0 = ntile * a.n_tile + 4 * (tid % nt4);
    if (k < tl.rows[j] && n0 < tl.cols[j]) {
      const int64_t i0 = tl.w_off[j] + int64_t(k) * tl.cols[j] + n0;
      const int nv = min(4, tl.cols[j] - n0);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < nv) {
          pf_p[e] = ad.params[i0 + e];
          pf_m[e] = ad.m[i0 + e];
          pf_v[e] = ad.v[i0 + e];
        }
    }
  }
  // 1. own partial by TMA tensor stores from the SW128 staging; once the writes are
  //    performed, arrive on the tile counter and wait for the tile's other splits
  if (tid == 0) {
    for (int m = 0; m < nm; ++m)
      for (int c = 0; c < ncg; ++c)
        tma_store_2d(pmap, smem + size_t(m * ncg + c) * 16384, ntile * a.n_tile + c * 32,
                     split * a.M_pad + (mt0 + m) * 128);
    bulk_commit();
  }
  const float bc1 = ad.bc[2 * s], bc2 = ad.bc[2 * s + 1];
  // while the stores drain and the tile's other splits finish: the work that does
  // not depend on the weight gradients (beta / bias / gamma, then block 0's loss /
  // StepResult -- after this CTA's arrival, so the tile's other splits never wait on it)
  wgrad_vec(rd, ad, bc1, bc2, clk);
  if (tid == 0) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (clk != nullptr) clk[8] = clock64();
    fence_proxy_async_global();
    __threadfence();
    atomicAdd(tl.tile_cnt + tile, 1u);
  }
  wgrad_loss(rd, ad, smem + size_t(nm) * ncg * 16384, s);
  if (tid == 0) {
    while (ld_acquire_gpu_u32(tl.tile_cnt + tile) < unsigned(S)) __nanosleep(32);
    fence_proxy_async_global();  // the bulk loads below see the other splits' partials
    if (clk != nullptr) clk[9] = clock64();
  }
  bar1(kWgProd);
  uint64_t* rbar = reinterpret_cast<uint64_t*>(smem + kWgRedBarOffset);
  const int rows_j = tl.rows[j], cols_j = tl.cols[j];
  const bool contig = a.n_tiles == 1;  // a tile's rows are one contiguous run per split
  int phase = 0;
  for (int c = r0; c < r1; c += cr, phase ^= 1) {
    const int nr = min(cr, r1 - c);
    if (warp == 0) {
      if (lane == 0) mbar_arrive_expect_tx(rbar, uint32_t(S) * uint32_t(nr) * rowb);
      __syncwarp();
      const int n_copies = contig ? S : S * nr;
      for (int q = lane; q < n_copies; q += 32) {
        const int sp = contig ? q : q / nr, rr = contig ? 0 : q % nr;
        const float* src = a.partial + (size_t(sp) * a.M_pad + mt0 * 128 + c + rr) * a.N_pad +
                           size_t(ntile) * a.n_tile;
        bulk_load(smem + (size_t(sp) * cr + rr) * rowb, src, contig ? uint32_t(nr) * rowb : rowb, rbar);
      }
    }
    mbar_wait(rbar, phase);
    if (clk != nullptr && tid == 0 && c == r0) clk[12] = clock64();
    for (int g = tid; g < nr * nt4; g += kWgProd) {
      const int rr = g / nt4, c4 = g % nt4;
      const int k = mt0 * 128 + c + rr, n0 = ntile * a.n_tile + 4 * c4;
      if (k >= rows_j || n0 >= cols_j) continue;
      const int64_t i0 = tl.w_off[j] + int64_t(k) * cols_j + n0;
      const int nv = min(4, cols_j - n0);
      float p0[4] = {0.f, 0.f, 0.f, 0.f}, m0[4] = {0.f, 0.f, 0.f, 0.f}, v0[4] = {0.f, 0.f, 0.f, 0.f};
      const bool pref = c == r0 && g == tid;  // prefetched before the tile wait
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < nv) {
          p0[e] = pref ? pf_p[e] : ad.params[i0 + e];
          m0[e] = pref ? pf_m[e] : ad.m[i0 + e];
          v0[e] = pref ? pf_v[e] : ad.v[i0 + e];
        }
      const float4* col = reinterpret_cast<const float4*>(smem + size_t(rr) * rowb) + c4;
      const size_t sstep = size_t(cr) * rowb / 16;  // float4s between splits
      float4 acc[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float4 a4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const int s1 = (q + 1) * S / 2;
        for (int sp = q * S / 2; sp < s1; sp += 8) {
          float4 x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (sp + u < s1) x[u] = col[(sp + u) * sstep];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (sp + u < s1) {
              a4.x = __fadd_rn(a4.x, x[u].x);
              a4.y = __fadd_rn(a4.y, x[u].y);
              a4.z = __fadd_rn(a4.z, x[u].z);
              a4.w = __fadd_rn(a4.w, x[u].w);
            }
        }
        acc[q] = a4;
      }
      const float gv[4] = {__fadd_rn(acc[0].x, acc[1].x), __fadd_rn(acc[0].y, acc[1].y),
                           __fadd_rn(acc[0].z, acc[1].z), __fadd_rn(acc[0].w, acc[1].w)};
      if (nv == 4 && (i0 & 3) == 0 && ad.planes[j].wt == nullptr) {
        adam4_planes(ad, rd.grads, j, i0, k, n0, gv, p0, m0, v0, bc1, bc2);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < nv) {
            rd.grads[i0 + e] = gv[e];
            refresh_planes(ad, j, k, n0 + e, adam_apply(ad, i0 + e, gv[e], p0[e], m0[e], v0[e], bc1, bc2));
          }
      }
    }
    bar1(kWgProd);  // the chunk's smem is reloaded next
    if (clk != nullptr && tid == 0 && c == r0) clk[13] = clock64();
  }
}

// One launch for every Linear layer: block -> (layer, m-group, n-tile, split), the
// split index innermost (a tile's CTAs are consecutive).
// A CTA accumulates mg M-tiles (mg x n_tile TMEM columns) so each dI stage
// loaded by TMA feeds mg MMAs.  kFused: the one-rank step tail runs in the
// epilogue (wgrad_fused_epilogue) instead of k_reduce_adam.
template <bool kFused>
__global__ void __launch_bounds__(kWgThreads, 1)
    k_wgrad(const __grid_constant__ WgradMaps maps, WgradArgs args, const __grid_constant__ ReduceArgs rd,
            const __grid_constant__ AdamArgs ad, const __grid_constant__ WgradTail tl) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  long long* clk = args.dbg_clk != nullptr ? args.dbg_clk + size_t(blockIdx.x) * kClkStride : nullptr;
  if (clk != nullptr && threadIdx.x == 0) {
    clk[0] = clock64();
    clk[6] = globaltimer();
  }
  int li = 0;
  while (li + 1 < args.n_layers && int(blockIdx.x) >= args.layer[li + 1].block_start) ++li;
  const WgradLayer a = args.layer[li];
  const CUtensorMap* tm_di = &maps.m[li];
  const int local = int(blockIdx.x) - a.block_start;
  const int split = local % a.splits, unit = local / a.splits;
  const int mgi = unit % a.m_groups, ntile = unit / a.m_groups;
  // fused tail: the step counter before any CTA can advance it (bias corrections)
  const int64_t step0 = kFused ? *reinterpret_cast<volatile const int64_t*>(rd.step) : 0;
  const int mt0 = mgi * a.mg;
  const int nm = min(a.mg, a.m_tiles - mt0);  // M-tiles of this CTA
  const int S = a.stages;
  const uint32_t stage_bytes = wg_stage_bytes(a.n_tile, a.mg);
  const uint32_t ptile = uint32_t(a.n_tile) * 128u;  // one plane: n_tile rows x 64 cols
  // kind 0: the dataset bytes of one (sample, 64-step block) are one contiguous
  // run of 8 * x_row_stride bytes -> one bulk copy per stage into xbuf
  const uint32_t xbytes = a.kind == 0 ? 8u * uint32_t(args.x_row_stride) : 0u;
  uint8_t* xbuf = smem + S * stage_bytes;
  // barriers live at the end of the (max-sized) dynamic smem, past every layer's stages
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kWgBarrierOffset);
  uint64_t* empty = full + S;
  uint64_t* xfull = empty + S;
  uint64_t* acc_full = xfull + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tq_per_b = args.T_pad / 64;
  // split s takes iterations [it0, it1) of the (sample, 64-step block) sequence:
  // finer than whole samples, so the splits of a tile finish closer together
  const int iters_all = args.B * tq_per_b;
  const int it0 = int((long long)iters_all * split / a.splits);
  const int total = int((long long)iters_all * (split + 1) / a.splits) - it0;
  const uint32_t tmem_cols = tmem_cols_for(a.mg * a.n_tile, 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1 + kWgProd);
      mbar_init(&empty[s], 1);
      mbar_init(&xfull[s], 1);
    }
    mbar_init(&acc_full[0], 1);
    if (kFused) mbar_init(reinterpret_cast<uint64_t*>(smem + kWgRedBarOffset), 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_any(tmem_cols, tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  if (clk != nullptr && threadIdx.x == 0) {
    clk[1] = clock64();
    clk[14] = globaltimer();  // span start: past the dependency wait
  }
  const uint32_t tmem = *tmem_slot;
  if (warp == kWgProdWarps) {
    if (elect_one()) {
      tma_prefetch(tm_di);
      const uint32_t* rows = batch_rows(args.rows, args.rows_slot, args.B);
      for (int it = 0; it < total; ++it) {
        const int s = it % S, ph = (it / S) & 1;
        const int bb = (it0 + it) / tq_per_b, tq = (it0 + it) % tq_per_b;
        mbar_wait(&empty[s], ph ^ 1);
        if (a.kind == 0) {
          mbar_arrive_expect_tx(&xfull[s], xbytes);
          bulk_load(xbuf + s * ((xbytes + 1023) & ~1023u),
                    args.x + (size_t(rows[bb]) * (args.T_pad / 8) + tq * 8) * args.x_row_stride,
                    xbytes, &xfull[s]);
        }
#if SNN_WG_EXP == 2
        const int kLoadPlanes = 1;  // timing experiment only
#else
        const int kLoadPlanes = args.planes;
#endif
        mbar_arrive_expect_tx(&full[s], kLoadPlanes * ptile);
        uint8_t* Bp = smem + s * stage_bytes + a.mg * kPlaneTile;
        for (int p = 0; p < kLoadPlanes; ++p)
          tma_load_2d(Bp + p * ptile, tm_di, &full[s], bb * args.T_pad + tq * 64,
                      p * a.N_pad + ntile * a.n_tile);
      }
    }
    __syncwarp();
  } else if (warp == kWgProdWarps + 1) {
    const uint32_t idesc = idesc_bf16(128, a.n_tile, false, false);
    if (elect_one()) {
      for (int it = 0; it < total; ++it) {
        const int s = it % S, ph = (it / S) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (clk != nullptr && it == 0) clk[2] = clock64();
        const uint32_t A = smem_u32(smem + s * stage_bytes);
        const uint32_t Bp = A + a.mg * kPlaneTile;
#pragma unroll
        for (int ks = 0; ks < (SNN_WG_EXP == 3 ? 0 : 4); ++ks) {
          for (int m = 0; m < nm; ++m) {
            const uint64_t ad = sdesc_sw128(A + m * kPlaneTile + ks * 32, 16, 1024);
            if (args.planes == 3) {
#pragma unroll
              for (int p = 2; p >= 0; --p) {
                const uint64_t bd = sdesc_sw128(Bp + p * ptile + ks * 32, 16, 1024);
                umma_bf16(tmem + m * a.n_tile, ad, bd, idesc, (it | ks | (2 - p)) != 0);
              }
            } else {
              for (int p = args.planes - 1; p >= 0; --p) {
                const uint64_t bd = sdesc_sw128(Bp + p * ptile + ks * 32, 16, 1024);
                umma_bf16(tmem + m * a.n_tile, ad, bd, idesc, (it | ks | (args.planes - 1 - p)) != 0);
              }
            }
          }
        }
        umma_commit(&empty[s]);
      }
      umma_commit(&acc_full[0]);
      if (clk != nullptr) clk[3] = clock64();
    }
    __syncwarp();
  } else {
    // A producers: nm tiles [128 k-rows][64 time cols], K-major SW128.  Thread p:
    // row p % 128 of every tile, 16-byte chunks 4h..4h+3 (h = p / 128: 32 steps).
    // kind 0 decodes the bulk-copied dataset bytes from smem; kind 1 loads the
    // time-packed spike word (L2-resident) one stage ahead.
    const int row = threadIdx.x & 127, h = threadIdx.x >> 7;
    auto fetch = [&](int it, int m) -> uint32_t {
      const int k = (mt0 + m) * 128 + row;
      if (a.kind == 0 || it >= total || m >= nm) return 0u;
      const int bb = (it0 + it) / tq_per_b, tq = (it0 + it) % tq_per_b;
      return __ldg(a.s_tp + size_t(k) * (size_t(args.B) * args.T_pad / 32) +
                   size_t(bb) * (args.T_pad / 32) + tq * 2 + h);
    };
    uint32_t cur[kWgMgMax], nxt[kWgMgMax];
    const int xsh = (a.kind == 0 && args.xshift != nullptr) ? *args.xshift : 0;
#pragma unroll
    for (int m = 0; m < kWgMgMax; ++m) cur[m] = fetch(0, m);
    for (int it = 0; it < total; ++it) {
      const int s = it % S, ph = (it / S) & 1;
#pragma unroll
      for (int m = 0; m < kWgMgMax; ++m) nxt[m] = fetch(it + 1, m);
      mbar_wait(&empty[s], ph ^ 1);
      if (a.kind == 0) {
        mbar_wait(&xfull[s], ph);
        const uint8_t* xs = xbuf + s * ((xbytes + 1023) & ~1023u) + 4 * h * args.x_row_stride;
#pragma unroll
        for (int m = 0; m < kWgMgMax; ++m) {
          if (m >= nm) break;
          const int k = (mt0 + m) * 128 + row;
          // rolled feature k reads staged feature (k - xsh) mod in (shift_augment)
          int src = k;
          if (xsh != 0)
            src = k >= args.in_features ? args.x_row_stride : (k >= xsh ? k - xsh : k - xsh + args.in_features);
          uint32_t v = 0;
          if (src < args.x_row_stride) {
#pragma unroll
            for (int j = 0; j < 4; ++j) v |= uint32_t(xs[j * args.x_row_stride + src]) << (8 * j);
          }
          cur[m] = v;
        }
      }
      const uint32_t A = smem_u32(smem + s * stage_bytes);
#pragma unroll
      for (int m = 0; m < (SNN_WG_EXP == 1 ? 0 : kWgMgMax); ++m) {
        if (m >= nm) break;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t byte = (cur[m] >> (8 * j)) & 0xFFu;
          st_shared_v4(A + m * kPlaneTile + sw128_off(row, 4 * h + j),
                       a.kind == 0 ? expand_bits_msb(byte) : expand_bits_lsb(byte));
        }
      }
      fence_async_smem();
      mbar_arrive(&full[s]);
#pragma unroll
      for (int m = 0; m < kWgMgMax; ++m) cur[m] = nxt[m];
    }
    // epilogue: TMEM -> smem (row per thread, rows padded by 16 bytes so the 8
    // rows of a quarter-warp hit distinct banks) -> one 1-D bulk store per row.
    // Warp w reads TMEM lanes 32 (w % 4)..; the two halves split the columns.
    mbar_wait(&acc_full[0], 0);
    tc_fence_after();
    if (clk != nullptr && threadIdx.x == 0) clk[4] = clock64();
    const uint32_t row_bytes = uint32_t(a.n_tile) * 4u;
    const uint32_t row_stride = wg_epi_row_stride(a.n_tile);
    const int nc = a.n_tile / 32, c0 = h * nc / 2, c1 = (h + 1) * nc / 2;
    if constexpr (kFused) {
      // SW128 staging for the TMA tensor stores: tile (m, 32-column group c) is
      // 128 rows x 128 bytes, 16-byte chunk j of row r at chunk j ^ (r & 7)
      for (int m = 0; m < nm; ++m)
        for (int c = c0; c < c1; ++c) {
          uint32_t r[32];
          tmem_ld32(tmem + (uint32_t((warp & 3) * 32) << 16) + m * a.n_tile + c * 32, r);
          tmem_ld_wait();
          const uint32_t base = smem_u32(smem) + uint32_t(m * nc + c) * 16384u + uint32_t(row) * 128u;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint4 v4 = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
            if (total == 0) v4 = make_uint4(0u, 0u, 0u, 0u);
            st_shared_v4(base + ((uint32_t(j) ^ uint32_t(row & 7)) << 4), v4);
          }
        }
      fence_async_smem();
      asm volatile("bar.sync 1, %0;" ::"r"(kWgProd) : "memory");
      wgrad_fused_epilogue(a, li, &maps.pm[li], split, mt0, nm, ntile, smem, rd, ad, tl, step0, clk);
    }
    for (int m = 0; m < (kFused ? 0 : nm); ++m) {
      uint8_t* srow = smem + (size_t(m) * 128 + row) * row_stride;  // stages are free now
      for (int c = c0; c < c1; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + (uint32_t((warp & 3) * 32) << 16) + m * a.n_tile + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint4 v4 = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
          if (total == 0) v4 = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(srow + c * 128 + j * 16) = v4;
        }
      }
    }
    if constexpr (!kFused) {
      fence_async_smem();
      asm volatile("bar.sync 1, %0;" ::"r"(kWgProd) : "memory");
      if (h == 0) {
        for (int m = 0; m < nm; ++m) {
          const int k = (mt0 + m) * 128 + row;
          bulk_store(a.partial + (size_t(split) * a.M_pad + k) * a.N_pad + ntile * a.n_tile,
                     smem + (size_t(m) * 128 + row) * row_stride, row_bytes);
        }
        bulk_commit_wait_all();
      }
    }
    tc_fence_before();
  }
  pdl_launch_dependents();
  __syncthreads();
  if (clk != nullptr && threadIdx.x == 0) {
    clk[5] = clock64();
    clk[7] = globaltimer();
    clk[15] = clk[7];
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_any(tmem_cols, tmem);
  }
  if constexpr (kFused) {
    // completion: the last CTA advances the step / schedule counters and re-arms
    // the tile counters (every CTA has passed its tile wait by now)
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(tl.done, 1u) == gridDim.x - 1) {
        for (int t = 0; t < tl.n_tiles_total; ++t) tl.tile_cnt[t] = 0u;
        *tl.done = 0u;
        *rd.step = step0 + 1;
        if (tl.rows_slot != nullptr) *tl.rows_slot += 1;
        __threadfence();
      }
    }
  }
}

// Single-rank step tail: k_reduce + k_adam in one launch (no allreduce between
// them).  Same block roles and the same fixed-order sums as k_reduce, each
// gradient consumed by Adam in the thread that produced it.  Every block reads
// the step counter first; the last block to finish (completion counter) advances
// it and the schedule slot, so no block can observe the advanced value.
__global__ void __launch_bounds__(256) k_reduce_adam(ReduceArgs r, AdamArgs a, unsigned int* done,
                                                     int64_t* rows_slot, long long* dbg_clk) {
  pdl_wait();
  const int tid = threadIdx.x;
  if (dbg_clk != nullptr && tid == 0) dbg_clk[size_t(blockIdx.x) * kClkStride + 14] = globaltimer();
  const int64_t s = *reinterpret_cast<volatile const int64_t*>(r.step);  // this step's bias corrections: table entry s (optimize.hpp:95-97)
  const float bc1 = a.bc[2 * s], bc2 = a.bc[2 * s + 1];
  // block 0: the serial batch-order loss sum (scheduled first, overlaps the rest);
  // blocks [1, 1 + vb_blocks): beta / bias; then one thread per W element
  const int vb_blocks = (r.n_vec + 7) / 8;
  const int wb0 = 1 + vb_blocks;
  if (blockIdx.x >= unsigned(wb0)) {
    const int64_t i = int64_t(blockIdx.x - wb0) * kRedElemsPerBlock + (tid >> 1);
    if (i < r.n_params) {
      const Entry en = r.entries[find_entry(r.entries, r.n_entries, i)];
      if (en.kind == kEntryW) {
        const int64_t li = i - en.offset;
        // Adam's operands are independent of the sum: issue them first
        float p0 = 0.0f, m0 = 0.0f, v0 = 0.0f;
        if ((tid & 1) == 0) {
          p0 = a.params[i];
          m0 = a.m[i];
          v0 = a.v[i];
        }
        const float g = sum_partials_pair(r, en, li, tid & 1);
        if ((tid & 1) == 0) {
          r.grads[i] = g;
          refresh_planes(a, en.layer, li / en.cols, li % en.cols, adam_apply(a, i, g, p0, m0, v0, bc1, bc2));
        }
      }
    }
  } else if (blockIdx.x >= 1u) {
    const int warp = tid >> 5, lane = tid & 31;
    const int v = (int(blockIdx.x) - 1) * 8 + warp;
    if (v < r.n_vec) {
      const int64_t i = r.vec_index[v];
      const Entry en = r.entries[find_entry(r.entries, r.n_entries, i)];
      const int64_t li = i - en.offset;
      const float* __restrict__ src =
          (en.kind == kEntryB ? r.dbias_part[en.layer]
                              : en.kind == kEntryGamma ? r.dgamma_part[en.layer] : r.dbeta_part[en.layer]) + li;
      float g = 0.0f;
      if (en.kind == kEntryBeta && en.beta_mode != 0) {
        // scalar beta: every (b, n) partial (mul_bcast backward, autodiff.hpp:191-205);
        // fixed beta is a tape constant -- no gradient, so Adam / SGD leave it as is
        if (en.beta_mode == 1)
          for (int q = lane; q < r.B * en.cols; q += 32) g = __fadd_rn(g, __ldg(src + q));
      } else {
        for (int b = lane; b < r.B; b += 32) g = __fadd_rn(g, __ldg(src + int64_t(b) * en.cols));
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) g = __fadd_rn(g, __shfl_xor_sync(0xffffffffu, g, off));
      if (lane == 0) {
        if (en.kind == kEntryBeta || en.kind == kEntryGamma) {
          const float beta = r.params[i];
          if (!(beta > 0.0f && beta < 1.0f)) g = 0.0f;  // clip01 gradient (autodiff.hpp:353-355)
        }
        r.grads[i] = g;
        adam_one(a, i, g, bc1, bc2);
      }
    }
  } else {
    // loss sum in batch order (objective.hpp:57-72) + hits -> StepResult
    float loss;
    int hits;
    loss_and_hits(r, loss, hits, tail_scratch(), 256);
    float l = __fdiv_rn(loss, a.loss_denom);
    for (int m = 0; m < r.n_mon; ++m) {  // loss = add(loss, regularizer) per monitor (optimize.hpp:185-191)
      const float v = activity_value(r, m, tail_scratch(), 256);
      if (tid == 0) {
        r.grads[r.n_params + 2 + m] = v;
        l = __fadd_rn(l, v);
      }
    }
    if (tid == 0) {
      r.grads[r.n_params] = loss;
      r.grads[r.n_params + 1] = float(hits);
      *a.loss_out = l;
      *a.acc_out = double(hits) / double(a.B_global);
    }
  }
  // completion: the last block advances the step (and schedule slot) counters
  __syncthreads();
  if (dbg_clk != nullptr && tid == 0) dbg_clk[size_t(blockIdx.x) * kClkStride + 15] = globaltimer();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *done = 0u;
      *r.step = s + 1;
      if (rows_slot != nullptr) *rows_slot += 1;
      __threadfence();
    }
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

// Host-batch layout [n][tp8][IN] (reference packed, data.hpp:105-126) -> the
// staged layout [n][tp8_pad][IN_pad], zero padded.  One thread per 4 output bytes;
// rows whose feature count is a multiple of 4 copy whole words (32-bit indexing:
// a host batch is far below 4 GB).
__global__ void k_relayout(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t n,
                           int tp8, int tp8_pad, int IN, int IN_pad) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t wpr = uint32_t(IN_pad) / 4;  // output words per row
  const uint32_t row = q / wpr, w = q - row * wpr;
  if (uint64_t(row) >= uint64_t(n) * tp8_pad) return;
  const uint32_t g = row % uint32_t(tp8_pad), i = row / uint32_t(tp8_pad);
  uint32_t word = 0;
  if (g < uint32_t(tp8)) {
    const uint32_t src = (i * uint32_t(tp8) + g) * uint32_t(IN);  // first byte of the source row
    if ((IN & 3) == 0) {
      if (4 * w < uint32_t(IN)) word = *reinterpret_cast<const uint32_t*>(in + src + 4 * w);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t k = 4 * w + e;
        if (k < uint32_t(IN)) word |= uint32_t(in[src + k]) << (8 * e);
      }
    }
  }
  reinterpret_cast<uint32_t*>(out)[q] = word;  // IN_pad is a multiple of 64
}

// StepResult of pipelined step k into mapped pinned host memory (no D2H copy on
// the compute stream between steps).
__global__ void k_result_out(const float* loss, const double* acc, float* host_loss, double* host_acc) {
  *host_loss = *loss;
  *host_acc = *acc;
}

// monitor_activity (neuron.hpp:106-114): counts[b][n] = spikes of (b, n) over the
// window, from the time-packed raster of the last forward.
__global__ void k_spike_counts(const uint32_t* __restrict__ s_tp, int B, int T_pad, int H,
                               float* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(B) * H) return;
  const int b = int(i / H), n = int(i % H), wpb = T_pad / 32;
  const uint32_t* w = s_tp + size_t(n) * (size_t(B) * wpb) + size_t(b) * wpb;
  int c = 0;
  for (int k = 0; k < wpb; ++k) c += __popc(__ldg(w + k));
  out[i] = float(c);
}

// StepResult{loss / B_global, hits / B_global}; advances the step counter.
__global__ void k_result(const float* tail, int B_global, float loss_denom, int64_t* step,
                         int do_step, float* loss_out, double* acc_out, int n_mon) {
  pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  float l = __fdiv_rn(tail[0], loss_denom);
  for (int m = 0; m < n_mon; ++m) l = __fadd_rn(l, tail[2 + m]);
  *loss_out = l;
  *acc_out = double(tail[1]) / double(B_global);
  if (do_step) *step += 1;
}

}  // namespace snn
