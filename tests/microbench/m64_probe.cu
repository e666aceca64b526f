// TMEM placement of a cta_group::1 M=64 tcgen05.mma accumulator (probe; not product code).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2402_18994_b200/csrc \
//        tests/microbench/m64_probe.cu -o /tmp/m64_probe && /tmp/m64_probe
// A[i][k] = (k == 0) ? i + 1 : 0 (64 x 64, K-major SW128), B[s][k] = (k == 0) ? s + 1 : 0
// (16 x 64): D[i][s] = (i + 1)(s + 1).  Prints, for every TMEM lane and column holding a
// nonzero value, which (i, s) it is.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda.h>
#include "sm100.cuh"
using namespace snn::sm100;

__global__ void probe(float* out, int N) {
  __shared__ __align__(1024) uint8_t sA[64 * 128];
  __shared__ __align__(1024) uint8_t sB[32 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    const uint32_t off = sw128_off(r, k / 8) + (k % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = __float2bfloat16(k == 0 ? float(r + 1) : 0.0f);
  }
  for (int i = tid; i < 32 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    const uint32_t off = sw128_off(r, k / 8) + (k % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = __float2bfloat16(k == 0 && r < N ? float(r + 1) : 0.0f);
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<32>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(64, N, false, false);
    umma_bf16(tmem, sdesc_sw128(smem_u32(sA), 16, 1024), sdesc_sw128(smem_u32(sB), 16, 1024), idesc, 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld32(tmem + (uint32_t(warp * 32) << 16), r);
  tmem_ld_wait();
  for (int c = 0; c < 32; ++c) out[(warp * 32 + (tid & 31)) * 32 + c] = __uint_as_float(r[c]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<32>(tmem);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 32 * 4);
  cudaMemset(d, 0, 128 * 32 * 4);
  for (int N : {16, 32}) {
    probe<<<1, 128>>>(d, N);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    std::printf("N=%d err=%s\n", N, cudaGetErrorString(e));
    for (int lane = 0; lane < 128; ++lane) {
      int first = -1, cnt = 0;
      for (int c = 0; c < 32; ++c)
        if (h[lane * 32 + c] != 0.0f) { if (first < 0) first = c; ++cnt; }
      if (cnt) {
        std::printf(" lane %3d: %d nonzero from col %d:", lane, cnt, first);
        for (int c = first; c < first + cnt && c < 32; ++c) std::printf(" %g", h[lane * 32 + c]);
        std::printf("\n");
      }
    }
  }
  return 0;
}
