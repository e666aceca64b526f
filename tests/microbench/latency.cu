// Dependent-chain latency microbenchmarks (cycles per op) on the target GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false latency.cu -o latency
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fadd(float* out, long long* cyc, int n, float a) {
  float v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = __fadd_rn(__fmul_rn(v, a), 1.0f);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_shfl(float* out, long long* cyc, int n) {
  float v = threadIdx.x;
  int src = threadIdx.x & 31;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    v = __shfl_sync(0xffffffffu, v, src);
    src = (int(v) + i) & 31;
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_lds(float* out, long long* cyc, int n) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i * 7 + 3) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = buf[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_idiv(float* out, long long* cyc, int n, int d) {
  int v = threadIdx.x + 1000000;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = v / d + v % d + 999999;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 4);
  cudaMalloc(&cyc, 8);
  const int n = 4096;
  long long h;
  for (int rep = 0; rep < 2; ++rep) {
    k_fadd<<<1, 32>>>(out, cyc, n, 0.999f);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("fmul+fadd dependent pair: %.2f cycles\n", double(h) / n);
    k_shfl<<<1, 32>>>(out, cyc, n);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("shfl.idx dependent (+cvt,add,and): %.2f cycles\n", double(h) / n);
    k_lds<<<1, 32>>>(out, cyc, n);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("lds pointer chase: %.2f cycles\n", double(h) / n);
    k_idiv<<<1, 32>>>(out, cyc, n, 4);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("int div+mod by runtime d (+add): %.2f cycles\n", double(h) / n);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
