// Microbenchmark: dependent-chain latency of DADD / DMUL / DFMA on the GPU
// (one thread, clock64 around N dependent ops), and the rate of a sequential
// sum fed from shared memory. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_add(double* out, long long* cyc, int n, double a) {
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, a);
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}

__global__ void chain_mul(double* out, long long* cyc, int n, double a) {
  double acc = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __dmul_rn(acc, a);
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}

__global__ void chain_smem(double* out, long long* cyc, int n) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 1e-3 * i;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double acc = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < n / 4096; ++rep) {
#pragma unroll 16
    for (int i = 0; i < 4096; ++i) acc = __dadd_rn(acc, __dmul_rn(buf[i], buf[4095 - i]));
  }
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 8);
  cudaMalloc(&c, 8);
  const int n = 1 << 20;
  long long h;
  chain_add<<<1, 1>>>(d, c, 1000, 1.0);
  chain_add<<<1, 1>>>(d, c, n, 1e-9);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / n);
  chain_mul<<<1, 1>>>(d, c, n, 1.0000001);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DMUL dependent latency: %.2f cycles\n", (double)h / n);
  chain_smem<<<1, 128>>>(d, c, n);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("smem-fed DMUL+DADD chain: %.2f cycles per element\n", (double)h / n);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SM clock attribute: %d kHz\n", clk);
  return 0;
}
