// Probe: FP64 DMMA (mma.sync m8n8k4 f64) vs DFMA throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double acc[NACC][2];
  #pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = threadIdx.x; acc[i][1] = i; }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NACC>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[NACC];
  #pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d cc %d.%d clock %d kHz\n", p.name, p.multiProcessorCount, p.major, p.minor, p.clockRate);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {128, 256, 512}) for (int cpsm : {1, 2, 4}) {
    int iters = 20000;
    int blocks = sms * cpsm;
    k_dmma<8><<<blocks, threads>>>(out, 100, 1.0, 1e-9);
    cudaEventRecord(e0);
    k_dmma<8><<<blocks, threads>>>(out, iters, 1.0, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
    printf("DMMA m8n8k4 threads %d ctas/sm %d: %.2f TFLOP/s (%.3f ms)\n", threads, cpsm, flops / ms / 1e9, ms);
  }
  for (int threads : {256, 512, 1024}) for (int cpsm : {1, 2}) {
    int iters = 20000;
    int blocks = sms * cpsm;
    k_dfma<8><<<blocks, threads>>>(out, 100, 1.0, 1e-9);
    cudaEventRecord(e0);
    k_dfma<8><<<blocks, threads>>>(out, iters, 1.0, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf("DFMA threads %d ctas/sm %d: %.2f TFLOP/s\n", threads, cpsm, flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
