#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, double a, double b, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; out[1] = (double)(t1 - t0) / n; }
}
__global__ void thr(double* out, double a, double b, int n) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < n; ++i) { x0 = fma(x0,a,b); x1 = fma(x1,a,b); x2 = fma(x2,a,b); x3 = fma(x3,a,b); x4 = fma(x4,a,b); x5 = fma(x5,a,b); x6 = fma(x6,a,b); x7 = fma(x7,a,b);}
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void thr32(float* out, float a, float b, int n) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < n; ++i) { x0 = fmaf(x0,a,b); x1 = fmaf(x1,a,b); x2 = fmaf(x2,a,b); x3 = fmaf(x3,a,b); x4 = fmaf(x4,a,b); x5 = fmaf(x5,a,b); x6 = fmaf(x6,a,b); x7 = fmaf(x7,a,b);}
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}
int main() {
  double* d; cudaMalloc(&d, 1 << 26);
  lat<<<1, 32>>>(d, 0.999, 0.001, 10000);
  double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("fp64 fma dependent latency: %.1f cycles\n", h[1]);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int n = 4096;
  thr<<<148 * 4, 512>>>(d, 0.999, 0.001, n);
  cudaEventRecord(e0); thr<<<148 * 4, 512>>>(d, 0.999, 0.001, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("fp64 FMA throughput: %.2f TFLOP/s\n", 2.0 * 8 * n * 148.0 * 4 * 512 / (ms * 1e-3) / 1e12);
  thr32<<<148 * 4, 512>>>((float*)d, 0.999f, 0.001f, n);
  cudaEventRecord(e0); thr32<<<148 * 4, 512>>>((float*)d, 0.999f, 0.001f, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("fp32 FMA throughput: %.2f TFLOP/s\n", 2.0 * 8 * n * 148.0 * 4 * 512 / (ms * 1e-3) / 1e12);
  return 0;
}
