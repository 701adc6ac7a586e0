// throughput probe: mma.sync m16n8k16 f64 vs DFMA on sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_k(double* out, int iters) {
  double a[8], b[4], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; i++) b[i] = threadIdx.x * 2e-3 + i;
  for (int it = 0; it < iters; it++) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0] + c[1] + c[2] + c[3];
}
__global__ void dfma_k(double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3 + i;
  const double m = 1.0000001, a = 1e-9;
  for (int it = 0; it < iters; it++)
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], m, a);
  double s = 0;
  for (int i = 0; i < 8; i++) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096, blocks = 148 * 8, threads = 256;
  dmma_k<<<blocks, threads>>>(out, 16);
  cudaEventRecord(a);
  dmma_k<<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fl = 2.0 * 16 * 8 * 16 * double(iters) * blocks * (threads / 32);
  printf("DMMA m16n8k16: %.1f TFLOP/s\n", fl / ms / 1e9);
  dfma_k<<<blocks, threads>>>(out, 16);
  cudaEventRecord(a);
  dfma_k<<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  fl = 2.0 * 8 * double(iters) * blocks * threads;
  printf("DFMA: %.1f TFLOP/s\n", fl / ms / 1e9);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
