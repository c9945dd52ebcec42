// DMMA (mma.sync m8n8k4 f64) latency and throughput at low occupancy.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 0.5;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH> void run(int warps, int blocks) {
  double* d; long long* c; cudaMalloc(&d, 8); cudaMalloc(&c, 8);
  int iters = 2000;
  k<CH><<<blocks, warps * 32>>>(d, c, iters); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<CH><<<blocks, warps * 32>>>(d, c, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  double tf = 2.0 * 256 * CH * iters * (double)warps * blocks / (ms * 1e9);
  printf("chains/warp %d warps/SM %d blocks %d: %.1f cycles per dmma per chain, %.2f TFLOP/s\n", CH, warps, blocks, (double)cy / iters, tf);
}
int main() {
  run<1>(1, 1); run<3>(1, 1); run<8>(1, 1);
  run<1>(16, 148); run<3>(16, 148); run<8>(16, 148); run<3>(32, 148);
}
