// FP64 pipe microbenchmarks for the B200 roofline denominator (MEASURED_PEAKS.json
// has no FP64 entry).  Measures: DFMA throughput, DMMA (mma.sync m8n8k4 f64)
// throughput, both running concurrently in one kernel, and the cost of FP64
// exp / sigmoid as used by the decoder.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double aa = a + threadIdx.x * 1e-9, bb = b;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i], aa, bb);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// even warps DFMA, odd warps DMMA: do the two share one pipe?
__global__ void k_mixed(double* out, double a, double b) {
  int w = threadIdx.x / 32;
  if (w & 1) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    double aa = a + threadIdx.x * 1e-9, bb = b;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i], aa, bb);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
  } else {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
  }
}

__global__ void k_exp(double* out, double a) {
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = (threadIdx.x % 64) * 1e-2 - 0.3 + i * 1e-3;
  double s = 0;
  for (int it = 0; it < ITERS / 16; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) { double e = exp(x[i]); s += e; x[i] = x[i] * a + 1e-7; }
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void k_sigmoid(double* out, double a) {
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = (threadIdx.x % 64) * 1e-2 - 0.3 + i * 1e-3;
  double s = 0;
  for (int it = 0; it < ITERS / 16; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double z = x[i];
      double sg = 1.0 / (1.0 + exp(-z));
      s += z * sg + sg * (1.0 + z * (1.0 - sg));
      x[i] = x[i] * a + 1e-7;
    }
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0;
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, dev));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, p.multiProcessorCount, clk_khz);
  double* d;
  CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    float ms;
    // DFMA
    k_dfma<<<blocks, tpb>>>(d, 0.999999, 1e-6);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_dfma<<<blocks, tpb>>>(d, 0.999999, 1e-6);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * ITERS * (double)blocks * tpb;
    printf("{\"test\": \"dfma\", \"tpb\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", tpb, ms, fl / ms / 1e9);
    // DMMA
    k_dmma<<<blocks, tpb>>>(d, 0.5, 0.25);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_dmma<<<blocks, tpb>>>(d, 0.5, 0.25);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 8 * (ITERS / 4) * (double)blocks * (tpb / 32);
    printf("{\"test\": \"dmma\", \"tpb\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", tpb, ms, fl / ms / 1e9);
    // mixed
    k_mixed<<<blocks, tpb>>>(d, 0.5, 0.25);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_mixed<<<blocks, tpb>>>(d, 0.5, 0.25);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 0.5 * (2.0 * 256 * 8 * (ITERS / 4) * (double)blocks * (tpb / 32))
       + 0.5 * (2.0 * 8 * ITERS * (double)blocks * tpb);
    printf("{\"test\": \"mixed\", \"tpb\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", tpb, ms, fl / ms / 1e9);
    // exp
    k_exp<<<blocks, tpb>>>(d, 0.9999);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_exp<<<blocks, tpb>>>(d, 0.9999);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double n = 4.0 * (ITERS / 16) * (double)blocks * tpb;
    printf("{\"test\": \"exp\", \"tpb\": %d, \"ms\": %.4f, \"gexp_per_s\": %.3f}\n", tpb, ms, n / ms / 1e6);
    k_sigmoid<<<blocks, tpb>>>(d, 0.9999);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_sigmoid<<<blocks, tpb>>>(d, 0.9999);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\": \"swish+deriv\", \"tpb\": %d, \"ms\": %.4f, \"g_per_s\": %.3f}\n", tpb, ms, n / ms / 1e6);
  }
  return 0;
}
