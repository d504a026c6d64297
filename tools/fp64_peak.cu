// FP64 throughput microbenchmark on sm_100a: scalar DFMA vs DMMA (mma.sync
// m8n8k4 f64).  Prints TFLOP/s for each; the bench's FP64 roofline denominator
// is the measured value (profiles/r1/fp64_peak.txt).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double acc[8][2];
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int tpb : {256, 512, 1024}) {
    int grid = sms * (2048 / tpb);
    k_dfma<<<grid, tpb>>>(d, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    k_dfma<<<grid, tpb>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)grid * tpb;
    printf("DFMA  tpb=%4d grid=%5d  %.2f TFLOP/s\n", tpb, grid, fl / ms / 1e9);
  }
  for (int tpb : {128, 256, 512}) {
    int grid = sms * (2048 / tpb);
    k_dmma<<<grid, tpb>>>(d, 100);
    cudaEventRecord(e0);
    k_dmma<<<grid, tpb>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid * (tpb / 32);
    printf("DMMA  tpb=%4d grid=%5d  %.2f TFLOP/s\n", tpb, grid, fl / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
