// Dependent-chain latencies on this GPU (cycles per op): DFMA, DMUL, DADD, FFMA, MUFU.RSQ64H-based
// rsqrt(double), fp64 division, LDS, SHFL, __syncwarp(partial mask), bar.sync (named, 64 threads).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, int n, double a) {
  __shared__ double sm[256];
  __shared__ int idx[256];
  sm[threadIdx.x] = a * threadIdx.x;
  idx[threadIdx.x] = (threadIdx.x + 1) & 255;
  __syncthreads();
  double x = a + threadIdx.x * 1e-9, y = 1.0 + 1e-9 * threadIdx.x;
  float f = (float)x;
  long long t0, t1;
  int slot = 0;
#define MEAS(k, body)                 \
  t0 = clock64();                     \
  for (int i = 0; i < n; ++i) { body; } \
  t1 = clock64();                     \
  if (threadIdx.x == 0) cyc[k] = (t1 - t0);
  MEAS(0, x = fma(x, y, 1e-9))
  MEAS(1, x = x * y)
  MEAS(2, x = x + y)
  MEAS(3, f = fmaf(f, 1.0000001f, 1e-9f))
  MEAS(4, x = rsqrt(x + 2.0))
  MEAS(5, x = 1.0 / (x + 2.0))
  MEAS(6, x = sqrt(x + 2.0))
  MEAS(7, slot = idx[slot])
  MEAS(8, x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9)
  MEAS(9, { x = sm[(int)(x) & 255] + 1e-9; })
  MEAS(10, { __syncwarp(0x0000ffffu << (16 * ((threadIdx.x >> 4) & 1))); x += 1e-9; })
  MEAS(11, { if (threadIdx.x < 64) asm volatile("bar.sync 1, 64;" ::: "memory"); x += 1e-9; })
  MEAS(12, { __syncthreads(); x += 1e-9; })
  MEAS(13, { float g = (float)x; x = (double)(g * 1.0000001f); })
  out[threadIdx.x] = x + f + slot;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256 * sizeof(double));
  cudaMallocManaged(&cyc, 32 * sizeof(long long));
  const int n = 4096;
  const char* names[] = {"DFMA", "DMUL", "DADD", "FFMA", "rsqrt(double)", "1.0/double", "sqrt(double)",
                         "LDS (int chase)", "SHFL.xor f64 + add", "LDS f64 + DADD", "syncwarp(16-lane mask)+DADD",
                         "bar.sync 64 + DADD", "__syncthreads (128) + DADD", "F2F pair + FMUL"};
  for (int warps : {4}) {
    k_lat<<<1, 32 * warps>>>(out, cyc, n, 0.5);
    cudaDeviceSynchronize();
    printf("threads %d\n", 32 * warps);
    for (int k = 0; k < 14; ++k) printf("  %-28s %.1f cyc/op\n", names[k], (double)cyc[k] / n);
  }
  return 0;
}
