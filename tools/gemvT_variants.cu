// Microbenchmark: variants of x = A^T y for A row-major m x lda (cfg2 shape).
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <cstdlib>

template <int NT, int U, int CP>
__global__ void __launch_bounds__(NT) gT_rows(const double* __restrict__ A, long lda, int m, const double* __restrict__ y,
                                              double* __restrict__ x, int r0g, int nrg, double* part) {
  // CP column pairs per thread (strided by NT), rows [r0, r1)
  __shared__ double ys[4096];
  const int rg = blockIdx.y;
  const int rows_per = (m + nrg - 1) / nrg;
  const int r0 = rg * rows_per, r1 = min(m, r0 + rows_per);
  for (int i = threadIdx.x; i < r1 - r0; i += NT) ys[i] = y[r0 + i];
  __syncthreads();
  const long ld2 = lda / 2;
  const long base = (long)blockIdx.x * NT * CP + threadIdx.x;
  double w[CP][2] = {};
  const double2* Ap = reinterpret_cast<const double2*>(A) + (long)r0 * ld2;
  int i = 0;
  const int nr = r1 - r0;
  for (; i + U <= nr; i += U) {
    double2 buf[U][CP];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < CP; ++c) buf[u][c] = __ldcs(Ap + (long)(i + u) * ld2 + base + c * NT);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        w[c][0] = fma(buf[u][c].x, ys[i + u], w[c][0]);
        w[c][1] = fma(buf[u][c].y, ys[i + u], w[c][1]);
      }
  }
  for (; i < nr; ++i)
#pragma unroll
    for (int c = 0; c < CP; ++c) {
      double2 a = __ldcs(Ap + (long)i * ld2 + base + c * NT);
      w[c][0] = fma(a.x, ys[i], w[c][0]);
      w[c][1] = fma(a.y, ys[i], w[c][1]);
    }
#pragma unroll
  for (int c = 0; c < CP; ++c) {
    long t = 2 * (base + c * NT);
    if (nrg == 1) { x[t] = w[c][0]; x[t + 1] = w[c][1]; }
    else { part[(long)rg * lda + t] = w[c][0]; part[(long)rg * lda + t + 1] = w[c][1]; }
  }
}

__global__ void reduce_parts(const double* part, int nrg, long lda, double* x) {
  long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= lda) return;
  double s = 0;
  for (int r = 0; r < nrg; ++r) s += part[(long)r * lda + t];
  x[t] = s;
}

// gemv-like pattern per tile: thread streams along a row; tile = RB rows x chunk
template <int RB>
__global__ void __launch_bounds__(256) gv(const double* __restrict__ A, long lda, int m, const double* __restrict__ v, int chunk, double* part) {
  const int row0 = blockIdx.x * RB;
  const long c0 = (long)blockIdx.y * chunk;
  const long c1 = (c0 + chunk < lda) ? c0 + chunk : lda;
  double acc[RB] = {};
  const double2* v2 = reinterpret_cast<const double2*>(v);
#pragma unroll 4
  for (long t = c0 / 2 + threadIdx.x; t < c1 / 2; t += 256) {
    const double2 vv = __ldg(v2 + t);
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const double2 aa = __ldcs(reinterpret_cast<const double2*>(A + (long)(row0 + r) * lda) + t);
      acc[r] = fma(aa.x, vv.x, acc[r]);
      acc[r] = fma(aa.y, vv.y, acc[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    double s = acc[r];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
    if ((threadIdx.x & 31) == 0) part[(long)blockIdx.y * m * 8 + (row0 + r) * 8 + (threadIdx.x >> 5)] = s;
  }
}

int main() {
  const int m = 2000;
  const long N = 164055, lda = 164064;
  double *A, *y, *x, *part;
  cudaMalloc(&A, (size_t)m * lda * 8);
  cudaMalloc(&y, m * 8);
  cudaMalloc(&x, lda * 8);
  cudaMalloc(&part, (size_t)32 * lda * 8);
  cudaMemset(A, 0, (size_t)m * lda * 8);
  std::vector<double> hy(m, 1.0);
  cudaMemcpy(y, hy.data(), m * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)m * N * 8;
  auto run = [&](const char* name, auto f) {
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(e0);
    const int R = 20;
    for (int i = 0; i < R; ++i) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= R;
    printf("%-40s %8.3f ms  %7.1f GB/s  err=%s\n", name, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  const long pairs = lda / 2;
  run("gT 128thr U16 CP1", [&] { gT_rows<128, 16, 1><<<dim3(pairs / 128 + 1, 1), 128>>>(A, lda, m, y, x, 0, 1, part); });
  run("gT 128thr U8 CP2", [&] { gT_rows<128, 8, 2><<<dim3(pairs / 256 + 1, 1), 128>>>(A, lda, m, y, x, 0, 1, part); });
  run("gT 256thr U8 CP1", [&] { gT_rows<256, 8, 1><<<dim3(pairs / 256 + 1, 1), 256>>>(A, lda, m, y, x, 0, 1, part); });
  run("gT 64thr U16 CP1", [&] { gT_rows<64, 16, 1><<<dim3(pairs / 64 + 1, 1), 64>>>(A, lda, m, y, x, 0, 1, part); });
  for (int nrg : {2, 4, 8, 16}) {
    char nm[64];
    sprintf(nm, "gT 128thr U16 CP1 rowgroups=%d", nrg);
    run(nm, [&] {
      gT_rows<128, 16, 1><<<dim3(pairs / 128 + 1, nrg), 128>>>(A, lda, m, y, x, 0, nrg, part);
      reduce_parts<<<(lda + 255) / 256, 256>>>(part, nrg, lda, x);
    });
    sprintf(nm, "gT 256thr U8 CP2 rowgroups=%d", nrg);
    run(nm, [&] {
      gT_rows<256, 8, 2><<<dim3(pairs / 512 + 1, nrg), 256>>>(A, lda, m, y, x, 0, nrg, part);
      reduce_parts<<<(lda + 255) / 256, 256>>>(part, nrg, lda, x);
    });
  }
  run("gemv RB4 chunk8192", [&] { gv<4><<<dim3(m / 4, (lda + 8191) / 8192), 256>>>(A, lda, m, y, 8192, part); });
  run("gemv RB8 chunk8192", [&] { gv<8><<<dim3(m / 8, (lda + 8191) / 8192), 256>>>(A, lda, m, y, 8192, part); });
  run("gemv RB4 chunk16384", [&] { gv<4><<<dim3(m / 4, (lda + 16383) / 16384), 256>>>(A, lda, m, y, 16384, part); });
  run("gemv RB2 chunk4096", [&] { gv<2><<<dim3(m / 2, (lda + 4095) / 4096), 256>>>(A, lda, m, y, 4096, part); });
  return 0;
}
