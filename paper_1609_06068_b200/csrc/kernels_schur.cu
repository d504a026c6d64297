// S^-1 of the KKT Schur complement S = A D^-1 A^T on the GPU (the factorisation cached once,
// P:233; the iteration applies the dense S^-1 as one mat-vec).
//
// Blocked Gauss-Jordan "sweep" of the symmetric positive definite S, pivot blocks K of 32 in order
// (no pivoting: S is SPD).  Sweeping block K of the current matrix M with D = M_KK:
//     M_KK <- -D^-1,   M_iK <- M_iK D^-1,   M_Kj <- D^-1 M_Kj,   M_ij <- M_ij - M_iK D^-1 M_Kj
// (i, j outside K).  Every sweep keeps M symmetric, and after all blocks M = -S^-1.  D at block K is
// the Schur complement of the blocks before it, so its pivots are the squared diagonal of the
// Cholesky factor: a pivot <= 1e-12 of its original diagonal entry (or not finite) marks S as
// singular, the same test as the host Cholesky.  Work 2 m^3, all of it in the rank-32 updates.
//
// Two kernels per block step: k_gj_diag (one CTA) forms -D^-1 by a 32 x 32 Gauss-Jordan sweep in
// shared memory; k_gj_sweep, out of place (M -> M'), one CTA per 64 x 64 tile of M', forms
// W_I = M_IK D^-1 for its rows and updates its tile with DMMA (mma.sync m8n8k4 f64):
// M'_IJ = M_IJ - W_I M_JK^T.  Tiles meeting row / column block K write W or -D^-1 instead.
#include "internal.h"

namespace sdp {

namespace {

constexpr int GJ_B = 32;      // pivot block
constexpr int GJ_T = 64;      // output tile
constexpr int GJ_NT = 256;    // threads
constexpr int GJ_LD = GJ_B + 4;  // smem row stride of the 64 x 32 panels (4 mod 32 words: conflict-free frags)
constexpr size_t kGjSmem = (size_t)(GJ_B * (GJ_B + 1) + 3 * GJ_T * GJ_LD) * sizeof(double);

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// -D^-1 of the current pivot block D = M_KK (32 x 32 Gauss-Jordan sweep in shared memory), with the
// pivot test; one CTA, once per block step
__global__ void __launch_bounds__(GJ_NT) k_gj_diag(const double* __restrict__ M, int m, int kb,
                                                    const double* __restrict__ diag0, int* bad, double* Dout) {
  __shared__ double Dm[GJ_B][GJ_B + 1];
  const int tid = threadIdx.x;
  const int bK = min(GJ_B, m - kb);
  for (int e = tid; e < GJ_B * GJ_B; e += GJ_NT) {
    const int r = e / GJ_B, c = e % GJ_B;
    Dm[r][c] = (r < bK && c < bK) ? M[(int64_t)(kb + r) * m + kb + c] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int p = 0; p < GJ_B; ++p) {
    double piv = Dm[p][p];
    if (p < bK && !(piv > 1e-12 * diag0[kb + p] && isfinite(piv))) {
      if (tid == 0) *bad = 1;
      piv = 1.0;
    }
    const double ip = 1.0 / piv;
    __syncthreads();
    // a_ij -= a_ip a_pj / piv (i, j != p); then row / column p scaled, a_pp = -1 / piv
    for (int e = tid; e < GJ_B * GJ_B; e += GJ_NT) {
      const int r = e / GJ_B, c = e % GJ_B;
      if (r != p && c != p) Dm[r][c] -= Dm[r][p] * Dm[p][c] * ip;
    }
    __syncthreads();
    if (tid < GJ_B && tid != p) {
      Dm[tid][p] *= ip;
      Dm[p][tid] *= ip;
    }
    if (tid == GJ_B) Dm[p][p] = -ip;
    __syncthreads();
  }
  for (int e = tid; e < GJ_B * GJ_B; e += GJ_NT) Dout[e] = Dm[e / GJ_B][e % GJ_B];
}

__global__ void __launch_bounds__(GJ_NT) k_gj_sweep(const double* __restrict__ M, double* __restrict__ Mn, int m,
                                                     int kb, const double* __restrict__ Dg, int last) {
  extern __shared__ double gj_smem[];
  // D (swept in place to -D^-1); M_IK (then W_J where rows of K are in the tile); M_JK; W_I
  double(*Dm)[GJ_B + 1] = reinterpret_cast<double(*)[GJ_B + 1]>(gj_smem);
  double(*PI)[GJ_LD] = reinterpret_cast<double(*)[GJ_LD]>(gj_smem + GJ_B * (GJ_B + 1));
  double(*PJ)[GJ_LD] = PI + GJ_T;
  double(*Wt)[GJ_LD] = PJ + GJ_T;
  const int tid = threadIdx.x;
  const int i0 = blockIdx.y * GJ_T, j0 = blockIdx.x * GJ_T;
  const int bK = min(GJ_B, m - kb);
  // ---- -D^-1 (k_gj_diag)
  for (int e = tid; e < GJ_B * GJ_B; e += GJ_NT) Dm[e / GJ_B][e % GJ_B] = Dg[e];
  // ---- panels M_IK, M_JK (zero beyond m / bK)
  for (int e = tid; e < GJ_T * GJ_B; e += GJ_NT) {
    const int r = e / GJ_B, c = e % GJ_B;
    const int gi = i0 + r, gj = j0 + r;
    PI[r][c] = (gi < m && c < bK) ? M[(int64_t)gi * m + kb + c] : 0.0;
    PJ[r][c] = (gj < m && c < bK) ? M[(int64_t)gj * m + kb + c] : 0.0;
  }
  __syncthreads();
  // ---- W_I = M_IK D^-1 = -(M_IK Dm)
  for (int e = tid; e < GJ_T * GJ_B; e += GJ_NT) {
    const int r = e / GJ_B, c = e % GJ_B;
    double s = 0.0;
#pragma unroll 8
    for (int l = 0; l < GJ_B; ++l) s = fma(PI[r][l], Dm[l][c], s);
    Wt[r][c] = -s;
  }
  __syncthreads();
  const bool rowsK = i0 < kb + bK && kb < i0 + GJ_T;  // tile rows meet K
  const bool colsK = j0 < kb + bK && kb < j0 + GJ_T;
  // ---- C = M_IJ - W_I M_JK^T (DMMA: warp w owns rows 16 (w / 2) .. +16, cols 32 (w % 2) .. +32)
  const int warp = tid >> 5, lane = tid & 31;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int r = i0 + wr + a * 8 + (lane >> 2);
      const int c = j0 + wc + b * 8 + (lane & 3) * 2;
      acc[a][b][0] = (r < m && c < m) ? M[(int64_t)r * m + c] : 0.0;
      acc[a][b][1] = (r < m && c + 1 < m) ? M[(int64_t)r * m + c + 1] : 0.0;
    }
#pragma unroll
  for (int k = 0; k < GJ_B; k += 4) {
    double af[2], bf[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) af[a] = -Wt[wr + a * 8 + (lane >> 2)][k + (lane & 3)];
#pragma unroll
    for (int b = 0; b < 4; ++b) bf[b] = PJ[wc + b * 8 + (lane >> 2)][k + (lane & 3)];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma(acc[a][b], af[a], bf[b]);
  }
  // W_J (for tile rows inside K: M'_ij = W_j,(i - kb))
  if (rowsK) {
    __syncthreads();
    for (int e = tid; e < GJ_T * GJ_B; e += GJ_NT) {
      const int r = e / GJ_B, c = e % GJ_B;
      double s = 0.0;
#pragma unroll 8
      for (int l = 0; l < GJ_B; ++l) s = fma(PJ[r][l], Dm[l][c], s);
      PI[r][c] = -s;  // PI is free now: W_J
    }
    __syncthreads();
  }
  const double sgn = last ? -1.0 : 1.0;  // the last sweep leaves -S^-1: store S^-1
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rl = wr + a * 8 + (lane >> 2), cl = wc + b * 8 + (lane & 3) * 2 + h;
        const int r = i0 + rl, c = j0 + cl;
        if (r >= m || c >= m) continue;
        const bool ri = r >= kb && r < kb + bK, ci = c >= kb && c < kb + bK;
        double v = acc[a][b][h];
        if (ri && ci)
          v = Dm[r - kb][c - kb];     // -D^-1
        else if (ci)
          v = Wt[rl][c - kb];          // W_i
        else if (ri)
          v = PI[cl][r - kb];          // W_j (rowsK)
        (void)colsK;
        Mn[(int64_t)r * m + c] = sgn * v;
      }
}

}  // namespace

// In-place-equivalent inversion: S (device, m x m row-major, symmetric positive definite) is
// overwritten; Sinv receives S^-1; work: m x m doubles; diag0: m + 1024 doubles; bad: 1 int (device).
// Returns false if S is not positive definite to the 1e-12 pivot test.
bool spd_inverse_gpu(double* S, int m, double* Sinv, double* work, double* diag0, int* bad, cudaStream_t s) {
  // (diag0 holds m doubles + the 32 x 32 -D^-1 of the current step)
  double* Dg = diag0 + m;
  SDP_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), s));
  // original diagonal (strided copy)
  SDP_CUDA_TRY(cudaMemcpy2DAsync(diag0, sizeof(double), S, (size_t)(m + 1) * sizeof(double), sizeof(double), m,
                                 cudaMemcpyDeviceToDevice, s));
  const int nblk = (m + GJ_B - 1) / GJ_B;
  const int nt = (m + GJ_T - 1) / GJ_T;
  SDP_CUDA_TRY(cudaFuncSetAttribute(k_gj_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGjSmem));
  // ping-pong S -> work -> S ...; the last sweep writes Sinv
  double* cur = S;
  double* nxt = work;
  for (int k = 0; k < nblk; ++k) {
    const bool last = k == nblk - 1;
    double* dst = last ? Sinv : nxt;
    k_gj_diag<<<1, GJ_NT, 0, s>>>(cur, m, k * GJ_B, diag0, bad, Dg);
    k_gj_sweep<<<dim3(nt, nt), GJ_NT, kGjSmem, s>>>(cur, dst, m, k * GJ_B, Dg, last ? 1 : 0);
    SDP_CUDA_TRY(cudaGetLastError());
    if (!last) {
      double* t = cur;
      cur = nxt;
      nxt = t;
    }
  }
  int hbad = 0;
  SDP_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  SDP_CUDA_TRY(cudaStreamSynchronize(s));
  return hbad == 0;
}

}  // namespace sdp
