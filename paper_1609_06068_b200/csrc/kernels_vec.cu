// Per-iteration vector kernels of Algorithms 1 and 2 (everything except the
// clique projection):
//   scatter   r1 = sum_k H_k^T(.)  (E:OptCondMinYPrimal / E:OptCondMinYDual rhs)
//   gemv      u  = A (D^-1 r1) - r2           (block elimination)
//   symv      y  = S^-1 u with the cached S^-1 = W^T W (W = L^-1); the kernel
//             also sums the gemv partials into u (single rank)
//   gemvT     x  = D^-1 (r1 - A^T y)
//   update    v_k, lambda_k of the dual (E:vkEqn, E:MultUpdateDualSDP)
//   finalize  eps_p, eps_d, objective, stop flag   (reading G9)
// All reductions are deterministic (fixed assignment and fixed tree order; no
// floating-point atomics), so two runs give bit-identical iterates.
#include <cstdlib>

#include "kernels_vec.h"

namespace sdp {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide deterministic sum of NV values per thread; result valid in thread 0.
template <int NV, int NT>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sm /* NV*NT/32 */) {
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) sm[j * (NT / 32) + w] = v[j];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = 0.0;
#pragma unroll 1
      for (int i = 0; i < NT / 32; ++i) s += sm[j * (NT / 32) + i];
      v[j] = s;
    }
  }
}

// ---------------------------------------------------------------- scatter
// Primal (E:OptCondMinYPrimal):  r1 = sum_k H_k^T (x_k + lam_k/rho) - c/rho
// Dual   (E:OptCondMinYDual):    r1 = c - sum_k H_k^T (z_k + lam_k/rho)
// Writes rD = r1 / D.  Residual partials: |sum H^T x_k - previous|^2 and
// (primal) |sum H^T lam_k|^2; previous <- sum H^T x_k.
// Coordinates with short segments: one thread each; long segments (listed
// in `longc`): one warp each.
template <int FORM>
__global__ void __launch_bounds__(256) k_scatter(ScatterArgs a) {
  if (a.done && *a.done) return;
  __shared__ double sm[2 * 8];
  double acc[2] = {0.0, 0.0};
  const int nb_short = (a.N + 255) / 256;
  if ((int)blockIdx.x < nb_short) {
    const int tt = blockIdx.x * 256 + threadIdx.x;
    const int t = (tt < a.N && a.list) ? a.list[tt] : tt;  // a subset of the coordinates (pipelined)
    if (tt < a.N) {
      const int b = a.seg_ptr[t], e = a.seg_ptr[t + 1];
      if (e - b <= kLongSeg) {
        double sr = 0.0, sx = 0.0, sl = 0.0;
        for (int i = b; i < e; ++i) {
          const int s = a.seg_idx[i];
          const double xv = a.xk[s], lv = a.lam[s];
          sr += xv + lv / a.rho;
          sx += xv;
          sl += lv;
        }
        const double r1 = (FORM == 0) ? sr - a.c[t] / a.rho : a.c[t] - sr;
        const int j = a.shared_idx ? a.shared_idx[t] : -1;
        if (j >= 0) {  // partial sums of a coordinate shared across ranks
          a.xbuf[3 * j] = r1;
          a.xbuf[3 * j + 1] = sx;
          a.xbuf[3 * j + 2] = sl;
        } else {
          a.rD[t] = r1 * a.Dinv[t];
          const double d = sx - a.sprev[t];
          a.sprev[t] = sx;
          acc[0] = d * d;
          acc[1] = sl * sl;
        }
      }
    }
  } else {
    const int warp = (blockIdx.x - nb_short) * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (warp < a.n_long) {
      const int t = a.longc[warp];
      const int b = a.seg_ptr[t], e = a.seg_ptr[t + 1];
      double sr = 0.0, sx = 0.0, sl = 0.0;
      for (int i = b + lane; i < e; i += 32) {
        const int s = a.seg_idx[i];
        const double xv = a.xk[s], lv = a.lam[s];
        sr += xv + lv / a.rho;
        sx += xv;
        sl += lv;
      }
      sr = warp_sum(sr);
      sx = warp_sum(sx);
      sl = warp_sum(sl);
      if (lane == 0) {
        const double r1 = (FORM == 0) ? sr - a.c[t] / a.rho : a.c[t] - sr;
        const int j = a.shared_idx ? a.shared_idx[t] : -1;
        if (j >= 0) {
          a.xbuf[3 * j] = r1;
          a.xbuf[3 * j + 1] = sx;
          a.xbuf[3 * j + 2] = sl;
        } else {
          a.rD[t] = r1 * a.Dinv[t];
          const double d = sx - a.sprev[t];
          a.sprev[t] = sx;
          acc[0] = d * d;
          acc[1] = sl * sl;
        }
      }
    }
  }
  block_sum<2, 256>(acc, sm);
  if (threadIdx.x == 0) {
    a.part[2 * blockIdx.x + 0] = acc[0];
    a.part[2 * blockIdx.x + 1] = acc[1];
  }
}

// ---------------------------------------------------------------- dense GEMV
// part[chunk][i] = sum_{t in chunk} A[i][t] * v[t]; A row-major m x lda (lda
// even, zero padded), v zero padded to lda.  Grid (m/RB, nchunks), 256 threads,
// every thread streams RB rows with 16-byte evict-first loads.
template <int RB>
__global__ void __launch_bounds__(256) k_gemv_dense(const double* __restrict__ A, int64_t lda, int m,
                                                     const double* __restrict__ v, int chunk,
                                                     double* __restrict__ part, const int* done) {
  if (done && *done) return;
  __shared__ double sm[RB * 8];
  const int row0 = blockIdx.x * RB;
  const int64_t c0 = (int64_t)blockIdx.y * chunk;
  const int64_t c1 = (c0 + chunk < lda) ? c0 + chunk : lda;
  double acc[RB];
  const double2* Ar[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    acc[r] = 0.0;
    const int rr = (row0 + r < m) ? row0 + r : m - 1;
    Ar[r] = reinterpret_cast<const double2*>(A + (int64_t)rr * lda);
  }
  const double2* v2 = reinterpret_cast<const double2*>(v);
#pragma unroll 4
  for (int64_t t = c0 / 2 + threadIdx.x; t < c1 / 2; t += 256) {
    const double2 vv = __ldg(v2 + t);
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const double2 aa = __ldcs(Ar[r] + t);
      acc[r] = fma(aa.x, vv.x, acc[r]);
      acc[r] = fma(aa.y, vv.y, acc[r]);
    }
  }
  block_sum<RB, 256>(acc, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (row0 + r < m) part[(int64_t)blockIdx.y * m + row0 + r] = acc[r];
  }
}

// y = S^-1 u with the cached dense S^-1 = W^T W (W = L^-1, S = L L^T),
// one warp per row, 8 independent 16-byte loads in flight per lane.  With
// `part` the kernel first forms u = sum_c part[c] - r2 (r2 = b primal, -b/rho
// dual) itself in shared memory (every CTA, fixed chunk order), so the GEMV
// partials need no separate reduction launch.
constexpr int SYMV_T = 512;
template <int FORM>
__global__ void __launch_bounds__(SYMV_T) k_symv(const double* __restrict__ Si, int m, const double* __restrict__ part,
                                                  int nchunks, const double* __restrict__ b, double rho,
                                                  const double* __restrict__ u, double* __restrict__ y,
                                                  const int* done) {
  if (done && *done) return;
  extern __shared__ double us[];
  // u = sum of the GEMV partials (chunk order) - r2: four entries per thread per round, all of
  // their partial loads in flight together
  for (int j0 = threadIdx.x; j0 < m; j0 += 4 * SYMV_T) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (part) {
      for (int c0 = 0; c0 < nchunks; c0 += 8) {
        double t[4][8];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int j = j0 + r * SYMV_T;
            t[r][q] = (j < m && c0 + q < nchunks) ? part[(int64_t)(c0 + q) * m + j] : 0.0;
          }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q) v[r] += t[r][q];
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int j = j0 + r * SYMV_T;
      if (j >= m) continue;
      us[j] = part ? ((FORM == 0) ? v[r] - b[j] : v[r] + b[j] / rho) : u[j];
    }
  }
  __syncthreads();
  const int row = blockIdx.x * (SYMV_T / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const double* Sr = Si + (int64_t)row * m;
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if ((m & 1) == 0) {
    const double2* S2 = reinterpret_cast<const double2*>(Sr);
    const int h = m / 2;
    for (int j = lane; j < h; j += 8 * 32) {  // 8 loads in flight per lane (the last batch masked)
      double2 a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = (j + 32 * q < h) ? __ldcs(S2 + j + 32 * q) : make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = 2 * min(j + 32 * q, h - 1);
        s[q] = fma(a[q].x, us[c], s[q]);
        s[q] = fma(a[q].y, us[c + 1], s[q]);
      }
    }
  } else {
    for (int j = lane; j < m; j += 32) s[0] = fma(Sr[j], us[j], s[0]);
  }
  double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  t = warp_sum(t);
  if (lane == 0) y[row] = t;
}

// u_i = sum_chunks part[.][i] - r2_i   (r2 = b primal, -b/rho dual);
// with a diagonal S the KKT solve is elementwise: y_i = u_i / S_ii.
template <int FORM>
__global__ void k_reduce_u(const double* __restrict__ part, int nchunks, int m, const double* __restrict__ b,
                           double rho, double* __restrict__ u, const double* __restrict__ sdiag,
                           double* __restrict__ y, const int* done) {
  if (done && *done) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += part[(int64_t)c * m + i];
  const double ui = !b ? s : (FORM == 0) ? s - b[i] : s - (-b[i] / rho);
  if (sdiag) {
    y[i] = ui / sdiag[i];
  } else {
    u[i] = ui;
  }
}


// ---------------------------------------------------------------- GEMV^T over the A^T copy
// x_t = rD_t - Dinv_t * (A^T y)_t with A^T stored row-major (lda x ldm): each
// warp streams whole rows of A^T (m doubles) with 16-byte evict-first loads
// issued in batches of TR_U per lane, y comes from L1; deterministic warp
// reduction.  8 warps x TR_ROWS rows per CTA; one partial per CTA.
constexpr int TR_ROWS = 2;
constexpr int TR_U = 16;
template <int FORM>
__global__ void __launch_bounds__(256) k_gemvT_rows(const double* __restrict__ AT, int64_t ldm, int m, int N,
                                                     const int32_t* __restrict__ rows,
                                                     const double* __restrict__ y, const double* __restrict__ rD,
                                                     const double* __restrict__ Dinv, const double* __restrict__ c,
                                                     const double* __restrict__ own, double* __restrict__ x,
                                                     double* __restrict__ part, const int* done) {
  if (done && *done) return;
  __shared__ double sm[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = (m + 1) / 2;  // column pairs (ldm even, zero padded)
  const double2* y2 = reinterpret_cast<const double2*>(y);
  double acc[1] = {0.0};
#pragma unroll
  for (int rr = 0; rr < TR_ROWS; ++rr) {
    const int64_t tt = ((int64_t)blockIdx.x * 8 + warp) * TR_ROWS + rr;
    if (tt >= N) break;
    const int64_t t = rows ? rows[tt] : tt;  // a subset of the coordinates (pipelined iteration)
    const double2* row = reinterpret_cast<const double2*>(AT + t * ldm);
    double w0 = 0.0, w1 = 0.0;
    // predicated batches: every load of a batch is issued before any is consumed
    for (int j0 = lane; j0 < np; j0 += 32 * TR_U) {
      double2 buf[TR_U];
#pragma unroll
      for (int u = 0; u < TR_U; ++u)
        buf[u] = (j0 + 32 * u < np) ? __ldcs(row + j0 + 32 * u) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < TR_U; ++u) {
        if (j0 + 32 * u < np) {
          const double2 yy = __ldg(y2 + j0 + 32 * u);
          w0 = fma(buf[u].x, yy.x, w0);
          w1 = fma(buf[u].y, yy.y, w1);
        }
      }
    }
    const double w = warp_sum(w0 + w1);
    if (lane == 0) {
      const double xv = rD[t] - Dinv[t] * w;
      x[t] = xv;
      acc[0] += (FORM == 0) ? c[t] * xv : own[t] * (xv / Dinv[t]) * (xv / Dinv[t]);
    }
  }
  block_sum<1, 256>(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
}

// AT[t][i] = A[i][t] (tiled transpose through shared memory, setup only)
__global__ void k_transpose(const double* __restrict__ A, int64_t lda, int m, double* __restrict__ AT, int64_t ldm,
                            int64_t ncols) {
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const int r0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int r = r0 + k;
    const int64_t cidx = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < m && cidx < ncols) ? A[(int64_t)r * lda + cidx] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t cidx = c0 + k;
    const int r = r0 + threadIdx.x;
    if (cidx < ncols && r < ldm) AT[cidx * ldm + r] = tile[threadIdx.x][k];
  }
}

// ---------------------------------------------------------------- sparse A (CSR / CSC)
template <int FORM>
__global__ void __launch_bounds__(256) k_gemv_csr(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                   const double* __restrict__ val, int m, const double* __restrict__ v,
                                                   const double* __restrict__ b, double rho, double* __restrict__ u,
                                                   const double* __restrict__ sdiag, double* __restrict__ y,
                                                   const int* done) {
  if (done && *done) return;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  double s = 0.0;
  for (int e = rp[row] + lane; e < rp[row + 1]; e += 32) s = fma(val[e], v[ci[e]], s);
  s = warp_sum(s);
  if (lane == 0) {
    const double ui = !b ? s : (FORM == 0) ? s - b[row] : s - (-b[row] / rho);
    if (sdiag)
      y[row] = ui / sdiag[row];
    else
      u[row] = ui;
  }
}

template <int FORM>
__global__ void __launch_bounds__(256) k_gemvT_csc(const int32_t* __restrict__ cp, const int32_t* __restrict__ ri,
                                                    const double* __restrict__ val, int N, const double* __restrict__ y,
                                                    const double* __restrict__ rD, const double* __restrict__ Dinv,
                                                    const double* __restrict__ c, const double* __restrict__ own,
                                                    double* __restrict__ x, double* __restrict__ part,
                                                    const int* done) {
  if (done && *done) return;
  __shared__ double sm[8];
  const int t = blockIdx.x * 256 + threadIdx.x;
  double acc[1] = {0.0};
  if (t < N) {
    double w = 0.0;
    for (int e = cp[t]; e < cp[t + 1]; ++e) w = fma(val[e], y[ri[e]], w);
    const double xv = rD[t] - Dinv[t] * w;
    x[t] = xv;
    acc[0] = (FORM == 0) ? c[t] * xv : own[t] * (xv / Dinv[t]) * (xv / Dinv[t]);
  }
  block_sum<1, 256>(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
}

// ---------------------------------------------------------------- dual update
// v_k = z_k + lam_k/rho + H_k x  (E:vkEqn);  lam_k = -rho H_k x  (G7)
__global__ void __launch_bounds__(256) k_update_dual(int64_t stot, const int32_t* __restrict__ G,
                                                      const double* __restrict__ x, const double* __restrict__ z,
                                                      double* __restrict__ lam, double* __restrict__ v, double rho,
                                                      double* __restrict__ part, const int* done,
                                                      const long long* iter_in, long long* iter_out) {
  // iter_out = iter_in + 1: the iteration index of the next projection, published before the
  // current finalize can run (pipelined dual schedule, api.cu pipe_dual_B)
  if (iter_out && blockIdx.x == 0 && threadIdx.x == 0) *iter_out = *iter_in + 1;
  if (done && *done) return;
  __shared__ double sm[3 * 8];
  const int64_t s = (int64_t)blockIdx.x * 256 + threadIdx.x;
  double acc[3] = {0.0, 0.0, 0.0};
  if (s < stot) {
    const double hx = __ldg(x + G[s]);
    const double zv = z[s];
    const double vv = zv + lam[s] / rho + hx;
    v[s] = vv;
    lam[s] = -rho * hx;
    const double d = zv - vv;
    acc[0] = d * d;
    acc[1] = zv * zv;
    acc[2] = vv * vv;
  }
  block_sum<3, 256>(acc, sm);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = acc[0];
    part[3 * blockIdx.x + 1] = acc[1];
    part[3 * blockIdx.x + 2] = acc[2];
  }
}

// ---------------------------------------------------------------- finalize
// Single CTA: fixed-order reduction of all partials, residuals (reading G9),
// objective (G17), history, stop flag.  PHASE 0: fused (one rank); PHASE 1:
// reduce the local partials into red[0..5] (to be all-reduced across ranks);
// PHASE 2: combine the all-reduced red[] on every rank.
template <int FORM, int PHASE>
__global__ void __launch_bounds__(256) k_finalize(FinalArgs a) {
  if (*a.done) return;
  __shared__ double sm[8 * 8];
  double v[6] = {0, 0, 0, 0, 0, 0};
  double w[1] = {0.0};
  if (PHASE != 2) {
    // partials in rounds of 4 per thread and array, all loads of a round in flight together
    // (the per-thread summation order is fixed, so the result is deterministic)
    auto gather = [&](const double* src, int n, int comps, int v0) {
      for (int i0 = threadIdx.x; i0 < n; i0 += 4 * 256) {
        double t[4][3];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int i = i0 + r * 256;
            t[r][q] = (q < comps && i < n) ? src[(int64_t)comps * i + q] : 0.0;
          }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if (q < comps) v[v0 + q] += t[r][q];
      }
    };
    if (FORM == 0)
      gather(a.proj_part, a.n_proj, 3, 0);
    else
      gather(a.upd_part, a.n_upd, 3, 0);
    gather(a.scat_part, a.n_scat, 2, 3);
    if (a.n_fix) gather(a.fix_part, a.n_fix, 2, 3);
    gather(a.gT_part, a.n_gT, 1, 5);
    block_sum<6, 256>(v, sm);
    __syncthreads();
    if (PHASE == 1) {
      if (threadIdx.x == 0)
        for (int j = 0; j < 6; ++j) a.red[j] = v[j];
      return;
    }
  } else if (a.n_fix2) {
    // packed primal exchange: the shared-coordinate eps_d partials are computed identically on
    // every rank after the all-reduce (k_shared_fixup, all shared coordinates) and added here
    auto gather2 = [&](const double* src, int n) {
      for (int i = threadIdx.x; i < n; i += 256) {
        v[3] += src[2 * (int64_t)i];
        v[4] += src[2 * (int64_t)i + 1];
      }
    };
    gather2(a.fix_part, a.n_fix2);
    block_sum<6, 256>(v, sm);
    __syncthreads();
  }
  if (FORM == 1)
    for (int i = threadIdx.x; i < a.m; i += 256) w[0] += a.b[i] * a.y[i];
  block_sum<1, 256>(w, sm + 48);
  if (threadIdx.x == 0) {
    if (PHASE == 2)
      for (int j = 0; j < 6; ++j) v[j] += a.red[j];
    const double np = sqrt(v[0]);
    const double den_p = fmax(fmax(sqrt(v[1]), sqrt(v[2])), 1.0);
    const double eps_p = np / den_p;
    double eps_d, obj;
    if (FORM == 0) {
      eps_d = a.rho * sqrt(v[3]) / fmax(sqrt(v[4]), 1.0);
      obj = v[5];
    } else {
      // |sum_k H_k^T lam_k| = rho |D x|
      eps_d = a.rho * sqrt(v[3]) / fmax(a.rho * sqrt(v[5]), 1.0);
      obj = w[0];
    }
    const long long it = *a.iter;
    a.res[0] = eps_p;
    a.res[1] = eps_d;
    a.res[2] = obj;
    if (it < a.hist_cap) {
      a.hist[3 * it + 0] = eps_p;
      a.hist[3 * it + 1] = eps_d;
      a.hist[3 * it + 2] = obj;
    }
    *a.iter = it + 1;
    const bool bad = !(isfinite(eps_p) && isfinite(eps_d) && isfinite(obj));
    if (bad) {
      *a.numerical = 1;
      *a.done = 1;
    } else if (fmax(eps_p, eps_d) < *a.tol) {
      *a.done = 1;
    }
  }
}

// ---------------------------------------------------------------- shared-coordinate fixup
// After the all-reduce of the scatter partials of coordinates shared across
// ranks: r1 -> rD, eps_d partials (counted by the owner only), reset buffer.
// With prevall != NULL (packed primal exchange) the eps_d partials cover EVERY shared coordinate,
// from a replicated copy of the previous sums, so that every rank computes the same values and no
// further all-reduce is needed.
__global__ void __launch_bounds__(256) k_shared_fixup(int nshared, const int32_t* __restrict__ shared_local,
                                                       double* __restrict__ xbuf, const double* __restrict__ Dinv,
                                                       const double* __restrict__ own, double* __restrict__ rD,
                                                       double* __restrict__ sprev, double* __restrict__ part,
                                                       const int* done, double* __restrict__ prevall) {
  if (done && *done) return;
  __shared__ double sm[2 * 8];
  const int j = blockIdx.x * 256 + threadIdx.x;
  double acc[2] = {0.0, 0.0};
  if (j < nshared) {
    const int t = shared_local[j];
    const double r1 = xbuf[3 * j], sx = xbuf[3 * j + 1], sl = xbuf[3 * j + 2];
    xbuf[3 * j] = 0.0;
    xbuf[3 * j + 1] = 0.0;
    xbuf[3 * j + 2] = 0.0;
    if (t >= 0) {
      rD[t] = r1 * Dinv[t];
      const double d = sx - sprev[t];
      sprev[t] = sx;
      if (!prevall && own[t] != 0.0) {
        acc[0] = d * d;
        acc[1] = sl * sl;
      }
    }
    if (prevall) {
      const double d = sx - prevall[j];
      prevall[j] = sx;
      acc[0] = d * d;
      acc[1] = sl * sl;
    }
  }
  block_sum<2, 256>(acc, sm);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x + 0] = acc[0];
    part[2 * blockIdx.x + 1] = acc[1];
  }
}

// ---------------------------------------------------------------- setup kernels
// S = A D^-1 A^T for dense A (m x lda): 64 x 64 output tiles (upper tiles only,
// mirrored), 256 threads with 4 x 4 outputs each, K tiles of 16 columns.
__global__ void __launch_bounds__(256) k_syrk_dense(const double* __restrict__ A, int64_t lda, int m,
                                                     const double* __restrict__ Dinv, double* __restrict__ S) {
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bi > bj) return;
  __shared__ double As[16][65];
  __shared__ double Bs[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4] = {};
  const int i0 = bi * 64, j0 = bj * 64;
  for (int64_t k0 = 0; k0 < lda; k0 += 16) {
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      const int r = e >> 4, kk = e & 15;
      const int64_t col = k0 + kk;
      double av = 0.0, bv = 0.0;
      if (col < lda) {
        if (i0 + r < m) av = A[(int64_t)(i0 + r) * lda + col] * Dinv[col];
        if (j0 + r < m) bv = A[(int64_t)(j0 + r) * lda + col];
      }
      As[kk][r] = av;
      Bs[kk][r] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a4[4], b4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a4[q] = As[kk][ty + 16 * q];
        b4[q] = Bs[kk][tx + 16 * q];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(a4[p], b4[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + ty + 16 * p, j = j0 + tx + 16 * q;
      // a diagonal tile computes both (i, j) and (j, i) with D^-1 on different
      // operands (different rounding): only i <= j writes, so S is deterministic
      if (i < m && j < m && (bi != bj || i <= j)) {
        S[(int64_t)i * m + j] = acc[p][q];
        S[(int64_t)j * m + i] = acc[p][q];
      }
    }
}

// S = A D^-1 A^T for dense A (m x lda, row-major) on the FP64 tensor path: 128 x 128 output tiles
// (upper tiles only: one wave of ~T(T+1)/2 CTAs for m = 2000, so A streams from DRAM about once),
// 8 warps of 64 x 32 DMMA (mma.sync m8n8k4 f64) accumulators, K staged in chunks of 16 columns by
// cp.async (double-buffered), D^-1 applied to the A fragments.  A diagonal tile writes only i <= j
// (its mirror has a different rounding), so S is deterministic and exactly symmetric.
constexpr int SY_T = 128, SY_K = 16, SY_LD = SY_K + 4, SY_NT = 256;
constexpr size_t kSyrkSmem = (size_t)(2 * 2 * SY_T * SY_LD + 2 * SY_K) * sizeof(double);

__device__ __forceinline__ void sy_cp16(double* sdst, const double* gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gsrc), "r"(n) : "memory");
}

__global__ void __launch_bounds__(SY_NT, 1) k_syrk_dmma(const double* __restrict__ A, int64_t lda, int m,
                                                         const double* __restrict__ Dinv, double* __restrict__ S) {
  const int nt = (m + SY_T - 1) / SY_T;
  int bi = 0, rem = blockIdx.x;  // upper tile (bi <= bj) of this CTA, row by row
  while (rem >= nt - bi) {
    rem -= nt - bi;
    ++bi;
  }
  const int bj = bi + rem;
  const int i0 = bi * SY_T, j0 = bj * SY_T;
  extern __shared__ double sy[];
  double* As = sy;                          // [buf][r][kk], row stride SY_LD
  double* Bs = As + 2 * SY_T * SY_LD;
  double* Dv = Bs + 2 * SY_T * SY_LD;       // [buf][kk]
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31, r4 = lane >> 2, c4 = lane & 3;
  const int wr = (wid >> 2) * 64, wc = (wid & 3) * 32;  // warp tile origin inside the CTA tile
  auto load = [&](int buf, int64_t k0) {
    for (int e = t; e < SY_T * (SY_K / 2); e += SY_NT) {
      const int r = e / (SY_K / 2), q = (e % (SY_K / 2)) * 2;
      sy_cp16(As + (buf * SY_T + r) * SY_LD + q, A + (int64_t)(i0 + r < m ? i0 + r : 0) * lda + k0 + q, i0 + r < m);
      sy_cp16(Bs + (buf * SY_T + r) * SY_LD + q, A + (int64_t)(j0 + r < m ? j0 + r : 0) * lda + k0 + q, j0 + r < m);
    }
    if (t < SY_K / 2) sy_cp16(Dv + buf * SY_K + 2 * t, Dinv + k0 + 2 * t, true);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int64_t nk = lda / SY_K;  // lda is a multiple of 32
  load(0, 0);
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < nk) {
      load(buf ^ 1, (kt + 1) * SY_K);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* as = As + (buf * SY_T + wr) * SY_LD;
    const double* bs = Bs + (buf * SY_T + wc) * SY_LD;
#pragma unroll
    for (int ks = 0; ks < SY_K / 4; ++ks) {
      const double dk = Dv[buf * SY_K + ks * 4 + c4];
      double af[8], bf[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) af[a] = as[(8 * a + r4) * SY_LD + ks * 4 + c4] * dk;
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = bs[(8 * b + r4) * SY_LD + ks * 4 + c4];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
              : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
              : "d"(af[a]), "d"(bf[b]));
    }
    __syncthreads();  // the next iteration's load overwrites this buffer
  }
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = i0 + wr + 8 * a + r4, j = j0 + wc + 8 * b + 2 * c4 + h;
        if (i < m && j < m && (bi != bj || i <= j)) {
          S[(int64_t)i * m + j] = acc[a][b][h];
          S[(int64_t)j * m + i] = acc[a][b][h];
        }
      }
}

// Zero the columns of A whose mask entry is 0 (non-owned coordinates of a rank).
__global__ void k_mask_cols(double* __restrict__ A, int64_t lda, int m, const double* __restrict__ mask) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= lda || mask[t] != 0.0) return;
  for (int i = 0; i < m; ++i) A[(int64_t)i * lda + t] = 0.0;
}

// Column permutation + svec scaling of the user's dense-on-pattern A.
// (sets *bad when an input value is not finite: the check runs on the device, not over the host array)
__global__ void k_place_dense(const double* __restrict__ raw, int64_t npat, int m, const int64_t* __restrict__ map,
                              const double* __restrict__ scale, double* __restrict__ A, int64_t lda, int* bad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (e >= npat || i >= m) return;
  const double v = raw[(int64_t)i * npat + e];
  if (!isfinite(v)) *bad = 1;
  if (map[e] >= 0) A[(int64_t)i * lda + map[e]] = v * scale[e];
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_scatter(int form, const ScatterArgs& a, cudaStream_t s) {
  const int grid = (a.N + 255) / 256 + (a.n_long + 7) / 8;
  if (grid <= 0) return;
  if (form == 0)
    k_scatter<0><<<grid, 256, 0, s>>>(a);
  else
    k_scatter<1><<<grid, 256, 0, s>>>(a);
}
int scatter_blocks(int N, int n_long) { return (N + 255) / 256 + (n_long + 7) / 8; }

// u partials over column pieces [pieces[2q], pieces[2q+1]) into part[(slot0 + q) * m ...]
template <int RB>
__global__ void __launch_bounds__(256) k_gemv_pieces(const double* __restrict__ A, int64_t lda, int m,
                                                      const double* __restrict__ v,
                                                      const int64_t* __restrict__ pieces, int slot0,
                                                      double* __restrict__ part, const int* done) {
  if (done && *done) return;
  __shared__ double sm[RB * 8];
  const int row0 = blockIdx.x * RB;
  const int64_t c0 = pieces[2 * blockIdx.y], c1 = pieces[2 * blockIdx.y + 1];
  double acc[RB];
  const double* Ar[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    acc[r] = 0.0;
    const int rr = (row0 + r < m) ? row0 + r : m - 1;
    Ar[r] = A + (int64_t)rr * lda;
  }
  // scalar head / tail for odd ends, 16-byte evict-first loads in between
  const int64_t e0 = (c0 + 1) & ~(int64_t)1, e1 = c1 & ~(int64_t)1;
  if (threadIdx.x == 0 && (c0 & 1) && c0 < c1) {
    const double vv = __ldg(v + c0);
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = fma(__ldcs(Ar[r] + c0), vv, acc[r]);
  }
  if (threadIdx.x == 1 && (c1 & 1) && e1 >= c0 && e1 < c1 && !(e1 == c0 && (c0 & 1))) {
    const double vv = __ldg(v + e1);
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = fma(__ldcs(Ar[r] + e1), vv, acc[r]);
  }
  const double2* v2 = reinterpret_cast<const double2*>(v);
#pragma unroll 4
  for (int64_t t = e0 / 2 + threadIdx.x; t < e1 / 2; t += 256) {
    const double2 vv = __ldg(v2 + t);
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const double2 aa = __ldcs(reinterpret_cast<const double2*>(Ar[r]) + t);
      acc[r] = fma(aa.x, vv.x, acc[r]);
      acc[r] = fma(aa.y, vv.y, acc[r]);
    }
  }
  block_sum<RB, 256>(acc, sm);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (row0 + r < m) part[(int64_t)(slot0 + blockIdx.y) * m + row0 + r] = acc[r];
  }
}

// the HBM-streaming kernels of the pipelined iteration (graph nodes that keep the default priority)
bool is_stream_kernel(const void* fn) {
  return fn == (const void*)k_gemv_pieces<4> || fn == (const void*)k_gemvT_rows<0> ||
         fn == (const void*)k_gemvT_rows<1> || fn == (const void*)k_symv<0> || fn == (const void*)k_symv<1>;
}

void launch_gemv_pieces(const double* A, int64_t lda, int m, const double* v, const int64_t* pieces, int npieces,
                        int slot0, double* part, const int* done, cudaStream_t s) {
  if (npieces <= 0) return;
  dim3 grid((m + 3) / 4, npieces);
  k_gemv_pieces<4><<<grid, 256, 0, s>>>(A, lda, m, v, pieces, slot0, part, done);
}

void launch_gemv_dense(const double* A, int64_t lda, int m, const double* v, int chunk, double* part,
                       const int* done, cudaStream_t s) {
  const int nch = (int)((lda + chunk - 1) / chunk);
  dim3 grid((m + 3) / 4, nch);
  k_gemv_dense<4><<<grid, 256, 0, s>>>(A, lda, m, v, chunk, part, done);
}

void launch_symv(int form, const double* Si, int m, const double* part, int nchunks, const double* b, double rho,
                 const double* u, double* y, const int* done, cudaStream_t s) {
  const size_t sm = (size_t)m * sizeof(double);
  const int rows = SYMV_T / 32;
  if (form == 0)
    k_symv<0><<<(m + rows - 1) / rows, SYMV_T, sm, s>>>(Si, m, part, nchunks, b, rho, u, y, done);
  else
    k_symv<1><<<(m + rows - 1) / rows, SYMV_T, sm, s>>>(Si, m, part, nchunks, b, rho, u, y, done);
}

void symv_init_attributes(int m) {
  const int sm = (int)(m * sizeof(double));
  cudaFuncSetAttribute(k_symv<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_symv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
}

void launch_reduce_u(int form, const double* part, int nchunks, int m, const double* b, double rho, double* u,
                     const double* sdiag, double* y, const int* done, cudaStream_t s) {
  if (form == 0)
    k_reduce_u<0><<<(m + 255) / 256, 256, 0, s>>>(part, nchunks, m, b, rho, u, sdiag, y, done);
  else
    k_reduce_u<1><<<(m + 255) / 256, 256, 0, s>>>(part, nchunks, m, b, rho, u, sdiag, y, done);
}



int gemvT_rows_blocks(int64_t N) { return (int)((N + 8 * TR_ROWS - 1) / (8 * TR_ROWS)); }

void launch_gemvT_rows(int form, const double* AT, int64_t ldm, int m, int N, const double* y, const double* rD,
                       const double* Dinv, const double* c, const double* own, double* x, double* part,
                       const int* done, cudaStream_t s, const int32_t* rows) {
  if (N <= 0) return;
  const int grid = gemvT_rows_blocks(N);
  if (form == 0)
    k_gemvT_rows<0><<<grid, 256, 0, s>>>(AT, ldm, m, N, rows, y, rD, Dinv, c, own, x, part, done);
  else
    k_gemvT_rows<1><<<grid, 256, 0, s>>>(AT, ldm, m, N, rows, y, rD, Dinv, c, own, x, part, done);
}

void launch_transpose(const double* A, int64_t lda, int m, double* AT, int64_t ldm, int64_t ncols, cudaStream_t s) {
  dim3 grid((unsigned)((ncols + 31) / 32), (unsigned)((ldm + 31) / 32));
  k_transpose<<<grid, dim3(32, 8), 0, s>>>(A, lda, m, AT, ldm, ncols);
}

void launch_gemv_csr(int form, const int32_t* rp, const int32_t* ci, const double* val, int m, const double* v,
                     const double* b, double rho, double* u, const double* sdiag, double* y, const int* done,
                     cudaStream_t s) {
  if (form == 0)
    k_gemv_csr<0><<<(m + 7) / 8, 256, 0, s>>>(rp, ci, val, m, v, b, rho, u, sdiag, y, done);
  else
    k_gemv_csr<1><<<(m + 7) / 8, 256, 0, s>>>(rp, ci, val, m, v, b, rho, u, sdiag, y, done);
}

int gemvT_csc_blocks(int N) { return (N + 255) / 256; }

void launch_gemvT_csc(int form, const int32_t* cp, const int32_t* ri, const double* val, int N, const double* y,
                      const double* rD, const double* Dinv, const double* c, const double* own, double* x,
                      double* part, const int* done, cudaStream_t s) {
  const int grid = gemvT_csc_blocks(N);
  if (form == 0)
    k_gemvT_csc<0><<<grid, 256, 0, s>>>(cp, ri, val, N, y, rD, Dinv, c, own, x, part, done);
  else
    k_gemvT_csc<1><<<grid, 256, 0, s>>>(cp, ri, val, N, y, rD, Dinv, c, own, x, part, done);
}

int update_blocks(int64_t stot) { return (int)((stot + 255) / 256); }

void launch_update_dual(int64_t stot, const int32_t* G, const double* x, const double* z, double* lam, double* v,
                        double rho, double* part, const int* done, cudaStream_t s, const long long* iter_in,
                        long long* iter_out) {
  if (stot <= 0 && !iter_out) return;
  k_update_dual<<<std::max(1, update_blocks(stot)), 256, 0, s>>>(stot, G, x, z, lam, v, rho, part, done, iter_in,
                                                                 iter_out);
}

void launch_finalize(int form, int phase, const FinalArgs& a, cudaStream_t s) {
  if (form == 0) {
    if (phase == 0) k_finalize<0, 0><<<1, 256, 0, s>>>(a);
    if (phase == 1) k_finalize<0, 1><<<1, 256, 0, s>>>(a);
    if (phase == 2) k_finalize<0, 2><<<1, 256, 0, s>>>(a);
  } else {
    if (phase == 0) k_finalize<1, 0><<<1, 256, 0, s>>>(a);
    if (phase == 1) k_finalize<1, 1><<<1, 256, 0, s>>>(a);
    if (phase == 2) k_finalize<1, 2><<<1, 256, 0, s>>>(a);
  }
}

int fixup_blocks(int nshared) { return (nshared + 255) / 256; }

void launch_shared_fixup(int nshared, const int32_t* shared_local, double* xbuf, const double* Dinv,
                         const double* own, double* rD, double* sprev, double* part, const int* done,
                         cudaStream_t s, double* prevall) {
  if (nshared <= 0) return;
  k_shared_fixup<<<fixup_blocks(nshared), 256, 0, s>>>(nshared, shared_local, xbuf, Dinv, own, rD, sprev, part,
                                                       done, prevall);
}

void launch_syrk_dense(const double* A, int64_t lda, int m, const double* Dinv, double* S, cudaStream_t s) {
  if (lda % 32 == 0 && getenv("SDP_SYRK_SCALAR") == nullptr) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_syrk_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSyrkSmem);
      attr = true;
    }
    const int nt = (m + SY_T - 1) / SY_T;
    k_syrk_dmma<<<nt * (nt + 1) / 2, SY_NT, kSyrkSmem, s>>>(A, lda, m, Dinv, S);
    return;
  }
  const int nt = (m + 63) / 64;
  dim3 grid(nt, nt);
  k_syrk_dense<<<grid, 256, 0, s>>>(A, lda, m, Dinv, S);
}

void launch_mask_cols(double* A, int64_t lda, int m, const double* mask, cudaStream_t s) {
  k_mask_cols<<<(unsigned)((lda + 255) / 256), 256, 0, s>>>(A, lda, m, mask);
}

void launch_place_dense(const double* raw, int64_t npat, int m, const int64_t* map, const double* scale, double* A,
                        int64_t lda, cudaStream_t s, int* bad) {
  dim3 grid((unsigned)((npat + 255) / 256), m);
  k_place_dense<<<grid, 256, 0, s>>>(raw, npat, m, map, scale, A, lda, bad);
}

}  // namespace sdp
