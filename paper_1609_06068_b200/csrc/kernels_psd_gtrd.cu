// Tridiagonal path of the giant tier: P_k(X) = V max(Lambda, 0) V^T
// (E:XkUpdate P:244-253, E:zkUpdate P:403-410) for 65 <= k <= 800, the
// max-cut clique blocks that carry > 90 % of cfg3's projection flops.
//
// Block Jacobi (kernels_psd_giant.cu) executes ~12 k^3 flops per sweep and
// needs several sweeps; this path executes ~4.5 k^3 (Golub & Van Loan 8.3),
// the LAPACK dsytrd -> dstebz -> dstein -> dormtr pipeline re-designed for the GPU:
//   1. k_gtrd_tridiag: blocked Householder reduction A = Q T Q^T (dsytrd / dlatrd,
//      panels of TC_NB columns), full-storage matrix in an L2-resident workspace;
//      orders >= SDP_GTRD_COOP_MIN are reduced by an 8-CTA thread-block cluster
//      (column chunks dealt to the CTAs, A22 v exchanged through DSMEM), smaller
//      ones one CTA each; tail: scaled T, Gershgorin bounds, exact inertia.
//   2. k_gtrd_bisect: every eigenvalue of T by multisection (3 Sturm chains).
//   3. k_gtrd_cluster: side of 0 to compute (fewer eigenvalues, or the side
//      without oversize clusters), clusters (gap <= 1e-3 ||T||), cuts of clusters
//      beyond a vector group at their largest gaps, vector-kernel groups.
//   4. k_gtrd_vec: inverse iteration (dstein): a CTA per group, a thread per
//      eigenvalue, LU factors in global memory, iterates in shared memory, MGS
//      inside cluster pieces, Rayleigh-quotient weights, residual check.
//   5. k_gtrd_wy + k_gtrd_back: V = H_0 ... H_{k-3} Z in compact-WY groups of 16
//      reflectors, S = Y^T Z, U = T S, Z -= Y U as DMMA products.
//   6. k_gtrd_recon + k_gtrd_fin: P_+ = [A] + sum_t w_t v_t v_t^T as DMMA
//      (mma.sync m8n8k4 f64) products over 32x32 tiles with the mode epilogue;
//      per-matrix partial sums in a fixed order.
// A matrix whose vectors fail the residual test, whose clusters cannot be cut
// safely, or with k > 800 is marked status = -1 and redone by the block-Jacobi
// kernel in the same projection call (GiantDev::only).  Eigenvalues are
// clipped at exactly 0.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "internal.h"

namespace sdp {

namespace {

constexpr int GT_KMAX = 800;
constexpr double kInvSqrt2 = 0.70710678118654752440;
constexpr double kSqrt2 = 1.41421356237309504880;
constexpr double kEps = 2.220446049250313e-16;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gmem_src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem_src) : "memory");
}
// 8-byte asynchronous copy, or 8 zero bytes when !valid (src-size 0)
__device__ __forceinline__ void cp_async8z(double* smem_dst, const double* gmem_src, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem_src), "r"(n) : "memory");
}

__device__ __forceinline__ void packed_rc(int e, int& r, int& c) {
  int cc = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while ((cc + 1) * (cc + 2) / 2 <= e) ++cc;
  while (cc * (cc + 1) / 2 > e) --cc;
  c = cc;
  r = e - cc * (cc + 1) / 2;
}

// projection input X_rc (r <= c), packed index e (absolute)
template <int MODE>
__device__ __forceinline__ double input_value(const ProjArgs& a, int64_t e, int r, int c) {
  if constexpr (MODE == PM_BATCH) {
    return a.in[e];
  } else if constexpr (MODE == PM_PRIMAL) {
    const double v = __ldg(a.x + a.G[e]) - a.lam[e] / a.rho;  // H_k x - lambda_k / rho
    return r == c ? v : v * kInvSqrt2;
  } else {
    const double v = a.vk[e] - a.lam[e] / a.rho;              // v_k - lambda_k / rho
    return r == c ? v : v * kInvSqrt2;
  }
}

// two-stage reduction (section 1b): bandwidth of stage A = reflectors per panel
constexpr int SB_NB = 8;
// bulge-chasing reflectors of stage B: per sweep s, ceil((k - 1 - s) / SB_NB) reflectors of
// SB_NB doubles (tau in slot 0, v_1 .. v_{NB-1} after it; v_0 = 1 implicit)
__host__ __device__ inline int64_t q2_doubles(int k) { return (int64_t)k * k / 2 + (int64_t)k * SB_NB + 64; }

// per-matrix workspace (doubles)
struct GView {
  double* p;
  int k, H;
  int ro = 1;  // row offset of the back-transform reflectors: v_j has its unit at row j + ro
               // (1: one-stage dsytrd reflectors; SB_NB: stage-A panel reflectors of the two-stage path)
  __host__ __device__ static int ld_of(int k) { return (k + 3) & ~3; }
  __device__ int ld() const { return ld_of(k); }
  __device__ double* M() const { return p; }                        // full symmetric, row-major; v_j in row j
  __device__ double* d() const { return p + (int64_t)k * ld(); }
  __device__ double* e() const { return d() + k; }
  __device__ double* tau() const { return e() + k; }
  __device__ double* lall() const { return tau() + k; }            // all eigenvalues (bisection)
  __device__ double* lsel() const { return lall() + k; }           // selected eigenvalues (shifts)
  __device__ double* lw() const { return lsel() + H; }             // reconstruction weights
  __device__ double* clst() const { return lw() + H; }             // cluster leaders
  __device__ double* gsr() const { return clst() + H; }            // vector-kernel groups: first index
  // hdr: nsel, side, ||T|| (scaled), pivmin, scale, Gershgorin lo, hi, index of the first selected
  __device__ double* hdr() const { return gsr() + H; }
  __device__ double* Z() const { return hdr() + 8; }               // selected vectors, column j at j * k
  __device__ double* iv() const { return Z() + (int64_t)k * H; }   // 3 x k x H LU factors + pivot words
  __device__ int nref() const { return k - 1 - ro; }                 // reflectors j = 0 .. k - 2 - ro
  __device__ int nwy() const { return (nref() + 15) / 16; }            // WY groups of 16 reflectors
  __device__ double* wyT() const { return iv() + 3 * (int64_t)k * H + ((k + 63) / 64) * (int64_t)H; }
  __device__ double* Q2() const {  // stage-B reflectors (64-byte aligned: written by bulk async copies)
    const uintptr_t raw = reinterpret_cast<uintptr_t>(wyT() + (int64_t)((k - 2 + 15) / 16) * 256 + 4);
    return reinterpret_cast<double*>((raw + 63) & ~uintptr_t(63));
  }
  __device__ double* Wg() const { return Q2() + q2_doubles(k); }     // stage-A W (k x SB_NB)
};
__host__ __device__ inline int64_t gview_doubles(int k) {
  const int64_t H = k;
  return (int64_t)k * GView::ld_of(k) + 4 * k + 4 * H + 8 + 4 * (int64_t)k * H + ((k + 63) / 64) * H +
         (int64_t)((k - 2 + 15) / 16) * 256 + 4 + 8 + q2_doubles(k) + (int64_t)k * SB_NB + 8;
}

// T (d, e raw, in shared memory, e[k-1] = 0) -> the workspace: T scaled by a power of two (max
// entry in [1, 2)), Gershgorin interval, ||T||, pivmin, inertia at 0 (exact Sturm count).  Called
// by every thread of one CTA (nt threads).
__device__ void tri_tail(const GView& W, double* d, double* e, int k, int t, int nt) {
  __syncthreads();
  if (t == 0) {
    double mx = 0.0;
    for (int i = 0; i < k; ++i) mx = fmax(mx, fmax(fabs(d[i]), fabs(e[i])));
    const double sc = mx > 0.0 ? scalbn(1.0, -ilogb(mx)) : 1.0;
    double gl = 0.0, gu = 0.0, tn = 0.0, me2 = 0.0;
    for (int i = 0; i < k; ++i) {
      d[i] *= sc;
      e[i] *= sc;
    }
    for (int i = 0; i < k; ++i) {
      const double rad = (i > 0 ? fabs(e[i - 1]) : 0.0) + fabs(e[i]);
      gl = i ? fmin(gl, d[i] - rad) : d[i] - rad;
      gu = i ? fmax(gu, d[i] + rad) : d[i] + rad;
      tn = fmax(tn, fabs(d[i]) + rad);
      me2 = fmax(me2, e[i] * e[i]);
    }
    const double pivmin = 1e-290 * fmax(1.0, me2);
    double q = d[0];
    if (fabs(q) < pivmin) q = -pivmin;
    int nneg = q < 0.0;
    for (int i = 1; i < k; ++i) {
      q = d[i] - e[i - 1] * e[i - 1] / q;
      if (fabs(q) < pivmin) q = -pivmin;
      nneg += q < 0.0;
    }
    const double w = gu - gl;
    double* h = W.hdr();
    h[0] = 0;  // k_gtrd_cluster decides the side and the count
    h[1] = 0;
    h[2] = tn;
    h[3] = pivmin;
    h[4] = sc;
    h[5] = gl - 2.0 * kEps * fabs(gl) - 2.0 * kEps * w - pivmin;
    h[6] = gu + 2.0 * kEps * fabs(gu) + 2.0 * kEps * w + pivmin;
    h[7] = nneg;
  }
  __syncthreads();
  for (int i = t; i < k; i += nt) {
    W.d()[i] = d[i];
    W.e()[i] = e[i];
  }
}

// ---------------------------------------------------------------- 1. tridiagonalization
// Jobs: a thread-block cluster of TC_CS CTAs either reduces one large matrix together ("coop",
// k >= SDP_GTRD_COOP_MIN) or each of its CTAs reduces one smaller matrix alone ("solo").
// In a coop job, CTA r owns the 32-column chunks r, r + TC_CS, ... of the matrix (full height):
// the symmetric product A22 v and the trailing update touch only owned columns, so the matrix
// streams from L2 into TC_CS SMs at once.  Everything that needs whole vectors (the updated row
// j, its norm, v, V^T v / W^T v, w) is computed redundantly and identically in every CTA from
// the replicated panel V / W; the one exchange per column is A22 v (each owner writes its part
// into every CTA's shared memory, double-buffered by column parity) followed by one cluster
// barrier; one more cluster barrier per panel publishes the trailing update.
namespace cg = cooperative_groups;
constexpr int TC_NT = 512;
constexpr int TC_NB = 6;
constexpr int TC_CS = GTRD_CLUSTER;  // CTAs per tridiagonalization cluster (16: non-portable size)
constexpr int TC_NR = 1 + 2 * TC_NB;  // block-reduced values per column: |x|^2, W^T x, V^T x
constexpr int TC_PS = GT_KMAX > TC_NT ? GT_KMAX : TC_NT;
constexpr size_t kTriSmem =
    (size_t)(2 * TC_NB * GT_KMAX + 3 * GT_KMAX + TC_PS + 32 * TC_NR + TC_NR + 32 + 4) * sizeof(double);

template <int MODE>
__global__ void __launch_bounds__(TC_NT, 1) k_gtrd_tridiag(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int job = blockIdx.x / TC_CS, rank = blockIdx.x % TC_CS;
  const bool coop = gt.job_coop[job] != 0;
  const int g = gt.job_g[job * TC_CS + (coop ? 0 : rank)];
  if (g < 0) return;  // unused solo slot (never inside a coop cluster)
  const int ncta = coop ? TC_CS : 1, r = coop ? rank : 0;
  const int task = gt.task[g];
  const int k = a.ksz[task];
  const int t = threadIdx.x;
  if (k > GT_KMAX) {
    if (r == 0 && t == 0) gt.status[g] = -1;
    return;
  }
  // SDP_GTRD_DEBUG=2: per-phase clock64 totals of CTA 0 of the first job (thread 0)
  const bool trace = gt.debug == 2 && blockIdx.x == 0 && t == 0;
  long long tr_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tr_last = clock64();
#define TR_MARK(ph)                         \
  if (trace) {                              \
    const long long now_ = clock64();       \
    tr_acc[ph] += now_ - tr_last;           \
    tr_last = now_;                         \
  }
  if (r == 0 && t == 0) gt.status[g] = 0;
  cg::cluster_group cl = cg::this_cluster();
  auto csync = [&]() {
    if (coop)
      cl.sync();
    else
      __syncthreads();
  };
  extern __shared__ double smem[];
  double* Vs = smem;                      // [q][i]
  double* Ws = Vs + TC_NB * GT_KMAX;
  double* pbuf = Ws + TC_NB * GT_KMAX;    // [2][GT_KMAX]: tau (A22 v - V y1 - W y2), all columns
  double* xrow = pbuf + 2 * GT_KMAX;      // updated row j
  double* psum = xrow + GT_KMAX;          // TC_PS partial sums
  double* red = psum + TC_PS;             // 32 x TC_NR
  double* yv = red + 32 * TC_NR;          // TC_NR
  double* red1 = yv + TC_NR;              // 32
  const GView W{gt.ws + gt.moff[g], k, gt.hsel[g]};
  const int LD = W.ld();
  double* M = W.M();
  const int64_t off = a.off[task];
  // load (both triangles), split over the job's CTAs
  const int ns = k * (k + 1) / 2;
  for (int e = r * TC_NT + t; e < ns; e += ncta * TC_NT) {
    int rr, c;
    packed_rc(e, rr, c);
    const double v = input_value<MODE>(a, off + e, rr, c);
    M[(int64_t)rr * LD + c] = v;
    M[(int64_t)c * LD + rr] = v;
  }
  for (int e = t; e < 2 * TC_NB * GT_KMAX; e += TC_NT) smem[e] = 0.0;
  csync();
  // column chunks of 16 (one 128-byte line per row) dealt round-robin to the job's CTAs
  constexpr int CW = 16;
  const int nchunk = (k + CW - 1) / CW;
  const int nown = (nchunk > r ? (nchunk - r + ncta - 1) / ncta : 0) * CW;  // owned columns (may pass k)
  auto own_col = [&](int oc) { return ((oc / CW) * ncta + r) * CW + (oc % CW); };
  auto first_oc = [&](int col) {  // first owned-column index of the chunks that reach column col
    const int cj = col / CW;
    return (cj > r ? (cj - r + ncta - 1) / ncta : 0) * CW;
  };
  const int wid = t >> 5, lane = t & 31;
  static_assert(GT_KMAX <= 2 * TC_NT, "row prefetch holds two entries per thread");
  for (int j0 = 0; j0 + 2 < k; j0 += TC_NB) {
    const int nbp = min(TC_NB, k - 2 - j0);
    double pre[2] = {0.0, 0.0};  // raw row j, prefetched during column j - 1 (inside a panel)
    for (int c = 0; c < nbp; ++c) {
      const int j = j0 + c;
      // (a) row j (== column j) from j on, with the panel's previous reflectors applied;
      //     partial sums of |x|^2, W^T x, V^T x over x = A(j+2:k, j)
      double part[TC_NR];
#pragma unroll
      for (int q = 0; q < TC_NR; ++q) part[q] = 0.0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = j + t + u * TC_NT;
        if (i >= k) continue;
        double x = c > 0 ? pre[u] : __ldcg(M + (int64_t)j * LD + i);
        for (int q = 0; q < c; ++q) x -= fma(Vs[q * GT_KMAX + i], Ws[q * GT_KMAX + j], Ws[q * GT_KMAX + i] * Vs[q * GT_KMAX + j]);
        xrow[i] = x;
        if (i >= j + 2) {
          part[0] = fma(x, x, part[0]);
#pragma unroll
          for (int q = 0; q < TC_NB; ++q) {
            part[1 + q] = fma(Ws[q * GT_KMAX + i], x, part[1 + q]);
            part[1 + TC_NB + q] = fma(Vs[q * GT_KMAX + i], x, part[1 + TC_NB + q]);
          }
        }
      }
      {
        // 16-value warp reduction in 15 exchanges (halving butterfly): lane L ends with the sum of
        // value ((L >> 1) & 15) bit-reversed over L's bits 4..1 (see idx below)
        double v16[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v16[q] = q < TC_NR ? part[q] : 0.0;
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1) {
          const int o = 2 * h;  // lane offsets 16, 8, 4, 2
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int q = 0; q < h; ++q) {
            const double send = up ? v16[q] : v16[q + h];
            const double keep = up ? v16[q + h] : v16[q];
            v16[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        const double tot = v16[0] + __shfl_xor_sync(0xffffffffu, v16[0], 1);
        const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
        if ((lane & 1) == 0 && idx < TC_NR) red[wid * TC_NR + idx] = tot;
      }
      __syncthreads();
      TR_MARK(1);
      if (t < TC_NR) {
        double sacc = 0.0;
        for (int w = 0; w < TC_NT / 32; ++w) sacc += red[w * TC_NR + t];
        yv[t] = sacc;
      }
      __syncthreads();
      TR_MARK(2);
      // (b) Householder vector of x (dlarfg); y1 = W^T v, y2 = V^T v
      const double alpha = xrow[j + 1], sig = yv[0];
      double tau = 0.0, beta = alpha, scl = 0.0;
      if (sig > 0.0) {
        const double nrm = sqrt(fma(alpha, alpha, sig));
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scl = 1.0 / (alpha - beta);
      }
      for (int i = j + 1 + t; i < k; i += TC_NT) {
        const double vi = i == j + 1 ? 1.0 : xrow[i] * scl;
        Vs[c * GT_KMAX + i] = vi;
        if (r == 0 && i >= j + 2) M[(int64_t)i * LD + j] = vi;  // v_j kept in column j (back-transform)
      }
      if (r == 0 && t == 0) {
        W.d()[j] = xrow[j];
        W.e()[j] = beta;
        W.tau()[j] = tau;
      }
      if (c + 1 < nbp) {  // rows of the panel are final (the trailing update ran before it)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int i = j + 1 + t + u * TC_NT;
          if (i < k) pre[u] = __ldcg(M + (int64_t)(j + 1) * LD + i);
        }
      }
      double y1[TC_NB], y2[TC_NB];
#pragma unroll
      for (int q = 0; q < TC_NB; ++q) {
        y1[q] = fma(scl, yv[1 + q], Ws[q * GT_KMAX + j + 1]);
        y2[q] = fma(scl, yv[1 + TC_NB + q], Vs[q * GT_KMAX + j + 1]);
      }
      __syncthreads();
      TR_MARK(3);
      if (tau != 0.0) {  // identical in every CTA of the job
        // (c) p = tau (A22 v - V y1 - W y2) on the owned columns, rows split in G groups
        const double* Vc = Vs + c * GT_KMAX;
        const int oc0 = first_oc(j + 1);
        const int nact = nown - oc0;
        const int G = nact > 0 ? max(1, min(8, TC_NT / nact)) : 1;
        for (int it = t; it < nact * G; it += TC_NT) {
          const int oc = oc0 + it % nact, gg = it / nact;
          const int col = own_col(oc);
          double pacc = 0.0;
          if (col > j && col < k) {
            int l = j + 1 + gg;
            const int64_t st = (int64_t)G * LD;
            const double* Ml = M + (int64_t)l * LD + col;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            for (; l < k; l += 24 * G, Ml += 24 * st) {  // 24 rows in flight (the last batch masked)
              double m[24];
#pragma unroll
              for (int u = 0; u < 24; ++u) m[u] = l + u * G < k ? __ldcg(Ml + u * st) : 0.0;
#pragma unroll
              for (int u = 0; u < 24; u += 4) {  // Vc beyond row k is zero (cleared per panel)
                a0 = fma(m[u], Vc[min(l + u * G, GT_KMAX - 1)], a0);
                a1 = fma(m[u + 1], Vc[min(l + (u + 1) * G, GT_KMAX - 1)], a1);
                a2 = fma(m[u + 2], Vc[min(l + (u + 2) * G, GT_KMAX - 1)], a2);
                a3 = fma(m[u + 3], Vc[min(l + (u + 3) * G, GT_KMAX - 1)], a3);
              }
            }
            pacc = (a0 + a1) + (a2 + a3);
          }
          psum[it] = pacc;
        }
        __syncthreads();
        TR_MARK(4);
        double* pb = pbuf + (j & 1) * GT_KMAX;
        for (int oc = oc0 + t; oc < nown; oc += TC_NT) {
          const int col = own_col(oc);
          if (col <= j || col >= k) continue;
          double p = 0.0;
          for (int gg = 0; gg < G; ++gg) p += psum[gg * nact + (oc - oc0)];
#pragma unroll
          for (int q = 0; q < TC_NB; ++q) p -= fma(Vs[q * GT_KMAX + col], y1[q], Ws[q * GT_KMAX + col] * y2[q]);
          p *= tau;
          if (coop) {
            for (int rr = 0; rr < TC_CS; ++rr) cl.map_shared_rank(pb, rr)[col] = p;
          } else {
            pb[col] = p;
          }
        }
        csync();
        TR_MARK(5);
        // K = (tau / 2) p.v ; w = p - K v   (whole vectors, every CTA)
        double kp = 0.0;
        for (int i = j + 1 + t; i < k; i += TC_NT) kp = fma(pb[i], Vc[i], kp);
        kp = warp_sum(kp);
        if (lane == 0) red1[wid] = kp;
        __syncthreads();
        double K = 0.0;
        for (int w = 0; w < TC_NT / 32; ++w) K += red1[w];
        K *= 0.5 * tau;
        for (int i = j + 1 + t; i < k; i += TC_NT) Ws[c * GT_KMAX + i] = pb[i] - K * Vc[i];
      }
      __syncthreads();
      TR_MARK(6);
    }
    // trailing rank-2*nbp update of the owned columns >= J, rows >= J
    const int J = j0 + nbp;
    {
      const int oc0 = first_oc(J);
      const int nact = nown - oc0;
      const int G = nact > 0 ? max(1, TC_NT / nact) : 1;
      for (int it = t; it < nact * G; it += TC_NT) {
        const int oc = oc0 + it % nact, gg = it / nact;
        const int col = own_col(oc);
        if (col < J || col >= k) continue;
        double vr[TC_NB], wr[TC_NB];
#pragma unroll
        for (int q = 0; q < TC_NB; ++q) {
          vr[q] = Vs[q * GT_KMAX + col];
          wr[q] = Ws[q * GT_KMAX + col];
        }
        auto upd = [&](int row) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < TC_NB; ++q) acc = fma(Vs[q * GT_KMAX + row], wr[q], fma(Ws[q * GT_KMAX + row], vr[q], acc));
          return acc;
        };
        int l = J + gg;
        const int64_t st = (int64_t)G * LD;
        double* Ml = M + (int64_t)l * LD + col;
        for (; l < k; l += 8 * G, Ml += 8 * st) {  // 8 rows per round (the last masked): loads, then stores
          double m[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) m[u] = l + u * G < k ? __ldcg(Ml + u * st) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (l + u * G < k) Ml[u * st] = m[u] - upd(l + u * G);
        }
      }
    }
    csync();
    TR_MARK(7);
    for (int e = t; e < 2 * TC_NB * GT_KMAX; e += TC_NT) smem[e] = 0.0;
    __syncthreads();
  }
  if (trace)
    printf("[gtrd tridiag k=%d coop=%d] cycles: reduce %lld | sum %lld | v %lld | A22v %lld | exchange %lld | w %lld | "
           "trailing %lld\n", k, (int)coop, tr_acc[1], tr_acc[2], tr_acc[3], tr_acc[4], tr_acc[5], tr_acc[6], tr_acc[7]);
#undef TR_MARK
  if (r != 0) return;
  // T (d, e) into shared memory; the last 2x2 block from the reduced matrix
  double* d = xrow;
  double* e = pbuf;
  for (int i = t; i < k; i += TC_NT) {
    d[i] = i < k - 2 ? W.d()[i] : __ldcg(M + (int64_t)i * LD + i);
    e[i] = i < k - 2 ? W.e()[i] : (i == k - 2 ? __ldcg(M + (int64_t)i * LD + i + 1) : 0.0);
  }
  tri_tail(W, d, e, k, t, TC_NT);
}

// ---------------------------------------------------------------- 2. eigenvalues and vectors of T
// Work items: per giant ceil(H / 32) warps, thread s of the giant <-> selected eigenvalue s.
__device__ __forceinline__ int find_item(const int32_t* pre, int ng, int item) {
  int lo = 0, hi = ng - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= item) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// 1/q to ~2^-44 relative (approximate reciprocal + one Newton step): a Sturm count with these
// quotients is the exact count of a relative ~1e-13 perturbation of T
__device__ __forceinline__ double rcp_fast(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  return fma(r, fma(-q, r, 1.0), r);
}

// Multisection (3 shifts per pass, 2 bits per pass) for every eigenvalue (the idx-th smallest) of the
// scaled T; Sturm counts of the LDL^T pivots with the LAPACK pivmin guard (dstebz), stopped at
// width <= 1e-11 ||T|| (the vectors then come from inverse iteration, the weights from Rayleigh
// quotients, so the shift only has to separate the eigenvalue from its neighbours' clusters)
__global__ void __launch_bounds__(32) k_gtrd_bisect(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int g = find_item(gt.ev_pre, gt.ng, blockIdx.x);
  if (gt.status[g] < 0) return;
  const int k = a.ksz[gt.task[g]];
  const GView W{gt.ws + gt.moff[g], k, gt.hsel[g]};
  const double* h = W.hdr();
  const int s = (blockIdx.x - gt.ev_pre[g]) * 32 + threadIdx.x;
  extern __shared__ double sm[];
  double* d = sm;
  double* e2 = sm + k;
  for (int i = threadIdx.x; i < k; i += 32) {
    d[i] = W.d()[i];
    const double ei = W.e()[i];
    e2[i] = ei * ei;
  }
  __syncwarp();
  if (s >= k) return;
  const int idx = s;
  const double pivmin = h[3], tol = 1e-11 * fmax(h[2], 1e-300);
  double lo = h[5], hi = h[6];
  for (int it = 0; it < 40 && hi - lo > tol; ++it) {
    const double w = 0.25 * (hi - lo);
    const double s1 = lo + w, s2 = lo + 2.0 * w, s3 = hi - w;
    double q1 = d[0] - s1, q2 = d[0] - s2, q3 = d[0] - s3;
    if (fabs(q1) < pivmin) q1 = -pivmin;
    if (fabs(q2) < pivmin) q2 = -pivmin;
    if (fabs(q3) < pivmin) q3 = -pivmin;
    int c1 = q1 < 0.0, c2 = q2 < 0.0, c3 = q3 < 0.0;
    for (int i = 1; i < k; ++i) {
      const double di = d[i], ei = e2[i - 1];
      q1 = (di - s1) - ei * rcp_fast(q1);
      q2 = (di - s2) - ei * rcp_fast(q2);
      q3 = (di - s3) - ei * rcp_fast(q3);
      if (fabs(q1) < pivmin) q1 = -pivmin;
      if (fabs(q2) < pivmin) q2 = -pivmin;
      if (fabs(q3) < pivmin) q3 = -pivmin;
      c1 += q1 < 0.0;
      c2 += q2 < 0.0;
      c3 += q3 < 0.0;
    }
    // count(x) <= idx  <=>  eigenvalue idx >= x
    if (c3 <= idx) lo = s3;
    else if (c2 <= idx) { lo = s2; hi = s3; }
    else if (c1 <= idx) { lo = s1; hi = s2; }
    else hi = s1;
  }
  W.lall()[s] = 0.5 * (lo + hi);
}

// Side and clusters.  Clusters: runs of eigenvalues with gaps <= 1e-3 ||T|| (dstein's ortol).
// The vector kernel orthogonalises a cluster inside one CTA whose shared memory holds the
// iterates: cap(k) = min(128, (26000 - 2k) / k) vectors.  The side of 0 whose eigenvectors are
// computed is the one with fewer eigenvalues, unless it has a cluster larger than cap(k) and the
// other side has none (ADMM iterates on max-cut cliques develop a dense band of negative
// eigenvalues while the positive side stays well separated).  A cluster larger than cap(k) is
// cut at its largest gaps into pieces of <= cap(k) (vectors of different pieces are then
// orthogonal to eps ||T|| / gap, gap being the largest gap in a window of cap(k) eigenvalues;
// a cut at a gap below 1e-6 ||T|| hands the matrix to the block-Jacobi fallback; the residual
// test below still guards every vector).  Then: distinct shifts inside the pieces
// and the groups of the vector kernel (consecutive pieces packed first-fit into <= cap(k)
// indices, <= 2 ceil(k / cap) + 1 groups).  One thread per giant.
__global__ void __launch_bounds__(32) k_gtrd_cluster(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int g = blockIdx.x;
  if (gt.status[g] < 0) return;
  const int k = a.ksz[gt.task[g]];
  const int cap = gtrd_vec_cap(k);
  const GView W{gt.ws + gt.moff[g], k, gt.hsel[g]};
  // the eigenvalues into shared memory (the scan below is sequential: one lane)
  extern __shared__ double la[];
  for (int i = threadIdx.x; i < k; i += 32) la[i] = W.lall()[i];
  __syncwarp();
  if (threadIdx.x != 0) return;
  double* h = W.hdr();
  const double tn = h[2], ortol = 1e-3 * tn, pertol = 10.0 * kEps * tn;
  const int nneg = (int)h[7];
  auto max_cluster = [&](int b, int e) {
    int m = 0, run = 0;
    for (int t = b; t < e; ++t) {
      if (t == b || la[t] - la[t - 1] > ortol) run = 0;
      m = max(m, ++run);
    }
    return m;
  };
  const bool okn = max_cluster(0, nneg) <= cap, okp = max_cluster(nneg, k) <= cap;
  int side = (k - nneg) <= nneg ? 0 : 1;
  if (side == 0 && !okp && okn) side = 1;
  if (side == 1 && !okn && okp) side = 0;
  const int nsel = side ? nneg : k - nneg, base = side ? 0 : nneg;
  h[0] = nsel;
  h[1] = side;
  double* ls = W.lsel();
  double* cl = W.clst();
  double* gs = W.gsr();
  int grp = 0, gbeg = 0, npiece = 0, pmax = 0, nsplit = 0;
  bool bad_cut = false;
  auto place = [&](int pb, int pe) {  // piece [pb, pe)
    for (int t = pb; t < pe; ++t) {
      cl[t] = (double)pb;
      double& lt = la[base + t];
      if (t > pb && lt - la[base + t - 1] < pertol) lt = la[base + t - 1] + pertol;
      ls[t] = lt;
    }
    if (pe - gbeg > cap) {  // does not fit the open group: close it at pb
      gs[grp++] = gbeg;
      gbeg = pb;
    }
    ++npiece;
    pmax = max(pmax, pe - pb);
  };
  for (int s0 = 0; s0 < nsel;) {
    int e = s0 + 1;
    while (e < nsel && la[base + e] - la[base + e - 1] <= ortol) ++e;
    int b = s0;
    while (e - b > cap) {  // cut at the largest gap among the first cap + 1 eigenvalues
      int best = b + cap;
      double bg = -1.0;
      for (int x = b + 1; x <= b + cap; ++x) {
        const double gap = la[base + x] - la[base + x - 1];
        if (gap > bg) {
          bg = gap;
          best = x;
        }
      }
      // vectors of different pieces are orthogonal only to ~(eps + 1e-11) ||T|| / gap: a cut inside
      // a (near-)degenerate run would leave them unorthogonalised -> block-Jacobi fallback
      if (bg < 1e-6 * tn) bad_cut = true;
      place(b, best);
      ++nsplit;
      b = best;
    }
    place(b, e);
    s0 = e;
  }
  if (nsel > 0) gs[grp++] = gbeg;
  gs[grp] = nsel;  // sentinel
  if (gt.debug == 1)
    printf("gtrd giant %d k %d nneg %d side %d nsel %d cap %d pieces %d max %d cuts %d groups %d\n", g, k, nneg, side,
           nsel, cap, npiece, pmax, nsplit, grp);
  gt.ngrp[g] = grp;
  if (bad_cut) gt.status[g] = -1;
}

// Inverse iteration (LAPACK dstein) for one group of <= cap(k) selected eigenvalues per CTA, one
// thread per eigenvalue: partial-pivoting LU of T - lam I in global memory ([i][s], coalesced,
// loads batched 8 deep), the iterate in shared memory (column per thread), kInvIters solves from a
// deterministic start vector, each followed by normalisation and modified Gram-Schmidt inside
// the cluster piece (its members are consecutive threads of the CTA).  Weight of vector z: its
// Rayleigh quotient z^T T z clipped at 0 on the selected side; a residual ||T z - rq z||_inf
// above 1e-9 ||T|| hands the matrix to the fallback.
constexpr int VB = 8;
constexpr int VT = 128;
// solves per vector: the shift is within 1e-11 ||T|| of the eigenvalue and clusters are
// orthogonalised explicitly, so two solves leave other components below (1e-8)^2 of a
// random start; the residual test below guards the exceptions
constexpr int kInvIters = 2;
__global__ void __launch_bounds__(VT) k_gtrd_vec(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int gi = find_item(gt.vg_pre, gt.ng, blockIdx.x);
  const int g = gt.vg_g[gi];
  const int grp = blockIdx.x - gt.vg_pre[gi];
  if (gt.status[g] < 0 || grp >= gt.ngrp[g]) return;
  const int k = a.ksz[gt.task[g]];
  const int H = gt.hsel[g];
  const int cap = gtrd_vec_cap(k);
  const GView W{gt.ws + gt.moff[g], k, H};
  const double* hd = W.hdr();
  const int side = (int)hd[1];
  const int sb = (int)W.gsr()[grp], se = (int)W.gsr()[grp + 1];
  const int t = threadIdx.x;
  const int s = sb + t;
  const bool act = s < se;
  extern __shared__ double sm[];
  double* d = sm;
  double* e = sm + k;
  double* xs = sm + 2 * k;  // [i][cap]
  for (int i = t; i < k; i += VT) {
    d[i] = W.d()[i];
    e[i] = W.e()[i];
  }
  const int lead = act ? (int)W.clst()[s] : -1;
  __syncthreads();
  const double tn = hd[2], sc = hd[4];
  const double tol = kEps * fmax(tn, 1e-300);
  double* ui = W.iv();
  double* u2 = ui + (int64_t)k * H;
  double* mu = u2 + (int64_t)k * H;
  uint64_t* pw = reinterpret_cast<uint64_t*>(mu + (int64_t)k * H);  // [i / 64][s]
  double* x = xs + t;  // element i at x[i * cap]
  __shared__ double nrm2s[VT];
  if (act) {
    const double lam = W.lsel()[s];
    // partial-pivoting LU of T - lam I (dlagtf); pivots below tol -> +-tol, stored inverted;
    // the second superdiagonal of U is e[i+1] where row i pivoted, else 0
    double r0 = d[0] - lam, r1 = e[0];
    uint64_t word = 0ull;
    for (int i = 0; i + 1 < k; ++i) {
      const double ci = e[i], ai = d[i + 1] - lam, bi = e[i + 1];  // e[k-1] == 0
      double p1, p2, m;
      const bool pv = fabs(ci) > fabs(r0);
      if (pv) {
        p1 = ci;
        p2 = ai;
        m = r0 / ci;
        r0 = r1 - m * ai;
        r1 = -m * bi;
      } else {
        p1 = r0;
        p2 = r1;
        m = r0 != 0.0 ? ci / r0 : 0.0;
        r0 = ai - m * r1;
        r1 = bi;
      }
      if (fabs(p1) < tol) p1 = p1 < 0.0 ? -tol : tol;
      ui[(int64_t)i * H + s] = 1.0 / p1;
      u2[(int64_t)i * H + s] = p2;
      mu[(int64_t)i * H + s] = m;
      word |= (uint64_t)pv << (i & 63);
      if ((i & 63) == 63) {
        pw[(int64_t)(i >> 6) * H + s] = word;
        word = 0ull;
      }
    }
    if (((k - 2) & 63) != 63) pw[(int64_t)((k - 2) >> 6) * H + s] = word;  // the last partial word
    if (fabs(r0) < tol) r0 = r0 < 0.0 ? -tol : tol;
    ui[(int64_t)(k - 1) * H + s] = 1.0 / r0;
    for (int i = 0; i < k; ++i) {  // deterministic start vector in [-1, 1]
      unsigned long long hh = (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ull ^
                              (unsigned long long)(s + 7) * 0xD1B54A32D192ED03ull;
      hh ^= hh >> 31;
      hh *= 0xBF58476D1CE4E5B9ull;
      hh ^= hh >> 29;
      x[i * cap] = (double)(hh >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
  }
  // does any cluster of this group have more than one member?
  const bool multi = __syncthreads_or(act && (s > lead || (s + 1 < se && (int)W.clst()[s + 1] == s)));
  for (int it = 0; it < kInvIters; ++it) {
    if (act) {
      // forward: L^{-1} x (row interchanges as recorded)
      double ry = x[0];
      int i = 0;
      for (; i + VB < k; i += VB) {
        double m[VB];
#pragma unroll
        for (int u = 0; u < VB; ++u) m[u] = mu[(int64_t)(i + u) * H + s];
        const uint64_t wd = pw[(int64_t)(i >> 6) * H + s];  // i .. i+7 share a word (VB | 64)
#pragma unroll
        for (int u = 0; u < VB; ++u) {
          const double yn = x[(i + 1 + u) * cap];
          if ((wd >> ((i + u) & 63)) & 1ull) {
            x[(i + u) * cap] = yn;
            ry = fma(-m[u], yn, ry);
          } else {
            x[(i + u) * cap] = ry;
            ry = fma(-m[u], ry, yn);
          }
        }
      }
      for (; i + 1 < k; ++i) {
        const double yn = x[(i + 1) * cap], m = mu[(int64_t)i * H + s];
        if ((pw[(int64_t)(i >> 6) * H + s] >> (i & 63)) & 1ull) {
          x[i * cap] = yn;
          ry = fma(-m, yn, ry);
        } else {
          x[i * cap] = ry;
          ry = fma(-m, ry, yn);
        }
      }
      // backward: U^{-1}
      double xn = ry * ui[(int64_t)(k - 1) * H + s], xn1 = 0.0;
      x[(k - 1) * cap] = xn;
      double mx = fabs(xn);
      i = k - 2;
      for (; i - (VB - 1) >= 0; i -= VB) {
        double a2[VB], ai[VB];
        uint64_t wd[2];
        wd[0] = pw[(int64_t)(i >> 6) * H + s];
        wd[1] = pw[(int64_t)((i - VB + 1) >> 6) * H + s];
#pragma unroll
        for (int u = 0; u < VB; ++u) {
          a2[u] = u2[(int64_t)(i - u) * H + s];
          ai[u] = ui[(int64_t)(i - u) * H + s];
        }
#pragma unroll
        for (int u = 0; u < VB; ++u) {
          const int r = i - u;
          const uint64_t w = ((r >> 6) == (i >> 6)) ? wd[0] : wd[1];
          const double u3 = ((w >> (r & 63)) & 1ull) ? e[r + 1] : 0.0;
          const double xi = (x[r * cap] - a2[u] * xn - u3 * xn1) * ai[u];
          x[r * cap] = xi;
          mx = fmax(mx, fabs(xi));
          xn1 = xn;
          xn = xi;
        }
      }
      for (; i >= 0; --i) {
        const double u3 = ((pw[(int64_t)(i >> 6) * H + s] >> (i & 63)) & 1ull) ? e[i + 1] : 0.0;
        const double xi = (x[i * cap] - u2[(int64_t)i * H + s] * xn - u3 * xn1) * ui[(int64_t)i * H + s];
        x[i * cap] = xi;
        mx = fmax(mx, fabs(xi));
        xn1 = xn;
        xn = xi;
      }
      // normalise (scaled by 1/max first so that the sum of squares cannot overflow)
      const double inv = mx > 0.0 ? 1.0 / mx : 1.0;
      double n4[4] = {0.0, 0.0, 0.0, 0.0};
      for (i = 0; i + 3 < k; i += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double v = x[(i + u) * cap] * inv;
          n4[u] = fma(v, v, n4[u]);
        }
      }
      for (; i < k; ++i) {
        const double v = x[i * cap] * inv;
        n4[0] = fma(v, v, n4[0]);
      }
      const double nrm = (n4[0] + n4[1]) + (n4[2] + n4[3]);
      const double in2 = nrm > 0.0 ? inv / sqrt(nrm) : 0.0;
      for (i = 0; i < k; ++i) x[i * cap] *= in2;
    }
    if (multi) {
      // modified Gram-Schmidt inside each cluster piece, all pieces of the group in step: at step
      // pr the member of rank pr (= s - lead) is the pivot of its piece and every member of higher
      // rank removes its component, x_q -= (x_p.x_q / |x_p|^2) x_p (pivots are left unnormalised;
      // |x|^2 is kept up to date by the fused update pass), then one final normalisation
      nrm2s[t] = 1.0;
      const int rank = act ? s - lead : 0;
      for (int pr = 0; __syncthreads_or(act && rank > pr); ++pr) {
        if (act && rank > pr) {
          const int pt = lead + pr - sb;  // pivot's thread = its column in xs
          const double* xp = xs + pt;
          const double np = nrm2s[pt];
          double d4[4] = {0.0, 0.0, 0.0, 0.0}, n4[4] = {0.0, 0.0, 0.0, 0.0};  // 4 chains (ILP)
          int i = 0;
          for (; i + 3 < k; i += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) d4[u] = fma(xp[(i + u) * cap], x[(i + u) * cap], d4[u]);
          }
          for (; i < k; ++i) d4[0] = fma(xp[i * cap], x[i * cap], d4[0]);
          const double coef = np > 0.0 ? ((d4[0] + d4[1]) + (d4[2] + d4[3])) / np : 0.0;
          for (i = 0; i + 3 < k; i += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double v = fma(-coef, xp[(i + u) * cap], x[(i + u) * cap]);
              x[(i + u) * cap] = v;
              n4[u] = fma(v, v, n4[u]);
            }
          }
          for (; i < k; ++i) {
            const double v = fma(-coef, xp[i * cap], x[i * cap]);
            x[i * cap] = v;
            n4[0] = fma(v, v, n4[0]);
          }
          nrm2s[t] = (n4[0] + n4[1]) + (n4[2] + n4[3]);
        }
      }
      if (act && rank > 0) {
        const double nq = nrm2s[t];
        const double in2 = nq > 0.0 ? 1.0 / sqrt(nq) : 0.0;
        for (int i = 0; i < k; ++i) x[i * cap] *= in2;
      }
      __syncthreads();  // rank-0 pivots are read by nobody after this; next solve reads only own x
    }
  }
  if (!act) return;
  // Rayleigh quotient, residual, output column
  double rq = 0.0;
  for (int i = 0; i < k; ++i) {
    double tz = d[i] * x[i * cap];
    if (i > 0) tz = fma(e[i - 1], x[(i - 1) * cap], tz);
    if (i + 1 < k) tz = fma(e[i], x[(i + 1) * cap], tz);
    rq = fma(x[i * cap], tz, rq);
  }
  double res = 0.0;
  double* Z = W.Z();
  for (int i = 0; i < k; ++i) {
    const double xi = x[i * cap];
    double tz = (d[i] - rq) * xi;
    if (i > 0) tz = fma(e[i - 1], x[(i - 1) * cap], tz);
    if (i + 1 < k) tz = fma(e[i], x[(i + 1) * cap], tz);
    res = fmax(res, fabs(tz));
    Z[(int64_t)s * k + i] = xi;
  }
  if (!(res <= 1e-9 * fmax(tn, 1e-300)) || gt.force_fallback) {  // includes NaN
    gt.status[g] = -1;
    if (gt.debug == 1)
      printf("gtrd giant %d k %d: vector %d (lam %.3e rq %.3e) residual %.2e ||T|| %.2e -> fallback\n", g, k, s,
             W.lsel()[s], rq, res, tn);
  }
  const double lw = side == 0 ? fmax(rq, 0.0) : fmax(-rq, 0.0);
  W.lw()[s] = lw / sc;
}

// ---------------------------------------------------------------- 1b. two-stage reduction
// For orders >= SDP_GTRD_SBR_MIN the one-column-at-a-time reduction above (one A22 v product
// and one cluster exchange per column: a latency chain of k steps) is replaced by successive
// band reduction (Bischof, Lang & Sun):
//  Stage A, k_sbr_band: dense -> band of bandwidth SB_NB.  Panel p (columns j0 = p NB .. J - 1,
//   J = j0 + NB): QR of the block below the band, A[J:k, j0:J] = (I - V T V^T) R, then the
//   trailing matrix A22 = A[J:k, J:k] <- Q^T A22 Q = A22 - V W^T - W V^T with X = A22 V T and
//   W = X - 1/2 V (T^T V^T X) (the rank-2nb form of dsytrd).  The m x 8 panel QR is computed
//   redundantly and identically in every CTA of the job from shared memory; X (rows = the CTA's
//   owned columns, A22 symmetric) and the trailing update of the owned columns are DMMA
//   (mma.sync m8n8k4 f64) products streamed from L2; per panel three cluster exchanges (the
//   V^T X partials through DSMEM, the W rows through L2, the updated matrix).  The panel
//   reflectors stay below the band (v_j with its unit at row j + NB) for the back-transform.
//  Stage B, k_sbr_chase: the band (plus room for the bulge: 2 NB subdiagonals) in one CTA's
//   shared memory is reduced to tridiagonal by bulge chasing (Schwarz; Lang): sweep s
//   annihilates column s below the subdiagonal with a reflector on rows s+1 .. s+NB and chases
//   the bulge this creates down the band, one NB-row block per step.  One warp per sweep; step i
//   of sweep s touches rows [s+1+i NB, s+(i+2) NB] and columns [s+1+(i-1) NB, s+(i+1) NB], so
//   it waits until sweep s-1 has finished its step i+2 (the last one whose elements overlap).
//  Back-transform V = Q1 Q2 Z: k_sbr_q2 applies the stage-B reflectors to Z (sweeps in reverse
//   order; the reflectors of one sweep touch disjoint rows and commute), then k_gtrd_wy /
//   k_gtrd_back apply the stage-A reflectors exactly like dsytrd's (row offset ro = NB).
constexpr int SA_NT = 512;
constexpr int SA_NW = SA_NT / 32;
constexpr int SA_CS = 8;
constexpr int SA_PAD = ((GT_KMAX + 7) / 8) * 8;
constexpr int SA_LC = 64;    // rows per partial-X task
constexpr int SA_MAXT = 64;  // partial X tiles held in shared memory at once
constexpr int SA_PLD = SB_NB + 1;  // row stride of the panel / V and of V T, W: conflict-free row-per-thread access
static_assert(SB_NB == 8, "the DMMA tiles and the chase lanes assume NB = 8");
constexpr size_t kSbrASmem =
    (size_t)(2 * SA_PAD * SA_PLD + SA_PAD * SB_NB + SA_MAXT * 64 + 2 * (SA_NW * 32 + 32) + 2 * 64 + SA_CS * 64 + 64) *
    sizeof(double);

// acquire-release fence at CTA scope (MEMBAR.ALL.CTA): orders this thread's shared-memory accesses
// around a progress flag without the sequentially consistent fence of __threadfence_block()
__device__ __forceinline__ void fence_cta() { asm volatile("fence.acq_rel.cta;\n" ::: "memory"); }

__device__ __forceinline__ void sb_mma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// CTA sum of one value per thread (every thread gets the total, fixed order); red: SA_NW
// doubles, used ping-pong by the caller so that one barrier per reduction suffices
__device__ __forceinline__ double sa_sum1(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < SA_NW; ++w) s += red[w];
  return s;
}

// CTA sums of NV = 8 or 32 values per thread (halving butterfly in the warp, then fixed-order sums
// of the warps' partials by the first NV threads); red: SA_NW * NV + NV doubles, used ping-pong by
// the caller (two barriers per reduction)
template <int NV>
__device__ __forceinline__ void sa_sumv(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int hh = NV / 2; hh >= 1; hh >>= 1) {
    const int o = (32 / NV) * hh;  // lane offsets: NV = 8: 16, 8, 4; NV = 32: 16, 8, 4, 2, 1
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int q = 0; q < hh; ++q) {
      const double send = up ? v[q] : v[q + hh];
      const double keep = up ? v[q + hh] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  double tot = v[0];
#pragma unroll
  for (int o = 32 / NV / 2; o >= 1; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  // lane L holds value idx = bit-reversal of L's bits (4 .. 5 - log2 NV)
  int idx = 0;
#pragma unroll
  for (int b = 0; (1 << b) < NV; ++b) idx = idx * 2 + ((lane >> (4 - b)) & 1);
  if ((lane & (32 / NV - 1)) == 0) red[(threadIdx.x >> 5) * NV + idx] = tot;
  __syncthreads();
  double* fin = red + SA_NW * NV;
  if (threadIdx.x < NV) {
    double sacc = 0.0;
#pragma unroll
    for (int w = 0; w < SA_NW; ++w) sacc += red[w * NV + threadIdx.x];
    fin[threadIdx.x] = sacc;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NV; ++c) v[c] = fin[c];
}

template <int MODE>
__global__ void __launch_bounds__(SA_NT, 1) k_sbr_band(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int job = blockIdx.x / SA_CS, rank = blockIdx.x % SA_CS;
  const bool coop = gt.job2_coop[job] != 0;
  const int g = gt.job2_g[job * SA_CS + (coop ? 0 : rank)];
  if (g < 0) return;
  const int ncta = coop ? SA_CS : 1, r = coop ? rank : 0;
  const int task = gt.task[g];
  const int k = a.ksz[task];
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31, r4 = lane >> 2, c4 = lane & 3;
  if (k > GT_KMAX) {
    if (r == 0 && t == 0) gt.status[g] = -1;
    return;
  }
  if (r == 0 && t == 0) gt.status[g] = 0;
  cg::cluster_group cl = cg::this_cluster();
  auto csync = [&]() {
    if (coop)
      cl.sync();
    else
      __syncthreads();
  };
  extern __shared__ double smem[];
  double* Pv = smem;                    // panel -> V, [l][q] (row stride SA_PLD), SA_PAD rows
  double* VT = Pv + SA_PAD * SA_PLD;    // V T, then W of all rows (row stride SA_PLD)
  double* Xo = VT + SA_PAD * SA_PLD;    // X -> W of the owned rows, [tile][r][q]
  double* Xp = Xo + SA_PAD * SB_NB;     // partial X tiles
  double* red = Xp + SA_MAXT * 64;      // 2 x (SA_NW x 32 + 32) (ping-pong)
  double* Mp = red + 2 * (SA_NW * 32 + 32);  // M' = T^T V^T X (8 x 8)
  double* Tm = Mp + 64;                 // T (8 x 8, upper)
  double* xch = Tm + 64;                // SA_CS x 64 partials of V^T X (DSMEM)
  GView W{gt.ws + gt.moff[g], k, gt.hsel[g]};
  const int LD = W.ld();
  double* M = W.M();
  double* Wg = W.Wg();
  const int64_t off = a.off[task];
  const int ns = k * (k + 1) / 2;
  for (int e = r * SA_NT + t; e < ns; e += ncta * SA_NT) {
    int rr, c;
    packed_rc(e, rr, c);
    const double v = input_value<MODE>(a, off + e, rr, c);
    M[(int64_t)rr * LD + c] = v;
    M[(int64_t)c * LD + rr] = v;
  }
  int rp = 0;  // ping-pong index of red
  auto R1 = [&]() { double* p = red + rp * (SA_NW * 32 + 32); rp ^= 1; return p; };
  const int nchunk = (k + SB_NB - 1) / SB_NB;
  csync();
  // SDP_GTRD_DEBUG=3: per-phase clock64 totals of thread 0 of CTA 0 of the first job
  const bool trace = gt.debug == 3 && blockIdx.x == 0 && t == 0;
  long long tr_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tr_last = clock64();
#define SA_MARK(ph)                         \
  if (trace) {                              \
    const long long now_ = clock64();       \
    tr_acc[ph] += now_ - tr_last;           \
    tr_last = now_;                         \
  }
  for (int p = 0;; ++p) {
    const int j0 = p * SB_NB, J = j0 + SB_NB, m = k - J;
    if (m < 2) break;
    const int nq = min(SB_NB, m - 1);
    // (1) panel A[J:k, j0:J] -> shared memory (rows >= m zero)
    for (int e = t; e < SA_PAD * SB_NB; e += SA_NT) {
      const int l = e >> 3, q = e & 7;
      Pv[l * SA_PLD + q] = l < m ? __ldcg(M + (int64_t)(J + l) * LD + j0 + q) : 0.0;
    }
    __syncthreads();
    // (2) Householder QR of the panel (dgeqr2), identical in every CTA
    double taus[SB_NB], betas[SB_NB];
#pragma unroll
    for (int q = 0; q < SB_NB; ++q) {
      taus[q] = 0.0;
      betas[q] = q < m ? Pv[q * SA_PLD + q] : 0.0;  // no reflector: the diagonal entry is R's
      if (q >= nq) continue;
      const double alpha = Pv[q * SA_PLD + q];
      double part = 0.0;
      for (int l = q + 1 + t; l < m; l += SA_NT) part = fma(Pv[l * SA_PLD + q], Pv[l * SA_PLD + q], part);
      const double sig = sa_sum1(part, R1());
      double tau = 0.0, beta = alpha, scl = 0.0;
      if (sig > 0.0) {
        const double nrm = sqrt(fma(alpha, alpha, sig));
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scl = 1.0 / (alpha - beta);
      }
      double wp[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) wp[c] = 0.0;
      for (int l = q + t; l < m; l += SA_NT) {
        double vl = 1.0;
        if (l > q) {
          vl = Pv[l * SA_PLD + q] * scl;
          Pv[l * SA_PLD + q] = vl;
        }
#pragma unroll
        for (int c = q + 1; c < 8; ++c) wp[c] = fma(vl, Pv[l * SA_PLD + c], wp[c]);
      }
      sa_sumv<8>(wp, R1());
      if (tau != 0.0)
        for (int l = q + t; l < m; l += SA_NT) {
          const double vl = l > q ? Pv[l * SA_PLD + q] : 1.0;
#pragma unroll
          for (int c = q + 1; c < 8; ++c) Pv[l * SA_PLD + c] -= tau * vl * wp[c];
        }
      __syncthreads();
      taus[q] = tau;
      betas[q] = beta;
    }
    SA_MARK(0);
    // (3) R and the reflectors back into the matrix (rank 0), tau
    if (r == 0) {
      for (int e = t; e < m * SB_NB; e += SA_NT) {
        const int l = e >> 3, q = e & 7;
        double v = Pv[l * SA_PLD + q];
#pragma unroll
        for (int qq = 0; qq < SB_NB; ++qq)
          if (qq == q && l == q) v = betas[qq];
        M[(int64_t)(J + l) * LD + j0 + q] = v;
      }
      if (t < SB_NB) {
        double tv = 0.0;
#pragma unroll
        for (int qq = 0; qq < SB_NB; ++qq)
          if (qq == t) tv = taus[qq];
        W.tau()[j0 + t] = tv;
      }
    }
    __syncthreads();
    // Pv -> V with an explicit unit diagonal and zeros above it
    if (t < 64) {
      const int l = t >> 3, q = t & 7;
      if (l < q) Pv[l * SA_PLD + q] = 0.0;
      if (l == q) Pv[l * SA_PLD + q] = 1.0;
    }
    __syncthreads();
    SA_MARK(1);
    // (4) T (dlarft forward, columnwise): T[q][q] = tau_q, T[0:q, q] = -tau_q T[0:q, 0:q] G[0:q, q],
    //     G = V^T V (one 32-value reduction: the 28 pairs a < b), T by warp 0 into shared memory
    {
      double gp[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) gp[u] = 0.0;
      for (int l = t; l < m; l += SA_NT) {
        double vr[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) vr[q] = Pv[l * SA_PLD + q];
        int u = 0;
#pragma unroll
        for (int x = 0; x < 8; ++x)
#pragma unroll
          for (int y = x + 1; y < 8; ++y) {
            gp[u] = fma(vr[x], vr[y], gp[u]);
            ++u;
          }
      }
      sa_sumv<32>(gp, R1());
      if (wid == 0) {
        // column c of T by lanes rr < c: T[rr][c] = -tau_c sum_{q = rr}^{c-1} T[rr][q] G[q][c]
        double trow[8];  // row `lane` of T (lanes 0..7)
#pragma unroll
        for (int c = 0; c < 8; ++c) trow[c] = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          double acc = 0.0;
          int u = 0;
#pragma unroll
          for (int x = 0; x < 8; ++x)
#pragma unroll
            for (int y = x + 1; y < 8; ++y) {
              if (y == c && x >= lane) acc = fma(trow[x], gp[u], acc);  // G[x][c], x in [lane, c)
              ++u;
            }
          double tc = 0.0;
#pragma unroll
          for (int qq = 0; qq < 8; ++qq)
            if (qq == c) tc = taus[qq];
          trow[c] = lane < c ? -tc * acc : (lane == c ? tc : 0.0);
        }
        if (lane < 8) {
#pragma unroll
          for (int c = 0; c < 8; ++c) Tm[lane * 8 + c] = trow[c];
        }
      }
      __syncthreads();
    }
    // (5) VT = V T for every row (rows >= m: 0)
    for (int l = t; l < SA_PAD; l += SA_NT) {
      double vr[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) vr[q] = Pv[l * SA_PLD + q];  // rows >= m are zero
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q <= c; ++q) acc = fma(vr[q], Tm[q * 8 + c], acc);
        VT[l * SA_PLD + c] = acc;
      }
    }
    __syncthreads();
    // owned column tiles (chunks of 8 columns, round-robin over the job's CTAs) at or after J
    const int ch0 = p + 1;                                        // first chunk of A22
    const int first = ch0 <= r ? r : r + ((ch0 - r + ncta - 1) / ncta) * ncta;
    const int nit = first < nchunk ? (nchunk - 1 - first) / ncta + 1 : 0;
    SA_MARK(2);
    // (6) X rows of the owned columns: X[i][:] = sum_l A22[l][i] VT[l][:] (DMMA, l split in
    //     chunks of SA_LC rows; partial tiles reduced in a fixed order)
    const int nlc = (m + SA_LC - 1) / SA_LC;
    for (int e = t; e < nit * 64; e += SA_NT) Xo[e] = 0.0;
    for (int tb = 0; tb < nit * nlc; tb += SA_MAXT) {
      const int nt = min(SA_MAXT, nit * nlc - tb);
      for (int u0 = wid; u0 < nt; u0 += 2 * SA_NW) {  // two tasks per warp: 32 loads in flight
        double av[2][SA_LC / 4];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int u = u0 + b * SA_NW;
          const int it = (tb + u) / nlc, lc = (tb + u) % nlc;
          const int icol = (first + it * ncta) * SB_NB + r4;
          const bool ok = u < nt && icol < k;
#pragma unroll
          for (int s4 = 0; s4 < SA_LC / 4; ++s4) {
            const int l = lc * SA_LC + s4 * 4 + c4;  // row of A22 (local)
            av[b][s4] = (ok && l < m) ? __ldcg(M + (int64_t)(J + l) * LD + icol) : 0.0;
          }
        }
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int u = u0 + b * SA_NW;
          if (u >= nt) break;
          const int lc = (tb + u) % nlc;
          double acc[2] = {0.0, 0.0};
#pragma unroll
          for (int s4 = 0; s4 < SA_LC / 4; ++s4) {
            const int l = lc * SA_LC + s4 * 4 + c4;
            sb_mma(acc, av[b][s4], l < SA_PAD ? VT[l * SA_PLD + r4] : 0.0);
          }
          Xp[u * 64 + r4 * 8 + 2 * c4] = acc[0];
          Xp[u * 64 + r4 * 8 + 2 * c4 + 1] = acc[1];
        }
      }
      __syncthreads();
      for (int e = t; e < nit * 64; e += SA_NT) {  // fixed order: batches, then chunks
        const int it = e >> 6;
        double sacc = Xo[e];
        for (int lc = 0; lc < nlc; ++lc) {
          const int u = it * nlc + lc - tb;
          if (u >= 0 && u < nt) sacc += Xp[u * 64 + (e & 63)];
        }
        Xo[e] = sacc;
      }
      __syncthreads();
    }
    SA_MARK(3);
    // (7) V^T X over the owned rows -> every CTA (DSMEM), summed in rank order; M' = T^T (V^T X)
    if (t < 64) {
      const int q = t >> 3, q2 = t & 7;
      double sacc = 0.0;
      for (int it = 0; it < nit; ++it) {
        const int i0 = (first + it * ncta) * SB_NB;
        for (int rr = 0; rr < 8; ++rr) {
          const int l = i0 + rr - J;
          if (i0 + rr < k) sacc = fma(Pv[l * SA_PLD + q], Xo[it * 64 + rr * 8 + q2], sacc);
        }
      }
      if (coop) {
        for (int rr = 0; rr < SA_CS; ++rr) cl.map_shared_rank(xch, rr)[r * 64 + t] = sacc;
      } else {
        xch[t] = sacc;
      }
    }
    csync();
    if (t < 64) {
      double m0[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double sacc = 0.0;
        for (int rr = 0; rr < ncta; ++rr) sacc += xch[rr * 64 + q * 8 + (t & 7)];
        m0[q] = sacc;
      }
      const int q = t >> 3;
      double mp = 0.0;
#pragma unroll
      for (int qq = 0; qq < 8; ++qq)
        if (qq <= q) mp = fma(Tm[qq * 8 + q], m0[qq], mp);  // (T^T)[q][qq] = T[qq][q]
      Mp[t] = mp;
    }
    __syncthreads();
    SA_MARK(4);
    // (8) W = X - 1/2 V M' for the owned rows -> Xo and the global W rows
    for (int e = t; e < nit * 64; e += SA_NT) {
      const int it = e >> 6, rr = (e >> 3) & 7, q = e & 7;
      const int i = (first + it * ncta) * SB_NB + rr;
      if (i >= k) {
        Xo[e] = 0.0;
        continue;
      }
      const int l = i - J;
      double vm = 0.0;
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) vm = fma(Pv[l * SA_PLD + qq], Mp[qq * 8 + q], vm);
      const double w = Xo[e] - 0.5 * vm;
      Xo[e] = w;
      Wg[(int64_t)l * SB_NB + q] = w;
    }
    csync();
    for (int e = t; e < SA_PAD * SB_NB; e += SA_NT) VT[(e >> 3) * SA_PLD + (e & 7)] = (e >> 3) < m ? __ldcg(Wg + e) : 0.0;
    __syncthreads();
    SA_MARK(5);
    // (9) A22[:, owned] -= V W^T + W V^T  (DMMA: [V | W](l, 16) x [W | V](i, 16)^T); every warp
    //     loads the C tiles of 8 of its tasks at once (L2 latency), then multiplies and stores
    const int nlt = (m + 7) / 8;
    const int ntask = nlt * nit;
    for (int u0 = wid; u0 < ntask; u0 += 16 * SA_NW) {
      double2 cur[16];
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const int u = u0 + b * SA_NW;
        cur[b] = make_double2(0.0, 0.0);
        if (u < ntask) {
          const int lt = u / nit, it = u % nit;
          const int row = J + lt * 8 + r4, col = (first + it * ncta) * SB_NB + 2 * c4;
          if (row < k && col < k) cur[b] = __ldcg(reinterpret_cast<const double2*>(M + (int64_t)row * LD + col));
        }
      }
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const int u = u0 + b * SA_NW;
        if (u >= ntask) break;
        const int lt = u / nit, it = u % nit;
        const int i0 = (first + it * ncta) * SB_NB;
        const int l0 = lt * 8;
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int q = (ks & 1) * 4 + c4;
          const double av = ks < 2 ? Pv[(l0 + r4) * SA_PLD + q] : VT[(l0 + r4) * SA_PLD + q];
          const double bv = ks < 2 ? Xo[it * 64 + r4 * 8 + q] : Pv[(i0 + r4 - J) * SA_PLD + q];
          sb_mma(acc, av, bv);
        }
        const int row = J + l0 + r4, col = i0 + 2 * c4;
        if (row < k && col < k) {
          double* pm = M + (int64_t)row * LD + col;
          pm[0] = cur[b].x - acc[0];
          if (col + 1 < k) pm[1] = cur[b].y - acc[1];
        }
      }
    }
    csync();
    SA_MARK(6);
  }
  if (trace)
    printf("[sbr band k=%d coop=%d] cycles: qr %lld | T,VT %lld | X %lld | VtX+exch %lld | W+exch %lld | update+sync %lld\n",
           k, (int)coop, tr_acc[0], tr_acc[1], tr_acc[2], tr_acc[3], tr_acc[4], tr_acc[6]);
#undef SA_MARK
  // the band stays in M (lower part, distance <= NB); stage B reads it
}

// Stage B.  AB[c * SB_LDB + d] = A[c + d][c], d = 0 .. SB_LDB - 1 (room for the bulge: d <= 2 NB - 1).
// Each warp chases SB_G consecutive sweeps in lockstep, one 8-lane group per sweep, group g lagging
// SB_LAG steps behind group g - 1 (step i of sweep s needs step i + 2 of sweep s - 1 finished, so a
// fixed lag of 4 satisfies every dependency inside the warp without waiting); group 0 waits for the
// previous warp's group SB_G - 1 through a per-block progress counter in shared memory.  The code of
// a step is branch-free across the lanes (inactive groups compute on a valid dummy block and store
// nothing), so the warp issues one instruction stream for SB_G sweeps.
constexpr int SB_LDB = 2 * SB_NB + 2;  // A[r][c] at c (SB_LDB - 1) + r: columns 17 doubles apart (conflict-free per lane)
constexpr int SB_NW = 8;
constexpr int SB_NT = SB_NW * 32;
constexpr int SB_G = 4;
constexpr int SB_LAG = 4;
constexpr int SB_NBLK = (GT_KMAX + SB_G - 1) / SB_G + 1;
constexpr size_t kSbrBSmem =
    (size_t)(GT_KMAX + 2 * SB_NB + 1) * SB_LDB * sizeof(double) + (size_t)(GT_KMAX + 1 + SB_NBLK) * sizeof(int);

__global__ void __launch_bounds__(SB_NT, 1) k_sbr_chase(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int g = gt.sb_g[blockIdx.x];
  if (gt.status[g] < 0) return;
  const int k = a.ksz[gt.task[g]];
  const GView W{gt.ws + gt.moff[g], k, gt.hsel[g]};
  const int LD = W.ld();
  const double* M = W.M();
  double* Q2 = W.Q2();
  extern __shared__ double smb2[];
  double* AB = smb2;
  int* qoff = reinterpret_cast<int*>(AB + (GT_KMAX + 2 * SB_NB + 1) * SB_LDB);
  int* sprog = qoff + (GT_KMAX + 1);  // per block of SB_G sweeps: super-steps completed
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31;
  for (int e = t; e < (k + 2 * SB_NB + 1) * SB_LDB; e += SB_NT) {
    const int c = e / SB_LDB, d = e % SB_LDB;
    AB[e] = (c < k && d <= SB_NB && c + d < k) ? __ldcg(M + (int64_t)(c + d) * LD + c) : 0.0;
  }
  const int nsw = k - 2;  // sweeps s = 0 .. k - 3 (s = k - 2 has nothing to annihilate)
  auto nsteps = [&](int s) { return (k - 1 - s + SB_NB - 1) / SB_NB; };
  const int nblk = nsw > 0 ? (nsw + SB_G - 1) / SB_G : 0;
  for (int b = t; b < SB_NBLK; b += SB_NT) sprog[b] = 0;
  if (t == 0) {
    int acc = 0;
    for (int s = 0; s < nsw; ++s) {
      qoff[s] = acc;
      acc += nsteps(s);
    }
  }
  __syncthreads();
  volatile int* vsp = sprog;
  auto A = [&](int rr, int c) -> double& { return AB[c * (SB_LDB - 1) + rr]; };  // rr >= c, rr - c <= 2 NB
  const int gq = lane >> 3, l = lane & 7;
  const bool trace = gt.debug == 3 && blockIdx.x == 0 && lane == 0;
  long long t_wait = 0, t_start = clock64(), nsup = 0;
  for (int b = wid; b < nblk; b += SB_NW) {
    const int s = b * SB_G + gq;  // this group's sweep
    const bool sv = s < nsw;
    const int nst = sv ? nsteps(s) : 0;
    int jmax = 0;
#pragma unroll
    for (int gg = 0; gg < SB_G; ++gg)
      if (b * SB_G + gg < nsw) jmax = max(jmax, nsteps(b * SB_G + gg) + SB_LAG * gg);
    const int sp = b * SB_G - 1;  // previous block's last sweep (group 0's dependency)
    const int nsp = sp >= 0 ? nsteps(sp) : 0;
    const int nst0 = nsteps(b * SB_G);
    for (int j = 0; j < jmax; ++j) {
      if (b > 0 && j < nst0) {  // group 0's step j needs sweep sp to have finished step j + 2
        const int need = min(j + 3, nsp) + SB_LAG * (SB_G - 1);
        const long long tw0 = trace ? clock64() : 0;
        while (vsp[b - 1] < need) __nanosleep(32);
        if (trace) t_wait += clock64() - tw0;
        fence_cta();
      }
      const int i = j - SB_LAG * gq;
      const bool act = sv && i >= 0 && i < nst;
      const int sg = act ? s : 0, ig = act ? i : 0;
      const int r0 = sg + 1 + ig * SB_NB;
      const int L = min(SB_NB, k - r0);
      const int cb = ig == 0 ? sg : r0 - SB_NB;  // column whose part in rows r0.. is annihilated
      // (a) reflector of x = A[r0 .. r0 + L - 1][cb]: beta = -sign(alpha) ||x||, v = x / (alpha - beta),
      //     tau = (beta - alpha) / beta, from one reciprocal 1 / (beta (alpha - beta))
      const double xl = l < L ? A(r0 + l, cb) : 0.0;
      const double alpha = __shfl_sync(0xffffffffu, xl, 0, SB_NB);
      double sq = (l >= 1) ? xl * xl : 0.0;
      sq += __shfl_xor_sync(0xffffffffu, sq, 1, SB_NB);
      sq += __shfl_xor_sync(0xffffffffu, sq, 2, SB_NB);
      sq += __shfl_xor_sync(0xffffffffu, sq, 4, SB_NB);
      const double nrm = sqrt(fma(alpha, alpha, sq));
      const double beta = sq > 0.0 ? (alpha >= 0.0 ? -nrm : nrm) : alpha;
      const double dd = alpha - beta;
      const double rr = sq > 0.0 ? 1.0 / (beta * dd) : 0.0;
      const double scl = beta * rr, tau = -dd * dd * rr;
      const double vl = l == 0 ? 1.0 : (l < L ? xl * scl : 0.0);
      if (act) {
        Q2[(int64_t)(qoff[sg] + ig) * SB_NB + l] = l == 0 ? tau : vl;
        if (l < L) A(r0 + l, cb) = l == 0 ? beta : 0.0;
      }
      double v[SB_NB];
#pragma unroll
      for (int r = 0; r < SB_NB; ++r) v[r] = __shfl_sync(0xffffffffu, vl, r, SB_NB);
      // (b) H from the left on the left block (columns cb + 1 .. cb + 7, steps i >= 1): lane = column
      {
        double z[SB_NB], d = 0.0;
#pragma unroll
        for (int r = 0; r < SB_NB; ++r) {
          z[r] = r < L ? A(r0 + r, cb + l) : 0.0;
          d = fma(v[r], z[r], d);
        }
        d *= tau;
        if (act && ig > 0 && l >= 1)
#pragma unroll
          for (int r = 0; r < SB_NB; ++r)
            if (r < L) A(r0 + r, cb + l) = fma(-d, v[r], z[r]);
      }
      // (c) two-sided on D = A[R][R]: lane = column l of D; y = tau D v, w = y - (tau/2)(y.v) v,
      //     D -= v w^T + w v^T (lower part, column l: rows r >= l)
      double dcol[SB_NB], y = 0.0;
#pragma unroll
      for (int r = 0; r < SB_NB; ++r) {
        dcol[r] = (r < L && l < L) ? (r >= l ? A(r0 + r, r0 + l) : A(r0 + l, r0 + r)) : 0.0;
        y = fma(dcol[r], v[r], y);
      }
      y *= tau;
      double vlv = v[0];
#pragma unroll
      for (int r = 1; r < SB_NB; ++r) vlv = (l == r) ? v[r] : vlv;
      double yv = y * vlv;
      yv += __shfl_xor_sync(0xffffffffu, yv, 1, SB_NB);
      yv += __shfl_xor_sync(0xffffffffu, yv, 2, SB_NB);
      yv += __shfl_xor_sync(0xffffffffu, yv, 4, SB_NB);
      const double wl = y - 0.5 * tau * yv * vlv;
      double w[SB_NB];
#pragma unroll
      for (int r = 0; r < SB_NB; ++r) w[r] = __shfl_sync(0xffffffffu, wl, r, SB_NB);
      if (act && l < L)
#pragma unroll
        for (int r = 0; r < SB_NB; ++r)
          if (r >= l && r < L) A(r0 + r, r0 + l) = dcol[r] - fma(v[r], wl, w[r] * vlv);
      // (d) E = A[r0 + 8 .. r0 + 8 + L2 - 1][R] <- E H: lane = row l of E
      {
        const int L2 = min(SB_NB, k - r0 - SB_NB);
        double e[SB_NB], u = 0.0;
#pragma unroll
        for (int c = 0; c < SB_NB; ++c) {
          e[c] = (l < L2 && c < L) ? A(r0 + SB_NB + l, r0 + c) : 0.0;
          u = fma(e[c], v[c], u);
        }
        u *= tau;
        if (act && l < L2)
#pragma unroll
          for (int c = 0; c < SB_NB; ++c)
            if (c < L) A(r0 + SB_NB + l, r0 + c) = fma(-u, v[c], e[c]);
      }
      __syncwarp();
      fence_cta();
      if (lane == 0) vsp[b] = j + 1;
      ++nsup;
    }
  }
  if (trace && (wid == 0 || wid == SB_NW - 1))
    printf("[sbr chase k=%d warp %d] super-steps %lld, cycles %lld, waiting %lld\n", k, wid, nsup, clock64() - t_start,
           t_wait);
  __syncthreads();
  // T: d = diagonal, e = first subdiagonal (raw) -> the tail
  double dv[(GT_KMAX + SB_NT - 1) / SB_NT], ev[(GT_KMAX + SB_NT - 1) / SB_NT];
#pragma unroll
  for (int u = 0; u < (GT_KMAX + SB_NT - 1) / SB_NT; ++u) {
    const int ii = t + u * SB_NT;
    dv[u] = ii < k ? A(ii, ii) : 0.0;
    ev[u] = ii + 1 < k ? A(ii + 1, ii) : 0.0;
  }
  __syncthreads();
  double* d0 = AB;
  double* e0 = AB + GT_KMAX;
#pragma unroll
  for (int u = 0; u < (GT_KMAX + SB_NT - 1) / SB_NT; ++u) {
    const int ii = t + u * SB_NT;
    if (ii < k) {
      d0[ii] = dv[u];
      e0[ii] = ev[u];
    }
  }
  tri_tail(W, d0, e0, k, t, SB_NT);
}

// Z <- Q2 Z (stage-B reflectors, applied in reverse generation order): a CTA per SQ_COLS columns
// of Z (k x 32 in shared memory, lane = column: each reflector is 8 loads, 16 FMAs and 8 stores per
// lane, no shuffles).  Reflector (s, i) acts on rows [s+1+8i, s+8+8i]; of the reflectors generated
// after it only (s+1, i-1) (row s+1+8i) overlaps it, and (s-1, i+1) is the next one down that
// overlaps it.  So the application is a wavefront without CTA barriers: the warp owning step index
// i applies (s, i) for s descending as soon as index i-1 has applied (s+1, i-1) (per-index
// progress counters in shared memory); the reflectors of the next sweeps are prefetched.
constexpr int SQ_NT = 1024;
constexpr int SQ_NW = SQ_NT / 32;
constexpr int SQ_COLS = 32;
constexpr int SQ_NI = (GT_KMAX + SB_NB - 1) / SB_NB + 1;
constexpr int SQ_RING = 4;  // per-warp cp.async ring of reflector slots
constexpr size_t kSbrQSmem = (size_t)GT_KMAX * SQ_COLS * sizeof(double) + (GT_KMAX + 1 + SQ_NI) * sizeof(int) +
                             (size_t)SQ_NW * SQ_RING * SB_NB * sizeof(double) + 64;

__global__ void __launch_bounds__(SQ_NT, 1) k_sbr_q2(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int item = blockIdx.x;
  const int g = find_item(gt.bt_pre, gt.ng, item);
  if (gt.status[g] < 0) return;
  const int k = a.ksz[gt.task[g]];
  if (k < gt.sbr_min) return;
  const int H = gt.hsel[g];
  const GView W{gt.ws + gt.moff[g], k, H};
  const int nsel = (int)W.hdr()[0];
  // bt_pre counts CTAs of kGtrdBackCols columns: the even ones take SQ_COLS = 2 x 16 columns
  const int local = item - gt.bt_pre[g];
  if (local & 1) return;
  const int col0 = local * kGtrdBackCols;
  if (col0 >= nsel) return;
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31;
  extern __shared__ double smq[];
  double* Zs = smq;                                        // [i][c], k x 32
  int* qoff = reinterpret_cast<int*>(Zs + GT_KMAX * SQ_COLS);
  int* prog = qoff + (GT_KMAX + 1);                        // per step index: lowest sweep applied
  double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(prog + SQ_NI) + 63) & ~uintptr_t(63)) +
                 wid * SQ_RING * SB_NB;                    // this warp's prefetch slots
  double* Z = W.Z();
  const double* Q2 = W.Q2();
  const int nsw = k - 2;
  auto nsteps = [&](int s) { return (k - 1 - s + SB_NB - 1) / SB_NB; };
  const int imax = nsw > 0 ? nsteps(0) : 0;
  if (t == 0) {
    int acc = 0;
    for (int s = 0; s < nsw; ++s) {
      qoff[s] = acc;
      acc += nsteps(s);
    }
  }
  for (int i = t; i < SQ_NI; i += SQ_NT) prog[i] = 1 << 30;
  for (int e = t; e < k * SQ_COLS; e += SQ_NT) {
    const int c = e / k, i = e % k;
    Zs[i * SQ_COLS + c] = col0 + c < nsel ? Z[(int64_t)(col0 + c) * k + i] : 0.0;
  }
  __syncthreads();
  volatile int* vprog = prog;
  auto shi_of = [&](int i) { return min(nsw - 1, k - 2 - SB_NB * i); };  // last sweep with a step i
  const bool trace = gt.debug == 3 && blockIdx.x == 0 && lane == 0 && (wid == 0 || wid == SQ_NW - 1);
  long long t_wait = 0, t_start = clock64(), nstep = 0;
  for (int i = wid; i < imax; i += SQ_NW) {
    const int shi = shi_of(i);
    const int shp = i > 0 ? shi_of(i - 1) : -1;
    // reflector (tau, v_1 .. v_7) of sweeps shi, shi-1, ... staged SQ_RING - 1 ahead by cp.async
    // (lanes 0..7, one element each; the fences below do not wait for them)
    __syncwarp();
    for (int u = 0; u < SQ_RING - 1; ++u) {
      if (lane < SB_NB && shi - u >= 0)
        cp_async8(ring + ((shi - u) & (SQ_RING - 1)) * SB_NB + lane, Q2 + (int64_t)(qoff[shi - u] + i) * SB_NB + lane);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    for (int s = shi; s >= 0; --s) {
      if (lane < SB_NB && s - (SQ_RING - 1) >= 0)
        cp_async8(ring + ((s - (SQ_RING - 1)) & (SQ_RING - 1)) * SB_NB + lane,
                  Q2 + (int64_t)(qoff[s - (SQ_RING - 1)] + i) * SB_NB + lane);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group %0;\n" ::"n"(SQ_RING - 1) : "memory");
      if (i > 0 && s + 1 <= shp) {  // (s+1, i-1) must be applied first (every lane polls: no divergence)
        const long long tw0 = trace ? clock64() : 0;
        while (vprog[i - 1] > s + 1) __nanosleep(20);
        if (trace) t_wait += clock64() - tw0;
        fence_cta();
      }
      __syncwarp();
      // tau, v_1 .. v_7 from the staged slot (broadcast loads); tau = 0 reflectors are applied as
      // identities (their stored v is 0), so the step has no lane-dependent branch
      const double2* rs = reinterpret_cast<const double2*>(ring + (s & (SQ_RING - 1)) * SB_NB);
      double v[SB_NB];
      double tau;
      {
        const double2 p0 = rs[0], p1 = rs[1], p2 = rs[2], p3 = rs[3];
        tau = p0.x;
        v[0] = 1.0;
        v[1] = p0.y;
        v[2] = p1.x;
        v[3] = p1.y;
        v[4] = p2.x;
        v[5] = p2.y;
        v[6] = p3.x;
        v[7] = p3.y;
      }
      const int r0 = s + 1 + SB_NB * i;
      const int L = min(SB_NB, k - r0);
      double z[SB_NB], d = 0.0;
#pragma unroll
      for (int r = 0; r < SB_NB; ++r) {
        z[r] = r < L ? Zs[(r0 + r) * SQ_COLS + lane] : 0.0;
        d = fma(v[r], z[r], d);
      }
      d *= tau;
#pragma unroll
      for (int r = 0; r < SB_NB; ++r)
        if (r < L) Zs[(r0 + r) * SQ_COLS + lane] = fma(-d, v[r], z[r]);
      __syncwarp();
      fence_cta();
      if (lane == 0) vprog[i] = s;
      ++nstep;
    }
  }
  if (trace) printf("[sbr q2 k=%d warp %d] steps %lld, cycles %lld, waiting %lld\n", k, wid, nstep, clock64() - t_start, t_wait);
  __syncthreads();
  for (int e = t; e < k * SQ_COLS; e += SQ_NT) {
    const int c = e / k, i = e % k;
    if (col0 + c < nsel) Z[(int64_t)(col0 + c) * k + i] = Zs[i * SQ_COLS + c];
  }
}

// ---------------------------------------------------------------- 3. back-transform V = Q Z
// Q = H_0 H_1 ... H_{k-3}; the reflectors are applied in groups of GB_NR from the last one down,
// each group in compact WY form H_lo ... H_hi = I - Y T Y^T (LAPACK dlarft, forward).
// k_gtrd_wy forms every group's T once per matrix (Y^T Y by the CTA's warps, T by warp 0);
// k_gtrd_back stages Y (double-buffered: the next group's loads are issued before the current
// group is applied) and, per column (a warp, the column in registers), z <- z - Y (T (Y^T z)):
// one 16-wide warp reduction per group.
constexpr int GB_NT = 512;   // 16 warps = 16 columns
constexpr int GB_NR = 16;    // reflectors per group

__global__ void __launch_bounds__(GB_NT) k_gtrd_wy(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int g = find_item(gt.wy_pre, gt.ng, blockIdx.x);
  if (gt.status[g] < 0) return;
  const int k = a.ksz[gt.task[g]];
  const GView W{gt.ws + gt.moff[g], k, gt.hsel[g], k >= gt.sbr_min ? SB_NB : 1};
  const int ro = W.ro;
  const int gi = blockIdx.x - gt.wy_pre[g];
  if (gi >= W.nwy()) return;
  const int jhi = W.nref() - 1 - gi * GB_NR;
  const int nr = min(GB_NR, jhi + 1);
  const int jlo = jhi - nr + 1;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ double vb[];          // Y: GB_NR x GT_KMAX
  double* Gm = vb + GB_NR * GT_KMAX;      // Y^T Y (upper)
  double* Tm = Gm + GB_NR * GB_NR;
  const double* M = W.M();
  const int LD = W.ld();
  for (int e = threadIdx.x; e < GB_NR * k; e += GB_NT) {  // v_j lives in column j: c fastest
    const int c = e % GB_NR, i = e / GB_NR;
    const int j = jlo + c;
    vb[c * GT_KMAX + i] = (c >= nr || i < j + ro) ? 0.0 : (i == j + ro ? 1.0 : M[(int64_t)i * LD + j]);
  }
  __syncthreads();
  for (int pr = wid; pr < GB_NR * (GB_NR - 1) / 2; pr += GB_NT / 32) {
    int aa = 0, rem = pr;
    while (rem >= GB_NR - 1 - aa) {
      rem -= GB_NR - 1 - aa;
      ++aa;
    }
    const int bb = aa + 1 + rem;
    double sacc = 0.0;
    if (bb < nr)
      for (int i = jlo + ro + lane; i < k; i += 32) sacc = fma(vb[aa * GT_KMAX + i], vb[bb * GT_KMAX + i], sacc);
    sacc = warp_sum(sacc);
    if (lane == 0) Gm[aa * GB_NR + bb] = sacc;
  }
  __syncthreads();
  if (wid == 0) {
    // T[c][c] = tau_c;  T[0:c, c] = -tau_c T[0:c, 0:c] (Y^T y_c)[0:c]
    for (int c = 0; c < GB_NR; ++c) {
      const double tau = c < nr ? W.tau()[jlo + c] : 0.0;
      double tv = 0.0;
      if (lane < c)
        for (int q = lane; q < c; ++q) tv = fma(Tm[lane * GB_NR + q], Gm[q * GB_NR + c], tv);
      __syncwarp();
      if (lane < c) Tm[lane * GB_NR + c] = -tau * tv;
      if (lane == c) Tm[c * GB_NR + c] = tau;
      if (lane > c && lane < GB_NR) Tm[lane * GB_NR + c] = 0.0;
      __syncwarp();
    }
    double* out = W.wyT() + (int64_t)gi * GB_NR * GB_NR;
    for (int e = lane; e < GB_NR * GB_NR; e += 32) out[e] = Tm[e];
  }
}

// k_gtrd_back: the columns of a CTA (kGtrdBackCols = 16) live in shared memory as a k x 16 block
// Zs; 8 warps own 8-row-aligned slices of its rows.  Per group: S = Y^T Zs (16 x 16, DMMA
// m8n8k4 over each warp's rows, partials summed in a fixed order), U = T S, Zs -= Y U (DMMA on
// the warp's rows).  Y is staged with cp.async; shared memory: Y 16 x (k_max + 4), Zs 832 x 16.
constexpr int BM_NW = 8;
constexpr int BM_NT = 32 * BM_NW;
constexpr int BM_ZROWS = 8 * (((GT_KMAX + 63) / 64) * 8);  // 8 warps x rows per warp (max)
constexpr int BM_YLD = BM_ZROWS + 4;  // >= the rows the warps sweep; == 4 (mod 16): conflict-free Y^T fragments
static_assert(BM_YLD % 16 == 4, "Y row stride");
static_assert(kGtrdBackCols == 16, "two 8-wide DMMA column tiles");

__device__ __forceinline__ void dmma_b(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(BM_NT, 1) k_gtrd_back(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int item = blockIdx.x;
  const int g = find_item(gt.bt_pre, gt.ng, item);
  if (gt.status[g] < 0) return;
  const int k = a.ksz[gt.task[g]];
  const int H = gt.hsel[g];
  const GView W{gt.ws + gt.moff[g], k, H, k >= gt.sbr_min ? SB_NB : 1};
  const int ro = W.ro;
  const int nsel = (int)W.hdr()[0];
  const int col0 = (item - gt.bt_pre[g]) * kGtrdBackCols;
  if (col0 >= nsel) return;
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31, r4 = lane >> 2, c4 = lane & 3;
  extern __shared__ double smb[];
  double* Ys = smb;                       // [c][i], 16 x BM_YLD
  double* Zs = Ys + 16 * BM_YLD;          // [i][col], BM_ZROWS x 16
  double* Sp = Zs + BM_ZROWS * 16;        // BM_NW x 256 partials of S, then S and U
  double* Ts = Sp + BM_NW * 256;          // T of the group (16 x 16)
  const double* M = W.M();
  const int LD = W.ld();
  double* Z = W.Z();
  const int RS = ((k + 63) / 64) * 8;     // rows per warp (8 | RS, 8 RS >= k)
  const int rb = wid * RS;
  for (int e = t; e < 16 * BM_YLD; e += BM_NT) Ys[e] = 0.0;
  for (int e = t; e < BM_ZROWS * 16; e += BM_NT) {
    const int col = e / BM_ZROWS, i = e % BM_ZROWS;  // coalesced along a column of Z
    Zs[i * 16 + col] = (i < k && col0 + col < nsel) ? Z[(int64_t)(col0 + col) * k + i] : 0.0;
  }
  const int ngr = W.nwy();
  for (int gi = 0; gi < ngr; ++gi) {
    const int jhi = W.nref() - 1 - gi * GB_NR;
    const int nr = min(GB_NR, jhi + 1);
    const int jlo = jhi - nr + 1;
    __syncthreads();  // previous group's Y / U no longer read
    for (int e = t; e < GB_NR * k; e += BM_NT) {  // v_j lives in column j of M: c fastest
      const int c = e % GB_NR, i = e / GB_NR;
      const int j = jlo + c;
      if (c >= nr || i < j + ro)
        Ys[c * BM_YLD + i] = 0.0;
      else if (i == j + ro)
        Ys[c * BM_YLD + i] = 1.0;
      else
        cp_async8(Ys + c * BM_YLD + i, M + (int64_t)i * LD + j);
    }
    for (int e = t; e < GB_NR * GB_NR; e += BM_NT) cp_async8(Ts + e, W.wyT() + (int64_t)gi * GB_NR * GB_NR + e);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    // S partial = Y(rows of this warp)^T Zs(rows of this warp)
    {
      double acc[2][2][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 2; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
      const int kb = max(rb, (jlo + ro) & ~3);  // rows < jlo + ro are zero in Y
      for (int kk = kb; kk < rb + RS; kk += 4) {
        const double a0 = Ys[r4 * BM_YLD + kk + c4], a1 = Ys[(8 + r4) * BM_YLD + kk + c4];
        const double b0 = Zs[(kk + c4) * 16 + r4], b1 = Zs[(kk + c4) * 16 + 8 + r4];
        dmma_b(acc[0][0], a0, b0);
        dmma_b(acc[0][1], a0, b1);
        dmma_b(acc[1][0], a1, b0);
        dmma_b(acc[1][1], a1, b1);
      }
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          Sp[wid * 256 + (m * 8 + r4) * 16 + n * 8 + 2 * c4] = acc[m][n][0];
          Sp[wid * 256 + (m * 8 + r4) * 16 + n * 8 + 2 * c4 + 1] = acc[m][n][1];
        }
    }
    __syncthreads();
    // S = sum of the partials (fixed order), then U = T S (T upper)
    double sv = 0.0;
    for (int w = 0; w < BM_NW; ++w) sv += Sp[w * 256 + t];
    __syncthreads();
    Sp[t] = sv;  // S[c][col], t = c * 16 + col
    __syncthreads();
    {
      const int c = t >> 4, col = t & 15;
      double u = 0.0;
      for (int q = c; q < GB_NR; ++q) u = fma(Ts[c * GB_NR + q], Sp[q * 16 + col], u);
      Sp[256 + t] = u;  // U[c][col]
    }
    __syncthreads();
    // Zs(rows of this warp) -= Y(rows) U
    const double* U = Sp + 256;
    for (int it = 0; it < RS; it += 8) {
      if (rb + it + 7 < jlo + ro) continue;  // Y rows < jlo + ro are zero
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const double av = Ys[(ks * 4 + c4) * BM_YLD + rb + it + r4];
        dmma_b(acc[0], av, U[(ks * 4 + c4) * 16 + r4]);
        dmma_b(acc[1], av, U[(ks * 4 + c4) * 16 + 8 + r4]);
      }
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        double* zp = Zs + (rb + it + r4) * 16 + n * 8 + 2 * c4;
        zp[0] -= acc[n][0];
        zp[1] -= acc[n][1];
      }
    }
  }
  __syncthreads();
  for (int e = t; e < k * 16; e += BM_NT) {
    const int col = e / k, i = e % k;
    if (col0 + col < nsel) Z[(int64_t)(col0 + col) * k + i] = Zs[i * 16 + col];
  }
}

// ---------------------------------------------------------------- 4. reconstruction
constexpr int GR_NW = 8;
constexpr int GR_LDS = 36;
struct GrSmem {
  double X[32 * GR_LDS];
  double Y[32 * GR_LDS];
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(GR_NW * 32) k_gtrd_recon(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  extern __shared__ __align__(16) unsigned char smraw[];
  GrSmem& sm = reinterpret_cast<GrSmem*>(smraw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31, r4 = lane >> 2, c4 = lane & 3;
  const int item = blockIdx.x * GR_NW + (threadIdx.x >> 5);
  if (item >= gt.tot_rc) return;
  int g = 0;
  {
    int lo = 0, hi = gt.ng - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (gt.rc_pre[mid] <= item) lo = mid; else hi = mid - 1;
    }
    g = lo;
  }
  if (gt.status[g] < 0) return;
  const int task = gt.task[g];
  const int k = a.ksz[task];
  const int H = gt.hsel[g];
  const GView W{gt.ws + gt.moff[g], k, H};
  const int nsel = (int)W.hdr()[0], side = (int)W.hdr()[1];
  int rb, cb;
  packed_rc(item - gt.rc_pre[g], rb, cb);
  const double* Z = W.Z();
  double acc[4][4][2];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q][0] = acc[p][q][1] = 0.0;
  const double* lwg = W.lw();
  for (int kk = 0; kk < nsel; kk += 32) {
    __syncwarp();
    // 64 asynchronous 8-byte copies per lane (lanes along the rows: Z is column-major), zero-filled
    // outside the matrix / the selected columns: one L2 round trip per K chunk instead of one per
    // few loads; the weights lw scale the A fragments below
    {
      const int rr = rb * 32 + lane, cc = cb * 32 + lane;
#pragma unroll 8
      for (int u = 0; u < 32; ++u) {
        const int uu = kk + u;
        const bool ok = uu < nsel;
        const double* zx = Z + (int64_t)(ok ? uu : 0) * k;
        cp_async8z(&sm.X[lane * GR_LDS + u], zx + (rr < k ? rr : 0), ok && rr < k);  // [m][k]
        cp_async8z(&sm.Y[lane * GR_LDS + u], zx + (cc < k ? cc : 0), ok && cc < k);  // [n][k]
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    const double lwl = kk + lane < nsel ? lwg[kk + lane] : 0.0;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const double w = __shfl_sync(0xffffffffu, lwl, ks * 4 + c4);
      double af[4], bf[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        af[q] = sm.X[(q * 8 + r4) * GR_LDS + ks * 4 + c4] * w;
        bf[q] = sm.Y[(q * 8 + r4) * GR_LDS + ks * 4 + c4];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma(acc[p][q], af[p], bf[q]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      sm.X[(p * 8 + r4) * GR_LDS + q * 8 + 2 * c4] = acc[p][q][0];
      sm.X[(p * 8 + r4) * GR_LDS + q * 8 + 2 * c4 + 1] = acc[p][q][1];
    }
  __syncwarp();
  const int64_t off = a.off[task];
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  for (int e = lane; e < 1024; e += 32) {
    const int jj = e >> 5, ii = e & 31;  // column-major walk: consecutive packed entries
    const int r = rb * 32 + ii, c = cb * 32 + jj;
    if (r > c || c >= k) continue;
    double v = sm.X[ii * GR_LDS + jj];
    const int64_t pe = off + (int64_t)c * (c + 1) / 2 + r;
    if (side == 1) v += input_value<MODE>(a, pe, r, c);
    if constexpr (MODE == PM_BATCH) {
      a.out[pe] = v;
    } else if constexpr (MODE == PM_PRIMAL) {
      const double xkv = (r == c) ? v : v * kSqrt2;
      const double hx = __ldg(a.x + a.G[pe]);
      const double dd = xkv - hx;
      a.xk[pe] = xkv;
      a.lam[pe] = a.lam[pe] + a.rho * dd;  // E:LambdakUpdate
      p0 += dd * dd;
      p1 += xkv * xkv;
      p2 += hx * hx;
    } else {
      a.xk[pe] = (r == c) ? v : v * kSqrt2;
    }
  }
  if constexpr (MODE == PM_PRIMAL) {
    p0 = warp_sum(p0);
    p1 = warp_sum(p1);
    p2 = warp_sum(p2);
    if (lane == 0) {
      gt.part[3 * (int64_t)item + 0] = p0;
      gt.part[3 * (int64_t)item + 1] = p1;
      gt.part[3 * (int64_t)item + 2] = p2;
    }
  }
}

__global__ void k_gtrd_fin(ProjArgs a) {
  if (a.done && *a.done) return;
  const GtrdDev& gt = a.gd.gt;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= gt.ng || gt.status[g] < 0) return;
  const int task = gt.task[g];
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  for (int t = gt.rc_pre[g]; t < gt.rc_pre[g + 1]; ++t) {
    p0 += gt.part[3 * (int64_t)t + 0];
    p1 += gt.part[3 * (int64_t)t + 1];
    p2 += gt.part[3 * (int64_t)t + 2];
  }
  a.part[3 * (int64_t)task + 0] = p0;
  a.part[3 * (int64_t)task + 1] = p1;
  a.part[3 * (int64_t)task + 2] = p2;
}


constexpr size_t kWySmem = (size_t)(GB_NR * GT_KMAX + 2 * GB_NR * GB_NR) * sizeof(double);
constexpr size_t kBackSmem = (size_t)(16 * BM_YLD + BM_ZROWS * 16 + BM_NW * 256 + GB_NR * GB_NR) * sizeof(double);

template <int MODE>
void launch_mode(const ProjArgs& a, cudaStream_t s) {
  const GtrdDev& gt = a.gd.gt;
  if (gt.njob) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gt.njob * TC_CS);
    cfg.blockDim = dim3(TC_NT);
    cfg.dynamicSmemBytes = kTriSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = TC_CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_gtrd_tridiag<MODE>, a);
  }
  if (gt.njob2) {  // two-stage: dense -> band (clusters of SA_CS CTAs) -> tridiagonal (a CTA each)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gt.njob2 * SA_CS);
    cfg.blockDim = dim3(SA_NT);
    cfg.dynamicSmemBytes = kSbrASmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = SA_CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_sbr_band<MODE>, a);
    k_sbr_chase<<<gt.nsb, SB_NT, kSbrBSmem, s>>>(a);
  }
  if (gt.tot_ev) {
    k_gtrd_bisect<<<gt.tot_ev, 32, (size_t)2 * gt.kmax * sizeof(double), s>>>(a);
    k_gtrd_cluster<<<gt.ng, 32, (size_t)gt.kmax * sizeof(double), s>>>(a);
    k_gtrd_vec<<<gt.tot_vg, VT, (size_t)kVecSmemDoubles * sizeof(double), s>>>(a);
  }
  if (gt.nsb && gt.tot_bt) k_sbr_q2<<<gt.tot_bt, SQ_NT, kSbrQSmem, s>>>(a);
  if (gt.tot_wy) k_gtrd_wy<<<gt.tot_wy, GB_NT, kWySmem, s>>>(a);
  if (gt.tot_bt) k_gtrd_back<<<gt.tot_bt, BM_NT, kBackSmem, s>>>(a);
  if (gt.tot_rc) k_gtrd_recon<MODE><<<(gt.tot_rc + GR_NW - 1) / GR_NW, GR_NW * 32, GR_NW * sizeof(GrSmem), s>>>(a);
  if (MODE == PM_PRIMAL) k_gtrd_fin<<<(gt.ng + 127) / 128, 128, 0, s>>>(a);
}

template <int MODE>
void set_attrs() {
  cudaFuncSetAttribute(k_gtrd_tridiag<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTriSmem);
  if (TC_CS > 8) cudaFuncSetAttribute(k_gtrd_tridiag<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_sbr_band<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSbrASmem);
  cudaFuncSetAttribute(k_gtrd_recon<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(GR_NW * sizeof(GrSmem)));
}

}  // namespace

void psd_gtrd_init_attributes() {
  set_attrs<PM_BATCH>();
  set_attrs<PM_PRIMAL>();
  set_attrs<PM_DUAL>();

  cudaFuncSetAttribute(k_gtrd_vec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kVecSmemDoubles * sizeof(double)));
  cudaFuncSetAttribute(k_gtrd_back, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBackSmem);
  cudaFuncSetAttribute(k_gtrd_wy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWySmem);
  cudaFuncSetAttribute(k_sbr_chase, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSbrBSmem);
  cudaFuncSetAttribute(k_sbr_q2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSbrQSmem);
}

int gtrd_max_order() { return GT_KMAX; }
int64_t gtrd_ws_doubles(int k) { return gview_doubles(k); }

void launch_projection_gtrd(int mode, const ProjArgs& a, cudaStream_t s) {
  if (a.gd.gt.ng <= 0) return;
  if (mode == PM_BATCH)
    launch_mode<PM_BATCH>(a, s);
  else if (mode == PM_PRIMAL)
    launch_mode<PM_PRIMAL>(a, s);
  else
    launch_mode<PM_DUAL>(a, s);
}

}  // namespace sdp
