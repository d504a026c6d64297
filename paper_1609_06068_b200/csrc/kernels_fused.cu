// Fused persistent iteration for small problems (cfg0 / cfg1 sizes): the whole ADMM iteration
// (Algorithm 1 lines 4-7 / Algorithm 2 lines 4-8, in the same order as api.cu's one-graph
// iteration) runs inside ONE cooperative kernel launch, looping over iterations, with grid-wide
// barriers between the phases instead of kernel boundaries.  For problems whose iteration is a few
// microseconds of work the separate launches (8-10 per iteration) are the cost; here a call of
// sdp_step(h, iters) is one launch.
//
// Phases (primal / dual):
//   U  u = A rD - r2 (r2 = b primal, -b/rho dual)            warp per row
//   Y  y = S^-1 u (cached dense S^-1) or u / diag(S)          warp per row
//   X  x = rD - D^-1 A^T y, objective partial                 warp per coordinate
//   P  x_k = P_+(H_k x - lam_k/rho), lam_k update (primal)    register-V Jacobi groups (psd_rv.cuh)
//      z_k = P_+(v_k - lam_k/rho) (dual)                        (E:XkUpdate / E:zkUpdate)
//   S  r1 = sum_k H_k^T(.) -> rD, eps_d partials              thread per coordinate
//   V  v_k, lam_k (dual)                                      thread per stacked entry (E:vkEqn)
//   F  residuals (reading G9), objective, history, stop flag  every CTA, same order
// Every CTA reduces its thread partials in a fixed order into a per-CTA slot; after the last
// barrier of the iteration every CTA sums the slots in the same order, so all CTAs take the same
// stop decision without another barrier, and CTA 0 publishes res / hist / iter / done.  The grid
// and the work assignment are fixed at setup, so two runs give bit-identical iterates.
//
// Global data written inside the kernel (x, y, u, rD, x_k, lam_k, v_k, partials) is read with
// coherent loads only; __ldg is kept for the constant problem data (A, A^T, S^-1, b, c, D^-1, maps).
#include <type_traits>

#include "kernels_fused.h"
#include "psd_rv.cuh"

namespace sdp {

namespace {

constexpr int FT = kFusedThreads;  // threads per CTA
constexpr int kLongSegF = kFusedLongSeg;
constexpr int FU = 8;              // phases U / X: 16-byte loads in flight per lane
constexpr int FW = FT / 32;        // warps per CTA

__device__ __forceinline__ double fwarp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Grid-wide barrier (all CTAs co-resident: cooperative launch).  One monotone arrival counter per
// launch: barrier j of the launch completes when the counter reaches j * gridDim.x, so a CTA pays
// one atomic and its polling, and nobody resets anything between barriers.  Launches alternate
// between two counters; CTA 0 zeroes the other one (idle since the previous launch) at the start.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier(unsigned* cnt, unsigned& target) {
  __syncthreads();
  if (gridDim.x == 1) return;
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt, 1u);
    while ((int)(ld_acquire_u32(cnt) - target) < 0) {
    }
  }
  __syncthreads();
}

// sum_e val[e] * v[idx[e]] over the entries ptr[r] + sl, + L, ... (v written in the kernel: coherent)
__device__ __forceinline__ double seg_dot(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                          const double* __restrict__ val, const double* v, int r, int sl, int L) {
  double s = 0.0;
  const int e1 = __ldg(ptr + r + 1);
  for (int e = __ldg(ptr + r) + sl; e < e1; e += L) s = fma(__ldg(val + e), v[__ldg(idx + e)], s);
  return s;
}

// block-wide deterministic sum of NV values per thread (fixed warp order); result in every thread
template <int NV>
__device__ __forceinline__ void block_sum_all(double (&v)[NV], double* sm /* NV * FW */) {
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = fwarp_sum(v[j]);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) sm[j * FW + w] = v[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < FW; ++i) s += sm[j * FW + i];
    v[j] = s;
  }
}

template <int KP, int Q>
struct FGroupLay {
  using Lay = RvLayout<KP, Q>;
  static constexpr int G = Lay::G;
  static constexpr int NG = FT / G;
  static constexpr int per_group = Lay::template per_group<3>();
  static constexpr int doubles = NG * per_group;
  static_assert(G <= FT && FT % G == 0, "group must divide the CTA");
};
using L8 = FGroupLay<8, 2>;
using L16 = FGroupLay<16, 4>;
using L32 = FGroupLay<32, 4>;
constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr int kGroupDoubles = cmax(L8::doubles, cmax(L16::doubles, L32::doubles));
constexpr int kTabInts = RvLayout<8, 2>::NBLK + RvLayout<16, 4>::NBLK + RvLayout<32, 4>::NBLK;

template <int KP>
__device__ void build_tab(int* tab) {
  constexpr int P = KP / 2;
  constexpr int NBLK = P * (P + 1) / 2;
  for (int b = threadIdx.x; b < NBLK; b += FT) {
    int i = 0, rem = b;
    while (rem >= P - i) {
      rem -= P - i;
      ++i;
    }
    tab[b] = (i << 16) | (i + rem);
  }
}

// one bucket of cliques: groups of G threads, slots strided over the grid
template <int KP, int Q, int MODE>
__device__ void fused_bucket(const ProjArgs& pa, const int32_t* __restrict__ ids, int count, double* smem,
                             const int* tab) {
  using FL = FGroupLay<KP, Q>;
  using Lay = RvLayout<KP, Q>;
  constexpr int G = FL::G;
  const int grp = threadIdx.x / G;
  RvGroup<G> g;
  g.tid = threadIdx.x % G;
  g.mask = (G >= 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) / G * G));
  g.bar = 1 + grp;
  double* base = smem + (size_t)grp * FL::per_group;
  double* A0 = base;
  double* A1 = base + KP * Lay::LD;
  double* T = A1 + KP * Lay::LD;
  double* rc = base + 3 * KP * Lay::LD;
  double* rs = rc + Lay::P;
  double* rt = rs + Lay::P;
  g.red = rt + Lay::P;
  // slot = grp * grid + CTA: consecutive cliques land on different SMs (the projections are
  // latency-bound chains; one group per SM runs them fastest)
  for (int slot = grp * gridDim.x + blockIdx.x; slot < count; slot += gridDim.x * FL::NG) {
    const int task = __ldg(ids + slot);
    project_rv<KP, Q, MODE, true>(g, __ldg(pa.ksz + task), __ldg(pa.off + task), task, A0, A1, T, rc, rs, rt, tab,
                                  pa);
  }
  __syncthreads();
}

// slots of the per-CTA partials
enum { CP_U0 = 0, CP_U1, CP_U2, CP_S0, CP_S1, CP_GT, CP_BY, CP_N = 8 };

template <int FORM>
__global__ void __launch_bounds__(FT, 1) k_fused_iter(FusedArgs a) {
  extern __shared__ double smem[];
  __shared__ double sred[8 * FW];
  __shared__ long long s_iter;
  __shared__ int s_stop;
  int* tab8 = reinterpret_cast<int*>(smem + kGroupDoubles);
  int* tab16 = tab8 + RvLayout<8, 2>::NBLK;
  int* tab32 = tab16 + RvLayout<16, 4>::NBLK;
  build_tab<8>(tab8);
  build_tab<16>(tab16);
  build_tab<32>(tab32);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * FW + warp, nw = gridDim.x * FW;
  const int gt = blockIdx.x * FT + threadIdx.x, nt = gridDim.x * FT;
  const double rho = a.rho;
  const long long it0 = *a.iter;
  unsigned* bar = a.bar + a.bar_parity;
  unsigned bar_target = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.bar[1 - a.bar_parity] = 0u;  // for the next launch
  if (*a.done) return;  // no writer before the first barrier: every CTA reads the same value
  ProjArgs pa = a.pa;
  pa.iter = &s_iter;  // the warm-start decision reads the CTA's copy of the iteration index
  pa.done = nullptr;
  pa.rvtrace = a.trace ? a.trace + 64 * 16 : nullptr;
  const double2* rD2 = reinterpret_cast<const double2*>(a.rD);
  const double2* y2 = reinterpret_cast<const double2*>(a.y);
  long long* trace = (a.trace && blockIdx.x == 0) ? a.trace : nullptr;
#define FMARK(ph)                                                                        \
  if (trace && threadIdx.x == 0) {                                                       \
    unsigned long long t_;                                                               \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
    trace[(int64_t)(i & 63) * 16 + (ph)] = (long long)t_;                                \
  }
  for (int i = 0; i < a.iters; ++i) {
    FMARK(0);
    if (threadIdx.x == 0) s_iter = it0 + i;
    __syncthreads();
    double acc[CP_N] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto projection = [&](auto mode_tag) {
      constexpr int MODE = decltype(mode_tag)::value;
      if (a.count[0]) fused_bucket<8, 2, MODE>(pa, a.ids[0], a.count[0], smem, tab8);
      if (a.count[1]) fused_bucket<16, 4, MODE>(pa, a.ids[1], a.count[1], smem, tab16);
      if (a.count[2]) fused_bucket<32, 4, MODE>(pa, a.ids[2], a.count[2], smem, tab32);
    };
    auto scatter = [&]() {
      // r1 = sum_k H_k^T (x_k + lam_k/rho) - c/rho  (primal) | c - sum_k H_k^T (z_k + lam_k/rho) (dual)
      auto finish = [&](int t, double sr, double sx, double sl) {
        const double ct = __ldg(a.c + t);
        const double r1 = (FORM == 0) ? sr - ct / rho : ct - sr;
        a.rD[t] = r1 * __ldg(a.Dinv + t);
        const double d = sx - a.sprev[t];
        a.sprev[t] = sx;
        acc[CP_S0] += d * d;
        acc[CP_S1] += sl * sl;
      };
      // short segments (<= kLongSegF entries): a thread each, all loads of the segment in flight
      for (int t = gt; t < a.N; t += nt) {
        const int b = __ldg(a.seg_ptr + t), e = __ldg(a.seg_ptr + t + 1);
        if (e - b > kLongSegF) continue;
        int si[kLongSegF];
#pragma unroll
        for (int q = 0; q < kLongSegF; ++q) si[q] = b + q < e ? __ldg(a.seg_idx + b + q) : -1;
        double xv[kLongSegF], lv[kLongSegF];
#pragma unroll
        for (int q = 0; q < kLongSegF; ++q) {
          xv[q] = si[q] >= 0 ? pa.xk[si[q]] : 0.0;
          lv[q] = si[q] >= 0 ? pa.lam[si[q]] : 0.0;
        }
        double sr = 0.0, sx = 0.0, sl = 0.0;
#pragma unroll
        for (int q = 0; q < kLongSegF; ++q)
          if (si[q] >= 0) {
            sr += xv[q] + lv[q] / rho;
            sx += xv[q];
            sl += lv[q];
          }
        finish(t, sr, sx, sl);
      }
      // long segments: a warp each (lane-strided, fixed-order warp sum)
      for (int w = gw; w < a.n_long; w += nw) {
        const int t = __ldg(a.longc + w);
        const int b = __ldg(a.seg_ptr + t), e = __ldg(a.seg_ptr + t + 1);
        double sr = 0.0, sx = 0.0, sl = 0.0;
        for (int q = b + lane; q < e; q += 32) {
          const int si = __ldg(a.seg_idx + q);
          const double xv = pa.xk[si], lv = pa.lam[si];
          sr += xv + lv / rho;
          sx += xv;
          sl += lv;
        }
        sr = fwarp_sum(sr);
        sx = fwarp_sum(sx);
        sl = fwarp_sum(sl);
        if (lane == 0) finish(t, sr, sx, sl);
      }
    };
    if constexpr (FORM == 1) {
      projection(std::integral_constant<int, PM_DUAL>{});
      FMARK(1);
      grid_barrier(bar, bar_target);
      FMARK(2);
      scatter();
      FMARK(3);
      grid_barrier(bar, bar_target);
      FMARK(4);
    }
    // ---- U: u = A rD - r2 (row i split over `usplit` warps; partials in upart)
    if (a.a_rp) {  // sparse A (CSR): ul lanes per row
      const int L = a.ul, per = 32 / L, sub = lane / L, sl = lane - sub * L;
      for (int base = gw * per; base < a.m; base += nw * per) {
        const int r = base + sub;
        double sum = (r < a.m) ? seg_dot(a.a_rp, a.a_ci, a.a_val, a.rD, r, sl, L) : 0.0;
        for (int o = L / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (r < a.m && sl == 0) a.upart[r] = sum;
      }
    } else {
      const int nwork = a.m * a.usplit;
      const int64_t np = a.lda / 2;
      const int64_t per = (np + a.usplit - 1) / a.usplit;
      for (int w = gw; w < nwork; w += nw) {
        const int row = w / a.usplit, part = w - row * a.usplit;
        const int64_t j0 = part * per, j1 = min(np, j0 + per);
        const double2* Ar = reinterpret_cast<const double2*>(a.A + (int64_t)row * a.lda);
        double s0 = 0.0, s1 = 0.0;
        for (int64_t j = j0 + lane; j < j1; j += 32 * FU) {
          double2 av[FU], rv[FU];
#pragma unroll
          for (int q = 0; q < FU; ++q) {
            const int64_t jj = j + 32 * q;
            av[q] = jj < j1 ? __ldg(Ar + jj) : make_double2(0.0, 0.0);
            rv[q] = jj < j1 ? rD2[jj] : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int q = 0; q < FU; ++q) {
            s0 = fma(av[q].x, rv[q].x, s0);
            s1 = fma(av[q].y, rv[q].y, s1);
          }
        }
        const double s = fwarp_sum(s0 + s1);
        if (lane == 0) a.upart[(int64_t)part * a.m + row] = s;
      }
    }
    FMARK(5);
    grid_barrier(bar, bar_target);
    FMARK(6);
    // ---- Y: y = S^-1 u  (u = sum of the row partials - r2, formed per use)
    if (a.sdiag) {
      for (int r = gt; r < a.m; r += nt) {
        double s = 0.0;
        for (int q = 0; q < a.usplit; ++q) s += a.upart[(int64_t)q * a.m + r];
        const double br = __ldg(a.b + r);
        const double u = (FORM == 0) ? s - br : s + br / rho;
        const double yv = u / __ldg(a.sdiag + r);
        a.y[r] = yv;
        if (FORM == 1) acc[CP_BY] += br * yv;
      }
    } else {
      double* us = smem;  // u, formed by every CTA (m doubles; m <= kFusedMaxM)
      for (int r = threadIdx.x; r < a.m; r += FT) {
        double s = 0.0;
        for (int q = 0; q < a.usplit; ++q) s += a.upart[(int64_t)q * a.m + r];
        const double br = __ldg(a.b + r);
        us[r] = (FORM == 0) ? s - br : s + br / rho;
      }
      __syncthreads();
      for (int r = gw; r < a.m; r += nw) {
        const double* Sr = a.Sinv + (int64_t)r * a.m;
        double s = 0.0;
        for (int j = lane; j < a.m; j += 32) s = fma(__ldg(Sr + j), us[j], s);
        s = fwarp_sum(s);
        if (lane == 0) {
          a.y[r] = s;
          if (FORM == 1) acc[CP_BY] += __ldg(a.b + r) * s;
        }
      }
      __syncthreads();  // us (smem) is reused by the projection
    }
    FMARK(7);
    grid_barrier(bar, bar_target);
    FMARK(8);
    // ---- X: x = rD - D^-1 A^T y, objective partial (c.x primal, |D x|^2 dual); xl lanes per
    // coordinate (rows of A^T are m long), 32 / xl coordinates per warp and round
    if (a.at_cp) {  // sparse A^T (CSC of A): xl lanes per coordinate
      const int L = a.xl, per = 32 / L, sub = lane / L, sl = lane - sub * L;
      for (int base = gw * per; base < a.N; base += nw * per) {
        const int t = base + sub;
        double w = (t < a.N) ? seg_dot(a.at_cp, a.at_ri, a.at_val, a.y, t, sl, L) : 0.0;
        for (int o = L / 2; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (t < a.N && sl == 0) {
          const double di = __ldg(a.Dinv + t);
          const double xv = a.rD[t] - di * w;
          a.x[t] = xv;
          acc[CP_GT] += (FORM == 0) ? __ldg(a.c + t) * xv : __ldg(a.own + t) * (xv / di) * (xv / di);
        }
      }
    } else {
      const int L = a.xl, per = 32 / L, sub = lane / L, sl = lane - sub * L;
      const int np = (a.m + 1) / 2;  // A^T rows and y are zero padded to an even length
      for (int base = gw * per; base < a.N; base += nw * per) {
        const int t = base + sub;
        const bool ok = t < a.N;
        const double2* row = reinterpret_cast<const double2*>(a.AT + (int64_t)(ok ? t : 0) * a.ldm);
        double w0 = 0.0, w1 = 0.0;
        for (int j = sl; j < np; j += L * FU) {
          double2 av[FU], yv[FU];
#pragma unroll
          for (int q = 0; q < FU; ++q) {
            const int jj = j + L * q;
            av[q] = (ok && jj < np) ? __ldg(row + jj) : make_double2(0.0, 0.0);
            yv[q] = (ok && jj < np) ? y2[jj] : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int q = 0; q < FU; ++q) {
            w0 = fma(av[q].x, yv[q].x, w0);
            w1 = fma(av[q].y, yv[q].y, w1);
          }
        }
        double w = w0 + w1;
        for (int o = L / 2; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (ok && sl == 0) {
          const double di = __ldg(a.Dinv + t);
          const double xv = a.rD[t] - di * w;
          a.x[t] = xv;
          acc[CP_GT] += (FORM == 0) ? __ldg(a.c + t) * xv : __ldg(a.own + t) * (xv / di) * (xv / di);
        }
      }
    }
    FMARK(9);
    grid_barrier(bar, bar_target);
    FMARK(10);
    if constexpr (FORM == 0) {
      projection(std::integral_constant<int, PM_PRIMAL>{});
      FMARK(11);
      grid_barrier(bar, bar_target);
      FMARK(12);
      scatter();
    } else {
      // ---- V: v_k = z_k + lam_k/rho + H_k x, lam_k = -rho H_k x (E:vkEqn, G7)
      for (int64_t s = gt; s < a.stot; s += nt) {
        const double hx = a.x[__ldg(pa.G + s)];
        const double zv = pa.xk[s];
        const double vv = zv + pa.lam[s] / rho + hx;
        a.vk[s] = vv;
        pa.lam[s] = -rho * hx;
        const double d = zv - vv;
        acc[CP_U0] += d * d;
        acc[CP_U1] += zv * zv;
        acc[CP_U2] += vv * vv;
      }
    }
    // per-CTA partials, then the last barrier of the iteration
    block_sum_all<CP_N>(acc, sred);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int j = 0; j < CP_N; ++j) a.cpart[(int64_t)blockIdx.x * CP_N + j] = acc[j];
    }
    FMARK(13);
    grid_barrier(bar, bar_target);
    FMARK(14);
    // ---- F: every CTA, same order (reading G9; objective G17)
    {
      double v[6] = {0, 0, 0, 0, 0, 0};
      if (FORM == 0) {
        for (int q = threadIdx.x; q < a.p; q += FT) {
          v[0] += pa.part[3 * (int64_t)q];
          v[1] += pa.part[3 * (int64_t)q + 1];
          v[2] += pa.part[3 * (int64_t)q + 2];
        }
      }
      for (int c = threadIdx.x; c < (int)gridDim.x; c += FT) {
        const double* cp = a.cpart + (int64_t)c * CP_N;
        if (FORM == 1) {
          v[0] += cp[CP_U0];
          v[1] += cp[CP_U1];
          v[2] += cp[CP_U2];
        }
        v[3] += cp[CP_S0];
        v[4] += cp[CP_S1];
        v[5] += cp[CP_GT];
      }
      double by[1] = {0.0};
      if (FORM == 1)
        for (int c = threadIdx.x; c < (int)gridDim.x; c += FT) by[0] += a.cpart[(int64_t)c * CP_N + CP_BY];
      block_sum_all<6>(v, sred);
      block_sum_all<1>(by, sred + 6 * FW);
      if (threadIdx.x == 0) {
        const double eps_p = sqrt(v[0]) / fmax(fmax(sqrt(v[1]), sqrt(v[2])), 1.0);
        double eps_d, obj;
        if (FORM == 0) {
          eps_d = rho * sqrt(v[3]) / fmax(sqrt(v[4]), 1.0);
          obj = v[5];
        } else {
          eps_d = rho * sqrt(v[3]) / fmax(rho * sqrt(v[5]), 1.0);
          obj = by[0];
        }
        const long long it = it0 + i;
        const bool bad = !(isfinite(eps_p) && isfinite(eps_d) && isfinite(obj));
        const bool stop = bad || fmax(eps_p, eps_d) < *a.tol;
        s_stop = stop;
        if (blockIdx.x == 0) {
          a.res[0] = eps_p;
          a.res[1] = eps_d;
          a.res[2] = obj;
          if (it < a.hist_cap) {
            a.hist[3 * it + 0] = eps_p;
            a.hist[3 * it + 1] = eps_d;
            a.hist[3 * it + 2] = obj;
          }
          *a.iter = it + 1;
          if (bad) *a.numerical = 1;
          if (stop) *a.done = 1;
        }
      }
      __syncthreads();
      FMARK(15);
      if (s_stop) break;
    }
  }
}

}  // namespace

size_t fused_smem_bytes() { return (size_t)kGroupDoubles * sizeof(double) + kTabInts * sizeof(int); }

int fused_max_ctas(int device) {
  static int cached[64] = {};
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  const size_t sm = fused_smem_bytes();
  cudaFuncSetAttribute(k_fused_iter<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k_fused_iter<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int per = 0, per1 = 0, nsm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fused_iter<0>, FT, sm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k_fused_iter<1>, FT, sm);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  const int r = std::min(per, per1) * nsm;
  if (device >= 0 && device < 64) cached[device] = r;
  return r;
}

void launch_fused(int form, const FusedArgs& a, cudaStream_t s) {
  if (a.iters <= 0) return;
  FusedArgs args = a;
  void* params[] = {&args};
  const size_t sm = fused_smem_bytes();
  const void* fn = form == 0 ? (const void*)k_fused_iter<0> : (const void*)k_fused_iter<1>;
  SDP_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(a.nb), dim3(FT), params, sm, s));
}

}  // namespace sdp
