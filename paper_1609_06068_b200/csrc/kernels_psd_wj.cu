// Warp-register Jacobi tier of the PSD projection P_k(X) = V max(Lambda, 0) V^T
// (E:XkUpdate P:244-253, E:zkUpdate P:403-410) for 16 < k <= 32 when few
// matrices share the size range (ADMM clique blocks, e.g. 400 cliques of 30):
// the latency-optimal layout, one warp per matrix, everything in registers.
//
// Same method as the other Jacobi tiers (two-sided cyclic Jacobi, round-robin
// ordering, Golub-Van Loan sym.schur2 rotations, stop at off(A)_F <= 1e-15
// ||A||_F (G16), cap 30 sweeps, clip at exactly 0 (G15)), with the data in
// "slot order" (the round-robin permutation applied physically, so the pairs
// of every step are the slots (2i, 2i+1); the permutation is the identity at
// every sweep boundary, tests/test_slot_schedule.py):
//   * lane j holds column j of A (a[0..31]) and row j of V (v[0..31]);
//   * J^T from the left and V <- V J rotate register pairs (static indices);
//   * A <- A J mixes the columns of the lane pair (2i, 2i+1): one xor shuffle;
//   * the slot permutation is a static register move for rows / V columns and
//     one shuffle per element for the columns of A.
// Warm start (ADMM modes): A <- V_prev^T A V_prev, V = V_prev, as two DMMA
// (mma.sync m8n8k4 f64) products; the reconstruction is a third.
#include <cmath>

#include "internal.h"
#include "jacobi_rot.cuh"
#include "jacobi_warp.cuh"

namespace sdp {

namespace {

constexpr int KP = 32;
constexpr int LDS = 36;  // conflict-free DMMA fragment loads
constexpr int NWARP = 4;
constexpr int kMaxSweeps = 30;
constexpr double kJacTol = 1e-15;
constexpr double kInvSqrt2 = 0.70710678118654752440;
constexpr double kSqrt2 = 1.41421356237309504880;
constexpr unsigned FULL = 0xffffffffu;
using wj::pick;

struct WjSmem {
  double S[32 * LDS];
  double W[32 * LDS];
  double2 cs[16];
  double lam[32];
};

__device__ __forceinline__ void packed_rc(int e, int& r, int& c) {
  int cc = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while ((cc + 1) * (cc + 2) / 2 <= e) ++cc;
  while (cc * (cc + 1) / 2 > e) --cc;
  c = cc;
  r = e - cc * (cc + 1) / 2;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// acc = op(X) op(Y) for 32x32 operands in shared memory (see kernels_psd_giant.cu)
template <bool TX, bool TY>
__device__ __forceinline__ void mma32(double (&acc)[4][4][2], const double* X, const double* Y, int lane) {
  const int r4 = lane >> 2, c4 = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    double af[4], bf[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      af[t] = TX ? X[(ks * 4 + c4) * LDS + t * 8 + r4] : X[(t * 8 + r4) * LDS + ks * 4 + c4];
      bf[t] = TY ? Y[(t * 8 + r4) * LDS + ks * 4 + c4] : Y[(ks * 4 + c4) * LDS + t * 8 + r4];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
  }
}

__device__ __forceinline__ void store32(double* S, const double (&acc)[4][4][2], int lane) {
  const int r4 = lane >> 2, c4 = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      S[(i * 8 + r4) * LDS + j * 8 + 2 * c4] = acc[i][j][0];
      S[(i * 8 + r4) * LDS + j * 8 + 2 * c4 + 1] = acc[i][j][1];
    }
}

template <int MODE>
__global__ void __launch_bounds__(NWARP * 32) k_psd_wj32(ProjArgs a) {
  if (a.done && *a.done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WjSmem& sm = reinterpret_cast<WjSmem*>(smem_raw)[wid];
  const int slot = blockIdx.x * NWARP + wid;
  if (slot >= a.count) return;
  const int task = a.ids ? a.ids[slot] : slot;
  const int k = a.ksz[task];
  const int64_t off = a.off[task];
  const int ns = k * (k + 1) / 2;
  // ---- load (zero padded, mirrored; gather H_k x for the primal form)
  for (int e = lane; e < KP * KP; e += 32) sm.S[(e >> 5) * LDS + (e & 31)] = 0.0;
  __syncwarp();
  // gathers batched: every lane's loads (index, then value) are issued before any is used
  constexpr int NE = (KP * (KP + 1) / 2 + 31) / 32;  // packed entries per lane (17)
  {
    double v[NE];
    if constexpr (MODE == PM_PRIMAL) {
      int32_t gi[NE];
#pragma unroll
      for (int u = 0; u < NE; ++u) gi[u] = lane + 32 * u < ns ? __ldg(a.G + off + lane + 32 * u) : 0;
#pragma unroll
      for (int u = 0; u < NE; ++u) {
        const int e = lane + 32 * u;
        v[u] = e < ns ? __ldg(a.x + gi[u]) - a.lam[off + e] / a.rho : 0.0;
      }
    } else {
#pragma unroll
      for (int u = 0; u < NE; ++u) {
        const int e = lane + 32 * u;
        v[u] = e >= ns ? 0.0 : (MODE == PM_BATCH) ? a.in[off + e] : a.vk[off + e] - a.lam[off + e] / a.rho;
      }
    }
#pragma unroll
    for (int u = 0; u < NE; ++u) {
      const int e = lane + 32 * u;
      if (e >= ns) continue;
      int r, c;
      packed_rc(e, r, c);
      const double w = (MODE != PM_BATCH && r != c) ? v[u] * kInvSqrt2 : v[u];
      sm.S[r * LDS + c] = w;
      sm.S[c * LDS + r] = w;
    }
  }
  __syncwarp();
  double av[KP], vv[KP];
  const bool warm = (MODE != PM_BATCH) && a.vprev != nullptr && a.warm_period > 0 && (*a.iter % a.warm_period) != 0;
  if (warm) {
    // A <- V_prev^T S V_prev, V = V_prev (stored 32 x 32 row-major)
    const double* Vp = a.vprev + a.voff[task];
    for (int e = lane; e < KP * KP; e += 32) sm.W[(e >> 5) * LDS + (e & 31)] = Vp[e];
    __syncwarp();
    double acc[4][4][2];
    mma32<false, false>(acc, sm.S, sm.W, lane);  // T = S Vp
    __syncwarp();
    store32(sm.S, acc, lane);
    __syncwarp();
    mma32<true, false>(acc, sm.W, sm.S, lane);   // B = Vp^T T
    __syncwarp();
    store32(sm.S, acc, lane);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < KP; ++r) {
      av[r] = 0.5 * (sm.S[r * LDS + lane] + sm.S[lane * LDS + r]);
      vv[r] = sm.W[lane * LDS + r];
    }
  } else {
#pragma unroll
    for (int r = 0; r < KP; ++r) {
      av[r] = sm.S[r * LDS + lane];
      vv[r] = (r == lane) ? 1.0 : 0.0;
    }
  }
  double fro2 = 0.0;
#pragma unroll
  for (int r = 0; r < KP; ++r) fro2 = fma(av[r], av[r], fro2);
  fro2 = warp_sum(fro2);
  const double thr = kJacTol * kJacTol * fro2;
  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    double o2 = 0.0;  // off-diagonal part of this column (no cancellation against the diagonal)
#pragma unroll
    for (int r = 0; r < KP; ++r) o2 = (r == lane) ? o2 : fma(av[r], av[r], o2);
    o2 = warp_sum(o2);
    if (o2 <= thr) break;
#pragma unroll 1
    for (int step = 0; step < KP - 1; ++step) wj::step(av, vv, sm.cs, lane);
  }
  if (sweep == kMaxSweeps && lane == 0 && a.capped) atomicAdd(a.capped, 1ull);
  if (lane == 0 && a.sweeps) atomicAdd(a.sweeps, (unsigned long long)sweep);
  // ---- eigenvalues (slot order == natural order at the sweep boundary)
  const double lam = pick(av, lane);
  sm.lam[lane] = lam > 0.0 ? lam : 0.0;
  if (MODE != PM_BATCH && a.vprev != nullptr) {
    double* Vp = a.vprev + a.voff[task];
#pragma unroll
    for (int c = 0; c < KP; ++c) Vp[lane * KP + c] = vv[c];
  }
  __syncwarp();
  // ---- P_+ = (V diag(max(l,0))) V^T as one DMMA product
#pragma unroll
  for (int c = 0; c < KP; ++c) {
    sm.W[lane * LDS + c] = vv[c] * sm.lam[c];  // [m][k]
    sm.S[lane * LDS + c] = vv[c];              // [n][k]
  }
  __syncwarp();
  double acc[4][4][2];
  mma32<false, true>(acc, sm.W, sm.S, lane);
  __syncwarp();
  store32(sm.W, acc, lane);
  __syncwarp();
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  if constexpr (MODE == PM_PRIMAL) {
    // H_k x and lambda_k gathered up front (batched), then x_k, the multiplier update and the
    // residual partials
    double hx[NE], lv[NE];
    {
      int32_t gi[NE];
#pragma unroll
      for (int u = 0; u < NE; ++u) gi[u] = lane + 32 * u < ns ? __ldg(a.G + off + lane + 32 * u) : 0;
#pragma unroll
      for (int u = 0; u < NE; ++u) {
        const int e = lane + 32 * u;
        hx[u] = e < ns ? __ldg(a.x + gi[u]) : 0.0;
        lv[u] = e < ns ? a.lam[off + e] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < NE; ++u) {
      const int e = lane + 32 * u;
      if (e >= ns) continue;
      int r, c;
      packed_rc(e, r, c);
      const double v = sm.W[r * LDS + c];
      const double xkv = (r == c) ? v : v * kSqrt2;
      const double d = xkv - hx[u];
      a.xk[off + e] = xkv;
      a.lam[off + e] = lv[u] + a.rho * d;  // E:LambdakUpdate
      p0 += d * d;
      p1 += xkv * xkv;
      p2 += hx[u] * hx[u];
    }
  } else {
    for (int e = lane; e < ns; e += 32) {
      int r, c;
      packed_rc(e, r, c);
      const double v = sm.W[r * LDS + c];
      if constexpr (MODE == PM_BATCH)
        a.out[off + e] = v;
      else
        a.xk[off + e] = (r == c) ? v : v * kSqrt2;
    }
  }
  if constexpr (MODE == PM_PRIMAL) {
    p0 = warp_sum(p0);
    p1 = warp_sum(p1);
    p2 = warp_sum(p2);
    if (lane == 0) {
      a.part[3 * (int64_t)task + 0] = p0;
      a.part[3 * (int64_t)task + 1] = p1;
      a.part[3 * (int64_t)task + 2] = p2;
    }
  }
}

template <int MODE>
void launch_wj(const ProjArgs& a, cudaStream_t s) {
  k_psd_wj32<MODE><<<(a.count + NWARP - 1) / NWARP, NWARP * 32, NWARP * sizeof(WjSmem), s>>>(a);
}

}  // namespace

void psd_wj_init_attributes() {
  cudaFuncSetAttribute(k_psd_wj32<PM_BATCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(NWARP * sizeof(WjSmem)));
  cudaFuncSetAttribute(k_psd_wj32<PM_PRIMAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(NWARP * sizeof(WjSmem)));
  cudaFuncSetAttribute(k_psd_wj32<PM_DUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(NWARP * sizeof(WjSmem)));
}

void launch_projection_wj(int mode, const ProjArgs& a, cudaStream_t s) {
  if (a.count <= 0) return;
  if (mode == PM_BATCH)
    launch_wj<PM_BATCH>(a, s);
  else if (mode == PM_PRIMAL)
    launch_wj<PM_PRIMAL>(a, s);
  else
    launch_wj<PM_DUAL>(a, s);
}

}  // namespace sdp
