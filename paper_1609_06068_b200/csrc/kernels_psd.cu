// Batched projection onto the PSD cone, P_k(X) = V max(Lambda, 0) V^T
// (E:XkUpdate P:244-253, E:zkUpdate P:403-410), for every clique block or
// every matrix of a batch.
//
// Eigendecomposition: two-sided cyclic Jacobi with the parallel round-robin
// ("circle") ordering: every step applies kp/2 disjoint rotations at once, a
// sweep is kp-1 steps and covers every pair once.  Rotations follow Golub &
// Van Loan's sym.schur2; the sweep stops when off(A)_F <= 1e-15 ||A||_F
// (reading G16) or after 30 sweeps (counted in `capped`).  Eigenvalues
// are clipped at exactly 0 (reading G15) and the projection is rebuilt as
// sum_t max(l_t,0) v_t v_t^T.
//
// Tiers (chosen per bucket by order k and by how many matrices share it,
// see bucket assignment in api.cu): a group of G threads owns one matrix whose
// A and V live in shared memory.
//   G8 / G16 / G32 : 8 / 16 / 32 lanes per matrix, k <= 8 / 16 / 32, many matrices
//   CTA32          : 128 threads per matrix, k <= 32, few matrices (fills the GPU)
//   CTA64          : 128 threads, k <= 64;  CTA96: 256 threads, k <= 96
//   GLOBAL (giant) : block Jacobi over the whole grid, k >= SDP_GIANT_MIN (kernels_psd_giant.cu)
// Odd k is padded with one zero row/column (exact: P_+(diag(X,0)) = diag(P_+(X),0)).
#include <cmath>
#include <cstdlib>
#include <string>

#include "internal.h"
#include "jacobi_rot.cuh"

namespace sdp {

namespace {

constexpr double kInvSqrt2 = 0.70710678118654752440;
constexpr double kSqrt2 = 1.41421356237309504880;
constexpr int kMaxSweeps = 30;
constexpr double kJacTol = 1e-15;

__device__ __forceinline__ void packed_rc(int e, int& r, int& c) {
  int cc = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while ((cc + 1) * (cc + 2) / 2 <= e) ++cc;
  while (cc * (cc + 1) / 2 > e) --cc;
  c = cc;
  r = e - cc * (cc + 1) / 2;
}

template <int G>
struct Group {
  int tid;
  unsigned mask;
  double* red;  // CTA-level reduction scratch (G > 32), >= G/32 doubles
  __device__ __forceinline__ void sync() const {
    if constexpr (G <= 32)
      __syncwarp(mask);
    else
      __syncthreads();
  }
  // Deterministic sum over the group; every member receives the same value.
  __device__ __forceinline__ double sum(double v) const {
    if constexpr (G <= 32) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, G);
      return v;
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const int w = tid >> 5;
      __syncthreads();
      if ((tid & 31) == 0) red[w] = v;
      __syncthreads();
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < G / 32; ++i) s += red[i];
      return s;
    }
  }
};

struct Rot {
  int* p;
  int* q;
  double* c;
  double* s;
  double* t;
  const int* blk;  // packed (i << 16 | j), i <= j, column-major over the pair triangle; nullptr = compute
};

// 2-D strided walk over an R x C index space starting at flat index `start`
// with flat stride G, without divisions in the loop.
struct Walk {
  int r, c, dr, dc, C;
  __device__ __forceinline__ Walk(int start, int G, int Cn) : C(Cn) {
    r = start / Cn;
    c = start - r * Cn;
    dr = G / Cn;
    dc = G - dr * Cn;
  }
  __device__ __forceinline__ void next() {
    c += dc;
    r += dr;
    if (c >= C) {
      c -= C;
      ++r;
    }
  }
};

template <int G, int MODE>
__device__ void project_matrix(const Group<G>& g, const int k, const int64_t off, const int task,
                               double* __restrict__ A, double* __restrict__ V, double* __restrict__ T,
                               const int ld, Rot rot, const ProjArgs& a) {
  const int kp = k + (k & 1);
  const int P = kp >> 1;
  const int ns = k * (k + 1) / 2;
  // ---- load (gather H_k x for the primal form) ----
  for (int e = g.tid; e < ns; e += G) {
    int r, c;
    packed_rc(e, r, c);
    double v;
    if constexpr (MODE == PM_BATCH) {
      v = a.in[off + e];
    } else if constexpr (MODE == PM_PRIMAL) {
      const double hx = __ldg(a.x + a.G[off + e]);
      v = hx - a.lam[off + e] / a.rho;
      if (r != c) v *= kInvSqrt2;
    } else {
      v = a.vk[off + e] - a.lam[off + e] / a.rho;
      if (r != c) v *= kInvSqrt2;
    }
    A[r * ld + c] = v;
    A[c * ld + r] = v;
  }
  if (k & 1) {
    for (int e = g.tid; e < kp; e += G) {
      A[k * ld + e] = 0.0;
      A[e * ld + k] = 0.0;
    }
  }
  // Warm start (ADMM modes, T != nullptr): V = V_prev, A <- V_prev^T A V_prev.
  const bool warm = (MODE != PM_BATCH) && T != nullptr && a.vprev != nullptr && a.warm_period > 0 &&
                    (*a.iter % a.warm_period) != 0;
  if (warm) {
    const double* Vp = a.vprev + a.voff[task];
    {
      Walk w(g.tid, G, kp);
      for (; w.r < kp; w.next()) V[w.r * ld + w.c] = Vp[w.r * kp + w.c];
    }
    g.sync();
    {  // T = A V
      Walk w(g.tid, G, kp);
      for (; w.r < kp; w.next()) {
        const double* Ar = A + w.r * ld;
        double acc = 0.0;
        for (int t = 0; t < kp; ++t) acc = fma(Ar[t], V[t * ld + w.c], acc);
        T[w.r * ld + w.c] = acc;
      }
    }
    g.sync();
    // A = V^T T (upper triangle, mirrored)
    for (int e = g.tid; e < kp * (kp + 1) / 2; e += G) {
      int r, c;
      packed_rc(e, r, c);
      double acc = 0.0;
      for (int t = 0; t < kp; ++t) acc = fma(V[t * ld + r], T[t * ld + c], acc);
      A[r * ld + c] = acc;
      A[c * ld + r] = acc;
    }
  } else {
    Walk w(g.tid, G, kp);
    for (; w.r < kp; w.next()) V[w.r * ld + w.c] = (w.r == w.c) ? 1.0 : 0.0;
  }
  g.sync();
  double fro2 = 0.0;
  {
    Walk w(g.tid, G, kp);
    for (; w.r < kp; w.next()) {
      if (w.r <= w.c) {
        const double v = A[w.r * ld + w.c];
        fro2 += (w.r == w.c ? 1.0 : 2.0) * v * v;
      }
    }
  }
  fro2 = g.sum(fro2);
  const double thr = kJacTol * kJacTol * fro2;
  const int nblk = P * (P + 1) / 2;
  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    double off2 = 0.0;
    {
      Walk w(g.tid, G, kp);
      for (; w.r < kp; w.next()) {
        if (w.r < w.c) {
          const double v = A[w.r * ld + w.c];
          off2 += 2.0 * v * v;
        }
      }
    }
    off2 = g.sum(off2);
    if (off2 <= thr) break;
    for (int step = 0; step < kp - 1; ++step) {
      // rotation parameters of the P disjoint pairs of this step
      for (int i = g.tid; i < P; i += G) {
        int p = 0, q;
        if (i != 0) {
          p = i - 1 + step;
          p = 1 + (p >= kp - 1 ? p - (kp - 1) : p);
        }
        q = kp - 2 - i + step;
        q = 1 + (q >= kp - 1 ? q - (kp - 1) : q);
        const double app = A[p * ld + p], aqq = A[q * ld + q], apq = A[min(p, q) * ld + max(p, q)];
        const JRot jr = jacobi_rotation(app, aqq, apq);
        const double cs = jr.c, sn = jr.s, t = 0.0;
        rot.p[i] = p;
        rot.q[i] = q;
        rot.c[i] = cs;
        rot.s[i] = sn;
        rot.t[i] = t;
      }
      g.sync();
      // A <- J^T A J on the 2x2 blocks (i <= j) of the pair partition.  Only the
      // upper triangle is kept current: every entry is read and written once at
      // (min, max) of its indices.
      for (int b = g.tid; b < nblk; b += G) {
        int i, j;
        if (rot.blk) {
          const int ij = rot.blk[b];
          i = ij >> 16;
          j = ij & 0xffff;
        } else {
          packed_rc(b, i, j);
        }
        const int p1 = rot.p[i], q1 = rot.q[i];
        const double c1 = rot.c[i], s1 = rot.s[i];
        if (i == j) {
          // full J^T B J (the rotation annihilates a_pq only to ~1e-14 relative)
          const int ipq = min(p1, q1) * ld + max(p1, q1);
          const double app = A[p1 * ld + p1], aqq = A[q1 * ld + q1], apq = A[ipq];
          const double r00 = c1 * app - s1 * apq, r01 = c1 * apq - s1 * aqq;
          const double r10 = s1 * app + c1 * apq, r11 = s1 * apq + c1 * aqq;
          A[p1 * ld + p1] = c1 * r00 - s1 * r01;
          A[q1 * ld + q1] = s1 * r10 + c1 * r11;
          A[ipq] = 0.5 * ((s1 * r00 + c1 * r01) + (c1 * r10 - s1 * r11));
        } else {
          const int p2 = rot.p[j], q2 = rot.q[j];
          const double c2 = rot.c[j], s2 = rot.s[j];
          const int i00 = min(p1, p2) * ld + max(p1, p2), i01 = min(p1, q2) * ld + max(p1, q2);
          const int i10 = min(q1, p2) * ld + max(q1, p2), i11 = min(q1, q2) * ld + max(q1, q2);
          const double b00 = A[i00], b01 = A[i01], b10 = A[i10], b11 = A[i11];
          // rows: J_i^T B
          const double r00 = c1 * b00 - s1 * b10, r01 = c1 * b01 - s1 * b11;
          const double r10 = s1 * b00 + c1 * b10, r11 = s1 * b01 + c1 * b11;
          // cols: (J_i^T B) J_j
          A[i00] = c2 * r00 - s2 * r01;
          A[i01] = s2 * r00 + c2 * r01;
          A[i10] = c2 * r10 - s2 * r11;
          A[i11] = s2 * r10 + c2 * r11;
        }
      }
      // V <- V J  (row r, pair i)
      {
        Walk w(g.tid, G, P);
        for (; w.r < kp; w.next()) {
          const int p = rot.p[w.c], q = rot.q[w.c];
          const double cs = rot.c[w.c], sn = rot.s[w.c];
          double* Vr = V + w.r * ld;
          const double vp = Vr[p], vq = Vr[q];
          Vr[p] = cs * vp - sn * vq;
          Vr[q] = sn * vp + cs * vq;
        }
      }
      g.sync();
    }
  }
  if (sweep == kMaxSweeps && g.tid == 0 && a.capped) atomicAdd(a.capped, 1ull);
  if (g.tid == 0 && a.sweeps) atomicAdd(a.sweeps, (unsigned long long)sweep);
  if (MODE != PM_BATCH && T != nullptr && a.vprev != nullptr) {
    double* Vp = a.vprev + a.voff[task];
    Walk w(g.tid, G, kp);
    for (; w.r < kp; w.next()) Vp[w.r * kp + w.c] = V[w.r * ld + w.c];
  }
  // ---- reconstruction sum_t max(l_t,0) v_t v_t^T, then the mode epilogue ----
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  for (int e = g.tid; e < ns; e += G) {
    int r, c;
    packed_rc(e, r, c);
    double acc = 0.0;
    const double* Vr = V + r * ld;
    const double* Vc = V + c * ld;
    for (int t = 0; t < kp; ++t) {
      const double l = A[t * ld + t];
      if (l > 0.0) acc += l * Vr[t] * Vc[t];
    }
    if constexpr (MODE == PM_BATCH) {
      a.out[off + e] = acc;
    } else if constexpr (MODE == PM_PRIMAL) {
      // E:LambdakUpdate: lambda_k += rho (x_k - H_k x)
      const double xkv = (r == c) ? acc : acc * kSqrt2;
      const double hx = __ldg(a.x + a.G[off + e]);
      const double d = xkv - hx;
      a.xk[off + e] = xkv;
      a.lam[off + e] = a.lam[off + e] + a.rho * d;
      p0 += d * d;
      p1 += xkv * xkv;
      p2 += hx * hx;
    } else {
      a.xk[off + e] = (r == c) ? acc : acc * kSqrt2;
    }
  }
  if constexpr (MODE == PM_PRIMAL) {
    p0 = g.sum(p0);
    p1 = g.sum(p1);
    p2 = g.sum(p2);
    if (g.tid == 0) {
      a.part[3 * (int64_t)task + 0] = p0;
      a.part[3 * (int64_t)task + 1] = p1;
      a.part[3 * (int64_t)task + 2] = p2;
    }
  }
  g.sync();
}

// Pair-block table (i << 16 | j), column-major over i <= j < PMAX: the first
// P(P+1)/2 entries are exactly the blocks of a matrix with P pairs.
template <int PMAX, int NT>
__device__ __forceinline__ void fill_blk_table(int* tab) {
  for (int b = threadIdx.x; b < PMAX * (PMAX + 1) / 2; b += NT) {
    int i, j;
    packed_rc(b, i, j);
    tab[b] = (i << 16) | j;
  }
  __syncthreads();
}

// --- small tiers: G lanes per matrix, NG groups per 128-thread CTA ---------
template <int G, int KMAX, int NBUF>
struct SmallLayout {
  static constexpr int NG = 128 / G;
  static constexpr int LD = KMAX + 1;
  static constexpr int P = KMAX / 2;
  static constexpr int PER = NBUF * KMAX * LD + 4 * P;  // doubles per group
  static constexpr int NBLK = P * (P + 1) / 2;
  static constexpr size_t bytes() { return (size_t)NG * PER * sizeof(double) + NBLK * sizeof(int); }
};

template <int G, int KMAX, int MODE>
__global__ void __launch_bounds__(128) k_psd_small(ProjArgs a) {
  if (a.done && *a.done) return;
  constexpr int NBUF = MODE == PM_BATCH ? 2 : 3;
  using Lay = SmallLayout<G, KMAX, NBUF>;
  extern __shared__ double smem[];
  int* tab = (int*)(smem + Lay::NG * Lay::PER);
  fill_blk_table<Lay::P, 128>(tab);
  const int grp = threadIdx.x / G;
  const int task_slot = blockIdx.x * Lay::NG + grp;
  if (task_slot >= a.count) return;
  double* base = smem + (size_t)grp * Lay::PER;
  double* A = base;
  double* V = base + KMAX * Lay::LD;
  double* T = NBUF == 3 ? V + KMAX * Lay::LD : nullptr;
  double* rc = V + (NBUF - 1) * KMAX * Lay::LD;
  double* rs = rc + Lay::P;
  double* rt = rs + Lay::P;
  int* rpq = (int*)(rt + Lay::P);
  Rot rot{rpq, rpq + Lay::P, rc, rs, rt, tab};
  Group<G> g;
  g.tid = threadIdx.x % G;
  g.mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) / G * G));
  g.red = nullptr;
  const int task = a.ids ? a.ids[task_slot] : task_slot;
  project_matrix<G, MODE>(g, a.ksz[task], a.off[task], task, A, V, T, Lay::LD, rot, a);
}

// --- CTA tiers: one CTA per matrix, A and V in shared memory ---------------
template <int G, int KMAX, int NBUF>
struct CtaLayout {
  static constexpr int LD = KMAX + 1;
  static constexpr int P = KMAX / 2;
  static constexpr int NBLK = P * (P + 1) / 2;
  static constexpr size_t bytes() {
    return (size_t)(NBUF * KMAX * LD + 4 * P + G / 32) * sizeof(double) + NBLK * sizeof(int);
  }
};
// warm start needs a third k x k buffer; the 96-tier cannot afford it in 227 KB
template <int KMAX, int MODE>
constexpr int cta_nbuf() {
  return (MODE == PM_BATCH || KMAX > 64) ? 2 : 3;
}

template <int G, int KMAX, int MODE>
__global__ void __launch_bounds__(G) k_psd_cta(ProjArgs a) {
  if (a.done && *a.done) return;
  constexpr int NBUF = cta_nbuf<KMAX, MODE>();
  using Lay = CtaLayout<G, KMAX, NBUF>;
  extern __shared__ double smem[];
  double* A = smem;
  double* V = A + KMAX * Lay::LD;
  double* T = NBUF == 3 ? V + KMAX * Lay::LD : nullptr;
  double* rc = V + (NBUF - 1) * KMAX * Lay::LD;
  double* rs = rc + Lay::P;
  double* rt = rs + Lay::P;
  int* rpq = (int*)(rt + Lay::P);
  double* red = (double*)(rpq + 2 * Lay::P);
  int* tab = (int*)(red + G / 32);
  fill_blk_table<Lay::P, G>(tab);
  Rot rot{rpq, rpq + Lay::P, rc, rs, rt, tab};
  Group<G> g;
  g.tid = threadIdx.x;
  g.mask = 0xffffffffu;
  g.red = red;
  for (int slot = blockIdx.x; slot < a.count; slot += gridDim.x) {
    const int task = a.ids ? a.ids[slot] : slot;
    project_matrix<G, MODE>(g, a.ksz[task], a.off[task], task, A, V, T, Lay::LD, rot, a);
  }
}

template <int MODE>
void launch_mode(int bucket, const ProjArgs& a, cudaStream_t s) {
  if (a.count <= 0) return;
  switch (bucket) {
    case B_G8:
      k_psd_small<8, 8, MODE><<<(a.count + 15) / 16, 128, SmallLayout<8, 8, MODE == PM_BATCH ? 2 : 3>::bytes(), s>>>(a);
      break;
    case B_G16:
      k_psd_small<16, 16, MODE><<<(a.count + 7) / 8, 128, SmallLayout<16, 16, MODE == PM_BATCH ? 2 : 3>::bytes(), s>>>(a);
      break;
    case B_G32:
      k_psd_small<32, 32, MODE><<<(a.count + 3) / 4, 128, SmallLayout<32, 32, MODE == PM_BATCH ? 2 : 3>::bytes(), s>>>(a);
      break;
    case B_CTA32:
      k_psd_cta<128, 32, MODE><<<a.count, 128, CtaLayout<128, 32, cta_nbuf<32, MODE>()>::bytes(), s>>>(a);
      break;
    case B_CTA64:
      k_psd_cta<128, 64, MODE><<<a.count, 128, CtaLayout<128, 64, cta_nbuf<64, MODE>()>::bytes(), s>>>(a);
      break;
    case B_CTA96:
      k_psd_cta<256, 96, MODE><<<a.count, 256, CtaLayout<256, 96, cta_nbuf<96, MODE>()>::bytes(), s>>>(a);
      break;
  }
}

template <int MODE>
void init_attrs_mode() {
  cudaFuncSetAttribute(k_psd_small<16, 16, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)SmallLayout<16, 16, MODE == PM_BATCH ? 2 : 3>::bytes());
  cudaFuncSetAttribute(k_psd_small<32, 32, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)SmallLayout<32, 32, MODE == PM_BATCH ? 2 : 3>::bytes());
  cudaFuncSetAttribute(k_psd_cta<128, 32, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)CtaLayout<128, 32, cta_nbuf<32, MODE>()>::bytes());
  cudaFuncSetAttribute(k_psd_cta<128, 64, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)CtaLayout<128, 64, cta_nbuf<64, MODE>()>::bytes());
  cudaFuncSetAttribute(k_psd_cta<256, 96, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)CtaLayout<256, 96, cta_nbuf<96, MODE>()>::bytes());
}

}  // namespace

// Opt the large-shared-memory tiers into > 48 KB (per device; call before capture).
void psd_rv_init_attributes();
void psd_trd_init_attributes();
void psd_wj_init_attributes();
void psd_gtrd_init_attributes();
void psd_init_attributes() {
  psd_wj_init_attributes();
  psd_gtrd_init_attributes();
  psd_rv_init_attributes();
  psd_trd_init_attributes();
  init_attrs_mode<PM_BATCH>();
  init_attrs_mode<PM_PRIMAL>();
  init_attrs_mode<PM_DUAL>();
}

// Tier of a matrix of order k when `count` matrices fall in its size range.
// Default tiers: k <= 16 register-resident-V Jacobi (kernels_psd_rv.cu),
// 16 < k <= 64 tridiagonal-QL (kernels_psd_trd.cu).  SDP_PSD_TIERS=jacobi keeps
// Jacobi for k <= 64; SDP_PSD_TIERS=smem selects the shared-memory-V Jacobi
// tiers; SDP_PSD_TIERS=trd uses tridiagonal-QL for every 16 < k <= 64 (tests,
// comparisons).
static int tier_mode() {  // 0 default, 1 smem Jacobi, 2 Jacobi (register V), 3 QL for every 16 < k <= 64
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SDP_PSD_TIERS");
    const std::string t = e ? e : "";
    v = t == "smem" ? 1 : t == "jacobi" ? 2 : t == "trd" ? 3 : 0;
  }
  return v;
}
static int use_smem_tiers() { return tier_mode() == 1; }
// orders above this take the QL tier when there are many of them: 4 (KP = 8 and 16 QL tiers);
// SDP_TRD8=0 keeps k <= 8 on register-V Jacobi (order 8), SDP_TRD16=0 every k <= 16 (order 16)
static int trd_min_order() {
  static int v = -1;
  if (v < 0) {
    const char* e16 = getenv("SDP_TRD16");
    const char* e8 = getenv("SDP_TRD8");
    v = (e16 && e16[0] == '0') ? 16 : (e8 && e8[0] == '0') ? 8 : 4;
  }
  return v;
}

int bucket_of(int k, int64_t count_in_range) {
  if (k >= giant_min_order()) return B_GLOBAL;
  const bool few = count_in_range < kFewMatrices;
  // many mid-size matrices: tridiagonal-QL (throughput); a few (e.g. 400 cliques of
  // 30): one CTA each with warm-started Jacobi is the lower-latency choice
  if (k > trd_min_order() && k <= 64 && (tier_mode() == 3 || (tier_mode() == 0 && count_in_range >= kFewMatrices)))
    return k <= 8 ? B_TRD8 : k <= 16 ? B_TRD16 : k <= 32 ? B_TRD32 : B_TRD64;
  if (!use_smem_tiers() && k <= 64) {
    // few mid-size matrices (e.g. 400 cliques of 30): one 128-thread CTA each is
    // the lower-latency choice; otherwise the register-V tiers
    if (few && k > 16) return k <= 32 ? (tier_mode() == 0 ? B_WJ32 : B_CTA32) : B_CTA64;
    return k <= 8 ? B_RV8 : k <= 16 ? B_RV16 : k <= 32 ? B_RV32 : B_RV64;
  }
  if (k <= 8) return few ? B_CTA32 : B_G8;
  if (k <= 16) return few ? B_CTA32 : B_G16;
  if (k <= 32) return few ? B_CTA32 : B_G32;
  if (k <= 64) return B_CTA64;
  if (k <= 96) return B_CTA96;
  return B_GLOBAL;
}

int size_range(int k) { return k <= 8 ? 0 : k <= 16 ? 1 : k <= 32 ? 2 : k <= 64 ? 3 : k <= 96 ? 4 : 5; }

void launch_projection(int bucket, int mode, const ProjArgs& a, cudaStream_t s) {
  if (bucket == B_GLOBAL) {
    launch_projection_giant(mode, a, s);
    return;
  }
  if (is_trd(bucket)) {
    launch_projection_trd(bucket, mode, a, s);
    return;
  }
  if (bucket == B_WJ32) {
    launch_projection_wj(mode, a, s);
    return;
  }
  if (is_rv(bucket)) {
    launch_projection_rv(bucket, mode, a, s);
    return;
  }
  if (mode == PM_BATCH)
    launch_mode<PM_BATCH>(bucket, a, s);
  else if (mode == PM_PRIMAL)
    launch_mode<PM_PRIMAL>(bucket, a, s);
  else
    launch_mode<PM_DUAL>(bucket, a, s);
}

}  // namespace sdp
