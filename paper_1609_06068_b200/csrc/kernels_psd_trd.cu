// Tridiagonal-QL tier of the PSD projection P_k(X) = V max(Lambda, 0) V^T
// (E:XkUpdate P:244-253, E:zkUpdate P:403-410) for orders 16 < k <= 64
// (padded storage KP = 32 or 64).
//
// Jacobi executes ~4k^3 instructions per sweep and needs 6-9 sweeps from a
// cold start; this tier uses the flop-lean textbook pipeline instead:
//   1. k_trd_tridiag_reg (KP threads per matrix, row i of A in thread i's
//      registers): Householder reduction to tridiagonal form A = Q T Q^T (LAPACK
//      dsytd2, lower; Golub & Van Loan Alg. 8.3.1); k_trd_tridiag is the
//      shared-memory variant (SDP_TRD_REG=0).
//   2. k_trd_ql (lane per matrix): implicit QL with Wilkinson shifts on T
//      (Golub & Van Loan Alg. 8.3.3 / "tqli"), eigenvalues only; the sequential
//      chain of one matrix runs in one lane, so a warp advances 32 matrices at
//      once and the chain latency is hidden across matrices.  P_+ needs only the
//      eigenvectors on one side of 0, so the smaller side is selected (P_+ =
//      sum_{l>0} l v v^T, or A + sum_{l<0} |l| v v^T).
//   3. k_trd_invit (thread per cluster of selected eigenvalues): their
//      eigenvectors of T by inverse iteration (LAPACK dstein: partial-pivoting
//      tridiagonal LU, clusters of gap <= 1e-3 ||T|| reorthogonalised), O(k) per
//      vector instead of the O(k^2) rotation accumulation of QL.
//   4. k_trd_apply (KP threads per matrix): V = Q Z with the Householder vectors
//      in compact-WY blocks of 8 (DMMA), then the reconstruction (DMMA) with the
//      mode epilogue (primal: lambda_k += rho (x_k - H_k x), E:LambdakUpdate).
// Every inverse-iteration vector is checked (||T z - lambda z|| <= 1e-9 ||T||);
// if one fails, or QL hit its iteration cap (50 per eigenvalue), the matrix is redone inside the
// apply kernel by QL with eigenvector accumulation (every thread runs the same
// chain on a private copy and rotates its own row).  Eigenvalues are clipped at
// exactly 0 (G15).
#include <cmath>
#include <cstdlib>
#include <utility>

#include "internal.h"

namespace sdp {

namespace {

constexpr double kInvSqrt2 = 0.70710678118654752440;
constexpr double kSqrt2 = 1.41421356237309504880;
constexpr int kQlMaxIter = 50;
constexpr int QL_T = 32;  // threads (= matrices) per CTA of the QL kernel

__device__ __forceinline__ void packed_rc(int e, int& r, int& c) {
  int cc = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while ((cc + 1) * (cc + 2) / 2 <= e) ++cc;
  while (cc * (cc + 1) / 2 > e) --cc;
  c = cc;
  r = e - cc * (cc + 1) / 2;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
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

// per-slot workspace (doubles): d, e, tau (KP each); the selected eigenvalues
// (ascending, used as inverse-iteration shifts), their reconstruction weights
// and cluster leaders (KP each); a header {nsel, side, ||T||, -}; the packed
// Householder vectors v_j (j = 0..k-3, entries j+2..k-1; v_j[j+1] = 1 implicit)
template <int KP>
struct HView {
  double* p;
  __device__ double* d() const { return p; }
  __device__ double* e() const { return p + KP; }
  __device__ double* tau() const { return p + 2 * KP; }
  __device__ double* lsel() const { return p + 3 * KP; }
  __device__ double* lw() const { return p + 4 * KP; }
  __device__ double* clst() const { return p + 5 * KP; }
  __device__ double* hdr() const { return p + 6 * KP; }
  __device__ double* v() const { return p + 6 * KP + 4; }
};

// A group of G = KP threads (one matrix row each); G = 64 spans two warps and
// synchronises on a named barrier, G = 16 is half a warp (its own lane mask: the two halves run
// independent matrices).  Sums are fixed-order (deterministic).
template <int G>
struct Grp {
  int tid;
  int bar;      // named barrier id (G > 32)
  double* red;  // 2 doubles of scratch (G > 32)
  __device__ __forceinline__ unsigned mask() const {
    if constexpr (G >= 32)
      return 0xffffffffu;
    else
      return ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
  }
  __device__ __forceinline__ void sync() const {
    if constexpr (G < 32)
      __syncwarp(mask());
    else if constexpr (G == 32)
      __syncwarp();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G) : "memory");
  }
  __device__ __forceinline__ double sum(double v) const {
    if constexpr (G < 32) {
      const unsigned m = mask();
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o);
      return v;
    }
    v = warp_sum(v);
    if constexpr (G > 32) {  // (the leading barrier: red may still be read by the previous sum)
      sync();
      if ((tid & 31) == 0) red[tid >> 5] = v;
      sync();
      v = red[0] + red[1];
#pragma unroll
      for (int w = 2; w < G / 32; ++w) v += red[w];  // (fixed order)
    }
    return v;
  }
  // sum() for call sites that alternate between two scratch slots (red[0..1], red[2..3]): a slot
  // is rewritten only after the other slot's sum and the caller's barriers in between, so the
  // leading WAR barrier is not needed (G = 64: 2 of the 6 barriers per tridiagonalization step)
  __device__ __forceinline__ double sum_slot(double v, int slot) const {
    if constexpr (G <= 32) {
      return sum(v);
    } else {
      static_assert(G == 64, "two warps per group");
      v = warp_sum(v);
      if ((tid & 31) == 0) red[2 * slot + (tid >> 5)] = v;
      sync();
      return red[2 * slot] + red[2 * slot + 1];
    }
  }
};

// ---------------------------------------------------------------- 1. tridiagonalization
// M is the packed LOWER triangle (row r at r(r+1)/2): 17.7 KB for k = 64, so
// 12 matrices fit on an SM; row reads at r(r+1)/2 + l are bank-conflict-free
// across 32 consecutive rows, column reads l(l+1)/2 + i are consecutive.
template <int KP>
struct TridiagLayout {
  static constexpr int PER = KP * (KP + 1) / 2 + 2 * KP + 2;  // M, v, w, reduction scratch
  static constexpr int NMAT = 128 / KP;                       // matrices per 128-thread CTA
};
__device__ __forceinline__ int tri(int r) { return r * (r + 1) / 2; }

template <int KP, int MODE>
__global__ void __launch_bounds__(128) k_trd_tridiag(ProjArgs a, int slot0, int nslots) {
  if (a.done && *a.done) return;
  using Lay = TridiagLayout<KP>;
  extern __shared__ double smem[];
  const int grp = threadIdx.x / KP;
  const int sl = blockIdx.x * Lay::NMAT + grp;
  if (sl >= nslots) return;  // whole groups leave together
  double* M = smem + (size_t)grp * Lay::PER;
  double* vv = M + KP * (KP + 1) / 2;
  double* wv = vv + KP;
  Grp<KP> g{(int)(threadIdx.x % KP), 1 + grp, wv + KP};
  const int i = g.tid;  // the row this thread owns
  const int slot = slot0 + sl;
  const int task = a.ids[slot];
  const int k = a.ksz[task];
  const int64_t off = a.off[task];
  const HView<KP> H{a.td.hbuf + a.td.hoff[slot]};
  const int ns = k * (k + 1) / 2;
  for (int e = i; e < ns; e += KP) {
    int r, c;
    packed_rc(e, r, c);
    M[tri(c) + r] = input_value<MODE>(a, off + e, r, c);  // (c, r), c >= r: lower
  }
  g.sync();
  double* Mi = M + tri(i);
  int64_t vpos = 0;
  for (int j = 0; j + 2 < k; ++j) {
    // Householder vector of x = M[j+1:k, j] (dlarfg): beta = -sign(alpha) ||x||,
    // tau = (beta - alpha) / beta, v = [1; x2 / (alpha - beta)]
    const double alpha = M[tri(j + 1) + j];
    const double xi = (i >= j + 2 && i < k) ? Mi[j] : 0.0;
    const double sig = g.sum(xi * xi);
    double tau = 0.0, beta = alpha, scl = 0.0;
    if (sig > 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, sig));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scl = 1.0 / (alpha - beta);
    }
    const bool in = i >= j + 1 && i < k;
    const double vi = in ? ((i == j + 1) ? 1.0 : xi * scl) : 0.0;
    if (in) vv[i] = vi;
    if (i >= j + 2 && i < k) H.v()[vpos + (i - j - 2)] = vi;
    if (i == 0) {
      H.e()[j] = beta;
      H.tau()[j] = tau;
    }
    vpos += k - j - 2;
    g.sync();
    if (tau != 0.0) {
      // p = tau A22 v ; w = p - (tau/2)(p.v) v ; A22 -= v w^T + w v^T
      // only the lower triangle is stored: row i reads M(i, l) for l <= i and
      // M(l, i) (column i) for l > i, with l uniform across the threads
      double pi = 0.0;
      if (in) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int l = j + 1;
        for (; l + 3 < k; l += 4) {
          const double m0 = (l <= i) ? Mi[l] : M[tri(l) + i];
          const double m1 = (l + 1 <= i) ? Mi[l + 1] : M[tri(l + 1) + i];
          const double m2 = (l + 2 <= i) ? Mi[l + 2] : M[tri(l + 2) + i];
          const double m3 = (l + 3 <= i) ? Mi[l + 3] : M[tri(l + 3) + i];
          a0 = fma(m0, vv[l], a0);
          a1 = fma(m1, vv[l + 1], a1);
          a2 = fma(m2, vv[l + 2], a2);
          a3 = fma(m3, vv[l + 3], a3);
        }
        for (; l < k; ++l) a0 = fma((l <= i) ? Mi[l] : M[tri(l) + i], vv[l], a0);
        pi = tau * ((a0 + a1) + (a2 + a3));
      }
      const double K = 0.5 * tau * g.sum(pi * vi);
      const double wi = pi - K * vi;
      if (in) wv[i] = wi;
      g.sync();
      if (in) {
        int l = j + 1;
        for (; l + 3 <= i; l += 4) {
          const double u0 = fma(vi, wv[l], wi * vv[l]), u1 = fma(vi, wv[l + 1], wi * vv[l + 1]);
          const double u2 = fma(vi, wv[l + 2], wi * vv[l + 2]), u3 = fma(vi, wv[l + 3], wi * vv[l + 3]);
          Mi[l] -= u0;
          Mi[l + 1] -= u1;
          Mi[l + 2] -= u2;
          Mi[l + 3] -= u3;
        }
        for (; l <= i; ++l) Mi[l] -= fma(vi, wv[l], wi * vv[l]);
      }
      g.sync();
    }
  }
  if (i < k) H.d()[i] = Mi[i];
  if (i == 0) {
    if (k >= 2) H.e()[k - 2] = M[tri(k - 1) + k - 2];
    H.e()[k - 1] = 0.0;
  }
}

// ---- 1'. register-resident tridiagonalization (default; SDP_TRD_REG=0 selects the one above)
// Thread i holds the whole row i of A in registers (KP doubles), so the symmetric
// product A22 v and the rank-2 update read only the broadcast vectors v, w from shared
// memory (one LDS.128 per 2 columns) instead of one shared-memory element per FMA: the
// shared-memory-bound loops above become FP64-issue-bound.  Full rows cost twice the
// flops of the packed triangle (both triangles are updated), in exchange for no
// per-element shared traffic.  Register indices must be compile-time constants, so the
// column loop is split into KP/8 unrolled blocks of 8 steps (block JB works on columns
// >= 8 JB; the few columns <= j inside the block see v = w = 0 and stay unchanged).
// Same reflectors (dlarfg), same outputs (d, e, tau, packed v) as the kernel above.
template <int KP>
struct RegLayout {
  static constexpr int NMAT = 128 / KP;
  static constexpr int TRI = KP * (KP + 1) / 2;
  static constexpr int PER = ((TRI + 1) & ~1) + 3 * KP + 4;  // staging (packed), xs, vs, ws, red
};

// (HKP, JO: the slot layout and the index of local step 0 in it -- the trailing-block kernel of the
// split k = 64 reduction runs KP = 32 registers on a KP = 64 slot from step 32)
template <int KP, int JB, int G, int HKP = KP, int JO = 0>
__device__ __forceinline__ void reg_block(double (&A)[KP], int i, int k, const Grp<G>& g, double* xs, double* vs,
                                          double* ws, const HView<HKP>& H, int64_t& vpos) {
  constexpr int L0 = 8 * JB;
  constexpr int UNR = KP <= 32 ? 8 : 1;  // KP = 32: steps unrolled too (all register indices static)
#pragma unroll UNR
  for (int j = L0; j < L0 + 8; ++j) {
    if (j + 2 >= k) break;
    double xi = A[L0];  // A(i, j), j dynamic inside the block
#pragma unroll
    for (int s = 1; s < 8; ++s)
      if (j == L0 + s) xi = A[L0 + s];
    const bool below = i >= j + 2 && i < k;
    if (i == j) H.d()[JO + j] = xi;  // row j is final: d_j = A(j, j)
    double alpha;
    if constexpr (G < 32) {
      alpha = __shfl_sync(g.mask(), xi, j + 1, G);
    } else if constexpr (G == 32) {
      alpha = __shfl_sync(0xffffffffu, xi, (j + 1) & 31);
    } else {
      xs[i] = xi;  // published by the barriers inside g.sum
    }
    const double sig = g.sum_slot(below ? xi * xi : 0.0, 0);
    if constexpr (G > 32) alpha = xs[j + 1];
    double tau = 0.0, beta = alpha, scl = 0.0;
    if (sig > 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, sig));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scl = 1.0 / (alpha - beta);
    }
    const bool in = i >= j + 1 && i < k;
    const double vi = in ? ((i == j + 1) ? 1.0 : xi * scl) : 0.0;
    vs[i] = vi;
    if (below) H.v()[vpos + (i - j - 2)] = vi;
    if (i == KP - 1) {  // (row KP-1 takes part in every block)
      H.e()[JO + j] = beta;
      H.tau()[JO + j] = tau;
    }
    vpos += k - j - 2;
    g.sync();  // vs visible; every thread has read alpha
    if (tau != 0.0) {
      // p = tau A22 v ; w = p - (tau/2)(p.v) v ; A22 -= v w^T + w v^T  (rows / columns <= j: v = w = 0)
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int l = L0; l < KP; l += 4) {
        const double2 v01 = *reinterpret_cast<const double2*>(vs + l);
        const double2 v23 = *reinterpret_cast<const double2*>(vs + l + 2);
        a0 = fma(A[l], v01.x, a0);
        a1 = fma(A[l + 1], v01.y, a1);
        a2 = fma(A[l + 2], v23.x, a2);
        a3 = fma(A[l + 3], v23.y, a3);
      }
      const double pi = tau * ((a0 + a1) + (a2 + a3));
      const double K = 0.5 * tau * g.sum_slot(pi * vi, 1);
      const double wi = in ? pi - K * vi : 0.0;
      ws[i] = wi;
      g.sync();
#pragma unroll
      for (int l = L0; l < KP; l += 2) {
        const double2 w2 = *reinterpret_cast<const double2*>(ws + l);
        const double2 v2 = *reinterpret_cast<const double2*>(vs + l);
        A[l] = fma(-vi, w2.x, fma(-wi, v2.x, A[l]));  // two DFMA (no DMUL + DADD)
        A[l + 1] = fma(-vi, w2.y, fma(-wi, v2.y, A[l + 1]));
      }
      // (the next column writes vs / ws only after the barriers of its g.sum)
    }
  }
}

// KP = 64: once j >= 32 (blocks JB >= 4) rows 0..31 are final, so the first warp waits at the
// closing barrier and the second continues alone with warp-level sums and syncs
template <int KP, int JB>
__device__ __forceinline__ void reg_block_any(double (&A)[KP], int i, int k, const Grp<KP>& g, double* xs, double* vs,
                                              double* ws, const HView<KP>& H, int64_t& vpos) {
  if constexpr (KP > 32 && 8 * JB >= 32) {
    if (i >= 32) reg_block<KP, JB, 32>(A, i, k, Grp<32>{i & 31, 0, nullptr}, xs, vs, ws, H, vpos);
  } else {
    reg_block<KP, JB, KP>(A, i, k, g, xs, vs, ws, H, vpos);
  }
}

template <int KP, int HKP, int JO, int... JB>
__device__ __forceinline__ void reg_blocks(double (&A)[KP], int i, int k, const Grp<KP>& g, double* xs, double* vs,
                                           double* ws, const HView<HKP>& H, int64_t vpos,
                                           std::integer_sequence<int, JB...>) {
  if constexpr (HKP == KP && JO == 0)
    (reg_block_any<KP, JB>(A, i, k, g, xs, vs, ws, H, vpos), ...);
  else
    (reg_block<KP, JB, KP, HKP, JO>(A, i, k, g, xs, vs, ws, H, vpos), ...);
}

// Split reduction (SDP_TRD_SPLIT, default on).  Once half of a group's steps are done, the rows of
// its first half are final: in the one-kernel form their threads (KP = 64: a whole warp waiting at
// the closing barrier; KP = 32: half of the warp's lanes) keep their registers without doing work.
// So a stage with STOP runs steps 0 .. KP/2 - 1 of its block, stores the trailing block
// A(KP/2:k, KP/2:k) column-major into the slot's eigenvector scratch (free until the eigenvector
// kernel) and exits, and a stage of half the width (KP = 32: one warp per matrix; KP = 16: two
// matrices per warp) reduces the trailing block, writing d, e, tau and the Householder vectors at
// their places in the slot (the vectors of later steps follow the earlier ones in the packed order
// and their entries are relative to the step, so only the step index JO is offset).
// k = 64 bucket: 64 -> 32 -> 16 -> 8 (steps 0..31, 32..47, 48..55, 56..); k = 32: 32 -> 16 -> 8;
// k = 16: 16 -> 8.  A matrix whose
// remaining order is <= 2 at a stage boundary finishes in the stage that reaches it.
static int g_trd_split = 1;
// scratch offset (doubles) of the block a stage starting at step jo reads: 64 | 32 | 16 | 8 wide
// blocks of one slot never overlap the block the same stage writes
__host__ __device__ constexpr int split_zoff(int jo) {
  return jo == 48 ? 1024 : jo == 56 ? 1280 : jo == 24 ? 256 : 0;
}

template <int KP, int MODE, int HKP = KP, int JO = 0, bool STOP = false>
__global__ void __launch_bounds__(128, KP <= 16 ? 6 : 3) k_trd_tridiag_reg(ProjArgs a, int slot0, int nslots) {
  if (a.done && *a.done) return;
  using Lay = RegLayout<KP>;
  extern __shared__ double smem[];
  const int grp = threadIdx.x / KP;
  const int sl = blockIdx.x * Lay::NMAT + grp;
  if (sl >= nslots) return;  // whole groups leave together
  double* st = smem + (size_t)grp * Lay::PER;
  double* xs = st + ((Lay::TRI + 1) & ~1);
  double* vs = xs + KP;
  double* ws = vs + KP;
  Grp<KP> g{(int)(threadIdx.x % KP), 1 + grp, ws + KP};
  const int i = g.tid;
  const int slot = slot0 + sl;
  const int task = a.ids[slot];
  const int kf = a.ksz[task];
  if (JO > 0 && kf <= JO + 2) return;  // finished by an earlier stage (whole groups leave together)
  const int k = kf - JO;               // order of this stage's block
  const HView<HKP> H{a.td.hbuf + a.td.hoff[slot]};
  double A[KP];
  if constexpr (JO == 0) {
    const int64_t off = a.off[task];
    const int ns = k * (k + 1) / 2;
    for (int e = i; e < ns; e += KP) {
      int r, c;
      packed_rc(e, r, c);
      st[e] = input_value<MODE>(a, off + e, r, c);  // (r, c), r <= c at c(c+1)/2 + r
    }
    g.sync();
#pragma unroll
    for (int l = 0; l < KP; ++l) A[l] = (i < k && l < k) ? st[l >= i ? tri(l) + i : tri(i) + l] : 0.0;
  } else {
    const double* zb = a.td.zbuf + a.td.zoff[slot] + split_zoff(JO);
#pragma unroll
    for (int l = 0; l < KP; ++l) A[l] = (i < k && l < k) ? zb[l * KP + i] : 0.0;
  }
  const int64_t vpos0 = (int64_t)JO * (kf - 2) - (int64_t)JO * (JO - 1) / 2;  // sum_{j < JO} (kf - j - 2)
  if constexpr (STOP) {
    reg_blocks<KP, HKP, JO>(A, i, k, g, xs, vs, ws, H, vpos0, std::make_integer_sequence<int, KP / 16>{});
    if (k > KP / 2 + 2) {  // steps remain: the trailing block for the next stage
      if (i >= KP / 2) {
        double* zb = a.td.zbuf + a.td.zoff[slot] + split_zoff(JO + KP / 2);
#pragma unroll
        for (int l = KP / 2; l < KP; ++l) zb[(l - KP / 2) * (KP / 2) + (i - KP / 2)] = A[l];
      }
      return;
    }
  } else {
    reg_blocks<KP, HKP, JO>(A, i, k, g, xs, vs, ws, H, vpos0, std::make_integer_sequence<int, KP / 8>{});
  }
  // d_j (j < k - 2) was stored at step j; the last 2 x 2 block of T from rows k-2, k-1 through the
  // (free) staging area, so that no register is indexed dynamically
  static_assert(Lay::TRI >= 2 * KP, "staging holds two rows");
  g.sync();  // every thread has loaded its row from the staging area (k <= 2 runs no step barrier)
  if (k >= 2 && (i == k - 1 || i == k - 2)) {
    double* row = st + (i == k - 1 ? KP : 0);
#pragma unroll
    for (int l = 0; l < KP; ++l) row[l] = A[l];
  } else if (k == 1 && i == 0) {
#pragma unroll
    for (int l = 0; l < KP; ++l) st[l] = A[l];
  }
  g.sync();
  if (i == 0) {
    if (k >= 2) {
      H.d()[JO + k - 2] = st[k - 2];
      H.d()[JO + k - 1] = st[KP + k - 1];
      H.e()[JO + k - 2] = st[KP + k - 2];
    } else {
      H.d()[JO] = st[0];
    }
    H.e()[JO + k - 1] = 0.0;
  }
}

static int g_trd_reg = 1;    // SDP_TRD_REG=0: the shared-memory tridiagonalization
static int g_ql_rsqrt = 1;  // SDP_TRD_QLRSQ=0: QL rotations with sqrt + reciprocal
static int g_trd_invit_order = 0;  // SDP_TRD_INVIT_ORDER=1: cluster eigenvectors scheduled first
static int g_trd_fusevec = 0;  // SDP_TRD_FUSEVEC=1: singleton eigenvectors in the apply kernel (measured slower)
__constant__ int g_ql_fused = 1;  // SDP_TRD_QLFUSED=0: tql's scan loop in the QL kernel

// ---------------------------------------------------------------- 2. implicit QL
// One tqli chain on T (d, e; e[i] couples i and i+1).  T is first scaled by a
// power of two so that max |entry| is in [1, 2): then f^2 + g^2 cannot
// overflow, hypot(f, g) = q rsqrt(q) with q = f^2 + g^2, and a coupling whose
// square underflows is below 1e-300 ||T|| and is deflated (the r == 0 branch).
// `emit(i, c, s)` receives every rotation acting on columns (i, i+1) of the
// eigenvector matrix: z_i <- c z_i - s z_{i+1}, z_{i+1} <- s z_i + c z_{i+1}.
// d, e are accessed as d[i * st], e[i * st].  Returns false if an eigenvalue
// needed more than kQlMaxIter iterations.  Eigenvalues are returned unscaled.
template <bool RSQ = false, class Emit>
__device__ __forceinline__ bool tql(int k, double* d, double* e, int st, Emit&& emit) {
  double mx = 0.0;
  for (int i = 0; i < k; ++i) mx = fmax(mx, fmax(fabs(d[i * st]), fabs(e[i * st])));
  if (mx == 0.0) return true;
  const int ex = ilogb(mx);
  const double sc = scalbn(1.0, -ex), usc = scalbn(1.0, ex);
  double tn = 0.0;  // ||T||_inf of the scaled T
  for (int i = 0; i < k; ++i) {
    d[i * st] *= sc;
    e[i * st] *= sc;
  }
  for (int i = 0; i < k; ++i)
    tn = fmax(tn, fabs(d[i * st]) + fabs(e[i * st]) + (i > 0 ? fabs(e[(i - 1) * st]) : 0.0));
  // a coupling is negligible if it is below the local test of tqli OR below
  // eps ||T||: P_+ needs eigenvalues to eps ||T|| absolute accuracy, and the
  // global test stops QL from iterating on noise-level blocks of graded T (e.g.
  // the tridiagonal form of a rank-one matrix), where the local test alone can
  // exhaust the iteration cap
  const double gtol = 2.220446049250313e-16 * tn;
  bool ok = true;
  for (int l = 0; l < k; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < k - 1; ++m) {
        const double dd = fabs(d[m * st]) + fabs(d[(m + 1) * st]);
        const double em = fabs(e[m * st]);
        if (em + dd == dd || em <= gtol) break;
      }
      if (m != l) {
        if (iter++ == kQlMaxIter) {
          ok = false;
          break;
        }
        double g = (d[(l + 1) * st] - d[l * st]) / (2.0 * e[l * st]);
        double r = fabs(g) > 1e150 ? fabs(g) : sqrt(fma(g, g, 1.0));
        g = d[m * st] - d[l * st] + e[l * st] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          const double ei = e[i * st];
          const double f = s * ei, b = c * ei;
          const double q = fma(f, f, g * g);
          if (q == 0.0) {
            e[(i + 1) * st] = 0.0;
            d[(i + 1) * st] -= p;
            e[m * st] = 0.0;
            r = 0.0;
            break;
          }
          double ri;
          if constexpr (RSQ) {  // one rsqrt instead of sqrt + reciprocal (c, s within 2 ulp)
            ri = rsqrt(q);
            r = q * ri;
          } else {
            r = sqrt(q);
            ri = 1.0 / r;
          }
          e[(i + 1) * st] = r;
          s = f * ri;
          c = g * ri;
          g = d[(i + 1) * st] - p;
          r = (d[i * st] - g) * s + 2.0 * c * b;
          p = s * r;
          d[(i + 1) * st] = g + p;
          g = c * r - b;
          emit(i, c, s);
        }
        if (r == 0.0 && i >= l) continue;
        d[l * st] -= p;
        e[l * st] = g;
        e[m * st] = 0.0;
      }
    } while (m != l);
    if (!ok) break;
  }
  for (int i = 0; i < k; ++i) d[i * st] *= usc;
  return ok;
}


// tql without eigenvectors, the same shifts, rotations and deflation tests (the same eigenvalues
// up to where the compiler contracts a multiply-add), with the chain shortened for the
// one-chain-per-lane QL kernel (k = 64 bucket of cfg4: 3.28 -> 2.48 ms):
//  * no separate scan for m: after the rotation at i, d[i+1], e[i+1] and d[i+2] hold their
//    final values for this sweep, so the test of position i+1 that tql's next scan makes is
//    made there (d[i+2] carried in a register), position l when the sweep ends, and the lowest
//    negligible position found is the next m (a full scan runs only when l passes m, i.e. at
//    the start of an unreduced block, and after the q == 0 early deflation);
//  * the next rotation's operands e[i-1], d[i-1] are loaded one rotation ahead (no rotation
//    writes them), so the shared-memory latency leaves the dependent chain.
template <bool RSQ = false>
__device__ __forceinline__ bool tql_vals(int k, double* d, double* e, int st) {
  double mx = 0.0;
  for (int i = 0; i < k; ++i) mx = fmax(mx, fmax(fabs(d[i * st]), fabs(e[i * st])));
  if (mx == 0.0) return true;
  const int ex = ilogb(mx);
  const double sc = scalbn(1.0, -ex), usc = scalbn(1.0, ex);
  double tn = 0.0;
  for (int i = 0; i < k; ++i) {
    d[i * st] *= sc;
    e[i * st] *= sc;
  }
  for (int i = 0; i < k; ++i)
    tn = fmax(tn, fabs(d[i * st]) + fabs(e[i * st]) + (i > 0 ? fabs(e[(i - 1) * st]) : 0.0));
  const double gtol = 2.220446049250313e-16 * tn;
  auto negl = [gtol](double dj, double dj1, double ej) {
    const double dd = fabs(dj) + fabs(dj1), em = fabs(ej);
    return em + dd == dd || em <= gtol;
  };
  auto scan = [&](int j) {
    while (j < k - 1 && !negl(d[j * st], d[(j + 1) * st], e[j * st])) ++j;
    return j;
  };
  bool ok = true;
  int m = scan(0);
  for (int l = 0; l < k && ok; ++l) {
    if (m < l) m = scan(l);
    int iter = 0, mnext = -1;
    while (m != l) {
      if (iter++ == kQlMaxIter) {
        ok = false;
        break;
      }
      double di = d[l * st];
      const double el = e[l * st];
      double g = (d[(l + 1) * st] - di) / (2.0 * el);
      double r = fabs(g) > 1e150 ? fabs(g) : sqrt(fma(g, g, 1.0));
      g = d[m * st] - di + el / (g + copysign(r, g));
      double s = 1.0, c = 1.0, p = 0.0, dprev = 0.0;
      int i = m - 1, mlo = m;
      double ei = e[i * st], di1 = d[m * st];
      di = d[i * st];
      bool early = false;
      for (;; --i) {
        double ein = 0.0, din = 0.0;
        if (i > l) {
          ein = e[(i - 1) * st];
          din = d[(i - 1) * st];
        }
        const double f = s * ei, b = c * ei;
        const double q = fma(f, f, g * g);
        if (q == 0.0) {
          e[(i + 1) * st] = 0.0;
          d[(i + 1) * st] = di1 - p;
          e[m * st] = 0.0;
          early = true;
          break;
        }
        double ri;
        if constexpr (RSQ) {
          ri = rsqrt(q);
          r = q * ri;
        } else {
          r = sqrt(q);
          ri = 1.0 / r;
        }
        const double en = r;
        e[(i + 1) * st] = en;
        s = f * ri;
        c = g * ri;
        g = di1 - p;
        r = (di - g) * s + 2.0 * c * b;
        p = s * r;
        const double dn = g + p;
        d[(i + 1) * st] = dn;
        g = c * r - b;
        if (i + 1 < m && negl(dn, dprev, en)) mlo = i + 1;
        dprev = dn;
        if (i == l) break;
        ei = ein;
        di1 = di;
        di = din;
      }
      if (early) {  // tql's r == 0 branch: rescan from l
        m = scan(l);
        continue;
      }
      const double dl = di - p;  // i == l: di = d[l]
      d[l * st] = dl;
      e[l * st] = g;
      e[m * st] = 0.0;
      if (negl(dl, dprev, g)) {
        mnext = mlo;  // first negligible position >= l + 1
        m = l;
      } else {
        m = mlo;
      }
    }
    if (mnext >= 0) m = mnext;
  }
  for (int j = 0; j < k; ++j) d[j * st] *= usc;
  return ok;
}

template <int KP, bool RSQ = false>
__global__ void __launch_bounds__(QL_T) k_trd_ql(ProjArgs a, int slot0, int nslots) {
  if (a.done && *a.done) return;
  extern __shared__ double smem[];
  const int t = threadIdx.x;
  const int sl = blockIdx.x * QL_T + t;
  if (sl >= nslots) return;
  double* d = smem + t;  // thread-minor: element i at [i * QL_T]
  double* e = smem + KP * QL_T + t;
  const int slot = slot0 + sl;
  const int k = a.ksz[a.ids[slot]];
  const HView<KP> H{a.td.hbuf + a.td.hoff[slot]};
  double tnorm = 0.0, eprev = 0.0;  // ||T||_inf of the unscaled T
  for (int i = 0; i < k; ++i) {
    const double di = H.d()[i], ei = H.e()[i];
    d[i * QL_T] = di;
    e[i * QL_T] = ei;
    tnorm = fmax(tnorm, fabs(di) + eprev + (i + 1 < k ? fabs(ei) : 0.0));
    eprev = fabs(ei);
  }
  const bool ok = g_ql_fused ? tql_vals<RSQ>(k, d, e, QL_T) : tql<RSQ>(k, d, e, QL_T, [](int, double, double) {});
  // the side of 0 with fewer eigenvectors: P_+ = sum_{l>0} l v v^T (side 0) or
  // A + sum_{l<0} |l| v v^T (side 1); selected eigenvalues sorted ascending,
  // clusters (gap <= 1e-3 ||T||, LAPACK dstein's ORTOL) and distinct shifts
  int npos = 0, nneg = 0;
  for (int i = 0; i < k; ++i) {
    const double l = d[i * QL_T];
    npos += l > 0.0;
    nneg += l < 0.0;
  }
  const int side = npos <= nneg ? 0 : 1;
  // the selected eigenvalues are sorted in shared memory (e is free after QL; the sort in the
  // global workspace put one L2 round trip into every comparison: ~10 % of the kernel)
  double* ls = e;  // element i at [i * QL_T]
  int n = 0;
  for (int i = 0; i < k; ++i) {
    const double l = d[i * QL_T];
    if (side == 0 ? l > 0.0 : l < 0.0) {
      int j = n++ - 1;  // insertion sort, ascending
      while (j >= 0 && ls[j * QL_T] > l) {
        ls[(j + 1) * QL_T] = ls[j * QL_T];
        --j;
      }
      ls[(j + 1) * QL_T] = l;
    }
  }
  const double ortol = 1e-3 * tnorm, pertol = 10.0 * 2.220446049250313e-16 * tnorm;
  int lead = 0;
  double prev = 0.0;
  for (int i = 0; i < n; ++i) {
    double li = ls[i * QL_T];
    H.lw()[i] = side == 0 ? li : -li;
    if (i == 0 || li - prev > ortol) lead = i;
    H.clst()[i] = (double)lead;
    if (i > lead && li - prev < pertol) li = prev + pertol;
    H.lsel()[i] = li;
    prev = li;
  }
  H.hdr()[0] = (double)n;
  H.hdr()[1] = (double)side;
  H.hdr()[2] = tnorm;
  a.td.rcount[slot] = ok ? 0 : -1;
}

// ---------------------------------------------------------------- 3. eigenvectors of T
// One thread per cluster of selected eigenvalues (gap <= 1e-3 ||T||, LAPACK dstein's ORTOL).
// A singleton (the usual case) takes the twisted factorization of T - lam I (Dhillon & Parlett's
// getvec, here on T itself: lam is accurate to eps ||T|| and its gap is > 1e-3 ||T||): the
// top-down T - lam I = L+ D+ L+^T and bottom-up U- D- U-^T pivots, the twist index
// r = argmin |gamma_i|, gamma_i = D+_i - e_i^2 / D-_{i+1}, then z_r = 1,
// z_i = -(e_i / D+_i) z_{i+1} below r and z_i = -(e_{i-1} / D-_i) z_{i-1} above r, for which
// (T - lam I) z = gamma_r e_r.  That is two pivot chains and one product pass, against the LU
// chain and two forward / back substitution pairs of inverse iteration, and two per-thread
// arrays (the reciprocal pivots) instead of three, so more threads are resident.  A cluster is
// handled by inverse iteration (dstein: partial-pivoting LU of T - lam I (dlagtf; pivots below
// tol replaced by +-tol, stored inverted), kTrdInvIters = 2 solves (dlagts) from a
// deterministic pseudo-random start, each followed by modified Gram-Schmidt against the
// cluster's previous vectors and normalisation), its iterate in the output column.  Every
// vector is then checked: ||T z - lam z||_inf > 1e-9 ||T|| ||z||_inf (NaN included) marks the
// matrix (rcount = -1) and the apply kernel redoes it by QL with eigenvector accumulation.
constexpr int IV_T = 32;  // threads per CTA
constexpr int kTrdInvIters = 2;  // solves per vector (eigenvalues from QL are accurate to eps ||T||)
template <int KP>
struct InvLayout {
  static constexpr int HALF = KP / 2;        // selected eigenvalues per matrix <= k / 2
  static constexpr int NMAT = IV_T / HALF;   // matrices per CTA
  // KP = 64: the second per-thread array (reciprocal D+ pivots / LU multipliers) lives in the
  // slot's global scratch, so twice as many CTAs are resident (k = 64 bucket 2.04 -> 1.88 ms);
  // smaller orders keep it in shared memory (measured faster there)
  static constexpr bool GLOBAL2 = KP >= 64;
  static constexpr size_t bytes() { return (size_t)((GLOBAL2 ? 1 : 2) * KP * IV_T + NMAT * 2 * KP) * sizeof(double); }
};

// 1 / x to full fp64 precision: hardware approximation + two Newton steps (no IEEE-division
// slow path on the pivot chains)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double t = fma(-x, r, 1.0);
  r = fma(r, t, r);
  t = fma(-x, r, 1.0);
  return fma(r, t, r);
}

// ROLE 0: every selected eigenvector.  ROLE 1: clusters only (the apply kernel forms the singleton
// vectors itself, twisted_vec below).  ROLE 2: a grid of two halves, the first for the clusters (so
// their long inverse-iteration chains start first and overlap the rest), the second for the
// singletons (SDP_TRD_INVIT_ORDER=1; same vectors bit for bit)
template <int KP, int ROLE = 0>
__global__ void __launch_bounds__(IV_T) k_trd_invit(ProjArgs a, int slot0, int nslots) {
  if (a.done && *a.done) return;
  using Lay = InvLayout<KP>;
  constexpr int ZL = KP / 2;  // row length of the output block
  extern __shared__ double smem[];
  const int t = threadIdx.x;
  int bid = blockIdx.x;
  bool cl_role = ROLE == 1;
  if constexpr (ROLE == 2) {
    const int nb = (nslots + Lay::NMAT - 1) / Lay::NMAT;
    cl_role = bid < nb;
    if (!cl_role) bid -= nb;
  }
  const int sl = bid * Lay::NMAT + t / Lay::HALF;
  const int j0 = t % Lay::HALF;  // cluster leader this thread may own
  if (sl >= nslots) return;
  const int slot = slot0 + sl;
  const HView<KP> H{a.td.hbuf + a.td.hoff[slot]};
  const int nsel = (int)H.hdr()[0];
  const int k = a.ksz[a.ids[slot]];
  if (cl_role) {  // a warp whose matrices have no cluster has nothing to do
    const bool need = j0 + 1 < nsel && (int)H.clst()[j0] == j0 && (int)H.clst()[j0 + 1] == j0;
    if (!__any_sync(__activemask(), need)) return;
  }
  // T (d, e) into shared memory: the recurrences below read it element by element, and the
  // workspace is far larger than L2 / L1, so global reads would each pay a DRAM round trip
  double* d = smem + (Lay::GLOBAL2 ? 1 : 2) * KP * IV_T + (t / Lay::HALF) * 2 * KP;
  double* e = d + KP;
  for (int i = j0; i < k; i += Lay::HALF) {
    d[i] = H.d()[i];
    e[i] = H.e()[i];
  }
  __syncwarp(Lay::HALF == 32 ? 0xffffffffu : (((1u << Lay::HALF) - 1u) << (Lay::HALF * ((t / Lay::HALF) % (32 / Lay::HALF)))));
  if (j0 >= nsel || (int)H.clst()[j0] != j0) return;
  const double tnorm = H.hdr()[2];
  const double tol = 2.220446049250313e-16 * fmax(tnorm, 1e-300);
  double* A0 = smem + t;  // per-thread array, element i at [i * IV_T]
  double* Zo0 = a.td.zbuf + a.td.zoff[slot];
  // the second per-thread array: shared memory [i * IV_T], or the unused half of the slot's
  // scratch [i * ZL] (GLOBAL2)
  double* A1 = Lay::GLOBAL2 ? Zo0 + ZL * KP + j0 : A0 + KP * IV_T;
  constexpr int S1 = Lay::GLOBAL2 ? ZL : IV_T;
  double* Zo = a.td.zbuf + a.td.zoff[slot];  // selected eigenvectors of T, [i][j], row length KP/2
  const bool single = j0 + 1 >= nsel || (int)H.clst()[j0 + 1] != j0;
  if (ROLE != 0 && single == cl_role) return;
  bool fail = false;
  if (single) {
    const double lam = H.lsel()[j0];
    double* rm = A0;  // 1 / D-_i (shared memory)
    double* zj = Zo + j0;  // the output column (z_i)
    double* rp = Lay::GLOBAL2 ? zj : A0 + KP * IV_T;  // 1 / D+_i: the output column (z_i overwrites
    constexpr int SP = Lay::GLOBAL2 ? ZL : IV_T;       // it), or shared memory
    double dm = d[k - 1] - lam;
    if (fabs(dm) < tol) dm = dm < 0.0 ? -tol : tol;
    double rmi = rcp_nr(dm);
    rm[(k - 1) * IV_T] = rmi;
    for (int i = k - 2; i >= 1; --i) {
      const double ei = e[i];
      dm = fma(-ei * ei, rmi, d[i] - lam);
      if (fabs(dm) < tol) dm = dm < 0.0 ? -tol : tol;
      rmi = rcp_nr(dm);
      rm[i * IV_T] = rmi;
    }
    double dp = 0.0, best = 0.0, rpi = 0.0;
    int r = 0;
    for (int i = 0; i < k; ++i) {
      const double ai = d[i] - lam;
      if (i == 0) {
        dp = ai;
      } else {
        const double em = e[i - 1];
        dp = fma(-em * em, rpi, ai);
      }
      if (fabs(dp) < tol) dp = dp < 0.0 ? -tol : tol;
      rpi = rcp_nr(dp);
      rp[i * SP] = rpi;
      const double gam = i + 1 < k ? fma(-e[i] * e[i], rm[(i + 1) * IV_T], dp) : dp;
      if (i == 0 || fabs(gam) < best) {
        best = fabs(gam);
        r = i;
      }
    }
    // z is written unnormalised; its residual rows and its norm are formed on the way, and the
    // reconstruction weight takes the 1 / ||z||^2 (w z z^T / ||z||^2 = w v v^T)
    double nrm = 1.0, mx = 1.0, res = 0.0, zr_up = 0.0, zr_dn = 0.0;
    double z1 = 1.0, z2 = 0.0;  // z at the last two rows of a chain
    for (int i = r + 1; i < k; ++i) {  // above r: z_i = -(e_{i-1} / D-_i) z_{i-1}
      const double z = z1 * (-e[i - 1] * rm[i * IV_T]);
      zj[i * ZL] = z;
      if (i >= r + 2) res = fmax(res, fabs(fma(e[i - 2], z2, fma(d[i - 1] - lam, z1, e[i - 1] * z))));
      else zr_up = z;
      z2 = z1;
      z1 = z;
      nrm = fma(z, z, nrm);
      mx = fmax(mx, fabs(z));
    }
    if (r + 1 < k) res = fmax(res, fabs(fma(e[k - 2], z2, (d[k - 1] - lam) * z1)));  // row k - 1
    z1 = 1.0;
    z2 = 0.0;
    // below r: z_i = -(e_i / D+_i) z_{i+1}, the reciprocal pivots read back from the column eight
    // at a time (the loads of a block are independent of the chain)
    for (int i0 = r - 1; i0 >= 0; i0 -= 8) {
      double rpb[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) rpb[q] = i0 - q >= 0 ? rp[(i0 - q) * SP] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = i0 - q;
        if (i < 0) break;
        const double z = z1 * (-e[i] * rpb[q]);
        zj[i * ZL] = z;
        if (i <= r - 2) res = fmax(res, fabs(fma(e[i], z, fma(d[i + 1] - lam, z1, e[i + 1] * z2))));
        else zr_dn = z;
        z2 = z1;
        z1 = z;
        nrm = fma(z, z, nrm);
        mx = fmax(mx, fabs(z));
      }
    }
    if (r >= 1) res = fmax(res, fabs(fma(e[0], z2, (d[0] - lam) * z1)));  // row 0
    zj[r * ZL] = 1.0;
    res = fmax(res, fabs((d[r] - lam) + (r >= 1 ? e[r - 1] * zr_dn : 0.0) + (r + 1 < k ? e[r] * zr_up : 0.0)));
    if (!(res <= 1e-9 * fmax(tnorm, 1e-300) * mx) || !(nrm < 1e300)) fail = true;  // NaN / Inf too
    else H.lw()[j0] /= nrm;
  } else {
    double* ui = A0;  // inverse pivots
    double* mu = A1;  // multipliers
    // the first superdiagonal of U is recomputed in the back substitution: u2_i = d_{i+1} - lam
    // where row i pivoted, else the carried r1 = e_0 (i = 0), -mu_{i-1} e_i (row i-1 pivoted) or
    // e_i; the second superdiagonal is e_{i+1} where row i pivoted, else 0
    for (int j = j0; j < nsel && (int)H.clst()[j] == j0; ++j) {
      const double lam = H.lsel()[j];
      double* x = Zo + j;  // the iterate lives in its output column (row stride KP/2)
      unsigned long long pv = 0ull;  // pivot flags (k <= 64)
      double r0 = d[0] - lam, r1 = k > 1 ? e[0] : 0.0;
      for (int i = 0; i + 1 < k; ++i) {
        const double ci = e[i], ai = d[i + 1] - lam, bi = (i + 2 < k) ? e[i + 1] : 0.0;
        double p1, m;
        if (fabs(ci) > fabs(r0)) {
          pv |= 1ull << i;
          p1 = ci;
          m = r0 / ci;
          r0 = r1 - m * ai;
          r1 = -m * bi;
        } else {
          p1 = r0;
          m = r0 != 0.0 ? ci / r0 : 0.0;
          r0 = ai - m * r1;
          r1 = bi;
        }
        if (fabs(p1) < tol) p1 = p1 < 0.0 ? -tol : tol;
        ui[i * IV_T] = 1.0 / p1;
        mu[i * S1] = m;
      }
      if (fabs(r0) < tol) r0 = r0 < 0.0 ? -tol : tol;
      ui[(k - 1) * IV_T] = 1.0 / r0;
      for (int i = 0; i < k; ++i) {
        unsigned long long h = (unsigned long long)(i + 1) * 0x9E3779B97F4A7C15ull ^
                               (unsigned long long)(j + 7) * 0xD1B54A32D192ED03ull;
        h ^= h >> 31;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
        x[i * ZL] = (double)(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;
      }
      for (int it = 0; it < kTrdInvIters; ++it) {
        double ry = x[0];
        for (int i = 0; i + 1 < k; ++i) {
          const double yn = x[(i + 1) * ZL];
          const double m = mu[i * S1];
          if ((pv >> i) & 1ull) {
            x[i * ZL] = yn;
            ry = fma(-m, yn, ry);
          } else {
            x[i * ZL] = ry;
            ry = fma(-m, ry, yn);
          }
        }
        double xn = ry * ui[(k - 1) * IV_T], xn1 = 0.0;
        x[(k - 1) * ZL] = xn;
        double mx = fabs(xn);
        for (int i = k - 2; i >= 0; --i) {
          const bool piv = (pv >> i) & 1ull;
          const double u3 = piv ? e[i + 1] : 0.0;  // i + 2 < k here
          const double u2 = piv ? d[i + 1] - lam
                                : (i == 0 ? e[0] : (((pv >> (i - 1)) & 1ull) ? -mu[(i - 1) * S1] * e[i] : e[i]));
          const double xi = (x[i * ZL] - u2 * xn - u3 * xn1) * ui[i * IV_T];
          x[i * ZL] = xi;
          mx = fmax(mx, fabs(xi));
          xn1 = xn;
          xn = xi;
        }
        const double inv = mx > 0.0 ? 1.0 / mx : 1.0;
        for (int i = 0; i < k; ++i) x[i * ZL] *= inv;
        for (int p = j0; p < j; ++p) {
          const double* zp = Zo + p;  // column p of the [i][j] block
          double dot = 0.0;
          for (int i = 0; i < k; ++i) dot = fma(zp[i * ZL], x[i * ZL], dot);
          for (int i = 0; i < k; ++i) x[i * ZL] = fma(-dot, zp[i * ZL], x[i * ZL]);
        }
        double nrm = 0.0;
        for (int i = 0; i < k; ++i) nrm = fma(x[i * ZL], x[i * ZL], nrm);
        const double in2 = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
        for (int i = 0; i < k; ++i) x[i * ZL] *= in2;
      }
    }
  }
  // check every vector of the cluster against T
  for (int j = j0; !single && j < nsel && (int)H.clst()[j] == j0; ++j) {
    const double lam = H.lsel()[j];
    double* zj = Zo + j;
    double res = 0.0, mx = 0.0, zprev = 0.0, zi = zj[0];
    for (int i = 0; i < k; ++i) {
      const double znext = i + 1 < k ? zj[(i + 1) * ZL] : 0.0;
      double tz = (d[i] - lam) * zi;
      if (i > 0) tz = fma(e[i - 1], zprev, tz);
      if (i + 1 < k) tz = fma(e[i], znext, tz);
      res = fmax(res, fabs(tz));
      mx = fmax(mx, fabs(zi));
      zprev = zi;
      zi = znext;
    }
    if (!(res <= 1e-9 * fmax(tnorm, 1e-300) * mx)) fail = true;  // includes NaN / Inf
  }
  if (fail) a.td.rcount[slot] = -1;
}

// ---------------------------------------------------------------- 4. back-transform, P_+
// Z holds at most KP/2 columns (the selected side has <= k/2 eigenvectors);
// row stride KP/2 + 4 == 4 (mod 16) keeps the DMMA fragment loads conflict-free.
// The back-transform applies the reflectors in blocks of 8 (compact WY, LAPACK dlarft /
// dlarfb): H_j0 ... H_j0+7 = I - Y T Y^T, Z <- Z - Y (T (Y^T Z)), all three products as
// DMMA (mma.sync m8n8k4 f64) on 8 x 8 tiles; each warp owns 8-column tiles of Z, so only
// the Y / T block is shared (2 CTA barriers per block instead of 3 per reflector).
template <int KP>
struct ApplyLayout {
  static constexpr int AT = KP < 32 ? 32 : KP;  // threads (a full warp for the DMMA fragments; 2 KP measured: no gain)
  static constexpr int LD = KP / 2 + 4;
  static constexpr int YLD = 12;  // Y block row stride (8 reflectors + pad)
  static constexpr int NW = AT / 32;
  // ... + d, e of T and the per-column cluster flags (fused eigenvector stage)
  static constexpr size_t bytes() {
    return (size_t)(KP * LD + AT * YLD + 128 + NW * 128 + KP + 12 + 3 * KP) * sizeof(double);
  }
};

// The singleton eigenvector of k_trd_invit (same twisted factorization, same operations in the
// same order, so the vector and its weight are bit-identical) formed in the apply kernel's shared
// Z column zc (row stride LDZ), so Z never goes through DRAM.  No per-thread pivot arrays: the
// bottom-up reciprocal pivots 1 / D-_i go into the column, the twist index r is found by a first
// top-down pass, and a second top-down pass up to r overwrites rows 0..r-1 with 1 / D+_i (rows
// below r need only D+, rows above r only D-).  Returns false where k_trd_invit sets rcount = -1.
template <int LDZ>
__device__ bool twisted_vec(int k, const double* d, const double* e, double lam, double tnorm, double* zc,
                            double& nrm_out) {
  const double tol = 2.220446049250313e-16 * fmax(tnorm, 1e-300);
  double dm = d[k - 1] - lam;
  if (fabs(dm) < tol) dm = dm < 0.0 ? -tol : tol;
  double rmi = rcp_nr(dm);
  zc[(k - 1) * LDZ] = rmi;
  for (int i = k - 2; i >= 1; --i) {
    const double ei = e[i];
    dm = fma(-ei * ei, rmi, d[i] - lam);
    if (fabs(dm) < tol) dm = dm < 0.0 ? -tol : tol;
    rmi = rcp_nr(dm);
    zc[i * LDZ] = rmi;
  }
  double dp = 0.0, best = 0.0, rpi = 0.0;
  int r = 0;
  for (int i = 0; i < k; ++i) {
    const double ai = d[i] - lam;
    if (i == 0) {
      dp = ai;
    } else {
      const double em = e[i - 1];
      dp = fma(-em * em, rpi, ai);
    }
    if (fabs(dp) < tol) dp = dp < 0.0 ? -tol : tol;
    rpi = rcp_nr(dp);
    const double gam = i + 1 < k ? fma(-e[i] * e[i], zc[(i + 1) * LDZ], dp) : dp;
    if (i == 0 || fabs(gam) < best) {
      best = fabs(gam);
      r = i;
    }
  }
  rpi = 0.0;
  for (int i = 0; i < r; ++i) {  // 1 / D+_i below the twist (the same recurrence again)
    const double ai = d[i] - lam;
    if (i == 0) {
      dp = ai;
    } else {
      const double em = e[i - 1];
      dp = fma(-em * em, rpi, ai);
    }
    if (fabs(dp) < tol) dp = dp < 0.0 ? -tol : tol;
    rpi = rcp_nr(dp);
    zc[i * LDZ] = rpi;
  }
  double nrm = 1.0, mx = 1.0, res = 0.0, zr_up = 0.0, zr_dn = 0.0;
  double z1 = 1.0, z2 = 0.0;
  for (int i = r + 1; i < k; ++i) {  // above r: z_i = -(e_{i-1} / D-_i) z_{i-1}
    const double z = z1 * (-e[i - 1] * zc[i * LDZ]);
    zc[i * LDZ] = z;
    if (i >= r + 2) res = fmax(res, fabs(fma(e[i - 2], z2, fma(d[i - 1] - lam, z1, e[i - 1] * z))));
    else zr_up = z;
    z2 = z1;
    z1 = z;
    nrm = fma(z, z, nrm);
    mx = fmax(mx, fabs(z));
  }
  if (r + 1 < k) res = fmax(res, fabs(fma(e[k - 2], z2, (d[k - 1] - lam) * z1)));
  z1 = 1.0;
  z2 = 0.0;
  for (int i = r - 1; i >= 0; --i) {  // below r: z_i = -(e_i / D+_i) z_{i+1}
    const double z = z1 * (-e[i] * zc[i * LDZ]);
    zc[i * LDZ] = z;
    if (i <= r - 2) res = fmax(res, fabs(fma(e[i], z, fma(d[i + 1] - lam, z1, e[i + 1] * z2))));
    else zr_dn = z;
    z2 = z1;
    z1 = z;
    nrm = fma(z, z, nrm);
    mx = fmax(mx, fabs(z));
  }
  if (r >= 1) res = fmax(res, fabs(fma(e[0], z2, (d[0] - lam) * z1)));
  zc[r * LDZ] = 1.0;
  res = fmax(res, fabs((d[r] - lam) + (r >= 1 ? e[r - 1] * zr_dn : 0.0) + (r + 1 < k ? e[r] * zr_up : 0.0)));
  nrm_out = nrm;
  return (res <= 1e-9 * fmax(tnorm, 1e-300) * mx) && (nrm < 1e300);
}

__device__ __forceinline__ void dmma8(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <int KP, int MODE, bool FV = false>
__global__ void __launch_bounds__(ApplyLayout<KP>::AT) k_trd_apply(ProjArgs a, int slot0, int nslots) {
  if (a.done && *a.done) return;
  using Lay = ApplyLayout<KP>;
  constexpr int LD = Lay::LD;
  extern __shared__ double smem[];
  const int sl = blockIdx.x;
  if (sl >= nslots) return;
  constexpr int YLD = Lay::YLD, NW = Lay::NW, AT = Lay::AT;
  double* Z = smem;  // selected eigenvectors (columns), then back-transformed
  double* Ys = Z + KP * LD;     // Y block [row][8]
  double* Gs = Ys + AT * YLD;   // Y^T Y (8 x 8)
  double* Ts = Gs + 64;         // T (8 x 8, upper)
  double* Wsm = Ts + 64;        // per warp: W = Y^T Z tile, then T W
  double* lw = Wsm + NW * 128;
  double* red = lw + KP;
  Grp<AT> g{(int)threadIdx.x, 1, red};
  const int tid = g.tid;
  const int slot = slot0 + sl;
  const int task = a.ids[slot];
  const int k = a.ksz[task];
  const int64_t off = a.off[task];
  const HView<KP> H{a.td.hbuf + a.td.hoff[slot]};
  int nsel = (int)H.hdr()[0];
  int side = (int)H.hdr()[1];
  bool fallback = a.td.rcount[slot] < 0 || a.td.force_fallback;
  for (int e = tid; e < KP * LD; e += AT) Z[e] = 0.0;  // rows >= k, columns >= nsel stay 0 (DMMA tiles)
  if constexpr (FV) {
    // fused eigenvector stage: thread j forms singleton vector j in Z's column j; cluster columns
    // (k_trd_invit<KP, 1>) are read from the workspace
    double* dsm = red + 12;
    double* esm = dsm + KP;
    double* cfl = esm + KP;
    if (!fallback) {
      for (int i = tid; i < k; i += AT) {
        dsm[i] = H.d()[i];
        esm[i] = H.e()[i];
      }
      if (tid < nsel) {
        const bool single = (int)H.clst()[tid] == tid && (tid + 1 >= nsel || (int)H.clst()[tid + 1] != tid);
        cfl[tid] = single ? 0.0 : 1.0;
        lw[tid] = H.lw()[tid];
      }
    }
    g.sync();
    bool fail = false;
    if (!fallback) {
      const double* Zo = a.td.zbuf + a.td.zoff[slot];
      for (int e = tid; e < k * (KP / 2); e += AT) {
        const int i = e / (KP / 2), j = e - i * (KP / 2);
        if (j < nsel && cfl[j] != 0.0) Z[i * LD + j] = Zo[e];
      }
      if (tid < nsel && cfl[tid] == 0.0) {
        double nrm;
        if (twisted_vec<LD>(k, dsm, esm, H.lsel()[tid], H.hdr()[2], Z + tid, nrm)) lw[tid] /= nrm;
        else fail = true;
      }
    }
    if (__syncthreads_or(fail) && !fallback) {
      fallback = true;
      for (int e = tid; e < KP * LD; e += AT) Z[e] = 0.0;
    }
  }
  g.sync();
  if (!FV && !fallback) {
    const double* Zo = a.td.zbuf + a.td.zoff[slot];  // [i][j], row length KP/2
    for (int e = tid; e < k * (KP / 2); e += AT) {
      const int i = e / (KP / 2), j = e - i * (KP / 2);
      if (j < nsel) Z[i * LD + j] = Zo[e];
    }
    if (tid < nsel) lw[tid] = H.lw()[tid];
  }
  if (fallback) {
    // QL with eigenvectors in the slot's global scratch (KP x KP), every thread
    // running the same chain on a private copy of (d, e) (identical arithmetic,
    // identical rotations) and rotating its own row; then the side of 0 with
    // fewer eigenvectors, in index order, into the shared Z
    const int row = tid;
    double* Zg = a.td.zbuf + a.td.zoff[slot];
    double* Zr = Zg + (size_t)row * KP;
    if (row < KP)
      for (int j = 0; j < KP; ++j) Zr[j] = (j == row) ? 1.0 : 0.0;
    double dl[KP], el[KP];
    for (int i = 0; i < k; ++i) {
      dl[i] = H.d()[i];
      el[i] = H.e()[i];
    }
    const bool ok = tql(k, dl, el, 1, [&](int i, double c, double s) {
      if (row < k) {
        const double zi = Zr[i], zi1 = Zr[i + 1];
        Zr[i + 1] = fma(s, zi, c * zi1);
        Zr[i] = fma(c, zi, -s * zi1);
      }
    });
    if (!ok && row == 0 && a.capped) atomicAdd(a.capped, 1ull);
    int npos = 0, nneg = 0;
    for (int t = 0; t < k; ++t) {
      npos += dl[t] > 0.0;
      nneg += dl[t] < 0.0;
    }
    side = npos <= nneg ? 0 : 1;
    int n = 0;
    for (int t = 0; t < k; ++t) {
      if (side == 0 ? dl[t] > 0.0 : dl[t] < 0.0) {
        if (row < k) Z[row * LD + n] = Zr[t];
        if (row == 0) lw[n] = side == 0 ? dl[t] : -dl[t];
        ++n;
      }
    }
    nsel = n;
  }
  g.sync();
  if (a.td.debug && slot == 0 && tid == 0) {
    printf("[trd] k=%d fallback=%d nsel=%d side=%d tnorm=%.3e rcount=%d\n", k, (int)fallback, nsel, side,
           H.hdr()[2], a.td.rcount[slot]);
    for (int i = 0; i < k; ++i) printf("  d[%d]=% .6e e=% .6e tau=% .6e\n", i, H.d()[i], H.e()[i], H.tau()[i]);
    for (int j = 0; j < nsel; ++j) printf("  sel %d: shift=% .6e w=% .6e clst=%d\n", j, H.lsel()[j], lw[j], (int)H.clst()[j]);
  }
  // back-transform the selected eigenvectors: V = H_0 H_1 ... H_{k-3} Z, blocks of 8 reflectors
  // from the last; reflector j (j <= k-3) has v_j = e_{j+1} + packed entries j+2 .. k-1
  {
    const int lane = tid & 31, warp = tid >> 5, r4 = lane >> 2, c4 = lane & 3;
    const int nref = k - 2;
    const int ntile = (nsel + 7) / 8;
    double* Wt = Wsm + warp * 128;
    double* taus = red + 4;  // tau of the block's reflectors
    // the next block's Y row (thread = row) and tau are fetched into registers while the current
    // block is applied (the reflectors come from DRAM)
    double ypre[8], tpre = 0.0;
    auto fetch = [&](int j0) {
      const int i = tid;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int j = j0 + c;
        double y = 0.0;
        if (j < nref) {
          if (i == j + 1)
            y = 1.0;
          else if (i >= j + 2 && i < k)
            y = H.v()[(int64_t)j * (k - 2) - (int64_t)j * (j - 1) / 2 + (i - j - 2)];
        }
        ypre[c] = y;
      }
      if (tid < 8) tpre = (j0 + tid < nref) ? H.tau()[j0 + tid] : 0.0;
    };
    const int jlast = nref > 0 ? ((nref - 1) / 8) * 8 : -1;
    if (jlast >= 0) fetch(jlast);
    for (int j0 = jlast; j0 >= 0; j0 -= 8) {
#pragma unroll
      for (int c = 0; c < 8; ++c) Ys[tid * YLD + c] = ypre[c];
      if (tid < 8) taus[tid] = tpre;
      if (j0 >= 8) fetch(j0 - 8);
      g.sync();
      const int kb = (j0 + 1) & ~3;  // first row (multiple of 4) where the block is nonzero
      if (warp == 0) {
        double gacc[2] = {0.0, 0.0}, gacc2[2] = {0.0, 0.0};  // G = Y^T Y (two accumulator chains)
        int k0 = kb;
        for (; k0 + 4 < k; k0 += 8) {
          const double y = Ys[(k0 + c4) * YLD + r4], y2 = Ys[(k0 + 4 + c4) * YLD + r4];
          dmma8(gacc, y, y);
          dmma8(gacc2, y2, y2);
        }
        if (k0 < k) {
          const double y = Ys[(k0 + c4) * YLD + r4];
          dmma8(gacc, y, y);
        }
        gacc[0] += gacc2[0];
        gacc[1] += gacc2[1];
        Gs[r4 * 8 + 2 * c4] = gacc[0];
        Gs[r4 * 8 + 2 * c4 + 1] = gacc[1];
        __syncwarp();
        if (lane < 8) {
          // row r = lane of T (dlarft, forward columnwise): T_rc = tau_c (r = c),
          // -tau_c sum_{q<c} T_rq G_qc (r < c), 0 (r > c)
          double trow[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const double tc = taus[c];
            double sacc = 0.0;
#pragma unroll
            for (int q = 0; q < c; ++q) sacc = fma(trow[q], Gs[q * 8 + c], sacc);
            trow[c] = lane < c ? -tc * sacc : (lane == c ? tc : 0.0);
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) Ts[lane * 8 + c] = trow[c];
        }
      }
      g.sync();
      for (int nt = warp; nt < ntile; nt += NW) {
        const int n0 = 8 * nt;
        double w[2] = {0.0, 0.0}, wb[2] = {0.0, 0.0};  // W = Y^T Z (8 reflectors x 8 columns), two chains
        int k0 = kb;
        for (; k0 + 4 < k; k0 += 8) {
          dmma8(w, Ys[(k0 + c4) * YLD + r4], Z[(k0 + c4) * LD + n0 + r4]);
          dmma8(wb, Ys[(k0 + 4 + c4) * YLD + r4], Z[(k0 + 4 + c4) * LD + n0 + r4]);
        }
        if (k0 < k) dmma8(w, Ys[(k0 + c4) * YLD + r4], Z[(k0 + c4) * LD + n0 + r4]);
        w[0] += wb[0];
        w[1] += wb[1];
        Wt[r4 * 8 + 2 * c4] = w[0];
        Wt[r4 * 8 + 2 * c4 + 1] = w[1];
        __syncwarp();
        double w2[2] = {0.0, 0.0};  // T W
#pragma unroll
        for (int kk = 0; kk < 8; kk += 4) dmma8(w2, Ts[r4 * 8 + kk + c4], Wt[(kk + c4) * 8 + r4]);
        Wt[64 + r4 * 8 + 2 * c4] = w2[0];
        Wt[64 + r4 * 8 + 2 * c4 + 1] = w2[1];
        __syncwarp();
        for (int m0 = ((j0 + 1) / 8) * 8; m0 < k; m0 += 8) {  // Z -= Y (T W)
          double* zr = Z + (m0 + r4) * LD + n0 + 2 * c4;
          double z[2] = {zr[0], zr[1]};
#pragma unroll
          for (int kk = 0; kk < 8; kk += 4) dmma8(z, -Ys[(m0 + r4) * YLD + kk + c4], Wt[64 + (kk + c4) * 8 + r4]);
          zr[0] = z[0];
          zr[1] = z[1];
        }
        __syncwarp();
      }
      g.sync();  // Y / T are rewritten by the next block
    }
  }
  // P_+ = [A] + sum_t w_t v_t v_t^T as DMMA (mma.sync m8n8k4 f64) 8x8 tiles over the
  // upper tile triangle, K = nsel; then the packed upper entries with the mode epilogue
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  {
    const int lane = tid & 31, warp = tid >> 5;
    const int r4 = lane >> 2, c4 = lane & 3;
    const int nt = (k + 7) / 8;
    const int ntile = nt * (nt + 1) / 2;
    for (int tl = warp; tl < ntile; tl += NW) {
      int rt, ct;
      packed_rc(tl, rt, ct);
      // the epilogue's global operands are loaded before the K loop (their latency then overlaps it)
      double pin[2] = {0.0, 0.0}, phx[2] = {0.0, 0.0}, plam[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * rt + r4, c = 8 * ct + 2 * c4 + h;
        if (r > c || c >= k) continue;
        const int64_t pe = off + (int64_t)c * (c + 1) / 2 + r;
        if (side == 1) pin[h] = input_value<MODE>(a, pe, r, c);
        if constexpr (MODE == PM_PRIMAL) {
          phx[h] = __ldg(a.x + a.G[pe]);
          plam[h] = a.lam[pe];
        }
      }
      double acc[2] = {0.0, 0.0};
      for (int u0 = 0; u0 < nsel; u0 += 4) {
        const int u = u0 + c4;
        const bool ok = u < nsel;
        const double a = ok ? lw[u] * Z[(8 * rt + r4) * LD + u] : 0.0;
        const double b = ok ? Z[(8 * ct + r4) * LD + u] : 0.0;
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
            : "+d"(acc[0]), "+d"(acc[1])
            : "d"(a), "d"(b));
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * rt + r4, c = 8 * ct + 2 * c4 + h;
        if (r > c || c >= k) continue;
        double v = acc[h];
        const int64_t pe = off + (int64_t)c * (c + 1) / 2 + r;
        if (side == 1) v += pin[h];
        if constexpr (MODE == PM_BATCH) {
          a.out[pe] = v;
        } else if constexpr (MODE == PM_PRIMAL) {
          const double xkv = (r == c) ? v : v * kSqrt2;
          const double hx = phx[h];
          const double dd = xkv - hx;
          a.xk[pe] = xkv;
          a.lam[pe] = plam[h] + a.rho * dd;  // E:LambdakUpdate
          p0 += dd * dd;
          p1 += xkv * xkv;
          p2 += hx * hx;
        } else {
          a.xk[pe] = (r == c) ? v : v * kSqrt2;
        }
      }
    }
  }
  if constexpr (MODE == PM_PRIMAL) {
    p0 = g.sum(p0);
    p1 = g.sum(p1);
    p2 = g.sum(p2);
    if (tid == 0) {
      a.part[3 * (int64_t)task + 0] = p0;
      a.part[3 * (int64_t)task + 1] = p1;
      a.part[3 * (int64_t)task + 2] = p2;
    }
  }
}

template <int KP, int MODE>
void launch_chunk(const ProjArgs& a, int c0, int n, cudaStream_t s) {
  using TL = TridiagLayout<KP>;
  using IL = InvLayout<KP>;
  using RL = RegLayout<KP>;
  bool split = false;
  if (KP >= 16 && g_trd_reg && g_trd_split) {
    using R32 = RegLayout<32>;
    using R16 = RegLayout<16>;
    using R8 = RegLayout<8>;
    if constexpr (KP >= 16)
      k_trd_tridiag_reg<KP, MODE, KP, 0, true>
          <<<(n + RL::NMAT - 1) / RL::NMAT, 128, RL::NMAT * RL::PER * sizeof(double), s>>>(a, c0, n);
    if constexpr (KP == 64)
      k_trd_tridiag_reg<32, PM_BATCH, 64, 32, true>
          <<<(n + R32::NMAT - 1) / R32::NMAT, 128, R32::NMAT * R32::PER * sizeof(double), s>>>(a, c0, n);
    if constexpr (KP >= 32)
      k_trd_tridiag_reg<16, PM_BATCH, KP, KP - 16, true>
          <<<(n + R16::NMAT - 1) / R16::NMAT, 128, R16::NMAT * R16::PER * sizeof(double), s>>>(a, c0, n);
    if constexpr (KP >= 16)
      k_trd_tridiag_reg<8, PM_BATCH, KP, KP - 8, false>
          <<<(n + R8::NMAT - 1) / R8::NMAT, 128, R8::NMAT * R8::PER * sizeof(double), s>>>(a, c0, n);
    split = true;
  }
  if (split) {
  } else if (g_trd_reg)
    k_trd_tridiag_reg<KP, MODE><<<(n + RL::NMAT - 1) / RL::NMAT, 128, RL::NMAT * RL::PER * sizeof(double), s>>>(a, c0, n);
  else
    k_trd_tridiag<KP, MODE><<<(n + TL::NMAT - 1) / TL::NMAT, 128, TL::NMAT * TL::PER * sizeof(double), s>>>(a, c0, n);
  if (g_ql_rsqrt)
    k_trd_ql<KP, true><<<(n + QL_T - 1) / QL_T, QL_T, 2 * KP * QL_T * sizeof(double), s>>>(a, c0, n);
  else
    k_trd_ql<KP><<<(n + QL_T - 1) / QL_T, QL_T, 2 * KP * QL_T * sizeof(double), s>>>(a, c0, n);
  if (g_trd_fusevec) {
    k_trd_invit<KP, 1><<<(n + IL::NMAT - 1) / IL::NMAT, IV_T, IL::bytes(), s>>>(a, c0, n);
    k_trd_apply<KP, MODE, true><<<n, ApplyLayout<KP>::AT, ApplyLayout<KP>::bytes(), s>>>(a, c0, n);
  } else {
    if (g_trd_invit_order)
      k_trd_invit<KP, 2><<<2 * ((n + IL::NMAT - 1) / IL::NMAT), IV_T, IL::bytes(), s>>>(a, c0, n);
    else
      k_trd_invit<KP><<<(n + IL::NMAT - 1) / IL::NMAT, IV_T, IL::bytes(), s>>>(a, c0, n);
    k_trd_apply<KP, MODE><<<n, ApplyLayout<KP>::AT, ApplyLayout<KP>::bytes(), s>>>(a, c0, n);
  }
}

template <int KP, int MODE>
void set_attrs() {
  using TL = TridiagLayout<KP>;
  cudaFuncSetAttribute(k_trd_tridiag<KP, MODE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_trd_tridiag_reg<KP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(RegLayout<KP>::NMAT * RegLayout<KP>::PER * sizeof(double)));
  if constexpr (KP >= 16)
    cudaFuncSetAttribute(k_trd_tridiag_reg<KP, MODE, KP, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(RegLayout<KP>::NMAT * RegLayout<KP>::PER * sizeof(double)));
  if constexpr (KP == 64)
    cudaFuncSetAttribute(k_trd_tridiag_reg<32, PM_BATCH, 64, 32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(RegLayout<32>::NMAT * RegLayout<32>::PER * sizeof(double)));
  if constexpr (KP >= 32)
    cudaFuncSetAttribute(k_trd_tridiag_reg<16, PM_BATCH, KP, KP - 16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(RegLayout<16>::NMAT * RegLayout<16>::PER * sizeof(double)));
  if constexpr (KP >= 16)
    cudaFuncSetAttribute(k_trd_tridiag_reg<8, PM_BATCH, KP, KP - 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(RegLayout<8>::NMAT * RegLayout<8>::PER * sizeof(double)));

  cudaFuncSetAttribute(k_trd_ql<KP>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_trd_invit<KP>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_trd_apply<KP, MODE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_trd_tridiag<KP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(TL::NMAT * TL::PER * sizeof(double)));
  cudaFuncSetAttribute(k_trd_ql<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * KP * QL_T * sizeof(double)));
  cudaFuncSetAttribute(k_trd_ql<KP, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_trd_ql<KP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * KP * QL_T * sizeof(double)));
  cudaFuncSetAttribute(k_trd_invit<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)InvLayout<KP>::bytes());
  cudaFuncSetAttribute(k_trd_apply<KP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)ApplyLayout<KP>::bytes());
  cudaFuncSetAttribute(k_trd_invit<KP, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_trd_invit<KP, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)InvLayout<KP>::bytes());
  cudaFuncSetAttribute(k_trd_invit<KP, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_trd_invit<KP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)InvLayout<KP>::bytes());
  cudaFuncSetAttribute(k_trd_apply<KP, MODE, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_trd_apply<KP, MODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)ApplyLayout<KP>::bytes());
}

}  // namespace

void psd_trd_init_attributes() {
  const char* ev = std::getenv("SDP_TRD_REG");
  g_trd_reg = (ev && ev[0] == '0') ? 0 : 1;
  const char* eq = std::getenv("SDP_TRD_QLRSQ");
  g_ql_rsqrt = (eq && eq[0] == '0') ? 0 : 1;
  const char* eio = std::getenv("SDP_TRD_INVIT_ORDER");
  g_trd_invit_order = (eio && eio[0] == '1') ? 1 : 0;
  const char* efv = std::getenv("SDP_TRD_FUSEVEC");
  g_trd_fusevec = (efv && efv[0] == '1') ? 1 : 0;
  const char* esp = std::getenv("SDP_TRD_SPLIT");
  g_trd_split = (esp && esp[0] == '0') ? 0 : 1;
  const char* eqf = std::getenv("SDP_TRD_QLFUSED");
  const int qf = (eqf && eqf[0] == '0') ? 0 : 1;
  cudaMemcpyToSymbol(g_ql_fused, &qf, sizeof(int));
  set_attrs<8, PM_BATCH>();
  set_attrs<8, PM_PRIMAL>();
  set_attrs<8, PM_DUAL>();
  set_attrs<16, PM_BATCH>();
  set_attrs<16, PM_PRIMAL>();
  set_attrs<16, PM_DUAL>();
  set_attrs<32, PM_BATCH>();
  set_attrs<32, PM_PRIMAL>();
  set_attrs<32, PM_DUAL>();
  set_attrs<64, PM_BATCH>();
  set_attrs<64, PM_PRIMAL>();
  set_attrs<64, PM_DUAL>();
}

int trd_launches_per_chunk(int bucket) {
  if (!(g_trd_reg && g_trd_split)) return 4;
  return bucket == B_TRD64 ? 7 : bucket == B_TRD32 ? 6 : bucket == B_TRD16 ? 5 : 4;
}

int64_t trd_hsize(int kp, int k) {
  const int64_t v = k >= 2 ? (int64_t)(k - 1) * (k - 2) / 2 : 0;
  return (6 * (int64_t)kp + 4 + v + 1) & ~(int64_t)1;
}

void launch_projection_trd(int bucket, int mode, const ProjArgs& a, cudaStream_t s) {
  const int count = a.td.count;
  if (count <= 0) return;
  for (int c0 = 0; c0 < count; c0 += a.td.chunk) {
    const int n = std::min(a.td.chunk, count - c0);
    if (bucket == B_TRD8) {
      if (mode == PM_BATCH) launch_chunk<8, PM_BATCH>(a, c0, n, s);
      else if (mode == PM_PRIMAL) launch_chunk<8, PM_PRIMAL>(a, c0, n, s);
      else launch_chunk<8, PM_DUAL>(a, c0, n, s);
    } else if (bucket == B_TRD16) {
      if (mode == PM_BATCH) launch_chunk<16, PM_BATCH>(a, c0, n, s);
      else if (mode == PM_PRIMAL) launch_chunk<16, PM_PRIMAL>(a, c0, n, s);
      else launch_chunk<16, PM_DUAL>(a, c0, n, s);
    } else if (bucket == B_TRD32) {
      if (mode == PM_BATCH) launch_chunk<32, PM_BATCH>(a, c0, n, s);
      else if (mode == PM_PRIMAL) launch_chunk<32, PM_PRIMAL>(a, c0, n, s);
      else launch_chunk<32, PM_DUAL>(a, c0, n, s);
    } else {
      if (mode == PM_BATCH) launch_chunk<64, PM_BATCH>(a, c0, n, s);
      else if (mode == PM_PRIMAL) launch_chunk<64, PM_PRIMAL>(a, c0, n, s);
      else launch_chunk<64, PM_DUAL>(a, c0, n, s);
    }
  }
}

}  // namespace sdp
