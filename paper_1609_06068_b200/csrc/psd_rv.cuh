// Register-resident-V Jacobi projection of one packed symmetric matrix by a
// group of G = KP * Q threads (device code shared by the register-V tier,
// kernels_psd_rv.cu, and the fused small-problem iteration, kernels_fused.cu).
// See kernels_psd_rv.cu for the method.  COH = true reads the global iterate x
// with coherent loads (x is written earlier in the same kernel by the fused
// iteration, so the read-only path may not be used).
#pragma once
#include <cmath>

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

// Circle-method slot rotation: slot 2i <-> position i, slot 2i+1 <-> position KP-1-i;
// positions 1..KP-1 advance by one each step, position 0 is fixed.
template <int KP>
__host__ __device__ constexpr int next_slot(int s) {
  return s == 0 ? 0 : (s & 1) ? (s == 1 ? 2 : s - 2) : (s == KP - 2 ? KP - 1 : s + 2);
}

template <int G>
struct RvGroup {
  int tid;
  unsigned mask;
  int bar;  // named barrier id (G > 32)
  double* red;
  __device__ __forceinline__ void sync() const {
    if constexpr (G <= 32)
      __syncwarp(mask);
    else
      asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G) : "memory");
  }
  __device__ __forceinline__ double sum(double v) const {
    if constexpr (G <= 32) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, G);
      return v;
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      sync();
      if ((tid & 31) == 0) red[tid >> 5] = v;
      sync();
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < G / 32; ++i) s += red[i];
      return s;
    }
  }
};

template <int KP, int Q>
struct RvLayout {
  static constexpr int G = KP * Q;   // threads per matrix
  static constexpr int S = KP / Q;   // V slots per lane
  static_assert(S >= 4, "each lane must hold at least 4 slots");
  static constexpr int LD = KP + 2;  // even: 16-byte aligned row pairs
  static constexpr int P = KP / 2;
  static constexpr int NBLK = P * (P + 1) / 2;
  template <int NBUF>
  static constexpr int per_group() {
    return NBUF * KP * LD + 3 * P + (G / 32 > 2 ? G / 32 : 2);
  }
  static constexpr int groups_per_cta() { return G < 128 ? 128 / G : 1; }
  static constexpr int threads() { return G < 128 ? 128 : G; }
  template <int NBUF>
  static constexpr size_t bytes() {
    return (size_t)groups_per_cta() * per_group<NBUF>() * sizeof(double) + NBLK * sizeof(int);
  }
};

template <int MODE>
constexpr int rv_nbuf() {
  return MODE == PM_BATCH ? 2 : 3;
}

template <int KP, int Q, int MODE, bool COH = false>
__device__ void project_rv(const RvGroup<KP * Q>& g, const int k, const int64_t off, const int task, double* Ac,
                           double* An, double* T, double* rc, double* rs, double* rt, const int* __restrict__ tab,
                           const ProjArgs& a) {
  using Lay = RvLayout<KP, Q>;
  constexpr int G = Lay::G;
  constexpr int S = Lay::S;
  constexpr int LD = Lay::LD;
  constexpr int P = Lay::P;
  const int ns = k * (k + 1) / 2;
  const int r = g.tid / Q;           // V row owned by this lane group
  const int q = g.tid - r * Q;       // part: slots [q*S, q*S + S)
  const unsigned qmask = Q == 1 ? 0u : (((1u << Q) - 1u) << ((threadIdx.x & 31) / Q * Q));
  // diagnostics: clock64 per phase of the first group of CTA 0 (slots: calls, load, warm start,
  // sweep loop, steps, sweeps, reconstruction + epilogue)
  long long* rtr = (a.rvtrace && blockIdx.x == 0 && threadIdx.x == 0) ? a.rvtrace : nullptr;
  long long rt0 = rtr ? clock64() : 0;
  // ---- load: zero padding, then the packed entries (gather H_k x)
  for (int e = g.tid; e < KP * KP; e += G) {
    const int rr = e / KP, cc = e - rr * KP;
    if (rr >= k || cc >= k) Ac[rr * LD + cc] = 0.0;
  }
  for (int e = g.tid; e < ns; e += G) {
    int rr, cc;
    packed_rc(e, rr, cc);
    double v;
    if constexpr (MODE == PM_BATCH) {
      v = a.in[off + e];
    } else if constexpr (MODE == PM_PRIMAL) {
      const double hx = COH ? a.x[a.G[off + e]] : __ldg(a.x + a.G[off + e]);
      v = hx - a.lam[off + e] / a.rho;
      if (rr != cc) v *= kInvSqrt2;
    } else {
      v = a.vk[off + e] - a.lam[off + e] / a.rho;
      if (rr != cc) v *= kInvSqrt2;
    }
    Ac[rr * LD + cc] = v;
    Ac[cc * LD + rr] = v;
  }
  if (rtr) {
    const long long now = clock64();
    rtr[0] += 1;
    rtr[1] += now - rt0;
    rt0 = now;
  }
  double v[S];
  const bool warm = (MODE != PM_BATCH) && T != nullptr && a.vprev != nullptr && a.warm_period > 0 &&
                    (*a.iter % a.warm_period) != 0;
  if (warm) {
    // A <- V_prev^T A V_prev (V_prev stored KP x KP row-major), V = V_prev
    const double* Vp = a.vprev + a.voff[task];
    for (int e = g.tid; e < KP * KP; e += G) An[(e / KP) * LD + (e % KP)] = Vp[e];
    g.sync();
    for (int e = g.tid; e < KP * KP; e += G) {
      const int rr = e / KP, cc = e - rr * KP;
      double acc = 0.0;
      for (int t = 0; t < KP; ++t) acc = fma(Ac[rr * LD + t], An[t * LD + cc], acc);
      T[rr * LD + cc] = acc;
    }
    g.sync();
    for (int e = g.tid; e < KP * (KP + 1) / 2; e += G) {
      int rr, cc;
      packed_rc(e, rr, cc);
      double acc = 0.0;
      for (int t = 0; t < KP; ++t) acc = fma(An[t * LD + rr], T[t * LD + cc], acc);
      Ac[rr * LD + cc] = acc;
      Ac[cc * LD + rr] = acc;
    }
#pragma unroll
    for (int c = 0; c < S; ++c) v[c] = An[r * LD + q * S + c];
  } else {
#pragma unroll
    for (int c = 0; c < S; ++c) v[c] = (q * S + c == r) ? 1.0 : 0.0;
  }
  g.sync();
  double fro2 = 0.0;
  for (int e = g.tid; e < KP * KP; e += G) {
    const int rr = e / KP, cc = e - rr * KP;
    if (rr <= cc) {
      const double x = Ac[rr * LD + cc];
      fro2 += (rr == cc ? 1.0 : 2.0) * x * x;
    }
  }
  fro2 = g.sum(fro2);
  if (rtr) {
    const long long now = clock64();
    rtr[2] += now - rt0;
    rt0 = now;
  }
  const double thr = kJacTol * kJacTol * fro2;
  // this thread's 2x2 blocks of the pair triangle (the same in every step: the slot permutation is
  // applied physically), with their source and destination offsets: A_next = (J^T A J) permuted by
  // ns(), upper triangle only; every block (i <= j, row-major over the pair triangle so that a
  // warp's lanes touch consecutive columns) writes each entry once, at (min, max) of its slots
  constexpr int NBU = (Lay::NBLK + G - 1) / G;
  int b_src[NBU], b_i[NBU], b_j[NBU], b_d[NBU][4];
#pragma unroll
  for (int u = 0; u < NBU; ++u) {
    const int b = g.tid + u * G;
    b_src[u] = -1;
    b_i[u] = b_j[u] = 0;
    b_d[u][0] = b_d[u][1] = b_d[u][2] = b_d[u][3] = 0;
    if (b < Lay::NBLK) {
      const int ij = tab[b];
      const int i = ij >> 16, j = ij & 0xffff;
      const int pi = next_slot<KP>(2 * i), qi = next_slot<KP>(2 * i + 1);
      b_src[u] = 2 * i * LD + 2 * j;
      b_i[u] = i;
      b_j[u] = j;
      if (i == j) {
        b_d[u][0] = pi * LD + pi;
        b_d[u][1] = qi * LD + qi;
        b_d[u][2] = min(pi, qi) * LD + max(pi, qi);
      } else {
        const int pj = next_slot<KP>(2 * j), qj = next_slot<KP>(2 * j + 1);
        b_d[u][0] = min(pi, pj) * LD + max(pi, pj);
        b_d[u][1] = min(pi, qj) * LD + max(pi, qj);
        b_d[u][2] = min(qi, pj) * LD + max(qi, pj);
        b_d[u][3] = min(qi, qj) * LD + max(qi, qj);
      }
    }
  }
  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    double off2 = 0.0;
    for (int e = g.tid; e < KP * KP; e += G) {
      const int rr = e / KP, cc = e - rr * KP;
      if (rr < cc) {
        const double x = Ac[rr * LD + cc];
        off2 += 2.0 * x * x;
      }
    }
    off2 = g.sum(off2);
    if (off2 <= thr) break;
#pragma unroll 1
    for (int step = 0; step < KP - 1; ++step) {
      // rotation of pair i = slots (2i, 2i+1) (Golub-Van Loan sym.schur2)
      for (int i = g.tid; i < P; i += G) {
        const double app = Ac[2 * i * LD + 2 * i], aqq = Ac[(2 * i + 1) * LD + 2 * i + 1];
        const double apq = Ac[2 * i * LD + 2 * i + 1];
        const JRot jr = jacobi_rotation(app, aqq, apq);
        rc[i] = jr.c;
        rs[i] = jr.s;
      }
      g.sync();
      // V <- V J in registers (this lane's S/2 pairs), then the slot permutation:
      // even slots move +2, odd slots -2; one element crosses to each neighbour lane
#pragma unroll
      for (int l = 0; l < S; l += 2) {
        const int i = (q * S + l) >> 1;
        const double cs = rc[i], sn = rs[i];
        const double vp = v[l], vq = v[l + 1];
        v[l] = cs * vp - sn * vq;
        v[l + 1] = sn * vp + cs * vq;
      }
      {
        double from_down = 0.0, from_up = 0.0;
        if constexpr (Q > 1) {
          from_down = __shfl_up_sync(qmask, v[S - 2], 1, Q);
          from_up = __shfl_down_sync(qmask, v[1], 1, Q);
        }
        double nv[S];
#pragma unroll
        for (int l = 0; l + 2 < S; l += 2) nv[l + 2] = v[l];       // even slots +2
#pragma unroll
        for (int l = 3; l < S; l += 2) nv[l - 2] = v[l];           // odd slots -2
        nv[0] = from_down;
        nv[S - 1] = from_up;
        if (q == 0) {        // slot 0 fixed, slot 1 -> 2
          nv[0] = v[0];
          nv[2] = v[1];
        }
        if (q == Q - 1) nv[S - 1] = v[S - 2];  // slot KP-2 -> KP-1
#pragma unroll
        for (int l = 0; l < S; ++l) v[l] = nv[l];
      }
#pragma unroll
      for (int u = 0; u < NBU; ++u) {
        if (b_src[u] < 0) continue;
        const int i = b_i[u], j = b_j[u];
        const double2 top = *reinterpret_cast<const double2*>(Ac + b_src[u]);
        const double2 bot = *reinterpret_cast<const double2*>(Ac + b_src[u] + LD);
        const double c1 = rc[i], s1 = rs[i];
        if (i == j) {
          // full J^T B J (the rotation annihilates a_pq only to ~1e-14 relative)
          const double app = top.x, apq = top.y, aqq = bot.y;
          const double r00 = c1 * app - s1 * apq, r01 = c1 * apq - s1 * aqq;
          const double r10 = s1 * app + c1 * apq, r11 = s1 * apq + c1 * aqq;
          const double n01 = 0.5 * ((s1 * r00 + c1 * r01) + (c1 * r10 - s1 * r11));
          An[b_d[u][0]] = c1 * r00 - s1 * r01;
          An[b_d[u][1]] = s1 * r10 + c1 * r11;
          An[b_d[u][2]] = n01;
        } else {
          const double c2 = rc[j], s2 = rs[j];
          const double r00 = c1 * top.x - s1 * bot.x, r01 = c1 * top.y - s1 * bot.y;
          const double r10 = s1 * top.x + c1 * bot.x, r11 = s1 * top.y + c1 * bot.y;
          An[b_d[u][0]] = c2 * r00 - s2 * r01;
          An[b_d[u][1]] = s2 * r00 + c2 * r01;
          An[b_d[u][2]] = c2 * r10 - s2 * r11;
          An[b_d[u][3]] = s2 * r10 + c2 * r11;
        }
      }
      g.sync();
      double* tmp = Ac;
      Ac = An;
      An = tmp;
    }
  }
  if (rtr) {
    const long long now = clock64();
    rtr[3] += now - rt0;
    rtr[4] += (long long)sweep * (KP - 1);
    rtr[5] += sweep;
    rt0 = now;
  }
  if (sweep == kMaxSweeps && g.tid == 0 && a.capped) atomicAdd(a.capped, 1ull);
  if (g.tid == 0 && a.sweeps) atomicAdd(a.sweeps, (unsigned long long)sweep);
  // sweep boundary: slot order == natural order.  V rows -> shared memory (An).
#pragma unroll
  for (int c = 0; c < S; ++c) An[r * LD + q * S + c] = v[c];
  if (MODE != PM_BATCH && T != nullptr && a.vprev != nullptr) {
    double* Vp = a.vprev + a.voff[task];
#pragma unroll
    for (int c = 0; c < S; ++c) Vp[r * KP + q * S + c] = v[c];
  }
  g.sync();
  // ---- reconstruction sum_t max(l_t,0) v_t v_t^T, then the mode epilogue ----
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  for (int e = g.tid; e < ns; e += G) {
    int rr, cc;
    packed_rc(e, rr, cc);
    double acc = 0.0;
    const double* Vr = An + rr * LD;
    const double* Vc = An + cc * LD;
#pragma unroll 4
    for (int t = 0; t < KP; ++t) {
      const double l = Ac[t * LD + t];
      if (l > 0.0) acc += l * Vr[t] * Vc[t];
    }
    if constexpr (MODE == PM_BATCH) {
      a.out[off + e] = acc;
    } else if constexpr (MODE == PM_PRIMAL) {
      const double xkv = (rr == cc) ? acc : acc * kSqrt2;
      const double hx = COH ? a.x[a.G[off + e]] : __ldg(a.x + a.G[off + e]);
      const double d = xkv - hx;
      a.xk[off + e] = xkv;
      a.lam[off + e] = a.lam[off + e] + a.rho * d;  // E:LambdakUpdate
      p0 += d * d;
      p1 += xkv * xkv;
      p2 += hx * hx;
    } else {
      a.xk[off + e] = (rr == cc) ? acc : acc * kSqrt2;
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
  if (rtr) rtr[6] += clock64() - rt0;
}

}  // namespace

}  // namespace sdp
