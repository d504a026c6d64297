// Tridiagonal-QL tier of the PSD projection P_k(X) = V max(Lambda, 0) V^T
// (E:XkUpdate P:244-253, E:zkUpdate P:403-410) for orders 16 < k <= 64
// (padded storage KP = 32 or 64).
//
// Jacobi executes ~4k^3 instructions per sweep and needs 6-9 sweeps from a
// cold start; this tier uses the flop-lean textbook pipeline instead:
//   1. k_trd_tridiag (KP threads per matrix, one row each): Householder
//      reduction to tridiagonal form A = Q T Q^T (LAPACK dsytd2, lower; Golub &
//      Van Loan Alg. 8.3.1), ~4/3 k^3 flops, matrix in shared memory.
//   2. k_trd_ql (lane per matrix): implicit QL with Wilkinson shifts on T
//      (Golub & Van Loan Alg. 8.3.3 / "tqli"), eigenvalues plus the list of
//      Givens rotations; the sequential rotation chain of one matrix runs in
//      one lane, so a warp advances 32 matrices at once and the chain latency
//      is hidden across matrices.
//   3. k_trd_apply (KP threads per matrix): replays the rotations on Z = I
//      (threads own rows, the rotation pair is thread-local, and inside one QL
//      sweep the descending pairs keep z_i in a register), back-transforms
//      V = Q Z with the Householder vectors (threads own columns; only
//      eigenvectors with lambda > 0 are formed), and rebuilds
//      P_+ = sum_{lambda_t > 0} lambda_t v_t v_t^T with the mode epilogue
//      (primal: lambda_k += rho (x_k - H_k x), E:LambdakUpdate).
// If a matrix needs more QL rotations than its list holds (or > 30 iterations
// for one eigenvalue), step 2 marks it and step 3 recomputes its QL inline
// (every thread runs the same chain on a private copy and rotates its row
// directly): same arithmetic, same result.  Eigenvalues are clipped at exactly 0 (G15).
#include <cmath>
#include <cstdlib>

#include "internal.h"

namespace sdp {

namespace {

constexpr double kInvSqrt2 = 0.70710678118654752440;
constexpr double kSqrt2 = 1.41421356237309504880;
constexpr int kQlMaxIter = 30;
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

// per-slot Householder workspace: d, e, tau, lambda (KP each), packed v_j (j = 0..k-3,
// entries j+2..k-1; v_j[j+1] = 1 implicit)
template <int KP>
struct HView {
  double* p;
  __device__ double* d() const { return p; }
  __device__ double* e() const { return p + KP; }
  __device__ double* tau() const { return p + 2 * KP; }
  __device__ double* lam() const { return p + 3 * KP; }
  __device__ double* v() const { return p + 4 * KP; }
};

// A group of G = KP threads (one matrix row each); G = 64 spans two warps and
// synchronises on a named barrier.  Sums are fixed-order (deterministic).
template <int G>
struct Grp {
  int tid;
  int bar;      // named barrier id (G > 32)
  double* red;  // 2 doubles of scratch (G > 32)
  __device__ __forceinline__ void sync() const {
    if constexpr (G <= 32)
      __syncwarp();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G) : "memory");
  }
  __device__ __forceinline__ double sum(double v) const {
    v = warp_sum(v);
    if constexpr (G > 32) {
      sync();
      if ((tid & 31) == 0) red[tid >> 5] = v;
      sync();
      v = red[0] + red[1];
    }
    return v;
  }
};

// ---------------------------------------------------------------- 1. tridiagonalization
template <int KP>
struct TridiagLayout {
  static constexpr int LD = KP + 1;
  static constexpr int PER = KP * LD + 2 * KP + 2;  // M, v, w, reduction scratch
  static constexpr int NMAT = 128 / KP;              // matrices per 128-thread CTA
};

template <int KP, int MODE>
__global__ void __launch_bounds__(128) k_trd_tridiag(ProjArgs a, int slot0, int nslots) {
  if (a.done && *a.done) return;
  using Lay = TridiagLayout<KP>;
  constexpr int LD = Lay::LD;
  extern __shared__ double smem[];
  const int grp = threadIdx.x / KP;
  const int sl = blockIdx.x * Lay::NMAT + grp;
  if (sl >= nslots) return;  // whole groups leave together
  double* M = smem + (size_t)grp * Lay::PER;
  double* vv = M + KP * LD;
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
    const double v = input_value<MODE>(a, off + e, r, c);
    M[r * LD + c] = v;
    M[c * LD + r] = v;
  }
  g.sync();
  double* Mi = M + i * LD;
  int64_t vpos = 0;
  for (int j = 0; j + 2 < k; ++j) {
    // Householder vector of x = M[j+1:k, j] (dlarfg): beta = -sign(alpha) ||x||,
    // tau = (beta - alpha) / beta, v = [1; x2 / (alpha - beta)]
    const double alpha = M[(j + 1) * LD + j];
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
      double pi = 0.0;
      if (in) {
        double a0 = 0.0, a1 = 0.0;
        int l = j + 1;
        for (; l + 1 < k; l += 2) {
          a0 = fma(Mi[l], vv[l], a0);
          a1 = fma(Mi[l + 1], vv[l + 1], a1);
        }
        if (l < k) a0 = fma(Mi[l], vv[l], a0);
        pi = tau * (a0 + a1);
      }
      const double K = 0.5 * tau * g.sum(pi * vi);
      const double wi = pi - K * vi;
      if (in) wv[i] = wi;
      g.sync();
      if (in)
        for (int l = j + 1; l < k; ++l) Mi[l] -= fma(vi, wv[l], wi * vv[l]);
      g.sync();
    }
  }
  if (i < k) H.d()[i] = Mi[i];
  if (i == 0) {
    if (k >= 2) H.e()[k - 2] = M[(k - 1) * LD + k - 2];
    H.e()[k - 1] = 0.0;
  }
}

// ---------------------------------------------------------------- 2. implicit QL
// One tqli chain on T (d, e; e[i] couples i and i+1).  T is first scaled by a
// power of two so that max |entry| is in [1, 2): then f^2 + g^2 cannot
// overflow, hypot(f, g) = q rsqrt(q) with q = f^2 + g^2, and a coupling whose
// square underflows is below 1e-300 ||T|| and is deflated (the r == 0 branch).
// `emit(i, c, s)` receives every rotation acting on columns (i, i+1) of the
// eigenvector matrix: z_i <- c z_i - s z_{i+1}, z_{i+1} <- s z_i + c z_{i+1}.
// d, e are accessed as d[i * st], e[i * st].  Returns false if an eigenvalue
// needed more than kQlMaxIter iterations.  Eigenvalues are returned unscaled.
template <class Emit>
__device__ __forceinline__ bool tql(int k, double* d, double* e, int st, Emit&& emit) {
  double mx = 0.0;
  for (int i = 0; i < k; ++i) mx = fmax(mx, fmax(fabs(d[i * st]), fabs(e[i * st])));
  if (mx == 0.0) return true;
  const int ex = ilogb(mx);
  const double sc = scalbn(1.0, -ex), usc = scalbn(1.0, ex);
  for (int i = 0; i < k; ++i) {
    d[i * st] *= sc;
    e[i * st] *= sc;
  }
  bool ok = true;
  for (int l = 0; l < k; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < k - 1; ++m) {
        const double dd = fabs(d[m * st]) + fabs(d[(m + 1) * st]);
        if (fabs(e[m * st]) + dd == dd) break;
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
          r = sqrt(q);
          const double ri = 1.0 / r;
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

template <int KP>
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
  for (int i = 0; i < k; ++i) {
    d[i * QL_T] = H.d()[i];
    e[i * QL_T] = H.e()[i];
  }
  double2* rot = a.td.rot + a.td.roff[slot];
  int16_t* ridx = a.td.ridx + a.td.roff[slot];
  const int64_t cap = a.td.rcap[slot];
  int64_t n = 0;
  const bool ok = tql(k, d, e, QL_T, [&](int i, double c, double s) {
    if (n < cap) {
      rot[n] = make_double2(c, s);
      ridx[n] = (int16_t)i;
    }
    ++n;
  });
  for (int i = 0; i < k; ++i) H.lam()[i] = d[i * QL_T];
  a.td.rcount[slot] = (ok && n <= cap) ? (int32_t)n : -1;
}

// ---------------------------------------------------------------- 3. rotations, back-transform, P_+
template <int KP>
struct ApplyLayout {
  static constexpr int LD = KP + 1;
  static constexpr int NR = 64;  // rotations staged per round
  static constexpr size_t bytes() {
    return (size_t)(KP * LD + 4 * KP + 2 + 2 * NR) * sizeof(double) + (KP + NR) * sizeof(int);
  }
};

template <int KP, int MODE>
__global__ void __launch_bounds__(KP) k_trd_apply(ProjArgs a, int slot0, int nslots) {
  if (a.done && *a.done) return;
  using Lay = ApplyLayout<KP>;
  constexpr int LD = Lay::LD;
  constexpr int NR = Lay::NR;
  extern __shared__ double smem[];
  const int sl = blockIdx.x;
  if (sl >= nslots) return;
  double* Z = smem;
  double* vv = Z + KP * LD;
  double* lp = vv + KP;
  double* dsm = lp + KP;
  double* esm = dsm + KP;
  double* red = esm + KP;
  double2* rsm = reinterpret_cast<double2*>(red + 2);
  int* pidx = reinterpret_cast<int*>(rsm + NR);
  int* ism = pidx + KP;
  Grp<KP> g{(int)threadIdx.x, 1, red};
  const int row = g.tid;
  const int slot = slot0 + sl;
  const int task = a.ids[slot];
  const int k = a.ksz[task];
  const int64_t off = a.off[task];
  const HView<KP> H{a.td.hbuf + a.td.hoff[slot]};
  double* Zr = Z + row * LD;
  for (int j = 0; j < KP; ++j) Zr[j] = (j == row) ? 1.0 : 0.0;
  const int nrot = a.td.rcount[slot];
  if (nrot >= 0) {
    // replay the QL rotations on this row; inside one QL sweep the pairs descend
    // (i+1, i+2), (i, i+1), ..., so z_i stays in a register ("carry")
    const double2* rot = a.td.rot + a.td.roff[slot];
    const int16_t* ridx = a.td.ridx + a.td.roff[slot];
    double carry = 0.0;
    int cur = -2;  // column held in `carry`
    for (int t0 = 0; t0 < nrot; t0 += NR) {
      const int nt = min(NR, nrot - t0);
      g.sync();
      for (int u = row; u < nt; u += KP) {
        rsm[u] = rot[t0 + u];
        ism[u] = ridx[t0 + u];
      }
      g.sync();
      if (row < k) {
        for (int u = 0; u < nt; ++u) {
          const double2 cs = rsm[u];
          const int i = ism[u];
          double zi1;
          if (i + 1 == cur) {
            zi1 = carry;
          } else {
            if (cur >= 0) Zr[cur] = carry;
            zi1 = Zr[i + 1];
          }
          const double zi = Zr[i];
          Zr[i + 1] = fma(cs.y, zi, cs.x * zi1);
          carry = fma(cs.x, zi, -cs.y * zi1);
          cur = i;
        }
      }
    }
    if (row < k && cur >= 0) Zr[cur] = carry;
    if (row < k) dsm[row] = H.lam()[row];
  } else {
    // fallback: the QL chain inline; every thread runs the same chain on a
    // private copy of (d, e) (identical arithmetic, so identical rotations) and
    // rotates its own row
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
    if (row < k) dsm[row] = dl[row];
    if (!ok && row == 0 && a.capped) atomicAdd(a.capped, 1ull);
  }
  g.sync();
  // positive eigenvalues, compacted in index order (deterministic)
  int npos = 0;
  for (int t0 = 0; t0 < k; t0 += 32) {
    const int t = t0 + (row & 31);
    const double l = t < k ? dsm[t] : 0.0;
    const bool pos = l > 0.0;
    const unsigned bal = __ballot_sync(0xffffffffu, pos);
    if (row < 32 && pos) {
      const int at = npos + __popc(bal & ((1u << row) - 1u));
      pidx[at] = t;
      lp[at] = l;
    }
    npos += __popc(bal);
  }
  g.sync();
  // back-transform the positive eigenvectors: V = H_0 H_1 ... H_{k-3} Z
  int64_t vpos = k >= 2 ? (int64_t)(k - 1) * (k - 2) / 2 : 0;
  for (int j = k - 3; j >= 0; --j) {
    vpos -= k - j - 2;
    const double tau = H.tau()[j];
    if (tau == 0.0) continue;
    if (row >= j + 1 && row < k) vv[row] = (row == j + 1) ? 1.0 : H.v()[vpos + (row - j - 2)];
    g.sync();
    for (int u = row; u < npos; u += KP) {
      const int c = pidx[u];
      double y0 = 0.0, y1 = 0.0;
      int i = j + 1;
      for (; i + 1 < k; i += 2) {
        y0 = fma(vv[i], Z[i * LD + c], y0);
        y1 = fma(vv[i + 1], Z[(i + 1) * LD + c], y1);
      }
      if (i < k) y0 = fma(vv[i], Z[i * LD + c], y0);
      const double y = tau * (y0 + y1);
      for (i = j + 1; i < k; ++i) Z[i * LD + c] = fma(-y, vv[i], Z[i * LD + c]);
    }
    g.sync();
  }
  // P_+ = sum_{lambda_t > 0} lambda_t v_t v_t^T, packed upper, mode epilogue
  const int ns = k * (k + 1) / 2;
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
  for (int e = row; e < ns; e += KP) {
    int r, c;
    packed_rc(e, r, c);
    const double* Zrr = Z + r * LD;
    const double* Zc = Z + c * LD;
    double acc = 0.0;
    for (int u = 0; u < npos; ++u) {
      const int t = pidx[u];
      acc = fma(lp[u] * Zrr[t], Zc[t], acc);
    }
    const int64_t pe = off + e;
    if constexpr (MODE == PM_BATCH) {
      a.out[pe] = acc;
    } else if constexpr (MODE == PM_PRIMAL) {
      const double xkv = (r == c) ? acc : acc * kSqrt2;
      const double hx = __ldg(a.x + a.G[pe]);
      const double dd = xkv - hx;
      a.xk[pe] = xkv;
      a.lam[pe] = a.lam[pe] + a.rho * dd;  // E:LambdakUpdate
      p0 += dd * dd;
      p1 += xkv * xkv;
      p2 += hx * hx;
    } else {
      a.xk[pe] = (r == c) ? acc : acc * kSqrt2;
    }
  }
  if constexpr (MODE == PM_PRIMAL) {
    p0 = g.sum(p0);
    p1 = g.sum(p1);
    p2 = g.sum(p2);
    if (row == 0) {
      a.part[3 * (int64_t)task + 0] = p0;
      a.part[3 * (int64_t)task + 1] = p1;
      a.part[3 * (int64_t)task + 2] = p2;
    }
  }
}

template <int KP, int MODE>
void launch_chunk(const ProjArgs& a, int c0, int n, cudaStream_t s) {
  using TL = TridiagLayout<KP>;
  k_trd_tridiag<KP, MODE><<<(n + TL::NMAT - 1) / TL::NMAT, 128, TL::NMAT * TL::PER * sizeof(double), s>>>(a, c0, n);
  k_trd_ql<KP><<<(n + QL_T - 1) / QL_T, QL_T, 2 * KP * QL_T * sizeof(double), s>>>(a, c0, n);
  k_trd_apply<KP, MODE><<<n, KP, ApplyLayout<KP>::bytes(), s>>>(a, c0, n);
}

template <int KP, int MODE>
void set_attrs() {
  using TL = TridiagLayout<KP>;
  cudaFuncSetAttribute(k_trd_tridiag<KP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(TL::NMAT * TL::PER * sizeof(double)));
  cudaFuncSetAttribute(k_trd_ql<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * KP * QL_T * sizeof(double)));
  cudaFuncSetAttribute(k_trd_apply<KP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)ApplyLayout<KP>::bytes());
}

}  // namespace

void psd_trd_init_attributes() {
  set_attrs<32, PM_BATCH>();
  set_attrs<32, PM_PRIMAL>();
  set_attrs<32, PM_DUAL>();
  set_attrs<64, PM_BATCH>();
  set_attrs<64, PM_PRIMAL>();
  set_attrs<64, PM_DUAL>();
}

// SDP_TRD_ROTCAP overrides the capacity (tests force the inline-QL fallback with it)
int64_t trd_rot_cap(int k) {
  const char* e = getenv("SDP_TRD_ROTCAP");
  if (e && *e) return std::max<int64_t>(0, atoll(e));
  return std::max<int64_t>(64, (int64_t)3 * k * k / 2);
}

int64_t trd_hsize(int kp, int k) {
  const int64_t v = k >= 2 ? (int64_t)(k - 1) * (k - 2) / 2 : 0;
  return (4 * (int64_t)kp + v + 1) & ~(int64_t)1;
}

void launch_projection_trd(int bucket, int mode, const ProjArgs& a, cudaStream_t s) {
  const int count = a.td.count;
  if (count <= 0) return;
  for (int c0 = 0; c0 < count; c0 += a.td.chunk) {
    const int n = std::min(a.td.chunk, count - c0);
    if (bucket == B_TRD32) {
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
