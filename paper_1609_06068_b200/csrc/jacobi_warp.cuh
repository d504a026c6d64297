// One step of the warp-register Jacobi on a 32x32 symmetric matrix in "slot
// order" (kernels_psd_wj.cu; the round-robin permutation applied physically so
// the pairs of every step are the slots (2i, 2i+1), identity again after 31
// steps): lane j holds column j of A (av) and row j of V (vv).  Applies
// A <- J^T A J, V <- V J for the 16 rotations of the step (Golub-Van Loan
// sym.schur2, jacobi_rot.cuh) and the slot permutation.  `cs` is 16 double2 of
// warp-private shared scratch.
#pragma once
#include <cuda_runtime.h>

#include "jacobi_rot.cuh"

namespace sdp {
namespace wj {

constexpr int KP = 32;
constexpr unsigned FULL = 0xffffffffu;

// round-robin slot rotation (same schedule as kernels_psd_rv.cu)
__host__ __device__ constexpr int next_slot(int s) {
  return s == 0 ? 0 : (s & 1) ? (s == 1 ? 2 : s - 2) : (s == KP - 2 ? KP - 1 : s + 2);
}
__host__ __device__ constexpr int prev_slot(int t) {
  return t == 0 ? 0 : t == 2 ? 1 : t == KP - 1 ? KP - 2 : (t & 1) ? t + 2 : t - 2;
}

// (x[2m], x[2m+1]) with m = lane / 2, by a select tree on the lane bits (no
// dynamic register indexing, which the compiler would move to local memory)
__device__ __forceinline__ void pick_pair(const double (&x)[KP], int lane, double& x0, double& x1) {
  double y0[8], y1[8], z0[4], z1[4], w0[2], w1[2];
  const bool b1 = lane & 2, b2 = lane & 4, b3 = lane & 8, b4 = lane & 16;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    y0[m] = b1 ? x[4 * m + 2] : x[4 * m];
    y1[m] = b1 ? x[4 * m + 3] : x[4 * m + 1];
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    z0[m] = b2 ? y0[2 * m + 1] : y0[2 * m];
    z1[m] = b2 ? y1[2 * m + 1] : y1[2 * m];
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    w0[m] = b3 ? z0[2 * m + 1] : z0[2 * m];
    w1[m] = b3 ? z1[2 * m + 1] : z1[2 * m];
  }
  x0 = b4 ? w0[1] : w0[0];
  x1 = b4 ? w1[1] : w1[0];
}
__device__ __forceinline__ double pick(const double (&x)[KP], int lane) {
  double x0, x1;
  pick_pair(x, lane, x0, x1);
  return (lane & 1) ? x1 : x0;
}

__device__ __forceinline__ void step(double (&av)[KP], double (&vv)[KP], double2* cs, int lane) {
  const bool odd = lane & 1;
  // rotation of this lane's pair (slots 2i, 2i+1); both lanes compute it
  double x0, x1;
  pick_pair(av, lane, x0, x1);
  const double dg = odd ? x1 : x0, of = odd ? x0 : x1;
  const double dp = __shfl_xor_sync(FULL, dg, 1);
  const double apq = __shfl_sync(FULL, of, lane & ~1);
  const JRot jr = jacobi_rotation(odd ? dp : dg, odd ? dg : dp, apq);
  if (!odd) cs[lane >> 1] = make_double2(jr.c, jr.s);
  __syncwarp();
  // J^T from the left on this column, V <- V J on this row
#pragma unroll
  for (int m = 0; m < KP / 2; ++m) {
    const double2 r = cs[m];
    const double p = av[2 * m], q = av[2 * m + 1];
    av[2 * m] = fma(r.x, p, -r.y * q);
    av[2 * m + 1] = fma(r.y, p, r.x * q);
    const double vp = vv[2 * m], vq = vv[2 * m + 1];
    vv[2 * m] = fma(r.x, vp, -r.y * vq);
    vv[2 * m + 1] = fma(r.y, vp, r.x * vq);
  }
  // A <- A J on the column pair (2i, 2i+1): p' = c p - s q, q' = s p + c q
  const double sg = odd ? jr.s : -jr.s;
#pragma unroll
  for (int r = 0; r < KP; ++r) {
    const double b = __shfl_xor_sync(FULL, av[r], 1);
    av[r] = fma(sg, b, jr.c * av[r]);
  }
  // slot permutation: content of slot s moves to next_slot(s)
  const int src = prev_slot(lane);
  double t[KP];
#pragma unroll
  for (int r = 0; r < KP; ++r) t[next_slot(r)] = __shfl_sync(FULL, av[r], src);
#pragma unroll
  for (int r = 0; r < KP; ++r) av[r] = t[r];
#pragma unroll
  for (int r = 0; r < KP; ++r) t[next_slot(r)] = vv[r];
#pragma unroll
  for (int r = 0; r < KP; ++r) vv[r] = t[r];
  __syncwarp();
}

}  // namespace wj
}  // namespace sdp
