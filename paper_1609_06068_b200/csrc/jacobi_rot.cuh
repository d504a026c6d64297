// Jacobi rotation for the symmetric 2x2 block [[app, apq], [apq, aqq]]
// (Golub & Van Loan, sym.schur2): J = [[c, s], [-s, c]] with t = s/c the
// smaller root of  apq t^2 + (aqq - app) t - apq = 0.
//
// Latency-lean evaluation: t is first computed in fp32 on inputs scaled by a
// power of two (no overflow/underflow), then refined with one fp64 Newton step
// on g(t) = apq t^2 + d t - apq, whose residual is evaluated exactly in fp64
// and divided by an fp32 approximation of g'(t); the refined t has relative
// error ~1e-14.  c = rsqrt(1 + t^2), s = t c in fp64, so J is orthogonal to
// fp64 rounding whatever the residual of t.  Because a_pq is then annihilated
// only to ~1e-14 relative, callers apply the full 2x2 transform to diagonal
// blocks instead of setting a_pq = 0.
#pragma once
#include <cuda_runtime.h>

namespace sdp {

struct JRot {
  double c, s;
};

__device__ __forceinline__ JRot jacobi_rotation(double app, double aqq, double apq) {
  // Branch-free (the rotation is on the critical chain of every Jacobi step).  Any orthogonal J is
  // a valid similarity, so the accuracy of t only affects how fast off(A) falls: the power-of-two
  // scaling is clamped instead of special-cased (mx outside [2^-1000, 2^1000] only slows the
  // estimate down), and apq == 0 selects the identity at the end.
  const double d = aqq - app;
  const double mx = fmax(fabs(d), fabs(apq));
  // 2^-e with e = ilogb(mx) from the exponent bits, clamped so that 2^-e stays a normal number
  int ex = ((__double2hiint(mx) >> 20) & 0x7ff) - 1023;
  ex = min(max(ex, -1000), 1000);
  const double sc = __hiloint2double((1023 - ex) << 20, 0);
  const double ds = d * sc, as = apq * sc;
  const float df = (float)ds, af = (float)as;
  // fp32 smaller root: t = 2 apq sign(d) / (|d| + sqrt(d^2 + 4 apq^2)).  Approximate fp32 square
  // root and divisions: the estimate only seeds the fp64 Newton step (q >= 1e-30 keeps rsqrtf finite;
  // q = 0 means apq = 0, selected away below)
  const float q = fmaxf(df * df + 4.0f * af * af, 1e-30f);
  const float rf = q * rsqrtf(q);
  const float den = fabsf(df) + rf;
  const float tf = __fdividef((df >= 0.0f ? 2.0f : -2.0f) * af, den);
  double t = (double)tf;
  // one fp64 Newton step on g(t) = apq t^2 + d t - apq (scaled coefficients); g'(t) in fp32 is
  // +-sqrt(d^2 + 4 apq^2) at the root, nonzero whenever apq != 0
  const double g = fma(fma(as, t, ds), t, -as);
  const float gp = 2.0f * af * tf + df;
  t -= g * (double)__fdividef(1.0f, gp);
  const double c = rsqrt(fma(t, t, 1.0));
  JRot r;
  const bool zero = apq == 0.0;
  r.c = zero ? 1.0 : c;
  r.s = zero ? 0.0 : t * c;
  return r;
}

}  // namespace sdp
