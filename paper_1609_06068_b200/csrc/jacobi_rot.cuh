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
  JRot r{1.0, 0.0};
  if (apq == 0.0) return r;
  const double d = aqq - app;
  // power-of-two scale so that max(|d|, |apq|) is in [1, 2)
  const double mx = fmax(fabs(d), fabs(apq));
  const int e = ilogb(mx);
  const float df = (float)scalbn(d, -e), af = (float)scalbn(apq, -e);
  // fp32 smaller root: t = 2 apq sign(d) / (|d| + sqrt(d^2 + 4 apq^2))
  const float rf = sqrtf(df * df + 4.0f * af * af);
  const float den = fabsf(df) + rf;
  float tf = (df >= 0.0f ? 2.0f : -2.0f) * af / den;
  double t = (double)tf;
  // one fp64 Newton step on g(t) = apq t^2 + d t - apq (scaled coefficients)
  const double as = scalbn(apq, -e), ds = scalbn(d, -e);
  const double g = fma(fma(as, t, ds), t, -as);
  const float gp = 2.0f * af * tf + df;  // g'(t) in fp32
  if (gp != 0.0f) t -= g * (double)(1.0f / gp);
  const double c = rsqrt(fma(t, t, 1.0));
  r.c = c;
  r.s = t * c;
  return r;
}

}  // namespace sdp
