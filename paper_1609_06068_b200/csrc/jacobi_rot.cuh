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
  // 2^-e with e = ilogb(mx), from the exponent bits (exact power of two, so
  // multiplying by it equals scalbn(., -e)); libm ilogb/scalbn only for
  // subnormal / extreme mx
  const int ex = ((__double2hiint(mx) >> 20) & 0x7ff) - 1023;
  double ds, as;
  if (ex > -1022 && ex < 1022) {
    const double sc = __hiloint2double((1023 - ex) << 20, 0);
    ds = d * sc;
    as = apq * sc;
  } else {
    const int e = ilogb(mx);
    ds = scalbn(d, -e);
    as = scalbn(apq, -e);
  }
  const float df = (float)ds, af = (float)as;
  // fp32 smaller root: t = 2 apq sign(d) / (|d| + sqrt(d^2 + 4 apq^2))
  // (approximate fp32 square root and divisions: the estimate only seeds the fp64 Newton step, and
  // the scaled operands keep every intermediate in [2^-60, 8], far from the approximations' limits)
  const float q = df * df + 4.0f * af * af;  // > 0: |as| >= 2^-53 |ds| or |ds| in [1, 2)
  const float rf = q * rsqrtf(q);
  const float den = fabsf(df) + rf;
  float tf = __fdividef((df >= 0.0f ? 2.0f : -2.0f) * af, den);
  double t = (double)tf;
  // one fp64 Newton step on g(t) = apq t^2 + d t - apq (scaled coefficients)
  const double g = fma(fma(as, t, ds), t, -as);
  const float gp = 2.0f * af * tf + df;  // g'(t) in fp32
  if (gp != 0.0f) t -= g * (double)__fdividef(1.0f, gp);
  const double c = rsqrt(fma(t, t, 1.0));
  r.c = c;
  r.s = t * c;
  return r;
}

}  // namespace sdp
