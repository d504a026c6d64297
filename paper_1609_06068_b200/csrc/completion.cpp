// PSD completion of the returned X on the chordal pattern (P:90-97 and Theorem 1,
// P:104-108).  The paper proves that a partial matrix whose maximal-clique blocks are PSD has a PSD
// completion; the completion written out here is the classical perfect-elimination construction
// (the maximum-determinant completion for definite blocks), the same one oracle/completion.py
// states: vertices are placed in reverse elimination order, and when v is placed its later
// neighbours alpha (a clique of the extended pattern) give every unknown
//     X[v, u] = X[v, alpha] X[alpha, alpha]^+ X[alpha, u]       (u already placed).
// Host code: an output transform run once per solve, O(n^2 |alpha|) plus one |alpha|^3
// pseudo-inverse per vertex (cyclic Jacobi, eigenvalues below rtol max|lambda| dropped).
#include <cmath>
#include <vector>

#include "internal.h"

namespace sdp {

namespace {

// pinv of the symmetric k x k matrix A (row-major) by cyclic Jacobi
void pinv_sym(int k, std::vector<double>& A, double rtol, std::vector<double>& P) {
  std::vector<double> V((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) V[(size_t)i * k + i] = 1.0;
  double fro = 0.0;
  for (double a : A) fro += a * a;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) off += 2.0 * A[(size_t)p * k + q] * A[(size_t)p * k + q];
    if (off <= 1e-30 * fro) break;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double apq = A[(size_t)p * k + q];
        if (apq == 0.0) continue;
        const double app = A[(size_t)p * k + p], aqq = A[(size_t)q * k + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < k; ++r) {  // A <- A J
          const double arp = A[(size_t)r * k + p], arq = A[(size_t)r * k + q];
          A[(size_t)r * k + p] = c * arp - s * arq;
          A[(size_t)r * k + q] = s * arp + c * arq;
        }
        for (int r = 0; r < k; ++r) {  // A <- J^T A
          const double apr = A[(size_t)p * k + r], aqr = A[(size_t)q * k + r];
          A[(size_t)p * k + r] = c * apr - s * aqr;
          A[(size_t)q * k + r] = s * apr + c * aqr;
        }
        for (int r = 0; r < k; ++r) {  // V <- V J
          const double vrp = V[(size_t)r * k + p], vrq = V[(size_t)r * k + q];
          V[(size_t)r * k + p] = c * vrp - s * vrq;
          V[(size_t)r * k + q] = s * vrp + c * vrq;
        }
      }
  }
  double lmax = 0.0;
  for (int i = 0; i < k; ++i) lmax = std::fmax(lmax, std::fabs(A[(size_t)i * k + i]));
  std::vector<double> inv(k, 0.0);
  for (int i = 0; i < k; ++i) {
    const double l = A[(size_t)i * k + i];
    inv[i] = std::fabs(l) > rtol * lmax ? 1.0 / l : 0.0;
  }
  P.assign((size_t)k * k, 0.0);
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < k; ++c) {
      double s = 0.0;
      for (int i = 0; i < k; ++i) s += V[(size_t)r * k + i] * inv[i] * V[(size_t)c * k + i];
      P[(size_t)r * k + c] = s;
    }
}

}  // namespace

void complete_psd_host(int32_t n, const ChordalResult& cr, const std::vector<uint8_t>& known, double rtol,
                       double* X) {
  for (int64_t i = 0; i < (int64_t)n * n; ++i)
    if (!known[i]) X[i] = 0.0;
  std::vector<int32_t> done;
  done.reserve(n);
  done.push_back(cr.order[n - 1]);
  std::vector<double> A, P, r;
  for (int t = n - 2; t >= 0; --t) {
    const int v = cr.order[t];
    const int32_t* al = cr.later_idx.data() + cr.later_ptr[v];
    const int k = (int)(cr.later_ptr[v + 1] - cr.later_ptr[v]);
    r.assign(k, 0.0);
    if (k > 0) {
      A.resize((size_t)k * k);
      for (int a = 0; a < k; ++a)
        for (int b = 0; b < k; ++b) A[(size_t)a * k + b] = X[(size_t)al[a] * n + al[b]];
      pinv_sym(k, A, rtol, P);
      for (int b = 0; b < k; ++b) {
        double s = 0.0;
        for (int a = 0; a < k; ++a) s += X[(size_t)v * n + al[a]] * P[(size_t)a * k + b];
        r[b] = s;
      }
    }
    const int64_t nd = (int64_t)done.size();
#pragma omp parallel for schedule(static)
    for (int64_t di = 0; di < nd; ++di) {
      const int u = done[di];
      if (u == v || known[(size_t)v * n + u]) continue;
      double s = 0.0;
      for (int b = 0; b < k; ++b) s += r[b] * X[(size_t)al[b] * n + u];
      X[(size_t)v * n + u] = s;
      X[(size_t)u * n + v] = s;
    }
    done.push_back(v);
  }
}

}  // namespace sdp
