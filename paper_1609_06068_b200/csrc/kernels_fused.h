// Fused persistent iteration for small problems (kernels_fused.cu).
#pragma once
#include "internal.h"

namespace sdp {

constexpr int kFusedThreads = 256;
constexpr int kFusedLongSeg = 8;  // scatter: segments longer than this get a warp

struct FusedArgs {
  int iters = 0;
  int nb = 1;           // CTAs (fixed at setup: the reduction order depends on it)
  int m = 0, N = 0, p = 0;
  int64_t lda = 0, ldm = 0, stot = 0;
  int usplit = 1;       // warps per row of A in phase U
  double rho = 1.0;
  const double *A = nullptr, *AT = nullptr, *Sinv = nullptr, *sdiag = nullptr;
  const double *b = nullptr, *c = nullptr, *Dinv = nullptr, *own = nullptr;
  double *rD = nullptr, *x = nullptr, *y = nullptr, *upart = nullptr, *sprev = nullptr, *vk = nullptr;
  const int32_t *seg_ptr = nullptr, *seg_idx = nullptr;
  // sparse A (A == nullptr): CSR of A and CSC (= CSR of A^T); ul lanes per row in phase U
  const int32_t *a_rp = nullptr, *a_ci = nullptr, *at_cp = nullptr, *at_ri = nullptr;
  const double *a_val = nullptr, *at_val = nullptr;
  int ul = 1;
  ProjArgs pa{};        // off, ksz, x, G, xk, lam, vk, rho, part, vprev, voff, warm_period, capped, sweeps
  const int32_t* ids[3] = {nullptr, nullptr, nullptr};  // B_RV8, B_RV16, B_RV32 task lists
  int count[3] = {0, 0, 0};
  double* cpart = nullptr;  // nb * 8 per-CTA partials
  unsigned* bar = nullptr;  // grid barrier: two arrival counters, used by alternate launches
  int bar_parity = 0;
  int xl = 32;              // lanes per coordinate in phase X (power of two)
  const int32_t* longc = nullptr;  // coordinates with more than kFusedLongSeg stacked entries
  int n_long = 0;
  double *res = nullptr, *hist = nullptr;
  long long hist_cap = 0;
  long long* iter = nullptr;
  int *done = nullptr, *numerical = nullptr;
  const double* tol = nullptr;
  long long* trace = nullptr;  // SDP_FUSED_TRACE: CTA 0's %globaltimer at the phase marks, 64 x 16
};

size_t fused_smem_bytes();
// most CTAs co-resident on `device` (cooperative launch limit)
int fused_max_ctas(int device);
// largest m for which phase Y stages u in shared memory
inline int fused_max_m() { return (int)(fused_smem_bytes() / sizeof(double)) - 64; }
void launch_fused(int form, const FusedArgs& a, cudaStream_t s);

}  // namespace sdp
