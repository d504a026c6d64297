#pragma once
#include "internal.h"

namespace sdp {

constexpr int kLongSeg = 16;  // scatter: segments longer than this get a warp

struct ScatterArgs {
  int N;
  const int32_t* seg_ptr;  // N+1
  const int32_t* seg_idx;  // stot, stacked positions of each coordinate (ascending)
  const int32_t* longc;    // coordinates with long segments
  int n_long;
  const double* xk;        // x_k (primal) / z_k (dual)
  const double* lam;
  const double* c;
  const double* Dinv;
  double rho;
  double* rD;              // out: r1 / D
  double* sprev;           // in/out: previous sum_k H_k^T x_k
  double* part;            // out: 2 per block
  const int* done;
  const int32_t* shared_idx;  // per coordinate: slot in xbuf if shared across ranks, else -1 (NULL: none)
  double* xbuf;               // 3 doubles per shared coordinate: r1, sum H^T x_k, sum H^T lam_k partials
  const int32_t* list = nullptr;  // short coordinates: list[0..N) instead of 0..N-1 (pipelined iteration)
};

struct FinalArgs {
  const double* proj_part;
  int n_proj;
  const double* upd_part;
  int n_upd;
  const double* scat_part;
  int n_scat;
  const double* gT_part;
  int n_gT;
  const double* fix_part;
  int n_fix;
  int n_fix2;         // PHASE 2 of the packed primal exchange: fix partials gathered here
  double* red;        // 6 partial sums (PHASE 1 out, PHASE 2 in)
  const double* b;
  const double* y;
  int m;
  double rho;
  double* res;        // eps_p, eps_d, objective
  double* hist;
  long long hist_cap;
  long long* iter;
  int* done;
  int* numerical;
  const double* tol;
};

void launch_scatter(int form, const ScatterArgs& a, cudaStream_t s);
int scatter_blocks(int N, int n_long);
void launch_gemv_dense(const double* A, int64_t lda, int m, const double* v, int chunk, double* part,
                       const int* done, cudaStream_t s);
// y = S^-1 u; with part != NULL, u = sum of the nchunks GEMV partials - r2 (formed in the kernel)
void launch_symv(int form, const double* Si, int m, const double* part, int nchunks, const double* b, double rho,
                 const double* u, double* y, const int* done, cudaStream_t s);
void symv_init_attributes(int m);
void launch_reduce_u(int form, const double* part, int nchunks, int m, const double* b, double rho, double* u,
                     const double* sdiag, double* y, const int* done, cudaStream_t s);
int gemvT_rows_blocks(int64_t N);
// rows != NULL: the N coordinates rows[0..N) instead of 0..N-1
void launch_gemvT_rows(int form, const double* AT, int64_t ldm, int m, int N, const double* y, const double* rD,
                       const double* Dinv, const double* c, const double* own, double* x, double* part,
                       const int* done, cudaStream_t s, const int32_t* rows = nullptr);
bool is_stream_kernel(const void* fn);
void launch_gemv_pieces(const double* A, int64_t lda, int m, const double* v, const int64_t* pieces, int npieces,
                        int slot0, double* part, const int* done, cudaStream_t s);
void launch_transpose(const double* A, int64_t lda, int m, double* AT, int64_t ldm, int64_t ncols, cudaStream_t s);
void launch_gemv_csr(int form, const int32_t* rp, const int32_t* ci, const double* val, int m, const double* v,
                     const double* b, double rho, double* u, const double* sdiag, double* y, const int* done,
                     cudaStream_t s);
int gemvT_csc_blocks(int N);
void launch_gemvT_csc(int form, const int32_t* cp, const int32_t* ri, const double* val, int N, const double* y,
                      const double* rD, const double* Dinv, const double* c, const double* own, double* x,
                      double* part, const int* done, cudaStream_t s);
int update_blocks(int64_t stot);
// iter_out (optional): *iter_out = *iter_in + 1 written by the kernel (next projection's iteration index)
void launch_update_dual(int64_t stot, const int32_t* G, const double* x, const double* z, double* lam, double* v,
                        double rho, double* part, const int* done, cudaStream_t s,
                        const long long* iter_in = nullptr, long long* iter_out = nullptr);
void launch_finalize(int form, int phase, const FinalArgs& a, cudaStream_t s);
int fixup_blocks(int nshared);
void launch_shared_fixup(int nshared, const int32_t* shared_local, double* xbuf, const double* Dinv,
                         const double* own, double* rD, double* sprev, double* part, const int* done,
                         cudaStream_t s, double* prevall = nullptr);
void launch_syrk_dense(const double* A, int64_t lda, int m, const double* Dinv, double* S, cudaStream_t s);
void launch_mask_cols(double* A, int64_t lda, int m, const double* mask, cudaStream_t s);
void launch_place_dense(const double* raw, int64_t npat, int m, const int64_t* map, const double* scale, double* A,
                        int64_t lda, cudaStream_t s, int* bad);

}  // namespace sdp
