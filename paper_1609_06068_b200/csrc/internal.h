// Internal declarations shared by the host setup, the kernels and the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/chordal_sdp.h"

namespace sdp {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
struct Error {
  int code;
  std::string msg;
};
#define SDP_CUDA_TRY(expr)                                                                   \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      throw ::sdp::Error{_e == cudaErrorMemoryAllocation ? SDP_E_OOM : SDP_E_CUDA,           \
                         std::string(#expr) + ": " + cudaGetErrorString(_e)};                \
  } while (0)

// ---------------------------------------------------------------- host setup
// Chordal analysis (setup_host.cpp).
struct ChordalResult {
  std::vector<std::vector<int32_t>> cliques;  // sorted inside, list sorted lexicographically
  // extended pattern, canonical (column-major upper) order
  std::vector<int32_t> coord_row, coord_col;
  std::vector<int64_t> col_ptr;  // coordinates of column j are [col_ptr[j], col_ptr[j+1])
  int64_t fill_edges = 0;
  std::vector<int32_t> order;                 // elimination order (a perfect elimination order of E')
  std::vector<int64_t> later_ptr;             // n + 1: later neighbours of v at [later_ptr[v], later_ptr[v+1])
  std::vector<int32_t> later_idx;
};
// PSD completion (completion.cpp): X (n x n row-major, known entries set) completed in place on the
// chordal pattern of cr (Theorem 1; see oracle/completion.py)
void complete_psd_host(int32_t n, const ChordalResult& cr, const std::vector<uint8_t>& known, double rtol,
                       double* X);
// edges: off-diagonal upper pairs (i<j), may contain duplicates
ChordalResult chordal_analysis(int32_t n, const std::vector<std::pair<int32_t, int32_t>>& edges);
int64_t coord_index(const ChordalResult& cr, int32_t i, int32_t j);  // -1 if absent

// Sparse Cholesky of S (sparse_chol.cpp): S given as CSR (both triangles); on success GT (m x ldg,
// row-major) holds G^T with G = L^-1 (S = L L^T in a minimum-degree order), so S^-1 = G^T G.
// Returns false with *why = "factor too dense" (nnz(L) > max_fill_frac m^2 and !force) or the
// rank-deficiency message.
// S^-1 of a symmetric positive definite S (device, m x m; clobbered) by a blocked Gauss-Jordan sweep
// (kernels_schur.cu); false if a pivot fails the 1e-12 relative test
bool spd_inverse_gpu(double* S, int m, double* Sinv, double* work, double* diag0, int* bad, cudaStream_t s);
bool sparse_inverse_factor(int m, const std::vector<int64_t>& sp, const std::vector<int32_t>& si,
                           const std::vector<double>& sv, int64_t ldg, std::vector<double>& GT, int64_t* nnz_l,
                           double max_fill_frac, bool force, std::string* why);

// ---------------------------------------------------------------- sharding (shard.cpp)
struct ShardPlan {
  int world = 1, rank = 0;
  std::vector<int32_t> clique_rank;    // per clique (canonical order): its rank (LPT on k^3)
  std::vector<int32_t> my_cliques;     // this rank's cliques, ascending
  std::vector<int32_t> local_coords;   // sorted global coordinates touched by this rank
  std::vector<uint8_t> owned;          // per local coordinate: 1 if this rank owns it
  std::vector<int32_t> shared_coords;  // sorted global coordinates touched by >= 2 ranks
  std::vector<int32_t> shared_local;   // per shared coordinate: local index here, or -1
};
ShardPlan make_shard_plan(const std::vector<int32_t>& ksz, const std::vector<int64_t>& off,
                          const std::vector<int32_t>& seg_ptr, const std::vector<int32_t>& seg_idx, int world,
                          int rank);

// NCCL via dlopen (nccl_dl.cpp); every call throws Error{SDP_E_NCCL} on failure
void nccl_unique_id(void* out128);
void* nccl_comm_init(const void* id128, int world, int rank);
void nccl_allreduce_sum(void* comm, double* buf, size_t count, cudaStream_t s);
void nccl_comm_destroy(void* comm);

// Communicator of a sharded handle (comm.cu): in-place sum all-reduce of a device buffer on a
// stream; NCCL across processes or the in-process loopback group (sdp_loopback_create).
struct Comm {
  int world = 1, rank = 0;
  virtual ~Comm() {}
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t s) = 0;
  virtual bool loopback() const { return false; }
};
Comm* make_nccl_comm(const void* id128, int world, int rank);
Comm* make_loop_comm(void* group, int world, int rank);

// ---------------------------------------------------------------- projection buckets
// Kernel tiers for the batched eigen-projection (kernels_psd.cu).
enum BucketKind {
  B_G8 = 0, B_G16, B_G32, B_CTA32, B_CTA64, B_CTA96, B_GLOBAL, B_RV8, B_RV16, B_RV32, B_RV64, B_TRD8, B_TRD16, B_TRD32, B_TRD64, B_WJ32, B_NUM
};
inline bool is_rv(int b) { return b >= B_RV8 && b <= B_RV64; }
inline bool is_trd(int b) { return b >= B_TRD8 && b <= B_TRD64; }
inline int trd_kp(int b) { return b == B_TRD8 ? 8 : b == B_TRD16 ? 16 : b == B_TRD32 ? 32 : 64; }
constexpr int kTrdTiers = 4;  // B_TRD8 .. B_TRD64 (TrdDev arrays indexed by b - B_TRD8)
// Size ranges (k <= 8, 16, 32, 64, 96, larger) with fewer than kFewMatrices
// members use one CTA per matrix so that a small batch still fills the GPU.
constexpr int64_t kFewMatrices = 2048;
int size_range(int k);
int bucket_of(int k, int64_t count_in_range);

// Projection modes
enum ProjMode { PM_BATCH = 0, PM_PRIMAL = 1, PM_DUAL = 2 };

// Tridiagonal path for the giant orders (kernels_psd_gtrd.cu): blocked Householder
// reduction of an L2-resident matrix (8-CTA clusters for the large orders),
// multisection bisection, inverse iteration on one side of the spectrum, WY
// back-transform and reconstruction as DMMA products.  status[g] = -1 hands
// matrix g to the block-Jacobi kernel (GiantDev::only).
struct GtrdDev {
  int ng = 0;
  int kmax = 0;
  const int32_t* task = nullptr;       // per giant (same order as GiantDev)
  const int64_t* moff = nullptr;       // per giant: offset (doubles) of its workspace in ws
  const int32_t* hsel = nullptr;       // per giant: H = k (max selected eigenvectors, row length of Z)
  double* ws = nullptr;
  int32_t* status = nullptr;           // per giant
  int njob = 0;                        // tridiagonalization jobs (thread-block clusters of 8 CTAs)
  const int32_t* job_g = nullptr;      // njob * 8: giant per CTA (solo) or in slot 0 (coop); -1 unused
  const int32_t* job_coop = nullptr;   // njob: 1 = the cluster reduces one matrix together
  const int32_t* ev_pre = nullptr;     // ng + 1: bisection warps (32 indices each)
  const int32_t* vg_pre = nullptr;     // ng + 1: inverse-iteration CTA slots (2 ceil(k / cap) + 1), giants by descending k
  const int32_t* vg_g = nullptr;       // ng: the giant of each vg_pre position (largest first: longest chains start first)
  int32_t* ngrp = nullptr;             // per giant: groups in use (device-computed)
  const int32_t* wy_pre = nullptr;     // ng + 1: WY groups (16 reflectors each)
  const int32_t* bt_pre = nullptr;     // ng + 1: back-transform CTAs (kGtrdBackCols columns each)
  const int32_t* rc_pre = nullptr;     // ng + 1: reconstruction tiles (32 x 32, upper)
  double* part = nullptr;              // 3 per reconstruction tile (primal residual partials)
  int tot_ev = 0, tot_vg = 0, tot_wy = 0, tot_bt = 0, tot_rc = 0;
  // two-stage reduction (dense -> band -> tridiagonal) for orders >= sbr_min (SDP_GTRD_SBR_MIN)
  int sbr_min = 1 << 30;
  int njob2 = 0;                       // stage-A jobs (clusters of 8 CTAs, like job_g / job_coop)
  const int32_t* job2_g = nullptr;
  const int32_t* job2_coop = nullptr;
  int nsb = 0;                         // stage-B CTAs: one per two-stage giant
  const int32_t* sb_g = nullptr;
  int force_fallback = 0;              // SDP_GTRD_FORCE_FALLBACK=1: mark every matrix failed (tests)
  int debug = 0;                       // SDP_GTRD_DEBUG=1: per-matrix spectrum / cluster printf
};

// Giant tier (kernels_psd_giant.cu): block-Jacobi over 16-wide blocks, one
// persistent grid for all matrices of order > the CTA tiers.  Per giant g:
// kp = k rounded up to 32, P = kp / 32 pair blocks per step, A / V / T are
// kp x kp row-major at ws + wsoff[g] (+ kp^2, + 2 kp^2), Q (P blocks of 32x32)
// at qbuf + qoff[g].  *_pre are prefix sums (ng + 1) of the per-giant item
// counts of each phase.
struct GiantDev {
  int ng = 0;
  int max_steps = 0;                    // max over giants of 2P - 1 (steps per sweep)
  int tot_inner = 0, tot_tile = 0, tot_rb = 0, tot_out = 0, tot_full = 0;
  int grid = 0;                         // CTAs of the persistent launch (all co-resident)
  const int32_t* task = nullptr;        // task id of giant g
  const int32_t* kp = nullptr;
  const int64_t* wsoff = nullptr;
  const int64_t* qoff = nullptr;
  const int32_t *inner_pre = nullptr, *tile_pre = nullptr, *rb_pre = nullptr, *out_pre = nullptr,
                *full_pre = nullptr;
  double* ws = nullptr;
  double* qbuf = nullptr;
  double* part_fro = nullptr;           // tot_rb (per 32-column block)
  double* part_off = nullptr;           // tot_out (per upper 32x32 tile)
  double* part_out = nullptr;           // 3 * tot_out
  int32_t* gsweeps = nullptr;           // ng
  int32_t* gflag = nullptr;             // ng: active in the current sweep
  unsigned* bar = nullptr;              // grid barrier {count, generation}
  int trace = 0;                        // SDP_GIANT_TRACE=1: CTA 0 printf's the per-phase times
  const int32_t* only = nullptr;        // if set: process only giants with only[g] < 0, cold start
  GtrdDev gt;                           // tridiagonal path (runs first; only = gt.status)
};

// Tridiagonal-QL tiers (kernels_psd_trd.cu), per bucket.  Slots = positions in
// the bucket list; processed in chunks of `chunk` slots whose workspace
// offsets (hoff: doubles into hbuf) are relative to the chunk's first slot.
// Per slot hbuf holds d, e, tau, lambda (KP each) followed by the packed
// Householder vectors.
struct TrdDev {
  int count = 0;
  int chunk = 0;
  int force_fallback = 0;     // SDP_TRD_FORCE_FALLBACK=1 (tests): QL with vectors for every matrix
  int debug = 0;              // SDP_TRD_DEBUG=1: printf slot 0's spectrum selection (diagnostics)
  const int64_t* hoff = nullptr;
  const int64_t* zoff = nullptr;  // per slot: offset (doubles) of its selected eigenvectors of T
  double* hbuf = nullptr;
  double* zbuf = nullptr;         // per slot KP x KP doubles
  int32_t* rcount = nullptr;  // per slot: 0, or -1 (QL iteration cap / inverse iteration residual)
};

struct ProjArgs {
  const int64_t* off;   // per task: offset of its packed values
  const int32_t* ksz;   // per task: order k
  const int32_t* ids;   // bucket list of task ids
  int32_t count;        // tasks in this bucket
  // batch mode
  const double* in;
  double* out;
  // ADMM modes
  const double* x;      // N, global iterate (primal gather source)
  const int32_t* G;     // stacked -> coordinate map
  double* xk;           // stacked x_k / z_k (output)
  double* lam;          // stacked lambda_k (primal: updated in place)
  const double* vk;     // dual: stacked v_k
  double rho;
  double* part;         // primal: per task 3 partials (|xk-hx|^2, |xk|^2, |hx|^2)
  GiantDev gd;          // B_GLOBAL (giant) tier: tridiagonal path + block-Jacobi fallback
  TrdDev td;            // tridiagonal-QL tier being launched
  unsigned long long* capped;  // count of sweep-capped projections
  unsigned long long* sweeps;  // total Jacobi sweeps (diagnostics)
  const int32_t* done;  // device stop flag (skip work when set)
  // warm start (ADMM modes): per task eigenvector basis of the previous iteration
  double* vprev;        // per task kp*kp doubles at voff[task]
  const int64_t* voff;
  const long long* iter;  // iteration counter; cold start when iter % warm_period == 0
  int32_t warm_period;    // 0 = never warm start
  long long* rvtrace = nullptr;  // diagnostics (SDP_FUSED_TRACE): register-V Jacobi phase clocks
};

void launch_projection(int bucket, int mode, const ProjArgs& a, cudaStream_t s);
void launch_projection_rv(int bucket, int mode, const ProjArgs& a, cudaStream_t s);
void launch_projection_giant(int mode, const ProjArgs& a, cudaStream_t s);
void launch_projection_gtrd(int mode, const ProjArgs& a, cudaStream_t s);
// CTAs per thread-block cluster of the giant one-stage tridiagonalization (k_gtrd_tridiag jobs)
#ifndef GTRD_CLUSTER
#define GTRD_CLUSTER 8
#endif
// columns per back-transform CTA of the giant tridiagonal path (one warp each)
constexpr int kGtrdBackCols = 16;
// vector-kernel group capacity of the giant tridiagonal path for order k (shared-memory bound)
constexpr int kVecSmemDoubles = 26000;
__host__ __device__ inline int gtrd_vec_cap(int k) {
  const int c = (kVecSmemDoubles - 2 * k) / (k > 0 ? k : 1);
  return c < 128 ? c : 128;
}
int gtrd_max_order();          // largest order the giant tridiagonal path takes (shared-memory bound)
int64_t gtrd_ws_doubles(int k);  // workspace of one matrix of order k
void launch_projection_trd(int bucket, int mode, const ProjArgs& a, cudaStream_t s);
void launch_projection_wj(int mode, const ProjArgs& a, cudaStream_t s);
int64_t trd_hsize(int kp, int k);  // doubles of per-slot Householder workspace
int trd_launches_per_chunk(int bucket);  // kernels per chunk of a QL tier (5 for the split k = 64 form)
int giant_grid();        // CTAs of the persistent giant kernel on the current device
int giant_min_order();   // smallest order routed to the giant tier (SDP_GIANT_MIN, default 65)
int rv_kp(int bucket);
// stride (kp) of the warm-start V storage of a matrix of order k in tier `bucket`
inline int store_kp(int bucket, int k) {
  return is_trd(bucket) ? 0 : bucket == B_WJ32 ? 32 : is_rv(bucket) ? rv_kp(bucket) : bucket == B_GLOBAL ? (k + 31) / 32 * 32 : k + (k & 1);
}

}  // namespace sdp
