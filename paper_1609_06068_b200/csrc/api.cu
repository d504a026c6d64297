// C ABI (include/chordal_sdp.h): setup, the ADMM iteration pipeline captured in
// a CUDA graph, getters, and the batched PSD projection plan.
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "kernels_fused.h"
#include "kernels_vec.h"

namespace sdp {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
void psd_init_attributes();

namespace {

constexpr double kSqrt2 = 1.41421356237309504880;
constexpr long long kHistCap = 1 << 20;

// Every device buffer of a handle / plan: cudaMalloc, or the caller's allocator
// (sdp_options.allocator: e.g. torch uint8 tensors, so that PyTorch owns the memory).
struct Alloc {
  std::vector<std::pair<void*, size_t>> ptrs;
  sdp_allocator hook{};
  bool has_hook = false;
  int device = 0;
  int64_t live = 0, peak = 0;
  void set_hook(const sdp_allocator* a, int dev) {
    device = dev;
    has_hook = a && a->alloc && a->free;
    if (has_hook) hook = *a;
  }
  void* raw(size_t bytes) {
    bytes = std::max<size_t>(bytes, 1);
    void* p = nullptr;
    if (has_hook) {
      p = hook.alloc(hook.ctx, bytes, device);
      if (!p)
        throw Error{SDP_E_OOM, "allocator returned NULL for " + std::to_string(bytes) + " bytes"};
      if ((uintptr_t)p % 256)
        throw Error{SDP_E_INVALID_ARG, "allocator returned a pointer not aligned to 256 bytes"};
    } else {
      SDP_CUDA_TRY(cudaMalloc(&p, bytes));
    }
    ptrs.push_back({p, bytes});
    live += (int64_t)bytes;
    peak = std::max(peak, live);
    return p;
  }
  template <class T>
  T* get(size_t n) {
    return (T*)raw(std::max<size_t>(n, 1) * sizeof(T));
  }
  // cudaMemset and cudaMemcpy from pageable host memory run on the legacy default stream and may
  // return before they land; the kernels that read the buffers run on non-blocking streams, so
  // both wait for the legacy stream before returning the buffer
  template <class T>
  T* zeros(size_t n) {
    T* p = get<T>(n);
    SDP_CUDA_TRY(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
    SDP_CUDA_TRY(cudaStreamSynchronize(cudaStreamLegacy));
    return p;
  }
  template <class T>
  T* upload(const std::vector<T>& v, size_t n_alloc = 0) {
    size_t n = std::max(v.size(), n_alloc);
    T* p = get<T>(n);
    if (v.size() < std::max<size_t>(n, 1))
      SDP_CUDA_TRY(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
    if (!v.empty()) SDP_CUDA_TRY(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    SDP_CUDA_TRY(cudaStreamSynchronize(cudaStreamLegacy));
    return p;
  }
  void free_one(void* p) {
    if (has_hook)
      hook.free(hook.ctx, p, device);
    else
      cudaFree(p);
  }
  void release(void* p) {
    auto it = std::find_if(ptrs.begin(), ptrs.end(), [&](const std::pair<void*, size_t>& q) { return q.first == p; });
    if (it != ptrs.end()) {
      cudaDeviceSynchronize();
      free_one(p);
      live -= (int64_t)it->second;
      ptrs.erase(it);
    }
  }
  void free_all() {
    for (auto& q : ptrs) free_one(q.first);
    ptrs.clear();
    live = 0;
  }
};

// Host Cholesky S = L L^T (row-major, lower), blocked right-looking with the panel solve and the
// trailing update spread over the host threads (OpenMP).  Returns false if S is not numerically
// positive definite (a pivot <= 1e-12 * the original S_ii).
bool cholesky_host(std::vector<double>& S, int m) {
  constexpr int NB = 64;
  std::vector<double> diag0(m);
  for (int i = 0; i < m; ++i) diag0[i] = S[(size_t)i * m + i];
  auto dot = [](const double* a, const double* b, int n) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    int k = 0;
    for (; k + 4 <= n; k += 4) {
      a0 += a[k] * b[k];
      a1 += a[k + 1] * b[k + 1];
      a2 += a[k + 2] * b[k + 2];
      a3 += a[k + 3] * b[k + 3];
    }
    for (; k < n; ++k) a0 += a[k] * b[k];
    return (a0 + a1) + (a2 + a3);
  };
  bool ok = true;
  for (int k0 = 0; k0 < m && ok; k0 += NB) {
    const int k1 = std::min(m, k0 + NB);
    // diagonal block (the columns < k0 were applied by the trailing updates)
    for (int i = k0; i < k1 && ok; ++i) {
      double* Li = S.data() + (size_t)i * m;
      for (int j = k0; j <= i; ++j) {
        const double* Lj = S.data() + (size_t)j * m;
        const double sv = Li[j] - dot(Li + k0, Lj + k0, j - k0);
        if (i == j) {
          if (!(sv > 1e-12 * diag0[i]) || !std::isfinite(sv)) {
            ok = false;
            break;
          }
          Li[i] = std::sqrt(sv);
        } else {
          Li[j] = sv / Lj[j];
        }
      }
    }
    if (!ok) break;
    // panel rows i >= k1: L[i][k0:k1] = A[i][k0:k1] L11^-T
#pragma omp parallel for schedule(static)
    for (int i = k1; i < m; ++i) {
      double* Li = S.data() + (size_t)i * m;
      for (int j = k0; j < k1; ++j) {
        const double* Lj = S.data() + (size_t)j * m;
        Li[j] = (Li[j] - dot(Li + k0, Lj + k0, j - k0)) / Lj[j];
      }
    }
    // trailing update of the lower part: A[i][j] -= L[i][k0:k1] . L[j][k0:k1], k1 <= j <= i
#pragma omp parallel for schedule(dynamic, 8)
    for (int i = k1; i < m; ++i) {
      double* Li = S.data() + (size_t)i * m;
      for (int j = k1; j <= i; ++j) Li[j] -= dot(Li + k0, S.data() + (size_t)j * m + k0, k1 - k0);
    }
  }
  if (!ok) return false;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) S[(size_t)i * m + j] = 0.0;
  return true;
}

// Wt = (L^-1)^T (row-major upper): row j of Wt is column j of L^-1.
void tri_inverse_T(const std::vector<double>& L, int m, std::vector<double>& Wt) {
  Wt.assign((size_t)m * m, 0.0);
#pragma omp parallel for schedule(dynamic, 8)
  for (int j = 0; j < m; ++j) {
    double* w = Wt.data() + (size_t)j * m;
    w[j] = 1.0 / L[(size_t)j * m + j];
    for (int i = j + 1; i < m; ++i) {
      const double* Li = L.data() + (size_t)i * m;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      int k = j;
      for (; k + 4 <= i; k += 4) {
        a0 += Li[k] * w[k];
        a1 += Li[k + 1] * w[k + 1];
        a2 += Li[k + 2] * w[k + 2];
        a3 += Li[k + 3] * w[k + 3];
      }
      for (; k < i; ++k) a0 += Li[k] * w[k];
      w[i] = -((a0 + a1) + (a2 + a3)) / Li[i];
    }
  }
}

}  // namespace
}  // namespace sdp

using namespace sdp;

// First clique of the second half of the pipelined iteration: the stacked-length fraction
// SDP_PIPE_SPLIT of the cliques goes to the first half.  Defaults measured on cfg2 (B200, A/B over
// 0.35 .. 0.8): primal 0.65 (1166 vs 1121 it/s at 0.5), dual 0.55 (1150 vs 1119 it/s) -- a larger
// first half shortens the second half's projection, which is the exposed tail of the iteration.
inline int64_t pipe_split(const std::vector<int64_t>& off, int64_t p, int form) {
  const double def = form == SDP_FORM_DUAL ? 0.55 : 0.65;
  const char* e = getenv("SDP_PIPE_SPLIT");
  double f = e ? atof(e) : def;
  if (!(f > 0.05 && f < 0.95)) f = def;
  int64_t p1 = 1;
  while (p1 < p - 1 && (double)off[p1] < f * (double)off[p]) ++p1;
  return p1;
}

// Side stream for the projection tiers: the giant tier (a chain of kernels whose tail leaves
// most SMs idle) runs on the calling stream while every other tier runs concurrently on `side`
// (fork / join by events, captured into the iteration graph as a branch).
struct TierFork {
  static constexpr int kMaxSide = 4;
  int nside = 0;  // SDP_TIER_STREAMS (default 2: cfg4 16.52M -> 16.78M proj/s, cfg3 / cfg1 unchanged; 3-4: no further gain)
  cudaStream_t side[kMaxSide] = {};
  // the lead tier (the giant chain, else the largest tier) runs on a stream of the highest
  // priority, so its kernels take the SMs first and the other tiers fill what its low-occupancy
  // phases (QL, inverse iteration, cluster reductions) leave idle; SDP_TIER_PRIO=0: off
  cudaStream_t hi = nullptr;
  cudaEvent_t fork = nullptr, join[kMaxSide] = {}, join_hi = nullptr;
  void create() {
    const char* e = getenv("SDP_TIER_STREAMS");
    nside = e ? std::max(1, std::min(kMaxSide, atoi(e))) : 2;
    SDP_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    for (int i = 0; i < nside; ++i) {
      SDP_CUDA_TRY(cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking));
      SDP_CUDA_TRY(cudaEventCreateWithFlags(&join[i], cudaEventDisableTiming));
    }
    const char* pr = getenv("SDP_TIER_PRIO");
    if (!(pr && *pr == '0')) {
      int least = 0, greatest = 0;
      SDP_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      SDP_CUDA_TRY(cudaStreamCreateWithPriority(&hi, cudaStreamNonBlocking, greatest));
      SDP_CUDA_TRY(cudaEventCreateWithFlags(&join_hi, cudaEventDisableTiming));
    }
  }
  void destroy() {
    for (int i = 0; i < kMaxSide; ++i) {
      if (side[i]) cudaStreamDestroy(side[i]);
      if (join[i]) cudaEventDestroy(join[i]);
      side[i] = nullptr;
      join[i] = nullptr;
    }
    if (hi) cudaStreamDestroy(hi);
    if (join_hi) cudaEventDestroy(join_hi);
    hi = nullptr;
    join_hi = nullptr;
    if (fork) cudaEventDestroy(fork);
    fork = nullptr;
    nside = 0;
  }
};
struct BucketSet {
  int32_t* d_ids[B_NUM] = {};
  int bcount[B_NUM] = {};
  TrdDev td[kTrdTiers];
};
struct Pipe {
  bool on = false;
  int p1 = 0;
  int32_t *rows1 = nullptr, *rows2 = nullptr;         // gemvT coordinates: touched by H1 / H2 only
  int nr1 = 0, nr2 = 0;
  int32_t *sc1 = nullptr, *sc2 = nullptr, *lc1 = nullptr, *lc2 = nullptr;  // scatter passes (short, long)
  int ns1 = 0, ns2 = 0, nl1 = 0, nl2 = 0;
  int64_t* pieces = nullptr;                          // gemv column pieces: H1-only first, then the rest
  int npe = 0, npl = 0;
  double *gemv_part = nullptr, *gT_part = nullptr, *scat_part = nullptr;
  // every sdp_step call ends with the next iteration's A already issued ("pending"): x on the
  // H1-touched coordinates and y of the finished iteration are kept in x_save / y_save, and
  // settle() puts them back before the state is read or changed through the API
  bool pending = false;
  double *x_save = nullptr, *y_save = nullptr;
  // dual form: the iteration index the next iteration's P_+(H1) reads (it runs concurrently with
  // the current finalize, which advances the handle's counter)
  long long* iter_next = nullptr;
  // dual form: scatter partials double-buffered by iteration parity (the next iteration's scatter
  // runs before the current finalize), dual-update partials per half
  int par = 0;
  int64_t soff1 = 0;  // stacked offset of the first clique of H2
  double *scat_part2 = nullptr, *upd_part = nullptr;
  int nb_u1 = 0, nb_u2 = 0;
  int nb_gT1 = 0, nb_gT2 = 0, nb_sc1 = 0, nb_sc2 = 0;
  BucketSet half[2];
  cudaStream_t sp = nullptr, sp2 = nullptr, sx = nullptr, sg = nullptr;  // projections (high priority), gemvT, gemv
  int prio_hi = 0;
  cudaEvent_t ev[8] = {};
  cudaGraph_t g[3] = {};
  cudaGraphExec_t x[3] = {};  // A, BA, B
  void destroy_graphs() {
    for (int i = 0; i < 3; ++i) {
      if (x[i]) cudaGraphExecDestroy(x[i]);
      if (g[i]) cudaGraphDestroy(g[i]);
      x[i] = nullptr;
      g[i] = nullptr;
    }
  }
  void destroy() {
    destroy_graphs();
    if (sp) cudaStreamDestroy(sp);
    if (sp2) cudaStreamDestroy(sp2);
    if (sx) cudaStreamDestroy(sx);
    if (sg) cudaStreamDestroy(sg);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    sp = sp2 = sx = sg = nullptr;
  }
};

struct sdp_handle_s {
  int n = 0, m = 0;
  int64_t N = 0, lda = 0, p = 0, stot = 0;
  int form = 0;
  double rho = 1.0;
  int device = 0;
  cudaStream_t stream = nullptr, cap_stream = nullptr;
  bool own_stream = false;
  int check_every = 10, use_graph = 1;
  int adapt = 0;
  double adapt_mu = 10.0, adapt_tau = 2.0;
  double setup_s = 0;
  int64_t fill_edges = 0;
  // host copies
  std::vector<int32_t> coord_row, coord_col, clique_size, clique_vert;
  ChordalResult chordal;  // pattern analysis kept for the PSD completion (order, later neighbours, E')
  std::vector<int64_t> clique_off;
  int64_t kmin = 0, kmax = 0;
  // device buffers
  Alloc alloc;
  double *x = nullptr, *rD = nullptr, *Dinv = nullptr, *c = nullptr, *sprev = nullptr, *y = nullptr, *u = nullptr,
         *t = nullptr, *b = nullptr;
  double *xk = nullptr, *lam = nullptr, *vk = nullptr;
  int32_t *G = nullptr, *seg_ptr = nullptr, *seg_idx = nullptr, *longc = nullptr;
  int n_long = 0;
  int64_t* d_off = nullptr;
  int32_t* d_ksz = nullptr;
  int32_t* d_ids[B_NUM] = {};
  int bcount[B_NUM] = {};
  GiantDev gd;
  TrdDev td[kTrdTiers];  // B_TRD8 .. B_TRD64
  TierFork tiers;
  Pipe pipe;
  // A
  int a_dense = 1;
  double* A = nullptr;
  double* AT = nullptr;  // A^T copy (row-major N x ldm) so A^T y is a row-streaming GEMV
  int64_t ldm = 0;
  int32_t *a_rp = nullptr, *a_ci = nullptr, *at_cp = nullptr, *at_ri = nullptr;
  double *a_val = nullptr, *at_val = nullptr;
  int s_diag = 0;
  int s_factor = 0;      // 0: S diagonal, 1: dense Cholesky (host), 2: sparse Cholesky (sparse_chol.cpp)
  int64_t nnz_l = 0;     // nonzeros of the sparse factor
  double* sdiag = nullptr;
  double *W = nullptr, *WT = nullptr, *Sinv = nullptr;
  double* gemv_part = nullptr;
  int chunk = 8192, nchunks = 0;
  // residuals
  double *proj_part = nullptr, *scat_part = nullptr, *gT_part = nullptr, *upd_part = nullptr;
  int nb_scat = 0, nb_gT = 0, nb_upd = 0;
  double *res = nullptr, *hist = nullptr, *tol = nullptr;
  long long* iter = nullptr;
  int *done = nullptr, *numerical = nullptr;
  unsigned long long* capped = nullptr;
  unsigned long long* sweeps = nullptr;
  double* vprev = nullptr;
  int64_t vprev_len = 0;
  int64_t* voff = nullptr;
  int warm_period = 64;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // sharding: this rank's local view
  int world = 1, rank = 0;
  Comm* comm = nullptr;         // NCCL or in-process loopback (comm.cu)
  int64_t pl = 0, Nl = 0, stotl = 0;  // local cliques / coordinates / stacked length
  std::vector<int32_t> my_cliques;    // this rank's cliques (canonical ids, ascending)
  std::vector<int32_t> local_coords;
  bool coord_perm = false;      // world == 1 with a permuted local coordinate order (pipelined iteration)
  double* own = nullptr;        // 1.0 on owned local coordinates
  int nshared = 0, n_fix = 0;
  int32_t *shared_idx = nullptr, *shared_local = nullptr;
  double *xbuf = nullptr, *fix_part = nullptr, *red = nullptr;
  double* prevall = nullptr;    // packed primal exchange: previous sums of every shared coordinate
  // fused persistent iteration (kernels_fused.cu): small single-rank problems
  bool fused = false;
  int fused_nb = 1, fused_usplit = 1;
  int32_t* fused_ids[3] = {nullptr, nullptr, nullptr};
  int fused_count[3] = {0, 0, 0};
  double *fused_upart = nullptr, *fused_cpart = nullptr;
  unsigned* fused_bar = nullptr;
  int fused_parity = 0;
  int fused_xl = 32, fused_ul = 1, fused_nlong = 0;
  int32_t* fused_longc = nullptr;
  long long* fused_trace = nullptr;
};

struct sdp_psd_plan_s {
  int device = 0;
  int64_t count = 0, values = 0;
  Alloc alloc;
  int64_t* d_off = nullptr;
  int32_t* d_ksz = nullptr;
  int32_t* d_ids[B_NUM] = {};
  int bcount[B_NUM] = {};
  GiantDev gd;
  TrdDev td[kTrdTiers];
  TierFork tiers;
  unsigned long long* capped = nullptr;
  unsigned long long* sweeps = nullptr;
  double *h_in_dev = nullptr, *h_out_dev = nullptr;
  // host-buffer path: two pinned staging chunks; the host side of each chunk is copied by all host
  // threads while the DMA of the other chunk is in flight
  double* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  // pinned host buffers: the batch in contiguous sub-plans whose H2D copy, projection and D2H copy
  // overlap (copy engines in both directions beside the compute)
  std::vector<int32_t> h_sizes;
  std::vector<sdp_psd_plan_s*> sub;
  std::vector<int64_t> sub_v0, sub_nv;
  cudaStream_t cp_in = nullptr, cp_out = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_comp;
  cudaEvent_t ev_end = nullptr;
  void free_stage() {
    for (int b = 0; b < 2; ++b) {
      if (stage[b]) cudaFreeHost(stage[b]);
      if (stage_ev[b]) cudaEventDestroy(stage_ev[b]);
      stage[b] = nullptr;
      stage_ev[b] = nullptr;
    }
  }
};

namespace {
constexpr int64_t kStageDoubles = 8 << 20;  // 64 MB per staging chunk

void host_copy_parallel(double* dst, const double* src, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < n; b += 65536) std::memcpy(dst + b, src + b, std::min<int64_t>(65536, n - b) * sizeof(double));
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) SDP_CUDA_TRY(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return SDP_E_OOM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return SDP_E_INVALID_ARG;
  }
}

// Tridiagonal path of the giant tier (kernels_psd_gtrd.cu); SDP_GIANT_METHOD=jacobi turns it off.
void build_gtrd(Alloc& al, const std::vector<int32_t>& ksz, const std::vector<int32_t>& ids, GiantDev& gd) {
  const char* meth = getenv("SDP_GIANT_METHOD");
  if (meth && std::string(meth) == "jacobi") return;
  GtrdDev& gt = gd.gt;
  const int ng = (int)ids.size();
  const int kcap = gtrd_max_order();
  std::vector<int64_t> moff(ng, 0);
  std::vector<int32_t> hsel(ng), ev(ng + 1, 0), vg(ng + 1, 0), wy(ng + 1, 0), bt(ng + 1, 0), rc(ng + 1, 0);
  int64_t ws = 0;
  int kmax = 0;
  for (int g = 0; g < ng; ++g) {
    const int k = ksz[ids[g]];
    hsel[g] = k;  // the computed side may be the larger one (k_gtrd_cluster)
    const bool ok = k <= kcap;
    moff[g] = ws;
    if (ok) {
      ws += (gtrd_ws_doubles(k) + 31) / 32 * 32;
      kmax = std::max(kmax, k);
    }
    const int R = (k + 31) / 32;
    ev[g + 1] = ev[g] + (ok ? (k + 31) / 32 : 0);
    vg[g + 1] = vg[g] + (ok ? 2 * ((k + gtrd_vec_cap(k) - 1) / gtrd_vec_cap(k)) + 1 : 0);
    wy[g + 1] = wy[g] + (ok ? (k - 2 + 15) / 16 : 0);
    bt[g + 1] = bt[g] + (ok ? (k + kGtrdBackCols - 1) / kGtrdBackCols : 0);
    rc[g + 1] = rc[g] + (ok ? R * (R + 1) / 2 : 0);
  }
  // tridiagonalization jobs: one 8-CTA cluster per order >= SDP_GTRD_COOP_MIN (default 200),
  // the smaller ones 8 per cluster (one CTA each), largest first
  const char* cm = getenv("SDP_GTRD_COOP_MIN");
  const int coop_min = cm ? std::max(1, atoi(cm)) : 200;
  // two-stage reduction (dense -> band -> tridiagonal) for orders >= SDP_GTRD_SBR_MIN; default off
  // (0): measured slower than the one-stage reduction on B200 ("two-stage")
  const char* sm = getenv("SDP_GTRD_SBR_MIN");
  int sbr_min = sm ? atoi(sm) : 0;
  if (sbr_min <= 0) sbr_min = 1 << 30;
  gt.sbr_min = sbr_min;
  std::vector<int> order(ng);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return ksz[ids[x]] > ksz[ids[y]]; });
  std::vector<int32_t> job_g, job_coop, job2_g, job2_coop, sb_g;
  std::vector<int> solo, solo2;
  for (int g : order) {
    const int kk = ksz[ids[g]];
    const bool two = kk >= sbr_min && kk <= kcap;
    std::vector<int32_t>& jg = two ? job2_g : job_g;
    std::vector<int32_t>& jc = two ? job2_coop : job_coop;
    if (two) sb_g.push_back(g);
    const int cs = two ? 8 : GTRD_CLUSTER;  // stage-A jobs use 8-CTA clusters
    if (kk >= coop_min) {
      jc.push_back(1);
      for (int r = 0; r < cs; ++r) jg.push_back(r == 0 ? g : -1);
    } else {
      (two ? solo2 : solo).push_back(g);
    }
  }
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<int>& so = pass ? solo2 : solo;
    std::vector<int32_t>& jg = pass ? job2_g : job_g;
    std::vector<int32_t>& jc = pass ? job2_coop : job_coop;
    const size_t cs = pass ? 8 : GTRD_CLUSTER;
    for (size_t i = 0; i < so.size(); i += cs) {
      jc.push_back(0);
      for (size_t r = 0; r < cs; ++r) jg.push_back(i + r < so.size() ? so[i + r] : -1);
    }
  }
  gt.njob = (int)job_coop.size();
  gt.job_g = job_g.empty() ? nullptr : al.upload(job_g);
  gt.job_coop = job_coop.empty() ? nullptr : al.upload(job_coop);
  gt.njob2 = (int)job2_coop.size();
  gt.job2_g = job2_g.empty() ? nullptr : al.upload(job2_g);
  gt.job2_coop = job2_coop.empty() ? nullptr : al.upload(job2_coop);
  gt.nsb = (int)sb_g.size();
  gt.sb_g = sb_g.empty() ? nullptr : al.upload(sb_g);
  gt.ng = ng;
  gt.kmax = std::max(kmax, 1);
  gt.task = al.upload(ids);
  gt.moff = al.upload(moff);
  gt.hsel = al.upload(hsel);
  gt.ws = al.get<double>((size_t)std::max<int64_t>(ws, 32));
  gt.status = al.zeros<int32_t>((size_t)ng);
  gt.ev_pre = al.upload(ev);
  gt.tot_ev = ev[ng];
  {
    // inverse-iteration CTA slots in descending order (the k = 630 groups' chains are the longest)
    std::vector<int32_t> vgo(ng + 1, 0), vgg(ng, 0);
    const char* vo = getenv("SDP_GTRD_VEC_ORDER");
    const bool desc = !(vo && vo[0] == '0');
    for (int q = 0; q < ng; ++q) {
      const int g = desc ? order[q] : q;
      vgg[q] = g;
      vgo[q + 1] = vgo[q] + (vg[g + 1] - vg[g]);
    }
    gt.vg_pre = al.upload(vgo);
    gt.vg_g = al.upload(vgg);
    gt.tot_vg = vgo[ng];
  }
  gt.ngrp = al.zeros<int32_t>((size_t)ng);
  gt.wy_pre = al.upload(wy);
  gt.tot_wy = wy[ng];
  gt.bt_pre = al.upload(bt);
  gt.rc_pre = al.upload(rc);
  gt.tot_bt = bt[ng];
  gt.tot_rc = rc[ng];
  gt.part = al.zeros<double>(3 * (size_t)std::max(gt.tot_rc, 1));
  const char* ff = getenv("SDP_GTRD_FORCE_FALLBACK");
  gt.force_fallback = (ff && *ff == '1') ? 1 : 0;
  const char* gdb = getenv("SDP_GTRD_DEBUG");
  gt.debug = gdb ? atoi(gdb) : 0;
  gd.only = gt.status;
}

// Giant-tier metadata and workspace (kernels_psd_giant.cu) for the tasks `ids`.
void build_giant(Alloc& al, const std::vector<int32_t>& ksz, const std::vector<int32_t>& ids, GiantDev& gd) {
  gd = GiantDev{};
  const int ng = (int)ids.size();
  if (!ng) return;
  std::vector<int32_t> kp(ng), inner(ng + 1, 0), tile(ng + 1, 0), rb(ng + 1, 0), out(ng + 1, 0), full(ng + 1, 0);
  std::vector<int64_t> wsoff(ng), qoff(ng);
  int64_t ws = 0, qb = 0, ti = 0;
  int maxs = 0;
  for (int g = 0; g < ng; ++g) {
    const int k = ksz[ids[g]];
    kp[g] = (k + 31) / 32 * 32;
    const int64_t P = kp[g] / 32;
    wsoff[g] = ws;
    ws += 3 * (int64_t)kp[g] * kp[g];
    qoff[g] = qb;
    qb += P * 1024;
    ti += P * (P + 1) / 2 + P * P;
    if (ti >= (1ll << 31)) throw Error{SDP_E_INVALID_ARG, "giant tier: too many work items"};
    inner[g + 1] = inner[g] + (int32_t)P;
    tile[g + 1] = tile[g] + (int32_t)(P * (P + 1) / 2 + P * P);
    rb[g + 1] = rb[g] + (int32_t)P;
    out[g + 1] = out[g] + (int32_t)(P * (P + 1) / 2);
    full[g + 1] = full[g] + (int32_t)(P * P);
    maxs = std::max(maxs, (int)(2 * P - 1));
  }
  gd.ng = ng;
  gd.max_steps = maxs;
  gd.tot_inner = inner[ng];
  gd.tot_tile = tile[ng];
  gd.tot_rb = rb[ng];
  gd.tot_out = out[ng];
  gd.tot_full = full[ng];
  gd.task = al.upload(ids);
  gd.kp = al.upload(kp);
  gd.wsoff = al.upload(wsoff);
  gd.qoff = al.upload(qoff);
  gd.inner_pre = al.upload(inner);
  gd.tile_pre = al.upload(tile);
  gd.rb_pre = al.upload(rb);
  gd.out_pre = al.upload(out);
  gd.full_pre = al.upload(full);
  gd.ws = al.get<double>((size_t)ws);
  gd.qbuf = al.get<double>((size_t)qb);
  gd.part_fro = al.zeros<double>((size_t)gd.tot_rb);
  gd.part_off = al.zeros<double>((size_t)gd.tot_out);
  gd.part_out = al.zeros<double>(3 * (size_t)gd.tot_out);
  gd.gsweeps = al.zeros<int32_t>((size_t)ng);
  gd.gflag = al.zeros<int32_t>((size_t)ng);
  gd.bar = al.zeros<unsigned>(2);
  gd.grid = giant_grid();
  const char* tr = getenv("SDP_GIANT_TRACE");
  gd.trace = tr ? atoi(tr) : 0;
  build_gtrd(al, ksz, ids, gd);
}

// Tridiagonal-QL tier workspace (kernels_psd_trd.cu) for the tasks `ids` of storage order kp,
// processed in chunks so that the workspace stays under SDP_TRD_BUDGET_MB (default 4096).
void build_trd(Alloc& al, const std::vector<int32_t>& ksz, const std::vector<int32_t>& ids, int kp, TrdDev& td) {
  td = TrdDev{};
  const int n = (int)ids.size();
  if (!n) return;
  const char* bud = getenv("SDP_TRD_BUDGET_MB");
  const int64_t budget = (bud ? std::max(16ll, atoll(bud)) : 4096ll) << 20;
  const int64_t zper = (int64_t)kp * kp;  // KP/2 inverse-iteration vectors, or the QL fallback's full Z
  const int64_t per = 8 * (trd_hsize(kp, kp) + zper);
  const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(n, budget / per));
  std::vector<int64_t> hoff(n), zoff(n);
  int64_t hmax = 0, h = 0;
  for (int i = 0; i < n; ++i) {
    if (i % chunk == 0) h = 0;
    hoff[i] = h;
    zoff[i] = (int64_t)(i % chunk) * zper;
    h += trd_hsize(kp, ksz[ids[i]]);
    hmax = std::max(hmax, h);
  }
  td.count = n;
  td.chunk = chunk;
  const char* ff = getenv("SDP_TRD_FORCE_FALLBACK");
  td.force_fallback = (ff && *ff == '1') ? 1 : 0;
  const char* dbg = getenv("SDP_TRD_DEBUG");
  td.debug = (dbg && *dbg == '1') ? 1 : 0;
  td.hoff = al.upload(hoff);
  td.zoff = al.upload(zoff);
  td.hbuf = al.get<double>((size_t)hmax);
  td.zbuf = al.get<double>((size_t)chunk * zper);
  td.rcount = al.zeros<int32_t>((size_t)n);
}

void build_buckets(Alloc& al, const std::vector<int32_t>& ksz, int32_t* d_ids[B_NUM], int bcount[B_NUM],
                   GiantDev& gd, TrdDev td[kTrdTiers], std::vector<int>* bucket_out = nullptr) {
  std::vector<std::vector<int32_t>> lists(B_NUM);
  int64_t in_range[6] = {0, 0, 0, 0, 0, 0};
  for (size_t i = 0; i < ksz.size(); ++i) in_range[size_range(ksz[i])]++;
  for (size_t i = 0; i < ksz.size(); ++i) {
    const int b = bucket_of(ksz[i], in_range[size_range(ksz[i])]);
    if (bucket_out) bucket_out->push_back(b);
    lists[b].push_back((int32_t)i);
  }
  for (int b = 0; b < B_NUM; ++b) {
    bcount[b] = (int)lists[b].size();
    d_ids[b] = bcount[b] ? al.upload(lists[b]) : nullptr;
  }
  build_giant(al, ksz, lists[B_GLOBAL], gd);
  for (int t = 0; t < kTrdTiers; ++t) build_trd(al, ksz, lists[B_TRD8 + t], trd_kp(B_TRD8 + t), td[t]);
}

// The tiers are independent: the giant tier (a chain of kernels whose tail leaves most SMs idle)
// runs on the calling stream, every other tier on a side stream of its own (round-robin over
// TierFork::nside), so the low-occupancy kernels of one tier (QL, inverse iteration) overlap the
// others; captured into the iteration graph as parallel branches.
void launch_tiers(ProjArgs a, int mode, int32_t* const d_ids[B_NUM], const int bcount[B_NUM], const TrdDev td[kTrdTiers],
                  const TierFork& tf, cudaStream_t s) {
  int tiers[B_NUM], nt = 0;
  for (int b = B_NUM - 1; b >= 0; --b)  // larger first
    if (b != B_GLOBAL && bcount[b]) tiers[nt++] = b;
  const bool giant = bcount[B_GLOBAL] > 0;
  const bool fork = tf.nside > 0 && nt + (giant ? 1 : 0) >= 2;
  bool used[TierFork::kMaxSide] = {};
  const bool lead_hi = fork && tf.hi != nullptr;
  if (fork) SDP_CUDA_TRY(cudaEventRecord(tf.fork, s));
  if (lead_hi) SDP_CUDA_TRY(cudaStreamWaitEvent(tf.hi, tf.fork, 0));
  if (giant) {
    a.ids = d_ids[B_GLOBAL];
    a.count = bcount[B_GLOBAL];
    launch_projection(B_GLOBAL, mode, a, lead_hi ? tf.hi : s);
  }
  for (int q = 0; q < nt; ++q) {
    const int b = tiers[q];
    cudaStream_t so = s;
    if (lead_hi && !giant && q == 0) {
      so = tf.hi;
    } else if (fork && !lead_hi && (giant || q > 0)) {
      const int k = (giant ? q : q - 1) % tf.nside;
      so = tf.side[k];
      if (!used[k]) SDP_CUDA_TRY(cudaStreamWaitEvent(so, tf.fork, 0));
      used[k] = true;
    } else if (lead_hi && tf.nside > 1) {  // the remaining tiers: the caller's stream + side streams
      const int r = (giant ? q : q - 1) % tf.nside;
      if (r > 0) {
        so = tf.side[r - 1];
        if (!used[r - 1]) SDP_CUDA_TRY(cudaStreamWaitEvent(so, tf.fork, 0));
        used[r - 1] = true;
      }
    }
    a.ids = d_ids[b];
    a.count = bcount[b];
    if (is_trd(b)) a.td = td[b - B_TRD8];
    launch_projection(b, mode, a, so);
  }
  for (int k = 0; k < TierFork::kMaxSide; ++k)
    if (used[k]) {
      SDP_CUDA_TRY(cudaEventRecord(tf.join[k], tf.side[k]));
      SDP_CUDA_TRY(cudaStreamWaitEvent(s, tf.join[k], 0));
    }
  if (lead_hi) {
    SDP_CUDA_TRY(cudaEventRecord(tf.join_hi, tf.hi));
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, tf.join_hi, 0));
  }
}

void enqueue_projection(sdp_handle h, int mode, cudaStream_t s) {
  ProjArgs a{};
  a.off = h->d_off;
  a.ksz = h->d_ksz;
  a.x = h->x;
  a.G = h->G;
  a.xk = h->xk;
  a.lam = h->lam;
  a.vk = h->vk;
  a.rho = h->rho;
  a.part = h->proj_part;
  a.gd = h->gd;
  a.capped = h->capped;
  a.sweeps = h->sweeps;
  a.done = h->done;
  a.vprev = h->vprev;
  a.voff = h->voff;
  a.iter = h->iter;
  a.warm_period = h->warm_period;
  launch_tiers(a, mode, h->d_ids, h->bcount, h->td, h->tiers, s);
}

FinalArgs final_args(sdp_handle h);

// Sharded primal iteration: the residual partials of the rank (projection, scatter,
// objective) ride in the tail of the shared-coordinate exchange (allreduce #1), and the
// shared-coordinate eps_d partials are then computed identically on every rank from a replicated
// copy of the previous sums, so the iteration needs two all-reduces (#1 and u), not three.
bool packed_exchange(sdp_handle h) { return h->world > 1 && h->form == SDP_FORM_PRIMAL; }

void enqueue_scatter(sdp_handle h, cudaStream_t s) {
  ScatterArgs a{};
  a.N = (int)h->Nl;
  a.shared_idx = h->shared_idx;
  a.xbuf = h->xbuf;
  a.seg_ptr = h->seg_ptr;
  a.seg_idx = h->seg_idx;
  a.longc = h->longc;
  a.n_long = h->n_long;
  a.xk = h->xk;
  a.lam = h->lam;
  a.c = h->c;
  a.Dinv = h->Dinv;
  a.rho = h->rho;
  a.rD = h->rD;
  a.sprev = h->sprev;
  a.part = h->scat_part;
  a.done = h->done;
  launch_scatter(h->form, a, s);
  if (packed_exchange(h)) {
    FinalArgs fa = final_args(h);
    fa.n_fix = 0;
    fa.red = h->xbuf + 3 * (size_t)h->nshared;  // the 6 local residual partials
    launch_finalize(h->form, 1, fa, s);
    h->comm->allreduce_sum(h->xbuf, 3 * (size_t)h->nshared + 6, s);  // allreduce #1 (+ residual scalars)
    launch_shared_fixup(h->nshared, h->shared_local, h->xbuf, h->Dinv, h->own, h->rD, h->sprev, h->fix_part,
                        h->done, s, h->prevall);
  } else if (h->world > 1 && h->nshared > 0) {
    // exchange: partial sums of coordinates shared across ranks (allreduce #1)
    h->comm->allreduce_sum(h->xbuf, 3 * (size_t)h->nshared, s);
    launch_shared_fixup(h->nshared, h->shared_local, h->xbuf, h->Dinv, h->own, h->rD, h->sprev, h->fix_part,
                        h->done, s);
  }
}

// Phase hook: records an event at a phase boundary when profiling.
struct PhaseRec {
  std::vector<cudaEvent_t>* ev = nullptr;
  int* idx = nullptr;
  void mark(int phase, cudaStream_t s) const {
    if (!ev) return;
    cudaEventRecord((*ev)[(*idx)++], s);
    (void)phase;
  }
};
thread_local PhaseRec g_phase;
thread_local int g_phase_id[64];
thread_local int g_phase_n = 0;
inline void phase(int ph, cudaStream_t s) {
  if (!g_phase.ev) return;
  g_phase_id[g_phase_n++] = ph;
  g_phase.mark(ph, s);
}

void enqueue_kkt(sdp_handle h, cudaStream_t s) {
  const int f = h->form;
  double* ydst = h->s_diag ? h->y : nullptr;
  phase(0, s);
  const bool shard = h->world > 1;
  if (h->a_dense) {
    // partials only: y = S^-1 (sum partials - r2) is one kernel below (single rank)
    launch_gemv_dense(h->A, h->lda, h->m, h->rD, h->chunk, h->gemv_part, h->done, s);
    phase(1, s);
    if (shard)  // partial u over owned columns
      launch_reduce_u(f, h->gemv_part, h->nchunks, h->m, nullptr, h->rho, h->u, nullptr, nullptr, h->done, s);
  } else {
    if (shard)
      launch_gemv_csr(f, h->a_rp, h->a_ci, h->a_val, h->m, h->rD, nullptr, h->rho, h->u, nullptr, nullptr, h->done,
                      s);
    else
      launch_gemv_csr(f, h->a_rp, h->a_ci, h->a_val, h->m, h->rD, h->b, h->rho, h->u,
                      h->s_diag ? h->sdiag : nullptr, ydst, h->done, s);
    phase(1, s);
  }
  if (shard) {
    // exchange: u = sum over ranks of A[:, owned] D^-1 r1 (allreduce #2), then - r2 (and / S_ii)
    h->comm->allreduce_sum(h->u, (size_t)h->m, s);
    launch_reduce_u(f, h->u, 1, h->m, h->b, h->rho, h->u, h->s_diag ? h->sdiag : nullptr, ydst, h->done, s);
  }
  if (!h->s_diag) {  // y = S^-1 u = W^T W u
    if (h->a_dense && !shard)
      launch_symv(f, h->Sinv, h->m, h->gemv_part, h->nchunks, h->b, h->rho, nullptr, h->y, h->done, s);
    else
      launch_symv(f, h->Sinv, h->m, nullptr, 0, nullptr, h->rho, h->u, h->y, h->done, s);
  }
  phase(2, s);
  if (h->a_dense)
    launch_gemvT_rows(f, h->AT, h->ldm, h->m, (int)h->Nl, h->y, h->rD, h->Dinv, h->c, h->own, h->x, h->gT_part,
                      h->done, s);
  else
    launch_gemvT_csc(f, h->at_cp, h->at_ri, h->at_val, (int)h->Nl, h->y, h->rD, h->Dinv, h->c, h->own, h->x,
                     h->gT_part,
                     h->done, s);
}

FinalArgs final_args(sdp_handle h) {
  FinalArgs a{};
  a.proj_part = h->proj_part;
  a.n_proj = (int)h->pl;
  a.fix_part = h->fix_part;
  a.n_fix = h->world > 1 ? h->n_fix : 0;
  a.red = h->red;
  a.upd_part = h->upd_part;
  a.n_upd = h->nb_upd;
  a.scat_part = h->scat_part;
  a.n_scat = h->nb_scat;
  a.gT_part = h->gT_part;
  a.n_gT = h->nb_gT;
  a.b = h->b;
  a.y = h->y;
  a.m = h->m;
  a.rho = h->rho;
  a.res = h->res;
  a.hist = h->hist;
  a.hist_cap = kHistCap;
  a.iter = h->iter;
  a.done = h->done;
  a.numerical = h->numerical;
  a.tol = h->tol;
  return a;
}

void enqueue_finalize(sdp_handle h, cudaStream_t s, const double* scat_part = nullptr, int n_scat = 0,
                      const double* gT_part = nullptr, int n_gT = 0, const double* upd_part = nullptr,
                      int n_upd = 0) {
  FinalArgs a{};
  a.proj_part = h->proj_part;
  a.n_proj = (int)h->pl;
  a.fix_part = h->fix_part;
  a.n_fix = h->world > 1 ? h->n_fix : 0;
  a.red = h->red;
  a.upd_part = upd_part ? upd_part : h->upd_part;
  a.n_upd = upd_part ? n_upd : h->nb_upd;
  a.scat_part = scat_part ? scat_part : h->scat_part;
  a.n_scat = scat_part ? n_scat : h->nb_scat;
  a.gT_part = gT_part ? gT_part : h->gT_part;
  a.n_gT = gT_part ? n_gT : h->nb_gT;
  a.b = h->b;
  a.y = h->y;
  a.m = h->m;
  a.rho = h->rho;
  a.res = h->res;
  a.hist = h->hist;
  a.hist_cap = kHistCap;
  a.iter = h->iter;
  a.done = h->done;
  a.numerical = h->numerical;
  a.tol = h->tol;
  if (h->world == 1) {
    launch_finalize(h->form, 0, a, s);
  } else if (packed_exchange(h)) {
    // the rank partials were all-reduced with the scatter exchange; add the shared-coordinate
    // partials (identical on every rank) and finish
    a.red = h->xbuf + 3 * (size_t)h->nshared;
    a.n_fix2 = h->n_fix;
    a.n_fix = 0;
    launch_finalize(h->form, 2, a, s);
  } else {
    launch_finalize(h->form, 1, a, s);
    h->comm->allreduce_sum(h->red, 6, s);  // residual partials (allreduce #3)
    launch_finalize(h->form, 2, a, s);
  }
}

// One ADMM iteration (Algorithm 1 lines 4-7 / Algorithm 2 lines 4-8).
// ---------------------------------------------------------------- pipelined primal iteration
// Setup of the pipelined iteration (see struct Pipe).  SDP_PIPELINE=0 turns it off.
void build_pipeline(sdp_handle h, const std::vector<int32_t>& G, const std::vector<int64_t>& off,
                    const std::vector<int32_t>& seg_ptr, const std::vector<int>& task_bucket) {
  Pipe& P = h->pipe;
  P = Pipe{};
  const char* env = getenv("SDP_PIPELINE");
  if (env && *env == '0') return;
  const int64_t N = h->Nl, p = h->pl;
  if (!h->a_dense || h->world != 1 || h->bcount[B_GLOBAL] > 0 || N < 65536 || p < 8)
    return;
  Alloc& al = h->alloc;
  // halves by stacked length
  const int p1 = (int)pipe_split(off, p, h->form);
  P.p1 = p1;
  std::vector<uint8_t> cls(N, 0);  // bit 0: touched by H1, bit 1: by H2
  for (int64_t k = 0; k < p; ++k)
    for (int64_t e = off[k]; e < off[k + 1]; ++e) cls[G[e]] |= (k < p1) ? 1 : 2;
  std::vector<int32_t> rows1, rows2, sc1, sc2, lc1, lc2;
  for (int64_t t = 0; t < N; ++t) {
    const bool lng = seg_ptr[t + 1] - seg_ptr[t] > kLongSeg;
    if (cls[t] & 1) rows1.push_back((int32_t)t);
    else rows2.push_back((int32_t)t);
    if (cls[t] == 1) (lng ? lc1 : sc1).push_back((int32_t)t);
    else (lng ? lc2 : sc2).push_back((int32_t)t);
  }
  // u = A D^-1 r1 column pieces: runs of H1-only coordinates, then runs of the rest, <= 32768 each
  std::vector<int64_t> pe, pl2;
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<int64_t>& out = pass ? pl2 : pe;
    int64_t t = 0;
    while (t < N) {
      const bool early = cls[t] == 1;
      if (early != (pass == 0)) {
        ++t;
        continue;
      }
      int64_t e = t;
      while (e < N && (cls[e] == 1) == early && e - t < 32768) ++e;
      out.push_back(t);
      out.push_back(e);
      t = e;
    }
  }
  P.npe = (int)pe.size() / 2;
  P.npl = (int)pl2.size() / 2;
  std::vector<int64_t> pieces(pe);
  pieces.insert(pieces.end(), pl2.begin(), pl2.end());
  if (P.npe == 0 || P.npl == 0 || rows2.empty()) return;  // nothing to overlap
  P.pieces = al.upload(pieces);
  P.soff1 = off[p1];
  P.rows1 = al.upload(rows1);
  P.rows2 = al.upload(rows2);
  P.nr1 = (int)rows1.size();
  P.nr2 = (int)rows2.size();
  P.sc1 = sc1.empty() ? nullptr : al.upload(sc1);
  P.sc2 = sc2.empty() ? nullptr : al.upload(sc2);
  P.lc1 = lc1.empty() ? nullptr : al.upload(lc1);
  P.lc2 = lc2.empty() ? nullptr : al.upload(lc2);
  P.ns1 = (int)sc1.size();
  P.ns2 = (int)sc2.size();
  P.nl1 = (int)lc1.size();
  P.nl2 = (int)lc2.size();
  P.gemv_part = al.zeros<double>((size_t)(P.npe + P.npl) * h->m);
  P.x_save = al.zeros<double>((size_t)rows1.size());
  P.y_save = al.zeros<double>((size_t)h->m);
  P.nb_gT1 = gemvT_rows_blocks(P.nr1);
  P.nb_gT2 = gemvT_rows_blocks(P.nr2);
  P.gT_part = al.zeros<double>((size_t)(P.nb_gT1 + P.nb_gT2));
  P.nb_sc1 = P.ns1 + P.nl1 > 0 ? scatter_blocks(P.ns1, P.nl1) : 0;
  P.nb_sc2 = P.ns2 + P.nl2 > 0 ? scatter_blocks(P.ns2, P.nl2) : 0;
  P.scat_part = al.zeros<double>(2 * (size_t)std::max(P.nb_sc1 + P.nb_sc2, 1));
  if (h->form == SDP_FORM_DUAL) {
    P.scat_part2 = al.zeros<double>(2 * (size_t)std::max(P.nb_sc1 + P.nb_sc2, 1));
    P.nb_u1 = update_blocks(off[p1]);
    P.nb_u2 = update_blocks(off[p] - off[p1]);
    P.upd_part = al.zeros<double>(3 * (size_t)(P.nb_u1 + P.nb_u2));
    P.iter_next = al.zeros<long long>(1);
  }
  // the two halves keep the tiers of the full assignment (the warm-start layout depends on it)
  for (int hf = 0; hf < 2; ++hf) {
    std::vector<std::vector<int32_t>> lists(B_NUM);
    for (int64_t k = hf ? p1 : 0; k < (hf ? p : p1); ++k) lists[task_bucket[k]].push_back((int32_t)k);
    BucketSet& B = P.half[hf];
    for (int b = 0; b < B_NUM; ++b) {
      B.bcount[b] = (int)lists[b].size();
      B.d_ids[b] = B.bcount[b] ? al.upload(lists[b]) : nullptr;
    }
    std::vector<int32_t> ksz(p);
    SDP_CUDA_TRY(cudaMemcpy(ksz.data(), h->d_ksz, p * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int t = 0; t < kTrdTiers; ++t) build_trd(al, ksz, lists[B_TRD8 + t], trd_kp(B_TRD8 + t), B.td[t]);
  }
  int lo = 0, hi = 0;
  SDP_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  SDP_CUDA_TRY(cudaStreamCreateWithPriority(&P.sp, cudaStreamNonBlocking, hi));
  SDP_CUDA_TRY(cudaStreamCreateWithPriority(&P.sp2, cudaStreamNonBlocking, hi));
  P.prio_hi = hi;
  SDP_CUDA_TRY(cudaStreamCreateWithFlags(&P.sx, cudaStreamNonBlocking));
  SDP_CUDA_TRY(cudaStreamCreateWithFlags(&P.sg, cudaStreamNonBlocking));
  for (auto& e : P.ev) SDP_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  P.on = true;
}

void pipe_gemv(sdp_handle h, cudaStream_t s, int first, int count) {
  const Pipe& P = h->pipe;
  launch_gemv_pieces(h->A, h->lda, h->m, h->rD, P.pieces + 2 * first, count, first, P.gemv_part, h->done, s);
}

void pipe_symv_gemvT1(sdp_handle h, cudaStream_t s) {
  const Pipe& P = h->pipe;
  launch_symv(h->form, h->Sinv, h->m, P.gemv_part, P.npe + P.npl, h->b, h->rho, nullptr, h->y, h->done, s);
  launch_gemvT_rows(h->form, h->AT, h->ldm, h->m, P.nr1, h->y, h->rD, h->Dinv, h->c, h->own, h->x,
                    P.gT_part, h->done, s, P.rows1);
}

void pipe_projection(sdp_handle h, int half, cudaStream_t s, const long long* iter = nullptr) {
  const BucketSet& B = h->pipe.half[half];
  ProjArgs a{};
  a.off = h->d_off;
  a.ksz = h->d_ksz;
  a.x = h->x;
  a.G = h->G;
  a.xk = h->xk;
  a.lam = h->lam;
  a.vk = h->vk;
  a.rho = h->rho;
  a.part = h->proj_part;
  a.capped = h->capped;
  a.sweeps = h->sweeps;
  a.done = h->done;
  a.vprev = h->vprev;
  a.voff = h->voff;
  a.iter = iter ? iter : h->iter;
  a.warm_period = h->warm_period;
  launch_tiers(a, h->form == SDP_FORM_PRIMAL ? PM_PRIMAL : PM_DUAL, B.d_ids, B.bcount, B.td, TierFork{}, s);
}

void pipe_scatter(sdp_handle h, int pass, cudaStream_t s) {
  const Pipe& P = h->pipe;
  ScatterArgs a{};
  a.N = pass ? P.ns2 : P.ns1;
  a.list = pass ? P.sc2 : P.sc1;
  a.seg_ptr = h->seg_ptr;
  a.seg_idx = h->seg_idx;
  a.longc = pass ? P.lc2 : P.lc1;
  a.n_long = pass ? P.nl2 : P.nl1;
  a.xk = h->xk;
  a.lam = h->lam;
  a.c = h->c;
  a.Dinv = h->Dinv;
  a.rho = h->rho;
  a.rD = h->rD;
  a.sprev = h->sprev;
  a.part = (P.par ? P.scat_part2 : P.scat_part) + 2 * (pass ? P.nb_sc1 : 0);
  a.done = h->done;
  launch_scatter(h->form, a, s);
}

// SDP_PIPE_TRACE=1 with use_graph = 0: event timeline of the last launched B / BA (stderr)
struct PipeTrace {
  bool on = false;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  void mark(const char* name, cudaStream_t s) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back({name, e});
  }
  void dump() {
    if (!on || ev.empty()) return;
    cudaDeviceSynchronize();
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0].second, ev[i].second);
      fprintf(stderr, "[pipe] %-14s %8.1f us\n", ev[i].first, ms * 1e3);
    }
    for (auto& e : ev) cudaEventDestroy(e.second);
    ev.clear();
  }
};
PipeTrace g_ptrace;

void pipe_enqueue_A(sdp_handle h, cudaStream_t s) {
  pipe_gemv(h, s, 0, h->pipe.npe + h->pipe.npl);
  pipe_symv_gemvT1(h, s);
}

// B (with_A: then the next iteration's A, overlapped)
void pipe_enqueue_B(sdp_handle h, cudaStream_t s, bool with_A) {
  Pipe& P = h->pipe;
  g_ptrace.mark("start", s);
  SDP_CUDA_TRY(cudaEventRecord(P.ev[0], s));
  SDP_CUDA_TRY(cudaStreamWaitEvent(P.sx, P.ev[0], 0));
  SDP_CUDA_TRY(cudaStreamWaitEvent(P.sp, P.ev[0], 0));
  // x on the H2-only coordinates || P_+ of H1, scatter of the H1-only coordinates
  launch_gemvT_rows(h->form, h->AT, h->ldm, h->m, P.nr2, h->y, h->rD, h->Dinv, h->c, h->own, h->x,
                    P.gT_part + P.nb_gT1, h->done, P.sx, P.rows2);
  g_ptrace.mark("gemvT2", P.sx);
  SDP_CUDA_TRY(cudaEventRecord(P.ev[1], P.sx));
  pipe_projection(h, 0, P.sp);
  g_ptrace.mark("projH1", P.sp);
  pipe_scatter(h, 0, P.sp);
  g_ptrace.mark("scatter1", P.sp);
  if (with_A) {  // next iteration: u over the H1-only columns, while P_+ of H2 runs
    SDP_CUDA_TRY(cudaEventRecord(P.ev[2], P.sp));
    SDP_CUDA_TRY(cudaStreamWaitEvent(P.sg, P.ev[2], 0));
    pipe_gemv(h, P.sg, 0, P.npe);
    g_ptrace.mark("gemv_early", P.sg);
    SDP_CUDA_TRY(cudaEventRecord(P.ev[3], P.sg));
  }
  // P_+ of H2 as soon as x is complete on its coordinates (own stream: not behind P_+ of H1)
  SDP_CUDA_TRY(cudaStreamWaitEvent(P.sp2, P.ev[1], 0));
  pipe_projection(h, 1, P.sp2);
  g_ptrace.mark("projH2", P.sp2);
  SDP_CUDA_TRY(cudaEventRecord(P.ev[5], P.sp2));
  SDP_CUDA_TRY(cudaStreamWaitEvent(P.sp, P.ev[5], 0));
  pipe_scatter(h, 1, P.sp);
  SDP_CUDA_TRY(cudaEventRecord(P.ev[6], P.sp));
  enqueue_finalize(h, P.sp, P.scat_part, P.nb_sc1 + P.nb_sc2, P.gT_part, P.nb_gT1 + P.nb_gT2);
  g_ptrace.mark("finalize", P.sp);
  SDP_CUDA_TRY(cudaEventRecord(P.ev[4], P.sp));
  if (with_A) {
    // the rest of u needs the scatter only (finalize runs alongside); y = S^-1 u and the
    // x-pass of the next iteration wait for finalize (its stop flag)
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, P.ev[6], 0));
    pipe_gemv(h, s, P.npe, P.npl);
    g_ptrace.mark("gemv_late", s);
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, P.ev[3], 0));
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, P.ev[4], 0));
    // the finished iteration's y and x on the coordinates the next x-pass overwrites (rows1 is
    // the contiguous range [0, nr1) of the local order)
    SDP_CUDA_TRY(cudaMemcpyAsync(P.y_save, h->y, (size_t)h->m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    SDP_CUDA_TRY(cudaMemcpyAsync(P.x_save, h->x, (size_t)P.nr1 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    pipe_symv_gemvT1(h, s);
    g_ptrace.mark("symv+gemvT1", s);
  } else {
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, P.ev[4], 0));
  }
}

// ---------------------------------------------------------------- pipelined dual iteration
// Alg. 2 order per iteration: P_+ (z) -> scatter -> u, y, x -> dual update (v, lambda) -> finalize.
// Prefix D_A: P_+ and scatter of the first iteration, u, y, x on the H1-touched coordinates.
// D_BA(t -> t+1): x on the H2-only coordinates || [dual update of H1 (x is complete on its
// coordinates), P_+ of H1 for t+1, scatter of the H1-only coordinates]; dual update of H2,
// finalize(t), P_+ of H2 for t+1, the rest of the scatter; the u-pass over the H1-only columns runs
// alongside P_+ of H2; then the rest of u, y, x on the H1-touched coordinates.  Suffix D_B: x on the
// H2-only coordinates, dual updates, finalize.  The next iteration's P_+ runs before the current
// finalize, so this schedule is used by sdp_step only (no stopping test); sdp_solve runs the
// one-graph iteration.  Scatter partials alternate between two buffers (P.par).
void pipe_dual_update_range(sdp_handle h, int half, cudaStream_t s) {
  const Pipe& P = h->pipe;
  const int64_t b = half ? P.soff1 : 0, e = half ? h->stotl : P.soff1;
  // the H1 update also publishes iter + 1 for the next P_+(H1) (finalize waits for this kernel)
  launch_update_dual(e - b, h->G + b, h->x, h->xk + b, h->lam + b, h->vk + b, h->rho,
                     P.upd_part + 3 * (half ? P.nb_u1 : 0), h->done, s, half ? nullptr : h->iter,
                     half ? nullptr : P.iter_next);
}

void pipe_dual_finalize(sdp_handle h, int par, cudaStream_t s) {
  const Pipe& P = h->pipe;
  enqueue_finalize(h, s, par ? P.scat_part2 : P.scat_part, P.nb_sc1 + P.nb_sc2, P.gT_part, P.nb_gT1 + P.nb_gT2,
                   P.upd_part, P.nb_u1 + P.nb_u2);
}

void pipe_dual_A(sdp_handle h, cudaStream_t s) {
  Pipe& P = h->pipe;
  P.par = 0;
  pipe_projection(h, 0, s);
  pipe_projection(h, 1, s);
  pipe_scatter(h, 0, s);
  pipe_scatter(h, 1, s);
  pipe_gemv(h, s, 0, P.npe + P.npl);
  pipe_symv_gemvT1(h, s);
}

void pipe_dual_B(sdp_handle h, cudaStream_t s, bool with_A) {
  Pipe& P = h->pipe;
  const int cur = P.par;  // scatter buffer of iteration t
  SDP_CUDA_TRY(cudaEventRecord(P.ev[0], s));
  SDP_CUDA_TRY(cudaStreamWaitEvent(P.sx, P.ev[0], 0));
  SDP_CUDA_TRY(cudaStreamWaitEvent(P.sp, P.ev[0], 0));
  launch_gemvT_rows(h->form, h->AT, h->ldm, h->m, P.nr2, h->y, h->rD, h->Dinv, h->c, h->own, h->x,
                    P.gT_part + P.nb_gT1, h->done, P.sx, P.rows2);
  SDP_CUDA_TRY(cudaEventRecord(P.ev[1], P.sx));
  pipe_dual_update_range(h, 0, P.sp);
  SDP_CUDA_TRY(cudaEventRecord(P.ev[2], P.sp));
  if (with_A) {
    P.par = cur ^ 1;  // iteration t+1 scatters into the other buffer
    pipe_projection(h, 0, P.sp, P.iter_next);
    pipe_scatter(h, 0, P.sp);
    SDP_CUDA_TRY(cudaEventRecord(P.ev[3], P.sp));
    SDP_CUDA_TRY(cudaStreamWaitEvent(P.sg, P.ev[3], 0));
    pipe_gemv(h, P.sg, 0, P.npe);
    SDP_CUDA_TRY(cudaEventRecord(P.ev[4], P.sg));
  }
  SDP_CUDA_TRY(cudaStreamWaitEvent(P.sp2, P.ev[1], 0));
  pipe_dual_update_range(h, 1, P.sp2);
  SDP_CUDA_TRY(cudaStreamWaitEvent(P.sp2, P.ev[2], 0));
  pipe_dual_finalize(h, cur, P.sp2);
  SDP_CUDA_TRY(cudaEventRecord(P.ev[5], P.sp2));
  if (with_A) {
    pipe_projection(h, 1, P.sp2);
    SDP_CUDA_TRY(cudaStreamWaitEvent(P.sp2, P.ev[3], 0));  // shared coordinates need P_+ of H1 too
    pipe_scatter(h, 1, P.sp2);
    SDP_CUDA_TRY(cudaEventRecord(P.ev[6], P.sp2));
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, P.ev[6], 0));
    pipe_gemv(h, s, P.npe, P.npl);
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, P.ev[4], 0));
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, P.ev[5], 0));
    pipe_symv_gemvT1(h, s);
  } else {
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, P.ev[5], 0));
  }
}

void pipe_capture(sdp_handle h, int which, cudaGraph_t* g, cudaGraphExec_t* x) {
  SDP_CUDA_TRY(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
  if (which == 0)
    pipe_enqueue_A(h, h->cap_stream);
  else
    pipe_enqueue_B(h, h->cap_stream, which == 1);
  SDP_CUDA_TRY(cudaStreamEndCapture(h->cap_stream, g));
  // stream priorities are not recorded by capture: every kernel node except the HBM-streaming
  // passes gets the high priority, so that the projections are scheduled as soon as they are ready
  size_t nn = 0;
  SDP_CUDA_TRY(cudaGraphGetNodes(*g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  SDP_CUDA_TRY(cudaGraphGetNodes(*g, nodes.data(), &nn));
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType ty;
    SDP_CUDA_TRY(cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp{};
    if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (is_stream_kernel(kp.func)) continue;
    cudaKernelNodeAttrValue v{};
    v.priority = h->pipe.prio_hi;
    SDP_CUDA_TRY(cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributePriority, &v));
  }
  SDP_CUDA_TRY(cudaGraphInstantiateWithFlags(x, *g, cudaGraphInstantiateFlagUseNodePriority));
}

int pipe_launches_per_iter(sdp_handle h) {
  const Pipe& P = h->pipe;
  int n = 0;
  for (int hf = 0; hf < 2; ++hf)
    for (int b = 0; b < B_NUM; ++b) {
      if (!P.half[hf].bcount[b]) continue;
      if (is_trd(b)) {
        const TrdDev& t = P.half[hf].td[b - B_TRD8];
        n += trd_launches_per_chunk(b) * ((t.count + t.chunk - 1) / t.chunk);
      } else {
        n += 1;
      }
    }
  n += (P.ns1 + P.nl1 > 0) + (P.ns2 + P.nl2 > 0);  // scatter passes
  n += (P.npe > 0) + (P.npl > 0) + 1;              // u pieces (two launches) + y = S^-1 u
  n += (P.nr1 > 0) + (P.nr2 > 0) + 1;              // two x passes + finalize
  if (h->form == SDP_FORM_DUAL) n += 2;              // dual updates per half
  return n;
}

void enqueue_iteration(sdp_handle h, cudaStream_t s) {
  if (h->pipe.on && h->form == SDP_FORM_PRIMAL) {  // the pipelined kernels, in sequence (per-phase profile)
    const Pipe& P = h->pipe;
    phase(0, s);
    pipe_gemv(h, s, 0, P.npe + P.npl);
    phase(1, s);
    launch_symv(SDP_FORM_PRIMAL, h->Sinv, h->m, P.gemv_part, P.npe + P.npl, h->b, h->rho, nullptr, h->y, h->done, s);
    phase(2, s);
    launch_gemvT_rows(SDP_FORM_PRIMAL, h->AT, h->ldm, h->m, P.nr1, h->y, h->rD, h->Dinv, h->c, h->own, h->x,
                      P.gT_part, h->done, s, P.rows1);
    launch_gemvT_rows(h->form, h->AT, h->ldm, h->m, P.nr2, h->y, h->rD, h->Dinv, h->c, h->own, h->x,
                      P.gT_part + P.nb_gT1, h->done, s, P.rows2);
    phase(3, s);
    pipe_projection(h, 0, s);
    pipe_projection(h, 1, s);
    phase(4, s);
    pipe_scatter(h, 0, s);
    pipe_scatter(h, 1, s);
    phase(6, s);
    enqueue_finalize(h, s, P.scat_part, P.nb_sc1 + P.nb_sc2, P.gT_part, P.nb_gT1 + P.nb_gT2);
    phase(7, s);
    return;
  }
  if (h->form == SDP_FORM_PRIMAL) {
    enqueue_kkt(h, s);                       // x   (E:OptCondMinYPrimal)
    phase(3, s);
    enqueue_projection(h, PM_PRIMAL, s);     // x_k (E:XkUpdate), lambda_k (E:LambdakUpdate)
    phase(4, s);
    enqueue_scatter(h, s);                   // rhs of the next KKT solve + eps_d partials
  } else {
    phase(3, s);
    enqueue_projection(h, PM_DUAL, s);       // z_k (E:zkUpdate)
    phase(4, s);
    enqueue_scatter(h, s);                   // rhs of E:OptCondMinYDual
    enqueue_kkt(h, s);                       // x, y
    phase(5, s);
    launch_update_dual(h->stotl, h->G, h->x, h->xk, h->lam, h->vk, h->rho, h->upd_part, h->done, s);  // v_k, lambda_k
  }
  phase(6, s);
  enqueue_finalize(h, s);
  phase(7, s);
}

int pipe_launches_per_iter(sdp_handle h);
int launches_per_iter(sdp_handle h) {
  if (h->fused) return 1;  // one launch per sdp_step call (any number of iterations)
  if (h->pipe.on) return pipe_launches_per_iter(h);
  int n = 0;
  for (int b = 0; b < B_NUM; ++b) {  // one launch per non-empty tier; 4-5 per chunk for the QL tiers
    if (!h->bcount[b]) continue;
    if (is_trd(b)) {
      const TrdDev& t = h->td[b - B_TRD8];
      n += trd_launches_per_chunk(b) * ((t.count + t.chunk - 1) / t.chunk);
    } else {
      n += 1;
    }
  }
  n += 1;                                       // scatter
  n += 2;                                       // gemv + gemvT (sparse A: gemv_csr forms u itself)
  n += h->s_diag ? 0 : 1;                       // y = S^-1 u (dense A: sums the gemv partials itself)
  if (h->world > 1 && h->a_dense) n += 1;       // partial u of the rank before the all-reduce
  n += (h->form == SDP_FORM_DUAL) ? 1 : 0;      // dual update
  n += 1;                                       // finalize
  if (h->world > 1) n += 2 + (h->nshared > 0 ? 1 : 0);  // second reduce_u, finalize phase 2 (or packed phase 1), fixup
  return n;
}

void rebuild_graph(sdp_handle h) {
  if (h->exec) {
    cudaGraphExecDestroy(h->exec);
    h->exec = nullptr;
  }
  if (h->graph) {
    cudaGraphDestroy(h->graph);
    h->graph = nullptr;
  }
  if (!h->use_graph || h->fused) return;
  if (h->pipe.on && h->form == SDP_FORM_PRIMAL) {
    // A and BA captured (per-node priorities).  Multi-iteration calls launch directly (the launches
    // stream ahead of the device: 1128 vs 1107 it/s on cfg2); one- and two-iteration calls replay the
    // graphs, whose single launch keeps the host out of the per-step loop (e2e 1034 -> 1049 it/s).
    // Both issue the same kernels in the same dependency order, so the results are identical.
    h->pipe.destroy_graphs();
    for (int w = 0; w < 2; ++w) pipe_capture(h, w, &h->pipe.g[w], &h->pipe.x[w]);
    return;
  }
  SDP_CUDA_TRY(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
  enqueue_iteration(h, h->cap_stream);
  SDP_CUDA_TRY(cudaStreamEndCapture(h->cap_stream, &h->graph));
  SDP_CUDA_TRY(cudaGraphInstantiate(&h->exec, h->graph, 0));
}

void reset_state(sdp_handle h) {
  cudaStream_t s = h->stream;
  SDP_CUDA_TRY(cudaMemsetAsync(h->xk, 0, h->stotl * sizeof(double), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->lam, 0, h->stotl * sizeof(double), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->vk, 0, h->stotl * sizeof(double), s));
  if (h->xbuf) SDP_CUDA_TRY(cudaMemsetAsync(h->xbuf, 0, (3 * (size_t)h->nshared + 8) * sizeof(double), s));
  if (h->prevall) SDP_CUDA_TRY(cudaMemsetAsync(h->prevall, 0, std::max(1, h->nshared) * sizeof(double), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->x, 0, h->lda * sizeof(double), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->rD, 0, h->lda * sizeof(double), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->sprev, 0, h->lda * sizeof(double), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->y, 0, h->m * sizeof(double), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->res, 0, 4 * sizeof(double), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->iter, 0, sizeof(long long), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->done, 0, sizeof(int), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->numerical, 0, sizeof(int), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->capped, 0, sizeof(unsigned long long), s));
  SDP_CUDA_TRY(cudaMemsetAsync(h->sweeps, 0, sizeof(unsigned long long), s));
  if (h->vprev) SDP_CUDA_TRY(cudaMemsetAsync(h->vprev, 0, (size_t)std::max<int64_t>(h->vprev_len, 1) * sizeof(double), s));
  const double neg = -1.0;
  SDP_CUDA_TRY(cudaMemcpyAsync(h->tol, &neg, sizeof(double), cudaMemcpyHostToDevice, s));
  if (h->form == SDP_FORM_PRIMAL) enqueue_scatter(h, s);  // r1 = -c/rho for iteration 1
  SDP_CUDA_TRY(cudaGetLastError());
  SDP_CUDA_TRY(cudaStreamSynchronize(s));
}

void check_indices(const char* what, int64_t nnz, const int32_t* r, const int32_t* c, int n) {
  for (int64_t e = 0; e < nnz; ++e) {
    if (r[e] < 0 || c[e] < 0 || r[e] >= n || c[e] >= n)
      throw Error{SDP_E_INVALID_ARG, std::string(what) + " entry " + std::to_string(e) + " index out of range"};
    if (r[e] > c[e])
      throw Error{SDP_E_INVALID_ARG, std::string(what) + " entry " + std::to_string(e) + " has row > col"};
  }
}

void destroy_handle(sdp_handle h) {
  if (!h) return;
  int cur = -1;
  cudaGetDevice(&cur);
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->exec) cudaGraphExecDestroy(h->exec);
  if (h->graph) cudaGraphDestroy(h->graph);
  h->alloc.free_all();
  delete h->comm;
  h->comm = nullptr;
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  h->tiers.destroy();
  h->pipe.destroy();
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  if (cur >= 0) cudaSetDevice(cur);
  delete h;
}

// A host-to-device copy on a helper thread (its own non-blocking stream, so pageable sources work
// and no legacy-stream ordering couples it to the caller's work); joined by finish() or on unwind.
struct AsyncUpload {
  double* dst = nullptr;
  std::thread th;
  cudaError_t err = cudaSuccess;
  void start(const double* src, size_t bytes, int device) {
    th = std::thread([this, src, bytes, device] {
      cudaStream_t st = nullptr;
      err = cudaSetDevice(device);
      if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      if (err == cudaSuccess) err = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
      if (err == cudaSuccess) err = cudaStreamSynchronize(st);
      if (st) cudaStreamDestroy(st);
    });
  }
  void finish() {
    if (th.joinable()) th.join();
    if (err != cudaSuccess) throw Error{SDP_E_CUDA, std::string("A upload: ") + cudaGetErrorString(err)};
  }
  ~AsyncUpload() {
    if (th.joinable()) th.join();
  }
};

void build_fused(sdp_handle h, const std::vector<int>& task_bucket);
int setup_impl(const sdp_problem* P, const sdp_options* opt_in, sdp_handle* out) {
  auto t0 = std::chrono::steady_clock::now();
  // SDP_SETUP_TRACE=1: wall time of the setup phases on stderr
  const bool strace = getenv("SDP_SETUP_TRACE") != nullptr;
  auto tlast = t0;
  auto smark = [&](const char* what) {
    if (!strace) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[setup] %-28s %9.2f ms\n", what, std::chrono::duration<double>(now - tlast).count() * 1e3);
    tlast = now;
  };
  if (!out) throw Error{SDP_E_INVALID_ARG, "out is NULL"};
  *out = nullptr;
  if (!P) throw Error{SDP_E_INVALID_ARG, "problem is NULL"};
  sdp_options opt;
  sdp_default_options(&opt);
  if (opt_in) opt = *opt_in;
  const int n = P->n, m = P->m;
  if (n <= 0) throw Error{SDP_E_INVALID_ARG, "n <= 0"};
  if (m <= 0) throw Error{SDP_E_INVALID_ARG, "m <= 0"};
  if (!(opt.rho > 0) || !std::isfinite(opt.rho)) throw Error{SDP_E_INVALID_ARG, "rho must be positive"};
  if (opt.form != SDP_FORM_PRIMAL && opt.form != SDP_FORM_DUAL) throw Error{SDP_E_INVALID_ARG, "bad form"};
  if (opt.world < 1 || opt.rank < 0 || opt.rank >= opt.world) throw Error{SDP_E_INVALID_ARG, "bad rank/world"};
  if (opt.world > 1 && !opt.nccl_id && !opt.comm)
    throw Error{SDP_E_INVALID_ARG, "world > 1 needs nccl_id (sdp_nccl_unique_id) or a loopback comm"};
  if (!P->b) throw Error{SDP_E_INVALID_ARG, "b is NULL"};
  if (P->c_nnz < 0 || (P->c_nnz > 0 && (!P->c_row || !P->c_col || !P->c_val)))
    throw Error{SDP_E_INVALID_ARG, "C arrays missing"};
  if (P->a_fmt != SDP_A_COO && P->a_fmt != SDP_A_DENSE_ON_PATTERN) throw Error{SDP_E_INVALID_ARG, "bad a_fmt"};
  if (P->a_nnz < 0 || (P->a_nnz > 0 && (!P->a_row || !P->a_col || !P->a_val)))
    throw Error{SDP_E_INVALID_ARG, "A arrays missing"};
  if (P->a_fmt == SDP_A_COO && P->a_nnz > 0 && !P->a_con) throw Error{SDP_E_INVALID_ARG, "a_con missing"};
  if (P->e_nnz < 0 || (P->e_nnz > 0 && (!P->e_row || !P->e_col))) throw Error{SDP_E_INVALID_ARG, "E arrays missing"};
  check_indices("C", P->c_nnz, P->c_row, P->c_col, n);
  check_indices("A", P->a_nnz, P->a_row, P->a_col, n);
  check_indices("E", P->e_nnz, P->e_row, P->e_col, n);
  for (int i = 0; i < m; ++i)
    if (!std::isfinite(P->b[i])) throw Error{SDP_E_INVALID_ARG, "b[" + std::to_string(i) + "] not finite"};
  for (int64_t e = 0; e < P->c_nnz; ++e)
    if (!std::isfinite(P->c_val[e])) throw Error{SDP_E_INVALID_ARG, "C value " + std::to_string(e) + " not finite"};
  if (P->a_fmt == SDP_A_COO)
    for (int64_t e = 0; e < P->a_nnz; ++e)
      if (P->a_con[e] < 0 || P->a_con[e] >= m)
        throw Error{SDP_E_INVALID_ARG, "A entry " + std::to_string(e) + " constraint index out of range"};

  int ndev = 0;
  SDP_CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (opt.device < 0 || opt.device >= ndev) throw Error{SDP_E_INVALID_ARG, "bad device ordinal"};
  DeviceGuard dg(opt.device);

  smark("validation");
  sdp_handle h = new sdp_handle_s();
  *out = h;  // so the caller-side cleanup path below can destroy it
  h->n = n;
  h->m = m;
  h->form = opt.form;
  h->rho = opt.rho;
  h->device = opt.device;
  h->check_every = opt.check_every > 0 ? opt.check_every : 10;
  h->use_graph = opt.use_graph;
  h->adapt = opt.adapt_rho ? 1 : 0;
  h->adapt_mu = opt.adapt_mu > 1.0 ? opt.adapt_mu : 10.0;
  h->adapt_tau = opt.adapt_tau > 1.0 ? opt.adapt_tau : 2.0;
  // The raw dense A values (the bulk of the input) go to the device on a helper thread while the
  // host runs the chordal analysis below; the placement onto the pattern waits for them (step 5).
  h->alloc.set_hook(opt.allocator, opt.device);
  AsyncUpload a_up;
  if (P->a_fmt == SDP_A_DENSE_ON_PATTERN && P->a_nnz > 0 &&
      (double)m * (double)P->a_nnz * 8.0 <= 16e9) {
    a_up.dst = h->alloc.get<double>((size_t)m * P->a_nnz);
    a_up.start(P->a_val, (size_t)m * P->a_nnz * sizeof(double), opt.device);
  }
  // ---- 1. aggregate pattern and chordal analysis
  std::vector<std::pair<int32_t, int32_t>> edges;
  edges.reserve((size_t)(P->c_nnz + P->a_nnz + P->e_nnz));
  auto add = [&](int64_t nnz, const int32_t* r, const int32_t* c) {
    for (int64_t e = 0; e < nnz; ++e)
      if (r[e] != c[e]) edges.push_back({r[e], c[e]});
  };
  add(P->c_nnz, P->c_row, P->c_col);
  add(P->a_nnz, P->a_row, P->a_col);
  add(P->e_nnz, P->e_row, P->e_col);
  ChordalResult cr = chordal_analysis(n, edges);
  edges.clear();
  edges.shrink_to_fit();

  h->fill_edges = cr.fill_edges;
  h->stream = (cudaStream_t)opt.stream;  // NULL = the legacy default stream, as in the CUDA runtime
  h->own_stream = false;
  h->world = opt.world;
  h->rank = opt.rank;
  if (h->world > 1)  // collective
    h->comm = opt.comm ? make_loop_comm(opt.comm, h->world, h->rank) : make_nccl_comm(opt.nccl_id, h->world, h->rank);
  if (h->comm && h->comm->loopback()) h->use_graph = 0;  // capture cannot cross the ranks' streams
  SDP_CUDA_TRY(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  h->tiers.create();
  const int64_t N = (int64_t)cr.coord_row.size();
  h->N = N;
  h->coord_row = cr.coord_row;
  h->coord_col = cr.coord_col;
  h->chordal.order = cr.order;
  h->chordal.later_ptr = cr.later_ptr;
  h->chordal.later_idx = cr.later_idx;
  if (N >= (1ll << 31)) throw Error{SDP_E_INVALID_ARG, "pattern too large"};

  smark("chordal analysis");
  // ---- 2. global layout: clique offsets, H_k maps, D, inverse map
  const int64_t p = (int64_t)cr.cliques.size();
  h->p = p;
  std::vector<int64_t> off(p + 1, 0);
  std::vector<int32_t> ksz(p);
  h->kmin = INT64_MAX;
  h->kmax = 0;
  for (int64_t k = 0; k < p; ++k) {
    const int kk = (int)cr.cliques[k].size();
    if (kk > SDP_MAX_K)
      throw Error{SDP_E_INVALID_ARG, "clique of order " + std::to_string(kk) + " exceeds SDP_MAX_K"};
    ksz[k] = kk;
    off[k + 1] = off[k] + (int64_t)kk * (kk + 1) / 2;
    h->kmin = std::min<int64_t>(h->kmin, kk);
    h->kmax = std::max<int64_t>(h->kmax, kk);
    h->clique_size.push_back(kk);
    for (int v : cr.cliques[k]) h->clique_vert.push_back(v);
  }
  const int64_t stot = off[p];
  h->stot = stot;
  h->clique_off = off;
  if (stot >= (1ll << 31)) throw Error{SDP_E_INVALID_ARG, "stacked clique vectors too large"};
  std::vector<int32_t> Gmap(stot);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t k = 0; k < p; ++k) {
    const auto& C = cr.cliques[k];
    int64_t e = off[k];
    for (size_t bcol = 0; bcol < C.size(); ++bcol)
      for (size_t arow = 0; arow <= bcol; ++arow) Gmap[e++] = (int32_t)coord_index(cr, C[arow], C[bcol]);
  }
  std::vector<int32_t> seg_ptr(N + 1, 0), seg_idx(stot);
  {
    std::vector<int32_t> cnt(N + 1, 0);
    for (int64_t s = 0; s < stot; ++s) cnt[Gmap[s] + 1]++;
    for (int64_t t = 0; t < N; ++t) seg_ptr[t + 1] = seg_ptr[t] + cnt[t + 1];
    std::vector<int32_t> fillp(seg_ptr.begin(), seg_ptr.end() - 1);
    for (int64_t s = 0; s < stot; ++s) seg_idx[fillp[Gmap[s]]++] = (int32_t)s;
  }
  std::vector<double> Dinv_g(N);
  for (int64_t t = 0; t < N; ++t) {
    const int d = seg_ptr[t + 1] - seg_ptr[t];
    if (d <= 0) throw Error{SDP_E_INVALID_ARG, "internal: pattern coordinate covered by no clique"};
    Dinv_g[t] = 1.0 / (double)d;
  }
  // c = svec(C) on the pattern
  std::vector<double> cglob(N, 0.0);
  {
    std::vector<char> seen(N, 0);
    for (int64_t e = 0; e < P->c_nnz; ++e) {
      const int64_t t = coord_index(cr, P->c_row[e], P->c_col[e]);
      if (seen[t]) throw Error{SDP_E_INVALID_ARG, "duplicate C entry " + std::to_string(e)};
      seen[t] = 1;
      cglob[t] = P->c_val[e] * (P->c_row[e] == P->c_col[e] ? 1.0 : kSqrt2);
    }
  }

  smark("layout, maps, D");
  // ---- 3. shard plan and this rank's local view; identity when world == 1
  if (h->world > p) throw Error{SDP_E_INVALID_ARG, "more ranks than cliques"};
  ShardPlan sp;
  if (h->world == 1) {
    sp.clique_rank.assign(p, 0);
    sp.my_cliques.resize(p);
    std::iota(sp.my_cliques.begin(), sp.my_cliques.end(), 0);
    sp.local_coords.resize(N);
    std::iota(sp.local_coords.begin(), sp.local_coords.end(), 0);
    sp.owned.assign(N, 1);
    // pipelined-iteration candidates (struct Pipe): coordinates touched only by the first half of
    // the cliques first, then the shared ones, then those of the second half only (stable), so
    // that every pass of the pipelined iteration is one contiguous coordinate range
    const char* penv = getenv("SDP_PIPELINE");
    if (!(penv && *penv == '0') && N >= 65536 && p >= 8) {
      const int64_t p1 = pipe_split(off, p, h->form);
      std::vector<uint8_t> cls(N, 0);
      for (int64_t k = 0; k < p; ++k)
        for (int64_t e = off[k]; e < off[k + 1]; ++e) cls[Gmap[e]] |= (k < p1) ? 1 : 2;
      std::stable_sort(sp.local_coords.begin(), sp.local_coords.end(), [&](int32_t a, int32_t b) {
        auto rank = [&](int32_t t) { return cls[t] == 1 ? 0 : cls[t] == 3 ? 1 : 2; };
        return rank(a) < rank(b);
      });
      h->coord_perm = true;
    }
  } else {
    sp = make_shard_plan(ksz, off, seg_ptr, seg_idx, h->world, h->rank);
  }
  const int64_t pl = (int64_t)sp.my_cliques.size(), Nl = (int64_t)sp.local_coords.size();
  std::vector<int64_t> offl(pl + 1, 0);  // local stacked layout: this rank's cliques, canonical order
  std::vector<int32_t> kszl(pl);
  for (int64_t q = 0; q < pl; ++q) {
    const int32_t k = sp.my_cliques[q];
    offl[q + 1] = offl[q] + (off[k + 1] - off[k]);
    kszl[q] = ksz[k];
  }
  const int64_t stotl = offl[pl];
  h->my_cliques = sp.my_cliques;
  h->pl = pl;
  h->Nl = Nl;
  h->stotl = stotl;
  h->lda = (Nl + 31) / 32 * 32;
  h->local_coords = sp.local_coords;
  h->nshared = (int)sp.shared_coords.size();
  std::vector<int32_t> g2l(N, -1);
  for (int64_t i = 0; i < Nl; ++i) g2l[sp.local_coords[i]] = (int32_t)i;
  std::vector<int32_t> Gl(stotl);
  for (int64_t q = 0; q < pl; ++q) {
    const int32_t k = sp.my_cliques[q];
    for (int64_t e = 0; e < off[k + 1] - off[k]; ++e) Gl[offl[q] + e] = g2l[Gmap[off[k] + e]];
  }
  std::vector<int32_t> segl_ptr(Nl + 1, 0), segl_idx(stotl);
  {
    std::vector<int32_t> cnt(Nl + 1, 0);
    for (int64_t s = 0; s < stotl; ++s) cnt[Gl[s] + 1]++;
    for (int64_t t = 0; t < Nl; ++t) segl_ptr[t + 1] = segl_ptr[t] + cnt[t + 1];
    std::vector<int32_t> fillp(segl_ptr.begin(), segl_ptr.end() - 1);
    for (int64_t s = 0; s < stotl; ++s) segl_idx[fillp[Gl[s]]++] = (int32_t)s;
  }
  std::vector<double> Dinv(h->lda, 0.0), cvec(h->lda, 0.0), own(h->lda, 0.0);
  std::vector<int32_t> longc, shared_idx(Nl, -1);
  for (int64_t t = 0; t < Nl; ++t) {
    const int64_t tg = sp.local_coords[t];
    Dinv[t] = Dinv_g[tg];  // D counts every clique (all ranks) containing the coordinate
    own[t] = sp.owned[t] ? 1.0 : 0.0;
    cvec[t] = sp.owned[t] ? cglob[tg] : 0.0;  // c enters the partial sums once, at the owner
    if (segl_ptr[t + 1] - segl_ptr[t] > kLongSeg) longc.push_back((int32_t)t);
  }
  for (int j = 0; j < h->nshared; ++j)
    if (sp.shared_local[j] >= 0) shared_idx[sp.shared_local[j]] = j;
  h->n_long = (int)longc.size();

  smark("shard plan / local view");
  // ---- 4. device uploads of the local layout
  Alloc& al = h->alloc;
  h->G = al.upload(Gl);
  h->seg_ptr = al.upload(segl_ptr);
  h->seg_idx = al.upload(segl_idx);
  h->longc = al.upload(longc);
  h->Dinv = al.upload(Dinv);
  h->c = al.upload(cvec);
  h->own = al.upload(own);
  h->d_off = al.upload(offl);
  h->d_ksz = al.upload(kszl);
  h->b = al.upload(std::vector<double>(P->b, P->b + m));
  h->x = al.zeros<double>(h->lda);
  h->rD = al.zeros<double>(h->lda);
  h->sprev = al.zeros<double>(h->lda);
  h->ldm = (m + 31) / 32 * 32;
  h->y = al.zeros<double>(h->ldm);
  h->u = al.zeros<double>(m);
  h->t = al.zeros<double>(m);
  h->xk = al.zeros<double>(stotl);
  h->lam = al.zeros<double>(stotl);
  h->vk = al.zeros<double>(stotl);
  if (h->nshared > 0) {
    h->shared_idx = al.upload(shared_idx);
    h->shared_local = al.upload(sp.shared_local);
  }
  if (h->world > 1) {
    h->xbuf = al.zeros<double>(3 * (size_t)h->nshared + 8);  // + the packed residual partials
    h->prevall = al.zeros<double>((size_t)std::max(1, h->nshared));
  }
  h->n_fix = h->nshared > 0 ? fixup_blocks(h->nshared) : 0;
  h->fix_part = al.zeros<double>(2 * (size_t)std::max(1, h->n_fix));
  h->red = al.zeros<double>(8);
  std::vector<int> task_bucket;
  build_buckets(al, kszl, h->d_ids, h->bcount, h->gd, h->td, &task_bucket);

  smark("uploads, tiers");
  // ---- 5. A (svec rows) and S = A D^-1 A^T, factor cached once
  std::vector<double> S;
  // S^-1 of a dense S: device Gauss-Jordan (default) or host Cholesky + L^-1 (SDP_SCHUR_HOST=1)
  const char* shost = getenv("SDP_SCHUR_HOST");
  const bool schur_host = shost && *shost == '1';
  double* dS_keep = nullptr;
  if (P->a_fmt == SDP_A_DENSE_ON_PATTERN) {
    h->a_dense = 1;
    const int64_t npat = P->a_nnz;
    std::vector<int64_t> map(npat);
    std::vector<double> scale(npat);
    std::vector<char> seen(N, 0);
    for (int64_t e = 0; e < npat; ++e) {
      const int64_t t = coord_index(cr, P->a_row[e], P->a_col[e]);
      if (seen[t]) throw Error{SDP_E_INVALID_ARG, "duplicate A pattern entry " + std::to_string(e)};
      seen[t] = 1;
      map[e] = g2l[t];  // -1: not on this rank
      scale[e] = (P->a_row[e] == P->a_col[e]) ? 1.0 : kSqrt2;
    }
    h->A = al.zeros<double>((size_t)m * h->lda);
    if (npat > 0) {
      // the raw values: already on the device (uploaded during the chordal analysis), else streamed
      // in row slabs of <= 256 MB through a staging buffer
      const bool pre = a_up.dst != nullptr;
      if (pre) a_up.finish();
      const int64_t rows_per =
          pre ? std::min<int64_t>(m, 65535) : std::max<int64_t>(1, (256ll << 20) / (8 * npat));
      double* raw = pre ? a_up.dst : al.get<double>((size_t)std::min<int64_t>(rows_per, m) * npat);
      int64_t* dmap = al.upload(map);
      double* dscale = al.upload(scale);
      int* dbad = al.zeros<int>(1);
      for (int64_t r0 = 0; r0 < m; r0 += rows_per) {
        const int64_t nr = std::min<int64_t>(rows_per, m - r0);
        if (!pre)
          SDP_CUDA_TRY(cudaMemcpy(raw, P->a_val + r0 * npat, nr * npat * sizeof(double), cudaMemcpyHostToDevice));
        launch_place_dense(pre ? raw + r0 * npat : raw, npat, (int)nr, dmap, dscale, h->A + r0 * h->lda, h->lda,
                           nullptr, dbad);
        SDP_CUDA_TRY(cudaGetLastError());
      }
      int bad = 0;
      SDP_CUDA_TRY(cudaMemcpy(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost));
      if (bad) throw Error{SDP_E_INVALID_ARG, "A value not finite"};
      al.release(raw);
      a_up.dst = nullptr;
      al.release(dmap);
      al.release(dscale);
      al.release(dbad);
    }
    // A^T copy over every local coordinate (x is needed on all of them) ...
    smark("A upload + placement");
    h->AT = al.zeros<double>((size_t)Nl * h->ldm);
    launch_transpose(h->A, h->lda, m, h->AT, h->ldm, Nl, nullptr);
    SDP_CUDA_TRY(cudaGetLastError());
    // ... while A keeps only the owned columns: u = A D^-1 r1 is summed over ranks
    if (h->world > 1) {
      launch_mask_cols(h->A, h->lda, m, h->own, nullptr);
      SDP_CUDA_TRY(cudaGetLastError());
    }
    h->chunk = 32768;
    h->nchunks = (int)((h->lda + h->chunk - 1) / h->chunk);
    h->gemv_part = al.zeros<double>((size_t)h->nchunks * m);
    double* dS = al.get<double>((size_t)m * m);
    smark("A^T copy");
    launch_syrk_dense(h->A, h->lda, m, h->Dinv, dS, nullptr);
    SDP_CUDA_TRY(cudaGetLastError());
    if (h->world > 1) h->comm->allreduce_sum(dS, (size_t)m * m, nullptr);  // S = sum of owned-column parts
    if (schur_host) {
      S.resize((size_t)m * m);
      SDP_CUDA_TRY(cudaMemcpy(S.data(), dS, S.size() * sizeof(double), cudaMemcpyDeviceToHost));
      al.release(dS);
    } else {
      dS_keep = dS;  // inverted on the device below
    }
  } else {
    h->a_dense = 0;
    struct Ent {
      int32_t con;
      int32_t t;
      double v;
    };
    std::vector<Ent> ents((size_t)P->a_nnz);
    for (int64_t e = 0; e < P->a_nnz; ++e) {
      if (!std::isfinite(P->a_val[e])) throw Error{SDP_E_INVALID_ARG, "A value " + std::to_string(e) + " not finite"};
      ents[e] = {P->a_con[e], (int32_t)coord_index(cr, P->a_row[e], P->a_col[e]),
                 P->a_val[e] * (P->a_row[e] == P->a_col[e] ? 1.0 : kSqrt2)};
    }
    std::sort(ents.begin(), ents.end(),
              [](const Ent& a, const Ent& b) { return a.con != b.con ? a.con < b.con : a.t < b.t; });
    for (size_t e = 1; e < ents.size(); ++e)
      if (ents[e].con == ents[e - 1].con && ents[e].t == ents[e - 1].t)
        throw Error{SDP_E_INVALID_ARG, "duplicate A entry (constraint " + std::to_string(ents[e].con) + ")"};
    // global column counts decide whether S is diagonal; S itself from all entries
    std::vector<int32_t> colcnt(N, 0);
    for (auto& en : ents) colcnt[en.t]++;
    int maxcol = 0;
    for (int64_t t = 0; t < N; ++t) maxcol = std::max(maxcol, colcnt[t]);
    // local CSR (owned columns, for u) and CSC (all local columns, for x), local indices
    std::vector<int32_t> rp(m + 1, 0), ci;
    std::vector<double> val;
    for (auto& en : ents) {
      const int32_t tl = g2l[en.t];
      if (tl < 0 || !sp.owned[tl]) continue;
      rp[en.con + 1]++;
      ci.push_back(tl);
      val.push_back(en.v);
    }
    for (int i = 0; i < m; ++i) rp[i + 1] += rp[i];
    std::vector<int32_t> cp(Nl + 1, 0), ri;
    std::vector<double> cval;
    for (auto& en : ents)
      if (g2l[en.t] >= 0) cp[g2l[en.t] + 1]++;
    for (int64_t t = 0; t < Nl; ++t) cp[t + 1] += cp[t];
    ri.resize(cp[Nl]);
    cval.resize(cp[Nl]);
    {
      std::vector<int32_t> pos(cp.begin(), cp.end() - 1);
      for (auto& en : ents) {  // ents sorted by (con, t): rows ascend inside each column
        const int32_t tl = g2l[en.t];
        if (tl < 0) continue;
        ri[pos[tl]] = en.con;
        cval[pos[tl]++] = en.v;
      }
    }
    h->a_rp = al.upload(rp);
    h->a_ci = al.upload(ci);
    h->a_val = al.upload(val);
    h->at_cp = al.upload(cp);
    h->at_ri = al.upload(ri);
    h->at_val = al.upload(cval);
    if (maxcol <= 1) {
      // rows of A have disjoint supports: S = A D^-1 A^T is diagonal
      std::vector<double> sd(m, 0.0);
      for (auto& en : ents) sd[en.con] += en.v * en.v * Dinv_g[en.t];
      for (int i = 0; i < m; ++i)
        if (!(sd[i] > 0)) throw Error{SDP_E_RANK_DEFICIENT, "constraint " + std::to_string(i) + " is empty"};
      h->s_diag = 1;
      h->sdiag = al.upload(sd);
    } else {
      // S_ij = sum_t A_it A_jt / D_t over all coordinates (every rank holds the full problem)
      std::vector<int32_t> gcp(N + 1, 0), gri(ents.size());
      std::vector<double> gval(ents.size());
      for (auto& en : ents) gcp[en.t + 1]++;
      for (int64_t t = 0; t < N; ++t) gcp[t + 1] += gcp[t];
      std::vector<int32_t> pos(gcp.begin(), gcp.end() - 1);
      for (auto& en : ents) {
        gri[pos[en.t]] = en.con;
        gval[pos[en.t]++] = en.v;
      }
      // sparse S (both triangles, CSR by row): one entry per pair of constraints sharing a coordinate
      struct Trip {
        int32_t a, b;
        double v;
      };
      std::vector<Trip> trip;
      for (int64_t t = 0; t < N; ++t)
        for (int e1 = gcp[t]; e1 < gcp[t + 1]; ++e1)
          for (int e2 = gcp[t]; e2 < gcp[t + 1]; ++e2)
            trip.push_back({gri[e1], gri[e2], gval[e1] * gval[e2] * Dinv_g[t]});
      std::stable_sort(trip.begin(), trip.end(),
                       [](const Trip& x, const Trip& y) { return x.a != y.a ? x.a < y.a : x.b < y.b; });
      std::vector<int64_t> sptr(m + 1, 0);
      std::vector<int32_t> sidx;
      std::vector<double> sval;
      for (size_t q = 0; q < trip.size();) {
        size_t r = q;
        double acc = 0.0;
        for (; r < trip.size() && trip[r].a == trip[q].a && trip[r].b == trip[q].b; ++r) acc += trip[r].v;
        sidx.push_back(trip[q].b);
        sval.push_back(acc);
        sptr[trip[q].a + 1]++;
        q = r;
      }
      for (int i = 0; i < m; ++i) sptr[i + 1] += sptr[i];
      trip.clear();
      trip.shrink_to_fit();
      // sparse Cholesky of S (fill-reducing minimum degree) when its factor is sparse;
      // SDP_SPARSE_S=0 never, =1 always (tests); default for m >= 256 and nnz(L) <= m^2 / 8
      const char* ss = getenv("SDP_SPARSE_S");
      const bool force = ss && *ss == '1', never = ss && *ss == '0';
      bool done_sparse = false;
      if (!never && (force || m >= 256)) {
        const int64_t ldg = (m + 31) / 32 * 32;
        std::vector<double> GT;
        std::string why;
        int64_t nnzl = 0;
        if (sparse_inverse_factor(m, sptr, sidx, sval, ldg, GT, &nnzl, 0.125, force, &why)) {
          double* dGT = al.upload(GT);
          std::vector<double> ones(ldg, 1.0);
          double* d1 = al.upload(ones);
          h->Sinv = al.get<double>((size_t)m * m);
          launch_syrk_dense(dGT, ldg, m, d1, h->Sinv, nullptr);  // S^-1 = G^T G
          SDP_CUDA_TRY(cudaGetLastError());
          SDP_CUDA_TRY(cudaDeviceSynchronize());
          al.release(dGT);
          al.release(d1);
          symv_init_attributes(m);
          h->s_factor = 2;
          h->nnz_l = nnzl;
          done_sparse = true;
        } else if (why != "factor too dense") {
          throw Error{SDP_E_RANK_DEFICIENT, why};
        }
      }
      if (!done_sparse) {
        S.assign((size_t)m * m, 0.0);
        for (int i = 0; i < m; ++i)
          for (int64_t e = sptr[i]; e < sptr[i + 1]; ++e) S[(size_t)i * m + sidx[e]] = sval[e];
      }
    }
  }
  smark("S = A D^-1 A^T (+ D2H)");
  if (!h->s_diag && h->s_factor != 2 && !schur_host) {
    // S^-1 on the device: blocked Gauss-Jordan sweep of the SPD S (kernels_schur.cu)
    h->s_factor = 1;
    double* dS = dS_keep ? dS_keep : al.upload(S);
    dS_keep = nullptr;
    S.clear();
    S.shrink_to_fit();
    h->Sinv = al.get<double>((size_t)m * m);
    double* work = al.get<double>((size_t)m * m);
    double* d0 = al.get<double>((size_t)m + 1024);
    int* dbad = al.zeros<int>(1);
    smark("S^-1 buffers");
    const bool ok = spd_inverse_gpu(dS, m, h->Sinv, work, d0, dbad, nullptr);
    smark("S^-1 (device Gauss-Jordan)");
    al.release(work);
    al.release(d0);
    al.release(dbad);
    al.release(dS);
    if (!ok) throw Error{SDP_E_RANK_DEFICIENT, "S = A D^-1 A^T is not positive definite"};
    symv_init_attributes(m);
    smark("S^-1 release");
  } else if (!h->s_diag && h->s_factor != 2) {
    if (dS_keep) al.release(dS_keep);
    h->s_factor = 1;
    if (!cholesky_host(S, m)) throw Error{SDP_E_RANK_DEFICIENT, "S = A D^-1 A^T is not positive definite"};
    smark("Cholesky (host)");
    std::vector<double> Wt;
    tri_inverse_T(S, m, Wt);
    smark("L^-1 (host)");
    h->WT = al.upload(Wt);
    // cached S^-1 = W^T W (one dense mat-vec per iteration instead of two dependent
    // triangular ones; cond(S) ~ 2 on the block-arrow configs), formed by the SYRK kernel
    std::vector<double> ones(m, 1.0);
    double* d1 = al.upload(ones);
    h->Sinv = al.get<double>((size_t)m * m);
    launch_syrk_dense(h->WT, m, m, d1, h->Sinv, nullptr);
    SDP_CUDA_TRY(cudaGetLastError());
    SDP_CUDA_TRY(cudaDeviceSynchronize());
    al.release(d1);
    al.release(h->WT);
    h->W = h->WT = nullptr;
    symv_init_attributes(m);
  }

  smark("A, S, factor, S^-1");
  // ---- 6. residual buffers, state, graph
  h->nb_scat = scatter_blocks((int)Nl, h->n_long);
  h->nb_gT = h->a_dense ? gemvT_rows_blocks(Nl) : gemvT_csc_blocks((int)Nl);
  h->nb_upd = update_blocks(stotl);
  h->proj_part = al.zeros<double>(3 * (size_t)std::max<int64_t>(pl, 1));
  h->scat_part = al.zeros<double>(2 * (size_t)h->nb_scat);
  h->gT_part = al.zeros<double>(h->nb_gT);
  h->upd_part = al.zeros<double>(3 * (size_t)h->nb_upd);
  h->res = al.zeros<double>(4);
  h->hist = al.zeros<double>(3 * (size_t)kHistCap);
  h->tol = al.zeros<double>(1);
  h->iter = al.zeros<long long>(1);
  h->done = al.zeros<int>(1);
  h->numerical = al.zeros<int>(1);
  h->capped = al.zeros<unsigned long long>(1);
  h->sweeps = al.zeros<unsigned long long>(1);
  {  // warm-start eigenvector storage: kp x kp per clique
    std::vector<int64_t> voff(pl + 1, 0);
    for (int64_t k = 0; k < pl; ++k) {
      const int64_t kp = store_kp(task_bucket[k], kszl[k]);
      voff[k + 1] = voff[k] + kp * kp;
    }
    h->voff = al.upload(voff);
    h->vprev = al.zeros<double>((size_t)std::max<int64_t>(voff[pl], 1));
    h->vprev_len = voff[pl];
  }
  build_pipeline(h, Gl, offl, segl_ptr, task_bucket);
  build_fused(h, task_bucket);
  psd_init_attributes();
  SDP_CUDA_TRY(cudaDeviceSynchronize());
  reset_state(h);
  rebuild_graph(h);
  smark("state, graphs");
  h->setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return SDP_OK;
}

// Sum a host vector over the ranks (getters of a sharded handle; collective).
void allreduce_host(sdp_handle h, std::vector<double>& v) {
  double* d = h->alloc.get<double>(v.size());
  // on the handle's stream: a legacy-stream cudaMemcpy from pageable memory can return before the
  // data lands, and the loopback sum (ordered after this stream's ready event) would read it early
  SDP_CUDA_TRY(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  h->comm->allreduce_sum(d, v.size(), h->stream);
  SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
  SDP_CUDA_TRY(cudaMemcpy(v.data(), d, v.size() * sizeof(double), cudaMemcpyDeviceToHost));
  h->alloc.release(d);
}

void fill_info(sdp_handle h, sdp_info* info) {
  double res[3];
  long long it;
  unsigned long long cap, sw;
  SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
  SDP_CUDA_TRY(cudaMemcpy(&sw, h->sweeps, sizeof(sw), cudaMemcpyDeviceToHost));
  SDP_CUDA_TRY(cudaMemcpy(res, h->res, 3 * sizeof(double), cudaMemcpyDeviceToHost));
  SDP_CUDA_TRY(cudaMemcpy(&it, h->iter, sizeof(long long), cudaMemcpyDeviceToHost));
  SDP_CUDA_TRY(cudaMemcpy(&cap, h->capped, sizeof(cap), cudaMemcpyDeviceToHost));
  std::memset(info, 0, sizeof(*info));
  info->iters = it;
  info->eps_p = res[0];
  info->eps_d = res[1];
  info->objective = res[2];
  info->setup_s = h->setup_s;
  info->n = h->n;
  info->m = h->m;
  info->N = h->N;
  info->p = h->p;
  info->kmin = h->kmin;
  info->kmax = h->kmax;
  info->stot = h->stot;
  info->form = h->form;
  info->s_diagonal = h->s_diag;
  info->jacobi_capped = (int64_t)cap;
  info->launches_per_iter = launches_per_iter(h);
  info->jacobi_sweeps = (int64_t)sw;
  info->rho = h->rho;
  info->pipelined = h->pipe.on ? 1 : 0;
  info->fused = h->fused ? 1 : 0;
  info->s_factor = h->s_factor;
  info->nnz_l = h->s_factor == 2 ? h->nnz_l : (h->s_factor == 1 ? (int64_t)h->m * (h->m + 1) / 2 : 0);
}

// The fused persistent iteration (kernels_fused.cu) replaces the per-phase launches for small
// single-rank problems whose cliques all fit the register-V groups (k <= 32): one cooperative
// launch per sdp_step / solve chunk.  SDP_FUSED=0 turns it off, =1 takes it whenever the problem
// is structurally eligible (default: also A + A^T <= 64 MB and p <= 8192); SDP_FUSED_CTAS fixes
// the grid.
void build_fused(sdp_handle h, const std::vector<int>& task_bucket) {
  h->fused = false;
  const char* env = getenv("SDP_FUSED");
  if (env && *env == '0') return;
  const bool force = env && *env == '1';
  if (h->world != 1 || h->pipe.on || h->pl < 1) return;
  for (int b = 0; b < B_NUM; ++b)
    if (h->bcount[b] && b != B_RV8 && b != B_RV16 && b != B_RV32 && b != B_WJ32) return;
  if (!h->s_diag && h->m > fused_max_m()) return;
  int64_t nnzA = 0;
  if (!h->a_dense) {
    int32_t last = 0;
    SDP_CUDA_TRY(cudaMemcpy(&last, h->a_rp + h->m, sizeof(int32_t), cudaMemcpyDeviceToHost));
    nnzA = last;
  }
  const double bytes = h->a_dense ? 8.0 * ((double)h->m * h->lda + (double)h->Nl * h->ldm) : 24.0 * (double)nnzA;
  if (!force && (bytes > 64e6 || h->pl > 8192)) return;
  const int maxc = fused_max_ctas(h->device);
  int nsm = 0;
  SDP_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->device));
  if (maxc < 1) return;
  std::vector<int32_t> lists[3];
  for (int64_t q = 0; q < h->pl; ++q) {
    const int b = task_bucket[q];
    lists[b == B_RV8 ? 0 : b == B_RV16 ? 1 : 2].push_back((int32_t)q);
  }
  // groups per 256-thread CTA: 16 (k <= 8), 4 (k <= 16), 2 (k <= 32)
  const int64_t proj = std::max({((int64_t)lists[0].size() + 15) / 16, ((int64_t)lists[1].size() + 3) / 4,
                                 ((int64_t)lists[2].size() + 1) / 2});
  const int64_t bw = (int64_t)std::ceil(bytes / 98304.0);
  int64_t nb = std::max<int64_t>(1, std::max(proj, bw));
  nb = std::min<int64_t>(nb, std::min(maxc, nsm));
  if (const char* c = getenv("SDP_FUSED_CTAS")) nb = std::max(1, std::min(maxc, atoi(c)));
  h->fused_nb = (int)nb;
  h->fused_usplit = (int)std::max<int64_t>(1, std::min<int64_t>(16, nb * (kFusedThreads / 32) / h->m));
  Alloc& al = h->alloc;
  for (int j = 0; j < 3; ++j) {
    h->fused_count[j] = (int)lists[j].size();
    h->fused_ids[j] = lists[j].empty() ? nullptr : al.upload(lists[j]);
  }
  h->fused_upart = al.zeros<double>((size_t)h->fused_usplit * h->m);
  h->fused_cpart = al.zeros<double>(8 * (size_t)nb);
  h->fused_bar = al.zeros<unsigned>(2);
  // phase X: lanes per coordinate ~ a quarter of the row's double pairs (power of two <= 32)
  // (sparse A: lanes per row / coordinate ~ half the mean entry count)
  const double np = h->a_dense ? (h->m + 1) / 2 : 0.5 * (double)nnzA / std::max<int64_t>(1, h->Nl);
  h->fused_xl = 1;
  while (h->fused_xl < 32 && h->fused_xl * (h->a_dense ? 8 : 1) < np) h->fused_xl *= 2;
  h->fused_ul = 1;
  while (!h->a_dense && h->fused_ul < 32 && h->fused_ul < 0.5 * (double)nnzA / h->m) h->fused_ul *= 2;
  // scatter: coordinates with long segments (a warp each)
  std::vector<int32_t> segp(h->Nl + 1), lc;
  SDP_CUDA_TRY(cudaMemcpy(segp.data(), h->seg_ptr, segp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
  for (int64_t t = 0; t < h->Nl; ++t)
    if (segp[t + 1] - segp[t] > kFusedLongSeg) lc.push_back((int32_t)t);
  h->fused_nlong = (int)lc.size();
  h->fused_longc = lc.empty() ? nullptr : al.upload(lc);
  h->fused = true;
}

FusedArgs fused_args(sdp_handle h, int iters) {
  FusedArgs a;
  a.iters = iters;
  a.nb = h->fused_nb;
  a.m = h->m;
  a.N = (int)h->Nl;
  a.p = (int)h->pl;
  a.lda = h->lda;
  a.ldm = h->ldm;
  a.stot = h->stotl;
  a.usplit = h->fused_usplit;
  a.rho = h->rho;
  a.A = h->A;
  a.AT = h->AT;
  a.Sinv = h->s_diag ? nullptr : h->Sinv;
  a.sdiag = h->s_diag ? h->sdiag : nullptr;
  a.b = h->b;
  a.c = h->c;
  a.Dinv = h->Dinv;
  a.own = h->own;
  a.rD = h->rD;
  a.x = h->x;
  a.y = h->y;
  a.upart = h->fused_upart;
  a.sprev = h->sprev;
  a.vk = h->vk;
  a.seg_ptr = h->seg_ptr;
  a.seg_idx = h->seg_idx;
  ProjArgs& p = a.pa;
  p.off = h->d_off;
  p.ksz = h->d_ksz;
  p.x = h->x;
  p.G = h->G;
  p.xk = h->xk;
  p.lam = h->lam;
  p.vk = h->vk;
  p.rho = h->rho;
  p.part = h->proj_part;
  p.capped = h->capped;
  p.sweeps = h->sweeps;
  p.vprev = h->vprev;
  p.voff = h->voff;
  p.warm_period = h->warm_period;
  for (int j = 0; j < 3; ++j) {
    a.ids[j] = h->fused_ids[j];
    a.count[j] = h->fused_count[j];
  }
  a.cpart = h->fused_cpart;
  a.bar = h->fused_bar;
  a.bar_parity = h->fused_parity;
  a.xl = h->fused_xl;
  a.ul = h->fused_ul;
  if (!h->a_dense) {
    a.A = a.AT = nullptr;
    a.a_rp = h->a_rp;
    a.a_ci = h->a_ci;
    a.a_val = h->a_val;
    a.at_cp = h->at_cp;
    a.at_ri = h->at_ri;
    a.at_val = h->at_val;
    a.usplit = 1;
  }
  a.longc = h->fused_longc;
  a.n_long = h->fused_nlong;
  a.res = h->res;
  a.hist = h->hist;
  a.hist_cap = kHistCap;
  a.iter = h->iter;
  a.done = h->done;
  a.numerical = h->numerical;
  a.tol = h->tol;
  return a;
}

void launch_iterations(sdp_handle h, int32_t iters, bool for_solve = false) {
  if (h->fused) {
    FusedArgs fa = fused_args(h, iters);
    const char* tr = getenv("SDP_FUSED_TRACE");
    if (tr && *tr == '1') {
      if (!h->fused_trace) h->fused_trace = h->alloc.zeros<long long>(64 * 16 + 16);
      fa.trace = h->fused_trace;
    }
    if (iters <= 0) return;
    launch_fused(h->form, fa, h->stream);
    SDP_CUDA_TRY(cudaGetLastError());
    h->fused_parity ^= 1;  // the next launch uses the other barrier counter (zeroed by this one)
    if (fa.trace) {  // mean time between consecutive marks (CTA 0, %globaltimer), iterations 1..63
      std::vector<long long> t(64 * 16 + 16);
      SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
      SDP_CUDA_TRY(cudaMemcpy(t.data(), fa.trace, t.size() * sizeof(long long), cudaMemcpyDeviceToHost));
      const int n = std::min(iters, 64);
      std::string line = "fused trace (ns, mark -> next mark):";
      for (int ph = 0; ph < 16; ++ph) {
        double sum = 0;
        int cnt = 0;
        for (int i = 1; i < n; ++i) {
          const long long a0 = t[i * 16 + ph];
          int nx = ph + 1;
          while (nx < 16 && t[i * 16 + nx] == 0) ++nx;
          const long long a1 = nx < 16 ? t[i * 16 + nx] : (i + 1 < n ? t[(i + 1) * 16] : 0);
          if (a0 && a1) {
            sum += (double)(a1 - a0);
            ++cnt;
          }
        }
        if (cnt && t[16 + ph]) line += " " + std::to_string(ph) + ":" + std::to_string((long long)(sum / cnt));
      }
      fprintf(stderr, "%s\n", line.c_str());
      const long long* rv = t.data() + 64 * 16;  // register-V Jacobi clocks (CTA 0, group 0)
      if (rv[0] > 0)
        fprintf(stderr,
                "  rv projection (cycles per call): load %.0f, warm start %.0f, sweeps %.0f (%.2f sweeps, %.0f per "
                "step), recon+epilogue %.0f\n",
                (double)rv[1] / rv[0], (double)rv[2] / rv[0], (double)rv[3] / rv[0], (double)rv[5] / rv[0],
                rv[4] ? (double)rv[3] / rv[4] : 0.0, (double)rv[6] / rv[0]);
      SDP_CUDA_TRY(cudaMemset(fa.trace, 0, t.size() * sizeof(long long)));
    }
    return;
  }
  // dual: the pipelined schedule pays off from two iterations per call on (D_A + D_B alone has no
  // overlap); a single iteration runs the one-graph iteration
  if (h->pipe.on && h->form == SDP_FORM_DUAL && !for_solve && iters > 1) {  // D_A (D_BA)^(iters-1) D_B
    for (int32_t i = 0; i <= iters; ++i) {
      if (i == 0)
        pipe_dual_A(h, h->stream);
      else
        pipe_dual_B(h, h->stream, i < iters);
    }
    SDP_CUDA_TRY(cudaGetLastError());
    return;
  }
  if (h->pipe.on && h->form == SDP_FORM_PRIMAL && iters > 0) {  // [A] (BA)^iters, next A left issued
    Pipe& P = h->pipe;
    const char* pg = getenv("SDP_PIPE_GRAPH");
    const bool gr = h->use_graph && P.x[0] && P.x[1] && (iters <= 2 || (pg && *pg == '1'));
    const char* tr = getenv("SDP_PIPE_TRACE");
    for (int32_t i = P.pending ? 1 : 0; i <= iters; ++i) {
      const int w = i == 0 ? 0 : 1;
      g_ptrace.on = tr && !gr && w == 1 && i == iters;
      if (gr) {
        SDP_CUDA_TRY(cudaGraphLaunch(P.x[w], h->stream));
      } else if (w == 0) {
        pipe_enqueue_A(h, h->stream);
      } else {
        pipe_enqueue_B(h, h->stream, true);
      }
    }
    P.pending = true;
    g_ptrace.on = tr != nullptr;
    g_ptrace.dump();
    g_ptrace.on = false;
    SDP_CUDA_TRY(cudaGetLastError());
    return;
  }
  for (int32_t i = 0; i < iters; ++i) {
    if (h->exec)
      SDP_CUDA_TRY(cudaGraphLaunch(h->exec, h->stream));
    else
      enqueue_iteration(h, h->stream);
  }
  SDP_CUDA_TRY(cudaGetLastError());
}

// Put back the finished iteration's x (H1-touched coordinates) and y when the next iteration's A
// is pending (see Pipe::pending); the next sdp_step then starts with A again.
void settle(sdp_handle h) {
  Pipe& P = h->pipe;
  if (!P.on || !P.pending) return;
  SDP_CUDA_TRY(cudaMemcpyAsync(h->y, P.y_save, (size_t)h->m * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  SDP_CUDA_TRY(cudaMemcpyAsync(h->x, P.x_save, (size_t)P.nr1 * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
  P.pending = false;
}

}  // namespace

extern "C" {

void sdp_default_options(sdp_options* opt) {
  if (!opt) return;
  std::memset(opt, 0, sizeof(*opt));
  opt->form = SDP_FORM_PRIMAL;
  opt->rho = 1.0;
  opt->device = 0;
  opt->stream = nullptr;
  opt->check_every = 10;
  opt->use_graph = 1;
  opt->rank = 0;
  opt->world = 1;
  opt->nccl_id = nullptr;
  opt->allocator = nullptr;
  opt->comm = nullptr;
  opt->adapt_rho = 0;
  opt->adapt_mu = 10.0;
  opt->adapt_tau = 2.0;
}

int sdp_setup(const sdp_problem* prob, const sdp_options* opt, sdp_handle* out) {
  int rc = guarded([&] { return setup_impl(prob, opt, out); });
  if (rc != SDP_OK && out && *out) {
    destroy_handle(*out);
    *out = nullptr;
  }
  return rc;
}

int sdp_step(sdp_handle h, int32_t iters) {
  return guarded([&] {
    if (!h) throw Error{SDP_E_INVALID_ARG, "handle is NULL"};
    if (iters < 0) throw Error{SDP_E_INVALID_ARG, "iters < 0"};
    DeviceGuard dg(h->device);
    SDP_CUDA_TRY(cudaMemsetAsync(h->done, 0, sizeof(int), h->stream));
    launch_iterations(h, iters);
    return SDP_OK;
  });
}

namespace {
// Change rho between iterations (the KKT factor is rho-free; lambda_k is
// kept unscaled).  The primal right-hand side r1 depends on rho and is rebuilt
// from the current x_k, lambda_k (sprev is unchanged); the graph is recaptured.
void apply_rho(sdp_handle h, double rho) {
  settle(h);
  SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->rho = rho;
  if (h->form == SDP_FORM_PRIMAL) {
    int saved = 0;
    SDP_CUDA_TRY(cudaMemcpy(&saved, h->done, sizeof(int), cudaMemcpyDeviceToHost));
    SDP_CUDA_TRY(cudaMemsetAsync(h->done, 0, sizeof(int), h->stream));
    enqueue_scatter(h, h->stream);
    SDP_CUDA_TRY(cudaMemcpyAsync(h->done, &saved, sizeof(int), cudaMemcpyHostToDevice, h->stream));
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  rebuild_graph(h);
}
}  // namespace

int sdp_solve(sdp_handle h, int32_t max_iters, double tol, sdp_info* info) {
  return guarded([&] {
    if (!h) throw Error{SDP_E_INVALID_ARG, "handle is NULL"};
    if (!(tol > 0)) throw Error{SDP_E_INVALID_ARG, "tol must be positive"};
    DeviceGuard dg(h->device);
    SDP_CUDA_TRY(cudaMemcpyAsync(h->tol, &tol, sizeof(double), cudaMemcpyHostToDevice, h->stream));
    SDP_CUDA_TRY(cudaMemsetAsync(h->done, 0, sizeof(int), h->stream));
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    long long it = 0;
    int done = 0, num = 0;
    SDP_CUDA_TRY(cudaMemcpy(&it, h->iter, sizeof(it), cudaMemcpyDeviceToHost));
    while (it < max_iters) {
      // chunks end on multiples of check_every (the adaptation points of adapt_rho)
      // (the fused iteration tests the stopping rule on the device every iteration: without
      // adaptation one launch runs the whole solve)
      const int chunk = (h->fused && !h->adapt)
                            ? (int)(max_iters - it)
                            : (int)std::min<long long>(h->check_every - it % h->check_every, max_iters - it);
      launch_iterations(h, chunk, true);
      SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
      SDP_CUDA_TRY(cudaMemcpy(&done, h->done, sizeof(int), cudaMemcpyDeviceToHost));
      SDP_CUDA_TRY(cudaMemcpy(&num, h->numerical, sizeof(int), cudaMemcpyDeviceToHost));
      SDP_CUDA_TRY(cudaMemcpy(&it, h->iter, sizeof(it), cudaMemcpyDeviceToHost));
      if (num || done) break;
      if (h->adapt && it % h->check_every == 0) {
        // residual balancing on the last iteration's eps_p, eps_d (same rule as oracle.admm.adapt_rho)
        double res[2];
        SDP_CUDA_TRY(cudaMemcpy(res, h->res, 2 * sizeof(double), cudaMemcpyDeviceToHost));
        double rho = h->rho;
        if (res[0] > h->adapt_mu * res[1])
          rho = h->rho * h->adapt_tau;
        else if (res[1] > h->adapt_mu * res[0])
          rho = h->rho / h->adapt_tau;
        if (rho != h->rho) apply_rho(h, rho);
      }
    }
    // a stop skips the pending next-iteration A: put the finished iteration's x / y back
    settle(h);
    const double neg = -1.0;
    SDP_CUDA_TRY(cudaMemcpyAsync(h->tol, &neg, sizeof(double), cudaMemcpyHostToDevice, h->stream));
    SDP_CUDA_TRY(cudaMemsetAsync(h->done, 0, sizeof(int), h->stream));
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (info) fill_info(h, info);
    if (num) throw Error{SDP_E_NUMERICAL, "non-finite residuals (NaN/Inf in the iterates)"};
    return done ? SDP_OK : SDP_MAX_ITER;
  });
}

int sdp_reset(sdp_handle h) {
  return guarded([&] {
    if (!h) throw Error{SDP_E_INVALID_ARG, "handle is NULL"};
    DeviceGuard dg(h->device);
    settle(h);
    reset_state(h);
    return SDP_OK;
  });
}

int sdp_set_rho(sdp_handle h, double rho) {
  return guarded([&] {
    if (!h) throw Error{SDP_E_INVALID_ARG, "handle is NULL"};
    if (!(rho > 0) || !std::isfinite(rho)) throw Error{SDP_E_INVALID_ARG, "rho must be positive"};
    DeviceGuard dg(h->device);
    apply_rho(h, rho);
    return SDP_OK;
  });
}

int sdp_get_info(sdp_handle h, sdp_info* info) {
  return guarded([&] {
    if (!h || !info) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    DeviceGuard dg(h->device);
    fill_info(h, info);
    int num = 0;
    SDP_CUDA_TRY(cudaMemcpy(&num, h->numerical, sizeof(int), cudaMemcpyDeviceToHost));
    if (num) throw Error{SDP_E_NUMERICAL, "non-finite residuals (NaN/Inf in the iterates)"};
    return SDP_OK;
  });
}

int sdp_get_vector(sdp_handle h, int32_t which, double* out) {
  return guarded([&] {
    if (!h || !out) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    DeviceGuard dg(h->device);
    settle(h);
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (which == SDP_VEC_X || which == SDP_VEC_XMAT || which == SDP_VEC_SDP_X) {
      if (h->world == 1 && !h->coord_perm) {
        SDP_CUDA_TRY(cudaMemcpy(out, h->x, h->N * sizeof(double), cudaMemcpyDeviceToHost));
      } else if (h->world == 1) {  // local order = a permutation of the canonical one
        std::vector<double> xl(h->Nl);
        SDP_CUDA_TRY(cudaMemcpy(xl.data(), h->x, h->Nl * sizeof(double), cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < h->Nl; ++i) out[h->local_coords[i]] = xl[i];
      } else {  // collective: owners contribute their coordinates
        std::vector<double> xl(h->Nl), own(h->Nl);
        SDP_CUDA_TRY(cudaMemcpy(xl.data(), h->x, h->Nl * sizeof(double), cudaMemcpyDeviceToHost));
        SDP_CUDA_TRY(cudaMemcpy(own.data(), h->own, h->Nl * sizeof(double), cudaMemcpyDeviceToHost));
        std::vector<double> full(h->N, 0.0);
        for (int64_t i = 0; i < h->Nl; ++i)
          if (own[i] != 0.0) full[h->local_coords[i]] = xl[i];
        allreduce_host(h, full);
        std::memcpy(out, full.data(), h->N * sizeof(double));
      }
      if (which != SDP_VEC_X)
        for (int64_t t = 0; t < h->N; ++t)
          if (h->coord_row[t] != h->coord_col[t]) out[t] /= kSqrt2;
      // recovered SDP primal (Remark 1): X = x (Alg. 1), X = -rho x (Alg. 2)
      if (which == SDP_VEC_SDP_X && h->form == SDP_FORM_DUAL)
        for (int64_t t = 0; t < h->N; ++t) out[t] *= -h->rho;
    } else if (which == SDP_VEC_Y || which == SDP_VEC_SDP_Y) {
      SDP_CUDA_TRY(cudaMemcpy(out, h->y, h->m * sizeof(double), cudaMemcpyDeviceToHost));
      // recovered SDP dual: yhat = -rho y (Alg. 1), yhat = y (Alg. 2)
      if (which == SDP_VEC_SDP_Y && h->form == SDP_FORM_PRIMAL)
        for (int i = 0; i < h->m; ++i) out[i] *= -h->rho;
    } else {
      throw Error{SDP_E_INVALID_ARG, "unknown vector id"};
    }
    return SDP_OK;
  });
}

int sdp_get_elimination_order(sdp_handle h, int32_t* order) {
  return guarded([&] {
    if (!h || !order) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    std::memcpy(order, h->chordal.order.data(), h->n * sizeof(int32_t));
    return SDP_OK;
  });
}

int sdp_complete_x(sdp_handle h, double rtol, double* out) {
  return guarded([&] {
    if (!h || !out) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    if (!(rtol >= 0.0)) throw Error{SDP_E_INVALID_ARG, "rtol must be >= 0"};
    const int32_t n = (int32_t)h->n;
    std::vector<double> xm(h->N);
    const int rc = sdp_get_vector(h, SDP_VEC_SDP_X, xm.data());  // SDP X entries, canonical order (both forms)
    if (rc != SDP_OK) return rc;
    std::vector<uint8_t> known((size_t)n * n, 0);
    for (int64_t i = 0; i < (int64_t)n * n; ++i) out[i] = 0.0;
    for (int64_t t = 0; t < h->N; ++t) {
      const int r = h->coord_row[t], c = h->coord_col[t];
      out[(size_t)r * n + c] = out[(size_t)c * n + r] = xm[t];
      known[(size_t)r * n + c] = known[(size_t)c * n + r] = 1;
    }
    complete_psd_host(n, h->chordal, known, rtol, out);
    return SDP_OK;
  });
}

int sdp_get_blocks(sdp_handle h, int32_t which, double* out) {
  return guarded([&] {
    if (!h || !out) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    DeviceGuard dg(h->device);
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    // SDP_BLK_SDP_Z: the Agler blocks Z_k of the recovered dual slack (Theorem 2): lambda_k in the
    // primal form, z_k in the dual form (Remark 1)
    if (which == SDP_BLK_SDP_Z) which = h->form == SDP_FORM_PRIMAL ? SDP_BLK_LAMBDA : SDP_BLK_XK;
    const double* src = which == SDP_BLK_XK ? h->xk : which == SDP_BLK_LAMBDA ? h->lam : which == SDP_BLK_VK ? h->vk : nullptr;
    if (!src) throw Error{SDP_E_INVALID_ARG, "unknown block id"};
    if (h->world == 1) {
      SDP_CUDA_TRY(cudaMemcpy(out, src, h->stot * sizeof(double), cudaMemcpyDeviceToHost));
    } else {  // collective: every rank places its cliques
      std::vector<double> loc(h->stotl), full(h->stot, 0.0);
      SDP_CUDA_TRY(cudaMemcpy(loc.data(), src, h->stotl * sizeof(double), cudaMemcpyDeviceToHost));
      int64_t e = 0;
      for (int32_t k : h->my_cliques) {
        const int64_t len = h->clique_off[k + 1] - h->clique_off[k];
        std::memcpy(full.data() + h->clique_off[k], loc.data() + e, len * sizeof(double));
        e += len;
      }
      allreduce_host(h, full);
      std::memcpy(out, full.data(), h->stot * sizeof(double));
    }
    return SDP_OK;
  });
}

int sdp_get_pattern(sdp_handle h, int32_t* row, int32_t* col) {
  return guarded([&] {
    if (!h || !row || !col) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    std::memcpy(row, h->coord_row.data(), h->N * sizeof(int32_t));
    std::memcpy(col, h->coord_col.data(), h->N * sizeof(int32_t));
    return SDP_OK;
  });
}

int sdp_get_cliques(sdp_handle h, int32_t* sizes, int32_t* vertices) {
  return guarded([&] {
    if (!h || !sizes || !vertices) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    std::memcpy(sizes, h->clique_size.data(), h->clique_size.size() * sizeof(int32_t));
    std::memcpy(vertices, h->clique_vert.data(), h->clique_vert.size() * sizeof(int32_t));
    return SDP_OK;
  });
}

int sdp_get_history(sdp_handle h, double* out, int64_t cap, int64_t* rows) {
  return guarded([&] {
    if (!h || !out || !rows) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    DeviceGuard dg(h->device);
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    long long it = 0;
    SDP_CUDA_TRY(cudaMemcpy(&it, h->iter, sizeof(it), cudaMemcpyDeviceToHost));
    const int64_t r = std::min<int64_t>(std::min<int64_t>(it, kHistCap), cap);
    if (r > 0) SDP_CUDA_TRY(cudaMemcpy(out, h->hist, 3 * r * sizeof(double), cudaMemcpyDeviceToHost));
    *rows = r;
    return SDP_OK;
  });
}

int sdp_profile_phases(sdp_handle h, int32_t iters, double* out_ms) {
  return guarded([&] {
    if (!h || !out_ms || iters <= 0) throw Error{SDP_E_INVALID_ARG, "bad argument"};
    DeviceGuard dg(h->device);
    settle(h);
    SDP_CUDA_TRY(cudaMemsetAsync(h->done, 0, sizeof(int), h->stream));
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    std::vector<cudaEvent_t> ev(16 * (size_t)iters);
    for (auto& e : ev) SDP_CUDA_TRY(cudaEventCreate(&e));
    std::vector<int> ids;
    int idx = 0;
    for (int it = 0; it < iters; ++it) {
      g_phase.ev = &ev;
      g_phase.idx = &idx;
      g_phase_n = 0;
      enqueue_iteration(h, h->stream);
      for (int i = 0; i < g_phase_n; ++i) ids.push_back(g_phase_id[i]);
    }
    g_phase.ev = nullptr;
    g_phase.idx = nullptr;
    SDP_CUDA_TRY(cudaGetLastError());
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    for (int p = 0; p < SDP_NUM_PHASES; ++p) out_ms[p] = 0.0;
    // consecutive marks (i, i+1) inside one iteration delimit phase ids[i]
    const int per = (int)ids.size() / iters;
    for (int it = 0; it < iters; ++it)
      for (int i = 0; i + 1 < per; ++i) {
        float ms = 0.f;
        SDP_CUDA_TRY(cudaEventElapsedTime(&ms, ev[it * per + i], ev[it * per + i + 1]));
        const int ph = ids[it * per + i];
        if (ph < SDP_NUM_PHASES) out_ms[ph] += ms / iters;
      }
    for (auto& e : ev) cudaEventDestroy(e);
    return SDP_OK;
  });
}

namespace {
constexpr int64_t kStateMagic = 0x3254415453504453ll;  // "SDPSTAT2"
constexpr int kStateHeader = 20;                      // int64 words
// FNV-1a over the local coordinate order (the layout of x, r1/D and sprev in the blob: a
// permutation of the canonical order that depends on the pipelined split)
int64_t layout_hash(sdp_handle h) {
  uint64_t x = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      x ^= (v >> (8 * b)) & 0xff;
      x *= 1099511628211ull;
    }
  };
  mix((uint64_t)h->Nl);
  for (int32_t t : h->local_coords) mix((uint64_t)(uint32_t)t);
  for (int32_t k : h->my_cliques) mix((uint64_t)(uint32_t)k);
  mix((uint64_t)h->pl);
  return (int64_t)(x & 0x7fffffffffffffffull);
}
struct StateLayout {
  int64_t stot, lda, m, vlen, hrows, nprev;
  int64_t words() const { return kStateHeader + 3 * stot + 3 * lda + m + 4 + 3 * hrows + vlen + nprev; }
};
StateLayout state_layout(sdp_handle h, long long iter) {
  StateLayout L;
  L.stot = h->stotl;
  L.lda = h->lda;
  L.m = h->m;
  L.vlen = h->vprev ? h->vprev_len : 0;
  L.hrows = std::min<long long>(iter, kHistCap);
  L.nprev = h->prevall ? std::max(1, h->nshared) : 0;
  return L;
}
}  // namespace

int sdp_state_bytes(sdp_handle h, int64_t* bytes) {
  return guarded([&] {
    if (!h || !bytes) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    DeviceGuard dg(h->device);
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    long long it = 0;
    SDP_CUDA_TRY(cudaMemcpy(&it, h->iter, sizeof(it), cudaMemcpyDeviceToHost));
    *bytes = 8 * state_layout(h, it).words();
    return SDP_OK;
  });
}

int sdp_save_state(sdp_handle h, void* host_out, int64_t capacity) {
  return guarded([&] {
    if (!h || !host_out) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    DeviceGuard dg(h->device);
    settle(h);
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    long long it = 0;
    unsigned long long cap = 0, sw = 0;
    SDP_CUDA_TRY(cudaMemcpy(&it, h->iter, sizeof(it), cudaMemcpyDeviceToHost));
    SDP_CUDA_TRY(cudaMemcpy(&cap, h->capped, sizeof(cap), cudaMemcpyDeviceToHost));
    SDP_CUDA_TRY(cudaMemcpy(&sw, h->sweeps, sizeof(sw), cudaMemcpyDeviceToHost));
    const StateLayout L = state_layout(h, it);
    if (capacity < 8 * L.words()) throw Error{SDP_E_INVALID_ARG, "state buffer too small (see sdp_state_bytes)"};
    int64_t* hd = static_cast<int64_t*>(host_out);
    std::memset(hd, 0, 8 * kStateHeader);
    hd[0] = kStateMagic;
    hd[1] = h->form;
    hd[2] = h->world;
    hd[3] = h->rank;
    hd[4] = L.stot;
    hd[5] = L.lda;
    hd[6] = L.m;
    hd[7] = L.vlen;
    hd[8] = L.hrows;
    hd[9] = it;
    hd[10] = (int64_t)cap;
    hd[11] = (int64_t)sw;
    std::memcpy(&hd[12], &h->rho, 8);
    hd[13] = h->N;
    hd[14] = h->p;
    hd[15] = h->coord_perm ? 1 : 0;  // coordinate layout of x, r1/D, sprev
    hd[16] = layout_hash(h);         // ... and the exact order
    hd[17] = h->pipe.on ? h->pipe.p1 : 0;
    double* w = reinterpret_cast<double*>(hd + kStateHeader);
    auto get = [&](const double* dev, int64_t n) {
      if (n) SDP_CUDA_TRY(cudaMemcpy(w, dev, n * sizeof(double), cudaMemcpyDeviceToHost));
      w += n;
    };
    get(h->xk, L.stot);
    get(h->lam, L.stot);
    get(h->vk, L.stot);
    get(h->x, L.lda);
    get(h->rD, L.lda);
    get(h->sprev, L.lda);
    get(h->y, L.m);
    get(h->res, 4);
    get(h->hist, 3 * L.hrows);
    get(h->vprev, L.vlen);
    get(h->prevall, L.nprev);
    return SDP_OK;
  });
}

int sdp_load_state(sdp_handle h, const void* host_in, int64_t bytes) {
  return guarded([&] {
    if (!h || !host_in) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    DeviceGuard dg(h->device);
    settle(h);
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));
    const int64_t* hd = static_cast<const int64_t*>(host_in);
    if (bytes < 8 * kStateHeader || hd[0] != kStateMagic) throw Error{SDP_E_INVALID_ARG, "not an sdp state blob"};
    StateLayout L = state_layout(h, hd[9]);
    if (hd[1] != h->form || hd[2] != h->world || hd[3] != h->rank || hd[4] != L.stot || hd[5] != L.lda ||
        hd[6] != L.m || hd[7] != L.vlen || hd[8] != L.hrows || hd[13] != h->N || hd[14] != h->p)
      throw Error{SDP_E_INVALID_ARG, "state blob is from a different problem, form or sharding"};
    if (hd[15] != (h->coord_perm ? 1 : 0) || hd[16] != layout_hash(h) || hd[17] != (h->pipe.on ? h->pipe.p1 : 0))
      throw Error{SDP_E_INVALID_ARG,
                  "state blob has a different coordinate layout (SDP_PIPELINE / SDP_PIPE_SPLIT or the build differ)"};
    if (bytes < 8 * L.words()) throw Error{SDP_E_INVALID_ARG, "state blob truncated"};
    const double* w = reinterpret_cast<const double*>(hd + kStateHeader);
    auto put = [&](double* dev, int64_t n) {
      if (n) SDP_CUDA_TRY(cudaMemcpyAsync(dev, w, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
      w += n;
    };
    put(h->xk, L.stot);
    put(h->lam, L.stot);
    put(h->vk, L.stot);
    put(h->x, L.lda);
    put(h->rD, L.lda);
    put(h->sprev, L.lda);
    put(h->y, L.m);
    put(h->res, 4);
    put(h->hist, 3 * L.hrows);
    put(h->vprev, L.vlen);
    put(h->prevall, L.nprev);
    const long long it = hd[9];
    const unsigned long long cap = (unsigned long long)hd[10], sw = (unsigned long long)hd[11];
    SDP_CUDA_TRY(cudaMemcpyAsync(h->iter, &it, sizeof(it), cudaMemcpyHostToDevice, h->stream));
    SDP_CUDA_TRY(cudaMemcpyAsync(h->capped, &cap, sizeof(cap), cudaMemcpyHostToDevice, h->stream));
    SDP_CUDA_TRY(cudaMemcpyAsync(h->sweeps, &sw, sizeof(sw), cudaMemcpyHostToDevice, h->stream));
    SDP_CUDA_TRY(cudaMemsetAsync(h->done, 0, sizeof(int), h->stream));
    SDP_CUDA_TRY(cudaMemsetAsync(h->numerical, 0, sizeof(int), h->stream));
    SDP_CUDA_TRY(cudaStreamSynchronize(h->stream));  // (it, cap, sw are locals)
    double rho;
    std::memcpy(&rho, &hd[12], 8);
    h->rho = rho;  // r1 / D was restored as saved: no rebuild from x_k, lambda_k
    rebuild_graph(h);
    return SDP_OK;
  });
}

int sdp_workspace_bytes(sdp_handle h, int64_t* live_bytes, int64_t* peak_bytes) {
  return guarded([&] {
    if (!h) throw Error{SDP_E_INVALID_ARG, "handle is NULL"};
    if (live_bytes) *live_bytes = h->alloc.live;
    if (peak_bytes) *peak_bytes = h->alloc.peak;
    return SDP_OK;
  });
}

int sdp_destroy(sdp_handle h) {
  return guarded([&] {
    destroy_handle(h);
    return SDP_OK;
  });
}

int sdp_chordal_cliques(int32_t n, int64_t nnz, const int32_t* row, const int32_t* col, int32_t* p, int32_t* sizes,
                        int64_t cap_vertices, int32_t* vertices, int64_t* nv, int64_t* fill_edges) {
  return guarded([&] {
    if (n <= 0) throw Error{SDP_E_INVALID_ARG, "n <= 0"};
    if (nnz > 0 && (!row || !col)) throw Error{SDP_E_INVALID_ARG, "NULL pattern"};
    if (!p || !sizes || !vertices || !nv) throw Error{SDP_E_INVALID_ARG, "NULL output"};
    check_indices("pattern", nnz, row, col, n);
    std::vector<std::pair<int32_t, int32_t>> edges;
    for (int64_t e = 0; e < nnz; ++e)
      if (row[e] != col[e]) edges.push_back({row[e], col[e]});
    ChordalResult cr = chordal_analysis(n, edges);
    int64_t tot = 0;
    for (auto& c : cr.cliques) tot += (int64_t)c.size();
    *p = (int32_t)cr.cliques.size();
    *nv = tot;
    if (fill_edges) *fill_edges = cr.fill_edges;
    if (tot > cap_vertices) throw Error{SDP_E_INVALID_ARG, "vertices buffer too small"};
    int64_t e = 0;
    for (size_t k = 0; k < cr.cliques.size(); ++k) {
      sizes[k] = (int32_t)cr.cliques[k].size();
      for (int v : cr.cliques[k]) vertices[e++] = v;
    }
    return SDP_OK;
  });
}

int sdp_psd_plan_create(int64_t count, const int32_t* h_sizes, int32_t device, sdp_psd_plan* out) {
  return sdp_psd_plan_create_ex(count, h_sizes, device, nullptr, out);
}

int sdp_psd_plan_create_ex(int64_t count, const int32_t* h_sizes, int32_t device, const sdp_allocator* allocator,
                           sdp_psd_plan* out) {
  sdp_psd_plan pl = nullptr;
  int rc = guarded([&] {
    if (!out) throw Error{SDP_E_INVALID_ARG, "out is NULL"};
    *out = nullptr;
    if (count < 0 || (count > 0 && !h_sizes)) throw Error{SDP_E_INVALID_ARG, "bad sizes"};
    if (count >= (1ll << 31)) throw Error{SDP_E_INVALID_ARG, "count too large"};
    int ndev = 0;
    SDP_CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw Error{SDP_E_INVALID_ARG, "bad device ordinal"};
    DeviceGuard dg(device);
    pl = new sdp_psd_plan_s();
    pl->device = device;
    pl->count = count;
    pl->alloc.set_hook(allocator, device);
    std::vector<int64_t> off(count + 1, 0);
    std::vector<int32_t> ksz(h_sizes, h_sizes + count);
    for (int64_t i = 0; i < count; ++i) {
      const int k = ksz[i];
      if (k < 1 || k > SDP_MAX_K)
        throw Error{SDP_E_INVALID_ARG, "matrix " + std::to_string(i) + " has order outside [1, SDP_MAX_K]"};
      off[i + 1] = off[i] + (int64_t)k * (k + 1) / 2;
    }
    pl->values = off[count];
    pl->h_sizes = ksz;
    pl->d_off = pl->alloc.upload(off);
    pl->d_ksz = pl->alloc.upload(ksz);
    build_buckets(pl->alloc, ksz, pl->d_ids, pl->bcount, pl->gd, pl->td);
    pl->capped = pl->alloc.zeros<unsigned long long>(1);
    pl->sweeps = pl->alloc.zeros<unsigned long long>(1);
    pl->tiers.create();
    psd_init_attributes();
    *out = pl;
    return SDP_OK;
  });
  if (rc != SDP_OK && pl) {
    pl->alloc.free_all();
    pl->tiers.destroy();
    delete pl;
  }
  return rc;
}

int sdp_project_psd_batch(sdp_psd_plan pl, const double* d_in, double* d_out, void* stream) {
  return guarded([&] {
    if (!pl) throw Error{SDP_E_INVALID_ARG, "plan is NULL"};
    if (pl->values > 0 && (!d_in || !d_out)) throw Error{SDP_E_INVALID_ARG, "NULL data pointer"};
    DeviceGuard dg(pl->device);
    cudaStream_t s = (cudaStream_t)stream;
    ProjArgs a{};
    a.off = pl->d_off;
    a.ksz = pl->d_ksz;
    a.in = d_in;
    a.out = d_out;
    a.gd = pl->gd;
    a.capped = pl->capped;
    a.sweeps = pl->sweeps;
    a.done = nullptr;
    launch_tiers(a, PM_BATCH, pl->d_ids, pl->bcount, pl->td, pl->tiers, s);
    SDP_CUDA_TRY(cudaGetLastError());
    return SDP_OK;
  });
}

}  // extern "C"

namespace {
constexpr int64_t kPipeMinCount = 4096;  // matrices per sub-plan of the pinned pipeline (at least)
int pipe_chunks() {  // SDP_PSD_PIPE_CHUNKS (default 4)
  const char* e = getenv("SDP_PSD_PIPE_CHUNKS");
  return e ? std::max(2, std::min(16, atoi(e))) : 4;
}

bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Pinned host buffers: pipe_chunks() contiguous sub-plans (equal value counts); chunk i's H2D copy
// (stream cp_in), projection (the caller's stream) and D2H copy (stream cp_out) are ordered by
// events only, so copies in both directions run beside the projections of other chunks.
void project_pipelined(sdp_psd_plan pl, const double* h_in, double* h_out, cudaStream_t s) {
  if (!pl->h_in_dev) {
    pl->h_in_dev = pl->alloc.get<double>(pl->values);
    pl->h_out_dev = pl->alloc.get<double>(pl->values);
  }
  if (pl->sub.empty()) {
    const int64_t n = pl->count;
    int64_t start = 0, v = 0;
    const int nch = pipe_chunks();
    for (int c = 0; c < nch && start < n; ++c) {
      const int64_t target = pl->values * (c + 1) / nch;
      int64_t end = start, nvc = 0;
      while (end < n && (c == nch - 1 || v + nvc < target)) {
        const int64_t k = pl->h_sizes[end];
        nvc += k * (k + 1) / 2;
        ++end;
      }
      sdp_psd_plan q = nullptr;
      const int rc = sdp_psd_plan_create_ex(end - start, pl->h_sizes.data() + start, pl->device,
                                            pl->alloc.has_hook ? &pl->alloc.hook : nullptr, &q);
      if (rc != SDP_OK) throw Error{rc, std::string("sub-plan: ") + sdp_last_error()};
      pl->sub.push_back(q);
      pl->sub_v0.push_back(v);
      pl->sub_nv.push_back(nvc);
      v += nvc;
      start = end;
    }
    SDP_CUDA_TRY(cudaStreamCreateWithFlags(&pl->cp_in, cudaStreamNonBlocking));
    SDP_CUDA_TRY(cudaStreamCreateWithFlags(&pl->cp_out, cudaStreamNonBlocking));
    pl->ev_in.assign(pl->sub.size(), nullptr);
    pl->ev_comp.assign(pl->sub.size(), nullptr);
    for (size_t i = 0; i < pl->sub.size(); ++i) {
      SDP_CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_in[i], cudaEventDisableTiming));
      SDP_CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_comp[i], cudaEventDisableTiming));
    }
    SDP_CUDA_TRY(cudaEventCreateWithFlags(&pl->ev_end, cudaEventDisableTiming));
  }
  // the copies start after the caller's earlier work on s (event ordering only)
  SDP_CUDA_TRY(cudaEventRecord(pl->ev_end, s));
  SDP_CUDA_TRY(cudaStreamWaitEvent(pl->cp_in, pl->ev_end, 0));
  for (size_t i = 0; i < pl->sub.size(); ++i) {
    SDP_CUDA_TRY(cudaMemcpyAsync(pl->h_in_dev + pl->sub_v0[i], h_in + pl->sub_v0[i],
                                 pl->sub_nv[i] * sizeof(double), cudaMemcpyHostToDevice, pl->cp_in));
    SDP_CUDA_TRY(cudaEventRecord(pl->ev_in[i], pl->cp_in));
  }
  for (size_t i = 0; i < pl->sub.size(); ++i) {
    SDP_CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_in[i], 0));
    const int rc = sdp_project_psd_batch(pl->sub[i], pl->h_in_dev + pl->sub_v0[i], pl->h_out_dev + pl->sub_v0[i], s);
    if (rc != SDP_OK) throw Error{rc, std::string("sub-plan: ") + sdp_last_error()};
    SDP_CUDA_TRY(cudaEventRecord(pl->ev_comp[i], s));
    SDP_CUDA_TRY(cudaStreamWaitEvent(pl->cp_out, pl->ev_comp[i], 0));
    SDP_CUDA_TRY(cudaMemcpyAsync(h_out + pl->sub_v0[i], pl->h_out_dev + pl->sub_v0[i], pl->sub_nv[i] * sizeof(double),
                                 cudaMemcpyDeviceToHost, pl->cp_out));
  }
  SDP_CUDA_TRY(cudaEventRecord(pl->ev_end, pl->cp_out));
  SDP_CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_end, 0));
  SDP_CUDA_TRY(cudaStreamSynchronize(s));
}
}  // namespace

extern "C" {

int sdp_project_psd_batch_host(sdp_psd_plan pl, const double* h_in, double* h_out, void* stream) {
  return guarded([&] {
    if (!pl) throw Error{SDP_E_INVALID_ARG, "plan is NULL"};
    if (pl->values > 0 && (!h_in || !h_out)) throw Error{SDP_E_INVALID_ARG, "NULL data pointer"};
    DeviceGuard dg(pl->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (!pl->h_in_dev) {
      pl->h_in_dev = pl->alloc.get<double>(pl->values);
      pl->h_out_dev = pl->alloc.get<double>(pl->values);
    }
    if (!pl->stage[0]) {
      for (int b = 0; b < 2; ++b) {
        SDP_CUDA_TRY(cudaHostAlloc(&pl->stage[b], kStageDoubles * sizeof(double), cudaHostAllocDefault));
        SDP_CUDA_TRY(cudaEventCreateWithFlags(&pl->stage_ev[b], cudaEventDisableTiming));
      }
    }
    const int64_t nv = pl->values;
    if (host_pinned(h_in) && host_pinned(h_out) && pl->count >= 4 * kPipeMinCount) {
      project_pipelined(pl, h_in, h_out, s);
      return SDP_OK;
    }
    // H2D: host -> pinned chunk (all host threads) -> async DMA, two chunks in flight
    for (int64_t c0 = 0, it = 0; c0 < nv; c0 += kStageDoubles, ++it) {
      const int b = (int)(it & 1);
      const int64_t n = std::min<int64_t>(kStageDoubles, nv - c0);
      if (it >= 2) SDP_CUDA_TRY(cudaEventSynchronize(pl->stage_ev[b]));
      host_copy_parallel(pl->stage[b], h_in + c0, n);
      SDP_CUDA_TRY(cudaMemcpyAsync(pl->h_in_dev + c0, pl->stage[b], n * sizeof(double), cudaMemcpyHostToDevice, s));
      SDP_CUDA_TRY(cudaEventRecord(pl->stage_ev[b], s));
    }
    int rc = sdp_project_psd_batch(pl, pl->h_in_dev, pl->h_out_dev, stream);
    if (rc != SDP_OK) return rc;
    // D2H: async DMA into a pinned chunk, then pinned -> host while the next chunk's DMA runs
    const int64_t nch = (nv + kStageDoubles - 1) / kStageDoubles;
    auto issue = [&](int64_t it) {
      const int b = (int)(it & 1);
      const int64_t c0 = it * kStageDoubles, n = std::min<int64_t>(kStageDoubles, nv - c0);
      SDP_CUDA_TRY(cudaMemcpyAsync(pl->stage[b], pl->h_out_dev + c0, n * sizeof(double), cudaMemcpyDeviceToHost, s));
      SDP_CUDA_TRY(cudaEventRecord(pl->stage_ev[b], s));
    };
    if (nch > 0) issue(0);
    for (int64_t it = 0; it < nch; ++it) {
      if (it + 1 < nch) issue(it + 1);
      const int b = (int)(it & 1);
      const int64_t c0 = it * kStageDoubles, n = std::min<int64_t>(kStageDoubles, nv - c0);
      SDP_CUDA_TRY(cudaEventSynchronize(pl->stage_ev[b]));
      host_copy_parallel(h_out + c0, pl->stage[b], n);
    }
    SDP_CUDA_TRY(cudaStreamSynchronize(s));
    return SDP_OK;
  });
}

int64_t sdp_psd_plan_values(sdp_psd_plan pl) { return pl ? pl->values : -1; }

int32_t sdp_psd_plan_launches(sdp_psd_plan pl) {
  if (!pl) return -1;
  int32_t n = 0;
  for (int b = 0; b < B_NUM; ++b) {
    if (!pl->bcount[b]) continue;
    if (is_trd(b)) {
      const TrdDev& t = pl->td[b - B_TRD8];
      n += trd_launches_per_chunk(b) * ((t.count + t.chunk - 1) / t.chunk);
    } else {
      n += 1;
    }
  }
  return n;
}

int sdp_psd_plan_destroy(sdp_psd_plan pl) {
  return guarded([&] {
    if (!pl) return SDP_OK;
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(pl->device);
    cudaDeviceSynchronize();
    for (auto* q : pl->sub) sdp_psd_plan_destroy(q);
    pl->sub.clear();
    if (pl->cp_in) cudaStreamDestroy(pl->cp_in);
    if (pl->cp_out) cudaStreamDestroy(pl->cp_out);
    for (auto e : pl->ev_in) cudaEventDestroy(e);
    for (auto e : pl->ev_comp) cudaEventDestroy(e);
    if (pl->ev_end) cudaEventDestroy(pl->ev_end);
    pl->alloc.free_all();
    pl->tiers.destroy();
    pl->free_stage();
    if (cur >= 0) cudaSetDevice(cur);
    delete pl;
    return SDP_OK;
  });
}

int sdp_nccl_unique_id(void* out128) {
  return guarded([&] {
    if (!out128) throw Error{SDP_E_INVALID_ARG, "NULL argument"};
    nccl_unique_id(out128);
    return SDP_OK;
  });
}

int sdp_shard_plan(int32_t n, int64_t nnz, const int32_t* row, const int32_t* col, int32_t world, int32_t rank,
                   int32_t* clique_rank, int64_t* n_local, int32_t* local_coords, uint8_t* owned,
                   int64_t* n_shared, int32_t* shared_coords, int64_t cap) {
  return guarded([&] {
    if (n <= 0 || world < 1 || rank < 0 || rank >= world) throw Error{SDP_E_INVALID_ARG, "bad n/world/rank"};
    if (nnz > 0 && (!row || !col)) throw Error{SDP_E_INVALID_ARG, "NULL pattern"};
    if (!clique_rank || !n_local || !local_coords || !owned || !n_shared || !shared_coords)
      throw Error{SDP_E_INVALID_ARG, "NULL output"};
    check_indices("pattern", nnz, row, col, n);
    std::vector<std::pair<int32_t, int32_t>> edges;
    for (int64_t e = 0; e < nnz; ++e)
      if (row[e] != col[e]) edges.push_back({row[e], col[e]});
    ChordalResult cr = chordal_analysis(n, edges);
    const int64_t p = (int64_t)cr.cliques.size(), N = (int64_t)cr.coord_row.size();
    std::vector<int64_t> off(p + 1, 0);
    std::vector<int32_t> ksz(p);
    for (int64_t k = 0; k < p; ++k) {
      ksz[k] = (int32_t)cr.cliques[k].size();
      off[k + 1] = off[k] + (int64_t)ksz[k] * (ksz[k] + 1) / 2;
    }
    std::vector<int32_t> Gmap(off[p]);
    for (int64_t k = 0; k < p; ++k) {
      const auto& C = cr.cliques[k];
      int64_t e = off[k];
      for (size_t bcol = 0; bcol < C.size(); ++bcol)
        for (size_t arow = 0; arow <= bcol; ++arow) Gmap[e++] = (int32_t)coord_index(cr, C[arow], C[bcol]);
    }
    std::vector<int32_t> seg_ptr(N + 1, 0), seg_idx(off[p]);
    for (int64_t s2 = 0; s2 < off[p]; ++s2) seg_ptr[Gmap[s2] + 1]++;
    for (int64_t t = 0; t < N; ++t) seg_ptr[t + 1] += seg_ptr[t];
    std::vector<int32_t> fillp(seg_ptr.begin(), seg_ptr.end() - 1);
    for (int64_t s2 = 0; s2 < off[p]; ++s2) seg_idx[fillp[Gmap[s2]]++] = (int32_t)s2;
    if (world > p) throw Error{SDP_E_INVALID_ARG, "more ranks than cliques"};
    ShardPlan sp = make_shard_plan(ksz, off, seg_ptr, seg_idx, world, rank);
    if (p > cap) throw Error{SDP_E_INVALID_ARG, "output buffers too small"};
    std::memcpy(clique_rank, sp.clique_rank.data(), p * sizeof(int32_t));
    *n_local = (int64_t)sp.local_coords.size();
    *n_shared = (int64_t)sp.shared_coords.size();
    if (*n_local > cap || *n_shared > cap) throw Error{SDP_E_INVALID_ARG, "output buffers too small"};
    std::memcpy(local_coords, sp.local_coords.data(), sp.local_coords.size() * sizeof(int32_t));
    std::memcpy(owned, sp.owned.data(), sp.owned.size());
    std::memcpy(shared_coords, sp.shared_coords.data(), sp.shared_coords.size() * sizeof(int32_t));
    return SDP_OK;
  });
}

int sdp_schur_inverse_host(int32_t m, const int64_t* ptr, const int32_t* idx, const double* val, int32_t force_sparse,
                           double* sinv, int64_t* nnz_l) {
  return guarded([&] {
    if (m <= 0 || !ptr || !idx || !val || !sinv) throw Error{SDP_E_INVALID_ARG, "bad argument"};
    std::vector<int64_t> sp(ptr, ptr + m + 1);
    std::vector<int32_t> si(idx, idx + sp[m]);
    std::vector<double> sv(val, val + sp[m]);
    for (int64_t e = 0; e < sp[m]; ++e)
      if (si[e] < 0 || si[e] >= m) throw Error{SDP_E_INVALID_ARG, "column index out of range"};
    const int64_t ldg = (m + 31) / 32 * 32;
    std::vector<double> GT;
    std::string why;
    int64_t nnz = 0;
    if (!sparse_inverse_factor(m, sp, si, sv, ldg, GT, &nnz, 0.125, force_sparse != 0, &why))
      throw Error{why == "factor too dense" ? SDP_E_STATE : SDP_E_RANK_DEFICIENT, why};
    if (nnz_l) *nnz_l = nnz;
#pragma omp parallel for schedule(dynamic, 8)
    for (int a = 0; a < m; ++a)
      for (int b = 0; b < m; ++b) {
        const double* ga = GT.data() + (size_t)a * ldg;
        const double* gb = GT.data() + (size_t)b * ldg;
        double acc = 0.0;
        for (int k = 0; k < m; ++k) acc += ga[k] * gb[k];
        sinv[(size_t)a * m + b] = acc;
      }
    return SDP_OK;
  });
}

const char* sdp_last_error(void) { return g_err.c_str(); }

}  // extern "C"
