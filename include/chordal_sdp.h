/*
 * chordal_sdp.h -- C ABI of the B200-native per-iteration hot path of the
 * chordally decomposed ADMM for sparse SDPs (arXiv 1609.06068).
 *
 * Citations: "P:L" = /root/reference/PAPER.md line L (LaTeX labels given too).
 *
 * Problem: given b in R^m, C in S^n and A_1..A_m in S^n,
 *   primal  E:PrimalSDP  min <C,X>  s.t. A(X) = b, X PSD
 *   dual    E:DualSDP    max <b,y>  s.t. A*(y) + Z = C, Z PSD.
 * sdp_setup() finds the aggregate pattern, its chordal extension
 * (exact minimum degree + symbolic elimination), the maximal cliques
 * C_1..C_p, the entry selectors H_k, D = sum H_k^T H_k
 * and the cached factor of S = A D^-1 A^T.  sdp_step()/sdp_solve()
 * run Algorithm 1 (primal) or Algorithm 2 (dual) on the
 * GPU.  sdp_project_psd_batch() exposes the clique projection P_k (E:XkUpdate,
 * P:244-253) on its own.
 *
 * Conventions
 *  - All indices are 0-based int32; matrix entries are given for the upper
 *    triangle (row <= col) and are UNSCALED matrix values.  Internally the
 *    library uses svec (off-diagonal x sqrt 2) over the extended pattern.
 *  - "Host" pointers are ordinary CPU memory owned by the caller and only read
 *    (or written, for getters) during the call.  "Device" pointers are CUDA
 *    global memory on the handle's device, owned by the caller.
 *  - Every call returns an int status: SDP_OK (0), SDP_MAX_ITER (1, not an
 *    error) or a negative SDP_E_* code; sdp_last_error() gives a thread-local
 *    message naming the offending argument.
 *  - Handles are not thread-safe; distinct handles are independent.
 *  - Pattern order ("canonical"): upper-triangle entries of the extended
 *    pattern sorted by column, then row.  Clique order: cliques sorted
 *    ascending inside, list sorted lexicographically.  Stacked clique vectors
 *    concatenate each clique's svec in packed-upper column-major local order.
 */
#ifndef CHORDAL_SDP_H
#define CHORDAL_SDP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SDP_OK 0
#define SDP_MAX_ITER 1             /* sdp_solve hit max_iters: not an error */
#define SDP_E_INVALID_ARG (-1)     /* bad index, i > j, duplicate entry, n or m <= 0, ...   */
#define SDP_E_RANK_DEFICIENT (-2)  /* S = A D^-1 A^T not positive definite          */
#define SDP_E_CUDA (-3)            /* CUDA runtime error (message has the CUDA error string)*/
#define SDP_E_NCCL (-4)            /* reserved: multi-GPU communication error               */
#define SDP_E_OOM (-5)             /* device or host allocation failed                      */
#define SDP_E_NUMERICAL (-6)       /* NaN/Inf in the iterates                       */
#define SDP_E_STATE (-7)           /* call not valid in the handle's current state          */

#define SDP_FORM_PRIMAL 0          /* Algorithm 1 */
#define SDP_FORM_DUAL 1            /* Algorithm 2, Remark 2 ordering */

#define SDP_A_COO 0                /* A given as (con, row, col, val) entries              */
#define SDP_A_DENSE_ON_PATTERN 1   /* A given as one (row, col) list + m x npat values     */

#define SDP_MAX_K 1024             /* largest clique / batch matrix order supported         */

/* ---- problem data ------------------------------------------- */
typedef struct {
  int32_t n;                 /* order of C, A_i (cone S^n)                          */
  int32_t m;                 /* number of equality constraints                      */
  /* C: upper-triangle COO, c_nnz entries, (c_row[t] <= c_col[t]) */
  int64_t c_nnz;
  const int32_t* c_row;
  const int32_t* c_col;
  const double* c_val;
  /* A_1..A_m */
  int32_t a_fmt;             /* SDP_A_COO or SDP_A_DENSE_ON_PATTERN                  */
  int64_t a_nnz;             /* COO: number of entries; DENSE: number of pattern entries npat */
  const int32_t* a_con;      /* COO: constraint index in [0,m) per entry; DENSE: unused (NULL) */
  const int32_t* a_row;      /* COO: per entry; DENSE: per pattern entry             */
  const int32_t* a_col;
  const double* a_val;       /* COO: a_nnz values; DENSE: m x npat row-major values  */
  const double* b;           /* m values                                             */
  /* optional user pattern E ("described by the graph G(V,E)"), may be NULL */
  int64_t e_nnz;
  const int32_t* e_row;
  const int32_t* e_col;
} sdp_problem;

/* Optional device-memory allocator (lets the caller -- e.g. PyTorch's caching
 * allocator through torch uint8 tensors -- own every device byte of a handle or plan).
 * alloc(ctx, bytes, device) returns a device pointer on `device` aligned to >= 256 B,
 * or NULL on failure (the call then fails with SDP_E_OOM); free(ctx, ptr, device)
 * releases it.  The library calls free only for pointers it got from alloc, after
 * synchronising the work that used them.  NULL allocator = cudaMalloc / cudaFree. */
typedef struct {
  void* (*alloc)(void* ctx, size_t bytes, int32_t device);
  void (*free)(void* ctx, void* ptr, int32_t device);
  void* ctx;
} sdp_allocator;

typedef struct {
  int32_t form;              /* SDP_FORM_PRIMAL or SDP_FORM_DUAL                     */
  double rho;                /* ADMM penalty rho > 0; default 1.0     */
  int32_t device;            /* CUDA device ordinal; default 0                        */
  void* stream;              /* cudaStream_t to enqueue on (NULL = default stream)   */
  int32_t check_every;       /* sdp_solve: host reads the stop flag every K iterations (default 10) */
  int32_t use_graph;         /* 1 (default): replay one captured CUDA graph per iteration */
  int32_t rank, world;       /* clique sharding over `world` ranks (one GPU each); default 0, 1 */
  const void* nccl_id;       /* world > 1: 128-byte id from sdp_nccl_unique_id on rank 0, same on all ranks */
  /* sdp_solve residual balancing (Boyd et al. 2011 Sec. 3.4.1, cited for the residuals at P:263-265):
   * after every check_every-th iteration that did not stop, rho <- adapt_tau * rho if
   * eps_p > adapt_mu * eps_d, rho <- rho / adapt_tau if eps_d > adapt_mu * eps_p.  The KKT
   * matrix is rho-free, so nothing is refactorised.  Default off (0), mu 10, tau 2. */
  int32_t adapt_rho;
  double adapt_mu;
  double adapt_tau;
  const sdp_allocator* allocator;  /* NULL: cudaMalloc; else every device buffer of the handle
                                    * (state, A, factor, workspaces, setup scratch) comes from it;
                                    * the struct is copied, ctx must outlive the handle */
  void* comm;                /* world > 1 without NCCL: an in-process loopback group
                              * (sdp_loopback_create) shared by the `world` handles of one
                              * process; NULL = NCCL (nccl_id) */
} sdp_options;

typedef struct {
  int64_t iters;             /* iterations run since the last reset                 */
  double eps_p, eps_d;       /* residuals of the last iteration (reading G9) */
  double objective;          /* primal <c,x> / dual <b,y> of the last iteration (G17) */
  double setup_s;            /* host wall time of sdp_setup                          */
  int64_t n, m, N, p;        /* sizes: pattern coordinates N, cliques p              */
  int64_t kmin, kmax, stot;  /* clique order range, stacked clique length sum k(k+1)/2 */
  int32_t form;
  int32_t s_diagonal;        /* 1 if S = A D^-1 A^T is diagonal (elementwise KKT)   */
  int64_t jacobi_capped;     /* count of projections that hit the sweep cap          */
  int32_t launches_per_iter; /* kernels launched per ADMM iteration                   */
  int64_t jacobi_sweeps;     /* total Jacobi sweeps over all projections since reset  */
  double rho;                /* penalty currently in force (changes with adapt_rho / sdp_set_rho) */
  int32_t pipelined;         /* 1: the pipelined primal iteration is in use:
                              * sdp_step(n) overlaps the projections with the A passes of the
                              * neighbouring iterations; SDP_PIPELINE=0 at setup turns it off */
  int32_t s_factor;          /* factorisation of S = A D^-1 A^T: 0 diagonal, 1 dense
                              * Cholesky, 2 sparse Cholesky in a minimum-degree order */
  int64_t nnz_l;             /* nonzeros of the Cholesky factor (0 when S is diagonal) */
  int32_t fused;             /* 1: the fused persistent iteration is in use (small single-rank
                              * problems, all cliques k <= 32): one
                              * cooperative kernel launch per sdp_step / sdp_solve call runs every
                              * phase of every iteration.  SDP_FUSED=0 at setup turns it off */
} sdp_info;

typedef struct sdp_handle_s* sdp_handle;

/* Fill *opt with the defaults listed above. */
void sdp_default_options(sdp_options* opt);

/* Build the decomposed problem and upload it (host setup, run once; timed
 * separately, "Setup: Chordal decomposition, KKT factorization").
 * Sharding (world > 1, collective: every rank calls it with the same full
 * problem): cliques are assigned to ranks by LPT on k^3 (sdp_shard_plan), each
 * rank runs the projections of its cliques and the affine step on the
 * coordinates they touch; per iteration the ranks all-reduce the partial sums of
 * shared coordinates (with the 6 residual scalars packed behind them in the
 * primal form) and the m-vector A D^-1 r1 over owned columns (the dual form adds
 * a third all-reduce for its residual scalars).  Getters of a sharded handle are
 * collective and return the full (global) vectors.
 * prob, opt: host, read during the call.  out: receives the handle.
 * Errors: SDP_E_INVALID_ARG (index out of range, row > col, duplicate entry,
 * n <= 0, m <= 0, clique order > SDP_MAX_K), SDP_E_RANK_DEFICIENT, SDP_E_CUDA,
 * SDP_E_OOM.  On error *out is NULL. */
int sdp_setup(const sdp_problem* prob, const sdp_options* opt, sdp_handle* out);

/* Run exactly `iters` ADMM iterations from the current state, no stopping test.
 * Asynchronous on the handle's stream; returns after enqueueing.  When
 * sdp_info.pipelined is 1 the iterations are issued as the pipelined schedule
 * (projections of one half of the cliques overlap the A
 * passes of the neighbouring iterations) on helper streams that fork from and
 * join back into the handle's stream.  The call also leaves the first part of
 * the next iteration issued; every getter, checkpoint, rho change and reset
 * first restores the finished iteration's x and y, so the state seen through
 * this API is always the iteration boundary. */
int sdp_step(sdp_handle h, int32_t iters);

/* Iterate until max(eps_p, eps_d) < tol (Algorithm 1/2 line 3) or until
 * max_iters iterations have run since the last reset.  The stop is exact (the
 * state is that of the first converged iteration).  Synchronises the stream.
 * info (host, may be NULL) receives the final info.
 * Returns SDP_OK, SDP_MAX_ITER, or SDP_E_NUMERICAL. */
int sdp_solve(sdp_handle h, int32_t max_iters, double tol, sdp_info* info);

/* Zero the ADMM state (initial guesses = 0, reading G12). */
int sdp_reset(sdp_handle h);

/* Change rho between iterations; the cached factor is rho-independent. */
int sdp_set_rho(sdp_handle h, double rho);

/* Synchronise and report sizes, residuals and objective (host out). */
int sdp_get_info(sdp_handle h, sdp_info* info);

/* PSD completion of the current SDP primal X (SDP_VEC_SDP_X: x in the primal form,
 * -rho x in the dual form; Theorem 1).
 * X is known on the extended chordal pattern E' only; out (host, n*n
 * doubles, row-major, written entirely) receives a completion that agrees with X
 * on E' and fills every other entry by the perfect-elimination construction:
 * vertices in reverse elimination order, X[v,u] = X[v,a] X[a,a]^+ X[a,u] with
 * a = the later neighbours of v (a clique of E'); the pseudo-inverse drops
 * eigenvalues below rtol * max|lambda| (take it near the solve accuracy, e.g.
 * 1e-8: separator blocks of a converged X are singular to that accuracy).  When every
 * maximal-clique block of X is PSD (a converged solve, either form) the result is PSD
 * (Grone); for definite blocks it is the maximum-determinant completion.  Host
 * computation, O(n^2 * max clique) once per call; world == 1 or collective.
 * Errors: SDP_E_INVALID_ARG. */
int sdp_complete_x(sdp_handle h, double rtol, double* out);

/* The elimination order of the chordal analysis (n vertices, host int32): a
 * perfect elimination order of E' (exact minimum degree, ties to the lowest
 * index; reading G13). */
int sdp_get_elimination_order(sdp_handle h, int32_t* order);

/* ---- getters: synchronise the stream, copy into host buffers ----------- */
/* Iterates of the decomposed problem (the state of Algorithm 1 / 2): */
#define SDP_VEC_X 0        /* N: KKT x (svec on the pattern; E:OptCondMinYPrimal / E:OptCondMinYDual) */
#define SDP_VEC_Y 1        /* m: KKT y                                               */
#define SDP_VEC_XMAT 2     /* N: unscaled matrix entries of the KKT x on the pattern */
/* The primal-dual SDP pair those iterates carry (Remark 1; the KKT
 * multipliers are rho*y, and rho*x), the same in both forms:
 *   primal form (Alg. 1): X = x,        yhat = -rho y,  Z_k = lambda_k
 *   dual form   (Alg. 2): X = -rho x,   yhat = y,       Z_k = z_k
 * with rho the penalty of the last iteration.  X satisfies A(X) = b exactly in both
 * forms (every iterate); <C,X> - <b,yhat> -> 0 and X, Z_k -> PSD at convergence. */
#define SDP_VEC_SDP_X 3    /* N: unscaled matrix entries X_ij of the SDP primal X on the pattern */
#define SDP_VEC_SDP_Y 4    /* m: the SDP dual yhat (E:DualSDP)                        */
#define SDP_BLK_XK 0       /* stacked x_k (primal) or z_k (dual)                      */
#define SDP_BLK_LAMBDA 1   /* stacked lambda_k                                       */
#define SDP_BLK_VK 2       /* stacked v_k (dual only)                                */
#define SDP_BLK_SDP_Z 3    /* stacked svec Z_k of the SDP dual slack Z = sum_k E_k^T Z_k E_k (Theorem 2) */
int sdp_get_vector(sdp_handle h, int32_t which, double* out);
int sdp_get_blocks(sdp_handle h, int32_t which, double* out);   /* stot values */
/* Pattern coordinates (row[N], col[N]) in canonical order. */
int sdp_get_pattern(sdp_handle h, int32_t* row, int32_t* col);
/* Clique sizes (p values) and the concatenated sorted vertex lists (sum of sizes). */
int sdp_get_cliques(sdp_handle h, int32_t* sizes, int32_t* vertices);
/* Per-iteration history since reset: rows of (eps_p, eps_d, objective); at most cap rows. */
int sdp_get_history(sdp_handle h, double* out, int64_t cap, int64_t* rows);

/* Per-phase timing: run `iters` iterations (no graph) with CUDA events recorded
 * on the handle's stream around every phase; out_ms[ph] (host, capacity
 * SDP_NUM_PHASES) receives the mean device time per iteration of phase ph:
 * 0 gemv (A.v), 1 kkt-small (y = S^-1 u), 2 gemvT (A^T.y + x),
 * 3 projection (all tiers), 4 scatter, 5 dual update, 6 finalize.
 * Advances the state like sdp_step.  Synchronises. */
#define SDP_NUM_PHASES 7
int sdp_profile_phases(sdp_handle h, int32_t iters, double* out_ms);

/* ---- checkpoint / resume (warm-start state I/O) -----------
 * The device-resident ADMM state at an iteration boundary -- x_k / z_k, lambda_k,
 * v_k, the KKT x and y, the next right-hand side r1 / D, sum_k H_k^T x_k of the
 * previous iteration (for eps_d), residuals, iteration count, rho, residual
 * history, warm-start eigenbases -- serialised into a caller-owned host buffer.
 * Loading it into a handle set up from the same problem, form and sharding
 * continues the run bit-identically (tested).  Sharded handles save their local
 * view (one blob per rank).  Errors: SDP_E_INVALID_ARG (NULL, buffer too small,
 * or a blob from a different problem / form / sharding). */
int sdp_state_bytes(sdp_handle h, int64_t* bytes);   /* size of the blob for the current state */
int sdp_save_state(sdp_handle h, void* host_out, int64_t capacity);
int sdp_load_state(sdp_handle h, const void* host_in, int64_t bytes);

/* Device bytes the handle currently holds (live allocations, from the allocator of
 * sdp_options or cudaMalloc) and the peak during setup (host out, either may be NULL). */
int sdp_workspace_bytes(sdp_handle h, int64_t* live_bytes, int64_t* peak_bytes);

/* Free all resources of the handle (synchronises). */
int sdp_destroy(sdp_handle h);

/* ---- chordal analysis only (host, no GPU) ------------------------------ */
/* Chordal extension + maximal cliques of the pattern given by (row, col) upper
 * entries (diagonal implicit).  sizes: host buffer of capacity n; vertices:
 * capacity cap_vertices; *p receives the clique count, *nv the vertex count.
 * Same rules as sdp_setup (exact minimum degree, lowest index on ties). */
int sdp_chordal_cliques(int32_t n, int64_t nnz, const int32_t* row, const int32_t* col,
                        int32_t* p, int32_t* sizes, int64_t cap_vertices, int32_t* vertices,
                        int64_t* nv, int64_t* fill_edges);

/* ---- batched PSD projection (E:XkUpdate) ---------------------- */
typedef struct sdp_psd_plan_s* sdp_psd_plan;

/* Plan for `count` matrices of orders h_sizes[i] (host, 1 <= k <= SDP_MAX_K).
 * Matrix i occupies k(k+1)/2 doubles at offset sum_{j<i} k_j(k_j+1)/2 of the
 * in/out arrays, packed upper column-major, UNSCALED entries. */
int sdp_psd_plan_create(int64_t count, const int32_t* h_sizes, int32_t device, sdp_psd_plan* out);
/* Same, with every device buffer of the plan (workspaces and the host-path staging
 * buffers) taken from `allocator` (copied; NULL = cudaMalloc). */
int sdp_psd_plan_create_ex(int64_t count, const int32_t* h_sizes, int32_t device, const sdp_allocator* allocator,
                           sdp_psd_plan* out);
/* out_i = argmin_{P PSD} ||P - in_i||_F for every i.  d_in, d_out: device,
 * may alias (in place).  Asynchronous on `stream` (cudaStream_t, NULL = default). */
int sdp_project_psd_batch(sdp_psd_plan plan, const double* d_in, double* d_out, void* stream);
/* Same, from/to HOST buffers (copies inside the call; synchronous).  h_in, h_out: host, owned by
 * the caller, `values` doubles each, must not alias.  Pageable buffers are staged through two
 * pinned chunks (host copies overlapping the DMA).  When BOTH buffers are pinned (cudaHostAlloc /
 * torch pin_memory) and the plan holds >= 16384 matrices, the batch is streamed as four contiguous
 * sub-plans (created on the first such call, from the plan's allocator) whose H2D copy, projection
 * and D2H copy overlap; each matrix may then take a different tier than in the whole-batch plan
 * (tier choice depends on the count per size range), so results agree to rounding, not bitwise. */
int sdp_project_psd_batch_host(sdp_psd_plan plan, const double* h_in, double* h_out, void* stream);
int64_t sdp_psd_plan_values(sdp_psd_plan plan);   /* total doubles of in/out */
/* Kernel launches one sdp_project_psd_batch call makes (diagnostics; -1 if plan is NULL). */
int32_t sdp_psd_plan_launches(sdp_psd_plan plan);
int sdp_psd_plan_destroy(sdp_psd_plan plan);

/* ---- multi-GPU helpers ----------------------------------------------------- */
/* 128-byte NCCL unique id (rank 0 calls it and broadcasts it, e.g. through
 * torch.distributed).  NCCL is loaded with dlopen("libnccl.so.2"). */
int sdp_nccl_unique_id(void* out128);
/* In-process loopback group for `world` sharded handles of ONE process (one host
 * thread per rank, handles on `device` or on devices with peer access to it): pass it
 * as sdp_options.comm with rank / world and no nccl_id.  Each all-reduce of the
 * iteration meets on the host (a barrier inside the call that enqueues it) and is
 * ordered on the devices by CUDA events only (no kernel waits for another rank):
 * rank 0 sums the ranks' buffers in rank order, every rank copies the sum back, so
 * results do not depend on timing.  It exists to run and test the sharded device
 * path on one GPU; one process per GPU over NCCL is the product path.
 * Handles using it do not capture CUDA graphs (use_graph is ignored).  Every call
 * on such handles must be made by all ranks (collective), each from its own thread.
 * world <= 16.  Destroy the group after its handles. */
int sdp_loopback_create(int32_t world, int32_t device, void** out);
int sdp_loopback_destroy(void* group);

/* Host-only shard plan of the pattern (row, col) for `rank` of `world`:
 * clique_rank[p] (the rank of every clique, canonical clique order: LPT on k^3 + 16, most
 * expensive clique first, each to the least-loaded rank), local_coords[n_local] (pattern
 * coordinates the rank's cliques touch, sorted), owned[n_local] (1 if the rank owns the coordinate:
 * the rank of its first clique), shared_coords[n_shared] (coordinates touched by >= 2 ranks).
 * cap = capacity of every output buffer (p <= cap). */
int sdp_shard_plan(int32_t n, int64_t nnz, const int32_t* row, const int32_t* col, int32_t world, int32_t rank,
                   int32_t* clique_rank, int64_t* n_local, int32_t* local_coords, uint8_t* owned,
                   int64_t* n_shared, int32_t* shared_coords, int64_t cap);

/* ---- sparse Cholesky of S (host only) ------------------------------------
 * The factorisation sdp_setup uses when S = A D^-1 A^T is sparse: minimum-degree order (the
 * chordal analysis of S's graph), left-looking S = L L^T, G = L^-1 along elimination-tree paths.
 * S given as CSR with both triangles (ptr[m+1], idx, val; host).  sinv (host, m*m row-major)
 * receives G^T G = S^-1.  Returns SDP_E_RANK_DEFICIENT for a pivot <= 1e-12 S_ii, SDP_E_STATE
 * if the factor is denser than m^2 / 8 and force_sparse == 0.  For tests and diagnostics. */
int sdp_schur_inverse_host(int32_t m, const int64_t* ptr, const int32_t* idx, const double* val, int32_t force_sparse,
                           double* sinv, int64_t* nnz_l);

const char* sdp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CHORDAL_SDP_H */
