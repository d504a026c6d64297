// Register-resident-V Jacobi tier for the PSD projection (E:XkUpdate P:244-253,
// E:zkUpdate P:403-410), orders k <= 64 (padded to KP in {8, 16, 32, 64}).
//
// Same method as kernels_psd.cu (two-sided cyclic Jacobi, parallel round-robin
// ordering, stop at off(A)_F <= 1e-15 ||A||_F, clip at 0), different data
// movement:
//  * "slot order": the round-robin permutation is applied physically, so the
//    P = KP/2 pairs of every step are the adjacent slots (2i, 2i+1).  The slot
//    map ns() is the circle method's rotation written on slots; it covers every
//    pair exactly once per sweep of KP-1 steps and is the identity again at
//    every sweep boundary (checked in tests/test_slot_schedule.py), so the
//    eigenpairs come out in natural order.
//  * A (symmetric, KP x KP) lives in shared memory, double-buffered: a 2x2 block
//    (2i..2i+1, 2j..2j+1) is read with two 16-byte loads from the current buffer
//    and written, already permuted by ns(), into the next buffer.
//  * V: row r of V lives in the registers of Q consecutive lanes (S = KP/Q
//    slots each, S >= 4); the column rotation V <- V J is register-local, the
//    slot permutation is a static register shuffle plus two warp shuffles (one
//    element moves to each neighbouring lane per step), so V costs no
//    shared-memory traffic until the reconstruction.
// Group = G = KP * Q threads per matrix (sub-warp, warp, or named-barrier group).
#include "psd_rv.cuh"

namespace sdp {

namespace {

template <int KP, int Q, int MODE>
__global__ void __launch_bounds__(RvLayout<KP, Q>::threads()) k_psd_rv(ProjArgs a) {
  if (a.done && *a.done) return;
  using Lay = RvLayout<KP, Q>;
  constexpr int G = Lay::G;
  constexpr int NBUF = rv_nbuf<MODE>();
  constexpr int NG = Lay::groups_per_cta();
  extern __shared__ double smem[];
  int* tab = (int*)(smem + NG * Lay::template per_group<NBUF>());
  for (int b = threadIdx.x; b < Lay::NBLK; b += Lay::threads()) {
    // row-major enumeration of i <= j < P: row i holds P - i blocks
    int i = 0, rem = b;
    while (rem >= Lay::P - i) {
      rem -= Lay::P - i;
      ++i;
    }
    tab[b] = (i << 16) | (i + rem);
  }
  __syncthreads();
  const int grp = threadIdx.x / G;
  RvGroup<G> g;
  g.tid = threadIdx.x % G;
  g.mask = (G >= 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) / G * G));
  g.bar = 1 + grp;
  double* base = smem + (size_t)grp * Lay::template per_group<NBUF>();
  double* A0 = base;
  double* A1 = base + KP * Lay::LD;
  double* T = NBUF == 3 ? A1 + KP * Lay::LD : nullptr;
  double* rc = base + NBUF * KP * Lay::LD;
  double* rs = rc + Lay::P;
  double* rt = rs + Lay::P;
  g.red = rt + Lay::P;
  for (int slot = blockIdx.x * NG + grp; slot < a.count; slot += gridDim.x * NG) {
    const int task = a.ids ? a.ids[slot] : slot;
    project_rv<KP, Q, MODE>(g, a.ksz[task], a.off[task], task, A0, A1, T, rc, rs, rt, tab, a);
  }
}

template <int KP, int Q, int MODE>
void launch_rv(const ProjArgs& a, cudaStream_t s) {
  using Lay = RvLayout<KP, Q>;
  constexpr int NG = Lay::groups_per_cta();
  const size_t sm = Lay::template bytes<rv_nbuf<MODE>()>();
  int grid = (a.count + NG - 1) / NG;
  k_psd_rv<KP, Q, MODE><<<grid, Lay::threads(), sm, s>>>(a);
}

template <int KP, int Q, int MODE>
void rv_attr() {
  cudaFuncSetAttribute(k_psd_rv<KP, Q, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)RvLayout<KP, Q>::template bytes<rv_nbuf<MODE>()>());
}

// (KP, Q) per tier: many matrices -> small groups; few matrices -> wide groups
#define RV_TIERS(X, MODE) X(8, 1, MODE) X(16, 2, MODE) X(32, 2, MODE) X(64, 4, MODE) X(32, 8, MODE) X(16, 4, MODE) X(8, 2, MODE)
#define RV_ATTR(KP, Q, MODE) rv_attr<KP, Q, MODE>();
template <int MODE>
void rv_attrs() {
  RV_TIERS(RV_ATTR, MODE)
}

}  // namespace

void psd_rv_init_attributes() {
  rv_attrs<PM_BATCH>();
  rv_attrs<PM_PRIMAL>();
  rv_attrs<PM_DUAL>();
}

// kp for warm-start storage of the register-V tiers
int rv_kp(int bucket) { return bucket == B_RV8 ? 8 : bucket == B_RV16 ? 16 : bucket == B_RV32 ? 32 : 64; }

void launch_projection_rv(int bucket, int mode, const ProjArgs& a, cudaStream_t s) {
  if (a.count <= 0) return;
  // few matrices: spread each over more lanes so the batch still fills the GPU
  const bool few = a.count < kFewMatrices;
#define RV_CASE(KP, Q)                  \
  if (mode == PM_BATCH)                 \
    launch_rv<KP, Q, PM_BATCH>(a, s);   \
  else if (mode == PM_PRIMAL)           \
    launch_rv<KP, Q, PM_PRIMAL>(a, s);  \
  else                                  \
    launch_rv<KP, Q, PM_DUAL>(a, s);
  switch (bucket) {
    case B_RV8:
      if (few) { RV_CASE(8, 2) } else { RV_CASE(8, 1) }
      break;
    case B_RV16:
      if (few) { RV_CASE(16, 4) } else { RV_CASE(16, 2) }
      break;
    case B_RV32:
      if (few) { RV_CASE(32, 8) } else { RV_CASE(32, 2) }
      break;
    case B_RV64: RV_CASE(64, 4) break;
  }
#undef RV_CASE
}

}  // namespace sdp
