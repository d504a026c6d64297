// Communicators of the clique-sharded iteration (the paper's "in
// parallel" over cliques).  The iteration needs one
// operation: an in-place sum all-reduce of a device fp64 buffer, enqueued on the
// handle's stream.
//
//  * NcclComm: one process per GPU, NCCL (dlopen, nccl_dl.cpp) -- the product path.
//  * LoopComm: an in-process group of `world` handles (one host thread each, any
//    devices of the process with peer access, typically all on one GPU).  It
//    exists so that the sharded device path -- the shard plan, the partial
//    scatter sums of shared coordinates, the owned-column GEMV, the shared-
//    coordinate fix-up and the residual reduction -- runs and is checked against
//    the oracle on the one GPU a test box has.  No kernel ever waits on another
//    rank's kernel: ranks meet on the host (a barrier), and the device order is
//    expressed with CUDA events only: every rank records "my buffer is ready";
//    rank 0's stream waits for all of them and sums the buffers in rank order into
//    a group scratch buffer (so results are bit-identical whatever the timing);
//    every rank's stream waits for that sum and copies it back.  Rank 0 waits for
//    all copies of the previous round before it overwrites the scratch.
#include <condition_variable>
#include <mutex>
#include <vector>

#include "internal.h"

namespace sdp {

namespace {

struct NcclComm final : Comm {
  void* comm = nullptr;
  NcclComm(const void* id, int w, int r) {
    world = w;
    rank = r;
    comm = nccl_comm_init(id, w, r);
  }
  ~NcclComm() override {
    if (comm) nccl_comm_destroy(comm);
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t s) override { nccl_allreduce_sum(comm, buf, n, s); }
};

constexpr int kLoopMax = 16;
struct LoopPtrs {
  const double* p[kLoopMax];
};

__global__ void k_loop_sum(LoopPtrs src, int world, double* __restrict__ dst, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double s = src.p[0][i];
    for (int r = 1; r < world; ++r) s += src.p[r][i];  // fixed rank order
    dst[i] = s;
  }
}

}  // namespace

struct LoopGroup {
  int world = 0;
  int device = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<double*> bufs;
  std::vector<size_t> counts;
  std::vector<cudaEvent_t> ready, copied;
  cudaEvent_t done = nullptr;
  double* scratch = nullptr;
  size_t cap = 0;
  bool first = true;
  bool ok = true;  // rank 0's count check of the current call (read after the second barrier)
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace {
struct LoopComm final : Comm {
  LoopGroup* g;
  LoopComm(LoopGroup* grp, int w, int r) : g(grp) {
    world = w;
    rank = r;
  }
  bool loopback() const override { return true; }
  void allreduce_sum(double* buf, size_t n, cudaStream_t s) override {
    LoopGroup& G = *g;
    G.bufs[rank] = buf;
    G.counts[rank] = n;
    SDP_CUDA_TRY(cudaEventRecord(G.ready[rank], s));
    G.barrier();
    bool ok = true;
    if (rank == 0) {
      for (int r = 0; r < world; ++r) ok &= G.counts[r] == n;
      G.ok = ok;
      if (ok && n > 0) {
        for (int r = 0; r < world; ++r) {
          SDP_CUDA_TRY(cudaStreamWaitEvent(s, G.ready[r], 0));
          if (!G.first) SDP_CUDA_TRY(cudaStreamWaitEvent(s, G.copied[r], 0));
        }
        if (n > G.cap) {
          SDP_CUDA_TRY(cudaStreamSynchronize(s));
          if (G.scratch) cudaFree(G.scratch);
          G.scratch = nullptr;
          SDP_CUDA_TRY(cudaMalloc(&G.scratch, n * sizeof(double)));
          G.cap = n;
        }
        LoopPtrs lp{};
        for (int r = 0; r < world; ++r) lp.p[r] = G.bufs[r];
        const int blocks = (int)std::min<size_t>((n + 255) / 256, 4 * 148);
        k_loop_sum<<<blocks, 256, 0, s>>>(lp, world, G.scratch, n);
        SDP_CUDA_TRY(cudaGetLastError());
      }
      SDP_CUDA_TRY(cudaEventRecord(G.done, s));
      G.first = false;
    }
    G.barrier();
    // (counts[] may already hold a fast rank's next call here: use rank 0's verdict)
    ok = G.ok;
    if (!ok) throw Error{SDP_E_INVALID_ARG, "loopback all-reduce: ranks passed different counts"};
    if (n > 0) {
      SDP_CUDA_TRY(cudaStreamWaitEvent(s, G.done, 0));
      SDP_CUDA_TRY(cudaMemcpyAsync(buf, G.scratch, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    SDP_CUDA_TRY(cudaEventRecord(G.copied[rank], s));
  }
};
}  // namespace

Comm* make_nccl_comm(const void* id128, int world, int rank) { return new NcclComm(id128, world, rank); }

Comm* make_loop_comm(void* group, int world, int rank) {
  LoopGroup* g = static_cast<LoopGroup*>(group);
  if (!g) throw Error{SDP_E_INVALID_ARG, "loopback group is NULL"};
  if (g->world != world) throw Error{SDP_E_INVALID_ARG, "loopback group size differs from world"};
  return new LoopComm(g, world, rank);
}

}  // namespace sdp

using namespace sdp;

extern "C" {

int sdp_loopback_create(int32_t world, int32_t device, void** out) {
  if (!out || world < 1 || world > kLoopMax) {
    set_error("sdp_loopback_create: need out != NULL and 1 <= world <= 16");
    return SDP_E_INVALID_ARG;
  }
  *out = nullptr;
  LoopGroup* g = new LoopGroup();
  g->world = world;
  g->device = device;
  g->bufs.assign(world, nullptr);
  g->counts.assign(world, 0);
  g->ready.assign(world, nullptr);
  g->copied.assign(world, nullptr);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  for (int r = 0; r < world && e == cudaSuccess; ++r) {
    e = cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->copied[r], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error(std::string("sdp_loopback_create: ") + cudaGetErrorString(e));
    delete g;
    return SDP_E_CUDA;
  }
  *out = g;
  return SDP_OK;
}

int sdp_loopback_destroy(void* group) {
  LoopGroup* g = static_cast<LoopGroup*>(group);
  if (!g) return SDP_OK;
  cudaDeviceSynchronize();
  for (auto e : g->ready)
    if (e) cudaEventDestroy(e);
  for (auto e : g->copied)
    if (e) cudaEventDestroy(e);
  if (g->done) cudaEventDestroy(g->done);
  if (g->scratch) cudaFree(g->scratch);
  delete g;
  return SDP_OK;
}

}  // extern "C"
