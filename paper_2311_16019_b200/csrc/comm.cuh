// comm.cuh — transports for row-sharded (multi-rank) contexts.
//
// A sharded context owns a contiguous range of grid planes (3-D) / lines (2-D).  Every
// block step exchanges, per sequence (north star, BASELINE.json):
//   * the ghost planes of the newest block Z_{j+1} with the two neighbour ranks (halo),
//   * the k r^2 Gram-Schmidt inner products and the r^2 Gram (allreduce, sum),
//   * the s x r partial sketch (allreduce, sum: S is linear in rows and hashed on GLOBAL
//     row indices, so the rank partials sum to S W exactly up to rounding order).
// Reductions must give bit-identical results on every rank (each rank then computes the
// same r x r coefficients and the same sketch-space QR); both transports guarantee it.
//
//   NcclComm   one process per GPU.  libnccl is dlopen'ed (the copy torch already loaded);
//              the caller creates the communicator from a unique id it broadcasts itself.
//              One split communicator per channel (U/V main, U/V side, setup), so the
//              collectives issued on different streams never share a communicator.
//   LocalComm  P virtual ranks in ONE process on one GPU, one host thread per rank (the
//              parity tests).  Host barriers + CUDA events order the streams; the sums and
//              ghost copies are ordinary kernels / device copies that never wait on another
//              kernel (no spin loops across ranks).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace sylv {

enum Chan : int { kChanUMain = 0, kChanVMain = 1, kChanUSide = 2, kChanVSide = 3, kChanSetup = 4, kNumChan = 5 };

struct CommError {
  std::string what;
};

struct Comm {
  int nranks = 1, rank = 0;
  std::vector<int64_t> rb, re;   // row ranges of all ranks (rank order = row order)
  virtual ~Comm() {}
  // in-place sum over ranks; identical result on every rank
  virtual void allreduce(double* buf, size_t n, cudaStream_t st, int chan) = 0;
  // recv[e] = sum over ranks of send[rank * n + e], e < n (send: nranks * n values): the rows of
  // the summed sketch that this rank's shard of the sketch space owns
  virtual void reduce_scatter(const double* send, double* recv, size_t n, cudaStream_t st, int chan) = 0;
  // fill the ghost rows of an SoA block (data = local row 0 of column 0): the gz rows
  // before each column from the lower neighbour's last gz rows, the gz rows after it from
  // the upper neighbour's first gz rows.  Ranks without a neighbour leave the ghosts alone.
  virtual void halo(double* data, int R, int64_t ld, int64_t gz, cudaStream_t st, int chan) = 0;
  // host-level allgather of this rank's row range (setup; blocking)
  virtual void gather_ranges(int64_t row_begin, int64_t row_end) = 0;
  // this rank failed inside a collective sequence: release peers blocked on it (LocalComm)
  virtual void abort() {}
  int lower() const { return rank > 0 ? rank - 1 : -1; }
  int upper() const { return rank + 1 < nranks ? rank + 1 : -1; }
  int64_t rows(int r) const { return re[r] - rb[r]; }
};

// ---------------------------------------------------------------------------------------
// NCCL
// ---------------------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);   // torch's copy if loaded
      if (!api.h) api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
#define SYLV_NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, "nccl" #f))
    SYLV_NCCL_SYM(GetUniqueId);
    SYLV_NCCL_SYM(CommInitRank);
    SYLV_NCCL_SYM(CommSplit);
    SYLV_NCCL_SYM(CommDestroy);
    SYLV_NCCL_SYM(CommCount);
    SYLV_NCCL_SYM(CommUserRank);
    SYLV_NCCL_SYM(AllReduce);
    SYLV_NCCL_SYM(AllGather);
    SYLV_NCCL_SYM(ReduceScatter);
    SYLV_NCCL_SYM(Send);
    SYLV_NCCL_SYM(Recv);
    SYLV_NCCL_SYM(GroupStart);
    SYLV_NCCL_SYM(GroupEnd);
    SYLV_NCCL_SYM(GetErrorString);
#undef SYLV_NCCL_SYM
  });
  return api;
}

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    NcclApi& a = nccl_api();
    throw CommError{std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "nccl error")};
  }
}

struct NcclComm : Comm {
  ncclComm_t base = nullptr;
  ncclComm_t ch[kNumChan] = {};
  double* dscratch = nullptr;   // setup allgather buffer (device)

  NcclComm(int n, int r, const ncclUniqueId& id) {
    NcclApi& a = nccl_api();
    if (!a.CommInitRank || !a.CommSplit || !a.AllReduce || !a.Send) throw CommError{"libnccl not loadable"};
    nranks = n;
    rank = r;
    nccl_check(a.CommInitRank(&base, n, id, r), "ncclCommInitRank");
    try {
      for (int i = 0; i < kNumChan; ++i) nccl_check(a.CommSplit(base, 0, r, &ch[i], nullptr), "ncclCommSplit");
    } catch (...) {   // the destructor does not run for a throwing constructor
      for (auto& c : ch)
        if (c) a.CommDestroy(c), c = nullptr;
      a.CommDestroy(base);
      base = nullptr;
      throw;
    }
  }
  // over a caller-owned communicator: the channels are split from it, it is never destroyed here
  explicit NcclComm(ncclComm_t caller) {
    NcclApi& a = nccl_api();
    if (!a.CommSplit || !a.AllReduce || !a.Send || !a.CommCount || !a.CommUserRank)
      throw CommError{"libnccl not loadable"};
    nccl_check(a.CommCount(caller, &nranks), "ncclCommCount");
    nccl_check(a.CommUserRank(caller, &rank), "ncclCommUserRank");
    try {
      for (int i = 0; i < kNumChan; ++i) nccl_check(a.CommSplit(caller, 0, rank, &ch[i], nullptr), "ncclCommSplit");
    } catch (...) {
      for (auto& c : ch)
        if (c) a.CommDestroy(c), c = nullptr;
      throw;
    }
  }
  ~NcclComm() override {
    NcclApi& a = nccl_api();
    for (auto& c : ch)
      if (c) a.CommDestroy(c);
    if (base) a.CommDestroy(base);   // only the library's own base communicator
    if (dscratch) cudaFree(dscratch);
  }
  void allreduce(double* buf, size_t n, cudaStream_t st, int chan) override {
    if (n == 0) return;   // (also at world size 1: keeps the transport exercised)
    nccl_check(nccl_api().AllReduce(buf, buf, n, ncclFloat64, ncclSum, ch[chan], st), "ncclAllReduce");
  }
  void reduce_scatter(const double* send, double* recv, size_t n, cudaStream_t st, int chan) override {
    if (n == 0) return;
    if (!nccl_api().ReduceScatter) throw CommError{"ncclReduceScatter not found"};
    nccl_check(nccl_api().ReduceScatter(send, recv, n, ncclFloat64, ncclSum, ch[chan], st), "ncclReduceScatter");
  }
  void halo(double* data, int R, int64_t ld, int64_t gz, cudaStream_t st, int chan) override {
    if (nranks == 1 || gz == 0) return;
    NcclApi& a = nccl_api();
    const int lo = lower(), up = upper();
    const int64_t n = rows(rank);
    nccl_check(a.GroupStart(), "ncclGroupStart");
    for (int c = 0; c < R; ++c) {
      double* col = data + (int64_t)c * ld;
      if (lo >= 0) {
        nccl_check(a.Send(col, (size_t)gz, ncclFloat64, lo, ch[chan], st), "ncclSend");
        nccl_check(a.Recv(col - gz, (size_t)gz, ncclFloat64, lo, ch[chan], st), "ncclRecv");
      }
      if (up >= 0) {
        nccl_check(a.Send(col + n - gz, (size_t)gz, ncclFloat64, up, ch[chan], st), "ncclSend");
        nccl_check(a.Recv(col + n, (size_t)gz, ncclFloat64, up, ch[chan], st), "ncclRecv");
      }
    }
    nccl_check(a.GroupEnd(), "ncclGroupEnd");
  }
  void gather_ranges(int64_t b, int64_t e) override {
    rb.assign(nranks, 0);
    re.assign(nranks, 0);
    if (!dscratch && cudaMalloc(&dscratch, (size_t)(2 + 2 * nranks) * sizeof(double)) != cudaSuccess)
      throw CommError{"cudaMalloc (range gather)"};
    const double mine[2] = {(double)b, (double)e};   // exact: row indices < 2^53
    std::vector<double> all(2 * nranks);
    cudaStream_t st = nullptr;
    if (cudaMemcpy(dscratch, mine, sizeof(mine), cudaMemcpyHostToDevice) != cudaSuccess)
      throw CommError{"cudaMemcpy (range gather)"};
    nccl_check(nccl_api().AllGather(dscratch, dscratch + 2, 2, ncclFloat64, ch[kChanSetup], st), "ncclAllGather");
    if (cudaMemcpy(all.data(), dscratch + 2, all.size() * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      throw CommError{"cudaMemcpy (range gather)"};
    for (int r = 0; r < nranks; ++r) {
      rb[r] = (int64_t)all[2 * r];
      re[r] = (int64_t)all[2 * r + 1];
    }
  }
};

// ---------------------------------------------------------------------------------------
// In-process group of virtual ranks on one GPU
// ---------------------------------------------------------------------------------------
constexpr int kMaxLocalRanks = 16;

struct PtrPack {
  const double* p[kMaxLocalRanks];
};

// out[e] = sum_{r < nr} in.p[r][e] (rank order: the same on every rank)
__global__ void k_sum_ranks(PtrPack in, int nr, size_t n, double* __restrict__ out) {
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nr; ++r) s += in.p[r][e];
    out[e] = s;
  }
}

struct LocalGroup {
  int P = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  bool aborted = false;
  std::vector<double*> ptr;
  std::vector<int64_t> ldv;                 // per-rank column stride of the block in a halo
  std::vector<cudaEvent_t> ev, ev2;
  std::vector<int64_t> rb, re;
  explicit LocalGroup(int p) : P(p), ptr(p, nullptr), ldv(p, 0), ev(p), ev2(p), rb(p, 0), re(p, 0) {
    for (int r = 0; r < p; ++r) {
      cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ev2[r], cudaEventDisableTiming);
    }
  }
  ~LocalGroup() {
    for (int r = 0; r < P; ++r) {
      cudaEventDestroy(ev[r]);
      cudaEventDestroy(ev2[r]);
    }
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) throw CommError{"local group aborted by a failing rank"};
    const uint64_t gen = generation;
    if (++arrived == P) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen || aborted; });
      if (aborted) throw CommError{"local group aborted by a failing rank"};
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

struct LocalComm : Comm {
  LocalGroup* g;
  // one scratch per channel: collectives of different channels run on different streams
  double* scratch[kNumChan] = {};
  size_t scratch_n[kNumChan] = {};
  bool trace = false;
  uint64_t seq = 0;
  LocalComm(LocalGroup* grp, int r) : g(grp) {
    nranks = grp->P;
    rank = r;
    trace = std::getenv("SYLV_TRACE") != nullptr;
  }
  void tr(const char* what, size_t n) {
    if (trace) std::fprintf(stderr, "[rank %d] #%llu %s %zu\n", rank, (unsigned long long)seq, what, n);
  }
  ~LocalComm() override {
    for (double* p : scratch)
      if (p) cudaFree(p);
  }
  void ck(cudaError_t e, const char* w) {
    if (e != cudaSuccess) {
      g->abort();
      throw CommError{std::string(w) + ": " + cudaGetErrorString(e)};
    }
  }
  void abort() override { g->abort(); }
  void allreduce(double* buf, size_t n, cudaStream_t st, int chan) override {
    if (nranks == 1 || n == 0) return;
    ++seq;
    tr("allreduce", n);
    if (n > scratch_n[chan]) {
      ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");    // previous use on this stream done
      if (scratch[chan]) cudaFree(scratch[chan]);
      ck(cudaMalloc(&scratch[chan], n * sizeof(double)), "cudaMalloc (local allreduce)");
      scratch_n[chan] = n;
    }
    double* sc = scratch[chan];
    g->ptr[rank] = buf;
    ck(cudaEventRecord(g->ev[rank], st), "cudaEventRecord");
    g->barrier();
    PtrPack pk{};
    for (int r = 0; r < nranks; ++r) {
      pk.p[r] = g->ptr[r];
      if (r != rank) ck(cudaStreamWaitEvent(st, g->ev[r], 0), "cudaStreamWaitEvent");
    }
    k_sum_ranks<<<(int)std::min<size_t>(1024, (n + 255) / 256), 256, 0, st>>>(pk, nranks, n, sc);
    ck(cudaGetLastError(), "k_sum_ranks");
    ck(cudaEventRecord(g->ev2[rank], st), "cudaEventRecord");
    g->barrier();                                        // every rank has enqueued its sum
    for (int r = 0; r < nranks; ++r)
      if (r != rank) ck(cudaStreamWaitEvent(st, g->ev2[r], 0), "cudaStreamWaitEvent");
    ck(cudaMemcpyAsync(buf, sc, n * sizeof(double), cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
    g->barrier();                                        // nobody re-records ev/ev2 early
  }
  void reduce_scatter(const double* send, double* recv, size_t n, cudaStream_t st, int) override {
    if (n == 0) return;
    ++seq;
    tr("reduce_scatter", n);
    g->ptr[rank] = const_cast<double*>(send);
    ck(cudaEventRecord(g->ev[rank], st), "cudaEventRecord");
    g->barrier();
    PtrPack pk{};
    for (int r = 0; r < nranks; ++r) {
      pk.p[r] = g->ptr[r] + (size_t)rank * n;      // this rank's slice of every rank's send buffer
      if (r != rank) ck(cudaStreamWaitEvent(st, g->ev[r], 0), "cudaStreamWaitEvent");
    }
    k_sum_ranks<<<(int)std::min<size_t>(1024, (n + 255) / 256), 256, 0, st>>>(pk, nranks, n, recv);
    ck(cudaGetLastError(), "k_sum_ranks");
    ck(cudaEventRecord(g->ev2[rank], st), "cudaEventRecord");
    g->barrier();                                        // every rank has read the send buffers
    for (int r = 0; r < nranks; ++r)
      if (r != rank) ck(cudaStreamWaitEvent(st, g->ev2[r], 0), "cudaStreamWaitEvent");
    g->barrier();
  }
  void halo(double* data, int R, int64_t ld, int64_t gz, cudaStream_t st, int) override {
    if (nranks == 1 || gz == 0) return;
    ++seq;
    tr("halo", (size_t)gz);
    g->ptr[rank] = data;
    g->ldv[rank] = ld;
    ck(cudaEventRecord(g->ev[rank], st), "cudaEventRecord");
    g->barrier();
    const int lo = lower(), up = upper();
    for (int nb : {lo, up}) {
      if (nb < 0) continue;
      ck(cudaStreamWaitEvent(st, g->ev[nb], 0), "cudaStreamWaitEvent");
      const double* src = g->ptr[nb];
      const int64_t sld = g->ldv[nb];            // the neighbour's column stride
      for (int c = 0; c < R; ++c) {
        double* col = data + (int64_t)c * ld;
        const double* scol = src + (int64_t)c * sld;
        if (nb == lo)
          ck(cudaMemcpyAsync(col - gz, scol + rows(lo) - gz, gz * sizeof(double), cudaMemcpyDeviceToDevice, st), "halo");
        else
          ck(cudaMemcpyAsync(col + rows(rank), scol, gz * sizeof(double), cudaMemcpyDeviceToDevice, st), "halo");
      }
    }
    ck(cudaEventRecord(g->ev2[rank], st), "cudaEventRecord");
    g->barrier();
    for (int nb : {lo, up})
      if (nb >= 0) ck(cudaStreamWaitEvent(st, g->ev2[nb], 0), "cudaStreamWaitEvent");
    g->barrier();
  }
  void gather_ranges(int64_t b, int64_t e) override {
    ++seq;
    tr("gather", 0);
    g->rb[rank] = b;
    g->re[rank] = e;
    g->barrier();
    rb = g->rb;
    re = g->re;
    g->barrier();
  }
};

}  // namespace sylv
