// engine.cu — context, step schedule and the extern "C" boundary of include/sylv_sketch.h.
//
// One sylv_ctx owns two Sequence objects (U: operator A, seed_u; V: operator B^T,
// seed_v).  A block step runs the n-space passes (nspace.cuh) and the sketch-space QR
// update (sspace.cuh) for U then V on the context stream; small coefficient mirrors
// are copied to pinned host memory for the host projected solve (host_solve.cpp).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "../../include/sylv_sketch.h"
#include "common.cuh"
#include "host_solve.hpp"
#include "nspace.cuh"
#include "sspace.cuh"
#include "stencil25d.cuh"
#include "sketch_pull.cuh"
#include "comm.cuh"
#include "proj_gpu.cuh"
#include "full_arnoldi.cuh"
#include "sketched_gs.cuh"
#include "srdct.cuh"

using namespace sylv;

#define SYLV_VERSION "sylv_sketch 0.1 (sm_100a)"

namespace {

struct CudaError {
  cudaError_t e;
  const char* what;
};

#define CK(call)                                         \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) throw CudaError{_e, #call};   \
  } while (0)

struct Status {
  sylv_status s;
  std::string msg;
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <typename T>
T* dalloc(size_t count) {
  // Stream-ordered allocation from the device's default memory pool, kept reserved after
  // frees (release threshold = max): a new context reuses the previous one's ~10 GB
  // instead of going back to the driver (context init 0.1-0.3 s -> ~0.05 s).
  static bool pool_set = [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    return true;
  }();
  (void)pool_set;
  T* p = nullptr;
  if (count == 0) count = 1;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), 0));
  CK(cudaStreamSynchronize(0));   // usable from any stream of the context
  return p;
}

// Free a dalloc'ed buffer (callers have synchronised the streams that used it).
void dfree(void* p) {
  if (p) cudaFreeAsync(p, 0);
}

// ----------------------------------------------------------------------------------
// Launch dispatch over the template parameters R in {1,2,4,8}, K in {1,2,3,4}
// ----------------------------------------------------------------------------------
#define SYLV_DISPATCH_R(Rv, ...)                          \
  switch (Rv) {                                           \
    case 1: { constexpr int R_ = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int R_ = 2; __VA_ARGS__; } break; \
    case 4: { constexpr int R_ = 4; __VA_ARGS__; } break; \
    case 8: { constexpr int R_ = 8; __VA_ARGS__; } break; \
    default: break;                                       \
  }
#define SYLV_DISPATCH_R124(Rv, ...)                                     \
  switch (Rv) {                                                         \
    case 1: { constexpr int R_ = 1; __VA_ARGS__; } break;               \
    case 2: { constexpr int R_ = 2; __VA_ARGS__; } break;               \
    case 4: { constexpr int R_ = 4; __VA_ARGS__; } break;               \
    default: break;                                                     \
  }
// K = 5..10 only for R <= 2 (the generic row kernels; the TMA / DMMA paths stay at K <= 4)
#define SYLV_KCASE_SMALL_R(KK, ...) \
    case KK: { constexpr int K_ = KK; if constexpr (R_ <= 2) { __VA_ARGS__; } } break;
#define SYLV_KCASES(...)                                                \
    case 1: { constexpr int K_ = 1; __VA_ARGS__; } break;               \
    case 2: { constexpr int K_ = 2; __VA_ARGS__; } break;               \
    case 3: { constexpr int K_ = 3; __VA_ARGS__; } break;               \
    case 4: { constexpr int K_ = 4; __VA_ARGS__; } break;               \
    SYLV_KCASE_SMALL_R(5, __VA_ARGS__)                                  \
    SYLV_KCASE_SMALL_R(6, __VA_ARGS__)                                  \
    SYLV_KCASE_SMALL_R(7, __VA_ARGS__)                                  \
    SYLV_KCASE_SMALL_R(8, __VA_ARGS__)                                  \
    SYLV_KCASE_SMALL_R(9, __VA_ARGS__)                                  \
    SYLV_KCASE_SMALL_R(10, __VA_ARGS__)                                 \
    default: break;
#define SYLV_DISPATCH_R124_K(Rv, Kv, ...)                               \
  SYLV_DISPATCH_R124(Rv, switch (Kv) { SYLV_KCASES(__VA_ARGS__) })
#define SYLV_DISPATCH_RK(Rv, Kv, ...)                                   \
  SYLV_DISPATCH_R(Rv, switch (Kv) { SYLV_KCASES(__VA_ARGS__) })

struct TimedPair {
  cudaEvent_t a, b;
  int kind;  // 0 pass1, 1 pass2, 2 skqr (sketch included), 3 sketch alone
};

}  // namespace

struct Sequence {
  // 2.5-D TMA passes (3-D stencil, r = 8, even N): tensor maps of the ring slots
  CUtensorMap mapH[kMaxKTma + 1];   // halo boxes
  CUtensorMap mapW[kMaxKTma + 1];   // window boxes
  bool tma = false;
  St25 st25{};
  int which = 0;
  int R = 1, K = 1, dmax = 0;
  int64_t n = 0, s = 0, ldT = 0, ld = 0;   // n: local rows; ld: SoA column stride
  int64_t sq = 0;                         // rows of the sketch-space QR on this rank: s, or s / P
                                          // when the sketch space is sharded
  double* skfull = nullptr;               // sharded sketch space: the s x R partial sketch
  // CSR pass 1 with the band window of Z_d in shared memory (k_pass1_csr_win): tile rows T
  // (0 = not eligible: the window of T + 2 band rows does not fit), band, grid, smem bytes
  int64_t csrT = 0, band = 0;
  int csr_grid = 0;
  size_t csr_smem = 0;
  int64_t* sell_ptr = nullptr;            // SELL-32 copy of the operator (k_pass1_sell_win)
  int32_t* sell_ci = nullptr;
  int16_t* sell_off = nullptr;            // 16-bit band offsets (k_pass1_sell_ring)
  int ringT = 0, ringCap = 0;             // sliding-ring pass 1: tile rows, ring rows per column
  double* sell_cv = nullptr;
  int64_t gz = 0;                         // ghost rows before/after a column (N^2 3-D, N 2-D, 0 CSR)
  OpParams op{};
  SketchParams sp{};
  // device
  double* ring = nullptr;     // (K+1) blocks, SoA R x ld
  double* Cdev = nullptr;     // SoA R x ld block (allocation; data at Cdev + gz)
  double* Yt = nullptr;       // CSR / sketched GS: A Z_d (SoA)
  double* skz = nullptr;      // sketched GS (f3): (K+1) ring of S Z_j, s x R row-major each
  // SRDCT sketch (f4, srdct.cuh): signs (n), selected rows (s), FFT buffers and plan
  bool srdct = false;
  double* sr_sign = nullptr;
  int64_t* sr_rows = nullptr;
  double* sr_v = nullptr;                 // R x n (Makhoul-ordered, signed columns)
  cufftDoubleComplex* sr_V = nullptr;     // R x (n/2 + 1)
  cufftHandle sr_plan = 0;
  double* Zaos = nullptr;     // CSR, r even: row-interleaved copy of Z_d for the pass-1 gathers
  double* sk = nullptr;       // s x R (row-major)
  double* skpart = nullptr;   // nchunk x R x s sketch partials
  // pull sketch (sketch_pull.cuh): groups sorted by (bucket, L2 chunk, window base)
  uint32_t* pl_list = nullptr;   // zeta x ngroups local group indices
  uint32_t* pl_off = nullptr;    // zeta x wpb + 1 per-warp segment offsets into pl_list
  double* pl_strips = nullptr;   // zeta x wpb x R x kPullS per-warp strips
  uint32_t pl_nch = 0, pl_wpb = 0, pl_bpw = 1, pl_kmax = 1;
  double* w = nullptr;        // s x R
  double* w2 = nullptr;       // s x R
  double* Q = nullptr;        // s x ldT (col-major)
  double* Tdev = nullptr;     // ldT x ldT col-major
  double* Rall = nullptr;     // (dmax+2) R^2
  double* Kc = nullptr;       // (dmax+1) (1+K) R^2
  double* Hc = nullptr;       // (dmax+1) (K+1) R^2
  double* hn2 = nullptr;      // (dmax+1)
  int* flags = nullptr;       // (dmax+2)
  double* part1 = nullptr;    // G x K R^2
  double* part2 = nullptr;    // G x R^2   (main stream: pass-2 Gram)
  double* part_s = nullptr;   // G x R^2   (side stream: CholQR2 Grams)
  double* cpart = nullptr;    // RT x ldT x R
  double* csum = nullptr;     // ldT x R
  double* c2 = nullptr;       // ldT x R
  double* qcpart = nullptr;   // CC x s x R
  double* small = nullptr;    // scratch r x r matrices
  int64_t* rp = nullptr;      // owned CSR (device)
  int32_t* ci = nullptr;
  double* cv = nullptr;
  // host mirrors (pinned)
  double* Hh = nullptr;       // (dmax+1) (K+1) R^2
  double* Th = nullptr;       // ldT x ldT col-major
  double* Rh = nullptr;       // (dmax+2) R^2 (filled on demand)
  int* flags_h = nullptr;
  // per-step events (ring of K+2).  Sketch on the side stream (push sketch, small n): ev_c2 =
  // step j's block ready (main -> side), ev_sk = the sketch of step j done reading ring slot
  // j+1 (side -> main, before pass 2 of step j+K+1 rewrites it).  Sketch on the main stream
  // (pull sketch): ev_c2 = sketch of step j done (main -> side QR), ev_sk = QR of step j done
  // with w (side -> main, before the next sketch writes it).
  std::vector<cudaEvent_t> ev_c2, ev_sk;
  double beta[kMaxR * kMaxR];
  double ell[kMaxR * kMaxR];

  // data pointer (local row 0 of column 0) of ring slot j; block base = data - gz
  double* slot(int j) const { return ring + (int64_t)(j % (K + 1)) * ld * R + gz; }
  double* cdata() const { return Cdev + gz; }
};

// Opaque transport handle of the C ABI (comm.cuh)
struct sylv_comm {
  Comm* impl = nullptr;
};

struct sylv_ctx {
  std::string err;
  cudaStream_t st = nullptr;
  cudaStream_t rst = nullptr;       // stream of the residual computation (= st, or st_solve)
  cudaStream_t st_solve = nullptr;  // solve driver: projected solves overlapping the next steps
  Comm* comm = nullptr;         // non-null: row-sharded context; not owned
  int64_t n_global = 0, row_begin = 0, row_end = 0;
  double* red = nullptr;        // multi-rank: reduced partials (k r^2 + r^2 per sequence)
  int R = 1, K = 1, dmax = 0, zeta = 8, chunk = 0, cflags = 0;
  int method = SYLV_METHOD_SKETCHED;   // sylv_config.method
  int RTn = 1, tpcN = 1, CCn = 1;      // full method: n-space Q^T w row chunks / tiles per CTA, Q c chunks
  int64_t sq = 0;                      // sketch-space rows per rank (s, or s / P: sharded sketch space)
  int64_t n = 0, s = 0;
  double tol = 1e-6, rank_tol = 1e-12;
  int sm = 148;
  int G = 0;          // grid of the n-space passes
  int G25 = 0;        // grid of the 2.5-D TMA passes (0: not used)
  size_t smem25_1 = 0, smem25_2 = 0;
  int RT = 1;         // row tiles of Q^T w
  int64_t tileQ = 0;
  int CC = 1;         // column chunks of Q c
  bool qmma = true;   // DMMA sweeps of Q (R >= 4); SYLV_QMMA=0: the FMA kernels (A/B)
  int nchunk = 1;     // row chunks of the sketch kernel (grid nchunk x R)
  int64_t gpc = 32;   // 32-row groups per sketch chunk
  size_t sk_smem = 0; // dynamic shared memory of the sketch kernel
  bool sk_pull = false;  // large n: pull formulation of the sketch (sketch_pull.cuh)
  // streams: main[0] = st (U passes), main[1] = st2 (V passes); side[q] = sketch + sketch-space
  // QR of sequence q, which overlaps the next step's n-space passes (all = st in serial mode)
  cudaStream_t st2 = nullptr, st3 = nullptr, st4 = nullptr;
  cudaEvent_t fork = nullptr, join[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t phase[3] = {nullptr, nullptr, nullptr};   // pass/sketch phase barriers (enqueue_steps)
  Sequence seq[2];
  int d_done = 0;
  int d_dev = 0;                // last step enqueued on the device (>= d_done; ring slots reflect it)
  bool broken = false;          // breakdown (R11): the Krylov space is invariant
  int breakdown_d = -1;
  bool halted = false;          // terminal for stepping: breakdown or lost independence
  sylv_status halt_status = SYLV_OK;
  std::string halt_msg;
  // last projected solution (host vector, or the device solver's C when y_dev)
  int y_d = -1;
  bool y_dev = false;
  std::vector<double> Y;
  GpuSylv* gsolve = nullptr;    // device projected solver (created on first use)
  cublasHandle_t blas = nullptr;  // second pass X accumulation (created on first use)
  int gpu_fail_d = 1 << 30;     // smallest d where the device solve fell back to the host
  int sign_fail_d = 1 << 30;    // smallest d where the sign iteration failed (eig solve from there)
  int eig_solve = 1;            // certified eigendecomposition solve (SYLV_EIG=0: off, 2: first; tests)
  int64_t eig_solves = 0;
  // solve driver, schedule phase: a device solve that converged off the identity (approximate;
  // c1's ill-conditioned projections) may decide a check "fail" when its rho_rel exceeds this
  // (3 tol; measured error of such solves at c1: <= 8 %), else the host solves it (0: off)
  double approx_thr = 0.0;
  std::vector<std::pair<int, double>> hist;
  sylv_stats stats{};
  std::vector<TimedPair> timed;
  std::vector<TimedPair> free_events;
};

namespace {

void count(sylv_ctx* c, int k = 1) { c->stats.launches += k; }

TimedPair ev_get(sylv_ctx* c, int kind) {
  TimedPair p;
  if (!c->free_events.empty()) {
    p = c->free_events.back();
    c->free_events.pop_back();
  } else {
    CK(cudaEventCreate(&p.a));
    CK(cudaEventCreate(&p.b));
  }
  p.kind = kind;
  return p;
}

void ev_collect(sylv_ctx* c) {
  for (auto& p : c->timed) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.a, p.b));
    if (p.kind == 0) { c->stats.ms_pass1 += ms; c->stats.n_pass1++; }
    else if (p.kind == 1) { c->stats.ms_pass2 += ms; c->stats.n_pass2++; }
    else if (p.kind == 2) { c->stats.ms_skqr += ms; c->stats.n_skqr++; }
    else { c->stats.ms_sketch += ms; c->stats.n_sketch++; }
    c->free_events.push_back(p);
  }
  c->timed.clear();
}

OpParams make_op(const sylv_operator* A, bool transpose) {
  OpParams op{};
  op.kind = A->kind;
  op.n = A->n;
  if (A->kind == SYLV_OP_STENCIL2D || A->kind == SYLV_OP_STENCIL3D) {
    const int dim = (A->kind == SYLV_OP_STENCIL2D) ? 2 : 3;
    const int N = A->grid[0];
    op.N = N;
    op.divN = make_fastdiv((uint32_t)N);
    const double h = 1.0 / (N + 1);
    const double nu = A->nu;
    const double sg = transpose ? -1.0 : 1.0;  // B^T = stencil with -w (R16)
    op.cd = 2.0 * dim * nu / (h * h);
    op.cxm = -nu / (h * h) - sg * A->w[0] / (2 * h);
    op.cxp = -nu / (h * h) + sg * A->w[0] / (2 * h);
    op.cym = -nu / (h * h) - sg * A->w[1] / (2 * h);
    op.cyp = -nu / (h * h) + sg * A->w[1] / (2 * h);
    if (dim == 3) {
      op.czm = -nu / (h * h) - sg * A->w[2] / (2 * h);
      op.czp = -nu / (h * h) + sg * A->w[2] / (2 * h);
    }
  }
  return op;
}

// ---- CSR upload; B^T by a stable device sort of the nonzeros by column -------------------
__global__ void k_row_of(const int64_t* __restrict__ rp, int64_t n, int32_t* __restrict__ row_of) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) row_of[p] = (int32_t)i;
}
__global__ void k_iota32(int32_t* __restrict__ x, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (int32_t)i;
}
// B^T in CSR = B in CSC: nonzero k of the sorted order is (col key[k], row row_of[perm[k]])
__global__ void k_csr_transpose_fill(const int32_t* __restrict__ key, const int32_t* __restrict__ perm,
                                     const int32_t* __restrict__ row_of, const double* __restrict__ cv, int64_t nnz,
                                     int64_t n, int32_t* __restrict__ tci, double* __restrict__ tcv,
                                     int64_t* __restrict__ tp) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t pk = perm[k];
    tci[k] = row_of[pk];
    tcv[k] = cv[pk];
    // row pointers of B^T: every column c in (key[k-1], key[k]] starts at k
    for (int64_t c = (k == 0 ? 0 : (int64_t)key[k - 1] + 1); c <= key[k]; ++c) tp[c] = k;
    if (k == nnz - 1)
      for (int64_t c = (int64_t)key[k] + 1; c <= n; ++c) tp[c] = nnz;
  }
}

// CSR of A (or B^T when transpose): host or device input arrays, uploaded as they are; the
// transpose is a stable radix sort of the nonzeros by column on the device (rows stay
// ascending inside each column, so B^T's rows are sorted and the result is deterministic).
// max |col - row| over the nonzeros (the halo width of a row-sharded CSR operator)
__global__ void k_csr_band(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n,
                           int* __restrict__ band) {
  int m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) m = max(m, abs(ci[p] - (int)i));
  atomicMax(band, m);
}

// rows [b, e) of a CSR matrix with column indices made local (col - b; ghosts are negative
// or >= e - b): rp_l[i] = rp[b+i] - rp[b], ci_l = ci - b, cv_l = cv
__global__ void k_csr_slice(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ cv,
                            int64_t b, int64_t e, int64_t p0, int64_t nnz_l, int64_t* __restrict__ rp_l,
                            int32_t* __restrict__ ci_l, double* __restrict__ cv_l) {
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, ts = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t0; i <= e - b; i += ts) rp_l[i] = rp[b + i] - p0;
  for (int64_t p = t0; p < nnz_l; p += ts) {
    ci_l[p] = ci[p0 + p] - (int32_t)b;
    cv_l[p] = cv[p0 + p];
  }
}

void upload_csr(Sequence& q, const sylv_operator* A, bool transpose, cudaStream_t st) {
  const int64_t n = A->n, nnz = A->nnz;
  const bool dev = is_device_ptr(A->row_ptr);
  const cudaMemcpyKind kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  q.rp = dalloc<int64_t>(n + 1);
  q.ci = dalloc<int32_t>(nnz);
  q.cv = dalloc<double>(nnz);
  if (n >= (1ll << 31) || nnz >= (1ll << 31)) throw Status{SYLV_E_INVALID, "CSR n and nnz must be < 2^31"};
  if (!transpose) {
    CK(cudaMemcpyAsync(q.rp, A->row_ptr, (n + 1) * sizeof(int64_t), kind, st));
    CK(cudaMemcpyAsync(q.ci, A->col_idx, nnz * sizeof(int32_t), kind, st));
    CK(cudaMemcpyAsync(q.cv, A->val, nnz * sizeof(double), kind, st));
  } else {
    int64_t* rp = dalloc<int64_t>(n + 1);
    int32_t *key = dalloc<int32_t>(nnz), *key2 = dalloc<int32_t>(nnz);
    int32_t *perm = dalloc<int32_t>(nnz), *perm2 = dalloc<int32_t>(nnz), *row_of = dalloc<int32_t>(nnz);
    double* cv = dalloc<double>(nnz);
    CK(cudaMemcpyAsync(rp, A->row_ptr, (n + 1) * sizeof(int64_t), kind, st));
    CK(cudaMemcpyAsync(key, A->col_idx, nnz * sizeof(int32_t), kind, st));
    CK(cudaMemcpyAsync(cv, A->val, nnz * sizeof(double), kind, st));
    k_row_of<<<1024, 256, 0, st>>>(rp, n, row_of);
    k_iota32<<<1024, 256, 0, st>>>(perm, nnz);
    int end_bit = 1;
    while ((1ll << end_bit) < n) ++end_bit;
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, key2, perm, perm2, (int)nnz, 0, end_bit, st));
    void* tmp = dalloc<char>(tmp_bytes);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key2, perm, perm2, (int)nnz, 0, end_bit, st));
    k_csr_transpose_fill<<<1024, 256, 0, st>>>(key2, perm2, row_of, cv, nnz, n, q.ci, q.cv, q.rp);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    for (void* p : {(void*)rp, (void*)key, (void*)key2, (void*)perm, (void*)perm2, (void*)row_of, (void*)cv, tmp})
      dfree(p);
  }
  CK(cudaStreamSynchronize(st));
  q.op.rp = q.rp;
  q.op.ci = q.ci;
  q.op.cv = q.cv;
}

void free_seq(Sequence& q) {
  for (cudaEvent_t e : q.ev_c2) cudaEventDestroy(e);
  for (cudaEvent_t e : q.ev_sk) cudaEventDestroy(e);
  double* dp[] = {q.ring, q.Cdev, q.Yt, q.Zaos, q.sk, q.skpart, q.w, q.w2, q.Q, q.Tdev, q.Rall, q.Kc, q.Hc, q.hn2,
                  q.part1, q.part2, q.part_s, q.cpart, q.csum, q.c2, q.qcpart, q.small, q.cv, q.skz, q.sr_sign,
                  q.sr_v, q.skfull};
  if (q.sr_plan) cufftDestroy(q.sr_plan);
  dfree(q.sr_rows);
  dfree(q.sr_V);
  dfree(q.sell_ptr);
  dfree(q.sell_ci);
  dfree(q.sell_off);
  dfree(q.sell_cv);
  for (double* p : dp) dfree(p);
  dfree(q.flags);
  dfree(q.pl_list);
  dfree(q.pl_off);
  dfree(q.pl_strips);
  dfree(q.rp);
  dfree(q.ci);
  if (q.Hh) cudaFreeHost(q.Hh);
  delete[] q.Th;
  if (q.Rh) cudaFreeHost(q.Rh);
  if (q.flags_h) cudaFreeHost(q.flags_h);
  q = Sequence{};
}

// CholQR2 of the s x R block `in` (destroyed): q written to Q[:, col0:col0+R]
// (column-major), R-factor tau (positive diagonal) to `tau_out` (device, R x R).
// out[e] = sum of the nparts per-CTA partials (block_sum_parts order), one CTA
__global__ void __launch_bounds__(kSmallThreads) k_sum_partials(const double* __restrict__ partial, int nparts, int len, double* __restrict__ out) {
  block_sum_parts(partial, nparts, len, len, out);
}

// General form: `rows` x R row-major `in` (destroyed; q.w2 holds rows x R scratch) -> `out`
// column-major with column stride out_ld.
// gram_chan >= 0: the rows are this rank's shard of a sketch-space block (sharded sketch space),
// the Gram is summed over the ranks (partials -> one vector -> allreduce on that channel).
void cholqr2_into(sylv_ctx* c, Sequence& q, double* in, int64_t rows, double* out, int64_t out_ld,
                  double* tau_out, int flag_slot, cudaStream_t st, int gram_chan = -1) {
  const int R = c->R;
  const int gs = (int)std::max<int64_t>(1, std::min<int64_t>(c->G, (rows + 255) / 256));
  double* ta = q.small;            // R^2
  double* tai = q.small + 64;      // R^2
  double* tbi = q.small + 128;     // R^2
  double* gsum = q.small + 448;    // R^2: the rank-summed Gram (sharded)
  auto gram = [&](const double* x) -> std::pair<const double*, int> {
    SYLV_DISPATCH_R(R, { k_gram_rowmajor<R_><<<gs, kThreads, 0, st>>>(rows, x, q.part_s); });
    if (gram_chan < 0 || !c->comm) return {q.part_s, gs};
    k_sum_partials<<<1, kSmallThreads, 0, st>>>(q.part_s, gs, R * R, gsum);
    c->comm->allreduce(gsum, (size_t)R * R, st, gram_chan);
    count(c);
    return {gsum, 1};
  };
  auto g1 = gram(in);
  SYLV_DISPATCH_R(R, {
    k_chol_small<R_><<<1, kSmallThreads, 0, st>>>(g1.first, g1.second, ta, tai, nullptr, q.flags, flag_slot);
    k_rmul<R_><<<gs, kThreads, 0, st>>>(rows, in, tai, q.w2, 0);
  });
  auto g2 = gram(q.w2);
  SYLV_DISPATCH_R(R, {
    k_chol_small<R_><<<1, kSmallThreads, 0, st>>>(g2.first, g2.second, tau_out, tbi, ta, q.flags, flag_slot);
    k_rmul<R_><<<gs, kThreads, 0, st>>>(rows, q.w2, tbi, out, out_ld);
  });
  count(c, 6);
  CK(cudaGetLastError());
}

void cholqr2(sylv_ctx* c, Sequence& q, double* in, int64_t col0, double* tau_out, int flag_slot,
             cudaStream_t st) {
  const bool shard = q.sq != q.s;
  const int chan = q.which == 0 ? kChanUSide : kChanVSide;
  cholqr2_into(c, q, in, q.sq, q.Q + col0 * q.sq, q.sq, tau_out, flag_slot, st, shard ? chan : -1);
}

// ---- 2.5-D TMA passes ------------------------------------------------------------------
constexpr int kTY25 = 4;   // tile height (lines) = warps per CTA

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

// SoA block (R columns of an N^3 grid, column stride ld) as an (x, y, z, column) tensor.
bool encode_block_map(CUtensorMap* m, const double* base, int N, int depth, int64_t ld, int R, int bx, int by) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)depth, (cuuint64_t)R};
  cuuint64_t strides[3] = {(cuuint64_t)N * 8, (cuuint64_t)N * N * 8, (cuuint64_t)ld * 8};
  cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, 1, (cuuint32_t)R};
  cuuint32_t es[4] = {1, 1, 1, 1};
  static const CUtensorMapL2promotion prom = [] {   // SYLV_TMA_L2PROM=0|64|128|256 (tuning)
    const char* e = std::getenv("SYLV_TMA_L2PROM");
    const int v = e ? std::atoi(e) : 256;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
           : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, prom,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int R, int K>
size_t smem25_bytes() {
  using Gm = Geo25<kTY25, R>;
  constexpr int ns = stages25<R>();
  return (size_t)ns * (Gm::HCOL * R + (K - 1) * Gm::WCOL * R) * 8 + ns * 8;
}

template <int R, int K>
void set_smem25(sylv_ctx* c) {
  c->smem25_1 = c->smem25_2 = smem25_bytes<R, K>();
  CK(cudaFuncSetAttribute(k_st3d<kTY25, R, K, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem25_1));
  CK(cudaFuncSetAttribute(k_st3d<kTY25, R, K, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem25_2));
  CK(cudaFuncSetAttribute(k_st3d<kTY25, R, K, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem25_2));
}

// Set up the TMA path for sequence q if eligible: 3-D stencil, r = 4 or 8, even N.
void setup_tma(sylv_ctx* c, Sequence& q) {
  q.tma = false;
  if ((c->cflags & 4) || q.op.kind != kStencil3D || (c->R != 8 && c->R != 4) || (q.op.N & 1) || q.op.N < 2 ||
      c->K > kMaxKTma)
    return;
  const int N = q.op.N;
  const int nz = (int)(q.n / ((int64_t)N * N));
  for (int j = 0; j <= c->K; ++j) {
    const double* base = q.ring + (int64_t)j * q.ld * c->R;     // ghost plane 0 of slot j
    if (!encode_block_map(&q.mapH[j], base, N, nz + 2, q.ld, c->R, Geo25<kTY25>::HX, Geo25<kTY25>::HY)) return;
    if (!encode_block_map(&q.mapW[j], base, N, nz + 2, q.ld, c->R, Geo25<kTY25>::WX, kTY25)) return;
  }
  St25& p = q.st25;
  p.N = N;
  p.nz = nz;
  p.ld = q.ld;
  p.tiles_x = (N + kTx - 1) / kTx;
  p.tiles_y = (N + kTY25 - 1) / kTY25;
  const int64_t tiles = (int64_t)p.tiles_x * p.tiles_y;
  // resident CTAs: r = 4 stages are half the size (4 stages of 11.6 KB; registers allow 4 CTAs)
  int gmul = c->R == 4 ? 4 : 2;
  if (const char* e = std::getenv("SYLV_G25MUL")) gmul = std::max(1, std::atoi(e));   // tuning
  const int grid = gmul * c->sm;
  int nseg = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(1, nz / 16), (8 * grid + tiles - 1) / tiles));
  if (const char* e = std::getenv("SYLV_NSEG")) nseg = std::max(1, std::min(nz, std::atoi(e)));   // tuning
  p.zseg = (nz + nseg - 1) / nseg;
  p.nseg = (nz + p.zseg - 1) / p.zseg;
  p.items = tiles * p.nseg;
  p.cd = q.op.cd;
  p.cxm = q.op.cxm; p.cxp = q.op.cxp;
  p.cym = q.op.cym; p.cyp = q.op.cyp;
  p.czm = q.op.czm; p.czp = q.op.czp;
  p.dbg = getenv("SYLV_DBG") ? atoi(getenv("SYLV_DBG")) : 0;
  c->G25 = (int)std::min<int64_t>(p.items, grid);
  if (c->R == 8) {
    switch (c->K) {
      case 1: set_smem25<8, 1>(c); break;
      case 2: set_smem25<8, 2>(c); break;
      case 3: set_smem25<8, 3>(c); break;
      case 4: set_smem25<8, 4>(c); break;
    }
  } else {
    switch (c->K) {
      case 1: set_smem25<4, 1>(c); break;
      case 2: set_smem25<4, 2>(c); break;
      case 3: set_smem25<4, 3>(c); break;
      case 4: set_smem25<4, 4>(c); break;
    }
  }
  q.tma = true;
}

Tma25 tma_args(const Sequence& q, int j, int nwin) {
  Tma25 tm;
  const int ns = q.K + 1;
  tm.zd = q.mapH[j % ns];
  for (int i = 0; i < nwin - 1; ++i) tm.win[i] = q.mapW[(j - nwin + 1 + i) % ns];
  return tm;
}

// Partials written by the pass kernels of sequence q (the coefficient kernels' nparts)
int pass_parts(const sylv_ctx* c, const Sequence& q) { return q.tma ? c->G25 : c->G; }
// partials written by pass 1 (the windowed CSR pass 1 runs its own grid)
int pass1_parts(const sylv_ctx* c, const Sequence& q) { return q.csrT > 0 ? q.csr_grid : pass_parts(c, q); }


// Multi-rank: reduce this rank's per-CTA partials to one vector of `len` values, sum it
// over the ranks (bit-identical on every rank), and return it as a single "partial" for
// the coefficient kernels (nparts = 1).  Single rank: the partials are used directly.
const double* reduce_partials(sylv_ctx* c, const double* partial, int nparts, int len, double* out,
                              cudaStream_t st, int chan, int* nparts_out) {
  if (!c->comm) {
    *nparts_out = nparts;
    return partial;
  }
  k_sum_partials<<<1, kSmallThreads, 0, st>>>(partial, nparts, len, out);
  count(c);
  CK(cudaGetLastError());
  c->comm->allreduce(out, (size_t)len, st, chan);
  *nparts_out = 1;
  return out;
}

// n-space pass launchers (2.5-D TMA kernels when eligible; else R <= 4: thread-per-row FMA
// kernels, R = 8: DMMA warp tiles).  j = step (1-based): Z_j is the newest window block.
void launch_pass1(sylv_ctx* c, Sequence& q, const Win& win, int nwin, int j, cudaStream_t st) {
  const int R = c->R, K = c->K;
  if (q.tma) {
    const Tma25 tm = tma_args(q, j, nwin);
    const int nw1 = nwin, slot0 = -1;
#define SYLV_ST3D_P1(RR, KK) k_st3d<kTY25, RR, KK, 1, false><<<c->G25, 32 * kTY25 * kWpl25, c->smem25_1, st>>>(tm, q.st25, nw1, nullptr, nullptr, q.part1, slot0)
    if (R == 8) {
      switch (K) {
        case 1: SYLV_ST3D_P1(8, 1); break;
        case 2: SYLV_ST3D_P1(8, 2); break;
        case 3: SYLV_ST3D_P1(8, 3); break;
        case 4: SYLV_ST3D_P1(8, 4); break;
      }
    } else {
      switch (K) {
        case 1: SYLV_ST3D_P1(4, 1); break;
        case 2: SYLV_ST3D_P1(4, 2); break;
        case 3: SYLV_ST3D_P1(4, 3); break;
        case 4: SYLV_ST3D_P1(4, 4); break;
      }
    }
#undef SYLV_ST3D_P1
  } else if (q.op.kind == kCSR && q.csrT > 0) {
    // band window of Z_d staged in shared memory (no AoS copy, gathers from shared memory)
    if (q.sell_off) {
      SYLV_DISPATCH_R124_K(R, K, {
        k_pass1_sell_ring<R_, K_><<<q.csr_grid, kSellThreads, q.csr_smem, st>>>(
            q.op, win, nwin, q.ld, q.gz, q.band, q.ringT, q.ringCap, q.sell_ptr, q.sell_off, q.sell_cv, q.Yt, q.part1);
      });
    } else if (q.sell_cv) {
      SYLV_DISPATCH_R124_K(R, K, {
        k_pass1_sell_win<R_, K_><<<q.csr_grid, kSellThreads, q.csr_smem, st>>>(
            q.op, win, nwin, q.ld, q.gz, q.band, q.csrT, q.sell_ptr, q.sell_ci, q.sell_cv, q.Yt, q.part1);
      });
    } else {
      SYLV_DISPATCH_R124_K(R, K, {
        k_pass1_csr_win<R_, K_><<<q.csr_grid, kCsrWinThreads, q.csr_smem, st>>>(q.op, win, nwin, q.ld, q.gz, q.band,
                                                                                q.csrT, q.Yt, q.part1);
      });
    }
    count(c);
  } else if (q.op.kind == kCSR && R <= 4) {
    if (R % 2 == 0) {   // AoS copy of Z_d for the gathers
      // rows -gz .. n+gz-1 (ghost rows of a sharded CSR operator included)
      SYLV_DISPATCH_R124(R, { k_soa_to_aos<R_><<<4 * c->sm, kThreads, 0, st>>>(c->n + 2 * q.gz, win.p[nwin - 1] - q.gz, q.ld, q.Zaos); });
      count(c);
    }
    SYLV_DISPATCH_R124_K(R, K, { k_pass1_csr<R_, K_><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, q.Zaos ? q.Zaos + q.gz * R : nullptr, q.Yt, q.part1); });
  } else if (R == 8) {
    switch (K) {
      case 1: k_pass1_r8<1><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, q.Yt, q.part1); break;
      case 2: k_pass1_r8<2><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, q.Yt, q.part1); break;
      case 3: k_pass1_r8<3><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, q.Yt, q.part1); break;
      case 4: k_pass1_r8<4><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, q.Yt, q.part1); break;
    }
  } else {
    SYLV_DISPATCH_R124_K(R, K, { k_pass1_rows<R_, K_><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, q.Yt, q.part1); });
  }
  count(c);
}

template <bool GRAM>
void launch_pass2(sylv_ctx* c, Sequence& q, const Win& win, int nwin, int j, const double* Yt, const double* coef,
                  double* out, cudaStream_t st, bool allow_tma = true) {
  const int R = c->R, K = c->K;
  if (q.tma && allow_tma) {
    const Tma25 tm = tma_args(q, j, nwin);
#define SYLV_ST3D_P2(RR, KK) k_st3d<kTY25, RR, KK, 2, GRAM><<<c->G25, 32 * kTY25 * kWpl25, c->smem25_2, st>>>(tm, q.st25, nwin, coef, out, q.part2)
    if (R == 8) {
      switch (K) {
        case 1: SYLV_ST3D_P2(8, 1); break;
        case 2: SYLV_ST3D_P2(8, 2); break;
        case 3: SYLV_ST3D_P2(8, 3); break;
        case 4: SYLV_ST3D_P2(8, 4); break;
      }
    } else {
      switch (K) {
        case 1: SYLV_ST3D_P2(4, 1); break;
        case 2: SYLV_ST3D_P2(4, 2); break;
        case 3: SYLV_ST3D_P2(4, 3); break;
        case 4: SYLV_ST3D_P2(4, 4); break;
      }
    }
#undef SYLV_ST3D_P2
  } else if (R == 8) {
    switch (K) {
      case 1: k_pass2_r8<1, GRAM><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, Yt, coef, out, q.part2); break;
      case 2: k_pass2_r8<2, GRAM><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, Yt, coef, out, q.part2); break;
      case 3: k_pass2_r8<3, GRAM><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, Yt, coef, out, q.part2); break;
      case 4: k_pass2_r8<4, GRAM><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, Yt, coef, out, q.part2); break;
    }
  } else {
    SYLV_DISPATCH_R124_K(R, K, {
      k_pass2_rows<R_, K_, GRAM><<<c->G, kThreads, 0, st>>>(q.op, win, nwin, q.ld, Yt, coef, out, q.part2);
    });
  }
  count(c);
}

// S X for an SoA block -> w (s x R row-major) = (S X) M  (M = nullptr: identity)
void launch_sketch(sylv_ctx* c, Sequence& q, const double* X, int R, const double* M, double* w, cudaStream_t st) {
  const int red_grid = (int)std::min<int64_t>(4 * c->sm, (q.s + 255) / 256);
  if (q.srdct) {                                   // S = sqrt(n/s) D N E (srdct.cuh)
    if (R != q.R) throw Status{SYLV_E_INVALID, "SRDCT: the sketched block must have r columns"};
    SYLV_DISPATCH_R(R, {
      k_srdct_pre<R_><<<(int)std::min<int64_t>(8 * c->sm, (c->n + 255) / 256), 256, 0, st>>>(c->n, X, q.ld, q.sr_sign,
                                                                                             q.sr_v);
    });
    if (cufftSetStream(q.sr_plan, st) != CUFFT_SUCCESS || cufftExecD2Z(q.sr_plan, q.sr_v, q.sr_V) != CUFFT_SUCCESS)
      throw Status{SYLV_E_CUDA, "cufftExecD2Z (SRDCT)"};
    SYLV_DISPATCH_R(R, {
      k_srdct_post<R_><<<(int)std::min<int64_t>(4 * c->sm, (q.s + 255) / 256), 256, 0, st>>>(c->n, q.s, q.sr_V,
                                                                                             q.sr_rows, M, w);
    });
    count(c, 2);
    return;
  }
  if (q.pl_list) {
    const int nw = (int)(q.sp.zeta * q.pl_wpb);
    SYLV_DISPATCH_R(R, {
      k_sketch_pull<R_><<<(nw + kPullWarps - 1) / kPullWarps, kPullWarps * 32, 0, st>>>(
          c->n, X, q.ld, q.sp, q.pl_list, q.pl_off, q.pl_wpb, q.pl_bpw, q.pl_strips);
      if (q.pl_kmax > 8) {   // many strips per slot (one or two bases per warp): warp per slot, lane = strip
        k_sketch_pull_fold_wide<R_><<<(int)std::min<int64_t>(16 * c->sm, (q.s + 3) / 4), 128, 0, st>>>(
            q.pl_strips, q.sp, q.pl_wpb, q.pl_bpw, q.pl_kmax, M, w);
      } else {
        k_sketch_pull_fold_apply<R_><<<(int)std::min<int64_t>(8 * c->sm, (q.s + 256 / R_ - 1) / (256 / R_)), 256, 0, st>>>(
            q.pl_strips, q.sp, q.pl_wpb, q.pl_bpw, q.pl_kmax, M, w);
      }
    });
    count(c, 2);
    return;
  }
  const dim3 g(c->nchunk, R);
  const int nchunk = c->nchunk;
  SYLV_DISPATCH_R(R, {
    k_sketch_cols<R_><<<g, kSkWarps * 32, c->sk_smem, st>>>(c->n, X, q.ld, q.sp, c->gpc, q.skpart);
    k_sketch_reduce<R_><<<red_grid, 256, 0, st>>>(q.skpart, nchunk, q.s, M, w);
  });
  count(c, 2);
}

// Pull-sketch lists (sketch_pull.cuh): the hash depends only on (seed, global group, bucket),
// so the groups of each bucket are sorted once by (L2 chunk, window base) — stable, so every
// later summation order is fixed.
void build_pull_lists(sylv_ctx* c, Sequence& q, cudaStream_t st) {
  const int64_t ngroups = (c->n + 31) / 32;
  int64_t gpch = std::max<int64_t>(1, (int64_t)(32 << 20) / (256 * q.R));   // ~32 MB of W per chunk
  if (const char* e = std::getenv("SYLV_PULL_CHUNK")) gpch = std::max<int64_t>(1, std::atoll(e));   // tests
  const int64_t nch = (ngroups + gpch - 1) / gpch;
  // warps per bucket: exactly the resident warps of the GPU (the warps sweep W's L2 chunks
  // together, a second wave would re-read W from HBM, and every SM gets the same load)
  int occ = 1;
  SYLV_DISPATCH_R(q.R, { CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sketch_pull<R_>, kPullWarps * 32, 0)); });
  const int64_t resident = (int64_t)std::max(1, occ) * c->sm * kPullWarps;
  const int64_t b = q.sp.b;
  int64_t wpb = std::max<int64_t>((b + kPullBpwMax - 1) / kPullBpwMax, std::min<int64_t>(b, resident / q.sp.zeta));
  if (const char* e = std::getenv("SYLV_PULL_BPW")) {   // tests: ranges of at most this many bases
    const int64_t bw = std::max(1, std::min(kPullBpwMax, std::atoi(e)));
    wpb = (b + bw - 1) / bw;
  }
  const int64_t bpw = (b + wpb - 1) / wpb;   // longest range
  const int64_t nkeys = (int64_t)q.sp.zeta * wpb * nch * bpw;
  const int64_t total = ngroups * q.sp.zeta;
  if (nkeys >= (1ll << 32) || total >= (1ll << 31) || c->n >= (1ll << 32) - 64) return;   // stays on k_sketch_cols
  q.pl_nch = (uint32_t)nch;
  q.pl_bpw = (uint32_t)bpw;
  q.pl_wpb = (uint32_t)wpb;
  // fold: warps whose strips can cover a slot (shortest range floor(b / wpb) >= 1 bases)
  q.pl_kmax = (uint32_t)std::min<int64_t>(wpb, (bpw + 31) / std::max<int64_t>(1, b / wpb) + 2);
  const int64_t nw = (int64_t)q.sp.zeta * wpb;
  uint32_t *keys = dalloc<uint32_t>(total), *keys2 = dalloc<uint32_t>(total), *vals = dalloc<uint32_t>(total);
  uint32_t* counts = dalloc<uint32_t>(nw + 1);
  q.pl_list = dalloc<uint32_t>(total);
  q.pl_off = dalloc<uint32_t>(nw + 1);
  q.pl_strips = dalloc<double>((size_t)nw * q.R * kPullS);
  CK(cudaMemsetAsync(counts, 0, (nw + 1) * sizeof(uint32_t), st));
  k_pull_keys<<<4 * c->sm, 256, 0, st>>>(ngroups, q.sp, gpch, (uint32_t)nch, q.pl_bpw, q.pl_wpb, keys, vals, counts);
  count(c);
  int end_bit = 1;
  while (end_bit < 32 && (1ll << end_bit) < nkeys) ++end_bit;
  size_t sort_bytes = 0, scan_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys, keys2, vals, q.pl_list, (int)total, 0, end_bit, st));
  CK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts, q.pl_off, (int)(nw + 1), st));
  void* tmp = dalloc<char>(std::max(sort_bytes, scan_bytes));
  CK(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, keys, keys2, vals, q.pl_list, (int)total, 0, end_bit, st));
  CK(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, counts, q.pl_off, (int)(nw + 1), st));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  for (void* p : {(void*)keys, (void*)keys2, (void*)vals, (void*)counts, tmp}) dfree(p);
}

// SYLV_TRACE_INIT=1: wall time of the init phases on stderr (development aid)
struct InitTrace {
  bool on = std::getenv("SYLV_TRACE_INIT") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, cudaStream_t st) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[init] %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Row-sharded CSR: keep rows [row_begin, row_end) of the global matrix
// uploaded by upload_csr, with local column indices.  The halo width is the matrix band
// max |col - row| (computed from the global matrix, hence the same on every rank); columns of
// the local rows reach at most band rows into the neighbour ranks, whose boundary rows the
// halo exchange copies into the ghost rows (gz = band) before and after each block column.
void shard_csr(sylv_ctx* c, Sequence& q) {
  cudaStream_t st = c->st;
  const int64_t ng = c->n_global, b = c->row_begin, e = c->row_end;
  int* band_d = dalloc<int>(1);
  CK(cudaMemsetAsync(band_d, 0, sizeof(int), st));
  k_csr_band<<<1024, 256, 0, st>>>(q.rp, q.ci, ng, band_d);
  count(c);
  int band = 0;
  int64_t pb[2];
  CK(cudaMemcpyAsync(&band, band_d, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&pb[0], q.rp + b, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&pb[1], q.rp + e, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  dfree(band_d);
  for (int r = 0; r < c->comm->nranks; ++r)
    if (c->comm->re[r] - c->comm->rb[r] < band)
      throw Status{SYLV_E_INVALID, "CSR sharding: every rank needs at least band = max|col-row| rows"};
  const int64_t nnz_l = pb[1] - pb[0];
  int64_t* rp_l = dalloc<int64_t>(e - b + 1);
  int32_t* ci_l = dalloc<int32_t>(nnz_l);
  double* cv_l = dalloc<double>(nnz_l);
  k_csr_slice<<<1024, 256, 0, st>>>(q.rp, q.ci, q.cv, b, e, pb[0], nnz_l, rp_l, ci_l, cv_l);
  count(c);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  dfree(q.rp);
  dfree(q.ci);
  dfree(q.cv);
  q.rp = rp_l;
  q.ci = ci_l;
  q.cv = cv_l;
  q.op.rp = q.rp;
  q.op.ci = q.ci;
  q.op.cv = q.cv;
  q.gz = band;
}

// Windowed CSR pass 1 (nspace.cuh k_pass1_csr_win) when the band window of a row tile fits in
// shared memory: tiles of T rows (multiple of 512), one CTA of 512 threads per SM.
void setup_csr_window(sylv_ctx* c, Sequence& q) {
  q.csrT = 0;
  const char* e = std::getenv("SYLV_CSR_WINDOW");      // "0": the global-gather kernel (A/B)
  if (e && std::strcmp(e, "0") == 0) return;
  int64_t band = q.gz;                                  // sharded: the halo width is the band
  if (!c->comm) {
    int* band_d = dalloc<int>(1);
    CK(cudaMemsetAsync(band_d, 0, sizeof(int), c->st));
    k_csr_band<<<1024, 256, 0, c->st>>>(q.rp, q.ci, c->n, band_d);
    count(c);
    int b = 0;
    CK(cudaMemcpyAsync(&b, band_d, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    dfree(band_d);
    band = b;
  }
  q.band = band;
  const int R = c->R, K = c->K;
  int dev = 0, max_optin = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int64_t rows_fit =
      ((int64_t)max_optin - (int64_t)std::max(kCsrWinWarps, kSellWarps) * K * R * R * 8 - 256) / (8 * R);
  int64_t T = (rows_fit - 2 * band - 2) / 512 * 512;
  if (T < 1024) return;
  T = std::min<int64_t>(T, (c->n + 511) / 512 * 512);
  {
    // balance the persistent CTAs: the same number of tiles per CTA (c4: 683 tiles of 6144 rows
    // on 148 CTAs = 5 or 4 per CTA -> 737 tiles of 5696 rows, 5 per CTA), tiles of 32-row slices
    const int64_t per_cta = (((c->n + T - 1) / T) + c->sm - 1) / c->sm;
    const int64_t Tb = ((c->n + per_cta * c->sm - 1) / (per_cta * c->sm) + 31) / 32 * 32;
    if (Tb >= 1024 && Tb <= T) T = Tb;
  }
  q.csrT = T;
  q.csr_smem = (size_t)R * (T + 2 * band + 2) * 8 + 16;
  q.csr_grid = (int)std::min<int64_t>(c->sm, (c->n + T - 1) / T);
  SYLV_DISPATCH_R124_K(R, K, {
    CK(cudaFuncSetAttribute(k_pass1_csr_win<R_, K_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)q.csr_smem));
    CK(cudaFuncSetAttribute(k_pass1_sell_win<R_, K_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)q.csr_smem));
  });
  // SELL-32 copy (SYLV_SELL=0: the CSR-stream kernel k_pass1_csr_win)
  const char* se = std::getenv("SYLV_SELL");
  if (se && std::strcmp(se, "0") == 0) return;
  const int64_t ns = (c->n + 31) / 32;
  int64_t* w = dalloc<int64_t>(ns + 1);
  q.sell_ptr = dalloc<int64_t>(ns + 1);
  CK(cudaMemsetAsync(w + ns, 0, sizeof(int64_t), c->st));
  k_sell_widths<<<(int)std::min<int64_t>(4096, (ns + 255) / 256), 256, 0, c->st>>>(q.rp, c->n, w);
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, w, q.sell_ptr, (int)(ns + 1), c->st));
  void* tmp = dalloc<char>(tb);
  CK(cub::DeviceScan::ExclusiveSum(tmp, tb, w, q.sell_ptr, (int)(ns + 1), c->st));
  int64_t total = 0;
  CK(cudaMemcpyAsync(&total, q.sell_ptr + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  dfree(w);
  dfree(tmp);
  q.sell_cv = dalloc<double>(std::max<int64_t>(1, total));
  // sliding ring (k_pass1_sell_ring) when two tiles of >= 1024 rows and the band fit in shared
  // memory and the band offsets fit in 16 bits; SYLV_SELL_RING=0: the static-window kernel (A/B)
  const char* re = std::getenv("SYLV_SELL_RING");
  const int64_t cap = rows_fit & ~(int64_t)1;
  const int64_t Tr = (cap - 2 * band - 2) / 2 / 1024 * 1024;
  const int fill_grid = (int)std::min<int64_t>(4096, (ns * 32 + 255) / 256);
  if (!(re && std::strcmp(re, "0") == 0) && Tr >= 1024 && band <= 32767) {
    q.ringT = (int)Tr;
    q.ringCap = (int)cap;
    q.csr_smem = (size_t)R * cap * 8 + 32;
    q.csr_grid = (int)std::min<int64_t>(c->sm, (ns + 31) / 32);
    SYLV_DISPATCH_R124_K(R, K, {
      CK(cudaFuncSetAttribute(k_pass1_sell_ring<R_, K_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)q.csr_smem));
    });
    q.sell_off = dalloc<int16_t>(std::max<int64_t>(1, total));
    k_sell_fill<int16_t><<<fill_grid, 256, 0, c->st>>>(q.rp, q.ci, q.cv, c->n, q.sell_ptr, q.sell_off, q.sell_cv);
  } else {
    q.sell_ci = dalloc<int32_t>(std::max<int64_t>(1, total));
    k_sell_fill<int32_t><<<fill_grid, 256, 0, c->st>>>(q.rp, q.ci, q.cv, c->n, q.sell_ptr, q.sell_ci, q.sell_cv);
  }
  count(c, 2);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->st));
}

void qtw_split(const sylv_ctx* c, int64_t rows, int m, bool mma, int R, int64_t* chunk, int* nrt);

void init_sequence(sylv_ctx* c, Sequence& q, int which, const sylv_operator* A, bool transpose,
                   const double* C, uint64_t seed, const int8_t* sr_sign, const int64_t* sr_rows) {
  InitTrace tr;
  q.which = which;
  q.R = c->R;
  q.K = c->K;
  q.dmax = c->dmax;
  q.n = c->n;
  q.s = c->s;
  q.sq = c->sq;
  q.op = make_op(A, transpose);
  q.op.n = c->n;   // this rank's rows
  q.gz = (A->kind == SYLV_OP_STENCIL3D) ? (int64_t)A->grid[0] * A->grid[0]
         : (A->kind == SYLV_OP_STENCIL2D) ? (int64_t)A->grid[0] : 0;
  if (A->kind == SYLV_OP_CSR) {
    upload_csr(q, A, transpose && !A->is_transposed, c->st);   // the global matrix (A, or B^T); sets q.op's arrays
    if (c->comm) shard_csr(c, q);                // this rank's rows; q.gz = band
  }
  q.ld = (c->n + 2 * q.gz + 63) / 64 * 64;
  if (A->kind == SYLV_OP_CSR && c->method != SYLV_METHOD_FULL) setup_csr_window(c, q);
  q.ldT = (int64_t)(c->dmax + 1) * c->R;
  q.sp.seed = (uint32_t)(seed ^ (seed >> 32));
  q.sp.zeta = (uint32_t)c->zeta;
  q.sp.b = (uint32_t)(c->s / c->zeta);
  q.sp.scale = 1.0 / std::sqrt((double)c->zeta);
  q.sp.m0 = (uint32_t)(c->row_begin >> 5);   // global group index of local row 0
  const int R = c->R, K = c->K;
  const int64_t blk = q.ld * R, sR = c->s * R, ldT = q.ldT;
  tr.mark("setup", c->st);
  const bool sgs = c->method == SYLV_METHOD_SKETCHED_GS;
  const bool sketched = c->method == SYLV_METHOD_SKETCHED || sgs;
  const bool full = c->method == SYLV_METHOD_FULL;
  // (+64: the windowed CSR pass 1 may read one element past the last column, see k_pass1_csr_win)
  q.ring = dalloc<double>((size_t)(K + 1) * blk + 64);   // full method: the retained basis (d_max + 1 slots)
  q.Cdev = dalloc<double>(blk);
  if (A->kind == SYLV_OP_CSR || sgs) q.Yt = dalloc<double>(blk);
  if (sgs) q.skz = dalloc<double>((size_t)(K + 1) * sR);
  if (A->kind == SYLV_OP_CSR && R % 2 == 0) q.Zaos = dalloc<double>((size_t)(c->n + 2 * q.gz) * R);
  if (sketched) {
    q.sk = dalloc<double>(sR);
    q.Q = dalloc<double>((size_t)q.sq * ldT);            // this rank's rows of Q (sharded: s / P)
    if (q.sq != q.s) q.skfull = dalloc<double>(sR);
    if (sr_sign) {
      // SRDCT (f4): signs -> doubles, rows (checked), cuFFT D2Z plan batched over the R columns
      q.srdct = true;
      std::vector<int8_t> sg((size_t)c->n);
      std::vector<int64_t> rw((size_t)c->s);
      CK(cudaMemcpy(sg.data(), sr_sign, (size_t)c->n, is_device_ptr(sr_sign) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
      CK(cudaMemcpy(rw.data(), sr_rows, (size_t)c->s * sizeof(int64_t),
                    is_device_ptr(sr_rows) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
      std::vector<double> sd((size_t)c->n);
      for (int64_t i = 0; i < c->n; ++i) {
        if (sg[i] != 1 && sg[i] != -1) throw Status{SYLV_E_INVALID, "SRDCT signs must be +1 or -1"};
        sd[i] = (double)sg[i];
      }
      for (int64_t v : rw)
        if (v < 0 || v >= c->n) throw Status{SYLV_E_INVALID, "SRDCT rows must lie in [0, n)"};
      q.sr_sign = dalloc<double>(c->n);
      q.sr_rows = reinterpret_cast<int64_t*>(dalloc<double>(c->s));
      q.sr_v = dalloc<double>((size_t)c->n * R);
      q.sr_V = reinterpret_cast<cufftDoubleComplex*>(dalloc<double>((size_t)2 * (c->n / 2 + 1) * R));
      CK(cudaMemcpy(q.sr_sign, sd.data(), (size_t)c->n * sizeof(double), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(q.sr_rows, rw.data(), (size_t)c->s * sizeof(int64_t), cudaMemcpyHostToDevice));
      int nn = (int)c->n;
      if (cufftPlanMany(&q.sr_plan, 1, &nn, nullptr, 1, nn, nullptr, 1, nn / 2 + 1, CUFFT_D2Z, R) != CUFFT_SUCCESS)
        throw Status{SYLV_E_CUDA, "cufftPlanMany (SRDCT)"};
    } else {
      q.skpart = dalloc<double>((size_t)c->nchunk * sR);
      if (c->sk_pull && q.sp.b >= 64) build_pull_lists(c, q, c->st);
    }
  }
  // w, w2: the s x R sketched block (sketched) / the n x R applied block (full method)
  const int64_t wrows = full ? c->n : (sketched ? c->s : 0);   // (sharded sketch space: only sq rows used)
  if (wrows) {
    q.w = dalloc<double>((size_t)wrows * R);
    q.w2 = dalloc<double>((size_t)wrows * R);
  }
  q.Tdev = dalloc<double>((size_t)ldT * ldT);
  q.Rall = dalloc<double>((size_t)(c->dmax + 2) * R * R);
  q.Kc = dalloc<double>((size_t)(c->dmax + 1) * (1 + K) * R * R);
  q.Hc = dalloc<double>((size_t)(c->dmax + 1) * (K + 1) * R * R);
  q.hn2 = dalloc<double>(c->dmax + 1);
  q.flags = dalloc<int>(c->dmax + 2);
  const int gmax = std::max(c->G, 3 * c->sm);
  q.part1 = dalloc<double>((size_t)gmax * K * R * R);
  q.part2 = dalloc<double>((size_t)gmax * R * R);
  q.part_s = dalloc<double>((size_t)c->G * R * R);
  q.ev_c2.resize(K + 2);
  q.ev_sk.resize(K + 2);
  for (int i = 0; i < K + 2; ++i) {
    CK(cudaEventCreateWithFlags(&q.ev_c2[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&q.ev_sk[i], cudaEventDisableTiming));
  }
  if (sketched || full) {
    size_t cpart_len = (size_t)(full ? c->RTn : c->RT) * ldT * R;
    if (sketched) {   // Q^T w partials: nrt(m) x m x R (qtw_split, both sweep kernels)
      for (int mm = R; mm <= ldT; mm += R)
        for (int mma = 0; mma < 2; ++mma) {
          int64_t ch = 0;
          int nrt = 0;
          qtw_split(c, q.sq, mm, mma != 0, R, &ch, &nrt);
          cpart_len = std::max(cpart_len, (size_t)nrt * mm * R);
        }
    }
    q.cpart = dalloc<double>(cpart_len);
    q.csum = dalloc<double>(ldT * R);
    q.c2 = dalloc<double>(ldT * R);
    q.qcpart = dalloc<double>(full ? (size_t)c->CCn * c->n * R : (size_t)c->CC * q.sq * R);
  }
  q.small = dalloc<double>(512);
  CK(cudaMemsetAsync(q.ring, 0, ((size_t)(K + 1) * blk + 64) * sizeof(double), c->st));
  tr.mark("device allocations + memsets", c->st);
  if (!full) setup_tma(c, q);
  tr.mark("tensor maps", c->st);
  CK(cudaMemsetAsync(q.Tdev, 0, (size_t)ldT * ldT * sizeof(double), c->st));
  CK(cudaMemsetAsync(q.flags, 0, (c->dmax + 2) * sizeof(int), c->st));
  CK(cudaMemsetAsync(q.Hc, 0, (size_t)(c->dmax + 1) * (K + 1) * R * R * sizeof(double), c->st));
  CK(cudaMallocHost(&q.Hh, (size_t)(c->dmax + 1) * (K + 1) * R * R * sizeof(double)));
  q.Th = new double[(size_t)ldT * ldT];   // host copy of T, filled on demand (sync_T)
  CK(cudaMallocHost(&q.Rh, (size_t)(c->dmax + 2) * R * R * sizeof(double)));
  CK(cudaMallocHost(&q.flags_h, (c->dmax + 2) * sizeof(int)));
  tr.mark("pinned host mirrors", c->st);
  std::memset(q.Hh, 0, (size_t)(c->dmax + 1) * (K + 1) * R * R * sizeof(double));

  // C (row-major, host or device) -> Cdev (SoA) and Z_1 (ring slot 1)
  {
    const bool dev = is_device_ptr(C);
    double* tmp = dalloc<double>((size_t)c->n * R);
    CK(cudaMemcpyAsync(tmp, C, (size_t)c->n * R * sizeof(double), dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
    CK(cudaMemsetAsync(q.Cdev, 0, blk * sizeof(double), c->st));
    SYLV_DISPATCH_R(R, { k_to_soa<R_><<<c->sm * 4, 256, 0, c->st>>>(c->n, tmp, q.cdata(), q.ld); });
    count(c);
    if (c->comm) c->comm->halo(q.cdata(), R, q.ld, q.gz, c->st, kChanSetup);   // ghosts of Z_1 = C
    CK(cudaMemcpyAsync(q.slot(1) - q.gz, q.Cdev, blk * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    dfree(tmp);
  }
  // Alg. 1 line 1: ell = chol(C^T C) (U_1 ell = C), S C -> CholQR2 -> beta, Q_1
  double* ell_d = q.small + 192;
  double* elli_d = q.small + 256;
  double* beta_d = q.small + 320;
  SYLV_DISPATCH_R(R, {
    k_gram_soa<R_><<<c->G, kThreads, 0, c->st>>>(c->n, q.cdata(), q.ld, q.part2);
  });
  {
    int npc = c->G;
    const double* pc = reduce_partials(c, q.part2, c->G, R * R, c->red ? c->red + (int64_t)q.which * (K + 1) * R * R : nullptr,
                                       c->st, kChanSetup, &npc);
    SYLV_DISPATCH_R(R, { k_chol_small<R_><<<1, kSmallThreads, 0, c->st>>>(pc, npc, ell_d, elli_d, nullptr, q.flags, 0); });
  }
  count(c, 2);
  CK(cudaGetLastError());
  tr.mark("C upload, SoA, halo, Gram", c->st);
  if (!sketched) {
    // Alg. 2 / full method, line 1: U_1 beta = C with beta = ell = R(C); no sketch, T = I
    // (the unwhitened projection: M_U = H_d), R_1 = ell^{-1}; the full method stores U_1
    // normalised in slot 1 (R_1 = I)
    k_set_identity<<<(int)std::min<int64_t>(1024, (ldT * ldT + 255) / 256), 256, 0, c->st>>>(q.Tdev, ldT);
    if (full) {
      SYLV_DISPATCH_R(R, { k_soa_rmul_inplace<R_><<<c->sm * 4, kThreads, 0, c->st>>>(c->n, q.slot(1), q.ld, elli_d); });
      k_set_identity<<<1, 64, 0, c->st>>>(q.Rall + R * R, R);
      k_set_identity<<<1, 64, 0, c->st>>>(q.Rall, R);
    } else {
      CK(cudaMemcpyAsync(q.Rall + R * R, elli_d, R * R * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    }
    count(c, full ? 4 : 1);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(q.ell, ell_d, R * R * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(q.flags_h, q.flags, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    std::memcpy(q.beta, q.ell, sizeof(q.beta));   // the projected right-hand side uses R(C)
    if (q.flags_h[0]) throw Status{SYLV_E_INVALID, "C1 or C2 is rank deficient"};
    return;
  }
  if (q.sq != q.s) {          // sharded sketch space: this rank keeps rows [rank sq, rank sq + sq) of S C
    launch_sketch(c, q, q.cdata(), R, nullptr, q.skfull, c->st);
    c->comm->reduce_scatter(q.skfull, q.sk, (size_t)q.sq * R, c->st, kChanSetup);
  } else {
    launch_sketch(c, q, q.cdata(), R, nullptr, q.sk, c->st);
    if (c->comm) c->comm->allreduce(q.sk, (size_t)q.s * R, c->st, kChanSetup);
  }
  CK(cudaGetLastError());
  tr.mark("sketch of C", c->st);
  // sketched GS (f3): S Z_1 = S C kept (the s-space ring), ell = R(S C) = beta, so U_1 = C beta^{-1}
  // is S-orthonormal and T_1 = beta ell^{-1} = I
  if (sgs) CK(cudaMemcpyAsync(q.skz + sR, q.sk, sR * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  cholqr2(c, q, q.sk, 0, beta_d, 0, c->st);
  if (sgs) CK(cudaMemcpyAsync(ell_d, beta_d, R * R * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  SYLV_DISPATCH_R(R, { k_init_tau<R_><<<1, 1, 0, c->st>>>(beta_d, ell_d, q.Tdev, ldT, q.Rall + R * R); });
  count(c);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(q.beta, beta_d, R * R * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(q.ell, ell_d, R * R * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(q.flags_h, q.flags, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  tr.mark("CholQR2, T_1, mirrors", c->st);
  if (q.flags_h[0]) throw Status{SYLV_E_INVALID, "C1 or C2 (or its sketch) is rank deficient"};
}

// One block step j (1-based) of one sequence: Alg. 1 lines 3-9, in two phases.
// step_passes (lines 3-8): the n-space passes and the coefficient kernels on `st`.
// step_sketch (line 9): the sketch of the new block on `st` (it reads the block just written
// and the ring slot is rewritten only by a later pass on the same stream), then the sketch-space
// QR update on `side`, which overlaps the next step's passes.
void qr_update(sylv_ctx* c, Sequence& q, int j, cudaStream_t st);

// Row split of the Q^T w sweeps for m columns over `rows` rows.  DMMA (k_qtw_mma): one warp per
// (32 columns, row chunk); FMA (k_qtw): a CTA per (64 columns, row tile <= qtw_tile<R>(), the w
// tile it stages in shared memory), i.e. ~8 columns per warp.  A fixed tile left most of the GPU
// idle at small m (c2, m <= 100: 13 CTAs, 40 us per sweep; c0 / c4: 1-2 CTAs), so the row chunks
// (multiples of 32 rows, >= 128) are chosen for about 16 busy warps per SM; deterministic for a
// given (rows, m).
void qtw_split(const sylv_ctx* c, int64_t rows, int m, bool mma, int R, int64_t* chunk, int* nrt) {
  const int64_t wn = mma ? (m + 31) / 32 : (m + 7) / 8;
  const int64_t target = (int64_t)c->sm * 16;
  const int64_t rt = std::max<int64_t>(1, std::min<int64_t>((rows + 127) / 128, (target + wn - 1) / wn));
  int64_t ch = ((rows + rt - 1) / rt + 31) / 32 * 32;
  if (!mma) {
    int64_t cap = 0;
    SYLV_DISPATCH_R(R, { cap = qtw_tile<R_>(); });
    ch = std::min(ch, cap);
  }
  *chunk = ch;
  *nrt = (int)((rows + ch - 1) / ch);
}

void step_passes(sylv_ctx* c, Sequence& q, int j, cudaStream_t st, bool sketch_on_side) {
  const int R = c->R, K = c->K;
  const int nwin = std::min(K, j);
  Win win{};
  for (int i = 0; i < nwin; ++i) win.p[i] = q.slot(j - nwin + 1 + i);
  const bool timing = (c->cflags & 1) != 0;
  const int G = pass_parts(c, q);
  const int G1 = pass1_parts(c, q);
  TimedPair t1{}, t2{};
  // ---- a1 + a2 coefficients: pass 1
  if (timing) { t1 = ev_get(c, 0); CK(cudaEventRecord(t1.a, st)); }
  launch_pass1(c, q, win, nwin, j, st);
  if (timing) { CK(cudaEventRecord(t1.b, st)); c->timed.push_back(t1); }
  const int chan_main = q.which == 0 ? kChanUMain : kChanVMain;
  double* red = c->red ? c->red + (int64_t)q.which * (K + 1) * R * R : nullptr;
  int np1 = G1;
  const double* p1 = reduce_partials(c, q.part1, G1, K * R * R, red, st, chan_main, &np1);
  SYLV_DISPATCH_RK(R, K, {
    k_coef1<R_, K_><<<1, kSmallThreads, 0, st>>>(p1, np1, nwin, j, q.Rall, q.Kc, q.Hc, q.hn2);
  });
  // ---- a2 update + a3 Gram: pass 2 (writes Z_{j+1} = W' into the ring slot that the
  //      sketch of step j-K-1 read: earlier on this stream, or on the side stream)
  if (sketch_on_side && j - K - 1 >= 1) CK(cudaStreamWaitEvent(st, q.ev_sk[(j - K - 1) % (K + 2)], 0));
  if (timing) { t2 = ev_get(c, 1); CK(cudaEventRecord(t2.a, st)); }
  launch_pass2<true>(c, q, win, nwin, j, q.Yt, q.Kc + (int64_t)j * (1 + K) * R * R, q.slot(j + 1), st);
  if (timing) { CK(cudaEventRecord(t2.b, st)); c->timed.push_back(t2); }
  int np2 = G;
  const double* p2 = reduce_partials(c, q.part2, G, R * R, red ? red + K * R * R : nullptr, st, chan_main, &np2);
  SYLV_DISPATCH_RK(R, K, {
    k_coef2<R_, K_><<<1, kSmallThreads, 0, st>>>(p2, np2, j, q.Rall, q.Hc, q.hn2, q.flags);
  });
  // ghost planes/lines of the new block for the next step's stencil (sharded contexts)
  if (c->comm) c->comm->halo(q.slot(j + 1), R, q.ld, q.gz, st, chan_main);
  count(c, 2);
  CK(cudaGetLastError());
  // ---- H column j mirror
  const size_t hb = (size_t)(K + 1) * R * R;
  CK(cudaMemcpyAsync(q.Hh + (size_t)j * hb, q.Hc + (size_t)j * hb, hb * sizeof(double),
                     cudaMemcpyDeviceToHost, st));
}

void step_sketch(sylv_ctx* c, Sequence& q, int j, cudaStream_t st, cudaStream_t side, bool sketch_on_side) {
  const int R = c->R, K = c->K;
  const bool timing = (c->cflags & 1) != 0;
  const int ne = K + 2;
  const int chan = q.which == 0 ? (sketch_on_side ? kChanUSide : kChanUMain) : (sketch_on_side ? kChanVSide : kChanVMain);
  TimedPair t3{}, t4{};
  if (side != st) {
    if (sketch_on_side) {
      CK(cudaEventRecord(q.ev_c2[j % ne], st));               // block j+1 written
      CK(cudaStreamWaitEvent(side, q.ev_c2[j % ne], 0));
      st = side;
    } else if (j >= 2) {
      CK(cudaStreamWaitEvent(st, q.ev_sk[(j - 1) % ne], 0));   // QR j-1 done with w
    }
  }
  // ---- a4: w = (S W') R_{j+1}   (a5 timing includes the sketch)
  if (timing) { t3 = ev_get(c, 2); CK(cudaEventRecord(t3.a, st)); }
  if (timing) { t4 = ev_get(c, 3); CK(cudaEventRecord(t4.a, st)); }
  if (q.sq != q.s) {   // sharded sketch space: reduce-scatter of the partial sketches (S linear in rows)
    launch_sketch(c, q, q.slot(j + 1), R, q.Rall + (int64_t)(j + 1) * R * R, q.skfull, st);
    c->comm->reduce_scatter(q.skfull, q.w, (size_t)q.sq * R, st, chan);
  } else {
    launch_sketch(c, q, q.slot(j + 1), R, q.Rall + (int64_t)(j + 1) * R * R, q.w, st);
    if (c->comm) c->comm->allreduce(q.w, (size_t)q.s * R, st, chan);   // S linear in rows
  }
  if (timing) { CK(cudaEventRecord(t4.b, st)); c->timed.push_back(t4); }
  if (side != st) {                                           // pull: QR on the side stream
    CK(cudaEventRecord(q.ev_c2[j % ne], st));
    CK(cudaStreamWaitEvent(side, q.ev_c2[j % ne], 0));
    st = side;
  } else if (sketch_on_side && st != c->st && st != c->st2) {
    CK(cudaEventRecord(q.ev_sk[j % ne], st));                 // ring slot j+1 read
  }
  qr_update(c, q, j, st);
  if (timing) { CK(cudaEventRecord(t3.b, st)); c->timed.push_back(t3); }
  if (!sketch_on_side && st != c->st && st != c->st2) CK(cudaEventRecord(q.ev_sk[j % ne], st));   // w free
}

// a5 (Alg. 1 line 9): block CGS2 of w = S U_{j+1} (s x R, q.w) against Q (m = j R
// columns), CholQR2 (positive diagonal) -> Q[:, m:m+R], T column [c1 + c2; tau] on `st`.
void qr_update(sylv_ctx* c, Sequence& q, int j, cudaStream_t st) {
  const int R = c->R;
  const int m = j * R;
  const int64_t rows = q.sq;                 // this rank's rows of w and Q (sharded: s / P)
  const bool shard = rows != q.s;
  const int chan = q.which == 0 ? kChanUSide : kChanVSide;
  // tensor-core sweeps (k_qtw_mma / k_qc_mma) for R >= 4 with 16-byte aligned columns
  const bool mma = R >= 4 && rows % 4 == 0 && c->qmma;
  int64_t qchunk = c->tileQ;
  int nrt = c->RT;
  qtw_split(c, rows, m, mma, R, &qchunk, &nrt);
  const dim3 gq(mma ? (unsigned)(((m + 31) / 32 + kWarps - 1) / kWarps) : (unsigned)((m + kQtwCols - 1) / kQtwCols),
                nrt);
  int cols_per_chunk = (m + c->CC - 1) / c->CC;
  if (mma) cols_per_chunk = (cols_per_chunk + 15) / 16 * 16;
  const int ncc = (m + cols_per_chunk - 1) / cols_per_chunk;
  const dim3 gc((unsigned)((rows + kThreads - 1) / kThreads), ncc);
  const int64_t mR = (int64_t)m * R;
  const int gr = (int)std::min<int64_t>(1024, (mR + 255) / 256);
  const int gw = (int)std::min<int64_t>(1024, (rows * R + 255) / 256);
  SYLV_DISPATCH_R(R, {
    auto qtw = [&]() {
      if constexpr (R_ >= 4) {
        if (mma) {
          k_qtw_mma<R_><<<gq, kThreads, 0, st>>>(q.Q, rows, rows, m, q.w, qchunk, q.cpart);
          return;
        }
      }
      k_qtw<R_><<<gq, kThreads, 0, st>>>(q.Q, rows, rows, m, q.w, qchunk, 1, q.cpart);
    };
    auto qc = [&](const double* cv) {
      if constexpr (R_ >= 4) {
        if (mma) {
          k_qc_mma<R_><<<gc, kThreads, 0, st>>>(q.Q, rows, rows, m, cv, cols_per_chunk, q.qcpart);
          return;
        }
      }
      k_qc_part<R_><<<gc, kThreads, 0, st>>>(q.Q, rows, rows, m, cv, cols_per_chunk, q.qcpart);
    };
    // sum of the nrt row-chunk partials: many parts of a short vector -> the part-parallel kernel
    auto red_parts = [&](const double* part, int np, int64_t len, double* out, double* acc) {
      if (np >= 32 && len <= (int64_t)np * 256)
        k_red_parts_wide<<<(unsigned)((len + 31) / 32), 32 * std::min(32, (np + 3) / 4), 0, st>>>(part, np, len, out, acc);
      else
        k_red_parts<<<gr, 256, 0, st>>>(part, np, len, out, acc);
    };
    // pass A: c1 = Q^T w (sharded: local rows, then the m R coefficients summed over the ranks)
    qtw();
    red_parts(q.cpart, nrt, mR, q.csum, nullptr);
    if (shard) c->comm->allreduce(q.csum, (size_t)mR, st, chan);
    // w -= Q c1
    qc(q.csum);
    k_wsub<<<gw, 256, 0, st>>>(q.w, q.qcpart, ncc, rows * R);
    // pass B: c2 = Q^T w, csum += c2
    qtw();
    if (shard) {
      red_parts(q.cpart, nrt, mR, q.c2, nullptr);
      c->comm->allreduce(q.c2, (size_t)mR, st, chan);
      k_axpy_inplace<<<gr, 256, 0, st>>>(q.c2, q.csum, mR);
    } else {
      red_parts(q.cpart, nrt, mR, q.c2, q.csum);
    }
    qc(q.c2);
    k_wsub<<<gw, 256, 0, st>>>(q.w, q.qcpart, ncc, rows * R);
  });
  count(c, 8);
  CK(cudaGetLastError());
  double* tau_d = q.small + 384;
  cholqr2(c, q, q.w, m, tau_d, j + 1, st);
  SYLV_DISPATCH_R(R, {
    k_tcol<R_><<<std::max(1, (int)std::min<int64_t>(256, ((int64_t)(m + R) * R + 255) / 256)), 256, 0, st>>>(
        q.csum, tau_d, q.Tdev, q.ldT, m);
  });
  count(c);
  CK(cudaGetLastError());
}

// Sketched inner products in the truncated GS (method 3, f3), step j of one
// sequence: n-space apply + sketch of the matvec, s-space coefficients (no reduction over n),
// the pass-2 update without Gram, s-space normalisation; the sketched QR update (a5) on `side`
// (sketched_gs.cuh).
void step_sgs(sylv_ctx* c, Sequence& q, int j, cudaStream_t st, cudaStream_t side) {
  const int R = c->R, K = c->K;
  const int nwin = std::min(K, j);
  const int ne = K + 2;
  const int64_t sR = q.s * R;
  auto skz = [&](int i) { return q.skz + (int64_t)(i % (K + 1)) * sR; };
  Win win{}, zs{};
  for (int i = 0; i < nwin; ++i) {
    win.p[i] = q.slot(j - nwin + 1 + i);
    zs.p[i] = skz(j - nwin + 1 + i);
  }
  const int ga = (int)std::min<int64_t>((int64_t)c->sm * 8, (c->n + kThreads - 1) / kThreads);
  SYLV_DISPATCH_R(R, { k_apply_soa<R_><<<ga, kThreads, 0, st>>>(q.op, q.slot(j), q.ld, q.Yt); });
  count(c);
  // the sketch buffer q.sk is reused every step: the previous step's s-space kernels ran on st
  launch_sketch(c, q, q.Yt, R, nullptr, q.sk, st);
  if (c->comm) c->comm->allreduce(q.sk, (size_t)sR, st, q.which == 0 ? kChanUMain : kChanVMain);
  const int gs = (int)std::max<int64_t>(1, std::min<int64_t>(c->G, (q.s + kThreads - 1) / kThreads));
  SYLV_DISPATCH_RK(R, K, {
    k_skpass1<R_, K_><<<dim3(gs, K_ * R_), kThreads, 0, st>>>(zs, nwin, q.s, q.sk, q.part1);
    k_coef1<R_, K_><<<1, kSmallThreads, 0, st>>>(q.part1, gs, nwin, j, q.Rall, q.Kc, q.Hc, q.hn2);
  });
  count(c, 2);
  const double* coef = q.Kc + (int64_t)j * (1 + K) * R * R;
  launch_pass2<false>(c, q, win, nwin, j, q.Yt, coef, q.slot(j + 1), st);
  if (c->comm) c->comm->halo(q.slot(j + 1), R, q.ld, q.gz, st, q.which == 0 ? kChanUMain : kChanVMain);
  SYLV_DISPATCH_RK(R, K, {
    k_skpass2<R_, K_><<<gs, kThreads, 0, st>>>(zs, nwin, q.s, q.sk, coef, skz(j + 1), q.part2);
    k_coef2<R_, K_><<<1, kSmallThreads, 0, st>>>(q.part2, gs, j, q.Rall, q.Hc, q.hn2, q.flags);
  });
  count(c, 2);
  CK(cudaGetLastError());
  const size_t hb = (size_t)(K + 1) * R * R;
  CK(cudaMemcpyAsync(q.Hh + (size_t)j * hb, q.Hc + (size_t)j * hb, hb * sizeof(double), cudaMemcpyDeviceToHost, st));
  // w = S U_{j+1} = (S Z_{j+1}) R_{j+1}, once the previous QR update is done with w
  if (j >= 2 && side != st) CK(cudaStreamWaitEvent(st, q.ev_sk[(j - 1) % ne], 0));
  const int gw = (int)std::min<int64_t>(c->G, (q.s + 255) / 256);
  SYLV_DISPATCH_R(R, { k_rmul<R_><<<gw, kThreads, 0, st>>>(q.s, skz(j + 1), q.Rall + (int64_t)(j + 1) * R * R, q.w, 0); });
  count(c);
  if (side != st) {
    CK(cudaEventRecord(q.ev_c2[j % ne], st));
    CK(cudaStreamWaitEvent(side, q.ev_c2[j % ne], 0));
  }
  qr_update(c, q, j, side);
  if (side != st) CK(cudaEventRecord(q.ev_sk[j % ne], side));
}

// Full Arnoldi (method 2), step j of one sequence on `st`: W~ = A U_j
// (row-major n x R in q.w), block CGS2 against ALL retained blocks U_1..U_j (two sweeps of the
// basis: c1 = U^T W~, W~ -= U c1, c2 = U^T W~, W~ -= U c2; h_{.,j} = c1 + c2), CholQR2 ->
// U_{j+1} normalised into ring slot j+1 (SoA) and h_{j+1,j}; H column j mirrored to the host.
void step_full(sylv_ctx* c, Sequence& q, int j, cudaStream_t st) {
  const int R = c->R, K = c->K;
  const int64_t n = c->n;
  const int m = j * R;
  const double* Ub = q.slot(1);   // basis column (b-1) R + c at Ub + ((b-1) R + c) ld (no ring wrap)
  const int ga = (int)std::min<int64_t>((int64_t)c->sm * 8, (n + kThreads - 1) / kThreads);
  SYLV_DISPATCH_R(R, { k_apply_rowmajor<R_><<<ga, kThreads, 0, st>>>(q.op, q.slot(j), q.ld, q.w); });
  const dim3 gq((m + kQtwCols - 1) / kQtwCols, c->RTn);
  const int cpc = (m + c->CCn - 1) / c->CCn;
  const int ncc = (m + cpc - 1) / cpc;
  const dim3 gc((unsigned)((n + kThreads - 1) / kThreads), ncc);
  const int64_t mR = (int64_t)m * R;
  const int gr = (int)std::min<int64_t>(1024, (mR + 255) / 256);
  const int gw = (int)std::min<int64_t>(4 * c->sm, (n * R + 255) / 256);
  SYLV_DISPATCH_R(R, {
    k_qtw<R_><<<gq, kThreads, 0, st>>>(Ub, n, q.ld, m, q.w, c->tileQ, c->tpcN, q.cpart);
    k_red_parts<<<gr, 256, 0, st>>>(q.cpart, c->RTn, mR, q.csum, nullptr);
    k_qc_part<R_><<<gc, kThreads, 0, st>>>(Ub, n, q.ld, m, q.csum, cpc, q.qcpart);
    k_wsub<<<gw, 256, 0, st>>>(q.w, q.qcpart, ncc, n * R);
    k_qtw<R_><<<gq, kThreads, 0, st>>>(Ub, n, q.ld, m, q.w, c->tileQ, c->tpcN, q.cpart);
    k_red_parts<<<gr, 256, 0, st>>>(q.cpart, c->RTn, mR, q.c2, q.csum);
    k_qc_part<R_><<<gc, kThreads, 0, st>>>(Ub, n, q.ld, m, q.c2, cpc, q.qcpart);
    k_wsub<<<gw, 256, 0, st>>>(q.w, q.qcpart, ncc, n * R);
  });
  count(c, 9);
  CK(cudaGetLastError());
  double* tau = q.small + 384;
  cholqr2_into(c, q, q.w, n, q.slot(j + 1), q.ld, tau, j + 1, st);
  SYLV_DISPATCH_R(R, { k_full_hcol<R_><<<1, kSmallThreads, 0, st>>>(q.csum, tau, m, j, K, q.Hc, q.Rall, q.flags); });
  count(c);
  CK(cudaGetLastError());
  const size_t hb = (size_t)(K + 1) * R * R;
  CK(cudaMemcpyAsync(q.Hh + (size_t)j * hb, q.Hc + (size_t)j * hb, hb * sizeof(double), cudaMemcpyDeviceToHost, st));
}

// Host copy of the leading rows x rows block of T (upper triangular, column-major, ldT).
// Called only after the streams have been joined (residual, solution, get_small).
// Uses the residual stream (c->rst: the context stream, or the solve driver's own stream
// while the next steps run on the context streams; the block read is final either way).
void sync_T(sylv_ctx* c, Sequence& q, int rows) {
  CK(cudaMemcpy2DAsync(q.Th, q.ldT * sizeof(double), q.Tdev, q.ldT * sizeof(double), (size_t)rows * sizeof(double),
                       rows, cudaMemcpyDeviceToHost, c->rst));
  CK(cudaStreamSynchronize(c->rst));
}

sylv_status fail(sylv_ctx* c, sylv_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

template <typename F>
sylv_status guard(sylv_ctx* c, F&& f) {
  try {
    return f();
  } catch (...) {
    // a rank that fails inside a collective sequence releases its peers (LocalComm)
    if (c && c->comm) c->comm->abort();
    try {
      throw;
    } catch (const CudaError& e) {
      return fail(c, SYLV_E_CUDA, std::string(e.what) + ": " + cudaGetErrorString(e.e));
    } catch (const Status& s) {
      return fail(c, s.s, s.msg);
    } catch (const std::bad_alloc&) {
      return fail(c, SYLV_E_NOMEM, "host allocation failed");
    } catch (const CommError& e) {
      return fail(c, SYLV_E_NCCL, e.what);
    }
  }
}

// Projected solve of check d on the device (sign iteration) or on the host (Bartels-Stewart)
// Sharded contexts solve the projected equation redundantly on every rank (identical small
// matrices).  The library solvers on that path need not be bitwise reproducible across ranks
// (cuSOLVER Xgeev's hybrid host part; a device solve certified on one rank, rejected on another),
// so the values a decision or an output rests on — rho, and Y for the second pass — are rank 0's
// on every rank: one allreduce on the setup channel with the other ranks contributing zeros.
void agree_rank0(sylv_ctx* c, double* host, size_t n) {
  if (!c->comm || c->comm->nranks <= 1 || n == 0) return;
  double* buf = dalloc<double>(n);
  if (c->comm->rank == 0)
    CK(cudaMemcpyAsync(buf, host, n * sizeof(double), cudaMemcpyHostToDevice, c->rst));
  else
    CK(cudaMemsetAsync(buf, 0, n * sizeof(double), c->rst));
  c->comm->allreduce(buf, n, c->rst, kChanSetup);
  CK(cudaMemcpyAsync(host, buf, n * sizeof(double), cudaMemcpyDeviceToHost, c->rst));
  CK(cudaStreamSynchronize(c->rst));
  dfree(buf);
}

bool device_solve(const sylv_ctx* c, int d) {
  // auto: device for d r >= 512, except at and beyond a d where it already fell back (the
  // conditioning of the projected matrices only grows with d: c1 needs the host there)
  return (c->cflags & 8) || (!(c->cflags & 16) && d * c->R >= 512 && d < c->gpu_fail_d);
}

// Enqueue block steps first..last (Alg. 1 lines 3-9 for both sequences) and the flag
// copies; no synchronisation (sylv_sketch_step = enqueue + finish; the solve driver
// enqueues the steps to the next check before solving the current one).
void enqueue_steps(sylv_ctx* c, int first, int last) {
  c->d_dev = std::max(c->d_dev, last);
  // U passes on the context stream, V passes on st2 (independent sequences); each
  // sequence's sketch-space work on its own side stream.  Serial mode: all on st.
  const bool serial = (c->cflags & 2) != 0;
  cudaStream_t others[3] = {c->st2, c->st3, c->st4};
  if (!serial) {
    CK(cudaEventRecord(c->fork, c->st));
    for (cudaStream_t s : others) CK(cudaStreamWaitEvent(s, c->fork, 0));
  }
  // Pull sketch (large n): per step, U and V passes concurrently (st, st2; each hides the
  // other's small coefficient kernels), then the U sketch, then the V sketch — the L2-resident
  // pull sketch (sketch_pull.cuh) must not share L2 with a streaming pass — then each
  // sequence's sketch-space QR on its side stream, overlapping the next step's passes.
  // Push sketch (small n): sketch + QR on the side streams, overlapping the next passes.
  const char* sched_env = std::getenv("SYLV_SCHED");   // "overlap" | "phase" (tuning)
  // CSR operators: the windowed pass 1 is latency-bound (HBM and L2 not saturated), so the pull
  // sketch overlaps it profitably (c4: 1.009 -> 0.922 ms per step); stencils keep the phases
  const bool on_side = sched_env ? std::strcmp(sched_env, "overlap") == 0
                                 : (!c->seq[0].pl_list || c->seq[0].op.kind == kCSR);
  for (int j = first; j <= last; ++j) {
    if (c->method == SYLV_METHOD_SKETCHED_GS) {   // f3: sketched inner products in the GS
      step_sgs(c, c->seq[0], j, c->st, serial ? c->st : c->st3);
      step_sgs(c, c->seq[1], j, serial ? c->st : c->st2, serial ? c->st : c->st4);
    } else if (c->method == SYLV_METHOD_FULL) {          // comparison method: full Arnoldi
      step_full(c, c->seq[0], j, c->st);
      step_full(c, c->seq[1], j, serial ? c->st : c->st2);
    } else if (c->method == SYLV_METHOD_TRUNCATED) {   // Alg. 2: the n-space passes only
      step_passes(c, c->seq[0], j, c->st, false);
      step_passes(c, c->seq[1], j, serial ? c->st : c->st2, false);
    } else if (serial) {
      step_passes(c, c->seq[0], j, c->st, false);
      step_sketch(c, c->seq[0], j, c->st, c->st, false);
      step_passes(c, c->seq[1], j, c->st, false);
      step_sketch(c, c->seq[1], j, c->st, c->st, false);
    } else if (on_side) {
      step_passes(c, c->seq[0], j, c->st, true);
      step_sketch(c, c->seq[0], j, c->st, c->st3, true);
      step_passes(c, c->seq[1], j, c->st2, true);
      step_sketch(c, c->seq[1], j, c->st2, c->st4, true);
    } else {
      step_passes(c, c->seq[0], j, c->st, false);
      step_passes(c, c->seq[1], j, c->st2, false);
      CK(cudaEventRecord(c->phase[0], c->st2));      // V passes done
      CK(cudaStreamWaitEvent(c->st, c->phase[0], 0));
      step_sketch(c, c->seq[0], j, c->st, c->st3, false);
      CK(cudaEventRecord(c->phase[1], c->st));       // U sketch done
      CK(cudaStreamWaitEvent(c->st2, c->phase[1], 0));
      step_sketch(c, c->seq[1], j, c->st2, c->st4, false);
      CK(cudaEventRecord(c->phase[2], c->st2));      // V sketch done
      CK(cudaStreamWaitEvent(c->st, c->phase[2], 0));
    }
  }
  if (!serial) {
    for (int i = 0; i < 3; ++i) {
      CK(cudaEventRecord(c->join[i], others[i]));
      CK(cudaStreamWaitEvent(c->st, c->join[i], 0));
    }
  }
  CK(cudaMemcpyAsync(c->seq[1].flags_h + first, c->seq[1].flags + first, (last - first + 2) * sizeof(int),
                     cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(c->seq[0].flags_h + first, c->seq[0].flags + first, (last - first + 2) * sizeof(int),
                     cudaMemcpyDeviceToHost, c->st));
}

// Wait for enqueued steps first..last, check breakdown / lost-independence flags, advance d_done.
sylv_status finish_steps(sylv_ctx* c, int first, int last) {
  CK(cudaStreamSynchronize(c->st));
  ev_collect(c);
  for (int j = first; j <= last; ++j) {
    const int f = c->seq[0].flags_h[j] | c->seq[1].flags_h[j];
    if (f & 1 || f & 2) {
      c->d_done = j;
      c->stats.steps += j - first + 1;
      c->broken = true;
      c->breakdown_d = j;
      c->halted = true;
      c->halt_status = SYLV_E_BREAKDOWN;
      c->halt_msg = "breakdown at step " + std::to_string(j);
      return fail(c, SYLV_E_BREAKDOWN, c->halt_msg);
    }
    const int g = c->seq[0].flags_h[j + 1] | c->seq[1].flags_h[j + 1];
    if (g & 4) {
      // terminal like a breakdown: steps j+1.. may already have run on the device (solve
      // driver prefetch) and overwritten the ring, so the state cannot be advanced from j
      c->d_done = j;
      c->stats.steps += j - first + 1;
      c->halted = true;
      c->halt_status = SYLV_E_LOST_INDEP;
      c->halt_msg = "sketched basis lost independence at step " + std::to_string(j);
      return fail(c, SYLV_E_LOST_INDEP, c->halt_msg);
    }
  }
  c->stats.steps += last - first + 1;
  c->d_done = last;
  return SYLV_OK;
}


// f1 (round 2): an APPROXIMATE rho_rel(d) from the device sign iteration, accepted off the
// identity (c1: M_V has eigenvalues with Re < 0 near the crossing, so the iteration solves a
// neighbouring equation; measured 0.25-8 % off).  Used only to choose WHERE the exact checks of
// the solve driver go; no decision rests on it, nothing is recorded (hist, y_d).  NaN on failure.
double probe_rho(sylv_ctx* c, int d) {
  const int r = c->R, m = d * r;
  if (d < 1 || d > c->d_done || m < 64) return NAN;
  try {
    Sequence& U = c->seq[0];
    Sequence& V = c->seq[1];
    double hhat[kMaxR * kMaxR], ghat[kMaxR * kMaxR], Bm[kMaxR * kMaxR];
    sync_T(c, U, m + r);
    sync_T(c, V, m + r);
    hat_coefficient(d, r, c->K, U.Th, U.ldT, U.Hh, hhat);
    hat_coefficient(d, r, c->K, V.Th, V.ldT, V.Hh, ghat);
    double bn = 0.0;
    for (int a = 0; a < r; ++a)
      for (int b = 0; b < r; ++b) {
        double sacc = 0.0;
        for (int p = 0; p < r; ++p) sacc += U.beta[a * r + p] * V.beta[b * r + p];
        Bm[a * r + b] = sacc;
        bn += sacc * sacc;
      }
    bn = std::sqrt(bn);
    if (!c->gsolve) {
      c->gsolve = new GpuSylv();
      c->gsolve->mcap = (c->dmax + 1) * r;
    }
    GpuSylv& gs = *c->gsolve;
    gs.allow_approx = true;
    const bool ok = gs.solve(U.Tdev, U.Hc, V.Tdev, V.Hc, U.ldT, d, r, c->K, Bm, c->rst);
    gs.allow_approx = false;
    if (!ok) return NAN;
    std::vector<double> lrow((size_t)m * r), lcol((size_t)m * r);
    CK(cudaMemcpy2DAsync(lrow.data(), (size_t)r * sizeof(double), gs.C + (m - r), (size_t)m * sizeof(double),
                         (size_t)r * sizeof(double), m, cudaMemcpyDeviceToHost, c->rst));
    CK(cudaMemcpyAsync(lcol.data(), gs.C + (size_t)(m - r) * m, (size_t)m * r * sizeof(double),
                       cudaMemcpyDeviceToHost, c->rst));
    CK(cudaStreamSynchronize(c->rst));
    if (c->y_dev) c->y_d = -1;              // the device Y buffer was overwritten by the probe
    double s1 = 0.0, s2 = 0.0;
    for (int col = 0; col < m; ++col)
      for (int a = 0; a < r; ++a) {
        double v = 0.0;
        for (int p = 0; p < r; ++p) v += hhat[a * r + p] * lrow[(size_t)col * r + p];
        s1 += v * v;
      }
    for (int row = 0; row < m; ++row)
      for (int a = 0; a < r; ++a) {
        double v = 0.0;
        for (int p = 0; p < r; ++p) v += lcol[(size_t)p * m + row] * ghat[a * r + p];
        s2 += v * v;
      }
    c->stats.gpu_approx_checks++;
    double pr = std::sqrt(s1 + s2) / bn;
    agree_rank0(c, &pr, 1);   // the check placement must not diverge across ranks
    return pr;
  } catch (const ProjError&) {
    cudaGetLastError();
    return NAN;
  }
}

}  // namespace

// ====================================================================================
// extern "C" boundary
// ====================================================================================
extern "C" {

const char* sylv_version(void) { return SYLV_VERSION; }

sylv_status sylv_host_projected(int32_t d, int32_t r, int32_t k, const double* T, int64_t ldT,
                                const double* H, double* M) {
  if (d < 1 || r < 1 || k < 1 || !T || !H || !M || ldT < (int64_t)(d + 1) * r) return SYLV_E_INVALID;
  if (!lapack_loaded()) return SYLV_E_LAPACK;
  std::vector<double> Mv;
  build_projected(d, r, k, T, ldT, H, Mv);
  std::memcpy(M, Mv.data(), Mv.size() * sizeof(double));
  return SYLV_OK;
}

sylv_status sylv_host_sylvester(int32_t m, int32_t r, double* MU, double* MV, const double* B, double* Y) {
  if (m < 1 || r < 1 || r > m || !MU || !MV || !B || !Y) return SYLV_E_INVALID;
  if (!lapack_loaded()) return SYLV_E_LAPACK;
  std::vector<double> a(MU, MU + (size_t)m * m), b(MV, MV + (size_t)m * m), y;
  std::string err;
  const int info = sylvester_bs(m, r, a, b, B, y, err);
  if (info < 0) return SYLV_E_LAPACK;
  if (info > 0) return SYLV_E_SINGULAR;
  std::memcpy(Y, y.data(), y.size() * sizeof(double));
  return SYLV_OK;
}

sylv_status sylv_set_lapack_path(const char* path) {
  std::string err;
  if (!path || !lapack_load(path, err)) {
    std::fprintf(stderr, "sylv_set_lapack_path: %s\n", err.c_str());
    return SYLV_E_LAPACK;
  }
  return SYLV_OK;
}

const char* sylv_sketch_last_error(const sylv_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

sylv_status sylv_partition(int32_t kind, int32_t N, int64_t n, int32_t nranks, int32_t rank, int64_t* row_begin,
                           int64_t* row_end) {
  if (!row_begin || !row_end || nranks < 1 || rank < 0 || rank >= nranks || N < 1) return SYLV_E_INVALID;
  int64_t unit;
  if (kind == SYLV_OP_STENCIL3D && n == (int64_t)N * N * N) unit = (int64_t)N * N;
  else if (kind == SYLV_OP_STENCIL2D && n == (int64_t)N * N) unit = N;
  else if (kind == SYLV_OP_CSR && n > 0) {
    // rows in groups of 32 (N is ignored)
    const int64_t ngrp = (n + 31) / 32;
    if (ngrp < nranks) return SYLV_E_INVALID;
    *row_begin = std::min<int64_t>(n, 32 * (ngrp * rank / nranks));
    *row_end = std::min<int64_t>(n, 32 * (ngrp * (rank + 1) / nranks));
    return *row_end > *row_begin ? SYLV_OK : SYLV_E_INVALID;
  } else return SYLV_E_INVALID;
  // planes/lines in groups of g so that every range starts at a multiple of 32 rows
  int64_t g = 1;
  while ((g * unit) % 32) ++g;
  const int64_t ngrp = (N + g - 1) / g;
  if (ngrp < nranks) return SYLV_E_INVALID;
  const int64_t gb = ngrp * rank / nranks, ge = ngrp * (rank + 1) / nranks;
  *row_begin = std::min<int64_t>(N, gb * g) * unit;
  *row_end = std::min<int64_t>(N, ge * g) * unit;
  return *row_end > *row_begin ? SYLV_OK : SYLV_E_INVALID;
}

sylv_status sylv_comm_nccl_unique_id(uint8_t id[128]) {
  if (!id) return SYLV_E_INVALID;
  NcclApi& a = nccl_api();
  if (!a.GetUniqueId) return SYLV_E_NCCL;
  ncclUniqueId u;
  if (a.GetUniqueId(&u) != ncclSuccess) return SYLV_E_NCCL;
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return SYLV_OK;
}

sylv_status sylv_comm_create_nccl(int32_t nranks, int32_t rank, const uint8_t id[128], sylv_comm** out) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return SYLV_E_INVALID;
  *out = nullptr;
  try {
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    std::unique_ptr<sylv_comm> c(new sylv_comm());
    c->impl = new NcclComm(nranks, rank, u);
    *out = c.release();
    return SYLV_OK;
  } catch (const CommError& e) {
    std::fprintf(stderr, "sylv_comm_create_nccl: %s\n", e.what.c_str());
    return SYLV_E_NCCL;
  }
}

sylv_status sylv_comm_wrap_nccl(void* nccl_comm, sylv_comm** out) {
  if (!out || !nccl_comm) return SYLV_E_INVALID;
  *out = nullptr;
  try {
    std::unique_ptr<sylv_comm> c(new sylv_comm());
    c->impl = new NcclComm(static_cast<ncclComm_t>(nccl_comm));
    *out = c.release();
    return SYLV_OK;
  } catch (const CommError& e) {
    std::fprintf(stderr, "sylv_comm_wrap_nccl: %s\n", e.what.c_str());
    return SYLV_E_NCCL;
  }
}

sylv_status sylv_local_group_create(int32_t nranks, void** group) {
  if (!group || nranks < 1 || nranks > kMaxLocalRanks) return SYLV_E_INVALID;
  *group = new LocalGroup(nranks);
  return SYLV_OK;
}

void sylv_local_group_destroy(void* group) { delete static_cast<LocalGroup*>(group); }

sylv_status sylv_comm_create_local(void* group, int32_t rank, sylv_comm** out) {
  if (!out || !group) return SYLV_E_INVALID;
  LocalGroup* g = static_cast<LocalGroup*>(group);
  if (rank < 0 || rank >= g->P) return SYLV_E_INVALID;
  sylv_comm* c = new sylv_comm();
  c->impl = new LocalComm(g, rank);
  *out = c;
  return SYLV_OK;
}

void sylv_comm_destroy(sylv_comm* comm) {
  if (!comm) return;
  delete comm->impl;
  delete comm;
}

void sylv_sketch_destroy(sylv_ctx* ctx) {
  if (!ctx) return;
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  for (cudaStream_t s : {ctx->st2, ctx->st3, ctx->st4, ctx->st_solve})
    if (s) cudaStreamSynchronize(s);
  for (auto& q : ctx->seq) free_seq(q);
  dfree(ctx->red);
  delete ctx->gsolve;
  if (ctx->blas) cublasDestroy(ctx->blas);
  for (cudaStream_t s : {ctx->st2, ctx->st3, ctx->st4, ctx->st_solve})
    if (s) cudaStreamDestroy(s);
  if (ctx->fork) cudaEventDestroy(ctx->fork);
  for (cudaEvent_t e : ctx->join)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->phase)
    if (e) cudaEventDestroy(e);
  for (auto& p : ctx->free_events) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto& p : ctx->timed) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  delete ctx;
}

sylv_status sylv_sketch_init(const sylv_operator* A, const sylv_operator* B, const double* C1,
                             const double* C2, const sylv_config* cfg, void* nccl_comm, void* stream,
                             sylv_ctx** out) {
  if (!out) return SYLV_E_INVALID;
  *out = nullptr;
  if (!A || !B || !C1 || !C2 || !cfg) return SYLV_E_INVALID;
  sylv_ctx* c = new sylv_ctx();
  *out = c;
  const int r = cfg->r;
  if (!(r == 1 || r == 2 || r == 4 || r == 8)) return fail(c, SYLV_E_INVALID, "r must be 1, 2, 4 or 8");
  const int method = cfg->method;
  if (method < SYLV_METHOD_SKETCHED || method > SYLV_METHOD_SKETCHED_GS) return fail(c, SYLV_E_INVALID, "unknown method");
  const bool sketched = method == SYLV_METHOD_SKETCHED || method == SYLV_METHOD_SKETCHED_GS;
  if (method != SYLV_METHOD_FULL && (cfg->k < 1 || cfg->k > (r <= 2 ? kMaxK : 4)))
    return fail(c, SYLV_E_INVALID, "k must be in [1, 4] (r = 4, 8) or [1, 10] (r = 1, 2)");
  if (cfg->d_max < 1) return fail(c, SYLV_E_INVALID, "d_max must be >= 1");
  const bool srdct = cfg->sketch_kind == SYLV_SKETCH_SRDCT;
  if (cfg->sketch_kind != SYLV_SKETCH_SPARSE_SIGN && !srdct) return fail(c, SYLV_E_INVALID, "unknown sketch kind");
  if (srdct && (!cfg->srdct_signs_u || !cfg->srdct_signs_v || !cfg->srdct_rows_u || !cfg->srdct_rows_v))
    return fail(c, SYLV_E_INVALID, "SRDCT: signs and rows of both sketches are required");
  if (srdct && nccl_comm) return fail(c, SYLV_E_INVALID, "SRDCT: single-rank only (the DCT mixes all rows)");
  if (srdct && A->n > INT32_MAX) return fail(c, SYLV_E_INVALID, "SRDCT: n must fit the FFT length");
  if (sketched && !srdct && (cfg->zeta < 1 || cfg->s <= 0 || cfg->s % cfg->zeta)) return fail(c, SYLV_E_INVALID, "s must be a positive multiple of zeta");
  if (srdct && (cfg->s <= 0 || cfg->s > A->n)) return fail(c, SYLV_E_INVALID, "SRDCT: 0 < s <= n");
  if (sketched && cfg->s < (int64_t)(cfg->d_max + 1) * r) return fail(c, SYLV_E_INVALID, "s must be >= (d_max+1) r");
  if (method == SYLV_METHOD_FULL && nccl_comm) return fail(c, SYLV_E_INVALID, "the full method is single-rank only");
  if (A->n != B->n || A->n <= 0) return fail(c, SYLV_E_INVALID, "A and B must be n x n with equal n");
  Comm* comm = nccl_comm ? static_cast<sylv_comm*>(nccl_comm)->impl : nullptr;
  if (comm && (A->kind != B->kind || (A->kind != SYLV_OP_CSR && A->grid[0] != B->grid[0])))
    return fail(c, SYLV_E_INVALID, "sharded contexts need A and B of the same kind (and grid for stencils)");
  if (sketched && !srdct && (uint64_t)A->n * cfg->zeta >= (1ull << 32)) return fail(c, SYLV_E_INVALID, "n*zeta must be < 2^32");
  for (const sylv_operator* o : {A, B}) {
    if (o->kind == SYLV_OP_STENCIL2D || o->kind == SYLV_OP_STENCIL3D) {
      const int64_t N = o->grid[0];
      const int64_t nn = (o->kind == SYLV_OP_STENCIL2D) ? N * N : N * N * N;
      if (N < 1 || nn != o->n) return fail(c, SYLV_E_INVALID, "stencil grid does not match n");
    } else if (o->kind == SYLV_OP_CSR) {
      if (!o->row_ptr || !o->col_idx || !o->val || o->nnz < 0) return fail(c, SYLV_E_INVALID, "CSR arrays missing");
    } else {
      return fail(c, SYLV_E_INVALID, "unknown operator kind");
    }
  }
  return guard(c, [&]() -> sylv_status {
    c->st = (cudaStream_t)stream;
    c->rst = c->st;
    c->R = r;
    c->method = method;
    c->K = method == SYLV_METHOD_FULL ? cfg->d_max : cfg->k;   // full: every block is in the window
    c->dmax = cfg->d_max;
    c->zeta = (sketched && cfg->sketch_kind == SYLV_SKETCH_SPARSE_SIGN) ? cfg->zeta : 8;
    c->n_global = A->n;
    c->row_begin = 0;
    c->row_end = A->n;
    if (comm) {
      // this rank's rows: given, or the balanced partition of sylv_partition
      int64_t rb = cfg->row_begin, re = cfg->row_end;
      if (rb == 0 && re == 0 &&
          sylv_partition(A->kind, A->grid[0], A->n, comm->nranks, comm->rank, &rb, &re) != SYLV_OK)
        throw Status{SYLV_E_INVALID, "cannot partition the grid over this many ranks"};
      comm->gather_ranges(rb, re);                                    // collective
      const bool csr = A->kind == SYLV_OP_CSR;
      const int64_t unit = (A->kind == SYLV_OP_STENCIL3D) ? (int64_t)A->grid[0] * A->grid[0]
                           : csr ? 32 : A->grid[0];
      for (int q = 0; q < comm->nranks; ++q) {
        const int64_t b = comm->rb[q], e = comm->re[q];
        if ((q == 0 && b != 0) || (q > 0 && b != comm->re[q - 1]) || (q == comm->nranks - 1 && e != A->n))
          throw Status{SYLV_E_INVALID, "row ranges must tile [0, n) in rank order"};
        if (e <= b || b % unit || (e % unit && e != A->n) || b % 32)
          throw Status{SYLV_E_INVALID, "row ranges must be whole, non-empty sets of grid planes (3-D) / lines (2-D) "
                                       "starting at multiples of 32 (CSR: multiples of 32 rows)"};
      }
      c->comm = comm;
      c->row_begin = rb;
      c->row_end = re;
      c->red = dalloc<double>((size_t)2 * (cfg->k + 1) * r * r);
    } else if (!(cfg->row_begin == 0 && (cfg->row_end == 0 || cfg->row_end == A->n))) {
      throw Status{SYLV_E_INVALID, "a row range needs a communicator"};
    }
    c->n = c->row_end - c->row_begin;
    c->s = sketched ? cfg->s : (int64_t)(cfg->d_max + 1) * r;   // unsketched: s only sizes unused scratch
    c->tol = cfg->tol;
    c->rank_tol = cfg->rank_tol > 0 ? cfg->rank_tol : 1e-12;
    c->chunk = cfg->chunk > 0 ? std::min(cfg->chunk, kMaxChunk) : 0;   // 0: auto (second pass)
    c->cflags = cfg->flags;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&c->sm, cudaDevAttrMultiProcessorCount, dev));
    const int64_t rows_per_cta = (int64_t)kWarps * (32 / r);
    c->G = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->sm * 4, (c->n + rows_per_cta - 1) / rows_per_cta));
    // Q^T w: (ceil(m / kQtwCols) x RT) CTAs, row tiles of qtw_tile<R>() rows
    // sketch space sharded by rows over the ranks: Alg. 1 with the hashed sparse
    // sign, several ranks, s a multiple of the rank count; else replicated on every rank
    c->sq = (comm && comm->nranks > 1 && method == SYLV_METHOD_SKETCHED && !srdct && c->s % comm->nranks == 0 &&
             !std::getenv("SYLV_SKETCH_REPLICATED"))
                ? c->s / comm->nranks : c->s;
    SYLV_DISPATCH_R(r, { c->tileQ = qtw_tile<R_>(); });
    if (const char* e = std::getenv("SYLV_QMMA")) c->qmma = std::atoi(e) != 0;   // A/B switch
    if (const char* e = std::getenv("SYLV_EIG")) c->eig_solve = std::atoi(e);   // A/B switch, tests
    c->RT = (int)((c->sq + c->tileQ - 1) / c->tileQ);
    // Q c: (ceil(s/256) x CC) CTAs, ~4 per SM at the full width (each thread streams a row
    // of its column chunk with 8 loads in flight)
    c->CC = (int)std::max<int64_t>(1, std::min<int64_t>(16, (4 * c->sm + (c->sq / 256)) / std::max<int64_t>(1, c->sq / 256)));
    if (method == SYLV_METHOD_FULL) {
      // n-space Q^T w over the retained basis: ~2 CTAs per SM of row chunks, each `tpcN` tiles
      const int64_t tiles = (c->n + c->tileQ - 1) / c->tileQ;
      c->tpcN = (int)std::max<int64_t>(1, (tiles + 2 * c->sm - 1) / (2 * c->sm));
      c->RTn = (int)((tiles + c->tpcN - 1) / c->tpcN);
      c->CCn = 1;
    }
    // sketch kernel: whole sketch column (s doubles) in shared memory per CTA
    c->sk_smem = (size_t)sketch_smem_doubles(c->s, c->zeta) * sizeof(double);
    int max_optin = 0;
    CK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (sketched && cfg->sketch_kind == SYLV_SKETCH_SPARSE_SIGN && c->sk_smem > (size_t)max_optin)
      throw Status{SYLV_E_INVALID, "s too large: the sketch column (8 s bytes) must fit in shared memory"};
    if (!sketched) c->sk_smem = 0;
    SYLV_DISPATCH_R(r, {
      CK(cudaFuncSetAttribute(k_sketch_cols<R_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->sk_smem));
    });
    int smem_sm = 0;
    CK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    const int per_sm = std::max(1, (int)(smem_sm / (c->sk_smem + 1024)));
    const int64_t ngroups = (c->n + 31) / 32;
    // a chunk also costs 2 s shared-memory ops (zero, write out) and s partial reads in the
    // reduction: give every chunk at least ~s scatter updates (32 zeta per group), so small n
    // does not end in one-group chunks (c0: 128 chunks of 1 group, a 25 us reduction)
    const int64_t min_gpc = std::max<int64_t>(1, c->s / (32 * std::max(1, c->zeta)));
    c->nchunk = (int)std::max<int64_t>(1, std::min<int64_t>((ngroups + min_gpc - 1) / min_gpc,
                                                            (int64_t)c->sm * per_sm / r));
    c->gpc = (ngroups + c->nchunk - 1) / c->nchunk;
    c->nchunk = (int)((ngroups + c->gpc - 1) / c->gpc);
    {
      // SYLV_SKETCH=cols|pull overrides the size rule (development / A-B timing)
      const char* e = std::getenv("SYLV_SKETCH");
      c->sk_pull = e ? std::strcmp(e, "pull") == 0 : ngroups >= kPullMinGroups;
    }
    CK(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->st3, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->st4, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->st_solve, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
    for (cudaEvent_t& e : c->join) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (cudaEvent_t& e : c->phase) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const bool srdct = cfg->sketch_kind == SYLV_SKETCH_SRDCT;
    init_sequence(c, c->seq[0], 0, A, false, C1, cfg->seed_u, srdct ? cfg->srdct_signs_u : nullptr,
                  srdct ? cfg->srdct_rows_u : nullptr);
    init_sequence(c, c->seq[1], 1, B, true, C2, cfg->seed_v, srdct ? cfg->srdct_signs_v : nullptr,
                  srdct ? cfg->srdct_rows_v : nullptr);
    return SYLV_OK;
  });
}

sylv_status sylv_sketch_step(sylv_ctx* c, int32_t nsteps, int32_t* d_done) {
  if (!c) return SYLV_E_INVALID;
  if (d_done) *d_done = c->d_done;
  if (c->halted) return fail(c, c->halt_status, c->halt_msg);
  return guard(c, [&]() -> sylv_status {
    const int first = c->d_done + 1;
    const int last = std::min(c->dmax, c->d_done + std::max(0, nsteps));
    if (last >= first) {
      enqueue_steps(c, first, last);
      const sylv_status st = finish_steps(c, first, last);
      if (d_done) *d_done = c->d_done;
      if (st != SYLV_OK) return st;
    }
    if (d_done) *d_done = c->d_done;
    if (nsteps > 0 && std::max(0, last - first + 1) < nsteps)
      return fail(c, SYLV_E_NOT_CONVERGED, "d_max reached");
    return SYLV_OK;
  });
}

sylv_status sylv_sketch_residual(sylv_ctx* c, int32_t d, double* rho, double* rho_rel) {
  if (!c) return SYLV_E_INVALID;
  if (d < 1 || d > c->d_done) return fail(c, SYLV_E_STATE, "residual(d) needs 1 <= d <= d_done");
  if (!lapack_loaded()) return fail(c, SYLV_E_LAPACK, "host LAPACK not loaded: call sylv_set_lapack_path");
  return guard(c, [&]() -> sylv_status {
    auto t0 = std::chrono::steady_clock::now();
    const int r = c->R, m = d * r;
    Sequence& U = c->seq[0];
    Sequence& V = c->seq[1];
    double hhat[kMaxR * kMaxR], ghat[kMaxR * kMaxR], Bm[kMaxR * kMaxR];
    sync_T(c, U, m + r);
    sync_T(c, V, m + r);
    hat_coefficient(d, r, c->K, U.Th, U.ldT, U.Hh, hhat);
    hat_coefficient(d, r, c->K, V.Th, V.ldT, V.Hh, ghat);
    double bn = 0.0;
    for (int a = 0; a < r; ++a)
      for (int b = 0; b < r; ++b) {
        double s = 0.0;
        for (int p = 0; p < r; ++p) s += U.beta[a * r + p] * V.beta[b * r + p];
        Bm[a * r + b] = s;
        bn += s * s;
      }
    bn = std::sqrt(bn);
    // Y's last r rows (lrow[col * r + p] = Y[m-r+p, col]) and last r columns
    // (lcol[p * m + row] = Y[row, m-r+p]) are all the residual needs
    std::vector<double> lrow((size_t)m * r), lcol((size_t)m * r);
    bool done = false, approx_used = false;
    // rho^2 = ||hhat E_d^T Y||^2 + ||Y E_d ghat^T||^2 from Y's last rows / columns
    auto rho_of = [&](const std::vector<double>& lr, const std::vector<double>& lc) {
      double s1 = 0.0, s2 = 0.0;
      for (int col = 0; col < m; ++col)
        for (int a = 0; a < r; ++a) {
          double v = 0.0;
          for (int p = 0; p < r; ++p) v += hhat[a * r + p] * lr[(size_t)col * r + p];
          s1 += v * v;
        }
      for (int row = 0; row < m; ++row)
        for (int a = 0; a < r; ++a) {
          double v = 0.0;
          for (int p = 0; p < r; ++p) v += lc[(size_t)p * m + row] * ghat[a * r + p];
          s2 += v * v;
        }
      return std::sqrt(s1 + s2);
    };
    const bool approx_mode = c->approx_thr > 0.0 && !(c->cflags & 16) && d * r >= 512;
    const bool want_gpu = device_solve(c, d) || approx_mode;
    if (want_gpu) {
      // f1: device sign-function solve; falls back to the host on non-convergence
      try {
        if (!c->gsolve) {
          c->gsolve = new GpuSylv();
          c->gsolve->mcap = (c->dmax + 1) * r;
        }
        GpuSylv& gs = *c->gsolve;
        gs.allow_approx = approx_mode;
        // the sign iteration first (it needs spec(M_U), spec(M_V) in Re > 0); where it failed
        // before (d >= sign_fail_d) or fails now, the certified eigendecomposition solve (f1, r2)
        bool ok = false;
        if ((d < c->sign_fail_d && c->eig_solve != 2) || approx_mode) {
          ok = gs.solve(U.Tdev, U.Hc, V.Tdev, V.Hc, U.ldT, d, r, c->K, Bm, c->rst);
          if (!ok && !approx_mode) c->sign_fail_d = std::min(c->sign_fail_d, d);
        }
        gs.allow_approx = false;
        if (!ok && !approx_mode && c->eig_solve) {
          ok = gs.solve_eig(U.Tdev, U.Hc, V.Tdev, V.Hc, U.ldT, d, r, c->K, Bm, c->rst);
          gs.off_identity = false;
          if (ok) c->eig_solves++;
        }
        if (ok) {
          CK(cudaMemcpy2DAsync(lrow.data(), (size_t)r * sizeof(double), gs.C + (m - r), (size_t)m * sizeof(double),
                               (size_t)r * sizeof(double), m, cudaMemcpyDeviceToHost, c->rst));
          CK(cudaMemcpyAsync(lcol.data(), gs.C + (size_t)(m - r) * m, (size_t)m * r * sizeof(double),
                             cudaMemcpyDeviceToHost, c->rst));
          CK(cudaStreamSynchronize(c->rst));
          done = true;
          if (gs.off_identity) {
            // approximate: usable only to decide "clearly above tol"
            const double rr_approx = rho_of(lrow, lcol) / bn;
            if (!(rr_approx > c->approx_thr)) done = false;
            else {
              c->stats.gpu_approx_checks++;
              approx_used = true;
            }
          }
          if (done) {
            c->y_dev = true;
            c->stats.gpu_solves++;
            c->stats.gpu_solve_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          }
        }
        if (!ok || !done) {
          c->stats.gpu_solve_fallbacks++;
          c->gpu_fail_d = std::min(c->gpu_fail_d, d);
          c->err = "device projected solve did not converge at d = " + std::to_string(d) + " (" +
                   std::to_string(c->gsolve->iterations) + " iterations); host fallback";
        }
      } catch (const ProjError& e) {
        c->stats.gpu_solve_fallbacks++;
        c->gpu_fail_d = std::min(c->gpu_fail_d, d);
        c->err = "device projected solve failed at d = " + std::to_string(d) + ": " + e.what + "; host fallback";
        if (std::getenv("SYLV_TRACE_PROJ")) std::fprintf(stderr, "[proj] %s\n", c->err.c_str());
        cudaGetLastError();
      }
    }
    if (!done) {
      std::vector<double> MU, MV;
      build_projected(d, r, c->K, U.Th, U.ldT, U.Hh, MU);
      build_projected(d, r, c->K, V.Th, V.ldT, V.Hh, MV);
      // a numerically singular T_d (sketched basis lost independence) gives non-finite M;
      // LAPACK's Schur iteration must not see it
      for (const std::vector<double>* Mx : {&MU, &MV})
        for (double v : *Mx)
          if (!std::isfinite(v)) {
            c->y_d = -1;
            if (rho) *rho = NAN;
            if (rho_rel) *rho_rel = NAN;
            return fail(c, SYLV_E_SINGULAR, "projected matrix not finite at d = " + std::to_string(d));
          }
      std::string err;
      const int info = sylvester_bs(m, r, MU, MV, Bm, c->Y, err);
      c->stats.host_solve_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      c->stats.host_solves++;
      if (info < 0) return fail(c, SYLV_E_LAPACK, err);
      if (info > 0) {
        c->hist.emplace_back(d, NAN);   // a failed check, kept in the history
        c->y_d = -1;
        if (rho) *rho = NAN;
        if (rho_rel) *rho_rel = NAN;
        return fail(c, SYLV_E_SINGULAR, err);
      }
      c->y_dev = false;
      for (int col = 0; col < m; ++col)
        for (int p = 0; p < r; ++p) {
          lrow[(size_t)col * r + p] = c->Y[(size_t)col * m + (m - r + p)];
          lcol[(size_t)p * m + col] = c->Y[(size_t)(m - r + p) * m + col];
        }
    }
    c->y_d = approx_used ? -1 : d;   // an approximate Y is never kept as the solution of d
    double rh = rho_of(lrow, lcol);
    if (c->method == SYLV_METHOD_TRUNCATED) {
      // Alg. 2 line 12 / Prop. 3.2: rho = sqrt(dr) (||Y E_d g^T|| + ||h E_d^T Y||)
      std::vector<double> zc((size_t)m * r, 0.0);
      const double a = rho_of(lrow, zc), b = rho_of(zc, lcol);
      rh = std::sqrt((double)m) * (a + b);
    }
    agree_rank0(c, &rh, 1);
    if (rho) *rho = rh;
    if (rho_rel) *rho_rel = rh / bn;
    c->hist.emplace_back(d, rh / bn);
    return SYLV_OK;
  });
}

sylv_status sylv_sketch_solution(sylv_ctx* c, int32_t d, double* X1, double* X2, int64_t ldx,
                                 int32_t max_rank, int32_t* rank) {
  if (!c) return SYLV_E_INVALID;
  if (d < 1 || d > c->d_done) return fail(c, SYLV_E_STATE, "solution(d) needs 1 <= d <= d_done");
  if (!X1 || !X2 || max_rank < 0 || ldx < max_rank) return fail(c, SYLV_E_INVALID, "bad output buffers");
  if (c->y_d != d) {
    double rho, rr;
    sylv_status s = sylv_sketch_residual(c, d, &rho, &rr);
    if (s != SYLV_OK) return s;
  }
  return guard(c, [&]() -> sylv_status {
    const int r = c->R, m = d * r, K = c->K;
    if (c->y_dev) {                                   // Y of the last (device) solve
      c->Y.resize((size_t)m * m);
      CK(cudaMemcpyAsync(c->Y.data(), c->gsolve->C, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      c->y_dev = false;
    }
    InitTrace tr;   // SYLV_TRACE_INIT=1: phase times on stderr
    std::vector<double> Y1, Y2;
    std::string err;
    agree_rank0(c, c->Y.data(), (size_t)m * m);   // sharded: rank 0's Y on every rank
    const int l = svd_truncate(m, c->Y, c->rank_tol, max_rank, Y1, Y2, err);
    tr.mark("solution: SVD of Y", c->st);
    if (l < 0) return fail(c, SYLV_E_LAPACK, err);
    if (rank) *rank = l;
    double* Xout[2] = {X1, X2};
    std::vector<double>* Ys[2] = {&Y1, &Y2};
    double* rbuf_keep = nullptr;   // replay ring, shared by the two sequences
    size_t rbuf_elems = 0;
    struct RbufFree {
      double*& p;
      ~RbufFree() { if (p) dfree(p); }
    } rbuf_guard{rbuf_keep};
    for (int qi = 0; qi < 2; ++qi) {
      int C = c->chunk;   // 0: chosen below from the free device memory
      Sequence& q = c->seq[qi];
      // Z = T_d^{-1} Y_q ; M_b = R_b Z[b-block]  (U_b = Z_b R_b)
      trsm_left_upper(m, l, q.Th, q.ldT, Ys[qi]->data());
      CK(cudaMemcpyAsync(q.Rh, q.Rall, (size_t)(d + 2) * r * r * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      std::vector<double> M((size_t)m * std::max(l, 1), 0.0);
      for (int b = 1; b <= d; ++b)
        for (int a = 0; a < r; ++a)
          for (int col = 0; col < l; ++col) {
            double s = 0.0;
            for (int p = 0; p < r; ++p)
              s += q.Rh[(size_t)b * r * r + a * r + p] * (*Ys[qi])[(size_t)col * m + (b - 1) * r + p];
            M[(size_t)((b - 1) * r + a) * l + col] = s;
          }
      tr.mark("solution: T^-1 Y, R_b blocks", c->st);
      const bool dev_out = is_device_ptr(Xout[qi]);
      double* Xd = dev_out ? Xout[qi] : dalloc<double>((size_t)c->n * ldx);
      CK(cudaMemsetAsync(Xd, 0, (size_t)c->n * ldx * sizeof(double), c->st));
      if (l > 0 && c->method == SYLV_METHOD_FULL) {
        // full method: the basis is retained and normalised (R_b = I, T = I): X = U_d Y_q,
        // one DGEMM over the d contiguous ring slots (X^T += M^T U^T)
        double* Md = dalloc<double>(M.size());
        CK(cudaMemcpyAsync(Md, M.data(), M.size() * sizeof(double), cudaMemcpyHostToDevice, c->st));
        cublasHandle_t hb = (c->gsolve && c->gsolve->hb) ? c->gsolve->hb : c->blas;
        if (!hb) {
          if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) throw Status{SYLV_E_CUDA, "cublasCreate"};
          hb = c->blas;
        }
        if (cublasSetStream(hb, c->st) != CUBLAS_STATUS_SUCCESS) throw Status{SYLV_E_CUDA, "cublasSetStream"};
        const double one = 1.0;
        if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, l, (int)c->n, m, &one, Md, l, q.slot(1), (int)q.ld, &one, Xd,
                        (int)ldx) != CUBLAS_STATUS_SUCCESS)
          throw Status{SYLV_E_CUDA, "cublasDgemm (X = U Y)"};
        CK(cudaStreamSynchronize(c->st));
        dfree(Md);
      } else if (l > 0) {
        double* Md = dalloc<double>(M.size());
        if (C <= 0) {
          // replay chunk: every chunk of C blocks is one pass over X (n x l) — with the default
          // C = k + 1 the X traffic dominated the second pass (c3 at rank 216: 58 passes over
          // 29 GB per sequence); use up to half the free memory for up to kMaxChunk blocks
          size_t fr = 0, tot = 0;
          CK(cudaMemGetInfo(&fr, &tot));
          const int64_t blkb = q.ld * r * (int64_t)sizeof(double);
          C = (int)std::max<int64_t>(c->K + 1, std::min<int64_t>(kMaxChunk, (int64_t)(fr / 2) / blkb - K));
          if (rbuf_keep)   // the second sequence: as many blocks as the kept ring holds
            C = (int)std::max<int64_t>(c->K + 1, std::min<int64_t>(kMaxChunk, (int64_t)rbuf_elems / (q.ld * r) - K));
        }
        // one replay ring for both sequences (a second cudaMalloc/cudaFree of tens of GB cost
        // ~0.4 s at c3); re-zeroed per sequence (ghosts = 0; the layouts may differ)
        const size_t rel = (size_t)(K + C) * q.ld * r;
        if (rel > rbuf_elems) {
          if (rbuf_keep) dfree(rbuf_keep);
          rbuf_keep = dalloc<double>(rel);
          rbuf_elems = rel;
        }
        double* rbuf = rbuf_keep;
        CK(cudaMemsetAsync(rbuf, 0, rel * sizeof(double), c->st));
        CK(cudaMemcpyAsync(Md, M.data(), M.size() * sizeof(double), cudaMemcpyHostToDevice, c->st));
        auto rslot = [&](int j) { return rbuf + (int64_t)(j % (K + C)) * q.ld * r + q.gz; };
        CK(cudaMemcpyAsync(rslot(1) - q.gz, q.Cdev, (size_t)q.ld * r * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
        // the 2.5-D TMA pass 2 for the replay too: tensor maps of the replay slots
        std::vector<CUtensorMap> rmapH, rmapW;
        bool rtma = q.tma;
        if (rtma) {
          rmapH.resize(K + C);
          rmapW.resize(K + C);
          const int N = q.st25.N, nz = q.st25.nz;
          for (int sl = 0; sl < K + C && rtma; ++sl) {
            const double* base = rbuf + (int64_t)sl * q.ld * r;
            rtma = encode_block_map(&rmapH[sl], base, N, nz + 2, q.ld, r, Geo25<kTY25>::HX, Geo25<kTY25>::HY) &&
                   encode_block_map(&rmapW[sl], base, N, nz + 2, q.ld, r, Geo25<kTY25>::WX, kTY25);
          }
        }
        int j0 = 1;
        for (int j = 1; j <= d; ++j) {
          if (j >= 2) {  // Z_j from Z_{j-nwin..j-1} with the stored pass-2 coefficients of step j-1
            const int jp = j - 1;
            const int nwin = std::min(K, jp);
            Win win{};
            for (int i = 0; i < nwin; ++i) win.p[i] = rslot(jp - nwin + 1 + i);
            const double* coef = q.Kc + (int64_t)jp * (1 + K) * r * r;
            if (rtma) {
              Tma25 tm;
              tm.zd = rmapH[jp % (K + C)];
              for (int i = 0; i < nwin - 1; ++i) tm.win[i] = rmapW[(jp - nwin + 1 + i) % (K + C)];
#define SYLV_ST3D_R(RR, KK) k_st3d<kTY25, RR, KK, 2, false><<<c->G25, 32 * kTY25 * kWpl25, c->smem25_2, c->st>>>(tm, q.st25, nwin, coef, rslot(j), q.part2)
              if (r == 8) {
                switch (K) {
                  case 1: SYLV_ST3D_R(8, 1); break;
                  case 2: SYLV_ST3D_R(8, 2); break;
                  case 3: SYLV_ST3D_R(8, 3); break;
                  case 4: SYLV_ST3D_R(8, 4); break;
                }
              } else {
                switch (K) {
                  case 1: SYLV_ST3D_R(4, 1); break;
                  case 2: SYLV_ST3D_R(4, 2); break;
                  case 3: SYLV_ST3D_R(4, 3); break;
                  case 4: SYLV_ST3D_R(4, 4); break;
                }
              }
#undef SYLV_ST3D_R
              count(c);
            } else {
              launch_pass2<false>(c, q, win, nwin, jp, nullptr, coef, rslot(j), c->st, /*allow_tma=*/false);
            }
            if (c->comm) c->comm->halo(rslot(j), r, q.ld, q.gz, c->st, kChanUMain);
          }
          if (j - j0 + 1 == C || j == d) {
            // X += [U_j0 .. U_j] M[j0..j] as DGEMMs over runs of adjacent replay slots (a run's
            // columns have the uniform stride ld): X^T (l x n, ld ldx) += M^T (l x kk) U^T
            // the device projected solver's cuBLAS handle when it exists (already initialised)
            cublasHandle_t hb = (c->gsolve && c->gsolve->hb) ? c->gsolve->hb : c->blas;
            if (!hb) {
              if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) throw Status{SYLV_E_CUDA, "cublasCreate"};
              hb = c->blas;
            }
            if (cublasSetStream(hb, c->st) != CUBLAS_STATUS_SUCCESS) throw Status{SYLV_E_CUDA, "cublasSetStream"};
            const double one = 1.0;
            int b0 = j0;
            while (b0 <= j) {
              int b1 = b0;
              while (b1 < j && (b1 + 1) % (K + C) != 0) ++b1;      // stop at the ring wrap
              const int kk = (b1 - b0 + 1) * r;
              if (cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, l, (int)c->n, kk, &one,
                              Md + (int64_t)(b0 - 1) * r * l, l, rslot(b0), (int)q.ld, &one, Xd, (int)ldx) !=
                  CUBLAS_STATUS_SUCCESS)
                throw Status{SYLV_E_CUDA, "cublasDgemm (X accumulation)"};
              b0 = b1 + 1;
            }
            j0 = j + 1;
          }
          CK(cudaGetLastError());
        }
        CK(cudaStreamSynchronize(c->st));
        tr.mark("solution: replay + X accumulation", c->st);
        dfree(Md);
      }
      if (!dev_out) {
        CK(cudaMemcpyAsync(Xout[qi], Xd, (size_t)c->n * ldx * sizeof(double), cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        dfree(Xd);
      }
    }
    CK(cudaStreamSynchronize(c->st));
    return SYLV_OK;
  });
}

sylv_status sylv_sketch_solve(sylv_ctx* c, int32_t* d_star, double* rho_rel) {
  if (!c) return SYLV_E_INVALID;
  // canonical schedule (R9; the paper's p = 10): every 10
  // steps while d r <= 800, then d_next = 10 ceil(1.15 d_prev / 10); d_max included;
  // bisection on the last bracket after the first pass.
  std::vector<int> sched;
  for (int d = 10; d <= c->dmax && d * c->R <= 800; d += 10) sched.push_back(d);
  int d = sched.empty() ? 10 : sched.back();
  while (true) {
    d = 10 * (int)std::ceil(1.15 * d / 10.0);
    if (d >= c->dmax) break;
    if (sched.empty() || d > sched.back()) sched.push_back(d);
  }
  if (sched.empty() || sched.back() != c->dmax) sched.push_back(c->dmax);
  int d_fail = 0, d_pass = -1, skips = 0;
  bool pass_by_breakdown = false;   // breakdown seen when the pass was decided (no bisection)
  double rr_pass = NAN, last_rr = NAN;
  // Before a check that is solved on the HOST, the steps up to the next scheduled check are
  // enqueued first: T and H of the checked d are final, the enqueued steps only append later
  // columns, so the CPU solve hides behind the GPU stepping (a passing check leaves at most
  // one batch of unneeded steps).  Device solves are not overlapped: measured on c3, their
  // GEMM/LU kernels and the pass kernels serialise on the SMs and the prefetched steps only
  // add work.
  int pend_first = 0, pend_last = -1;
  auto finish_pending = [&]() -> sylv_status {
    if (pend_last < pend_first) return SYLV_OK;
    const int f = pend_first, l = pend_last;
    pend_first = 0;
    pend_last = -1;
    return guard(c, [&]() -> sylv_status { return finish_steps(c, f, l); });
  };
  auto ok_step = [](sylv_status s) { return s == SYLV_OK || s == SYLV_E_BREAKDOWN || s == SYLV_E_NOT_CONVERGED; };
  // valid checks so far (d, rho_rel): the crossing prediction below uses the last two
  std::vector<std::pair<int, double>> seen;
  auto predict = [&](int d1, double r1, int d2, double r2) -> double {   // log-linear crossing
    if (!(r1 > r2) || !(r2 > 0) || !std::isfinite(r1) || d2 <= d1) return NAN;
    const double slope = (std::log(r2) - std::log(r1)) / (d2 - d1);
    return d2 + (std::log(c->tol) - std::log(r2)) / slope;
  };
  bool probe_walk = false;   // the last check was placed by approximate probes (f1, round 2)
  // schedule phase: approximate device checks may decide clear fails (rho_rel > 3 tol); the
  // search for the first crossing below uses exact solves only
  // (opt-in, SYLV_APPROX_CHECKS=1: an off-identity sign iteration solves a different
  // equation, so its rho_rel has no error bound; by default every check is exact)
  {
    const char* e = std::getenv("SYLV_APPROX_CHECKS");
    c->approx_thr = (e && std::strcmp(e, "1") == 0) ? 3.0 * c->tol : 0.0;
  }
  struct ApproxOff {   // every exit of the driver leaves residual() exact
    sylv_ctx* c;
    ~ApproxOff() { c->approx_thr = 0.0; }
  } approx_off{c};
  for (size_t idx = 0; idx < sched.size(); ++idx) {
    // past the every-10 regime: when the log-linear extrapolation of the last two checks puts
    // the crossing well before the next scheduled check, check just past the prediction
    // instead (same first crossing after the search below; fewer large projected solves)
    // (round 2) inside the every-10 regime a check is skipped while the predicted crossing lies
    // more than 10 steps past it and the next check is still in that regime (skipping into the
    // geometric regime overshot c1's crossing by 250 steps: one m = 4148 solve, ~20 s)
    if (seen.size() >= 2) {
      const auto& a = seen[seen.size() - 2];
      const auto& b = seen.back();
      const double dh = predict(a.first, a.second, b.first, b.second);
      if (std::isfinite(dh) && (int64_t)sched[idx] * c->R > 800 && dh + 2 < sched[idx]) {
        sched[idx] = std::max(b.first + 1, (int)std::ceil(dh) + 2);
        // f1 (round 2): when that check will be a host Bartels-Stewart solve (the device sign
        // iteration failed at or below it: c1), refine where it goes with approximate device
        // solves around the predicted crossing (they only move the check; SYLV_PROBE=0: off)
        // opt-in (SYLV_PROBE=1): the probes move checks away from the oracle's R9 schedule, so
        // with a non-monotone rho (Ex. 6.1 nu = 0.001, kappa(T) ~ 1e16) the search can find a
        // different crossing or none (d_max reached; B200 r2): off by default
        const char* pe = std::getenv("SYLV_PROBE");
        if ((pe && std::strcmp(pe, "1") == 0) && !device_solve(c, sched[idx]) && sched[idx] * c->R >= 512 &&
            c->d_done >= b.first) {
          const int target = std::min(c->dmax, sched[idx] + 12);
          if (c->d_done < target && !c->halted) {
            const sylv_status s0 = finish_pending();
            if (!ok_step(s0) && s0 != SYLV_E_LOST_INDEP) return s0;
            int dd = 0;
            if (c->d_done < target && !c->halted) sylv_sketch_step(c, target - c->d_done, &dd);
          }
          // probes at the predicted crossing and 10 steps on: log-linear through them (and the
          // last exact check) -> the first d predicted below tol, checked one step above it
          double xs[3], ys[3];
          int np = 0;
          xs[np] = b.first;
          ys[np++] = std::log(b.second);
          for (int pd : {std::max(b.first + 1, (int)std::ceil(dh)), std::max(b.first + 2, (int)std::ceil(dh) + 10)}) {
            const int pdc = std::min(pd, c->d_done);
            const double pr = probe_rho(c, pdc);
            if (std::isfinite(pr) && pr > 0.0) {
              xs[np] = pdc;
              ys[np++] = std::log(pr);
            }
          }
          if (np == 3) {
            // least-squares line through the last two (the probes): the local slope near the crossing
            const double sl = (ys[2] - ys[1]) / (xs[2] - xs[1]);
            if (sl < 0.0) {
              const double x = xs[1] + (std::log(c->tol) - ys[1]) / sl;
              if (std::isfinite(x)) {
                sched[idx] = std::max(b.first + 1, std::min(c->dmax, (int)std::ceil(x)));
                probe_walk = true;      // the exact checks walk one step at a time from here
              }
            }
          }
        }
      } else if (std::isfinite(dh) && dh - 10 > sched[idx] && idx + 1 < sched.size() &&
                 (int64_t)sched[idx + 1] * c->R <= 800 && sched[idx + 1] - b.first <= 50) {
        continue;   // every-10 regime, crossing far ahead: skip (R9; a valid check every <= 50 steps)
      }
    }
    const int dc = sched[idx];
    if (dc > c->dmax) break;
    if (c->d_done < dc && !c->halted) {
      sylv_status s = finish_pending();
      if (!ok_step(s) && s != SYLV_E_LOST_INDEP) return s;
      if (c->d_done < dc && !c->halted) {
        int dd = 0;
        s = sylv_sketch_step(c, dc - c->d_done, &dd);
        if (!ok_step(s) && s != SYLV_E_LOST_INDEP) return s;
      }
    }
    if (!c->halted && idx + 1 < sched.size() && !device_solve(c, std::min(dc, c->d_done))) {
      const int nx = std::min(sched[idx + 1], c->dmax);
      if (nx > c->d_done) {
        const int f = c->d_done + 1;
        const sylv_status s = guard(c, [&]() -> sylv_status {
          enqueue_steps(c, f, nx);
          return SYLV_OK;
        });
        if (s != SYLV_OK) return s;
        pend_first = f;
        pend_last = nx;
      }
    }
    const int dchk = std::min(dc, c->d_done);
    double rho, rr;
    c->rst = c->st_solve;
    sylv_status s = sylv_sketch_residual(c, dchk, &rho, &rr);
    c->rst = c->st;
    if (s == SYLV_E_SINGULAR) {
      if (++skips >= 5) break;
      continue;
    }
    if (s != SYLV_OK) {
      finish_pending();
      return s;
    }
    skips = 0;
    last_rr = rr;
    if (std::isfinite(rr)) seen.emplace_back(dchk, rr);
    // a breakdown decides a pass only at (or before) the checked d: with the crossing
    // prediction a check can be moved below steps that were already prefetched, and a
    // breakdown found while finishing those steps says nothing about dchk
    const bool brk = c->broken && c->breakdown_d <= dchk;
    if (rr < c->tol || brk) {
      d_pass = dchk;
      rr_pass = rr;
      pass_by_breakdown = brk;
      break;
    }
    d_fail = dchk;
    if (c->halted && c->d_done <= dchk) break;   // lost independence: no later d to check
    // a probe-placed check that failed: the crossing is just above it (walk up by 2, not to the
    // next geometric point)
    if (probe_walk && idx + 1 < sched.size()) sched[idx + 1] = std::min(sched[idx + 1], std::min(c->dmax, dchk + 2));
    probe_walk = false;
  }
  c->approx_thr = 0.0;
  {
    const sylv_status s = finish_pending();   // the last prefetched batch
    if (!ok_step(s) && s != SYLV_E_LOST_INDEP) return s;
  }
  if (d_pass < 0) {
    if (d_star) *d_star = c->d_done;
    if (rho_rel) *rho_rel = last_rr;
    return fail(c, SYLV_E_NOT_CONVERGED, "tolerance not reached by d_max");
  }
  // first crossing inside the bracket (d_fail, d_pass]: safeguarded regula falsi on
  // log rho_rel (Illinois), a bisection step whenever the bracket does not halve; with
  // rho_rel monotone on the bracket this returns the same d* as bisection
  // the projected solution of the best passing check so far (host-solved checks), so the
  // final d* need not be solved again (c1: one m ~ 3100 solve ~ 12 s)
  // (host-solved checks: a host copy of Y; device-solved checks: a device copy of the solver's Y)
  std::vector<double> best_Y;
  int best_d = -1;
  bool best_on_dev = false;
  struct DevBuf {
    double* p = nullptr;
    size_t cap = 0;
    ~DevBuf() { dfree(p); }
  } best_dev;
  auto keep_if_pass = [&](int d) {
    if (c->y_d != d) return;
    if (!c->y_dev) {
      best_Y = c->Y;
      best_on_dev = false;
    } else {
      const size_t mm = (size_t)d * c->R * d * c->R;
      const sylv_status st = guard(c, [&]() -> sylv_status {
        if (best_dev.cap < mm) {
          dfree(best_dev.p);
          best_dev.p = nullptr;
          best_dev.p = dalloc<double>(mm);
          best_dev.cap = mm;
        }
        CK(cudaMemcpyAsync(best_dev.p, c->gsolve->C, mm * sizeof(double), cudaMemcpyDeviceToDevice, c->rst));
        CK(cudaStreamSynchronize(c->rst));
        return SYLV_OK;
      });
      if (st != SYLV_OK) return;      // not kept: d* is re-solved at the end
      best_on_dev = true;
    }
    best_d = d;
  };
  keep_if_pass(d_pass);
  int lo = d_fail, hi = d_pass;
  double rlo = NAN, rhi = rr_pass;
  for (const auto& e : seen)
    if (e.first == lo) rlo = e.second;
  int slow = 0;
  int walk = probe_walk ? 3 : 0;   // after a probe-placed pass: step down one d at a time (<= 3)
  while (hi - lo > 1 && !pass_by_breakdown) {
    int mid0 = (lo + hi) / 2;
    if (walk > 0) {
      mid0 = hi - 1;
      --walk;
    } else if (slow < 2 && std::isfinite(rlo) && std::isfinite(rhi) && rlo > rhi && rhi > 0) {
      const double x = lo + (std::log(rlo) - std::log(c->tol)) / (std::log(rlo) - std::log(rhi)) * (hi - lo);
      mid0 = std::min(hi - 1, std::max(lo + 1, (int)std::ceil(x)));
      if (hi - mid0 <= 2) mid0 = hi - 1;   // crossing predicted just below hi: settle it at once
    }
    // a check that fails numerically (non-converged Schur iteration, non-finite projected
    // matrix: ill-conditioned sketched basis) decides nothing: the nearest d inside the
    // bracket with a valid check is used instead (mid, mid+1, mid-1, mid+2, ...)
    int mid = -1;
    double rho, rr = NAN;
    for (int t = 0; t < 8; ++t) {
      const int cand = mid0 + ((t & 1) ? (t + 1) / 2 : -(t / 2));
      if (cand <= lo || cand >= hi) continue;
      if (sylv_sketch_residual(c, cand, &rho, &rr) == SYLV_OK && std::isfinite(rr)) {
        mid = cand;
        break;
      }
    }
    const int width = hi - lo;
    if (mid < 0) {               // no valid check near the middle: keep the old rule
      lo = mid0;
      rlo = NAN;
      continue;
    }
    if (rr < c->tol) {
      hi = mid;
      rhi = rr;
      rr_pass = rr;
      keep_if_pass(mid);
    } else {
      lo = mid;
      rlo = rr;
      walk = 0;
    }
    slow = (walk > 0 || 2 * (hi - lo) > width) ? 0 : slow;
    if (walk == 0 && 2 * (hi - lo) > width) ++slow;
  }
  if (c->y_d != hi) {
    if (best_d == hi && !best_on_dev) {   // restore the kept solution of d* (no re-solve)
      c->Y.swap(best_Y);
      c->y_d = hi;
      c->y_dev = false;
    } else if (best_d == hi && guard(c, [&]() -> sylv_status {
                 const size_t mm = (size_t)hi * c->R * hi * c->R;
                 CK(cudaMemcpyAsync(c->gsolve->C, best_dev.p, mm * sizeof(double), cudaMemcpyDeviceToDevice, c->rst));
                 CK(cudaStreamSynchronize(c->rst));
                 return SYLV_OK;
               }) == SYLV_OK) {
      c->y_d = hi;
      c->y_dev = true;
    } else {
      double rho, rr;
      sylv_sketch_residual(c, hi, &rho, &rr);
    }
  }
  if (d_star) *d_star = hi;
  if (rho_rel) *rho_rel = rr_pass;
  return SYLV_OK;
}

sylv_status sylv_sketch_apply_sketch(sylv_ctx* c, int32_t which, const double* X, int32_t r, double* Yout) {
  if (!c || !X || !Yout || (which != 0 && which != 1)) return SYLV_E_INVALID;
  if (c->method == SYLV_METHOD_TRUNCATED || c->method == SYLV_METHOD_FULL)
    return fail(c, SYLV_E_STATE, "this context has no sketch (method 1 / 2)");
  if (!(r == 1 || r == 2 || r == 4 || r == 8)) return fail(c, SYLV_E_INVALID, "r must be 1, 2, 4 or 8");
  return guard(c, [&]() -> sylv_status {
    Sequence& q = c->seq[which];
    const bool xin = is_device_ptr(X), yout = is_device_ptr(Yout);
    double* Xtmp = dalloc<double>((size_t)c->n * r);
    double* Xs = dalloc<double>((size_t)q.ld * r);
    CK(cudaMemcpyAsync(Xtmp, X, (size_t)c->n * r * sizeof(double), xin ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
    CK(cudaMemsetAsync(Xs, 0, (size_t)q.ld * r * sizeof(double), c->st));
    SYLV_DISPATCH_R(r, { k_to_soa<R_><<<c->sm * 4, 256, 0, c->st>>>(c->n, Xtmp, Xs + q.gz, q.ld); });
    count(c);
    double* Yd = yout ? Yout : dalloc<double>((size_t)c->s * r);
    if (r != c->R) {
      // the sketch kernel's shared memory attribute is set for R = c->R at init
      SYLV_DISPATCH_R(r, {
        CK(cudaFuncSetAttribute(k_sketch_cols<R_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->sk_smem));
      });
    }
    // partials buffer is sized for nchunk x R x s; r <= R fits, larger r needs a temporary
    double* saved = q.skpart;
    double* saved_strips = q.pl_strips;
    if (r > c->R) {
      q.skpart = dalloc<double>((size_t)c->nchunk * c->s * r);
      if (q.pl_list) q.pl_strips = dalloc<double>((size_t)q.sp.zeta * q.pl_wpb * r * kPullS);
    }
    launch_sketch(c, q, Xs + q.gz, r, nullptr, Yd, c->st);
    if (c->comm) c->comm->allreduce(Yd, (size_t)c->s * r, c->st, kChanSetup);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->st));
    if (q.skpart != saved) {
      dfree(q.skpart);
      q.skpart = saved;
    }
    if (q.pl_strips != saved_strips) {
      dfree(q.pl_strips);
      q.pl_strips = saved_strips;
    }
    dfree(Xtmp);
    dfree(Xs);
    if (!yout) {
      CK(cudaMemcpyAsync(Yout, Yd, (size_t)c->s * r * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    }
    CK(cudaStreamSynchronize(c->st));
    if (!yout) dfree(Yd);
    return SYLV_OK;
  });
}

sylv_status sylv_sketch_get_small(sylv_ctx* c, int32_t which, int32_t d, double* H, double* T, double* beta) {
  if (!c || (which != 0 && which != 1)) return SYLV_E_INVALID;
  if (d < 0 || d > c->d_done) return fail(c, SYLV_E_STATE, "get_small(d) needs 0 <= d <= d_done");
  const Sequence& q = c->seq[which];
  const int r = c->R, K = c->K, m = d * r;
  if (H) {
    std::fill(H, H + (size_t)(m + r) * m, 0.0);
    for (int j = 1; j <= d; ++j) {
      const int nwin = std::min(K, j);
      for (int ii = 0; ii <= nwin; ++ii) {
        const int i = (ii < nwin) ? (j - nwin + 1 + ii) : (j + 1);
        const double* h = q.Hh + (size_t)j * (K + 1) * r * r + (size_t)((ii < nwin) ? ii : K) * r * r;
        for (int a = 0; a < r; ++a)
          for (int b = 0; b < r; ++b) H[(size_t)((i - 1) * r + a) * m + (j - 1) * r + b] = h[a * r + b];
      }
    }
  }
  if (T) {
    sylv_status st = guard(c, [&]() -> sylv_status {
      sync_T(c, const_cast<Sequence&>(q), m + r);
      return SYLV_OK;
    });
    if (st != SYLV_OK) return st;
    for (int a = 0; a < m + r; ++a)
      for (int b = 0; b < m + r; ++b) T[(size_t)a * (m + r) + b] = q.Th[(int64_t)b * q.ldT + a];
  }
  if (beta) std::memcpy(beta, q.beta, r * r * sizeof(double));
  return SYLV_OK;
}

sylv_status sylv_sketch_get_block(sylv_ctx* c, int32_t which, int32_t j, double* out) {
  if (!c || !out || (which != 0 && which != 1)) return SYLV_E_INVALID;
  // the ring reflects the last ENQUEUED step (d_dev >= d_done after a halt inside a prefetched batch)
  if (j < 1 || j > c->d_done + 1 || j < c->d_dev + 1 - c->K)
    return fail(c, SYLV_E_STATE, "block j is not in the window");
  return guard(c, [&]() -> sylv_status {
    Sequence& q = c->seq[which];
    const int r = c->R;
    const bool dev = is_device_ptr(out);
    double* od = dev ? out : dalloc<double>((size_t)c->n * r);
    SYLV_DISPATCH_R(r, { k_soa_mul_rowmajor<R_><<<c->sm * 4, 256, 0, c->st>>>(c->n, q.slot(j), q.ld, q.Rall + (int64_t)j * r * r, od); });
    count(c);
    CK(cudaGetLastError());
    if (!dev) CK(cudaMemcpyAsync(out, od, (size_t)c->n * r * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (!dev) dfree(od);
    return SYLV_OK;
  });
}

sylv_status sylv_sketch_history(sylv_ctx* c, int32_t cap, int32_t* d, double* rho_rel, int32_t* cnt) {
  if (!c) return SYLV_E_INVALID;
  const int n = (int)std::min<size_t>(c->hist.size(), (size_t)std::max(0, cap));
  for (int i = 0; i < n; ++i) {
    if (d) d[i] = c->hist[i].first;
    if (rho_rel) rho_rel[i] = c->hist[i].second;
  }
  if (cnt) *cnt = (int32_t)c->hist.size();
  return SYLV_OK;
}

sylv_status sylv_sketch_stats(sylv_ctx* c, sylv_stats* out) {
  if (!c || !out) return SYLV_E_INVALID;
  *out = c->stats;
  return SYLV_OK;
}

void sylv_sketch_reset_stats(sylv_ctx* c) {
  if (!c) return;
  const int64_t l = c->stats.launches, s = c->stats.steps;
  c->stats = sylv_stats{};
  c->stats.launches = l;
  c->stats.steps = s;
}

}  // extern "C"
