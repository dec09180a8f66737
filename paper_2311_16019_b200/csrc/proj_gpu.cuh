// proj_gpu.cuh — GPU projected Sylvester solve for Alg. 1 line 12
// (eq. reduced_sk):  M_U Y + Y M_V^T = E1 beta1 beta2^T E1^T.
//
// M_U = [T_d | T_H] H_und_d T_d^{-1} (R6) is formed on the device from the
// device-resident T (sketch-space QR) and the H coefficients (cuBLAS GEMM + TRSM), and
// likewise M_V.  The equation A Y + Y B = C (A = M_U, B = M_V^T) is solved by the scaled
// Newton iteration for the matrix sign function of the block-triangular matrix
// [[A, -C], [0, -B]]  (H_{k+1} = (mu H_k + H_k^{-1} / mu) / 2, block by block):
//      A_{k+1} = (mu A_k + A_k^{-1} / mu) / 2,     B_{k+1} = (mu B_k + B_k^{-1} / mu) / 2,
//      C_{k+1} = (mu C_k + A_k^{-1} C_k B_k^{-1} / mu) / 2,      Y = C_inf / 2,
// with determinantal scaling mu = |det H_k|^{-1/(2m)} = (|det A_k| |det B_k|)^{-1/(2m)}
// while the relative change exceeds 1e-2, then plain Newton (Roberts 1980; Higham,
// Functions of Matrices, §5.5; Benner, Quintana-Orti, Quintana-Orti 2004).  It converges when spec(A) and spec(-B) are
// separated by the imaginary axis (Re spec(M_U), Re spec(M_V) > 0: the projected
// convection-diffusion operators); the solver reports non-convergence and the caller
// falls back to the host Bartels-Stewart solve.  LU factorisations: cuSOLVER getrf/getrs;
// products: cuBLAS DGEMM (library routines on an O(m^3) dense step that is not the hot
// path).  Every O(m^3) operation stays on the device; only r x m and m x r slices of Y
// come back for the residual (Alg. 1 line 13).
#pragma once
#include <cuComplex.h>
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

namespace sylv {

struct ProjError {
  std::string what;
};

// Dense H_und_d ((m+r) x m, column-major, ld = m + r) from the stored coefficients
// Hc[j] = [h_{j-nwin+1,j} .. h_{j,j}, 0.., h_{j+1,j}] (row-major r x r each), j = 1..d.
__global__ void k_build_hbar(const double* __restrict__ Hc, int d, int r, int K, double* __restrict__ Hb) {
  const int m = d * r, ldh = m + r;
  const int64_t total = (int64_t)ldh * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(e / ldh), row = (int)(e - (int64_t)col * ldh);
    const int j = col / r + 1, c = col % r;          // block column j (1-based)
    const int i = row / r + 1, a = row % r;          // block row i
    const int nwin = j < K ? j : K;
    double v = 0.0;
    if (i == j + 1) {
      v = Hc[(int64_t)j * (K + 1) * r * r + (int64_t)K * r * r + a * r + c];
    } else if (i >= j - nwin + 1 && i <= j) {
      const int ii = i - (j - nwin + 1);
      v = Hc[(int64_t)j * (K + 1) * r * r + (int64_t)ii * r * r + a * r + c];
    }
    Hb[e] = v;
  }
}

__global__ void k_eye(double* __restrict__ X, int m) {
  const int64_t total = (int64_t)m * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    X[e] = (e % (m + 1) == 0) ? 1.0 : 0.0;
}

__global__ void k_add_diag(double* __restrict__ X, int m, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) X[(int64_t)i * (m + 1)] += v;
}

// out[0] = sum_i log|LU_ii|  (one CTA, fixed order)
__global__ void k_logdet(const double* __restrict__ LU, int m, double* __restrict__ out) {
  __shared__ double sm[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) s += log(fabs(LU[(int64_t)i * (m + 1)]));
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sm[0];
}

// ---- eigendecomposition solve (round 2, f1 at c1): complex helpers
// LAPACK real-eigenvector packing -> complex columns: a real eigenvalue j has v_j = VR(:, j); a
// conjugate pair (j, j+1) (pair[j] = 1) has v_j = VR(:, j) + i VR(:, j+1), v_{j+1} = conj(v_j).
__global__ void k_unpack_vr(const double* __restrict__ VR, const int* __restrict__ pair, int m,
                            cuDoubleComplex* __restrict__ V) {
  const int64_t total = (int64_t)m * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(e / m);
    const int p = pair[col];   // 0 real, 1 first of a pair, 2 second of a pair
    double re, im;
    if (p == 0) {
      re = VR[e];
      im = 0.0;
    } else if (p == 1) {
      re = VR[e];
      im = VR[e + m];
    } else {
      re = VR[e - m];
      im = -VR[e];
    }
    V[e] = make_cuDoubleComplex(re, im);
  }
}

__global__ void k_real_to_complex(const double* __restrict__ X, int64_t n, cuDoubleComplex* __restrict__ Z) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    Z[e] = make_cuDoubleComplex(X[e], 0.0);
}

// G[i, j] /= (la_i + lb_j)
__global__ void k_div_eig(cuDoubleComplex* __restrict__ G, int m, const cuDoubleComplex* __restrict__ la,
                          const cuDoubleComplex* __restrict__ lb) {
  const int64_t total = (int64_t)m * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / m);
    const int i = (int)(e - (int64_t)j * m);
    G[e] = cuCdiv(G[e], cuCadd(la[i], lb[j]));
  }
}

__global__ void k_ceye(cuDoubleComplex* __restrict__ X, int m) {
  const int64_t total = (int64_t)m * m;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    X[e] = make_cuDoubleComplex((e % (m + 1) == 0) ? 1.0 : 0.0, 0.0);
}

// Y[e] += Re Z[e]
__global__ void k_add_real(const cuDoubleComplex* __restrict__ Z, int64_t n, double* __restrict__ Y) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    Y[e] += cuCreal(Z[e]);
}

struct GpuSylv {
  cublasHandle_t hb = nullptr;
  cusolverDnHandle_t hs = nullptr;
  // second lane: the B inversion of a Newton step runs concurrently with the A one
  // (cuSOLVER getrf is latency-bound at these sizes)
  cusolverDnHandle_t hs2 = nullptr;
  cudaStream_t st2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double *LU2 = nullptr, *work2 = nullptr;
  int *ipiv2 = nullptr, *info2 = nullptr;
  int cap = 0, capr = 0, lwork = 0;
  int mcap = 1 << 30;            // largest m ever needed ((d_max + 1) r)
  cudaStream_t cur = nullptr;    // stream of the current solve
  int dev = 0;                   // device of the context (the lane-1 thread sets it)
  double *A = nullptr, *B = nullptr, *C = nullptr, *Ai = nullptr, *Bi = nullptr, *W = nullptr, *LU = nullptr;
  double *Hb = nullptr, *work = nullptr, *dlog = nullptr;
  int *ipiv = nullptr, *info = nullptr;
  int iterations = 0;
  bool allow_approx = false;   // accept a converged iteration that ends off the identity
  bool off_identity = false;   // the last accepted solve ended off the identity (approximate)
  int newton_steps = 0, ns_steps = 0;
  double t_build = 0, t_newton = 0, t_ns = 0;   // seconds (SYLV_TRACE_PROJ)

  // eigendecomposition solve (solve_eig): complex eigenvectors, their inverses, work, eigenvalues
  cuDoubleComplex *VA = nullptr, *VB = nullptr, *VAi = nullptr, *VBi = nullptr, *G1 = nullptr, *G2 = nullptr;
  cuDoubleComplex *wA = nullptr, *wB = nullptr;
  int* pairs = nullptr;                  // 2 m packing flags (A then B)
  void* gbuf = nullptr;                  // Xgeev / zgetrf device workspace
  std::vector<char> ghost;               // Xgeev host workspace
  size_t gws = 0;
  cusolverDnParams_t gparams = nullptr;
  int ecap = 0;
  int eig_refine = 0;                    // refinement steps of the last solve_eig
  double eig_res = 0.0;                  // its final relative projected residual
  double t_eig = 0.0, t_refine = 0.0;

  ~GpuSylv() { release(); }
  void free_eig() {
    for (cuDoubleComplex* p : {VA, VB, VAi, VBi, G1, G2, wA, wB})
      if (p) cudaFree(p);
    if (pairs) cudaFree(pairs);
    if (gbuf) cudaFree(gbuf);
    VA = VB = VAi = VBi = G1 = G2 = wA = wB = nullptr;
    pairs = nullptr;
    gbuf = nullptr;
    gws = 0;
    ecap = 0;
  }
  void free_bufs() {
    free_eig();
    for (double* p : {A, B, C, Ai, Bi, W, LU, Hb, work, dlog, LU2, work2})
      if (p) cudaFree(p);
    for (int* p : {ipiv, info, ipiv2, info2})
      if (p) cudaFree(p);
    A = B = C = Ai = Bi = W = LU = Hb = work = dlog = LU2 = work2 = nullptr;
    ipiv = info = ipiv2 = info2 = nullptr;
  }
  void release() {
    if (st2) cudaStreamSynchronize(st2);
    free_bufs();
    cap = 0;
    if (hb) cublasDestroy(hb);
    if (hs) cusolverDnDestroy(hs);
    if (hs2) cusolverDnDestroy(hs2);
    if (gparams) cusolverDnDestroyParams(gparams);
    gparams = nullptr;
    if (st2) cudaStreamDestroy(st2);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    hb = nullptr;
    hs = hs2 = nullptr;
    st2 = nullptr;
    ev_fork = ev_join = nullptr;
  }
  static void ck(cudaError_t e, const char* w) {
    if (e != cudaSuccess) throw ProjError{std::string(w) + ": " + cudaGetErrorString(e)};
  }
  static void ckb(cublasStatus_t e, const char* w) {
    if (e != CUBLAS_STATUS_SUCCESS) throw ProjError{std::string(w) + ": cublas status " + std::to_string((int)e)};
  }
  static void cks(cusolverStatus_t e, const char* w) {
    if (e != CUSOLVER_STATUS_SUCCESS) throw ProjError{std::string(w) + ": cusolver status " + std::to_string((int)e)};
  }

  void ensure(int m, int r, cudaStream_t st) {
    cur = st;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    if (!hb) {
      ckb(cublasCreate(&hb), "cublasCreate");
      cks(cusolverDnCreate(&hs), "cusolverDnCreate");
      cks(cusolverDnCreate(&hs2), "cusolverDnCreate");
      ck(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking), "cudaStreamCreate");
      ck(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "cudaEventCreate");
      ck(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "cudaEventCreate");
      cks(cusolverDnSetStream(hs2, st2), "cusolverDnSetStream");
    }
    ckb(cublasSetStream(hb, st), "cublasSetStream");
    cks(cusolverDnSetStream(hs, st), "cusolverDnSetStream");
    if (m <= cap && r <= capr) return;
    if (m > cap) m = std::max(m, std::min(mcap, cap + cap / 2));   // grow geometrically (<= mcap)
    ck(cudaStreamSynchronize(st), "sync");
    free_bufs();
    const size_t mm = (size_t)m * m;
    for (double** p : {&A, &B, &C, &Ai, &Bi, &W, &LU, &LU2}) ck(cudaMalloc(p, mm * sizeof(double)), "cudaMalloc (proj)");
    ck(cudaMalloc(&Hb, (size_t)(m + r) * m * sizeof(double)), "cudaMalloc (proj)");
    ck(cudaMalloc(&dlog, 2 * sizeof(double)), "cudaMalloc (proj)");
    for (int** p : {&ipiv, &ipiv2}) ck(cudaMalloc(p, (size_t)m * sizeof(int)), "cudaMalloc (proj)");
    for (int** p : {&info, &info2}) ck(cudaMalloc(p, sizeof(int)), "cudaMalloc (proj)");
    cks(cusolverDnDgetrf_bufferSize(hs, m, m, LU, m, &lwork), "getrf_bufferSize");
    ck(cudaMalloc(&work, (size_t)std::max(lwork, 1) * sizeof(double)), "cudaMalloc (proj)");
    ck(cudaMalloc(&work2, (size_t)std::max(lwork, 1) * sizeof(double)), "cudaMalloc (proj)");
    cap = m;
    capr = r;
  }

  // out = [T_d | T_H] H_und_d T_d^{-1} (m x m, column-major): T (ldT, device), Hc (device)
  void build_M(const double* T, int64_t ldT, const double* Hc, int d, int r, int K, double* out, cudaStream_t st) {
    const int m = d * r;
    const int64_t tot = (int64_t)(m + r) * m;
    k_build_hbar<<<(int)std::min<int64_t>(4096, (tot + 255) / 256), 256, 0, st>>>(Hc, d, r, K, Hb);
    ck(cudaGetLastError(), "k_build_hbar");
    const double one = 1.0, zero = 0.0;
    ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m + r, &one, T, (int)ldT, Hb, m + r, &zero, out, m),
        "dgemm (T Hbar)");
    ckb(cublasDtrsm(hb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, m, &one, T,
                    (int)ldT, out, m),
        "dtrsm (X T_d^-1)");
  }

  // X (m x m, in/out of `src`) -> Xinv; returns log|det X|
  // Enqueue X -> X^{-1} (LU) on lane 0 (st, hs) or lane 1 (st2, hs2); log|det X| -> dlog[lane]
  void invert_async(const double* src, double* dst, int m, int lane, cudaStream_t st) {
    cudaStream_t s = lane ? st2 : st;
    cusolverDnHandle_t h = lane ? hs2 : hs;
    double* lu = lane ? LU2 : LU;
    ck(cudaMemcpyAsync(lu, src, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy (LU)");
    cks(cusolverDnDgetrf(h, m, m, lu, m, lane ? work2 : work, lane ? ipiv2 : ipiv, lane ? info2 : info), "getrf");
    k_logdet<<<1, 256, 0, s>>>(lu, m, dlog + lane);
    k_eye<<<(int)std::min<int64_t>(4096, ((int64_t)m * m + 255) / 256), 256, 0, s>>>(dst, m);
    cks(cusolverDnDgetrs(h, CUBLAS_OP_N, m, m, lu, m, lane ? ipiv2 : ipiv, dst, m, lane ? info2 : info), "getrs");
  }

  // A^{-1} and B^{-1} concurrently; returns log|det A|, log|det B|
  void invert_pair(const double* Am, double* Ainv, const double* Bm, double* Binv, int m, cudaStream_t st,
                   double* la, double* lb) {
    ck(cudaEventRecord(ev_fork, st), "event");
    ck(cudaStreamWaitEvent(st2, ev_fork, 0), "event");
    invert_async(Am, Ainv, m, 0, st);
    invert_async(Bm, Binv, m, 1, st);
    ck(cudaEventRecord(ev_join, st2), "event");
    ck(cudaStreamWaitEvent(st, ev_join, 0), "event");
    double ld[2] = {0.0, 0.0};
    int inf[2] = {0, 0};
    ck(cudaMemcpyAsync(ld, dlog, 2 * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaMemcpyAsync(&inf[0], info, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaMemcpyAsync(&inf[1], info2, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    if (inf[0] != 0 || inf[1] != 0 || !std::isfinite(ld[0]) || !std::isfinite(ld[1]))
      throw ProjError{"singular projected matrix"};
    *la = ld[0];
    *lb = ld[1];
  }

  // the sign iteration must end at A = B = I (sign of matrices with spectra in Re > 0)
  bool near_identity(const double* X, int m, cudaStream_t st) {
    ck(cudaMemcpyAsync(LU, X, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy");
    k_add_diag<<<(m + 255) / 256, 256, 0, st>>>(LU, m, -1.0);
    return fro(LU, (int64_t)m * m) <= 1e-8 * std::sqrt((double)m);
  }

  double fro(const double* X, int64_t n) {
    double v = 0.0;
    ckb(cublasDnrm2(hb, (int)n, X, 1, &v), "dnrm2");
    return v;
  }

  // Solve M_U Y + Y M_V^T = C0 (C0 nonzero only in its leading r x r block: Bm, row-major).
  // On success Y (= C/2) is left in `C`; returns false if the iteration did not converge.
  bool solve(const double* TU, const double* HcU, const double* TV, const double* HcV, int64_t ldT, int d, int r,
             int K, const double* Bm, cudaStream_t st) {
    if (solve_once(TU, HcU, TV, HcV, ldT, d, r, K, Bm, st, true)) return true;
    return solve_once(TU, HcU, TV, HcV, ldT, d, r, K, Bm, st, false);   // pure Newton retry
  }

  // ||X^2 - I||_F / sqrt(m) (Newton-Schulz converges when this is < 1)
  double sq_dev(const double* X, int m) {
    const double one = 1.0, zero = 0.0;
    ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, X, m, X, m, &zero, LU, m), "dgemm (X^2)");
    k_add_diag<<<(m + 255) / 256, 256, 0, cur>>>(LU, m, -1.0);
    return fro(LU, (int64_t)m * m) / std::sqrt((double)m);
  }

  bool solve_once(const double* TU, const double* HcU, const double* TV, const double* HcV, int64_t ldT, int d, int r,
                  int K, const double* Bm, cudaStream_t st, bool allow_ns) {
    const bool trace = std::getenv("SYLV_TRACE_PROJ") != nullptr;
    auto now = [&]() {
      if (trace) cudaStreamSynchronize(st);
      return std::chrono::steady_clock::now();
    };
    auto t0 = now();
    newton_steps = ns_steps = 0;
    const int m = d * r;
    ensure(m, r, st);
    build_M(TU, ldT, HcU, d, r, K, A, st);
    build_M(TV, ldT, HcV, d, r, K, W, st);
    const double one = 1.0, zero = 0.0;
    ckb(cublasDgeam(hb, CUBLAS_OP_T, CUBLAS_OP_N, m, m, &one, W, m, &zero, W, m, B, m), "geam (M_V^T)");
    ck(cudaMemsetAsync(C, 0, (size_t)m * m * sizeof(double), st), "memset");
    std::vector<double> cb((size_t)r * r);
    for (int a = 0; a < r; ++a)
      for (int b = 0; b < r; ++b) cb[(size_t)b * r + a] = Bm[a * r + b];   // column-major r x r
    ck(cudaMemcpy2DAsync(C, (size_t)m * sizeof(double), cb.data(), (size_t)r * sizeof(double),
                         (size_t)r * sizeof(double), r, cudaMemcpyHostToDevice, st),
       "H2D (rhs)");
    const int64_t mm = (int64_t)m * m;
    auto t1 = now();
    t_build = std::chrono::duration<double>(t1 - t0).count();
    t_newton = t_ns = 0.0;
    const double mone = -1.0, half = 0.5, c15 = 1.5, cm05 = -0.5;
    bool scale = true, last = false, ns = false;
    for (iterations = 1; iterations <= 60; ++iterations) {
      double dA, nA, dB, nB;
      auto ti = now();
      if (!ns) ++newton_steps; else ++ns_steps;
      if (!ns) {
        // scaled Newton step (needs A^{-1}, B^{-1}: LU)
        double la = 0.0, lb = 0.0;
        invert_pair(A, Ai, B, Bi, m, st, &la, &lb);
        const double mu = scale ? std::exp(-(la + lb) / (2.0 * m)) : 1.0;
        const double a1 = 0.5 / mu, b1 = 0.5 * mu;
        // C <- (mu C + Ai C Bi / mu) / 2
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, Ai, m, C, m, &zero, W, m), "dgemm (Ai C)");
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &a1, W, m, Bi, m, &b1, C, m), "dgemm (Ai C Bi)");
        // A <- (mu A + Ai / mu) / 2, B likewise (W = new, old - new kept for the change)
        ckb(cublasDgeam(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, &b1, A, m, &a1, Ai, m, W, m), "geam (A)");
        ckb(cublasDaxpy(hb, (int)mm, &mone, W, 1, A, 1), "daxpy");
        dA = fro(A, mm);
        nA = fro(W, mm);
        std::swap(A, W);
        ckb(cublasDgeam(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, &b1, B, m, &a1, Bi, m, W, m), "geam (B)");
        ckb(cublasDaxpy(hb, (int)mm, &mone, W, 1, B, 1), "daxpy");
        dB = fro(B, mm);
        nB = fro(W, mm);
        std::swap(B, W);
      } else {
        // Newton-Schulz step, inverse-free (valid once ||I - H^2|| < 1): H <- H (3I - H^2) / 2,
        //   C <- (3C - C B^2 - A^2 C + A (C B)) / 2,  A <- (3A - A^3) / 2,  B <- (3B - B^3) / 2
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, A, m, A, m, &zero, Ai, m), "dgemm (A^2)");
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, B, m, B, m, &zero, Bi, m), "dgemm (B^2)");
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, C, m, B, m, &zero, W, m), "dgemm (C B)");
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, A, m, W, m, &zero, LU, m), "dgemm (A C B)");
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &mone, C, m, Bi, m, &one, LU, m), "dgemm (C B^2)");
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &mone, Ai, m, C, m, &one, LU, m), "dgemm (A^2 C)");
        ckb(cublasDgeam(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, &c15, C, m, &half, LU, m, W, m), "geam (C)");
        std::swap(C, W);
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, A, m, Ai, m, &zero, LU, m), "dgemm (A^3)");
        ckb(cublasDgeam(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, &c15, A, m, &cm05, LU, m, W, m), "geam (A)");
        ckb(cublasDaxpy(hb, (int)mm, &mone, W, 1, A, 1), "daxpy");
        dA = fro(A, mm);
        nA = fro(W, mm);
        std::swap(A, W);
        ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, B, m, Bi, m, &zero, LU, m), "dgemm (B^3)");
        ckb(cublasDgeam(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, &c15, B, m, &cm05, LU, m, W, m), "geam (B)");
        ckb(cublasDaxpy(hb, (int)mm, &mone, W, 1, B, 1), "daxpy");
        dB = fro(B, mm);
        nB = fro(W, mm);
        std::swap(B, W);
      }
      const double rel = std::max(dA / nA, dB / nB);
      {
        const double dt = std::chrono::duration<double>(now() - ti).count();
        if (ns_steps && newton_steps + ns_steps > 0 && ns) t_ns += dt; else t_newton += dt;
      }
      if (!std::isfinite(rel)) {
        if (trace) std::fprintf(stderr, "[proj] m=%d non-finite step after %d iterations\n", m, iterations);
        return false;
      }
      if (rel < 1e-2) scale = false;                      // quadratic phase: unscaled
      if (last || rel < 1e-14) {                          // one step after rel < 1e-7: error ~ rel^2
        off_identity = false;
        if (!near_identity(A, m, st) || !near_identity(B, m, st)) {          // wrong fixed point
          if (trace) std::fprintf(stderr, "[proj] m=%d identity check failed after %d iterations\n", m, iterations);
          if (!allow_approx && !std::getenv("SYLV_PROJ_ACCEPT")) return false;   // (development switch)
          off_identity = true;          // approximate: the caller decides whether it may be used
        }
        ckb(cublasDscal(hb, (int)mm, &half, C, 1), "dscal (Y = C/2)");
        if (trace)
          std::fprintf(stderr, "[proj] m=%d build %.1f ms, %d Newton %.1f ms, %d NS %.1f ms\n", m, 1e3 * t_build,
                       newton_steps, 1e3 * t_newton, ns_steps, 1e3 * t_ns);
        return true;
      }
      if (rel < 1e-7) last = true;
      // Newton-Schulz once inside its basin: ||A^2 - I||, ||B^2 - I|| well below 1 (checked,
      // not inferred from the step size: the projected matrices can be far from normal)
      if (allow_ns && !ns && rel < 5e-2 && sq_dev(A, m) < 0.3 && sq_dev(B, m) < 0.3) ns = true;
    }
    if (trace) std::fprintf(stderr, "[proj] m=%d no convergence in 60 iterations (rel step history above)\n", m);
    return false;
  }

  // ---- f1 (round 2): eigendecomposition solve with iterative refinement, for projected
  // equations the sign iteration cannot solve (c1: M_V has eigenvalues with Re < 0, so
  // sign(M_V) != I).  With A = V_A diag(la) V_A^{-1}, B = V_B diag(lb) V_B^{-1}
  // (cuSOLVER Xgeev, complex right eigenvectors), A Y + Y B = R is solved by
  //   Y = V_A [ (V_A^{-1} R V_B) ./ (la_i + lb_j) ] V_B^{-1}      (apply(R), 4 ZGEMMs),
  // then refined: Y += apply(C - A Y - Y B) until the projected residual is at rounding level,
  // ||C - A Y - Y B||_F <= 1e-12 (||A||_F + ||B||_F) ||Y||_F — the backward error of a
  // backward-stable (Bartels-Stewart) solve — else the caller falls back to the host.  The
  // accuracy of the first apply depends on kappa(V_A) kappa(V_B); the refinement converges
  // while that times the unit roundoff is well below 1, and the residual test certifies it.
  void ensure_eig(int m) {
    if (m <= ecap) return;
    ck(cudaStreamSynchronize(cur), "sync");
    free_eig();
    const size_t mm = (size_t)cap * cap;             // sized like the real buffers (cap >= m)
    for (cuDoubleComplex** p : {&VA, &VB, &VAi, &VBi, &G1, &G2})
      ck(cudaMalloc(p, mm * sizeof(cuDoubleComplex)), "cudaMalloc (eig)");
    ck(cudaMalloc(&wA, (size_t)cap * sizeof(cuDoubleComplex)), "cudaMalloc (eig)");
    ck(cudaMalloc(&wB, (size_t)cap * sizeof(cuDoubleComplex)), "cudaMalloc (eig)");
    ck(cudaMalloc(&pairs, 2 * (size_t)cap * sizeof(int)), "cudaMalloc (eig)");
    if (!gparams) cks(cusolverDnCreateParams(&gparams), "cusolverDnCreateParams");
    size_t wd = 0, wh = 0;
    cks(cusolverDnXgeev_bufferSize(hs, gparams, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, cap, CUDA_R_64F,
                                   LU, cap, CUDA_C_64F, wA, CUDA_R_64F, nullptr, cap, CUDA_R_64F, Ai, cap, CUDA_R_64F,
                                   &wd, &wh),
        "Xgeev_bufferSize");
    int lw = 0;
    cks(cusolverDnZgetrf_bufferSize(hs, cap, cap, G1, cap, &lw), "zgetrf_bufferSize");
    gws = 2 * std::max(wd, (size_t)lw * sizeof(cuDoubleComplex));   // margin: queries at m <= cap
    ck(cudaMalloc(&gbuf, gws + 16), "cudaMalloc (eig)");
    ghost.assign(wh + 16, 0);
    ecap = cap;
  }

  // eigenvalues w, complex right eigenvectors V and Vi = V^{-1} of the real m x m matrix X (X is
  // copied; VR in Ai, the LU of V in G1) on the solve's stream
  void eig_inv(const double* X, int m, cuDoubleComplex* w, cuDoubleComplex* V, cuDoubleComplex* Vi, int* pair_dev) {
    cusolverDnHandle_t h = hs;
    cudaStream_t s = cur;
    double* in = LU;
    double* vr = Ai;
    void* gb = gbuf;
    std::vector<char>& gh = ghost;
    int* inf_d = info;
    int* piv = ipiv;
    cuDoubleComplex* lu = G1;
    ck(cudaMemcpyAsync(in, X, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy (geev)");
    size_t wd = 0, wh = 0;
    cks(cusolverDnXgeev_bufferSize(h, gparams, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, m, CUDA_R_64F,
                                   in, m, CUDA_C_64F, w, CUDA_R_64F, nullptr, m, CUDA_R_64F, vr, m, CUDA_R_64F, &wd,
                                   &wh),
        "Xgeev_bufferSize");
    if (wd > gws) throw ProjError{"Xgeev device workspace grew (" + std::to_string(wd) + " > " + std::to_string(gws) + ")"};
    if (wh + 16 > gh.size()) gh.assign(wh + 16, 0);
    cks(cusolverDnXgeev(h, gparams, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, m, CUDA_R_64F, in, m,
                        CUDA_C_64F, w, CUDA_R_64F, nullptr, m, CUDA_R_64F, vr, m, CUDA_R_64F, gb, gws, gh.data(), wh,
                        inf_d),
        "Xgeev");
    int inf = 0;
    std::vector<cuDoubleComplex> wh_((size_t)m);
    ck(cudaMemcpyAsync(&inf, inf_d, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaMemcpyAsync(wh_.data(), w, (size_t)m * sizeof(cuDoubleComplex), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    if (inf != 0) throw ProjError{"Xgeev info " + std::to_string(inf)};
    std::vector<int> pr((size_t)m, 0);
    for (int j = 0; j < m; ++j) {
      if (!std::isfinite(cuCreal(wh_[j])) || !std::isfinite(cuCimag(wh_[j]))) throw ProjError{"Xgeev: non-finite eigenvalue"};
      if (pr[j] == 0 && cuCimag(wh_[j]) != 0.0) {
        if (j + 1 >= m) throw ProjError{"Xgeev: unpaired complex eigenvalue"};
        pr[j] = 1;
        pr[j + 1] = 2;
      }
    }
    ck(cudaMemcpyAsync(pair_dev, pr.data(), (size_t)m * sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
    const int64_t mm = (int64_t)m * m;
    const int g = (int)std::min<int64_t>(4096, (mm + 255) / 256);
    k_unpack_vr<<<g, 256, 0, s>>>(vr, pair_dev, m, V);
    ck(cudaGetLastError(), "k_unpack_vr");
    // Vi = V^{-1}: complex LU, then solves against the identity
    ck(cudaMemcpyAsync(lu, V, (size_t)mm * sizeof(cuDoubleComplex), cudaMemcpyDeviceToDevice, s), "copy");
    cks(cusolverDnZgetrf(h, m, m, lu, m, reinterpret_cast<cuDoubleComplex*>(gb), piv, inf_d), "zgetrf");
    k_ceye<<<g, 256, 0, s>>>(Vi, m);
    cks(cusolverDnZgetrs(h, CUBLAS_OP_N, m, m, lu, m, piv, Vi, m, inf_d), "zgetrs");
    ck(cudaMemcpyAsync(&inf, inf_d, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");   // also: pr (host) was read by the async copy
    if (inf != 0) throw ProjError{"singular eigenvector matrix"};
  }

  // Y += Re(V_A [(V_A^{-1} R V_B) ./ (la_i + lb_j)] V_B^{-1})
  void eig_apply(const double* Rr, double* Y, int m) {
    const int64_t mm = (int64_t)m * m;
    const int g = (int)std::min<int64_t>(4096, (mm + 255) / 256);
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
    k_real_to_complex<<<g, 256, 0, cur>>>(Rr, mm, G2);
    ckb(cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, VAi, m, G2, m, &zero, G1, m), "zgemm (VA^-1 R)");
    ckb(cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, G1, m, VB, m, &zero, G2, m), "zgemm (. VB)");
    k_div_eig<<<g, 256, 0, cur>>>(G2, m, wA, wB);
    ckb(cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, VA, m, G2, m, &zero, G1, m), "zgemm (VA .)");
    ckb(cublasZgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, G1, m, VBi, m, &zero, G2, m), "zgemm (. VB^-1)");
    k_add_real<<<g, 256, 0, cur>>>(G2, mm, Y);
    ck(cudaGetLastError(), "eig_apply");
  }

  // Solve M_U Y + Y M_V^T = E1 Bm E1^T; Y left in C.  false: not certified (caller: host).
  bool solve_eig(const double* TU, const double* HcU, const double* TV, const double* HcV, int64_t ldT, int d, int r,
                 int K, const double* Bm, cudaStream_t st) {
    const bool trace = std::getenv("SYLV_TRACE_PROJ") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    const int m = d * r;
    ensure(m, r, st);
    ensure_eig(m);
    build_M(TU, ldT, HcU, d, r, K, A, st);
    build_M(TV, ldT, HcV, d, r, K, W, st);
    const double one = 1.0, zero = 0.0, mone = -1.0;
    ckb(cublasDgeam(hb, CUBLAS_OP_T, CUBLAS_OP_N, m, m, &one, W, m, &zero, W, m, B, m), "geam (M_V^T)");
    const int64_t mm = (int64_t)m * m;
    // right-hand side F (in Bi: kept for the residuals)
    ck(cudaMemsetAsync(Bi, 0, (size_t)mm * sizeof(double), st), "memset");
    std::vector<double> cb((size_t)r * r);
    for (int a = 0; a < r; ++a)
      for (int b = 0; b < r; ++b) cb[(size_t)b * r + a] = Bm[a * r + b];
    ck(cudaMemcpy2DAsync(Bi, (size_t)m * sizeof(double), cb.data(), (size_t)r * sizeof(double),
                         (size_t)r * sizeof(double), r, cudaMemcpyHostToDevice, st),
       "H2D (rhs)");
    // A = M_U and B = M_V^T in turn on the context's stream: two concurrent Xgeev calls (two
    // handles, two host threads) failed intermittently with CUSOLVER_STATUS_INTERNAL_ERROR on
    // B200 (c1, m = 2000), so the halves are serial
    eig_inv(A, m, wA, VA, VAi, pairs);
    eig_inv(B, m, wB, VB, VBi, pairs + m);
    auto t1 = std::chrono::steady_clock::now();
    t_eig = std::chrono::duration<double>(t1 - t0).count();
    const double nA = fro(A, mm), nB = fro(B, mm), nF = fro(Bi, mm);
    ck(cudaMemsetAsync(C, 0, (size_t)mm * sizeof(double), st), "memset");
    eig_apply(Bi, C, m);
    double prev = INFINITY;
    bool okc = false;
    for (eig_refine = 0; eig_refine < 8; ++eig_refine) {
      // W = F - A Y - Y B
      ck(cudaMemcpyAsync(W, Bi, (size_t)mm * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy");
      ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &mone, A, m, C, m, &one, W, m), "dgemm (A Y)");
      ckb(cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &mone, C, m, B, m, &one, W, m), "dgemm (Y B)");
      const double rn = fro(W, mm), yn = fro(C, mm);
      eig_res = rn / nF;
      if (!std::isfinite(rn) || !std::isfinite(yn)) break;
      if (rn <= 1e-12 * (nA + nB) * yn) {
        okc = true;
        break;
      }
      if (eig_refine >= 2 && rn > 0.5 * prev) break;   // stagnated: not certified
      prev = rn;
      eig_apply(W, C, m);
    }
    t_refine = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    if (trace)
      std::fprintf(stderr, "[proj] m=%d eig %.1f ms, %d refinements %.1f ms, residual %.2e (%s)\n", m, 1e3 * t_eig,
                   eig_refine, 1e3 * t_refine, eig_res, okc ? "certified" : "rejected");
    return okc;
  }
};

}  // namespace sylv
