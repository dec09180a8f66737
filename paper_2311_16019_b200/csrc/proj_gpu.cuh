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
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cmath>
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

struct GpuSylv {
  cublasHandle_t hb = nullptr;
  cusolverDnHandle_t hs = nullptr;
  int cap = 0, capr = 0, lwork = 0;
  int mcap = 1 << 30;            // largest m ever needed ((d_max + 1) r)
  cudaStream_t cur = nullptr;    // stream of the current solve
  double *A = nullptr, *B = nullptr, *C = nullptr, *Ai = nullptr, *Bi = nullptr, *W = nullptr, *LU = nullptr;
  double *Hb = nullptr, *work = nullptr, *dlog = nullptr;
  int *ipiv = nullptr, *info = nullptr;
  int iterations = 0;

  ~GpuSylv() { release(); }
  void release() {
    for (double* p : {A, B, C, Ai, Bi, W, LU, Hb, work, dlog})
      if (p) cudaFree(p);
    if (ipiv) cudaFree(ipiv);
    if (info) cudaFree(info);
    A = B = C = Ai = Bi = W = LU = Hb = work = dlog = nullptr;
    ipiv = info = nullptr;
    cap = 0;
    if (hb) cublasDestroy(hb);
    if (hs) cusolverDnDestroy(hs);
    hb = nullptr;
    hs = nullptr;
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
    if (!hb) {
      ckb(cublasCreate(&hb), "cublasCreate");
      cks(cusolverDnCreate(&hs), "cusolverDnCreate");
    }
    ckb(cublasSetStream(hb, st), "cublasSetStream");
    cks(cusolverDnSetStream(hs, st), "cusolverDnSetStream");
    if (m <= cap && r <= capr) return;
    if (m > cap) m = std::max(m, std::min(mcap, cap + cap / 2));   // grow geometrically (<= mcap)
    for (double* p : {A, B, C, Ai, Bi, W, LU, Hb, work, dlog})
      if (p) cudaFree(p);
    if (ipiv) cudaFree(ipiv);
    if (info) cudaFree(info);
    const size_t mm = (size_t)m * m;
    for (double** p : {&A, &B, &C, &Ai, &Bi, &W, &LU}) ck(cudaMalloc(p, mm * sizeof(double)), "cudaMalloc (proj)");
    ck(cudaMalloc(&Hb, (size_t)(m + r) * m * sizeof(double)), "cudaMalloc (proj)");
    ck(cudaMalloc(&dlog, 2 * sizeof(double)), "cudaMalloc (proj)");
    ck(cudaMalloc(&ipiv, (size_t)m * sizeof(int)), "cudaMalloc (proj)");
    ck(cudaMalloc(&info, sizeof(int)), "cudaMalloc (proj)");
    cks(cusolverDnDgetrf_bufferSize(hs, m, m, LU, m, &lwork), "getrf_bufferSize");
    ck(cudaMalloc(&work, (size_t)std::max(lwork, 1) * sizeof(double)), "cudaMalloc (proj)");
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
  double invert(const double* src, double* dst, int m, cudaStream_t st) {
    ck(cudaMemcpyAsync(LU, src, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy (LU)");
    cks(cusolverDnDgetrf(hs, m, m, LU, m, work, ipiv, info), "getrf");
    k_logdet<<<1, 256, 0, st>>>(LU, m, dlog);
    k_eye<<<(int)std::min<int64_t>(4096, ((int64_t)m * m + 255) / 256), 256, 0, st>>>(dst, m);
    cks(cusolverDnDgetrs(hs, CUBLAS_OP_N, m, m, LU, m, ipiv, dst, m, info), "getrs");
    double ld = 0.0;
    int inf = 0;
    ck(cudaMemcpyAsync(&ld, dlog, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaMemcpyAsync(&inf, info, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    if (inf != 0 || !std::isfinite(ld)) throw ProjError{"singular projected matrix"};
    return ld;
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
    const double mone = -1.0, half = 0.5, c15 = 1.5, cm05 = -0.5;
    bool scale = true, last = false, ns = false;
    for (iterations = 1; iterations <= 60; ++iterations) {
      double dA, nA, dB, nB;
      if (!ns) {
        // scaled Newton step (needs A^{-1}, B^{-1}: LU)
        const double la = invert(A, Ai, m, st);
        const double lb = invert(B, Bi, m, st);
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
      if (!std::isfinite(rel)) return false;
      if (rel < 1e-2) scale = false;                      // quadratic phase: unscaled
      if (last || rel < 1e-14) {                          // one step after rel < 1e-7: error ~ rel^2
        if (!near_identity(A, m, st) || !near_identity(B, m, st)) return false;   // wrong fixed point
        ckb(cublasDscal(hb, (int)mm, &half, C, 1), "dscal (Y = C/2)");
        return true;
      }
      if (rel < 1e-7) last = true;
      // Newton-Schulz once inside its basin: ||A^2 - I||, ||B^2 - I|| well below 1 (checked,
      // not inferred from the step size: the projected matrices can be far from normal)
      if (allow_ns && !ns && rel < 5e-2 && sq_dev(A, m) < 0.3 && sq_dev(B, m) < 0.3) ns = true;
    }
    return false;
  }
};

}  // namespace sylv
