// full_arnoldi.cuh — kernels of the comparison methods:
//   * Alg. 2, truncated Arnoldi without a sketch: the n-space passes of
//     nspace.cuh / stencil25d.cuh unchanged, no sketch, T = I;
//   * the full Arnoldi (Galerkin) method: every basis block retained and
//     orthonormalised against ALL previous blocks by block CGS2 (two sweeps over the basis:
//     the tall-skinny Q^T w / Q c kernels of sspace.cuh with the n-space basis as Q), then
//     CholQR2 — the O(d^2) orthogonalisation cost the paper's truncation removes.
// Layout: the retained basis lives in the context's ring, one SoA block per step (ring of
// d_max + 1 slots, no wrap); U_j is stored normalised (R_j = I).
#pragma once
#include "nspace.cuh"

namespace sylv {

// out[row*R + c] = (A Z)[row, c] for an SoA block Z (ghost rows zero / halo), row-major output.
template <int R>
__global__ void __launch_bounds__(kThreads) k_apply_rowmajor(OpParams op, const double* __restrict__ Z, int64_t ld,
                                                             double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < op.n; row += stride) {
    if (op.kind == kCSR) {
#pragma unroll
      for (int c = 0; c < R; ++c) out[row * R + c] = csr_col(op, Z + c * ld, row);
    } else {
      const Coord q = coords(op, (uint32_t)row);
#pragma unroll
      for (int c = 0; c < R; ++c) {
        double center;
        out[row * R + c] = stencil_col(op, Z + c * ld, (uint32_t)row, q, center);
      }
    }
  }
}

// X (SoA, R columns of stride ld) := X M in place, M R x R row-major.
template <int R>
__global__ void __launch_bounds__(kThreads) k_soa_rmul_inplace(int64_t n, double* __restrict__ X, int64_t ld,
                                                               const double* __restrict__ M) {
  __shared__ double ms[R * R];
  if (threadIdx.x < R * R) ms[threadIdx.x] = M[threadIdx.x];
  __syncthreads();
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < n; row += (int64_t)gridDim.x * kThreads) {
    double x[R];
#pragma unroll
    for (int a = 0; a < R; ++a) x[a] = X[a * ld + row];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < R; ++a) s = fma(x[a], ms[a * R + c], s);
      X[c * ld + row] = s;
    }
  }
}

// Full method, step j: H column from the CGS2 coefficients csum (m = jR rows, row-major m x R:
// h_{i,j}[a][c] = csum[((i-1)R + a) R + c]) and h_{j+1,j} = tau; R_{j+1} = I (normalised
// storage); breakdown flag (bit 0, R11) when min diag tau <= 1e-14 ||W~||_F with
// ||W~||_F^2 = ||tau||_F^2 + ||csum||_F^2 (orthonormal basis).  One CTA.
template <int R>
__global__ void k_full_hcol(const double* __restrict__ csum, const double* __restrict__ tau, int m, int j, int K,
                            double* __restrict__ Hc, double* __restrict__ Rall, int* __restrict__ flags) {
  __shared__ double red[kSmallThreads];
  double* Hj = Hc + (int64_t)j * (K + 1) * R * R;
  double acc = 0.0;
  for (int e = threadIdx.x; e < m * R; e += blockDim.x) {
    const int row = e / R, c = e % R;
    const int i = row / R, a = row % R;               // block i (0-based), row a
    const double v = csum[e];
    Hj[(int64_t)i * R * R + a * R + c] = v;
    acc += v * v;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) s += red[t];   // fixed order
    double tn = 0.0, mind = 1e300;
    for (int e = 0; e < R * R; ++e) {
      Hj[(int64_t)K * R * R + e] = tau[e];
      tn += tau[e] * tau[e];
    }
    for (int a = 0; a < R; ++a) mind = fmin(mind, tau[a * R + a]);
    for (int e = 0; e < R * R; ++e) Rall[(int64_t)(j + 1) * R * R + e] = (e / R == e % R) ? 1.0 : 0.0;
    if (mind <= 1e-14 * sqrt(tn + s)) atomicOr(flags + j, 1);
  }
}

// T := I (ldT x ldT, column-major): methods without a sketch (Alg. 2, full) use the unwhitened
// projected matrices, i.e. the whitening factor is the identity.
__global__ void k_set_identity(double* __restrict__ T, int64_t ldT) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ldT * ldT;
       e += (int64_t)gridDim.x * blockDim.x)
    T[e] = (e / ldT == e % ldT) ? 1.0 : 0.0;
}

}  // namespace sylv
