// sketched_gs.cuh — f3: the sketched inner product inside the truncated
// Gram-Schmidt, "avoiding any inner product in R^n".
//
// Per block step j of one sequence (blocks stored unnormalised, U_i = Z_i R_i, as in nspace.cuh):
//   Yt  = A Z_j                                   (n-space, k_apply_soa)
//   Ys  = S Yt                                    (the hashed sketch of the matvec)
//   P_i = (S Z_i)^T Ys  for the window i          (s-space, k_skpass1) -> k_coef1:
//         h_{i,j} = R_i^T P_i R_j = (S U_i)^T (S W~),  K_i = R_i h_{i,j}
//   Z_{j+1} = W' = Yt R_j - sum_i Z_i K_i          (n-space, the pass-2 kernel without Gram)
//   S Z_{j+1} = Ys R_j - sum_i (S Z_i) K_i        (s-space, k_skpass2; S is linear) and its Gram
//         -> k_coef2: h_{j+1,j} = chol((S W')^T (S W')), R_{j+1} = h^{-1}  (S-normalisation)
//   w = S U_{j+1} = (S Z_{j+1}) R_{j+1}           -> the sketched QR update (a5), unchanged.
// The only reductions over n are gone: the coefficients come from s x R sketches (on several
// ranks: one allreduce of Ys, S being linear in rows; no allreduce of inner products).
#pragma once
#include "nspace.cuh"

namespace sylv {

// Yt (SoA, R columns of stride ld) = A Z (SoA).
template <int R>
__global__ void __launch_bounds__(kThreads) k_apply_soa(OpParams op, const double* __restrict__ Z, int64_t ld,
                                                        double* __restrict__ Yt) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < op.n; row += stride) {
    if (op.kind == kCSR) {
#pragma unroll
      for (int c = 0; c < R; ++c) Yt[c * ld + row] = csr_col(op, Z + c * ld, row);
    } else {
      const Coord q = coords(op, (uint32_t)row);
#pragma unroll
      for (int c = 0; c < R; ++c) {
        double center;
        Yt[c * ld + row] = stencil_col(op, Z + c * ld, (uint32_t)row, q, center);
      }
    }
  }
}

// partial[blk * (K R R) + (i R + a) R + c] = sum_{rows of blk} zs_i[row, a] ys[row, c]
// (the k_coef1 partial layout); blockIdx.y = i R + a, i < nwin; s x R row-major sketches.
template <int R, int K>
__global__ void __launch_bounds__(kThreads) k_skpass1(Win zs, int nwin, int64_t s, const double* __restrict__ ys,
                                                      double* __restrict__ partial) {
  __shared__ double sm[kWarps * R];
  const int ia = blockIdx.y, i = ia / R, a = ia % R;
  if (i >= nwin) return;                                   // block-uniform
  const double* __restrict__ z = zs.p[i];
  double acc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < s; row += (int64_t)gridDim.x * kThreads) {
    const double zv = z[row * R + a];
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] = fma(zv, ys[row * R + c], acc[c]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < R; ++c) {
    double v = acc[c];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(SYLV_FULL_MASK, v, off);
    if (lane == 0) sm[warp * R + c] = v;
  }
  __syncthreads();
  if (threadIdx.x < R) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v += sm[w * R + threadIdx.x];   // fixed order
    partial[(int64_t)blockIdx.x * (K * R * R) + ia * R + threadIdx.x] = v;
  }
}

// out = ys R_j - sum_i zs_i K_i  (coef = [R_j, K_0 .. K_{nwin-1}], R x R row-major each) and the
// Gram partials of out (k_coef2 layout: partial[blk * R R + a R + c]).
template <int R, int K>
__global__ void __launch_bounds__(kThreads) k_skpass2(Win zs, int nwin, int64_t s, const double* __restrict__ ys,
                                                      const double* __restrict__ coef, double* __restrict__ out,
                                                      double* __restrict__ partial) {
  __shared__ double cf[(1 + K) * R * R];
  __shared__ double sm[kWarps * R * R];
  for (int e = threadIdx.x; e < (1 + nwin) * R * R; e += kThreads) cf[e] = coef[e];
  __syncthreads();
  double g[R * R];
#pragma unroll
  for (int e = 0; e < R * R; ++e) g[e] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < s; row += (int64_t)gridDim.x * kThreads) {
    double y[R], o[R];
#pragma unroll
    for (int a = 0; a < R; ++a) y[a] = ys[row * R + a];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double v = 0.0;
#pragma unroll
      for (int a = 0; a < R; ++a) v = fma(y[a], cf[a * R + c], v);
      o[c] = v;
    }
    for (int i = 0; i < nwin; ++i) {
      double z[R];
#pragma unroll
      for (int a = 0; a < R; ++a) z[a] = zs.p[i][row * R + a];
#pragma unroll
      for (int c = 0; c < R; ++c) {
        double v = o[c];
#pragma unroll
        for (int a = 0; a < R; ++a) v = fma(-z[a], cf[(1 + i) * R * R + a * R + c], v);
        o[c] = v;
      }
    }
#pragma unroll
    for (int c = 0; c < R; ++c) out[row * R + c] = o[c];
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int c = 0; c < R; ++c) g[a * R + c] = fma(o[a], o[c], g[a * R + c]);
  }
  cta_reduce_store<R * R>(g, partial, sm);
}

}  // namespace sylv
