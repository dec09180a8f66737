// nspace.cuh — n-space kernels of the hot path.
//
// Storage: basis blocks are kept UNNORMALISED as Z_j with U_j = Z_j R_j (R_j upper
// triangular r x r; R_1 = ell^{-1}, R_{j+1} = h_{j+1,j}^{-1}).  Every normalisation
// is folded into r x r coefficients, so no pass rescales an n x r block:
//
//   pass 1  Yt = A Z_d (a1, on the fly),  P_i = Z_i^T Yt  for the k window blocks
//           -> h_{i,d} = U_i^T W~ = R_i^T P_i R_d            (a2 coefficients, CGS)
//   pass 2  W' = Yt R_d - sum_i Z_i (R_i h_{i,d})  = W~ - sum_i U_i h_{i,d}  (a2 update)
//           written as Z_{d+1};  G = W'^T W' (a3 Gram);  S W' scattered (a4)
//           -> h_{d+1,d} = chol(G),  R_{d+1} = h_{d+1,d}^{-1},  S U_{d+1} = (S W') R_{d+1}
//
// CGS over the k-window equals the paper's MGS in exact arithmetic because the
// window blocks are mutually orthonormal (R5).  Blocks are row-major n x R
// ("row-interleaved": the R values of one grid row are contiguous).
#pragma once
#include "common.cuh"

namespace sylv {

struct Win {
  const double* p[kMaxK];  // window blocks Z_{d-nwin+1..d}, oldest first
};

// Reduce acc (per-lane column c = lane % R) over the lanes of a warp with equal c.
template <int R>
__device__ __forceinline__ double warp_sum_same_col(double v) {
#pragma unroll
  for (int off = R; off < 32; off <<= 1) v += __shfl_xor_sync(SYLV_FULL_MASK, v, off);
  return v;
}

// ---------------------------------------------------------------------------------
// pass 1: Yt = A Z_d,  partial[blk][(i*R + a)*R + c] = sum_rows Z_i[row,a] Yt[row,c]
// ---------------------------------------------------------------------------------
template <int R, int K>
__global__ void __launch_bounds__(kThreads) k_pass1(OpParams op, Win win, int nwin,
                                                    double* __restrict__ Yt,
                                                    double* __restrict__ partial) {
  constexpr int RPW = 32 / R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % R, rl = lane / R;
  const double* __restrict__ Zd = win.p[nwin - 1];
  double acc[K][R];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int a = 0; a < R; ++a) acc[i][a] = 0.0;

  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t rg = (int64_t)blockIdx.x * kWarps + warp; rg * RPW < op.n; rg += nwarps) {
    const int64_t row = rg * RPW + rl;
    if (row < op.n) {
      const double y = op_apply<R>(op, Zd, row, c);
      if (Yt) Yt[row * R + c] = y;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i < nwin) {
          const double* __restrict__ zi = win.p[i] + row * R;
#pragma unroll
          for (int a = 0; a < R; ++a) acc[i][a] = fma(__ldg(zi + a), y, acc[i][a]);
        }
      }
    }
  }
  __shared__ double sm[kWarps][K * R * R];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const double v = warp_sum_same_col<R>(acc[i][a]);
      if (lane < R) sm[warp][(i * R + a) * R + lane] = v;
    }
  __syncthreads();
  for (int e = threadIdx.x; e < K * R * R; e += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += sm[w][e];
    partial[(int64_t)blockIdx.x * K * R * R + e] = s;
  }
}

// ---------------------------------------------------------------------------------
// pass 2: W' = Yt R_d - sum_i Z_i K_i (coef = [R_d, K_0..K_{nwin-1}]), write W';
//         optional Gram partial (G[a][c]) and sparse-sign scatter of W' into sk.
// Also the replay kernel of the second pass (GRAM_SKETCH = false).
// ---------------------------------------------------------------------------------
template <int R, int K, bool GRAM_SKETCH>
__global__ void __launch_bounds__(kThreads) k_pass2(OpParams op, Win win, int nwin,
                                                    const double* __restrict__ Yt,
                                                    const double* __restrict__ coef,
                                                    double* __restrict__ Wout,
                                                    double* __restrict__ partial,
                                                    SketchParams sp, double* __restrict__ sk) {
  constexpr int RPW = 32 / R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % R, rl = lane / R;
  __shared__ double cs[(K + 1) * R * R];
  for (int e = threadIdx.x; e < (1 + nwin) * R * R; e += kThreads) cs[e] = coef[e];
  __syncthreads();
  const double* __restrict__ Zd = win.p[nwin - 1];
  double g[R];
#pragma unroll
  for (int a = 0; a < R; ++a) g[a] = 0.0;

  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t rg = (int64_t)blockIdx.x * kWarps + warp; rg * RPW < op.n; rg += nwarps) {
    const int64_t row = rg * RPW + rl;
    const bool valid = row < op.n;
    double y = 0.0;
    if (valid) y = Yt ? Yt[row * R + c] : op_apply<R>(op, Zd, row, c);
    double wv = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const double ya = (R == 1) ? y : __shfl_sync(SYLV_FULL_MASK, y, rl * R + a);
      wv = fma(ya, cs[a * R + c], wv);
    }
    if (valid) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i < nwin) {
          const double* __restrict__ zi = win.p[i] + row * R;
          const double* ki = cs + (1 + i) * R * R;
#pragma unroll
          for (int a = 0; a < R; ++a) wv = fma(-__ldg(zi + a), ki[a * R + c], wv);
        }
      }
      Wout[row * R + c] = wv;
    } else {
      wv = 0.0;
    }
    if (GRAM_SKETCH) {
#pragma unroll
      for (int a = 0; a < R; ++a) {
        const double wa = (R == 1) ? wv : __shfl_sync(SYLV_FULL_MASK, wv, rl * R + a);
        g[a] = fma(wa, wv, g[a]);
      }
      if (valid && sk) {
        const uint32_t m = (uint32_t)(row >> 5), l = (uint32_t)(row & 31);
        for (uint32_t t = 0; t < sp.zeta; ++t) {
          const SkEntry e = sk_entry(sp, m, l, t);
          atomicAdd(sk + (int64_t)e.row * R + c, e.val * wv);
        }
      }
    }
  }
  if (GRAM_SKETCH) {
    __shared__ double sm[kWarps][R * R];
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const double v = warp_sum_same_col<R>(g[a]);
      if (lane < R) sm[warp][a * R + lane] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += kThreads) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += sm[w][e];
      partial[(int64_t)blockIdx.x * R * R + e] = s;
    }
  }
}

// ---------------------------------------------------------------------------------
// Standalone sketch of an n x R block (init: S C; test entry apply_sketch), and the
// Gram partial of the same block (init: C^T C).  out must be zeroed.
// ---------------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(kThreads) k_sketch_gram(int64_t n, const double* __restrict__ X,
                                                          SketchParams sp, double* __restrict__ out,
                                                          double* __restrict__ partial) {
  constexpr int RPW = 32 / R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % R, rl = lane / R;
  double g[R];
#pragma unroll
  for (int a = 0; a < R; ++a) g[a] = 0.0;
  const int64_t nwarps = (int64_t)gridDim.x * kWarps;
  for (int64_t rg = (int64_t)blockIdx.x * kWarps + warp; rg * RPW < n; rg += nwarps) {
    const int64_t row = rg * RPW + rl;
    const bool valid = row < n;
    const double x = valid ? X[row * R + c] : 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const double xa = (R == 1) ? x : __shfl_sync(SYLV_FULL_MASK, x, rl * R + a);
      g[a] = fma(xa, x, g[a]);
    }
    if (valid && out) {
      const uint32_t m = (uint32_t)(row >> 5), l = (uint32_t)(row & 31);
      for (uint32_t t = 0; t < sp.zeta; ++t) {
        const SkEntry e = sk_entry(sp, m, l, t);
        atomicAdd(out + (int64_t)e.row * R + c, e.val * x);
      }
    }
  }
  if (partial) {
    __shared__ double sm[kWarps][R * R];
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const double v = warp_sum_same_col<R>(g[a]);
      if (lane < R) sm[warp][a * R + lane] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < R * R; e += kThreads) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s += sm[w][e];
      partial[(int64_t)blockIdx.x * R * R + e] = s;
    }
  }
}

// ---------------------------------------------------------------------------------
// Second pass accumulation X[row, l] += sum_b sum_a Z_b[row, a] M[(b*R + a)*ell + l]
// for a chunk of nb blocks (a7).  One thread per (row, l).
// ---------------------------------------------------------------------------------
constexpr int kMaxChunk = 16;
struct ChunkPtrs {
  const double* p[kMaxChunk];
};

template <int R>
__global__ void __launch_bounds__(kThreads) k_xacc(int64_t n, ChunkPtrs zb, int nb,
                                                   const double* __restrict__ M, int ell,
                                                   double* __restrict__ X, int64_t ldx) {
  const int64_t total = n * (int64_t)ell;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * kThreads) {
    const int64_t row = e / ell;
    const int l = (int)(e - row * ell);
    double acc = X[row * ldx + l];
    for (int b = 0; b < nb; ++b) {
      const double* z = zb.p[b] + row * R;
#pragma unroll
      for (int a = 0; a < R; ++a) acc = fma(__ldg(z + a), __ldg(M + (int64_t)(b * R + a) * ell + l), acc);
    }
    X[row * ldx + l] = acc;
  }
}

// Normalised block out = Z R (introspection entry get_block).
template <int R>
__global__ void k_zr(int64_t n, const double* __restrict__ Z, const double* __restrict__ Rm,
                     double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * R;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / R;
    const int c = (int)(e - row * R);
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a) s = fma(Z[row * R + a], Rm[a * R + c], s);
    out[e] = s;
  }
}

}  // namespace sylv
