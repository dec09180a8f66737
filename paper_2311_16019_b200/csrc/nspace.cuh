// nspace.cuh — n-space kernels of the hot path.
//
// Storage: basis blocks are kept UNNORMALISED as Z_j with U_j = Z_j R_j (R_j upper
// triangular r x r; R_1 = ell^{-1}, R_{j+1} = h_{j+1,j}^{-1}).  Every normalisation
// is folded into r x r coefficients, so no pass rescales an n x r block:
//
//   pass 1  Yt = A Z_d (a1, on the fly),  P_i = Z_i^T Yt  for the k window blocks
//           -> h_{i,d} = U_i^T W~ = R_i^T P_i R_d            (a2 coefficients, CGS)
//   pass 2  W' = Yt R_d - sum_i Z_i (R_i h_{i,d})  = W~ - sum_i U_i h_{i,d}  (a2 update)
//           written as Z_{d+1};  G = W'^T W' (a3 Gram)
//           -> h_{d+1,d} = chol(G),  R_{d+1} = h_{d+1,d}^{-1}
//   sketch  S W' with the hashed sparse-sign S (a4), shared-memory privatised per column
//           -> S U_{d+1} = (S W') R_{d+1}
//
// CGS over the k-window equals the paper's MGS in exact arithmetic because the window
// blocks are mutually orthonormal (R5).
//
// Layout ("SoA"): an n x R block is R columns of length ld (ld = n rounded up to 64),
// element (row, c) at X[c*ld + row].  Warps read 32/64-byte column segments, so every
// 32-byte sector fetched is fully used for any R.
//
// r = 8 uses the fp64 tensor-core MMA (mma.sync.m8n8k4.f64, DMMA) for the block inner
// products, the block update and the Gram: one instruction per 256 FMAs and 2 accumulator
// registers per lane per r x r product.  r <= 4 uses one thread per row with FMAs.
#pragma once
#include "common.cuh"

namespace sylv {

struct Win {
  const double* p[kMaxK];  // window blocks Z_{d-nwin+1..d}, oldest first (Z_d = p[nwin-1])
};

// Stencil grid coordinates of `row` (x fastest).
struct Coord {
  uint32_t x, y, z;
};
__device__ __forceinline__ Coord coords(const OpParams& op, uint32_t row) {
  Coord c;
  const uint32_t q1 = fdiv(row, op.divN);
  c.x = row - q1 * (uint32_t)op.N;
  if (op.kind == kStencil2D) {
    c.y = q1;
    c.z = 0;
  } else {
    c.z = fdiv(q1, op.divN);
    c.y = q1 - c.z * (uint32_t)op.N;
  }
  return c;
}

// (A Z)[row] for one SoA column `z` (= Z + c*ld), row local to this rank's block.
// `center` returns z[row].  The last grid direction (y in 2-D, z in 3-D) is read
// unconditionally: the block's ghost lines/planes hold the neighbour rank's boundary data,
// or zeros at the Dirichlet boundary (fma(c, 0, v) = v exactly).
__device__ __forceinline__ double stencil_col(const OpParams& op, const double* __restrict__ z,
                                              uint32_t row, const Coord& q, double& center) {
  const uint32_t N = (uint32_t)op.N;
  const double* p = z + row;
  center = __ldg(p);
  double v = op.cd * center;
  if (q.x > 0) v = fma(op.cxm, __ldg(p - 1), v);
  if (q.x + 1 < N) v = fma(op.cxp, __ldg(p + 1), v);
  if (op.kind == kStencil3D) {
    if (q.y > 0) v = fma(op.cym, __ldg(p - N), v);
    if (q.y + 1 < N) v = fma(op.cyp, __ldg(p + N), v);
    const uint32_t NN = N * N;
    v = fma(op.czm, __ldg(p - NN), v);
    v = fma(op.czp, __ldg(p + NN), v);
  } else {
    v = fma(op.cym, __ldg(p - N), v);
    v = fma(op.cyp, __ldg(p + N), v);
  }
  return v;
}

__device__ __forceinline__ double csr_col(const OpParams& op, const double* __restrict__ z, int64_t row) {
  double v = 0.0;
  const int64_t p1 = __ldg(op.rp + row + 1);
  for (int64_t p = __ldg(op.rp + row); p < p1; ++p) v = fma(__ldg(op.cv + p), __ldg(z + __ldg(op.ci + p)), v);
  return v;
}

// Deterministic CTA reduction of NV per-thread values -> partial[blockIdx.x*NV + e].
template <int NV>
__device__ __forceinline__ void cta_reduce_store(const double (&v)[NV], double* __restrict__ partial,
                                                 double* sm /* kWarps*NV */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int e = 0; e < NV; ++e) {
    double s = v[e];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(SYLV_FULL_MASK, s, off);
    if (lane == 0) sm[warp * NV + e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NV; e += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += sm[w * NV + e];
    partial[(int64_t)blockIdx.x * NV + e] = s;
  }
}

// =====================================================================================
// r <= 4: one thread per row
// =====================================================================================

// pass 1: partial[blk][(i*R + a)*R + c] = sum_rows Z_i[row,a] Yt[row,c]
template <int R, int K>
__global__ void __launch_bounds__(kThreads) k_pass1_rows(OpParams op, Win win, int nwin, int64_t ld,
                                                         double* __restrict__ Yt,
                                                         double* __restrict__ partial) {
  __shared__ double sm[kWarps * K * R * R];
  double acc[K * R * R];
#pragma unroll
  for (int e = 0; e < K * R * R; ++e) acc[e] = 0.0;
  const double* __restrict__ Zd = win.p[nwin - 1];
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < op.n; row += stride) {
    double y[R], zc[R];
    if (op.kind == kCSR) {
#pragma unroll
      for (int c = 0; c < R; ++c) {
        y[c] = csr_col(op, Zd + c * ld, row);
        zc[c] = __ldg(Zd + c * ld + row);
      }
      if (Yt) {
#pragma unroll
        for (int c = 0; c < R; ++c) Yt[c * ld + row] = y[c];
      }
    } else {
      const Coord q = coords(op, (uint32_t)row);
#pragma unroll
      for (int c = 0; c < R; ++c) y[c] = stencil_col(op, Zd + c * ld, (uint32_t)row, q, zc[c]);
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i < nwin) {
        double z[R];
        if (i == nwin - 1) {
#pragma unroll
          for (int a = 0; a < R; ++a) z[a] = zc[a];
        } else {
#pragma unroll
          for (int a = 0; a < R; ++a) z[a] = __ldg(win.p[i] + a * ld + row);
        }
#pragma unroll
        for (int a = 0; a < R; ++a)
#pragma unroll
          for (int c = 0; c < R; ++c) acc[(i * R + a) * R + c] = fma(z[a], y[c], acc[(i * R + a) * R + c]);
      }
    }
  }
  cta_reduce_store<K * R * R>(acc, partial, sm);
}

// pass 2: W' = Yt R_d - sum_i Z_i K_i  (coef = [R_d, K_0..K_{nwin-1}]); Gram partial.
// GRAM = false: the second-pass replay (no Gram).
template <int R, int K, bool GRAM>
__global__ void __launch_bounds__(kThreads) k_pass2_rows(OpParams op, Win win, int nwin, int64_t ld,
                                                         const double* __restrict__ Yt,
                                                         const double* __restrict__ coef,
                                                         double* __restrict__ Wout,
                                                         double* __restrict__ partial) {
  __shared__ double cs[(K + 1) * R * R];
  __shared__ double sm[GRAM ? kWarps * R * R : 1];
  for (int e = threadIdx.x; e < (1 + nwin) * R * R; e += blockDim.x) cs[e] = coef[e];
  __syncthreads();
  double g[R * R];
#pragma unroll
  for (int e = 0; e < R * R; ++e) g[e] = 0.0;
  const double* __restrict__ Zd = win.p[nwin - 1];
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < op.n; row += stride) {
    double y[R], zc[R];
    if (Yt) {
#pragma unroll
      for (int c = 0; c < R; ++c) {
        y[c] = __ldg(Yt + c * ld + row);
        zc[c] = __ldg(Zd + c * ld + row);
      }
    } else if (op.kind == kCSR) {
#pragma unroll
      for (int c = 0; c < R; ++c) {
        y[c] = csr_col(op, Zd + c * ld, row);
        zc[c] = __ldg(Zd + c * ld + row);
      }
    } else {
      const Coord q = coords(op, (uint32_t)row);
#pragma unroll
      for (int c = 0; c < R; ++c) y[c] = stencil_col(op, Zd + c * ld, (uint32_t)row, q, zc[c]);
    }
    double w[R];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < R; ++a) s = fma(y[a], cs[a * R + c], s);
      w[c] = s;
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i < nwin) {
        double z[R];
        if (i == nwin - 1) {
#pragma unroll
          for (int a = 0; a < R; ++a) z[a] = zc[a];
        } else {
#pragma unroll
          for (int a = 0; a < R; ++a) z[a] = __ldg(win.p[i] + a * ld + row);
        }
        const double* ki = cs + (1 + i) * R * R;
#pragma unroll
        for (int c = 0; c < R; ++c)
#pragma unroll
          for (int a = 0; a < R; ++a) w[c] = fma(-z[a], ki[a * R + c], w[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < R; ++c) Wout[c * ld + row] = w[c];
    if (GRAM) {
#pragma unroll
      for (int a = 0; a < R; ++a)
#pragma unroll
        for (int c = 0; c < R; ++c) g[a * R + c] = fma(w[a], w[c], g[a * R + c]);
    }
  }
  if (GRAM) cta_reduce_store<R * R>(g, partial, sm);
}

// =====================================================================================
// CSR pass 1 (a1 + a2 inner products): 4 lanes per row
// =====================================================================================
// Each 4-lane sub-warp owns one row at a time (8 rows per warp): lanes stride over the row's
// nonzeros, issue all value/index loads of their first 6 nonzeros before the gathers, gather
// the rows of Z_d from a row-interleaved copy (one sector per nonzero for r <= 4), accumulate
// all R columns of (A Z_d)[row] from ONE sweep of the row, and reduce with two xor-shuffles;
// the next row's row pointers are loaded one iteration ahead.  The sub-warp's lane 0 stores
// Yt[row] (pass 2 streams it instead of re-reading A) and accumulates P_i += Z_i[row]^T Yt[row].
// c4 (r = 2): 0.76 ms -> 0.48 ms per launch (8 lanes, SoA gathers -> this).
constexpr int kCsrLanes = 4;

// Row-interleaved (AoS) copy of an SoA block for the CSR gathers: Za[row*R + c] = Z[c*ld + row].
// One gathered row is then R contiguous doubles (one 32-byte sector for R <= 4) instead of R
// separate sectors: half (R = 2) or a quarter (R = 4) of the L1 wavefronts of pass 1.
template <int R>
__global__ void __launch_bounds__(kThreads) k_soa_to_aos(int64_t n, const double* __restrict__ Z, int64_t ld,
                                                         double* __restrict__ Za) {
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < n; row += (int64_t)gridDim.x * kThreads) {
    double v[R];
#pragma unroll
    for (int c = 0; c < R; ++c) v[c] = __ldg(Z + c * ld + row);
    if (R % 2 == 0) {
#pragma unroll
      for (int c = 0; c < R; c += 2) reinterpret_cast<double2*>(Za + row * R)[c / 2] = make_double2(v[c], v[c + 1]);
    } else {
#pragma unroll
      for (int c = 0; c < R; ++c) Za[row * R + c] = v[c];
    }
  }
}

template <int R, int K>
__global__ void __launch_bounds__(kThreads) k_pass1_csr(OpParams op, Win win, int nwin, int64_t ld,
                                                        const double* __restrict__ Za,
                                                        double* __restrict__ Yt, double* __restrict__ partial) {
  __shared__ double sm[kWarps * K * R * R];
  double acc[K * R * R];
#pragma unroll
  for (int e = 0; e < K * R * R; ++e) acc[e] = 0.0;
  const int sub = threadIdx.x & (kCsrLanes - 1);
  const double* __restrict__ Zd = win.p[nwin - 1];
  const int64_t nsub = (int64_t)gridDim.x * (kThreads / kCsrLanes);
  // warp-uniform trip count: every lane of a warp runs the same iterations (the shuffles
  // below use the full mask); sub-warps past the last row do no work
  const int64_t wfirst = (int64_t)blockIdx.x * (kThreads / kCsrLanes) + (threadIdx.x & ~31) / kCsrLanes;
  // row pointers of the next row are loaded one iteration ahead
  const int64_t r0 = wfirst + (threadIdx.x & 31) / kCsrLanes;
  int64_t q0 = r0 < op.n ? __ldg(op.rp + r0) : 0, q1 = r0 < op.n ? __ldg(op.rp + r0 + 1) : 0;
  for (int64_t wrow = wfirst; wrow < op.n; wrow += nsub) {
    const int64_t row = wrow + (threadIdx.x & 31) / kCsrLanes;
    const bool valid = row < op.n;
    double y[R];
#pragma unroll
    for (int c = 0; c < R; ++c) y[c] = 0.0;
    const int64_t p0 = q0, p1 = q1;
    {
      const int64_t rn = row + nsub;
      q0 = rn < op.n ? __ldg(op.rp + rn) : 0;
      q1 = rn < op.n ? __ldg(op.rp + rn + 1) : 0;
    }
    // gather of Z_d row `col` into y (AoS copy for even R)
    auto gather = [&](double a, int64_t col) {
      if (R % 2 == 0) {
        const double2* zr = reinterpret_cast<const double2*>(Za + col * R);
#pragma unroll
        for (int c = 0; c < R; c += 2) {
          const double2 z = __ldg(zr + c / 2);
          y[c] = fma(a, z.x, y[c]);
          y[c + 1] = fma(a, z.y, y[c + 1]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < R; ++c) y[c] = fma(a, __ldg(Zd + c * ld + col), y[c]);
      }
    };
    // the first kCsrU nonzeros per lane: all value/index loads issued before the gathers
    // (rows of the BASELINE CSR have 21 nonzeros: <= 6 per lane); longer rows continue below
    constexpr int kCsrU = 6;
    // (column indices of a row-sharded operator are local and may be negative: ghost rows)
    double av[kCsrU];
    int32_t cl[kCsrU];
#pragma unroll
    for (int u = 0; u < kCsrU; ++u) {
      const int64_t p = p0 + sub + u * kCsrLanes;
      av[u] = p < p1 ? __ldg(op.cv + p) : 0.0;
      cl[u] = p < p1 ? __ldg(op.ci + p) : 0;
    }
#pragma unroll
    for (int u = 0; u < kCsrU; ++u)
      if (p0 + sub + u * kCsrLanes < p1) gather(av[u], cl[u]);
    for (int64_t p = p0 + sub + kCsrU * kCsrLanes; p < p1; p += kCsrLanes) gather(__ldg(op.cv + p), __ldg(op.ci + p));
#pragma unroll
    for (int c = 0; c < R; ++c) {
#pragma unroll
      for (int off = kCsrLanes / 2; off > 0; off >>= 1) y[c] += __shfl_xor_sync(SYLV_FULL_MASK, y[c], off);
    }
    if (sub == 0 && valid) {
      if (Yt) {
#pragma unroll
        for (int c = 0; c < R; ++c) Yt[c * ld + row] = y[c];
      }
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i < nwin) {
          double z[R];
#pragma unroll
          for (int a = 0; a < R; ++a) z[a] = __ldg(win.p[i] + a * ld + row);
#pragma unroll
          for (int a = 0; a < R; ++a)
#pragma unroll
            for (int c = 0; c < R; ++c) acc[(i * R + a) * R + c] = fma(z[a], y[c], acc[(i * R + a) * R + c]);
        }
      }
    }
  }
  cta_reduce_store<K * R * R>(acc, partial, sm);
}

// =====================================================================================
// r = 8: DMMA warp tiles
// =====================================================================================

// pass 1, 4-row tiles: lane <-> element (row0 + (lane&3), col lane>>2) of every block.
template <int K>
__global__ void __launch_bounds__(kThreads) k_pass1_r8(OpParams op, Win win, int nwin, int64_t ld,
                                                       double* __restrict__ Yt,
                                                       double* __restrict__ partial) {
  constexpr int R = 8;
  __shared__ double sm[kWarps * K * 64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rr = lane & 3, c = lane >> 2;
  double acc[K][2];
#pragma unroll
  for (int i = 0; i < K; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double* __restrict__ Zd = win.p[nwin - 1] + c * ld;
  const int64_t ntiles = (op.n + 3) >> 2;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + warp; t < ntiles; t += wstride) {
    const int64_t row = t * 4 + rr;
    double y = 0.0, zc = 0.0;
    if (row < op.n) {
      if (op.kind == kCSR) {
        y = csr_col(op, Zd, row);
        zc = __ldg(Zd + row);
        if (Yt) Yt[c * ld + row] = y;
      } else {
        const Coord q = coords(op, (uint32_t)row);
        y = stencil_col(op, Zd, (uint32_t)row, q, zc);
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i < nwin) {
        const double z = (i == nwin - 1) ? zc : (row < op.n ? __ldg(win.p[i] + c * ld + row) : 0.0);
        dmma(acc[i], z, y);  // P_i[a][c'] += Z_i[row][a] Yt[row][c']
      }
    }
  }
  // D fragment: lane holds P_i[lane>>2][2*(lane&3) + e]
#pragma unroll
  for (int i = 0; i < K; ++i) {
    sm[(warp * K + i) * 64 + c * 8 + 2 * rr] = acc[i][0];
    sm[(warp * K + i) * 64 + c * 8 + 2 * rr + 1] = acc[i][1];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < K * 64; e += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += sm[w * K * 64 + e];
    partial[(int64_t)blockIdx.x * K * 64 + e] = s;
  }
  (void)R;
}

// pass 2, 8-row tiles.  A fragments: lane holds X[row0 + (lane>>2)][(lane&3) + 4h], h = 0, 1.
template <int K, bool GRAM>
__global__ void __launch_bounds__(kThreads) k_pass2_r8(OpParams op, Win win, int nwin, int64_t ld,
                                                       const double* __restrict__ Yt,
                                                       const double* __restrict__ coef,
                                                       double* __restrict__ Wout,
                                                       double* __restrict__ partial) {
  __shared__ double sm[GRAM ? kWarps * 64 : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ra = lane >> 2, ka = lane & 3;  // A: row ra, k-col ka (+4h); B: k-row ka (+4h), col ra
  // B fragments of the coefficient matrices (row-major 8x8): R_d and -K_i
  double bR[2], bK[K][2];
#pragma unroll
  for (int h = 0; h < 2; ++h) bR[h] = __ldg(coef + (ka + 4 * h) * 8 + ra);
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) bK[i][h] = (i < nwin) ? -__ldg(coef + (1 + i) * 64 + (ka + 4 * h) * 8 + ra) : 0.0;
  double G[2] = {0.0, 0.0};
  const double* __restrict__ Zd = win.p[nwin - 1];
  const int64_t ntiles = (op.n + 7) >> 3;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + warp; t < ntiles; t += wstride) {
    const int64_t row = t * 8 + ra;
    const bool valid = row < op.n;
    double y[2] = {0.0, 0.0}, zc[2] = {0.0, 0.0};
    if (valid) {
      if (Yt) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          y[h] = __ldg(Yt + (ka + 4 * h) * ld + row);
          zc[h] = __ldg(Zd + (ka + 4 * h) * ld + row);
        }
      } else if (op.kind == kCSR) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          y[h] = csr_col(op, Zd + (ka + 4 * h) * ld, row);
          zc[h] = __ldg(Zd + (ka + 4 * h) * ld + row);
        }
      } else {
        const Coord q = coords(op, (uint32_t)row);
#pragma unroll
        for (int h = 0; h < 2; ++h) y[h] = stencil_col(op, Zd + (ka + 4 * h) * ld, (uint32_t)row, q, zc[h]);
      }
    }
    double D[2] = {0.0, 0.0};
    dmma(D, y[0], bR[0]);
    dmma(D, y[1], bR[1]);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i < nwin) {
        double z0, z1;
        if (i == nwin - 1) {
          z0 = zc[0];
          z1 = zc[1];
        } else {
          z0 = valid ? __ldg(win.p[i] + ka * ld + row) : 0.0;
          z1 = valid ? __ldg(win.p[i] + (ka + 4) * ld + row) : 0.0;
        }
        dmma(D, z0, bK[i][0]);
        dmma(D, z1, bK[i][1]);
      }
    }
    // D: lane holds W'[row0 + ra][2*ka + e]
    const int64_t orow = t * 8 + ra;
    if (orow < op.n) {
      Wout[(2 * ka) * ld + orow] = D[0];
      Wout[(2 * ka + 1) * ld + orow] = D[1];
    }
    if (GRAM) {
      // Gram: A = B = element (row0 + 4q + (lane&3), col lane>>2), held by lane 4r + (col>>1), reg col&1
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const int r = 4 * qq + (lane & 3);
        const int col = lane >> 2;
        const int src = 4 * r + (col >> 1);
        const double v0 = __shfl_sync(SYLV_FULL_MASK, D[0], src);
        const double v1 = __shfl_sync(SYLV_FULL_MASK, D[1], src);
        const double v = (col & 1) ? v1 : v0;
        dmma(G, v, v);
      }
    }
  }
  if (GRAM) {
    sm[warp * 64 + ra * 8 + 2 * ka] = G[0];
    sm[warp * 64 + ra * 8 + 2 * ka + 1] = G[1];
    __syncthreads();
    for (int e = threadIdx.x; e < 64; e += kThreads) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += sm[w * 64 + e];
      partial[(int64_t)blockIdx.x * 64 + e] = s;
    }
  }
}

// =====================================================================================
// Sparse-sign sketch of an SoA block, shared-memory privatised (a4)
// =====================================================================================
// grid (nchunk, R), one CTA per SM (the whole sketch column lives in shared memory).
// CTA (chunk, c) accumulates column c of S X over the rows of its chunk.
//
// Tiles of kSkWarps x kSkG groups of 32 rows: warp w loads ITS OWN kSkG groups into
// registers (coalesced 256-byte loads, double-buffered: the next tile is in flight while
// this one is scattered), so every element is read from HBM exactly once.
// Per tile, each warp first evaluates the three hashes of all its
// (group, bucket) pairs (4 pairs per lane, independent chains) and stores one 16-byte
// record per pair in its own shared-memory area: {byte offset of the slot window, a, 8c,
// sign bits}.  The scatter then runs in
// P = max(zeta, 8) phases separated by __syncthreads(); in phase p warp w owns bucket
// t = (w + p) mod P, so no two warps ever touch the same bucket at the same time and no
// atomics are needed.  A group's record is one broadcast LDS.128; its 32 rows hit the 32
// distinct consecutive slots base .. base+31 of a bucket padded to b + 32 slots (no wrap
// test; the pad is folded back onto slots 0..31 at the end), conflict-free; the sign is
// applied by flipping the sign bit.  Two groups whose windows are disjoint issue their
// read-modify-writes together.
// Output: partial[(chunk*R + c)*s + q].
constexpr int kSkWarps = 8;
constexpr int kSkG = 16;           // groups per warp per tile

__host__ __device__ constexpr int64_t sketch_smem_doubles(int64_t s, int zeta) {
  return s + 32 * (int64_t)zeta + (int64_t)kSkWarps * kSkG * zeta * 2;   // buckets + hash records
}

template <int R>
__global__ void __launch_bounds__(kSkWarps * 32, 1) k_sketch_cols(int64_t n, const double* __restrict__ X,
                                                                  int64_t ld, SketchParams sp,
                                                                  int64_t groups_per_chunk,
                                                                  double* __restrict__ partial) {
  extern __shared__ __align__(16) double skm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.y;
  const uint32_t b = sp.b, bp = sp.b + 32u;           // bucket height, padded height
  const uint32_t zeta = sp.zeta;
  const int64_t s = (int64_t)b * zeta;
  const int64_t sz = (int64_t)bp * zeta;
  uint4* rec = reinterpret_cast<uint4*>(skm + sz) + (size_t)warp * kSkG * zeta;   // [g][t]
  for (int64_t e = threadIdx.x; e < sz; e += kSkWarps * 32) skm[e] = 0.0;
  const int64_t ngroups = (n + 31) >> 5;
  const int64_t g0 = (int64_t)blockIdx.x * groups_per_chunk;
  const int64_t g1 = min(ngroups, g0 + groups_per_chunk);
  const double* __restrict__ xc = X + c * ld;
  const uint32_t P = zeta > (uint32_t)kSkWarps ? zeta : (uint32_t)kSkWarps;
  constexpr int64_t kTile = (int64_t)kSkWarps * kSkG;   // groups per tile
  const uint32_t l8 = 8u * (uint32_t)lane;
  const uint32_t npairs = (uint32_t)kSkG * zeta;      // (group, bucket) pairs per warp per tile
  char* const sb = reinterpret_cast<char*>(skm);

  double v[kSkG], vn[kSkG];
#pragma unroll
  for (int g = 0; g < kSkG; ++g) {
    const int64_t grp = g0 + (int64_t)warp * kSkG + g;
    const int64_t row = (grp << 5) + lane;
    vn[g] = (grp < g1 && row < n) ? __ldg(xc + row) : 0.0;
  }
  __syncthreads();
  for (int64_t tg = g0; tg < g1; tg += kTile) {
#pragma unroll
    for (int g = 0; g < kSkG; ++g) v[g] = vn[g];
    if (tg + kTile < g1) {                               // prefetch the next tile
#pragma unroll
      for (int g = 0; g < kSkG; ++g) {
        const int64_t grp = tg + kTile + (int64_t)warp * kSkG + g;
        const int64_t row = (grp << 5) + lane;
        vn[g] = (grp < g1 && row < n) ? __ldg(xc + row) : 0.0;
      }
    }
    const int64_t mybase = tg + (int64_t)warp * kSkG;      // first group of this warp
    // hash records of this warp's (group, bucket) pairs
    for (uint32_t e = lane; e < npairs; e += 32) {
      const uint32_t g = e / zeta, t = e - g * zeta;
      const uint32_t m = sp.m0 + (uint32_t)mybase + g;          // global group index
      const uint32_t h0 = group_hash(sp, m, t, 0);
      const uint32_t h1 = group_hash(sp, m, t, 1);
      const uint32_t h2 = group_hash(sp, m, t, 2);
      rec[e] = make_uint4(8u * (t * bp + __umulhi(h0, b)),   // byte offset of the slot window
                          2u * (h1 & 15u) + 1u,              // a
                          ((h1 >> 4) & 31u) * 8u,            // 8 c
                          h2);                               // sign bits
    }
    __syncwarp();
    for (uint32_t p = 0; p < P; ++p) {
      const uint32_t t = (warp + p) % P;
      if (t < zeta && mybase < g1) {
        if (b >= 32u) {
#pragma unroll
          for (int g8 = 0; g8 < kSkG; g8 += 8) {
            uint32_t adr[8], wof[8];
            double val[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {          // records first (broadcast loads, no aliasing)
              const uint4 r4 = rec[(g8 + u) * zeta + t];
              wof[u] = r4.x;
              adr[u] = r4.x + ((r4.y * l8 + r4.z) & 248u);
              val[u] = __hiloint2double(__double2hiint(v[g8 + u]) ^ (int)((r4.w << (31 - lane)) & 0x80000000u),
                                        __double2loint(v[g8 + u]));
            }
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
              double* pa = reinterpret_cast<double*>(sb + adr[u]);
              double* pb = reinterpret_cast<double*>(sb + adr[u + 1]);
              const uint32_t dist = wof[u] > wof[u + 1] ? wof[u] - wof[u + 1] : wof[u + 1] - wof[u];
              if (dist >= 256u) {                  // disjoint windows: both loads in flight
                const double oa = *pa, ob = *pb;
                *pa = oa + val[u];
                *pb = ob + val[u + 1];
              } else {
                *pa += val[u];
                *pb += val[u + 1];
              }
            }
          }
        } else {
          // tiny buckets (b < 32): the 32 rows of a group collide; shared atomics
          double* bucket = skm + (int64_t)t * bp;
#pragma unroll
          for (int g = 0; g < kSkG; ++g) {
            const uint4 r4 = rec[g * zeta + t];
            const uint32_t base = r4.x / 8u - t * bp;
            const uint32_t sl = (base + ((r4.y * (uint32_t)lane + r4.z / 8u) & 31u)) % b;
            atomicAdd(bucket + sl, ((r4.w >> lane) & 1u) ? -v[g] : v[g]);
          }
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  // fold the pad slots b .. b+31 of every bucket onto slots 0 .. 31, scale, write
  double* out = partial + ((int64_t)blockIdx.x * R + c) * s;
  for (int64_t q = threadIdx.x; q < s; q += kSkWarps * 32) {
    const int64_t t = q / b, i = q - t * b;
    double v0 = skm[t * bp + i];
    if (i < 32 && b >= 32u) v0 += skm[t * bp + b + i];
    out[q] = v0 * sp.scale;
  }
}

// w[q*R + c] = sum_a (sum_chunk partial[(chunk*R + a)*s + q]) M[a*R + c]  (M = identity if null)
template <int R>
__global__ void k_sketch_reduce(const double* __restrict__ partial, int nchunk, int64_t s,
                                const double* __restrict__ M, double* __restrict__ w) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < s; q += (int64_t)gridDim.x * blockDim.x) {
    double v[R];
#pragma unroll
    for (int a = 0; a < R; ++a) {
      double acc = 0.0;
      for (int ch = 0; ch < nchunk; ++ch) acc += partial[((int64_t)ch * R + a) * s + q];
      v[a] = acc;
    }
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double o;
      if (M) {
        o = 0.0;
#pragma unroll
        for (int a = 0; a < R; ++a) o = fma(v[a], __ldg(M + a * R + c), o);
      } else {
        o = v[c];
      }
      w[q * R + c] = o;
    }
  }
}

// Gram partial of an SoA block (init: C^T C), one thread per row.
template <int R>
__global__ void __launch_bounds__(kThreads) k_gram_soa(int64_t n, const double* __restrict__ X, int64_t ld,
                                                       double* __restrict__ partial) {
  __shared__ double sm[kWarps * R * R];
  double g[R * R];
#pragma unroll
  for (int e = 0; e < R * R; ++e) g[e] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < n; row += (int64_t)gridDim.x * kThreads) {
    double x[R];
#pragma unroll
    for (int c = 0; c < R; ++c) x[c] = __ldg(X + c * ld + row);
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int c = 0; c < R; ++c) g[a * R + c] = fma(x[a], x[c], g[a * R + c]);
  }
  cta_reduce_store<R * R>(g, partial, sm);
}

// Gram partial of a row-major rows x R block (sketch space CholQR2), one thread per row.
template <int R>
__global__ void __launch_bounds__(kThreads) k_gram_rowmajor(int64_t rows, const double* __restrict__ X,
                                                            double* __restrict__ partial) {
  __shared__ double sm[kWarps * R * R];
  double g[R * R];
#pragma unroll
  for (int e = 0; e < R * R; ++e) g[e] = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x; row < rows; row += (int64_t)gridDim.x * kThreads) {
    double x[R];
#pragma unroll
    for (int c = 0; c < R; ++c) x[c] = __ldg(X + row * R + c);
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int c = 0; c < R; ++c) g[a * R + c] = fma(x[a], x[c], g[a * R + c]);
  }
  cta_reduce_store<R * R>(g, partial, sm);
}

// Row-major (n x R, ld_in) <-> SoA (R columns, ld).
template <int R>
__global__ void k_to_soa(int64_t n, const double* __restrict__ in, double* __restrict__ out, int64_t ld) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * R; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / R;
    const int c = (int)(e - row * R);
    out[c * ld + row] = in[e];
  }
}

// out (row-major n x R) = Z (SoA) M  (get_block: U_j = Z_j R_j)
template <int R>
__global__ void k_soa_mul_rowmajor(int64_t n, const double* __restrict__ Z, int64_t ld,
                                   const double* __restrict__ M, double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * R; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / R;
    const int c = (int)(e - row * R);
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a) s = fma(Z[a * ld + row], M[a * R + c], s);
    out[e] = s;
  }
}

// Second pass (a7): blocks per X accumulation (the replay keeps k + chunk blocks; the
// accumulation X += [U_j0 .. U_j] M is a cuBLAS DGEMM per run of adjacent replay slots, engine.cu)
constexpr int kMaxChunk = 32;   // replay blocks per X accumulation chunk (second pass)

}  // namespace sylv

namespace sylv {

// =====================================================================================
// CSR pass 1 with the band window of Z_d in shared memory (c4: band = max |col - row| = 4096)
// =====================================================================================
// A CTA owns tiles of T consecutive rows.  Every column index of rows [i0, i1) lies in
// [i0 - band, i1 + band), so the window Z_d[w0, w1) (all R columns, SoA) arrives in shared
// memory by bulk copies (cp.async.bulk, one mbarrier) and the 21 gathers per row read shared
// memory instead of L1/L2 (which the global-gather kernel above is bound by).  The CSR
// values / indices stream from HBM once.  4 lanes per row, CGS inner products with the window
// blocks as in k_pass1_csr; the same per-row arithmetic order (parity with k_pass1_csr is exact
// up to the order of the 4-lane shuffle sums, which is the same).
constexpr int kCsrWinThreads = 1024;   // 32 warps: the CSR streams are latency-bound per warp
constexpr int kCsrWinWarps = kCsrWinThreads / 32;
constexpr int kCsrWinRows = kCsrWinThreads / kCsrLanes;   // rows per sweep of the CTA

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

template <int R, int K>
__global__ void __launch_bounds__(kCsrWinThreads, 1)
    k_pass1_csr_win(OpParams op, Win win, int nwin, int64_t ld, int64_t gz, int64_t band, int64_t T,
                    double* __restrict__ Yt, double* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char csr_smraw[];
  const int64_t Wcap = T + 2 * band + 2;
  double* zw = reinterpret_cast<double*>(csr_smraw);                       // R x Wcap
  uint64_t* bar = reinterpret_cast<uint64_t*>(zw + (int64_t)R * Wcap);
  __shared__ double red[kCsrWinWarps * K * R * R];
  double acc[K * R * R];
#pragma unroll
  for (int e = 0; e < K * R * R; ++e) acc[e] = 0.0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int sub = threadIdx.x & (kCsrLanes - 1);
  const int rsub = threadIdx.x / kCsrLanes;
  const double* __restrict__ Zd = win.p[nwin - 1];
  const int64_t n = op.n;
  const int64_t ntiles = (n + T - 1) / T;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * T, i1 = min(n, i0 + T);
    int64_t w0 = max(-gz, i0 - band);
    if ((gz + w0) & 1) --w0;                   // 16-byte aligned source (column data start is)
    int64_t w1 = min(n + gz, i1 + band);
    if ((w1 - w0) & 1) ++w1;                   // whole 16-byte units (the ring is padded)
    __syncthreads();                           // the previous tile's gathers are done
    if (threadIdx.x == 0) {
      const uint64_t bytes = (uint64_t)(w1 - w0) * 8;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(bar)),
                   "r"((uint32_t)(bytes * R))
                   : "memory");
      for (int c = 0; c < R; ++c)
        for (uint64_t off = 0; off < bytes; off += 32768)
          bulk_g2s(reinterpret_cast<char*>(zw + c * Wcap) + off, reinterpret_cast<const char*>(Zd + c * ld + w0) + off,
                   (uint32_t)min((uint64_t)32768, bytes - off), bar);
    }
    {
      uint32_t ok = 0;
      while (!ok) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(phase)
            : "memory");
      }
      phase ^= 1u;
    }
    // row pointers one sweep ahead (the value / index loads of a row depend on them)
    int64_t q0 = (i0 + rsub < i1) ? __ldg(op.rp + i0 + rsub) : 0;
    int64_t q1 = (i0 + rsub < i1) ? __ldg(op.rp + i0 + rsub + 1) : 0;
    for (int64_t rb = i0; rb < i1; rb += kCsrWinRows) {        // block-uniform trip count
      const int64_t row = rb + rsub;
      const bool valid = row < i1;
      const int64_t p0 = q0, p1 = q1;
      {
        const int64_t rn = row + kCsrWinRows;
        q0 = rn < i1 ? __ldg(op.rp + rn) : 0;
        q1 = rn < i1 ? __ldg(op.rp + rn + 1) : 0;
      }
      double y[R];
#pragma unroll
      for (int c = 0; c < R; ++c) y[c] = 0.0;
      // the older window blocks' values of this row, issued with the CSR loads (independent of
      // them: one memory latency per sweep instead of two)
      double zo[K > 1 ? K - 1 : 1][R];
#pragma unroll
      for (int i = 0; i < K - 1; ++i)
#pragma unroll
        for (int a = 0; a < R; ++a) zo[i][a] = (sub == 0 && valid && i < nwin - 1) ? __ldg(win.p[i] + a * ld + row) : 0.0;
      constexpr int kCsrU = 6;
      double av[kCsrU];
      int32_t cl[kCsrU];
#pragma unroll
      for (int u = 0; u < kCsrU; ++u) {
        const int64_t p = p0 + sub + u * kCsrLanes;
        av[u] = p < p1 ? __ldg(op.cv + p) : 0.0;
        cl[u] = p < p1 ? __ldg(op.ci + p) : (int32_t)w0;
      }
#pragma unroll
      for (int u = 0; u < kCsrU; ++u) {
        if (p0 + sub + u * kCsrLanes < p1) {
          const int64_t off = cl[u] - w0;
#pragma unroll
          for (int c = 0; c < R; ++c) y[c] = fma(av[u], zw[c * Wcap + off], y[c]);
        }
      }
      for (int64_t p = p0 + sub + kCsrU * kCsrLanes; p < p1; p += kCsrLanes) {
        const double a = __ldg(op.cv + p);
        const int64_t off = __ldg(op.ci + p) - w0;
#pragma unroll
        for (int c = 0; c < R; ++c) y[c] = fma(a, zw[c * Wcap + off], y[c]);
      }
#pragma unroll
      for (int c = 0; c < R; ++c) {
#pragma unroll
        for (int o = kCsrLanes / 2; o > 0; o >>= 1) y[c] += __shfl_xor_sync(SYLV_FULL_MASK, y[c], o);
      }
      if (sub == 0 && valid) {
        if (Yt) {
#pragma unroll
          for (int c = 0; c < R; ++c) Yt[c * ld + row] = y[c];
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i < nwin) {
            double z[R];
#pragma unroll
            for (int a = 0; a < R; ++a) z[a] = (i == nwin - 1) ? zw[a * Wcap + (row - w0)] : zo[i < K - 1 ? i : 0][a];
#pragma unroll
            for (int a = 0; a < R; ++a)
#pragma unroll
              for (int c = 0; c < R; ++c) acc[(i * R + a) * R + c] = fma(z[a], y[c], acc[(i * R + a) * R + c]);
          }
        }
      }
    }
  }
  // deterministic CTA reduction (fixed warp order)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int e = 0; e < K * R * R; ++e) {
    double s = acc[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(SYLV_FULL_MASK, s, o);
    if (lane == 0) red[warp * K * R * R + e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < K * R * R; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kCsrWinWarps; ++w) s += red[w * K * R * R + e];
    partial[(int64_t)blockIdx.x * K * R * R + e] = s;
  }
}

}  // namespace sylv

namespace sylv {

// =====================================================================================
// SELL-32 copy of a CSR operator (built once at init) for the windowed pass 1
// =====================================================================================
// Slice s holds rows 32 s .. 32 s + 31; its width w_s = max nnz of those rows; entry k of the
// slice's row (32 s + l) is at sptr[s] + 32 k + l (padding: value 0, column = the row itself,
// which always lies in the band window).  A warp then streams a slice with one coalesced
// 256-byte value load and one 128-byte index load per k, lane = row: no per-row shuffles.
__global__ void k_sell_widths(const int64_t* __restrict__ rp, int64_t n, int64_t* __restrict__ width) {
  const int64_t ns = (n + 31) / 32;
  for (int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; sl < ns; sl += (int64_t)gridDim.x * blockDim.x) {
    int64_t w = 0;
    for (int64_t r = sl * 32; r < min(n, sl * 32 + 32); ++r) w = max(w, rp[r + 1] - rp[r]);
    width[sl] = w * 32;
  }
}

// IdxT = int32_t: column indices; IdxT = int16_t: band offsets col - row (k_pass1_sell_ring; the
// caller checks band <= 32767; padding = offset 0)
template <typename IdxT>
__global__ void k_sell_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ cv, int64_t n, const int64_t* __restrict__ sptr,
                            IdxT* __restrict__ sci, double* __restrict__ scv) {
  constexpr bool kOff = sizeof(IdxT) == 2;
  const int64_t ns = (n + 31) / 32;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < ns * 32; row += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sl = row / 32, l = row % 32;
    const int64_t w = (sptr[sl + 1] - sptr[sl]) / 32;
    const int64_t p0 = row < n ? rp[row] : 0, p1 = row < n ? rp[row + 1] : 0;
    const int64_t self = min(row, n - 1);
    for (int64_t k = 0; k < w; ++k) {
      const int64_t p = p0 + k;
      const bool ok = p < p1;
      const int64_t col = ok ? (int64_t)ci[p] : self;
      sci[sptr[sl] + 32 * k + l] = (IdxT)(kOff ? col - self : col);
      scv[sptr[sl] + 32 * k + l] = ok ? cv[p] : 0.0;
    }
  }
}

// Windowed pass 1 on the SELL-32 copy: CTA = tiles of T rows (T multiple of 32), band window of
// Z_d in shared memory (bulk copies, as k_pass1_csr_win), warp = slice, lane = row.
// kSellNE slice entries (value + column index) in flight per lane (A/B: -DSYLV_SELL_NE=8,
// -DSYLV_SELL_THREADS=512 — fewer warps with more registers each)
#ifndef SYLV_SELL_THREADS
#define SYLV_SELL_THREADS 1024
#endif
#ifndef SYLV_SELL_NE
#define SYLV_SELL_NE 4
#endif
constexpr int kSellThreads = SYLV_SELL_THREADS;
constexpr int kSellWarps = kSellThreads / 32;
constexpr int kSellNE = SYLV_SELL_NE;
template <int R, int K>
__global__ void __launch_bounds__(kSellThreads, 1)
    k_pass1_sell_win(OpParams op, Win win, int nwin, int64_t ld, int64_t gz, int64_t band, int64_t T,
                     const int64_t* __restrict__ sptr, const int32_t* __restrict__ sci,
                     const double* __restrict__ scv, double* __restrict__ Yt, double* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char sell_smraw[];
  const int64_t Wcap = T + 2 * band + 2;
  double* zw = reinterpret_cast<double*>(sell_smraw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(zw + (int64_t)R * Wcap);
  __shared__ double red[kSellWarps * K * R * R];
  double acc[K * R * R];
#pragma unroll
  for (int e = 0; e < K * R * R; ++e) acc[e] = 0.0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* __restrict__ Zd = win.p[nwin - 1];
  const int64_t n = op.n;
  const int64_t ntiles = (n + T - 1) / T;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * T, i1 = min(n, i0 + T);
    int64_t w0 = max(-gz, i0 - band);
    if ((gz + w0) & 1) --w0;
    int64_t w1 = min(n + gz, i1 + band);
    if ((w1 - w0) & 1) ++w1;
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t bytes = (uint64_t)(w1 - w0) * 8;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(bar)),
                   "r"((uint32_t)(bytes * R))
                   : "memory");
      for (int c = 0; c < R; ++c)
        for (uint64_t off = 0; off < bytes; off += 32768)
          bulk_g2s(reinterpret_cast<char*>(zw + c * Wcap) + off, reinterpret_cast<const char*>(Zd + c * ld + w0) + off,
                   (uint32_t)min((uint64_t)32768, bytes - off), bar);
    }
    {
      uint32_t ok = 0;
      while (!ok) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(phase)
            : "memory");
      }
      phase ^= 1u;
    }
    for (int64_t sl = i0 / 32 + warp; sl * 32 < i1; sl += kSellWarps) {
      const int64_t row = sl * 32 + lane;
      const bool valid = row < i1;
      // window blocks' values of this row (independent of the slice stream)
      double zo[K > 1 ? K - 1 : 1][R];
#pragma unroll
      for (int i = 0; i < K - 1; ++i)
#pragma unroll
        for (int a = 0; a < R; ++a) zo[i][a] = (valid && i < nwin - 1) ? __ldg(win.p[i] + a * ld + row) : 0.0;
      const int64_t b0 = __ldg(sptr + sl), b1 = __ldg(sptr + sl + 1);
      double y[R];
#pragma unroll
      for (int c = 0; c < R; ++c) y[c] = 0.0;
      int64_t p = b0 + lane;
      for (; p + (kSellNE - 1) * 32 < b1; p += kSellNE * 32) {   // kSellNE entries in flight
        double v[kSellNE];
        int32_t cl[kSellNE];
#pragma unroll
        for (int u = 0; u < kSellNE; ++u) {
          v[u] = __ldg(scv + p + 32 * u);
          cl[u] = __ldg(sci + p + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < kSellNE; ++u) {
          const int64_t off = cl[u] - w0;
#pragma unroll
          for (int c = 0; c < R; ++c) y[c] = fma(v[u], zw[c * Wcap + off], y[c]);
        }
      }
      for (; p < b1; p += 32) {
        const double v = __ldg(scv + p);
        const int64_t off = __ldg(sci + p) - w0;
#pragma unroll
        for (int c = 0; c < R; ++c) y[c] = fma(v, zw[c * Wcap + off], y[c]);
      }
      if (valid) {
        if (Yt) {
#pragma unroll
          for (int c = 0; c < R; ++c) Yt[c * ld + row] = y[c];
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i < nwin) {
            double z[R];
#pragma unroll
            for (int a = 0; a < R; ++a) z[a] = (i == nwin - 1) ? zw[a * Wcap + (row - w0)] : zo[i < K - 1 ? i : 0][a];
#pragma unroll
            for (int a = 0; a < R; ++a)
#pragma unroll
              for (int c = 0; c < R; ++c) acc[(i * R + a) * R + c] = fma(z[a], y[c], acc[(i * R + a) * R + c]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < K * R * R; ++e) {
    double s = acc[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(SYLV_FULL_MASK, s, o);
    if (lane == 0) red[warp * K * R * R + e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < K * R * R; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kSellWarps; ++w) s += red[w * K * R * R + e];
    partial[(int64_t)blockIdx.x * K * R * R + e] = s;
  }
}

// Sliding-ring pass 1 on the SELL-32 copy (round 2, default when two tiles and the band fit):
// a CTA owns a CONTIGUOUS range of slices, so the band window of Z_d slides: only the T new rows
// of the next tile are loaded (the static-window kernel reloads T + 2 band rows per tile, 2.4x at
// c4, and waits for them).  Z_d lives in a shared-memory ring of `cap` rows per column, row
// u = i + gz at position u mod cap; 2 T + 2 band + 2 <= cap, so the rows of tile i + 1 arrive
// (cp.async.bulk on full[(i+1)&1]) while tile i is streamed.  No CTA-wide barrier in the loop:
// every warp arrives on done[i&1] after its slices of tile i; warp 0 waits for done(i-1) — all
// warps are past the rows tile i + 1 overwrites — before it issues that load.  Warp w streams
// slices s0 + w + 32 k in order; a tile is T/32 consecutive slices (T a multiple of 1024: the same
// number of slices per warp and tile).  Column indices are 16-bit band offsets (col - row):
// 10 instead of 12 bytes per stored entry.
__device__ __forceinline__ void sell_mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity)
        : "memory");
  }
}

template <int R, int K>
__global__ void __launch_bounds__(kSellThreads, 1)
    k_pass1_sell_ring(OpParams op, Win win, int nwin, int64_t ld, int64_t gz, int64_t band, int T, int cap,
                      const int64_t* __restrict__ sptr, const int16_t* __restrict__ soff,
                      const double* __restrict__ scv, double* __restrict__ Yt, double* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char sell_smraw[];
  double* zw = reinterpret_cast<double*>(sell_smraw);                    // [R][cap]
  uint64_t* full = reinterpret_cast<uint64_t*>(zw + (int64_t)R * cap);   // [2]
  uint64_t* done = full + 2;                                             // [2]
  __shared__ double red[kSellWarps * K * R * R];
  double acc[K * R * R];
#pragma unroll
  for (int e = 0; e < K * R * R; ++e) acc[e] = 0.0;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(full + b)) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(done + b)),
                   "r"(kSellWarps)
                   : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* __restrict__ Zs = win.p[nwin - 1] - gz;   // row u = i + gz >= 0; Zs 16-byte aligned, ld even
  const int64_t n = op.n;
  const int64_t ns = (n + 31) / 32;
  const int64_t s0 = ns * blockIdx.x / gridDim.x, s1 = ns * (blockIdx.x + 1) / gridDim.x;
  const int Ts = T / 32;
  const int nt = (int)((s1 - s0 + Ts - 1) / Ts);
  const int64_t utop = n + 2 * gz;
  // window of tile i in u coordinates: [ulo(i), uhi(i)), even bounds
  auto ulo = [&](int i) -> int64_t { return max((int64_t)0, (s0 + (int64_t)i * Ts) * 32 + gz - band) & ~(int64_t)1; };
  auto uhi = [&](int i) -> int64_t {
    const int64_t h = min(utop, min(s1, s0 + (int64_t)(i + 1) * Ts) * 32 + gz + band);
    return h + (h & 1);
  };
  // rows [a, b) of every column into the ring, completing on bar (thread 0)
  auto load = [&](int64_t a, int64_t b, uint64_t* bar) {
    const uint32_t tx = (uint32_t)((b - a) * 8 * R);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(tx)
                 : "memory");
    int64_t u = a;
    while (u < b) {
      const int64_t pos = u % cap;
      const int64_t len = min(min(b - u, (int64_t)cap - pos), (int64_t)4096);   // <= 32 KB per copy
      for (int c = 0; c < R; ++c)
        bulk_g2s(zw + (int64_t)c * cap + pos, Zs + (int64_t)c * ld + u, (uint32_t)(len * 8), bar);
      u += len;
    }
  };
  if (nt > 0 && threadIdx.x == 0) load(ulo(0), uhi(0), full);
  for (int i = 0; i < nt; ++i) {
    if (warp == 0 && i + 1 < nt) {
      if (i >= 1) sell_mbar_wait(done + ((i - 1) & 1), (uint32_t)(((i - 1) >> 1) & 1));
      if (lane == 0) load(uhi(i), uhi(i + 1), full + ((i + 1) & 1));
      __syncwarp();
    }
    sell_mbar_wait(full + (i & 1), (uint32_t)((i >> 1) & 1));
    const int64_t lo = ulo(i);
    const int plo = (int)(lo % cap);
    const int64_t sle = min(s1, s0 + (int64_t)(i + 1) * Ts);
    for (int64_t sl = s0 + (int64_t)i * Ts + warp; sl < sle; sl += kSellWarps) {
      const int64_t row = sl * 32 + lane;
      const bool valid = row < n;
      double zo[K > 1 ? K - 1 : 1][R];
#pragma unroll
      for (int i2 = 0; i2 < K - 1; ++i2)
#pragma unroll
        for (int a = 0; a < R; ++a) zo[i2][a] = (valid && i2 < nwin - 1) ? __ldg(win.p[i2] + a * ld + row) : 0.0;
      const int64_t b0 = __ldg(sptr + sl), b1 = __ldg(sptr + sl + 1);
      // ring position of this lane's own row (padding rows of the last slice: row n - 1)
      const int rb = plo + (int)(min(row, n - 1) + gz - lo);
      double y[R];
#pragma unroll
      for (int c = 0; c < R; ++c) y[c] = 0.0;
      int64_t p = b0 + lane;
      for (; p + (kSellNE - 1) * 32 < b1; p += kSellNE * 32) {   // kSellNE entries in flight
        double v[kSellNE];
        int cl[kSellNE];
#pragma unroll
        for (int u = 0; u < kSellNE; ++u) {
          v[u] = __ldg(scv + p + 32 * u);
          cl[u] = (int)__ldg(soff + p + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < kSellNE; ++u) {
          int off = rb + cl[u];
          off -= off >= cap ? cap : 0;
#pragma unroll
          for (int c = 0; c < R; ++c) y[c] = fma(v[u], zw[c * cap + off], y[c]);
        }
      }
      for (; p < b1; p += 32) {
        const double v = __ldg(scv + p);
        int off = rb + (int)__ldg(soff + p);
        off -= off >= cap ? cap : 0;
#pragma unroll
        for (int c = 0; c < R; ++c) y[c] = fma(v, zw[c * cap + off], y[c]);
      }
      if (valid) {
        if (Yt) {
#pragma unroll
          for (int c = 0; c < R; ++c) Yt[c * ld + row] = y[c];
        }
        const int own = rb - (rb >= cap ? cap : 0);
#pragma unroll
        for (int i2 = 0; i2 < K; ++i2) {
          if (i2 < nwin) {
            double z[R];
#pragma unroll
            for (int a = 0; a < R; ++a) z[a] = (i2 == nwin - 1) ? zw[a * cap + own] : zo[i2 < K - 1 ? i2 : 0][a];
#pragma unroll
            for (int a = 0; a < R; ++a)
#pragma unroll
              for (int c = 0; c < R; ++c) acc[(i2 * R + a) * R + c] = fma(z[a], y[c], acc[(i2 * R + a) * R + c]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(done + (i & 1))) : "memory");
  }
#pragma unroll
  for (int e = 0; e < K * R * R; ++e) {
    double s = acc[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(SYLV_FULL_MASK, s, o);
    if (lane == 0) red[warp * K * R * R + e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < K * R * R; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kSellWarps; ++w) s += red[w * K * R * R + e];
    partial[(int64_t)blockIdx.x * K * R * R + e] = s;
  }
}

}  // namespace sylv
