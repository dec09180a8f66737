// sspace.cuh — coefficient kernels (one CTA) and sketch-space QR update kernels
// (SURVEY §8(a) rows a2/a3 coefficients and a5; Alg. 1 line 9).
//
// Sketch-space data: Q (s x m, column-major, ld = s, orthonormal columns), T (mT x mT,
// column-major, upper triangular), w (s x R row-major, the new sketched block).
// The update is block CGS2:  c1 = Q^T w, w -= Q c1, c2 = Q^T w, w -= Q c2,
// w = q tau (CholQR2, positive diagonal), T_H = c1 + c2  (R7).
#pragma once
#include "common.cuh"

namespace sylv {

// Deterministic column sums of per-CTA partials: out[e] = sum_p partial[p*len + e].
__device__ __forceinline__ double sum_parts(const double* __restrict__ partial, int nparts,
                                            int64_t len, int64_t e) {
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += partial[(int64_t)p * len + e];
  return s;
}

// Block-wide deterministic sums of per-CTA partials: out[e] = sum_p partial[p*len + e] for
// e < nelem.  Warp w reduces elements w, w + nwarps, ...; lane l adds parts l, l + 32, ...
// and the 32 lane sums are combined by a fixed butterfly (same order on every run).
__device__ __forceinline__ void block_sum_parts(const double* __restrict__ partial, int nparts, int64_t len,
                                                int nelem, double* __restrict__ out) {
  // nc chunks of parts per element, one thread per (element, chunk) — coalesced over the
  // elements, 8 independent loads in flight per thread — then the chunk sums in chunk order
  // (fixed order: deterministic).  Launched with kSmallThreads threads; nelem <= len <=
  // kMaxK R^2.  The chunking depends on len, not nelem, so a sum over all len elements
  // (k_sum_partials, sharded contexts) adds each element in the same order as a sum over a
  // prefix (k_coef1 with nwin < K): bit-identical results.
  __shared__ double acc[kSmallThreads];
  const int nt = blockDim.x;
  const int nc = max(1, min(nt / (len > 0 ? (int)len : 1), nparts));
  for (int idx = threadIdx.x; idx < nelem * nc; idx += nt) {
    const int e = idx % nelem, c = idx / nelem;
    double s = 0.0;
#pragma unroll 8
    for (int p = c; p < nparts; p += nc) s += partial[(int64_t)p * len + e];
    acc[idx] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nelem; e += nt) {
    double s = 0.0;
    for (int c = 0; c < nc; ++c) s += acc[c * nelem + e];
    out[e] = s;
  }
}

// h_{i,j} = R_i^T P_i R_j, K_i = R_i h_{i,j}; Kc[j] = [R_j, K_0..]; Hc[j] = [h_.., 0.., h_{j+1,j}]
// (one CTA; thread per matrix entry for the r x r products)
template <int R, int K>
__global__ void __launch_bounds__(kSmallThreads) k_coef1(const double* __restrict__ partial, int nparts, int nwin, int j,
                        const double* __restrict__ Rall, double* __restrict__ Kc,
                        double* __restrict__ Hc, double* __restrict__ hnorm2) {
  constexpr int RR = R * R;
  __shared__ double P[K * RR], T1[K * RR], Hs[K * RR];
  block_sum_parts(partial, nparts, K * RR, nwin * RR, P);
  __syncthreads();
  const double* Rd = Rall + (int64_t)j * RR;
  double* Kout = Kc + (int64_t)j * (1 + K) * RR;
  double* Hout = Hc + (int64_t)j * (K + 1) * RR;
  for (int e = threadIdx.x; e < K * RR; e += blockDim.x) {      // T1_i = R_i^T P_i
    const int i = e / RR, a = (e % RR) / R, c = e % R;
    double v = 0.0;
    if (i < nwin) {
      const double* Ri = Rall + (int64_t)(j - nwin + 1 + i) * RR;
      for (int p = 0; p < R; ++p) v += Ri[p * R + a] * P[i * RR + p * R + c];
    }
    T1[e] = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < K * RR; e += blockDim.x) {      // h_i = T1_i R_d
    const int i = e / RR, a = (e % RR) / R, c = e % R;
    double v = 0.0;
    if (i < nwin)
      for (int p = 0; p < R; ++p) v += T1[i * RR + a * R + p] * Rd[p * R + c];
    Hs[e] = v;
    Hout[e] = v;
  }
  for (int e = threadIdx.x; e < RR; e += blockDim.x) Kout[e] = Rd[e];
  __syncthreads();
  for (int e = threadIdx.x; e < K * RR; e += blockDim.x) {      // K_i = R_i h_i
    const int i = e / RR, a = (e % RR) / R, c = e % R;
    double v = 0.0;
    if (i < nwin) {
      const double* Ri = Rall + (int64_t)(j - nwin + 1 + i) * RR;
      for (int p = 0; p < R; ++p) v += Ri[a * R + p] * Hs[i * RR + p * R + c];
    }
    Kout[RR + e] = v;
  }
  if (threadIdx.x < 32) {                                       // ||h_{.,j}||_F^2, fixed order
    double hn = 0.0;
    for (int e = threadIdx.x; e < nwin * RR; e += 32) hn += Hs[e] * Hs[e];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) hn += __shfl_xor_sync(SYLV_FULL_MASK, hn, off);
    if (threadIdx.x == 0) hnorm2[j] = hn;
  }
}

// Warp-cooperative Cholesky G = U^T U (upper, positive diagonal) and V = U^{-1}, R <= 8, run by
// one full warp: lane j < R keeps column j of U in registers; row k of U needs the column-k
// entries above it, broadcast by shuffles (R^2/2 shuffles, no serial thread-0 loops).  U, V:
// R x R row-major in shared memory.  Returns false (on every lane) when G is not positive
// definite; U = V = I then.
template <int R>
__device__ __forceinline__ bool warp_chol_inv(const double* G, double* U, double* V) {
  const int lane = threadIdx.x & 31;
  const int jj = lane < R ? lane : 0;
  double u[R];
#pragma unroll
  for (int p = 0; p < R; ++p) u[p] = 0.0;
  bool ok = true;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    double t = G[k * R + jj];
#pragma unroll
    for (int p = 0; p < k; ++p) t -= __shfl_sync(SYLV_FULL_MASK, u[p], k) * u[p];   // U[p][k] U[p][j]
    const double dk = __shfl_sync(SYLV_FULL_MASK, t, k);
    if (!(dk > 0.0)) ok = false;                       // warp-uniform
    const double d = ok ? sqrt(dk) : 1.0;
    u[k] = (jj == k) ? d : (jj > k ? t / d : 0.0);
  }
  if (!ok) {
#pragma unroll
    for (int p = 0; p < R; ++p) u[p] = (p == jj) ? 1.0 : 0.0;
  }
  if (lane < R)
#pragma unroll
    for (int p = 0; p < R; ++p) U[p * R + lane] = u[p];
  __syncwarp();
  // column j of V by back substitution: V[j][j] = 1/U[j][j], V[i][j] = -sum_{p=i+1..j} U[i][p] V[p][j] / U[i][i]
  if (lane < R) {
    double v[R];
#pragma unroll
    for (int i = R - 1; i >= 0; --i) {
      double val = 0.0;
      if (i == lane) {
        val = 1.0 / U[i * R + i];
      } else if (i < lane) {
        double s = 0.0;
#pragma unroll
        for (int p = i + 1; p < R; ++p)
          if (p <= lane) s += U[i * R + p] * v[p];
        val = -s / U[i * R + i];
      }
      v[i] = val;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) V[i * R + lane] = v[i];
  }
  __syncwarp();
  return ok;
}

// G = W'^T W' -> h_{j+1,j} = chol(G) (upper, positive diagonal), R_{j+1} = h^{-1};
// breakdown flag (bit 0) if min diag h <= 1e-14 ||W~||_F  (R11), with
// ||W~||_F^2 = ||W'||_F^2 + sum_i ||h_{i,j}||_F^2 (window orthonormal); bit 1 if G not PD.
template <int R, int K>
__global__ void __launch_bounds__(kSmallThreads) k_coef2(const double* __restrict__ partial, int nparts, int j,
                        double* __restrict__ Rall, double* __restrict__ Hc,
                        const double* __restrict__ hnorm2, int* __restrict__ flags) {
  __shared__ double G[R * R], h[R * R], hi[R * R];
  block_sum_parts(partial, nparts, R * R, R * R, G);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const bool ok = warp_chol_inv<R>(G, h, hi);
  if (threadIdx.x != 0) {
    double* Hout = Hc + (int64_t)j * (K + 1) * R * R + K * R * R;
    double* Rn = Rall + (int64_t)(j + 1) * R * R;
    for (int e = threadIdx.x - 1; e < R * R; e += 31) {
      Hout[e] = h[e];
      Rn[e] = hi[e];
    }
    return;
  }
  int fl = ok ? 0 : 2;
  double tr = 0.0, mind = 1e300;
  for (int a = 0; a < R; ++a) {
    tr += G[a * R + a];
    mind = fmin(mind, h[a * R + a]);
  }
  const double wn = sqrt(tr + hnorm2[j]);
  if (mind <= 1e-14 * wn) fl |= 1;
  if (fl) atomicOr(flags + j, fl);
}

// tau = chol(sum of Gram partials) (upper); tinv = tau^{-1}; if prev: tau_out = tau * prev.
// Sets flags[slot] bit 2 if not positive definite (lost independence).
template <int R>
__global__ void __launch_bounds__(kSmallThreads) k_chol_small(const double* __restrict__ partial, int nparts,
                             double* __restrict__ tau_out, double* __restrict__ tinv_out,
                             const double* __restrict__ prev, int* __restrict__ flags, int slot) {
  __shared__ double G[R * R], t[R * R], ti[R * R];
  block_sum_parts(partial, nparts, R * R, R * R, G);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const bool ok = warp_chol_inv<R>(G, t, ti);
  if (!ok && threadIdx.x == 0) atomicOr(flags + slot, 4);
  for (int e = threadIdx.x; e < R * R; e += 32) {
    tinv_out[e] = ti[e];
    if (prev) {
      const int a = e / R, c = e % R;
      double sacc = 0.0;
      for (int p = 0; p < R; ++p) sacc += t[a * R + p] * prev[p * R + c];   // (t prev)[a][c]
      tau_out[e] = sacc;
    } else {
      tau_out[e] = t[e];
    }
  }
}

// out = A M for a rows x R row-major A; if colmajor_ld > 0 the result is written
// column-major (out[c*ld + row], the Q layout), else row-major.
template <int R>
__global__ void __launch_bounds__(kThreads) k_rmul(int64_t rows, const double* __restrict__ A,
                                                   const double* __restrict__ M, double* __restrict__ out,
                                                   int64_t colmajor_ld) {
  __shared__ double ms[R * R];
  if (threadIdx.x < R * R) ms[threadIdx.x] = M[threadIdx.x];
  __syncthreads();
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < rows * R;
       e += (int64_t)gridDim.x * kThreads) {
    const int64_t row = e / R;
    const int c = (int)(e - row * R);
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a) s = fma(A[row * R + a], ms[a * R + c], s);
    if (colmajor_ld > 0)
      out[(int64_t)c * colmajor_ld + row] = s;
    else
      out[e] = s;
  }
}

// partial[(rt*m + j)*R + c] = sum_{rows in tile rt} Q[j*s + row] w[row*R + c]   (a5: Q^T w)
//
// One CTA per (row tile of qtw_tile<R>() rows, group of kQtwCols columns).  The tile of w is staged
// once in shared memory, column-major (lane-consecutive rows: conflict-free reads), so every
// element of w is read from L2 once per column group instead of once per column; each warp
// register-blocks kQtwU columns (kQtwU coalesced 256-byte Q loads per 32 rows, R FMAs per
// loaded w value and column) and reduces its kQtwU x R sums by a fixed shuffle tree at the end
// of the tile (deterministic).  Q (s x m, column-major) is read exactly once from HBM.
template <int R> constexpr int qtw_tile() { return 4096 / R; }   // rows per tile (w tile: 32 KB)
constexpr int kQtwU = 4;                       // columns per warp and pass
constexpr int kQtwCols = kWarps * kQtwU * 2;   // columns per CTA (two passes of the warps)
// Q may be any column-major matrix of `s` rows with column stride ldq (the sketched basis:
// ldq = s; the retained n-space basis of the full method: ldq = the SoA block stride).  A CTA
// processes `tpc` consecutive row tiles of its row chunk (blockIdx.y), keeping its column sums
// in registers across them, so the partials stay small when s is large.
template <int R>
__global__ void __launch_bounds__(kThreads, 2) k_qtw(const double* __restrict__ Q, int64_t s, int64_t ldq, int m,
                                                  const double* __restrict__ w, int64_t tile, int tpc,
                                                  double* __restrict__ partial) {
  __shared__ double ws[R][qtw_tile<R>() + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rt = blockIdx.y;
  for (int pass = 0; pass < 2; ++pass) {
    const int j0 = blockIdx.x * kQtwCols + pass * kWarps * kQtwU + warp * kQtwU;
    double acc[kQtwU][R];
#pragma unroll
    for (int u = 0; u < kQtwU; ++u)
#pragma unroll
      for (int c = 0; c < R; ++c) acc[u][c] = 0.0;
   for (int tt = 0; tt < tpc; ++tt) {
    const int64_t r0 = ((int64_t)rt * tpc + tt) * tile;
    if (r0 >= s) break;                                   // block-uniform
    const int nr = (int)(tile < s - r0 ? tile : s - r0);
    __syncthreads();                                      // previous tile's readers done
    for (int e = threadIdx.x; e < nr * R; e += kThreads) ws[e % R][e / R] = __ldg(w + r0 * R + e);
    __syncthreads();
    if (j0 >= m) continue;                                // (no early exit: barriers above)
    const double* __restrict__ q0 = Q + r0;
    const double* __restrict__ qc[kQtwU];
#pragma unroll
    for (int u = 0; u < kQtwU; ++u) qc[u] = q0 + (int64_t)min(j0 + u, m - 1) * ldq;   // clamped: zero-weighted below
    // 4 row strides of kQtwU loads in flight per warp (HBM latency x bandwidth)
    int row = lane;
    for (; row + 96 < nr; row += 128) {
      double qv[4][kQtwU];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int u = 0; u < kQtwU; ++u) qv[i][u] = __ldg(qc[u] + row + 32 * i);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < R; ++c) {
          const double wv = ws[c][row + 32 * i];
#pragma unroll
          for (int u = 0; u < kQtwU; ++u) acc[u][c] = fma(qv[i][u], wv, acc[u][c]);
        }
    }
    for (; row < nr; row += 32) {
      double qv[kQtwU];
#pragma unroll
      for (int u = 0; u < kQtwU; ++u) qv[u] = __ldg(qc[u] + row);
#pragma unroll
      for (int c = 0; c < R; ++c) {
        const double wv = ws[c][row];
#pragma unroll
        for (int u = 0; u < kQtwU; ++u) acc[u][c] = fma(qv[u], wv, acc[u][c]);
      }
    }
   }
    if (j0 >= m) continue;
#pragma unroll
    for (int u = 0; u < kQtwU; ++u)
#pragma unroll
      for (int c = 0; c < R; ++c) {
        double v = acc[u][c];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(SYLV_FULL_MASK, v, off);
        acc[u][c] = v;
      }
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < kQtwU; ++u)
        if (j0 + u < m)
#pragma unroll
          for (int c = 0; c < R; ++c) partial[((int64_t)rt * m + j0 + u) * R + c] = acc[u][c];
    }
  }
}

// out[e] = sum_rt partial[rt*len + e]  (+ optional accumulation into acc_out: acc_out[e] += out[e])
__global__ void k_red_parts(const double* __restrict__ partial, int nparts, int64_t len,
                            double* __restrict__ out, double* __restrict__ acc_out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = sum_parts(partial, nparts, len, e);
    out[e] = v;
    if (acc_out) acc_out[e] += v;
  }
}

// The same sum for many parts (the row-split Q^T w sweeps at small m: ~200 parts of a few
// hundred elements): a CTA takes 32 consecutive elements (lane = element, coalesced) and
// blockDim / 32 part chunks (warp c sums parts c, c + nc, ... in order), then the chunk sums
// in chunk order — a fixed order, deterministic.  blockDim = 32 * nc, nc <= 32.
__global__ void k_red_parts_wide(const double* __restrict__ partial, int nparts, int64_t len,
                                 double* __restrict__ out, double* __restrict__ acc_out) {
  __shared__ double sm[32][33];
  const int lane = threadIdx.x & 31, ci = threadIdx.x >> 5, nc = blockDim.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (e < len) {
#pragma unroll 8
    for (int p = ci; p < nparts; p += nc) s += __ldg(partial + (int64_t)p * len + e);
  }
  sm[ci][lane] = s;
  __syncthreads();
  if (ci == 0 && e < len) {
    double v = 0.0;
    for (int c = 0; c < nc; ++c) v += sm[c][lane];
    out[e] = v;
    if (acc_out) acc_out[e] += v;
  }
}

// acc[e] += x[e]  (sharded sketch space: csum += the rank-summed c2)
__global__ void k_axpy_inplace(const double* __restrict__ x, double* __restrict__ acc, int64_t len) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x)
    acc[e] += x[e];
}

// partial2[(cc*s + row)*R + c] = sum_{j in chunk cc} Q[j*s + row] cvec[j*R + c]
template <int R>
__global__ void __launch_bounds__(kThreads) k_qc_part(const double* __restrict__ Q, int64_t s, int64_t ldq, int m,
                                                      const double* __restrict__ cvec, int cols_per_chunk,
                                                      double* __restrict__ partial2) {
  constexpr int kStage = 256;
  __shared__ double cs[kStage * R];
  const int cc = blockIdx.y;
  const int j0 = cc * cols_per_chunk;
  const int j1 = min(m, j0 + cols_per_chunk);
  const int64_t row = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  double acc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.0;
  for (int jj = j0; jj < j1; jj += kStage) {
    const int nj = min(kStage, j1 - jj);
    __syncthreads();
    for (int e = threadIdx.x; e < nj * R; e += kThreads) cs[e] = cvec[(int64_t)jj * R + e];
    __syncthreads();
    if (row < s) {
      const double* __restrict__ q = Q + (int64_t)jj * ldq + row;
      int t = 0;
      for (; t + 8 <= nj; t += 8) {          // 8 column loads in flight per thread
        double qv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) qv[u] = __ldg(q + (int64_t)(t + u) * ldq);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int c = 0; c < R; ++c) acc[c] = fma(qv[u], cs[(t + u) * R + c], acc[c]);
      }
      for (; t < nj; ++t) {
        const double qv = __ldg(q + (int64_t)t * ldq);
#pragma unroll
        for (int c = 0; c < R; ++c) acc[c] = fma(qv, cs[t * R + c], acc[c]);
      }
    }
  }
  if (row < s) {
#pragma unroll
    for (int c = 0; c < R; ++c) partial2[((int64_t)cc * s + row) * R + c] = acc[c];
  }
}

// ---- Tensor-core (DMMA) sweeps of Q for R >= 4 (round 2): the two products of a CGS2 sweep
// are (m x s)(s x R) and (s x m)(m x R) contractions with R <= 8 = the DMMA n width, so one
// mma.sync.m8n8k4.f64 does 8 x 8 x 4 FMAs and every lane loads one 32-byte run of one Q column
// per four DMMAs (the k index of a fragment is free: lane l's four consecutive rows are the k
// slots t = 0..3 of four DMMAs).  Few registers per lane (accumulators are 2 doubles per 8 x 8
// tile), so two row steps of loads stay in flight per lane; Q is read exactly once, coalesced
// (a warp's loads cover 256-byte runs of 4 columns / 32 rows).  Requires ldq % 4 == 0 and a
// 32-byte aligned Q (checked by the caller).  Deterministic: fixed summation order per lane.

// partial[(rt*m + j)*R + c] = sum_{rows of chunk rt} Q[j*ldq + row] w[row*R + c]
// Warp = (32 columns j0..j0+31 = four 8-column tiles, one row chunk); CTA = 8 warps on 256
// consecutive columns of the same row chunk (they share w's rows through L1).
template <int R>
__global__ void __launch_bounds__(kThreads, 2) k_qtw_mma(const double* __restrict__ Q, int64_t s, int64_t ldq, int m,
                                                      const double* __restrict__ w, int64_t chunk,
                                                      double* __restrict__ partial) {
  static_assert(R >= 4 && R <= 8, "DMMA sweep: R in 4..8");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q4 = lane & 3, mc = lane >> 2;
  const int rt = blockIdx.y;
  const int j0 = (blockIdx.x * kWarps + warp) * 32;
  if (j0 >= m) return;                                 // warp-uniform (no barriers below)
  const int64_t r0 = (int64_t)rt * chunk;
  const int64_t r1 = r0 + chunk < s ? r0 + chunk : s;
  const double* __restrict__ qc[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) qc[u] = Q + (int64_t)min(j0 + 8 * u + mc, m - 1) * ldq;   // clamped: dropped below
  const bool wl = mc < R;
  double acc[4][2];
#pragma unroll
  for (int u = 0; u < 4; ++u) acc[u][0] = acc[u][1] = 0.0;
  int64_t k0 = r0;
  for (; k0 + 32 <= r1; k0 += 32) {                    // two 16-row steps in flight
    double2 qa[2][4][2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2* p = reinterpret_cast<const double2*>(qc[u] + k0 + 16 * h + 4 * q4);
        qa[h][u][0] = __ldg(p);
        qa[h][u][1] = __ldg(p + 1);
      }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t rb = k0 + 16 * h + 4 * q4;
      double wb[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) wb[t] = wl ? __ldg(w + (rb + t) * R + mc) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        dmma(acc[u], qa[h][u][0].x, wb[0]);
        dmma(acc[u], qa[h][u][0].y, wb[1]);
        dmma(acc[u], qa[h][u][1].x, wb[2]);
        dmma(acc[u], qa[h][u][1].y, wb[3]);
      }
    }
  }
  for (; k0 < r1; k0 += 16) {                          // ragged tail: guarded scalar loads
    const int64_t rb = k0 + 4 * q4;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const bool in = rb + t < r1;
      const double wv = (in && wl) ? __ldg(w + (rb + t) * R + mc) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma(acc[u], in ? __ldg(qc[u] + rb + t) : 0.0, wv);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = j0 + 8 * u + mc;
    if (j < m) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (2 * q4 + e < R) partial[((int64_t)rt * m + j) * R + 2 * q4 + e] = acc[u][e];
    }
  }
}

// partial2[(cc*s + row)*R + c] = sum_{j in chunk cc} Q[j*ldq + row] cvec[j*R + c]
// Warp = 32 rows x one column chunk (blockIdx.y); DMMA t covers rows i0 + 4 m + t (m = 0..7),
// k = 4 consecutive columns: lane l loads rows i0 + 4 (l>>2) .. +3 of column j + (l&3).
template <int R>
__global__ void __launch_bounds__(kThreads) k_qc_mma(const double* __restrict__ Q, int64_t s, int64_t ldq, int m,
                                                     const double* __restrict__ cvec, int cols_per_chunk,
                                                     double* __restrict__ partial2) {
  static_assert(R >= 4 && R <= 8, "DMMA sweep: R in 4..8");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q4 = lane & 3, mr = lane >> 2;
  const int cc = blockIdx.y;
  const int ja = cc * cols_per_chunk;
  const int jb = min(m, ja + cols_per_chunk);
  const int64_t i0 = ((int64_t)blockIdx.x * kWarps + warp) * 32;
  if (i0 >= s) return;                                 // warp-uniform
  const int64_t rb = i0 + 4 * mr;
  const bool full = rb + 4 <= s;
  const bool cl = mr < R;                              // B fragment: c = l>>2
  double acc[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = 0.0;
  int j = ja;
  for (; j + 16 <= jb; j += 16) {                      // four 4-column steps in flight
    double2 qa[4][2];
    double bv[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const double* col = Q + (int64_t)(j + 4 * h + q4) * ldq + rb;
      if (full) {
        qa[h][0] = __ldg(reinterpret_cast<const double2*>(col));
        qa[h][1] = __ldg(reinterpret_cast<const double2*>(col) + 1);
      } else {
        qa[h][0].x = rb < s ? __ldg(col) : 0.0;
        qa[h][0].y = rb + 1 < s ? __ldg(col + 1) : 0.0;
        qa[h][1].x = rb + 2 < s ? __ldg(col + 2) : 0.0;
        qa[h][1].y = rb + 3 < s ? __ldg(col + 3) : 0.0;
      }
      bv[h] = cl ? __ldg(cvec + (int64_t)(j + 4 * h + q4) * R + mr) : 0.0;
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      dmma(acc[0], qa[h][0].x, bv[h]);
      dmma(acc[1], qa[h][0].y, bv[h]);
      dmma(acc[2], qa[h][1].x, bv[h]);
      dmma(acc[3], qa[h][1].y, bv[h]);
    }
  }
  for (; j < jb; j += 4) {                             // ragged column tail
    const int jj = j + q4;
    const bool in = jj < jb;
    const double* col = Q + (int64_t)(in ? jj : ja) * ldq + rb;
    double a[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) a[t] = (in && rb + t < s) ? __ldg(col + t) : 0.0;
    const double bvv = (in && cl) ? __ldg(cvec + (int64_t)jj * R + mr) : 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) dmma(acc[t], a[t], bvv);
  }
  // D_t[mr'][c]: row i0 + 4 (lane>>2) + t, columns c = 2 (lane&3) + e
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int64_t row = i0 + 4 * mr + t;
    if (row < s) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (2 * q4 + e < R) partial2[((int64_t)cc * s + row) * R + 2 * q4 + e] = acc[t][e];
    }
  }
}

// w[row*R + c] -= sum_cc partial2[(cc*s + row)*R + c]
__global__ void k_wsub(double* __restrict__ w, const double* __restrict__ partial2, int ncc,
                       int64_t len) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < ncc; ++p) s += partial2[(int64_t)p * len + e];
    w[e] -= s;
  }
}

// T[:, m:m+R] = [c1 + c2 (m x R); tau (R x R)]  (column-major, ld = ldT)
template <int R>
__global__ void k_tcol(const double* __restrict__ csum, const double* __restrict__ tau,
                       double* __restrict__ T, int64_t ldT, int m) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (m + R) * R; e += gridDim.x * blockDim.x) {
    const int cc = e / (m + R);
    const int i = e - cc * (m + R);
    const double v = (i < m) ? csum[(int64_t)i * R + cc] : tau[(i - m) * R + cc];
    T[(int64_t)(m + cc) * ldT + i] = v;
  }
}

// tau_1 = beta ell^{-1}  (R3), written to T[0:R, 0:R]; ell = chol(C^T C)
template <int R>
__global__ void k_init_tau(const double* __restrict__ beta, const double* __restrict__ ell,
                           double* __restrict__ T, int64_t ldT, double* __restrict__ R1) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double li[R * R], t[R * R];
  inv_upper<R>(ell, li);
  mm<R>(beta, li, t);
  for (int a = 0; a < R; ++a)
    for (int c = 0; c < R; ++c) T[(int64_t)c * ldT + a] = t[a * R + c];
  for (int e = 0; e < R * R; ++e) R1[e] = li[e];
}

}  // namespace sylv
