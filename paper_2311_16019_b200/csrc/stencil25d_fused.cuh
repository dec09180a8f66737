// stencil25d_fused.cuh — pass 2 of step j fused with the old-block part of pass 1 of step j+1
// (Alg. 1 lines 3-8) for the 3-D stencil, r = 4/8.
//
// Pass 1 of step j+1 needs P_i = Z_i^T (A Z_{j+1}) for the window blocks i = j+2-k .. j+1.
// For the old blocks i <= j this is P_i = (A^T Z_i)^T W' with W' = Z_{j+1} the block that pass 2
// of step j produces (lazy normalisation: both sides unnormalised, R5): the transpose
// stencil is applied to the old blocks, which pass 2 streams anyway, and the product needs W'
// only at the tile's own points.  Only P_{j+1} = W'^T A W' (W' with its halo) is left to a
// one-block pass 1 (k_st3d<.., PASS 1> with nwin = 1, writing one slot of the partials).  Per
// block step and sequence: 2k+1 block transfers become k+2 (c3: 7 -> 5).
//
// Tiles, z-streaming, TMA stages and DMMA fragments as in stencil25d.cuh (pass 2).  A^T Z_d comes
// from the same neighbour values as A Z_d (transposed coefficients: x -> -x etc. swap); the other
// A^T blocks (the newest k-2 window blocks) arrive as halo boxes of Z_d's geometry (38 wide; two
// CTAs per SM still fit at r = 8, k = 3) with their z neighbours rolled in registers.  A^T Z_i is produced in the pass-2 element
// pattern (B) and moved to the pass-1 pattern (A) by two shuffles per element, W' in pattern A is
// the Gram's shuffle output, and P_i += (A^T Z_i)^T W' is one DMMA per 4 points.
//
// Stage layout (doubles): [Z_d halo: HCOL*R][NE extra halo boxes: HCOL2*R each][NW window boxes:
// WCOL*R each], NE = na-1, NW = nwin-1-NE, na = min(k-1, nwin) A^T blocks.
#pragma once
#include "stencil25d.cuh"

namespace sylv {

template <int TY>
struct Geo25x {
  static constexpr int HX2 = kTx + 6;                  // extra halo box width: Z_d's (38; a 36-wide box
                                                       // gave 36 % bank conflicts)
  static constexpr int HCOL2 = HX2 * (TY + 2);
};

struct Tma25F {
  CUtensorMap zd;                // halo box (38 wide) of Z_d
  CUtensorMap hx[kMaxKTma];         // extra halo boxes (Z_d's geometry) of the A^T window blocks, oldest first
  CUtensorMap win[kMaxKTma];        // window boxes of the other window blocks, oldest first
};

template <int TY, int R, int K>
constexpr int fused_stage_doubles() {
  return Geo25<TY, R>::HCOL * R + (K >= 3 ? (K - 2) : 0) * Geo25x<TY>::HCOL2 * R + Geo25<TY, R>::WCOL * R;
}

template <int TY, int R>
__device__ __forceinline__ void issue_plane_fused(const Tma25F& tm, int ne, int nw, double* stage, uint64_t* bar,
                                                  int x0, int y0, int p, bool with_win) {
  using Gm = Geo25<TY, R>;
  constexpr int HB2 = Geo25x<TY>::HCOL2 * R * 8;
  const uint32_t bytes = Gm::HBYTES + (uint32_t)ne * HB2 + (with_win ? (uint32_t)nw * Gm::WBYTES : 0u);
  mbar_expect_tx(bar, bytes);
  const int hx0 = x0 > 0 ? x0 - 2 : 0, hy0 = y0 > 0 ? y0 - 1 : 0;
  tma_load_4d(stage, &tm.zd, hx0, hy0, p, 0, bar);
  double* e0 = stage + Gm::HCOL * R;
  for (int e = 0; e < ne; ++e) tma_load_4d(e0 + e * Geo25x<TY>::HCOL2 * R, &tm.hx[e], hx0, hy0, p, 0, bar);
  if (with_win) {
    double* w0 = e0 + ne * Geo25x<TY>::HCOL2 * R;
    for (int w = 0; w < nw; ++w) tma_load_4d(w0 + w * Gm::WCOL * R, &tm.win[w], x0, y0, p, 0, bar);
  }
}

// Wout = W' (SoA); gram[blk][a*R + c] = (W'^T W')[a][c]; pp[blk][(slot*R + a)*R + c] =
// ((A^T Z_slot)^T W')[a][c] for the A^T slots 0 .. na-1 (window blocks j-na+1 .. j; slot na-1 =
// Z_d); other slots of pp are not written.  coef = [R_d, K_0 .. K_{nwin-1}] row-major R x R.
#define DMMA25F(...) dmma(__VA_ARGS__)
template <int TY, int R, int K>
__global__ void __launch_bounds__(32 * TY, (TY <= 4 ? 2 : 1))
    k_st3d_fused(const __grid_constant__ Tma25F tm, St25 p, int nwin, const double* __restrict__ coef,
                 double* __restrict__ Wout, double* __restrict__ gram, double* __restrict__ pp) {
  static_assert(R == 4 || R == 8, "R = 4 or 8");
  static_assert(K >= 2, "the fused pass needs k >= 2");
  constexpr int kNS = 3;
  constexpr int NEmax = K - 2;
  using Gm = Geo25<TY, R>;
  constexpr int HX2 = Geo25x<TY>::HX2;
  constexpr int HCOL2 = Geo25x<TY>::HCOL2;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* stages = reinterpret_cast<double*>(smraw);
  constexpr int kStageD = fused_stage_doubles<TY, R, K>();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw + (size_t)kNS * kStageD * 8);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int N = p.N;
  const int na = min(K - 1, nwin);            // A^T blocks (the newest na window blocks)
  const int ne = na - 1;                      // extra halo boxes
  const int nw = nwin - 1 - ne;               // plain window boxes (0 or 1)
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // pattern B: element e = 2q + h is (point 8q + (L>>2), column (L&3) + 4h)
  int px[8], col[8];
  bool cok[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    px[e] = 8 * (e >> 1) + (lane >> 2);
    col[e] = (lane & 3) + 4 * (e & 1);
    cok[e] = col[e] < R;
    if (!cok[e]) col[e] = 0;
  }
  double aR[2] = {0.0, 0.0}, aK[K][2];
  {
    const int mm = lane >> 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = (lane & 3) + 4 * h;
      const bool ok = mm < R && kk < R;
      aR[h] = ok ? __ldg(coef + kk * R + mm) : 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) aK[i][h] = (ok && i < nwin) ? -__ldg(coef + (1 + i) * R * R + kk * R + mm) : 0.0;
    }
  }
  double gacc[2] = {0.0, 0.0}, gacc2[2] = {0.0, 0.0};
  double pacc[K - 1][2], pacc2[K - 1][2];
#pragma unroll
  for (int a = 0; a < K - 1; ++a) pacc[a][0] = pacc[a][1] = pacc2[a][0] = pacc2[a][1] = 0.0;

  uint32_t phase = 0;
  for (int64_t item = blockIdx.x; item < p.items; item += gridDim.x) {
    const int seg = (int)(item % p.nseg);
    const int64_t t2 = item / p.nseg;
    const int tx = (int)(t2 % p.tiles_x), ty = (int)(t2 / p.tiles_x);
    const int x0 = tx * kTx, y0 = ty * TY;
    const int z0 = 1 + seg * p.zseg, z1 = min(p.nz + 1, z0 + p.zseg);
    auto stage_of = [&](int q) { return (q - z0 + 1) % kNS; };
    if (threadIdx.x == 0) {
      for (int q = z0 - 1; q < z0 - 1 + kNS && q <= z1; ++q) {
        const int s = stage_of(q);
        issue_plane_fused<TY, R>(tm, ne, nw, stages + (size_t)s * kStageD, &bars[s], x0, y0, q, q >= z0 && q < z1);
      }
    }
    const int sx = x0 > 0 ? 2 : 0, sy = y0 > 0 ? 1 : 0;
    const int yrow = warp + sy;
    const bool yok = (y0 + warp) < N;
    const bool has_ym = (y0 + warp) > 0;
    double zm[8], zc[8], zp[8];
    double em[NEmax > 0 ? NEmax : 1][8], ec[NEmax > 0 ? NEmax : 1][8], ep[NEmax > 0 ? NEmax : 1][8];
    // wait for plane q and read the centres of Z_d and of the extra halo blocks
    auto read_centers = [&](int q, double (&dst)[8], double (&edst)[NEmax > 0 ? NEmax : 1][8]) {
      const int s = stage_of(q);
      mbar_wait(&bars[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      const double* H = stages + (size_t)s * kStageD;
#pragma unroll
      for (int e = 0; e < 8; ++e) dst[e] = cok[e] ? H[(col[e] * Gm::HY + yrow) * Gm::HX + px[e] + sx] : 0.0;
#pragma unroll
      for (int b = 0; b < NEmax; ++b) {
        const double* E = H + Gm::HCOL * R + b * HCOL2 * R;
#pragma unroll
        for (int e = 0; e < 8; ++e)
          edst[b][e] = (b < ne && cok[e]) ? E[(col[e] * Gm::HY + yrow) * HX2 + px[e] + sx] : 0.0;
      }
    };
    read_centers(z0 - 1, zm, em);
    read_centers(z0, zc, ec);
    __syncthreads();
    if (threadIdx.x == 0 && z0 - 1 + kNS <= z1) {
      const int q = z0 - 1 + kNS;
      const int s = stage_of(q);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_plane_fused<TY, R>(tm, ne, nw, stages + (size_t)s * kStageD, &bars[s], x0, y0, q, q < z1);
    }
    for (int z = z0; z < z1; ++z) {
      read_centers(z + 1, zp, ep);
      const double* H = stages + (size_t)stage_of(z) * kStageD;
      const double* Eb = H + Gm::HCOL * R;
      const double* Wb = Eb + ne * HCOL2 * R;
      // y = A Z_d and xt[0] = A^T Z_d (slot na-1) from the same neighbours; xt[1+b] = A^T Z_extra_b
      double y[8], xt[K - 1][8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (!cok[e]) {
          y[e] = 0.0;
#pragma unroll
          for (int a = 0; a < K - 1; ++a) xt[a][e] = 0.0;
          continue;
        }
        const bool has_xm = (x0 + px[e]) > 0;
        {
          const double* hc = H + (col[e] * Gm::HY + yrow) * Gm::HX + px[e] + sx;
          const double xm = has_xm ? hc[-1] : 0.0;
          const double ym = has_ym ? hc[-Gm::HX] : 0.0;
          const double xp = hc[1], yp = hc[Gm::HX];
          double v = p.cd * zc[e];
          v = fma(p.cxm, xm, v);
          v = fma(p.cxp, xp, v);
          v = fma(p.cym, ym, v);
          v = fma(p.cyp, yp, v);
          v = fma(p.czm, zm[e], v);
          v = fma(p.czp, zp[e], v);
          y[e] = v;
          double u = p.cd * zc[e];                     // transpose: neighbour coefficients swapped
          u = fma(p.cxp, xm, u);
          u = fma(p.cxm, xp, u);
          u = fma(p.cyp, ym, u);
          u = fma(p.cym, yp, u);
          u = fma(p.czp, zm[e], u);
          u = fma(p.czm, zp[e], u);
          xt[0][e] = u;
        }
#pragma unroll
        for (int b = 0; b < NEmax; ++b) {
          double u = 0.0;
          if (b < ne) {
            const double* hc = Eb + b * HCOL2 * R + (col[e] * Gm::HY + yrow) * HX2 + px[e] + sx;
            const double xm = has_xm ? hc[-1] : 0.0;
            const double ym = has_ym ? hc[-HX2] : 0.0;
            u = p.cd * ec[b][e];
            u = fma(p.cxp, xm, u);
            u = fma(p.cxm, hc[1], u);
            u = fma(p.cyp, ym, u);
            u = fma(p.cym, hc[HX2], u);
            u = fma(p.czp, em[b][e], u);
            u = fma(p.czm, ep[b][e], u);
          }
          xt[1 + b][e] = u;
        }
      }
      const int64_t rowbase = ((int64_t)(z - 1) * N + (y0 + warp)) * N + x0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double D[2] = {0.0, 0.0};
        DMMA25F(D, aR[0], y[2 * q]);
        if (R == 8) DMMA25F(D, aR[1], y[2 * q + 1]);
        // window slots i = 0 .. nwin-1 (oldest first): plain window boxes (i < nw), extra halo
        // boxes (nw <= i < nwin-1), Z_d (i = nwin-1)
#pragma unroll
        for (int i = 0; i < K; ++i) {
          if (i >= nwin) continue;
          double w0, w1;
          if (i == nwin - 1) {
            w0 = zc[2 * q];
            w1 = zc[2 * q + 1];
          } else if (i >= nw) {
            const int b = i - nw;                // extra halo block b (select: no dynamic register index)
            w0 = 0.0;
            w1 = 0.0;
#pragma unroll
            for (int bb = 0; bb < NEmax; ++bb)
              if (bb == b) {
                w0 = ec[bb][2 * q];
                w1 = ec[bb][2 * q + 1];
              }
          } else {
            const double* wi = Wb + i * Gm::WCOL * R;
            w0 = cok[2 * q] ? wi[(col[2 * q] * TY + warp) * Gm::WX + px[2 * q]] : 0.0;
            w1 = wi[(col[2 * q + 1] * TY + warp) * Gm::WX + px[2 * q + 1]];
          }
          DMMA25F(D, aK[i][0], w0);
          if (R == 8) DMMA25F(D, aK[i][1], w1);
        }
        // D: lane holds W'[point 8q + 2(L&3) + e][column L>>2]
        const int xo = 8 * q + 2 * (lane & 3);
        const bool cw = (lane >> 2) < R;
        const bool ok0 = cw && yok && (x0 + xo) < N, ok1 = cw && yok && (x0 + xo + 1) < N;
        D[0] = ok0 ? D[0] : 0.0;
        D[1] = ok1 ? D[1] : 0.0;
        double* dst = Wout + (int64_t)(cw ? (lane >> 2) : 0) * p.ld + rowbase + xo;
        if (ok1) {
          *reinterpret_cast<double2*>(dst) = make_double2(D[0], D[1]);
        } else if (ok0) {
          dst[0] = D[0];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          // W' in pattern A: v = W'[point 8q + 4u + (L&3)][column L>>2]
          const int src = (lane & ~3) | (((lane & 3) + 4 * u) >> 1);
          const double v0 = __shfl_sync(SYLV_FULL_MASK, D[0], src);
          const double v1 = __shfl_sync(SYLV_FULL_MASK, D[1], src);
          const double v = (lane & 1) ? v1 : v0;
          if (u) DMMA25F(gacc2, v, v); else DMMA25F(gacc, v, v);
          // (A^T Z)^T in pattern A from pattern B: point 8q + 4u + (L&3) is held by lane
          // 4(4u + (L&3)) + ((L>>2)&3) in element 2q + (L>>4)
          const int s2 = 4 * (4 * u + (lane & 3)) + ((lane >> 2) & 3);
#pragma unroll
          for (int a = 0; a < K - 1; ++a) {
            if (a >= na) continue;
            const double a0 = __shfl_sync(SYLV_FULL_MASK, xt[a][2 * q], s2);
            const double a1 = __shfl_sync(SYLV_FULL_MASK, xt[a][2 * q + 1], s2);
            const double xa = (lane >> 4) ? a1 : a0;
            if (u) DMMA25F(pacc2[a], xa, v); else DMMA25F(pacc[a], xa, v);
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        zm[e] = zc[e];
        zc[e] = zp[e];
#pragma unroll
        for (int b = 0; b < NEmax; ++b) {
          em[b][e] = ec[b][e];
          ec[b][e] = ep[b][e];
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const int q = z + kNS;
        if (q <= z1) {
          const int s = stage_of(q);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_plane_fused<TY, R>(tm, ne, nw, stages + (size_t)s * kStageD, &bars[s], x0, y0, q, q < z1);
        }
      }
    }
  }
  // CTA reduction (stage memory is free: every issued plane has been consumed).  D layout:
  // lane holds [L>>2][2(L&3)+e].  Slots: 0 = Gram, 1 + a = P of A^T slot a.
  double* red = stages;                        // [TY][K][64]
  __syncthreads();
  red[(warp * K + 0) * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = gacc[0] + gacc2[0];
  red[(warp * K + 0) * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = gacc[1] + gacc2[1];
#pragma unroll
  for (int a = 0; a < K - 1; ++a) {
    red[(warp * K + 1 + a) * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = pacc[a][0] + pacc2[a][0];
    red[(warp * K + 1 + a) * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = pacc[a][1] + pacc2[a][1];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < (1 + na) * R * R; e += blockDim.x) {
    const int i = e / (R * R), a = (e / R) % R, c = e % R;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < TY; ++w) s += red[(w * K + i) * 64 + a * 8 + c];
    if (i == 0) {
      gram[(int64_t)blockIdx.x * R * R + a * R + c] = s;
    } else {
      // xt[0] = A^T Z_d is the newest old block of step j+1's window (slot na-1); xt[1+b] =
      // extra halo block b = slot b
      const int slot = (i == 1) ? na - 1 : i - 2;
      pp[(int64_t)blockIdx.x * K * R * R + (slot * R + a) * R + c] = s;
    }
  }
}
#undef DMMA25F

}  // namespace sylv
