// stencil25d.cuh — 2.5-D streaming n-space passes for the 3-D stencil with r = 8
// (SURVEY §8(a) rows a1-a3 at configs c3; Alg. 1 lines 3-8).
//
// Same arithmetic as nspace.cuh's pass 1 / pass 2 (lazy normalisation, CGS over the
// k-window, R5), re-tiled for B200:
//
//  * A CTA owns a kTx x TY tile of the (x, y) plane and walks z over a segment of planes.
//    Every plane of every block it needs arrives in shared memory by TMA
//    (cp.async.bulk.tensor.4d over the SoA block viewed as an (x, y, z, column) tensor),
//    kNS planes in flight, one mbarrier per stage.  L1 is not used for block data.
//  * The stencil's z-neighbours are kept in registers (planes z-1, z, z+1 of Z_d roll
//    through three register arrays), x/y neighbours come from the halo'd plane in shared
//    memory.  Missing neighbours contribute 0 (homogeneous Dirichlet boundary): on the high
//    side TMA zero-fills the out-of-range part of the box; on the low side the box starts at
//    x = 0 / y = 0 (measured on this driver: a negative box coordinate, or an innermost
//    coordinate whose byte offset is not a multiple of 16, raises an illegal-instruction
//    fault) and the x-1 / y-1 neighbours of x = 0 / y = 0 are masked to 0.  In z the block
//    carries ghost planes (zeros at the domain boundary, the neighbour rank's boundary
//    plane when sharded), so the tensor's planes 0 .. nz+1 are all real memory.
//  * The r x r block products are fp64 tensor-core MMAs (mma.sync.m8n8k4.f64):
//      pass 1  P_i += Z_i(plane)^T Y(plane)             (3 DMMA per 4 points for k = 3)
//      pass 2  W'^T = R_d^T Y^T - sum_i K_i^T Z_i^T      (8 DMMA per 8 points)
//              G   += W'^T W'                            (2 DMMA per 8 points)
//  * Persistent grid (2 CTAs per SM): one partial per CTA.
//
// Shared-memory layout of one stage (TMA boxes are dense, innermost first):
//   halo  Z_d(p)   box (kTx+6, TY+2, 1, 8) at (x0-sx, y0-sy, p, 0): [c][y'][x'],
//                  sx = 2 (x0 > 0) or 0, sy = 1 (y0 > 0) or 0 (x0 - sx stays 16-byte aligned);
//                  point (x0+px, y0+w) is at [y' = w+sy][x' = px+sx]
//   win_i Z_i(p)   box (kTx+2, TY,   1, 8) at (x0,   y0,   p, 0): [c][y][x]  (i < nwin-1)
// The box widths (38 and 34 doubles) pad the column strides to 228 and 136 doubles, which
// makes the MMA-fragment reads bank-conflict-free.
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "nspace.cuh"

namespace sylv {

constexpr int kTx = 32;          // tile width in x (points)
// pipeline stages (planes in flight): enough bytes in flight per SM to cover HBM latency
// (r = 4 tiles carry half the bytes of r = 8 ones)
#ifndef SYLV_ST25_NS8
#define SYLV_ST25_NS8 3        // stages for r = 8 (development A/B: -DSYLV_ST25_NS8=2)
#endif
template <int R>
constexpr int stages25() { return R >= 8 ? SYLV_ST25_NS8 : 4; }
// warps per tile line: 2 splits a line's 32 points between two warps (each half the elements,
// twice the warps per SM to hide the shared-memory / DMMA latency chains)
#ifndef SYLV_ST25_WPL
#define SYLV_ST25_WPL 2
#endif
constexpr int kWpl25 = SYLV_ST25_WPL;

struct Tma25 {
  CUtensorMap zd;                // halo box map of Z_d's ring slot
  CUtensorMap win[kMaxKTma];     // window-box maps of the window blocks, oldest first
};

struct St25 {
  int N;                         // grid size (even)
  int nz;                        // planes of this rank's block; the TMA tensor has nz + 2 planes
                                 // (ghost plane 0, local planes 1..nz, ghost plane nz + 1)
  int tiles_x, tiles_y, nseg, zseg;
  int64_t items;                 // tiles_x * tiles_y * nseg
  int64_t ld;                    // SoA column stride
  double cd, cxm, cxp, cym, cyp, czm, czp;
  int dbg;                       // development switches (SYLV_DBG), 0 in production
};

template <int TY, int R = 8>
struct Geo25 {
  static constexpr int HX = kTx + 6, HY = TY + 2;      // halo box
  static constexpr int WX = kTx + 2;                   // window box width
  static constexpr int HCOL = HX * HY;                 // doubles per column, halo box
  static constexpr int WCOL = WX * TY;                 // doubles per column, window box
  static constexpr int HBYTES = R * HCOL * 8;
  static constexpr int WBYTES = R * WCOL * 8;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Wait for the phase with the given parity; the loop is visible to the compiler and the
// warp is reconverged before the caller's mma.sync.aligned instructions.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
  __syncwarp();
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x, int y, int z, int c,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(x), "r"(y), "r"(z), "r"(c), "r"(smem_u32(bar))
      : "memory");
}

// Issue the loads of plane p into stage `st` (thread 0 only).  Window blocks are needed
// only for the planes the CTA computes (with_win).
template <int TY, int R>
__device__ __forceinline__ void issue_plane(const Tma25& tm, int nwin, double* stage, uint64_t* bar, int x0,
                                            int y0, int p, bool with_win, int dbg = 0) {
  if (dbg & 1) with_win = false;
  using Gm = Geo25<TY, R>;
  const uint32_t bytes = Gm::HBYTES + (with_win ? (uint32_t)(nwin - 1) * Gm::WBYTES : 0u);
  mbar_expect_tx(bar, bytes);
  tma_load_4d(stage, &tm.zd, x0 > 0 ? x0 - 2 : 0, y0 > 0 ? y0 - 1 : 0, p, 0, bar);
  if (with_win)
    for (int i = 0; i < nwin - 1; ++i)
      tma_load_4d(stage + Gm::HCOL * R + i * Gm::WCOL * R, &tm.win[i], x0, y0, p, 0, bar);
}

// ---------------------------------------------------------------------------------------
// The kernel (R = 8 or 4 block columns; the DMMA fragments are 8 wide, columns >= R are
// zero and never loaded or stored).  PASS = 1: partial[blk][(i*R + a)*R + c] =
// sum Z_i[.,a] Y[.,c] (P_i).  PASS = 2: Wout = W' (SoA), partial[blk][a*R + c] =
// (W'^T W')[a][c] when GRAM.  coef (pass 2) = [R_d, K_0 .. K_{nwin-1}] row-major R x R.
// Element patterns (lane L, warp w owns line y0 + w of the tile; 32 points x0 .. x0+31):
//   pass 1 (pattern A): element e = 0..7 is (point 4e + (L&3), column L>>2)
//   pass 2 (pattern B): element e = 2q + h is (point 8q + (L>>2), column (L&3) + 4h)
// ---------------------------------------------------------------------------------------
#define DMMA25(...) do { if (!(p.dbg & 2)) dmma(__VA_ARGS__); } while (0)
template <int TY, int R, int K, int PASS, bool GRAM>
__global__ void __launch_bounds__(32 * TY * kWpl25, (TY <= 4 ? 2 : 1))
    k_st3d(const __grid_constant__ Tma25 tm, St25 p, int nwin, const double* __restrict__ coef,
           double* __restrict__ Wout, double* __restrict__ partial, int slot0 = -1) {
  static_assert(R == 4 || R == 8, "R = 4 or 8");
  constexpr int kNS = stages25<R>();
  using Gm = Geo25<TY, R>;
  extern __shared__ __align__(128) unsigned char smraw[];
  double* stages = reinterpret_cast<double*>(smraw);
  constexpr int kStageD = Gm::HCOL * R + (K - 1) * Gm::WCOL * R;   // doubles per stage
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw + (size_t)kNS * kStageD * 8);
  constexpr int EL = 8 / kWpl25;                // elements per lane (of the line's 8)
  // pass 1 with R = 4: two 4-point slices per DMMA (lanes 0-15 slice a, lanes 16-31 slice b:
  // P_a and P_b are the diagonal 4 x 4 blocks of the 8 x 8 product), half the elements
  constexpr bool kPack = PASS == 1 && R == 4;
  constexpr int NE = kPack ? EL / 2 : EL;
  __shared__ double red[TY * kWpl25][64 * (PASS == 1 ? K : 1)];

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int warp = wid / kWpl25, half = wid % kWpl25;   // warp = tile line; half = element range
  const int N = p.N;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // element coordinates inside the tile (point offset px in [0,32), column col); this warp owns
  // elements half*EL .. half*EL + EL - 1 of its line
  int px[NE], col[NE];
  bool cok[NE];                                 // column < R (else the element is zero)
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int eg = half * NE + e;
    if (kPack) {
      px[e] = 4 * (2 * eg + (lane >> 4)) + (lane & 3);
      col[e] = (lane >> 2) & 3;
    } else if (PASS == 1) {
      px[e] = 4 * eg + (lane & 3);
      col[e] = lane >> 2;
    } else {
      px[e] = 8 * (eg >> 1) + (lane >> 2);
      col[e] = (lane & 3) + 4 * (eg & 1);
    }
    cok[e] = col[e] < R;
    if (!cok[e]) col[e] = 0;                    // keeps the (unused) addresses in range
  }
  // pass 2: A fragments of R_d^T and -K_i^T (A[m][k] = M^T[m][k'] = M[k'][m], k' = (L&3) + 4h)
  double aR[2] = {0.0, 0.0}, aK[K][2];
  if (PASS == 2) {
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
  // two accumulator sets (even / odd slices) halve the dependent DMMA chains
  double acc[PASS == 1 ? K : 1][2], acc2[PASS == 1 ? K : 1][2];
#pragma unroll
  for (int i = 0; i < (PASS == 1 ? K : 1); ++i) acc[i][0] = acc[i][1] = acc2[i][0] = acc2[i][1] = 0.0;

  if (p.dbg & 8) return;
  uint32_t phase = 0;   // bit s = parity of the next wait on stage s
  const int NN = N;
  for (int64_t item = blockIdx.x; item < p.items; item += gridDim.x) {
    const int seg = (int)(item % p.nseg);
    const int64_t t2 = item / p.nseg;
    const int tx = (int)(t2 % p.tiles_x), ty = (int)(t2 / p.tiles_x);
    const int x0 = tx * kTx, y0 = ty * TY;
    const int z0 = 1 + seg * p.zseg, z1 = min(p.nz + 1, z0 + p.zseg);   // tensor planes
    // planes z0-1 .. z1 go through the stages; plane q uses stage (q - z0 + 1) % kNS
    auto stage_of = [&](int q) { return (q - z0 + 1) % kNS; };
    if (threadIdx.x == 0) {
      for (int q = z0 - 1; q < z0 - 1 + kNS && q <= z1; ++q) {
        if (q < 0) continue;                    // plane -1: Dirichlet zeros, never loaded
        const int s = stage_of(q);
        issue_plane<TY, R>(tm, nwin, stages + (size_t)s * kStageD, &bars[s], x0, y0, q, q >= z0 && q < z1, p.dbg);
      }
    }
    const int sx = x0 > 0 ? 2 : 0, sy = y0 > 0 ? 1 : 0;
    const int yrow = warp + sy;                // line inside the halo box
    const bool yok = (y0 + warp) < NN;
    const bool has_ym = (y0 + warp) > 0;       // y-1 neighbour exists
    double zm[NE], zc[NE], zp[NE];
    auto read_centers = [&](int q, double (&dst)[NE]) {
      if (q < 0) {
#pragma unroll
        for (int e = 0; e < NE; ++e) dst[e] = 0.0;
        return;
      }
      const int s = stage_of(q);
      mbar_wait(&bars[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      const double* H = stages + (size_t)s * kStageD;
#pragma unroll
      for (int e = 0; e < NE; ++e) dst[e] = cok[e] ? H[(col[e] * Gm::HY + yrow) * Gm::HX + px[e] + sx] : 0.0;
    };
    read_centers(z0 - 1, zm);
    read_centers(z0, zc);
    __syncthreads();                            // stage of plane z0-1 is free
    if (threadIdx.x == 0 && z0 - 1 + kNS <= z1) {
      const int q = z0 - 1 + kNS;
      const int s = stage_of(q);
      if (!(p.dbg & 4)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_plane<TY, R>(tm, nwin, stages + (size_t)s * kStageD, &bars[s], x0, y0, q, q < z1, p.dbg);
    }
    for (int z = z0; z < z1; ++z) {
      read_centers(z + 1, zp);                  // waits for plane z+1 (plane z is ready since z-1)
      const double* H = stages + (size_t)stage_of(z) * kStageD;
      const double* Wb = H + Gm::HCOL * R;
      double y[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        if (!cok[e]) {
          y[e] = 0.0;
          continue;
        }
        const double* hc = H + (col[e] * Gm::HY + yrow) * Gm::HX + px[e] + sx;
        const double xm = (x0 + px[e] > 0) ? hc[-1] : 0.0;
        const double ym = has_ym ? hc[-Gm::HX] : 0.0;
        double v = p.cd * zc[e];
        v = fma(p.cxm, xm, v);
        v = fma(p.cxp, hc[1], v);
        v = fma(p.cym, ym, v);
        v = fma(p.cyp, hc[Gm::HX], v);
        v = fma(p.czm, zm[e], v);
        v = fma(p.czp, zp[e], v);
        y[e] = v;
      }
      if (PASS == 1) {
        // P_i += Z_i^T Y over the 4-point slices e (pattern A: lane (col L>>2, point L&3))
#pragma unroll
        for (int e = 0; e < NE; ++e) {
#pragma unroll
          for (int i = 0; i < K; ++i) {
            if (i < nwin - 1) {
              const double zi = cok[e] ? Wb[i * Gm::WCOL * R + (col[e] * TY + warp) * Gm::WX + px[e]] : 0.0;
              if (e & 1) DMMA25(acc2[i], zi, y[e]); else DMMA25(acc[i], zi, y[e]);
            } else if (i == nwin - 1) {
              if (e & 1) DMMA25(acc2[i], zc[e], y[e]); else DMMA25(acc[i], zc[e], y[e]);
            }
          }
        }
      } else {
        const int64_t rowbase = ((int64_t)(z - 1) * NN + (y0 + warp)) * NN + x0;   // local row
#pragma unroll
        for (int ql = 0; ql < EL / 2; ++ql) {
          const int q = half * (EL / 2) + ql;     // 8-point slice of the line (pair of elements 2ql, 2ql+1)
          double D[2] = {0.0, 0.0};
          DMMA25(D, aR[0], y[2 * ql]);
          if (R == 8) DMMA25(D, aR[1], y[2 * ql + 1]);
#pragma unroll
          for (int i = 0; i < K; ++i) {
            if (i < nwin - 1) {
              const double* wi = Wb + i * Gm::WCOL * R;
              DMMA25(D, aK[i][0], cok[2 * ql] ? wi[(col[2 * ql] * TY + warp) * Gm::WX + px[2 * ql]] : 0.0);
              if (R == 8) DMMA25(D, aK[i][1], wi[(col[2 * ql + 1] * TY + warp) * Gm::WX + px[2 * ql + 1]]);
            } else if (i == nwin - 1) {
              DMMA25(D, aK[i][0], zc[2 * ql]);
              if (R == 8) DMMA25(D, aK[i][1], zc[2 * ql + 1]);
            }
          }
          // D: lane holds W'[point 8q + 2(L&3) + e][column L>>2]
          const int xo = 8 * q + 2 * (lane & 3);
          const bool cw = (lane >> 2) < R;      // output column exists
          const bool ok0 = cw && yok && (x0 + xo) < NN, ok1 = cw && yok && (x0 + xo + 1) < NN;
          D[0] = ok0 ? D[0] : 0.0;
          D[1] = ok1 ? D[1] : 0.0;
          double* dst = Wout + (int64_t)(cw ? (lane >> 2) : 0) * p.ld + rowbase + xo;
          if (ok1) {
            *reinterpret_cast<double2*>(dst) = make_double2(D[0], D[1]);
          } else if (ok0) {
            dst[0] = D[0];
          }
          if (GRAM) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int src = (lane & ~3) | (((lane & 3) + 4 * u) >> 1);
              const double v0 = __shfl_sync(SYLV_FULL_MASK, D[0], src);
              const double v1 = __shfl_sync(SYLV_FULL_MASK, D[1], src);
              const double v = (lane & 1) ? v1 : v0;
              if (u) DMMA25(acc2[0], v, v); else DMMA25(acc[0], v, v);
            }
          }
        }
      }
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        zm[e] = zc[e];
        zc[e] = zp[e];
      }
      __syncthreads();                          // stage of plane z is free
      if (threadIdx.x == 0) {
        const int q = z + kNS;
        if (q <= z1) {
          const int s = stage_of(q);
          if (!(p.dbg & 4)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue_plane<TY, R>(tm, nwin, stages + (size_t)s * kStageD, &bars[s], x0, y0, q, q < z1, p.dbg);
        }
      }
    }
    // plane z1 was consumed as zp of the last step; every issued plane has been waited on
  }
  // CTA reduction of the accumulators (D layout: lane holds [L>>2][2(L&3)+e])
  if (PASS == 1 || GRAM) {
    constexpr int NA = (PASS == 1 ? K : 1);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      red[wid][i * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = acc[i][0] + acc2[i][0];
      red[wid][i * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = acc[i][1] + acc2[i][1];
    }
    __syncthreads();
    // slot0 >= 0 (pass 1 with nwin = 1 after the fused pass, stencil25d_fused.cuh): only
    // P_{j} = Z_j^T A Z_j, written to slot slot0 of the K-slot record; the other slots hold the
    // fused pass's P and are left alone
    const int ne = slot0 >= 0 ? R * R : NA * R * R;
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
      const int i = e / (R * R), a = (e / R) % R, c = e % R;      // R x R blocks of the 8 x 8 D
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < TY * kWpl25; ++w) {
        s += red[w][i * 64 + a * 8 + c];
        if (kPack) s += red[w][i * 64 + (a + 4) * 8 + (c + 4)];   // slice b's diagonal block
      }
      partial[(int64_t)blockIdx.x * NA * R * R + (slot0 >= 0 ? slot0 * R * R + e : e)] = s;
    }
  }
}

#undef DMMA25
}  // namespace sylv
