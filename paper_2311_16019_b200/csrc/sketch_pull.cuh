// a4: S·W for the hashed sparse-sign sketch, "pull" formulation for large n.
//
// The sketch of one column x is y_t[(base_t(m) + π_{t,m}(l)) mod b] += σ_{t,m}(l) x[32m + l]
// (common.cuh: sk_entry; P:965 with BJ's sparse-sign, ζ buckets of b = s/ζ slots, group hash per
// 32 rows).  k_sketch_cols pushes every (group, bucket) window into a shared-memory copy of the
// column — 16 bytes of shared-memory read-modify-write per update.  Here the scatter is turned
// around.  The hash depends only on (seed, global group, bucket), so at init the groups of each
// bucket are sorted by window base (stable device radix sort; the sort is chunked by L2-sized row
// ranges so all warps sweep W chunk by chunk while it is L2-resident).  A warp owns bpw
// consecutive bases of one bucket; for every group whose window starts there, lane j loads
// x[32m + π⁻¹(j)] for all R columns — one coalesced 256-byte segment per column, permuted across
// lanes — and accumulates in registers while the base is unchanged (≈ n/(32 b) groups share a
// base).  Only on a base change is the register window added into the warp's private strip of
// bpw + 31 slots (bpw <= kPullBpwMax bases per warp, chosen at init so the grid fills the GPU).  A fold kernel adds the strips covering each slot in a fixed order
// and applies the r x r factor.  Every summation order is fixed by the stable sort: results are deterministic.
//
// Cost per (group, bucket, column): one 256-B L2 read (W is read from HBM once per chunk and
// ζ times from L2) instead of a shared-memory read-modify-write chain.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace sylv {

constexpr int kPullWarps = 8;
constexpr int kPullBpwMax = 16;           // window bases per warp (runtime ceil(b / wpb) <= this)
constexpr int kPullS = kPullBpwMax + 32;  // strip slots per warp and column (bpw + 31 used)
// list entries whose R column loads are in flight together (16-32 loads of 256 B per warp)
template <int R> constexpr int pull_u() { return R >= 4 ? 2 : 4; }
template <int R> constexpr int pull_min_blocks() { return R >= 8 ? 2 : 3; }   // registers: 2 U R + R doubles
constexpr int64_t kPullMinGroups = 4096;  // default: pull for n >= 131072 rows (with b >= 64)

// Warp w of a bucket owns the window bases [q0(w), q0(w+1)), q0(w) = floor(w b / wpb): ranges of
// floor(b/wpb) or ceil(b/wpb) = bpw bases, so wpb can be chosen to fill the resident warps of
// the GPU exactly (every SM gets the same load).
__host__ __device__ __forceinline__ uint32_t pull_q0(uint32_t w, uint32_t b, uint32_t wpb) {
  return (uint32_t)(((uint64_t)w * b) / wpb);
}
__host__ __device__ __forceinline__ uint32_t pull_owner(uint32_t p, uint32_t b, uint32_t wpb) {
  return (uint32_t)((((uint64_t)p + 1) * wpb - 1) / b);   // max w with q0(w) <= p
}

// Sort keys: entry (group g, bucket t) with window base p belongs to warp w = pull_owner(p) of
// bucket t; within the warp's list segment the order is (L2 chunk of g, p), and the radix sort
// is stable, so equal keys keep increasing g.
//   keys[t * ngroups + g] = ((t * wpb + w) * nch + g / gpch) * bpw + (p - q0(w)), vals = g,
//   counts[t * wpb + w] += 1 (-> exclusive scan = per-warp segment offsets)
__global__ void k_pull_keys(int64_t ngroups, SketchParams sp, int64_t gpch, uint32_t nch, uint32_t bpw,
                            uint32_t wpb, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                            uint32_t* __restrict__ counts) {
  const int64_t total = ngroups * sp.zeta;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(i / ngroups);
    const int64_t g = i - (int64_t)t * ngroups;
    const uint32_t base = __umulhi(group_hash(sp, sp.m0 + (uint32_t)g, t, 0), sp.b);
    const uint32_t w = pull_owner(base, sp.b, wpb);
    keys[i] = ((t * wpb + w) * nch + (uint32_t)(g / gpch)) * bpw + (base - pull_q0(w, sp.b, wpb));
    vals[i] = (uint32_t)g;
    atomicAdd(counts + t * wpb + w, 1u);
  }
}

// Hash record of list entry e (lane-private): group, packed (base - q0 | ainv << 8 | c << 16), signs
struct PullRec {
  uint32_t g, pk, sg;
};

__device__ __forceinline__ PullRec pull_rec(const SketchParams& sp, const uint32_t* __restrict__ list, uint32_t e,
                                            uint32_t e1, uint32_t t, uint32_t q0) {
  PullRec r{0u, 0u, 0u};
  if (e < e1) {
    r.g = __ldg(list + e);
    const uint32_t m = sp.m0 + r.g;
    const uint32_t h0 = group_hash(sp, m, t, 0);
    const uint32_t h1 = group_hash(sp, m, t, 1);
    r.sg = group_hash(sp, m, t, 2);
    const uint32_t a = 2u * (h1 & 15u) + 1u;
    const uint32_t ainv = (a * (2u - a * a)) & 31u;   // a·a ≡ 1 (mod 8) -> one Newton step
    const uint32_t c = (h1 >> 4) & 31u;
    r.pk = (__umulhi(h0, sp.b) - q0) | (ainv << 8) | (c << 16);
  }
  return r;
}

// Loads of U list entries eb + i .. eb + i + U - 1 (records in lanes i ..): lane j gets
// x[32 g + π⁻¹(j)] for the R columns and the multiplier σ ∈ {+1, -1} (0 for rows of the ragged
// last group past n, whose index is clamped to n - 1); bi = relative base, or ~0 past the
// segment end.  acc += σ x is one exact DFMA (σ x is exact).
template <int R, int U>
__device__ __forceinline__ void pull_load(const double* const (&xc)[R], uint32_t n, const PullRec& rc, uint32_t eb,
                                          uint32_t i, uint32_t e1, int lane, double (&v)[U][R], double (&sg)[U],
                                          uint32_t (&bi)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t idx = i + u;
    const uint32_t gi = __shfl_sync(0xffffffffu, rc.g, idx);
    const uint32_t pki = __shfl_sync(0xffffffffu, rc.pk, idx);
    const uint32_t sgi = __shfl_sync(0xffffffffu, rc.sg, idx);
    bi[u] = eb + idx < e1 ? (pki & 255u) : 0xffffffffu;
    const uint32_t l = (((pki >> 8) & 31u) * ((uint32_t)lane - (pki >> 16))) & 31u;   // π⁻¹(lane)
    const uint32_t row = (gi << 5) + l;
    sg[u] = row < n ? (((sgi >> l) & 1u) ? -1.0 : 1.0) : 0.0;
    const uint32_t rr = min(row, n - 1u);
#pragma unroll
    for (int c = 0; c < R; ++c) v[u][c] = __ldg(xc[c] + rr);
  }
}

template <int R, int U>
__device__ __forceinline__ void pull_accumulate(const double (&v)[U][R], const double (&sg)[U], const uint32_t (&bi)[U],
                                                double (&acc)[R], uint32_t& cur, double* st, int lane) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (bi[u] == 0xffffffffu) continue;
    if (bi[u] != cur) {
#pragma unroll
      for (int c = 0; c < R; ++c) {
        st[c * kPullS + cur + lane] += acc[c];
        acc[c] = 0.0;
      }
      cur = bi[u];
    }
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] = fma(v[u][c], sg[u], acc[c]);
  }
}

// y partial for one (bucket, base range) per warp -> strips[wg][R][kPullS].  The warp walks its
// list segment in steps of U entries with two register buffers: the loads of step k+1 are in
// flight while step k is accumulated.  Row indices are 32-bit (n < 2^32 is checked at init).
template <int R>
__global__ void __launch_bounds__(kPullWarps * 32, pull_min_blocks<R>()) k_sketch_pull(int64_t n, const double* __restrict__ X, int64_t ld,
                                                                 SketchParams sp, const uint32_t* __restrict__ list,
                                                                 const uint32_t* __restrict__ woff, uint32_t wpb,
                                                                 uint32_t bpw, double* __restrict__ strips) {
  constexpr int U = pull_u<R>();
  __shared__ double sm[kPullWarps][R * kPullS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t wg = blockIdx.x * kPullWarps + warp;
  if (wg >= sp.zeta * wpb) return;               // whole warp; no block-wide barrier below
  const uint32_t t = wg / wpb;
  const uint32_t q0 = pull_q0(wg - t * wpb, sp.b, wpb);
  const uint32_t n32 = (uint32_t)n;
  const double* xc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) xc[c] = X + (int64_t)c * ld;
  double* st = sm[warp];
  for (int i = lane; i < R * kPullS; i += 32) st[i] = 0.0;
  __syncwarp();
  double acc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.0;
  uint32_t cur = 0;                               // current base, relative to q0
  const uint32_t e0 = __ldg(woff + wg), e1 = __ldg(woff + wg + 1);
  if (e0 < e1) {
    uint32_t eb = e0, i = 0;                      // step position: entry eb + i
    PullRec rc = pull_rec(sp, list, eb + lane, e1, t, q0);
    double va[U][R], vb[U][R], sa[U], sb[U];
    uint32_t ba[U], bb[U];
    pull_load<R, U>(xc, n32, rc, eb, i, e1, lane, va, sa, ba);
    // advance (eb, i) by one step; refresh the records every 32 entries
    auto next = [&]() -> bool {
      i += U;
      if (i == 32u) {
        eb += 32u;
        i = 0;
        if (eb < e1) rc = pull_rec(sp, list, eb + lane, e1, t, q0);
      }
      return eb + i < e1;
    };
    while (true) {
      const bool more_b = next();
      if (more_b) pull_load<R, U>(xc, n32, rc, eb, i, e1, lane, vb, sb, bb);
      pull_accumulate<R, U>(va, sa, ba, acc, cur, st, lane);
      if (!more_b) break;
      const bool more_a = next();
      if (more_a) pull_load<R, U>(xc, n32, rc, eb, i, e1, lane, va, sa, ba);
      pull_accumulate<R, U>(vb, sb, bb, acc, cur, st, lane);
      if (!more_a) break;
    }
  }
#pragma unroll
  for (int c = 0; c < R; ++c) st[c * kPullS + cur + lane] += acc[c];
  __syncwarp();
  double* out = strips + (size_t)wg * R * kPullS;
  for (int i = lane; i < R * kPullS; i += 32) out[i] = st[i];
}

// Fold and right-multiply: w[q*R + c] = sum_a (scale * sum of the strips covering slot q of its
// bucket, column a) M[a*R + c]  (M = nullptr: identity).  The strips covering slot p are those
// of the warps whose bases q0 .. q0+bpw-1 reach it (slots q0 .. q0+bpw+30 mod b; zero past the
// warp's own bases + 30), summed nearest first — a fixed order.  Needs b >= bpw + 31 so a
// strip never covers a slot twice (b >= 64 is required at init).
template <int R>
__global__ void __launch_bounds__(256) k_sketch_pull_fold_apply(const double* __restrict__ strips, SketchParams sp,
                                                                uint32_t wpb, uint32_t bpw, uint32_t kmax,
                                                                const double* __restrict__ M, double* __restrict__ w) {
  // one thread per (slot, column): the strip sums; then one per (slot, output column): x M.
  // kmax bounds the candidate warps (their distance grows with k; the predicated loop keeps
  // every candidate's load in flight, and adds them nearest first like the break-loop did)
  constexpr int SPB = 256 / R;                         // slots per block
  __shared__ double vs[SPB][R];
  const uint32_t b = sp.b;
  const int64_t s = (int64_t)b * sp.zeta;
  const int ls = threadIdx.x / R, a = threadIdx.x % R;
  for (int64_t q0 = (int64_t)blockIdx.x * SPB; q0 < s; q0 += (int64_t)gridDim.x * SPB) {
    const int64_t q = q0 + ls;
    if (q < s) {
      const uint32_t t = (uint32_t)(q / b), p = (uint32_t)(q - (int64_t)t * b);
      const uint32_t wl = pull_owner(p, b, wpb);
      double v = 0.0;
      for (uint32_t k = 0; k < kmax; ++k) {
        const uint32_t wq = (wl + wpb - k) % wpb;
        const uint32_t dd = (p + b - pull_q0(wq, b, wpb)) % b;
        if (dd < bpw + 31u) v += strips[((size_t)(t * wpb + wq) * R + a) * kPullS + dd];
      }
      vs[ls][a] = v * sp.scale;
    }
    __syncthreads();
    if (q < s) {
      const int c = a;
      double o;
      if (M) {
        o = 0.0;
#pragma unroll
        for (int e = 0; e < R; ++e) o = fma(vs[ls][e], __ldg(M + e * R + c), o);
      } else {
        o = vs[ls][c];
      }
      w[q * R + c] = o;
    }
    __syncthreads();
  }
}

// The same fold for many candidate strips per slot (bpw small: c4 has one base per warp, so ~33
// warps' strips cover a slot and the per-thread candidate loop above — a 64-bit division per
// candidate — ran 20 us on 25 CTAs): one warp per slot, lane = candidate (k = lane, lane + 32),
// xor-butterfly sum (a fixed order: deterministic), lanes c < R apply the r x r factor.
template <int R>
__global__ void __launch_bounds__(128) k_sketch_pull_fold_wide(const double* __restrict__ strips, SketchParams sp,
                                                               uint32_t wpb, uint32_t bpw, uint32_t kmax,
                                                               const double* __restrict__ M, double* __restrict__ w) {
  const uint32_t b = sp.b;
  const int64_t s = (int64_t)b * sp.zeta;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < s; q += nw) {
    const uint32_t t = (uint32_t)(q / b), p = (uint32_t)(q - (int64_t)t * b);
    const uint32_t wl = pull_owner(p, b, wpb);
    double va[R];
#pragma unroll
    for (int a = 0; a < R; ++a) va[a] = 0.0;
    for (uint32_t k = (uint32_t)lane; k < kmax; k += 32u) {
      const uint32_t wq = (wl + wpb - k % wpb) % wpb;
      const uint32_t dd = (p + b - pull_q0(wq, b, wpb)) % b;
      if (dd < bpw + 31u) {
        const double* sp0 = strips + ((size_t)(t * wpb + wq) * R) * kPullS + dd;
#pragma unroll
        for (int a = 0; a < R; ++a) va[a] += sp0[(size_t)a * kPullS];
      }
    }
#pragma unroll
    for (int a = 0; a < R; ++a) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) va[a] += __shfl_xor_sync(0xffffffffu, va[a], o);
      va[a] *= sp.scale;
    }
    if (lane < R) {
      double o = 0.0;
      if (M) {
#pragma unroll
        for (int e = 0; e < R; ++e) o = fma(va[e], __ldg(M + e * R + lane), o);
      } else {
#pragma unroll
        for (int e = 0; e < R; ++e) o = (e == lane) ? va[e] : o;
      }
      w[q * R + lane] = o;
    }
  }
}

}  // namespace sylv
