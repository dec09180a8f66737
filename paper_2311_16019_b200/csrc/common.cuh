// common.cuh — shared device definitions of the sylv_sketch CUDA library (sm_100a).
//
// Everything here is the product path; nothing is shared with oracle/ (DESIGN.md
// "Independence").  The sparse-sign hash below is the counter-based generator of
// DESIGN.md §"Sparse-sign hash", implemented independently of oracle/sparse_sign.py.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define SYLV_FULL_MASK 0xffffffffu

namespace sylv {

constexpr int kMaxR = 8;
constexpr int kMaxK = 10;      // k <= 4 for every r; 5..10 for r <= 2 (generic passes)
constexpr int kMaxKTma = 4;    // window blocks of the 2.5-D TMA passes
constexpr int kThreads = 256;            // CTA size of the streaming kernels
constexpr int kSmallThreads = 1024;      // CTA size of the one-CTA coefficient kernels (sspace.cuh)
constexpr int kWarps = kThreads / 32;

// ---- hashed sparse-sign S (never stored) ------------------------------------------
struct SketchParams {
  uint32_t seed;    // seed32 = seed ^ (seed >> 32)
  uint32_t zeta;    // nonzeros per column
  uint32_t b;       // bucket height s / zeta
  uint32_t m0;      // global index of this rank's first 32-row group (row_begin / 32)
  double scale;     // 1 / sqrt(zeta)
};

__host__ __device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__host__ __device__ __forceinline__ uint32_t group_hash(const SketchParams& sp, uint32_t m,
                                                        uint32_t t, uint32_t q) {
  return mix32(mix32(((m * sp.zeta + t) << 2) | q) ^ sp.seed);
}

// Row (in [0, s)) and sign of the bucket-t nonzero of column j = 32*m + lane.
struct SkEntry { uint32_t row; double val; };

__device__ __forceinline__ SkEntry sk_entry(const SketchParams& sp, uint32_t m, uint32_t lane,
                                            uint32_t t) {
  const uint32_t g0 = group_hash(sp, m, t, 0);
  const uint32_t g1 = group_hash(sp, m, t, 1);
  const uint32_t g2 = group_hash(sp, m, t, 2);
  const uint32_t base = __umulhi(g0, sp.b);
  const uint32_t a = 2u * (g1 & 15u) + 1u;
  const uint32_t c = (g1 >> 4) & 31u;
  uint32_t slot = base + ((a * lane + c) & 31u);
  slot = (sp.b >= 32u) ? (slot >= sp.b ? slot - sp.b : slot) : (slot % sp.b);
  SkEntry e;
  e.row = t * sp.b + slot;
  e.val = ((g2 >> lane) & 1u) ? -sp.scale : sp.scale;
  return e;
}

// ---- fast 32-bit division by a runtime constant (round-up method, exact for all x) ----
struct FastDiv {
  uint32_t d, m, s;
};

inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;
  f.s = s;
  f.m = (uint32_t)((((1ull << s) - d) << 32) / d + 1);
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
  return (uint32_t)(((uint64_t)__umulhi(x, f.m) + x) >> f.s);
}

// ---- operator descriptors -----------------------------------------------------------
enum OpKind : int { kStencil2D = 1, kStencil3D = 2, kCSR = 3 };

struct OpParams {
  int kind;
  int64_t n;          // rows of this rank's block (stencil: whole lines/planes); blocks carry
                      // ghost lines (2-D) / planes (3-D) before and after them
  int N;              // stencil grid size
  FastDiv divN;       // division by N
  double cd;          // diagonal 2*dim*nu/h^2
  double cxm, cxp;    // x-1 / x+1 neighbour coefficients
  double cym, cyp;
  double czm, czp;
  const int64_t* rp;  // CSR (device)
  const int32_t* ci;
  const double* cv;
};

// ---- tiny dense r x r helpers (row-major, one thread) ------------------------------
template <int R>
__device__ inline bool chol_upper(const double* G, double* U) {  // G = U^T U
  for (int i = 0; i < R * R; ++i) U[i] = 0.0;
  for (int j = 0; j < R; ++j) {
    double s = G[j * R + j];
    for (int p = 0; p < j; ++p) s -= U[p * R + j] * U[p * R + j];
    if (!(s > 0.0)) return false;
    const double d = sqrt(s);
    U[j * R + j] = d;
    for (int i = j + 1; i < R; ++i) {
      double t = G[j * R + i];
      for (int p = 0; p < j; ++p) t -= U[p * R + j] * U[p * R + i];
      U[j * R + i] = t / d;
    }
  }
  return true;
}

template <int R>
__device__ inline void inv_upper(const double* U, double* V) {  // V = U^{-1}
  for (int i = 0; i < R * R; ++i) V[i] = 0.0;
  for (int j = R - 1; j >= 0; --j) {
    V[j * R + j] = 1.0 / U[j * R + j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int p = i + 1; p <= j; ++p) s += U[i * R + p] * V[p * R + j];
      V[i * R + j] = -s / U[i * R + i];
    }
  }
}

template <int R>
__device__ inline void mm(const double* A, const double* B, double* C) {  // C = A B
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) {
      double s = 0.0;
      for (int p = 0; p < R; ++p) s += A[i * R + p] * B[p * R + j];
      C[i * R + j] = s;
    }
}

template <int R>
__device__ inline void mtm(const double* A, const double* B, double* C) {  // C = A^T B
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) {
      double s = 0.0;
      for (int p = 0; p < R; ++p) s += A[p * R + i] * B[p * R + j];
      C[i * R + j] = s;
    }
}

// D(8x8) += A(8x4) B(4x8), fp64; fragments per PTX ISA m8n8k4 .f64:
// A: lane holds A[lane>>2][lane&3]; B: B[lane&3][lane>>2]; D: D[lane>>2][2*(lane&3)+{0,1}].
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

}  // namespace sylv
