// srdct.cuh — the paper's own sketch: subsampled randomized DCT,
// S = sqrt(n/s) D N E  (the printed sqrt(s/n) read as sqrt(n/s), R2):
// E = Rademacher signs, N = orthonormal DCT-II along the n rows, D = s selected rows.
// The signs and rows are inputs (synth/ draws them), copied to the device at init.
//
// DCT-II by one real-to-complex FFT of length n (Makhoul 1980): with v_k = x_{2k} for
// k < ceil(n/2) and v_{n-1-k} = x_{2k+1}, X_k = sum_j x_j cos(pi k (2j+1) / (2n)) =
// Re(exp(-i pi k / (2n)) V_k), V = FFT(v); orthonormal scaling sqrt(1/n) (k = 0), sqrt(2/n).
// The FFT is cuFFT (a library transform on an optional sketch; the hot-path sketch is the hashed
// sparse sign).  Only the s selected outputs are formed, each times the r x r factor M.
#pragma once
#include <cufft.h>

#include "common.cuh"

namespace sylv {

// v[c][k] (R columns of length n, contiguous) = sign[src] X[c*ld + src], src = Makhoul order of k
template <int R>
__global__ void __launch_bounds__(256) k_srdct_pre(int64_t n, const double* __restrict__ X, int64_t ld,
                                                   const double* __restrict__ sign, double* __restrict__ v) {
  const int64_t half = (n + 1) / 2;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t src = k < half ? 2 * k : 2 * (n - 1 - k) + 1;
    const double sg = __ldg(sign + src);
#pragma unroll
    for (int c = 0; c < R; ++c) v[(int64_t)c * n + k] = sg * __ldg(X + (int64_t)c * ld + src);
  }
}

// w[i*R + c] = sum_a (sqrt(n/s) X_{rows[i]}[a]) M[a*R + c]  (M = nullptr: identity), X = DCT-II of
// the pre-processed columns from V (R columns of n/2 + 1 complex values)
template <int R>
__global__ void __launch_bounds__(256) k_srdct_post(int64_t n, int64_t s, const cufftDoubleComplex* __restrict__ V,
                                                    const int64_t* __restrict__ rows, const double* __restrict__ M,
                                                    double* __restrict__ w) {
  const int64_t nh = n / 2 + 1;
  const double pi = 3.141592653589793238462643383279502884;
  const double sc = sqrt((double)n / (double)s);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = __ldg(rows + i);
    const double nrm = sc * (k == 0 ? sqrt(1.0 / (double)n) : sqrt(2.0 / (double)n));
    double sn, cs;
    sincospi(-(double)k / (2.0 * (double)n), &sn, &cs);
    double x[R];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double re, im;
      if (k < nh) {
        re = V[(int64_t)c * nh + k].x;
        im = V[(int64_t)c * nh + k].y;
      } else {                                        // V_k = conj(V_{n-k}) (real input)
        re = V[(int64_t)c * nh + (n - k)].x;
        im = -V[(int64_t)c * nh + (n - k)].y;
      }
      x[c] = nrm * (cs * re - sn * im);               // Re(exp(-i pi k/(2n)) V_k)
    }
    (void)pi;
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double o = x[c];
      if (M) {
        o = 0.0;
#pragma unroll
        for (int a = 0; a < R; ++a) o = fma(x[a], __ldg(M + a * R + c), o);
      }
      w[i * R + c] = o;
    }
  }
}

}  // namespace sylv
