// host_solve.hpp — host-side small dense algebra of Alg. 1 (SURVEY §8(a) row a6, a7 prep):
// projected matrices, Bartels-Stewart for the projected Sylvester equation, sketched
// residual, SVD truncation.  LAPACK is the `scipy_`-prefixed LP64 OpenBLAS shipped
// with SciPy, loaded with dlopen (a library routine, like cuBLAS on the device).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace sylv {

bool lapack_load(const char* path, std::string& err);
bool lapack_loaded();

// M = [T_d | T_H] H_und_d T_d^{-1}  (R6), m = d r, col-major m x m.
// Th: T (col-major, ld ldT) holding at least T_{d+1}; Hh: per step j, (K+1) r x r
// row-major blocks [h_{j-nwin+1,j} .. h_{j,j}, pad.., h_{j+1,j} in slot K], nwin = min(k, j).
void build_projected(int d, int r, int k, const double* Th, int64_t ldT, const double* Hh,
                     std::vector<double>& M);

// hhat = tau_{d+1} h_{d+1,d} tau_d^{-1}  (r x r row-major; R4)
void hat_coefficient(int d, int r, int k, const double* Th, int64_t ldT, const double* Hh,
                     double* hhat);

// Solve MU Y + Y MV^T = F, F = E1 B E1^T with B = beta1 beta2^T (r x r row-major).
// MU, MV destroyed.  Y col-major m x m.  Returns 0 ok, 1 (near-)singular, <0 error.
int sylvester_bs(int m, int r, std::vector<double>& MU, std::vector<double>& MV,
                 const double* B, std::vector<double>& Y, std::string& err);

// Y = W S V^T; keep sigma_i > rank_tol sigma_1 (at most max_rank); Y1 = W_l S^{1/2},
// Y2 = V_l S^{1/2} (col-major m x l).  Returns l (>= 0) or < 0 on error.
int svd_truncate(int m, const std::vector<double>& Y, double rank_tol, int max_rank,
                 std::vector<double>& Y1, std::vector<double>& Y2, std::string& err);

// X <- T_d^{-1} X for upper triangular T (col-major ld ldT), X col-major m x l.
void trsm_left_upper(int m, int l, const double* T, int64_t ldT, double* X);

}  // namespace sylv
