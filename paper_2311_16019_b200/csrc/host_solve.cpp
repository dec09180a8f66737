// host_solve.cpp — see host_solve.hpp.  Bartels-Stewart (Schur of both projected
// matrices with dgees, quasi-triangular solve with dtrsyl3/dtrsyl, back-transform with
// dgemm) for Alg. 1 line 12 (eq. reduced_sk).
#include "host_solve.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <thread>

namespace sylv {
namespace {

using fstrlen = size_t;
typedef void (*dgees_t)(const char*, const char*, void*, const int*, double*, const int*, int*,
                        double*, double*, double*, const int*, double*, const int*, int*, int*,
                        fstrlen, fstrlen);
typedef void (*dtrsyl_t)(const char*, const char*, const int*, const int*, const int*,
                         const double*, const int*, const double*, const int*, double*,
                         const int*, double*, int*, fstrlen, fstrlen);
typedef void (*dtrsyl3_t)(const char*, const char*, const int*, const int*, const int*,
                          const double*, const int*, const double*, const int*, double*,
                          const int*, double*, int*, const int*, double*, const int*, int*,
                          fstrlen, fstrlen);
typedef void (*dgemm_t)(const char*, const char*, const int*, const int*, const int*,
                        const double*, const double*, const int*, const double*, const int*,
                        const double*, double*, const int*, fstrlen, fstrlen);
typedef void (*dtrsm_t)(const char*, const char*, const char*, const char*, const int*,
                        const int*, const double*, const double*, const int*, double*,
                        const int*, fstrlen, fstrlen, fstrlen, fstrlen);
typedef void (*dgesvd_t)(const char*, const char*, const int*, const int*, double*, const int*,
                         double*, double*, const int*, double*, const int*, double*,
                         const int*, int*, fstrlen, fstrlen);

typedef void (*dgesdd_t)(const char*, const int*, const int*, double*, const int*, double*, double*,
                         const int*, double*, const int*, double*, const int*, int*, int*, fstrlen);

typedef int (*set_threads_local_t)(int);

struct Lapack {
  void* h = nullptr;
  set_threads_local_t set_threads_local = nullptr;   // OpenBLAS: BLAS threads of the calling thread
  dgees_t dgees = nullptr;
  dtrsyl_t dtrsyl = nullptr;
  dtrsyl3_t dtrsyl3 = nullptr;
  dgemm_t dgemm = nullptr;
  dtrsm_t dtrsm = nullptr;
  dgesvd_t dgesvd = nullptr;
  dgesdd_t dgesdd = nullptr;   // optional: divide and conquer (what numpy's svd calls)
};
Lapack g_lapack;
std::mutex g_mu;

template <typename F>
bool sym(void* h, const char* name, F& out, std::string& err) {
  std::string full = std::string("scipy_") + name + "_";
  out = reinterpret_cast<F>(dlsym(h, full.c_str()));
  if (!out) {
    out = reinterpret_cast<F>(dlsym(h, (std::string(name) + "_").c_str()));
  }
  if (!out) {
    err = "LAPACK symbol not found: " + full;
    return false;
  }
  return true;
}

void gemm(char ta, char tb, int m, int n, int k, double alpha, const double* A, int lda,
          const double* B, int ldb, double beta, double* C, int ldc) {
  g_lapack.dgemm(&ta, &tb, &m, &n, &k, &alpha, A, &lda, B, &ldb, &beta, C, &ldc, 1, 1);
}

}  // namespace

bool lapack_load(const char* path, std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_lapack.h) return true;
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    err = std::string("dlopen failed: ") + (dlerror() ? dlerror() : path);
    return false;
  }
  Lapack L;
  L.h = h;
  if (!sym(h, "dgees", L.dgees, err) || !sym(h, "dtrsyl", L.dtrsyl, err) ||
      !sym(h, "dgemm", L.dgemm, err) || !sym(h, "dtrsm", L.dtrsm, err) ||
      !sym(h, "dgesvd", L.dgesvd, err)) {
    dlclose(h);
    return false;
  }
  std::string ignore;
  sym(h, "dtrsyl3", L.dtrsyl3, ignore);  // optional (LAPACK >= 3.11)
  sym(h, "dgesdd", L.dgesdd, ignore);    // optional
  L.set_threads_local = reinterpret_cast<set_threads_local_t>(dlsym(h, "openblas_set_num_threads_local"));
  g_lapack = L;
  return true;
}

bool lapack_loaded() { return g_lapack.h != nullptr; }

void build_projected(int d, int r, int k, const double* Th, int64_t ldT, const double* Hh,
                     std::vector<double>& M) {
  const int m = d * r;
  const int K = k;
  M.assign((size_t)m * m, 0.0);
  // X[:, block j] = sum_i T[0:m, block i] h_{i,j},  i = j-nwin+1 .. j+1
  for (int j = 1; j <= d; ++j) {
    const int nwin = std::min(k, j);
    const double* Hj = Hh + (size_t)j * (K + 1) * r * r;
    for (int ii = 0; ii <= nwin; ++ii) {
      const int i = (ii < nwin) ? (j - nwin + 1 + ii) : (j + 1);
      const double* h = (ii < nwin) ? (Hj + (size_t)ii * r * r) : (Hj + (size_t)K * r * r);
      for (int c = 0; c < r; ++c) {
        double* xcol = M.data() + (size_t)((j - 1) * r + c) * m;
        for (int a = 0; a < r; ++a) {
          const double hv = h[a * r + c];
          if (hv == 0.0) continue;
          const double* tcol = Th + (int64_t)((i - 1) * r + a) * ldT;
          const int rows = std::min(m, i * r);  // T upper triangular: rows < i*r nonzero
          for (int row = 0; row < rows; ++row) xcol[row] += tcol[row] * hv;
        }
      }
    }
  }
  // M = X T_d^{-1}
  const char side = 'R', uplo = 'U', trans = 'N', diag = 'N';
  const double one = 1.0;
  const int ld = (int)ldT;
  g_lapack.dtrsm(&side, &uplo, &trans, &diag, &m, &m, &one, Th, &ld, M.data(), &m, 1, 1, 1, 1);
}

void hat_coefficient(int d, int r, int k, const double* Th, int64_t ldT, const double* Hh,
                     double* hhat) {
  const int K = k;
  const double* h = Hh + (size_t)d * (K + 1) * r * r + (size_t)K * r * r;
  std::vector<double> tau1(r * r), taud(r * r), tmp(r * r), inv(r * r, 0.0);
  for (int a = 0; a < r; ++a)
    for (int c = 0; c < r; ++c) {
      tau1[a * r + c] = Th[(int64_t)(d * r + c) * ldT + d * r + a];
      taud[a * r + c] = Th[(int64_t)((d - 1) * r + c) * ldT + (d - 1) * r + a];
    }
  // inv = taud^{-1} (upper triangular)
  for (int j = r - 1; j >= 0; --j) {
    inv[j * r + j] = 1.0 / taud[j * r + j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int p = i + 1; p <= j; ++p) s += taud[i * r + p] * inv[p * r + j];
      inv[i * r + j] = -s / taud[i * r + i];
    }
  }
  for (int a = 0; a < r; ++a)
    for (int c = 0; c < r; ++c) {
      double s = 0.0;
      for (int p = 0; p < r; ++p) s += tau1[a * r + p] * h[p * r + c];
      tmp[a * r + c] = s;
    }
  for (int a = 0; a < r; ++a)
    for (int c = 0; c < r; ++c) {
      double s = 0.0;
      for (int p = 0; p < r; ++p) s += tmp[a * r + p] * inv[p * r + c];
      hhat[a * r + c] = s;
    }
}

static int schur(int m, std::vector<double>& A, std::vector<double>& Z, std::string& err) {
  const char jobvs = 'V', sort = 'N';
  int sdim = 0, info = 0, lwork = -1;
  std::vector<double> wr(m), wi(m);
  Z.assign((size_t)m * m, 0.0);
  double wq = 0.0;
  g_lapack.dgees(&jobvs, &sort, nullptr, &m, A.data(), &m, &sdim, wr.data(), wi.data(), Z.data(),
                 &m, &wq, &lwork, nullptr, &info, 1, 1);
  lwork = std::max(1, (int)wq);
  std::vector<double> work(lwork);
  g_lapack.dgees(&jobvs, &sort, nullptr, &m, A.data(), &m, &sdim, wr.data(), wi.data(), Z.data(),
                 &m, work.data(), &lwork, nullptr, &info, 1, 1);
  if (info != 0) {
    err = "dgees info=" + std::to_string(info);
    return -1;
  }
  return 0;
}

int sylvester_bs(int m, int r, std::vector<double>& MU, std::vector<double>& MV, const double* B,
                 std::vector<double>& Y, std::string& err) {
  if (!lapack_loaded()) {
    err = "LAPACK not loaded (sylv_set_lapack_path)";
    return -2;
  }
  // SYLV_TRACE_INIT=1: phase times of the host solve on stderr (development aid)
  const bool trace = std::getenv("SYLV_TRACE_INIT") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[host] %-24s m=%d %8.1f ms\n", what, m, std::chrono::duration<double, std::milli>(now - t0).count());
    t0 = now;
  };
  std::vector<double> ZU, ZV;
  // a Schur iteration that does not converge (badly scaled M of an ill-conditioned sketched
  // basis) is a failed check at this d, not a missing library
  // The two independent Schur decompositions on two host threads with half of the BLAS threads
  // each (OpenBLAS per-thread thread counts) for m >= 512 (SYLV_HOST_PARALLEL=0: one after the
  // other).  c1 at m = 3128: 10.0 s -> 6.0 s.  Not bit-reproducible run to run: at c1's crossing
  // (kappa(T) ~ 1e13-1e15) rho_rel moved by 1.4e-4 relative between two solves of the same
  // matrices — the same order as any change of BLAS blocking; d* is a valid crossing of the
  // search either way (R20) and is tested against the oracle's (+-2).
  const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
  const char* hp = std::getenv("SYLV_HOST_PARALLEL");
  if (m >= 512 && g_lapack.set_threads_local && !(hp && std::strcmp(hp, "0") == 0)) {
    int su = 0, sv = 0;
    std::string erru, errv;
    const int half = (int)std::max(1u, hw / 2);
    std::thread tu([&]() {
      const int prev = g_lapack.set_threads_local(half);
      su = schur(m, MU, ZU, erru);
      g_lapack.set_threads_local(prev);
    });
    const int prev = g_lapack.set_threads_local(half);
    sv = schur(m, MV, ZV, errv);
    g_lapack.set_threads_local(prev);
    tu.join();
    lap("dgees M_U || M_V");
    if (su || sv) {
      err = su ? erru : errv;
      return 1;
    }
  } else {
    if (schur(m, MU, ZU, err)) return 1;
    lap("dgees M_U");
    if (schur(m, MV, ZV, err)) return 1;
    lap("dgees M_V");
  }
  // Ft = ZU^T F ZV = ZU[0:r,:]^T (B ZV[0:r,:])
  std::vector<double> Bc(r * r), tmp((size_t)r * m), F((size_t)m * m);
  for (int a = 0; a < r; ++a)
    for (int c = 0; c < r; ++c) Bc[c * r + a] = B[a * r + c];  // col-major
  gemm('N', 'N', r, m, r, 1.0, Bc.data(), r, ZV.data(), m, 0.0, tmp.data(), r);   // B * ZV[0:r,:]
  gemm('T', 'N', m, m, r, 1.0, ZU.data(), m, tmp.data(), r, 0.0, F.data(), m);    // ZU[0:r,:]^T tmp
  // TU X + X TV^T = scale F
  const char ta = 'N', tb = 'T';
  const int isgn = 1;
  double scale = 1.0;
  int info = 0;
  bool done = false;
  if (g_lapack.dtrsyl3) {
    int liwork = -1, ldsw = -1;
    int iwq = 0;
    double swq[2] = {0, 0};
    g_lapack.dtrsyl3(&ta, &tb, &isgn, &m, &m, MU.data(), &m, MV.data(), &m, F.data(), &m, &scale,
                     &iwq, &liwork, swq, &ldsw, &info, 1, 1);
    if (info == 0) {
      liwork = std::max(1, iwq);
      ldsw = std::max(2, (int)swq[0]);
      const int cols = std::max(2, (int)swq[1]);
      std::vector<int> iw(liwork);
      std::vector<double> sw((size_t)ldsw * cols);
      g_lapack.dtrsyl3(&ta, &tb, &isgn, &m, &m, MU.data(), &m, MV.data(), &m, F.data(), &m,
                       &scale, iw.data(), &liwork, sw.data(), &ldsw, &info, 1, 1);
      done = (info >= 0);
    }
  }
  if (!done) {
    g_lapack.dtrsyl(&ta, &tb, &isgn, &m, &m, MU.data(), &m, MV.data(), &m, F.data(), &m, &scale,
                    &info, 1, 1);
  }
  lap("dtrsyl3");
  if (info < 0) {
    err = "dtrsyl info=" + std::to_string(info);
    return -1;
  }
  if (!(scale > 0.0) || !std::isfinite(scale)) {
    err = "dtrsyl scale underflow";
    return 1;
  }
  // Y = ZU (F/scale) ZV^T
  std::vector<double> W((size_t)m * m);
  gemm('N', 'N', m, m, m, 1.0 / scale, ZU.data(), m, F.data(), m, 0.0, W.data(), m);
  Y.assign((size_t)m * m, 0.0);
  gemm('N', 'T', m, m, m, 1.0, W.data(), m, ZV.data(), m, 0.0, Y.data(), m);
  lap("back-transform GEMMs");
  for (double v : Y)
    if (!std::isfinite(v)) {
      err = "non-finite projected solution";
      return 1;
    }
  if (info == 1) err = "dtrsyl: close eigenvalues of M_U and -M_V (perturbed)";
  return 0;
}

int svd_truncate(int m, const std::vector<double>& Yin, double rank_tol, int max_rank,
                 std::vector<double>& Y1, std::vector<double>& Y2, std::string& err) {
  std::vector<double> A(Yin), S(m), U((size_t)m * m), VT((size_t)m * m);
  int info = 0, lwork = -1;
  double wq = 0;
  bool done = false;
  if (g_lapack.dgesdd) {
    // divide and conquer (c3, m = 1872: ~9 s with dgesvd on the host); dgesvd if it fails
    const char jobz = 'S';
    std::vector<int> iwork((size_t)8 * m);
    g_lapack.dgesdd(&jobz, &m, &m, A.data(), &m, S.data(), U.data(), &m, VT.data(), &m, &wq, &lwork,
                    iwork.data(), &info, 1);
    if (info == 0) {
      lwork = std::max(1, (int)wq);
      std::vector<double> work(lwork);
      g_lapack.dgesdd(&jobz, &m, &m, A.data(), &m, S.data(), U.data(), &m, VT.data(), &m, work.data(), &lwork,
                      iwork.data(), &info, 1);
      done = info == 0;
    }
    if (!done) A = Yin;
  }
  if (!done) {
    const char jobu = 'S', jobvt = 'S';
    lwork = -1;
    g_lapack.dgesvd(&jobu, &jobvt, &m, &m, A.data(), &m, S.data(), U.data(), &m, VT.data(), &m, &wq,
                    &lwork, &info, 1, 1);
    lwork = std::max(1, (int)wq);
    std::vector<double> work(lwork);
    g_lapack.dgesvd(&jobu, &jobvt, &m, &m, A.data(), &m, S.data(), U.data(), &m, VT.data(), &m,
                    work.data(), &lwork, &info, 1, 1);
    if (info != 0) {
      err = "dgesvd info=" + std::to_string(info);
      return -1;
    }
  }
  int l = 0;
  if (m > 0 && S[0] > 0.0)
    while (l < m && S[l] > rank_tol * S[0]) ++l;
  l = std::min(l, max_rank);
  Y1.assign((size_t)m * l, 0.0);
  Y2.assign((size_t)m * l, 0.0);
  for (int c = 0; c < l; ++c) {
    const double sq = std::sqrt(S[c]);
    for (int i = 0; i < m; ++i) {
      Y1[(size_t)c * m + i] = U[(size_t)c * m + i] * sq;
      Y2[(size_t)c * m + i] = VT[(size_t)i * m + c] * sq;  // V = VT^T
    }
  }
  return l;
}

void trsm_left_upper(int m, int l, const double* T, int64_t ldT, double* X) {
  if (l == 0) return;
  const char side = 'L', uplo = 'U', trans = 'N', diag = 'N';
  const double one = 1.0;
  const int ld = (int)ldT;
  g_lapack.dtrsm(&side, &uplo, &trans, &diag, &m, &l, &one, T, &ld, X, &m, 1, 1, 1, 1);
}

}  // namespace sylv
