// geev_probe.cu — timing probe (development tool, not product): cuSOLVER Xgeev on m x m
// nonsymmetric matrices (real input / complex eigenpairs; complex input), to decide whether
// an eigendecomposition-based projected Sylvester solve can replace host Schur solves at c1.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/geev_probe.cu -lcusolver -lcublas -o tools/geev_probe
#include <cuComplex.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { auto e_ = (x); if (e_ != 0) { printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__); exit(1); } } while (0)

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  cusolverDnHandle_t h;
  CK(cusolverDnCreate(&h));
  cusolverDnParams_t p;
  CK(cusolverDnCreateParams(&p));
  for (int ai = 1; ai < argc; ++ai) {
    const int64_t m = atoll(argv[ai]);
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    std::vector<double> A(m * m);
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < m; ++i) A[j * m + i] = (i <= j + 4 ? nd(g) / sqrt((double)m) : 0.0) + (i == j ? 10.0 + 0.01 * i : 0.0);
    for (int cplx = 0; cplx < 2; ++cplx) {
      const size_t es = cplx ? 16 : 8;
      void *dA, *dW, *dV;
      CK(cudaMalloc(&dA, m * m * es));
      CK(cudaMalloc(&dW, m * 16));
      CK(cudaMalloc(&dV, m * m * es));
      std::vector<double> Ah(cplx ? 2 * m * m : m * m, 0.0);
      for (int64_t e = 0; e < m * m; ++e) Ah[cplx ? 2 * e : e] = A[e];
      const cudaDataType ta = cplx ? CUDA_C_64F : CUDA_R_64F;
      size_t wd = 0, wh = 0;
      CK(cusolverDnXgeev_bufferSize(h, p, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, m, ta, dA, m,
                                    CUDA_C_64F, dW, ta, nullptr, m, ta, dV, m, ta, &wd, &wh));
      void* bd;
      CK(cudaMalloc(&bd, wd + 1));
      std::vector<char> bh(wh + 1);
      int* info;
      CK(cudaMalloc(&info, 4));
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemcpy(dA, Ah.data(), Ah.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaDeviceSynchronize());
        const double t0 = now();
        CK(cusolverDnXgeev(h, p, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, m, ta, dA, m, CUDA_C_64F, dW,
                           ta, nullptr, m, ta, dV, m, ta, bd, wd, bh.data(), wh, info));
        CK(cudaDeviceSynchronize());
        const double t1 = now();
        int inf = -1;
        CK(cudaMemcpy(&inf, info, 4, cudaMemcpyDeviceToHost));
        printf("m=%lld %s rep %d: %.3f s info %d (ws dev %zu MB host %zu MB)\n", (long long)m, cplx ? "complex" : "real",
               rep, t1 - t0, inf, wd >> 20, wh >> 20);
        fflush(stdout);
      }
      cudaFree(dA); cudaFree(dW); cudaFree(dV); cudaFree(bd); cudaFree(info);
    }
  }
  return 0;
}
