// Development probe: green-context SM partitions with runtime-API launches (not product code).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

__global__ void k_where(unsigned* smid, unsigned long long* t, int spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  double x = threadIdx.x;
  for (int i = 0; i < spin; ++i) x = x * 1.0000001 + 1e-9;
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) {
    smid[blockIdx.x] = s;
    t[2 * blockIdx.x] = t0;
    t[2 * blockIdx.x + 1] = t1 + (x == -1.0);
  }
}

#define DRV(name) auto name = reinterpret_cast<PFN_##name##_v12040>(sym(#name))
static void* sym(const char* n) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint(n, &p, cudaEnableDefault, &q);
  if (!p) printf("missing %s\n", n);
  return p;
}

int main() {
  cudaFree(0);
  CUdevice dev = 0;
  auto getres = reinterpret_cast<CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType)>(sym("cuDeviceGetDevResource"));
  auto split = reinterpret_cast<CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned)>(sym("cuDevSmResourceSplitByCount"));
  auto gendesc = reinterpret_cast<CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned)>(sym("cuDevResourceGenerateDesc"));
  auto gcreate = reinterpret_cast<CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned)>(sym("cuGreenCtxCreate"));
  auto gstream = reinterpret_cast<CUresult (*)(CUstream*, CUgreenCtx, unsigned, int)>(sym("cuGreenCtxStreamCreate"));
  CUdevResource all, grp, rem;
  printf("getres %d\n", (int)getres(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("SMs %u\n", all.sm.smCount);
  unsigned n = 1;
  printf("split %d\n", (int)split(&grp, &n, &all, &rem, 0, 64));
  printf("group %u SMs, remaining %u SMs\n", grp.sm.smCount, rem.sm.smCount);
  CUdevResourceDesc dA, dB;
  printf("desc %d %d\n", (int)gendesc(&dA, &grp, 1), (int)gendesc(&dB, &rem, 1));
  CUgreenCtx gA, gB;
  printf("gctx %d %d\n", (int)gcreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM), (int)gcreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sA, sB;
  printf("gstream %d %d\n", (int)gstream(&sA, gA, CU_STREAM_NON_BLOCKING, 0), (int)gstream(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
  const int nb = 600;
  unsigned *smA, *smB;
  unsigned long long *tA, *tB;
  cudaMalloc(&smA, nb * 4); cudaMalloc(&smB, nb * 4);
  cudaMalloc(&tA, nb * 16); cudaMalloc(&tB, nb * 16);
  k_where<<<nb, 128, 0, (cudaStream_t)sA>>>(smA, tA, 200000);
  printf("launch A: %s\n", cudaGetErrorString(cudaGetLastError()));
  k_where<<<nb, 128, 0, (cudaStream_t)sB>>>(smB, tB, 200000);
  printf("launch B: %s\n", cudaGetErrorString(cudaGetLastError()));
  printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<unsigned> a(nb), b(nb);
  std::vector<unsigned long long> ta(2 * nb), tb(2 * nb);
  cudaMemcpy(a.data(), smA, nb * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), smB, nb * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(ta.data(), tA, nb * 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(tb.data(), tB, nb * 16, cudaMemcpyDeviceToHost);
  std::set<unsigned> SA(a.begin(), a.end()), SB(b.begin(), b.end());
  int inter = 0;
  for (unsigned x : SA) inter += SB.count(x);
  unsigned long long a0 = ~0ull, a1 = 0, b0 = ~0ull, b1 = 0;
  for (int i = 0; i < nb; ++i) {
    a0 = std::min(a0, ta[2 * i]); a1 = std::max(a1, ta[2 * i + 1]);
    b0 = std::min(b0, tb[2 * i]); b1 = std::max(b1, tb[2 * i + 1]);
  }
  printf("A on %zu SMs, B on %zu SMs, shared %d; A [%llu, %llu] us, B [%llu, %llu] us (rel. to A start)\n", SA.size(),
         SB.size(), inter, 0ull, (a1 - a0) / 1000, (b0 - a0) / 1000, (b1 - a0) / 1000);
  return 0;
}
