// Development probe: isolate the 4-D TMA load of an SoA block (not product code).
// Usage: tma_probe <variant>   0: map as a direct __grid_constant__ param
//                              1: map inside a __grid_constant__ struct
//                              2: variant 1 + mbarrier wait loop + DMMA afterwards
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

struct Maps { CUtensorMap a; CUtensorMap b[4]; };

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ void load4d(void* dst, const CUtensorMap* m, int x, int y, int z, int c, uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(su32(dst)), "l"((uint64_t)m), "r"(x), "r"(y), "r"(z), "r"(c),
               "r"(su32(bar)) : "memory");
}
__device__ void load2d(void* dst, const CUtensorMap* m, int x, int y, uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)), "l"((uint64_t)m), "r"(x), "r"(y),
               "r"(su32(bar)) : "memory");
}
__device__ void waitp(uint64_t* bar, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(bar)), "r"(par) : "memory");
  }
  __syncwarp();
}

__global__ void k_2d(const __grid_constant__ CUtensorMap m, float* out) {
  __shared__ __align__(128) float buf[32 * 8];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) load2d(buf, &m, 0, 0, &bar, sizeof(buf));
  waitp(&bar, 0);
  for (int e = threadIdx.x; e < 256; e += blockDim.x) out[e] = buf[e];
}
template <int V>
__global__ void k_probe(const __grid_constant__ CUtensorMap m0, const __grid_constant__ Maps ms, double* out, int nbox,
                        int cx, int cy, int cz) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* buf = (double*)sm;
  uint64_t* bar = (uint64_t*)(sm + nbox * 8);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) load4d(buf, V == 0 ? &m0 : &ms.b[2], cx, cy, cz, 0, bar, nbox * 8);
  waitp(bar, 0);
  double d0 = 0, d1 = 0;
  if (V == 2) {
    double a = buf[threadIdx.x], b = buf[threadIdx.x + 32];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  }
  for (int e = threadIdx.x; e < nbox; e += blockDim.x) out[e] = buf[e];
  if (V == 2 && threadIdx.x < 32) out[nbox + threadIdx.x] = d0 + d1;
}

int main(int argc, char** argv) {
  const int V = argc > 1 ? atoi(argv[1]) : 0;
  if (V == 9) {   // rank-2 fp32 sanity
    float* g; cudaMalloc(&g, 64 * 64 * 4);
    std::vector<float> hg(64 * 64); for (int i = 0; i < 64 * 64; ++i) hg[i] = i;
    cudaMemcpy(g, hg.data(), 64 * 64 * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr; cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap m; cuuint64_t dims[2] = {64, 64}; cuuint64_t str[1] = {64 * 4};
    cuuint32_t box[2] = {32, 8}; cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    float* o; cudaMalloc(&o, 256 * 4);
    k_2d<<<1, 128>>>(m, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(256); cudaMemcpy(ho.data(), o, 1024, cudaMemcpyDeviceToHost);
    printf("variant 9 (2d fp32): encode %d, %s, o[33]=%g (want 65)\n", (int)r, cudaGetErrorString(e), ho[33]);
    return 0;
  }
  const int N = 34, R = 8;
  const long n = (long)N * N * N, ld = (n + 63) / 64 * 64;
  std::vector<double> h(ld * R);
  for (long c = 0; c < R; ++c)
    for (long i = 0; i < n; ++i) h[c * ld + i] = c * 1e6 + i;
  double* d;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)R};
  cuuint64_t str[3] = {(cuuint64_t)N * 8, (cuuint64_t)N * N * 8, (cuuint64_t)ld * 8};
  const int bx = 34, by = 6;
  cuuint32_t box[4] = {bx, by, 1, (cuuint32_t)R};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d (qr %d)\n", (int)r, (int)qr);
  Maps ms;
  ms.a = m;
  for (auto& x : ms.b) x = m;
  const int nbox = bx * by * R;
  double* o;
  cudaMalloc(&o, (nbox + 64) * 8);
  const size_t smem = nbox * 8 + 16;
  cudaError_t e;
  const int cx = argc > 2 ? atoi(argv[2]) : 0, cy = argc > 3 ? atoi(argv[3]) : 0, cz = argc > 4 ? atoi(argv[4]) : 3;
  if (V == 0) { cudaFuncSetAttribute(k_probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k_probe<0><<<1, 128, smem>>>(m, ms, o, nbox, cx, cy, cz); }
  if (V == 1) { cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k_probe<1><<<1, 128, smem>>>(m, ms, o, nbox, cx, cy, cz); }
  if (V == 2) { cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); k_probe<2><<<1, 128, smem>>>(m, ms, o, nbox, cx, cy, cz); }
  e = cudaDeviceSynchronize();
  printf("variant %d: %s\n", V, cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<double> ho(nbox);
  cudaMemcpy(ho.data(), o, nbox * 8, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int c = 0; c < R; ++c)
    for (int y = 0; y < by; ++y)
      for (int x = 0; x < bx; ++x) {
        const int gx = x + cx, gy = y + cy, gz = cz;
        const double want = (gx < 0 || gx >= N || gy < 0 || gy >= N || gz < 0 || gz >= N) ? 0.0 : c * 1e6 + ((long)gz * N + gy) * N + gx;
        if (ho[(c * by + y) * bx + x] != want) ++bad;
      }
  printf("variant %d: %ld mismatches of %d\n", V, bad, nbox);
  return 0;
}
