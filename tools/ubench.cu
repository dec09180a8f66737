// Microbenchmarks for design decisions (development tool, not product).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d0[2] = {0, 0}, d1[2] = {0, 0}, d2[2] = {0, 0}, d3[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
#define MMA(D) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" \
                             : "+d"(D[0]), "+d"(D[1]) : "d"(a), "d"(b));
    MMA(d0) MMA(d1) MMA(d2) MMA(d3)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = d0[0] + d0[1] + d1[0] + d1[1] + d2[0] + d2[1] + d3[0] + d3[1];
}

// Smem scatter: each warp owns a 2400-double bucket, lanes hit 32 consecutive (cyclic) slots.
__global__ void k_smem_scatter(const double* __restrict__ x, int64_t n, double* out, int b) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* bucket = sm + warp * b;
  for (int i = lane; i < b; i += 32) bucket[i] = 0;
  __syncwarp();
  uint32_t h = 12345u + warp * 777u + blockIdx.x;
  for (int64_t g = blockIdx.x; g < n / 32; g += gridDim.x) {
    h = h * 1664525u + 1013904223u;
    const uint32_t base = __umulhi(h, (uint32_t)b);
    uint32_t slot = base + ((5u * lane + (h >> 7)) & 31u);
    slot = slot >= (uint32_t)b ? slot - b : slot;
    const double v = x[g * 32 + lane];
    bucket[slot] += (h >> lane & 1) ? -v : v;
    __syncwarp();
  }
  for (int i = lane; i < b; i += 32) atomicAdd(out + i, bucket[i]);
}

// Global REDG scatter, r=8 contiguous per row (4 rows per warp instr)
__global__ void k_redg(const double* __restrict__ x, int64_t n, double* sk, uint32_t s) {
  const int lane = threadIdx.x & 31;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * 8; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e >> 3;
    uint32_t h = (uint32_t)row * 2654435761u;
    h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
    const uint32_t tgt = __umulhi(h, s);
    atomicAdd(sk + (int64_t)tgt * 8 + (lane & 7), x[e]);
  }
}

__global__ void k_copy(const double4* __restrict__ a, double4* __restrict__ b, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  int sm; cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sm, clk);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int iters = 20000;
  k_dfma<<<sm * 8, 256>>>(out, 10); cudaDeviceSynchronize();
  cudaEventRecord(e0); k_dfma<<<sm * 8, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 8 * iters * (double)sm * 8 * 256;
  printf("DFMA: %.1f TFLOP/s\n", fl / ms / 1e9);
  k_dmma<<<sm * 8, 256>>>(out, 10); cudaDeviceSynchronize();
  cudaEventRecord(e0); k_dmma<<<sm * 8, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 256 * 4 * iters * (double)sm * 8 * 8;   // per warp: 4 mma of 8x8x4
  printf("DMMA m8n8k4: %.1f TFLOP/s  (%s)\n", fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  // smem scatter
  int64_t n = 1ll << 27; double* x; cudaMalloc(&x, n * 8); cudaMemset(x, 0, n * 8);
  int b = 2400;
  cudaFuncSetAttribute(k_smem_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * b * 8);
  k_smem_scatter<<<sm, 256, 8 * b * 8>>>(x, n, out, b); cudaDeviceSynchronize();
  cudaEventRecord(e0); k_smem_scatter<<<sm, 256, 8 * b * 8>>>(x, n, out, b); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  // each of 8 warps scatters all n/gridDim rows... per CTA: (n/32/sm) groups * 8 warps * 32 updates
  double upd = (double)(n / 32) * 8 * 32;
  printf("smem scatter (8 warps, conflict-free): %.3f ms, %.2f updates/clk/SM (%s)\n", ms, upd / (ms * 1e-3) / sm / (clk * 1e3), cudaGetErrorString(cudaGetLastError()));
  // REDG
  int64_t nr = 1ll << 24; double* sk; cudaMalloc(&sk, 19200 * 8 * 8);
  k_redg<<<sm * 8, 256>>>(x, nr, sk, 19200); cudaDeviceSynchronize();
  cudaEventRecord(e0); k_redg<<<sm * 8, 256>>>(x, nr, sk, 19200); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("REDG f64 r=8 rows: %.3f ms for %lld updates = %.2f Gupd/s\n", ms, (long long)nr * 8, nr * 8 / (ms * 1e-3) / 1e9);
  // copy bandwidth
  int64_t nb = 1ll << 30;  // bytes per buffer... 1 GiB
  double4 *a4, *b4; cudaMalloc(&a4, nb); cudaMalloc(&b4, nb);
  k_copy<<<sm * 8, 256>>>(a4, b4, nb / 32); cudaDeviceSynchronize();
  cudaEventRecord(e0); for (int i = 0; i < 5; ++i) k_copy<<<sm * 8, 256>>>(a4, b4, nb / 32); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy: %.0f GB/s\n", 5 * 2.0 * nb / (ms * 1e-3) / 1e9);
  return 0;
}
