// Streaming ceiling probe (diagnostic, not product code): the K2 access pattern without LARS — read w, g, m
// (fp32), write w, m — as a plain grid-stride kernel with 256-bit accesses, timed with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/stream_probe tools/stream_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct F8 { float v[8]; };
__device__ __forceinline__ F8 ld8(const float* p) {
  F8 o; uint32_t* r = reinterpret_cast<uint32_t*>(o.v);
  asm volatile("ld.global.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(p));
  return o;
}
__device__ __forceinline__ void st8(float* p, const F8& o) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(o.v);
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
}
template <int U>
__global__ void __launch_bounds__(256, 4) k2_shape(float* w, const float* g, float* m, long n8) {
  for (long i = (long)blockIdx.x * 256 + threadIdx.x; i < n8; i += (long)gridDim.x * 256 * U) {
    F8 a[U], b[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * gridDim.x * 256L < n8) {
      long j = 8 * (i + u * gridDim.x * 256L);
      a[u] = ld8(w + j); b[u] = ld8(g + j); c[u] = ld8(m + j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * gridDim.x * 256L < n8) {
      long j = 8 * (i + u * gridDim.x * 256L);
#pragma unroll
      for (int k = 0; k < 8; ++k) { c[u].v[k] = 0.9f * c[u].v[k] + 1e-3f * b[u].v[k]; a[u].v[k] -= c[u].v[k]; }
      st8(w + j, a[u]); st8(m + j, c[u]);
    }
  }
}
__global__ void rd_only(const float* g, long n8, float* sink) {
  float acc = 0.f;
  for (long i = (long)blockIdx.x * 256 + threadIdx.x; i < n8; i += (long)gridDim.x * 256) {
    F8 b = ld8(g + 8 * i);
    for (int k = 0; k < 8; ++k) acc += b.v[k];
  }
  if (acc == 12345.f) *sink = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (long n : {25557032L / 8 * 8, 256L << 20}) {
    float *w, *g, *m, *sink, *flush;
    cudaMalloc(&w, n * 4); cudaMalloc(&g, n * 4); cudaMalloc(&m, n * 4); cudaMalloc(&sink, 4);
    cudaMalloc(&flush, 512L << 20);
    cudaMemset(w, 0, n * 4); cudaMemset(g, 0, n * 4); cudaMemset(m, 0, n * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int U : {1, 2}) for (int cps : {4}) {
      float best = 1e9;
      for (int rep = 0; rep < 20; ++rep) {
        cudaMemsetAsync(flush, rep, 512L << 20);
        cudaEventRecord(e0);
        if (U == 1) k2_shape<1><<<sms * cps, 256>>>(w, g, m, n / 8);
        else k2_shape<2><<<sms * cps, 256>>>(w, g, m, n / 8);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("K2-shape n=%ld U=%d ctas/SM=%d: %.1f us, %.0f GB/s (20 B/elem)\n", n, U, cps, best * 1e3, 20.0 * n / (best * 1e-3) / 1e9);
    }
    float best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      cudaMemsetAsync(flush, rep, 512L << 20);
      cudaEventRecord(e0); rd_only<<<sms * 8, 256>>>(g, n / 8, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("read-only n=%ld: %.1f us, %.0f GB/s\n", n, best * 1e3, 4.0 * n / (best * 1e-3) / 1e9);
    cudaFree(w); cudaFree(g); cudaFree(m); cudaFree(flush);
  }
  return 0;
}
