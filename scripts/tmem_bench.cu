// TMEM -> register load bandwidth microbenchmark (tcgen05.ld.32x32b.x32), B200 sm_100a.
// W warps per CTA (one CTA per SM) each load 32 lanes x 32 columns x 4 B = 4 KB per instruction,
// repeatedly, with tcgen05.wait::ld after every `batch` loads; reports bytes per SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tmem_bench scripts/tmem_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define LD32(taddr, v)                                                                                             \
  asm volatile(                                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                              \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),           \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),     \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),   \
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])    \
      : "r"(taddr))

template <int BATCH>
__global__ void bench(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[BATCH][32];
#pragma unroll
    for (int b = 0; b < BATCH; ++b) LD32(tmem + (uint32_t)(((i * BATCH + b + warp) & 15) * 32), v[b]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int b = 0; b < BATCH; ++b) acc += __uint_as_float(v[b][31]) + __uint_as_float(v[b][0]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 1234.f) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  }
}

template <int BATCH>
double run(int sms, int warps, unsigned long long* d, unsigned long long* h, float* sink) {
  const int iters = 2048;
  bench<BATCH><<<sms, warps * 32>>>(iters, d, sink);
  bench<BATCH><<<sms, warps * 32>>>(iters, d, sink);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += h[i];
  const double cyc = s / sms;
  return (double)warps * iters * BATCH * 4096.0 / cyc;   // bytes per clock per SM
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *d, h[1024];
  float* sink;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&sink, 4);
  printf("{\"B_per_clk_sm\": {\"w4_b1\": %.1f, \"w4_b2\": %.1f, \"w8_b2\": %.1f, \"w16_b2\": %.1f, \"w16_b1\": %.1f, \"w8_b4\": %.1f}, \"err\": \"%s\"}\n",
         run<1>(sms, 4, d, h, sink), run<2>(sms, 4, d, h, sink), run<2>(sms, 8, d, h, sink), run<2>(sms, 16, d, h, sink),
         run<1>(sms, 16, d, h, sink), run<4>(sms, 8, d, h, sink), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
