// Pipe-rate microbenchmarks on B200: MUFU ex2, FP32 FFMA/FADD, FMNMX.
// Each kernel runs 148*k CTAs of 256 threads with 8 independent dependency chains per thread;
// the rate is (ops executed) / (CUDA-event time) / (SMs * SM clock).  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks scripts/peaks.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_ex2(float* out, float seed) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j) * 1e-9f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma(float* out, float seed) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j);
  const float m = seed * 0.999f, c = seed * 1e-3f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[j]) : "f"(m), "f"(c));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_fadd(float* out, float seed) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j);
  const float c = seed * 1e-3f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[j]) : "f"(c));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_fmax(float* out, float seed) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j);
  float c = seed * 1e-3f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[j]) : "f"(c));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_fadd2(float* out, float seed) {
  float2 a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = make_float2(seed * (threadIdx.x + j), seed * j);
  const float2 c = make_float2(seed * 1e-3f, seed * 2e-3f);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __fadd2_rn(a[j], c);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j].x + a[j].y;
  if (s == 1234.5f) out[0] = s;
}

// MUFU with one broadcast LDS.128 per 4 ex2 (the reverse pass's ht loads): MIO sharing
__global__ void k_ex2_lds(float* out, float seed) {
  __shared__ float4 sh[256];
  sh[threadIdx.x] = make_float4(seed, seed * 2, seed * 3, seed * 4);
  __syncthreads();
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j) * 1e-9f;
  for (int i = 0; i < ITERS; ++i) {
    const float4 q0 = sh[(i * 2) & 255], q1 = sh[(i * 2 + 1) & 255];   // warp-uniform address: broadcast
    const float qq[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float y = a[j] + qq[j];
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(y));
      a[j] = y;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1234.5f) out[0] = s;
}

// MUFU ex2 + one cvt.rn.f16x2.f32 (F2FP) per 2 ex2 (+ optional f16x2 -> f32 unpack): which pipe converts?
template <int UNPACK>
__global__ void k_ex2_cvt(float* out, float seed) {
  float a[8];
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j) * 1e-9f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      uint32_t h;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a[j]), "f"(a[j + 1]));
      if (UNPACK) {
        float lo, hi;
        asm volatile("{.reg .f16 l, u;\n mov.b32 {l, u}, %2;\n cvt.f32.f16 %0, l;\n cvt.f32.f16 %1, u;}" : "=f"(lo), "=f"(hi) : "r"(h));
        a[j] += lo * 1e-30f;
        a[j + 1] += hi * 1e-30f;
      }
      acc ^= h;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1234.5f || acc == 0x12345u) out[0] = s;
}

// mixed: what the forward softmax does per pair (FADD bias, FMNMX, FFMA-folded subtract in ex2 arg, FADD sum)
__global__ void k_mixed(float* out, float seed) {
  float x[8], s[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { x[j] = seed * (threadIdx.x + j) * 1e-9f; s[j] = 0.f; }
  float mx = -1e30f;
  const float cb = seed * 1e-7f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v;
      asm volatile("add.f32 %0, %1, %2;" : "=f"(v) : "f"(x[j]), "f"(cb));
      asm volatile("max.f32 %0, %0, %1;" : "+f"(mx) : "f"(v));
      float e;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(v));
      asm volatile("add.f32 %0, %0, %1;" : "+f"(s[j]) : "f"(e));
      x[j] = v;
    }
  }
  float t = mx;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += s[j];
  if (t == 1234.5f) out[0] = t;
}

template <typename F>
float run(F kern, int sms, float* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) kern<<<sms * 8, 256>>>(out, 1.0f);
  cudaEventRecord(a);
  const int REP = 5;
  for (int r = 0; r < REP; ++r) kern<<<sms * 8, 256>>>(out, 1.0f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / REP;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4);
  const double ops = (double)sms * 8 * 256 * ITERS * 8;
  const double ghz = clk_khz * 1e-6;
  auto rate = [&](float ms) { return ops / (ms * 1e-3); };
  float t_ex2 = run(k_ex2, sms, out), t_ffma = run(k_ffma, sms, out), t_fadd = run(k_fadd, sms, out),
        t_fmax = run(k_fmax, sms, out), t_mixed = run(k_mixed, sms, out), t_fadd2 = run(k_fadd2, sms, out), t_ex2lds = run(k_ex2_lds, sms, out),
        t_cvt = run(k_ex2_cvt<0>, sms, out), t_cvt2 = run(k_ex2_cvt<1>, sms, out);
  printf("{\"sms\": %d, \"clock_attr_ghz\": %.3f, "
         "\"ex2_per_s\": %.4e, \"ffma_per_s\": %.4e, \"fadd_per_s\": %.4e, \"fmax_per_s\": %.4e, "
         "\"mixed_pairs_per_s\": %.4e, \"fadd2_lanes_per_clk_sm_at_attr\": %.2f, \"ex2_with_lds_per_clk_sm\": %.2f, \"ex2_with_f2fp_per_clk_sm\": %.2f, \"ex2_with_f2fp_unpack_per_clk_sm\": %.2f, "
         "\"ex2_per_clk_sm_at_attr\": %.2f, \"ffma_per_clk_sm_at_attr\": %.2f, \"fadd_per_clk_sm_at_attr\": %.2f, "
         "\"fmax_per_clk_sm_at_attr\": %.2f, \"mixed_pairs_per_clk_sm_at_attr\": %.2f}\n",
         sms, ghz, rate(t_ex2), rate(t_ffma), rate(t_fadd), rate(t_fmax), rate(t_mixed), 2 * rate(t_fadd2) / sms / (ghz * 1e9), rate(t_ex2lds) / sms / (ghz * 1e9), rate(t_cvt) / sms / (ghz * 1e9), rate(t_cvt2) / sms / (ghz * 1e9),
         rate(t_ex2) / sms / (ghz * 1e9), rate(t_ffma) / sms / (ghz * 1e9), rate(t_fadd) / sms / (ghz * 1e9),
         rate(t_fmax) / sms / (ghz * 1e9), rate(t_mixed) / sms / (ghz * 1e9));
  return 0;
}
