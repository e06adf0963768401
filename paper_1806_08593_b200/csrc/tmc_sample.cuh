// reparameterisation noise eps ~ N(0, I) for the proposal samples
// z_i = mu_q + sigma_q * eps, drawn on the device, bit-exact with a host
// implementation.
//
//   Philox4x32-10 (Salmon et al., SC'11): key = (seed lo, seed hi), counter =
//   (tag, global datapoint b, latent i, k * ceil(D/4) + d/4); the 4 output words give eps for
//   d = 4j .. 4j+3 of sample k (two Box-Muller pairs).
//   uniform u = ((x >> 8) + 0.5) * 2^-24 in (0, 1); Box-Muller eps = sqrt(-2 ln u1) * (cos, sin)(2 pi u2)
//   with ln and sincos as fixed fp32 polynomials (coefficients: the fp32 values nearest 1/(2j+1),
//   +-1/n!, ln 2, 2 pi, sqrt 2, written as exact hex literals) evaluated with explicitly rounded fma / mul / add /
//   div / sqrt only, so any IEEE fp32 implementation that performs the same operations (the host
//   side lives in oracle/, written independently from the same definition) produces the same bits.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmc {
namespace rng {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u, kPhiloxW1 = 0xBB67AE85u;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(kPhiloxM0, c.x), lo0 = kPhiloxM0 * c.x;
    const uint32_t hi1 = __umulhi(kPhiloxM1, c.z), lo1 = kPhiloxM1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += kPhiloxW0;
    k.y += kPhiloxW1;
  }
  return c;
}

__device__ __forceinline__ float u01(uint32_t x) {       // (0, 1), exact in fp32
  return __fmul_rn(__fadd_rn((float)(x >> 8), 0.5f), 5.9604644775390625e-8f);   // 2^-24
}

// ln(u) for u in (0, 1]: u = 2^e m with m in [sqrt(1/2), sqrt(2)); ln m = 2 atanh(s),
// s = (m - 1)/(m + 1), |s| <= 0.1716: odd series to s^13 (truncation < 1e-12 relative).
__device__ __forceinline__ float ln_poly(float u) {
  uint32_t bits = __float_as_uint(u);
  int e = (int)((bits >> 23) & 0xFF) - 127;
  float m = __uint_as_float((bits & 0x007FFFFFu) | 0x3F800000u);      // [1, 2)
  if (m > 0x1.6a09e6p+0f) { m = __fmul_rn(m, 0.5f); e += 1; }
  const float s = __fdiv_rn(__fadd_rn(m, -1.0f), __fadd_rn(m, 1.0f));
  const float s2 = __fmul_rn(s, s);
  float p = 0x1.3b13b2p-4f;                                             // fp32(1/13)
  p = __fmaf_rn(p, s2, 0x1.745d18p-4f);                                 // 1/11
  p = __fmaf_rn(p, s2, 0x1.c71c72p-4f);                                 // 1/9
  p = __fmaf_rn(p, s2, 0x1.24924ap-3f);                                 // 1/7
  p = __fmaf_rn(p, s2, 0x1.99999ap-3f);                                 // 1/5
  p = __fmaf_rn(p, s2, 0x1.555556p-2f);                                 // 1/3
  p = __fmaf_rn(p, s2, 1.0f);
  const float lnm = __fmul_rn(__fmul_rn(2.0f, s), p);
  return __fmaf_rn((float)e, 0x1.62e430p-1f, lnm);                         // fp32(ln 2)
}

// (cos, sin)(2 pi v) for v in [0, 1): quadrant q = rint(4v), w = v - q/4 in [-1/8, 1/8],
// x = 2 pi w, Taylor polynomials (|x| <= pi/4: sin to x^11, cos to x^12), then the quadrant rotation.
__device__ __forceinline__ void sincos2pi_poly(float v, float& c, float& s) {
  const float q = rintf(__fmul_rn(v, 4.0f));
  const float w = __fadd_rn(v, __fmul_rn(q, -0.25f));
  const float x = __fmul_rn(w, 0x1.921fb6p+2f);                            // fp32(2 pi)
  const float x2 = __fmul_rn(x, x);
  float ps = -0x1.ae6456p-26f;                                          // fp32(-1/11!)
  ps = __fmaf_rn(ps, x2, 0x1.71de3ap-19f);                              //  1/9!
  ps = __fmaf_rn(ps, x2, -0x1.a01a02p-13f);                             // -1/7!
  ps = __fmaf_rn(ps, x2, 0x1.111112p-7f);                               //  1/5!
  ps = __fmaf_rn(ps, x2, -0x1.555556p-3f);                              // -1/3!
  ps = __fmaf_rn(__fmul_rn(ps, x2), x, x);
  float pc = 0x1.1eed8ep-29f;                                           //  fp32(1/12!)
  pc = __fmaf_rn(pc, x2, -0x1.27e4fcp-22f);                             // -1/10!
  pc = __fmaf_rn(pc, x2, 0x1.a01a02p-16f);                              //  1/8!
  pc = __fmaf_rn(pc, x2, -0x1.6c16c2p-10f);                             // -1/6!
  pc = __fmaf_rn(pc, x2, 0x1.555556p-5f);                               //  1/4!
  pc = __fmaf_rn(pc, x2, -0.5f);
  pc = __fmaf_rn(pc, x2, 1.0f);
  const int qi = ((int)q) & 3;
  c = (qi == 0) ? pc : (qi == 1) ? -ps : (qi == 2) ? -pc : ps;
  s = (qi == 0) ? ps : (qi == 1) ? pc : (qi == 2) ? -ps : -pc;
}

__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& n0, float& n1) {
  const float r = __fsqrt_rn(__fmul_rn(-2.0f, ln_poly(u01(a))));
  float c, s;
  sincos2pi_poly(u01(b), c, s);
  n0 = __fmul_rn(r, c);
  n1 = __fmul_rn(r, s);
}

// eps[b][k][d] for datapoints b0 .. b0+B-1 (global ids), one thread per (b, k, 4-dim group).
__global__ void __launch_bounds__(256) normal_kernel(uint64_t seed, uint32_t tag, int B, int64_t b0, int latent,
                                                     int K, int D, float* __restrict__ eps) {
  const int G = (D + 3) >> 2;
  const int64_t n = (int64_t)B * K * G;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(t % G);
    const int64_t bk = t / G;
    const int k = (int)(bk % K);
    const int b = (int)(bk / K);
    const uint4 x = philox4x32_10(make_uint4(tag, (uint32_t)(b0 + b), (uint32_t)latent, (uint32_t)(k * G + g)),
                                  make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    float e[4];
    box_muller(x.x, x.y, e[0], e[1]);
    box_muller(x.z, x.w, e[2], e[3]);
    float* out = eps + ((int64_t)b * K + k) * D + 4 * g;
    const int nd = min(4, D - 4 * g);
    if (nd == 4 && (D & 3) == 0) {
      *reinterpret_cast<float4*>(out) = make_float4(e[0], e[1], e[2], e[3]);
    } else {
      for (int q = 0; q < nd; ++q) out[q] = e[q];
    }
  }
}

}  // namespace rng
}  // namespace tmc
