// the IWAE estimator at equal K on the same inputs as TMC, so the
// two can be timed side by side ("TMC cost ~ IWAE cost").  The K joint samples
// are the index tuples (k, ..., k): latent i's k-th sample with its conditional at the parent's
// k-th sample (the root at its prior, column 0).
//   log w[b,k] = sum_i [ log N(z_i[b,k]; mu_i[b,c], exp(v_i[b,c])) - logq_i[b,k] + logobs_i[b,k] ],  c = k (root: 0)
//   L[b] = LSE_k log w[b,k] - ln K;  pi[b,k] = dlogp[b] softmax_k(log w[b,:])
//   dlogobs = pi, dlogq = -pi, dz = pi (mu - z) lam, dmu[c] = pi (z - mu) lam, dv[c] = pi/2 ((z - mu)^2 lam - 1)
// (root: dmu, dv summed over k).  O(B n K D) work: HBM-bound; three launches per latent chunk.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/tmc.h"

namespace tmc {
namespace iwae {

constexpr int kMaxLat = 48;
struct LatDesc {
  const float *z, *mu, *lv, *logq, *logobs;
  float *gz, *gmu, *glv, *gq, *go;
  int D, root;
};
struct Batch {
  LatDesc l[kMaxLat];
  int count, B, K;
  float alpha;
};

// log w[b,k] (+)= sum over this chunk's latents; one warp per (b, k) row, lanes over d (coalesced).
__global__ void __launch_bounds__(256) logw_kernel(const __grid_constant__ Batch bt, double* __restrict__ w, int first) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= (int64_t)bt.B * bt.K) return;
  const int b = (int)(row / bt.K), k = (int)(row % bt.K);
  double acc = first ? 0.0 : w[row];   // per-latent terms in fp32, their sum in fp64
  // unrolled over latents so several latents' row loads are in flight at once (HBM latency)
#pragma unroll 4
  for (int j = 0; j < bt.count; ++j) {
    const LatDesc& L = bt.l[j];
    const int c = L.root ? 0 : k, Kp = L.root ? 1 : bt.K, D = L.D;
    const float* z = L.z + row * D;
    const float* mu = L.mu + ((int64_t)b * Kp + c) * D;
    const float* lv = L.lv + ((int64_t)b * Kp + c) * D;
    float q = 0.f;
    for (int d = lane; d < D; d += 32) {
      const float df = __ldg(z + d) - __ldg(mu + d);
      const float v = __ldg(lv + d);
      q += df * df * __expf(-v) + v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    float t = -0.5f * (q + D * 1.8378770664093453f) - L.logq[row];
    if (L.logobs) t += L.logobs[row];
    acc += (double)(bt.alpha * t);
  }
  if (lane == 0) w[row] = acc;
}

// Vectorised variants (every latent's D % 4 == 0): 4 rows per warp, 8 lanes per row, float4 loads,
// so each warp keeps 4x the bytes in flight of the one-row-per-warp kernels (HBM latency bound).
__global__ void __launch_bounds__(256) logw4_kernel(const __grid_constant__ Batch bt, double* __restrict__ w, int first) {
  const int lane = threadIdx.x & 31, sub = lane & 7;
  const int64_t row = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 4 + (lane >> 3);
  const bool ok = row < (int64_t)bt.B * bt.K;
  const int64_t rr = ok ? row : 0;
  const int b = (int)(rr / bt.K), k = (int)(rr % bt.K);
  double acc = (first || !ok) ? 0.0 : w[rr];
#pragma unroll 2
  for (int j = 0; j < bt.count; ++j) {
    const LatDesc& L = bt.l[j];
    const int c = L.root ? 0 : k, Kp = L.root ? 1 : bt.K, D4 = L.D >> 2;
    const float4* z = reinterpret_cast<const float4*>(L.z + rr * L.D);
    const float4* mu = reinterpret_cast<const float4*>(L.mu + ((int64_t)b * Kp + c) * L.D);
    const float4* lv = reinterpret_cast<const float4*>(L.lv + ((int64_t)b * Kp + c) * L.D);
    float q = 0.f;
    for (int d = sub; d < D4; d += 8) {
      const float4 zz = __ldg(z + d), mm = __ldg(mu + d), vv = __ldg(lv + d);
      const float d0 = zz.x - mm.x, d1 = zz.y - mm.y, d2 = zz.z - mm.z, d3 = zz.w - mm.w;
      q += d0 * d0 * __expf(-vv.x) + vv.x + d1 * d1 * __expf(-vv.y) + vv.y;
      q += d2 * d2 * __expf(-vv.z) + vv.z + d3 * d3 * __expf(-vv.w) + vv.w;
    }
#pragma unroll
    for (int o = 4; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    float t = -0.5f * (q + L.D * 1.8378770664093453f) - __ldg(L.logq + rr);
    if (L.logobs) t += __ldg(L.logobs + rr);
    acc += (double)(bt.alpha * t);
  }
  if (ok && sub == 0) w[rr] = acc;
}

__global__ void __launch_bounds__(256) grad4_kernel(const __grid_constant__ Batch bt, const double* __restrict__ pi) {
  const int lane = threadIdx.x & 31, sub = lane & 7;
  const int64_t row = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 4 + (lane >> 3);
  if (row >= (int64_t)bt.B * bt.K) return;
  const float p = (float)(bt.alpha * pi[row]);
#pragma unroll 2
  for (int j = 0; j < bt.count; ++j) {
    const LatDesc& L = bt.l[j];
    if (sub == 0) {
      if (L.go) L.go[row] = p;
      if (L.gq) L.gq[row] = -p;
    }
    if (L.root) continue;
    const int D4 = L.D >> 2;
    const float4* z = reinterpret_cast<const float4*>(L.z + row * L.D);
    const float4* mu = reinterpret_cast<const float4*>(L.mu + row * L.D);
    const float4* lv = reinterpret_cast<const float4*>(L.lv + row * L.D);
    for (int d = sub; d < D4; d += 8) {
      const float4 zz = __ldg(z + d), mm = __ldg(mu + d), vv = __ldg(lv + d);
      const float4 lam = make_float4(__expf(-vv.x), __expf(-vv.y), __expf(-vv.z), __expf(-vv.w));
      const float4 df = make_float4(zz.x - mm.x, zz.y - mm.y, zz.z - mm.z, zz.w - mm.w);
      if (L.gz) reinterpret_cast<float4*>(L.gz + row * L.D)[d] =
          make_float4(-p * df.x * lam.x, -p * df.y * lam.y, -p * df.z * lam.z, -p * df.w * lam.w);
      if (L.gmu) reinterpret_cast<float4*>(L.gmu + row * L.D)[d] =
          make_float4(p * df.x * lam.x, p * df.y * lam.y, p * df.z * lam.z, p * df.w * lam.w);
      if (L.glv) reinterpret_cast<float4*>(L.glv + row * L.D)[d] =
          make_float4(0.5f * p * (df.x * df.x * lam.x - 1.f), 0.5f * p * (df.y * df.y * lam.y - 1.f),
                      0.5f * p * (df.z * df.z * lam.z - 1.f), 0.5f * p * (df.w * df.w * lam.w - 1.f));
    }
  }
}

// logp[b] = LSE_k w - ln K (fp64 result), then w <- pi = dlogp[b] softmax(w) in place.
__global__ void __launch_bounds__(256) lse_kernel(double* __restrict__ w, int K, const double* dlogp, double* logp) {
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double red[32];
  __shared__ double dred[32];
  double* wb = w + (int64_t)b * K;
  double m = -INFINITY;
  for (int k = tid; k < K; k += 256) m = fmax(m, wb[k]);
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (tid == 0) {
    double v = red[0];
    for (int j = 1; j < 8; ++j) v = fmax(v, red[j]);
    red[16] = v;
  }
  __syncthreads();
  const double M = red[16];
  double s = 0.0;
  if (M > -INFINITY)
    for (int k = tid; k < K; k += 256) s += (double)__expf((float)(wb[k] - M));
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) dred[warp] = s;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int j = 0; j < 8; ++j) t += dred[j];
    dred[16] = t;
    logp[b] = (M == -INFINITY || t <= 0.0) ? -INFINITY : M + log(t) - log((double)K);
  }
  __syncthreads();
  const double S = dred[16];
  const double scale = (S > 0.0) ? (dlogp ? dlogp[b] : 1.0) / S : 0.0;
  for (int k = tid; k < K; k += 256) wb[k] = (M > -INFINITY) ? scale * (double)__expf((float)(wb[k] - M)) : 0.0;
}

// Non-root latents: one warp per (b, k) row, lanes over d.
__global__ void __launch_bounds__(256) grad_kernel(const __grid_constant__ Batch bt, const double* __restrict__ pi) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= (int64_t)bt.B * bt.K) return;
  const float p = (float)(bt.alpha * pi[row]);
#pragma unroll 4
  for (int j = 0; j < bt.count; ++j) {
    const LatDesc& L = bt.l[j];
    if (lane == 0) {
      if (L.go) L.go[row] = p;
      if (L.gq) L.gq[row] = -p;
    }
    if (L.root) continue;
    const int D = L.D;
    for (int d = lane; d < D; d += 32) {
      const float z = __ldg(L.z + row * D + d), mu = __ldg(L.mu + row * D + d), lv = __ldg(L.lv + row * D + d);
      const float lam = __expf(-lv), df = z - mu;
      if (L.gz) L.gz[row * D + d] = -p * df * lam;
      if (L.gmu) L.gmu[row * D + d] = p * df * lam;
      if (L.glv) L.glv[row * D + d] = 0.5f * p * (df * df * lam - 1.f);
    }
  }
}

// Root latents of the chunk: dz per (b, k); dmu / dv of the prior summed over k.  One CTA per
// (b, root): 8 warps stride over k, lanes over d (up to 8 chunks of 32 dims), then a shared-memory
// reduction over the warps.
constexpr int kRootMaxChunks = 8;                     // D <= 256
constexpr int kRootWarps = 16;
__global__ void __launch_bounds__(kRootWarps * 32) root_grad_kernel(const __grid_constant__ Batch bt, const double* __restrict__ pi) {
  const int b = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ float red[3][kRootWarps][kRootMaxChunks * 32];
  int seen = -1;
  for (int j = 0; j < bt.count; ++j) {
    if (!bt.l[j].root) continue;
    if (++seen != (int)blockIdx.y) continue;
    const LatDesc& L = bt.l[j];
    const int D = L.D, nch = (D + 31) / 32;
    const float* mu = L.mu + (int64_t)b * D;
    const float* lv = L.lv + (int64_t)b * D;
    float s1[kRootMaxChunks], s2[kRootMaxChunks], sp = 0.f;
#pragma unroll
    for (int q = 0; q < kRootMaxChunks; ++q) { s1[q] = 0.f; s2[q] = 0.f; }
#pragma unroll 4
    for (int k = warp; k < bt.K; k += kRootWarps) {
      const int64_t r = (int64_t)b * bt.K + k;
      const float p = (float)(bt.alpha * pi[r]);
      sp += p;
#pragma unroll
      for (int q = 0; q < kRootMaxChunks; ++q) {
        const int d = q * 32 + lane;
        if (q >= nch || d >= D) continue;
        const float lam = __expf(-lv[d]), df = L.z[r * D + d] - mu[d];
        if (L.gz) L.gz[r * D + d] = -p * df * lam;
        s1[q] += p * df;
        s2[q] += p * df * df;
      }
    }
#pragma unroll
    for (int q = 0; q < kRootMaxChunks; ++q) {
      red[0][warp][q * 32 + lane] = s1[q];
      red[1][warp][q * 32 + lane] = s2[q];
    }
    red[2][warp][lane] = sp;
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      float a1 = 0.f, a2 = 0.f, ap = 0.f;
      for (int w2 = 0; w2 < kRootWarps; ++w2) { a1 += red[0][w2][d]; a2 += red[1][w2][d]; ap += red[2][w2][0]; }
      const float lam = __expf(-lv[d]);
      if (L.gmu) L.gmu[(int64_t)b * D + d] = lam * a1;
      if (L.glv) L.glv[(int64_t)b * D + d] = 0.5f * (lam * a2 - ap);
    }
    __syncthreads();
  }
}

}  // namespace iwae
}  // namespace tmc
