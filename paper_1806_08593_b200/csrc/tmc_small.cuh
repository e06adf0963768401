// Small problems (C0 and C1 are launch-latency bound; target one launch per call).
// One CTA per datapoint runs the whole estimator for a tree with K_i <= 64, D_i <= 128, n <= 32 in
// shared memory: the upward elimination, the final LSE, and - for the reverse
// pass - the top-down marginals and every input gradient.  Factors are recomputed in the
// direct form in fp32; messages, h and the LSEs are carried in fp64, so no offset
// bookkeeping is needed.  tmc_forward = one launch (mode 0); tmc_backward = one launch that redoes
// the (cheap) forward and then the reverse pass (mode 1); the workspace is not used.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmc {
namespace small {

constexpr int kMaxN = 32, kMaxK = 64, kMaxD = 128, kThreads = 256;

struct Lat {
  const float *z, *mu, *lv, *logq, *logobs;   // inputs
  float *gz, *gmu, *glv, *gq, *go, *pair;      // gradient outputs (any may be NULL)
  int K, Kp, D, parent;
  double lnK;                                  // ln K (host-computed)
};
static_assert(sizeof(Lat) % 16 == 0, "Lat is copied to shared memory in 16-byte units");
struct Args {
  Lat l[kMaxN];
  int n, B, mode;                              // mode 0: logp only; 1: logp + gradients
  int cache;                                   // 1: keep every latent's factor tile from the forward sweep (mode 1)
  float alpha;
  const double* dlogp;
  double* logp;
};

// shared-memory bytes for the graph (per CTA): fp64 h_i, msg_i; fp32 pi_i, the staged inputs
// z_i [K][D], mu_i and lam_i = exp(-v_i) [Kp][D], ldet_i [Kp] = sum_d v_i, and a K x Kp scratch.
__host__ inline size_t smem_bytes(const Args& a) {
  size_t d = 0, f = 0;
  int kk = 1, kp = 1;
  auto r4 = [](size_t x) { return (x + 3) & ~size_t(3); };      // every fp32 array 16-byte aligned
  for (int i = 0; i < a.n; ++i) {
    const Lat& L = a.l[i];
    d += (size_t)L.K + L.Kp;
    f += 3 * r4(L.K) + r4((size_t)L.K * L.D) + 2 * r4((size_t)L.Kp * L.D) + r4(L.Kp);   // pi, logq, logobs, z, mu, lam, ldet
    kk = L.K > kk ? L.K : kk;
    kp = L.Kp > kp ? L.Kp : kp;
  }
  f += (size_t)kk * kp;
  if (a.cache)
    for (int i = 0; i < a.n; ++i) f += r4((size_t)a.l[i].K * a.l[i].Kp);   // per-latent factor tiles
  return 8 * d + 4 * f + 64;
}

struct Staged { float *z, *mu, *lam, *ldet, *lq, *lo; };

// 4-byte asynchronous global -> shared copy (LDGSTS): every staging copy of the CTA is in flight
// at once, so the whole datapoint arrives in about one memory latency.
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// F[a*Kp + c] = alpha * (sum_d log N(z[a,d]; mu[c,d], exp(v[c,d])))   (logq enters through h)
template <int NT>
__device__ void factor(const Lat& L, const Staged& S, float alpha, float* F) {
  const int D = L.D;
  for (int t = threadIdx.x; t < L.K * L.Kp; t += NT) {
    const int a = t / L.Kp, c = t - a * L.Kp;
    float q = 0.f, q2 = 0.f;
    if ((D & 3) == 0) {                       // 16-byte shared-memory loads, two accumulators
      const float4* z4 = reinterpret_cast<const float4*>(S.z + a * D);
      const float4* m4 = reinterpret_cast<const float4*>(S.mu + c * D);
      const float4* l4 = reinterpret_cast<const float4*>(S.lam + c * D);
      for (int d = 0; d < (D >> 2); ++d) {
        const float4 zz = z4[d], mm = m4[d], ll = l4[d];
        const float d0 = zz.x - mm.x, d1 = zz.y - mm.y, d2 = zz.z - mm.z, d3 = zz.w - mm.w;
        q = fmaf(d0 * d0, ll.x, q);
        q2 = fmaf(d1 * d1, ll.y, q2);
        q = fmaf(d2 * d2, ll.z, q);
        q2 = fmaf(d3 * d3, ll.w, q2);
      }
    } else {
      for (int d = 0; d < D; ++d) {
        const float df = S.z[a * D + d] - S.mu[c * D + d];
        q = fmaf(df * df, S.lam[c * D + d], q);
      }
    }
    F[t] = alpha * (-0.5f * ((q + q2) + S.ldet[c] + D * 1.8378770664093453f));
  }
}

__device__ __forceinline__ int kkmax(const Lat* l, int n) { int m = 1; for (int i = 0; i < n; ++i) m = l[i].K > m ? l[i].K : m; return m; }
__device__ __forceinline__ int kpmax(const Lat* l, int n) { int m = 1; for (int i = 0; i < n; ++i) m = l[i].Kp > m ? l[i].Kp : m; return m; }

// NT = kThreads threads per CTA (128 measured slower at C0 and C1: more work per thread, same barrier count).
template <int NT>
__global__ void __launch_bounds__(NT) small_kernel(const __grid_constant__ Args A) {
  constexpr int kThreads = NT;
  extern __shared__ __align__(16) unsigned char smraw[];
  // the per-latent descriptors, copied once from the parameter space in parallel (a chain of
  // constant-cache misses through the latent loops cost ~6000 clk at C0)
  __shared__ __align__(16) Lat sL[kMaxN];
  const int b = blockIdx.x, tid = threadIdx.x;
  {
    const uint4* src = reinterpret_cast<const uint4*>(&A.l[0]);
    uint4* dst = reinterpret_cast<uint4*>(sL);
    const int nq = A.n * (int)(sizeof(Lat) / 16);
    for (int q = tid; q < nq; q += NT) dst[q] = src[q];
    __syncthreads();
  }
#ifdef TMC_INSTRUMENT
  long long _ph = clock64();
#define SMALL_MARK(k) do { if (tid == 0) { const long long _n = clock64(); tc::g_tmc_prof[b & 1023][50 + (k)] += _n - _ph; _ph = _n; } } while (0)
#else
#define SMALL_MARK(k) do {} while (0)
#endif
  double* dp = reinterpret_cast<double*>(smraw);
  double* H[kMaxN];
  double* M[kMaxN];
  for (int i = 0; i < A.n; ++i) { H[i] = dp; dp += sL[i].K; M[i] = dp; dp += sL[i].Kp; }
  if ((reinterpret_cast<uintptr_t>(dp) & 15) != 0) ++dp;      // fp32 region 16-byte aligned (slack in smem_bytes)
  float* fp = reinterpret_cast<float*>(dp);
  float* PI[kMaxN];
  Staged ST[kMaxN];
  auto r4 = [](int x) { return (x + 3) & ~3; };            // matches smem_bytes: 16-byte aligned arrays
  for (int i = 0; i < A.n; ++i) {
    const Lat& L = sL[i];
    PI[i] = fp; fp += r4(L.K);
    ST[i].lq = fp; fp += r4(L.K);
    ST[i].lo = fp; fp += r4(L.K);
    ST[i].z = fp; fp += r4(L.K * L.D);
    ST[i].mu = fp; fp += r4(L.Kp * L.D);
    ST[i].lam = fp; fp += r4(L.Kp * L.D);
    ST[i].ldet = fp; fp += r4(L.Kp);
  }
  float* F = fp;
  float* FC[kMaxN];                           // per-latent factor tiles (cache) or the shared scratch
  {
    float* q = fp + r4(kkmax(sL, A.n) * kpmax(sL, A.n));
    for (int i = 0; i < A.n; ++i) {
      if (A.cache) { FC[i] = q; q += r4(sL[i].K * sL[i].Kp); }
      else FC[i] = F;
    }
  }
  // stage this datapoint's inputs once (all copies in flight together); later phases read shared memory
  for (int i = 0; i < A.n; ++i) {
    const Lat& L = sL[i];
    const float* z = L.z + (int64_t)b * L.K * L.D;
    const float* mu = L.mu + (int64_t)b * L.Kp * L.D;
    const float* lv = L.lv + (int64_t)b * L.Kp * L.D;
    for (int t = tid; t < L.K * L.D; t += kThreads) cp_async4(ST[i].z + t, z + t);
    for (int t = tid; t < L.Kp * L.D; t += kThreads) { cp_async4(ST[i].mu + t, mu + t); cp_async4(ST[i].lam + t, lv + t); }
    for (int t = tid; t < L.K; t += kThreads) {
      cp_async4(ST[i].lq + t, L.logq + (int64_t)b * L.K + t);
      if (L.logobs) cp_async4(ST[i].lo + t, L.logobs + (int64_t)b * L.K + t);
    }
  }
  SMALL_MARK(0);
  cp_async_wait_all();
  __syncthreads();
  SMALL_MARK(1);
  for (int i = 0; i < A.n; ++i) {              // ldet from the raw log-variances
    const Lat& L = sL[i];
    for (int c = tid; c < L.Kp; c += kThreads) {
      float sd = 0.f;
      for (int d = 0; d < L.D; ++d) sd += ST[i].lam[c * L.D + d];
      ST[i].ldet[c] = sd;
    }
  }
  // ---- upward: h_i = alpha (logobs_i - logq_i) + sum_children msg; msg_i[c] = LSE_a(F + h) - ln K_i
  for (int i = 0; i < A.n; ++i) {
    const Lat& L = sL[i];
    for (int a = tid; a < L.K; a += kThreads) {
      double u = -(double)ST[i].lq[a];
      if (L.logobs) u += (double)ST[i].lo[a];
      H[i][a] = (double)A.alpha * u;
    }
  }
  __syncthreads();
  for (int i = 0; i < A.n; ++i) {              // lam = exp(-v) in place (after ldet read v)
    const Lat& L = sL[i];
    for (int t = tid; t < L.Kp * L.D; t += kThreads) ST[i].lam[t] = __expf(-ST[i].lam[t]);
  }
  __syncthreads();
  SMALL_MARK(2);
  double logp = 0.0;
  for (int i = A.n - 1; i >= 0; --i) {          // parent[i] < i: children come first
    const Lat& L = sL[i];
    float* Fi = FC[i];
    factor<NT>(L, ST[i], A.alpha, Fi);
    __syncthreads();
    SMALL_MARK(3);
    // one warp per column c, lanes over a (K <= 64): warp-shuffle max and sum
    const int warp = tid >> 5, lane = tid & 31;
    const double lnK = L.lnK;
    for (int c = warp; c < L.Kp; c += kThreads / 32) {
      const double x0 = lane < L.K ? (double)Fi[lane * L.Kp + c] + H[i][lane] : -INFINITY;
      const double x1 = lane + 32 < L.K ? (double)Fi[(lane + 32) * L.Kp + c] + H[i][lane + 32] : -INFINITY;
      double m = fmax(x0, x1);
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      float s = 0.f;                            // terms <= 1 after the max: fp32 exp and sum
      if (m > -INFINITY) s = __expf((float)(x0 - m)) + __expf((float)(x1 - m));
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) M[i][c] = (m > -INFINITY) ? m + (double)__logf(s) - lnK : -INFINITY;
    }
    __syncthreads();
    if (L.parent >= 0) {
      for (int c = tid; c < L.Kp; c += kThreads) H[L.parent][c] += M[i][c];
    } else {
      logp += M[i][0];                          // a root's message is its (K_p = 1) evidence
    }
    __syncthreads();
    SMALL_MARK(4);
  }
  if (tid == 0) A.logp[b] = logp;
  if (A.mode == 0) return;

  // ---- reverse: pi_root = w softmax(F_root + h_root); P_i[a,c] = pi_p[c] softmax_a(F_i + h_i)[a,c]
  const double w = (logp == -INFINITY) ? 0.0 : (A.dlogp ? A.dlogp[b] : 1.0);
  for (int i = 0; i < A.n; ++i) {
    const Lat& L = sL[i];
    float* F = FC[i];                        // the forward sweep's factor tile when cached
    if (!A.cache) factor<NT>(L, ST[i], A.alpha, F);
    __syncthreads();
    SMALL_MARK(5);
    // P (in place of F): weight of pair (a, c)
    for (int t = tid; t < L.K * L.Kp; t += kThreads) {
      const int a = t / L.Kp, c = t - a * L.Kp;
      const double up = (L.parent >= 0) ? (double)PI[L.parent][c] : w;
      const double lm = M[i][c] + L.lnK;
      F[t] = (up == 0.0 || lm == -INFINITY) ? 0.f : (float)up * __expf((float)((double)F[t] + H[i][a] - lm));
    }
    __syncthreads();
    SMALL_MARK(6);
    const float al = A.alpha;
    {
      const int warp = tid >> 5, lane = tid & 31;   // one warp per row a, lanes over c
      for (int a = warp; a < L.K; a += kThreads / 32) {
        float s = 0.f;
        for (int c = lane; c < L.Kp; c += 32) s += F[a * L.Kp + c];
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
          PI[i][a] = s;
          if (L.go) L.go[(int64_t)b * L.K + a] = al * s;
          if (L.gq) L.gq[(int64_t)b * L.K + a] = -al * s;
        }
      }
    }
    SMALL_MARK(7);
    if (L.pair)
      for (int t = tid; t < L.K * L.Kp; t += kThreads) L.pair[(int64_t)b * L.K * L.Kp + t] = al * F[t];
    const int D = L.D;
    const float* z = ST[i].z;
    const float* mu = ST[i].mu;
    const float* lamv = ST[i].lam;
    if (L.gz)
      for (int t = tid; t < L.K * D; t += kThreads) {          // dz[a,d] = sum_c P (mu - z) lam
        const int a = t / D, d = t - a * D;
        float acc = 0.f;
        for (int c = 0; c < L.Kp; ++c)
          acc += F[a * L.Kp + c] * (mu[c * D + d] - z[a * D + d]) * lamv[c * D + d];
        L.gz[(int64_t)b * L.K * D + t] = al * acc;
      }
    if (L.gmu || L.glv)
      for (int t = tid; t < L.Kp * D; t += kThreads) {         // dmu, dlogvar of parent sample c
        const int c = t / D, d = t - c * D;
        const float lam = lamv[c * D + d];
        float s1 = 0.f, s2 = 0.f, sp = 0.f;
        for (int a = 0; a < L.K; ++a) {
          const float p = F[a * L.Kp + c], df = z[a * D + d] - mu[c * D + d];
          s1 += p * df;
          s2 += p * df * df;
          sp += p;
        }
        if (L.gmu) L.gmu[(int64_t)b * L.Kp * D + t] = al * lam * s1;
        if (L.glv) L.glv[(int64_t)b * L.Kp * D + t] = al * 0.5f * (lam * s2 - sp);
      }
    SMALL_MARK(8);
    __syncthreads();
    SMALL_MARK(9);
  }
}
#undef SMALL_MARK

}  // namespace small
}  // namespace tmc
