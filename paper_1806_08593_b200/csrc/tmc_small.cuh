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

constexpr int kMaxN = 32, kMaxK = 64, kMaxD = 128;
// Threads per CTA: 256 for tiny graphs, 512 when the per-datapoint work is larger (measured: C0
// 17.0 vs 17.6 us per launch, C1 30.9 vs 26.6 us; interleaved A/B, scripts/gpu_r2s.sh).
constexpr int kThreadsSmall = 256, kThreadsLarge = 512, kLargeWork = 1024;

struct Lat {
  const float *z, *mu, *lv, *logq, *logobs;   // inputs
  float *gz, *gmu, *glv, *gq, *go, *pair;      // gradient outputs (any may be NULL)
  int K, Kp, D, parent;
  double lnK;                                  // ln K (host-computed)
  // byte offsets into the dynamic shared memory (host-computed by layout()): fp64 h, msg; fp32 pi,
  // logq, logobs, z, mu, lam, ldet, and this latent's factor tile (the shared scratch when not cached)
  int o_h, o_m, o_pi, o_lq, o_lo, o_z, o_mu, o_lam, o_ldet, o_f, pad_[2];
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

// Shared-memory layout of one CTA (per-latent byte offsets written into A.l[i].o_*; computed on the
// host so the kernel addresses every array from a shared-memory descriptor instead of building
// per-thread pointer tables): fp64 h_i [K], msg_i [Kp]; then, 16-byte aligned, fp32 pi_i, logq_i,
// logobs_i [K], z_i [K][D], mu_i and lam_i = exp(-v_i) [Kp][D], ldet_i [Kp]; a K x Kp scratch; and
// with A.cache every latent's factor tile.  Returns the bytes.
__host__ inline size_t layout(Args& a) {
  size_t off = 0;
  for (int i = 0; i < a.n; ++i) {
    Lat& L = a.l[i];
    L.o_h = (int)off; off += 8 * (size_t)L.K;
    L.o_m = (int)off; off += 8 * (size_t)L.Kp;
  }
  off = (off + 15) & ~size_t(15);
  auto r4 = [](size_t x) { return 4 * ((x + 3) & ~size_t(3)); };   // bytes of a 16-byte aligned fp32 array
  int kk = 1, kp = 1;
  for (int i = 0; i < a.n; ++i) {
    Lat& L = a.l[i];
    L.o_pi = (int)off; off += r4(L.K);
    L.o_lq = (int)off; off += r4(L.K);
    L.o_lo = (int)off; off += r4(L.K);
    L.o_z = (int)off; off += r4((size_t)L.K * L.D);
    L.o_mu = (int)off; off += r4((size_t)L.Kp * L.D);
    L.o_lam = (int)off; off += r4((size_t)L.Kp * L.D);
    L.o_ldet = (int)off; off += r4(L.Kp);
    kk = L.K > kk ? L.K : kk;
    kp = L.Kp > kp ? L.Kp : kp;
  }
  const size_t scratch = off;
  off += r4((size_t)kk * kp);
  for (int i = 0; i < a.n; ++i) {
    if (a.cache) { a.l[i].o_f = (int)off; off += r4((size_t)a.l[i].K * a.l[i].Kp); }
    else a.l[i].o_f = (int)scratch;
  }
  return off;
}
__host__ inline size_t smem_bytes(const Args& a) {
  Args t = a;
  return layout(t);
}
// sum over latents of the staged elements (K D + Kp D): selects the CTA size
__host__ inline bool large_work(const Args& a) {
  long long w = 0;
  for (int i = 0; i < a.n; ++i) w += (long long)(a.l[i].K + a.l[i].Kp) * a.l[i].D;
  return w > kLargeWork;
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
__device__ void factor(const Lat& L, const Staged& S, float alpha, float* F, int t0 = -1) {
  const int D = L.D;
  for (int t = t0 < 0 ? (int)threadIdx.x : t0; t < L.K * L.Kp; t += NT) {
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

// NT threads per CTA (128 measured slower at C0 and C1: more work per thread, same barrier count).
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
  // every shared-memory array is addressed from the latent's descriptor (host-computed offsets)
  auto H = [&](int i) { return reinterpret_cast<double*>(smraw + sL[i].o_h); };
  auto M = [&](int i) { return reinterpret_cast<double*>(smraw + sL[i].o_m); };
  auto PI = [&](int i) { return reinterpret_cast<float*>(smraw + sL[i].o_pi); };
  auto FC = [&](int i) { return reinterpret_cast<float*>(smraw + sL[i].o_f); };
  auto ST = [&](int i) {
    const Lat& L = sL[i];
    return Staged{reinterpret_cast<float*>(smraw + L.o_z), reinterpret_cast<float*>(smraw + L.o_mu),
                  reinterpret_cast<float*>(smraw + L.o_lam), reinterpret_cast<float*>(smraw + L.o_ldet),
                  reinterpret_cast<float*>(smraw + L.o_lq), reinterpret_cast<float*>(smraw + L.o_lo)};
  };
  // Per-latent loops over small item counts start at a rotating thread: thread tid takes the items
  // t of latent i with (base_i + t) % NT == tid (base_i = the items of the latents before i), so the
  // latents of a small graph are spread over the CTA instead of all landing on threads 0.. .
  auto first = [&](int base) { const int f = (tid - base) % kThreads; return f < 0 ? f + kThreads : f; };
  // stage this datapoint's inputs once (all copies in flight together); later phases read shared memory
  {
    int base = 0;
    for (int i = 0; i < A.n; ++i) {
      const Lat& L = sL[i];
      const Staged S = ST(i);
      const float* z = L.z + (int64_t)b * L.K * L.D;
      const float* mu = L.mu + (int64_t)b * L.Kp * L.D;
      const float* lv = L.lv + (int64_t)b * L.Kp * L.D;
      for (int t = first(base); t < L.K * L.D; t += kThreads) cp_async4(S.z + t, z + t);
      base += L.K * L.D;
      for (int t = first(base); t < L.Kp * L.D; t += kThreads) { cp_async4(S.mu + t, mu + t); cp_async4(S.lam + t, lv + t); }
      base += L.Kp * L.D;
      for (int t = first(base); t < L.K; t += kThreads) {
        cp_async4(S.lq + t, L.logq + (int64_t)b * L.K + t);
        if (L.logobs) cp_async4(S.lo + t, L.logobs + (int64_t)b * L.K + t);
      }
      base += L.K;
    }
  }
  SMALL_MARK(0);
  cp_async_wait_all();
  __syncthreads();
  SMALL_MARK(1);
  // ldet = sum_d v, lam = exp(-v) in place (one thread per parameter row), h_i = alpha (logobs - logq)
  for (int i = 0, base = 0; i < A.n; ++i) {
    const Lat& L = sL[i];
    const Staged S = ST(i);
    for (int c = first(base); c < L.Kp; c += kThreads) {
      float sd = 0.f;
      for (int d = 0; d < L.D; ++d) {
        const float v = S.lam[c * L.D + d];
        sd += v;
        S.lam[c * L.D + d] = __expf(-v);
      }
      S.ldet[c] = sd;
    }
    base += L.Kp;
    for (int a = first(base); a < L.K; a += kThreads) {
      double u = -(double)S.lq[a];
      if (L.logobs) u += (double)S.lo[a];
      H(i)[a] = (double)A.alpha * u;
    }
    base += L.K;
  }
  __syncthreads();
  SMALL_MARK(2);
  // ---- upward: h_i = alpha (logobs_i - logq_i) + sum_children msg; msg_i[c] = LSE_a(F + h) - ln K_i
  __shared__ double s_logp;
  if (tid == 0) s_logp = 0.0;
  if (A.cache) {                                // every factor tile in one phase (they are independent)
    for (int i = 0, base = 0; i < A.n; ++i) {
      factor<NT>(sL[i], ST(i), A.alpha, FC(i), first(base));
      base += sL[i].K * sL[i].Kp;
    }
    __syncthreads();
  }
  for (int i = A.n - 1; i >= 0; --i) {          // parent[i] < i: children come first
    const Lat& L = sL[i];
    float* Fi = FC(i);
    if (!A.cache) {
      factor<NT>(L, ST(i), A.alpha, Fi);
      __syncthreads();
    }
    SMALL_MARK(3);
    // one warp per column c, lanes over a (K <= 64): warp-shuffle max and sum; lane 0 adds the
    // message into the parent's h (each column has one owner warp) or, at a root, into logp
    const int warp = tid >> 5, lane = tid & 31;
    const double lnK = L.lnK;
    // reductions over the lowest W lanes only (W = the power of two covering min(K, 32)); the
    // max is taken in fp32 (any value near the max stabilises the sum; x - m stays fp64)
    const int W = L.K >= 32 ? 32 : L.K > 16 ? 32 : L.K > 8 ? 16 : L.K > 4 ? 8 : L.K > 2 ? 4 : 2;
    for (int c = warp; c < L.Kp; c += kThreads / 32) {
      const double x0 = lane < L.K ? (double)Fi[lane * L.Kp + c] + H(i)[lane] : -INFINITY;
      const double x1 = lane + 32 < L.K ? (double)Fi[(lane + 32) * L.Kp + c] + H(i)[lane + 32] : -INFINITY;
      float mf = (float)fmax(x0, x1);
      for (int o = W >> 1; o; o >>= 1) mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, o));
      const double m = (double)mf;
      float s = 0.f;                            // terms ~<= 1 after the max: fp32 exp and sum
      if (mf > -INFINITY) s = __expf((float)(x0 - m)) + __expf((float)(x1 - m));
      for (int o = W >> 1; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        const double msg = (mf > -INFINITY) ? m + (double)__logf(s) - lnK : -INFINITY;
        M(i)[c] = msg;
        if (L.parent >= 0) H(L.parent)[c] += msg;
        else s_logp += msg;                     // a root's message is its (K_p = 1) evidence
      }
    }
    __syncthreads();
    SMALL_MARK(4);
  }
  const double logp = s_logp;
  if (tid == 0) A.logp[b] = logp;
  if (A.mode == 0) return;

  // ---- reverse: pi_root = w softmax(F_root + h_root); P_i[a,c] = pi_p[c] softmax_a(F_i + h_i)[a,c]
  const double w = (logp == -INFINITY) ? 0.0 : (A.dlogp ? A.dlogp[b] : 1.0);
  const float al = A.alpha;
  const int warp = tid >> 5, lane = tid & 31;
  // P (in place of the factor tile) of the rows a = warp, warp + 8, ... with lanes over c, and the
  // row sums pi_i[a] = sum_c P[a,c] (the marginal of z_i^a) from the same warp
  auto pair_rows = [&](int i, float* F) {
    const Lat& L = sL[i];
    const int W = L.Kp >= 32 ? 32 : L.Kp > 16 ? 32 : L.Kp > 8 ? 16 : L.Kp > 4 ? 8 : L.Kp > 2 ? 4 : 2;
    for (int a = warp; a < L.K; a += kThreads / 32) {
      float s = 0.f;
      for (int c = lane; c < L.Kp; c += 32) {
        const double up = (L.parent >= 0) ? (double)PI(L.parent)[c] : w;
        const double lm = M(i)[c] + L.lnK;
        const float pv = (up == 0.0 || lm == -INFINITY) ? 0.f
                         : (float)up * __expf((float)((double)F[a * L.Kp + c] + H(i)[a] - lm));
        F[a * L.Kp + c] = pv;
        s += pv;
      }
      for (int o = W >> 1; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        PI(i)[a] = s;
        if (L.go) L.go[(int64_t)b * L.K + a] = al * s;
        if (L.gq) L.gq[(int64_t)b * L.K + a] = -al * s;
      }
    }
  };
  // The gradients of latent i as items g = 0 .. nz + nm - 1: g < nz = K*D -> dz[a,d] = sum_c P (mu - z) lam;
  // else dmu, dlogvar of parameter row c (sums over a).  Thread tid takes the items of latent i
  // with (base + g) % NT == tid, where base counts the items of the latents before i: one
  // round-robin over every latent's items (small latents share the CTA), with the latent's
  // constants hoisted out of the item loop.
  auto grads = [&](int i, int base, const float* F) {
    const Lat& L = sL[i];
    const int D = L.D, K = L.K, Kp = L.Kp;
    const int nz = L.gz ? K * D : 0, nm = (L.gmu || L.glv) ? Kp * D : 0;
    const Staged S = ST(i);
    int g = (tid - base) % kThreads;
    if (g < 0) g += kThreads;
    for (; g < nz; g += kThreads) {
      const int a = g / D, d = g - a * D;
      const float zz = S.z[a * D + d];
      float acc = 0.f;
      for (int c = 0; c < Kp; ++c) acc += F[a * Kp + c] * (S.mu[c * D + d] - zz) * S.lam[c * D + d];
      L.gz[(int64_t)b * K * D + g] = al * acc;
    }
    for (g -= nz; g < nm; g += kThreads) {
      const int c = g / D, d = g - c * D;
      const float lam = S.lam[c * D + d], mu = S.mu[c * D + d];
      float s1 = 0.f, s2 = 0.f, sp = 0.f;
      for (int a = 0; a < K; ++a) {
        const float pv = F[a * Kp + c], df = S.z[a * D + d] - mu;
        s1 += pv * df;
        s2 += pv * df * df;
        sp += pv;
      }
      if (L.gmu) L.gmu[(int64_t)b * Kp * D + g] = al * lam * s1;
      if (L.glv) L.glv[(int64_t)b * Kp * D + g] = al * 0.5f * (lam * s2 - sp);
    }
    return nz + nm;
  };
  if (A.cache) {
    // every latent keeps its own tile: the top-down P sweep (one phase per latent), then every
    // latent's gradients and pair marginals in one flattened phase
    for (int i = 0; i < A.n; ++i) {
      pair_rows(i, FC(i));
      __syncthreads();
    }
    SMALL_MARK(6);
    int base = 0;
    for (int i = 0; i < A.n; ++i) base += grads(i, base, FC(i));
    for (int i = 0; i < A.n; ++i) {
      const Lat& L = sL[i];
      if (L.pair)
        for (int t = tid; t < L.K * L.Kp; t += kThreads) L.pair[(int64_t)b * L.K * L.Kp + t] = al * FC(i)[t];
    }
    SMALL_MARK(8);
  } else {
    for (int i = 0; i < A.n; ++i) {
      const Lat& L = sL[i];
      float* F = FC(i);
      factor<NT>(L, ST(i), A.alpha, F);
      __syncthreads();
      SMALL_MARK(5);
      pair_rows(i, F);
      __syncthreads();
      SMALL_MARK(7);
      if (L.pair)
        for (int t = tid; t < L.K * L.Kp; t += kThreads) L.pair[(int64_t)b * L.K * L.Kp + t] = al * F[t];
      grads(i, 0, F);
      SMALL_MARK(8);
      __syncthreads();                          // the next latent reuses the scratch tile
      SMALL_MARK(9);
    }
  }
}
#undef SMALL_MARK

}  // namespace small
}  // namespace tmc
