// General TMC elimination on a factor graph over sample indices.
//
// PAPER.md §"Efficient averaging" (Fig[factor:loop] P:145-215): the TMC estimate of a
// loopy factor graph is computed by summing the indices out one at a time,
//   f_new^{kappa'} = 1/K_v sum_{k_v} prod_{j: v in kappa_j} f_j^{kappa_j},   kappa' = U kappa_j \ {v},
// e.g. f_12^{k2 k3} = 1/K1 sum_{k1} f_1^{k1 k2} f_2^{k1 k3} (a K^3 log-domain contraction whose
// output never materialises the K^3 summand).  One elimination step is one launch:
//   elim_step_kernel      thread = one entry o of the new factor; online-max log2-sum-exp2 over k_v
//                         of s(o, k_v) = sum_j f_j (ex2.approx on MUFU), no K^3 tensor in memory;
//   elim_norm_kernel      per datapoint: subtract the max of the new table (fp32 residual) and carry
//                         it in an fp64 offset (reading A17, as the chain path does);
//   elim_grad_kernel      reverse of one step: thread = one entry e of an input factor,
//                         g_j[e] = sum over the consistent (o, k_v) of g_out[o] exp(s(o,k_v) - LSE_v s(o,.)),
//                         each thread owns its entry (deterministic, no atomics);
//   elim_final_kernel     logp[b] = sum of the remaining 0-index factors (fp64).
// Factor tables are fp32 [B][K_s0][K_s1][K_s2] row-major in scope order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "tmc_internal.h"

namespace tmc {
namespace elim {

constexpr int kMaxArity = 3;          // of any factor, input or intermediate
constexpr int kMaxTouch = 8;          // factors that contain one eliminated index
constexpr int kMaxUnion = kMaxArity + 1;

struct Step {
  int nin;                            // factors touching v
  int nu;                             // |union of their scopes| (v included), <= 4
  int Ku[kMaxUnion];                  // K of each union variable (union order = ascending variable id)
  int vpos;                           // position of v in the union
  float lnK;                          // ln K_v (natural)
  const float* tab[kMaxTouch];        // input residual tables [B][size]
  long long tsize[kMaxTouch];         // entries per datapoint of each input
  int tstride[kMaxTouch][kMaxUnion];  // stride of each union variable in input j (0 if absent)
  int tar[kMaxTouch];                 // arity of input j
  int tpos[kMaxTouch][kMaxArity];     // union position of the a-th scope variable of input j
  const double* toff[kMaxTouch];      // [B] fp64 offsets of the inputs (NULL = 0)
  float* out;                         // [B][osize] new factor (residual, normalised by elim_norm_kernel)
  long long osize;
  int ostride[kMaxUnion];             // stride of each union variable in the output (0 for v)
  double* ooff;                       // [B] offset of the new factor
  float* shift;                       // [B] max subtracted by elim_norm_kernel + ln K_v (for the reverse)
  // reverse
  const float* gout;                  // [B][osize] dJ/d(new factor)
  float* gin[kMaxTouch];              // [B][tsize] dJ/d(input j) or NULL (not wanted)
};

// log2-domain online sum: (m, s) represents 2^m * s
__device__ __forceinline__ void lse2_push(float& m, float& s, float x) {
  if (x > m) {
    s = (m == -INFINITY) ? 1.f : fmaf(s, exp2f(m - x), 1.f);
    m = x;
  } else if (x > -INFINITY) {
    s += exp2f(x - m);
  }
}

__global__ void __launch_bounds__(256) elim_step_kernel(const __grid_constant__ Step st) {
  const int b = blockIdx.y;
  const long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= st.osize) return;
  // decode the output entry into union values (output layout = union order without v, row-major)
  int val[kMaxUnion] = {0, 0, 0, 0};
  long long r = o;
  for (int u = st.nu - 1; u >= 0; --u) {
    if (u == st.vpos) continue;
    val[u] = (int)(r % st.Ku[u]);
    r /= st.Ku[u];
  }
  const float* p[kMaxTouch];
  int sv[kMaxTouch];
#pragma unroll
  for (int j = 0; j < kMaxTouch; ++j) {
    if (j >= st.nin) break;
    long long base = 0;
    for (int u = 0; u < st.nu; ++u) base += (long long)val[u] * st.tstride[j][u];
    p[j] = st.tab[j] + (size_t)b * st.tsize[j] + base;
    sv[j] = st.tstride[j][st.vpos];
  }
  float m = -INFINITY, s = 0.f;
  const int Kv = st.Ku[st.vpos];
  for (int k = 0; k < Kv; ++k) {
    float x = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxTouch; ++j) {
      if (j >= st.nin) break;
      x += __ldg(p[j] + (size_t)k * sv[j]);
    }
    lse2_push(m, s, x * kLog2E);
  }
  st.out[(size_t)b * st.osize + o] = (m == -INFINITY) ? -INFINITY : kLn2 * (m + __log2f(s)) - st.lnK;
}

// per datapoint: subtract the max entry of the new factor; offset = sum of input offsets + max
__global__ void __launch_bounds__(256) elim_norm_kernel(const __grid_constant__ Step st) {
  const int b = blockIdx.x, tid = threadIdx.x;
  float* t = st.out + (size_t)b * st.osize;
  __shared__ float red[8];
  float m = -INFINITY;
  for (long long i = tid; i < st.osize; i += 256) m = fmaxf(m, t[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((tid & 31) == 0) red[tid >> 5] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
  const bool dead = (m == -INFINITY);
  if (!dead)
    for (long long i = tid; i < st.osize; i += 256) t[i] -= m;
  if (tid == 0) {
    double off = 0.0;
    for (int j = 0; j < st.nin; ++j)
      if (st.toff[j]) off += st.toff[j][b];
    st.ooff[b] = dead ? -INFINITY : off + (double)m;
    st.shift[b] = dead ? 0.f : m + st.lnK;
  }
}

// Reverse of one step for input factor jj: thread = one entry e of that input.
__global__ void __launch_bounds__(256) elim_grad_kernel(const __grid_constant__ Step st, int jj) {
  const int b = blockIdx.y;
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= st.tsize[jj]) return;
  int val[kMaxUnion] = {0, 0, 0, 0};
  bool fixed[kMaxUnion] = {false, false, false, false};
  long long r = e;
  for (int a = st.tar[jj] - 1; a >= 0; --a) {
    const int u = st.tpos[jj][a];
    val[u] = (int)(r % st.Ku[u]);
    r /= st.Ku[u];
    fixed[u] = true;
  }
  long long nfree = 1;
  for (int u = 0; u < st.nu; ++u)
    if (!fixed[u]) nfree *= st.Ku[u];
  const float sh = st.shift[b];
  const float* gout = st.gout + (size_t)b * st.osize;
  const float* outb = st.out + (size_t)b * st.osize;
  float acc = 0.f;
  for (long long f = 0; f < nfree; ++f) {
    long long q = f;
    for (int u = st.nu - 1; u >= 0; --u) {
      if (fixed[u]) continue;
      val[u] = (int)(q % st.Ku[u]);
      q /= st.Ku[u];
    }
    long long o = 0;
    for (int u = 0; u < st.nu; ++u) o += (long long)val[u] * st.ostride[u];
    const float g = gout[o], lo = outb[o];
    if (g == 0.f || lo == -INFINITY) continue;
    float x = 0.f;
    for (int j = 0; j < st.nin; ++j) {
      long long idx = 0;
      for (int u = 0; u < st.nu; ++u) idx += (long long)val[u] * st.tstride[j][u];
      x += __ldg(st.tab[j] + (size_t)b * st.tsize[j] + idx);
    }
    acc += g * exp2f((x - lo - sh) * kLog2E);
  }
  st.gin[jj][(size_t)b * st.tsize[jj] + e] = acc;
}

constexpr int kMaxFinal = 64;
struct Final {
  int count;
  const float* res[kMaxFinal];        // [B] residual of each remaining 0-index factor
  const double* off[kMaxFinal];       // [B] its offset (NULL = 0)
  float* grad[kMaxFinal];             // [B] dJ/d(factor) (reverse), or NULL
};

__global__ void elim_final_kernel(const __grid_constant__ Final f, int B, double* logp) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double s = 0.0;
  for (int j = 0; j < f.count; ++j) s += (double)f.res[j][b] + (f.off[j] ? f.off[j][b] : 0.0);
  logp[b] = s;
}

__global__ void elim_final_bwd_kernel(const __grid_constant__ Final f, int B, const double* logp, const double* dlogp) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double w = dlogp ? dlogp[b] : 1.0;
  const float g = (logp[b] == -INFINITY) ? 0.f : (float)w;   // an impossible datapoint: zero gradients
  for (int j = 0; j < f.count; ++j)
    if (f.grad[j]) f.grad[j][b] = g;
}

}  // namespace elim
}  // namespace tmc
