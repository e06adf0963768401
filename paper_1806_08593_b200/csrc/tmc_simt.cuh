// SIMT (CUDA-core, fp32) kernels of the TMC message pass — the generic path (any K, D <= 256,
// chains and trees, Gaussian or dense factors).  The tensor-core path (tmc_tc.cuh) replaces the
// hot contraction for aligned shapes; these kernels remain the small-K / ragged-D path.
//
// One edge contraction is run as "passes" over the K_rows x K_cols pair matrix of one datapoint
// (sum/product swap, log-domain inner product):
//   MODE 0 (forward, row owner):   ell[r] = LSE_c(g[r,c] + cb[c] - cbmax);  out[r] = rb[r] + ell[r] - ln C
//   MODE 1 (reverse, row owner):   P[r,c] = w[r] exp(g[r,c] + cb[c] - cbmax - ell[r]);  row-side grads
//   MODE 2 (reverse, column owner): same P; colsum[c] = sum_r P[r,c] and column-side grads
// P is dJ/dlogf (the pair marginal scaled by the upstream weight).  A CTA owns 32 owners
// (rows or columns) of one datapoint, streams the other side through shared memory in chunks of 64,
// and each warp owns 4 owners; phase 1 (lanes over streamed entries) forms g and P, phase 2 (lanes
// over the D dimensions) accumulates the owner-side Gaussian gradients.  No atomics: every output
// element has exactly one writer, so results are deterministic.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "tmc_internal.h"

namespace tmc {
namespace simt {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kOPW = 4;                  // owners per warp
constexpr int kOPC = kOPW * kWarps;      // owners per CTA
constexpr int kTC = 64;                  // streamed chunk
constexpr int kTCSmall = 512;            // streamed chunk of the D <= 4 variant (no P buffer): the
                                         // per-chunk staging latency is amortised over 8x the pairs

__host__ __device__ inline int padded(int D) { return D | 1; }   // odd stride: conflict-free lanes

// Dynamic shared memory bytes of pass_kernel for dimension D.
__host__ inline size_t pass_smem_bytes(int D, bool dense) {
  if (dense) return sizeof(float) * (4 * kTC + 4 * kOPC + kWarps * kOPW * kTC + 32);
  int SD = padded(D);
  const bool small = D <= 4;                 // pass_kernel<..., MAXDL = 0>
  const size_t tck = small ? kTCSmall : kTC;
  size_t f = 2 * tck * SD + tck              // streamed vectors (+beta)
           + 2 * (size_t)kOPC * SD + kOPC    // owner vectors (+beta)
           + 2 * tck + 2 * kOPC              // scalars
           + (small ? 0 : (size_t)kWarps * kOPW * tck)   // P buffer
           + 32;
  return f * sizeof(float);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// merge two (max, scaled-sum) logsumexp states
__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2) {
  float M = fmaxf(m, m2);
  if (M == -INFINITY) { m = M; s = 0.f; return; }
  s = s * __expf(m - M) + s2 * __expf(m2 - M);
  m = M;
}

template <bool ZROWS, int MODE, bool DENSE, int MAXDL>
__device__ __forceinline__ void pass_body(const PassArgs& a) {
  constexpr bool OWNER_ROW = (MODE != 2);
  constexpr bool OWNER_Z = ZROWS ? (MODE != 2) : (MODE == 2);   // owner vectors are z-side
  const int b = blockIdx.y;
  const int D = a.D;
  const int SD = padded(D);
  const int NO = OWNER_ROW ? a.R : a.C;
  const int NS = OWNER_ROW ? a.C : a.R;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int obase = blockIdx.x * kOPC;
  constexpr bool SMALL = (MAXDL <= 0);       // 0: D <= 4; -1: D == 1 exactly
  constexpr int TCK = (SMALL && !DENSE) ? kTCSmall : kTC;

  extern __shared__ float sm[];
  float *sv0, *sv1, *sbeta, *ov0, *ov1, *obeta, *ss0, *ss1, *os0, *os1, *pbuf, *red;
  {
    float* p = sm;
    if (!DENSE) {
      sv0 = p; p += TCK * SD;
      sv1 = p; p += TCK * SD;
      sbeta = p; p += TCK;
      ov0 = p; p += kOPC * SD;
      ov1 = p; p += kOPC * SD;
      obeta = p; p += kOPC;
    } else {
      p += 2 * kTC;  // keep layout simple
    }
    ss0 = p; p += TCK;
    ss1 = p; p += TCK;
    os0 = p; p += kOPC;
    os1 = p; p += kOPC;
    pbuf = p; p += (SMALL && !DENSE) ? 0 : kWarps * kOPW * TCK;
    red = p;
  }

  const float* zb = DENSE ? nullptr : a.z + (int64_t)b * a.Kz * D;
  const float* mub = DENSE ? nullptr : a.mu + (int64_t)b * a.Kp * D;
  const float* lvb = DENSE ? nullptr : a.lv + (int64_t)b * a.Kp * D;
  const float* cbb = a.cb + (int64_t)b * a.C;

  // ---- column-bias maximum (offset pulled out of the LSE; exact in fp64 bookkeeping)
  float cbmax;
  if (MODE == 0) {
    float m = -INFINITY;
    for (int c = tid; c < a.C; c += kThreads) m = fmaxf(m, cbb[c]);
    m = warp_max(m);
    if (lane == 0) red[warp] = m;
    __syncthreads();
    if (tid < 32) {
      float v = tid < kWarps ? red[tid] : -INFINITY;
      v = warp_max(v);
      if (tid == 0) red[31] = (v == -INFINITY) ? 0.f : v;
    }
    __syncthreads();
    cbmax = red[31];
    if (blockIdx.x == 0 && tid == 0) {
      a.cbmax[b] = cbmax;
      double off = (double)cbmax;
      if (a.off_cb) off += a.off_cb[b];
      if (a.off_rb) off += a.off_rb[b];
      a.off_out[b] = off;
    }
  } else {
    cbmax = a.cbmax[b];
  }

  // ---- stage owner vectors and scalars
  if (!DENSE) {
    for (int idx = tid; idx < kOPC * D; idx += kThreads) {
      int ol = idx / D, d = idx - ol * D, o = obase + ol;
      float v0 = 0.f, v1 = 0.f;
      if (o < NO) {
        if (OWNER_Z) {
          v0 = zb[(int64_t)o * D + d];
        } else {
          v0 = mub[(int64_t)o * D + d];
          v1 = __expf(-lvb[(int64_t)o * D + d]);
        }
      }
      ov0[ol * SD + d] = v0;
      ov1[ol * SD + d] = v1;
    }
    if (!OWNER_Z) {
      for (int j = 0; j < kOPW; ++j) {
        int ol = warp * kOPW + j, o = obase + ol;
        float s = 0.f;
        if (o < NO)
          for (int d = lane; d < D; d += 32) s += lvb[(int64_t)o * D + d] + kLog2Pi;
        s = warp_sum(s);
        if (lane == 0) obeta[ol] = -0.5f * s;
      }
    }
  }
  for (int ol = tid; ol < kOPC; ol += kThreads) {
    int o = obase + ol;
    float s0 = 0.f, s1 = 0.f;
    if (o < NO) {
      if (MODE == 1) { s0 = a.w[(int64_t)b * a.R + o]; s1 = a.ell[(int64_t)b * a.R + o]; }
      if (MODE == 2) { s0 = cbb[o]; }
    }
    os0[ol] = s0;
    os1[ol] = s1;
  }

  // per-lane state.  SMALL (MAXDL == 0, D <= 4): each lane accumulates the owner-side Gaussian
  // gradient sums over its own streamed entries in phase 1 (warp-reduced in the epilogue) instead
  // of the lanes-over-dimensions phase 2, which would leave 31 of 32 lanes idle.
  constexpr int NDL = (MAXDL == -1) ? 1 : (SMALL ? 4 : MAXDL);
  float lm[kOPW], ls[kOPW], ptot[kOPW];
  float acc0[kOPW][NDL], acc1[kOPW][NDL];
#pragma unroll
  for (int j = 0; j < kOPW; ++j) {
    lm[j] = -INFINITY; ls[j] = 0.f; ptot[j] = 0.f;
#pragma unroll
    for (int q = 0; q < NDL; ++q) { acc0[j][q] = 0.f; acc1[j][q] = 0.f; }
  }

  for (int s0 = 0; s0 < NS; s0 += TCK) {
    const int tc = min(TCK, NS - s0);
    __syncthreads();
    // ---- stage streamed chunk
    if (!DENSE) {
      for (int idx = tid; idx < tc * D; idx += kThreads) {
        int sl = idx / D, d = idx - sl * D, s = s0 + sl;
        if (!OWNER_Z) {   // streamed entries are z-side
          sv0[sl * SD + d] = zb[(int64_t)s * D + d];
        } else {
          sv0[sl * SD + d] = mub[(int64_t)s * D + d];
          sv1[sl * SD + d] = __expf(-lvb[(int64_t)s * D + d]);
        }
      }
      if (OWNER_Z) {
        for (int sl = warp; sl < tc; sl += kWarps) {
          float s = 0.f;
          for (int d = lane; d < D; d += 32) s += lvb[(int64_t)(s0 + sl) * D + d] + kLog2Pi;
          s = warp_sum(s);
          if (lane == 0) sbeta[sl] = -0.5f * s;
        }
      }
    }
    for (int sl = tid; sl < tc; sl += kThreads) {
      int s = s0 + sl;
      if (MODE == 2) { ss0[sl] = a.w[(int64_t)b * a.R + s]; ss1[sl] = a.ell[(int64_t)b * a.R + s]; }
      else { ss0[sl] = cbb[s]; }
    }
    __syncthreads();

    // ---- phase 1: lanes over streamed entries
#pragma unroll
    for (int j = 0; j < kOPW; ++j) {
      const int ol = warp * kOPW + j, o = obase + ol;
      if (o >= NO) continue;
      for (int sl = lane; sl < tc; sl += 32) {
        const int s = s0 + sl;
        const int row = OWNER_ROW ? o : s, col = OWNER_ROW ? s : o;
        const int ai = ZROWS ? row : col, pi = ZROWS ? col : row;
        float g;
        if (DENSE) {
          g = a.logf[((int64_t)b * a.Kz + ai) * a.Kp + pi];
        } else {
          const float* zv = OWNER_Z ? ov0 + ol * SD : sv0 + sl * SD;
          const float* mv = OWNER_Z ? sv0 + sl * SD : ov0 + ol * SD;
          const float* lam = OWNER_Z ? sv1 + sl * SD : ov1 + ol * SD;
          float q = 0.f;
          for (int d = 0; d < D; ++d) {
            float df = zv[d] - mv[d];
            q = fmaf(lam[d] * df, df, q);
          }
          g = (OWNER_Z ? sbeta[sl] : obeta[ol]) - 0.5f * q;
        }
        g *= a.alpha;
        if (MODE == 0) {
          float x = g + ss0[sl] - cbmax;
          if (x > lm[j]) { ls[j] = ls[j] * __expf(lm[j] - x) + 1.f; lm[j] = x; }
          else if (x > -INFINITY) { ls[j] += __expf(x - lm[j]); }
        } else {
          float wr = MODE == 1 ? os0[ol] : ss0[sl];
          float el = MODE == 1 ? os1[ol] : ss1[sl];
          float cbv = MODE == 1 ? ss0[sl] : os0[ol];
          float P = 0.f;
          if (wr != 0.f && el > -INFINITY) P = wr * __expf(g + cbv - cbmax - el);
          if constexpr (SMALL && !DENSE) {
            const float* zv = OWNER_Z ? ov0 + ol * SD : sv0 + sl * SD;
            const float* mv = OWNER_Z ? sv0 + sl * SD : ov0 + ol * SD;
#pragma unroll
            for (int q = 0; q < NDL; ++q) {
              if (q >= D) break;
              if (OWNER_Z) {     // dz_o,q += P (mu_s,q - z_o,q) lam_s,q
                acc0[j][q] = fmaf(P * (mv[q] - zv[q]), sv1[sl * SD + q], acc0[j][q]);
              } else {           // sum_s P (z_s,q - mu_o,q) and sum_s P (z_s,q - mu_o,q)^2
                const float df = zv[q] - mv[q], pd = P * df;
                acc0[j][q] += pd;
                acc1[j][q] = fmaf(pd, df, acc1[j][q]);
              }
            }
          } else {
            pbuf[(warp * kOPW + j) * TCK + sl] = P;
          }
          ptot[j] += P;
          if (MODE == 1 && a.pair) a.pair[((int64_t)b * a.Kz + ai) * a.Kp + pi] = a.alpha * P;
        }
      }
    }
    // ---- phase 2: lanes over dimensions (owner-side Gaussian gradients)
    if (MODE != 0 && !DENSE && !SMALL) {
      __syncwarp();
#pragma unroll
      for (int j = 0; j < kOPW; ++j) {
        const int ol = warp * kOPW + j, o = obase + ol;
        if (o >= NO) continue;
        const float* pw = pbuf + (warp * kOPW + j) * TCK;
#pragma unroll
        for (int q = 0; q < MAXDL; ++q) {
          const int d = lane + 32 * q;
          if (d >= D) continue;
          if (OWNER_Z) {     // dz_o,d = sum_s P (mu_s,d - z_o,d) lam_s,d
            const float zo = ov0[ol * SD + d];
            float acc = acc0[j][q];
            for (int sl = 0; sl < tc; ++sl) {
              float p = pw[sl];
              acc = fmaf(p * (sv0[sl * SD + d] - zo), sv1[sl * SD + d], acc);
            }
            acc0[j][q] = acc;
          } else {           // sum_s P (z_s,d - mu_o,d) and sum_s P (z_s,d - mu_o,d)^2
            const float mo = ov0[ol * SD + d];
            float x0 = acc0[j][q], x1 = acc1[j][q];
            for (int sl = 0; sl < tc; ++sl) {
              float p = pw[sl];
              float df = sv0[sl * SD + d] - mo;
              float pd = p * df;
              x0 += pd;
              x1 = fmaf(pd, df, x1);
            }
            acc0[j][q] = x0; acc1[j][q] = x1;
          }
        }
      }
      __syncwarp();
    }
  }

  // ---- epilogue
#pragma unroll
  for (int j = 0; j < kOPW; ++j) {
    const int ol = warp * kOPW + j, o = obase + ol;
    if (o >= NO) continue;   // warp-uniform
    if (MODE == 0) {
      float m = lm[j], s = ls[j];
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        float m2 = __shfl_xor_sync(0xffffffffu, m, off);
        float s2 = __shfl_xor_sync(0xffffffffu, s, off);
        lse_merge(m, s, m2, s2);
      }
      if (lane == 0) {
        float e = (m == -INFINITY) ? -INFINITY : m + logf(s);
        a.ell[(int64_t)b * a.R + o] = e;
        float rbv = a.rb ? a.rb[(int64_t)b * a.R + o] : 0.f;
        a.out[(int64_t)b * a.R + o] = rbv + e - a.lnC;
      }
    } else {
      float tot = warp_sum(ptot[j]);
      if (MODE == 2 && lane == 0 && a.colsum) a.colsum[(int64_t)b * a.C + o] = tot;
      if (DENSE) continue;
      if constexpr (SMALL) {
#pragma unroll
        for (int q = 0; q < NDL; ++q) {
          if (q >= D) break;
          const float s0 = warp_sum(acc0[j][q]), s1 = warp_sum(acc1[j][q]);
          if (lane) continue;
          if (OWNER_Z) {
            if (a.gz) a.gz[((int64_t)b * a.Kz + o) * D + q] = a.alpha * s0;
          } else {
            const float lam = ov1[ol * SD + q];
            if (a.gmu) a.gmu[((int64_t)b * a.Kp + o) * D + q] = a.alpha * lam * s0;
            if (a.glv) a.glv[((int64_t)b * a.Kp + o) * D + q] = a.alpha * 0.5f * (lam * s1 - tot);
          }
        }
        continue;
      }
#pragma unroll
      for (int q = 0; q < MAXDL; ++q) {
        const int d = lane + 32 * q;
        if (d >= D) continue;
        if (OWNER_Z) {
          if (a.gz) a.gz[((int64_t)b * a.Kz + o) * D + d] = a.alpha * acc0[j][q];
        } else {
          const float lam = ov1[ol * SD + d];
          if (a.gmu) a.gmu[((int64_t)b * a.Kp + o) * D + d] = a.alpha * lam * acc0[j][q];
          if (a.glv) a.glv[((int64_t)b * a.Kp + o) * D + d] = a.alpha * 0.5f * (lam * acc1[j][q] - tot);
        }
      }
    }
  }
}

template <bool ZROWS, int MODE, bool DENSE, int MAXDL>
__global__ void __launch_bounds__(kThreads) pass_kernel(const PassArgs a) {
  pass_body<ZROWS, MODE, DENSE, MAXDL>(a);
}

// The same pass over up to kMaxPassBatch independent edges of one tree level (blockIdx.z = edge):
// many small edges (e.g. the N data points of a shared-root star) fill the GPU in one
// launch instead of one under-filled launch each.
constexpr int kMaxPassBatch = 16;
struct PassBatch { PassArgs e[kMaxPassBatch]; };
template <bool ZROWS, int MODE, bool DENSE, int MAXDL>
__global__ void __launch_bounds__(kThreads) pass_batch_kernel(const __grid_constant__ PassBatch pb) {
  const PassArgs& a = pb.e[blockIdx.z];
  if ((int)blockIdx.x * kOPC >= ((MODE != 2) ? a.R : a.C)) return;
  pass_body<ZROWS, MODE, DENSE, MAXDL>(a);
}

// ------------------------------------------------------------------------------ small kernels
// Unary prep: u = (logobs - max logobs) - logq, uoff = max logobs (fp64 offset).
__global__ void __launch_bounds__(256) unary_prep_kernel(const UnaryBatch ub) {
  const UnaryDesc& d = ub.d[blockIdx.y];
  const int b = blockIdx.x;
  __shared__ float red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float m = 0.f;
  if (d.logobs) {
    m = -INFINITY;
    for (int k = tid; k < d.K; k += 256) m = fmaxf(m, d.logobs[(int64_t)b * d.K + k]);
    m = warp_max(m);
    if (lane == 0) red[warp] = m;
    __syncthreads();
    if (tid < 32) {
      float v = tid < 8 ? red[tid] : -INFINITY;
      v = warp_max(v);
      if (tid == 0) red[31] = v;
    }
    __syncthreads();
    m = red[31];
  }
  const float shift = (m == -INFINITY) ? 0.f : m;
  const float al = ub.alpha;
  for (int k = tid; k < d.K; k += 256) {
    float v = d.logobs ? d.logobs[(int64_t)b * d.K + k] - shift : 0.f;
    if (d.logq) v -= d.logq[(int64_t)b * d.K + k];
    d.u[(int64_t)b * d.K + k] = al * v;
  }
  if (tid == 0) d.uoff[b] = (double)al * (double)shift;
}

// h_i = u_i + sum_j msg_{j->i}  (UP direction), offsets added in fp64.
__global__ void __launch_bounds__(256) hbuild_kernel(const HBuild h) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * 256 + threadIdx.x;
  if (k < h.K) {
    float v = h.u[(int64_t)b * h.K + k];
    for (int j = 0; j < h.nchild; ++j) v += h.msg[j][(int64_t)b * h.K + k];
    h.h[(int64_t)b * h.K + k] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double o = h.uoff[b];
    for (int j = 0; j < h.nchild; ++j) o += h.moff[j][b];
    h.hoff[b] = o;
  }
}

// Shared-root exchange.  x[b][r] (r < K) accumulates the fp32 residuals of the root's
// child messages in fp64, x[b][K] their fp64 offsets; `first` overwrites instead of accumulating.
__global__ void __launch_bounds__(256) xmsg_kernel(const HBuild h, double* x, bool first) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * 256 + threadIdx.x;
  if (k > h.K) return;
  double v = first ? 0.0 : x[(int64_t)b * (h.K + 1) + k];
  for (int j = 0; j < h.nchild; ++j) v += k < h.K ? (double)h.msg[j][(int64_t)b * h.K + k] : h.moff[j][b];
  x[(int64_t)b * (h.K + 1) + k] = v;
}

// h_root = u_root + x (x = shard sums of xmsg_kernel, summed over shards by the caller).
__global__ void __launch_bounds__(256) hroot_kernel(const float* u, const double* uoff, const double* x, int K,
                                                    float* h, double* hoff) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * 256 + threadIdx.x;
  if (k < K) h[(int64_t)b * K + k] = u[(int64_t)b * K + k] + (float)x[(int64_t)b * (K + 1) + k];
  if (blockIdx.x == 0 && threadIdx.x == 0) hoff[b] = uoff[b] + x[(int64_t)b * (K + 1) + K];
}

// Tensor-core padding (tmc_api.cu): rows of Di floats -> rows of Dt floats (tail = fill), and back;
// one launch per batch of up to kMaxPad arrays (blockIdx.y = array).
constexpr int kMaxPad = 48;
struct PadDesc { const float* src; float* dst; int64_t rows; int Di, Dt; float fill; };
struct PadBatch { PadDesc d[kMaxPad]; int count; };
__global__ void __launch_bounds__(256) pad_batch_kernel(const __grid_constant__ PadBatch pb, int unpad) {
  const PadDesc& q = pb.d[blockIdx.y];
  if (unpad) {
    const int64_t n = q.rows * q.Di;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = t / q.Di;
      q.dst[t] = q.src[r * q.Dt + (t - r * q.Di)];
    }
    return;
  }
  // padded rows of Dt = 32 / 64 floats written as float4 (Dt / 4 = 8 or 16 per row: shift, no divide)
  const int sh = q.Dt == 64 ? 4 : 3;
  const int64_t n4 = q.rows << sh;
  float4* dst4 = reinterpret_cast<float4*>(q.dst);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n4; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t >> sh;
    const int d0 = (int)(t - (r << sh)) * 4;
    const float* sr = q.src + r * q.Di;
    float4 v;
    v.x = d0 < q.Di ? sr[d0] : q.fill;
    v.y = d0 + 1 < q.Di ? sr[d0 + 1] : q.fill;
    v.z = d0 + 2 < q.Di ? sr[d0 + 2] : q.fill;
    v.w = d0 + 3 < q.Di ? sr[d0 + 3] : q.fill;
    dst4[t] = v;
  }
}
__global__ void __launch_bounds__(256) pad_rows_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                       int64_t rows, int Di, int Dt, float fill) {
  const int64_t n = rows * Dt;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / Dt;
    const int d = (int)(t - r * Dt);
    dst[t] = d < Di ? src[r * Di + d] : fill;
  }
}
__global__ void __launch_bounds__(256) unpad_rows_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                         int64_t rows, int Di, int Dt) {
  const int64_t n = rows * Di;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / Di;
    dst[t] = src[r * Dt + (t - r * Di)];
  }
}

// DOWN final: logp = off + LSE_a m[a] - ln K; save lse for the reverse pass.
__global__ void __launch_bounds__(256) final_down_fwd_kernel(const float* m, const double* off, int K,
                                                             float lnK, float* lse, double* logp) {
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float red[64];
  float mx = -INFINITY;
  for (int k = tid; k < K; k += 256) mx = fmaxf(mx, m[(int64_t)b * K + k]);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (tid < 32) {
    float v = tid < 8 ? red[tid] : -INFINITY;
    v = warp_max(v);
    if (tid == 0) red[40] = v;
  }
  __syncthreads();
  mx = red[40];
  float s = 0.f;
  if (mx > -INFINITY)
    for (int k = tid; k < K; k += 256) s += __expf(m[(int64_t)b * K + k] - mx);
  s = warp_sum(s);
  __syncthreads();
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (tid == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    float l = (mx == -INFINITY) ? -INFINITY : mx + logf(t);
    lse[b] = l;
    logp[b] = (l == -INFINITY) ? -INFINITY : off[b] + (double)l - (double)lnK;
  }
}

// DOWN final reverse: w[a] = dlogp * softmax(m)[a].
__global__ void __launch_bounds__(256) final_down_bwd_kernel(const float* m, const float* lse, int K,
                                                             const double* dlogp, float* w) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * 256 + threadIdx.x;
  if (k >= K) return;
  float l = lse[b];
  float g = dlogp ? (float)dlogp[b] : 1.f;
  w[(int64_t)b * K + k] = (l == -INFINITY || g == 0.f) ? 0.f : g * __expf(m[(int64_t)b * K + k] - l);
}

// UP final: logp = sum over roots of (off_root + out_root[0]).
__global__ void final_up_fwd_kernel(const RootList r, double* logp) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= r.B) return;
  double s = 0.0;
  for (int j = 0; j < r.count; ++j) {
    float o = r.out[j][b];
    s += (o == -INFINITY) ? -INFINITY : r.off[j][b] + (double)o;
  }
  logp[b] = s;
}

// UP reverse seed: w_root[b] = dlogp[b]; zero if the datapoint is impossible.
__global__ void final_up_bwd_kernel(const RootList r, const double* dlogp) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= r.B) return;
  for (int j = 0; j < r.count; ++j) r.w[j][b] = dlogp ? (float)dlogp[b] : 1.f;
}

// dlogobs = pi, dlogq = -pi.
__global__ void unary_grad_kernel(const UnaryGradBatch g) {
  const UnaryGradDesc& d = g.d[blockIdx.y];
  const int64_t n = (int64_t)g.B * d.K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float p = g.alpha * d.pi[i];
    if (d.dlogobs) d.dlogobs[i] = p;
    if (d.dlogq) d.dlogq[i] = -p;
  }
}

// tmc_factors: logf[b][a][c] = sum_d log N(z_a; mu_c, exp v_c) - logq[a] (direct form, fp32).
__global__ void __launch_bounds__(256) factors_kernel(const float* z, const float* mu, const float* lv,
                                                      const float* logq, float* logf, int Ki, int Kp, int D) {
  const int b = blockIdx.z;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int a = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (a >= Ki || c >= Kp) return;
  const float* zv = z + ((int64_t)b * Ki + a) * D;
  const float* mv = mu + ((int64_t)b * Kp + c) * D;
  const float* vv = lv + ((int64_t)b * Kp + c) * D;
  float q = 0.f, sv = 0.f;
  for (int d = 0; d < D; ++d) {
    float df = zv[d] - mv[d];
    q = fmaf(__expf(-vv[d]) * df, df, q);
    sv += vv[d] + kLog2Pi;
  }
  logf[((int64_t)b * Ki + a) * Kp + c] = -0.5f * (q + sv) - logq[(int64_t)b * Ki + a];
}

// TMC_FLAG_VALIDATE: flag NaN / +inf (and -inf where not allowed) in a buffer.
__global__ void validate_kernel(const float* x, int64_t n, int allow_neginf, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float v = x[i];
    bool bad = isnan(v) || v == INFINITY || (!allow_neginf && v == -INFINITY);
    if (bad) *flag = 1;
  }
}

// ---------------------------------------------------------------------------------------------
// Root edge of a DOWN chain (K_p = 1: the prior P(z_0)).  The pair matrix is K x 1, so
// the "contraction" is elementwise in a: one warp per sample row, lanes over the D dimensions.
//   fwd:  ell[a] = g[a] + cb[0] - cbmax,  out[a] = rb[a] + ell[a] - lnC      (g = log N(z_a; mu_0, e^{v_0}))
//   row owner (MODE 1): P[a] = w[a] (softmax over one column), dz = P (mu - z) lam, pair = P
//   column owner (MODE 2): colsum = sum_a P[a], dmu = sum_a P (z - mu) lam, dv = 1/2 sum_a P ((z-mu)^2 lam - 1)
// Same arithmetic as pass_kernel<true, MODE, false, *> with C = 1.
__global__ void __launch_bounds__(256) root_down_fwd_kernel(const PassArgs a) {
  // one thread per (datapoint, sample row): the row's D values are contiguous (float4 when D % 4 == 0)
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)a.B * a.R) return;
  const int b = (int)(idx / a.R), r = (int)(idx % a.R);
  const int D = a.D;
  const float cb0 = a.cb[b];
  const float cbmax = (cb0 == -INFINITY) ? 0.f : cb0;
  if (r == 0) {
    a.cbmax[b] = cbmax;
    double off = (double)cbmax;
    if (a.off_cb) off += a.off_cb[b];
    if (a.off_rb) off += a.off_rb[b];
    a.off_out[b] = off;
  }
  const float* mu = a.mu + (int64_t)b * D;
  const float* lv = a.lv + (int64_t)b * D;
  const float* z = a.z + ((int64_t)b * a.Kz + r) * D;
  float s = 0.f;
  if ((D & 3) == 0) {
    for (int d = 0; d < D; d += 4) {
      const float4 z4 = *reinterpret_cast<const float4*>(z + d);
      const float4 m4 = *reinterpret_cast<const float4*>(mu + d);
      const float4 v4 = *reinterpret_cast<const float4*>(lv + d);
      const float zz[4] = {z4.x, z4.y, z4.z, z4.w}, mm[4] = {m4.x, m4.y, m4.z, m4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float df = zz[e] - mm[e];
        s += df * df * __expf(-vv[e]) + vv[e] + kLog2Pi;
      }
    }
  } else {
    for (int d = 0; d < D; ++d) {
      const float df = z[d] - mu[d], v = lv[d];
      s += df * df * __expf(-v) + v + kLog2Pi;
    }
  }
  const float e = (cb0 == -INFINITY) ? -INFINITY : -0.5f * a.alpha * s + (cb0 - cbmax);
  a.ell[(int64_t)b * a.R + r] = e;
  const float rb = a.rb ? a.rb[(int64_t)b * a.R + r] : 0.f;
  a.out[(int64_t)b * a.R + r] = rb + e - a.lnC;
}

__global__ void __launch_bounds__(256) root_down_row_kernel(const PassArgs a) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)a.B * a.R) return;
  const int b = (int)(idx / a.R), r = (int)(idx % a.R);
  const int D = a.D;
  const float e = a.ell[(int64_t)b * a.R + r];
  const float P = (e == -INFINITY) ? 0.f : a.alpha * a.w[(int64_t)b * a.R + r];   // alpha * dJ/d(alpha logf)
  if (a.pair) a.pair[(int64_t)b * a.R + r] = P;
  if (!a.gz) return;
  const float* mu = a.mu + (int64_t)b * D;
  const float* lv = a.lv + (int64_t)b * D;
  const float* z = a.z + ((int64_t)b * a.Kz + r) * D;
  float* gz = a.gz + ((int64_t)b * a.Kz + r) * D;
  if ((D & 3) == 0) {
    for (int d = 0; d < D; d += 4) {
      const float4 z4 = *reinterpret_cast<const float4*>(z + d);
      const float4 m4 = *reinterpret_cast<const float4*>(mu + d);
      const float4 v4 = *reinterpret_cast<const float4*>(lv + d);
      *reinterpret_cast<float4*>(gz + d) =
          make_float4(P * (m4.x - z4.x) * __expf(-v4.x), P * (m4.y - z4.y) * __expf(-v4.y),
                      P * (m4.z - z4.z) * __expf(-v4.z), P * (m4.w - z4.w) * __expf(-v4.w));
    }
  } else {
    for (int d = 0; d < D; ++d) gz[d] = P * (mu[d] - z[d]) * __expf(-lv[d]);
  }
}

// one CTA per datapoint: reduce over the K rows
__global__ void __launch_bounds__(256) root_down_col_kernel(const PassArgs a) {
  const int b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int D = a.D;
  __shared__ float red[3][8][33];
  const float* mu = a.mu + (int64_t)b * D;
  const float* lv = a.lv + (int64_t)b * D;
  const float* w = a.w + (int64_t)b * a.R;
  const float* ell = a.ell + (int64_t)b * a.R;
  float psum = 0.f;
  for (int d0 = 0; d0 < D; d0 += 32) {
    const int d = d0 + lane;
    float am = 0.f, av = 0.f;
    const float m = d < D ? mu[d] : 0.f, lam = d < D ? __expf(-lv[d]) : 0.f;
    // 4 rows in flight per warp (independent loads), fixed summation order
    for (int r0 = warp * 4; r0 < a.R; r0 += 32) {
      float P[4], zv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = r0 + q;
        P[q] = (r < a.R && ell[r] != -INFINITY) ? w[r] : 0.f;
        zv[q] = (r < a.R && d < D) ? a.z[((int64_t)b * a.Kz + r) * D + d] : 0.f;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (d0 == 0) psum += P[q];
        if (d < D) {
          const float df = zv[q] - m;
          am += P[q] * df * lam;
          av += P[q] * (df * df * lam - 1.f);
        }
      }
    }
    red[0][warp][lane] = am;
    red[1][warp][lane] = av;
    if (d0 == 0) red[2][warp][lane] = psum;
    __syncthreads();
    if (warp == 0) {
      float sm = 0.f, sv = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) { sm += red[0][k][lane]; sv += red[1][k][lane]; }
      if (d < D) {
        if (a.gmu) a.gmu[(int64_t)b * D + d] = a.alpha * sm;
        if (a.glv) a.glv[(int64_t)b * D + d] = a.alpha * 0.5f * sv;
      }
      if (d0 == 0) {
        float sp = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) sp += red[2][k][lane];   // lanes hold per-warp partials
        if (lane == 0 && a.colsum) a.colsum[b] = sp;           // every lane of a warp added the same P
      }
    }
    __syncthreads();
  }
}

}  // namespace simt
}  // namespace tmc
