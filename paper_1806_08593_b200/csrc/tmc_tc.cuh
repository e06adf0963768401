// Tensor-core (tcgen05) path of the TMC message pass, sm_100a.
//
// The pairwise log-factor of a diagonal-Gaussian conditional ("nominally quadratic
// cost ... dominated by the linear cost") is a dense contraction once the square is expanded:
//   log N(z_a; mu_c, diag e^{v_c}) = S[a,c] + beta[c],   S = X . Y^T,
//   X[a] = [z'^2, z'],  Y[c] = [-lam/2, lam mu'] * log2(e),  lam = e^{-v},
//   beta[c] = -1/2 sum_d (lam mu'^2 + v + ln 2 pi),  z' = z - s,  mu' = mu - s
// with a per-(datapoint, latent) centering shift s (the posterior-weighted mean of the samples the
// message pass already weighted; an exact identity that keeps the expanded terms small).  Every operand is split into an fp16 pair (hi, lo = fp16(x - hi)) and
// S = X_hi Y_hi + X_hi Y_lo + X_lo Y_hi is accumulated in fp32 in TMEM by tcgen05.mma kind::f16
// (relative error ~2^-21 per product).
//
//   tc_prep_kernel   (K1): per (datapoint, latent): s, X/Y hi/lo tile images (pre-swizzled 128B,
//                          the exact shared-memory image a bulk copy lands), beta.
//   tc_colbias_kernel:     per (datapoint, edge): cbmax, fp64 offset, column bias in log2 units.
//   tc_fwd_kernel    (K3): persistent, warp-specialised: a producer warp streams tiles with
//                          cp.async.bulk (TMA engine) into a 3-stage mbarrier ring, an MMA warp
//                          issues tcgen05.mma (+ one K=16 bias MMA) into double-buffered TMEM
//                          accumulators, 8*RB softmax warps drain TMEM with tcgen05.ld and run the
//                          online-max log2-sum-exp2 (ex2.approx on MUFU, 4/16 on a packed FMA polynomial).
//   tc_rowterm_kernel:     per (datapoint, edge): reverse-pass row terms, their bias tiles, live flags.
//   tc_bwd_kernel    (K4): one owner pass of the reverse contraction (below).
//   tc_factors_kernel(K2): materialised logf (tmc_factors).
#pragma once
#include <cstdio>
#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../../include/tmc.h"
#include "tmc_internal.h"

namespace tmc {
namespace tc {

constexpr int kTileRows = 128;
constexpr int kAtomBytes = 128 * 128;        // 128 rows x 128 B (one SWIZZLE_128B K-atom)

// tcgen05 flops issued per kernel family while the launch profiler is on (tmc_profile_begin/end)
__device__ unsigned long long g_tmc_mma_flops[PF_COUNT];

template <int D>
struct Geo {
  static constexpr int W = 2 * D;                    // fp16 elements per part
  static constexpr int ATOMS = W / 64;               // 128-byte K atoms per part
  static constexpr int PART = ATOMS * kAtomBytes;    // bytes of one part (hi or lo) of a 128-row tile
  static constexpr int TILE = 2 * PART;              // hi + lo
  static constexpr int RB = (D <= 32) ? 2 : 1;       // 128-row blocks per CTA work unit
  static constexpr int STAGES = (D <= 32) ? 3 : 2;   // B-tile ring depth
  static constexpr int SOFTMAX_WARPS = 8 * RB;        // 2 per (TMEM lane quarter, row block): column halves
  static constexpr int THREADS = 64 + 32 * SOFTMAX_WARPS;
  static constexpr int TMEM_COLS = RB * 2 * 128;
  static constexpr size_t SMEM = 1024 /*align*/ + (size_t)RB * TILE + (size_t)STAGES * TILE +
                                 (size_t)(STAGES + 1) * 4096 /*bias operand ring + constant ones*/ +
                                 2 * (size_t)RB * 128 * 8 /*half merge, unit parity*/ + 512 /*barriers*/;
};

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#if defined(TMC_DEBUG_SYNC)
// Debug build (libtmc_debug.so): every mbarrier wait has a deadline of 2^34 SM clocks
// (~9 s); a pipeline that loses a phase (wrong parity, a missing arrive / commit / expect_tx)
// reports the barrier and traps, so the launch fails with an error instead of hanging the GPU.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.b32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __noinline__ void mbar_timeout(uint64_t* bar, uint32_t parity) {
  printf("libtmc (debug): mbarrier wait timed out: block %d thread %d barrier smem 0x%x parity %u\n", blockIdx.x,
         threadIdx.x, smem_u32(bar), parity);
  __trap();
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const long long t0 = clock64();
  while (!mbar_try(bar, parity))
    if (clock64() - t0 > (1ll << 34)) mbar_timeout(bar, parity);
}
#elif !defined(TMC_SPIN_WAIT)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#endif
// Optional instrumentation (-DTMC_INSTRUMENT builds libtmc_instr.so only): cycles each role spends
// waiting on each barrier, per CTA, read back with tmc_debug_counters().
#ifdef TMC_INSTRUMENT
__device__ unsigned long long g_tmc_prof[1024][64];
#define TMC_PROF_WAIT(cond, slot, call)                                                   \
  do {                                                                                    \
    const long long _t0 = clock64();                                                      \
    call;                                                                                 \
    if (cond) atomicAdd(&g_tmc_prof[blockIdx.x & 1023][slot], (unsigned long long)(clock64() - _t0)); \
  } while (0)
#define TMC_PROF_T0(var) const long long var = clock64()
#define TMC_PROF_END(cond, slot, var) \
  if (cond) atomicAdd(&g_tmc_prof[blockIdx.x & 1023][slot], (unsigned long long)(clock64() - var))
#else
#define TMC_PROF_WAIT(cond, slot, call) call
#define TMC_PROF_T0(var)
#define TMC_PROF_END(cond, slot, var)
#endif
// reverse-pass MMA-warp probes (off with -DTMC_MMA_PROF=0 to measure the others without them)
#ifndef TMC_MMA_PROF
#define TMC_MMA_PROF 1
#endif
#if TMC_MMA_PROF == 2
// register-accumulated MMA-warp probes (no atomics in the loop; flushed once at the end)
#define TMC_PROF_WAIT_M(slot, call) do { const long long _t0 = clock64(); call; mprof[slot - 3] += clock64() - _t0; } while (0)
#define TMC_PROF_T0_M(var) const long long var = clock64()
#define TMC_PROF_END_M(slot, var) mprof[slot - 3] += clock64() - var
#elif TMC_MMA_PROF
#define TMC_PROF_WAIT_M(slot, call) TMC_PROF_WAIT(lane == 0, slot, call)
#define TMC_PROF_T0_M(var) TMC_PROF_T0(var)
#define TMC_PROF_END_M(slot, var) TMC_PROF_END(lane == 0, slot, var)
#else
#define TMC_PROF_WAIT_M(slot, call) call
#define TMC_PROF_T0_M(var)
#define TMC_PROF_END_M(slot, var)
#endif
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, SWIZZLE_128B shared-memory matrix descriptor (start, LBO=16B, SBO=1024B, version 1).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// descriptor of (base + off) from the descriptor of base: the address field is (addr & 0x3FFFF) >> 4
// and every shared-memory address here is < 2^18, so the offset adds without carry.
__device__ __forceinline__ uint64_t dadd(uint64_t desc, uint32_t off_bytes) { return desc + (off_bytes >> 4); }
// Instruction descriptor: kind::f16, A/B fp16 K-major, D fp32, M=128, N=128.
constexpr uint32_t kIdescF16M128N128 = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

// The MMA warp runs converged (descriptors stay in uniform registers); one elected lane issues.
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

#define TMC_LD32(taddr, v)                                                                                          \
  asm volatile(                                                                                                     \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                               \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),            \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),      \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),    \
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])     \
      : "r"(taddr))

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (Cody-Waite range reduction + degree-5 minimax polynomial on [-1/2, 1/2],
// max relative error 8e-8, below ex2.approx's 2^-22): used to move a fixed share of the forward's
// exponentials off the MUFU pipe.  Valid for x <= 127 (callers guarantee x <= 8); x < -125 -> ~0.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;            // 1.5 * 2^23: round(x) lands in the low mantissa bits
  const float f = x - (t - 12582912.f);       // f in [-1/2, 1/2]
  float p = fmaf(1.3277400e-3f, f, 9.6758800e-3f);
  p = fmaf(p, f, 5.5507130e-2f);
  p = fmaf(p, f, 2.4022112e-1f);
  p = fmaf(p, f, 6.9314696e-1f);
  p = fmaf(p, f, 1.0000001f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// The same polynomial on a pair (FADD2 / FFMA2 on packed fp32 pairs, LEA for the exponent add):
// 12 issue slots per two exponentials instead of ~20.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x = make_float2(fmaxf(x.x, -125.f), fmaxf(x.y, -125.f));
  const float2 M = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, M);
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 p = __ffma2_rn(make_float2(1.3277400e-3f, 1.3277400e-3f), f, make_float2(9.6758800e-3f, 9.6758800e-3f));
  p = __ffma2_rn(p, f, make_float2(5.5507130e-2f, 5.5507130e-2f));
  p = __ffma2_rn(p, f, make_float2(2.4022112e-1f, 2.4022112e-1f));
  p = __ffma2_rn(p, f, make_float2(6.9314696e-1f, 6.9314696e-1f));
  p = __ffma2_rn(p, f, make_float2(1.0000001f, 1.0000001f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Byte offset of element k (fp16 index within the part's row vector) of row r in a tile part
// laid out as ATOMS x [128 rows][128 B] with the 128-byte XOR swizzle (16B chunk ^= row % 8).
__host__ __device__ __forceinline__ uint32_t swz_off(int r, int k) {
  const int atom = k >> 6, kk = k & 63;
  const int chunk = (kk >> 3) ^ (r & 7);
  return (uint32_t)(atom * kAtomBytes + r * 128 + chunk * 16 + (kk & 7) * 2);
}

// Extra K=16 operand of the forward (column bias on the tensor core): 128 rows x 16 fp16, K-major,
// no swizzle, 8-row x 16-byte core matrices: (row r, k) at (r/8)*256 + (k/8)*128 + (r%8)*16 + (k%8)*2.
constexpr int kBxBytes = 128 * 16 * 2;
__host__ __device__ __forceinline__ uint32_t bx_off(int r, int k) {
  return (uint32_t)((r >> 3) * 256 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
// K-major SWIZZLE_NONE descriptor for that layout: LBO = 128 B (next core matrix along K),
// SBO = 256 B (next 8-row group), version 1.
__device__ __forceinline__ uint64_t sdesc_bx(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}

// ------------------------------------------------------------------------------ K1: operand prep
struct PrepArgs {
  const float *z, *mu, *lv;   // [B][Kz][D], [B][Kp][D]
  int Kz, Kp, KzPad, KpPad;   // padded row counts (multiple of 256)
  uint8_t *Xt, *Yt;           // tile images [B][KzPad/128][TILE], [B][KpPad/128][TILE]
  float* beta;                // [B][KpPad]
  float* shift;               // [B][D] centering shift s (the reverse pass needs z', mu')
  const float* wsrc;          // [B][wlen] log-weights of the centering mean (messages), or NULL
  int wlen;
  int wz;                     // 1: s = sum_a softmax(wsrc)[a] z[a] ; 0: s = sum_c softmax(wsrc)[c] mu[c]
  float alpha;                // factor power: Y and beta scaled by alpha (S becomes alpha * S)
};

// hi/lo fp16 split of x (exact sum to ~2^-22 relative); lo may be subnormal.
__device__ __forceinline__ void split16(float x, __half& hi, __half& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));
}

// K1a: per-datapoint centering shift s[d]: the posterior-weighted mean of the samples the message
// pass has already weighted (UP: softmax(h_i) over z_i; DOWN: softmax(m_pa) over mu_i), else mean_c mu.
// Any s is exact algebra; a posterior-centred s keeps the expanded terms of the pairs that carry
// weight small, so the fp32 tensor-core accumulator never holds large cancelling partial sums.
constexpr int kMaxPrepBatch = 16;
struct PrepBatch { PrepArgs e[kMaxPrepBatch]; int ne; };

template <int D>
__global__ void __launch_bounds__(256) tc_shift_kernel(const __grid_constant__ PrepBatch pb) {
  const PrepArgs& p = pb.e[blockIdx.z];
  const int b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ float s_part[256];
  __shared__ float s_ws[256];
  __shared__ float s_w[2048 + 32];
  const float* mub = p.mu + (size_t)b * p.Kp * D;
  const float* zb = p.z + (size_t)b * p.Kz * D;
  const float* vec = mub;
  int nrow = p.Kp;
  bool weighted = false;
  if (p.wsrc && p.wlen <= 2048) {
    vec = p.wz ? zb : mub;
    nrow = p.wz ? p.Kz : p.Kp;
    const float* wb = p.wsrc + (size_t)b * p.wlen;
    float m = -INFINITY;
    for (int k = tid; k < nrow; k += 256) m = fmaxf(m, wb[k]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_part[warp] = m;
    __syncthreads();
    if (tid == 0) {
      float v = s_part[0];
      for (int w = 1; w < 8; ++w) v = fmaxf(v, s_part[w]);
      s_w[2048] = v;
    }
    __syncthreads();
    const float mx = s_w[2048];
    weighted = mx > -INFINITY;
    if (weighted)
      for (int k = tid; k < nrow; k += 256) s_w[k] = __expf(wb[k] - mx);
    __syncthreads();
  }
  constexpr int G_ = 256 / D;
  const int d = tid % D, g = tid / D;
  float acc0 = 0.f, acc1 = 0.f, ws0 = 0.f, ws1 = 0.f;     // two independent chains (loads in flight)
  if (weighted) {
    int k = g;
    for (; k + G_ < nrow; k += 2 * G_) {
      const float w0 = s_w[k], w1 = s_w[k + G_];
      acc0 += w0 * vec[(size_t)k * D + d];
      acc1 += w1 * vec[(size_t)(k + G_) * D + d];
      ws0 += w0; ws1 += w1;
    }
    if (k < nrow) { acc0 += s_w[k] * vec[(size_t)k * D + d]; ws0 += s_w[k]; }
  } else {
    for (int c = g; c < p.Kp; c += G_) acc0 += mub[(size_t)c * D + d];
  }
  s_part[tid] = acc0 + acc1;
  s_ws[tid] = ws0 + ws1;
  __syncthreads();
  if (tid < D) {
    float t = 0.f, ws = 0.f;
    for (int j = 0; j < G_; ++j) { t += s_part[j * D + tid]; ws += s_ws[j * D]; }
    if (!weighted) ws = (float)p.Kp;
    p.shift[(size_t)b * D + tid] = t / ws;
  }
}

// K1b: operand tile images of rows [blockIdx.y * 256, +256) of both sides (Y rows then X rows
// share the grid: y < KpPad/256 -> param rows, else z rows).
template <int D>
__global__ void __launch_bounds__(256) tc_prep_kernel(const __grid_constant__ PrepBatch pb) {
  using G = Geo<D>;
  const PrepArgs& p = pb.e[blockIdx.z];
  if ((int)blockIdx.y >= p.KpPad / 256 + p.KzPad / 256) return;
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  __shared__ float s_shift[D];
  if (tid < D) s_shift[tid] = p.shift[(size_t)b * D + tid];
  __syncthreads();
  const float* mub = p.mu + (size_t)b * p.Kp * D;
  const float* lvb = p.lv + (size_t)b * p.Kp * D;
  const float* zb = p.z + (size_t)b * p.Kz * D;
  const int ychunks = p.KpPad / 256;
  const bool yside = (int)blockIdx.y < ychunks;
  const int rbase = (yside ? (int)blockIdx.y : (int)blockIdx.y - ychunks) * 256;
  // Tile images: one thread per (row, 8-feature chunk) writes 16 B of the hi part and 16 B of the lo
  // part (8 consecutive chunk-threads fill one 128-byte swizzled row of an atom: coalesced).
  constexpr int CPR = D / 4;           // 8-feature chunks per row (2D features)
  constexpr int HC = D / 8;            // chunks of the first half ([z'^2] / [-lam/2])
  constexpr int RPI = 256 / CPR;       // rows per iteration of the CTA
  const int j = tid % CPR, rsub = tid / CPR;
  const int dj = (j < HC ? j : j - HC) * 8;
  uint8_t* Yb = p.Yt + (size_t)b * (p.KpPad / kTileRows) * G::TILE;
  uint8_t* Xb = p.Xt + (size_t)b * (p.KzPad / kTileRows) * G::TILE;
  float sh[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) sh[e] = s_shift[dj + e];
  auto store = [&](uint8_t* img, int row, const float* vals) {
    uint8_t* tile = img + (size_t)(row / kTileRows) * G::TILE;
    const int r = row % kTileRows;
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __half2 h = __floats2half2_rn(vals[2 * q], vals[2 * q + 1]);
      const float2 hf = __half22float2(h);
      __half2 l = __floats2half2_rn(vals[2 * q] - hf.x, vals[2 * q + 1] - hf.y);
      hi[q] = *reinterpret_cast<uint32_t*>(&h);
      lo[q] = *reinterpret_cast<uint32_t*>(&l);
    }
    const uint32_t off = swz_off(r, j * 8);
    *reinterpret_cast<uint4*>(tile + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(tile + G::PART + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  };
  // param rows -> Y tile image, beta
  if (yside)
  for (int c0 = rbase; c0 < rbase + 256; c0 += RPI) {
    const int c = c0 + rsub;
    float y[8];
    float bsum = 0.f;
    if (c < p.Kp) {
      const float4* lv4 = reinterpret_cast<const float4*>(lvb + (size_t)c * D + dj);
      const float4* mu4 = reinterpret_cast<const float4*>(mub + (size_t)c * D + dj);
      const float4 va = lv4[0], vb = lv4[1], ma = mu4[0], mb = mu4[1];
      const float vv[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
      const float mm[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float lam = __expf(-vv[e]);
        const float mp = mm[e] - sh[e];
        if (j < HC) {
          y[e] = -0.5f * p.alpha * lam * kLog2E;
          bsum += lam * mp * mp + vv[e] + kLog2Pi;
        } else {
          y[e] = p.alpha * lam * mp * kLog2E;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) y[e] = 0.f;
    }
    if (c < p.KpPad) store(Yb, c, y);
    // beta: sum over the HC first-half chunk-threads of the row (lane groups of CPR)
#pragma unroll
    for (int o = CPR / 2; o; o >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
    if (j == 0 && c < p.KpPad) p.beta[(size_t)b * p.KpPad + c] = (c < p.Kp) ? -0.5f * p.alpha * bsum : 0.f;
  }
  // z rows -> X tile image
  if (!yside)
  for (int a0 = rbase; a0 < rbase + 256; a0 += RPI) {
    const int a = a0 + rsub;
    float x[8];
    if (a < p.Kz) {
      const float4* z4 = reinterpret_cast<const float4*>(zb + (size_t)a * D + dj);
      const float4 za = z4[0], zc = z4[1];
      const float zz[8] = {za.x, za.y, za.z, za.w, zc.x, zc.y, zc.z, zc.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float zp = zz[e] - sh[e];
        x[e] = (j < HC) ? zp * zp : zp;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = 0.f;
    }
    if (a < p.KzPad) store(Xb, a, x);
  }
}

// ------------------------------------------------------------------------------ per-edge column bias
struct ColbiasArgs {
  const float* cb;       // [B][C] message bias (natural units)
  const float* beta;     // [B][betaStride] or NULL (DOWN: beta of the column/param side)
  int betaStride;
  int C, Cpad;
  float* cb2;            // [B][Cpad] out: (cb + beta - cbmax) * log2e, -inf padded
  uint8_t* bx;           // [B][Cpad/128][kBxBytes] out: the same bias as an extra K=16 MMA operand, or NULL
  int* live;             // [B][Cpad/128] out: 1 if any column of the 128-column tile is finite
  float* cbmax;          // [B]
  const double *off_cb, *off_rb;
  double* off_out;
};

// Edges per batched launch (forward, reverse, column bias, row terms): the siblings of one tree
// level share a persistent grid.  Kernel parameters up to 32 KB (CUDA >= 12.1) hold the batch.
constexpr int kMaxBatch = 32;
struct ColbiasBatch { ColbiasArgs e[kMaxBatch]; int ne; };

// Row r of a K=16 bias operand tile (the extra MMA that adds a per-column term to S): the value as
// four fp16-representable parts (each within +-60000 log2 units), every part as fp16 hi + lo in
// slots k = 2j, 2j+1 (the constant A operand has ones in k = 0..7); exact to ~2^-22 relative over
// +-240000 log2 units (beyond that, a dead entry, clamped).
__device__ __forceinline__ void store_bias_row(uint8_t* tiles, int r, float v) {
  uint32_t w[4];
  float rest = fminf(fmaxf(v, -240000.f), 240000.f);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float part = (j < 3) ? fminf(fmaxf(rest, -60000.f), 60000.f) : rest;
    rest -= part;
    __half hh, ll;
    split16(part, hh, ll);
    w[j] = (uint32_t)__half_as_ushort(hh) | ((uint32_t)__half_as_ushort(ll) << 16);
  }
  uint8_t* tile = tiles + (size_t)(r / kTileRows) * kBxBytes;
  const int rr = r % kTileRows;
  *reinterpret_cast<uint4*>(tile + bx_off(rr, 0)) = make_uint4(w[0], w[1], w[2], w[3]);
  *reinterpret_cast<uint4*>(tile + bx_off(rr, 8)) = make_uint4(0u, 0u, 0u, 0u);
}

// live[t] = 1 if any of the 128 log2 terms of tile t is finite (any number of tiles): one warp per
// tile, block-stride over tiles, read back from the values this block has just stored.
__device__ __forceinline__ void tile_live_flags(const float* vals, int ntiles, int* live) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = warp; t < ntiles; t += nw) {
    const float* v = vals + (size_t)t * kTileRows;
    const bool any = (v[lane] > -INFINITY) || (v[lane + 32] > -INFINITY) || (v[lane + 64] > -INFINITY) ||
                     (v[lane + 96] > -INFINITY);
    const unsigned m = __ballot_sync(0xffffffffu, any);
    if (lane == 0) live[t] = m ? 1 : 0;
  }
}

__global__ void __launch_bounds__(256) tc_colbias_kernel(const __grid_constant__ ColbiasBatch cbb_) {
  const ColbiasArgs& a = cbb_.e[blockIdx.y];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float red[32];
  const float* cbb = a.cb + (size_t)b * a.C;
  float m = -INFINITY;
  for (int c = tid; c < a.C; c += 256) m = fmaxf(m, cbb[c]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (tid == 0) {
    float v = red[0];
    for (int w = 1; w < 8; ++w) v = fmaxf(v, red[w]);
    red[16] = (v == -INFINITY) ? 0.f : v;
    red[17] = (v == -INFINITY) ? 1.f : 0.f;   // no live column: every message of this datapoint is -inf
  }
  __syncthreads();
  const float cmax = red[16];
  for (int c = tid; c < a.Cpad; c += 256) {
    float v = -INFINITY;
    if (c < a.C) {
      v = cbb[c] - cmax;
      if (a.beta) v += a.beta[(size_t)b * a.betaStride + c];
      v *= kLog2E;
    }
    a.cb2[(size_t)b * a.Cpad + c] = v;
    if (a.bx) {
      store_bias_row(a.bx + (size_t)b * (a.Cpad / kTileRows) * kBxBytes, c, v);
    }
  }
  __syncthreads();   // the block's cb2 stores are visible to the whole block
  if (a.live) tile_live_flags(a.cb2 + (size_t)b * a.Cpad, a.Cpad / kTileRows, a.live + (size_t)b * (a.Cpad / kTileRows));
  if (tid == 0) {
    a.cbmax[b] = cmax;
    double off = (double)cmax;
    if (a.off_cb) off += a.off_cb[b];
    if (a.off_rb) off += a.off_rb[b];
    // All columns dead: the clamped biases above would leave a finite (-6e4-scale) LSE, so the
    // offset carries the exact -inf (a sum of zero weights).
    a.off_out[b] = red[17] != 0.f ? -INFINITY : off;
  }
}

// ------------------------------------------------------------------------------ K3: forward contraction
struct FwdArgs {
  const uint8_t *At, *Bt;      // row / column operand tile images [B][tiles][TILE]
  int a_tiles, b_tiles;        // 128-row tiles per datapoint (a_tiles multiple of RB)
  const float* cb2;            // [B][b_tiles*128]
  const uint8_t* Bx;           // [B][b_tiles][kBxBytes] column bias as the extra K=16 MMA operand
  const float* ell_add;        // [B][ell_stride] added to ell (UP: beta of the row/param side) or NULL
  int ell_stride;
  const float* out_add;        // [B][R] added to out (DOWN: unary of the row/z side) or NULL
  int R, B;
  float lnC;
  float *out, *ell;            // [B][R]
};

// Several independent edges (siblings of a tree level) in one persistent launch: unit u belongs to
// edge e with ustart[e] <= u < ustart[e+1].  All edges of a batch share D.
// (kMaxBatch is defined with the colbias batch above)
struct FwdBatch {
  FwdArgs e[kMaxBatch];
  int ustart[kMaxBatch + 1];
  int ne;
  int count;                          // launch profiler on: add issued MMA flops to g_tmc_mma_flops
  unsigned long long flops_per_tile;  // tcgen05 flops issued per 128 x 128 pair tile
};
template <typename Batch>
__device__ __forceinline__ int batch_edge(const Batch& fb, int u) {
  int e = 0;
  while (e + 1 < fb.ne && u >= fb.ustart[e + 1]) ++e;
  return e;
}

// 2 of every 8 exponential pairs of the forward run on the FMA pipe (ex2_poly2, packed); DESIGN.md §12c.
#ifndef TMC_FWD_NPOLY2
#define TMC_FWD_NPOLY2 2
#endif
constexpr int kFwdPolyPairs = TMC_FWD_NPOLY2;

template <int D>
__global__ void __launch_bounds__(Geo<D>::THREADS, 1) tc_fwd_kernel(const __grid_constant__ FwdBatch fb) {
  using G = Geo<D>;
  constexpr int NPOLY2 = kFwdPolyPairs;
  constexpr int RB = G::RB, ST = G::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps the shared window
  uint8_t* sA = smem;                                   // RB tiles
  uint8_t* sB = sA + (size_t)RB * G::TILE;              // ST tiles
  uint8_t* sBx = sB + (size_t)ST * G::TILE;                            // ST x kBxBytes (bias operand ring)
  uint8_t* sAx = sBx + (size_t)ST * kBxBytes;                          // constant ones operand
  float2* sMerge = reinterpret_cast<float2*>(sAx + kBxBytes);          // [2][RB x 128] (max, sum) of half 1
  uint64_t* bars = reinterpret_cast<uint64_t*>(sMerge + 2 * RB * 128);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 1;
  uint64_t* b_full = bars + 2;            // [ST]
  uint64_t* b_empty = bars + 2 + ST;      // [ST]
  uint64_t* acc_full = bars + 2 + 2 * ST; // [2]
  uint64_t* acc_empty = bars + 4 + 2 * ST;// [2]
  uint64_t* cb_full = bars + 6 + 2 * ST;  // [ST] column-bias ring (consumed by the softmax warps)
  uint64_t* cb_empty = bars + 6 + 3 * ST; // [ST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6 + 4 * ST);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int units = fb.ustart[fb.ne];
#define TMC_FWD_UNIT()                                                   \
  const int e_ = batch_edge(fb, u);                                      \
  const FwdArgs& a = fb.e[e_];                                           \
  const int groups = a.a_tiles / RB;                                     \
  const int uu_ = u - fb.ustart[e_];                                     \
  const int b = uu_ / groups, g = uu_ % groups;                          \
  (void)b; (void)g

  if (tid == 0) {
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
      mbar_init(&cb_full[s], 1);
      mbar_init(&cb_empty[s], G::SOFTMAX_WARPS);
    }
    for (int s = 0; s < 2; ++s) { mbar_init(&acc_full[s], 1); mbar_init(&acc_empty[s], G::SOFTMAX_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // constant A operand of the bias MMA: k = 0..7 are ones (times the bias parts' hi and lo)
  for (int r = tid; r < kTileRows; r += blockDim.x) {
    *reinterpret_cast<uint4*>(sAx + bx_off(r, 0)) = make_uint4(0x3C003C00u, 0x3C003C00u, 0x3C003C00u, 0x3C003C00u);
    *reinterpret_cast<uint4*>(sAx + bx_off(r, 8)) = make_uint4(0u, 0u, 0u, 0u);
  }
  fence_proxy_async();
  if (warp == G::SOFTMAX_WARPS + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(G::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == G::SOFTMAX_WARPS) {
    TMC_PROF_T0(_tr0);
    // ===================== producer: bulk copies (TMA engine) =====================
    if (lane == 0) {
      uint32_t t = 0, ua = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++ua) {
        TMC_FWD_UNIT();
        TMC_PROF_WAIT(true, 2, mbar_wait(a_empty, (ua & 1) ^ 1));
        mbar_expect_tx(a_full, RB * G::TILE);
        bulk_g2s(sA, a.At + ((size_t)b * a.a_tiles + (size_t)g * RB) * G::TILE, RB * G::TILE, a_full);
        for (int j = 0; j < a.b_tiles; ++j, ++t) {
          const int s = t % ST;
          const uint32_t ph = ((t / ST) & 1) ^ 1;
          TMC_PROF_WAIT(true, 0, mbar_wait(&b_empty[s], ph));
          mbar_expect_tx(&b_full[s], G::TILE + kBxBytes);
          bulk_g2s(sB + (size_t)s * G::TILE, a.Bt + ((size_t)b * a.b_tiles + j) * G::TILE, G::TILE, &b_full[s]);
          bulk_g2s(sBx + (size_t)s * kBxBytes, a.Bx + ((size_t)b * a.b_tiles + j) * kBxBytes, kBxBytes, &b_full[s]);
        }
        if (fb.count) atomicAdd(&g_tmc_mma_flops[PF_TC_FWD], (unsigned long long)a.b_tiles * RB * fb.flops_per_tile);
      }
    }
    TMC_PROF_END(lane == 0, 14, _tr0);
  } else if (warp == G::SOFTMAX_WARPS + 1) {
    TMC_PROF_T0(_tr1);
    // ===================== MMA issuer (whole warp, one elected lane issues) =====================
    {
      uint32_t t = 0, ua = 0;
      const uint32_t aBase = smem_u32(sA), bBase = smem_u32(sB), axBase = smem_u32(sAx), bxBase = smem_u32(sBx);
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++ua) {
        TMC_FWD_UNIT();
        TMC_PROF_WAIT(lane == 0, 6, mbar_wait(a_full, ua & 1));
        for (int j = 0; j < a.b_tiles; ++j, ++t) {
          const int s = t % ST, as = t & 1;
          TMC_PROF_WAIT(lane == 0, 3, mbar_wait(&b_full[s], (t / ST) & 1));
          TMC_PROF_WAIT(lane == 0, 4, mbar_wait(&acc_empty[as], ((t >> 1) & 1) ^ 1));
          tc_fence_after();
#pragma unroll
          for (int rb = 0; rb < RB; ++rb) {
            const uint32_t d = tmem + (uint32_t)((rb * 2 + as) * 128);
            const uint64_t dA = sdesc(aBase + rb * G::TILE), dB = sdesc(bBase + s * G::TILE);
            // small cross terms first, the large hi*hi products last: fewer fp32 accumulator
            // roundings at large partial-sum magnitude
#pragma unroll
            for (int at = 0; at < G::ATOMS; ++at) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint32_t o = at * kAtomBytes + kk * 32;
                mma_f16(d, dadd(dA, o), dadd(dB, G::PART + o), kIdescF16M128N128, (at | kk) ? 1u : 0u);
                mma_f16(d, dadd(dA, G::PART + o), dadd(dB, o), kIdescF16M128N128, 1u);
              }
            }
#pragma unroll
            for (int at = 0; at < G::ATOMS; ++at) {
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint32_t o = at * kAtomBytes + kk * 32;
                mma_f16(d, dadd(dA, o), dadd(dB, o), kIdescF16M128N128, 1u);
              }
            }
            // + column bias: ones(128 x 16) . [cb_hi, cb_lo, 0..]^T
            mma_f16(d, sdesc_bx(axBase), sdesc_bx(bxBase + s * kBxBytes), kIdescF16M128N128, 1u);
          }
          mma_commit(&b_empty[s]);
          mma_commit(&acc_full[as]);
        }
        mma_commit(a_empty);
      }
    }
    TMC_PROF_END(lane == 0, 12, _tr1);
  } else {
    TMC_PROF_T0(_tr2);
    // ===================== softmax warps: TMEM -> online log2-sum-exp2 =====================
    // warp -> (TMEM lane quarter, row block rb, column half): each thread owns one row of one
    // 64-column half of every S tile; the two halves' (max, sum) states merge at the unit's end.
    const int sw = warp;
    const int rb = (sw >> 2) % RB;
    const int half = sw / (4 * RB);
    const int quarter = warp & 3;               // TMEM lane quarter this warp may access
    const int rloc = rb * 128 + quarter * 32 + lane;
    uint32_t t = 0, ua = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++ua) {
      TMC_FWD_UNIT();
      // the unit's row terms, loaded now and used after the last tile (their latency is off the
      // critical path at the unit boundary)
      const int r = g * RB * 128 + rloc;
      float ea = 0.f, oa = 0.f;
      if (half == 0 && r < a.R) {
        if (a.ell_add) ea = a.ell_add[(size_t)b * a.ell_stride + r];
        if (a.out_add) oa = a.out_add[(size_t)b * a.R + r];
      }
      float mref = -INFINITY, sum = 0.f;
      for (int j = 0; j < a.b_tiles; ++j, ++t) {
        const int as = t & 1;
        TMC_PROF_WAIT(sw == 0 && lane == 0, 8, mbar_wait(&acc_full[as], (t >> 1) & 1));
        tc_fence_after();
        uint32_t v[64];
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)((rb * 2 + as) * 128 + half * 64);
        TMC_LD32(taddr + 0, (v + 0));
        TMC_LD32(taddr + 32, (v + 32));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[as]);
        // x = S + colbias, both from the tensor core (the bias is the extra K=16 MMA)
        float2 x2[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) x2[q] = make_float2(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1]));
        // row max of this tile half (4 independent 3-input max chains, FMNMX3)
        auto tile_max = [&]() {
          float mx[4];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int c = q & 3;
            const float m4 = fmaxf(fmaxf(x2[2 * q].x, x2[2 * q].y), fmaxf(x2[2 * q + 1].x, x2[2 * q + 1].y));
            mx[c] = (q < 4) ? m4 : fmaxf(mx[c], m4);
          }
          return fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        };
        auto tile_sum = [&](float m) {
          // NPOLY2 of every 8 exponential pairs run on the FMA pipe (ex2_poly2), the rest on MUFU;
          // arguments and partial sums on packed pairs (4 independent float2 accumulators)
          const float2 nm = make_float2(-m, -m);
          float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float2 y = __fadd2_rn(x2[q], nm);
            const float2 e = ((q & 7) >= 8 - NPOLY2) ? ex2_poly2(y) : make_float2(ex2(y.x), ex2(y.y));
            acc[q & 3] = __fadd2_rn(acc[q & 3], e);
          }
          const float2 t01 = __fadd2_rn(acc[0], acc[1]), t23 = __fadd2_rn(acc[2], acc[3]);
          const float2 tt = __fadd2_rn(t01, t23);
          return tt.x + tt.y;
        };
        const float tmax = tile_max();
        if (tmax > mref + 8.f) {          // lazy rescale: only when the max grows by > 2^8
          sum = (mref == -INFINITY) ? 0.f : sum * ex2(mref - tmax);
          mref = tmax;
        }
        if (mref > -INFINITY) sum += tile_sum(mref);
      }
      // merge the two column halves of each row (half 1 -> SMEM -> half 0): only the two warps
      // holding the halves of the same rows meet (one named barrier per (row block, lane quarter),
      // ids 1..4 RB); the merge slots alternate with the unit parity, so half 1 can write the next
      // unit's slot while half 0 still reads this one (one barrier per unit)
      float2* mslot = sMerge + (ua & 1) * (RB * 128);
      if (half == 1) mslot[rloc] = make_float2(mref, sum);
      named_bar(1 + rb * 4 + quarter, 64);
      if (half == 0) {
        const float2 o = mslot[rloc];
        const float M = fmaxf(mref, o.x);
        float tot = 0.f;
        if (M > -INFINITY) tot = (mref > -INFINITY ? sum * ex2(mref - M) : 0.f) + (o.x > -INFINITY ? o.y * ex2(o.x - M) : 0.f);
        if (r < a.R) {
          float e = (tot > 0.f) ? kLn2 * (M + __log2f(tot)) : -INFINITY;
          if (a.ell_add) e += ea;
          a.ell[(size_t)b * a.R + r] = e;
          a.out[(size_t)b * a.R + r] = oa + e - a.lnC;
        }
      }
    }
    TMC_PROF_END(warp == 0 && lane == 0, 13, _tr2);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == G::SOFTMAX_WARPS + 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(G::TMEM_COLS));
  }
}
#undef TMC_FWD_UNIT


// ------------------------------------------------------------------------------ K4: reverse pass
// One "owner" pass of the reverse contraction.  The CTA owns 128 rows m of one
// datapoint and streams the other side in 128-wide tiles n:
//   P~[m,n] = ex2(S2[m,n] + ho[m] + ht[n] + 14)          (= 2^14 |w|/wscale exp(logf + bias - ell))
//   G[m,:] += sum_n P~[m,n] T[n,:]                         (tcgen05, P~ and T both fp16 hi/lo)
//   rowsum[m] = sum_n P~[m,n]
// S is recomputed on tensor cores exactly as in the forward, and the streamed term ht is added by
// the tensor core too (a K=16 bias MMA on pre-split tiles), so the softmax computes
// ex2(S + ho + 14) with one FADD2 per pair.  P~ is split into fp16 hi/lo and stored back into the
// TMEM columns its S tile came from (hi in the first 16 of each 32-column quarter, lo in the last
// 16), where it is the A operand (tcgen05.mma A-from-TMEM) of the gradient GEMM whose B operand is
// the streamed tile itself read MN-major; the S buffer is released to the next S MMA by the commit
// of that gradient GEMM.  Two MMA-issuing warps (S MMAs / gradient GEMMs), eight softmax warps (SG =
// 3: TMEM lane quarter x column half, two 32-column quarters each), four epilogue warps that turn G
// into dz (T = Y tiles) or dmu/dlogvar (T = X tiles).
struct BwdArgs {
  const uint8_t *Ot, *Tt;      // owned / streamed tile images [B][tiles][TILE]
  int o_tiles, t_tiles;
  const float* ho;             // [B][o_tiles*128] owned log2 term
  const float* ht;             // [B][t_tiles*128] streamed log2 term (-inf padded)
  const uint8_t* Hx;           // [B][t_tiles][kBxBytes] the same term as the K=16 bias operand (added by the tensor core)
  const float* sgn;            // [B] signed scale of the upstream weights (w = sgn * |w|/|sgn|)
  float alpha;                 // factor power (param-side gradients scale by alpha; the Y tiles carry it already)
  int M, B;
  int owner_z;                 // 1: G = sum P Y -> dz ; 0: G = sum P X -> dmu, dlogvar
  const float *z, *mu, *lv;    // owner-side fp32 inputs [B][M][D]
  const float* shift;          // [B][D]
  float *gz, *gmu, *glv;       // gradient outputs [B][M][D]
  float* rowsum;               // [B][M] sum_n P (the edge's column sum) or NULL
  const int *olive, *tlive;    // [B][o_tiles], [B][t_tiles]: 0 = every P~ of the tile is exactly 0 (skipped)
  int* tflag;                  // row-owner pass: [B][t_tiles] set to 1 when any P~ of a streamed tile is nonzero in fp16
  const int* oflag;            // column-owner pass: those flags for the owned tiles (0: the tile's sums are 0, R6)
};

template <int D>
#ifndef TMC_BWD_NPOLY
#define TMC_BWD_NPOLY 0   // reverse-pass softmax: groups (of 8) of 4 exponentials evaluated on the FMA pipe
#endif
#ifndef TMC_EPI_PREFETCH
#define TMC_EPI_PREFETCH 1   // reverse-pass epilogue (D <= 32): owner rows loaded before the accumulator waits
#endif
#ifndef TMC_BWD_SPLIT
#define TMC_BWD_SPLIT 1   // 1: S MMAs and gradient MMAs issued by two warps (see tc_bwd_kernel)
#endif
struct BGeo {
  static constexpr int TILE = Geo<D>::TILE;
  static constexpr int PART = Geo<D>::PART;
  static constexpr int ATOMS = Geo<D>::ATOMS;
#ifndef TMC_BWD_ST32
#define TMC_BWD_ST32 4
#endif
  static constexpr int ST = (D <= 32) ? TMC_BWD_ST32 : 2;      // streamed-tile ring depth
  static constexpr int SMW = 16;                               // softmax warps (4 per TMEM lane quarter)
  static constexpr int EW = 4;                                 // epilogue warps (1 per TMEM lane quarter)
  static constexpr int THREADS = 32 * (SMW + EW + 2 + TMC_BWD_SPLIT);
  static constexpr size_t SMEM = 1024 + (size_t)TILE + (size_t)ST * TILE + (size_t)(ST + 1) * 4096 /*bias ring + ones*/ +
                                 2 * 4 * 128 * 4 + 512;
};

// MN-major SWIZZLE_128B descriptor: LBO = stride of 64-element MN chunks, SBO = 8-row K groups.
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// D[tmem] (+)= A[tmem] * B[smem]  (A K-major in TMEM: lane = row, fp16 pairs per 32-bit column)
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}

#define TMC_ST32(taddr, v)                                                                                          \
  asm volatile(                                                                                                     \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"  \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                                 \
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),           \
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),    \
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),   \
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])                                                    \
      : "memory")

#define TMC_ST16(taddr, v)                                                                                          \
  asm volatile(                                                                                                     \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"      \
      ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),         \
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])                 \
      : "memory")

#define TMC_LD8(taddr, v)                                                                                           \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                             \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])    \
               : "r"(taddr))

#define TMC_LD16(taddr, v)                                                                                          \
  asm volatile(                                                                                                     \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"       \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),            \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])       \
      : "r"(taddr))

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// GT = fp16 terms of the gradient GEMM:
//   1 = P_hi T_hi, 2 = P_hi (T_lo + T_hi), 3 = P_lo T_hi + P_hi T_lo + P_hi T_hi  (N = 2D MMAs), and the
//   packed forms, where one MMA of N = 4D reads the streamed tile's hi and lo parts side by side
//   ([T_hi | T_lo] is exactly the tile image seen MN-major with LBO = one atom) and the epilogue adds
//   the two column halves:  4 = P_hi [T_hi | T_lo],  5 = (P_hi + P_lo) [T_hi | T_lo].
struct BwdBatch {
  BwdArgs e[kMaxBatch];
  int ustart[kMaxBatch + 1];
  int ne;
  int count;                          // launch profiler on: add issued MMA flops to g_tmc_mma_flops
  unsigned long long flops_per_tile;  // tcgen05 flops issued per live 128 x 128 pair tile
};

// SG = softmax groups: 1 = all 16 softmax warps on every tile (one 32-column quarter each);
// 2 = two groups of 8 alternating tiles (each warp two 32-column quarters), so two tiles are in
// the softmax stage at once and the S -> P~ -> gradient-GEMM handoffs of one group overlap the other.
// SG: 1 = 16 softmax warps, one 32-column quarter each; 2 = two groups of 8 on alternating tiles;
// 3 = 8 softmax warps, two column quarters each with both TMEM loads in flight together.
// (4 softmax warps with all four quarters, loads in two pairs, measured 34% slower: one warp per
// SMSP cannot keep the MUFU fed.)
__host__ __device__ constexpr int bwd_smw(int SG) { return SG == 3 ? 8 : 16; }
template <int D, int SG>
__host__ __device__ constexpr int bwd_threads() { return 32 * (bwd_smw(SG) + BGeo<D>::EW + 2 + TMC_BWD_SPLIT); }

// CF: the row-owner pass records which streamed (column) tiles carry fp16 weight (BwdArgs::tflag); the
// column-owner instantiation (CF = false) has no trace of it in its softmax loop.
template <int D, int GT, int SG, bool CF>
__global__ void __launch_bounds__(bwd_threads<D, SG>(), 1) tc_bwd_kernel(const __grid_constant__ BwdBatch fb) {
  using G = BGeo<D>;
  constexpr int ST = G::ST, SMW = bwd_smw(SG), EW = G::EW;
  constexpr int SMX_ARRIVE = (SG == 2) ? SMW / 2 : SMW;     // softmax warps per tile
  constexpr int W_PROD = SMW + EW, W_MMA = SMW + EW + 1;     // role warps take the highest ids
  constexpr int W_MMAG = TMC_BWD_SPLIT ? W_MMA + 1 : W_MMA;  // gradient-MMA issuer (split mode)
  constexpr uint32_t IDESC_S = kIdescF16M128N128;
  constexpr bool PACKED = GT >= 4;
  constexpr uint32_t GN = PACKED ? 4 * D : 2 * D;            // N of the gradient MMA
  constexpr bool PLO = (GT == 3 || GT == 5);                 // P~ lo part needed
  constexpr uint32_t IDESC_G = (1u << 4) | (1u << 16) | (GN >> 3 << 17) | ((128u >> 4) << 24);
  // TMEM: NSB S/P~ buffers of 128 columns, then GB gradient accumulators of GN columns.  Three S
  // buffers let S(j+1) run while the gradient GEMM of j-1 still reads its P~; two accumulators let
  // the epilogue warps drain unit u while the MMAs of unit u+1 already accumulate.
  constexpr int NSB = (3 * 128 + 2 * GN <= 512) ? 3 : 2;
  constexpr int GB = (NSB * 128 + 2 * GN <= 512) ? 2 : 1;
  constexpr uint32_t GCOL = NSB * 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sO = smem;
  uint8_t* sT = sO + G::TILE;
  uint8_t* sHx = sT + (size_t)ST * G::TILE;                 // [ST] streamed-term bias operand tiles
  uint8_t* sOnes = sHx + (size_t)ST * kBxBytes;             // constant ones A operand of the bias MMA
  float* sRs = reinterpret_cast<float*>(sOnes + kBxBytes);  // [2 (unit parity)][4 (column quarter)][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRs + 1024);
  uint64_t* o_full = bars + 0;
  uint64_t* o_empty = bars + 1;
  uint64_t* t_full = bars + 2;              // [ST]
  uint64_t* t_empty = bars + 2 + ST;        // [ST]
  uint64_t* h_full = bars + 2 + 2 * ST;     // [ST]
  uint64_t* h_empty = bars + 2 + 3 * ST;    // [ST]
  uint64_t* s_full = bars + 2 + 4 * ST;     // [3]  S tile ready in TMEM buffer
  uint64_t* s_empty = bars + 5 + 4 * ST;    // [3]  buffer free (its P~ consumed by the gradient GEMM)
  uint64_t* p_full = bars + 8 + 4 * ST;     // [3]  P~ written back into the buffer
  uint64_t* g_full = bars + 11 + 4 * ST;    // [2]  gradient accumulator complete
  uint64_t* g_empty = bars + 13 + 4 * ST;   // [2]  accumulator drained by the epilogue warps
  uint64_t* r_full = bars + 15 + 4 * ST;    // [2]  row sums of the unit written to sRs
  uint64_t* r_empty = bars + 17 + 4 * ST;   // [2]  row sums consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 19 + 4 * ST);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int units = fb.ustart[fb.ne];
  // Exact sparsity: a tile whose owner rows (or streamed rows) all carry weight exactly 0 has
  // P~ == 0 everywhere, so every role skips it consistently (phase counters count live work only).
  auto olive = [](const BwdArgs& a, int b, int mt) -> bool { return !a.olive || a.olive[(size_t)b * a.o_tiles + mt]; };
  auto tlive = [](const BwdArgs& a, int b, int j) -> bool { return !a.tlive || a.tlive[(size_t)b * a.t_tiles + j]; };
  // The streamed-tile flags of one datapoint as a register bitmask, loaded once per unit by a whole
  // warp (a per-tile global load sat on every role's critical path: ~750 clk per tile).
  auto tmask = [](const BwdArgs& a, int b) -> uint64_t {
    if (!a.tlive) return ~0ull;
    if (a.t_tiles > 64) return 0ull;                      // callers fall back to tlive()
    const int l = threadIdx.x & 31;
    const int f0 = l < a.t_tiles ? a.tlive[(size_t)b * a.t_tiles + l] : 0;
    const int f1 = l + 32 < a.t_tiles ? a.tlive[(size_t)b * a.t_tiles + l + 32] : 0;
    return (uint64_t)__ballot_sync(0xffffffffu, f0) | ((uint64_t)__ballot_sync(0xffffffffu, f1) << 32);
  };
  auto live = [&](const BwdArgs& a, int b, uint64_t msk, int j) -> bool {
    return a.t_tiles <= 64 ? ((msk >> j) & 1ull) != 0 : tlive(a, b, j);
  };
#define TMC_BWD_UNIT()                                                   \
  const int e_ = batch_edge(fb, u);                                      \
  const BwdArgs& a = fb.e[e_];                                           \
  const int uu_ = u - fb.ustart[e_];                                     \
  const int b = uu_ / a.o_tiles, mt = uu_ % a.o_tiles
  if (tid == 0) {
    mbar_init(o_full, 1);
    mbar_init(o_empty, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&t_full[s], 1); mbar_init(&t_empty[s], 1);
      mbar_init(&h_full[s], 1); mbar_init(&h_empty[s], 1);      // bias tile: read by the S MMAs only
    }
    for (int s = 0; s < NSB; ++s) { mbar_init(&s_full[s], 1); mbar_init(&s_empty[s], 1); mbar_init(&p_full[s], SMX_ARRIVE); }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&g_full[s], 1); mbar_init(&g_empty[s], EW);
      mbar_init(&r_full[s], SMW); mbar_init(&r_empty[s], EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int r = tid; r < kTileRows; r += blockDim.x) {       // ones in k = 0..7 (times the bias parts)
    *reinterpret_cast<uint4*>(sOnes + bx_off(r, 0)) = make_uint4(0x3C003C00u, 0x3C003C00u, 0x3C003C00u, 0x3C003C00u);
    *reinterpret_cast<uint4*>(sOnes + bx_off(r, 8)) = make_uint4(0u, 0u, 0u, 0u);
  }
  fence_proxy_async();
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == W_PROD) {
    TMC_PROF_T0(_tr0);
    if (lane == 0) {   // ---------------- producer
      uint32_t t = 0, ua = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        TMC_BWD_UNIT();
        if (!olive(a, b, mt)) continue;
        TMC_PROF_WAIT(true, 2, mbar_wait(o_empty, (ua & 1) ^ 1));
        ++ua;
        mbar_expect_tx(o_full, G::TILE);
        bulk_g2s(sO, a.Ot + ((size_t)b * a.o_tiles + mt) * G::TILE, G::TILE, o_full);
        unsigned long long nlive = 0;
        for (int j = 0; j < a.t_tiles; ++j) {
          if (!tlive(a, b, j)) continue;
          ++nlive;
          const int s = t % ST;
          const uint32_t ph = ((t / ST) & 1) ^ 1;
          TMC_PROF_WAIT(true, 0, mbar_wait(&t_empty[s], ph));
          mbar_expect_tx(&t_full[s], G::TILE);
          bulk_g2s(sT + (size_t)s * G::TILE, a.Tt + ((size_t)b * a.t_tiles + j) * G::TILE, G::TILE, &t_full[s]);
          TMC_PROF_WAIT(true, 1, mbar_wait(&h_empty[s], ph));
          mbar_expect_tx(&h_full[s], kBxBytes);
          bulk_g2s(sHx + (size_t)s * kBxBytes, a.Hx + ((size_t)b * a.t_tiles + j) * kBxBytes, kBxBytes, &h_full[s]);
          ++t;
        }
        if (fb.count) atomicAdd(&g_tmc_mma_flops[PF_TC_BWD], nlive * fb.flops_per_tile);
      }
    }
    TMC_PROF_END(lane == 0, 14, _tr0);
  } else if (warp == W_MMA || warp == W_MMAG) {
    TMC_PROF_T0(_tr1);
    {   // ---------------- MMA issuer (whole warp, one elected lane issues)
#if defined(TMC_INSTRUMENT) && TMC_MMA_PROF == 2
      long long mprof[16] = {0};
#endif
      uint32_t t = 0, ua = 0;
      const uint32_t oBase = smem_u32(sO), tBase = smem_u32(sT);
      auto grad = [&](const BwdArgs& a, uint32_t tt, bool first) {
        const uint32_t as = tt % NSB;
        const uint32_t gb = ua % GB;
        TMC_PROF_WAIT_M(5, mbar_wait(&p_full[as], (tt / NSB) & 1));
        if (first) TMC_PROF_WAIT_M(7, mbar_wait(&g_empty[gb], ((ua / GB) & 1) ^ 1));
        tc_fence_after();
        const uint32_t Ts = tBase + (tt % ST) * G::TILE;
        const uint32_t pA = tmem + as * 128;
        const uint32_t gD = tmem + GCOL + gb * GN;
        const uint64_t dT = sdesc_mn(Ts, kAtomBytes);
        TMC_PROF_T0_M(_tg);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          // P~ of K-step kk: 16 tile columns held by column quarter kk/2, hi then lo (16 TMEM columns each)
          const uint32_t phi = pA + (kk >> 1) * 32 + (kk & 1) * 8, plo = phi + 16;
          const uint64_t thi = dadd(dT, kk * 2048), tlo = dadd(dT, G::PART + kk * 2048);
          const uint32_t acc0 = (!first || kk) ? 1u : 0u;
          if constexpr (PACKED) {
            if constexpr (GT == 5) mma_f16_ts(gD, plo, thi, IDESC_G, acc0);
            mma_f16_ts(gD, phi, thi, IDESC_G, GT == 5 ? 1u : acc0);
          } else {
            if constexpr (GT >= 3) mma_f16_ts(gD, plo, thi, IDESC_G, acc0);
            if constexpr (GT >= 2) mma_f16_ts(gD, phi, tlo, IDESC_G, GT >= 3 ? 1u : acc0);
            mma_f16_ts(gD, phi, thi, IDESC_G, GT >= 2 ? 1u : acc0);
          }
        }
        TMC_PROF_END_M(11, _tg);
        TMC_PROF_T0_M(_tc);
        mma_commit(&t_empty[tt % ST]);
        mma_commit(&s_empty[as]);
        TMC_PROF_END_M(16, _tc);
      };
      // Split mode: a second warp issues the gradient GEMMs, so the S issue stream never stalls on
      // the P~ hand-off of the previous tile (each thread's tcgen05.commit tracks its own MMAs; the
      // gradient MMA of tile j is issued after p_full(j), which implies S(j) completed, so its
      // commit may free both the S buffer and the streamed tile).
      if (TMC_BWD_SPLIT && warp == W_MMAG) {
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
          TMC_BWD_UNIT();
          if (!olive(a, b, mt)) continue;
          const uint64_t tm = tmask(a, b);
          int jj = 0;
          for (int j = 0; j < a.t_tiles; ++j) {
            if (!live(a, b, tm, j)) continue;
            grad(a, t, jj == 0);
            ++jj;
            ++t;
          }
          mma_commit(&g_full[ua % GB]);
          ++ua;
        }
      } else
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        TMC_BWD_UNIT();
        if (!olive(a, b, mt)) continue;
        const uint64_t tm = tmask(a, b);
        TMC_PROF_WAIT_M(6, mbar_wait(o_full, ua & 1));
        int jj = 0;                      // live streamed tiles so far in this unit
        for (int j = 0; j < a.t_tiles; ++j) {
          if (!live(a, b, tm, j)) continue;
          const int s = t % ST, as = t % NSB;
          TMC_PROF_WAIT_M(3, mbar_wait(&t_full[s], (t / ST) & 1));
          mbar_wait(&h_full[s], (t / ST) & 1);
          TMC_PROF_WAIT_M(4, mbar_wait(&s_empty[as], ((t / NSB) & 1) ^ 1));
          TMC_PROF_WAIT_M(17, tc_fence_after());
          const uint32_t d = tmem + (uint32_t)(as * 128);
          const uint64_t dO = sdesc(oBase), dS = sdesc(tBase + s * G::TILE);
          TMC_PROF_T0_M(_ts);
#pragma unroll
          for (int at = 0; at < G::ATOMS; ++at) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t o = at * kAtomBytes + kk * 32;
              mma_f16(d, dadd(dO, o), dadd(dS, G::PART + o), IDESC_S, (at | kk) ? 1u : 0u);
              mma_f16(d, dadd(dO, G::PART + o), dadd(dS, o), IDESC_S, 1u);
            }
          }
#pragma unroll
          for (int at = 0; at < G::ATOMS; ++at) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t o = at * kAtomBytes + kk * 32;
              mma_f16(d, dadd(dO, o), dadd(dS, o), IDESC_S, 1u);
            }
          }
          // + the streamed term ht (log2 units) on the tensor core: ones(128 x 16) . [parts hi/lo]^T
          mma_f16(d, sdesc_bx(smem_u32(sOnes)), sdesc_bx(smem_u32(sHx) + s * kBxBytes), IDESC_S, 1u);
          TMC_PROF_END_M(15, _ts);
          TMC_PROF_T0_M(_tc2);
          mma_commit(&s_full[as]);
          mma_commit(&h_empty[s]);
          TMC_PROF_END_M(18, _tc2);
          if (!TMC_BWD_SPLIT && jj > 0) grad(a, t - 1, jj == 1);
          ++jj;
          ++t;
        }
        if (!TMC_BWD_SPLIT) {
          if (jj > 0) grad(a, t - 1, jj == 1);
          mma_commit(&g_full[ua % GB]);
        }
        mma_commit(o_empty);
        ++ua;
      }
#if defined(TMC_INSTRUMENT) && TMC_MMA_PROF == 2
      if (lane == 0)
        for (int q = 0; q < 16; ++q) atomicAdd(&g_tmc_prof[blockIdx.x & 1023][3 + q], (unsigned long long)mprof[q]);
#endif
    }
    TMC_PROF_END(lane == 0, 12, _tr1);
  } else if (warp < SMW) {
    TMC_PROF_T0(_tr2);
    // ---------------- softmax / P~ warps (16)
    // warp -> (TMEM lane quarter, column quarter cq): 32 columns of every S tile; P~ hi/lo go back
    // into those same 32 columns (hi in the first 16, lo in the last 16), so no warp writes TMEM
    // columns another warp still has to read.
    const int sw = warp;
    const int quarter = warp & 3;               // TMEM lane quarter this warp may access
    const int grp = (SG == 2) ? (sw >> 3) : 0;  // tile parity this warp processes (SG = 2)
    const int slot = (SG == 2) ? ((sw >> 2) & 1) : (SG == 3) ? (sw >> 2) * 2 : (sw >> 2);   // row-sum slot (4 per row)
    const int m = quarter * 32 + lane;          // owned row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t t = 0, ua = 0;
#if defined(TMC_INSTRUMENT) && defined(TMC_SMX_PROF)
    long long sprof[6] = {0, 0, 0, 0, 0, 0};   // waits, TMEM ld, math, TMEM st + release, unit start, row-sum handoff
    long long _sp = clock64();
#define TMC_SMX_MARK(q) do { const long long _n = clock64(); sprof[q] += _n - _sp; _sp = _n; } while (0)
#else
#define TMC_SMX_MARK(q) do {} while (0)
#endif
    // P~ of 32 columns: arguments S + ht + (ho + 14) on packed pairs, ex2, row-sum accumulation,
    // fp16 hi/lo split
    float pmax = 0.f;   // CF: largest P~ this thread computed in the current streamed tile
    auto chunk_math = [&](const uint32_t* v, float2 hom2, float2* racc, uint32_t* hi, uint32_t* lo) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        // S already carries the streamed term (bias MMA); + the owned term (ho + 14)
        const float2 y01 = __fadd2_rn(make_float2(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1])), hom2);
        const float2 y23 = __fadd2_rn(make_float2(__uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])), hom2);
        const bool poly = q >= 8 - TMC_BWD_NPOLY;
        const float2 p01 = poly ? make_float2(ex2_poly(y01.x), ex2_poly(y01.y)) : make_float2(ex2(y01.x), ex2(y01.y));
        const float2 p23 = poly ? make_float2(ex2_poly(y23.x), ex2_poly(y23.y)) : make_float2(ex2(y23.x), ex2(y23.y));
        racc[0] = __fadd2_rn(racc[0], p01);
        racc[1] = __fadd2_rn(racc[1], p23);
        if constexpr (CF) {
          pmax = fmaxf(pmax, fmaxf(p01.x, p01.y));
          pmax = fmaxf(pmax, fmaxf(p23.x, p23.y));
        }
        __half2 h01 = __floats2half2_rn(p01.x, p01.y), h23 = __floats2half2_rn(p23.x, p23.y);
        hi[2 * q] = *reinterpret_cast<uint32_t*>(&h01);
        hi[2 * q + 1] = *reinterpret_cast<uint32_t*>(&h23);
        if constexpr (PLO) {
          const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
          const float2 d01 = __fadd2_rn(p01, make_float2(-f01.x, -f01.y));
          const float2 d23 = __fadd2_rn(p23, make_float2(-f23.x, -f23.y));
          __half2 l01 = __floats2half2_rn(d01.x, d01.y), l23 = __floats2half2_rn(d23.x, d23.y);
          lo[2 * q] = *reinterpret_cast<uint32_t*>(&l01);
          lo[2 * q + 1] = *reinterpret_cast<uint32_t*>(&l23);
        }
      }
    };
    // the per-unit global loads (owned-tile live flag, owned row term, streamed-tile live flags) of
    // unit u + gridDim.x are issued while unit u runs: their latency leaves the unit boundary
    struct UnitPre { int olv; float ho; int f0, f1; };
    auto unit_pre = [&](int un) -> UnitPre {
      UnitPre r{0, 0.f, 0, 0};
      if (un >= units) return r;
      const int en = batch_edge(fb, un);
      const BwdArgs& an = fb.e[en];
      const int uun = un - fb.ustart[en];
      const int bn = uun / an.o_tiles, mtn = uun % an.o_tiles;
      r.olv = olive(an, bn, mtn) ? 1 : 0;
      r.ho = an.ho[(size_t)bn * an.o_tiles * 128 + mtn * 128 + m];
      if (an.tlive && an.t_tiles <= 64) {
        r.f0 = lane < an.t_tiles ? an.tlive[(size_t)bn * an.t_tiles + lane] : 0;
        r.f1 = lane + 32 < an.t_tiles ? an.tlive[(size_t)bn * an.t_tiles + lane + 32] : 0;
      }
      return r;
    };
    UnitPre nxt = unit_pre(blockIdx.x);
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      TMC_BWD_UNIT();
      (void)mt;
      const UnitPre cur = nxt;
      nxt = unit_pre(u + gridDim.x);
      if (!cur.olv) continue;
      const float hom = cur.ho + 14.f;
      const float2 hom2 = make_float2(hom, hom);
      float2 racc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      uint32_t fmask = 0;                // CF: bit j = this thread saw fp16 weight in streamed tile j
      TMC_SMX_MARK(4);
      const uint64_t tm = !a.tlive ? ~0ull : a.t_tiles > 64 ? 0ull
                        : ((uint64_t)__ballot_sync(0xffffffffu, cur.f0) | ((uint64_t)__ballot_sync(0xffffffffu, cur.f1) << 32));
      for (int j = 0; j < a.t_tiles; ++j) {
        if (!live(a, b, tm, j)) continue;
        if (SG == 2 && (int)(t & 1) != grp) { ++t; continue; }
        const int as = t % NSB;
        TMC_PROF_WAIT(lane == 0, 32 + sw, mbar_wait(&s_full[as], (t / NSB) & 1));
        tc_fence_after();
        TMC_SMX_MARK(0);
        if constexpr (CF) pmax = 0.f;
        if constexpr (SG == 3) {
          // two column quarters, both TMEM loads in flight before the first wait
          const int cq0 = (sw >> 2) * 2;
          const uint32_t ta0 = tmem + lane_off + (uint32_t)(as * 128 + cq0 * 32), ta1 = ta0 + 32;
          uint32_t v0[32], v1[32];
          TMC_LD32(ta0, v0);
          TMC_LD32(ta1, v1);
          tmem_ld_wait();
          TMC_SMX_MARK(1);
          uint32_t hi[16], lo[16];
          if (hom > -INFINITY) chunk_math(v0, hom2, racc, hi, lo);
          else for (int q = 0; q < 16; ++q) { hi[q] = 0u; lo[q] = 0u; }
          TMC_ST16(ta0, hi);
          if constexpr (PLO) TMC_ST16(ta0 + 16, lo);
          if (hom > -INFINITY) chunk_math(v1, hom2, racc, hi, lo);
          TMC_SMX_MARK(2);
          TMC_ST16(ta1, hi);
          if constexpr (PLO) TMC_ST16(ta1 + 16, lo);
        } else
#pragma unroll 1
        for (int c = 0; c < (SG == 2 ? 2 : 1); ++c) {
          // column quarter handled now: 32 S columns; P~ hi/lo go back into the same 32 columns
          const int cq = (SG == 2) ? (((sw >> 2) & 1) * 2 + c) : (sw >> 2);
          uint32_t v[32];
          const uint32_t taddr = tmem + lane_off + (uint32_t)(as * 128 + cq * 32);
          TMC_LD32(taddr, v);
          tmem_ld_wait();
          TMC_SMX_MARK(1);
          uint32_t hi[16], lo[16];
          if (hom > -INFINITY) {
            chunk_math(v, hom2, racc, hi, lo);
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) { hi[q] = 0u; lo[q] = 0u; }
          }
          TMC_SMX_MARK(2);
          TMC_ST16(taddr, hi);
          if constexpr (PLO) TMC_ST16(taddr + 16, lo);
        }
        __syncwarp();
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[as]);
        // Row-owner pass: does this streamed (column) tile carry fp16 weight?  P~ <= 2^-27 everywhere is
        // a factor 4 below the 2^-25 that rounds to a nonzero fp16, so the column-owner pass's
        // recomputed P~ of an unflagged tile are zero in both parts whatever its last-bit differences
        // in S.  NaN counts as weight (fmaxf drops NaN: test the row sums too).  One bit per tile in
        // a per-thread mask, published once per unit; tiles past 32 (K > 4096) publish at once.
        if constexpr (CF) {
          const float rs = (racc[0].x + racc[0].y) + (racc[1].x + racc[1].y);
          const bool wt = pmax > 0x1p-27f || rs != rs;
          if (j < 32) fmask |= (uint32_t)wt << j;
          else if (a.tflag && __any_sync(0xffffffffu, wt) && lane == 0) a.tflag[(size_t)b * a.t_tiles + j] = 1;
        }
        TMC_SMX_MARK(3);
        ++t;
      }
      if constexpr (CF) {
        if (a.tflag) {   // publish the unit's streamed-tile flags (idempotent stores of 1)
          const uint32_t m0 = __reduce_or_sync(0xffffffffu, fmask);
          if ((m0 >> lane) & 1u) a.tflag[(size_t)b * a.t_tiles + lane] = 1;
        }
      }
      // this warp's row sums -> the epilogue warps
      mbar_wait(&r_empty[ua & 1], ((ua >> 1) & 1) ^ 1);
      const float2 rr = __fadd2_rn(racc[0], racc[1]);
      sRs[(ua & 1) * 512 + (grp * 2 + slot) % 4 * 128 + m] = rr.x + rr.y;
      if (SG == 3) sRs[(ua & 1) * 512 + (slot + 1) * 128 + m] = 0.f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&r_full[ua & 1]);
      TMC_SMX_MARK(5);
      ++ua;
    }
#if defined(TMC_INSTRUMENT) && defined(TMC_SMX_PROF)
    if (lane == 0 && (sw == 0 || sw == 15))
      for (int q = 0; q < 6; ++q) atomicAdd(&g_tmc_prof[blockIdx.x & 1023][19 + q + (sw ? 6 : 0)], (unsigned long long)sprof[q]);
#endif
#undef TMC_SMX_MARK
    TMC_PROF_END(lane == 0, 48 + sw, _tr2);
  } else {
    // ---------------- epilogue warps (4, one per TMEM lane quarter): G -> gradients, off the
    // softmax warps' critical path (they already stream the next unit's tiles).
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t ua = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      TMC_BWD_UNIT();
      const int gm = mt * 128 + m;
      if (!olive(a, b, mt)) {
        // no owner row carries weight: every gradient of these rows is exactly 0
        if (gm < a.M) {
          const size_t row = ((size_t)b * a.M + gm) * D;
#pragma unroll 1
          for (int d = 0; d < D; d += 4) {
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (a.owner_z) { if (a.gz) *reinterpret_cast<float4*>(a.gz + row + d) = z4; }
            else {
              if (a.gmu) *reinterpret_cast<float4*>(a.gmu + row + d) = z4;
              if (a.glv) *reinterpret_cast<float4*>(a.glv + row + d) = z4;
            }
          }
          if (a.rowsum) a.rowsum[(size_t)b * a.M + gm] = 0.f;
        }
        continue;
      }
      // D <= 32: the rows this thread combines with G (z, or mu and logvar) are loaded into registers
      // before the row-sum and accumulator waits, so the epilogue pays no dependent global-load
      // latency per 8 features (C4 reverse -1.6%, C3 neutral; at D = 64 the 64 extra registers cost
      // more than the latency: C2 reverse +3%, so D = 64 keeps the per-8-feature loads).
      constexpr bool EPI_PRE = TMC_EPI_PREFETCH && D <= 32;
      const size_t prow = ((size_t)b * a.M + (gm < a.M ? gm : 0)) * D;
      const float* pA_ = a.owner_z ? a.z : a.mu;
      float4 pa[8], pb[8];
      if constexpr (EPI_PRE) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          pa[q] = *reinterpret_cast<const float4*>(pA_ + prow + 4 * q);
          pb[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (!a.owner_z) {
#pragma unroll
          for (int q = 0; q < 8; ++q) pb[q] = *reinterpret_cast<const float4*>(a.lv + prow + 4 * q);
        }
      }
      int nl = 0;
      if (a.t_tiles <= 64) {
        nl = __popcll(tmask(a, b) & (a.t_tiles == 64 ? ~0ull : ((1ull << a.t_tiles) - 1)));
      } else {
        for (int j = 0; j < a.t_tiles; ++j) nl += tlive(a, b, j) ? 1 : 0;
      }
      const uint32_t gb = ua % GB;
      mbar_wait(&r_full[ua & 1], (ua >> 1) & 1);
      const float* rs = sRs + (ua & 1) * 512;
      const float rtot = (rs[m] + rs[128 + m]) + (rs[256 + m] + rs[384 + m]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&r_empty[ua & 1]);
      TMC_PROF_WAIT(warp == SMW && lane == 0, 10, mbar_wait(&g_full[gb], (ua / GB) & 1));
      tc_fence_after();
      const float sc = a.sgn[b] * (1.f / 16384.f);
      // R6: an owned tile no P~ of which is nonzero in fp16 carries no weight; its sums are 0 (the
      // skipping pass never computes it, the dense pass computes exact-zero gradients for it)
      const bool oz = a.oflag && !a.oflag[(size_t)b * a.o_tiles + mt];
      const float pi = oz ? 0.f : rtot * sc;
      const bool live = gm < a.M;
      const float* sh = a.shift + (size_t)b * D;
      const size_t row = ((size_t)b * a.M + (live ? gm : 0)) * D;
      const uint32_t gaddr = tmem + lane_off + GCOL + gb * GN;
      if constexpr (EPI_PRE) {
      {
        constexpr int c0 = 0;
#pragma unroll
        for (int dd = 0; dd < 32; dd += 16) {
          const int d0 = c0 + dd;
          uint32_t r0[16], r1[16];
          TMC_LD16(gaddr + d0, r0);
          TMC_LD16(gaddr + D + d0, r1);
          if constexpr (PACKED) {     // + the T_lo column half
            uint32_t q0[16], q1[16];
            TMC_LD16(gaddr + 2 * D + d0, q0);
            TMC_LD16(gaddr + 3 * D + d0, q1);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              r0[e] = __float_as_uint(__uint_as_float(r0[e]) + __uint_as_float(q0[e]));
              r1[e] = __float_as_uint(__uint_as_float(r1[e]) + __uint_as_float(q1[e]));
            }
          }
          tmem_ld_wait();
          if (live) {
#pragma unroll
            for (int d4 = 0; d4 < 16; d4 += 4) {
              float g0[4], g1[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {   // no live streamed tile: the accumulator was never written
                g0[e] = nl ? __uint_as_float(r0[d4 + e]) : 0.f;
                g1[e] = nl ? __uint_as_float(r1[d4 + e]) : 0.f;
              }
              const float4 a4 = pa[(dd + d4) >> 2];
              const float av[4] = {a4.x, a4.y, a4.z, a4.w};
              if (a.owner_z) {
                // G = sum P (Y = [-lam/2, lam mu'] log2e): dz = sum P lam (mu' - z') = (G1 + 2 z' G0) / log2e
                if (a.gz) {
                  float o[4];
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float zp = av[e] - sh[d0 + d4 + e];
                    o[e] = (g1[e] + 2.f * zp * g0[e]) * (sc * kLn2);
                  }
                  *reinterpret_cast<float4*>(a.gz + row + d0 + d4) = make_float4(o[0], o[1], o[2], o[3]);
                }
              } else {
                // G = sum P (X = [z'^2, z']): A2 = sum P z'^2, A1 = sum P z'
                const float4 v4 = pb[(dd + d4) >> 2];
                const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
                float om[4], ov[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float mp = av[e] - sh[d0 + d4 + e];
                  const float lam = __expf(-vv[e]);
                  const float A1 = g1[e] * sc, A2 = g0[e] * sc;
                  om[e] = a.alpha * lam * (A1 - mp * pi);
                  ov[e] = a.alpha * 0.5f * (lam * (A2 - 2.f * mp * A1 + mp * mp * pi) - pi);
                }
                if (a.gmu) *reinterpret_cast<float4*>(a.gmu + row + d0 + d4) = make_float4(om[0], om[1], om[2], om[3]);
                if (a.glv) *reinterpret_cast<float4*>(a.glv + row + d0 + d4) = make_float4(ov[0], ov[1], ov[2], ov[3]);
              }
            }
          }
        }
      }
      } else {
#pragma unroll 1
      for (int d0 = 0; d0 < D; d0 += 8) {
        uint32_t r0[8], r1[8];
        TMC_LD8(gaddr + d0, r0);
        TMC_LD8(gaddr + D + d0, r1);
        if constexpr (PACKED) {     // + the T_lo column half
          uint32_t q0[8], q1[8];
          TMC_LD8(gaddr + 2 * D + d0, q0);
          TMC_LD8(gaddr + 3 * D + d0, q1);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            r0[e] = __float_as_uint(__uint_as_float(r0[e]) + __uint_as_float(q0[e]));
            r1[e] = __float_as_uint(__uint_as_float(r1[e]) + __uint_as_float(q1[e]));
          }
        }
        tmem_ld_wait();
        if (!live) continue;
        float g0[8], g1[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {   // no live streamed tile: the accumulator was never written
          g0[e] = nl ? __uint_as_float(r0[e]) : 0.f;
          g1[e] = nl ? __uint_as_float(r1[e]) : 0.f;
        }
        if (a.owner_z) {
          // G = sum P (Y = [-lam/2, lam mu'] log2e): dz = sum P lam (mu' - z') = (G1 + 2 z' G0) / log2e
          if (a.gz) {
#pragma unroll
            for (int d4 = 0; d4 < 8; d4 += 4) {
              const float4 z4 = *reinterpret_cast<const float4*>(a.z + row + d0 + d4);
              const float zz[4] = {z4.x, z4.y, z4.z, z4.w};
              float o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float zp = zz[e] - sh[d0 + d4 + e];
                o[e] = (g1[d4 + e] + 2.f * zp * g0[d4 + e]) * (sc * kLn2);
              }
              *reinterpret_cast<float4*>(a.gz + row + d0 + d4) = make_float4(o[0], o[1], o[2], o[3]);
            }
          }
        } else {
          // G = sum P (X = [z'^2, z']): A2 = sum P z'^2, A1 = sum P z'
#pragma unroll
          for (int d4 = 0; d4 < 8; d4 += 4) {
            const float4 m4 = *reinterpret_cast<const float4*>(a.mu + row + d0 + d4);
            const float4 v4 = *reinterpret_cast<const float4*>(a.lv + row + d0 + d4);
            const float mm[4] = {m4.x, m4.y, m4.z, m4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
            float om[4], ov[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float mp = mm[e] - sh[d0 + d4 + e];
              const float lam = __expf(-vv[e]);
              const float A1 = g1[d4 + e] * sc, A2 = g0[d4 + e] * sc;
              om[e] = a.alpha * lam * (A1 - mp * pi);
              ov[e] = a.alpha * 0.5f * (lam * (A2 - 2.f * mp * A1 + mp * mp * pi) - pi);
            }
            if (a.gmu) *reinterpret_cast<float4*>(a.gmu + row + d0 + d4) = make_float4(om[0], om[1], om[2], om[3]);
            if (a.glv) *reinterpret_cast<float4*>(a.glv + row + d0 + d4) = make_float4(ov[0], ov[1], ov[2], ov[3]);
          }
        }
      }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&g_empty[gb]);
      if (live && a.rowsum) a.rowsum[(size_t)b * a.M + gm] = pi;
      ++ua;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}
#undef TMC_BWD_UNIT

// Per-row terms of the reverse pass: rterm2[r] = log2(|w[r]|/ws) - (ell[r] - beta[r]) log2e (-inf when
// the row carries no weight) and sgn[b] = +-ws, where ws = 2^ceil(log2 max_r |w[r]|) keeps the fp16
// P~ <= 2^14 whatever the magnitude of dlogp, and the sign is that of the (uniformly signed, R2)
// upstream weights.
struct RowtermArgs {
  const float *ell, *w, *beta;   // [B][R], [B][R], [B][betaStride] (UP: beta of the row side) or NULL
  int betaStride, R, Rpad;
  float* rterm2;                 // [B][Rpad]
  uint8_t* bx;                   // [B][Rpad/128][kBxBytes]: rterm2 as the bias operand of the column-owner pass
  float* sgn;                    // [B]
  int* live;                     // [B][Rpad/128] 1 if any row of the 128-row tile carries weight
  int* cflag;                    // [B][ctiles] column-tile fp16-weight flags, zeroed here for the row-owner pass (or NULL)
  int ctiles;
};

struct RowtermBatch { RowtermArgs e[kMaxBatch]; int ne; };
#ifndef TMC_FLUSH_LOG2
#define TMC_FLUSH_LOG2 -41.f
#endif
constexpr float kFlushLog2 = TMC_FLUSH_LOG2;   // log2 of the row-weight flush threshold relative to the scale ws

__global__ void __launch_bounds__(256) tc_rowterm_kernel(const __grid_constant__ RowtermBatch rb_) {
  const RowtermArgs& a = rb_.e[blockIdx.y];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float red[8];
  __shared__ int neg;
  if (tid == 0) neg = 0;
  float wm = 0.f;
  for (int r = tid; r < a.R; r += 256) wm = fmaxf(wm, fabsf(a.w[(size_t)b * a.R + r]));
#pragma unroll
  for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
  if (lane == 0) red[warp] = wm;
  __syncthreads();
  wm = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) wm = fmaxf(wm, red[w]);
  // power-of-two scale (exact division); 1 when all weights are 0
  const float lw = (wm > 0.f) ? ceilf(__log2f(wm)) : 0.f;
  const float ws = exp2f(lw);
  for (int r = tid; r < a.Rpad; r += 256) {
    float v = -INFINITY;
    if (r < a.R) {
      const float e = a.ell[(size_t)b * a.R + r], w = a.w[(size_t)b * a.R + r];
      if (w < 0.f) neg = 1;
      // P~[r, n] = 2^14 |w[r]|/ws * (pair term / row total) <= 2^14 |w[r]|/ws (1 + rounding): a row
      // below 2^-41 of the scale has every P~ <= 2^-27, which rounds to zero in both fp16 parts, so
      // its gradient-GEMM contribution is exactly 0 already; flushing the row (kFlushLog2) also zeroes
      // its row sum (<= 2^-41 relative) and lets the zero-tile skip drop tiles that carry no fp16 weight.
      const float lr = (w != 0.f) ? __log2f(fabsf(w)) - lw : -INFINITY;
      if (e > -INFINITY && lr >= kFlushLog2) {
        const float bt = a.beta ? a.beta[(size_t)b * a.betaStride + r] : 0.f;
        v = lr - (e - bt) * kLog2E;
      }
    }
    a.rterm2[(size_t)b * a.Rpad + r] = v;
    if (a.bx) store_bias_row(a.bx + (size_t)b * (a.Rpad / kTileRows) * kBxBytes, r, v);
  }
  __syncthreads();
  if (tid == 0) a.sgn[b] = neg ? -ws : ws;
  tile_live_flags(a.rterm2 + (size_t)b * a.Rpad, a.Rpad / kTileRows, a.live + (size_t)b * (a.Rpad / kTileRows));
  if (a.cflag)
    for (int t = tid; t < a.ctiles; t += 256) a.cflag[(size_t)b * a.ctiles + t] = 0;
}

}  // namespace tc

// ================================================================================ host side
// The reverse pass's gradient GEMM uses the 3-term fp16 product (P_lo T_hi + P_hi T_lo + P_hi T_hi,
// DESIGN.md §6) and 8 wide softmax warps (SG = 3).  Zero-weight tile skipping is exact; the graph
// flag TMC_FLAG_DENSE_REVERSE disables it (every tile computed, for measurement).
#ifndef TMC_GRAD_TERMS
#define TMC_GRAD_TERMS 3
#endif
constexpr int kGradTerms = TMC_GRAD_TERMS;
constexpr int kBwdGroups = 3;

struct TcLatentBuf {
  bool ok = false;          // this latent's (non-root) edge runs on tensor cores
  int D = 0, KzPad = 0, KpPad = 0;
  size_t xt = 0, yt = 0, beta = 0, cb2 = 0, bx = 0, shift = 0, rterm2 = 0, rbx = 0, sgn = 0, rlive = 0, clive = 0, clive2 = 0;
  bool bwd_ok = false;      // reverse pass on tensor cores
};

inline bool tc_dim_ok(int D) { return D == 32 || D == 64; }

inline bool tc_supported(const std::vector<int>& parent, const std::vector<int>& K, const std::vector<int>& D) {
  bool any = false;
  for (size_t i = 0; i < parent.size(); ++i)
    if (parent[i] >= 0 && tc_dim_ok(D[i]) && K[i] >= 1) any = true;
  return any;
}

inline size_t tc_carve(size_t& cur, size_t bytes) {
  size_t at = (cur + 1023) & ~size_t(1023);
  cur = at + bytes;
  return at;
}

inline int pad256(int k) { return (k + 255) / 256 * 256; }

inline size_t tc_tile_bytes(int D) { return D == 32 ? tc::Geo<32>::TILE : tc::Geo<64>::TILE; }

inline void tc_plan(const std::vector<int>& parent, const std::vector<int>& K, const std::vector<int>& D,
                    const std::vector<int>& Kp, int B, int dir, size_t& cur, std::vector<TcLatentBuf>& bufs) {
  const size_t Bn = (size_t)(B > 0 ? B : 1);
  bufs.assign(parent.size(), TcLatentBuf{});
  for (size_t i = 0; i < parent.size(); ++i) {
    if (parent[i] < 0 || !tc_dim_ok(D[i])) continue;
    TcLatentBuf& t = bufs[i];
    t.ok = true;
    t.D = D[i];
    t.KzPad = pad256(K[i]);
    t.KpPad = pad256(Kp[i]);
    const size_t tb = tc_tile_bytes(D[i]);
    t.xt = tc_carve(cur, Bn * (t.KzPad / 128) * tb);
    t.yt = tc_carve(cur, Bn * (t.KpPad / 128) * tb);
    t.beta = tc_carve(cur, Bn * t.KpPad * 4);
    const int Cpad = (dir == TMC_DIR_DOWN) ? t.KpPad : t.KzPad;
    const int Rpad = (dir == TMC_DIR_DOWN) ? t.KzPad : t.KpPad;
    t.cb2 = tc_carve(cur, Bn * Cpad * 4);
    t.bx = tc_carve(cur, Bn * (Cpad / 128) * tc::kBxBytes);
    t.shift = tc_carve(cur, Bn * D[i] * 4);
    t.rterm2 = tc_carve(cur, Bn * Rpad * 4);
    t.rbx = tc_carve(cur, Bn * (Rpad / 128) * tc::kBxBytes);
    t.rlive = tc_carve(cur, Bn * (Rpad / 128) * 4);
    t.clive = tc_carve(cur, Bn * (Cpad / 128) * 4);
    t.clive2 = tc_carve(cur, Bn * (Cpad / 128) * 4);
    t.sgn = tc_carve(cur, Bn * 4);
    t.bwd_ok = true;
  }
}

inline bool tc_edge_ok(const TcLatentBuf& b) { return b.ok; }

template <int D>
inline void tc_prep_launch(const tc::PrepBatch& pb, int B, cudaStream_t s) {
  int chunks = 0;
  for (int k = 0; k < pb.ne; ++k) chunks = std::max(chunks, pb.e[k].KpPad / 256 + pb.e[k].KzPad / 256);
  tc::tc_shift_kernel<D><<<dim3(B, 1, pb.ne), 256, 0, s>>>(pb);
  tc::tc_prep_kernel<D><<<dim3(B, chunks, pb.ne), 256, 0, s>>>(pb);
}

// Operand prep of tensor-core edges (one launch pair for up to kMaxPrepBatch edges of equal D):
// X/Y tile images, beta and the centering shift.  wsrc/wlen/wz: the message weights each edge's
// shift is centred on (see tc_shift_kernel).
struct PrepJob {
  int Ki, Kpi, Di;
  const tmc_latent_in* in;
  const TcLatentBuf* t;
  const float* wsrc;
  int wlen, wz;
  float alpha;
};

inline int tc_prep_batch(const PrepJob* jobs, int ne, int B, void* ws, cudaStream_t s) {
  if (B == 0 || ne == 0) return 0;
  int launched = 0;
  for (int e0 = 0; e0 < ne; e0 += tc::kMaxPrepBatch) {
    tc::PrepBatch pb{};
    pb.ne = std::min(tc::kMaxPrepBatch, ne - e0);
    for (int k = 0; k < pb.ne; ++k) {
      const PrepJob& j = jobs[e0 + k];
      tc::PrepArgs& p = pb.e[k];
      p.z = j.in->z; p.mu = j.in->mu; p.lv = j.in->logvar;
      p.Kz = j.Ki; p.Kp = j.Kpi; p.KzPad = j.t->KzPad; p.KpPad = j.t->KpPad;
      p.Xt = static_cast<uint8_t*>(ws) + j.t->xt;
      p.Yt = static_cast<uint8_t*>(ws) + j.t->yt;
      p.beta = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + j.t->beta);
      p.shift = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + j.t->shift);
      p.wsrc = j.wsrc; p.wlen = j.wlen; p.wz = j.wz;
      p.alpha = j.alpha;
    }
    ProfScope ps(PF_TC_PREP, s);
    if (jobs[e0].Di == 32) tc_prep_launch<32>(pb, B, s);
    else tc_prep_launch<64>(pb, B, s);
    launched += 2;   // shift + image kernels
  }
  return launched;
}

inline int tc_prep_edge(int Ki, int Kpi, int Di, int B, const tmc_latent_in& in, void* ws, const TcLatentBuf& t,
                        const float* wsrc, int wlen, int wz, float alpha, cudaStream_t s) {
  if (!t.ok) return 0;
  PrepJob j{Ki, Kpi, Di, &in, &t, wsrc, wlen, wz, alpha};
  return tc_prep_batch(&j, 1, B, ws, s);
}

template <int D>
inline void tc_fwd_launch(const tc::FwdBatch& fb, cudaStream_t s) {
  using G = tc::Geo<D>;
  static bool attr[kMaxDevices] = {};
  ensure_smem_attr(tc::tc_fwd_kernel<D>, (int)G::SMEM, attr);
  const int sms = sm_count();
  const int units = fb.ustart[fb.ne];
  const int grid = units < sms ? units : sms;
  if (grid > 0) tc::tc_fwd_kernel<D><<<grid, G::THREADS, G::SMEM, s>>>(fb);
}

// Forward contraction of ne edges (same D) on tensor cores: per-edge column bias, then ONE persistent
// launch over the units of every edge (siblings of a tree level run together).  zrows = DOWN (rows =
// z side).  Returns the number of kernels launched.
inline int tc_pass_forward_batch(const PassArgs* as, const TcLatentBuf* const* ts, int ne, void* ws, bool zrows,
                                 cudaStream_t s) {
  uint8_t* w = static_cast<uint8_t*>(ws);
  int launched = 0;
  for (int e0 = 0; e0 < ne; e0 += tc::kMaxBatch) {
    tc::FwdBatch fb{};
    tc::ColbiasBatch cb{};
    fb.ne = std::min(tc::kMaxBatch, ne - e0);
    cb.ne = fb.ne;
    fb.ustart[0] = 0;
    for (int k = 0; k < fb.ne; ++k) {
      const PassArgs& a = as[e0 + k];
      const TcLatentBuf& t = *ts[e0 + k];
      const int Cpad = zrows ? t.KpPad : t.KzPad;
      tc::ColbiasArgs& cbA = cb.e[k];
      cbA.cb = a.cb;
      cbA.beta = zrows ? reinterpret_cast<const float*>(w + t.beta) : nullptr;
      cbA.betaStride = t.KpPad;
      cbA.C = a.C; cbA.Cpad = Cpad;
      cbA.cb2 = reinterpret_cast<float*>(w + t.cb2);
      cbA.bx = w + t.bx;
      cbA.live = reinterpret_cast<int*>(w + t.clive);
      cbA.cbmax = a.cbmax;
      cbA.off_cb = a.off_cb; cbA.off_rb = a.off_rb; cbA.off_out = a.off_out;
      tc::FwdArgs& f = fb.e[k];
      f.At = zrows ? w + t.xt : w + t.yt;
      f.Bt = zrows ? w + t.yt : w + t.xt;
      f.a_tiles = (zrows ? t.KzPad : t.KpPad) / 128;
      f.b_tiles = Cpad / 128;
      f.cb2 = cbA.cb2;
      f.Bx = cbA.bx;
      f.ell_add = zrows ? nullptr : reinterpret_cast<const float*>(w + t.beta);
      f.ell_stride = t.KpPad;
      f.out_add = a.rb;
      f.R = a.R; f.B = a.B; f.lnC = a.lnC;
      f.out = a.out; f.ell = a.ell;
      const int rb = (t.D == 32) ? tc::Geo<32>::RB : tc::Geo<64>::RB;
      fb.ustart[k + 1] = fb.ustart[k] + a.B * (f.a_tiles / rb);
    }
    {
      ProfScope ps(PF_TC_PREP, s);
      tc::tc_colbias_kernel<<<dim3(as[e0].B, cb.ne), 256, 0, s>>>(cb);
    }
    fb.count = prof_on() ? 1 : 0;
    fb.flops_per_tile = (unsigned long long)(12 * ts[e0]->D + 32) * 128 * 128;   // 3-term S (K = 2D) + bias MMA (K = 16)
    ProfScope ps(PF_TC_FWD, s);
    if (ts[e0]->D == 32) tc_fwd_launch<32>(fb, s);
    else tc_fwd_launch<64>(fb, s);
    launched += 2;
  }
  return launched;
}

inline int tc_pass_forward(const PassArgs& a, const TcLatentBuf& t, void* ws, bool zrows, cudaStream_t s) {
  const TcLatentBuf* tp = &t;
  return tc_pass_forward_batch(&a, &tp, 1, ws, zrows, s);
}

template <int D, int GT, int SG, bool CF>
inline void tc_bwd_launch_t(const tc::BwdBatch& fb, cudaStream_t s) {
  using G = tc::BGeo<D>;
  static bool attr[kMaxDevices] = {};
  ensure_smem_attr(tc::tc_bwd_kernel<D, GT, SG, CF>, (int)G::SMEM, attr);
  const int sms = sm_count();
  const int units = fb.ustart[fb.ne];
  const int grid = units < sms ? units : sms;
  if (grid > 0) tc::tc_bwd_kernel<D, GT, SG, CF><<<grid, tc::bwd_threads<D, SG>(), G::SMEM, s>>>(fb);
}

template <int D>
inline void tc_bwd_launch(const tc::BwdBatch& fb, bool colflags, cudaStream_t s) {
  if (colflags) tc_bwd_launch_t<D, kGradTerms, kBwdGroups, true>(fb, s);
  else tc_bwd_launch_t<D, kGradTerms, kBwdGroups, false>(fb, s);
}

constexpr int kColFlagMaxTiles = 8;   // column-tile weight flags (R6) for edges with K_column <= 1024

inline bool tc_bwd_edge_ok(const TcLatentBuf& t, const PassArgs& a) { return t.ok && t.bwd_ok && !a.pair; }

// Reverse pass of ne edges (same D) on tensor cores: row-owner pass (mode 1) or column-owner pass
// (mode 2), ONE persistent launch over every edge's units.  The row terms are prepared per edge
// before the row-owner pass.  Returns kernels launched.
inline int tc_pass_backward_batch(const PassArgs* as, const TcLatentBuf* const* ts, int ne, void* ws, bool zrows,
                                  int mode, bool dense_reverse, cudaStream_t s) {
  uint8_t* w = static_cast<uint8_t*>(ws);
  int launched = 0;
  for (int e0 = 0; e0 < ne; e0 += tc::kMaxBatch) {
    tc::BwdBatch fb{};
    tc::RowtermBatch rtb{};
    fb.ne = std::min(tc::kMaxBatch, ne - e0);
    // Column-tile weight flags (reading R6) for batches whose edges have at most kColFlagMaxTiles
    // column tiles: recording them costs the row-owner pass ~2% where it is tensor-bound (K = 2048,
    // where it also found nothing more to skip) and nothing where the per-unit latency binds.
    bool colflags = true;
    for (int k = 0; k < fb.ne; ++k) {
      const TcLatentBuf& t = *ts[e0 + k];
      if ((zrows ? t.KpPad : t.KzPad) / 128 > kColFlagMaxTiles) colflags = false;
    }
    rtb.ne = fb.ne;
    fb.ustart[0] = 0;
    for (int k = 0; k < fb.ne; ++k) {
      const PassArgs& a = as[e0 + k];
      const TcLatentBuf& t = *ts[e0 + k];
      const int Rpad = zrows ? t.KzPad : t.KpPad, Cpad = zrows ? t.KpPad : t.KzPad;
      float* rterm2 = reinterpret_cast<float*>(w + t.rterm2);
      float* sgn = reinterpret_cast<float*>(w + t.sgn);
      if (mode == 1) {
        tc::RowtermArgs& r = rtb.e[k];
        r.ell = a.ell; r.w = a.w;
        r.beta = zrows ? nullptr : reinterpret_cast<const float*>(w + t.beta);
        r.betaStride = t.KpPad; r.R = a.R; r.Rpad = Rpad;
        r.rterm2 = rterm2; r.sgn = sgn;
        r.bx = w + t.rbx;
        r.live = reinterpret_cast<int*>(w + t.rlive);
        r.cflag = reinterpret_cast<int*>(w + t.clive2);
        r.ctiles = Cpad / 128;
      }
      tc::BwdArgs& f = fb.e[k];
      const bool own_rows = (mode == 1);
      const uint8_t* rowT = zrows ? w + t.xt : w + t.yt;
      const uint8_t* colT = zrows ? w + t.yt : w + t.xt;
      f.Ot = own_rows ? rowT : colT;
      f.Tt = own_rows ? colT : rowT;
      f.o_tiles = (own_rows ? Rpad : Cpad) / 128;
      f.t_tiles = (own_rows ? Cpad : Rpad) / 128;
      f.ho = own_rows ? rterm2 : reinterpret_cast<const float*>(w + t.cb2);
      f.ht = own_rows ? reinterpret_cast<const float*>(w + t.cb2) : rterm2;
      // the same streamed term as bias-operand tiles: the forward's column-bias tiles (row-owner
      // pass) or the row-term tiles written by tc_rowterm_kernel (column-owner pass)
      f.Hx = own_rows ? w + t.bx : w + t.rbx;
      f.sgn = sgn;
      f.M = own_rows ? a.R : a.C;
      f.B = a.B;
      const bool owner_is_z = (own_rows == zrows);
      f.owner_z = owner_is_z ? 1 : 0;
      f.z = a.z; f.mu = a.mu; f.lv = a.lv;
      f.shift = reinterpret_cast<const float*>(w + t.shift);
      f.gz = a.gz; f.gmu = a.gmu; f.glv = a.glv;
      f.rowsum = own_rows ? nullptr : a.colsum;
      // Column tiles: the exact flags of the forward (a message of -inf) for the row-owner pass, which
      // records the tiles that carry fp16 weight (clive2); the column-owner pass owns only those.
      int* cl2 = reinterpret_cast<int*>(w + t.clive2);
      f.tflag = (own_rows && colflags) ? cl2 : nullptr;
      f.oflag = (!own_rows && colflags) ? cl2 : nullptr;
      if (!dense_reverse) {
        const int* rl = reinterpret_cast<const int*>(w + t.rlive);
        const int* cl = reinterpret_cast<const int*>(w + t.clive);
        f.olive = own_rows ? rl : (colflags ? cl2 : cl);
        f.tlive = own_rows ? cl : rl;
      }
      f.alpha = a.alpha;
      fb.ustart[k + 1] = fb.ustart[k] + a.B * f.o_tiles;
    }
    if (mode == 1) {
      ProfScope ps(PF_TC_PREP, s);
      tc::tc_rowterm_kernel<<<dim3(as[e0].B, rtb.ne), 256, 0, s>>>(rtb);
      ++launched;
    }
    fb.count = prof_on() ? 1 : 0;
    // per live tile of one owner pass: S recompute (3 terms x K = 2D) + bias MMA (K = 16) + the 3-term
    // gradient GEMM (K = 128 streamed rows, N = 2D): (12 D + 32 + 12 D) flops per pair
    fb.flops_per_tile = (unsigned long long)((12 + 4 * (kGradTerms > 3 ? 2 : kGradTerms)) * ts[e0]->D + 32) * 128 * 128;
    ProfScope ps(PF_TC_BWD, s);
    if (ts[e0]->D == 32) tc_bwd_launch<32>(fb, mode == 1 && colflags, s);
    else tc_bwd_launch<64>(fb, mode == 1 && colflags, s);
    ++launched;
  }
  return launched;
}

inline int tc_pass_backward(const PassArgs& a, const TcLatentBuf& t, void* ws, bool zrows, int mode,
                            bool dense_reverse, cudaStream_t s) {
  const TcLatentBuf* tp = &t;
  return tc_pass_backward_batch(&a, &tp, 1, ws, zrows, mode, dense_reverse, s);
}

// ------------------------------------------------------------------------------ K2: tmc_factors on tensor cores
namespace tc {
// Materialised pairwise log-factor of one latent:
//   logf[b][a][c] = log N(z_a; mu_c, diag e^{v_c}) - logq[a] = S[a,c] + beta[c] - logq[a],
//   S = X.Y^T (X = [z'^2, z'], Y = [-lam/2, lam mu'], z' = z - s, mu' = mu - s), 3-term fp16 split,
//   beta[c] = -1/2 sum_d (lam mu'^2 + v + ln 2 pi)  ("norm + log-det" in the epilogue).
// No workspace: the CTA builds its operand images in shared memory from the fp32 inputs.  Persistent;
// unit = (datapoint, 128-row tile of z).  8 convert/epilogue warps (TMEM lane quarter x column half)
// build the X image once per unit and the Y image + beta of every column tile (double buffered),
// the MMA warp runs the 3-term product into double-buffered TMEM accumulators, and the same warps
// drain S, add the norm/log-det/-logq terms and store logf rows (HBM-write bound: 4 B per pair).
// The shift s (any s is exact algebra) is the mean of mu over the unit's first column tile.
struct FacArgs {
  const float *z, *mu, *lv, *logq;
  float* logf;
  int B, Kz, Kp;
};

template <int D>
struct FGeo {
  static constexpr int TILE = Geo<D>::TILE, PART = Geo<D>::PART, ATOMS = Geo<D>::ATOMS;
  static constexpr int CW = 8;                         // convert / epilogue warps
  static constexpr int THREADS = 32 * (CW + 1);        // + MMA warp
  static constexpr size_t SMEM = 1024 + 3 * (size_t)TILE + 4 * 128 * 4 + 128 * 4 + 64 * 4 + 256;
};

template <int D>
__global__ void __launch_bounds__(FGeo<D>::THREADS, 1) tc_factors_kernel(const FacArgs a) {
  using G = FGeo<D>;
  constexpr int CW = G::CW, W_MMA = CW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;                                            // X image (hi, lo)
  uint8_t* sY = sX + G::TILE;                                    // 2 Y images
  // beta ring of 4: a warp can be building Y(ct) while a slower warp still reads beta of ct-3
  float* sBeta = reinterpret_cast<float*>(sY + 2 * (size_t)G::TILE);   // [4][128]
  float* sLq = sBeta + 512;                                      // [128] logq of the unit's rows
  float* sSh = sLq + 128;                                        // [64] shift
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSh + 64);
  uint64_t* y_full = bars;        // [2] Y image + beta ready (CW warps)
  uint64_t* y_empty = bars + 2;   // [2] MMA done reading it
  uint64_t* acc_full = bars + 4;  // [2]
  uint64_t* acc_empty = bars + 6; // [2] (CW warps)
  uint64_t* x_full = bars + 8;    // X image ready (CW warps)
  uint64_t* x_empty = bars + 9;   // MMA done with the unit's X image
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rtiles = (a.Kz + 127) / 128, ctiles = (a.Kp + 127) / 128;
  const int units = a.B * rtiles;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&y_full[i], CW); mbar_init(&y_empty[i], 1);
      mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], CW);
    }
    mbar_init(x_full, CW); mbar_init(x_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == W_MMA) {
    uint32_t t = 0, ua = 0;
    const uint32_t xBase = smem_u32(sX), yBase = smem_u32(sY);
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++ua) {
      mbar_wait(x_full, ua & 1);
      for (int ct = 0; ct < ctiles; ++ct, ++t) {
        const uint32_t buf = t & 1, ph = (t >> 1) & 1;
        mbar_wait(&y_full[buf], ph);
        mbar_wait(&acc_empty[buf], ph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * 128;
        const uint64_t dX = sdesc(xBase), dY = sdesc(yBase + buf * G::TILE);
#pragma unroll
        for (int at = 0; at < G::ATOMS; ++at) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t o = at * kAtomBytes + kk * 32;
            mma_f16(d, dadd(dX, o), dadd(dY, G::PART + o), kIdescF16M128N128, (at | kk) ? 1u : 0u);
            mma_f16(d, dadd(dX, G::PART + o), dadd(dY, o), kIdescF16M128N128, 1u);
          }
        }
#pragma unroll
        for (int at = 0; at < G::ATOMS; ++at) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t o = at * kAtomBytes + kk * 32;
            mma_f16(d, dadd(dX, o), dadd(dY, o), kIdescF16M128N128, 1u);
          }
        }
        mma_commit(&y_empty[buf]);
        mma_commit(&acc_full[buf]);
      }
      mma_commit(x_empty);
    }
  } else {
    // ---------------- convert / epilogue warps
    const int quarter = warp & 3, half = warp >> 2;
    const int m = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    constexpr int CPR = D / 4, HC = D / 8, RPI = 256 / CPR;   // 8-feature chunks per image row
    const int j = tid % CPR, rsub = tid / CPR;
    const int dj = (j < HC ? j : j - HC) * 8;
    uint32_t t = 0, ua = 0;
    auto store16 = [&](uint8_t* img, int r, const float* vals) {
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        __half2 h = __floats2half2_rn(vals[2 * q], vals[2 * q + 1]);
        const float2 hf = __half22float2(h);
        __half2 l = __floats2half2_rn(vals[2 * q] - hf.x, vals[2 * q + 1] - hf.y);
        hi[q] = *reinterpret_cast<uint32_t*>(&h);
        lo[q] = *reinterpret_cast<uint32_t*>(&l);
      }
      const uint32_t off = swz_off(r, j * 8);
      *reinterpret_cast<uint4*>(img + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(img + G::PART + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    };
    auto build_y = [&](int b, int ct, uint32_t buf, uint32_t bb) {
      const float* mub = a.mu + (size_t)b * a.Kp * D;
      const float* lvb = a.lv + (size_t)b * a.Kp * D;
      uint8_t* img = sY + buf * G::TILE;
      for (int r0 = 0; r0 < 128; r0 += RPI) {
        const int r = r0 + rsub, c = ct * 128 + r;
        float y[8];
        float bsum = 0.f;
        if (c < a.Kp) {
          const float4* lv4 = reinterpret_cast<const float4*>(lvb + (size_t)c * D + dj);
          const float4* mu4 = reinterpret_cast<const float4*>(mub + (size_t)c * D + dj);
          const float4 va = lv4[0], vb = lv4[1], ma = mu4[0], mb = mu4[1];
          const float vv[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
          const float mm[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float lam = __expf(-vv[e]);
            const float mp = mm[e] - sSh[dj + e];
            if (j < HC) {
              y[e] = -0.5f * lam;
              bsum += lam * mp * mp + vv[e] + kLog2Pi;
            } else {
              y[e] = lam * mp;
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) y[e] = 0.f;
        }
        store16(img, r, y);
#pragma unroll
        for (int o = CPR / 2; o; o >>= 1) bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
        if (j == 0) sBeta[bb * 128 + r] = -0.5f * bsum;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&y_full[buf]);
    };
    auto epilogue = [&](int b, int rt, int ct, uint32_t buf, uint32_t ph, uint32_t bb) {
      mbar_wait(&acc_full[buf], ph);
      tc_fence_after();
      uint32_t v[64];
      const uint32_t taddr = tmem + lane_off + buf * 128 + half * 64;
      TMC_LD32(taddr, v);
      TMC_LD32(taddr + 32, (v + 32));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      const int arow = rt * 128 + m;
      if (arow < a.Kz) {
        const float lq = sLq[m];
        const float* bt = sBeta + bb * 128 + half * 64;
        const int c0 = ct * 128 + half * 64;
        float* dst = a.logf + ((size_t)b * a.Kz + arow) * a.Kp + c0;
        const int nc = min(64, a.Kp - c0);
        if (nc == 64 && (a.Kp & 3) == 0) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            *reinterpret_cast<float4*>(dst + 4 * q) =
                make_float4(__uint_as_float(v[4 * q]) + bt[4 * q] - lq, __uint_as_float(v[4 * q + 1]) + bt[4 * q + 1] - lq,
                            __uint_as_float(v[4 * q + 2]) + bt[4 * q + 2] - lq, __uint_as_float(v[4 * q + 3]) + bt[4 * q + 3] - lq);
        } else {
#pragma unroll
          for (int q = 0; q < 64; ++q)
            if (q < nc) dst[q] = __uint_as_float(v[q]) + bt[q] - lq;
        }
      }
    };
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++ua) {
      const int b = u / rtiles, rt = u % rtiles;
      // all CW warps must be done with the previous unit's shift / X image / logq before rewriting
      named_bar(1, 32 * CW);
      // shift: mean of mu over the first column tile
      if (tid < D) {
        const float* mub = a.mu + (size_t)b * a.Kp * D;
        const int n = min(128, a.Kp);
        float acc = 0.f;
        for (int c = 0; c < n; ++c) acc += mub[(size_t)c * D + tid];
        sSh[tid] = acc / (float)n;
      }
      if (tid < 128) {
        const int arow = rt * 128 + tid;
        sLq[tid] = arow < a.Kz ? a.logq[(size_t)b * a.Kz + arow] : 0.f;
      }
      named_bar(1, 32 * CW);
      // X image of the unit (after the MMA has finished with the previous one)
      mbar_wait(x_empty, (ua & 1) ^ 1);
      {
        const float* zb = a.z + (size_t)b * a.Kz * D;
        for (int r0 = 0; r0 < 128; r0 += RPI) {
          const int r = r0 + rsub, arow = rt * 128 + r;
          float x[8];
          if (arow < a.Kz) {
            const float4* z4 = reinterpret_cast<const float4*>(zb + (size_t)arow * D + dj);
            const float4 za = z4[0], zc = z4[1];
            const float zz[8] = {za.x, za.y, za.z, za.w, zc.x, zc.y, zc.z, zc.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float zp = zz[e] - sSh[dj + e];
              x[e] = (j < HC) ? zp * zp : zp;
            }
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = 0.f;
          }
          store16(sX, r, x);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(x_full);
      }
      // column tiles: build Y(ct) (double buffered), then drain S(ct-1)
      for (int ct = 0; ct < ctiles; ++ct) {
        const uint32_t tt = t + ct, buf = tt & 1, ph = (tt >> 1) & 1;
        mbar_wait(&y_empty[buf], ph ^ 1);
        build_y(b, ct, buf, tt & 3);
        if (ct > 0) epilogue(b, rt, ct - 1, (tt - 1) & 1, ((tt - 1) >> 1) & 1, (tt - 1) & 3);
      }
      {
        const uint32_t tt = t + ctiles - 1;
        epilogue(b, rt, ctiles - 1, tt & 1, (tt >> 1) & 1, tt & 3);
      }
      t += ctiles;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}
}  // namespace tc

inline bool tc_factors_ok(int Ki, int Kp, int D) { return (D == 32 || D == 64) && Ki >= 1 && Kp >= 1; }

template <int D>
inline void tc_factors_launch(const tc::FacArgs& f, cudaStream_t s) {
  using G = tc::FGeo<D>;
  static bool attr[kMaxDevices] = {};
  ensure_smem_attr(tc::tc_factors_kernel<D>, (int)G::SMEM, attr);
  const int sms = sm_count();
  const int units = f.B * ((f.Kz + 127) / 128);
  const int grid = units < sms ? units : sms;
  tc::tc_factors_kernel<D><<<grid, G::THREADS, G::SMEM, s>>>(f);
}

inline tmc_status tc_factors(const tmc_latent_in* in, float* logf, int B, int Ki, int Kp, int D, cudaStream_t s) {
  tc::FacArgs f{};
  f.z = in->z; f.mu = in->mu; f.lv = in->logvar; f.logq = in->logq; f.logf = logf;
  f.B = B; f.Kz = Ki; f.Kp = Kp;
  if (D == 32) tc_factors_launch<32>(f, s);
  else tc_factors_launch<64>(f, s);
  return TMC_OK;
}

}  // namespace tmc
