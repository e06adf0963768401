// Single-pass reverse contraction of one edge on tensor cores (K4', D = 32), sm_100a.
//
// The reverse pass needs, for every pair (a, c) of an edge, the pair weight
//   P[a,c] = w_a exp(logf[a,c] + bias - ell_a)            (= dJ/dlogf)
// and three contractions: S = X Y^T (recomputed), G_row = P Y (-> dz) and G_col = P^T X (-> dmu, dv).
// The two-owner-pass kernel (tc_bwd_kernel) recomputes S and P in each orientation.  Here every
// S tile and every P~ tile is computed ONCE: the CTA owns a whole (edge, datapoint) and sweeps the
// column tiles in pairs (outer) and the row tiles (inner):
//   * S(i,j) = X_i Y_j^T + column term (bias MMA), 3-term fp16 split, fp32 in TMEM (2 buffers);
//   * 8 softmax warps: P~ = ex2(S + row term + 14) (MUFU), split to fp16 hi/lo, stored back into the
//     S buffer (A operand of G_row, A-from-TMEM MMA) AND as an MN-major SWIZZLE_128B shared-memory
//     image (A operand of G_col: P~^T without a transpose);
//   * G_col(j) += P~^T X_i accumulates over the row tiles in TMEM (N = 80: the 64 features of X plus
//     16 columns of ones at the descriptor's LBO, so the column sums sum_a P~ come out of the same
//     MMA); drained once per column-tile pair into dmu, dlogvar and the column sums;
//   * G_row(i) = P~ Y_j over the pair's two column tiles, drained once per (row tile, pair) by 4
//     epilogue warps into dz as an fp32 read-add-write of the row's 32 floats, in a fixed column
//     order (deterministic, no atomics) — plus the row sums when the edge needs them (UP trees).
// Rows are always the z side (X tiles) and columns the parameter side (Y tiles), whatever the
// direction of the forward pass: the row and column terms and the live flags are swapped by the
// host for UP trees.  Tiles whose pair weights are all exactly zero are skipped (exact).
#pragma once
#include "tmc_tc.cuh"

namespace tmc {
namespace tc {

struct Bwd1Args {
  const uint8_t *Xt, *Yt;      // row (z) / column (parameter) tile images [B][tiles][TILE]
  int r_tiles, c_tiles;        // 128-row tiles per datapoint (c_tiles even, both <= 64)
  const float* rterm;          // [B][r_tiles*128] row log2 term (-inf padded), added by the softmax warps
  const uint8_t* Cx;           // [B][c_tiles][kBxBytes] column log2 term as the bias-MMA operand
  const float* sgn;            // [B] signed scale of the upstream weights
  float alpha;                 // factor power (parameter-side gradients)
  int Mr, Mc;                  // valid rows (z samples) / columns (parameter rows)
  const float *z, *mu, *lv, *shift;   // z [B][Mr][32]; mu, lv [B][Mc][32]; shift [B][32]
  float *gz, *gmu, *glv;       // gradient outputs (any may be NULL)
  float* rowsum;               // [B][Mr] sum_c P (UP: the child's weights) or NULL
  float* colsum;               // [B][Mc] sum_a P (DOWN: the parent edge's weights) or NULL
  const int *rlive, *clive;    // [B][r_tiles], [B][c_tiles]: 0 = every weight of the tile is exactly 0
};

struct Bwd1Batch {
  Bwd1Args e[kMaxBatch];
  int ustart[kMaxBatch + 1];   // unit = (edge, datapoint)
  int ne;
  int count;                   // launch profiler on: add issued MMA flops to g_tmc_mma_flops
  unsigned long long flops_per_tile;
};

struct B1Geo {
  static constexpr int D = 32;
  static constexpr int TILE = Geo<32>::TILE;       // 32 KB: hi part then lo part, one 16 KB atom each
  static constexpr int PART = Geo<32>::PART;
  static constexpr int SMW = 8;                    // softmax warps (lane quarter x 64-column half)
  static constexpr int EW = 4;                     // epilogue warps
  static constexpr int W_PROD = SMW + EW, W_MMA = SMW + EW + 1;
  static constexpr int THREADS = 32 * (SMW + EW + 2);
  static constexpr int PIMG = 2 * 16384;           // one part (hi or lo) of the P~ image: 2 M-chunks of 64 columns
  // TMEM columns: S/P~ buffers 0, 128; G_col accumulators 256, 336 (N = 80); G_row 416 (N = 64)
  static constexpr uint32_t GCOL = 256, GCN = 80, GROW = 416;
  static constexpr size_t SMEM = 1024 /*align*/ + 2 * (size_t)TILE /*X ring*/ + 2 * (size_t)TILE /*Y pair*/ +
                                 2 * (size_t)PIMG /*P~ hi + lo*/ + 2 * kBxBytes /*column-term pair*/ +
                                 kBxBytes /*ones (bias MMA A)*/ + 2048 /*ones (column sums)*/ +
                                 2 * 2 * 128 * 4 /*row-sum handoff*/ + 128 /*shift*/ + 512 /*barriers*/;
};

template <int GN>
__host__ __device__ constexpr uint32_t idesc_f16(bool a_mn, bool b_mn) {
  return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(GN >> 3) << 17) |
         ((128u >> 4) << 24);
}

__global__ void __launch_bounds__(B1Geo::THREADS, 1) tc_bwd1_kernel(const __grid_constant__ Bwd1Batch fb) {
  using G = B1Geo;
  constexpr int D = G::D, SMW = G::SMW, EW = G::EW;
  constexpr uint32_t IDESC_S = kIdescF16M128N128;
  constexpr uint32_t IDESC_GR = idesc_f16<64>(false, true);    // TS: A = P~ (TMEM), B = Y MN-major
  constexpr uint32_t IDESC_GC80 = idesc_f16<80>(true, true);   // SS: A = P~^T image, B = [X_hi | ones]
  constexpr uint32_t IDESC_GC64 = idesc_f16<64>(true, true);   // SS: A = P~^T image, B = X_lo
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;                                   // [2] row-tile images
  uint8_t* sY = sX + 2 * (size_t)G::TILE;               // [2] the pair's column-tile images
  uint8_t* sP = sY + 2 * (size_t)G::TILE;               // P~ image: hi (2 chunks x 16 KB) then lo
  uint8_t* sCx = sP + 2 * (size_t)G::PIMG;              // [2] column-term bias operands
  uint8_t* sOnesB = sCx + 2 * kBxBytes;                 // constant A operand of the bias MMA
  uint8_t* sOnesC = sOnesB + kBxBytes;                  // 2 KB of fp16 ones (column sums), 1024-aligned
  float* sRs = reinterpret_cast<float*>(sOnesC + 2048); // [2 (visit parity)][2 (column half)][128]
  float* sSh = sRs + 512;                               // [32] centering shift of the unit's datapoint
  uint64_t* bars = reinterpret_cast<uint64_t*>(sSh + 32);
  uint64_t* x_full = bars + 0;      // [2]
  uint64_t* x_empty = bars + 2;     // [2]
  uint64_t* y_full = bars + 4;
  uint64_t* y_empty = bars + 5;
  uint64_t* s_full = bars + 6;      // [2]
  uint64_t* p_full = bars + 8;      // [2]  P~ of the tile written (TMEM + shared image)
  uint64_t* pimg_empty = bars + 10; //      the shared P~ image consumed by G_col
  uint64_t* grow_full = bars + 11;
  uint64_t* grow_empty = bars + 12;
  uint64_t* gcol_full = bars + 13;  // [2]
  uint64_t* gcol_empty = bars + 15; // [2]
  uint64_t* r_full = bars + 17;     // [2]
  uint64_t* r_empty = bars + 19;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 21);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int units = fb.ustart[fb.ne];
  // live-tile masks of a datapoint (<= 64 tiles per side), loaded by a whole warp
  auto mask64 = [&](const int* flags, int n, int b) -> uint64_t {
    if (!flags) return n >= 64 ? ~0ull : ((1ull << n) - 1);
    const int f0 = lane < n ? flags[(size_t)b * n + lane] : 0;
    const int f1 = lane + 32 < n ? flags[(size_t)b * n + lane + 32] : 0;
    return (uint64_t)__ballot_sync(0xffffffffu, f0) | ((uint64_t)__ballot_sync(0xffffffffu, f1) << 32);
  };
#define TMC_BWD1_UNIT()                                                    \
  const int e_ = batch_edge(fb, u);                                        \
  const Bwd1Args& a = fb.e[e_];                                            \
  const int b = u - fb.ustart[e_];                                         \
  const uint64_t rmask = mask64(a.rlive, a.r_tiles, b);                    \
  const uint64_t cmask = mask64(a.clive, a.c_tiles, b);                    \
  const int npairs = a.c_tiles / 2
  auto pair_bits = [](uint64_t cmask, int p) -> uint32_t { return (uint32_t)(cmask >> (2 * p)) & 3u; };

  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&x_full[s], 1); mbar_init(&x_empty[s], 1);
      mbar_init(&s_full[s], 1); mbar_init(&p_full[s], SMW);
      mbar_init(&gcol_full[s], 1); mbar_init(&gcol_empty[s], EW);
      mbar_init(&r_full[s], SMW); mbar_init(&r_empty[s], EW);
    }
    mbar_init(y_full, 1); mbar_init(y_empty, 1);
    mbar_init(pimg_empty, 1);
    mbar_init(grow_full, 1); mbar_init(grow_empty, EW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int r = tid; r < kTileRows; r += blockDim.x) {
    *reinterpret_cast<uint4*>(sOnesB + bx_off(r, 0)) = make_uint4(0x3C003C00u, 0x3C003C00u, 0x3C003C00u, 0x3C003C00u);
    *reinterpret_cast<uint4*>(sOnesB + bx_off(r, 8)) = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int q = tid; q < 2048 / 16; q += blockDim.x)
    reinterpret_cast<uint4*>(sOnesC)[q] = make_uint4(0x3C003C00u, 0x3C003C00u, 0x3C003C00u, 0x3C003C00u);
  fence_proxy_async();
  if (warp == G::W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  TMC_PROF_T0(_tot);
  if (warp == G::W_PROD) {
    // ---------------- producer: the pair's Y tiles + column-term operands, then the row tiles
    uint32_t v = 0, pa = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      TMC_BWD1_UNIT();
      unsigned long long nlive = 0;
      for (int p = 0; p < npairs; ++p) {
        const uint32_t pb = pair_bits(cmask, p);
        if (!pb || !rmask) continue;
        if (lane == 0) {
          TMC_PROF_WAIT(true, 43, mbar_wait(y_empty, (pa & 1) ^ 1));
          mbar_expect_tx(y_full, 2 * G::TILE + 2 * kBxBytes);
          for (int h = 0; h < 2; ++h) {
            const int j = 2 * p + h;
            bulk_g2s(sY + (size_t)h * G::TILE, a.Yt + ((size_t)b * a.c_tiles + j) * G::TILE, G::TILE, y_full);
            bulk_g2s(sCx + (size_t)h * kBxBytes, a.Cx + ((size_t)b * a.c_tiles + j) * kBxBytes, kBxBytes, y_full);
          }
        }
        ++pa;
        for (int i = 0; i < a.r_tiles; ++i) {
          if (!((rmask >> i) & 1)) continue;
          nlive += __popc(pb);
          const uint32_t s = v & 1;
          if (lane == 0) {
            TMC_PROF_WAIT(true, 44, mbar_wait(&x_empty[s], ((v >> 1) & 1) ^ 1));
            mbar_expect_tx(&x_full[s], G::TILE);
            bulk_g2s(sX + (size_t)s * G::TILE, a.Xt + ((size_t)b * a.r_tiles + i) * G::TILE, G::TILE, &x_full[s]);
          }
          ++v;
        }
      }
      if (fb.count && lane == 0) atomicAdd(&g_tmc_mma_flops[PF_TC_BWD], nlive * fb.flops_per_tile);
    }
  } else if (warp == G::W_MMA) {
    // ---------------- MMA issuer (one warp, one elected lane; MMAs execute in issue order)
    uint32_t t = 0, v = 0, pa = 0;
    const uint32_t xBase = smem_u32(sX), yBase = smem_u32(sY), pBase = smem_u32(sP);
    const uint32_t onesC = smem_u32(sOnesC);
    // the gradient GEMMs of live tile tt (issued one tile late, after S of the next tile)
    struct Pend { uint32_t t, xs, h, first_row, first_col, last_visit, last_pair, valid; };
    Pend pend{0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t gc_uses = 0;                   // bit h: parity of the uses of G_col accumulator h
    uint32_t gr_uses = 0;                   // G_row accumulator uses (visits)
    auto issue_g = [&](const Pend& q) {
      const uint32_t buf = q.t & 1;
      TMC_PROF_WAIT(lane == 0, 26, mbar_wait(&p_full[buf], (q.t >> 1) & 1));
      tc_fence_after();
      // G_col(j) += P~^T X_i  (A = shared P~ image, MN-major; B = X tile MN-major, ones at LBO)
      if (q.first_col) {
        TMC_PROF_WAIT(lane == 0, 27, mbar_wait(&gcol_empty[q.h], ((gc_uses >> q.h) & 1) ^ 1));
        gc_uses ^= 1u << q.h;
        tc_fence_after();
      }
      const uint32_t gcD = tmem + G::GCOL + q.h * G::GCN;
      const uint32_t xs = xBase + q.xs * G::TILE;
      TMC_PROF_T0(_gc);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t ko = kk * 2048;
        const uint64_t aHi = sdesc_mn(pBase + ko, 16384), aLo = sdesc_mn(pBase + G::PIMG + ko, 16384);
        const uint64_t bHi1 = sdesc_mn(xs + ko, onesC - (xs + ko));          // [X_hi | ones]
        const uint64_t bLo = sdesc_mn(xs + G::PART + ko, 16384);              // X_lo
        mma_f16(gcD, aLo, bHi1, IDESC_GC80, (q.first_col && kk == 0) ? 0u : 1u);
        mma_f16(gcD, aHi, bLo, IDESC_GC64, 1u);
        mma_f16(gcD, aHi, bHi1, IDESC_GC80, 1u);
      }
      mma_commit(pimg_empty);
      TMC_PROF_END(lane == 0, 46, _gc);
      if (q.last_visit) mma_commit(&x_empty[q.xs]);
      if (q.last_pair) mma_commit(&gcol_full[q.h]);   // the last row tile of the pair: acc h complete
      // G_row(i) += P~ Y_j  (A = P~ in TMEM, B = Y tile MN-major)
      if (q.first_row) {
        TMC_PROF_WAIT(lane == 0, 28, mbar_wait(grow_empty, (gr_uses & 1) ^ 1));
        ++gr_uses;
        tc_fence_after();
      }
      const uint32_t pA = tmem + buf * 128;
      const uint32_t grD = tmem + G::GROW;
      TMC_PROF_T0(_gr);
      const uint64_t dT = sdesc_mn(yBase + q.h * G::TILE, kAtomBytes);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t phi = pA + (kk >> 1) * 32 + (kk & 1) * 8, plo = phi + 16;
        const uint64_t thi = dadd(dT, kk * 2048), tlo = dadd(dT, G::PART + kk * 2048);
        mma_f16_ts(grD, plo, thi, IDESC_GR, (q.first_row && kk == 0) ? 0u : 1u);
        mma_f16_ts(grD, phi, tlo, IDESC_GR, 1u);
        mma_f16_ts(grD, phi, thi, IDESC_GR, 1u);
      }
      TMC_PROF_END(lane == 0, 47, _gr);
      if (q.last_visit) mma_commit(grow_full);
      if (q.last_pair && q.last_visit) mma_commit(y_empty);
    };
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      TMC_BWD1_UNIT();
      for (int p = 0; p < npairs; ++p) {
        const uint32_t pb = pair_bits(cmask, p);
        if (!pb || !rmask) continue;
        TMC_PROF_WAIT(lane == 0, 24, mbar_wait(y_full, pa & 1));
        ++pa;
        // the last live visit of this pair
        const int ilast = 63 - __clzll((long long)rmask);
        uint32_t first_col = 3u;            // bit h: acc h not yet written in this pair
        for (int i = 0; i < a.r_tiles; ++i) {
          if (!((rmask >> i) & 1)) continue;
          const uint32_t xs = v & 1;
          TMC_PROF_WAIT(lane == 0, 25, mbar_wait(&x_full[xs], (v >> 1) & 1));
          ++v;
          const int hlast = (pb & 2) ? 1 : 0;
          bool first_row = true;
          for (int h = 0; h < 2; ++h) {
            if (!((pb >> h) & 1)) continue;
            const uint32_t buf = t & 1;
            tc_fence_after();
            // S(i, 2p+h) = X_i Y^T (3-term fp16 split, small terms first) + the column term
            const uint32_t d = tmem + buf * 128;
            const uint64_t dA = sdesc(xBase + xs * G::TILE), dB = sdesc(yBase + h * G::TILE);
            TMC_PROF_T0(_s);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t o = kk * 32;
              mma_f16(d, dadd(dA, o), dadd(dB, G::PART + o), IDESC_S, kk ? 1u : 0u);
              mma_f16(d, dadd(dA, G::PART + o), dadd(dB, o), IDESC_S, 1u);
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t o = kk * 32;
              mma_f16(d, dadd(dA, o), dadd(dB, o), IDESC_S, 1u);
            }
            mma_f16(d, sdesc_bx(smem_u32(sOnesB)), sdesc_bx(smem_u32(sCx) + h * kBxBytes), IDESC_S, 1u);
            mma_commit(&s_full[buf]);
            TMC_PROF_END(lane == 0, 48, _s);
            if (pend.valid) issue_g(pend);
            pend = Pend{t, xs, (uint32_t)h, first_row ? 1u : 0u, (first_col >> h) & 1u,
                        h == hlast ? 1u : 0u, (i == ilast) ? 1u : 0u, 1u};
            first_row = false;
            first_col &= ~(1u << h);
            ++t;
          }
        }
        // the pair's Y tiles are replaced next: finish its gradient GEMMs first
        if (pend.valid) { issue_g(pend); pend.valid = 0; }
      }
    }
    if (pend.valid) issue_g(pend);
  } else if (warp < SMW) {
    // ---------------- softmax / P~ warps: (TMEM lane quarter, 64-column half)
    const int quarter = warp & 3, half = warp >> 2;
    const int m = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t sw = (uint32_t)(m & 7);
    uint8_t* prow_hi = sP + half * 16384 + (m >> 3) * 1024 + (m & 7) * 128;   // this thread's row of chunk `half`
    uint8_t* prow_lo = prow_hi + G::PIMG;
    uint32_t t = 0, v = 0;
    auto chunk_math = [&](const uint32_t* x, float2 hom2, float2* racc, uint32_t* hi, uint32_t* lo) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float2 y01 = __fadd2_rn(make_float2(__uint_as_float(x[4 * q]), __uint_as_float(x[4 * q + 1])), hom2);
        const float2 y23 = __fadd2_rn(make_float2(__uint_as_float(x[4 * q + 2]), __uint_as_float(x[4 * q + 3])), hom2);
        const float2 p01 = make_float2(ex2(y01.x), ex2(y01.y));
        const float2 p23 = make_float2(ex2(y23.x), ex2(y23.y));
        racc[0] = __fadd2_rn(racc[0], p01);
        racc[1] = __fadd2_rn(racc[1], p23);
        __half2 h01 = __floats2half2_rn(p01.x, p01.y), h23 = __floats2half2_rn(p23.x, p23.y);
        hi[2 * q] = *reinterpret_cast<uint32_t*>(&h01);
        hi[2 * q + 1] = *reinterpret_cast<uint32_t*>(&h23);
        const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
        const float2 d01 = __fadd2_rn(p01, make_float2(-f01.x, -f01.y));
        const float2 d23 = __fadd2_rn(p23, make_float2(-f23.x, -f23.y));
        __half2 l01 = __floats2half2_rn(d01.x, d01.y), l23 = __floats2half2_rn(d23.x, d23.y);
        lo[2 * q] = *reinterpret_cast<uint32_t*>(&l01);
        lo[2 * q + 1] = *reinterpret_cast<uint32_t*>(&l23);
      }
    };
    // 32 columns (hi or lo words w[16] = 32 fp16) -> 16-byte units u0..u0+3 of this thread's image row
    auto sts_units = [&](uint8_t* row, int u0, const uint32_t* w) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(row + (((uint32_t)(u0 + q) ^ sw) << 4)) =
            make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    };
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      TMC_BWD1_UNIT();
      for (int p = 0; p < npairs; ++p) {
        const uint32_t pb = pair_bits(cmask, p);
        if (!pb || !rmask) continue;
        for (int i = 0; i < a.r_tiles; ++i) {
          if (!((rmask >> i) & 1)) continue;
          const float hom = a.rterm[(size_t)b * a.r_tiles * 128 + i * 128 + m] + 14.f;
          const float2 hom2 = make_float2(hom, hom);
          float2 racc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
          for (int h = 0; h < 2; ++h) {
            if (!((pb >> h) & 1)) continue;
            const uint32_t buf = t & 1;
            TMC_PROF_WAIT(warp == 0 && lane == 0, 30, mbar_wait(&s_full[buf], (t >> 1) & 1));
            tc_fence_after();
            const uint32_t ta0 = tmem + lane_off + (uint32_t)(buf * 128 + half * 64);
            // two 32-column quarters, one after the other (keeps the register footprint small)
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
              const uint32_t ta = ta0 + 32 * c;
              uint32_t x[32];
              TMC_PROF_T0(_l);
              TMC_LD32(ta, x);
              tmem_ld_wait();
              TMC_PROF_END(warp == 0 && lane == 0, 32, _l);
              TMC_PROF_T0(_mth);
              uint32_t hi[16], lo[16];
              if (hom > -INFINITY) chunk_math(x, hom2, racc, hi, lo);
              else for (int q = 0; q < 16; ++q) { hi[q] = 0u; lo[q] = 0u; }
              TMC_PROF_END(warp == 0 && lane == 0, 33, _mth);
              TMC_PROF_T0(_st);
              TMC_ST16(ta, hi);
              TMC_ST16(ta + 16, lo);
              // the shared image is free once the previous tile's G_col has read it
              if (c == 0) TMC_PROF_WAIT(warp == 0 && lane == 0, 31, mbar_wait(pimg_empty, (t & 1) ^ 1));
              sts_units(prow_hi, 4 * c, hi);
              sts_units(prow_lo, 4 * c, lo);
              TMC_PROF_END(warp == 0 && lane == 0, 34, _st);
            }
            tmem_st_wait();
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[buf]);
            ++t;
          }
          if (a.rowsum) {   // this warp's row sums of the visit -> the epilogue warps
            TMC_PROF_WAIT(warp == 0 && lane == 0, 35, mbar_wait(&r_empty[v & 1], ((v >> 1) & 1) ^ 1));
            const float2 rr = __fadd2_rn(racc[0], racc[1]);
            sRs[(v & 1) * 256 + half * 128 + m] = rr.x + rr.y;
            __syncwarp();
            if (lane == 0) mbar_arrive(&r_full[v & 1]);
          }
          ++v;
        }
      }
    }
  } else if (warp < SMW + EW) {
    // ---------------- epilogue warps (one per TMEM lane quarter): dz per visit, dmu/dlogvar per pair
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint32_t v = 0, gr = 0, gcp = 0;        // gcp bit h: parity of acc h's drains
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      TMC_BWD1_UNIT();
      const float sc = a.sgn[b] * (1.f / 16384.f);
      // the datapoint's centering shift, staged once in shared memory (broadcast reads)
      named_bar(2, 32 * EW);
      if (warp == SMW && lane < D) sSh[lane] = a.shift[(size_t)b * D + lane];
      named_bar(2, 32 * EW);
      const float* sh = sSh;
      uint64_t init = 0;                    // row tiles whose dz rows hold a partial sum
      for (int p = 0; p < npairs; ++p) {
        const uint32_t pb = pair_bits(cmask, p);
        const bool pact = pb && rmask;
        for (int i = 0; i < a.r_tiles && pact; ++i) {
          if (!((rmask >> i) & 1)) continue;
          // ---- G_row(i) over this pair -> dz partial (read-add-write in column-pair order)
          const int gm = i * 128 + m;
          const bool rowok = gm < a.Mr;
          const size_t row = ((size_t)b * a.Mr + (rowok ? gm : 0)) * D;
          const bool first = !((init >> i) & 1);
          // the row's z and its dz partial so far, loaded before G_row(i) is ready: all 16 loads in
          // flight at once (one memory latency per visit instead of one per float4); G_row is then
          // read 8 dimensions at a time (register budget: 64 prefetched + 16 accumulator values)
          TMC_PROF_T0(_dz);
          float4 zq[D / 4], dq[D / 4];
          const bool wz = a.gz && rowok;
#pragma unroll
          for (int q = 0; q < D / 4; ++q) {
            zq[q] = wz ? __ldg(reinterpret_cast<const float4*>(a.z + row) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            dq[q] = (wz && !first) ? __ldcg(reinterpret_cast<const float4*>(a.gz + row) + q)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          const float rprev = (a.rowsum && rowok && !first) ? __ldcg(a.rowsum + (size_t)b * a.Mr + gm) : 0.f;
          TMC_PROF_END(warp == SMW && lane == 0, 40, _dz);
          TMC_PROF_WAIT(warp == SMW && lane == 0, 37, mbar_wait(grow_full, gr & 1));
          ++gr;
          tc_fence_after();
          // dz partial (G1 + 2 z' G0) sgn/2^14 ln 2 added to the running sum
#pragma unroll
          for (int d8 = 0; d8 < D; d8 += 8) {
            uint32_t g0[8], g1[8];
            TMC_LD8(tmem + lane_off + G::GROW + d8, g0);       // G0 = sum P~ Y0
            TMC_LD8(tmem + lane_off + G::GROW + 32 + d8, g1);  // G1 = sum P~ Y1
            tmem_ld_wait();
            if (d8 + 8 == D) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(grow_empty);
            }
#pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
              const int d4 = d8 + 4 * hq;
              const float4 z4 = zq[d4 / 4], p4 = dq[d4 / 4];
              const float zz[4] = {z4.x, z4.y, z4.z, z4.w}, pp[4] = {p4.x, p4.y, p4.z, p4.w};
              float o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e)
                o[e] = pp[e] + (__uint_as_float(g1[4 * hq + e]) + 2.f * (zz[e] - sh[d4 + e]) *
                                __uint_as_float(g0[4 * hq + e])) * (sc * kLn2);
              if (wz) *reinterpret_cast<float4*>(a.gz + row + d4) = make_float4(o[0], o[1], o[2], o[3]);
            }
          }
          float rs = 0.f;
          if (a.rowsum) {
            TMC_PROF_WAIT(warp == SMW && lane == 0, 38, mbar_wait(&r_full[v & 1], (v >> 1) & 1));
            rs = sRs[(v & 1) * 256 + m] + sRs[(v & 1) * 256 + 128 + m];
            __syncwarp();
            if (lane == 0) mbar_arrive(&r_empty[v & 1]);
          }
          ++v;
          if (a.rowsum && rowok) a.rowsum[(size_t)b * a.Mr + gm] = rprev + rs * sc;
          init |= 1ull << i;
        }
        // ---- G_col of the pair's two column tiles -> dmu, dlogvar, column sums
        for (int h = 0; h < 2; ++h) {
          const int j = 2 * p + h;
          const bool got = pact && ((pb >> h) & 1);
          const int gc_ = j * 128 + m;
          const bool colok = gc_ < a.Mc;
          const size_t row = ((size_t)b * a.Mc + (colok ? gc_ : 0)) * D;
          // mu / logvar of the column's row, loaded before the accumulator is ready (read-only inputs)
          const bool ld = got && colok;
          float4 mq[D / 4], vq[D / 4];
#pragma unroll
          for (int q = 0; q < D / 4; ++q) {
            mq[q] = ld ? __ldg(reinterpret_cast<const float4*>(a.mu + row) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            vq[q] = ld ? __ldg(reinterpret_cast<const float4*>(a.lv + row) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          uint32_t ga = 0;
          float pi = 0.f;
          if (got) {
            TMC_PROF_WAIT(warp == SMW && lane == 0, 39, mbar_wait(&gcol_full[h], (gcp >> h) & 1));
            gcp ^= 1u << h;
            tc_fence_after();
            ga = tmem + lane_off + G::GCOL + h * G::GCN;
            uint32_t cs[8];
            TMC_LD8(ga + 64, cs);
            tmem_ld_wait();
            pi = __uint_as_float(cs[0]) * sc;
          }
#pragma unroll
          for (int d8 = 0; d8 < D; d8 += 8) {
            uint32_t c0[8], c1[8];
            if (got) {
              TMC_LD8(ga + d8, c0);
              TMC_LD8(ga + 32 + d8, c1);
              tmem_ld_wait();
              if (d8 + 8 == D) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&gcol_empty[h]);
              }
            }
#pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
              const int d4 = d8 + 4 * hq;
              float om[4] = {0.f, 0.f, 0.f, 0.f}, ov[4] = {0.f, 0.f, 0.f, 0.f};
              if (got) {
                const float4 m4 = mq[d4 / 4], v4 = vq[d4 / 4];
                const float mm[4] = {m4.x, m4.y, m4.z, m4.w}, vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float mp = mm[e] - sh[d4 + e];
                  const float lam = __expf(-vv[e]);
                  const float A1 = __uint_as_float(c1[4 * hq + e]) * sc, A2 = __uint_as_float(c0[4 * hq + e]) * sc;
                  om[e] = a.alpha * lam * (A1 - mp * pi);
                  ov[e] = a.alpha * 0.5f * (lam * (A2 - 2.f * mp * A1 + mp * mp * pi) - pi);
                }
              }
              if (colok && a.gmu) *reinterpret_cast<float4*>(a.gmu + row + d4) = make_float4(om[0], om[1], om[2], om[3]);
              if (colok && a.glv) *reinterpret_cast<float4*>(a.glv + row + d4) = make_float4(ov[0], ov[1], ov[2], ov[3]);
            }
          }
          if (colok && a.colsum) a.colsum[(size_t)b * a.Mc + gc_] = pi;
        }
      }
      // row tiles that never received a contribution: exact zeros
      for (int i = 0; i < a.r_tiles; ++i) {
        if ((init >> i) & 1) continue;
        const int gm = i * 128 + m;
        if (gm >= a.Mr) continue;
        const size_t row = ((size_t)b * a.Mr + gm) * D;
        if (a.gz)
          for (int d4 = 0; d4 < D; d4 += 4) *reinterpret_cast<float4*>(a.gz + row + d4) = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a.rowsum) a.rowsum[(size_t)b * a.Mr + gm] = 0.f;
      }
    }
  }
  TMC_PROF_END(lane == 0 && (warp == G::W_PROD || warp == G::W_MMA || warp == 0 || warp == SMW),
               warp == G::W_PROD ? 45 : warp == G::W_MMA ? 29 : warp == 0 ? 36 : 42, _tot);
  tc_fence_before();
  __syncthreads();
  if (warp == G::W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}
#undef TMC_BWD1_UNIT

}  // namespace tc

// ================================================================================ host side
// Single-pass reverse when the edge is D = 32, both sides <= 64 tiles and the tile grid is big
// enough for the per-(edge, datapoint) pipeline (>= 16 tiles); pair marginals use the SIMT path.
inline bool tc_bwd1_ok(const TcLatentBuf& t, const PassArgs& a) {
  const int rt = t.KzPad / 128, ct = t.KpPad / 128;
  return t.ok && t.bwd_ok && !a.pair && t.D == 32 && rt <= 64 && ct <= 64 && rt * ct >= 16;
}

// ne edges (same D = 32), one batched launch: the per-edge row terms / bias tiles / live flags
// (tc_rowterm_kernel), then tc_bwd1_kernel over every (edge, datapoint).  zrows = DOWN.  Each
// PassArgs carries gz/gmu/glv, w (row weights of the forward's rows) and colsum (DOWN: the parent
// edge's weights; UP: the z side's marginal).  Returns kernels launched.
inline int tc_pass_backward1_batch(const PassArgs* as, const TcLatentBuf* const* ts, int ne, void* ws, bool zrows,
                                   bool dense_reverse, cudaStream_t s) {
  uint8_t* w = static_cast<uint8_t*>(ws);
  int launched = 0;
  static bool attr[kMaxDevices] = {};
  ensure_smem_attr(tc::tc_bwd1_kernel, (int)tc::B1Geo::SMEM, attr);
  for (int e0 = 0; e0 < ne; e0 += tc::kMaxBatch) {
    tc::Bwd1Batch fb{};
    tc::RowtermBatch rtb{};
    fb.ne = std::min(tc::kMaxBatch, ne - e0);
    rtb.ne = fb.ne;
    fb.ustart[0] = 0;
    for (int k = 0; k < fb.ne; ++k) {
      const PassArgs& a = as[e0 + k];
      const TcLatentBuf& t = *ts[e0 + k];
      const int Rpad = zrows ? t.KzPad : t.KpPad;        // the forward's rows
      float* rterm2 = reinterpret_cast<float*>(w + t.rterm2);
      float* sgn = reinterpret_cast<float*>(w + t.sgn);
      tc::RowtermArgs& r = rtb.e[k];
      r.ell = a.ell; r.w = a.w;
      r.beta = zrows ? nullptr : reinterpret_cast<const float*>(w + t.beta);
      r.betaStride = t.KpPad; r.R = a.R; r.Rpad = Rpad;
      r.rterm2 = rterm2; r.sgn = sgn;
      r.bx = w + t.rbx;
      r.live = reinterpret_cast<int*>(w + t.rlive);
      tc::Bwd1Args& f = fb.e[k];
      f.Xt = w + t.xt;
      f.Yt = w + t.yt;
      f.r_tiles = t.KzPad / 128;
      f.c_tiles = t.KpPad / 128;
      const int* rl = reinterpret_cast<const int*>(w + t.rlive);   // over the forward's rows
      const int* cl = reinterpret_cast<const int*>(w + t.clive);   // over the forward's columns
      if (zrows) {            // DOWN: forward rows = z samples
        f.rterm = rterm2;
        f.Cx = w + t.bx;
        f.Mr = a.R; f.Mc = a.C;
        f.rlive = dense_reverse ? nullptr : rl;
        f.clive = dense_reverse ? nullptr : cl;
        f.rowsum = nullptr;
        f.colsum = a.colsum;
      } else {                // UP: forward rows = parent samples
        f.rterm = reinterpret_cast<const float*>(w + t.cb2);
        f.Cx = w + t.rbx;
        f.Mr = a.C; f.Mc = a.R;
        f.rlive = dense_reverse ? nullptr : cl;
        f.clive = dense_reverse ? nullptr : rl;
        f.rowsum = a.colsum;
        f.colsum = nullptr;
      }
      f.sgn = sgn;
      f.alpha = a.alpha;
      f.z = a.z; f.mu = a.mu; f.lv = a.lv;
      f.shift = reinterpret_cast<const float*>(w + t.shift);
      f.gz = a.gz; f.gmu = a.gmu; f.glv = a.glv;
      fb.ustart[k + 1] = fb.ustart[k] + a.B;
    }
    {
      ProfScope ps(PF_TC_PREP, s);
      tc::tc_rowterm_kernel<<<dim3(as[e0].B, rtb.ne), 256, 0, s>>>(rtb);
    }
    ++launched;
    fb.count = prof_on() ? 1 : 0;
    // per live tile: S (3 terms, K = 2D) + bias MMA (K = 16) + G_row (3 x N = 64) + G_col (N = 80, 64, 80)
    fb.flops_per_tile = (unsigned long long)(12 * 32 + 32 + 12 * 32 + 2 * 224) * 128 * 128;
    const int sms = sm_count();
    const int units = fb.ustart[fb.ne];
    const int grid = units < sms ? units : sms;
    ProfScope ps(PF_TC_BWD, s);
    if (grid > 0) tc::tc_bwd1_kernel<<<grid, tc::B1Geo::THREADS, tc::B1Geo::SMEM, s>>>(fb);
    ++launched;
  }
  return launched;
}

}  // namespace tmc
