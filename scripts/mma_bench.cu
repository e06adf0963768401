// tcgen05.mma issue-rate microbenchmark on B200 (sm_100a): cycles per instruction for the MMA
// shapes the TMC kernels use.  One CTA per SM, one elected thread issues N back-to-back MMAs into
// TMEM (operands: a 128x64 fp16 SWIZZLE_128B K-major tile pair in shared memory, or A from TMEM),
// then commits and waits; the kernel reports clock64 cycles / N.  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_bench scripts/mma_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <int MODE>   // 0: SS K-major N=128; 1: SS N=64; 2: TS (A in TMEM) B MN-major N=64; 3: TS N=128; 4: SS N=256
                      // 5: the reverse pass's tile mix (12 SS N=128 into cols 0.., 24 TS N=64 into cols 384..); n = tiles
                      // 6: as 5 while warps 1-3 stream tcgen05.ld/st over TMEM columns 128..383 (softmax-like traffic)
                      // 7: as 5 while warps 1-3 stream LDS.128 reads of shared memory (port contention)
                      // 8: as 5 with the S MMAs in TS mode (A from TMEM cols 448..511)
                      // 9: as 5 while 20 other warps (5 per SMSP) run an ex2/FADD2 loop (softmax-like issue load)
                      // 10: as 5 with a tcgen05.commit after the S MMAs and two after the gradient MMAs (per tile)
                      // 11: single-pass reverse tile mix: 12 SS N=128 (S) + 24 TS N=64 (G_row, A = P~ in TMEM)
                      //     + 24 SS N=64 with A MN-major in shared memory (G_col, A = P~^T)
                      // 12: as 11 while 4 warps store 64 KB per tile to shared memory (the P~ images)
                      // 13: packed two-pass gradient: 12 SS N=128 + per K-step P_hi [T_hi|T_lo] (TS N=128)
                      //     + P_lo T_hi (TS N=64), 8 K-steps
                      // 14: SS, A and B both MN-major, N=64 (the G_col MMA alone); 15: the same at N=80
                      // 16: tc_bwd1_kernel's exact tile mix: 12 SS N=128 + bias K=16 + 8 x (N=80, 64, 80)
                      //     A-MN-major SS (G_col) + 24 TS N=64 (G_row)
__global__ void __launch_bounds__(704, 1) bench(int n, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint64_t dbar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&dbar[q])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t A = smem_u32(smem), Bs = A + 32768;
    constexpr uint32_t N = (MODE == 1 || MODE == 2) ? 64 : (MODE == 4 ? 256 : 128);
    constexpr uint32_t bmaj = (MODE >= 2 && MODE <= 3) ? 1u : 0u;
    constexpr uint32_t idesc = (1u << 4) | (bmaj << 16) | ((N >> 3) << 17) | ((128u >> 4) << 24);
    long long t0 = clock64();
    if constexpr (MODE == 8) {
      constexpr uint32_t idS = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t idG = (1u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
      for (int i = 0; i < n; ++i) {
        for (int k = 0; k < 12; ++k) {
          const uint64_t b = sdesc(Bs + (k & 3) * 32);
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + (i % 3) * 128),
                       "r"(tmem + 448 + (k & 7) * 8), "l"(b), "r"(idS), "r"((uint32_t)(k != 0)));
        }
        for (int k = 0; k < 24; ++k) {
          const uint64_t b = sdesc_mn(Bs + (k & 7) * 2048, 16384);
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 384),
                       "r"(tmem + ((i + 2) % 3) * 128 + (k & 7) * 8), "l"(b), "r"(idG), "r"(1u));
        }
      }
    } else if constexpr (MODE == 14 || MODE == 15) {
      constexpr uint32_t NN = MODE == 14 ? 64u : 80u;
      constexpr uint32_t idC = (1u << 4) | (1u << 15) | (1u << 16) | ((NN >> 3) << 17) | ((128u >> 4) << 24);
      for (int i = 0; i < n; ++i) {
        const uint64_t a = sdesc_mn(A + (i & 7) * 2048, 16384), b = sdesc_mn(Bs + (i & 7) * 2048, 16384);
        asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 256),
                     "l"(a), "l"(b), "r"(idC), "r"(1u));
      }
    } else if constexpr (MODE == 16) {
      constexpr uint32_t idS = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t idG = (1u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t idC64 = (1u << 4) | (1u << 15) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t idC80 = (1u << 4) | (1u << 15) | (1u << 16) | ((80u >> 3) << 17) | ((128u >> 4) << 24);
      for (int i = 0; i < n; ++i) {
        for (int k = 0; k < 13; ++k) {
          const uint64_t a = sdesc(A + (k & 3) * 32), b = sdesc(Bs + (k & 3) * 32);
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (i % 2) * 128),
                       "l"(a), "l"(b), "r"(idS), "r"((uint32_t)(k != 0)));
        }
        for (int k = 0; k < 24; ++k) {
          const uint64_t a = sdesc_mn(A + (k & 7) * 2048, 16384), b = sdesc_mn(Bs + (k & 7) * 2048, 16384);
          const uint32_t id = (k % 3 == 1) ? idC64 : idC80;
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 256),
                       "l"(a), "l"(b), "r"(id), "r"(1u));
        }
        for (int k = 0; k < 24; ++k) {
          const uint64_t b = sdesc_mn(Bs + (k & 7) * 2048, 16384);
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 416),
                       "r"(tmem + ((i + 1) % 2) * 128 + (k & 7) * 8), "l"(b), "r"(idG), "r"(1u));
        }
      }
    } else if constexpr (MODE == 11 || MODE == 12 || MODE == 13) {
      constexpr uint32_t idS = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t idG = (1u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t idG2 = (1u << 4) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t idC = (1u << 4) | (1u << 15) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
      for (int i = 0; i < n; ++i) {
        for (int k = 0; k < 12; ++k) {
          const uint64_t a = sdesc(A + (k & 3) * 32), b = sdesc(Bs + (k & 3) * 32);
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (i % 2) * 128),
                       "l"(a), "l"(b), "r"(idS), "r"((uint32_t)(k != 0)));
        }
        if constexpr (MODE == 13) {
          for (int k = 0; k < 8; ++k) {
            const uint64_t b = sdesc_mn(Bs + (k & 7) * 2048, 16384);
            asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 256),
                         "r"(tmem + ((i + 1) % 2) * 128 + (k & 7) * 8), "l"(b), "r"(idG2), "r"(1u));
            asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 384),
                         "r"(tmem + ((i + 1) % 2) * 128 + (k & 7) * 8), "l"(b), "r"(idG), "r"(1u));
          }
        } else {
          for (int k = 0; k < 24; ++k) {
            const uint64_t b = sdesc_mn(Bs + (k & 7) * 2048, 16384);
            asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 256),
                         "r"(tmem + ((i + 1) % 2) * 128 + (k & 7) * 8), "l"(b), "r"(idG), "r"(1u));
          }
          for (int k = 0; k < 24; ++k) {
            const uint64_t a = sdesc_mn(A + (k & 7) * 2048, 16384), b = sdesc_mn(Bs + (k & 7) * 2048, 16384);
            asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 384),
                         "l"(a), "l"(b), "r"(idC), "r"(1u));
          }
        }
      }
    } else if constexpr (MODE >= 5 && MODE != 9 || MODE == 9) {
      constexpr uint32_t idS = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      constexpr uint32_t idG = (1u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
      for (int i = 0; i < n; ++i) {
        for (int k = 0; k < 12; ++k) {
          const uint64_t a = sdesc(A + (k & 3) * 32), b = sdesc(Bs + (k & 3) * 32);
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (i % 3) * 128),
                       "l"(a), "l"(b), "r"(idS), "r"((uint32_t)(k != 0)));
        }
        if (MODE == 10)
          asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                       "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&dbar[0])) : "memory");
        for (int k = 0; k < 24; ++k) {
          const uint64_t b = sdesc_mn(Bs + (k & 7) * 2048, 16384);
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 384),
                       "r"(tmem + ((i + 2) % 3) * 128 + (k & 7) * 8), "l"(b), "r"(idG), "r"(1u));
        }
        if (MODE == 10) {
          asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                       "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&dbar[1])) : "memory");
          asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                       "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&dbar[2])) : "memory");
        }
      }
    } else
    for (int i = 0; i < n; ++i) {
      const uint32_t acc = i ? 1u : 0u;
      const uint32_t koff = (i & 3) * 32;
      if constexpr (MODE <= 1 || MODE == 4) {
        const uint64_t a = sdesc(A + koff), b = sdesc(Bs + koff);
        asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 256),
                     "l"(a), "l"(b), "r"(idesc), "r"(acc));
      } else {
        const uint64_t b = sdesc_mn(Bs + (i & 7) * 2048, 16384);
        asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 256),
                     "r"(tmem + (i & 7) * 8), "l"(b), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
        smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  if (MODE == 9 && warp != 0) {
    float2 acc = make_float2(0.f, 0.f), x = make_float2(threadIdx.x * 1e-9f, 1e-9f);
    for (int i = 0; i < n * 96; ++i) {
      const float2 y = __fadd2_rn(x, make_float2(-1e-3f, -2e-3f));
      float e0, e1;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(y.x));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(y.y));
      acc = __fadd2_rn(acc, make_float2(e0, e1));
      x = __fadd2_rn(x, make_float2(1e-7f, 1e-7f));
    }
    if (acc.x == 1234.f) out[1023] = 1;
  }
  if (MODE == 12 && warp != 0) {
    // 4 warps x 16 KB per tile of 16-byte stores (the P~ hi/lo images of a 128 x 128 tile)
    uint4* p4 = reinterpret_cast<uint4*>(smem + 49152);
    const uint4 v = make_uint4(threadIdx.x, 1u, 2u, 3u);
    for (int i = 0; i < n * 32; ++i) {
      p4[(i * 32 + (threadIdx.x & 31) + (warp - 1) * 256) & 1023] = v;
      __syncwarp();
    }
  }
  if (MODE == 7 && warp != 0) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* p4 = reinterpret_cast<const float4*>(smem);
    for (int i = 0; i < n * 64; ++i) {
      const float4 q = p4[(i * 32 + (threadIdx.x & 31) + warp * 1024) & 4095];
      acc.x += q.x; acc.y += q.y; acc.z += q.z; acc.w += q.w;
    }
    if (acc.x == 1234.f) out[1023] = 1;
  }
  if (MODE == 6 && warp != 0) {
    // 3 warps (lane quarters 1-3) read and write back 64 columns per "tile", like the softmax warps
    uint32_t v[32];
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 128;
    for (int i = 0; i < n * 4; ++i) {
      const uint32_t ta = base + (uint32_t)((i & 3) * 64);
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   :: "r"(ta + 32), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int MODE>
double run(int sms, unsigned long long* d, unsigned long long* h, int n) {
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int threads = MODE == 9 ? 704 : MODE == 12 ? 160 : 128;
  bench<MODE><<<sms, threads, 70 * 1024>>>(n, d);
  bench<MODE><<<sms, threads, 70 * 1024>>>(n, d);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += h[i];
  return s / sms / n;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *d, h[1024];
  cudaMalloc(&d, sizeof(h));
  const int n = 4096;
  printf("{\"clk_per_mma_ss_n128\": %.1f, \"clk_per_mma_ss_n64\": %.1f, \"clk_per_mma_ts_mn_n64\": %.1f, "
         "\"clk_per_mma_ts_mn_n128\": %.1f, \"clk_per_mma_ss_n256\": %.1f, \"clk_per_bwd_tile_mix\": %.1f, "
         "\"clk_per_bwd_tile_mix_with_tmem_traffic\": %.1f, \"clk_per_bwd_tile_mix_with_lds\": %.1f, "
         "\"clk_per_bwd_tile_mix_S_in_TS_mode\": %.1f, \"clk_per_bwd_tile_mix_busy_smsp\": %.1f, \"clk_per_bwd_tile_mix_3_commits\": %.1f, "
         "\"clk_per_single_pass_tile_mix\": %.1f, \"clk_per_single_pass_tile_mix_with_p_stores\": %.1f, "
         "\"clk_per_packed_grad_tile_mix\": %.1f, \"clk_per_mma_ss_amn_n64\": %.1f, \"clk_per_mma_ss_amn_n80\": %.1f, "
         "\"clk_per_bwd1_exact_tile_mix\": %.1f, \"err\": \"%s\"}\n",
         run<0>(sms, d, h, n), run<1>(sms, d, h, n), run<2>(sms, d, h, n), run<3>(sms, d, h, n), run<4>(sms, d, h, n),
         run<5>(sms, d, h, 256), run<6>(sms, d, h, 256), run<7>(sms, d, h, 256), run<8>(sms, d, h, 256), run<9>(sms, d, h, 256), run<10>(sms, d, h, 256),
         run<11>(sms, d, h, 256), run<12>(sms, d, h, 256), run<13>(sms, d, h, 256),
         run<14>(sms, d, h, n), run<15>(sms, d, h, n), run<16>(sms, d, h, 256),
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
