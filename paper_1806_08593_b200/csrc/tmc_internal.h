// Internal structures shared by the libtmc host code and kernels (NOT part of the ABI).
#pragma once
#include <cstdint>
#include <mutex>
#include <vector>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

namespace tmc {

// NVTX ranges (header-only nvtx3; free when no tool is attached): one range per ABI call and one
// per kernel-family launch scope, so a timeline / `ncu --nvtx` shows which call and which stage
// every kernel belongs to (launch-gap evidence).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Per-device one-time state (kernel attributes, SM counts): a process may drive several GPUs.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDevices) ? d : 0;
}
inline int sm_count() {
  static int sms[kMaxDevices] = {};
  const int d = current_device();
  if (!sms[d]) cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, d);
  return sms[d];
}
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel instantiation, device)
template <typename Kernel>
inline void ensure_smem_attr(Kernel k, int bytes, bool* done) {
  const int d = current_device();
  if (!done[d]) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done[d] = true;
  }
}

// ------------------------------------------------------------------ launch profiler (diagnostics)
// tmc_profile_begin/end (include/tmc.h): while enabled, every launch of a kernel family is
// bracketed by a CUDA event pair recorded on the launching stream, and the tensor-core kernels add
// the tcgen05 flops they issue to a device counter.  Off by default: a disabled scope is one load.
enum ProfFamily { PF_TC_FWD = 0, PF_TC_BWD, PF_TC_PREP, PF_SIMT, PF_SMALL, PF_AUX, PF_COUNT };
inline const char* prof_name(int f) {
  static const char* n[PF_COUNT] = {"tc_fwd_kernel", "tc_bwd_kernel", "tc_prep (shift/prep/colbias/rowterm)",
                                    "simt", "small_kernel", "aux (unary/final/pad/iwae/sampler)"};
  return n[f];
}
struct Profiler {
  std::mutex mu;
  bool on = false;
  std::vector<cudaEvent_t> pool;   // reused across sessions
  size_t used = 0;
  struct Rec { int fam; cudaEvent_t a, b; };
  std::vector<Rec> recs;
};
inline Profiler& profiler() {
  static Profiler p;
  return p;
}
inline bool prof_on() { return profiler().on; }
struct ProfScope {
  int fam;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  NvtxRange nvtx;
  ProfScope(int fam_, cudaStream_t s_) : fam(fam_), s(s_), nvtx(prof_name(fam_)) {
    Profiler& p = profiler();
    if (!p.on) return;
    std::lock_guard<std::mutex> lk(p.mu);
    while (p.pool.size() < p.used + 2) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      p.pool.push_back(e);
    }
    a = p.pool[p.used++];
    b = p.pool[p.used++];
    cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!a) return;
    Profiler& p = profiler();
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(p.mu);
    p.recs.push_back({fam, a, b});
  }
};

constexpr float kLog2Pi = 1.8378770664093453f;
constexpr float kLog2E = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// One edge contraction ("pass") of the message pass.  Rows are the index that is kept,
// columns the index that is summed.  The pair log-factor is
//   g[r,c] = log N(z_a ; mu_p, diag exp(v_p))           (Gaussian path)
//          = logf[b][a][p]                               (dense path)
// with (a, p) = (r, c) if zrows else (c, r).
struct PassArgs {
  int B, R, C, D;
  int Kz, Kp;                  // leading sizes of z [B][Kz][D] and mu/logvar [B][Kp][D]
  const float *z, *mu, *lv;    // Gaussian inputs
  const float *logf;           // dense [B][Kz][Kp] (or NULL)
  const float *cb;             // [B][C] column bias (messages from the summed side)
  const float *rb;             // [B][R] row add (unary of the kept side) or NULL
  float *cbmax;                // [B] max_c cb (forward writes, backward reads)
  float *out, *ell;            // [B][R] message out (= rb + ell - lnC), row LSE (saved)
  const double *off_cb, *off_rb;  // [B] fp64 offsets carried by cb / rb (NULL = 0)
  double *off_out;             // [B] offset of `out`
  float lnC;                   // ln(#columns): the 1/K of the summed index
  float alpha;                 // factor power: pair log-factor used = alpha * logf (1 = the TMC estimate)
  const float *w;              // [B][R] upstream gradient of out (backward)
  float *colsum;               // [B][C] sum_r P[r,c] (backward, column owner)
  float *gz, *gmu, *glv;       // owner-side gradient outputs (overwritten)
  float *pair;                 // [B][Kz][Kp] pair marginals / dlogf (row owner) or NULL
};

struct UnaryDesc {            // per-latent unary preparation
  const float *logobs, *logq; // [B][K] (either may be NULL)
  float *u;                   // [B][K] out: (logobs - max_a logobs) - logq
  double *uoff;               // [B]   out: max_a logobs (0 if absent / all -inf)
  int K;
};
constexpr int kMaxUnaryPerLaunch = 48;
struct UnaryBatch { UnaryDesc d[kMaxUnaryPerLaunch]; int count; int B; float alpha; };

constexpr int kMaxChildren = 24;
struct HBuild {               // h_i = u_i + sum_children msg_j   (UP direction)
  const float *u; const double *uoff;
  const float *msg[kMaxChildren]; const double *moff[kMaxChildren];
  int nchild; int B, K;
  float *h; double *hoff;
};

struct UnaryGradDesc { const float *pi; float *dlogq, *dlogobs; int K; };
struct UnaryGradBatch { UnaryGradDesc d[kMaxUnaryPerLaunch]; int count; int B; float alpha; };

constexpr int kMaxRoots = 16;
struct RootList { const float *out[kMaxRoots]; const double *off[kMaxRoots]; float *w[kMaxRoots]; int count; int B; };

}  // namespace tmc
