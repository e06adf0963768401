// Internal structures shared by the libtmc host code and kernels (NOT part of the ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmc {

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
