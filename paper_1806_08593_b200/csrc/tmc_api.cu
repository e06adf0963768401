// libtmc host side: validation, workspace plan, and the launch schedule of the TMC message pass.
// The ABI is declared (and documented) in include/tmc.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tmc.h"
#include "tmc_internal.h"
#include "tmc_elim.cuh"
#include "tmc_iwae.cuh"
#include "tmc_sample.cuh"
#include "tmc_simt.cuh"
#include "tmc_tc.cuh"
#include "tmc_small.cuh"
#include "tmc_bwd1.cuh"

namespace tmc {
namespace {
// Default tensor-core reverse pass (measured): the two owner passes until the single
// pass is faster on the bench configurations.
constexpr bool kDefaultTwoPassReverse = true;

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
#define TMC_COUNT_LAUNCH() g_launches.fetch_add(1, std::memory_order_relaxed)

tmc_status fail(tmc_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

// ------------------------------------------------------------------------------------ plan
struct EdgeBuf {
  int R = 0, C = 0;
  size_t out = 0, ell = 0, cbmax = 0, off = 0, h = 0, hoff = 0, w = 0, colsum = 0;
};

struct Plan {
  int n = 0, B = 0, dir = 0, prec = 0;
  int requested_prec = 0;          // the caller's tmc_precision (prec is the resolved path)
  int requested_dir = 0;           // the caller's tmc_direction (dir is the resolved one)
  float alpha = 1.f;
  bool dense = false;
  bool dense_reverse = false;      // TMC_FLAG_DENSE_REVERSE: no zero-weight tile skipping
  bool two_pass_reverse = false;   // TMC_FLAG_TWO_PASS_REVERSE: two owner passes instead of one
  std::vector<int> parent, K, D, Kp;
  std::vector<std::vector<int>> children;
  std::vector<int> roots;
  std::vector<EdgeBuf> e;
  std::vector<size_t> u, uoff;
  size_t zero = 0, lse = 0, flag = 0;
  std::vector<TcLatentBuf> tc;   // tensor-core operand buffers (per latent), empty for SIMT
  // Tensor-core padding: a non-root latent whose D is not 32/64 (D < 64) is run on the D' = 32/64
  // tensor-core path from zero-padded copies of its inputs in the workspace (padded dims: z = mu = 0,
  // logvar = -ln 2 pi, so each contributes log N(0; 0, 1/(2 pi)) = 0 exactly to every pair), and its
  // gradients are copied back unpadded.  Din = the caller's D; D = the internal (padded) one.
  std::vector<int> Din;
  std::vector<size_t> pz, pmu, plv, pgz, pgmu, pglv;
  bool any_pad = false;
  size_t total = 0;
};

size_t carve(size_t& cur, size_t bytes) {
  size_t at = (cur + 255) & ~size_t(255);
  cur = at + bytes;
  return at;
}

bool is_chain(const std::vector<int>& parent) {
  for (size_t i = 0; i < parent.size(); ++i)
    if (parent[i] != (int)i - 1) return false;
  return true;
}

tmc_status make_plan(const tmc_graph* g, bool dense, Plan& p) {
  if (!g) return fail(TMC_ERR_INVALID_ARG, "graph is NULL");
  if (g->n <= 0) return fail(TMC_ERR_SHAPE, "n must be >= 1");
  if (g->B < 0) return fail(TMC_ERR_SHAPE, "B must be >= 0");
  if (!g->parent || !g->K || !g->D) return fail(TMC_ERR_INVALID_ARG, "graph parent/K/D arrays must be non-NULL");
  if (g->direction < 0 || g->direction > 2) return fail(TMC_ERR_INVALID_ARG, "bad direction");
  if (g->precision < 0 || g->precision > 2) return fail(TMC_ERR_INVALID_ARG, "bad precision");
  p.n = g->n;
  p.B = g->B;
  if (!(g->factor_power >= 0.f) || g->factor_power > 64.f)
    return fail(TMC_ERR_INVALID_ARG, "factor_power must be in [0, 64] (0 = 1)");
  p.alpha = g->factor_power == 0.f ? 1.f : g->factor_power;
  p.dense = dense;
  p.dense_reverse = (g->flags & TMC_FLAG_DENSE_REVERSE) != 0;
  if ((g->flags & TMC_FLAG_TWO_PASS_REVERSE) && (g->flags & TMC_FLAG_SINGLE_PASS_REVERSE))
    return fail(TMC_ERR_INVALID_ARG, "TMC_FLAG_TWO_PASS_REVERSE and TMC_FLAG_SINGLE_PASS_REVERSE are exclusive");
  p.two_pass_reverse = (g->flags & TMC_FLAG_SINGLE_PASS_REVERSE) ? false
                       : (g->flags & TMC_FLAG_TWO_PASS_REVERSE) ? true : kDefaultTwoPassReverse;
  p.parent.assign(g->parent, g->parent + g->n);
  p.K.assign(g->K, g->K + g->n);
  p.D.assign(g->D, g->D + g->n);
  p.Din = p.D;
  p.children.assign(p.n, {});
  for (int i = 0; i < p.n; ++i) {
    if (p.K[i] <= 0) return fail(TMC_ERR_SHAPE, "K[" + std::to_string(i) + "] must be >= 1");
    if (p.D[i] <= 0) return fail(TMC_ERR_SHAPE, "D[" + std::to_string(i) + "] must be >= 1");
    if (!dense && p.D[i] > 256 && g->precision != TMC_PREC_TC)
      return fail(TMC_ERR_SHAPE, "SIMT path supports D <= 256");
    if (p.parent[i] < -1 || p.parent[i] >= i)
      return fail(TMC_ERR_GRAPH, "parent[" + std::to_string(i) + "] must satisfy -1 <= parent[i] < i");
    if (p.parent[i] >= 0) p.children[p.parent[i]].push_back(i);
    else p.roots.push_back(i);
  }
  if ((int)p.roots.size() > kMaxRoots) return fail(TMC_ERR_GRAPH, "too many roots");
  p.Kp.resize(p.n);
  for (int i = 0; i < p.n; ++i) p.Kp[i] = p.parent[i] < 0 ? 1 : p.K[p.parent[i]];
  const bool chain = is_chain(p.parent);
  p.dir = g->direction == TMC_DIR_AUTO ? (chain ? TMC_DIR_DOWN : TMC_DIR_UP) : g->direction;
  if (p.dir == TMC_DIR_DOWN && !chain) return fail(TMC_ERR_GRAPH, "TMC_DIR_DOWN requires a chain (parent[i] == i-1)");
  // tensor-core padding of small / odd D (large K only under AUTO; any K when TC is requested)
  if (!dense && g->precision != TMC_PREC_SIMT)
    for (int i = 0; i < p.n; ++i)
      if (p.parent[i] >= 0 && p.D[i] < 64 && p.D[i] != 32 &&
          (g->precision == TMC_PREC_TC || (p.K[i] >= 128 && p.Kp[i] >= 128))) {
        p.D[i] = p.D[i] < 32 ? 32 : 64;
        p.any_pad = true;
      }
  // precision
  p.requested_prec = g->precision;
  p.requested_dir = g->direction;
  p.prec = TMC_PREC_SIMT;
  if (!dense && g->precision != TMC_PREC_SIMT) {
    bool ok = tc_supported(p.parent, p.K, p.D);
    if (g->precision == TMC_PREC_TC && !ok)
      return fail(TMC_ERR_SHAPE, "TMC_PREC_TC needs D_i <= 64 on some non-root latent");
    if (ok) p.prec = TMC_PREC_TC;
  }

  const size_t B = (size_t)std::max(p.B, 1);
  size_t cur = 0;
  p.e.resize(p.n);
  p.u.resize(p.n);
  p.uoff.resize(p.n);
  for (int i = 0; i < p.n; ++i) {
    p.u[i] = carve(cur, 4 * B * p.K[i]);
    p.uoff[i] = carve(cur, 8 * B);
  }
  for (int i = 0; i < p.n; ++i) {
    EdgeBuf& e = p.e[i];
    if (p.dir == TMC_DIR_DOWN) { e.R = p.K[i]; e.C = p.Kp[i]; }
    else { e.R = p.Kp[i]; e.C = p.K[i]; }
    e.out = carve(cur, 4 * B * e.R);
    e.ell = carve(cur, 4 * B * e.R);
    e.cbmax = carve(cur, 4 * B);
    e.off = carve(cur, 8 * B);
    e.w = carve(cur, 4 * B * e.R);
    e.colsum = carve(cur, 4 * B * e.C);
    if (p.dir == TMC_DIR_UP) {
      e.h = carve(cur, 4 * B * e.C);
      e.hoff = carve(cur, 8 * B);
    }
  }
  p.zero = carve(cur, 4 * B);
  p.lse = carve(cur, 4 * B);
  p.flag = carve(cur, 16);
  if (p.prec == TMC_PREC_TC) tc_plan(p.parent, p.K, p.D, p.Kp, p.B, p.dir, cur, p.tc);
  p.pz.assign(p.n, 0); p.pmu.assign(p.n, 0); p.plv.assign(p.n, 0);
  p.pgz.assign(p.n, 0); p.pgmu.assign(p.n, 0); p.pglv.assign(p.n, 0);
  if (p.prec == TMC_PREC_TC)
    for (int i = 0; i < p.n; ++i)
      if (p.D[i] != p.Din[i]) {
        const size_t zk = 4 * B * p.K[i] * p.D[i], mk = 4 * B * p.Kp[i] * p.D[i];
        p.pz[i] = carve(cur, zk); p.pmu[i] = carve(cur, mk); p.plv[i] = carve(cur, mk);
        p.pgz[i] = carve(cur, zk); p.pgmu[i] = carve(cur, mk); p.pglv[i] = carve(cur, mk);
      }
  if (p.prec != TMC_PREC_TC) { p.D = p.Din; p.any_pad = false; }   // padding only serves the TC path
  p.total = (cur + 255) & ~size_t(255);
  return TMC_OK;
}

// ------------------------------------------------------------------------------------ device
tmc_status check_device() {
  static int cached[64];
  static std::once_flag once;
  std::call_once(once, [] { for (int& c : cached) c = -1; });
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(TMC_ERR_UNSUPPORTED_DEVICE, "no CUDA device");
  if (dev < 0 || dev >= 64) return fail(TMC_ERR_UNSUPPORTED_DEVICE, "device index out of range");
  if (cached[dev] < 0) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cached[dev] = major * 10 + minor;
  }
  if (cached[dev] != 100)
    return fail(TMC_ERR_UNSUPPORTED_DEVICE, "libtmc is built for sm_100a (B200); device cc = " +
                                                std::to_string(cached[dev] / 10) + "." + std::to_string(cached[dev] % 10));
  return TMC_OK;
}

tmc_status launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TMC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return TMC_OK;
}

template <typename T>
T* at(void* ws, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(ws) + off); }

// ------------------------------------------------------------------------------------ SIMT pass dispatch
template <bool ZR, int MODE, bool DENSE, int MAXDL>
void launch_pass_t(const PassArgs& a, cudaStream_t s) {
  const int NO = (MODE != 2) ? a.R : a.C;
  const size_t smem = simt::pass_smem_bytes(a.D, DENSE);
  auto kern = simt::pass_kernel<ZR, MODE, DENSE, MAXDL>;
  static bool attr[kMaxDevices] = {};
  ensure_smem_attr(kern, 200 * 1024, attr);
  dim3 grid((NO + simt::kOPC - 1) / simt::kOPC, a.B);
  ProfScope ps(PF_SIMT, s);
  kern<<<grid, simt::kThreads, smem, s>>>(a);
    TMC_COUNT_LAUNCH();
}

template <bool ZR, int MODE>
void launch_pass_m(const PassArgs& a, bool dense, cudaStream_t s) {
  if (dense) return launch_pass_t<ZR, MODE, true, 1>(a, s);
  if (a.D == 1) return launch_pass_t<ZR, MODE, false, -1>(a, s);
  if (a.D <= 4) return launch_pass_t<ZR, MODE, false, 0>(a, s);
  if (a.D <= 32) return launch_pass_t<ZR, MODE, false, 1>(a, s);
  if (a.D <= 64) return launch_pass_t<ZR, MODE, false, 2>(a, s);
  if (a.D <= 128) return launch_pass_t<ZR, MODE, false, 4>(a, s);
  return launch_pass_t<ZR, MODE, false, 8>(a, s);
}

void launch_pass(const PassArgs& a, bool zrows, int mode, bool dense, cudaStream_t s) {
  if (a.B == 0) return;
  if (zrows && !dense && a.C == 1) {   // root of a DOWN chain: K x 1 pair matrix (prior)
    const unsigned grid = (unsigned)(((int64_t)a.B * a.R + 255) / 256);
    ProfScope ps(PF_SIMT, s);
    if (mode == 0) simt::root_down_fwd_kernel<<<grid, 256, 0, s>>>(a);
    else if (mode == 1) simt::root_down_row_kernel<<<grid, 256, 0, s>>>(a);
    else simt::root_down_col_kernel<<<a.B, 256, 0, s>>>(a);
    TMC_COUNT_LAUNCH();
    return;
  }
  if (zrows) {
    if (mode == 0) launch_pass_m<true, 0>(a, dense, s);
    else if (mode == 1) launch_pass_m<true, 1>(a, dense, s);
    else launch_pass_m<true, 2>(a, dense, s);
  } else {
    if (mode == 0) launch_pass_m<false, 0>(a, dense, s);
    else if (mode == 1) launch_pass_m<false, 1>(a, dense, s);
    else launch_pass_m<false, 2>(a, dense, s);
  }
}

template <bool ZR, int MODE, bool DENSE, int MAXDL>
void launch_pass_batch_t(const PassArgs* as, int ne, cudaStream_t s) {
  auto kern = simt::pass_batch_kernel<ZR, MODE, DENSE, MAXDL>;
  static bool attr[kMaxDevices] = {};
  ensure_smem_attr(kern, 200 * 1024, attr);
  for (int e0 = 0; e0 < ne; e0 += simt::kMaxPassBatch) {
    simt::PassBatch pb{};
    const int n = std::min(simt::kMaxPassBatch, ne - e0);
    int maxNO = 0, maxD = 1;
    for (int k = 0; k < n; ++k) {
      pb.e[k] = as[e0 + k];
      maxNO = std::max(maxNO, MODE != 2 ? pb.e[k].R : pb.e[k].C);
      maxD = std::max(maxD, pb.e[k].D);
    }
    dim3 grid((maxNO + simt::kOPC - 1) / simt::kOPC, as[0].B, n);
    ProfScope ps(PF_SIMT, s);
    kern<<<grid, simt::kThreads, simt::pass_smem_bytes(maxD, DENSE), s>>>(pb);
    TMC_COUNT_LAUNCH();
  }
}

template <int MODE, bool DENSE, int MAXDL>
void launch_pass_batch_c(const std::vector<PassArgs>& v, cudaStream_t s) {
  if (!v.empty()) launch_pass_batch_t<false, MODE, DENSE, MAXDL>(v.data(), (int)v.size(), s);
}

template <int MODE>
void launch_pass_batch_m(const std::vector<PassArgs>& as, bool dense, cudaStream_t s) {
  if (dense) return launch_pass_batch_c<MODE, true, 1>(as, s);
  std::vector<PassArgs> cls[6];
  for (const PassArgs& a : as) cls[a.D == 1 ? 5 : a.D <= 4 ? 4 : a.D <= 32 ? 0 : a.D <= 64 ? 1 : a.D <= 128 ? 2 : 3].push_back(a);
  launch_pass_batch_c<MODE, false, -1>(cls[5], s);
  launch_pass_batch_c<MODE, false, 0>(cls[4], s);
  launch_pass_batch_c<MODE, false, 1>(cls[0], s);
  launch_pass_batch_c<MODE, false, 2>(cls[1], s);
  launch_pass_batch_c<MODE, false, 4>(cls[2], s);
  launch_pass_batch_c<MODE, false, 8>(cls[3], s);
}

// SIMT passes of the independent edges of one UP level (rows = parent samples), batched.
void launch_pass_batch(const std::vector<PassArgs>& as, int mode, bool dense, cudaStream_t s) {
  if (as.empty() || as[0].B == 0) return;
  if (mode == 0) launch_pass_batch_m<0>(as, dense, s);
  else if (mode == 1) launch_pass_batch_m<1>(as, dense, s);
  else launch_pass_batch_m<2>(as, dense, s);
}

// Common PassArgs of edge i (inputs, geometry, forward state).
PassArgs edge_args(const Plan& p, int i, const tmc_latent_in* in, const float* const* dense, void* ws) {
  PassArgs a{};
  const EdgeBuf& e = p.e[i];
  a.B = p.B; a.R = e.R; a.C = e.C; a.D = p.D[i];
  a.Kz = p.K[i]; a.Kp = p.Kp[i];
  a.alpha = p.alpha;
  if (dense) a.logf = dense[i];
  else { a.z = in[i].z; a.mu = in[i].mu; a.lv = in[i].logvar; }
  a.cbmax = at<float>(ws, e.cbmax);
  a.out = at<float>(ws, e.out);
  a.ell = at<float>(ws, e.ell);
  a.off_out = at<double>(ws, e.off);
  if (p.dir == TMC_DIR_DOWN) {
    const int par = p.parent[i];
    a.cb = par < 0 ? at<float>(ws, p.zero) : at<float>(ws, p.e[par].out);
    a.off_cb = par < 0 ? nullptr : at<double>(ws, p.e[par].off);
    a.rb = at<float>(ws, p.u[i]);
    a.off_rb = at<double>(ws, p.uoff[i]);
    a.lnC = par < 0 ? 0.f : std::log((float)p.Kp[i]);
  } else {
    // h_i = u_i + child messages; a non-root leaf's h is its unary (no copy is built)
    const bool leaf = p.children[i].empty() && p.parent[i] >= 0;   // roots keep h (shared-root exchange)
    a.cb = leaf ? at<float>(ws, p.u[i]) : at<float>(ws, e.h);
    a.off_cb = leaf ? at<double>(ws, p.uoff[i]) : at<double>(ws, e.hoff);
    a.rb = nullptr;
    a.off_rb = nullptr;
    a.lnC = std::log((float)p.K[i]);
  }
  return a;
}

tmc_status check_inputs(const Plan& p, const tmc_latent_in* in, const float* const* dense) {
  if (!in && !dense) return fail(TMC_ERR_INVALID_ARG, "inputs are NULL");
  if (p.B == 0) return TMC_OK;            // an empty batch reads no input (empty tensors may be NULL)
  for (int i = 0; i < p.n; ++i) {
    if (dense) {
      if (!dense[i]) return fail(TMC_ERR_INVALID_ARG, "logf_dense[" + std::to_string(i) + "] is NULL");
      continue;
    }
    if (!in[i].z || !in[i].mu || !in[i].logvar || !in[i].logq)
      return fail(TMC_ERR_INVALID_ARG, "latent " + std::to_string(i) + ": z/mu/logvar/logq must be non-NULL");
    if (p.prec == TMC_PREC_TC && p.D[i] == p.Din[i]) {      // padded latents are copied (no alignment need)
      for (const void* q : {(const void*)in[i].z, (const void*)in[i].mu, (const void*)in[i].logvar})
        if (reinterpret_cast<uintptr_t>(q) % 16)
          return fail(TMC_ERR_ALIGNMENT, "tensor-core path needs 16-byte aligned z/mu/logvar");
    }
  }
  return TMC_OK;
}

tmc_status validate_inputs(const Plan& p, const tmc_latent_in* in, const float* const* dense, void* ws,
                           cudaStream_t s) {
  int* flag = at<int>(ws, p.flag);
  cudaMemsetAsync(flag, 0, sizeof(int), s);
  auto scan = [&](const float* x, int64_t n, int allow) {
    if (x && n > 0) simt::validate_kernel<<<256, 256, 0, s>>>(x, n, allow, flag);
    TMC_COUNT_LAUNCH();
  };
  const int64_t B = p.B;
  for (int i = 0; i < p.n; ++i) {
    if (dense) { scan(dense[i], B * p.K[i] * p.Kp[i], 1); }
    else {
      scan(in[i].z, B * p.K[i] * p.Din[i], 0);
      scan(in[i].mu, B * p.Kp[i] * p.Din[i], 0);
      scan(in[i].logvar, B * p.Kp[i] * p.Din[i], 0);
      scan(in[i].logq, B * p.K[i], 1);
    }
    if (in && in[i].logobs) scan(in[i].logobs, B * p.K[i], 1);
  }
  int host = 0;
  cudaMemcpyAsync(&host, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return launch_check("validate");
  if (host) return fail(TMC_ERR_NONFINITE, "NaN or +inf (or -inf in z/mu/logvar) found in an input");
  return TMC_OK;
}

// ------------------------------------------------------------------------------- padding
bool padded(const Plan& p, int i) { return p.prec == TMC_PREC_TC && p.D[i] != p.Din[i]; }

void launch_pad(const std::vector<simt::PadDesc>& jobs, int unpad, cudaStream_t s) {
  for (size_t j0 = 0; j0 < jobs.size(); j0 += simt::kMaxPad) {
    simt::PadBatch pb{};
    pb.count = (int)std::min<size_t>(simt::kMaxPad, jobs.size() - j0);
    int64_t mx = 1;
    for (int k = 0; k < pb.count; ++k) {
      pb.d[k] = jobs[j0 + k];
      mx = std::max<int64_t>(mx, pb.d[k].rows * (unpad ? pb.d[k].Di : pb.d[k].Dt / 4));
    }
    const unsigned gx = (unsigned)std::min<int64_t>((mx + 255) / 256, 1024);
    ProfScope ps(PF_AUX, s);
    simt::pad_batch_kernel<<<dim3(gx, pb.count), 256, 0, s>>>(pb, unpad);
    TMC_COUNT_LAUNCH();
  }
}

// The inputs the kernels see: padded latents point at their workspace copies (filled when
// `fill`, i.e. on the forward; the reverse pass reuses the forward's copies).
std::vector<tmc_latent_in> kernel_inputs(const Plan& p, const tmc_latent_in* in, void* ws, cudaStream_t s, bool fill) {
  std::vector<tmc_latent_in> v(in, in + p.n);
  if (!p.any_pad) return v;
  std::vector<simt::PadDesc> jobs;
  for (int i = 0; i < p.n; ++i) {
    if (!padded(p, i)) continue;
    float* z = at<float>(ws, p.pz[i]);
    float* mu = at<float>(ws, p.pmu[i]);
    float* lv = at<float>(ws, p.plv[i]);
    const int64_t rz = (int64_t)p.B * p.K[i], rm = (int64_t)p.B * p.Kp[i];
    jobs.push_back({in[i].z, z, rz, p.Din[i], p.D[i], 0.f});
    jobs.push_back({in[i].mu, mu, rm, p.Din[i], p.D[i], 0.f});
    jobs.push_back({in[i].logvar, lv, rm, p.Din[i], p.D[i], -1.8378770664093453f});   // -ln(2 pi): adds exactly 0
    v[i].z = z; v[i].mu = mu; v[i].logvar = lv;
  }
  if (fill && p.B > 0) launch_pad(jobs, 0, s);
  return v;
}

// Gradient outputs the kernels write: padded latents write into workspace buffers (copied back
// unpadded by unpad_outputs).
std::vector<tmc_latent_grad> kernel_outputs(const Plan& p, const tmc_latent_grad* out, void* ws) {
  std::vector<tmc_latent_grad> v(p.n);
  for (int i = 0; i < p.n; ++i) {
    v[i] = out ? out[i] : tmc_latent_grad{};
    if (!out || !padded(p, i)) continue;
    if (out[i].dz) v[i].dz = at<float>(ws, p.pgz[i]);
    if (out[i].dmu) v[i].dmu = at<float>(ws, p.pgmu[i]);
    if (out[i].dlogvar) v[i].dlogvar = at<float>(ws, p.pglv[i]);
  }
  return v;
}

void unpad_outputs(const Plan& p, const tmc_latent_grad* out, void* ws, cudaStream_t s) {
  if (!out || !p.any_pad || p.B == 0) return;
  std::vector<simt::PadDesc> jobs;
  for (int i = 0; i < p.n; ++i) {
    if (!padded(p, i)) continue;
    const int64_t rz = (int64_t)p.B * p.K[i], rm = (int64_t)p.B * p.Kp[i];
    if (out[i].dz) jobs.push_back({at<float>(ws, p.pgz[i]), out[i].dz, rz, p.Din[i], p.D[i], 0.f});
    if (out[i].dmu) jobs.push_back({at<float>(ws, p.pgmu[i]), out[i].dmu, rm, p.Din[i], p.D[i], 0.f});
    if (out[i].dlogvar) jobs.push_back({at<float>(ws, p.pglv[i]), out[i].dlogvar, rm, p.Din[i], p.D[i], 0.f});
  }
  launch_pad(jobs, 1, s);
}

// ------------------------------------------------------------------------------------ forward
// Small problems (K_i <= 64, D_i <= 128, n <= 32; TMC_PREC_AUTO and TMC_DIR_AUTO, Gaussian path):
// one CTA per datapoint does the whole forward (mode 0) or forward + reverse (mode 1) in one
// launch.  An explicit direction or precision selects the general kernels (the shared-root
// exchange requires TMC_DIR_UP, so its backward never recomputes a shard-local forward here).
bool small_ok(const Plan& p, bool dense, small::Args* A, const tmc_latent_in* in, const tmc_latent_grad* out,
              double* logp, const double* dlogp, int mode) {
  if (dense || p.requested_prec != TMC_PREC_AUTO || p.requested_dir != TMC_DIR_AUTO || p.n > small::kMaxN)
    return false;
  for (int i = 0; i < p.n; ++i)
    if (p.K[i] > small::kMaxK || p.Kp[i] > small::kMaxK || p.D[i] > small::kMaxD) return false;
  if (!A) return true;
  *A = small::Args{};
  A->n = p.n; A->B = p.B; A->mode = mode; A->alpha = p.alpha; A->dlogp = dlogp; A->logp = logp;
  for (int i = 0; i < p.n; ++i) {
    small::Lat& L = A->l[i];
    L.z = in[i].z; L.mu = in[i].mu; L.lv = in[i].logvar; L.logq = in[i].logq; L.logobs = in[i].logobs;
    if (out) {
      L.gz = out[i].dz; L.gmu = out[i].dmu; L.glv = out[i].dlogvar; L.gq = out[i].dlogq; L.go = out[i].dlogobs;
      L.pair = out[i].pair_marginal;
    }
    L.K = p.K[i]; L.Kp = p.Kp[i]; L.D = p.D[i]; L.parent = p.parent[i]; L.lnK = std::log((double)p.K[i]);
  }
  A->cache = 0;
  if (small::smem_bytes(*A) > 160 * 1024) return false;
  // keep every latent's factor tile (one factor phase; the reverse sweep reuses them) if they fit
  A->cache = 1;
  if (small::smem_bytes(*A) > 160 * 1024) A->cache = 0;
  small::layout(*A);                          // the shared-memory offsets the kernel addresses by
  return true;
}

tmc_status launch_small(const small::Args& A, cudaStream_t s) {
  const size_t smem = small::smem_bytes(A);
  static bool attr[kMaxDevices] = {}, attr2[kMaxDevices] = {};
  ProfScope ps(PF_SMALL, s);
  if (small::large_work(A)) {
    ensure_smem_attr(small::small_kernel<small::kThreadsLarge>, 160 * 1024, attr2);
    small::small_kernel<small::kThreadsLarge><<<A.B, small::kThreadsLarge, smem, s>>>(A);
  } else {
    ensure_smem_attr(small::small_kernel<small::kThreadsSmall>, 160 * 1024, attr);
    small::small_kernel<small::kThreadsSmall><<<A.B, small::kThreadsSmall, smem, s>>>(A);
  }
  TMC_COUNT_LAUNCH();
  return launch_check("tmc (small-problem kernel)");
}

// phase: 0 = the whole forward; 1 = every latent below the (single) root, then the root's child
// messages summed into xout [B][K_root+1] (fp64 residual sums, then the offset sum); 2 = the root's
// elimination from h_root = u_root + xin (xin = the sum of phase-1 outputs over the shards of the
// root's children) and logp.  Phases 1 + 2 on one shard equal phase 0.
tmc_status forward_impl(const Plan& p, const tmc_latent_in* in, const float* const* dense, double* logp,
                        void* ws, cudaStream_t s, int phase = 0, double* xout = nullptr,
                        const double* xin = nullptr) {
  if (p.B == 0) return TMC_OK;
  if (phase == 0) {
    small::Args A;
    if (small_ok(p, dense != nullptr, &A, in, nullptr, logp, nullptr, 0)) return launch_small(A, s);
  }
  // unary prep (all latents)
  if (phase != 2)
  for (int i0 = 0; i0 < p.n; i0 += kMaxUnaryPerLaunch) {
    UnaryBatch ub{};
    ub.B = p.B;
    ub.alpha = p.alpha;
    ub.count = std::min(kMaxUnaryPerLaunch, p.n - i0);
    for (int j = 0; j < ub.count; ++j) {
      int i = i0 + j;
      ub.d[j].logobs = in ? in[i].logobs : nullptr;
      ub.d[j].logq = dense ? nullptr : in[i].logq;
      ub.d[j].u = at<float>(ws, p.u[i]);
      ub.d[j].uoff = at<double>(ws, p.uoff[i]);
      ub.d[j].K = p.K[i];
    }
    ProfScope ps(PF_AUX, s);
    simt::unary_prep_kernel<<<dim3(p.B, ub.count), 256, 0, s>>>(ub);
    TMC_COUNT_LAUNCH();
  }
  if (p.dir == TMC_DIR_DOWN) {
    cudaMemsetAsync(at<float>(ws, p.zero), 0, 4 * (size_t)p.B, s);
    for (int i = 0; i < p.n; ++i) {
      PassArgs a = edge_args(p, i, in, dense, ws);
      if (p.prec == TMC_PREC_TC && tc_edge_ok(p.tc[i])) {
        // centre on the parent's filtering weights m_pa (predicted location of z_i)
        g_launches.fetch_add(tc_prep_edge(p.K[i], p.Kp[i], p.D[i], p.B, in[i], ws, p.tc[i],
                                          at<float>(ws, p.e[p.parent[i]].out), p.Kp[i], 0, p.alpha, s));
        g_launches.fetch_add(tc_pass_forward(a, p.tc[i], ws, /*zrows=*/true, s));
      }
      else launch_pass(a, /*zrows=*/true, 0, dense != nullptr, s);
    }
    const EdgeBuf& last = p.e[p.n - 1];
    ProfScope ps(PF_AUX, s);
    simt::final_down_fwd_kernel<<<p.B, 256, 0, s>>>(at<float>(ws, last.out), at<double>(ws, last.off),
                                                     p.K[p.n - 1], std::log((float)p.K[p.n - 1]),
                                                     at<float>(ws, p.lse), logp);
    TMC_COUNT_LAUNCH();
  } else {
    // Leaves -> roots by height (height 0 = leaf); the edges of one height are independent, so
    // their tensor-core contractions (same D) run as ONE batched persistent launch.
    std::vector<int> height(p.n, 0);
    int maxh = 0;
    for (int i = p.n - 1; i >= 0; --i) {
      for (int c : p.children[i]) height[i] = std::max(height[i], height[c] + 1);
      maxh = std::max(maxh, height[i]);
    }
    const int root0 = p.roots.empty() ? 0 : p.roots[0];
    for (int h = 0; h <= maxh; ++h) {
      if ((phase == 1 && h == maxh) || (phase == 2 && h < maxh)) continue;
      std::vector<int> level;
      for (int i = p.n - 1; i >= 0; --i)
        if (height[i] == h) level.push_back(i);
      std::vector<PassArgs> tcA;
      std::vector<const TcLatentBuf*> tcT;
      int tcD = 0;
      std::vector<PrepJob> prepJ;
      std::vector<PassArgs> simtA;
      auto flush_tc = [&]() {
        if (!tcA.empty()) {
          g_launches.fetch_add(tc_prep_batch(prepJ.data(), (int)prepJ.size(), p.B, ws, s));
          g_launches.fetch_add(tc_pass_forward_batch(tcA.data(), tcT.data(), (int)tcA.size(), ws, false, s));
        }
        tcA.clear();
        tcT.clear();
        prepJ.clear();
      };
      for (int i : level) {
        // h_i = u_i + sum of child messages
        const std::vector<int>& ch = p.children[i];
        int done = 0;
        if (phase == 2 && i == root0) {
          simt::hroot_kernel<<<dim3((p.K[i] + 255) / 256, p.B), 256, 0, s>>>(
              at<float>(ws, p.u[i]), at<double>(ws, p.uoff[i]), xin, p.K[i], at<float>(ws, p.e[i].h),
              at<double>(ws, p.e[i].hoff));
          TMC_COUNT_LAUNCH();
          done = (int)ch.size();
        } else if (!ch.empty() || p.parent[i] < 0)
        do {
          HBuild hb{};
          hb.B = p.B; hb.K = p.K[i];
          hb.u = done == 0 ? at<float>(ws, p.u[i]) : at<float>(ws, p.e[i].h);
          hb.uoff = done == 0 ? at<double>(ws, p.uoff[i]) : at<double>(ws, p.e[i].hoff);
          hb.nchild = std::min<int>(kMaxChildren, (int)ch.size() - done);
          for (int j = 0; j < hb.nchild; ++j) {
            hb.msg[j] = at<float>(ws, p.e[ch[done + j]].out);
            hb.moff[j] = at<double>(ws, p.e[ch[done + j]].off);
          }
          hb.h = at<float>(ws, p.e[i].h);
          hb.hoff = at<double>(ws, p.e[i].hoff);
          ProfScope ps(PF_AUX, s);
          simt::hbuild_kernel<<<dim3((p.K[i] + 255) / 256, p.B), 256, 0, s>>>(hb);
          TMC_COUNT_LAUNCH();
          done += hb.nchild;
        } while (done < (int)ch.size());
        PassArgs a = edge_args(p, i, in, dense, ws);
        if (p.prec == TMC_PREC_TC && tc_edge_ok(p.tc[i])) {
          // centre on softmax(h_i): z_i weighted by its subtree evidence
          if (!tcA.empty() && tcD != p.D[i]) flush_tc();
          tcD = p.D[i];
          tcA.push_back(a);
          tcT.push_back(&p.tc[i]);
          prepJ.push_back(PrepJob{p.K[i], p.Kp[i], p.D[i], &in[i], &p.tc[i], a.cb, p.K[i], 1, p.alpha});
        } else {
          simtA.push_back(a);
        }
      }
      flush_tc();
      launch_pass_batch(simtA, 0, dense != nullptr, s);
    }
    if (phase == 1) {
      // the root's incoming messages, summed over this shard's children (fp64)
      const std::vector<int>& ch = p.children[root0];
      for (int done = 0; done < (int)ch.size() || done == 0;) {
        HBuild hb{};
        hb.B = p.B; hb.K = p.K[root0];
        hb.nchild = std::min<int>(kMaxChildren, (int)ch.size() - done);
        for (int j = 0; j < hb.nchild; ++j) {
          hb.msg[j] = at<float>(ws, p.e[ch[done + j]].out);
          hb.moff[j] = at<double>(ws, p.e[ch[done + j]].off);
        }
        simt::xmsg_kernel<<<dim3((p.K[root0] + 1 + 255) / 256, p.B), 256, 0, s>>>(hb, xout, done == 0);
        TMC_COUNT_LAUNCH();
        done += std::max(hb.nchild, 1);
        if (done >= (int)ch.size()) break;
      }
      return launch_check("tmc_forward_children");
    }
    RootList rl{};
    rl.B = p.B;
    rl.count = (int)p.roots.size();
    for (int j = 0; j < rl.count; ++j) {
      rl.out[j] = at<float>(ws, p.e[p.roots[j]].out);
      rl.off[j] = at<double>(ws, p.e[p.roots[j]].off);
    }
    ProfScope ps(PF_AUX, s);
    simt::final_up_fwd_kernel<<<(p.B + 127) / 128, 128, 0, s>>>(rl, logp);
    TMC_COUNT_LAUNCH();
  }
  return launch_check("tmc_forward");
}

// ------------------------------------------------------------------------------------ backward
tmc_status backward_impl(const Plan& p, const tmc_latent_in* in, const float* const* dense, void* ws,
                         const double* dlogp, tmc_latent_grad* out, float* const* dlogf, cudaStream_t s) {
  if (p.B == 0) return TMC_OK;
  {
    // small problems: one launch that redoes the forward (logp into the workspace) and the reverse pass
    small::Args A;
    if (small_ok(p, dense != nullptr, &A, in, out, static_cast<double*>(ws), dlogp, 1)) return launch_small(A, s);
  }
  std::vector<const float*> pi(p.n);
  auto grad = [&](int i) -> tmc_latent_grad { return out ? out[i] : tmc_latent_grad{}; };
  if (p.dir == TMC_DIR_DOWN) {
    const int L = p.n - 1;
    {
      ProfScope ps(PF_AUX, s);
      simt::final_down_bwd_kernel<<<dim3((p.K[L] + 255) / 256, p.B), 256, 0, s>>>(
          at<float>(ws, p.e[L].out), at<float>(ws, p.lse), p.K[L], dlogp, at<float>(ws, p.e[L].w));
    }
    TMC_COUNT_LAUNCH();
    for (int i = L; i >= 0; --i) {
      PassArgs a = edge_args(p, i, in, dense, ws);
      tmc_latent_grad g = grad(i);
      a.w = at<float>(ws, p.e[i].w);
      // row owner (z side): dz_i and pair marginals
      a.gz = g.dz;
      a.pair = dense ? (dlogf ? dlogf[i] : nullptr) : g.pair_marginal;
      if (p.prec == TMC_PREC_TC && !p.two_pass_reverse && tc_bwd1_ok(p.tc[i], a)) {
        // single pass: dz, dmu, dlogvar and the parent edge's weights from one S / P~ per tile
        PassArgs f = a;
        f.gmu = g.dmu; f.glv = g.dlogvar;
        f.colsum = p.parent[i] >= 0 ? at<float>(ws, p.e[p.parent[i]].w) : at<float>(ws, p.e[i].colsum);
        const TcLatentBuf* tp = &p.tc[i];
        g_launches.fetch_add(tc_pass_backward1_batch(&f, &tp, 1, ws, true, p.dense_reverse, s));
        pi[i] = at<float>(ws, p.e[i].w);
        continue;
      }
      const bool tcb = p.prec == TMC_PREC_TC && tc_bwd_edge_ok(p.tc[i], a);
      if (tcb) g_launches.fetch_add(tc_pass_backward(a, p.tc[i], ws, true, 1, p.dense_reverse, s));
      else launch_pass(a, true, 1, dense != nullptr, s);
      // column owner (param side): colsum -> w of the parent edge; dmu_i, dlogvar_i
      a.gz = nullptr; a.pair = nullptr;
      a.gmu = g.dmu; a.glv = g.dlogvar;
      a.colsum = p.parent[i] >= 0 ? at<float>(ws, p.e[p.parent[i]].w) : at<float>(ws, p.e[i].colsum);
      if (tcb) g_launches.fetch_add(tc_pass_backward(a, p.tc[i], ws, true, 2, p.dense_reverse, s));
      else launch_pass(a, true, 2, dense != nullptr, s);
      pi[i] = at<float>(ws, p.e[i].w);
    }
  } else {
    RootList rl{};
    rl.B = p.B;
    rl.count = (int)p.roots.size();
    for (int j = 0; j < rl.count; ++j) rl.w[j] = at<float>(ws, p.e[p.roots[j]].w);
    {
      ProfScope ps(PF_AUX, s);
      simt::final_up_bwd_kernel<<<(p.B + 127) / 128, 128, 0, s>>>(rl, dlogp);
    }
    TMC_COUNT_LAUNCH();
    // Roots -> leaves by depth: an edge's row-owner pass needs its parent edge's column sums;
    // the edges of one depth are independent and run batched (same D) on tensor cores.
    std::vector<int> depth(p.n, 0);
    int maxd = 0;
    for (int i = 0; i < p.n; ++i) {
      depth[i] = p.parent[i] < 0 ? 0 : depth[p.parent[i]] + 1;
      maxd = std::max(maxd, depth[i]);
    }
    for (int dl = 0; dl <= maxd; ++dl) {
      std::vector<PassArgs> rowA, colA, simtRow, simtCol;
      std::vector<const TcLatentBuf*> tcT;
      std::vector<int> tcI;
      for (int i = 0; i < p.n; ++i) {
        if (depth[i] != dl) continue;
        PassArgs a = edge_args(p, i, in, dense, ws);
        tmc_latent_grad g = grad(i);
        a.w = p.parent[i] >= 0 ? at<float>(ws, p.e[p.parent[i]].colsum) : at<float>(ws, p.e[i].w);
        // row owner (param side): dmu_i, dlogvar_i, pair marginals
        a.gmu = g.dmu; a.glv = g.dlogvar;
        a.pair = dense ? (dlogf ? dlogf[i] : nullptr) : g.pair_marginal;
        PassArgs c = a;
        // column owner (z side): colsum = pi_i, dz_i
        c.gmu = nullptr; c.glv = nullptr; c.pair = nullptr;
        c.gz = g.dz;
        c.colsum = at<float>(ws, p.e[i].colsum);
        pi[i] = at<float>(ws, p.e[i].colsum);
        const bool tcb = p.prec == TMC_PREC_TC && tc_bwd_edge_ok(p.tc[i], a);
        if (tcb) {
          rowA.push_back(a);
          colA.push_back(c);
          tcT.push_back(&p.tc[i]);
          tcI.push_back(i);
        } else {
          simtRow.push_back(a);
          simtCol.push_back(c);
        }
      }
      launch_pass_batch(simtRow, 1, dense != nullptr, s);
      launch_pass_batch(simtCol, 2, dense != nullptr, s);
      // single-pass tensor-core reverse for the eligible edges of the level (one batched launch)
      {
        std::vector<PassArgs> fa;
        std::vector<const TcLatentBuf*> ft;
        for (size_t k = 0; k < tcI.size(); ++k) {
          if (p.two_pass_reverse || !tc_bwd1_ok(*tcT[k], rowA[k])) continue;
          PassArgs f = rowA[k];
          f.gz = colA[k].gz;
          f.colsum = colA[k].colsum;
          fa.push_back(f);
          ft.push_back(tcT[k]);
          tcT[k] = nullptr;                    // done
        }
        if (!fa.empty())
          g_launches.fetch_add(tc_pass_backward1_batch(fa.data(), ft.data(), (int)fa.size(), ws, false, p.dense_reverse, s));
      }
      // batched tensor-core passes, grouped by D (row-owner passes of the level, then column owners)
      for (int Dv : {32, 64}) {
        std::vector<PassArgs> ra, ca;
        std::vector<const TcLatentBuf*> tt;
        for (size_t k = 0; k < tcI.size(); ++k)
          if (tcT[k] && p.D[tcI[k]] == Dv) { ra.push_back(rowA[k]); ca.push_back(colA[k]); tt.push_back(tcT[k]); }
        if (ra.empty()) continue;
        g_launches.fetch_add(tc_pass_backward_batch(ra.data(), tt.data(), (int)ra.size(), ws, false, 1, p.dense_reverse, s));
        g_launches.fetch_add(tc_pass_backward_batch(ca.data(), tt.data(), (int)ca.size(), ws, false, 2, p.dense_reverse, s));
      }
    }
  }
  for (int i0 = 0; i0 < p.n; i0 += kMaxUnaryPerLaunch) {
    UnaryGradBatch gb{};
    gb.B = p.B;
    gb.alpha = p.alpha;
    gb.count = std::min(kMaxUnaryPerLaunch, p.n - i0);
    for (int j = 0; j < gb.count; ++j) {
      int i = i0 + j;
      tmc_latent_grad g = grad(i);
      gb.d[j].pi = pi[i];
      gb.d[j].dlogobs = g.dlogobs;
      gb.d[j].dlogq = dense ? nullptr : g.dlogq;
      gb.d[j].K = p.K[i];
    }
    ProfScope ps(PF_AUX, s);
    simt::unary_grad_kernel<<<dim3(std::min<int64_t>(((int64_t)p.B * 64 + 255) / 256, 1024), gb.count), 256, 0, s>>>(gb);
    TMC_COUNT_LAUNCH();
  }
  return launch_check("tmc_backward");
}

}  // namespace
}  // namespace tmc



// ====================================================================== general elimination (NEXT-4)
// tmc_elim_*: the TMC estimate of an arbitrary factor graph over sample indices by summing the
// indices out in a given order; see tmc_elim.cuh and include/tmc.h.
namespace tmc {
namespace {

struct ElimFac {
  std::vector<int> scope;     // variable ids, table layout order
  long long size = 1;         // entries per datapoint
  int user = -1;              // index into the caller's logf[] (-1: intermediate in the workspace)
  size_t tab = 0, off = 0, grad = 0, shift = 0;
};
struct ElimStepDesc {
  int v = 0;
  std::vector<int> in;        // factor ids
  int out = -1;
  std::vector<int> uni;       // union of the input scopes, ascending
};
struct ElimPlan {
  int nvar = 0, B = 0;
  std::vector<int> K;
  std::vector<ElimFac> facs;
  std::vector<ElimStepDesc> steps;
  std::vector<int> finals;    // 0-index factors left after the last step
  size_t total = 0;
};

tmc_status make_elim_plan(const tmc_factor_graph* g, ElimPlan& p) {
  if (!g) return fail(TMC_ERR_INVALID_ARG, "factor graph is NULL");
  if (g->nvar <= 0 || g->nfac <= 0) return fail(TMC_ERR_SHAPE, "nvar and nfac must be >= 1");
  if (g->B < 0 || g->B > 65535) return fail(TMC_ERR_SHAPE, "B must be in [0, 65535]");
  if (!g->K || !g->arity || !g->scope) return fail(TMC_ERR_INVALID_ARG, "K/arity/scope must be non-NULL");
  p.nvar = g->nvar;
  p.B = g->B;
  p.K.assign(g->K, g->K + g->nvar);
  for (int v = 0; v < p.nvar; ++v)
    if (p.K[v] <= 0) return fail(TMC_ERR_SHAPE, "K[" + std::to_string(v) + "] must be >= 1");
  for (int j = 0; j < g->nfac; ++j) {
    ElimFac f;
    const int a = g->arity[j];
    if (a < 1 || a > elim::kMaxArity) return fail(TMC_ERR_SHAPE, "factor arity must be in [1, 3]");
    for (int q = 0; q < a; ++q) {
      const int v = g->scope[j * elim::kMaxArity + q];
      if (v < 0 || v >= p.nvar) return fail(TMC_ERR_GRAPH, "factor " + std::to_string(j) + ": scope variable out of range");
      if (std::find(f.scope.begin(), f.scope.end(), v) != f.scope.end())
        return fail(TMC_ERR_GRAPH, "factor " + std::to_string(j) + ": repeated scope variable");
      f.scope.push_back(v);
      f.size *= p.K[v];
    }
    if (f.size > INT32_MAX) return fail(TMC_ERR_SHAPE, "factor table too large");
    f.user = j;
    p.facs.push_back(f);
  }
  std::vector<int> order(p.nvar);
  if (g->order) order.assign(g->order, g->order + p.nvar);
  else for (int v = 0; v < p.nvar; ++v) order[v] = v;
  {
    std::vector<int> seen(p.nvar, 0);
    for (int v : order) {
      if (v < 0 || v >= p.nvar || seen[v]) return fail(TMC_ERR_GRAPH, "order must be a permutation of 0..nvar-1");
      seen[v] = 1;
    }
  }
  const size_t B = (size_t)std::max(p.B, 1);
  size_t cur = 0;
  std::vector<int> live;                       // factor ids not yet consumed
  for (int j = 0; j < (int)p.facs.size(); ++j) live.push_back(j);
  for (int v : order) {
    ElimStepDesc st;
    st.v = v;
    std::vector<int> keep;
    for (int f : live) {
      const std::vector<int>& sc = p.facs[f].scope;
      if (std::find(sc.begin(), sc.end(), v) != sc.end()) st.in.push_back(f);
      else keep.push_back(f);
    }
    if (st.in.empty()) continue;              // 1/K_v sum_{k_v} 1 = 1
    if ((int)st.in.size() > elim::kMaxTouch)
      return fail(TMC_ERR_SHAPE, "more than 8 factors contain index " + std::to_string(v));
    for (int f : st.in)
      for (int u : p.facs[f].scope)
        if (std::find(st.uni.begin(), st.uni.end(), u) == st.uni.end()) st.uni.push_back(u);
    std::sort(st.uni.begin(), st.uni.end());
    if ((int)st.uni.size() > elim::kMaxUnion)
      return fail(TMC_ERR_SHAPE, "eliminating index " + std::to_string(v) +
                                     " creates a factor over more than 3 indices (choose another order)");
    ElimFac nf;
    for (int u : st.uni)
      if (u != v) { nf.scope.push_back(u); nf.size *= p.K[u]; }
    if (nf.size > INT32_MAX) return fail(TMC_ERR_SHAPE, "intermediate factor too large");
    nf.tab = carve(cur, 4 * B * nf.size);
    nf.grad = carve(cur, 4 * B * nf.size);
    nf.off = carve(cur, 8 * B);
    nf.shift = carve(cur, 4 * B);
    st.out = (int)p.facs.size();
    p.facs.push_back(nf);
    keep.push_back(st.out);
    live = keep;
    p.steps.push_back(st);
  }
  for (int f : live) {
    if (!p.facs[f].scope.empty()) return fail(TMC_ERR_GRAPH, "internal: factor left with free indices");
    p.finals.push_back(f);
  }
  if ((int)p.finals.size() > elim::kMaxFinal) return fail(TMC_ERR_SHAPE, "too many disconnected components");
  p.total = (cur + 255) & ~size_t(255);
  return TMC_OK;
}

// Kernel descriptor of step k (pointers resolved against the caller's tables and the workspace).
elim::Step elim_step_desc(const ElimPlan& p, int k, const float* const* logf, void* ws, float* const* dlogf) {
  const ElimStepDesc& sd = p.steps[k];
  elim::Step st{};
  st.nin = (int)sd.in.size();
  st.nu = (int)sd.uni.size();
  st.vpos = (int)(std::find(sd.uni.begin(), sd.uni.end(), sd.v) - sd.uni.begin());
  st.lnK = std::log((float)p.K[sd.v]);
  for (int u = 0; u < st.nu; ++u) st.Ku[u] = p.K[sd.uni[u]];
  auto strides_of = [&](const std::vector<int>& sc, int* out) {
    for (int u = 0; u < elim::kMaxUnion; ++u) out[u] = 0;
    long long s = 1;
    for (int a = (int)sc.size() - 1; a >= 0; --a) {
      const int u = (int)(std::find(sd.uni.begin(), sd.uni.end(), sc[a]) - sd.uni.begin());
      out[u] = (int)s;
      s *= p.K[sc[a]];
    }
  };
  for (int j = 0; j < st.nin; ++j) {
    const ElimFac& f = p.facs[sd.in[j]];
    st.tab[j] = f.user >= 0 ? logf[f.user] : at<float>(ws, f.tab);
    st.toff[j] = f.user >= 0 ? nullptr : at<double>(ws, f.off);
    st.tsize[j] = f.size;
    st.tar[j] = (int)f.scope.size();
    for (int a = 0; a < st.tar[j]; ++a)
      st.tpos[j][a] = (int)(std::find(sd.uni.begin(), sd.uni.end(), f.scope[a]) - sd.uni.begin());
    strides_of(f.scope, st.tstride[j]);
    st.gin[j] = f.user >= 0 ? (dlogf ? dlogf[f.user] : nullptr) : at<float>(ws, f.grad);
  }
  const ElimFac& o = p.facs[sd.out];
  st.out = at<float>(ws, o.tab);
  st.osize = o.size;
  strides_of(o.scope, st.ostride);
  st.ooff = at<double>(ws, o.off);
  st.shift = at<float>(ws, o.shift);
  st.gout = at<float>(ws, o.grad);
  return st;
}

elim::Final elim_final_desc(const ElimPlan& p, void* ws) {
  elim::Final f{};
  f.count = (int)p.finals.size();
  for (int j = 0; j < f.count; ++j) {
    const ElimFac& e = p.facs[p.finals[j]];
    f.res[j] = at<float>(ws, e.tab);
    f.off[j] = at<double>(ws, e.off);
    f.grad[j] = at<float>(ws, e.grad);
  }
  return f;
}

}  // namespace
}  // namespace tmc


// ============================================================ host-input streamed estimate (e2e)
// tmc_estimate_host: the batch is cut into chunks of datapoints (independent problems),
// chunk c+1's inputs are copied host->device on an internal copy stream into one of two staging
// slots while chunk c runs on the caller's stream, so PCIe transfer and kernels overlap.
namespace tmc {
namespace {

struct HostPipe {            // per device: the copy stream and slot events (created once, never freed)
  cudaStream_t copy = nullptr;
  cudaEvent_t start = nullptr, copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
  std::mutex enqueue;        // calls from several host threads on one device enqueue one at a time
};

tmc_status host_pipe(HostPipe*& hp) {
  static std::mutex mu;
  static HostPipe pipes[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail(TMC_ERR_CUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(mu);
  HostPipe& h = pipes[dev];
  if (!h.copy) {
    if (cudaStreamCreateWithFlags(&h.copy, cudaStreamNonBlocking) != cudaSuccess) return fail(TMC_ERR_CUDA, "copy stream");
    cudaEvent_t* evs[5] = {&h.start, &h.copied[0], &h.copied[1], &h.done[0], &h.done[1]};
    for (cudaEvent_t* e : evs)
      if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return fail(TMC_ERR_CUDA, "event");
  }
  hp = &h;
  return TMC_OK;
}

// Floats one datapoint's inputs take, per latent field, in staging order (z, mu, logvar, logq, logobs).
struct StageLayout {
  std::vector<size_t> off[5];   // [field][latent] byte offset inside a slot for chunk datapoints
  size_t slot_bytes = 0, dlogp_off = 0, ws_off = 0, total = 0;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

void stage_layout(const tmc_graph* g, int chunk, size_t ws_chunk, StageLayout& L) {
  size_t cur = 0;
  for (int f = 0; f < 5; ++f) L.off[f].assign(g->n, 0);
  for (int i = 0; i < g->n; ++i) {
    const size_t K = g->K[i], D = g->D[i], Kp = g->parent[i] < 0 ? 1 : g->K[g->parent[i]];
    const size_t per[5] = {K * D, Kp * D, Kp * D, K, K};
    for (int f = 0; f < 5; ++f) {
      L.off[f][i] = cur;
      cur = align256(cur + (size_t)chunk * per[f] * sizeof(float));
    }
  }
  L.dlogp_off = cur;
  cur = align256(cur + (size_t)chunk * sizeof(double));
  L.slot_bytes = cur;
  L.ws_off = align256(2 * L.slot_bytes + (size_t)chunk * sizeof(double) * 2);
  L.total = L.ws_off + ws_chunk;
}

}  // namespace
}  // namespace tmc

// ====================================================================================== C ABI
using namespace tmc;

extern "C" {

size_t tmc_workspace_size(const tmc_graph* g) {
  Plan p;
  if (make_plan(g, false, p) != TMC_OK) return 0;
  return p.total;
}

tmc_status tmc_factors(const tmc_graph* g, int32_t i, const tmc_latent_in* in_i, float* logf, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_factors");
  try {
    Plan p;
    tmc_status st = make_plan(g, false, p);
    if (st != TMC_OK) return st;
    if (i < 0 || i >= p.n) return fail(TMC_ERR_SHAPE, "latent index out of range");
    if (!in_i || !in_i->z || !in_i->mu || !in_i->logvar || !in_i->logq || !logf)
      return fail(TMC_ERR_INVALID_ARG, "tmc_factors: NULL buffer");
    if ((st = check_device()) != TMC_OK) return st;
    if (p.B == 0) return TMC_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int Ki = p.K[i], Kp = p.Kp[i];
    if (p.prec == TMC_PREC_TC && tc_factors_ok(Ki, Kp, p.Din[i])) {
      st = tc_factors(in_i, logf, p.B, Ki, Kp, p.Din[i], s);
      if (st != TMC_OK) return st;
    } else {
      dim3 grid((Kp + 31) / 32, (Ki + 7) / 8, p.B);
      simt::factors_kernel<<<grid, 256, 0, s>>>(in_i->z, in_i->mu, in_i->logvar, in_i->logq, logf, Ki, Kp, p.Din[i]);
    TMC_COUNT_LAUNCH();
    }
    return launch_check("tmc_factors");
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

tmc_status tmc_forward(const tmc_graph* g, const tmc_latent_in* in, const float* const* logf_dense, double* logp,
                       void* ws, size_t ws_bytes, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_forward");
  try {
    Plan p;
    tmc_status st = make_plan(g, logf_dense != nullptr, p);
    if (st != TMC_OK) return st;
    if ((st = check_inputs(p, in, logf_dense)) != TMC_OK) return st;
    if (!logp && p.B > 0) return fail(TMC_ERR_INVALID_ARG, "logp is NULL");
    if (!ws || ws_bytes < p.total) return fail(TMC_ERR_WORKSPACE, "workspace too small: need " + std::to_string(p.total));
    if ((st = check_device()) != TMC_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (g->flags & TMC_FLAG_VALIDATE)
      if ((st = validate_inputs(p, in, logf_dense, ws, s)) != TMC_OK) return st;
    if (logf_dense) return forward_impl(p, in, logf_dense, logp, ws, s);
    const std::vector<tmc_latent_in> kin = kernel_inputs(p, in, ws, s, true);
    return forward_impl(p, kin.data(), nullptr, logp, ws, s);
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

tmc_status tmc_backward(const tmc_graph* g, const tmc_latent_in* in, const float* const* logf_dense, void* ws,
                        size_t ws_bytes, const double* dlogp, tmc_latent_grad* out, float* const* dlogf_dense,
                        tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_backward");
  try {
    Plan p;
    tmc_status st = make_plan(g, logf_dense != nullptr, p);
    if (st != TMC_OK) return st;
    if ((st = check_inputs(p, in, logf_dense)) != TMC_OK) return st;
    if (!ws || ws_bytes < p.total) return fail(TMC_ERR_WORKSPACE, "workspace too small: need " + std::to_string(p.total));
    if ((st = check_device()) != TMC_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (logf_dense) return backward_impl(p, in, logf_dense, ws, dlogp, out, dlogf_dense, s);
    const std::vector<tmc_latent_in> kin = kernel_inputs(p, in, ws, s, false);
    std::vector<tmc_latent_grad> kout = kernel_outputs(p, out, ws);
    st = backward_impl(p, kin.data(), nullptr, ws, dlogp, out ? kout.data() : nullptr, nullptr, s);
    if (st != TMC_OK) return st;
    unpad_outputs(p, out, ws, s);
    return launch_check("tmc_backward");
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

tmc_status tmc_estimate(const tmc_graph* g, const tmc_latent_in* in, double* logp, const double* dlogp,
                        tmc_latent_grad* out, void* ws, size_t ws_bytes, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_estimate");
  try {
    // small problems: the reverse launch of the small-problem kernel redoes the forward anyway, so the
    // whole estimate is ONE launch that writes logp and every gradient
    Plan p;
    tmc_status st = make_plan(g, false, p);
    if (st != TMC_OK) return st;
    if ((st = check_inputs(p, in, nullptr)) != TMC_OK) return st;
    if (!logp && p.B > 0) return fail(TMC_ERR_INVALID_ARG, "logp is NULL");
    if (!ws || ws_bytes < p.total) return fail(TMC_ERR_WORKSPACE, "workspace too small: need " + std::to_string(p.total));
    if ((st = check_device()) != TMC_OK) return st;
    small::Args A;
    if (p.B > 0 && !p.any_pad && small_ok(p, false, &A, in, out, logp, dlogp, 1)) {
      cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
      if (g->flags & TMC_FLAG_VALIDATE)
        if ((st = validate_inputs(p, in, nullptr, ws, s)) != TMC_OK) return st;
      return launch_small(A, s);
    }
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
  tmc_status st = tmc_forward(g, in, nullptr, logp, ws, ws_bytes, stream);
  if (st != TMC_OK) return st;
  return tmc_backward(g, in, nullptr, ws, ws_bytes, dlogp, out, nullptr, stream);
}


namespace {
tmc_status exchange_plan(const tmc_graph* g, const tmc_latent_in* in, void* ws, size_t ws_bytes, Plan& p) {
  tmc_status st = make_plan(g, false, p);
  if (st != TMC_OK) return st;
  if (p.dir != TMC_DIR_UP) return fail(TMC_ERR_GRAPH, "shared-root exchange needs direction = TMC_DIR_UP");
  if (p.roots.size() != 1) return fail(TMC_ERR_GRAPH, "shared-root exchange needs exactly one root");
  if ((st = check_inputs(p, in, nullptr)) != TMC_OK) return st;
  if (!ws || ws_bytes < p.total) return fail(TMC_ERR_WORKSPACE, "workspace too small: need " + std::to_string(p.total));
  return check_device();
}
}  // namespace

tmc_status tmc_forward_children(const tmc_graph* g, const tmc_latent_in* in, double* root_msg, void* ws,
                                size_t ws_bytes, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_forward_children");
  try {
    Plan p;
    tmc_status st = exchange_plan(g, in, ws, ws_bytes, p);
    if (st != TMC_OK) return st;
    if (!root_msg && p.B > 0) return fail(TMC_ERR_INVALID_ARG, "root_msg is NULL");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (g->flags & TMC_FLAG_VALIDATE)
      if ((st = validate_inputs(p, in, nullptr, ws, s)) != TMC_OK) return st;
    const std::vector<tmc_latent_in> kin = kernel_inputs(p, in, ws, s, true);
    return forward_impl(p, kin.data(), nullptr, nullptr, ws, s, 1, root_msg, nullptr);
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

tmc_status tmc_forward_root(const tmc_graph* g, const tmc_latent_in* in, const double* root_msg_total, double* logp,
                            void* ws, size_t ws_bytes, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_forward_root");
  try {
    Plan p;
    tmc_status st = exchange_plan(g, in, ws, ws_bytes, p);
    if (st != TMC_OK) return st;
    if ((!root_msg_total || !logp) && p.B > 0) return fail(TMC_ERR_INVALID_ARG, "root_msg_total / logp is NULL");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const std::vector<tmc_latent_in> kin = kernel_inputs(p, in, ws, s, false);
    return forward_impl(p, kin.data(), nullptr, logp, ws, s, 2, nullptr, root_msg_total);
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

tmc_status tmc_sample_normal(uint64_t seed, uint32_t tag, int32_t B, int64_t b0, int32_t latent, int32_t K, int32_t D,
                             float* eps, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_sample_normal");
  try {
    if (B < 0 || K < 0 || D <= 0 || b0 < 0 || latent < 0) return fail(TMC_ERR_SHAPE, "tmc_sample_normal: bad shape");
    if ((int64_t)K * ((D + 3) / 4) > INT32_MAX || b0 + (int64_t)B > UINT32_MAX)
      return fail(TMC_ERR_SHAPE, "tmc_sample_normal: K*ceil(D/4) and b0+B must fit the 32-bit counter words");
    if ((int64_t)B * K == 0) return TMC_OK;
    if (!eps) return fail(TMC_ERR_INVALID_ARG, "eps is NULL");
    if (reinterpret_cast<uintptr_t>(eps) % 4) return fail(TMC_ERR_ALIGNMENT, "eps must be 4-byte aligned");
    tmc_status st = check_device();
    if (st != TMC_OK) return st;
    if ((D & 3) == 0 && reinterpret_cast<uintptr_t>(eps) % 16)
      return fail(TMC_ERR_ALIGNMENT, "eps must be 16-byte aligned when D % 4 == 0");
    const int64_t n = (int64_t)B * K * ((D + 3) / 4);
    const int sms = sm_count();
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 16);
    rng::normal_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(seed, tag, B, b0, latent, K, D, eps);
    TMC_COUNT_LAUNCH();
    return launch_check("tmc_sample_normal");
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

size_t tmc_iwae_workspace_size(const tmc_graph* g) {
  if (!g || g->n <= 0 || g->B < 0 || !g->K) return 0;
  return (size_t)std::max(g->B, 1) * (size_t)std::max(g->K[0], 1) * sizeof(double);
}

tmc_status tmc_iwae(const tmc_graph* g, const tmc_latent_in* in, double* logp, const double* dlogp,
                    tmc_latent_grad* out, void* ws, size_t ws_bytes, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_iwae");
  try {
    Plan p;
    tmc_status st = make_plan(g, false, p);
    if (st != TMC_OK) return st;
    for (int i = 0; i < p.n; ++i) {
      if (p.K[i] != p.K[0]) return fail(TMC_ERR_SHAPE, "tmc_iwae needs equal K on every latent");
      if (p.parent[i] < 0 && p.Din[i] > 32 * iwae::kRootMaxChunks) return fail(TMC_ERR_SHAPE, "tmc_iwae: root D > 256");
    }
    if ((st = check_inputs(p, in, nullptr)) != TMC_OK) return st;
    if (p.B == 0) return TMC_OK;
    if (!logp) return fail(TMC_ERR_INVALID_ARG, "logp is NULL");
    const size_t need = tmc_iwae_workspace_size(g);
    if (!ws || ws_bytes < need) return fail(TMC_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
    if ((st = check_device()) != TMC_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    double* w = static_cast<double*>(ws);
    const int K = p.K[0];
    auto fill = [&](int i0, int cnt, iwae::Batch& bt) {
      bt = iwae::Batch{};
      bt.count = cnt; bt.B = p.B; bt.K = K; bt.alpha = p.alpha;
      int roots = 0;
      for (int j = 0; j < cnt; ++j) {
        const int i = i0 + j;
        iwae::LatDesc& L = bt.l[j];
        L.z = in[i].z; L.mu = in[i].mu; L.lv = in[i].logvar; L.logq = in[i].logq; L.logobs = in[i].logobs;
        if (out) { L.gz = out[i].dz; L.gmu = out[i].dmu; L.glv = out[i].dlogvar; L.gq = out[i].dlogq; L.go = out[i].dlogobs; }
        L.D = p.Din[i]; L.root = p.parent[i] < 0;
        roots += L.root;
      }
      return roots;
    };
    bool vec4 = true;                                                 // every D % 4 == 0: float4 kernels
    for (int i = 0; i < p.n; ++i) vec4 = vec4 && (p.Din[i] % 4 == 0);
    for (int i = 0; i < p.n && vec4; ++i)
      for (const void* q : {(const void*)in[i].z, (const void*)in[i].mu, (const void*)in[i].logvar})
        vec4 = vec4 && (reinterpret_cast<uintptr_t>(q) % 16 == 0);
    if (out)
      for (int i = 0; i < p.n && vec4; ++i)
        for (const void* q : {(const void*)out[i].dz, (const void*)out[i].dmu, (const void*)out[i].dlogvar})
          vec4 = vec4 && (reinterpret_cast<uintptr_t>(q) % 16 == 0);
    const int64_t rows = (int64_t)p.B * K;
    const unsigned grid = (unsigned)(vec4 ? (rows + 31) / 32 : (rows + 7) / 8);   // 4 or 1 rows per warp
    for (int i0 = 0; i0 < p.n; i0 += iwae::kMaxLat) {
      iwae::Batch bt;
      fill(i0, std::min(iwae::kMaxLat, p.n - i0), bt);
      if (vec4) iwae::logw4_kernel<<<grid, 256, 0, s>>>(bt, w, i0 == 0);
      else iwae::logw_kernel<<<grid, 256, 0, s>>>(bt, w, i0 == 0);
      TMC_COUNT_LAUNCH();
    }
    iwae::lse_kernel<<<p.B, 256, 0, s>>>(w, K, dlogp, logp);
    TMC_COUNT_LAUNCH();
    if (out) {
      for (int i0 = 0; i0 < p.n; i0 += iwae::kMaxLat) {
        iwae::Batch bt;
        const int roots = fill(i0, std::min(iwae::kMaxLat, p.n - i0), bt);
        if (vec4) iwae::grad4_kernel<<<grid, 256, 0, s>>>(bt, w);
        else iwae::grad_kernel<<<grid, 256, 0, s>>>(bt, w);
        TMC_COUNT_LAUNCH();
        if (roots) {
          iwae::root_grad_kernel<<<dim3(p.B, roots), iwae::kRootWarps * 32, 0, s>>>(bt, w);
          TMC_COUNT_LAUNCH();
        }
      }
    }
    return launch_check("tmc_iwae");
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

size_t tmc_estimate_host_workspace_size(const tmc_graph* g, int32_t chunk) {
  if (!g || chunk <= 0) return 0;
  tmc_graph gc = *g;
  gc.B = std::min<int32_t>(chunk, std::max<int32_t>(g->B, 1));
  Plan p;
  if (make_plan(&gc, false, p) != TMC_OK) return 0;
  StageLayout L;
  stage_layout(g, gc.B, p.total, L);
  return L.total;
}

tmc_status tmc_estimate_host(const tmc_graph* g, const tmc_latent_in* in, double* logp_host, const double* dlogp_host,
                             tmc_latent_grad* out, int32_t chunk, void* ws, size_t ws_bytes, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_estimate_host");
  try {
    Plan p;
    tmc_status st = make_plan(g, false, p);
    if (st != TMC_OK) return st;
    if (chunk <= 0) return fail(TMC_ERR_INVALID_ARG, "chunk must be > 0");
    if (!in || (!logp_host && p.B > 0)) return fail(TMC_ERR_INVALID_ARG, "tmc_estimate_host: NULL input/logp");
    for (int i = 0; i < p.n; ++i)
      if (!in[i].z || !in[i].mu || !in[i].logvar || !in[i].logq) return fail(TMC_ERR_INVALID_ARG, "NULL input buffer");
    if (p.B == 0) return TMC_OK;
    const int cb = std::min<int>(chunk, p.B);
    const size_t need = tmc_estimate_host_workspace_size(g, cb);
    if (!ws || ws_bytes < need) return fail(TMC_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
    if ((st = check_device()) != TMC_OK) return st;
    tmc_graph gc = *g;
    gc.B = cb;
    Plan pc;
    if ((st = make_plan(&gc, false, pc)) != TMC_OK) return st;
    StageLayout L;
    stage_layout(g, cb, pc.total, L);
    HostPipe* hp = nullptr;
    if ((st = host_pipe(hp)) != TMC_OK) return st;
    std::lock_guard<std::mutex> lk(hp->enqueue);     // the slot events are shared per device
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    uint8_t* w = static_cast<uint8_t*>(ws);
    double* logp_dev = reinterpret_cast<double*>(w + 2 * L.slot_bytes);
    // the copy stream may overwrite the staging slots only after earlier work on `stream`
    cudaEventRecord(hp->start, s);
    cudaStreamWaitEvent(hp->copy, hp->start, 0);
    const int nchunks = (p.B + cb - 1) / cb;
    std::vector<tmc_latent_in> cin(p.n);
    std::vector<tmc_latent_grad> cout(p.n);
    for (int c = 0; c < nchunks; ++c) {
      const int b0 = c * cb, bc = std::min(cb, p.B - b0), sl = c & 1;
      uint8_t* slot = w + (size_t)sl * L.slot_bytes;
      if (c >= 2) cudaStreamWaitEvent(hp->copy, hp->done[sl], 0);
      for (int i = 0; i < p.n; ++i) {
        const size_t K = p.K[i], D = p.Din[i], Kp = p.Kp[i];
        const size_t per[5] = {K * D, Kp * D, Kp * D, K, K};
        const float* src[5] = {in[i].z, in[i].mu, in[i].logvar, in[i].logq, in[i].logobs};
        float* dst[5];
        for (int f = 0; f < 5; ++f) {
          dst[f] = reinterpret_cast<float*>(slot + L.off[f][i]);
          if (src[f] && cudaMemcpyAsync(dst[f], src[f] + (size_t)b0 * per[f], (size_t)bc * per[f] * sizeof(float),
                                        cudaMemcpyHostToDevice, hp->copy) != cudaSuccess)
            return fail(TMC_ERR_CUDA, "host->device copy failed");
        }
        cin[i] = tmc_latent_in{dst[0], dst[1], dst[2], dst[3], in[i].logobs ? dst[4] : nullptr};
        tmc_latent_grad o{};
        if (out) {
          const tmc_latent_grad& O = out[i];
          o.dz = O.dz ? O.dz + (size_t)b0 * K * D : nullptr;
          o.dmu = O.dmu ? O.dmu + (size_t)b0 * Kp * D : nullptr;
          o.dlogvar = O.dlogvar ? O.dlogvar + (size_t)b0 * Kp * D : nullptr;
          o.dlogq = O.dlogq ? O.dlogq + (size_t)b0 * K : nullptr;
          o.dlogobs = O.dlogobs ? O.dlogobs + (size_t)b0 * K : nullptr;
          o.pair_marginal = O.pair_marginal ? O.pair_marginal + (size_t)b0 * K * Kp : nullptr;
        }
        cout[i] = o;
      }
      double* dl = nullptr;
      if (dlogp_host) {
        dl = reinterpret_cast<double*>(slot + L.dlogp_off);
        if (cudaMemcpyAsync(dl, dlogp_host + b0, (size_t)bc * sizeof(double), cudaMemcpyHostToDevice, hp->copy) != cudaSuccess)
          return fail(TMC_ERR_CUDA, "host->device copy failed");
      }
      cudaEventRecord(hp->copied[sl], hp->copy);
      cudaStreamWaitEvent(s, hp->copied[sl], 0);
      gc.B = bc;
      st = out ? tmc_estimate(&gc, cin.data(), logp_dev + b0 % (2 * cb), dl, cout.data(), w + L.ws_off, pc.total, stream)
               : tmc_forward(&gc, cin.data(), nullptr, logp_dev + b0 % (2 * cb), w + L.ws_off, pc.total, stream);
      if (st != TMC_OK) return st;
      if (cudaMemcpyAsync(logp_host + b0, logp_dev + b0 % (2 * cb), (size_t)bc * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return fail(TMC_ERR_CUDA, "device->host copy failed");
      cudaEventRecord(hp->done[sl], s);
    }
    return launch_check("tmc_estimate_host");
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

size_t tmc_elim_workspace_size(const tmc_factor_graph* g) {
  ElimPlan p;
  if (make_elim_plan(g, p) != TMC_OK) return 0;
  return std::max<size_t>(p.total, 256);
}

tmc_status tmc_elim_forward(const tmc_factor_graph* g, const float* const* logf, double* logp, void* ws,
                            size_t ws_bytes, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_elim_forward");
  try {
    ElimPlan p;
    tmc_status st = make_elim_plan(g, p);
    if (st != TMC_OK) return st;
    if (p.B == 0) return TMC_OK;
    if (!logf || !logp) return fail(TMC_ERR_INVALID_ARG, "logf / logp is NULL");
    for (int j = 0; j < g->nfac; ++j)
      if (!logf[j]) return fail(TMC_ERR_INVALID_ARG, "logf[" + std::to_string(j) + "] is NULL");
    if (!ws || ws_bytes < p.total) return fail(TMC_ERR_WORKSPACE, "workspace too small: need " + std::to_string(p.total));
    if ((st = check_device()) != TMC_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    ProfScope ps(PF_AUX, s);
    for (int k = 0; k < (int)p.steps.size(); ++k) {
      const elim::Step sd = elim_step_desc(p, k, logf, ws, nullptr);
      dim3 grid((unsigned)((sd.osize + 255) / 256), p.B);
      elim::elim_step_kernel<<<grid, 256, 0, s>>>(sd);
      elim::elim_norm_kernel<<<p.B, 256, 0, s>>>(sd);
      TMC_COUNT_LAUNCH();
      TMC_COUNT_LAUNCH();
    }
    const elim::Final f = elim_final_desc(p, ws);
    elim::elim_final_kernel<<<(p.B + 127) / 128, 128, 0, s>>>(f, p.B, logp);
    TMC_COUNT_LAUNCH();
    return launch_check("tmc_elim_forward");
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

tmc_status tmc_elim_backward(const tmc_factor_graph* g, const float* const* logf, const double* logp, void* ws,
                             size_t ws_bytes, const double* dlogp, float* const* dlogf, tmc_stream_t stream) {
  NvtxRange nvtx_("tmc_elim_backward");
  try {
    ElimPlan p;
    tmc_status st = make_elim_plan(g, p);
    if (st != TMC_OK) return st;
    if (p.B == 0) return TMC_OK;
    if (!logf || !logp || !dlogf) return fail(TMC_ERR_INVALID_ARG, "logf / logp / dlogf is NULL");
    if (!ws || ws_bytes < p.total) return fail(TMC_ERR_WORKSPACE, "workspace too small: need " + std::to_string(p.total));
    if ((st = check_device()) != TMC_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    ProfScope ps(PF_AUX, s);
    const elim::Final f = elim_final_desc(p, ws);
    elim::elim_final_bwd_kernel<<<(p.B + 127) / 128, 128, 0, s>>>(f, p.B, logp, dlogp);
    TMC_COUNT_LAUNCH();
    for (int k = (int)p.steps.size() - 1; k >= 0; --k) {
      const elim::Step sd = elim_step_desc(p, k, logf, ws, dlogf);
      for (int j = 0; j < sd.nin; ++j) {
        if (!sd.gin[j]) continue;
        dim3 grid((unsigned)((sd.tsize[j] + 255) / 256), p.B);
        elim::elim_grad_kernel<<<grid, 256, 0, s>>>(sd, j);
        TMC_COUNT_LAUNCH();
      }
    }
    return launch_check("tmc_elim_backward");
  } catch (...) {
    return fail(TMC_ERR_CUDA, "internal error");
  }
}

const char* tmc_last_error(void) { return g_err.c_str(); }

int32_t tmc_profile_begin(void) {
  Profiler& p = profiler();
  std::lock_guard<std::mutex> lk(p.mu);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(TMC_ERR_CUDA, "tmc_profile_begin: device error");
  static const unsigned long long zeros[PF_COUNT] = {};
  if (cudaMemcpyToSymbol(tc::g_tmc_mma_flops, zeros, sizeof(zeros)) != cudaSuccess)
    return fail(TMC_ERR_CUDA, "tmc_profile_begin: counter reset failed");
  p.recs.clear();
  p.used = 0;
  p.on = true;
  return TMC_OK;
}

int32_t tmc_profile_end(tmc_profile_entry* out, int32_t max_entries) {
  Profiler& p = profiler();
  std::lock_guard<std::mutex> lk(p.mu);
  if (!p.on) return fail(TMC_ERR_INVALID_ARG, "tmc_profile_end without tmc_profile_begin");
  p.on = false;
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(TMC_ERR_CUDA, "tmc_profile_end: device error");
  unsigned long long flops[PF_COUNT] = {};
  cudaMemcpyFromSymbol(flops, tc::g_tmc_mma_flops, sizeof(flops));
  tmc_profile_entry acc[PF_COUNT];
  for (int f = 0; f < PF_COUNT; ++f) acc[f] = tmc_profile_entry{prof_name(f), 0, 0.0, (double)flops[f]};
  for (const Profiler::Rec& r : p.recs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) continue;
    acc[r.fam].launches += 1;
    acc[r.fam].ms += ms;
  }
  p.recs.clear();
  p.used = 0;
  int n = 0;
  for (int f = 0; f < PF_COUNT && n < max_entries; ++f)
    if (acc[f].launches) out[n++] = acc[f];
  return n;
}

int32_t tmc_version(void) { return 100; }

uint64_t tmc_launch_count(void) { return g_launches.load(); }

#ifdef TMC_INSTRUMENT
// Instrumented build only (libtmc_instr.so): copy (and optionally clear) the per-CTA wait counters.
int tmc_debug_counters(unsigned long long* host, int n, int clear) {
  const size_t bytes = sizeof(unsigned long long) * (size_t)std::min(n, 1024 * 64);
  if (cudaMemcpyFromSymbol(host, tc::g_tmc_prof, bytes) != cudaSuccess) return -1;
  if (clear) {
    static unsigned long long zeros[1024 * 64];
    if (cudaMemcpyToSymbol(tc::g_tmc_prof, zeros, sizeof(zeros)) != cudaSuccess) return -1;
  }
  return 0;
}
#endif

}  // extern "C"
