// TMC ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, fp64 CPU implementation of the Tensor Monte Carlo estimator
// (arXiv 1806.08593) and its gradient, used ONLY by tests/, by
// __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
// leg.  It shares no code, header, table or helper with the CUDA path
// (paper_1806_08593_b200/csrc, include/tmc.h) and neither imports the other.
//
// What it computes (PAPER.md line numbers, "P:n"):
//   * factor   logf_i[a,r] = log P(z_i^a | z_pa^r) - log Q(z_i^a)          P:571-576 (Appendix, typical factors)
//              with P(z_i|z_pa) = N(mu_i(z_pa), diag exp(logvar_i(z_pa)))   P:365-369 (§Computational costs)
//   * estimate log P_TMC = log (1/prod K_i) sum_{k_1..k_n} prod_j f_j        P:136-140 (Eq. is)
//              evaluated by variable elimination (sum/product swap)        P:316-331 (§Efficient averaging)
//              with one 1/K_i per eliminated index
//              and a joint-max logsumexp (P:661-677 logmmexp is the
//              matrix case; its separate x_i / y_k maxima are replaced by the joint max).
//   * gradient d log P_TMC / d logf_i = pair marginal of (k_i, k_pa) under the
//              normalised weights (autodiff of P:332 derived by marginals), then
//              the chain rule through the Gaussian density (direct form).
// Every routine is a literal loop over the definitions; there is no blocking,
// fusion or reordering.  Parity pins: tests/test_oracle.py.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>
#include <algorithm>

namespace {

const double kNegInf = -std::numeric_limits<double>::infinity();
const double kLog2Pi = std::log(2.0 * M_PI);

// log sum_j exp(x_j) with the joint max M = max_j x_j; M = -inf => -inf.
double lse(const std::vector<double>& x) {
  double M = kNegInf;
  for (double v : x) M = std::max(M, v);
  if (M == kNegInf) return kNegInf;
  if (std::isinf(M)) return M;  // +inf
  double s = 0.0;
  for (double v : x) s += std::exp(v - M);
  return M + std::log(s);
}

// softmax_j(x_j); all -inf => all zeros (probability-zero slice).
std::vector<double> softmax(const std::vector<double>& x) {
  std::vector<double> p(x.size(), 0.0);
  double L = lse(x);
  if (L == kNegInf) return p;
  for (size_t j = 0; j < x.size(); ++j) p[j] = std::exp(x[j] - L);
  return p;
}

struct Graph {
  int n, B;
  const int *parent, *K, *D;
  int Kp(int i) const { return parent[i] < 0 ? 1 : K[parent[i]]; }
};

struct Inputs {
  const float *const *z, *const *mu, *const *logvar, *const *logq, *const *logobs, *const *logf_dense;
  // factor power: every log-factor and observation term times alpha.  alpha = 2 is "running TMC
  // again, with squared weights", the sum of squared weights the DReGs surrogate needs.
  double alpha = 1.0;
};

struct Outputs {
  double* logp;
  double *const *pair, *const *dz, *const *dmu, *const *dlogvar, *const *dlogq, *const *dlogobs;
  const double* dlogp;
};

// Direct-form log density of one pair: sum_d log N(z_d; mu_d, exp(v_d)).
double log_normal_pair(const float* z, const float* mu, const float* v, int D) {
  double s = 0.0;
  for (int d = 0; d < D; ++d) {
    double zz = z[d], mm = mu[d], vv = v[d];
    double diff = zz - mm;
    s += -0.5 * (diff * diff * std::exp(-vv) + vv + kLog2Pi);
  }
  return s;
}

// logf_i[a][r] for datapoint b: P:573-576 factor = P(z_i^a | z_pa^r) / Q(z_i^a).
std::vector<double> factor(const Graph& g, const Inputs& in, int i, int b) {
  const int Ki = g.K[i], Kp = g.Kp(i), D = g.D[i];
  std::vector<double> f((size_t)Ki * Kp);
  if (in.logf_dense) {
    const float* src = in.logf_dense[i] + (size_t)b * Ki * Kp;
    for (size_t j = 0; j < f.size(); ++j) f[j] = src[j];
    return f;
  }
  const float* z = in.z[i] + (size_t)b * Ki * D;
  const float* mu = in.mu[i] + (size_t)b * Kp * D;
  const float* v = in.logvar[i] + (size_t)b * Kp * D;
  const float* lq = in.logq[i] + (size_t)b * Ki;
  for (int a = 0; a < Ki; ++a)
    for (int r = 0; r < Kp; ++r)
      f[(size_t)a * Kp + r] = log_normal_pair(z + (size_t)a * D, mu + (size_t)r * D, v + (size_t)r * D, D)
                              - (double)lq[a];
  return f;
}

double obs(const Inputs& in, const Graph& g, int i, int b, int a) {
  if (!in.logobs || !in.logobs[i]) return 0.0;
  return in.logobs[i][(size_t)b * g.K[i] + a];
}

// One datapoint: upward elimination (leaves -> roots), optional downward pass
// (chains, the north_star recursion), marginals top-down, gradients.
void run_datapoint(const Graph& g, const Inputs& in, const Outputs& out, int direction, int b) {
  const int n = g.n;
  std::vector<std::vector<double>> f(n), h(n), msg(n);
  for (int i = 0; i < n; ++i) {
    f[i] = factor(g, in, i, b);
    for (double& v : f[i]) v *= in.alpha;
  }

  // O3: upward elimination, reverse topological order (parent[i] < i).
  for (int i = 0; i < n; ++i) {
    h[i].assign(g.K[i], 0.0);
    for (int a = 0; a < g.K[i]; ++a) h[i][a] = in.alpha * obs(in, g, i, b, a);
  }
  double L_up = 0.0;
  for (int i = n - 1; i >= 0; --i) {
    const int Ki = g.K[i], Kp = g.Kp(i);
    msg[i].assign(Kp, 0.0);
    for (int r = 0; r < Kp; ++r) {
      std::vector<double> t(Ki);
      for (int a = 0; a < Ki; ++a) t[a] = f[i][(size_t)a * Kp + r] + h[i][a];
      msg[i][r] = lse(t) - std::log((double)Ki);   // (1/K_i) sum_{k_i}
    }
    if (g.parent[i] >= 0) {
      for (int r = 0; r < Kp; ++r) h[g.parent[i]][r] += msg[i][r];
    } else {
      L_up += msg[i][0];
    }
  }
  double L = L_up;

  // O3': downward recursion m_i[a] = obs_i[a] + LSE_c(logf_i[a,c] + m_p[c]) - ln K_p (chains).
  if (direction == 1) {
    std::vector<double> m;
    for (int i = 0; i < n; ++i) {
      const int Ki = g.K[i], Kp = g.Kp(i);
      std::vector<double> mi(Ki);
      for (int a = 0; a < Ki; ++a) {
        std::vector<double> t(Kp);
        for (int c = 0; c < Kp; ++c) t[c] = f[i][(size_t)a * Kp + c] + (i == 0 ? 0.0 : m[c]);
        mi[a] = in.alpha * obs(in, g, i, b, a) + lse(t) - (i == 0 ? 0.0 : std::log((double)Kp));
      }
      m.swap(mi);
    }
    L = lse(m) - std::log((double)g.K[n - 1]);
  }
  out.logp[b] = L;

  // O4: marginals top-down.  pi_root = softmax(logf_root + h_root); for a child c of p:
  // P_c[a,r] = pi_p[r] * softmax_a(logf_c[a,r] + h_c[a]);  pi_c[a] = sum_r P_c[a,r].
  const double w = out.dlogp ? out.dlogp[b] : 1.0;
  std::vector<std::vector<double>> pi(n), P(n);
  for (int i = 0; i < n; ++i) {
    const int Ki = g.K[i], Kp = g.Kp(i);
    P[i].assign((size_t)Ki * Kp, 0.0);
    pi[i].assign(Ki, 0.0);
    for (int r = 0; r < Kp; ++r) {
      double wr = g.parent[i] < 0 ? w : pi[g.parent[i]][r];
      std::vector<double> t(Ki);
      for (int a = 0; a < Ki; ++a) t[a] = f[i][(size_t)a * Kp + r] + h[i][a];
      std::vector<double> s = softmax(t);
      for (int a = 0; a < Ki; ++a) P[i][(size_t)a * Kp + r] = wr * s[a];
    }
    for (int a = 0; a < Ki; ++a)
      for (int r = 0; r < Kp; ++r) pi[i][a] += P[i][(size_t)a * Kp + r];
  }

  // O5: gradients.  dL/dlogf_i = P_i; dL/dlogobs_i = pi_i; dL/dlogq_i = -pi_i;
  // then d logN / d{z, mu, v} in the direct form.
  for (int i = 0; i < n; ++i) {
    const int Ki = g.K[i], Kp = g.Kp(i), D = g.D[i];
    // with factor power alpha every input enters as alpha * (its log-term): chain rule factor alpha
    const double al = in.alpha;
    if (out.pair && out.pair[i])
      for (size_t j = 0; j < P[i].size(); ++j) out.pair[i][(size_t)b * Ki * Kp + j] = al * P[i][j];
    if (out.dlogobs && out.dlogobs[i])
      for (int a = 0; a < Ki; ++a) out.dlogobs[i][(size_t)b * Ki + a] = al * pi[i][a];
    if (in.logf_dense) continue;
    if (out.dlogq && out.dlogq[i])
      for (int a = 0; a < Ki; ++a) out.dlogq[i][(size_t)b * Ki + a] = -al * pi[i][a];
    const float* z = in.z[i] + (size_t)b * Ki * D;
    const float* mu = in.mu[i] + (size_t)b * Kp * D;
    const float* v = in.logvar[i] + (size_t)b * Kp * D;
    std::vector<double> dz((size_t)Ki * D, 0.0), dmu((size_t)Kp * D, 0.0), dv((size_t)Kp * D, 0.0);
    for (int a = 0; a < Ki; ++a)
      for (int r = 0; r < Kp; ++r) {
        double p = al * P[i][(size_t)a * Kp + r];
        if (p == 0.0) continue;
        for (int d = 0; d < D; ++d) {
          double zz = z[(size_t)a * D + d], mm = mu[(size_t)r * D + d], vv = v[(size_t)r * D + d];
          double lam = std::exp(-vv), diff = zz - mm;
          dz[(size_t)a * D + d] += p * (-diff * lam);                 // d/dz   logN = -(z-mu)/s2
          dmu[(size_t)r * D + d] += p * (diff * lam);                 // d/dmu  logN =  (z-mu)/s2
          dv[(size_t)r * D + d] += p * 0.5 * (diff * diff * lam - 1.0);  // d/dv logN
        }
      }
    if (out.dz && out.dz[i]) std::memcpy(out.dz[i] + (size_t)b * Ki * D, dz.data(), sizeof(double) * Ki * D);
    if (out.dmu && out.dmu[i]) std::memcpy(out.dmu[i] + (size_t)b * Kp * D, dmu.data(), sizeof(double) * Kp * D);
    if (out.dlogvar && out.dlogvar[i])
      std::memcpy(out.dlogvar[i] + (size_t)b * Kp * D, dv.data(), sizeof(double) * Kp * D);
  }
}

bool valid_graph(int n, int B, const int* parent, const int* K, const int* D) {
  if (n <= 0 || B < 0 || !parent || !K || !D) return false;
  for (int i = 0; i < n; ++i) {
    if (K[i] <= 0 || D[i] <= 0) return false;
    if (parent[i] >= i || parent[i] < -1) return false;
  }
  return true;
}

bool is_chain(int n, const int* parent) {
  for (int i = 0; i < n; ++i)
    if (parent[i] != i - 1) return false;
  return true;
}

}  // namespace


// ============================================================================================
// the reparameterisation noise eps ~ N(0,1), defined exactly as
// include/tmc.h (tmc_sample_normal) states it, written here from that definition so the device
// sampler can be checked bit for bit.  Philox4x32-10 (Salmon et al., SC'11: multipliers
// 0xD2511F53 / 0xCD9E8D57, Weyl key increments 0x9E3779B9 / 0xBB67AE85, 10 rounds), uniforms
// ((w >> 8) + 1/2) 2^-24, Box-Muller with ln / cos / sin as the stated fp32 polynomials; every fp32
// operation below is a single correctly rounded IEEE operation (this file is built with
// -ffp-contract=off; fma is std::fma).
namespace a1 {

void philox_4x32_10(const uint32_t in[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
  uint32_t x0 = in[0], x1 = in[1], x2 = in[2], x3 = in[3];
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * x0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
    const uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0;
    const uint32_t y1 = (uint32_t)p1;
    const uint32_t y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
    const uint32_t y3 = (uint32_t)p0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

float uniform(uint32_t w) { return ((float)(w >> 8) + 0.5f) * 0x1p-24f; }

float log_fp32(float u) {
  uint32_t b;
  std::memcpy(&b, &u, 4);
  int ex = (int)((b >> 23) & 0xFFu) - 127;
  const uint32_t mb = (b & 0x7FFFFFu) | 0x3F800000u;
  float m;
  std::memcpy(&m, &mb, 4);
  if (m > 0x1.6a09e6p+0f) {          // fp32(sqrt 2)
    m = m * 0.5f;
    ex = ex + 1;
  }
  const float t = (m - 1.0f) / (m + 1.0f);
  const float t2 = t * t;
  // 1 + t^2/3 + t^4/5 + ... + t^12/13, Horner from the top, coefficients fp32(1/(2j+1))
  const float coef[6] = {0x1.3b13b2p-4f, 0x1.745d18p-4f, 0x1.c71c72p-4f, 0x1.24924ap-3f, 0x1.99999ap-3f, 0x1.555556p-2f};
  float h = coef[0];
  for (int j = 1; j < 6; ++j) h = std::fma(h, t2, coef[j]);
  h = std::fma(h, t2, 1.0f);
  const float lm = (2.0f * t) * h;
  return std::fma((float)ex, 0x1.62e430p-1f, lm);     // fp32(ln 2)
}

void cos_sin_2pi(float v, float* c, float* s) {
  const float q = std::nearbyint(v * 4.0f);
  const float w = v + q * -0.25f;
  const float x = w * 0x1.921fb6p+2f;                  // fp32(2 pi)
  const float x2 = x * x;
  const float sc[5] = {-0x1.ae6456p-26f, 0x1.71de3ap-19f, -0x1.a01a02p-13f, 0x1.111112p-7f, -0x1.555556p-3f};
  float sp = sc[0];
  for (int j = 1; j < 5; ++j) sp = std::fma(sp, x2, sc[j]);
  sp = std::fma(sp * x2, x, x);                         // x - x^3/3! + ... - x^11/11!
  const float cc[7] = {0x1.1eed8ep-29f, -0x1.27e4fcp-22f, 0x1.a01a02p-16f, -0x1.6c16c2p-10f, 0x1.555556p-5f, -0.5f, 1.0f};
  float cp = cc[0];
  for (int j = 1; j < 7; ++j) cp = std::fma(cp, x2, cc[j]);   // 1 - x^2/2! + ... + x^12/12!
  switch (((int)q) & 3) {
    case 0: *c = cp; *s = sp; break;
    case 1: *c = -sp; *s = cp; break;
    case 2: *c = -cp; *s = -sp; break;
    default: *c = sp; *s = -cp; break;
  }
}

void gauss_pair(uint32_t w0, uint32_t w1, float* n0, float* n1) {
  const float r = std::sqrt(-2.0f * log_fp32(uniform(w0)));
  float c, s;
  cos_sin_2pi(uniform(w1), &c, &s);
  *n0 = r * c;
  *n1 = r * s;
}

}  // namespace a1

extern "C" {

// Joint-max logsumexp of x[0..n).  Returns -inf for n == 0.
double or_logsumexp(const double* x, int64_t n) {
  std::vector<double> v(x, x + n);
  return lse(v);
}

// Z[i][k] = log sum_j exp(X[i][j] + Y[j][k])  (P:661-677 logmmexp; joint max, A2).
int or_logmmexp(const double* X, const double* Y, int64_t I, int64_t J, int64_t Kk, double* Z) {
  for (int64_t i = 0; i < I; ++i)
    for (int64_t k = 0; k < Kk; ++k) {
      std::vector<double> t(J);
      for (int64_t j = 0; j < J; ++j) t[j] = X[i * J + j] + Y[j * Kk + k];
      Z[i * Kk + k] = lse(t);
    }
  return 0;
}

// logf_i[b][a][r] (fp64) of the typical directed factorisation.
int or_factor(int n, int B, const int* parent, const int* K, const int* D, int i,
              const float* z, const float* mu, const float* logvar, const float* logq, double* logf) {
  if (!valid_graph(n, B, parent, K, D) || i < 0 || i >= n) return -1;
  Graph g{n, B, parent, K, D};
  std::vector<const float*> zz(n, nullptr), mm(n, nullptr), vv(n, nullptr), qq(n, nullptr);
  zz[i] = z; mm[i] = mu; vv[i] = logvar; qq[i] = logq;
  Inputs in{zz.data(), mm.data(), vv.data(), qq.data(), nullptr, nullptr};
  const size_t sz = (size_t)K[i] * g.Kp(i);
  for (int b = 0; b < B; ++b) {
    std::vector<double> f = factor(g, in, i, b);
    std::memcpy(logf + b * sz, f.data(), sizeof(double) * sz);
  }
  return 0;
}

// Full estimator + gradient.  direction: 1 = downward recursion (chains only), 2 = upward.
// Any output pointer array (or entry) may be NULL.  Returns 0, or -1 bad graph, -2 down on non-chain.
int or_estimate(int n, int B, const int* parent, const int* K, const int* D,
                const float* const* z, const float* const* mu, const float* const* logvar,
                const float* const* logq, const float* const* logobs, const float* const* logf_dense,
                int direction, const double* dlogp, double* logp,
                double* const* pair, double* const* dz, double* const* dmu, double* const* dlogvar,
                double* const* dlogq, double* const* dlogobs, int nthreads, double alpha) {
  if (!valid_graph(n, B, parent, K, D) || !logp) return -1;
  if (direction == 1 && !is_chain(n, parent)) return -2;
  Graph g{n, B, parent, K, D};
  Inputs in{z, mu, logvar, logq, logobs, logf_dense, alpha};
  Outputs out{logp, pair, dz, dmu, dlogvar, dlogq, dlogobs, dlogp};
  if (nthreads <= 1 || B <= 1) {
    for (int b = 0; b < B; ++b) run_datapoint(g, in, out, direction, b);
    return 0;
  }
  nthreads = std::min(nthreads, B);
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&, t]() {
      for (int b = t; b < B; b += nthreads) run_datapoint(g, in, out, direction, b);
    });
  for (auto& x : th) x.join();
  return 0;
}


// eps[b][k][d], b = 0..B-1 <-> global datapoint b0 + b (tmc_sample_normal's definition).
int or_sample_normal(uint64_t seed, uint32_t tag, int B, int64_t b0, int latent, int K, int D, float* eps) {
  if (B < 0 || K < 0 || D <= 0 || !eps) return -1;
  const int groups = (D + 3) / 4;
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < K; ++k)
      for (int g = 0; g < groups; ++g) {
        const uint32_t ctr[4] = {tag, (uint32_t)(b0 + b), (uint32_t)latent, (uint32_t)(k * groups + g)};
        uint32_t w[4];
        a1::philox_4x32_10(ctr, (uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32), w);
        float e[4];
        a1::gauss_pair(w[0], w[1], &e[0], &e[1]);
        a1::gauss_pair(w[2], w[3], &e[2], &e[3]);
        for (int q = 0; q < 4 && 4 * g + q < D; ++q) eps[((size_t)b * K + k) * D + 4 * g + q] = e[q];
      }
  return 0;
}

// Raw Philox4x32-10 (known-answer tests) and the fp32 polynomials (accuracy pins).
void or_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) { a1::philox_4x32_10(ctr, key[0], key[1], out); }
float or_log_fp32(float u) { return a1::log_fp32(u); }
void or_cos_sin_2pi(float v, float* c, float* s) { a1::cos_sin_2pi(v, c, s); }


// NEXT-3: the IWAE estimator at equal K, by its definition: the K joint
// samples are the index tuples (k, k, ..., k) (every latent's k-th sample, its conditional taken at
// the parent's k-th sample), log w_k = sum_i [log p(z_i^k | z_pa^k) - log q_i(z_i^k) + log p(x_i | z_i^k)],
// L = log (1/K) sum_k w_k.  Gradients of J = sum_b dlogp[b] L_b: with pi_k = dlogp * softmax_k(log w),
// dlogobs_i[k] = pi_k, dlogq_i[k] = -pi_k, and the Gaussian terms of the (k, k) pair of each edge.
// All K_i must be equal.  Returns 0, -1 bad graph / unequal K.
int or_iwae(int n, int B, const int* parent, const int* K, const int* D,
            const float* const* z, const float* const* mu, const float* const* logvar,
            const float* const* logq, const float* const* logobs, const double* dlogp, double* logp,
            double* const* dz, double* const* dmu, double* const* dlogvar, double* const* dlogq,
            double* const* dlogobs) {
  if (!valid_graph(n, B, parent, K, D) || !logp) return -1;
  for (int i = 1; i < n; ++i)
    if (K[i] != K[0]) return -1;
  const int Kk = K[0];
  for (int b = 0; b < B; ++b) {
    std::vector<double> lw(Kk, 0.0);
    for (int k = 0; k < Kk; ++k) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) {
        const int c = parent[i] < 0 ? 0 : k;
        const int Kp = parent[i] < 0 ? 1 : K[parent[i]];
        const size_t zo = ((size_t)b * K[i] + k) * D[i], mo = ((size_t)b * Kp + c) * D[i];
        s += log_normal_pair(z[i] + zo, mu[i] + mo, logvar[i] + mo, D[i]);
        s -= (double)logq[i][(size_t)b * K[i] + k];
        if (logobs && logobs[i]) s += (double)logobs[i][(size_t)b * K[i] + k];
      }
      lw[k] = s;
    }
    double M = -std::numeric_limits<double>::infinity();
    for (double v : lw) M = std::max(M, v);
    double S = 0.0;
    if (M > -std::numeric_limits<double>::infinity())
      for (double v : lw) S += std::exp(v - M);
    logp[b] = (M == -std::numeric_limits<double>::infinity()) ? M : M + std::log(S) - std::log((double)Kk);
    const double wb = dlogp ? dlogp[b] : 1.0;
    for (int i = 0; i < n; ++i) {
      const int Kp = parent[i] < 0 ? 1 : K[parent[i]];
      if (dmu && dmu[i]) std::fill(dmu[i] + (size_t)b * Kp * D[i], dmu[i] + (size_t)(b + 1) * Kp * D[i], 0.0);
      if (dlogvar && dlogvar[i]) std::fill(dlogvar[i] + (size_t)b * Kp * D[i], dlogvar[i] + (size_t)(b + 1) * Kp * D[i], 0.0);
    }
    for (int k = 0; k < Kk; ++k) {
      const double pk = (S > 0.0) ? wb * std::exp(lw[k] - M) / S : 0.0;
      for (int i = 0; i < n; ++i) {
        const int c = parent[i] < 0 ? 0 : k;
        const int Kp = parent[i] < 0 ? 1 : K[parent[i]];
        const size_t zo = ((size_t)b * K[i] + k) * D[i], mo = ((size_t)b * Kp + c) * D[i];
        if (dlogobs && dlogobs[i]) dlogobs[i][(size_t)b * K[i] + k] = pk;
        if (dlogq && dlogq[i]) dlogq[i][(size_t)b * K[i] + k] = -pk;
        for (int d = 0; d < D[i]; ++d) {
          const double diff = (double)z[i][zo + d] - (double)mu[i][mo + d];
          const double lam = std::exp(-(double)logvar[i][mo + d]);
          if (dz && dz[i]) dz[i][zo + d] = -pk * diff * lam;
          if (dmu && dmu[i]) dmu[i][mo + d] += pk * diff * lam;
          if (dlogvar && dlogvar[i]) dlogvar[i][mo + d] += 0.5 * pk * (diff * diff * lam - 1.0);
        }
      }
    }
  }
  return 0;
}

}  // extern "C"
