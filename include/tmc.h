/*
 * tmc.h — C ABI of libtmc, the B200 (sm_100a) Tensor Monte Carlo hot path.
 *
 * Paper: L. Aitchison, "Tensor Monte Carlo: particle methods for the GPU era",
 * arXiv 1806.08593.  Citations "P:n" are PAPER.md line numbers.
 *
 * WHAT IS COMPUTED
 *   A directed model over latents z_0..z_{n-1} whose parent structure is a tree
 *   or forest (parent[i] < i, -1 = root).  Every latent i carries K_i proposal
 *   samples z_i^{k}.  The conditional P(z_i | z_pa) is a
 *   diagonal Gaussian N(mu_i(z_pa), diag exp(logvar_i(z_pa))),
 *   evaluated by the caller at every parent sample (the root's "parent" is a
 *   single prior, K_p = 1).  The typical factorisation gives one
 *   pairwise factor per latent,
 *       logf_i[b,a,c] = log N(z_i^a ; mu_i[b,c], exp(logvar_i[b,c])) - logq_i[b,a]
 *   and observation factors logobs_i[b,a] = log P(x | z_i^a).  The TMC estimate
 *   (Eq. is; Eq. fac) for datapoint b is
 *       logp[b] = log( (1/prod_i K_i) * sum_{k_0..k_{n-1}} prod_i f_i * prod_i obs_i ),
 *   evaluated by sum/product swapping as a chain/tree of log-domain
 *   tensor inner products, never by enumeration:
 *     DOWN (chains, the north_star recursion):
 *       m_i[a] = logobs_i[a] + LSE_c( logf_i[a,c] + m_{i-1}[c] ) - ln K_{i-1}
 *       logp   = LSE_a m_{n-1}[a] - ln K_{n-1}
 *     UP (trees, leaves -> roots):
 *       msg_{i->p}[r] = LSE_a( logf_i[a,r] + logobs_i[a] + sum_{j child of i} msg_{j->i}[a] ) - ln K_i
 *       logp   = sum over roots of msg_{root}[0]
 *   Non-factorised proposals (Eq. 2) enter through logq_i, which is
 *   indexed only by k_i.  The reverse pass returns the gradient of
 *   J = sum_b dlogp[b] * logp[b] w.r.t. every input, and optionally the pair
 *   marginals dJ/dlogf_i[b,a,c].
 *
 * CONVENTIONS (all calls)
 *   - Graph metadata (tmc_graph.parent/K/D, the pointer arrays themselves) are
 *     HOST memory.  Every float/double buffer is DEVICE memory owned by the
 *     caller, contiguous row-major, 4-byte aligned (16-byte for the tensor-core
 *     path, see TMC_PREC_TC).  The library allocates no device memory
 *     (tmc_estimate_host keeps one copy stream and five events per device).
 *   - Calls are asynchronous and stream-ordered on `stream`; they are reentrant
 *     across streams given distinct workspaces.  Shape/graph/argument errors
 *     are detected synchronously and nothing is launched.  Launch failures
 *     return TMC_ERR_CUDA.  No C++ exception crosses this boundary.
 *   - B = 0 is valid: nothing is read or launched, and buffer pointers may be NULL.
 *   - -inf is allowed in logq/logobs/logf (probability-zero event).  A
 *     datapoint whose every tuple is impossible gets logp = -inf and all-zero
 *     gradients (never NaN).  NaN inputs are not checked unless TMC_FLAG_VALIDATE.
 *   - Outputs are deterministic: identical inputs give bit-identical outputs,
 *     independent of batch position (no atomics on the data path).
 */
#ifndef TMC_H_
#define TMC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same object as cudaStream_t; NULL = legacy default stream. */
typedef struct CUstream_st *tmc_stream_t;

typedef enum {
  TMC_OK = 0,
  TMC_ERR_INVALID_ARG = -1,        /* NULL where a buffer is required, bad enum value      */
  TMC_ERR_SHAPE = -2,              /* n<=0, B<0, K_i<=0, D_i<=0, i out of range            */
  TMC_ERR_GRAPH = -3,              /* parent[i] >= i or < -1; DOWN requested on a non-chain */
  TMC_ERR_ALIGNMENT = -4,          /* buffer misaligned for the requested precision path   */
  TMC_ERR_WORKSPACE = -5,          /* ws NULL or ws_bytes < tmc_workspace_size()           */
  TMC_ERR_UNSUPPORTED_DEVICE = -6, /* current device is not compute capability 10.0       */
  TMC_ERR_CUDA = -7,               /* a kernel launch failed (message in tmc_last_error)   */
  TMC_ERR_NONFINITE = -8           /* TMC_FLAG_VALIDATE found NaN/+inf in an input         */
} tmc_status;

typedef enum { TMC_DIR_AUTO = 0, TMC_DIR_DOWN = 1, TMC_DIR_UP = 2 } tmc_direction;
/* AUTO = DOWN for chains (parent[i] == i-1), UP otherwise. Both give the same logp. */

typedef enum {
  TMC_PREC_AUTO = 0, /* TC where the shape allows it, SIMT otherwise; small problems (all   */
                     /* K_i <= 64, D_i <= 128, n <= 32, direction AUTO) run as one fused   */
                     /* launch per tmc_forward / tmc_backward (one CTA per datapoint)      */
  TMC_PREC_SIMT = 1, /* fp32 CUDA-core direct form sum_d (z-mu)^2/s^2                        */
  TMC_PREC_TC = 2    /* expanded quadratic form on tcgen05 tensor cores, 3-term fp16 split; */
                     /* a non-root latent with D not in {32,64} (D <= 64) runs from zero-    */
                     /* padded workspace copies (padded dims contribute exactly 0); AUTO     */
                     /* pads only when K_i, K_p >= 128                                       */
} tmc_precision;

enum {
  TMC_FLAG_VALIDATE = 1u,      /* scan every input for NaN/+inf first (TMC_ERR_NONFINITE), synchronous   */
  TMC_FLAG_DENSE_REVERSE = 2u, /* reverse pass computes every tile, including tiles whose pair weights  */
                               /* are all exactly 0 (skipped by default; identical results, measurement). */
                               /* On the tensor-core path "weight 0" includes pair terms that are zero in */
                               /* both fp16 parts of their weight (below 2^-41 of the edge's largest      */
                               /* upstream weight, R5/R6): their rows and column sums are 0 in  */
                               /* both modes, so the two stay bit-identical                               */
  TMC_FLAG_TWO_PASS_REVERSE = 4u, /* tensor-core reverse pass as two owner passes (S and P~ recomputed   */
                               /* per orientation); equal to the single pass within fp32 rounding        */
  TMC_FLAG_SINGLE_PASS_REVERSE = 8u /* tensor-core reverse pass as one pass (one S and P~ per tile, D = 32 */
                               /* edges); the library picks per build which of the two is the default;  */
                               /* setting both flags is TMC_ERR_INVALID_ARG                              */
};

typedef struct {
  int32_t n;              /* number of latent variables, >= 1                                 */
  int32_t B;              /* number of datapoints (independent problems), >= 0                */
  const int32_t *parent;  /* HOST [n]: parent index, -1 for a root, parent[i] < i             */
  const int32_t *K;       /* HOST [n]: samples per latent K_i >= 1                      */
  const int32_t *D;       /* HOST [n]: dimension of latent i, >= 1                             */
  int32_t direction;      /* tmc_direction                                                    */
  int32_t precision;      /* tmc_precision                                                    */
  uint32_t flags;         /* TMC_FLAG_*                                                       */
  float factor_power;     /* alpha: every log-factor and observation term is multiplied by    */
                          /* alpha, i.e. logp = log((1/prod K_i) sum prod f^alpha obs^alpha);  */
                          /* 0 or 1 = the TMC estimate; 2 = the sum of squared importance      */
                          /* weights of the DReGs surrogate ("running TMC again, with squared  */
                          /* weights").  Gradients are of that logp.  tmc_factors   */
                          /* ignores it (it materialises logf itself).                          */
} tmc_graph;

/* Per-latent inputs (DEVICE).  K_p = K[parent[i]], or 1 for a root (its prior).             */
typedef struct {
  const float *z;       /* [B][K_i][D_i]  proposal samples z_i^k                               */
  const float *mu;      /* [B][K_p][D_i]  mean of P(z_i | z_pa^c) for every parent sample c    */
  const float *logvar;  /* [B][K_p][D_i]  log-variance of the same conditional                */
  const float *logq;    /* [B][K_i]       log Q(z_i^k | ...)  (ignored on the dense path)      */
  const float *logobs;  /* [B][K_i] or NULL (= 0): log P(x_i | z_i^k) of attached observations */
} tmc_latent_in;

/* Per-latent gradient outputs (DEVICE, overwritten).  Any pointer may be NULL (not wanted). */
typedef struct {
  float *dz;            /* [B][K_i][D_i]                                                     */
  float *dmu;           /* [B][K_p][D_i]                                                     */
  float *dlogvar;       /* [B][K_p][D_i]                                                     */
  float *dlogq;         /* [B][K_i]   = -pi_i (marginal of k_i under the normalised weights) */
  float *dlogobs;       /* [B][K_i]   =  pi_i                                                */
  float *pair_marginal; /* [B][K_i][K_p] = dJ/dlogf_i; O(K^2) memory, small K only    */
} tmc_latent_grad;

/* Bytes of device workspace tmc_forward/tmc_backward/tmc_estimate need for this graph.
 * Returns 0 if the graph is invalid (see tmc_last_error). */
size_t tmc_workspace_size(const tmc_graph *g);

/* Materialise the pairwise log-factor of latent i:
 *   logf[b][a][c] = sum_d log N(z_i[b,a,d]; mu_i[b,c,d], exp(logvar_i[b,c,d])) - logq_i[b,a]
 * logf is DEVICE [B][K_i][K_p] fp32.  O(B K_i K_p) HBM writes: for inspection/export; the
 * estimator never materialises it. */
tmc_status tmc_factors(const tmc_graph *g, int32_t i, const tmc_latent_in *in_i, float *logf,
                       tmc_stream_t stream);

/* Forward pass: logp[b] (DEVICE fp64 [B]).  in = HOST array of n tmc_latent_in.
 * logf_dense: NULL for the fused Gaussian path, else a HOST array of n DEVICE pointers
 * logf_i [B][K_i][K_p] (already containing -logq); then only in[i].logobs is read.
 * ws/ws_bytes: device workspace; it holds the state tmc_backward needs. */
tmc_status tmc_forward(const tmc_graph *g, const tmc_latent_in *in, const float *const *logf_dense,
                       double *logp, void *ws, size_t ws_bytes, tmc_stream_t stream);

/* Reverse pass for J = sum_b dlogp[b] logp[b] (dlogp DEVICE fp64 [B], NULL = all ones).
 * Requires the workspace of a tmc_forward on the same graph/inputs, earlier on `stream`.
 * out = HOST array of n tmc_latent_grad.  On the dense path dlogf_dense (HOST array of n
 * DEVICE pointers, entries may be NULL) receives dJ/dlogf_i, and dz/dmu/dlogvar/dlogq are
 * not written. */
tmc_status tmc_backward(const tmc_graph *g, const tmc_latent_in *in, const float *const *logf_dense,
                        void *ws, size_t ws_bytes, const double *dlogp, tmc_latent_grad *out,
                        float *const *dlogf_dense, tmc_stream_t stream);

/* tmc_forward + tmc_backward on the fused Gaussian path (same results, same workspace).  Small
 * problems (every K_i <= 64, D_i <= 128, n <= 32, AUTO precision and direction) run as ONE kernel
 * launch that writes logp and every gradient; the workspace is then left untouched. */
tmc_status tmc_estimate(const tmc_graph *g, const tmc_latent_in *in, double *logp, const double *dlogp,
                        tmc_latent_grad *out, void *ws, size_t ws_bytes, tmc_stream_t stream);

/* Shared-root trees sharded over processes (the star graph of P:334-346: a global latent theta
 * with K_theta samples shared by N data points, each with its own latent z_i).  Each shard holds
 * the root and a subset of its children (subtrees); the root's incoming messages are additive in
 * the log domain, so the TMC estimate needs ONE exchange:
 *   1. tmc_forward_children on every shard: the forward pass of every latent below the root;
 *      root_msg (DEVICE fp64 [B][K_root+1]) receives, for datapoint b, the sum over this shard's
 *      root children j of msg_{j->root}[b][r] as fp32 residuals summed in fp64 (r < K_root) and
 *      the sum of their fp64 offsets (entry K_root).  A shard without children writes zeros.
 *   2. the caller sums root_msg over shards (e.g. ncclAllReduce SUM, fp64).
 *   3. tmc_forward_root on every shard with the summed root_msg: h_root = u_root + sum, the
 *      root's elimination and logp (identical on every shard).
 *   4. tmc_backward as usual: gradients of this shard's latents under the global root marginal.
 *      The root's own gradients (dz/dmu/dlogvar/dlogq/dlogobs of the root) are computed on every
 *      shard identically; count them once.
 * Requirements: exactly one root, direction = TMC_DIR_UP (explicitly: a shard holding one child
 * is a chain), the same workspace for steps 1, 3 and 4 on the same stream. */
tmc_status tmc_forward_children(const tmc_graph *g, const tmc_latent_in *in, double *root_msg, void *ws,
                                size_t ws_bytes, tmc_stream_t stream);
tmc_status tmc_forward_root(const tmc_graph *g, const tmc_latent_in *in, const double *root_msg_total,
                            double *logp, void *ws, size_t ws_bytes, tmc_stream_t stream);

/* Streamed estimate from HOST inputs (the end-to-end path of a caller whose samples live in
 * host memory).  Datapoints are independent problems, so the batch is cut into
 * chunks of `chunk` datapoints: chunk c+1's inputs are copied host->device on an internal
 * copy stream (one per device, created on first use) into one of two staging slots of `ws`
 * while chunk c runs tmc_estimate on `stream`; PCIe transfer and kernels overlap.
 *   in         HOST array of n tmc_latent_in whose buffers are HOST memory, same layouts as
 *              tmc_latent_in (page-locked for the overlap; pageable memory works, serialised).
 *   logp_host  HOST fp64 [B]; written by the time `stream` passes the call's last operation
 *              (page-locked for an asynchronous copy).
 *   dlogp_host HOST fp64 [B] or NULL (= all ones).
 *   out        DEVICE gradients in the full-batch layout of tmc_latent_grad, or NULL for
 *              logp only.
 *   ws         DEVICE workspace of tmc_estimate_host_workspace_size(g, chunk) bytes: two
 *              input staging slots + the tmc_estimate workspace of one chunk.
 * The host buffers must stay valid and unmodified until `stream` completes the call's work. */
size_t tmc_estimate_host_workspace_size(const tmc_graph *g, int32_t chunk);
tmc_status tmc_estimate_host(const tmc_graph *g, const tmc_latent_in *in, double *logp_host,
                             const double *dlogp_host, tmc_latent_grad *out, int32_t chunk, void *ws,
                             size_t ws_bytes, tmc_stream_t stream);

/* IWAE at equal K on the same inputs, for side-by-side cost and
 * bound comparisons with TMC: the K joint samples are the index tuples (k, ..., k) (latent i's k-th
 * sample, its conditional at the parent's k-th sample, a root at its prior row 0):
 *   logp[b] = log (1/K) sum_k exp( sum_i [log N(z_i[b,k]; mu_i[b,c], e^{v_i[b,c]}) - logq_i[b,k] + logobs_i[b,k]] ),
 * c = k (root: 0), times factor_power like tmc_forward.  Requires K_i equal on every latent
 * (else TMC_ERR_SHAPE).  out (may be NULL) receives the gradient of J = sum_b dlogp[b] logp[b]
 * in tmc_latent_grad's layout; only the diagonal rows c = k of dmu/dlogvar are written (the other
 * rows have zero gradient and are left untouched); pair_marginal is ignored.
 * ws: DEVICE workspace of tmc_iwae_workspace_size(g) bytes. */
size_t tmc_iwae_workspace_size(const tmc_graph *g);
tmc_status tmc_iwae(const tmc_graph *g, const tmc_latent_in *in, double *logp, const double *dlogp,
                    tmc_latent_grad *out, void *ws, size_t ws_bytes, tmc_stream_t stream);

/* Reparameterisation noise for the proposal samples z = mu_q + sigma_q * eps (SURVEY
 * §8a row a1): eps[b][k][d] ~ N(0, 1), DEVICE fp32 [B][K][D] (16-byte aligned when D % 4 == 0),
 * for global datapoints b0 .. b0+B-1 of latent `latent`.  Counter-based and bit-exact across
 * devices, batch splits and world sizes: Philox4x32-10 with key = seed (lo, hi words) and counter
 * (tag, b0 + b, latent, k * ceil(D/4) + d/4) gives the 4 words of dims 4j..4j+3; each word pair
 * (w0, w1) -> u = ((w >> 8) + 0.5) 2^-24 -> Box-Muller sqrt(-2 ln u0) (cos, sin)(2 pi u1), with ln,
 * cos and sin as fixed fp32 polynomials in correctly rounded fma/mul/add/div/sqrt (no libm), so a
 * host implementation performing the same operations reproduces every bit.
 * Limits: K * ceil(D/4) <= 2^31 - 1 and b0 + B <= 2^32 - 1 (32-bit counter words), else
 * TMC_ERR_SHAPE. */
tmc_status tmc_sample_normal(uint64_t seed, uint32_t tag, int32_t B, int64_t b0, int32_t latent, int32_t K,
                             int32_t D, float *eps, tmc_stream_t stream);


/* ---------------------------------------------------------------- general elimination (NEXT-4)
 * The TMC estimate of an arbitrary (loopy) factor graph over sample indices, PAPER.md "Efficient
 * averaging" (Fig[factor:loop] P:145-215):
 *     logp[b] = log( 1/(K_0 ... K_{nvar-1}) sum_{k_0..k_{nvar-1}} prod_j f_j^{kappa_j} )
 * computed by summing the indices out one at a time in `order`:
 *     f_new^{kappa'} = 1/K_v sum_{k_v} prod_{j: v in kappa_j} f_j^{kappa_j},  kappa' = (U kappa_j) \ {v}
 * e.g. Fig[factor:loop]: f_12^{k2 k3} = 1/K1 sum_{k1} f_1^{k1 k2} f_2^{k1 k3}.  Log-domain, online
 * max (never the appendix's separate maxima, reading A2); the K^{|kappa'|+1} summand of a step is
 * never stored.  Discrete latents summed out exactly are the special case of one
 * "sample" per state with uniform Q.
 *   logf[j]   DEVICE fp32 [B][K_{s0}][K_{s1}][K_{s2}] (row-major in the order of scope[j][.]) = log f_j;
 *             -inf allowed (a probability-zero event; an all -inf datapoint gives logp = -inf and
 *             zero gradients).
 *   arity[j]  1..3; scope[3 j + a] = the a-th index variable of factor j (a < arity[j]).
 *   order     HOST [nvar] permutation (NULL = 0, 1, ..., nvar-1).  Every factor created by an
 *             elimination must have <= 3 indices and every index may appear in <= 8 factors at its
 *             turn, else TMC_ERR_SHAPE (choose another order).  An index no factor contains
 *             contributes exactly 1 (1/K_v sum_{k_v} 1).
 * tmc_elim_forward writes logp (DEVICE fp64 [B]) and keeps the intermediate factors in ws.
 * tmc_elim_backward (after tmc_elim_forward on the same graph, tables and ws, same stream) writes
 * dlogf[j] = dJ/dlogf_j for J = sum_b dlogp[b] logp[b] (dlogp DEVICE fp64 [B] or NULL = ones; a
 * NULL entry of dlogf = not wanted) = dlogp[b] times the marginal of kappa_j under the normalised
 * summand.  Deterministic (no atomics).  B <= 65535. */
typedef struct {
  int32_t nvar;           /* index variables k_0 .. k_{nvar-1}, >= 1                            */
  int32_t B;              /* datapoints (independent problems), >= 0                            */
  const int32_t *K;       /* HOST [nvar] samples (or states) per index, >= 1                     */
  int32_t nfac;           /* factors, >= 1                                                      */
  const int32_t *arity;   /* HOST [nfac] 1..3                                                   */
  const int32_t *scope;   /* HOST [nfac][3] index variables of each factor (table axis order)   */
  const int32_t *order;   /* HOST [nvar] elimination order, or NULL                             */
} tmc_factor_graph;
size_t tmc_elim_workspace_size(const tmc_factor_graph *g);   /* 0 if the graph/order is invalid */
tmc_status tmc_elim_forward(const tmc_factor_graph *g, const float *const *logf, double *logp, void *ws,
                            size_t ws_bytes, tmc_stream_t stream);
tmc_status tmc_elim_backward(const tmc_factor_graph *g, const float *const *logf, const double *logp, void *ws,
                             size_t ws_bytes, const double *dlogp, float *const *dlogf, tmc_stream_t stream);

/* Thread-local message describing the last non-OK status on this thread. */
const char *tmc_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
int32_t tmc_version(void);

/* Diagnostics: number of kernels libtmc has launched in this process so far (all streams). */
uint64_t tmc_launch_count(void);

/* Diagnostics: per-kernel-family device time (bench.py's roofline).  tmc_profile_begin
 * synchronises the device, clears the counters and enables recording: until tmc_profile_end,
 * every libtmc launch is bracketed by a CUDA event pair recorded on its launching stream, and the
 * tensor-core kernels add the tcgen05 MMA flops they issue (live tiles only) to a device counter.
 * tmc_profile_end synchronises, disables recording and writes one entry per family that launched
 * (at most max_entries) to HOST `out`; it returns the number of entries or a negative tmc_status.
 * Not thread-safe against concurrent begin/end; not for use during CUDA-graph capture. */
typedef struct {
  const char *family;   /* static string: kernel family name                                */
  uint64_t launches;    /* launches recorded                                                */
  double ms;            /* summed device time between each launch's event pair              */
  double mma_flops;     /* tcgen05 flops the family issued (0 for non-tensor-core families) */
} tmc_profile_entry;
int32_t tmc_profile_begin(void);
int32_t tmc_profile_end(tmc_profile_entry *out, int32_t max_entries);

#ifdef __cplusplus
}
#endif
#endif /* TMC_H_ */
