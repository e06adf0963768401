"""Pins for the fp64 CPU oracle (oracle/), against things other than itself.

Each test names the passage or mathematical fact it pins.  These run without a GPU.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import logsumexp
from scipy.stats import multivariate_normal, norm

import oracle
import tmc_workload as tw
from bruteforce import log_factor, log_weights, pair_marginals, tmc_bruteforce, workload_datapoint

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TINY = ["S_chain", "S_tree", "S_mnist", "S_mlp", "S_mlp_bern", "S_hier", "C0"]


def _f(v):
    return -math.inf if v == "-inf" else (math.inf if v == "inf" else v)


# ----------------------------------------------------------------------------- log-domain primitives
def test_logsumexp_spec_examples():
    g = json.load(open(os.path.join(GOLDEN, "logdomain_examples.json")))
    for case in g["logsumexp"]:
        x = [_f(v) for v in case["x"]]
        got = oracle.logsumexp(x)
        exp = _f(case["expect"])
        if math.isinf(exp):
            assert got == exp, case["cite"]
        else:
            assert abs(got - exp) <= 1e-12 * max(1.0, abs(exp)), case["cite"]
    assert oracle.logsumexp([]) == -math.inf


def test_logmmexp_spec_examples_and_A2_counterexample():
    g = json.load(open(os.path.join(GOLDEN, "logdomain_examples.json")))
    for case in g["logmmexp"]:
        Z = oracle.logmmexp(np.array(case["X"]), np.array(case["Y"]))
        np.testing.assert_allclose(Z, np.array(case["expect"]), rtol=1e-13, atol=1e-12, err_msg=case["cite"])


def test_logmmexp_matches_exp_domain_product():
    # S:94 invariant: for |entries| <= 50, logmmexp == log(exp(X) @ exp(Y)) within 1e-12.
    rng = np.random.default_rng(1)
    X = rng.uniform(-50, 50, (5, 7))
    Y = rng.uniform(-50, 50, (7, 3))
    np.testing.assert_allclose(oracle.logmmexp(X, Y), np.log(np.exp(X) @ np.exp(Y)), rtol=1e-13, atol=1e-12)


# ----------------------------------------------------------------------------- factor
def test_factor_hand_computed_D1():
    # log N(1; 0, 1) = -1/2 - ln(2 pi)/2 ; logq subtracted.
    z = np.array([[[1.0]]], np.float32)
    mu = np.zeros((1, 1, 1), np.float32)
    lv = np.zeros((1, 1, 1), np.float32)
    lq = np.array([[0.25]], np.float32)
    f = oracle.factor([-1], [1], [1], 0, z, mu, lv, lq)
    assert abs(f[0, 0, 0] - (-0.5 - 0.5 * math.log(2 * math.pi) - 0.25)) < 1e-15


@pytest.mark.parametrize("name", ["C0", "S_tree", "S_mnist", "S_mlp"])
def test_factor_matches_scipy(name):
    wl = tw.make_workload(name)
    for i in range(len(wl.parent)):
        f = oracle.factor(wl.parent, wl.K, wl.D, i, wl.z[i], wl.mu[i], wl.logvar[i], wl.logq[i])
        for b in range(wl.B):
            ref = log_factor(wl.z[i][b], wl.mu[i][b], wl.logvar[i][b], wl.logq[i][b])
            np.testing.assert_allclose(f[b], ref, rtol=1e-12, atol=1e-10)


# ----------------------------------------------------------------------------- estimator value
@pytest.mark.parametrize("name", TINY)
def test_estimate_equals_bruteforce(name):
    """Eq. is: message passing == explicit sum over all prod K_i tuples."""
    wl = tw.make_workload(name)
    up = oracle.estimate_workload(wl, direction="up", grads=False)["logp"]
    chain = all(p == i - 1 for i, p in enumerate(wl.parent))
    down = oracle.estimate_workload(wl, direction="down", grads=False)["logp"] if chain else up
    for b in range(wl.B):
        fac, obs = workload_datapoint(wl, b)
        ref = tmc_bruteforce(wl.parent, wl.K, fac, obs)
        assert abs(up[b] - ref) <= 1e-10 * max(1.0, abs(ref)), (b, up[b], ref)
        assert abs(down[b] - ref) <= 1e-10 * max(1.0, abs(ref)), (b, down[b], ref)


def test_fault_injection_breaks_bruteforce():
    """+ln 2 on one factor entry must be detected by the brute-force pin."""
    wl = tw.make_workload("S_chain")
    fac, obs = workload_datapoint(wl, 0)
    ref = tmc_bruteforce(wl.parent, wl.K, fac, obs)
    dense = [oracle.factor(wl.parent, wl.K, wl.D, i, wl.z[i], wl.mu[i], wl.logvar[i], wl.logq[i]).astype(np.float32)
             for i in range(len(wl.parent))]
    good = oracle.estimate(wl.parent, wl.K, wl.D, None, None, None, None, wl.logobs, logf_dense=dense,
                           grads=False)["logp"][0]
    dense[2][0, 1, 2] += math.log(2.0)
    bad = oracle.estimate(wl.parent, wl.K, wl.D, None, None, None, None, wl.logobs, logf_dense=dense,
                          grads=False)["logp"][0]
    assert abs(good - ref) < 1e-5          # fp32 rounding of the dense factors only
    assert abs(bad - ref) > 1e-3


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_up_down_and_dense_agree_on_large_family(name):
    """Order invariance and dense-factor path == Gaussian path, on 2 datapoints at reduced K."""
    wl = tw.make_workload(name, b_ids=[0, 7], K=24)
    up = oracle.estimate_workload(wl, direction="up", grads=False)["logp"]
    if all(p == i - 1 for i, p in enumerate(wl.parent)):
        down = oracle.estimate_workload(wl, direction="down", grads=False)["logp"]
        np.testing.assert_allclose(down, up, rtol=1e-12, atol=1e-9)
    dense = [oracle.factor(wl.parent, wl.K, wl.D, i, wl.z[i], wl.mu[i], wl.logvar[i], wl.logq[i])
             for i in range(len(wl.parent))]
    # dense path reads float32 factors: compare against the brute-force-free identity at fp32 rounding
    d = oracle.estimate(wl.parent, wl.K, wl.D, None, None, None, None, wl.logobs,
                        logf_dense=[x.astype(np.float32) for x in dense], grads=False)["logp"]
    np.testing.assert_allclose(d, up, rtol=1e-6, atol=1e-3)


def test_K1_reduces_to_single_sample_elbo():
    """K=1: P_TMC = P(x,z)/Q(z), computed monolithically from the model."""
    wl = tw.make_workload("C0", K=1)
    got = oracle.estimate_workload(wl, grads=False)["logp"]
    p = wl.params
    for b in range(wl.B):
        z = [wl.z[i][b, 0].astype(np.float64) for i in range(4)]
        lp = multivariate_normal.logpdf(z[0], np.zeros(2), np.eye(2))
        for i in range(1, 4):
            lp += multivariate_normal.logpdf(z[i], p["W"][i] @ z[i - 1], 0.5 * np.eye(2))
        lp += multivariate_normal.logpdf(wl.x[b][0], p["C"][3] @ z[3], 0.1 * np.eye(4))
        lq = sum(multivariate_normal.logpdf(z[i], np.zeros(2), 2.0 * np.eye(2)) for i in range(4))
        assert abs(got[b] - (lp - lq)) < 1e-5 * max(1, abs(lp)), b   # logq/logobs are fp32 inputs


def test_W0_decouples_into_independent_averages():
    """W=0: every conditional ignores its parent, so sum_k prod_i f_i(k_i) = prod_i sum_{k_i} f_i(k_i)."""
    wl = tw.make_workload("C0", w_var=0.0)
    got = oracle.estimate_workload(wl, grads=False)["logp"]
    for b in range(wl.B):
        tot = 0.0
        for i in range(4):
            t = norm.logpdf(wl.z[i][b].astype(np.float64), 0.0, math.sqrt(1.0 if i == 0 else 0.5)).sum(-1)
            t = t - wl.logq[i][b]
            if wl.logobs[i] is not None:
                t = t + wl.logobs[i][b]
            tot += logsumexp(t) - math.log(wl.K[i])
        assert abs(got[b] - tot) < 1e-5, (b, got[b], tot)


def test_neg_inf_handling():
    """-inf entries are probability-zero events; an all -inf slice gives -inf and zero gradients, no NaN."""
    wl = tw.make_workload("S_chain")
    wl.logobs[3][0, 1] = -np.inf                  # one impossible sample
    wl.logobs[3][1, :] = -np.inf                  # datapoint 1 impossible
    r = oracle.estimate_workload(wl, direction="up")
    fac, obs = workload_datapoint(wl, 0)
    assert abs(r["logp"][0] - tmc_bruteforce(wl.parent, wl.K, fac, obs)) < 1e-10
    assert r["logp"][1] == -np.inf
    for key in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs"):
        for g in r[key]:
            assert not np.isnan(g).any()
            assert np.all(g[1] == 0.0)
    assert r["dlogobs"][3][0, 1] == 0.0


# ----------------------------------------------------------------------------- unbiasedness E[exp L] = p(x)
def _mc_check(logp, logpx, nsig=4.0):
    w = np.exp(logp - logpx)
    m, se = w.mean(), w.std(ddof=1) / math.sqrt(len(w))
    assert abs(m - 1.0) <= nsig * se, (m, se)
    assert logp.mean() <= logpx + 1e-9          # Jensen: L = E log P <= log p(x)
    return m, se


@pytest.mark.parametrize("K", [1, 3, 8])
def test_unbiased_hierarchical_toy(K):
    """Toy 1: star graph theta -> z_i -> x_i, closed-form evidence."""
    g = json.load(open(os.path.join(GOLDEN, "toy_evidence.json")))["hierarchical"]
    for case in g["cases"]:
        x = np.array(case["x"])
        N = len(x)
        R = 100_000
        rng = np.random.default_rng([17, K, N])
        n = N + 1
        parent = [-1] + [0] * N
        th = rng.normal(0, 1, (R, K, 1)).astype(np.float32)
        z = [th] + [rng.normal(0, math.sqrt(2), (R, K, 1)).astype(np.float32) for _ in range(N)]
        mu = [np.zeros((R, 1, 1), np.float32)] + [th.copy() for _ in range(N)]
        lv = [np.zeros((R, 1, 1), np.float32)] + [np.zeros((R, K, 1), np.float32) for _ in range(N)]
        lq = [norm.logpdf(th[..., 0], 0, 1).astype(np.float32)] + \
             [norm.logpdf(z[i][..., 0], 0, math.sqrt(2)).astype(np.float32) for i in range(1, n)]
        lo = [None] + [norm.logpdf(x[i - 1], z[i][..., 0], 1.0).astype(np.float32) for i in range(1, n)]
        logp = oracle.estimate(parent, [K] * n, [1] * n, z, mu, lv, lq, lo, grads=False)["logp"]
        _mc_check(logp, case["logpx"])


@pytest.mark.parametrize("proposal", ["factorised", "nonfactorised"])
def test_unbiased_chain_toy(proposal):
    """Toy 2: z_i|z_{i-1} ~ N(z_{i-1}, 1/N), x|z_N ~ N(z_N, 1); x ~ N(0, 2).
    Factorised Q(z_i) = N(0, i/N); non-factorised Q(z_i|z_{i-1}) with diagonal pairing,
    whose factors are indexed only by k_i (Eq. 2)."""
    g = json.load(open(os.path.join(GOLDEN, "toy_evidence.json")))["chain"]
    for case in g["cases"]:
        N, x, K, R = case["N"], case["x"], 4, 100_000
        rng = np.random.default_rng([23, N, proposal == "factorised"])
        s = math.sqrt(1.0 / N)
        z, lq = [], []
        for i in range(N):
            if proposal == "factorised":
                zi = rng.normal(0, math.sqrt((i + 1) / N), (R, K, 1))
                lqi = norm.logpdf(zi[..., 0], 0, math.sqrt((i + 1) / N))
            else:
                prev = np.zeros((R, K, 1)) if i == 0 else z[i - 1].astype(np.float64)
                zi = prev + s * rng.normal(0, 1, (R, K, 1))
                zi = zi.astype(np.float32)
                lqi = norm.logpdf(zi[..., 0], prev[..., 0], s)
            z.append(zi.astype(np.float32))
            lq.append(lqi.astype(np.float32))
        mu = [np.zeros((R, 1, 1), np.float32)] + [z[i - 1].copy() for i in range(1, N)]
        lv = [np.full((R, 1 if i == 0 else K, 1), math.log(1.0 / N), np.float32) for i in range(N)]
        lo = [None] * (N - 1) + [norm.logpdf(x, z[N - 1][..., 0], 1.0).astype(np.float32)]
        parent = [-1] + list(range(N - 1))
        logp = oracle.estimate(parent, [K] * N, [1] * N, z, mu, lv, lq, lo, grads=False)["logp"]
        _mc_check(logp, case["logpx"])


def test_unbiased_C0_closed_form():
    """C0 (BASELINE configs[0]): x ~ N(0, C S4 C^T + 0.1 I), S1 = I, Si = Wi S(i-1) Wi^T + 0.5 I."""
    wl = tw.make_workload("C0")
    p = wl.params
    S = np.eye(2)
    for i in range(1, 4):
        S = p["W"][i] @ S @ p["W"][i].T + 0.5 * np.eye(2)
    cov = p["C"][3] @ S @ p["C"][3].T + 0.1 * np.eye(4)
    R, K = 100_000, 8
    for b in (2, 3):      # datapoints with moderate evidence (well-conditioned MC)
        x = wl.x[b][0]
        logpx = multivariate_normal.logpdf(x, np.zeros(4), cov)
        rng = np.random.default_rng([29, b])
        z = [rng.normal(0, math.sqrt(2), (R, K, 2)).astype(np.float32) for _ in range(4)]
        lq = [norm.logpdf(zi.astype(np.float64), 0, math.sqrt(2)).sum(-1).astype(np.float32) for zi in z]
        mu = [np.zeros((R, 1, 2), np.float32)] + [(z[i - 1].astype(np.float64) @ p["W"][i].T).astype(np.float32)
                                                   for i in range(1, 4)]
        lv = [np.zeros((R, 1, 2), np.float32)] + [np.full((R, K, 2), math.log(0.5), np.float32) for _ in range(3)]
        m = z[3].astype(np.float64) @ p["C"][3].T
        lo = [None] * 3 + [(-0.5 * (((x - m) ** 2) / 0.1 + math.log(0.1) + math.log(2 * math.pi)).sum(-1)).astype(np.float32)]
        logp = oracle.estimate([-1, 0, 1, 2], [K] * 4, [2] * 4, z, mu, lv, lq, lo, grads=False)["logp"]
        _mc_check(logp, logpx)


# ----------------------------------------------------------------------------- gradients
@pytest.mark.parametrize("name", ["S_chain", "S_tree", "S_mnist", "S_mlp", "S_hier"])
def test_pair_marginals_match_bruteforce(name):
    """dL/dlogf_i = pair marginal of (k_i, k_pa) under normalised weights (autodiff of P:332)."""
    wl = tw.make_workload(name)
    r = oracle.estimate_workload(wl, pair=True)
    for b in range(wl.B):
        fac, obs = workload_datapoint(wl, b)
        P = pair_marginals(wl.parent, wl.K, fac, obs)
        for i in range(len(wl.parent)):
            np.testing.assert_allclose(r["pair"][i][b], P[i], atol=1e-10)
            np.testing.assert_allclose(r["dlogobs"][i][b], P[i].sum(1), atol=1e-10)
            np.testing.assert_allclose(r["dlogq"][i][b], -P[i].sum(1), atol=1e-10)
            assert abs(P[i].sum() - 1.0) < 1e-12


def _bf_value(wl, b, i, which, arr):
    """Brute-force log P_TMC of datapoint b with input `which` of latent i replaced by arr (fp64)."""
    n = len(wl.parent)
    fac, obs = [], []
    for j in range(n):
        z, mu, lv, lq = wl.z[j][b], wl.mu[j][b], wl.logvar[j][b], wl.logq[j][b]
        if j == i:
            z = arr if which == "z" else z
            mu = arr if which == "mu" else mu
            lv = arr if which == "logvar" else lv
        fac.append(log_factor(z, mu, lv, lq))
        obs.append(None if wl.logobs[j] is None else np.asarray(wl.logobs[j][b], np.float64))
    return tmc_bruteforce(wl.parent, wl.K, fac, obs)


@pytest.mark.parametrize("name", ["S_chain", "S_tree", "S_mlp"])
def test_gradients_match_central_finite_differences(name):
    """gradient vs central FD (h=1e-5) of the brute-force value, relative error < 1e-6."""
    wl = tw.make_workload(name)
    r = oracle.estimate_workload(wl)
    h = 1e-5
    key = {"z": "dz", "mu": "dmu", "logvar": "dlogvar"}
    for b in range(min(wl.B, 2)):
        for i in range(len(wl.parent)):
            for which, src in (("z", wl.z), ("mu", wl.mu), ("logvar", wl.logvar)):
                base = src[i][b].astype(np.float64)
                fd = np.zeros_like(base)
                for idx in np.ndindex(base.shape):
                    e = np.zeros_like(base)
                    e[idx] = h
                    fd[idx] = (_bf_value(wl, b, i, which, base + e) - _bf_value(wl, b, i, which, base - e)) / (2 * h)
                got = r[key[which]][i][b]
                scale = max(1e-3, np.abs(fd).max())
                assert np.abs(got - fd).max() / scale < 1e-6, (b, i, which, got, fd)


def test_dlogp_scales_gradients():
    wl = tw.make_workload("S_tree")
    r1 = oracle.estimate_workload(wl)
    w = np.array([0.5, -2.0, 0.0, 3.0])
    r2 = oracle.estimate_workload(wl, dlogp=w)
    for i in range(len(wl.parent)):
        np.testing.assert_allclose(r2["dz"][i], r1["dz"][i] * w[:, None, None], atol=1e-14)
        np.testing.assert_allclose(r2["dlogq"][i], r1["dlogq"][i] * w[:, None], atol=1e-14)


# ----------------------------------------------------------------------------- factor power (NEXT-1)
@pytest.mark.parametrize("name", ["S_chain", "S_tree", "S_mlp", "S_mnist"])
def test_alpha2_is_sum_of_squared_weights(name):
    """alpha = 2: "running TMC again, with squared weights" == log((1/prod K) sum w^2),
    the second quantity of the DReGs surrogate, by brute-force enumeration."""
    wl = tw.make_workload(name)
    r = oracle.estimate_workload(wl, alpha=2.0, grads=False)
    for b in range(wl.B):
        fac, obs = workload_datapoint(wl, b)
        fac2 = [2.0 * f for f in fac]
        obs2 = [None if o is None else 2.0 * o for o in obs]
        assert abs(r["logp"][b] - tmc_bruteforce(wl.parent, wl.K, fac2, obs2)) < 1e-10


def test_alpha2_gradients_match_finite_differences():
    wl = tw.make_workload("S_tree")
    r = oracle.estimate_workload(wl, alpha=2.0)
    h = 1e-5
    b = 1

    def val(i, which, arr):
        fac, obs = [], []
        for j in range(len(wl.parent)):
            z, mu, lv, lq = wl.z[j][b], wl.mu[j][b], wl.logvar[j][b], wl.logq[j][b]
            if j == i:
                z = arr if which == "z" else z
                mu = arr if which == "mu" else mu
            fac.append(2.0 * log_factor(z, mu, lv, lq))
            obs.append(None if wl.logobs[j] is None else 2.0 * np.asarray(wl.logobs[j][b], np.float64))
        return tmc_bruteforce(wl.parent, wl.K, fac, obs)

    for i in range(len(wl.parent)):
        for which, src, key in (("z", wl.z, "dz"), ("mu", wl.mu, "dmu")):
            base = src[i][b].astype(np.float64)
            fd = np.zeros_like(base)
            for idx in np.ndindex(base.shape):
                e = np.zeros_like(base)
                e[idx] = h
                fd[idx] = (val(i, which, base + e) - val(i, which, base - e)) / (2 * h)
            assert np.abs(r[key][i][b] - fd).max() / max(1e-3, np.abs(fd).max()) < 1e-6


def test_dregs_surrogate_identity():
    """d/dz of 1/2 (sum w^2 / (sum w)^2) log sum w_hat^2 equals
    sum_i w_i^2/(sum w)^2 d log w_i / dz.  With L_a = log((1/prod K) sum w^a) from the oracle:
    1/2 exp(L_2 - 2 L_1 - sum ln K) * dL_2/dz  ==  the brute-force weighted sum (here w.r.t. z)."""
    wl = tw.make_workload("S_chain")
    r1 = oracle.estimate_workload(wl, alpha=1.0, grads=False)
    r2 = oracle.estimate_workload(wl, alpha=2.0)
    lnK = sum(math.log(k) for k in wl.K)
    for b in range(wl.B):
        fac, obs = workload_datapoint(wl, b)
        combos, lw = log_weights(wl.parent, wl.K, fac, obs)
        c = np.exp(2 * lw - 2 * logsumexp(lw))          # w_i^2 / (sum w)^2
        # d log w_i / d z_j[a, d]: log w_i depends on z_j[k_j] through factor j and its children
        for j in range(len(wl.parent)):
            g = np.zeros_like(wl.z[j][b], dtype=np.float64)
            h = 1e-6
            for idx in np.ndindex(g.shape):
                zp = wl.z[j][b].astype(np.float64).copy(); zp[idx] += h
                zm = wl.z[j][b].astype(np.float64).copy(); zm[idx] -= h
                def lwz(zz):
                    f2, o2 = list(fac), list(obs)
                    f2[j] = log_factor(zz, wl.mu[j][b], wl.logvar[j][b], wl.logq[j][b])
                    return log_weights(wl.parent, wl.K, f2, o2)[1]
                g[idx] = np.sum(c * (lwz(zp) - lwz(zm)) / (2 * h))
            scale = 0.5 * math.exp(r2["logp"][b] - 2 * r1["logp"][b] - lnK)
            np.testing.assert_allclose(scale * r2["dz"][j][b], g, rtol=1e-5, atol=1e-7)


# ----------------------------------------------------------------------------- row a1: sampling
def test_philox_known_answers():
    """Philox4x32-10 against the published known-answer vectors (tests/golden/philox_kat.json)."""
    kat = json.load(open(os.path.join(GOLDEN, "philox_kat.json")))["vectors"]
    for v in kat:
        h = lambda xs: [int(x, 16) for x in xs]
        assert oracle.philox4x32_10(h(v["ctr"]), h(v["key"])).tolist() == h(v["out"])


def test_box_muller_polynomials_accuracy():
    """The fixed fp32 ln / cos / sin polynomials of the sampler definition against numpy (fp64)."""
    u = np.concatenate([np.linspace(2.0 ** -24, 1.0, 20001), 2.0 ** -np.arange(1, 25)]).astype(np.float32)
    got = np.array([oracle.log_fp32(x) for x in u], np.float64)
    ref = np.log(u.astype(np.float64))
    assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30)) <= 1e-6 or np.max(np.abs(got - ref)) <= 2e-7
    assert np.max(np.abs(got - ref)) <= 4e-6                 # |ln u| <= 16.6: a few fp32 ulps
    v = np.linspace(0.0, 1.0, 20001, endpoint=False).astype(np.float32)
    cs = np.array([oracle.cos_sin_2pi(x) for x in v], np.float64)
    ang = 2 * np.pi * v.astype(np.float64)
    assert np.max(np.abs(cs[:, 0] - np.cos(ang))) <= 1e-6
    assert np.max(np.abs(cs[:, 1] - np.sin(ang))) <= 1e-6


def test_sample_normal_distribution_and_keying():
    """eps ~ N(0,1): moments and Kolmogorov-Smirnov on 2^20 draws; the draws of a datapoint do not
    depend on which batch slice produced them (counter = global id); ragged D uses a prefix of the
    4-wide group."""
    from scipy.stats import kstest
    e = oracle.sample_normal(7, 4, 64, 0, 3, 1024, 16).ravel().astype(np.float64)
    n = e.size
    assert abs(e.mean()) <= 5 / math.sqrt(n)
    assert abs(e.var() - 1) <= 5 * math.sqrt(2 / n)
    assert kstest(e, "norm").pvalue > 1e-3
    full = oracle.sample_normal(7, 4, 10, 0, 1, 33, 5)
    part = oracle.sample_normal(7, 4, 3, 6, 1, 33, 5)
    assert np.array_equal(full[6:9], part)
    d8 = oracle.sample_normal(7, 4, 2, 0, 1, 3, 8)
    d5 = oracle.sample_normal(7, 4, 2, 0, 1, 3, 5)
    assert np.array_equal(d8[..., :5], d5)       # same ceil(D/4): D = 5 is a prefix of D = 8
    d9 = oracle.sample_normal(7, 4, 2, 0, 1, 3, 9)
    assert np.array_equal(d9[:, 0, :8], d8[:, 0])   # k = 0 shares counters; k >= 1 moves with ceil(D/4)
    assert not np.array_equal(d9[:, 1, :8], d8[:, 1])
    other = oracle.sample_normal(8, 4, 10, 0, 1, 33, 5)
    assert not np.any(other == full)


# ----------------------------------------------------------------------------- NEXT-3: IWAE
def _iwae_wl(wl, **kw):
    return oracle.iwae(wl.parent, wl.K, wl.D, wl.z, wl.mu, wl.logvar, wl.logq, wl.logobs, **kw)


@pytest.mark.parametrize("name", TINY)
def test_iwae_equals_diagonal_bruteforce(name):
    """IWAE = log mean over the K diagonal index tuples of the brute-force weights."""
    from bruteforce import iwae_bruteforce
    wl = tw.make_workload(name)
    r = _iwae_wl(wl, grads=False)
    for b in range(wl.B):
        fac, obs = workload_datapoint(wl, b)
        assert abs(r["logp"][b] - iwae_bruteforce(wl.parent, wl.K, fac, obs)) <= 1e-10


def test_iwae_K1_equals_tmc_K1():
    """With one sample per latent IWAE and TMC are both the single-sample ELBO estimator."""
    wl = tw.make_workload("C0", K=1)
    a = _iwae_wl(wl, grads=False)["logp"]
    b = oracle.estimate_workload(wl, grads=False)["logp"]
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-10)


@pytest.mark.parametrize("name", ["S_chain", "S_tree", "S_mlp"])
def test_iwae_gradients_match_finite_differences(name):
    """Oracle IWAE gradients vs central differences of the brute-force diagonal value (scipy)."""
    from bruteforce import iwae_bruteforce, log_factor
    wl = tw.make_workload(name)
    r = _iwae_wl(wl, dlogp=np.ones(wl.B))
    rng = np.random.default_rng(5)
    b = 1
    h = 1e-3

    def value(zz, mm, vv):
        fac = [log_factor(zz[i], mm[i], vv[i], wl.logq[i][b]) for i in range(len(wl.parent))]
        obs = [None if wl.logobs[i] is None else wl.logobs[i][b].astype(np.float64) for i in range(len(wl.parent))]
        return iwae_bruteforce(wl.parent, wl.K, fac, obs)
    base = [[x[b].astype(np.float64) for x in arrs] for arrs in (wl.z, wl.mu, wl.logvar)]
    for which, key in ((0, "dz"), (1, "dmu"), (2, "dlogvar")):
        for _ in range(4):
            i = int(rng.integers(len(wl.parent)))
            arr = base[which][i]
            idx = tuple(int(rng.integers(s)) for s in arr.shape)
            vals = []
            for sgn in (1, -1):
                mod = [[a.copy() for a in lst] for lst in base]
                mod[which][i][idx] += sgn * h
                vals.append(value(*mod))
            fd = (vals[0] - vals[1]) / (2 * h)
            assert abs(fd - r[key][i][b][idx]) <= 1e-6 * max(1.0, abs(fd)), (key, i, idx, fd, r[key][i][b][idx])


def test_iwae_unbiased_C0_closed_form():
    """E[exp L_IWAE] = p(x) on C0's closed-form evidence, by Monte Carlo."""
    wl = tw.make_workload("C0")
    p = wl.params
    S = np.eye(2)
    for i in range(1, 4):
        S = p["W"][i] @ S @ p["W"][i].T + 0.5 * np.eye(2)
    cov = p["C"][3] @ S @ p["C"][3].T + 0.1 * np.eye(4)
    R, K = 100_000, 8
    b = 2
    x = wl.x[b][0]
    logpx = multivariate_normal.logpdf(x, np.zeros(4), cov)
    rng = np.random.default_rng([31, b])
    z = [rng.normal(0, math.sqrt(2), (R, K, 2)).astype(np.float32) for _ in range(4)]
    lq = [norm.logpdf(zi.astype(np.float64), 0, math.sqrt(2)).sum(-1).astype(np.float32) for zi in z]
    mu = [np.zeros((R, 1, 2), np.float32)] + [(z[i - 1].astype(np.float64) @ p["W"][i].T).astype(np.float32)
                                               for i in range(1, 4)]
    lv = [np.zeros((R, 1, 2), np.float32)] + [np.full((R, K, 2), math.log(0.5), np.float32) for _ in range(3)]
    m = z[3].astype(np.float64) @ p["C"][3].T
    lo = [None] * 3 + [(-0.5 * (((x - m) ** 2) / 0.1 + math.log(0.1) + math.log(2 * math.pi)).sum(-1)).astype(np.float32)]
    logp = oracle.iwae([-1, 0, 1, 2], [K] * 4, [2] * 4, z, mu, lv, lq, lo, grads=False)["logp"]
    _mc_check(logp, logpx, nsig=5.0)


# ----------------------------------------------------------------------------- exact discrete marginalisation
def test_oracle_dense_path_exact_discrete_marginalisation():
    """with K_i = number of states, stratified samples and uniform Q, the TMC estimate of
    an all-discrete chain IS log p(x) (the forward algorithm), and enumerating a discrete z_1 in a
    mixed model equals TMC on the model with z_1 marginalised out."""
    import discrete
    logf, obs, pi, A, _ = discrete.hmm(B=3, n=5, M=6)
    n, M = 5, 6
    r = oracle.estimate([-1] + list(range(n - 1)), [M] * n, [1] * n, None, None, None, None, obs,
                        logf_dense=logf, grads=False)
    np.testing.assert_allclose(r["logp"], discrete.hmm_forward_algorithm(logf, obs), rtol=0, atol=1e-9)
    lf, ob, p = discrete.mixed(B=3, M=4, K=7)
    r = oracle.estimate([-1, 0], [4, 7], [1, 1], None, None, None, None, ob, logf_dense=lf, grads=False)
    np.testing.assert_allclose(r["logp"], discrete.mixed_marginalised_reference(lf, ob, 7), rtol=0, atol=1e-9)
