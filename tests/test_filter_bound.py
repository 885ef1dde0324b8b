"""The K2-F error bound checked numerically on the CPU.

The kernel computes f_q = sum over octets of fp32(fp16 octet sum of
fp16(eta_hat) * fp16(lambda_hat)), with eta_hat = eta * sigma / tau_j and
lambda_hat = lambda * tau_j, and claims |f_q / sigma - score| <= eps_q. Here
score is the reference's sequential fp32 sum of fp32(eta * lambda). This test
replays that arithmetic in numpy with *unfused* fp16 multiply-then-add, which
is a harsher case than the kernel's HFMA2. It checks the bound, with the kernel's
sigma / tau / eps formulas, on random tables and codes across magnitudes."""
import numpy as np
import pytest


def frexp_e(x):
    return int(np.frexp(np.float64(x))[1]) if x > 0 else 0


def tables(rng, m, k, s, eta_scale, lam_scale):
    eta = (rng.standard_normal((m, k)) * eta_scale).astype(np.float32)
    lam = (rng.uniform(-1.5, 1.5, (m, s)) * lam_scale).astype(np.float32)
    return eta, lam


def kernel_constants(eta, lam):
    m = eta.shape[0]
    maxlam = np.abs(lam).max(axis=1).astype(np.float64)
    me = np.abs(eta).max(axis=1).astype(np.float64)
    pr = me * maxlam
    M, A = pr.max(), pr.sum()
    e = frexp_e(M)
    sigma = 2.0 ** (10 - e)
    u = 2.0 ** -11
    eps = (12 * u + 2.0 ** -20) * A + m * 1e-4 / sigma + (m + 1.0) * 1.02 * 2.0 ** -24 * A
    tau = np.array([2.0 ** -frexp_e(x) if x > 0 else 1.0 for x in maxlam])
    return sigma, tau, eps, maxlam


def filter_scores(eta, lam, codes_c, codes_l, sigma, tau, maxlam):
    m = eta.shape[0]
    live = maxlam > 0
    eh = np.where(live[:, None], eta.astype(np.float64) * sigma / tau[:, None], 0.0).astype(np.float16)
    lh = (lam.astype(np.float64) * tau[:, None]).astype(np.float16)
    n = codes_c.shape[0]
    f = np.zeros(n, np.float32)
    for o in range(0, m, 8):
        acc = np.zeros(n, np.float16)
        for j in range(o, min(o + 8, m)):
            prod = (eh[j, codes_c[:, j]] * lh[j, codes_l[:, j]]).astype(np.float16)  # rounded product
            acc = (acc + prod).astype(np.float16)                                     # rounded sum
        f = (f + acc.astype(np.float32)).astype(np.float32)
    return f


def reference_scores(eta, lam, codes_c, codes_l):
    n, m = codes_c.shape
    acc = np.full(n, -0.0, np.float32)
    for j in range(m):
        t = (eta[j, codes_c[:, j]] * lam[j, codes_l[:, j]]).astype(np.float32)
        acc = (acc + t).astype(np.float32)
    return acc


@pytest.mark.parametrize("m,eta_scale,lam_scale,seed", [(50, 0.05, 1.0, 1), (16, 1.0, 1e-3, 2), (64, 3.0, 40.0, 3),
                                                        (13, 1e-6, 1e6, 4), (50, 1e3, 1e-12, 5)])
def test_filter_bound_holds(m, eta_scale, lam_scale, seed):
    rng = np.random.default_rng(seed)
    k, s, n = 16, 8, 20000
    eta, lam = tables(rng, m, k, s, eta_scale, lam_scale)
    lam[rng.integers(0, m)] = 0.0  # a section without scale
    codes_c = rng.integers(0, k, (n, m))
    codes_l = rng.integers(0, s, (n, m))
    # points that stress the sums: every section at its largest |eta * lambda|
    jc = np.abs(eta).argmax(axis=1)
    jl = np.abs(lam).argmax(axis=1)
    codes_c[:50] = jc
    codes_l[:50] = jl
    sigma, tau, eps, maxlam = kernel_constants(eta, lam)
    f = filter_scores(eta, lam, codes_c, codes_l, sigma, tau, maxlam)
    ref = reference_scores(eta, lam, codes_c, codes_l)
    err = np.abs(f.astype(np.float64) / sigma - ref.astype(np.float64))
    assert np.all(np.isfinite(f))
    assert err.max() <= eps, (err.max(), eps)
    # and the bound is not vacuous: observed eps / max error is 15-51 on these cases
    assert eps < 200 * max(err.max(), 1e-300) or err.max() == 0.0
