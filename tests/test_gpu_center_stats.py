"""Lloyd center statistics on the GPU: bit-identical to the sequential
restatement (pinned to pcpq::center_anisotropic by test_oracle.py), for all
sections at once, and chainable through `init` (the multi-GPU ordered chain)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dbar,k,nsec", [(4, 16, 3), (2, 16, 2), (4, 7, 1)])
def test_center_stats_bit_exact_and_chainable(port, dbar, k, nsec):
    import torch
    import paper_2112_02179_b200 as P
    rng = np.random.default_rng(dbar * 31 + k)
    n = 30000
    x = (rng.standard_normal((nsec, n, dbar)) * 0.5).astype(np.float32)
    x[:, ::97] = 0.0
    assign = rng.integers(0, k, (nsec, n)).astype(np.int32)
    alpha = rng.standard_normal((nsec, n))
    hp = rng.uniform(0.01, 0.2, (nsec, n))
    hb = hp * rng.uniform(0.01, 0.9, (nsec, n))
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    got = P.center_stats(T(x), T(assign), T(alpha), T(hp), T(hb), k).cpu().numpy()
    for j in range(nsec):
        want = port.center_stats(x[j], assign[j], alpha[j], hp[j], hb[j], k)
        assert got[j].tobytes() == want.tobytes()
    # chain: points [0, h) then [h, n) continuing from the partials
    h = 12345
    first = P.center_stats(T(x[:, :h]), T(assign[:, :h]), T(alpha[:, :h]), T(hp[:, :h]), T(hb[:, :h]), k)
    second = P.center_stats(T(x[:, h:]), T(assign[:, h:]), T(alpha[:, h:]), T(hp[:, h:]), T(hb[:, h:]), k,
                            init=first)
    assert second.cpu().numpy().tobytes() == got.tobytes()


def test_assign_anisotropic_prev_fallback(port):
    """With a previous assignment, points keep their old center whenever that
    has the lower score-aware loss (clustering.cpp:339-349)."""
    import torch
    import paper_2112_02179_b200 as P
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((8000, 4)) * 0.4).astype(np.float32)
    c = rng.standard_normal((16, 4)).astype(np.float32)
    hp = rng.uniform(0.01, 0.2, 8000)
    hb = hp * rng.uniform(0.01, 0.9, 8000)
    prev = rng.integers(0, 16, 8000).astype(np.int32)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    a0, al0, lo0 = P.assign_anisotropic(T(x), T(c), T(hp), T(hb))
    a1, al1, lo1 = P.assign_anisotropic(T(x), T(c), T(hp), T(hb), prev=T(prev))
    a0, a1, lo0, lo1 = (v.cpu().numpy() for v in (a0, a1, lo0, lo1))
    ra, ral, rlo = port.assign_anisotropic(x, c, hp, hb)
    assert np.array_equal(a0.astype(np.uint32), ra)
    changed = a1 != a0
    assert np.all(a1[changed] == prev[changed])      # only ever falls back to prev
    assert np.all(lo1 <= lo0 + 0.0)                   # never a higher own loss
