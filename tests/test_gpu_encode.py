"""Encode kernels (secondary path) against the reference's own assignment
functions (oracle/_ref when built, else the C restatement pinned to it):
center codes, alphas and per-point losses bit-for-bit (fp64)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _checker():
    from oracle.oracle import Port, Ref
    return Ref() if Ref.available() else Port()


def _weights(x, t, dbar):
    """aniso_weights per point (host-side, the reference's libm sin) — only
    via the reference library; the restatement keeps zeros for zero rows."""
    from oracle.oracle import Ref
    hp = np.zeros(len(x))
    hb = np.zeros(len(x))
    if not Ref.available():
        pytest.skip("aniso weights need oracle/_ref (glibc sin, SURVEY App. C.9)")
    R = Ref()
    for i in range(len(x)):
        nrm = float(np.sqrt(np.dot(x[i].astype(np.float64), x[i].astype(np.float64))))
        if nrm > 0:
            hp[i], hb[i] = R.aniso_weights(nrm, t, dbar)
    return hp, hb


@pytest.mark.parametrize("dbar,k", [(2, 16), (4, 16), (4, 256), (3, 7)])
def test_assign_projective_bit_exact(dbar, k):
    import torch
    import paper_2112_02179_b200 as P
    rng = np.random.default_rng(dbar * 100 + k)
    x = rng.standard_normal((20000, dbar)).astype(np.float32)
    x[::97] = 0.0
    c = rng.standard_normal((k, dbar)).astype(np.float32)
    a, al, lo = P.assign_projective(torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda())
    torch.cuda.synchronize()
    ra, ral, rlo = _checker().assign_projective(x, c)
    assert np.array_equal(a.cpu().numpy().astype(np.uint32), ra)
    assert al.cpu().numpy().tobytes() == ral.tobytes()
    assert lo.cpu().numpy().tobytes() == rlo.tobytes()


@pytest.mark.parametrize("dbar,k", [(2, 16), (4, 16), (4, 64)])
def test_assign_anisotropic_and_alpha_codes_bit_exact(dbar, k):
    import torch
    import paper_2112_02179_b200 as P
    from oracle.oracle import Port
    rng = np.random.default_rng(dbar * 7 + k)
    x = (rng.standard_normal((5000, dbar)) * 0.3).astype(np.float32)
    x[::53] = 0.0
    c = rng.standard_normal((k, dbar)).astype(np.float32)
    hp, hb = _weights(x, 0.2, dbar)
    tx = torch.from_numpy(x).cuda()
    tc = torch.from_numpy(c).cuda()
    thp, thb = torch.from_numpy(hp).cuda(), torch.from_numpy(hb).cuda()
    a, al, lo = P.assign_anisotropic(tx, tc, thp, thb)
    torch.cuda.synchronize()
    ra, ral, rlo = _checker().assign_anisotropic(x, c, hp, hb)
    assert np.array_equal(a.cpu().numpy().astype(np.uint32), ra)
    assert al.cpu().numpy().tobytes() == ral.tobytes()
    assert lo.cpu().numpy().tobytes() == rlo.tobytes()
    values = np.sort(rng.standard_normal(8)).astype(np.float32)
    codes = P.aniso_alpha_codes(tx, tc, a, thp, thb, torch.from_numpy(values).cuda())
    torch.cuda.synchronize()
    want = Port().alpha_codes_aniso(x, c, ra, hp, hb, values)
    assert np.array_equal(codes.cpu().numpy(), want)
