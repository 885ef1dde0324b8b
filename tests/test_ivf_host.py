"""IVF host-side checks that need no GPU: the PCPQIVF1 container error
classes of pcpqg_ivf_load (validation happens before any device work) against
the reference's codes for the same corrupted containers (golden, made by
tests/golden/make_golden_ivf.py from pcpq::deserialize_ivf, proj/core/src/ivf.cpp:256-316),
and the numpy container round trip."""
import numpy as np
import pytest

import paper_2112_02179_b200 as P
from paper_2112_02179_b200 import pcpqivf
from tests.test_oracle_ivf import NAMES, corruptions, load_ivf


@pytest.mark.parametrize("name", NAMES)
def test_container_roundtrip(name):
    data, _ = load_ivf(name)
    iv = pcpqivf.deserialize(data)
    assert pcpqivf.serialize(iv) == data
    assert sorted(np.concatenate(iv.members).tolist()) == list(range(iv.n))


@pytest.mark.parametrize("name", NAMES)
def test_ivf_load_error_classes_match_reference(name):
    data, g = load_ivf(name)
    for (label, bad), code in zip(corruptions(data), g["error_codes"]):
        if code == 0:
            continue  # accepted containers go on to the device upload
        with pytest.raises(P.PcpqError) as e:
            P.deserialize_ivf(bad)
        assert e.value.status == code, (label, e.value)
