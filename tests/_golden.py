"""Loader for the golden fixtures in tests/golden/ (made by the unmodified
reference library; see tests/golden/make_golden.py)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.idx")))


def load(name):
    with open(os.path.join(GOLDEN, name + ".idx"), "rb") as f:
        data = f.read()
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return data, {k: z[k] for k in z.files}


def corruptions(name, data):
    """Re-create the corrupted images of make_golden.corrupt_cases."""
    import sys
    sys.path.insert(0, GOLDEN)
    from make_golden import corrupt_cases  # noqa: E402
    from paper_2112_02179_b200 import pcpqidx
    return corrupt_cases(data, pcpqidx.deserialize(data))
