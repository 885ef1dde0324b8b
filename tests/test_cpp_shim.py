"""The C++ shim (include/pcpq_gpu.hpp) compiles against the C ABI here, and
on a GPU reproduces the reference's golden scores / LUT / top-n bit-for-bit."""
import os
import shutil
import subprocess

import pytest

from tests import _golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2112_02179_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "shim_parity")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_parity.cpp"), "-L", LIBDIR, "-lpcpqg",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_shim_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pcpq_q_m8_k16_s16", "apcpq_q_m10_k16_s8", "pcpq_raw16_m4_k16", "kmeans_k300_wide",
                                  "pcpq_q_ties"])
def test_shim_parity_on_gpu(tmp_path, name):
    exe = _build(tmp_path)
    data, g = _golden.load(name)
    files = {}
    for key, arr in [("q", g["queries"]), ("s", g["scores"]), ("i", g["ids10"]), ("t", g["top10"]), ("e", g["eta"])]:
        p = tmp_path / f"{key}.bin"
        p.write_bytes(arr.tobytes())
        files[key] = str(p)
    idx = tmp_path / "x.idx"
    idx.write_bytes(data)
    r = subprocess.run([exe, str(idx), files["q"], str(g["queries"].shape[0]), files["s"], files["i"], files["t"],
                        files["e"]], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
