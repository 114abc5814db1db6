"""The C ABI from plain C (examples/lik_demo.c): the header compiles as C99 and the
program links against liblik.so (CPU); on a GPU its output equals the Python
binding's bitwise on the same inputs, and the call-level error path reports
EDOMAIN with the offending index."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2305_04318_b200")


def _compile(tmp_path):
    from paper_2305_04318_b200 import build
    build.build()
    exe = str(tmp_path / "lik_demo")
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-Wall", "-Werror", os.path.join(ROOT, "examples", "lik_demo.c"),
                           "-I", os.path.join(ROOT, "include"), "-L", LIBDIR, "-llik",
                           f"-Wl,-rpath,{LIBDIR}", "-lm", "-o", exe])
    return exe


def test_c_client_compiles_and_links(tmp_path):
    exe = _compile(tmp_path)
    assert os.access(exe, os.X_OK)


def _inputs():
    """The LCG of lik_demo.c."""
    s = 2305043180
    mask = (1 << 64) - 1

    def u():
        nonlocal s
        s = (s * 6364136223846793005 + 1442695040888963407) & mask
        return (s >> 11) * (1.0 / 9007199254740992.0)

    n, p = 96, 2
    coords, y, X = np.empty((n, 2)), np.empty(n), np.empty((n, p))
    for i in range(n):
        coords[i, 0] = 10000.0 * u()
        coords[i, 1] = 10000.0 * u()
        y[i] = 1.0 + 2.0 * u()
        X[i] = (1.0, coords[i, 0] / 1e4)
    P = np.array([[1500.0, 0.5, 0.2, 1.0, 0.0], [800.0, 2.0, 0.05, 2.5, 0.6], [3000.0, 7.5, 0.5, 0.5, -1.0]])
    return coords, y, X, P, np.array([0.0, 0.5])


@pytest.mark.gpu
def test_c_client_matches_python_binding(tmp_path):
    import paper_2305_04318_b200 as lik
    exe = _compile(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    ctx = lik.create(0)
    ref = ctx.eval_batch(*_inputs())
    ctx.close()
    for k in range(3):
        f = lines[k].split()
        assert int(f[3]) == ref["status"][k]
        assert float(f[5]) == ref["logdetV"][k]
        assert [float(f[7]), float(f[9])] == list(ref["loglik"][k])
    assert lines[3].startswith("error -2 ") and "7" in lines[3], lines[3]
