"""CPU-side checks of the boundary (-m "not gpu"): the C-ABI library builds,
loads, and exports every symbol include/lik.h declares; the binding has no
CPU fallback; the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "lik.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(lik_\w+)\s*\(", src, re.M)))


def test_header_declares_expected_entry_points():
    syms = _header_symbols()
    for s in ("lik_create", "lik_eval_batch", "lik_eval_batch_device", "lik_last_error", "lik_destroy"):
        assert s in syms


def test_library_builds_loads_and_exports_every_symbol():
    from paper_2305_04318_b200 import build
    path = build.build()
    L = ctypes.CDLL(path)
    for s in _header_symbols():
        assert hasattr(L, s), s
    import paper_2305_04318_b200 as lik
    assert sorted(lik.ABI_SYMBOLS) == _header_symbols()
    nm = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for s in _header_symbols():
        assert re.search(rf"\bT {s}\b", nm), s


def test_sass_uses_fp64_tensor_cores_and_bulk_copies():
    from paper_2305_04318_b200 import build
    path = build.build()
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass
    assert "UBLKCP" in sass


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2305_04318_b200 as lik
    with pytest.raises(lik.LikError):
        lik.create(0)


def test_product_package_does_not_touch_oracle():
    pkg = os.path.join(ROOT, "paper_2305_04318_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle/" not in txt, f
