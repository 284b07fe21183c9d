"""The drop-in boundary: libbvc_b200.so loads and exports every entry point that
include/bvc_b200.h declares; compute calls fail loudly without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2302_11825_b200 as B
from tests.conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "bvc_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bvc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = B.lib()
    names = declared_symbols()
    assert len(names) >= 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(B.api.SYMBOLS) == names
    version = int(re.search(r"#define BVC_ABI_VERSION (\d+)", open(os.path.join(ROOT, "include", "bvc_b200.h")).read())[1])
    assert lib.bvc_abi_version() == version


def test_library_is_built_for_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {B.library_path()} 2>&1").read()
    assert "sm_100a" in out, out


def _has_device():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.mark.skipif(_has_device(), reason="checks the no-GPU behaviour")
def test_compute_calls_fail_loudly_without_device():
    with pytest.raises(B.NoDeviceError):
        B.EvaluationPoints(np.zeros((4, 2)))
    with pytest.raises(B.NoDeviceError):
        B.eval_bessel(0, [1.0])
    sc = B.Scene(np.array([[0, 0], [1, 0], [0, 1]], float), [[0, 1], [1, 2], [2, 0]], [0, 0, 0])
    with pytest.raises(B.NoDeviceError):
        sc.closest_point([[0.2, 0.2]])


def test_error_codes_map_to_reference_exceptions():
    assert issubclass(B.ParseError, B.BvcError) and issubclass(B.SolverError, B.BvcError)
    msg = B.lib().bvc_last_error()
    assert isinstance(msg, bytes)


def test_library_has_no_unresolved_internal_symbols():
    """A declaration/definition mismatch between translation units links into a .so
    that only fails when it is loaded; catch it at build time."""
    import shutil
    import subprocess

    if shutil.which("nm") is None:
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--undefined-only", B.library_path()], capture_output=True, text=True).stdout
    bad = [line for line in out.splitlines() if "bvc_impl" in line or "bvc_capi" in line or "bvc_host" in line]
    assert not bad, bad
