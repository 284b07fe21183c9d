"""A compiled C++ caller of the C ABI (include/bvc_b200.h): INTEGRATION.md's
runSolveInMemory snippet as a real program (tests/cpp/integration_example.cpp), built
with g++ against libbvc_b200.so. On a host without a GPU it must build, load and
report BVC_ERR_NO_DEVICE from its first compute call (no CPU fallback); on the GPU it
solves square-mixed-linear (u = x) to tolerance."""
import json
import os
import shutil
import subprocess

import pytest

import paper_2302_11825_b200 as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_example(tmp_path):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    lib = B.library_path()
    exe = str(tmp_path / "integration_example")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "integration_example.cpp"), "-L", os.path.dirname(lib), "-lbvc_b200",
           f"-Wl,-rpath,{os.path.dirname(lib)}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_caller_builds_and_fails_loudly_without_device(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by test_cpp_caller_solves_on_gpu")
    exe = build_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 3, (r.returncode, r.stdout, r.stderr)
    assert "no device" in r.stdout


@pytest.mark.gpu
def test_cpp_caller_solves_on_gpu(tmp_path):
    exe = build_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["max_abs_err_u"] < 0.06 and out["max_solution_reconstruction_err"] < 1e-12, out
