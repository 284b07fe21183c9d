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


CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build_example(tmp_path, name="integration_example", cudart=False):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    lib = B.library_path()
    exe = str(tmp_path / name)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-pthread", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L", os.path.dirname(lib), "-lbvc_b200",
           f"-Wl,-rpath,{os.path.dirname(lib)}", "-o", exe]
    if cudart:  # the example's own host-staged all-gather copies device buffers
        if not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime.h")):
            pytest.skip("CUDA headers not available")
        cmd += ["-I", os.path.join(CUDA, "include"), "-L", os.path.join(CUDA, "lib64"), "-lcudart",
                f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"]
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


def test_cpp_sharded_threads_builds_and_fails_loudly_without_device(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by test_cpp_sharded_threads_on_gpu")
    exe = build_example(tmp_path, "sharded_threads", cudart=True)
    r = subprocess.run([exe, "2"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 3, (r.returncode, r.stdout, r.stderr)


@pytest.mark.gpu
@pytest.mark.parametrize("ranks", [2, 3])
def test_cpp_sharded_threads_on_gpu(tmp_path, ranks):
    """tests/cpp/sharded_threads.cpp: one host thread per rank (per-thread library state),
    a host-staged all-gather written in C++ (bvc_comm_init_callback), every rank's points
    bitwise equal to the single-rank round."""
    exe = build_example(tmp_path, "sharded_threads", cudart=True)
    r = subprocess.run([exe, str(ranks)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["bitwise_equal"] and out["ranks"] == ranks, out
