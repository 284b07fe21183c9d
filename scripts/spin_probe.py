"""(Build the spinning kernel first: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
-o paper_2302_11825_b200/_build/libspin.so scripts/cuda/spin.cu)
Which of the library's kernels can share an SM with a resident 1-CTA-per-SM kernel of a
given shared-memory carve-out? A spinning kernel (scripts/cuda/spin.cu) holds one CTA on
every SM for ~T s on one stream; the gather / the walks run on another and report how long
they took. Usage: python scripts/spin_probe.py"""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402

spin = C.CDLL(os.path.join(os.path.dirname(B.library_path()), "libspin.so"))
spin.spin_launch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_longlong, C.c_int]
configs.CONFIGS[5] = lambda: configs.config5(n_points=2_097_152)
c, scene, region = bench.build_problem(5, B, configs, abi)
cfg = c.cache
N = int(cfg.nBoundary)
pts = B.EvaluationPoints(c.points, c.dim)
B.mark_evaluation_points(scene, region, cfg, pts)
spec = B.make_splat_config(scene, c.problem, cfg)
cache0 = B.generate_boundary_cache(scene, c.problem, region, cfg, c.seed, 0)
s_spin = torch.cuda.Stream()
s_lib = torch.cuda.Stream()
B.set_stream(s_lib.cuda_stream)


def gather():
    t = time.perf_counter()
    B.splat_range(cache0, None, pts, spec, 0, 1 << 62, True, False)
    B.synchronize()
    return time.perf_counter() - t


def walks():
    t = time.perf_counter()
    cc = B.generate_boundary_cache(scene, c.problem, region, cfg, c.seed, 1, begin=0, end=N // 8)
    B.synchronize()
    dt = time.perf_counter() - t
    del cc
    return dt


gather(); walks()
print("alone: gather", round(gather(), 3), "walks", round(walks(), 3), flush=True)
SPIN_S = 3.0
for carve in (-1, 44):
    for name, fn, env in (("gather", gather, "BVC_GATHER_CARVEOUT"), ("walks", walks, "BVC_WALK_CARVEOUT")):
        for lib_carve in (None, 44):
            if lib_carve is None:
                os.environ.pop(env, None)
            else:
                os.environ[env] = str(lib_carve)
            torch.cuda.synchronize()
            spin.spin_launch(C.c_void_p(s_spin.cuda_stream), 148, 256, int(SPIN_S * 1.965e9), carve)
            time.sleep(0.05)
            dt = fn()
            torch.cuda.synchronize()
            print(f"spin carve {carve} ({SPIN_S} s resident): {name} with {env}={lib_carve}: {dt:.3f} s", flush=True)
            os.environ.pop(env, None)
