"""(Build the spinning kernel first: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
-o paper_2302_11825_b200/_build/libspin.so scripts/cuda/spin.cu)
Does a kernel with shared memory start while the library's walks (1-3 blocks per SM) are
resident? Thread W runs a cache generation; the main thread launches a 0.2 s spinning
kernel with 16 KB of shared memory per CTA on another stream and times it."""
import ctypes as C
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402

spin = C.CDLL(os.path.join(os.path.dirname(B.library_path()), "libspin.so"))
for f in (spin.spin_launch, spin.spin_launch_smem):
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_longlong, C.c_int]
configs.CONFIGS[5] = lambda: configs.config5(n_points=1_048_576)
c, scene, region = bench.build_problem(5, B, configs, abi)
cfg = c.cache
N = int(cfg.nBoundary)
s_w, s_g = torch.cuda.Stream(), torch.cuda.Stream()


def walks():
    B.set_stream(s_w.cuda_stream)
    t = time.perf_counter()
    cc = B.generate_boundary_cache(scene, c.problem, region, cfg, c.seed, 1, begin=0, end=N // 4)
    B.synchronize()
    res["w"] = time.perf_counter() - t
    del cc


res = {}
walks()
for wocc in (1,):
    for wcarve in (None,):
        for smem in (0, 1):
            os.environ["BVC_WALK_OCC"] = str(wocc)
            if wcarve is None:
                os.environ.pop("BVC_WALK_CARVEOUT", None)
            else:
                os.environ["BVC_WALK_CARVEOUT"] = str(wcarve)
            torch.cuda.synchronize()
            th = threading.Thread(target=walks)
            th.start()
            time.sleep(0.5)
            t = time.perf_counter()
            fn = spin.spin_launch_smem if smem else spin.spin_launch
            fn(C.c_void_p(s_g.cuda_stream), 592, 128, int(0.2 * 1.965e9), -1)
            t_launch = time.perf_counter() - t
            s_g.synchronize()
            dt = time.perf_counter() - t
            th.join()
            print(f"walk occ {wocc} carve {wcarve}: walks {res['w']:.3f} s; 0.2 s spin kernel (smem {16 * smem} KB) done after {dt:.3f} s (launch call {t_launch * 1e3:.2f} ms)",
                  flush=True)
