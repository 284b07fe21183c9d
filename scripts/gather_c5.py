"""C5-shaped gather timing (screened 3D values, sigma = 1): a 1M-sample cache on a unit
sphere shell, K uniform points inside, CUDA events over repeated splats.
    [BVC_LIB=...] python scripts/gather_c5.py [K] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N = 1 << 20
rng = np.random.default_rng(0)
z = rng.normal(size=(N, 3))
z /= np.linalg.norm(z, axis=1)[:, None]
order = np.lexsort((z[:, 0], np.floor(z[:, 1] * 64), np.floor(z[:, 2] * 64)))  # spatially coherent like leaf order
z = z[order]
x = rng.uniform(-0.55, 0.55, (K, 3))
bc = B.BoundaryCache.from_arrays(z, z, np.full(N, 1 / (4 * np.pi)), rng.uniform(-1, 1, N), rng.uniform(-1, 1, N))
pts = B.EvaluationPoints(x, 3)
spec = abi.SplatConfig(abi.KernelSpec(abi.KERNEL_SCREENED, 1.0, 3, 2.0), 2e-12, 0, 0)
B.splat_range(bc, None, pts, spec, 0, K, True, False)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    B.splat_range(bc, None, pts, spec, 0, K, True, False)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
st = pts.download()
t = min(ts)
bound = 148 * 1965e6 * 8  # 16 FP32 ops and 2 MUFU per pair: 8 pairs/clk/SM
print(f"[{os.environ.get('BVC_LIB', 'default')}] K={K} N={N} t={t*1e3:.1f} ms pairs/s={K*N/t:.4e} "
      f"frac_of_8pairs_per_clk={K*N/t/bound:.3f} checksum={np.sum(st['boundarySum']):.12e}", flush=True)
