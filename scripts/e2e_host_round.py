"""Wall time of bvc_update_solution_host (C2) against the device time it reports
(generateSeconds + splatSeconds): the difference is readout, host round trips and
call overhead."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402
from bench import build_problem  # noqa: E402

c, scene, region = build_problem(2, B, configs, abi)
src = torch.from_numpy(np.ascontiguousarray(c.points)).pin_memory().numpy()
u = torch.empty(len(src), dtype=torch.float64).pin_memory().numpy()
g = torch.empty((len(src), 2), dtype=torch.float64).pin_memory().numpy()
for k in range(8):
    st = {}
    torch.cuda.synchronize()
    t = time.perf_counter()
    B.update_solution_host(scene, c.problem, region, c.cache, src, c.seed, 50 + k, gradients=True, out=(u, g), stats=st)
    w = time.perf_counter() - t
    if k >= 3:
        dev = st["generateSeconds"] + st["splatSeconds"]
        print(f"wall {w * 1e3:.3f} ms, device (e0..e2) {dev * 1e3:.3f} ms, outside {1e3 * (w - dev):.3f} ms", flush=True)
