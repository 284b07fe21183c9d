"""Scene BVH build time per builder (BVC_BVH = host | sah | lbvh), per config."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import configs  # noqa: E402

for cid in (2, 3, 4, 5):
    c = getattr(configs, f"config{cid}")()
    for mode in ("host", "sah", "lbvh"):
        os.environ["BVC_BVH"] = mode
        dim = c.extra.get("dim", 2) if c.extra else 2
        if dim == 2:
            sc = B.Scene(c.vertices, c.segments, c.labels)
        else:
            sc = B.Scene.mesh3(c.vertices, c.segments, c.labels)
        B.synchronize()
        t0 = time.perf_counter()
        x = np.zeros((1, dim))
        sc.closest_point(x)  # first device query triggers the upload + BVH build
        B.synchronize()
        print(f"C{cid} {mode}: scene upload incl. BVH build {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
