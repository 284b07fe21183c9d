"""Cache-generation (walk) wall time of a BASELINE config at full size, for A/B runs of
walk-kernel variants selected by environment knobs:
    BVC_SHSTACK=8 python scripts/walk_time.py 5 [reps] [scale]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402

cid = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
c = configs.CONFIGS[cid](scale=scale) if cid in (4, 5) else configs.CONFIGS[cid]()
if c.extra.get("dim") == 3:
    if "components" in c.extra:
        c.segments, c.labels = configs.soup_shell(c)
    sc = B.Scene.mesh3(c.vertices, c.segments, c.labels)
    region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
else:
    sc = B.Scene(c.vertices, c.segments, c.labels)
    if c.region_mode == abi.REGION_SUBDOMAIN:
        sub = B.Scene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
        region = B.SolveRegion(sc, abi.REGION_SUBDOMAIN, c.region_offset, sub, epsilon=c.epsilon)
    else:
        region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
ts = []
chk = 0.0
for r in range(reps + 1):
    B.synchronize()
    t = time.perf_counter()
    st = {}
    cc = B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, r, stats=st)
    B.synchronize()
    ts.append(time.perf_counter() - t)
    if r == 0:
        d = cc.download()
        chk = float(np.sum(d["uHat"]) + np.sum(d["dHat"]))
    del cc
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("BVC_"))
print(f"C{cid} [{tag}] walks s: first {ts[0]:.3f} min {min(ts[1:]):.4f} all {[round(x, 4) for x in ts[1:]]} steps {st.get('cacheSteps')} "
      f"checksum {chk:.9e}", flush=True)
