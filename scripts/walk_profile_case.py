"""One cache generation of a BASELINE config at reduced sample count (for ncu captures
of the walk kernel): python scripts/walk_profile_case.py CONFIG SCALE"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402

cid, scale = int(sys.argv[1]), float(sys.argv[2])
c = configs.CONFIGS[cid](scale=scale)
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
for r in range(2):
    st = {}
    B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, r, stats=st)
    print(st, flush=True)
