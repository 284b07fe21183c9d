"""Child process of tests/test_gpu_walk_accel.py: small versions of the BASELINE
configs; dumps the walk outputs (cache u-hat / d-hat) of one round. Run with one
walk-query acceleration switched off (BVC_HINTGRID / BVC_ENTRY = 0) and
with the defaults."""
import sys

import numpy as np

import paper_2302_11825_b200 as B
from paper_2302_11825_b200 import abi, configs

SCALES = {2: 1 / 64, 3: 1 / 256, 4: 1 / 256, 5: 1 / 1024}


def scene_region(cid):
    c = configs.CONFIGS[cid](scale=SCALES[cid])
    if c.extra.get("dim") == 3:
        if "components" in c.extra:
            c.segments, c.labels = configs.soup_shell(c)
        sc = B.Scene.mesh3(c.vertices, c.segments, c.labels)
        return c, sc, B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
    sc = B.Scene(c.vertices, c.segments, c.labels)
    if c.region_mode == abi.REGION_SUBDOMAIN:
        sub = B.Scene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
        return c, sc, B.SolveRegion(sc, abi.REGION_SUBDOMAIN, c.region_offset, sub, epsilon=c.epsilon)
    return c, sc, B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)


if __name__ == "__main__":
    res = {}
    for cid in SCALES:
        c, sc, region = scene_region(cid)
        st = {}
        cache = B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, 0, stats=st).download()
        res[f"c{cid}_u"], res[f"c{cid}_d"] = cache["uHat"], cache["dHat"]
        res[f"c{cid}_steps"] = np.array([st["cacheSteps"]])
    np.savez(sys.argv[1], **res)
