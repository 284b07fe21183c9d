import numpy as np
import paper_2302_11825_b200 as B
from paper_2302_11825_b200 import abi, configs
from tests.test_gpu_3d import HARMONIC, g_exact, grad_exact
V, F = configs.icosphere(4)
sc = B.Scene.mesh3(V, F, np.zeros(len(F), np.int32))
pb = B.problem(B.poisson(3), g=HARMONIC)
region = B.SolveRegion(sc, offset=0.02, epsilon=1e-3)
cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=8192, nWalksNeumann=64, nWalksDirichlet=256, offset=0.02)
c = B.generate_boundary_cache(sc, pb, region, cfg, 3, 0).download()
z, n = c["z"], c["n"]
du = c["uHat"] - g_exact(z); dd = c["dHat"] - np.sum(n * grad_exact(z), 1)
print("uHat bias %.5f +- %.5f   dHat bias %.4f +- %.4f" % (du.mean(), du.std() / np.sqrt(len(du)), dd.mean(), dd.std() / np.sqrt(len(dd))))
print("pdf*area", c["pdf"][0] * region.vertices.shape[0], "pdf", c["pdf"][0], "normals |n|", np.linalg.norm(n, axis=1).min())
# region area
Vr, Fr = region.vertices, region.segments
area = 0.5 * np.linalg.norm(np.cross(Vr[Fr[:, 1]] - Vr[Fr[:, 0]], Vr[Fr[:, 2]] - Vr[Fr[:, 0]]), axis=1).sum()
print("region area", area, "1/pdf", 1 / c["pdf"][0])
rng = np.random.default_rng(0)
x = rng.normal(size=(500, 3)); x *= (0.8 * rng.uniform(0, 1, 500) ** (1 / 3) / np.linalg.norm(x, axis=1))[:, None]
exact = B.BoundaryCache.from_arrays(z, n, c["pdf"], g_exact(z), np.sum(n * grad_exact(z), 1))
one = B.BoundaryCache.from_arrays(z, n, c["pdf"], np.ones(len(z)), np.zeros(len(z)))
spec = abi.SplatConfig(abi.KernelSpec(0, 0.0, 3, sc.diagonal), 1e-12 * sc.diagonal, 0, 0)
for name, cc in [("exact", exact), ("one", one), ("estimated", B.BoundaryCache.from_arrays(z, n, c["pdf"], c["uHat"], c["dHat"]))]:
    p = B.EvaluationPoints(x, 3); B.splat_solution(cc, None, p, spec); u = p.solution()
    ref = np.ones(len(x)) if name == "one" else g_exact(x)
    print(name, "mean err %.5f rms %.5f" % ((u - ref).mean(), np.sqrt(np.mean((u - ref) ** 2))))
