"""Quick GPU sanity pass used during development (prints, does not assert)."""
import time
import numpy as np
import paper_2302_11825_b200 as B
from oracle import oracle as O

np.set_printoptions(precision=6, linewidth=150)
# Bessel
t = np.array([0.05, 0.5, 1.0, 1.99, 2.01, 3.0, 5.0, 10.0])
L = O.oracle_lib()
for w, f in enumerate([L.or_bessel_k0, L.or_bessel_k1, L.or_bessel_i0, L.or_bessel_i1]):
    g = B.eval_bessel(w, t); r = np.array([f(x) for x in t])
    print("bessel", w, np.max(np.abs(g / r - 1)))
# kernels
rng = np.random.default_rng(0)
for spec in [B.poisson(2), B.screened(3.0, 2), B.poisson(3), B.screened(1.0, 3)]:
    d = spec.dim
    x = rng.uniform(-1, 1, (64, d)); y = rng.uniform(-1, 1, (64, d)); n = rng.normal(size=(64, d)); n /= np.linalg.norm(n, axis=1)[:, None]
    gk = B.eval_kernels(spec, x, y, n); rk = np.zeros_like(gk)
    import ctypes as C
    L.or_eval_kernels(C.byref(spec), x.ravel(), y.ravel(), n.ravel(), len(x), rk.ravel())
    print("kernels", spec.kind, d, np.max(np.abs(gk - rk) / (np.abs(rk) + 1e-3)))
# gather parity C1-like
v, s, l = O.circle_geometry(segments=1024)
scene = B.Scene(v, s, l)
pb = B.problem(B.poisson(2), g=B.field(B.abi.FIELD_HARMONIC_POLY, 2, 1, 0))
region = B.SolveRegion(scene, epsilon=1e-3)
cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=4096, nWalksNeumann=256, nWalksDirichlet=256)
st = {}
t0 = time.time(); cache = B.generate_boundary_cache(scene, pb, region, cfg, 11, 0, stats=st); B.synchronize(); t1 = time.time()
print("C1 cache", st, "wall", t1 - t0)
c = cache.download()
zz = c["z"]; exact_u = zz[:, 0] ** 2 - zz[:, 1] ** 2
print("uHat err mean", np.mean(c["uHat"] - exact_u), "sd", np.std(c["uHat"] - exact_u))
nrm = c["n"]; exact_d = 2 * zz[:, 0] * nrm[:, 0] - 2 * zz[:, 1] * nrm[:, 1]
print("dHat err mean", np.mean(c["dHat"] - exact_d), "sd", np.std(c["dHat"] - exact_d))
g = np.linspace(-1, 1, 256); X, Y = np.meshgrid(g, g); xs = np.stack([X.ravel(), Y.ravel()], 1); xs = xs[np.hypot(xs[:, 0], xs[:, 1]) < 0.95]
print("K", len(xs))
pts = B.EvaluationPoints(xs)
spec = B.splat_config(B.poisson(2), scene.diagonal)
B.splat_solution(cache, None, pts, spec); B.synchronize()
t0 = time.time()
for _ in range(10): B.splat_solution(cache, None, pts, spec)
B.synchronize(); t1 = time.time()
print("gather 10x wall ms", (t1 - t0) * 100, "pairs/s", len(xs) * 4096 * 10 / (t1 - t0))
pts = B.EvaluationPoints(xs); B.splat_solution(cache, None, pts, spec)
gs = pts.download(); ug = pts.solution(gs)
sub = slice(0, 2000)
ref = O.oracle_splat(spec.kernel, spec.coincidenceTol, c, None, xs[sub], value=True)
ur = O.solution(ref)
print("gather rel err", np.max(np.abs(ug[sub] - ur)) / max(np.max(np.abs(ur)), np.sqrt(np.mean(ur ** 2))))
print("u err vs exact", np.sqrt(np.mean((ug - (xs[:, 0] ** 2 - xs[:, 1] ** 2)) ** 2)))
# C2 round
v = []; segs = []; labels = []
n = 512
corners = [(-1, -1), (1, -1), (1, 1), (-1, 1)]
side_labels = [1, 0, 1, 0]
for k in range(4):
    a = np.array(corners[k]); b = np.array(corners[(k + 1) % 4])
    for j in range(n):
        v.append(a + (b - a) * j / n); labels.append(side_labels[k])
V = np.array(v); S = np.array([[i, (i + 1) % len(V)] for i in range(len(V))])
scene2 = B.Scene(V, S, labels)
pb2 = B.problem(B.poisson(2), g=B.field(B.abi.FIELD_LINEAR, 1, 0, 0, 0))
region2 = B.SolveRegion(scene2, epsilon=1e-3)
cfg2 = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=16384, nWalksNeumann=512, nWalksDirichlet=512)
g = np.linspace(-1, 1, 512); X, Y = np.meshgrid(g, g); xs2 = np.stack([X.ravel(), Y.ravel()], 1)
pts2 = B.EvaluationPoints(xs2)
B.mark_evaluation_points(scene2, region2, cfg2, pts2)
for r in range(2):
    t0 = time.time(); st = B.update_solution(scene2, pb2, region2, cfg2, pts2, 5, r, gradients=True); t1 = time.time()
    print("C2 round", r, st, "wall", t1 - t0)
s2 = pts2.download(); u2 = pts2.solution(s2); g2 = pts2.gradient(s2)
print("fallback", s2["fallback"].sum(), "u rmse", np.sqrt(np.mean((u2 - xs2[:, 0]) ** 2)), "grad rmse", np.sqrt(np.mean((g2 - [1, 0]) ** 2, axis=0)))
print("launches", B.launch_count())
