"""Generates tests/golden/*.npz from the REFERENCE (oracle/_ref, built from
/root/reference/proj/core by oracle/Makefile). Run in this container:

    python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/bvc_oracle.c) and the product's host
logic on machines where /root/reference is absent, and give the GPU tests
reference outputs on identical inputs. Inputs are seeded; nothing here is copied
from the reference's test files — the cases mirror the situations its tests
exercise (test_kernels.cpp, test_geometry.cpp, test_cache.cpp, test_pointwise.cpp).
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2302_11825_b200 import abi  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def star_geometry(seed, n=24, mixed=True):
    """random star polygon with mixed labels (the shape test_geometry.cpp builds)."""
    rng = np.random.default_rng(seed)
    th = np.sort(rng.uniform(0, 2 * np.pi, n))
    r = rng.uniform(0.4, 1.0, n)
    v = np.stack([r * np.cos(th), r * np.sin(th)], 1)
    s = np.stack([np.arange(n), (np.arange(n) + 1) % n], 1).astype(np.int32)
    lab = (rng.uniform(size=n) < 0.5).astype(np.int32) if mixed else np.zeros(n, np.int32)
    if mixed:
        lab[0] = 0
    return v, s, lab


def spec(kind, sigma, dim, scale=1.0):
    return abi.KernelSpec(kind, sigma, dim, scale)


def main():
    R = O.ref_lib()
    # --- RNG (rng.h) --------------------------------------------------------
    rng_cases = [(0, 0), (1, 2), (2302118250, 0x1001), (17, 0xFFFFFFFFFFFF)]
    ru = np.zeros((len(rng_cases), 16))
    for i, (sd, st) in enumerate(rng_cases):
        R.ref_rng_uniforms(sd, st, 16, ru[i])
    mk = np.array([R.ref_mixkey(a, b) for a, b in [(0, 0), (0x1002, 3), (123456789, 42)]], dtype=np.uint64)
    np.savez(os.path.join(OUT, "rng.npz"), cases=np.array(rng_cases, dtype=np.uint64), uniforms=ru, mixkey=mk)

    # --- Bessel functions (kernels.cpp:7-29) ----------------------------------
    t = np.concatenate([np.geomspace(1e-4, 50.0, 60), [0.1, 0.5, 1.0, 2.0, 5.0, 10.0]])
    bes = np.zeros((4, len(t)))
    out = C.c_double()
    for w in range(4):
        for j, x in enumerate(t):
            R.ref_bessel(w, x, C.byref(out))
            bes[w, j] = out.value
    np.savez(os.path.join(OUT, "bessel.npz"), t=t, values=bes)

    # --- free-space kernels (kernels.h:78-129) ---------------------------------
    g = np.random.default_rng(5)
    kern = {}
    for name, sp in [("p2", spec(0, 0.0, 2)), ("s2", spec(1, 3.0, 2)), ("p3", spec(0, 0.0, 3)),
                     ("s3", spec(1, 1.0, 3)), ("s2big", spec(1, 10.0, 2))]:
        d = sp.dim
        x = g.uniform(-1, 1, (200, d))
        r = np.exp(g.uniform(np.log(0.01), np.log(3.0), 200))
        dirs = g.normal(size=(200, d))
        dirs /= np.linalg.norm(dirs, axis=1)[:, None]
        y = x + r[:, None] * dirs
        n = g.normal(size=(200, d))
        n /= np.linalg.norm(n, axis=1)[:, None]
        o = np.zeros((200, 2 + 2 * d))
        assert R.ref_eval_kernels(C.byref(sp), x.ravel(), y.ravel(), n.ravel(), 200, o.ravel()) == 0
        kern[name + "_x"], kern[name + "_y"], kern[name + "_n"], kern[name + "_out"] = x, y, n, o
        kern[name + "_spec"] = np.array([sp.kind, sp.sigma, sp.dim, sp.scale])
    np.savez(os.path.join(OUT, "kernels.npz"), **kern)

    # --- geometry queries (scene.cpp:133-254) -----------------------------------
    geo = {}
    for k in range(3):
        v, s, lab = star_geometry(100 + k)
        sc = O.RefScene(v, s, lab)
        q = g.uniform(-1.1, 1.1, (400, 2))
        d = g.normal(size=(400, 2))
        d /= np.linalg.norm(d, axis=1)[:, None]
        res = {}
        for filt in (abi.FILTER_ANY, abi.FILTER_DIRICHLET, abi.FILTER_NEUMANN):
            p, dist, seg, tt = sc.closest_point(q, filt)
            res[f"cp{filt}_dist"], res[f"cp{filt}_seg"], res[f"cp{filt}_point"] = dist, seg, p
        res["sil"] = sc.silhouette_distance(q)
        for filt in (abi.FILTER_ANY, abi.FILTER_NEUMANN):
            tt, seg, p, sp_ = sc.intersect_ray(q, d, np.inf, filt, 0.0)
            res[f"ray{filt}_t"], res[f"ray{filt}_seg"] = tt, seg
        res["inside"] = sc.inside(q)
        for key, val in res.items():
            geo[f"s{k}_{key}"] = val
        geo[f"s{k}_v"], geo[f"s{k}_s"], geo[f"s{k}_lab"], geo[f"s{k}_q"], geo[f"s{k}_d"] = v, s, lab, q, d
    np.savez(os.path.join(OUT, "geometry.npz"), **geo)

    # --- samplers (sampling.cpp) -----------------------------------------------------
    v, s, lab = O.circle_geometry(segments=64)
    sc = O.RefScene(v, s, lab)
    p, n, pdf, seg, arc = sc.boundary_sample(128, True, 777)
    p2, n2, pdf2, seg2, arc2 = sc.boundary_sample(128, False, 778)
    rp, rpdf = sc.region_sample(200, True, 779)
    rp2, rpdf2 = sc.region_sample(200, False, 780)
    np.savez(os.path.join(OUT, "sampler.npz"), v=v, s=s, lab=lab, strat_p=p, strat_n=n, strat_pdf=pdf,
             strat_seg=seg, strat_arc=arc, plain_p=p2, plain_seg=seg2, region_strat=rp, region_plain=rp2,
             region_pdf=rpdf)

    # --- regions (cache.cpp:137-246) ----------------------------------------------
    reg = {}
    cases = {
        "square_d": (O.rectangle_geometry([0, 0], [1, 1], [0, 0, 0, 0]), 0.1),
        "square_mixed": (O.rectangle_geometry([0, 0], [1, 1], [1, 0, 1, 0]), 0.05),
        "disk": (O.circle_geometry(segments=256), 0.05),
        "annulus": (O.annulus_geometry((0, 0), 1.0, np.e, 256), 0.05),
        "star": (star_geometry(7, 16, True), 0.01),
    }
    for name, ((v, s, lab), off) in cases.items():
        sc = O.RefScene(v, s, lab)
        try:
            r = O.RefRegion(sc, abi.REGION_WHOLE_DOMAIN, off, eps=1e-3)
            reg[name + "_v"], reg[name + "_s"], reg[name + "_lab"] = r.vertices, r.segments, r.labels
            reg[name + "_kinds"], reg[name + "_src"] = r.kinds, r.source
            reg[name + "_area"] = np.array([r.area])
        except ValueError as e:
            reg[name + "_error"] = np.array([str(e)])
        reg[name + "_in_v"], reg[name + "_in_s"], reg[name + "_in_lab"] = v, s, lab
        reg[name + "_offset"] = np.array([off])
    np.savez(os.path.join(OUT, "regions.npz"), **reg)

    # --- walks (pointwise.cpp) -----------------------------------------------------
    walks = {}

    def run(name, v, s, lab, pb, x, kind, nw, seed, normal=None, grad=False):
        sc = O.RefScene(v, s, lab)
        cfg = abi.default_walk_config()
        cfg.nWalks, cfg.seed = nw, seed
        if grad or normal is not None:
            walks[name] = sc.gradient(pb, x, cfg, normal)
        else:
            walks[name] = sc.solve(pb, x, cfg, kind)
        walks[name + "_x"] = np.array(x)

    disk = O.circle_geometry(segments=256)
    sq_mixed = O.rectangle_geometry([0, 0], [1, 1], [1, 0, 1, 0])
    sq_d = O.rectangle_geometry([0, 0], [1, 1], [0, 0, 0, 0])
    lin = abi.Problem()
    lin.kernel = spec(0, 0.0, 2)
    lin.g = abi.make_field(abi.FIELD_LINEAR, [1, 0, 0, 0])
    dpo = abi.Problem()
    dpo.kernel = spec(0, 0.0, 2)
    dpo.f = abi.make_field(abi.FIELD_CONSTANT, [1.0])
    dpo.g = abi.make_field(abi.FIELD_RADIAL, [0, 0, 0.25, 2, -0.25])
    vert = abi.Problem()
    vert.kernel = spec(0, 0.0, 2)
    vert.g = abi.make_field(abi.FIELD_LINEAR, [0, 1, 0, 0])
    vert.h = abi.make_field(abi.FIELD_LINEAR, [0, 2, -1, 0])  # = n.(0,1) on y = 0 and y = 1
    scr = abi.Problem()
    scr.kernel = spec(1, 2.0, 2)
    scr.g = abi.make_field(abi.FIELD_CONSTANT, [1.0])
    scr.f = abi.make_field(abi.FIELD_CONSTANT, [-2.0])
    run("disk_linear", *disk, lin, [0.3, 0.4], 0, 20000, 2)
    run("disk_poisson", *disk, dpo, [0.0, 0.0], 0, 20000, 3)
    run("mixed", *sq_mixed, lin, [0.25, 0.5], 1, 20000, 6)
    run("vertical", *sq_mixed, vert, [0.3, 0.7], 1, 20000, 7)
    run("screened", *sq_d, scr, [0.2, 0.4], 0, 20000, 4)
    run("grad_disk_poisson", *disk, dpo, [0.5, 0.0], 1, 20000, 12, grad=True)
    run("dn_disk_poisson", *disk, dpo, [0.95, 0.0], 1, 20000, 13, normal=[1.0, 0.0])
    run("grad_screened", *sq_d, scr, [0.3, 0.6], 1, 20000, 14, grad=True)
    np.savez(os.path.join(OUT, "walks.npz"), **walks)

    # --- splats on identical exact-data caches (cache.cpp:426-497) -------------------
    spl = {}
    g2 = np.random.default_rng(11)
    for name, (geom, kspec, ufun, dfun, ffun) in {
        "square_ux": (sq_d, spec(0, 0.0, 2), lambda z: z[:, 0], lambda z, n: n[:, 0], None),
        "disk_poisson": (disk, spec(0, 0.0, 2), lambda z: 0.25 * (np.sum(z * z, 1) - 1),
                         lambda z, n: 0.5 * np.sum(z * n, 1), lambda y: np.ones(len(y))),
        "screened_disk": (disk, spec(1, 2.0, 2), lambda z: np.ones(len(z)), lambda z, n: np.zeros(len(z)),
                          lambda y: -2.0 * np.ones(len(y))),
    }.items():
        v, s, lab = geom
        sc = O.RefScene(v, s, lab)
        z, n, pdf, seg, arc = sc.boundary_sample(512, False, int(g2.integers(1 << 30)))
        cache = dict(z=z, n=n, pdf=pdf, uHat=ufun(z), dHat=dfun(z, n), weight=np.zeros(len(z)))
        scache = None
        if ffun is not None:
            yy, ypdf = sc.region_sample(256, False, int(g2.integers(1 << 30)))
            scache = dict(y=yy, pdf=ypdf, f=ffun(yy))
        lo, hi = v.min(0) + 0.1, v.max(0) - 0.1
        xs = g2.uniform(lo, hi, (64, 2))
        xs = xs[sc.inside(xs)]
        kspec.scale = sc.diagonal
        st = O.ref_splat(kspec, 1e-12 * sc.diagonal, cache, scache, xs, value=True, gradient=True, threads=1)
        for key, val in cache.items():
            spl[f"{name}_b_{key}"] = val
        if scache is not None:
            for key, val in scache.items():
                spl[f"{name}_s_{key}"] = val
        spl[f"{name}_x"] = xs
        spl[f"{name}_spec"] = np.array([kspec.kind, kspec.sigma, kspec.dim, kspec.scale])
        for key in ("boundarySum", "sourceSum", "nBoundary", "mSource", "boundaryGradSum", "sourceGradSum",
                    "skipped"):
            spl[f"{name}_{key}"] = st[key]
    np.savez(os.path.join(OUT, "splat.npz"), **spl)

    # --- boundary cache generation (cache.cpp:301-390) ------------------------------
    v, s, lab = sq_mixed
    sc = O.RefScene(v, s, lab)
    rg = O.RefRegion(sc, abi.REGION_WHOLE_DOMAIN, 0.05, eps=1e-3)
    cfg = abi.default_cache_config()
    cfg.nBoundary, cfg.nWalksNeumann, cfg.nWalksDirichlet, cfg.threads = 48, 8, 16, 1
    cfg.offset = 0.05
    cfg.walk.epsilon = 1e-3
    c = O.ref_generate_boundary_cache(sc, lin, rg, cfg, 11, 0)
    np.savez(os.path.join(OUT, "cache.npz"), **{k: np.asarray(v_) for k, v_ in c.items() if k != "seconds"})
    # --- clamped / ball-kernel splats (cache.cpp:410-416, 499-597) ------------------
    # the deterministic loops of correctedBoundarySplat (ClampOnly) and
    # correctedSourceSplat (no f: no sampled term), and markEvaluationPoints' ball radius
    cl = {}
    g3 = np.random.default_rng(23)
    v, s, lab = O.circle_geometry(segments=256)
    sc = O.RefScene(v, s, lab)
    loop = O.RefScene(v, s, lab)
    rg = O.RefRegion(sc, abi.REGION_SUBDOMAIN, 0.0, subdomain=loop, eps=1e-3)
    z, n, pdf, seg, arc = sc.boundary_sample(512, False, int(g3.integers(1 << 30)))
    cache = dict(z=z, n=n, pdf=pdf, uHat=z[:, 0] + 0.5, dHat=n[:, 0] - 0.25, weight=np.zeros(len(z)))
    yy, ypdf = sc.region_sample(256, False, int(g3.integers(1 << 30)))
    scache = dict(y=yy, pdf=ypdf, f=1.0 + yy[:, 0] ** 2)
    rr = np.concatenate([[0.0, 0.3, 0.9, 0.95, 0.99], g3.uniform(0, 0.995, 27)])
    ph = g3.uniform(0, 2 * np.pi, len(rr))
    xs = np.stack([rr * np.cos(ph), rr * np.sin(ph)], 1)
    R = O.ref_ball_radius(sc, rg, xs)
    k2 = spec(0, 0.0, 2, sc.diagonal)
    for key, val in cache.items():
        cl[f"b_{key}"] = val
    for key, val in scache.items():
        cl[f"s_{key}"] = val
    cl["x"], cl["ballRadius"], cl["region_v"] = xs, R, rg.vertices
    cases = [(1, 1.0), (1, 0.05), (2, 0.0), (3, 1.0), (6, 0.2), (7, 0.2)]
    cl["cases"] = np.array(cases)
    for i, (mode, c) in enumerate(cases):
        st = O.ref_clamped_splat(k2, 1e-12 * sc.diagonal, cache, scache, xs, mode, c, R)
        for key in ("boundarySum", "sourceSum", "nBoundary", "mSource", "skipped"):
            cl[f"{i}_{key}"] = st[key]
    np.savez(os.path.join(OUT, "clamp.npz"), **cl)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
