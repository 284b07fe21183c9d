"""ctypes wrappers for the test oracles (TEST INFRASTRUCTURE ONLY).

* `Oracle*`  -> oracle/_build/liboracle.so : the C restatement (bvc_oracle.c)
* `Ref*`     -> oracle/_ref/libbvc_ref.so  : the reference's own core (ref_driver.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2302_11825_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbvc_ref.so")
REF_SRC = "/root/reference/proj/core"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build(quiet: bool = True) -> None:
    """make the restatement (always) and oracle/_ref (when the reference sources exist)."""
    targets = ["_build/liboracle.so"]
    if os.path.isdir(REF_SRC):
        targets.append("ref")
    out = subprocess.run(["make", "-C", HERE, *targets], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.or_mix64.restype = C.c_uint64
        L.or_mix64.argtypes = [C.c_uint64]
        L.or_mixkey.restype = C.c_uint64
        L.or_mixkey.argtypes = [C.c_uint64, C.c_uint64]
        L.or_rng_uniforms.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _dp]
        L.or_rng_key_uniforms.argtypes = [C.c_uint64, C.c_int, _dp]
        for nm in ("or_bessel_k0", "or_bessel_k1", "or_bessel_i0", "or_bessel_i1"):
            getattr(L, nm).restype = C.c_double
            getattr(L, nm).argtypes = [C.c_double]
        L.or_eval_kernels.argtypes = [C.POINTER(abi.KernelSpec), _dp, _dp, _dp, C.c_size_t, _dp]
        for nm in ("or_ball_greens", "or_ball_sphere_weight"):
            getattr(L, nm).restype = C.c_double
            getattr(L, nm).argtypes = [C.POINTER(abi.KernelSpec), C.c_double, C.c_double]
        L.or_ball_greens_mass.restype = C.c_double
        L.or_ball_greens_mass.argtypes = [C.POINTER(abi.KernelSpec), C.c_double]
        L.or_field_eval.restype = C.c_double
        L.or_field_eval.argtypes = [C.POINTER(abi.Field), _dp, C.c_int, C.c_int]
        L.or_scene_create.restype = C.c_void_p
        L.or_scene_create.argtypes = [_dp, C.c_int, _ip, _ip, C.c_int]
        L.or_scene_free.argtypes = [C.c_void_p]
        L.or_scene_diagonal.restype = C.c_double
        L.or_scene_diagonal.argtypes = [C.c_void_p]
        L.or_scene_closed.argtypes = [C.c_void_p]
        L.or_loop_area.restype = C.c_double
        L.or_loop_area.argtypes = [C.c_void_p]
        L.or_scene_closest_point.argtypes = [C.c_void_p, _dp, C.c_size_t, C.c_int, _dp, _dp, _ip, _dp]
        L.or_scene_silhouette_distance.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp]
        L.or_scene_intersect_ray.argtypes = [C.c_void_p, _dp, _dp, C.c_size_t, C.c_double, C.c_int,
                                             C.c_double, _dp, _ip, _dp, _dp]
        L.or_scene_inside.argtypes = [C.c_void_p, _dp, C.c_size_t, _u8p]
        L.or_boundary_sample.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                         C.c_uint64, C.c_uint64, _dp, _dp, _dp, _ip, _dp]
        L.or_region_sample.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                       C.c_uint64, _dp, _dp]
        L.or_solve.argtypes = [C.c_void_p, C.POINTER(abi.Problem), _dp, C.POINTER(abi.WalkConfig),
                               C.c_int, _dp]
        L.or_gradient.argtypes = [C.c_void_p, C.POINTER(abi.Problem), _dp, C.c_void_p,
                                  C.POINTER(abi.WalkConfig), _dp]
        L.or_generate_boundary_cache.argtypes = [
            C.c_void_p, C.POINTER(abi.Problem), C.c_void_p, _ip, _ip, C.POINTER(abi.CacheConfig),
            C.c_uint64, C.c_uint64, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _ip, _dp,
            np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")]
        L.or_generate_source_cache.argtypes = [C.POINTER(abi.Problem), C.c_void_p,
                                               C.POINTER(abi.CacheConfig), C.c_uint64, C.c_uint64,
                                               _dp, _dp, _dp]
        L.or_splat.argtypes = [C.POINTER(abi.KernelSpec), C.c_double, C.c_int, C.c_int, _dp, _dp, _dp,
                               _dp, _dp, _dp, C.c_int, _dp, _dp, _dp, C.c_size_t, _dp, C.c_void_p,
                               C.c_int, C.c_int, _dp, _dp, _i64p, _i64p, _dp, _dp, _i64p, _i64p, _i64p]
        L.or_clamped_splat.argtypes = [C.POINTER(abi.KernelSpec), C.c_double, C.c_int, C.c_int, _dp, _dp, _dp,
                                       _dp, _dp, _dp, C.c_int, _dp, _dp, _dp, C.c_size_t, _dp, C.c_void_p,
                                       C.c_int, C.c_double, C.c_void_p, _dp, _dp, _i64p, _i64p, _i64p]
        _oracle = L
    return _oracle


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            if not os.path.isdir(REF_SRC):
                raise FileNotFoundError("oracle/_ref is not built and the reference is absent")
            build()
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mixkey.restype = C.c_uint64
        L.ref_mixkey.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_mix64.restype = C.c_uint64
        L.ref_mix64.argtypes = [C.c_uint64]
        L.ref_rng_uniforms.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _dp]
        L.ref_rng_key_uniforms.argtypes = [C.c_uint64, C.c_int, _dp]
        L.ref_bessel.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_double)]
        L.ref_eval_kernels.argtypes = [C.POINTER(abi.KernelSpec), _dp, _dp, _dp, C.c_size_t, _dp]
        L.ref_ball.argtypes = [C.c_int, C.POINTER(abi.KernelSpec), C.c_double, C.c_double,
                               C.POINTER(C.c_double)]
        L.ref_scene_create.restype = C.c_void_p
        L.ref_scene_create.argtypes = [_dp, C.c_int, _ip, _ip, C.c_int]
        L.ref_scene_free.argtypes = [C.c_void_p]
        L.ref_scene_diagonal.restype = C.c_double
        L.ref_scene_diagonal.argtypes = [C.c_void_p]
        L.ref_scene_closed.argtypes = [C.c_void_p]
        L.ref_scene_closest_point.argtypes = [C.c_void_p, _dp, C.c_size_t, C.c_int, _dp, _dp, _ip, _dp]
        L.ref_scene_silhouette_distance.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp]
        L.ref_scene_intersect_ray.argtypes = [C.c_void_p, _dp, _dp, C.c_size_t, C.c_double, C.c_int,
                                              C.c_double, _dp, _ip, _dp, _dp]
        L.ref_scene_inside.argtypes = [C.c_void_p, _dp, C.c_size_t, _u8p]
        L.ref_boundary_sample.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, _dp, _dp,
                                          _dp, _ip, _dp]
        L.ref_region_sample.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, _dp, _dp]
        L.ref_region_build.restype = C.c_void_p
        L.ref_region_build.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_double]
        L.ref_region_free.argtypes = [C.c_void_p]
        L.ref_region_scene.restype = C.c_void_p
        L.ref_region_scene.argtypes = [C.c_void_p]
        L.ref_region_info.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.ref_region_export.argtypes = [C.c_void_p, _dp, _ip, _ip, _ip, _ip]
        L.ref_solve.argtypes = [C.c_void_p, C.POINTER(abi.Problem), _dp, C.POINTER(abi.WalkConfig),
                                C.c_int, _dp]
        L.ref_gradient.argtypes = [C.c_void_p, C.POINTER(abi.Problem), _dp, C.c_void_p,
                                   C.POINTER(abi.WalkConfig), _dp]
        L.ref_generate_boundary_cache.argtypes = [
            C.c_void_p, C.POINTER(abi.Problem), C.c_void_p, C.POINTER(abi.CacheConfig), C.c_uint64,
            C.c_uint64, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _dp, _i64p, C.POINTER(C.c_double)]
        L.ref_generate_source_cache.argtypes = [C.POINTER(abi.Problem), C.c_void_p,
                                                C.POINTER(abi.CacheConfig), C.c_uint64, C.c_uint64,
                                                _dp, _dp, _dp, C.POINTER(C.c_int)]
        L.ref_splat.argtypes = [C.POINTER(abi.KernelSpec), C.c_double, C.c_int, C.c_int, _dp, _dp, _dp,
                                _dp, _dp, C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_size_t, _dp,
                                C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, _dp, _i64p, _i64p, _dp,
                                _dp, _i64p, _i64p, _i64p, C.POINTER(C.c_double)]
        L.ref_clamped_splat.argtypes = [C.POINTER(abi.KernelSpec), C.c_double, C.c_int, C.c_int, _dp, _dp, _dp,
                                        _dp, _dp, C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_size_t, _dp, C.c_int,
                                        C.c_double, C.c_void_p, _dp, _dp, _i64p, _i64p, _i64p]
        L.ref_ball_radius.argtypes = [C.c_void_p, C.c_void_p, _dp, C.c_size_t, _dp]
        L.ref_grid_save_csv.argtypes = [C.c_char_p, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, _dp,
                                        C.c_void_p]
        L.ref_grid_load_rmse.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_double)]
        L.ref_mark_points.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(abi.CacheConfig), _dp,
                                      C.c_size_t, _u8p, _u8p]
        L.ref_update_solution.argtypes = [C.c_void_p, C.POINTER(abi.Problem), C.c_void_p,
                                          C.POINTER(abi.CacheConfig), _dp, C.c_size_t, C.c_uint64,
                                          C.c_uint64, C.c_int, _dp, C.c_void_p, _u8p, _i64p, _dp]
        L.ref_thread_count.argtypes = [C.c_int]
        L.ref_splat3.argtypes = [C.POINTER(abi.KernelSpec), C.c_double, C.c_int, _dp, _dp, _dp, _dp, _dp,
                                 C.c_size_t, _dp, C.c_int, _dp, _i64p, _i64p, C.POINTER(C.c_double)]
        _ref = L
    return _ref


def _check_ref(code: int) -> None:
    if code != 0:
        raise RuntimeError(f"reference error {code}: {ref_lib().ref_last_error().decode()}")


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


# ----------------------------------------------------------------------------------------
# scenes (restated scene makers of problems.cpp:12-51)
# ----------------------------------------------------------------------------------------
def circle_geometry(center=(0.0, 0.0), radius=1.0, segments=256, label=abi.DIRICHLET, ccw=True):
    """makeCircleScene problems.cpp:12-23."""
    k = np.arange(segments)
    a = 2.0 * np.pi * k / segments * (1.0 if ccw else -1.0)
    v = np.stack([center[0] + radius * np.cos(a), center[1] + radius * np.sin(a)], axis=1)
    s = np.stack([k, (k + 1) % segments], axis=1).astype(np.int32)
    return v, s, np.full(segments, label, dtype=np.int32)


def rectangle_geometry(lo, hi, sides):
    """makeRectangleScene problems.cpp:25-31; sides ordered bottom, right, top, left."""
    v = np.array([lo, [hi[0], lo[1]], hi, [lo[0], hi[1]]], dtype=np.float64)
    s = np.array([[k, (k + 1) % 4] for k in range(4)], dtype=np.int32)
    return v, s, np.array(sides, dtype=np.int32)


def annulus_geometry(center, r_in, r_out, segments):
    """makeAnnulusScene problems.cpp:33-51 (outer CCW, inner hole CW)."""
    k = np.arange(segments)
    ao = 2.0 * np.pi * k / segments
    ai = -2.0 * np.pi * k / segments
    vo = np.stack([center[0] + r_out * np.cos(ao), center[1] + r_out * np.sin(ao)], axis=1)
    vi = np.stack([center[0] + r_in * np.cos(ai), center[1] + r_in * np.sin(ai)], axis=1)
    so = np.stack([k, (k + 1) % segments], axis=1)
    si = segments + np.stack([k, (k + 1) % segments], axis=1)
    return (np.concatenate([vo, vi]), np.concatenate([so, si]).astype(np.int32),
            np.zeros(2 * segments, dtype=np.int32))


class _SceneBase:
    def __init__(self, vertices, segments, labels):
        self.v = _f64(vertices).reshape(-1, 2)
        self.s = np.ascontiguousarray(segments, dtype=np.int32).reshape(-1, 2)
        self.labels = np.ascontiguousarray(labels, dtype=np.int32)

    def _pts(self, x):
        return _f64(x).reshape(-1, 2)


class OracleScene(_SceneBase):
    """The restated Scene (bvc_oracle.c) with brute-force queries."""

    def __init__(self, vertices, segments, labels):
        super().__init__(vertices, segments, labels)
        L = oracle_lib()
        self.h = L.or_scene_create(self.v.ravel(), len(self.v), self.s.ravel(), self.labels, len(self.s))
        if not self.h:
            raise ValueError("oracle scene build failed (ParseError)")
        self.diagonal = L.or_scene_diagonal(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            oracle_lib().or_scene_free(self.h)
            self.h = None

    def closest_point(self, x, filt=abi.FILTER_ANY):
        x = self._pts(x)
        n = len(x)
        p, d, sg, t = np.zeros((n, 2)), np.zeros(n), np.zeros(n, np.int32), np.zeros(n)
        oracle_lib().or_scene_closest_point(self.h, x.ravel(), n, filt, p.ravel(), d, sg, t)
        return p, d, sg, t

    def silhouette_distance(self, x):
        x = self._pts(x)
        out = np.zeros(len(x))
        oracle_lib().or_scene_silhouette_distance(self.h, x.ravel(), len(x), out)
        return out

    def intersect_ray(self, o, d, t_max=np.inf, filt=abi.FILTER_ANY, t_min=0.0):
        o, d = self._pts(o), self._pts(d)
        n = len(o)
        t, sg, p, s = np.zeros(n), np.zeros(n, np.int32), np.zeros((n, 2)), np.zeros(n)
        oracle_lib().or_scene_intersect_ray(self.h, o.ravel(), d.ravel(), n, t_max, filt, t_min, t, sg,
                                            p.ravel(), s)
        return t, sg, p, s

    def inside(self, x):
        x = self._pts(x)
        out = np.zeros(len(x), np.uint8)
        oracle_lib().or_scene_inside(self.h, x.ravel(), len(x), out)
        return out.astype(bool)

    def area(self):
        return oracle_lib().or_loop_area(self.h)

    def boundary_sample(self, count, stratified, key=None, seed=0, stream=0, filt=abi.FILTER_ANY):
        p, n, pdf = np.zeros((count, 2)), np.zeros((count, 2)), np.zeros(count)
        sg, arc = np.zeros(count, np.int32), np.zeros(count)
        e = oracle_lib().or_boundary_sample(self.h, filt, count, int(stratified), key or 0,
                                            int(key is not None), seed, stream, p.ravel(), n.ravel(),
                                            pdf, sg, arc)
        if e:
            raise ValueError("boundary sampler: no segments match the filter")
        return p, n, pdf, sg, arc

    def region_sample(self, count, stratified, key=None, seed=0, stream=0):
        p, pdf = np.zeros((count, 2)), np.zeros(count)
        e = oracle_lib().or_region_sample(self.h, count, int(stratified), seed, stream,
                                          int(key is not None), key or 0, p.ravel(), pdf)
        if e:
            raise ValueError("region sampler failed")
        return p, pdf

    def solve(self, problem, x, cfg, kind=1):
        out = np.zeros(5)
        e = oracle_lib().or_solve(self.h, C.byref(problem), _f64(x), C.byref(cfg), kind, out)
        if e:
            raise RuntimeError(f"oracle solve error {e}")
        return out  # mean, se, count, truncated, steps

    def gradient(self, problem, x, cfg, normal=None):
        out = np.zeros(7)
        nrm = None if normal is None else _f64(normal)
        e = oracle_lib().or_gradient(self.h, C.byref(problem), _f64(x),
                                     None if nrm is None else nrm.ctypes.data, C.byref(cfg), out)
        if e:
            raise RuntimeError(f"oracle gradient error {e}")
        return out


class RefScene(_SceneBase):
    """The reference's own Scene (oracle/_ref)."""

    def __init__(self, vertices, segments, labels, _handle=None, _owner=None):
        super().__init__(vertices, segments, labels)
        L = ref_lib()
        if _handle is not None:
            self.h, self.owned, self._owner = _handle, False, _owner
        else:
            self.h = L.ref_scene_create(self.v.ravel(), len(self.v), self.s.ravel(), self.labels,
                                        len(self.s))
            self.owned = True
            if not self.h:
                raise ValueError("reference Scene::build: " + L.ref_last_error().decode())
        self.diagonal = L.ref_scene_diagonal(self.h)

    def __del__(self):
        if getattr(self, "owned", False) and getattr(self, "h", None):
            ref_lib().ref_scene_free(self.h)
            self.h = None

    def closest_point(self, x, filt=abi.FILTER_ANY):
        x = self._pts(x)
        n = len(x)
        p, d, sg, t = np.zeros((n, 2)), np.zeros(n), np.zeros(n, np.int32), np.zeros(n)
        _check_ref(ref_lib().ref_scene_closest_point(self.h, x.ravel(), n, filt, p.ravel(), d, sg, t))
        return p, d, sg, t

    def silhouette_distance(self, x):
        x = self._pts(x)
        out = np.zeros(len(x))
        _check_ref(ref_lib().ref_scene_silhouette_distance(self.h, x.ravel(), len(x), out))
        return out

    def intersect_ray(self, o, d, t_max=np.inf, filt=abi.FILTER_ANY, t_min=0.0):
        o, d = self._pts(o), self._pts(d)
        n = len(o)
        t, sg, p, s = np.zeros(n), np.zeros(n, np.int32), np.zeros((n, 2)), np.zeros(n)
        _check_ref(ref_lib().ref_scene_intersect_ray(self.h, o.ravel(), d.ravel(), n, t_max, filt, t_min,
                                                     t, sg, p.ravel(), s))
        return t, sg, p, s

    def inside(self, x):
        x = self._pts(x)
        out = np.zeros(len(x), np.uint8)
        _check_ref(ref_lib().ref_scene_inside(self.h, x.ravel(), len(x), out))
        return out.astype(bool)

    def boundary_sample(self, count, stratified, key, filt=abi.FILTER_ANY):
        p, n, pdf = np.zeros((count, 2)), np.zeros((count, 2)), np.zeros(count)
        sg, arc = np.zeros(count, np.int32), np.zeros(count)
        _check_ref(ref_lib().ref_boundary_sample(self.h, filt, count, int(stratified), key, p.ravel(),
                                                 n.ravel(), pdf, sg, arc))
        return p, n, pdf, sg, arc

    def region_sample(self, count, stratified, key):
        p, pdf = np.zeros((count, 2)), np.zeros(count)
        _check_ref(ref_lib().ref_region_sample(self.h, count, int(stratified), key, p.ravel(), pdf))
        return p, pdf

    def solve(self, problem, x, cfg, kind=1):
        out = np.zeros(4)
        _check_ref(ref_lib().ref_solve(self.h, C.byref(problem), _f64(x), C.byref(cfg), kind, out))
        return out

    def gradient(self, problem, x, cfg, normal=None):
        out = np.zeros(6)
        nrm = None if normal is None else _f64(normal)
        _check_ref(ref_lib().ref_gradient(self.h, C.byref(problem), _f64(x),
                                          None if nrm is None else nrm.ctypes.data, C.byref(cfg), out))
        return out


class RefRegion:
    """buildSolveRegion of the reference (cache.cpp:137-246)."""

    def __init__(self, scene: RefScene, mode=abi.REGION_WHOLE_DOMAIN, offset=0.0, subdomain=None,
                 eps=1e-3):
        L = ref_lib()
        self.scene = scene
        self.h = L.ref_region_build(scene.h, mode, offset, subdomain.h if subdomain else None, eps)
        if not self.h:
            raise ValueError("reference buildSolveRegion: " + L.ref_last_error().decode())
        nv, ns, off, area, whole = C.c_int(), C.c_int(), C.c_double(), C.c_double(), C.c_int()
        L.ref_region_info(self.h, C.byref(nv), C.byref(ns), C.byref(off), C.byref(area), C.byref(whole))
        self.offset, self.area, self.whole_domain = off.value, area.value, bool(whole.value)
        v, s = np.zeros((nv.value, 2)), np.zeros((ns.value, 2), np.int32)
        lab, kinds, src = (np.zeros(ns.value, np.int32) for _ in range(3))
        L.ref_region_export(self.h, v.ravel(), s.ravel(), lab, kinds, src)
        self.vertices, self.segments, self.labels, self.kinds, self.source = v, s, lab, kinds, src
        self.boundary = RefScene(v, s, lab, _handle=L.ref_region_scene(self.h), _owner=self)

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_region_free(self.h)
            self.h = None


def ref_generate_boundary_cache(scene: RefScene, problem, region: RefRegion, cfg, seed, round_):
    L = ref_lib()
    N = max(1, cfg.nBoundary)
    z, n = np.zeros((N, 2)), np.zeros((N, 2))
    pdf, u, d, w, arc = (np.zeros(N) for _ in range(5))
    seg = np.zeros(N, np.int32)
    stats = np.zeros(3, np.int64)
    sec = C.c_double()
    _check_ref(L.ref_generate_boundary_cache(scene.h, C.byref(problem), region.h, C.byref(cfg), seed,
                                             round_, z.ravel(), n.ravel(), pdf, u, d, w, seg, arc, stats,
                                             C.byref(sec)))
    return dict(z=z, n=n, pdf=pdf, uHat=u, dHat=d, weight=w, segment=seg, arc=arc, stats=stats,
                seconds=sec.value)


def ref_generate_source_cache(problem, region: RefRegion, cfg, seed, round_):
    M = max(1, cfg.nSource)
    y, pdf, f = np.zeros((M, 2)), np.zeros(M), np.zeros(M)
    m = C.c_int()
    _check_ref(ref_lib().ref_generate_source_cache(C.byref(problem), region.h, C.byref(cfg), seed, round_,
                                                   y.ravel(), pdf, f, C.byref(m)))
    m = m.value
    return dict(y=y[:m], pdf=pdf[:m], f=f[:m])


def _splat_arrays(K, dim):
    return dict(boundarySum=np.zeros(K), sourceSum=np.zeros(K), nBoundary=np.zeros(K, np.int64),
                mSource=np.zeros(K, np.int64), boundaryGradSum=np.zeros((K, dim)),
                sourceGradSum=np.zeros((K, dim)), nBoundaryGrad=np.zeros(K, np.int64),
                mSourceGrad=np.zeros(K, np.int64), skipped=np.zeros(K, np.int64))


def _cache_args(bcache, scache, dim):
    N = len(bcache["pdf"]) if bcache is not None else 0
    M = len(scache["pdf"]) if scache is not None else 0
    e = np.zeros(1)
    bz = _f64(bcache["z"]).ravel() if N else e
    bn = _f64(bcache["n"]).ravel() if N else e
    bp = _f64(bcache["pdf"]) if N else e
    bu = _f64(bcache["uHat"]) if N else e
    bd = _f64(bcache["dHat"]) if N else e
    bw = _f64(bcache.get("weight", np.zeros(N))) if N else e
    sy = _f64(scache["y"]).ravel() if M else e
    sp = _f64(scache["pdf"]) if M else e
    sf = _f64(scache["f"]) if M else e
    return N, bz, bn, bp, bu, bd, bw, M, sy, sp, sf


def oracle_splat(spec, tol, bcache, scache, x, fallback=None, value=True, gradient=False,
                 voronoi=False, state=None):
    """splatSolution / splatGradient restated (cache.cpp:426-497), 2D or 3D."""
    dim = spec.dim
    x = _f64(x).reshape(-1, dim)
    K = len(x)
    st = state if state is not None else _splat_arrays(K, dim)
    N, bz, bn, bp, bu, bd, bw, M, sy, sp, sf = _cache_args(bcache, scache, dim)
    fb = None if fallback is None else np.ascontiguousarray(fallback, dtype=np.uint8)
    e = oracle_lib().or_splat(C.byref(spec), tol, int(voronoi), N, bz, bn, bp, bu, bd, bw, M, sy, sp, sf,
                              K, x.ravel(), None if fb is None else fb.ctypes.data, int(value),
                              int(gradient), st["boundarySum"], st["sourceSum"], st["nBoundary"],
                              st["mSource"], st["boundaryGradSum"].ravel(), st["sourceGradSum"].ravel(),
                              st["nBoundaryGrad"], st["mSourceGrad"], st["skipped"])
    if e:
        raise RuntimeError(f"oracle splat error {e}")
    return st


def ref_splat(spec, tol, bcache, scache, x, fallback=None, value=True, gradient=False, voronoi=False,
              threads=0, state=None):
    """The reference's splatSolution / splatGradient on an identical host cache (2D)."""
    x = _f64(x).reshape(-1, 2)
    K = len(x)
    st = state if state is not None else _splat_arrays(K, 2)
    N, bz, bn, bp, bu, bd, bw, M, sy, sp, sf = _cache_args(bcache, scache, 2)
    fb = None if fallback is None else np.ascontiguousarray(fallback, dtype=np.uint8)
    sec = C.c_double()
    _check_ref(ref_lib().ref_splat(C.byref(spec), tol, int(voronoi), N, bz, bn, bp, bu, bd, bw.ctypes.data,
                                   M, sy, sp, sf, K, x.ravel(), None if fb is None else fb.ctypes.data,
                                   int(value), int(gradient), threads, st["boundarySum"], st["sourceSum"],
                                   st["nBoundary"], st["mSource"], st["boundaryGradSum"].ravel(),
                                   st["sourceGradSum"].ravel(), st["nBoundaryGrad"], st["mSourceGrad"],
                                   st["skipped"], C.byref(sec)))
    st["seconds"] = sec.value
    return st


def ref_splat3(spec, tol, bcache, x, threads=0):
    """cache.cpp:426-461's loop with Vector3 over the reference's own kernel templates
    (kernels.h:78-129), threaded by its parallelFor: the CPU counterpart of the 3D gather."""
    x = _f64(x).reshape(-1, 3)
    K = len(x)
    N = len(bcache["pdf"])
    bsum, nb, sk = np.zeros(K), np.zeros(K, np.int64), np.zeros(K, np.int64)
    sec = C.c_double()
    _check_ref(ref_lib().ref_splat3(C.byref(spec), tol, N, _f64(bcache["z"]).ravel(), _f64(bcache["n"]).ravel(),
                                    _f64(bcache["pdf"]), _f64(bcache["uHat"]), _f64(bcache["dHat"]), K, x.ravel(),
                                    threads, bsum, nb, sk, C.byref(sec)))
    return {"boundarySum": bsum, "nBoundary": nb, "skipped": sk, "seconds": sec.value}


def _clamped_args(bcache, scache, x, ball_radius):
    x = _f64(x).reshape(-1, 2)
    K = len(x)
    st = _splat_arrays(K, 2)
    R = None if ball_radius is None else _f64(ball_radius).reshape(K)
    return x, K, st, R


def oracle_clamped_splat(spec, tol, bcache, scache, x, mode, clamp, ball_radius=None, voronoi=False,
                         fallback=None):
    """The clamped / ball-kernel splat loops restated (cache.cpp:410-416, 512-524, 573-582);
    mode bits 1 clamp dG/dn, 2 ball kernel G^B, 4 clamp the source G^B."""
    x, K, st, R = _clamped_args(bcache, scache, x, ball_radius)
    N, bz, bn, bp, bu, bd, bw, M, sy, sp, sf = _cache_args(bcache, scache, 2)
    fb = None if fallback is None else np.ascontiguousarray(fallback, dtype=np.uint8)
    e = oracle_lib().or_clamped_splat(C.byref(spec), C.c_double(tol), int(voronoi), N, bz, bn, bp, bu, bd, bw, M,
                                      sy, sp, sf, C.c_size_t(K), x.ravel(),
                                      None if fb is None else fb.ctypes.data, int(mode), C.c_double(clamp),
                                      None if R is None else R.ctypes.data, st["boundarySum"], st["sourceSum"],
                                      st["nBoundary"], st["mSource"], st["skipped"])
    if e:
        raise RuntimeError(f"oracle clamped splat error {e}")
    return st


def ref_clamped_splat(spec, tol, bcache, scache, x, mode, clamp, ball_radius=None, voronoi=False):
    """The reference's correctedBoundarySplat (ClampOnly) / correctedSourceSplat without
    their sampled terms, or splatSolution, on an identical host cache."""
    x, K, st, R = _clamped_args(bcache, scache, x, ball_radius)
    N, bz, bn, bp, bu, bd, bw, M, sy, sp, sf = _cache_args(bcache, scache, 2)
    _check_ref(ref_lib().ref_clamped_splat(C.byref(spec), C.c_double(tol), int(voronoi), N, bz, bn, bp, bu, bd,
                                           bw.ctypes.data, M, sy, sp, sf, C.c_size_t(K), x.ravel(), int(mode),
                                           C.c_double(clamp), None if R is None else R.ctypes.data,
                                           st["boundarySum"], st["sourceSum"], st["nBoundary"], st["mSource"],
                                           st["skipped"]))
    return st


def ref_ball_radius(scene: "RefScene", region: "RefRegion", x):
    """markEvaluationPoints with sourceBall: ballRadius per point (cache.cpp:268-274)."""
    x = _f64(x).reshape(-1, 2)
    R = np.zeros(len(x))
    _check_ref(ref_lib().ref_ball_radius(scene.h, region.h, x.ravel(), C.c_size_t(len(x)), R))
    return R


def ref_grid_save_csv(path, origin, spacing, values, valid=None):
    """The reference's saveGridCsv (grid.cpp:22-34)."""
    v = _f64(values)
    ny, nx = v.shape
    ok = None if valid is None else np.ascontiguousarray(valid, dtype=np.uint8)
    _check_ref(ref_lib().ref_grid_save_csv(str(path).encode(), origin[0], origin[1], spacing, nx, ny, v.ravel(),
                                           None if ok is None else ok.ctypes.data))


def ref_grid_load_rmse(path_a, path_b):
    """rmse(loadGridCsv(a), loadGridCsv(b)) of the reference (grid.cpp:36-96)."""
    out = C.c_double()
    _check_ref(ref_lib().ref_grid_load_rmse(str(path_a).encode(), str(path_b).encode(), C.byref(out)))
    return out.value


def ref_streamlines(scene, region, cfg, spec, tol, caches, seeds, h, steps):
    """runStreamlines' tracing loop (tools/src/runner.cpp:310-369) restated in Python over
    the reference's own Scene::inside, markEvaluationPoints and splatGradient, on given
    (boundary, source) cache pairs. Returns (polylines, reasons) like api.trace_streamlines."""
    def direction(p):
        if not scene.inside(np.array([p]))[0]:
            return None, "outside"
        if not region.whole_domain and not region.boundary.inside(np.array([p]))[0]:
            return None, "outside"
        fb, _ = ref_mark_points(scene, region, cfg, [p])
        if fb[0]:
            return None, "outside"
        st = None
        for bc, sc in caches:
            st = ref_splat(spec, tol, bc, sc, [p], value=False, gradient=True, threads=1, state=st)
        g = gradient(st)[0]
        n = float(np.linalg.norm(g))
        if n < 1e-12:
            return None, "zero-gradient"
        return g / n, ""

    lines, reasons = [], []
    for x0 in np.asarray(seeds, float):
        x = x0.copy()
        _, reason = direction(x)
        if reason == "outside":
            lines.append(np.zeros((0, 2)))
            reasons.append("outside")
            continue
        pts = [x.copy()]
        stop = reason
        k = 1
        while k <= steps and not stop:
            k1, stop = direction(x)
            if stop:
                break
            k2, probe = direction(x + h * k1)
            nxt = x + 0.5 * h * (k1 + k2) if not probe else x + h * k1
            _, landed = direction(nxt)
            if landed == "outside":
                stop = "outside"
                break
            x = nxt
            pts.append(x.copy())
            k += 1
        lines.append(np.array(pts))
        reasons.append(stop or "ok")
    return lines, reasons


def solution(st):
    """EvaluationPoint::solution() (cache.h:91-96) for non-fallback points."""
    nb, ms = st["nBoundary"], st["mSource"]
    v = np.where(nb > 0, st["boundarySum"] / np.maximum(nb, 1), 0.0)
    return v + np.where(ms > 0, st["sourceSum"] / np.maximum(ms, 1), 0.0)


def gradient(st):
    """EvaluationPoint::gradient() (cache.h:97-105) for non-fallback points."""
    nb, ms = st["nBoundaryGrad"][:, None], st["mSourceGrad"][:, None]
    v = np.where(nb > 0, st["boundaryGradSum"] / np.maximum(nb, 1), 0.0)
    return v + np.where(ms > 0, st["sourceGradSum"] / np.maximum(ms, 1), 0.0)


def ref_update_solution(scene: RefScene, problem, region: RefRegion, cfg, x, seed, round_,
                        gradients=False):
    """One updateSolution round (cache.cpp:622-684) on fresh points; returns u, grad, stats."""
    x = _f64(x).reshape(-1, 2)
    K = len(x)
    u, fb = np.zeros(K), np.zeros(K, np.uint8)
    g = np.zeros((K, 2)) if gradients else None
    stats, sec = np.zeros(3, np.int64), np.zeros(2)
    _check_ref(ref_lib().ref_update_solution(scene.h, C.byref(problem), region.h, C.byref(cfg), x.ravel(), K,
                                             seed, round_, int(gradients), u,
                                             None if g is None else g.ctypes.data, fb, stats, sec))
    return dict(u=u, grad=g, fallback=fb.astype(bool), stats=stats, generateSeconds=sec[0],
                splatSeconds=sec[1])


def ref_mark_points(scene: RefScene, region: RefRegion, cfg, x):
    x = _f64(x).reshape(-1, 2)
    fb, gu = np.zeros(len(x), np.uint8), np.zeros(len(x), np.uint8)
    _check_ref(ref_lib().ref_mark_points(scene.h, region.h, C.byref(cfg), x.ravel(), len(x), fb, gu))
    return fb.astype(bool), gu.astype(bool)
