"""Python mirror of the reference's BVC operator API over the C ABI (include/bvc_b200.h).

Names, argument meaning and error behaviour follow /root/reference/proj/core/include/bvc/
(`Scene::build` scene.h:84, `buildSolveRegion` cache.h:41, `generateBoundaryCache`
cache.h:159, `splatSolution` cache.h:168, `updateSolution` cache.h:195, the
pointwise estimators pointwise.h:62-76). Every call runs the sm_100a kernels of
libbvc_b200.so; there is no CPU fallback — without a GPU the calls raise
`NoDeviceError`.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi

# BVC_LIB: another build of the library (A/B runs of compile-time variants)
_LIB_PATH = os.environ.get("BVC_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build",
                                                      "libbvc_b200.so")
_lib = None

# exported symbols declared in include/bvc_b200.h (kept in sync by tests/test_abi.py)
SYMBOLS = (
    "bvc_last_error bvc_abi_version bvc_set_device bvc_set_stream bvc_synchronize bvc_kernel_launch_count "
    "bvc_scene_create bvc_scene_create_mesh3 bvc_scene_destroy bvc_scene_info bvc_scene_closest_point "
    "bvc_scene_silhouette_distance bvc_scene_intersect_ray bvc_scene_inside bvc_region_build bvc_region_destroy "
    "bvc_region_info bvc_region_export bvc_region_boundary bvc_points_create bvc_points_destroy bvc_points_download "
    "bvc_points_upload bvc_points_solution bvc_points_reset bvc_mark_evaluation_points bvc_generate_boundary_cache "
    "bvc_generate_boundary_cache_shard bvc_generate_source_cache bvc_boundary_cache_create bvc_boundary_cache_size "
    "bvc_boundary_cache_download bvc_boundary_cache_packed bvc_boundary_cache_from_packed bvc_boundary_cache_destroy "
    "bvc_source_cache_create bvc_source_cache_size bvc_source_cache_download bvc_source_cache_destroy "
    "bvc_make_splat_config bvc_splat_solution bvc_splat_gradient bvc_splat_solution_gradient bvc_splat_range "
    "bvc_update_solution bvc_wos_solve bvc_wost_solve bvc_wost_gradient bvc_wost_normal_derivative "
    "bvc_walk_traffic_profile bvc_eval_kernels bvc_eval_bessel bvc_corrected_boundary_splat "
    "bvc_corrected_source_splat bvc_trace_streamlines bvc_grid_save_csv bvc_grid_load_csv bvc_grid_rmse "
    "bvc_grid_save_pgm bvc_streamlines_write_csv bvc_pipe_probe bvc_boundary_cache_assign_voronoi "
    "bvc_fallback_walks bvc_update_solution_host bvc_update_solution_with_evaluator bvc_generate_boundary_cache_shard_fallback "
    "bvc_points_set_index_base bvc_comm_unique_id bvc_comm_init_nccl bvc_comm_init_callback bvc_comm_info "
    "bvc_comm_destroy bvc_shard_layout bvc_update_solution_sharded bvc_update_solution_sharded_host bvc_wost_gradient3 "
    "bvc_last_round_kernel_seconds"
).split()


class BvcError(RuntimeError):
    """Base class; `code` is the bvc_status."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InvalidArgument(BvcError, ValueError):
    pass


class ParseError(BvcError):
    """ParseError (scene.h:14-16)."""


class SolverError(BvcError):
    """SolverError (pointwise.h:13-15)."""


class KernelSingularity(BvcError):
    """KernelSingularity (kernels.h:12-14)."""


class DomainError(BvcError, ValueError):
    pass


class CudaError(BvcError):
    pass


class NoDeviceError(BvcError):
    pass


_ERRORS = {abi.BVC_ERR_INVALID_ARGUMENT: InvalidArgument, abi.BVC_ERR_PARSE: ParseError,
           abi.BVC_ERR_SOLVER: SolverError, abi.BVC_ERR_SINGULARITY: KernelSingularity,
           abi.BVC_ERR_DOMAIN: DomainError, abi.BVC_ERR_CUDA: CudaError, abi.BVC_ERR_NO_DEVICE: NoDeviceError}


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Loads libbvc_b200.so; raises ImportError when the CUDA library was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"libbvc_b200.so is not built ({_LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(_LIB_PATH)
        L.bvc_last_error.restype = C.c_char_p
        L.bvc_kernel_launch_count.restype = C.c_longlong
        L.bvc_region_boundary.restype = C.c_void_p
        L.bvc_region_boundary.argtypes = [C.c_void_p]
        for name in SYMBOLS:
            if name not in ("bvc_last_error", "bvc_kernel_launch_count", "bvc_region_boundary"):
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(code: int) -> None:
    if code != abi.BVC_OK:
        msg = lib().bvc_last_error().decode(errors="replace")
        raise _ERRORS.get(code, BvcError)(code, msg)


def _f64(a, cols=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if cols is None else a.reshape(-1, cols)


def _ptr(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


def launch_count() -> int:
    return int(lib().bvc_kernel_launch_count())


def last_round_kernel_seconds() -> dict:
    """Device time of the main cache-walk launch and the main gather launch of this
    thread's last updateSolution round (bvc_last_round_kernel_seconds; 0 = not launched)."""
    w, g = C.c_double(0.0), C.c_double(0.0)
    _check(lib().bvc_last_round_kernel_seconds(C.byref(w), C.byref(g)))
    return {"walk": w.value, "gather": g.value}


def set_stream(stream_ptr: int | None) -> None:
    _check(lib().bvc_set_stream(C.c_void_p(stream_ptr or 0)))


def synchronize() -> None:
    _check(lib().bvc_synchronize())


# ----------------------------------------------------------------------------
# problems
# ----------------------------------------------------------------------------
def kernel_spec(kind=abi.KERNEL_POISSON, sigma=0.0, dim=2, scale=1.0) -> abi.KernelSpec:
    return abi.KernelSpec(kind, float(sigma), dim, float(scale))


def poisson(dim=2, scale=1.0):
    """KernelSpec::poisson (kernels.h:38-40)."""
    return kernel_spec(abi.KERNEL_POISSON, 0.0, dim, scale)


def screened(sigma, dim=2, scale=1.0):
    """KernelSpec::screened (kernels.h:41-43)."""
    return kernel_spec(abi.KERNEL_SCREENED, sigma, dim, scale)


def field(kind=abi.FIELD_NONE, *params, n=0):
    return abi.make_field(kind, params, n)


def gaussian_sum(sigma, centers, amps):
    """f = sum a_m exp(-|x - c_m|^2 / (2 sigma^2))."""
    centers = np.asarray(centers, dtype=np.float64)
    p = [sigma]
    for c, a in zip(centers, amps):
        cz = c[2] if len(c) > 2 else 0.0
        p += [c[0], c[1], cz, a]
    return abi.make_field(abi.FIELD_GAUSSIAN_SUM, p, len(amps))


def problem(kernel=None, f=None, g=None, h=None) -> abi.Problem:
    """PdeProblem (pointwise.h:19-26); None fields are empty callbacks."""
    pb = abi.Problem()
    pb.kernel = kernel if kernel is not None else poisson(2)
    pb.f = f if f is not None else abi.make_field()
    pb.g = g if g is not None else abi.make_field()
    pb.h = h if h is not None else abi.make_field()
    return pb


def walk_config(**kw) -> abi.WalkConfig:
    c = abi.default_walk_config()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def cache_config(walk=None, **kw) -> abi.CacheConfig:
    c = abi.default_cache_config()
    if walk is not None:
        c.walk = walk
    for k, v in kw.items():
        setattr(c, k, v)
    return c


# ----------------------------------------------------------------------------
# scene / region
# ----------------------------------------------------------------------------
class Scene:
    """Scene::build (scene.h:84): a 2D segment mesh (or a 3D triangle soup via `mesh3`)."""

    def __init__(self, vertices, segments, labels, _handle=None, _owner=None):
        L = lib()
        if _handle is not None:
            self.h, self.owned, self._owner = C.c_void_p(_handle), False, _owner
        else:
            v = _f64(vertices, 2)
            s = np.ascontiguousarray(segments, dtype=np.int32).reshape(-1, 2)
            lb = np.ascontiguousarray(labels, dtype=np.int32)
            self.h = C.c_void_p()
            _check(L.bvc_scene_create(_ptr(v), len(v), _ptr(s, C.c_int), _ptr(lb, C.c_int), len(s), C.byref(self.h)))
            self.owned = True
        self._info()

    @classmethod
    def mesh3(cls, vertices, tris, labels):
        self = cls.__new__(cls)
        v = _f64(vertices, 3)
        t = np.ascontiguousarray(tris, dtype=np.int32).reshape(-1, 3)
        lb = np.ascontiguousarray(labels, dtype=np.int32)
        self.h = C.c_void_p()
        _check(lib().bvc_scene_create_mesh3(_ptr(v), len(v), _ptr(t, C.c_int), _ptr(lb, C.c_int), len(t),
                                            C.byref(self.h)))
        self.owned = True
        self._info()
        return self

    def _info(self):
        dim, diag, dl, nl, closed, nloops = C.c_int(), C.c_double(), C.c_double(), C.c_double(), C.c_int(), C.c_int()
        lo, hi = (C.c_double * 3)(), (C.c_double * 3)()
        _check(lib().bvc_scene_info(self.h, C.byref(dim), C.byref(diag), lo, hi, C.byref(dl), C.byref(nl),
                                    C.byref(closed), C.byref(nloops)))
        self.dim, self.diagonal = dim.value, diag.value
        self.lo, self.hi = np.array(lo[:dim.value]), np.array(hi[:dim.value])
        self.dirichlet_length, self.neumann_length = dl.value, nl.value
        self.closed, self.n_loops = bool(closed.value), nloops.value

    def __del__(self):
        if getattr(self, "owned", False) and getattr(self, "h", None):
            lib().bvc_scene_destroy(self.h)
            self.h = None

    def has_neumann(self):
        return self.neumann_length > 0.0

    def closest_point(self, x, filt=abi.FILTER_ANY):
        """Scene::closestPoint (scene.h:95); returns point, dist, segment (triangle in 3D), t."""
        x = _f64(x, self.dim)
        n = len(x)
        p, d, sg, t = np.zeros((n, self.dim)), np.zeros(n), np.zeros(n, np.int32), np.zeros(n)
        _check(lib().bvc_scene_closest_point(self.h, _ptr(x), C.c_size_t(n), filt, _ptr(p), _ptr(d),
                                             _ptr(sg, C.c_int), _ptr(t)))
        return p, d, sg, t

    def silhouette_distance(self, x):
        x = _f64(x, 2)
        out = np.zeros(len(x))
        _check(lib().bvc_scene_silhouette_distance(self.h, _ptr(x), C.c_size_t(len(x)), _ptr(out)))
        return out

    def intersect_ray(self, o, d, t_max=np.inf, filt=abi.FILTER_ANY, t_min=0.0):
        o, d = _f64(o, 2), _f64(d, 2)
        n = len(o)
        t, sg, p, s = np.zeros(n), np.zeros(n, np.int32), np.zeros((n, 2)), np.zeros(n)
        _check(lib().bvc_scene_intersect_ray(self.h, _ptr(o), _ptr(d), C.c_size_t(n), C.c_double(t_max), filt,
                                             C.c_double(t_min), _ptr(t), _ptr(sg, C.c_int), _ptr(p), _ptr(s)))
        return t, sg, p, s

    def inside(self, x):
        x = _f64(x, self.dim)
        out = np.zeros(len(x), np.uint8)
        _check(lib().bvc_scene_inside(self.h, _ptr(x), C.c_size_t(len(x)), _ptr(out, C.c_uint8)))
        return out.astype(bool)


class SolveRegion:
    """buildSolveRegion (cache.h:41): whole-domain offset region or a user subdomain loop."""

    def __init__(self, scene: Scene, mode=abi.REGION_WHOLE_DOMAIN, offset=0.0, subdomain: Scene | None = None,
                 epsilon=1e-3):
        self.scene = scene
        self._sub = subdomain
        req = abi.RegionRequest(mode, float(offset), subdomain.h.value if subdomain is not None else None)
        self.h = C.c_void_p()
        _check(lib().bvc_region_build(scene.h, C.byref(req), C.c_double(epsilon), C.byref(self.h)))
        nv, ns, off, area, whole = C.c_int(), C.c_int(), C.c_double(), C.c_double(), C.c_int()
        _check(lib().bvc_region_info(self.h, C.byref(nv), C.byref(ns), C.byref(off), C.byref(area), C.byref(whole)))
        self.offset, self.area, self.whole_domain = off.value, area.value, bool(whole.value)
        d = scene.dim  # 3D regions are triangle meshes (area = enclosed volume)
        v, s = np.zeros((nv.value, d)), np.zeros((ns.value, d), np.int32)
        lb, kinds, src = (np.zeros(ns.value, np.int32) for _ in range(3))
        _check(lib().bvc_region_export(self.h, _ptr(v), _ptr(s, C.c_int), _ptr(lb, C.c_int), _ptr(kinds, C.c_int),
                                       _ptr(src, C.c_int)))
        self.vertices, self.segments, self.labels, self.kinds, self.source = v, s, lb, kinds, src
        self.boundary = Scene(None, None, None, _handle=lib().bvc_region_boundary(self.h), _owner=self)

    def __del__(self):
        if getattr(self, "h", None):
            lib().bvc_region_destroy(self.h)
            self.h = None


# ----------------------------------------------------------------------------
# evaluation points and caches
# ----------------------------------------------------------------------------
class EvaluationPoints:
    """Device-resident std::vector<EvaluationPoint> (cache.h:73-110)."""

    def __init__(self, x, dim=2, index_base=0):
        x = _f64(x, dim)
        self.n, self.dim = len(x), dim
        self.h = C.c_void_p()
        _check(lib().bvc_points_create(_ptr(x), C.c_size_t(self.n), dim, C.byref(self.h)))
        if index_base:  # this set is a shard of a larger one: per-point streams use global indices
            _check(lib().bvc_points_set_index_base(self.h, C.c_longlong(index_base)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().bvc_points_destroy(self.h)
            self.h = None

    def download(self) -> dict:
        n, d = self.n, self.dim
        st = dict(x=np.zeros((n, d)), fallback=np.zeros(n, np.uint8), gradientUnreliable=np.zeros(n, np.uint8),
                  boundarySum=np.zeros(n), sourceSum=np.zeros(n), nBoundary=np.zeros(n, np.int64),
                  mSource=np.zeros(n, np.int64), boundaryGradSum=np.zeros((n, d)), sourceGradSum=np.zeros((n, d)),
                  nBoundaryGrad=np.zeros(n, np.int64), mSourceGrad=np.zeros(n, np.int64), walkSum=np.zeros(n),
                  walkCount=np.zeros(n, np.int64), walkTruncated=np.zeros(n, np.int64),
                  gradientWalkSum=np.zeros((n, d)), gradientWalkCount=np.zeros(n, np.int64),
                  skipped=np.zeros(n, np.int64), ballRadius=np.zeros(n))
        ps = abi.PointState()
        ps.count, ps.dim = n, d
        for name, arr in st.items():
            t = {np.float64: C.c_double, np.uint8: C.c_uint8, np.int64: C.c_longlong}[arr.dtype.type]
            setattr(ps, name, _ptr(arr, t))
        _check(lib().bvc_points_download(self.h, C.byref(ps)))
        st["fallback"] = st["fallback"].astype(bool)
        st["gradientUnreliable"] = st["gradientUnreliable"].astype(bool)
        return st

    def set_fallback(self, flags):
        f = np.ascontiguousarray(flags, dtype=np.uint8)
        ps = abi.PointState()
        ps.count, ps.dim = self.n, self.dim
        ps.fallback = _ptr(f, C.c_uint8)
        _check(lib().bvc_points_upload(self.h, C.byref(ps)))

    def set_ball_radius(self, radius):
        """EvaluationPoint::ballRadius (cache.h:77), as markEvaluationPoints would set it."""
        r = np.ascontiguousarray(radius, dtype=np.float64)
        ps = abi.PointState()
        ps.count, ps.dim = self.n, self.dim
        ps.ballRadius = _ptr(r)
        _check(lib().bvc_points_upload(self.h, C.byref(ps)))

    def reset(self):
        _check(lib().bvc_points_reset(self.h))

    def read_solution(self, gradient=True, out=None):
        """u (and grad u) computed on the device (EvaluationPoint::solution/gradient, cache.h:91-105);
        only these arrays cross to the host. `out` = (u, grad) host arrays to fill (e.g. pinned)."""
        if out is not None:
            u, g = out
        else:
            u = np.zeros(self.n)
            g = np.zeros((self.n, self.dim)) if gradient else None
        _check(lib().bvc_points_solution(self.h, _ptr(u), _ptr(g) if g is not None else None))
        return (u, g) if gradient else u

    def solution(self, st=None):
        """EvaluationPoint::solution() (cache.h:91-96)."""
        st = st or self.download()
        nb, ms = st["nBoundary"], st["mSource"]
        v = np.where(nb > 0, st["boundarySum"] / np.maximum(nb, 1), 0.0)
        v = v + np.where(ms > 0, st["sourceSum"] / np.maximum(ms, 1), 0.0)
        wc = st["walkCount"]
        return np.where(st["fallback"], np.where(wc > 0, st["walkSum"] / np.maximum(wc, 1), 0.0), v)

    def gradient(self, st=None):
        """EvaluationPoint::gradient() (cache.h:97-105)."""
        st = st or self.download()
        nb, ms = st["nBoundaryGrad"][:, None], st["mSourceGrad"][:, None]
        v = np.where(nb > 0, st["boundaryGradSum"] / np.maximum(nb, 1), 0.0)
        v = v + np.where(ms > 0, st["sourceGradSum"] / np.maximum(ms, 1), 0.0)
        gc = st["gradientWalkCount"][:, None]
        fb = st["fallback"][:, None]
        return np.where(fb, np.where(gc > 0, st["gradientWalkSum"] / np.maximum(gc, 1), 0.0), v)


class BoundaryCache:
    """BoundaryCache (cache.h:54-59), device-resident."""

    def __init__(self, handle):
        self.h = handle
        n, d = C.c_int(), C.c_int()
        _check(lib().bvc_boundary_cache_size(self.h, C.byref(n), C.byref(d)))
        self.n, self.dim = n.value, d.value

    @classmethod
    def from_arrays(cls, z, n, pdf, uHat, dHat, weight=None, segment=None, arc=None, voronoi=False, length=0.0):
        z = _f64(z)
        dim = z.shape[1]
        N = len(z)
        arr = (abi.BoundarySample * max(N, 1))()
        nn = _f64(n)
        for i in range(N):
            s = arr[i]
            for k in range(dim):
                s.z[k] = z[i, k]
                s.n[k] = nn[i, k]
            s.pdf, s.uHat, s.dHat = float(pdf[i]), float(uHat[i]), float(dHat[i])
            s.weight = float(weight[i]) if weight is not None else 0.0
            s.segment = int(segment[i]) if segment is not None else -1
            s.arc = float(arc[i]) if arc is not None else 0.0
        h = C.c_void_p()
        _check(lib().bvc_boundary_cache_create(arr, N, dim, int(voronoi), C.c_double(length), C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().bvc_boundary_cache_destroy(self.h)
            self.h = None

    def download(self) -> dict:
        arr = (abi.BoundarySample * max(self.n, 1))()
        _check(lib().bvc_boundary_cache_download(self.h, arr))
        raw = np.ctypeslib.as_array(C.cast(arr, C.POINTER(C.c_double)), shape=(max(self.n, 1) * 12,))
        raw = raw.reshape(max(self.n, 1), 12)[: self.n]
        seg = np.array([arr[i].segment for i in range(self.n)], dtype=np.int32)
        d = self.dim
        return dict(z=raw[:, 0:d].copy(), n=raw[:, 3:3 + d].copy(), pdf=raw[:, 6].copy(), uHat=raw[:, 7].copy(),
                    dHat=raw[:, 8].copy(), weight=raw[:, 9].copy(), segment=seg, arc=raw[:, 11].copy())

    def assign_voronoi(self, region: "SolveRegion"):
        """assignVoronoiWeights (cache.cpp:280-297) over this (whole-round) cache."""
        _check(lib().bvc_boundary_cache_assign_voronoi(self.h, region.h))

    def packed(self):
        p, b = C.c_void_p(), C.c_size_t()
        _check(lib().bvc_boundary_cache_packed(self.h, C.byref(p), C.byref(b)))
        return p.value, b.value


class SourceCache:
    """SourceCache (cache.h:67-70), device-resident."""

    def __init__(self, handle):
        self.h = handle
        m, d = C.c_int(), C.c_int()
        _check(lib().bvc_source_cache_size(self.h, C.byref(m), C.byref(d)))
        self.m, self.dim = m.value, d.value

    @classmethod
    def from_arrays(cls, y, pdf, f, area=0.0):
        y = _f64(y)
        M, dim = y.shape
        arr = (abi.SourceSample * max(M, 1))()
        for i in range(M):
            for k in range(dim):
                arr[i].y[k] = y[i, k]
            arr[i].pdf, arr[i].f = float(pdf[i]), float(f[i])
        h = C.c_void_p()
        _check(lib().bvc_source_cache_create(arr, M, dim, C.c_double(area), C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().bvc_source_cache_destroy(self.h)
            self.h = None

    def download(self) -> dict:
        arr = (abi.SourceSample * max(self.m, 1))()
        _check(lib().bvc_source_cache_download(self.h, arr))
        raw = np.ctypeslib.as_array(C.cast(arr, C.POINTER(C.c_double)), shape=(max(self.m, 1) * 5,))
        raw = raw.reshape(max(self.m, 1), 5)[: self.m]
        return dict(y=raw[:, 0:self.dim].copy(), pdf=raw[:, 3].copy(), f=raw[:, 4].copy())


def _stats_dict(st: abi.RoundStats) -> dict:
    return dict(resampled=st.resampled, cacheWalks=st.cacheWalks, cacheTruncated=st.cacheTruncated,
                cacheSteps=st.cacheSteps, generateSeconds=st.generateSeconds, splatSeconds=st.splatSeconds)


def generate_boundary_cache(scene: Scene, pb, region: SolveRegion, cfg, seed, round_, begin=None, end=None,
                            stats: dict | None = None) -> BoundaryCache:
    """generateBoundaryCache (cache.h:159-161); a shard [begin, end) of the N samples if given."""
    st = abi.RoundStats()
    h = C.c_void_p()
    if begin is None:
        _check(lib().bvc_generate_boundary_cache(scene.h, C.byref(pb), region.h, C.byref(cfg), C.c_uint64(seed),
                                                 C.c_uint64(round_), C.byref(st), C.byref(h)))
    else:
        _check(lib().bvc_generate_boundary_cache_shard(scene.h, C.byref(pb), region.h, C.byref(cfg), C.c_uint64(seed),
                                                       C.c_uint64(round_), int(begin), int(end), C.byref(st),
                                                       C.byref(h)))
    if stats is not None:
        stats.update(_stats_dict(st))
    return BoundaryCache(h)


def generate_boundary_cache_with_fallback(scene: Scene, pb, region: SolveRegion, cfg, seed, round_, begin, end,
                                         pts: "EvaluationPoints", gradients=False,
                                         stats: dict | None = None) -> BoundaryCache:
    """A shard [begin, end) of the round's cache plus the fallback-band walks of `pts`
    (updateSolution cache.cpp:665-681), the latter overlapping the shard's walks."""
    st = abi.RoundStats()
    h = C.c_void_p()
    _check(lib().bvc_generate_boundary_cache_shard_fallback(scene.h, C.byref(pb), region.h, C.byref(cfg),
                                                            C.c_uint64(seed), C.c_uint64(round_), int(begin),
                                                            int(end), pts.h, int(gradients), C.byref(st),
                                                            C.byref(h)))
    if stats is not None:
        stats.update(_stats_dict(st))
    return BoundaryCache(h)


def generate_source_cache(pb, region: SolveRegion, cfg, seed, round_) -> SourceCache:
    """generateSourceCache (cache.h:163-164)."""
    h = C.c_void_p()
    _check(lib().bvc_generate_source_cache(C.byref(pb), region.h, C.byref(cfg), C.c_uint64(seed),
                                           C.c_uint64(round_), C.byref(h)))
    return SourceCache(h)


def make_splat_config(scene: Scene, pb, cfg) -> abi.SplatConfig:
    """makeSplatConfig (cache.h:151)."""
    out = abi.SplatConfig()
    _check(lib().bvc_make_splat_config(scene.h, C.byref(pb), C.byref(cfg), C.byref(out)))
    return out


def splat_config(kernel, diagonal, voronoi=False, fp64=False) -> abi.SplatConfig:
    k = abi.KernelSpec(kernel.kind, kernel.sigma, kernel.dim, diagonal)
    return abi.SplatConfig(k, 1e-12 * diagonal, int(voronoi), 0, int(fp64))


def splat_solution(bcache, scache, pts: EvaluationPoints, cfg):
    """splatSolution (cache.h:168-169)."""
    _check(lib().bvc_splat_solution(bcache.h if bcache else None, scache.h if scache else None, pts.h,
                                    C.byref(cfg)))


def splat_gradient(bcache, scache, pts: EvaluationPoints, cfg):
    """splatGradient (cache.h:172-173)."""
    _check(lib().bvc_splat_gradient(bcache.h if bcache else None, scache.h if scache else None, pts.h,
                                    C.byref(cfg)))


def splat_solution_gradient(bcache, scache, pts: EvaluationPoints, cfg):
    _check(lib().bvc_splat_solution_gradient(bcache.h if bcache else None, scache.h if scache else None, pts.h,
                                             C.byref(cfg)))


def splat_range(bcache, scache, pts: EvaluationPoints, cfg, begin, end, value=True, gradient=False):
    _check(lib().bvc_splat_range(bcache.h if bcache else None, scache.h if scache else None, pts.h, C.byref(cfg),
                                 C.c_size_t(begin), C.c_size_t(end), int(value), int(gradient)))


def field_evaluator(f) -> abi.BoundaryEvaluator:
    """A BoundaryEvaluator returning exact data u(z) = f(z) (e.g. the constant 1 of
    test_cache.cpp:785)."""
    ev = abi.BoundaryEvaluator()
    ev.kind = abi.EVALUATOR_FIELD
    ev.field = f
    return ev


def walk_evaluator(scene: Scene, pb, cfg) -> abi.BoundaryEvaluator:
    """makeDefaultEvaluator (cache.cpp:600-620): cfg.correctionWalks WoSt walks per crossing."""
    ev = abi.BoundaryEvaluator()
    ev.kind = abi.EVALUATOR_WALKS
    ev.scene = scene.h
    ev._keep = (pb, cfg)  # the struct holds raw pointers to these
    ev.problem = C.pointer(pb)
    ev.cfg = C.pointer(cfg)
    return ev


def corrected_boundary_splat(bcache, pts: EvaluationPoints, region: SolveRegion, cfg, clamp_bound, mode,
                             evaluator=None, seed=0, stream=0):
    """correctedBoundarySplat (cache.h:178-184; cache.cpp:499-553)."""
    _check(lib().bvc_corrected_boundary_splat(bcache.h if bcache else None, pts.h, region.h, C.byref(cfg),
                                              C.c_double(clamp_bound), int(mode),
                                              C.byref(evaluator) if evaluator is not None else None,
                                              C.c_uint64(seed), C.c_uint64(stream)))


def corrected_source_splat(scache, pts: EvaluationPoints, region: SolveRegion, cfg, clamp_bound, f=None, seed=0,
                           stream=0):
    """correctedSourceSplat (cache.h:186-191; cache.cpp:555-597); f is a field descriptor or None."""
    _check(lib().bvc_corrected_source_splat(scache.h if scache else None, pts.h, region.h, C.byref(cfg),
                                            C.c_double(clamp_bound), C.byref(f) if f is not None else None,
                                            C.c_uint64(seed), C.c_uint64(stream)))


def mark_evaluation_points(scene: Scene, region: SolveRegion, cfg, pts: EvaluationPoints):
    """markEvaluationPoints (cache.h:154-155)."""
    _check(lib().bvc_mark_evaluation_points(scene.h, region.h, C.byref(cfg), pts.h))


def update_solution(scene: Scene, pb, region: SolveRegion, cfg, pts: EvaluationPoints, seed, round_,
                    gradients=False, correction_eval=None) -> dict:
    """updateSolution (cache.h:195-198): one progressive round; returns RoundStats.
    correction_eval: a BoundaryEvaluator (field_evaluator / walk_evaluator) for the
    ClampCorrect correction; None = the reference's default (makeDefaultEvaluator)."""
    st = abi.RoundStats()
    if correction_eval is None:
        _check(lib().bvc_update_solution(scene.h, C.byref(pb), region.h, C.byref(cfg), pts.h, C.c_uint64(seed),
                                         C.c_uint64(round_), int(gradients), C.byref(st)))
    else:
        _check(lib().bvc_update_solution_with_evaluator(scene.h, C.byref(pb), region.h, C.byref(cfg), pts.h,
                                                        C.c_uint64(seed), C.c_uint64(round_), int(gradients),
                                                        C.byref(correction_eval), C.byref(st)))
    return _stats_dict(st)


def update_solution_host(scene: Scene, pb, region: SolveRegion, cfg, x, seed, round_, gradients=False, out=None,
                         stats=None):
    """runSolveInMemory's round on host points (runner.cpp:116-169): upload, classify, one
    updateSolution round, read u (and grad u). Returns u or (u, grad). `out` = host arrays
    to fill (e.g. pinned); the upload and classification overlap the cache walks."""
    x = _f64(x, scene.dim)
    n = len(x)
    if out is not None:
        u, g = out
    else:
        u = np.zeros(n)
        g = np.zeros((n, scene.dim)) if gradients else None
    st = abi.RoundStats()
    _check(lib().bvc_update_solution_host(scene.h, C.byref(pb), region.h, C.byref(cfg), _ptr(x), C.c_size_t(n),
                                          C.c_uint64(seed), C.c_uint64(round_), int(gradients), _ptr(u),
                                          _ptr(g) if g is not None else None, C.byref(st)))
    if stats is not None:
        stats.update(_stats_dict(st))
    return (u, g) if gradients else u


# --- multi-GPU rounds inside the library (bvc_comm, bvc_update_solution_sharded) ---------

ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


def comm_unique_id() -> bytes:
    """ncclGetUniqueId through the library: 128 bytes for the caller's bootstrap to share."""
    buf = (C.c_char * 128)()
    _check(lib().bvc_comm_unique_id(buf))
    return bytes(buf)


def shard_layout(n: int, nranks: int, rank: int) -> tuple[int, int, int]:
    """Rank's [begin, end) of n units and the padded per-rank count the all-gather moves."""
    b, e, cap = C.c_longlong(), C.c_longlong(), C.c_longlong()
    _check(lib().bvc_shard_layout(C.c_longlong(n), nranks, rank, C.byref(b), C.byref(e), C.byref(cap)))
    return b.value, e.value, cap.value


class Communicator:
    """bvc_comm: the ranks of a multi-GPU job, one GPU each (the device current at init)."""

    def __init__(self, handle, keep=None):
        self.h = handle
        self._keep = keep  # a callback must outlive the communicator
        n, r = C.c_int(), C.c_int()
        _check(lib().bvc_comm_info(self.h, C.byref(n), C.byref(r)))
        self.nranks, self.rank = n.value, r.value

    @classmethod
    def nccl(cls, unique_id: bytes, nranks: int, rank: int) -> "Communicator":
        h = C.c_void_p()
        _check(lib().bvc_comm_init_nccl(C.c_char_p(unique_id), nranks, rank, C.byref(h)))
        return cls(h)

    @classmethod
    def from_allgather(cls, nranks: int, rank: int, fn) -> "Communicator":
        """Host-staged exchange: fn(send_ptr, recv_ptr, nbytes) must fill the device buffer
        recv_ptr (nranks * nbytes) with every rank's send buffer before returning."""
        def tramp(send, recv, nbytes, user, stream):
            try:
                fn(send or 0, recv or 0, int(nbytes))
                return 0
            except Exception:  # noqa: BLE001 - reported to the library as a failed exchange
                import traceback

                traceback.print_exc()
                return 1

        cb = ALLGATHER_FN(tramp)
        h = C.c_void_p()
        _check(lib().bvc_comm_init_callback(nranks, rank, cb, None, C.byref(h)))
        return cls(h, keep=cb)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().bvc_comm_destroy(self.h)
                self.h = None
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def update_solution_sharded(comm: Communicator, scene: Scene, pb, region: SolveRegion, cfg, pts: EvaluationPoints,
                            seed, round_, gradients=False) -> dict:
    """updateSolution sharded over `comm` (bvc_update_solution_sharded): this rank's
    samples and band walks, one all-gather of the cache, this rank's points `pts`."""
    st = abi.RoundStats()
    _check(lib().bvc_update_solution_sharded(comm.h, scene.h, C.byref(pb), region.h, C.byref(cfg), pts.h,
                                             C.c_uint64(seed), C.c_uint64(round_), int(gradients), C.byref(st)))
    return _stats_dict(st)


def update_solution_sharded_host(comm: Communicator, scene: Scene, pb, region: SolveRegion, cfg, x, index_base, seed,
                                 round_, gradients=False, out=None, stats=None):
    """The sharded round on host buffers (bvc_update_solution_sharded_host): x = this
    rank's points (global indices index_base ...); returns u or (u, grad)."""
    x = _f64(x, scene.dim)
    n = len(x)
    if out is not None:
        u, g = out
    else:
        u = np.zeros(n)
        g = np.zeros((n, scene.dim)) if gradients else None
    st = abi.RoundStats()
    _check(lib().bvc_update_solution_sharded_host(comm.h, scene.h, C.byref(pb), region.h, C.byref(cfg), _ptr(x),
                                                  C.c_size_t(n), C.c_longlong(index_base), C.c_uint64(seed),
                                                  C.c_uint64(round_), int(gradients), _ptr(u),
                                                  _ptr(g) if g is not None else None, C.byref(st)))
    if stats is not None:
        stats.update(_stats_dict(st))
    return (u, g) if gradients else u


def fallback_walks(scene: Scene, pb, cfg, pts: EvaluationPoints, seed, round_, gradients=False):
    """updateSolution's fallback-band loop (cache.cpp:665-681) on its own (sharded rounds)."""
    _check(lib().bvc_fallback_walks(scene.h, C.byref(pb), C.byref(cfg), pts.h, C.c_uint64(seed), C.c_uint64(round_),
                                    int(gradients)))


def _estimates(fn, scene, pb, x, cfg, streams, normal=None, vector=False):
    x = _f64(x, scene.dim)
    n = len(x)
    out = (abi.VectorEstimate * max(n, 1))() if vector else (abi.ScalarEstimate * max(n, 1))()
    st = None
    if streams is not None:
        st = np.ascontiguousarray(streams, dtype=np.uint64)
    sp = _ptr(st, C.c_uint64) if st is not None else None
    if normal is not None:
        nrm = _f64(normal, scene.dim)
        _check(fn(scene.h, C.byref(pb), _ptr(x), _ptr(nrm), C.c_size_t(n), C.byref(cfg), sp, out))
    else:
        _check(fn(scene.h, C.byref(pb), _ptr(x), C.c_size_t(n), C.byref(cfg), sp, out))
    if vector:
        return dict(mean=np.array([list(out[i].mean) for i in range(n)]), se=np.array([list(out[i].se) for i in range(n)]),
                    count=np.array([out[i].count for i in range(n)]),
                    truncated=np.array([out[i].truncated for i in range(n)]))
    return dict(mean=np.array([out[i].mean for i in range(n)]), se=np.array([out[i].se for i in range(n)]),
                count=np.array([out[i].count for i in range(n)]), truncated=np.array([out[i].truncated for i in range(n)]))


def wos_solve(scene, pb, x, cfg, streams=None):
    """wosSolve (pointwise.h:62-63), batched."""
    return _estimates(lib().bvc_wos_solve, scene, pb, x, cfg, streams)


def wost_solve(scene, pb, x, cfg, streams=None):
    """wostSolve (pointwise.h:66-67), batched."""
    return _estimates(lib().bvc_wost_solve, scene, pb, x, cfg, streams)


def wost_gradient(scene, pb, x, cfg, streams=None):
    """wostGradient (pointwise.h:71-72), batched; 3D meshes through bvc_wost_gradient3."""
    if scene.dim == 3:
        x = _f64(x, 3)
        n = len(x)
        mean, se = np.zeros((n, 3)), np.zeros((n, 3))
        count, trunc = np.zeros(n, np.int64), np.zeros(n, np.int64)
        st = np.ascontiguousarray(streams, dtype=np.uint64) if streams is not None else None
        _check(lib().bvc_wost_gradient3(scene.h, C.byref(pb), _ptr(x), C.c_size_t(n), C.byref(cfg),
                                        _ptr(st, C.c_uint64) if st is not None else None, _ptr(mean), _ptr(se),
                                        _ptr(count, C.c_longlong), _ptr(trunc, C.c_longlong)))
        return dict(mean=mean, se=se, count=count, truncated=trunc)
    return _estimates(lib().bvc_wost_gradient, scene, pb, x, cfg, streams, vector=True)


def wost_normal_derivative(scene, pb, x, normal, cfg, streams=None):
    """wostNormalDerivative (pointwise.h:75-76), batched."""
    return _estimates(lib().bvc_wost_normal_derivative, scene, pb, x, cfg, streams, normal=normal)


def walk_traffic_profile(scene: Scene, pb, region: SolveRegion, cfg, seed, round_) -> dict:
    """Counts BVH node / primitive fetches of one cache generation (diagnostic launch)."""
    out = (C.c_double * 4)()
    _check(lib().bvc_walk_traffic_profile(scene.h, C.byref(pb), region.h, C.byref(cfg), C.c_uint64(seed),
                                          C.c_uint64(round_), out))
    return dict(steps=out[0], node_fetches=out[1], prim_fetches=out[2], walks=out[3])


def eval_kernels(spec, x, y, n):
    """Device FP32 [G, dG/dx, dG/dn_y, d2G/dx dn_y] (kernels.h:78-129) per row."""
    d = spec.dim
    x, y, n = _f64(x, d), _f64(y, d), _f64(n, d)
    out = np.zeros((len(x), 2 + 2 * d))
    _check(lib().bvc_eval_kernels(C.byref(spec), _ptr(x), _ptr(y), _ptr(n), C.c_size_t(len(x)), _ptr(out)))
    return out


def eval_bessel(which, t):
    """Device FP32 K0 (0), K1 (1), I0 (2), I1 (3)."""
    t = _f64(t)
    out = np.zeros(len(t))
    _check(lib().bvc_eval_bessel(int(which), _ptr(t), C.c_size_t(len(t)), _ptr(out)))
    return out


# ----------------------------------------------------------------------------
# streamlines and data formats
# ----------------------------------------------------------------------------

STREAM_REASONS = ("ok", "outside", "zero-gradient")


def trace_streamlines(scene: Scene, pb, region: SolveRegion, cfg, seed, rounds, seeds, step, steps) -> dict:
    """runStreamlines (tools/src/runner.cpp:285-373) on the device: Heun steps along the
    unit gradient of `rounds` retained cache rounds. Returns the polylines (one (m, 2)
    array per seed, empty for a seed outside the region) and the stop reasons."""
    seeds = _f64(seeds, 2)
    n = len(seeds)
    pts = np.zeros((n, steps + 1, 2))
    counts = np.zeros(n, np.int32)
    reasons = np.zeros(n, np.int32)
    _check(lib().bvc_trace_streamlines(scene.h, C.byref(pb), region.h, C.byref(cfg), C.c_uint64(seed), int(rounds),
                                       _ptr(seeds), n, C.c_double(step), int(steps), _ptr(pts),
                                       _ptr(counts, C.c_int), _ptr(reasons, C.c_int)))
    return dict(seeds=seeds, points=pts, counts=counts, reason_codes=reasons, steps=steps,
                polylines=[pts[i, :counts[i]].copy() for i in range(n)],
                reasons=[STREAM_REASONS[r] for r in reasons])


def write_streamlines_csv(path, traced: dict):
    """The streamline CSV of runStreamlines (`seed,step,x,y,reason`, %.17g)."""
    _check(lib().bvc_streamlines_write_csv(str(path).encode(), _ptr(traced["seeds"]), len(traced["seeds"]),
                                           int(traced["steps"]), _ptr(traced["points"]),
                                           _ptr(traced["counts"], C.c_int), _ptr(traced["reason_codes"], C.c_int)))


def save_grid_csv(path, origin, spacing, values, valid=None):
    """saveGridCsv (grid.h:35-37): values shaped (ny, nx), row-major y-rows."""
    v = _f64(values)
    ny, nx = v.shape
    ok = None if valid is None else np.ascontiguousarray(valid, dtype=np.uint8)
    _check(lib().bvc_grid_save_csv(str(path).encode(), C.c_double(origin[0]), C.c_double(origin[1]),
                                   C.c_double(spacing), nx, ny, _ptr(v),
                                   None if ok is None else _ptr(ok, C.c_uint8)))


def load_grid_csv(path):
    """loadGridCsv (grid.cpp:36-80): returns (origin, spacing, values (ny, nx), valid (ny, nx))."""
    ox, oy, h, nx, ny = C.c_double(), C.c_double(), C.c_double(), C.c_int(), C.c_int()
    b = str(path).encode()
    _check(lib().bvc_grid_load_csv(b, C.byref(ox), C.byref(oy), C.byref(h), C.byref(nx), C.byref(ny), None, None,
                                   C.c_size_t(0)))
    v = np.zeros((ny.value, nx.value))
    ok = np.zeros((ny.value, nx.value), np.uint8)
    _check(lib().bvc_grid_load_csv(b, None, None, None, C.byref(nx), C.byref(ny), _ptr(v), _ptr(ok, C.c_uint8),
                                   C.c_size_t(v.size)))
    return (ox.value, oy.value), h.value, v, ok.astype(bool)


def grid_rmse(a, b, valid_a=None, valid_b=None) -> float:
    """rmse over jointly valid nodes (grid.cpp:82-96)."""
    a, b = _f64(a).ravel(), _f64(b).ravel()
    if a.shape != b.shape:
        raise ParseError(abi.BVC_ERR_PARSE, "rmse: grid layouts do not match")
    va = None if valid_a is None else np.ascontiguousarray(valid_a, dtype=np.uint8).ravel()
    vb = None if valid_b is None else np.ascontiguousarray(valid_b, dtype=np.uint8).ravel()
    out = C.c_double()
    _check(lib().bvc_grid_rmse(_ptr(a), None if va is None else _ptr(va, C.c_uint8), _ptr(b),
                               None if vb is None else _ptr(vb, C.c_uint8), C.c_size_t(a.size), C.byref(out)))
    return out.value


def save_grid_pgm(path, values, valid=None, auto_range=True, lo=0.0, hi=1.0):
    """saveGridImage (tools/src/image.cpp:12-51): binary PGM plus a `.txt` legend."""
    v = _f64(values)
    ny, nx = v.shape
    ok = None if valid is None else np.ascontiguousarray(valid, dtype=np.uint8)
    _check(lib().bvc_grid_save_pgm(str(path).encode(), nx, ny, _ptr(v), None if ok is None else _ptr(ok, C.c_uint8),
                                   int(auto_range), C.c_double(lo), C.c_double(hi)))


PROBES = ("ffma", "mufu_lg2", "mufu_rcp", "dfma", "mufu_rsq", "mufu_ex2", "l2_read_bytes", "ffma_reg", "fmul_reg",
          "fadd_reg", "ffma2_fp32_ops")


def pipe_probe() -> dict:
    """Measured FP32/MUFU/FP64 issue rates (instructions/s) and L2 read bandwidth (B/s)."""
    out = {}
    for i, name in enumerate(PROBES):
        v = C.c_double()
        _check(lib().bvc_pipe_probe(i, C.byref(v)))
        out[name] = v.value
    return out
