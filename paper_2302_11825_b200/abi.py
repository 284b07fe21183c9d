"""ctypes mirror of the structs in include/bvc_b200.h (layouts only, no library load).

The names follow the reference's C++ API (`/root/reference/proj/core/include/bvc/*.h`):
`bvc_walk_config` is `WalkConfig` (pointwise.h:28-45), `bvc_cache_config` is
`CacheConfig` (cache.h:114-132), `bvc_problem` is `PdeProblem` (pointwise.h:19-26)
with the std::function fields replaced by device-evaluable `bvc_field` descriptors.
"""
from __future__ import annotations

import ctypes as C

# status codes (exception classes of the reference)
BVC_OK = 0
BVC_ERR_INVALID_ARGUMENT = 1
BVC_ERR_PARSE = 2
BVC_ERR_SOLVER = 3
BVC_ERR_SINGULARITY = 4
BVC_ERR_DOMAIN = 5
BVC_ERR_CUDA = 6
BVC_ERR_NO_DEVICE = 7

DIRICHLET, NEUMANN = 0, 1
FILTER_ANY, FILTER_DIRICHLET, FILTER_NEUMANN = 0, 1, 2
KERNEL_POISSON, KERNEL_SCREENED = 0, 1
REGION_WHOLE_DOMAIN, REGION_SUBDOMAIN = 0, 1
SEG_KNOWN_NEUMANN, SEG_ESTIMATED_OFFSET, SEG_USER_LOOP = 0, 1, 2
CLAMP_OFF, CLAMP_ONLY, CLAMP_CORRECT = 0, 1, 2

FIELD_NONE = 0
FIELD_CONSTANT = 1
FIELD_LINEAR = 2
FIELD_RADIAL = 3
FIELD_HARMONIC_POLY = 4
FIELD_CHECKERBOARD = 5
FIELD_SIN_COS = 6
FIELD_GAUSSIAN_SUM = 7
FIELD_QUADRATIC3 = 8
FIELD_TRIG3 = 9
FIELD_MAX_PARAMS = 68


class KernelSpec(C.Structure):
    _fields_ = [("kind", C.c_int), ("sigma", C.c_double), ("dim", C.c_int), ("scale", C.c_double)]


class Field(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_int), ("p", C.c_double * FIELD_MAX_PARAMS)]


class Problem(C.Structure):
    _fields_ = [("kernel", KernelSpec), ("f", Field), ("g", Field), ("h", Field)]


class WalkConfig(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("rMin", C.c_double), ("maxSteps", C.c_int),
                ("nWalks", C.c_int), ("seed", C.c_uint64), ("stream", C.c_uint64)]


class CacheConfig(C.Structure):
    _fields_ = [("nBoundary", C.c_int), ("nSource", C.c_int), ("nWalksNeumann", C.c_int),
                ("nWalksDirichlet", C.c_int), ("offset", C.c_double), ("clamp", C.c_double),
                ("clampMode", C.c_int), ("sourceBall", C.c_int), ("correctionWalks", C.c_int),
                ("voronoi", C.c_int), ("stratified", C.c_int), ("walk", WalkConfig),
                ("threads", C.c_int)]


class RegionRequest(C.Structure):
    _fields_ = [("mode", C.c_int), ("offset", C.c_double), ("subdomain", C.c_void_p)]


class RoundStats(C.Structure):
    _fields_ = [("resampled", C.c_longlong), ("cacheWalks", C.c_longlong),
                ("cacheTruncated", C.c_longlong), ("cacheSteps", C.c_longlong),
                ("generateSeconds", C.c_double), ("splatSeconds", C.c_double)]


class ScalarEstimate(C.Structure):
    _fields_ = [("mean", C.c_double), ("se", C.c_double), ("count", C.c_longlong),
                ("truncated", C.c_longlong)]


class VectorEstimate(C.Structure):
    _fields_ = [("mean", C.c_double * 2), ("se", C.c_double * 2), ("count", C.c_longlong),
                ("truncated", C.c_longlong)]


class SplatConfig(C.Structure):
    _fields_ = [("kernel", KernelSpec), ("coincidenceTol", C.c_double), ("voronoi", C.c_int),
                ("useBallGreens", C.c_int), ("fp64", C.c_int)]


class BoundarySample(C.Structure):
    _fields_ = [("z", C.c_double * 3), ("n", C.c_double * 3), ("pdf", C.c_double),
                ("uHat", C.c_double), ("dHat", C.c_double), ("weight", C.c_double),
                ("segment", C.c_int), ("arc", C.c_double)]


class SourceSample(C.Structure):
    _fields_ = [("y", C.c_double * 3), ("pdf", C.c_double), ("f", C.c_double)]


_P = C.POINTER


class PointState(C.Structure):
    _fields_ = [("count", C.c_size_t), ("dim", C.c_int), ("x", _P(C.c_double)),
                ("fallback", _P(C.c_uint8)), ("gradientUnreliable", _P(C.c_uint8)),
                ("boundarySum", _P(C.c_double)), ("sourceSum", _P(C.c_double)),
                ("nBoundary", _P(C.c_longlong)), ("mSource", _P(C.c_longlong)),
                ("boundaryGradSum", _P(C.c_double)), ("sourceGradSum", _P(C.c_double)),
                ("nBoundaryGrad", _P(C.c_longlong)), ("mSourceGrad", _P(C.c_longlong)),
                ("walkSum", _P(C.c_double)), ("walkCount", _P(C.c_longlong)),
                ("walkTruncated", _P(C.c_longlong)), ("gradientWalkSum", _P(C.c_double)),
                ("gradientWalkCount", _P(C.c_longlong)), ("skipped", _P(C.c_longlong)),
                ("ballRadius", _P(C.c_double))]


# BoundaryEvaluator (cache.h:175-176) kinds
EVALUATOR_NONE, EVALUATOR_FIELD, EVALUATOR_WALKS = 0, 1, 2


class BoundaryEvaluator(C.Structure):
    _fields_ = [("kind", C.c_int), ("field", Field), ("scene", C.c_void_p), ("problem", _P(Problem)),
                ("cfg", _P(CacheConfig))]


def make_field(kind: int = FIELD_NONE, params=(), n: int = 0) -> Field:
    f = Field()
    f.kind = kind
    f.n = n
    for i, v in enumerate(params):
        f.p[i] = float(v)
    return f


def default_walk_config() -> WalkConfig:
    """WalkConfig defaults (pointwise.h:28-35)."""
    return WalkConfig(0.0, 0.0, 10000, 128, 0, 0)


def default_cache_config() -> CacheConfig:
    """CacheConfig defaults (cache.h:114-127)."""
    return CacheConfig(1024, 1024, 16, 160, 0.0, 0.0, CLAMP_OFF, 0, 4, 0, 1,
                       default_walk_config(), 0)
