"""Shared test helpers: problems from the reference's analytic registry
(problems.cpp:65-156) as device field descriptors, and small statistics."""
import math

import numpy as np

from oracle import oracle as O
from paper_2302_11825_b200 import abi


def kspec(kind=0, sigma=0.0, dim=2, scale=1.0):
    return abi.KernelSpec(kind, float(sigma), dim, float(scale))


def make_problem(kernel, f=None, g=None, h=None):
    pb = abi.Problem()
    pb.kernel = kernel
    pb.f = f if f is not None else abi.make_field()
    pb.g = g if g is not None else abi.make_field()
    pb.h = h if h is not None else abi.make_field()
    return pb


def disk_linear():
    """disk-linear (problems.cpp:65-76): u = x on the 256-gon."""
    return O.circle_geometry(segments=256), make_problem(kspec(), g=abi.make_field(abi.FIELD_LINEAR, [1, 0, 0, 0]))


def disk_poisson():
    """disk-poisson (problems.cpp:78-92): f = 1, u = (|x|^2 - 1)/4."""
    return O.circle_geometry(segments=256), make_problem(
        kspec(), f=abi.make_field(abi.FIELD_CONSTANT, [1.0]), g=abi.make_field(abi.FIELD_RADIAL, [0, 0, 0.25, 2, -0.25]))


def square_mixed():
    """square-mixed-linear (problems.cpp:94-108): Neumann y = 0,1; Dirichlet x = 0,1; u = x."""
    return O.rectangle_geometry([0, 0], [1, 1], [1, 0, 1, 0]), make_problem(
        kspec(), g=abi.make_field(abi.FIELD_LINEAR, [1, 0, 0, 0]))


def vertical():
    """the reflecting-data problem of test_pointwise.cpp:22-34: u = y, h = n_y."""
    return O.rectangle_geometry([0, 0], [1, 1], [1, 0, 1, 0]), make_problem(
        kspec(), g=abi.make_field(abi.FIELD_LINEAR, [0, 1, 0, 0]), h=abi.make_field(abi.FIELD_LINEAR, [0, 2, -1, 0]))


def screened_constant():
    """screened-constant (problems.cpp:110-124): sigma = 2, f = -sigma, u = 1."""
    return O.rectangle_geometry([0, 0], [1, 1], [0, 0, 0, 0]), make_problem(
        kspec(1, 2.0), f=abi.make_field(abi.FIELD_CONSTANT, [-2.0]), g=abi.make_field(abi.FIELD_CONSTANT, [1.0]))


def star_geometry(seed, n=24, mixed=True):
    rng = np.random.default_rng(seed)
    th = np.sort(rng.uniform(0, 2 * np.pi, n))
    r = rng.uniform(0.4, 1.0, n)
    v = np.stack([r * np.cos(th), r * np.sin(th)], 1)
    s = np.stack([np.arange(n), (np.arange(n) + 1) % n], 1).astype(np.int32)
    lab = (rng.uniform(size=n) < 0.5).astype(np.int32) if mixed else np.zeros(n, np.int32)
    if mixed:
        lab[0] = 0
    return v, s, lab


def zscore(m1, s1, m2, s2):
    return (m1 - m2) / math.sqrt(s1 * s1 + s2 * s2)


def rel_err(got, ref):
    """SURVEY §8d parity metric: max |got - ref| / max(|ref|_max, RMS(ref))."""
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    scale = max(np.max(np.abs(ref)), float(np.sqrt(np.mean(ref ** 2))), 1e-300)
    return float(np.max(np.abs(got - ref)) / scale)


def rel_err_pointwise(got, ref):
    """SURVEY §8d's per-point form: max_k |got_k - ref_k| / max(|ref_k|, RMS(ref))."""
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    rms = max(float(np.sqrt(np.mean(ref ** 2))), 1e-300)
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), rms)))
