"""Gather-only timing across kernel kinds (CUDA events, warm)."""
import sys, json, numpy as np, torch
import paper_2302_11825_b200 as B
from paper_2302_11825_b200 import abi

def run(kind, sigma, dim, N, M, K, val=True, grad=True, reps=10, ordered=True):
    rng = np.random.default_rng(0)
    if dim == 2:
        th = rng.uniform(0, 2 * np.pi, N)
        if ordered:  # caches come out ordered along the loop (stratified sampler)
            th = np.sort(th)
        z = np.stack([np.cos(th), np.sin(th)], 1)
        x = rng.uniform(-0.65, 0.65, (K, 2))
        ys = rng.uniform(-0.6, 0.6, (M, 2))
    else:
        z = rng.normal(size=(N, 3)); z /= np.linalg.norm(z, axis=1)[:, None]
        x = rng.uniform(-0.5, 0.5, (K, 3)); ys = rng.uniform(-0.5, 0.5, (M, 3))
    bc = B.BoundaryCache.from_arrays(z, z, np.full(N, 0.2), rng.uniform(-1, 1, N), rng.uniform(-1, 1, N))
    sc = B.SourceCache.from_arrays(ys, np.ones(M), rng.uniform(-1, 1, M)) if M else None
    pts = B.EvaluationPoints(x, dim)
    spec = abi.SplatConfig(abi.KernelSpec(kind, sigma, dim, 2.0), 2e-12, 0, 0)
    B.splat_range(bc, sc, pts, spec, 0, K, val, grad); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): B.splat_range(bc, sc, pts, spec, 0, K, val, grad)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    return K * (N + M) / t, t

if __name__ != "__main__":  # imported by gather_one.py: run a single case
    import os
    case = int(os.environ.get("GATHER_CASE", "1"))
    sel = [("C1", 0, 0.0, 2, 4096, 0, 46112, True, False), ("C2", 0, 0.0, 2, 16384, 0, 261120, True, True)][case]
    run(*sel[1:], reps=2)
    raise SystemExit(0)
props = torch.cuda.get_device_properties(0); sms = props.multi_processor_count
f = 1965e6
cases = [("C1 lap2 u", 0, 0.0, 2, 4096, 0, 46112, True, False, (9, 2)),
         ("C2 lap2 u+grad", 0, 0.0, 2, 16384, 0, 261120, True, True, (18, 2)),
         ("C3 scr2 u+grad (+src)", 1, 10.0, 2, 65536, 65536, 40000, True, True, (50, 3)),
         ("C4 lap3 u", 0, 0.0, 3, 262144, 0, 131072, True, False, (14, 1)),
         ("C5 scr3 u", 1, 1.0, 3, 262144, 0, 131072, True, False, (20, 2))]
for name, kind, sg, dim, N, M, K, v, g, (F, S) in cases:
    for ordered in ([True, False] if dim == 2 else [True]):
        rate, t = run(kind, sg, dim, N, M, K, v, g, ordered=ordered)
        bound = sms * f / max(F / 128, S / 16)
        print(json.dumps({"case": name, "ordered": ordered, "pairs_per_s": rate, "ms": t * 1e3, "bound": bound,
                          "frac": rate / bound}))
