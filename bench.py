"""BVC hot-path benchmark (BASELINE.json metric); BASELINE config 5 by default.

A step is one progressive BVC round, updateSolution (cache.cpp:622-684). The default
workload is C5 (BASELINE.json configs[4], the largest single-GPU config): the 3D
screened (sigma = 1) mixed problem on the outer shell of 8 overlapping displaced
level-6 icospheres — 1,048,576 boundary samples x (128 u-walks + 128 du/dn walks),
then the u gather at exactly 16,777,216 uniform interior query points. `--config
1..4` runs the other configs. Inputs are seeded synthetic data of those shapes (no
dataset exists for this path).

value  = interactions/s = (non-fallback points x cache samples) per round / round time,
         whole job (all ranks). Walk steps/s (closest-Dirichlet queries) are reported
         next to it.
e2e    = the same metric through the public API with host buffers: each call
         uploads the query points (H2D), runs the round and reads u back (D2H).
--impl reference: the reference's own CPU implementation on a bounded sample of the
         same workload (oracle/_ref, compiled from /root/reference's sources; for the
         3D configs, which the reference cannot run, the threaded port of its splat
         loop over its own kernel templates).

Multi-GPU (torchrun): cache samples and query points are sharded by rank; the
packed cache shards are all-gathered with NCCL; each rank gathers its points.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return dict(PEAKS_FALLBACK)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.samples = []  # (time, fields)
        self.proc = None
        self.t_start = self.t_end = None

    def mark(self, which):
        """bracket the timed region; samples are taken from the whole run, kept inside it"""
        setattr(self, "t_" + which, time.time())

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))

    def __exit__(self, *a):
        t0 = time.time()
        while self.proc and time.time() - t0 < 3.0 and not any(t >= (self.t_end or 0) for t, _ in self.samples):
            time.sleep(0.05)  # a short region: wait for the first sample after it
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        inside = [f for t, f in self.samples if self.t_start is not None and self.t_start <= t <= (self.t_end or t)]
        where = "inside the timed region"
        if not inside and self.samples and self.t_end is not None:  # region shorter than the 100 ms period
            inside = [min(self.samples, key=lambda tf: abs(tf[0] - self.t_end))[1]]
            where = "nearest sample to the end of the timed region (region < 100 ms)"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        samples = inside
        sm = [float(s[0]) for s in samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in samples for i in range(4) if len(s) > 4 + i and "Active" in s[4 + i]
                          and "Not" not in s[4 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(samples), "sampled": where}


def build_problem(cfg_id, B, configs, abi):
    c = configs.CONFIGS[cfg_id]()
    if c.extra.get("dim") == 3:
        if "components" in c.extra:
            # soup of 8 closed meshes: the walks and the cache live on its outer shell;
            # inside the union = inside any component
            tris, labels = configs.soup_shell(c)
            comps = configs.soup_components(c)

            def inside(x):
                keep = np.zeros(len(x), bool)
                for comp in comps:
                    keep |= comp.inside(x)
                return keep

            c.extra["shell_triangles"] = int(len(tris))
            c.segments, c.labels = tris, labels
            scene = B.Scene.mesh3(c.vertices, c.segments, c.labels)
        else:
            scene = B.Scene.mesh3(c.vertices, c.segments, c.labels)
            inside = scene.inside
        region = B.SolveRegion(scene, offset=c.region_offset, epsilon=c.epsilon)
        c.points = configs.interior_points(c, inside)  # exactly n_points interior points
        c.dim = 3
        return c, scene, region
    c.dim = 2
    scene = B.Scene(c.vertices, c.segments, c.labels)
    if c.region_mode == abi.REGION_SUBDOMAIN:
        sub = B.Scene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
        region = B.SolveRegion(scene, abi.REGION_SUBDOMAIN, c.region_offset, sub, epsilon=c.epsilon)
        keep = region.boundary.inside(c.points)
    else:
        region = B.SolveRegion(scene, offset=c.region_offset, epsilon=c.epsilon)
        keep = scene.inside(c.points)
    c.points = c.points[keep]
    return c, scene, region


def workload_config(c, cfg_id):
    """The `config` dict both arms print — identical by construction: it describes the
    workload only (sizes, walk budgets, the query set), no measured counts."""
    cfg = c.cache
    M = cfg.nSource if c.problem.f.kind else 0
    d = {"workload": c.name, "config_index": cfg_id, "boundary_samples": int(cfg.nBoundary), "source_samples": int(M),
         "walks_u": int(cfg.nWalksNeumann), "walks_dudn": int(cfg.nWalksDirichlet), "epsilon": c.epsilon,
         "region_offset": cfg.offset, "gradients": bool(c.gradients),
         "l2": "flushed between timed steps (256 MB write)"}
    if c.extra.get("n_points"):
        d["query_points"] = int(c.extra["n_points"])  # exactly this many interior points (configs.interior_points)
        d["query_set"] = "uniform interior points (bbox rejection, seeded)"
    else:
        d["query_set"] = c.extra.get("query_set", "grid")
    return d


METRIC = "BVC eval interactions/s and walk steps/s per GPU; % of FP32/SFU roofline"


class _StdoutToStderr:
    """Native libraries (NCCL prints its version line at communicator init) write to fd 1;
    the bench's stdout must hold exactly one JSON line, so fd 1 points at stderr meanwhile."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def run_gpu(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or os.environ.get("BVC_BENCH_SHARDED") == "1":
        import torch.distributed as dist

        with _StdoutToStderr():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2302_11825_b200 as B
    from paper_2302_11825_b200 import abi, configs

    B.lib().bvc_set_device(local)
    c, scene, region = build_problem(args.config, B, configs, abi)
    cfg = c.cache
    N, M = cfg.nBoundary, (cfg.nSource if c.problem.f.kind else 0)
    K_all = len(c.points)
    # points of this rank: a contiguous slice (the library sorts each rank's points spatially)
    lo_p, hi_p = rank * K_all // world, (rank + 1) * K_all // world
    my_points = c.points[lo_p:hi_p]
    pts = B.EvaluationPoints(my_points, c.dim, index_base=lo_p)
    B.mark_evaluation_points(scene, region, cfg, pts)
    st0 = pts.download()
    k_active = int((~st0["fallback"]).sum())
    del st0
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2

    comm = None

    def round_multi(p, rnd):
        """the library's sharded round (bvc_update_solution_sharded): shard walks by global
        sample index with the rank's band walks overlapped, one ncclAllGather of the
        48-byte samples on the library's stream, then each rank gathers its own points"""
        return B.update_solution_sharded(comm, scene, c.problem, region, cfg, p, c.seed, rnd,
                                         gradients=bool(c.gradients))

    def round_single(p, rnd):
        return B.update_solution(scene, c.problem, region, cfg, p, c.seed, rnd, gradients=bool(c.gradients))

    # BVC_BENCH_SHARDED=1 runs the sharded path (NCCL all-gather) even at N=1, to
    # exercise the multi-GPU plumbing on a single device
    sharded = world > 1 or os.environ.get("BVC_BENCH_SHARDED") == "1"
    if sharded:
        from paper_2302_11825_b200 import distributed

        with _StdoutToStderr():
            comm = distributed.library_comm(B, dist, rank, world)
    step = round_multi if sharded else round_single

    def barrier():
        if dist is not None:
            dist.barrier()

    clk = ClockSampler(local).__enter__()  # running before the timed region; samples kept inside it
    for w in range(args.warmup):
        step(pts, 1000 + w)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches0 = B.launch_count()
    times, per_step = [], []
    clk.mark("start")
    for k in range(args.steps):
        flush.fill_(float(k))  # L2 flush on the library's stream (the legacy default stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = step(pts, k)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        st = dict(st)
        st["kernelSeconds"] = B.last_round_kernel_seconds()  # the round's main walk / gather launches
        per_step.append(st)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk.mark("end")
    clk.__exit__(None, None, None)
    launches = B.launch_count() - launches0
    t_step = float(np.mean(times))
    steps_total = sum(s.get("cacheSteps", 0) for s in per_step)
    walks_total = sum(s.get("cacheWalks", 0) for s in per_step)
    if dist is not None:
        t = torch.tensor([t_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step = float(t.item())
        tot = torch.tensor([k_active, steps_total, walks_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(tot)
        k_active_all, steps_total, walks_total = (float(v) for v in tot.tolist())
    else:
        k_active_all = k_active
    pairs = k_active_all * (N + M)
    value = pairs / t_step
    out = {"metric": METRIC, "value": value, "unit": "interactions/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f32 (f64 accumulation)", "data": "synthetic (seeded, configs.py)",
           "gpu_launches": int(launches / max(args.steps, 1))}
    out["step_ms"] = {"min": min(times) * 1e3, "median": float(np.median(times)) * 1e3, "max": max(times) * 1e3,
                      "mean": float(np.mean(times)) * 1e3, "rank": "this rank's steps (rank 0)"}
    out["resampled_per_step"] = [int(s.get("resampled", 0)) for s in per_step]
    out["walk_steps_per_s"] = steps_total / (t_step * args.steps)
    out["walks_per_s"] = walks_total / (t_step * args.steps)
    out["config"] = workload_config(c, args.config)
    out["counts"] = {"query_points": int(K_all), "nonfallback_points": int(k_active_all),
                     "fallback_points": int(K_all - k_active_all), "pairs_per_step": pairs,
                     "parallelism": f"dp{world} (samples and points sharded)" if sharded else "1 GPU"}
    if "shell_triangles" in c.extra:
        out["counts"]["shell_triangles"] = c.extra["shell_triangles"]
    out["clocks"] = clk.summary()
    # e2e on every rank (the sharded host-buffer round is collective); rank 0 reports the
    # slowest rank's call time over the whole job's interactions
    e2e = e2e_measure(B, c, scene, region, my_points, args, world, t_step, comm=comm if sharded else None,
                      index_base=lo_p, k_active_all=k_active_all, dist=dist)
    if rank == 0:
        # phase times measured live inside the timed steps: the round's own CUDA events on
        # the library stream (RoundStats generateSeconds / splatSeconds)
        live = {"cache_generation": float(np.mean([s["generateSeconds"] for s in per_step])),
                "gather": float(np.mean([s["splatSeconds"] for s in per_step])),
                "walk_kernel": float(np.mean([s["kernelSeconds"]["walk"] for s in per_step])),
                "gather_kernel": float(np.mean([s["kernelSeconds"]["gather"] for s in per_step]))}
        out.update(phase_breakdown(B, c, scene, region, pts, args, per_step[-1], live, k_active))
        out["e2e"] = e2e
        if world == 1 and not args.no_cpu:
            out["cpu_baseline"] = cpu_baseline(c, args.cpu_sample_s)
            wps = out["cpu_baseline"].get("walks_per_s")
            if wps and out.get("walk_stats"):
                out["cpu_baseline"]["steps_per_s_derived"] = wps * out["walk_stats"]["steps_per_walk"]
        if world == 1 and args.extra_configs:
            out["other_configs"] = other_configs(args)
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def ncu_traffic(kernel, cfg_id):
    """DRAM bytes (read + write) per launch of `kernel` ("walk" / "gather") on config
    cfg_id, from the latest committed ncu --set full summary
    (profiles/<round>_<kernel>_c<cfg>_ncu.txt), or None."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_{kernel}_c{cfg_id}_ncu.txt")))
    if not files:
        return None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total = 0.0
    for line in open(files[-1]):
        for key in ("dram__bytes_read.sum =", "dram__bytes_write.sum ="):
            if line.startswith(key):
                parts = line.split("=")[1].split()
                total += float(parts[0]) * scale.get(parts[1] if len(parts) > 1 else "byte", 1.0)
    scale_note = None
    for line in open(files[-1]):
        if line.startswith("# scale "):  # profiled at a reduced size: bytes per launch scaled to the bench's
            scale_note = line[2:].strip()
            total *= float(line.split()[2])
    return {"bytes": total, "source": os.path.relpath(files[-1], ROOT), "scaled": scale_note}


# per-pair FP32-pipe instructions F and SFU ops S
PER_PAIR = {"lap2_u": (9, 2), "lap2_ugrad": (18, 2), "scr2_ugrad": (50, 3), "lap3_u": (14, 1), "scr3_u": (20, 2)}


def phase_breakdown(B, c, scene, region, pts, args, stats, live, k_active):
    """Rooflines of the round's two kernels. Phase times come from the timed steps
    themselves (`live`: the round's device events); without them (sharded rounds) one
    extra round-equivalent is timed here with CUDA events."""
    import torch

    cfg = c.cache
    N, M = cfg.nBoundary, (cfg.nSource if c.problem.f.kind else 0)
    pairs = k_active * (N + M)
    extra = {}
    if live is None or args.config == 1:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        st = {}
        cache = B.generate_boundary_cache(scene, c.problem, region, cfg, c.seed, 77, stats=st)
        ev[1].record()
        scache = B.generate_source_cache(c.problem, region, cfg, c.seed, 77) if M else None
        spec = B.make_splat_config(scene, c.problem, cfg)
        ev[2].record()
        B.splat_range(cache, scache, pts, spec, 0, 1 << 62, True, bool(c.gradients))
        ev[3].record()
        torch.cuda.synchronize()
        if live is None:
            live = {"cache_generation": ev[0].elapsed_time(ev[1]) / 1e3, "gather": ev[2].elapsed_time(ev[3]) / 1e3}
            stats = st
        if args.config == 1:  # BASELINE C1 also asks for fp64: the FP64 gather on the same cache
            spec64 = B.make_splat_config(scene, c.problem, cfg)
            spec64.fp64 = 1
            B.splat_range(cache, scache, pts, spec64, 0, 1 << 62, True, bool(c.gradients))
            torch.cuda.synchronize()
            reps = 5
            ev[2].record()
            for _ in range(reps):
                B.splat_range(cache, scache, pts, spec64, 0, 1 << 62, True, bool(c.gradients))
            ev[3].record()
            torch.cuda.synchronize()
            t64 = ev[2].elapsed_time(ev[3]) / 1e3 / reps
            extra["gather_fp64"] = {"ms": t64 * 1e3, "pairs_per_s": pairs / t64,
                                    "note": "every pair in FP64 (rcp/rsqrt: FP32 seed + 2 Newton steps, libdevice "
                                            "log); parity with the reference's double loop <= 1e-12 (tests)"}
    t_gen, t_gather = live["cache_generation"], live["gather"]
    # the rooflines divide by the dominant launches' own durations (events around the main
    # cache-walk launch and the main gather launch inside each timed round); the phase
    # times (pack/prologue, finalize, sampling, reductions included) are reported beside them
    k_walk, k_gather = live.get("walk_kernel") or t_gen, live.get("gather_kernel") or t_gather
    peaks = load_peaks()
    # walk traffic: SURVEY §8(d) algorithmic bytes per step (packed fp32 node 32 B, 2D segment
    # 16 + 4 B, 3D triangle 36 + 4 B, walk state 32 B) x the fetch counts of a counting launch
    prof = B.walk_traffic_profile(scene, c.problem, region, cfg, c.seed, 77)
    steps = max(prof["steps"], 1.0)
    node_b, prim_b = 32, (40 if c.dim == 3 else 20)
    bytes_per_step = (prof["node_fetches"] * node_b + prof["prim_fetches"] * prim_b) / steps + 32.0
    walk_bytes = bytes_per_step * stats["cacheSteps"]
    walk_achieved = walk_bytes / k_walk / 1e9
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    # gather bound: SMs * f_SM / max(F/128, S/16) pairs/s
    props = torch.cuda.get_device_properties(0)
    sms = props.multi_processor_count
    f_sm = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    if c.dim == 3:
        key = "scr3_u" if c.problem.kernel.kind else "lap3_u"
    else:
        key = ("scr2_ugrad" if c.problem.kernel.kind else "lap2_ugrad") if c.gradients else "lap2_u"
    F, S = PER_PAIR[key]
    bound = sms * f_sm / max(F / 128.0, S / 16.0)
    gather_rate = pairs / k_gather
    if args.no_probe:  # profiling runs: reuse the committed measurement
        pipes = json.load(open(os.path.join(ROOT, "profiles", "r1_pipe_peaks.json")))["rates"]
        pipes = {k: v["per_s"] for k, v in pipes.items()}
    else:
        pipes = B.pipe_probe()
    mufu = min(pipes["mufu_lg2"], pipes["mufu_rcp"]) if c.dim == 2 else pipes["mufu_rsq"]
    bound_meas = min(pipes["ffma"] / F, mufu / S)
    gtraffic = ncu_traffic("gather", args.config) or {}
    wtraffic = ncu_traffic("walk", args.config) or {}
    walk_roof = {"bound": "hbm", "kernel": "bvc walk_kernel (cache generation)", "achieved": walk_achieved,
                 "peak": hbm, "unit": "GB/s", "frac": walk_achieved / hbm, "traffic": wtraffic.get("bytes"),
                 "traffic_source": wtraffic.get("source"), "algorithmic_bytes_per_launch": walk_bytes,
                 "algorithmic_bytes_per_step": bytes_per_step,
                 "node_fetches_per_step": prof["node_fetches"] / steps,
                 "prim_fetches_per_step": prof["prim_fetches"] / steps, "peak_source": peaks["source"],
                 "l2_read_peak_gbs": pipes["l2_read_bytes"] / 1e9,
                 "frac_of_l2_read_peak": walk_achieved / (pipes["l2_read_bytes"] / 1e9),
                 "note": ("SURVEY §8(d) bytes: node 32 B, primitive 20 B (2D) / 40 B (3D), 32 B walk state per step; "
                          "the scene is L1/L2-resident, the kernel is latency/divergence-bound (see profiles/)")}
    gather_roof = {"bound": "fp32+sfu", "kernel": f"bvc gather_kernel ({key})", "achieved": gather_rate,
                   "peak": bound, "unit": "pairs/s", "frac": gather_rate / bound,
                   "peak_formula": f"{sms} SMs x {f_sm / 1e6:.0f} MHz / max({F}/128, {S}/16)",
                   "peak_measured_pipes": bound_meas, "frac_measured_pipes": gather_rate / bound_meas,
                   "pairs_per_launch": pairs, "traffic": gtraffic.get("bytes"),
                   "traffic_source": gtraffic.get("source"),
                   "algorithmic_bytes_per_launch": (k_active * (12 if c.dim == 3 else 8) + (N + M) * 32),
                   "note": "compute-bound N-body gather: no tensor-core or HBM roofline applies (SURVEY §8d)"}
    dominant = "walk" if t_gen >= t_gather else "gather"
    roof = dict(walk_roof if dominant == "walk" else gather_roof)
    roof["dominant"] = dominant
    roof["timing"] = ("live: mean over the timed steps of the launch's own device events" if args.config != 1 or live
                      else "one extra round")
    return {
        **extra,
        "pipe_peaks": {k: v for k, v in pipes.items()},
        "walk_stats": {"steps_per_walk": stats["cacheSteps"] / max(stats["cacheWalks"], 1),
                       "truncated_fraction": stats["cacheTruncated"] / max(stats["cacheWalks"], 1),
                       "walks": stats["cacheWalks"]},
        "phases_s": {"cache_generation": t_gen, "gather": t_gather},
        "kernel_s": {"walk": k_walk, "gather": k_gather,
                     "note": "the round's main cache-walk and gather launches (events on the library stream)"},
        "roofline": roof,
        "walk_roofline": walk_roof,
        "gather_roofline": gather_roof,
    }


def e2e_measure(B, c, scene, region, points, args, world, t_step, comm=None, index_base=0, k_active_all=None,
                dist=None):
    """Public API with host buffers: H2D points, one round, D2H of u (and grad u). With a
    communicator (N > 1, or BVC_BENCH_SHARDED) the sharded host-buffer round: this rank's
    points, its share of the walks, the all-gather, its gather."""
    import torch

    times = []
    reps = max(2, min(args.steps, 5)) if t_step < 1.0 else 3
    # pinned host buffers for the step's input points and its u / grad u results
    src = torch.from_numpy(np.ascontiguousarray(points, dtype=np.float64)).pin_memory().numpy()
    u_out = torch.empty(len(points), dtype=torch.float64).pin_memory().numpy()
    g_out = torch.empty((len(points), c.dim), dtype=torch.float64).pin_memory().numpy() if c.gradients else None
    for k in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # one call (runSolveInMemory's round): H2D of the points from pinned memory,
        # classification, the round, D2H of u and grad u into pinned memory; the
        # upload and classification overlap the cache walks (second stream)
        if comm is not None:
            res = B.update_solution_sharded_host(comm, scene, c.problem, region, c.cache, src, index_base, c.seed,
                                                 500 + k, gradients=bool(c.gradients), out=(u_out, g_out))
        else:
            res = B.update_solution_host(scene, c.problem, region, c.cache, src, c.seed, 500 + k,
                                         gradients=bool(c.gradients), out=(u_out, g_out))
        torch.cuda.synchronize()
        if k:
            times.append(time.perf_counter() - t0)
        u = res[0] if c.gradients else res
        assert np.all(np.isfinite(u))
    N, M = c.cache.nBoundary, (c.cache.nSource if c.problem.f.kind else 0)
    if k_active_all is None:
        pts = B.EvaluationPoints(src, c.dim)
        B.mark_evaluation_points(scene, region, c.cache, pts)
        k_active_all = int((~pts.download()["fallback"]).sum())
    t = float(np.mean(times))
    if dist is not None:  # the job's call time is the slowest rank's
        tt = torch.tensor([t], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    d2h = len(points) * 8 * (1 + (c.dim if c.gradients else 0))
    return {"value": k_active_all * (N + M) / t, "unit": "interactions/s", "ms_per_step": t * 1e3,
            "ms_min": min(times) * 1e3, "ms_median": float(np.median(times)) * 1e3, "ms_max": max(times) * 1e3,
            "calls": len(times),
            "h2d_bytes_per_step": int(points.size * 8), "d2h_bytes_per_step": int(d2h),
            "note": "wall clock per bvc_update_solution_host call (bvc_update_solution_sharded_host per rank for "
                    "N > 1, max over ranks) from pinned host buffers: point upload (H2D) and classification "
                    "(overlapping the cache walks on a second stream), one round, u/grad-u readout (D2H), per rank's "
                    "points; no L2 flush between calls"}


_ACTIVE = {}  # the reference's non-fallback query points per config object (computed once)


def reference_round_estimate(c, sample_s=20.0, threads=0):
    """Time the reference's own updateSolution pieces (oracle/_ref) on a bounded sample of
    the round: generateBoundaryCache on n_sub samples (cost ~ #walks) and
    splatSolution(+splatGradient) on k_sub points against a full-size cache (cost ~ K (N+M)).
    The rate is the full round's pairs over the round time extrapolated from the sample;
    `seconds` is the sample's measured wall time."""
    from oracle import oracle as O
    from paper_2302_11825_b200 import abi

    t_all = time.perf_counter()
    O.ref_lib()
    rs = O.RefScene(c.vertices, c.segments, c.labels)
    if c.region_mode == abi.REGION_SUBDOMAIN:
        sub = O.RefScene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
        rr = O.RefRegion(rs, abi.REGION_SUBDOMAIN, c.region_offset, sub, eps=c.epsilon)
    else:
        rr = O.RefRegion(rs, abi.REGION_WHOLE_DOMAIN, c.region_offset, eps=c.epsilon)
    cfg = c.cache
    N, M = cfg.nBoundary, (cfg.nSource if c.problem.f.kind else 0)
    cfg.threads = threads
    cores = O.ref_lib().ref_thread_count(threads)
    # walks: grow the sample until ~40% of the budget is spent
    n_sub, t_gen = 8, 0.0
    while True:
        sub_cfg = abi.CacheConfig.from_buffer_copy(cfg)
        sub_cfg.nBoundary = n_sub
        t0 = time.perf_counter()
        small = O.ref_generate_boundary_cache(rs, c.problem, rr, sub_cfg, c.seed, 0)
        t_gen = time.perf_counter() - t0
        if t_gen > 0.4 * sample_s or n_sub >= N:
            break
        n_sub = min(N, int(n_sub * max(2.0, 0.4 * sample_s / max(t_gen, 1e-3) * 0.8)))
    gen_full = t_gen * N / n_sub
    # the reference's walk throughput (RoundStats cacheWalks / generation time, cache.cpp:381-387)
    sample_walks = int(small["stats"][1]) if "stats" in small else 0
    # gather: the reference splats on a point subset against a full-size cache
    rng = np.random.default_rng(0)
    reps = int(np.ceil(N / n_sub))
    cache = {k: np.tile(v, (reps, 1) if np.ndim(v) == 2 else reps)[:N] for k, v in small.items()
             if k in ("z", "n", "pdf", "uHat", "dHat", "weight")}
    scache = None
    if M:
        scache = O.ref_generate_source_cache(c.problem, rr, cfg, c.seed, 0)
    # the query set: the config's points inside the scene (the reference's own inside test),
    # then markEvaluationPoints' fallback split
    act = _ACTIVE.get(id(c))
    if act is None:
        pts = c.points
        if c.region_mode == abi.REGION_SUBDOMAIN:
            sub = O.RefScene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
            pts = pts[sub.inside(pts)]
        else:
            pts = pts[rs.inside(pts)]
        fb, _ = O.ref_mark_points(rs, rr, cfg, pts)
        act = _ACTIVE[id(c)] = pts[~fb]
    k_sub = 64
    while True:
        xs = act[rng.choice(len(act), size=min(k_sub, len(act)), replace=False)]
        spec = abi.KernelSpec(c.problem.kernel.kind, c.problem.kernel.sigma, 2, rs.diagonal)
        st = O.ref_splat(spec, 1e-12 * rs.diagonal, cache, scache, xs, value=True, gradient=bool(c.gradients),
                         threads=threads)
        t_spl = st["seconds"]
        if t_spl > 0.4 * sample_s or k_sub >= len(act):
            break
        k_sub = min(len(act), int(k_sub * max(2.0, 0.4 * sample_s / max(t_spl, 1e-3) * 0.8)))
    splat_full = t_spl * len(act) / len(xs)
    t_round = gen_full + splat_full
    pairs = len(act) * (N + M)
    return {"value": pairs / t_round, "unit": "interactions/s", "cores": int(cores), "kind": "reference",
            "cpu": cpu_model(), "host_threads": os.cpu_count(), "seconds": time.perf_counter() - t_all,
            "sample": (f"the reference's generateBoundaryCache on {n_sub}/{N} samples ({t_gen:.2f} s) + splatSolution"
                       f"{'+splatGradient' if c.gradients else ''} on {len(xs)}/{len(act)} points vs a full "
                       f"{N}+{M}-sample cache ({t_spl:.2f} s); rate = full-round pairs / round time extrapolated "
                       "linearly from the sample (cost ~ walks, ~ K(N+M))"),
            "round_seconds_extrapolated": t_round,
            "walks_per_s": sample_walks / t_gen if t_gen > 0 and sample_walks else None,
            "walks_note": "the reference's walks/s in its generateBoundaryCache sample (RoundStats.cacheWalks / time); "
                          "CPU steps/s = walks/s x the GPU's mean steps per walk (derived, the reference counts no steps)"}


def port_gather_3d(c, sample_s, threads=0):
    """3D has no reference path (pointwise.cpp:23: the solver is 2D-only), so there are no
    CPU walks to time. The CPU number is splatSolution's loop (cache.cpp:426-461) over
    Vector3 calling the reference's own kernel templates (kernels.h:78-129), threaded with
    its parallelFor (oracle/ref_driver.cpp ref_splat3), on k points against a full-size
    N-sample cache (the per-pair cost does not depend on the values). Gather only."""
    from oracle import oracle as O
    from paper_2302_11825_b200 import abi

    t_all = time.perf_counter()
    N = c.cache.nBoundary
    cache = _ACTIVE.get(("cache3", id(c)))
    if cache is None:
        rng = np.random.default_rng(0)
        z = c.vertices[rng.integers(0, len(c.vertices), N)]
        n = rng.normal(size=(N, 3))
        n /= np.linalg.norm(n, axis=1)[:, None]
        cache = _ACTIVE[("cache3", id(c))] = dict(z=z, n=n, pdf=np.full(N, 0.1), uHat=rng.uniform(-1, 1, N),
                                                   dHat=rng.uniform(-1, 1, N))
    diag = float(np.linalg.norm(c.vertices.max(0) - c.vertices.min(0)))
    spec = abi.KernelSpec(c.problem.kernel.kind, c.problem.kernel.sigma, 3, diag)
    cores = O.ref_lib().ref_thread_count(threads)
    # size the sample once per (config, budget); later steps time that size directly
    k, fixed = _ACTIVE.get(("k3", id(c), sample_s), 4 * cores), ("k3", id(c), sample_s) in _ACTIVE
    while True:
        xs = c.points[:k]
        st = O.ref_splat3(spec, 1e-12 * diag, cache, xs, threads=threads)
        t = st["seconds"]
        if fixed or t > 0.5 * sample_s or k >= len(c.points):
            break
        k = min(len(c.points), int(k * max(2.0, 0.5 * sample_s / max(t, 1e-3) * 0.8)))
    _ACTIVE[("k3", id(c), sample_s)] = k
    return {"value": k * N / t, "unit": "interactions/s", "cores": int(cores), "kind": "port", "cpu": cpu_model(),
            "host_threads": os.cpu_count(), "seconds": time.perf_counter() - t_all,
            "sample": (f"splatSolution's loop (cache.cpp:426-461) over Vector3 with the reference's kernel templates "
                       f"(kernels.h:78-129) and parallelFor, {cores} threads, on {k} points x {N} samples "
                       f"({t:.2f} s); gather only: the reference has no 3D walk path (pointwise.cpp:23), so the "
                       "CPU round's walk time is not counted (the GPU value includes its walks)")}


def cpu_model():
    """`model name` of the host CPU (SURVEY 8d asks for the core count and model per run)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_estimate(c, sample_s, threads=0):
    if c.extra.get("dim") == 3:
        return port_gather_3d(c, sample_s, threads)
    return reference_round_estimate(c, sample_s, threads)


def cpu_baseline(c, sample_s):
    try:
        return cpu_estimate(c, sample_s)
    except Exception as e:  # oracle/_ref missing on this host
        return {"value": None, "unit": "interactions/s", "cores": os.cpu_count(),
                "kind": "port" if c.extra.get("dim") == 3 else "reference", "sample": f"unavailable: {e}"}


def run_reference(args):
    """The reference arm: the reference's own CPU implementation of the path (oracle/_ref,
    compiled from /root/reference's sources; for the 3D configs the threaded port of its
    splat loop over its kernel templates), all host threads, rank 0 only. Each step is a
    bounded sample of the same workload, timed; `ms_per_step` is that measured sample's
    wall time, `value` the rate it implies for the full round."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2302_11825_b200 import configs

    c = configs.CONFIGS[args.config]()
    budget = min(args.cpu_sample_s, 150.0 / max(args.steps + args.warmup, 1))
    vals, secs = [], []
    t0 = time.perf_counter()
    for k in range(args.warmup + args.steps):
        est = cpu_estimate(c, budget)
        if k >= args.warmup:
            vals.append(est)
            secs.append(est["seconds"])
    value = float(np.mean([v["value"] for v in vals]))
    kind = vals[-1]["kind"]
    out = {"metric": METRIC, "value": value, "unit": "interactions/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(secs)) * 1e3,
           "ms_per_step_note": "measured wall time of one bounded-sample step (not an extrapolated round)",
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded, configs.py)", "impl": "reference",
           "config": workload_config(c, args.config),
           "cpu_baseline": {"value": value, "unit": "interactions/s", "cores": vals[-1]["cores"],
                            "cpu": vals[-1]["cpu"], "kind": kind, "sample": vals[-1]["sample"]},
           "e2e": {"value": value, "unit": "interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "wall_s": time.perf_counter() - t0}
    if "round_seconds_extrapolated" in vals[-1]:
        out["round_seconds_extrapolated"] = float(np.mean([v["round_seconds_extrapolated"] for v in vals]))
    print(json.dumps(out), flush=True)


_T_START = time.perf_counter()


def other_configs(args):
    """The other BASELINE configs (not the headline): a short bench.py run of each in a
    fresh process (3 timed rounds, 2 warm-up), so one driver run leaves evidence for all
    five. Skipped once the run has used 7 minutes; each run is capped at 80 s."""
    res = {}
    for cid in (1, 2, 3, 4):
        if cid == args.config:
            continue
        if time.perf_counter() - _T_START > 420.0:
            res[f"C{cid}"] = {"skipped": "time budget of the default run"}
            continue
        cmd = [sys.executable, os.path.abspath(__file__), "--config", str(cid), "--steps", "3", "--warmup", "2",
               "--no-cpu", "--no-probe", "--no-extra"]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=80, cwd=ROOT,
                               env={k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE")})
            line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
            d = json.loads(line)
            res[f"C{cid}"] = {"workload": d["config"]["workload"], "ms_per_step": d["ms_per_step"],
                              "step_ms": d["step_ms"], "value": d["value"], "unit": d["unit"],
                              "e2e_ms_per_call": d["e2e"]["ms_per_step"], "phases_s": d.get("phases_s"),
                              "kernel_s": d.get("kernel_s"),
                              "gather_frac_of_bound": d.get("gather_roofline", {}).get("frac"),
                              "walk_steps_per_s": d.get("walk_steps_per_s"), "clocks": d.get("clocks")}
            if "gather_fp64" in d:  # C1's fp64 variant (BASELINE configs[0])
                res[f"C{cid}"]["gather_fp64"] = d["gather_fp64"]
        except Exception as e:  # noqa: BLE001 - reported, the headline line stands
            res[f"C{cid}"] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-probe", action="store_true", help="skip the pipe microbenchmarks (profiling runs)")
    ap.add_argument("--no-extra", dest="extra_configs", action="store_false",
                    help="skip the short runs of the other configs (other_configs key)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
