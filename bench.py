#!/usr/bin/env python
"""Benchmark of the RTG-SLAM mapping hot path on B200 (contract: DESIGN.md §7).

Workloads (BASELINE.json configs; `--config`, default C3 at one GPU and C5 under torchrun):
  C3 / C2  one STEP = one pass of every §8(a) row over one synthetic frame:
      ingest     A1 project -> A2 bin (all tiles) -> A3/A4 FULL render -> A7 classify + sample
      iteration  A1 project -> A0 coverage + tile keep -> A2 bin (kept tiles) -> A3/A4 MASKED render
                 -> A5 masked backward -> A6 Adam
      `value` counts one mapping iteration per step (each step also carries a full frame ingest, so
      it is conservative w.r.t. the paper's 'mapping / iteration').
  C4       render-only novel views: A1 + A2 + A3/A4 FULL per step (frames/s).
  C5       the keyframe batch: 64 C3 views split over N ranks; per view a FULL
           render, its top-40 % colour-error pixels and the masked backward over ALL Gaussians; an
           in-place NCCL reduce-scatter of the gradients, Adam on each rank's block of rows, in-place
           NCCL all-gathers of the map (dist.global_step_sharded).  `value` = views/s of the whole job
           (strong scaling: the 64-view batch is fixed), plus T_1 / (N T_N) measured in the same run.

    python bench.py [--gpus N --steps K --warmup W] [--config C2|C3|C4|C5] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "mapping iters/sec (fwd+masked bwd) and Gaussian-pixel blends/s vs roofline"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1965.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 20 ms during the timed region."""

    def __init__(self, idx: int):
        self.idx = idx
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


_SCENES = {}


def _scene(cfg_name):
    from synth import CONFIGS, make_frame, make_pose, make_scene
    if cfg_name not in _SCENES:
        cfg = CONFIGS[cfg_name]
        scene = make_scene(cfg)
        R, t = make_pose(cfg)
        _SCENES[cfg_name] = (cfg, scene, R, t, make_frame(cfg))
    return _SCENES[cfg_name]


def _oracle_active_count(cfg_name):
    """|P| of the config's primary-view iteration by the ORACLE (O4 coverage by splatting the unstable
    support rects, the 50 % tile rule): the workload size the CPU leg extrapolates to (setup, untimed)."""
    import torch
    from oracle import projection as OP, raster as OR
    cfg, scene, R, t, _ = _scene(cfg_name)
    with torch.no_grad():
        pr = OP.project(OP.params_from_scene(scene), R, t, OP.camera(cfg), scene["sh_degree"])
    cov, _ = OR.unstable_coverage_splat(pr, (scene["flags"] & 2) == 0, cfg.width, cfg.height)
    return int(OR.active_set(cov, OR.tile_keep(cov)).sum())


def oracle_sample(cfg_name: str, k_fwd: int, k_bwd: int, seed: int = 0):
    """The oracle (float64 CPU, as it stands) on a bounded sample of the step: projection of ALL
    Gaussians, the forward render (Eq.1-5) of `k_fwd` pixels, and the masked iteration's loss (colour
    AND depth, Eq.7 with the full-frame normalisations) + autograd backward over `k_bwd` active
    pixels (the projection is part of the autograd graph, as in the iteration).  Returns the timings
    of the three parts."""
    import torch
    from oracle import loss as OL, projection as OP, raster as OR
    cfg, scene, R, t, (col, dep) = _scene(cfg_name)
    cam = OP.camera(cfg)
    threads = torch.get_num_threads()
    rng = np.random.default_rng(seed)
    t0 = time.perf_counter()
    with torch.no_grad():
        proj = OP.project(OP.params_from_scene(scene), R, t, cam, scene["sh_degree"])
    t_proj = time.perf_counter() - t0
    pix = np.stack([rng.integers(0, cfg.width, k_fwd), rng.integers(0, cfg.height, k_fwd)], 1)
    t1 = time.perf_counter()
    with torch.no_grad():
        OR.render_pixels(proj, pix, cam, R, chunk=8, want_margin=False)
    t_fwd = time.perf_counter() - t1
    # active pixels: the slab (the unstable Gaussians' image-x range)
    u = scene["u_img"][(scene["flags"] & 2) == 0]
    x_lo = int(np.percentile(u, 5))
    act = np.zeros((cfg.height, cfg.width), bool)
    act[rng.integers(0, cfg.height, k_bwd), rng.integers(max(x_lo, 0), cfg.width, k_bwd)] = True
    t2 = time.perf_counter()
    res = OL.iteration_loss(scene, R, t, cam, col, dep, act)
    res["L"].backward()
    t_bwd = time.perf_counter() - t2
    return dict(t_proj=t_proj, t_fwd=t_fwd, t_bwd=t_bwd, k_fwd=k_fwd, k_bwd=int(act.sum()), threads=threads,
                t_sample=time.perf_counter() - t0)


def oracle_step_seconds(r, cfg, n_active):
    """The oracle doing the bench's step, extrapolated from the sample: ingest (projection of all
    Gaussians + forward render of every pixel) + one uncached mapping iteration (projection again,
    part of the timed backward sample, + render / loss / backward of the |P| active pixels)."""
    return (r["t_proj"] + r["t_fwd"] * cfg.width * cfg.height / r["k_fwd"]
            + r["t_bwd"] * n_active / r["k_bwd"])


ORACLE_SAMPLE = ("per step: projection of all {n} Gaussians + forward render of {kf} pixels + colour+depth loss "
                 "and autograd backward of {kb} active pixels (float64 torch CPU, {th} threads), {ts:.1f} s; "
                 "extrapolated linearly to the step (projection + forward of all {wh} pixels + iteration over "
                 "|P| = {p} active pixels, |P| from the oracle's own coverage)")


def oracle_c1_measured():
    """Supplementary, MEASURED (no extrapolation): the oracle's whole C1 step (BASELINE configs[0]):
    ingest (projection, FULL render of every pixel, Eq.6 classify) + one iteration (coverage + tile
    keep, projection + render + loss + backward of P, Adam) - on all host threads and on one."""
    import torch
    from oracle import classify as OC, loss as OL, optim as OO, projection as OP, raster as OR
    from synth import CONFIGS, make_frame, make_pose, make_scene
    cfg = CONFIGS["C1"]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    col, dep = make_frame(cfg)
    cam = OP.camera(cfg)
    K = (scene["sh_degree"] + 1) ** 2

    def step():
        with torch.no_grad():
            pr = OP.project(OP.params_from_scene(scene), R, t, cam, scene["sh_degree"])
            img = OR.render_image(pr, cam, R, want_margin=False)
        OC.classify(img["color"].numpy(), img["trans"].numpy(), img["depth"].numpy(), img["index"], col, dep,
                    scene["flags"])
        unstable = (scene["flags"] & 2) == 0
        cov, _ = OR.unstable_coverage(pr, unstable, OR.all_pixels(cfg.width, cfg.height))
        cov = cov.reshape(cfg.height, cfg.width)
        act = OR.active_set(cov, OR.tile_keep(cov))
        gid = np.nonzero(unstable)[0]
        res = OL.iteration_grads(scene, R, t, cam, col, dep, act, gid)
        theta = np.concatenate([scene["pos"][gid], scene["log_scale"][gid], scene["rot"][gid],
                                scene["sh"][gid].reshape(len(gid), -1)], 1).astype(np.float64)
        z = np.zeros_like(theta)
        OO.unstable_step(theta, res["grad"], z, z.copy(), theta[:, :10].copy(), (scene["flags"][gid] & 1) != 0,
                         1000.0, OO.lr_vector(K, 1e-3, 5e-4, 2.5e-5, 4e-3, 1e-3), 1, np.zeros(len(gid), np.int64))

    out = {}
    nt = torch.get_num_threads()
    for label, threads in (("all_threads", nt), ("one_thread", 1)):
        torch.set_num_threads(threads)
        step()  # warm
        t0 = time.perf_counter()
        step()
        out[label] = {"s_per_step": round(time.perf_counter() - t0, 3), "threads": threads}
    torch.set_num_threads(nt)
    return out


def reference_arm(args, rank, world):
    """--impl reference: the oracle timed on the host cores (rank 0 only), one bounded sample of the
    workload per step (ms_per_step is the sample's measured time; value extrapolates the sample to
    the whole step, the fraction is stated).  The workload is the GPU arm's: C3 at one GPU, the C5
    keyframe batch under torchrun (64 views: per view projection + forward of every pixel + the
    backward of the top-40 % pixels over every Gaussian)."""
    if rank != 0:
        return
    from synth import CONFIGS
    eff = args.config or ("C5" if world > 1 else "C3")
    cfg_name = "C3" if eff == "C5" else eff
    cfg = CONFIGS[cfg_name]
    HW = cfg.width * cfg.height
    n_active = int(round(0.4 * HW)) if eff == "C5" else _oracle_active_count(cfg_name)
    rows = []
    # the per-step sample shrinks with the run length so that warmup + steps samples stay within a
    # few minutes (~0.7 s of projection + ~45 ms per sampled pixel at C3, 16 host threads)
    n_run = args.warmup + args.steps
    kp = args.ref_pixels if n_run <= 30 else max(8, int(round(args.ref_pixels * 30 / n_run)))
    for s in range(n_run):
        r = oracle_sample(cfg_name, kp, kp, seed=s)
        if s >= args.warmup:
            rows.append(r)
    t_sample = statistics.mean(r["t_sample"] for r in rows)
    t_unit = statistics.mean(oracle_step_seconds(r, cfg, n_active) for r in rows)
    if eff == "C5":   # value in views / s: the batch step is 64 such views
        v, t_step = 1.0 / t_unit, N_C5_VIEWS * t_unit
        config = batch_config(cfg, world)
        what = (f"one C5 view (projection + forward of all {HW} pixels + backward of the top-40 % = {n_active} "
                f"pixels), x {N_C5_VIEWS} views per step")
    else:
        v, t_step = 1.0 / t_unit, t_unit
        config = mapping_config(cfg, True, "CUDA graph of the whole step (2 streams)", world)
        what = None
    cpu = {"value": v, "unit": "iters/s", "cores": rows[0]["threads"], "kind": "oracle", "extrapolated": True,
           "sample_fraction": t_sample / t_step,
           "sample": ORACLE_SAMPLE.format(n=cfg.n, kf=rows[0]["k_fwd"], kb=rows[0]["k_bwd"], th=rows[0]["threads"],
                                          ts=t_sample, wh=HW, p=n_active) + (f"; {what}" if what else "")}
    line = {"metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_sample, "higher_is_better": True,
            "scaling": "strong" if eff == "C5" else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config, "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def batch_config(cfg, world):
    return {"workload": (f"C5 keyframe batch: {N_C5_VIEWS} views of the C3 Replica-shaped "
                         f"{cfg.width}x{cfg.height} 1M-Gaussian scene (+-0.3 m / 15 deg around the "
                         f"primary view); iteration = one view's FULL render + top-40 % colour-error "
                         f"pixels + masked backward over ALL Gaussians; step = {N_C5_VIEWS} views + "
                         f"in-place NCCL reduce-scatter + Adam on each rank's row block (position lr "
                         f"0, others x 0.1) + in-place NCCL all-gathers (P:284)"),
            "l2": "flushed between timed steps (256 MB write)", "launch": "eager (NCCL in the step)",
            "parallelism": f"{world} ranks x {N_C5_VIEWS // world} views, sharded optimiser"}


def mapping_config(cfg, cached, launch, world):
    return {"workload": workload_name(cfg, cached),
            "l2": "flushed between timed steps (256 MB write); Gaussian SoA 237 MB > L2",
            "launch": launch, "parallelism": "single GPU" if world == 1 else f"{world} replicas"}


SHAPES = {"C1": "small synthetic", "C2": "TUM-shaped", "C3": "Replica-shaped", "C4": "ScanNet++-shaped"}


def workload_name(cfg, cached=True):
    head = (f"{cfg.name} {SHAPES.get(cfg.name, 'synthetic')} {cfg.width}x{cfg.height}, {cfg.n} Gaussians "
            f"({int(round(cfg.frac_transparent * 100))}% transparent), "
            f"{int(cfg.frac_unstable * 100)}% unstable slab, SH deg {cfg.sh_degree}; ")
    if cached:
        return head + ("step = frame ingest (A1,A2,A3/A4 FULL,A7, f3 stable cache) + one masked mapping "
                       "iteration (A1 on the unstable slots,A0,A2 merged with the cache,A3/A4,A5,A6)")
    return head + "step = frame ingest (A1,A2,A3/A4 FULL,A7) + one masked mapping iteration (A1,A0,A2,A3/A4,A5,A6)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="C2 | C3 | C4 | C5 (default: C3, or C5 under torchrun)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-pixels", type=int, default=64, help="oracle sample: forward and backward pixels")
    ap.add_argument("--phases", action="store_true", help="print per-call timings to stderr")
    ap.add_argument("--no-graph", action="store_true", help="launch every step eagerly (no CUDA graph)")
    ap.add_argument("--no-cache", action="store_true", help="iteration without the f3 stable-projection cache")
    ap.add_argument("--no-fuse-adam", action="store_true", help="separate A5 backward and A6 Adam calls")
    ap.add_argument("--no-restore", action="store_true", help="diagnostic: let the map drift between timed steps")
    ap.add_argument("--no-window", action="store_true", help="skip the supplementary mapping-window measurement")
    ap.add_argument("--no-reorder", action="store_true",
                    help="keep the generator's Gaussian order instead of the engine's Morton layout")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if args.config is None:   # the keyframe batch is the workload that shards (north star)
        args.config = "C5" if world > 1 else "C3"

    import torch
    import torch.distributed as dist
    # harness check only (RTGS_BENCH_ONE_GPU=1): every rank on cuda:0 with gloo, to exercise the N > 1
    # code path on a one-GPU box; a real multi-GPU run is one process per GPU over NCCL
    one_gpu = os.environ.get("RTGS_BENCH_ONE_GPU", "") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2404_19706_b200 as P
    from paper_2404_19706_b200 import build as B
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    if args.config == "C5":
        run_batch(args, rank, world, local)
    elif args.config == "C4":
        run_render_only(args, rank, world, local)
    else:
        if world > 1:
            raise SystemExit("a single frame stays on one GPU (north star): multi-GPU runs use --config C5")
        run_mapping(args, rank, world, local)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def measure_ablation(P, eng, gm, cam, pose, col, dep, restore, flush, reps=10):
    """Table stable_gaussian_ablation on the bench's frame: time per optimisation iteration
    (device, median of `reps`, map restored and L2 flushed between iterations, outside the events) for
    (a) all Gaussians optimised over the whole image, (b) only the unstable Gaussians over the whole
    image, (c) only the unstable Gaussians over the pixels they cover (P = Eq.12 + the 50 % tiles, the
    production iteration, uncached and f3-cached).  (a) and (b): A1 + A2 + a FULL render + every pixel
    active + the backward over the Gaussians of the row + Adam over them."""
    import torch
    from paper_2404_19706_b200 import mapping as M
    stream = torch.cuda.current_stream()
    restore()
    eng.ingest(col, dep, pose)   # eager: the f3 cache (and its ready event) outside any graph capture
    eng._global_state(1)
    rb = eng.g_rb

    def full_all_pixels():
        P.project_and_bin(gm, pose, cam, eng.proj, eng.bins, eng.ws_bin)
        P.render_color_depth(gm, eng.proj, eng.bins, pose, cam, P.RTGS_RENDER_FULL, rb)
        P.topk_error_mask(rb, col, cam, 1.0, rb, eng.g_ws_topk)   # ratio 1: every pixel, every tile

    def it_all():
        full_all_pixels()
        M.render_backward_masked(gm, eng.proj, eng.bins, pose, cam, rb, col, dep, eng.weights, eng.g_slot,
                                 eng.g_gid, eng.g_grad, eng.g_loss, eng.g_ws_bwd)
        eng.global_adam_block(0, eng.g_rows, lr_scale=1.0)

    def it_unstable_all_px():
        full_all_pixels()
        M.render_backward_masked(gm, eng.proj, eng.bins, pose, cam, rb, col, dep, eng.weights, eng.slot_of_gid,
                                 eng.gid_of_slot, eng.grad, eng.loss, eng.ws_bwd)
        eng.optimizer_step()

    def it_masked(cached):
        def f():
            eng.use_cache = cached
            eng.forward_masked(pose)
            eng.backward_adam(col, dep, pose)
        return f

    out = {}
    use_cache0 = eng.use_cache
    for name, fn in (("S_all_pixels", it_all), ("S_unstable_all_pixels", it_unstable_all_px),
                     ("S_unstable_P_uncached", it_masked(False)), ("S_unstable_P", it_masked(True))):
        ts = []
        for _ in range(reps + 2):
            restore()
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name + "_ms"] = round(statistics.median(ts[2:]), 4)
    eng.use_cache = use_cache0
    restore()
    out["trend_holds"] = bool(out["S_all_pixels_ms"] > out["S_unstable_all_pixels_ms"] > out["S_unstable_P_ms"])
    out["paper_ms"] = {"Storeroom": [9.8, 7.4, 5.2], "Hotel room": [8.4, 6.5, 4.7], "Home": [8.9, 6.4, 4.3],
                       "note": "P:753-755, RTX 4090, order S / S_unstable all px / S_unstable unstable px; context"}
    return out


def c5_views(P, cfg, idx):
    """The C5 keyframe views `idx` of the C3 scene (synth.make_pose view v: +-0.3 m / 15 deg around the
    primary view), as device (colour, depth, pose) triples."""
    import torch
    from synth import make_frame, make_pose
    out = []
    for v in idx:
        R, t = make_pose(cfg, view=v)
        c, d = make_frame(cfg, (R, t))
        out.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), P.make_pose(R, t)))
    return out


N_C5_VIEWS = 64


def measure_c5_one_gpu(P, eng, cfg, restore, flush, reps=3):
    """One C5 global step (64 views, every Gaussian, one Adam step) on this GPU: the T_1 of the
    multi-GPU keyframe-batch runs (dist.global_step_sharded with one rank)."""
    import torch
    from paper_2404_19706_b200.dist import global_step_sharded
    stream = torch.cuda.current_stream()
    views = c5_views(P, cfg, range(N_C5_VIEWS))
    global_step_sharded(eng, views)  # warm: allocates the all-Gaussian state
    ts = []
    for _ in range(reps):
        restore()
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        global_step_sharded(eng, views)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = statistics.median(ts)
    del views
    return {"views": N_C5_VIEWS, "ms_per_global_step": round(t, 3), "views_per_s": round(N_C5_VIEWS * 1e3 / t, 1),
            "note": "BASELINE configs[4] at N = 1: per view FULL render + top-40 % pixels + masked backward over "
                    "all 1M Gaussians; one Adam step (position lr 0, others x 0.1); eager"}


def cpu_leg(args, cfg):
    """`cpu_baseline` of the GPU line: the oracle as it stands on the host cores, a bounded sample of
    the same step extrapolated (stated), plus the MEASURED whole C1 step (all threads / one)."""
    try:
        n_active = _oracle_active_count(cfg.name)
        k = 4 * args.ref_pixels   # ~10-30 s of oracle work at C3 (16 host threads)
        r = oracle_sample(cfg.name, k, k)
        t_step = oracle_step_seconds(r, cfg, n_active)
        out = {"value": 1.0 / t_step, "unit": "iters/s", "cores": r["threads"], "kind": "oracle",
               "extrapolated": True, "sample_fraction": r["t_sample"] / t_step,
               "sample": ORACLE_SAMPLE.format(n=cfg.n, kf=r["k_fwd"], kb=r["k_bwd"], th=r["threads"],
                                              ts=r["t_sample"], wh=cfg.width * cfg.height, p=n_active)}
        out["c1_measured"] = oracle_c1_measured()
        return out
    except Exception as e:  # report, never fake
        return {"value": None, "error": repr(e)[:200]}


def run_mapping(args, rank, world, local):
    """C3 / C2: the mapping step (ingest + one masked iteration), CUDA graph, single GPU."""
    import torch
    import torch.distributed as dist
    import paper_2404_19706_b200 as P
    from synth import CONFIGS, make_frame, make_pose, make_scene, trajectory_pose
    cfg = CONFIGS[args.config]
    scene = make_scene(cfg)
    # each rank optimises the shared map from its own keyframe view (rank 0 = the primary view)
    R, t = make_pose(cfg) if rank == 0 else make_pose(cfg, view=rank)
    col_h, dep_h = make_frame(cfg, (R, t))
    gm = P.GaussianMap.from_arrays(scene, capacity=cfg.n + 1 + cfg.width * cfg.height // 2)  # room for f2 rows
    cam = P.camera_of(cfg)
    pose = P.make_pose(R, t)
    eng = P.MappingEngine(gm, cam, capacity=4 * cfg.n)
    if not args.no_reorder:
        eng.reorder_spatially()   # the framework's map layout (rtgs_morton_order), before any timing
    eng.use_cache = not args.no_cache
    eng.fused_adam = not args.no_fuse_adam
    col = torch.as_tensor(col_h, device="cuda")
    dep = torch.as_tensor(dep_h, device="cuda")
    stream = torch.cuda.current_stream()

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    # Stationary workload: every timed step starts from the same map and optimiser state (the first
    # iteration of a window), restored outside the timed events like the L2 flush.  Without
    # this, hundreds of Adam steps on one frame drift the unstable Gaussians and change the work.
    snap = {k: getattr(gm, k).clone() for k in ("pos", "log_scale", "rot", "sh")}
    snap_eta = eng.eta.clone()

    def restore():
        for k, v in snap.items():
            getattr(gm, k).copy_(v)
        eng.m.zero_()
        eng.v.zero_()
        eng.grad.zero_()
        eng.eta.copy_(snap_eta)
        eng.step_dev.zero_()

    def between_steps():
        if not args.no_restore:
            restore()
        flush.zero_()

    def step(c, d, frame_idx):
        # ingest (side stream) || masked iteration (current stream); Adam waits for the ingest projection
        eng.step(c, d, pose, seed=1234, frame_idx=frame_idx)

    for i in range(args.warmup):
        step(col, dep, i)
    torch.cuda.synchronize()
    l_eager = P.launch_count()
    step(col, dep, args.warmup)
    torch.cuda.synchronize()
    launches_per_step = P.launch_count() - l_eager
    # CUDA graph of one whole step (both streams); the Adam step counter lives on the device, so each
    # replay is a genuine next iteration.  Eager under torchrun (NCCL inside the step).
    use_graph = (not args.no_graph) and world == 1
    graph = None
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step(col, dep, args.warmup + 1)
        torch.cuda.synchronize()

    def run_step(i):
        if graph is not None:
            graph.replay()
        else:
            step(col, dep, args.warmup + i)
    n_inst_iter0 = int(eng.bins.n_instances.item())
    n_inst = int(eng.bins_full.n_instances.item())     # full-frame instance count (ingest binning)
    if max(n_inst, n_inst_iter0) > eng.capacity:
        raise RuntimeError(f"instance capacity {eng.capacity} < {max(n_inst, n_inst_iter0)}")


    # ---- device-timed region: K steps, L2 flushed between steps (outside the events) -------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = P.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_spin = time.perf_counter()
        while time.perf_counter() - t_spin < 0.25:  # keep the GPU busy while nvidia-smi starts sampling
            run_step(0)
        torch.cuda.synchronize()
        for i in range(args.steps):
            between_steps()
            starts[i].record(stream)
            run_step(i)
            ends[i].record(stream)
        torch.cuda.synchronize()
    launches = launches_per_step * args.steps
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_step = sum(ms) / len(ms)
    if world > 1:
        tt = torch.tensor([t_step], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
        dist.barrier()

    # ---- per-call phase timing (one instrumented step, same stream) ------------------------------
    phases = {}
    if rank == 0:
        ev = {}

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            ev.setdefault(name, []).append(e)

        def hold(ms):
            # keep the GPU busy while the host enqueues the timed calls, so host-side marshalling
            # latency never lands between two events
            torch.cuda._sleep(int(ms * 2.0e6))

        between_steps()
        hold(5.0)
        mark("start")
        P.project_and_bin(gm, pose, cam, eng.proj_full, eng.bins_full, eng.ws_bin_full,
                          cache=eng.cache if eng.use_cache else None)
        mark("ingest.project_bin_cache")
        P.render_color_depth(gm, eng.proj_full, eng.bins_full, pose, cam, P.RTGS_RENDER_FULL, eng.full, normals=False); mark("ingest.render_full")
        P.classify_and_add_pixels(eng.full, col, dep, gm.flags, cam, P.add_params(seed=1234), eng.pixel_class,
                                  eng.samples, eng.add_counts, eng.ws_cls); mark("ingest.classify")
        if eng.use_cache:  # the iteration through the f3 stable cache, as eng.step runs it
            n_slots = int(eng.gid_of_slot.numel())
            P.project_subset(gm, eng.gid_of_slot, pose, cam, eng.proj_sub); mark("iter.project_subset")
            P.coverage_subset(eng.proj_sub, n_slots, cam, eng.out, eng.capacity, eng.ws_bin_cached)
            mark("iter.coverage_subset")
            P.merge_cached(eng.proj_full, eng.cache, eng.proj_sub, eng.gid_of_slot, cam, eng.out, eng.bins,
                           eng.ws_bin_cached); mark("iter.merge_cached")
            eng.proj_iter = eng.proj_full
        else:
            P.project_gaussians(gm, pose, cam, eng.proj); mark("iter.project")
            P.render_color_depth(gm, eng.proj, None, pose, cam, P.RTGS_RENDER_COVERAGE, eng.out); mark("iter.coverage")
            P.bin_and_sort(eng.proj, gm.n, cam, eng.out.tile_keep, eng.bins, eng.ws_bin); mark("iter.bin_and_sort")
            eng.bins.sub = None
            eng.proj_iter = eng.proj
        P.render_color_depth(gm, eng.proj_iter, eng.bins, pose, cam, P.RTGS_RENDER_MASKED, eng.out)
        mark("iter.render_masked")
        if eng.fused_adam:
            eng.backward_adam(col, dep, pose); mark("iter.backward_adam")
        else:
            eng.backward(col, dep, pose); mark("iter.backward")
            eng.optimizer_step(); mark("iter.adam")
        torch.cuda.synchronize()
        names = list(ev)
        for a, b in zip(names[:-1], names[1:]):
            phases[b] = ev[a][0].elapsed_time(ev[b][0])
        # project kernel alone, averaged over several launches (HBM roofline of A1)
        reps = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pt = []
        for _ in range(reps):
            flush.zero_()
            hold(0.5)
            e0.record(stream)
            P.project_gaussians(gm, pose, cam, eng.proj)
            e1.record(stream)
            torch.cuda.synchronize()
            pt.append(e0.elapsed_time(e1))
        phases["project_alone_ms"] = statistics.mean(pt)
        # the FULL render alone (dominant kernel of the step), same protocol
        rt = []
        for _ in range(reps):
            flush.zero_()
            hold(0.5)
            e0.record(stream)
            P.render_color_depth(gm, eng.proj_full, eng.bins_full, pose, cam, P.RTGS_RENDER_FULL, eng.full, normals=False)
            e1.record(stream)
            torch.cuda.synchronize()
            rt.append(e0.elapsed_time(e1))
        phases["render_full_alone_ms"] = statistics.mean(rt)
        # A2 alone (count, offsets, emission, tile sort of the full map; same lists as the ingest's)
        bt = []
        for _ in range(reps):
            flush.zero_()
            hold(0.5)
            e0.record(stream)
            P.bin_and_sort(eng.proj_full, gm.n, cam, None, eng.bins_full, eng.ws_bin_full)
            e1.record(stream)
            torch.cuda.synchronize()
            bt.append(e0.elapsed_time(e1))
        phases["bin_alone_ms"] = statistics.mean(bt)
        phases["bin_instances"] = int(eng.bins_full.n_instances.item())
        # NEXT f1 (once per window, not part of the step): Eq.9 fusion and the state transitions
        from paper_2404_19706_b200 import mapping as M
        hold(0.5)
        e0.record(stream)
        M.fuse_window(gm, eng.gid_of_slot, eng.before, eng.eta_before, eng.eta)
        e1.record(stream)
        torch.cuda.synchronize()
        phases["window.fuse_ms"] = e0.elapsed_time(e1)
        flags_keep = gm.flags.clone()
        hold(0.5)
        e0.record(stream)
        M.manage_states(eng.full, col, dep, cam, gm.flags, eng.err_count, eng.eta, eng.t_created,
                        M.state_params(1), eng.state_counts, eng.ws_state)
        e1.record(stream)
        torch.cuda.synchronize()
        phases["window.manage_states_ms"] = e0.elapsed_time(e1)
        gm.flags.copy_(flags_keep)
        # NEXT f2 (once per frame, not part of the step): insertion for this frame's A7 samples
        # (grids over the 1M existing Gaussians, exact 3-NN, Eq.11); the map is not resized after
        P.classify_and_add_pixels(eng.full, col, dep, gm.flags, cam, P.add_params(seed=1234), eng.pixel_class,
                                  eng.samples, eng.add_counts, eng.ws_cls)
        hold(0.5)
        e0.record(stream)
        eng.insert(col, dep, pose, frame_idx=1, sync=False)
        e1.record(stream)
        torch.cuda.synchronize()
        phases["frame.add_gaussians_ms"] = e0.elapsed_time(e1)
        insert_result = eng.insert_result.cpu().numpy().tolist()
        # NEXT f4 (once per frame, not part of the step): model render at the previous pose + ICP
        icp_pose = P.pose_device(R, t)
        eng.track(dep, pose, init_pose=icp_pose)   # warm (allocates the ICP workspace)
        icp_pose.copy_(P.pose_device(R, t))
        torch.cuda.synchronize()
        hold(0.5)
        e0.record(stream)
        eng.track(dep, pose, init_pose=icp_pose)
        e1.record(stream)
        torch.cuda.synchronize()
        phases["frame.track_ms"] = e0.elapsed_time(e1)
        icp_rows = eng.icp_diag.cpu().numpy().reshape(-1, 4)
        icp_rows = icp_rows[icp_rows[:, 0] >= 0]
        restore()
        # blended-pair statistic of the FULL render: one extra launch of the counting variant (the
        # timed step and render_full_alone_ms use the production kernel, which does not count)
        eng.full.count_blends = True
        P.render_color_depth(gm, eng.proj_full, eng.bins_full, pose, cam, P.RTGS_RENDER_FULL, eng.full)
        eng.out.count_blends = True   # and of the last iteration's MASKED render (same lists)
        P.render_color_depth(gm, eng.proj_iter, eng.bins, pose, cam, P.RTGS_RENDER_MASKED, eng.out)
        torch.cuda.synchronize()
        eng.full.count_blends = False
        eng.out.count_blends = False
        blends_full = int(eng.full.counts[3].item())
        blends_masked = int(eng.out.counts[3].item())
        counts_full = None
        counts = eng.out.counts.cpu().numpy().tolist()
        ninst_iter = int(eng.bins.n_instances.item())
        if args.phases:
            print(json.dumps({"phases_ms": phases, "counts": counts, "n_inst_iter": ninst_iter,
                              "n_inst_full": n_inst}), file=sys.stderr)
        _ = counts_full

    # ---- e2e: host frames in pinned memory -> device, step, loss + add counts back to the host ------
    # Streamed like a live system: the H2D copy of frame i+1 (copy stream, double-buffered staging)
    # overlaps the step of frame i; each step's copy and its D2H read-back are inside the timed span.
    # The frames arrive sensor-native (8-bit interleaved RGB, 16-bit depth at 5000 units / m, as TUM /
    # Replica store them) and are decoded on the device (rtgs_decode_rgbd) into the graph's inputs.
    n_e2e = max(20, args.steps)  # (the first frame's copy is not overlapped: amortised over >= 20)
    DEPTH_SCALE = 5000.0
    rgb_h = np.clip(np.rint(np.moveaxis(col_h, 0, -1) * 255.0), 0, 255).astype(np.uint8)
    raw_h = np.clip(np.rint(dep_h * DEPTH_SCALE), 0, 65535).astype(np.uint16)
    col_pin = torch.as_tensor(rgb_h).pin_memory()
    dep_pin = torch.as_tensor(raw_h.view(np.int16)).pin_memory()
    loss_h = torch.empty((n_e2e, 4), dtype=torch.float32).pin_memory()
    cnt_h = torch.empty((n_e2e, 5), dtype=torch.int32).pin_memory()
    st_col = [torch.empty_like(col_pin, device="cuda") for _ in range(2)]
    st_dep = [torch.empty_like(dep_pin, device="cuda") for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    ev_copied = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    # single GPU: one CUDA graph per staging buffer = decode + the whole step + the D2H read-back of
    # the step's loss and add counts (into that graph's pinned slot), so a frame costs one launch
    e2e_graphs = []
    if graph is not None:
        res_pin = [(torch.empty(4, dtype=torch.float32).pin_memory(), torch.empty(5, dtype=torch.int32).pin_memory())
                   for _ in range(2)]
        for bsel in range(2):
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2):
                P.decode_rgbd(st_col[bsel], st_dep[bsel], DEPTH_SCALE, col, dep)
                step(col, dep, args.warmup + 1)
                res_pin[bsel][0].copy_(eng.loss, non_blocking=True)
                res_pin[bsel][1].copy_(eng.add_counts, non_blocking=True)
            e2e_graphs.append(g2)
    restore()
    flush.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    copy_stream.wait_stream(stream)

    def h2d(i):
        with torch.cuda.stream(copy_stream):
            if i >= 2:
                copy_stream.wait_event(ev_free[i % 2])
            st_col[i % 2].copy_(col_pin, non_blocking=True)
            st_dep[i % 2].copy_(dep_pin, non_blocking=True)
            ev_copied[i % 2].record(copy_stream)

    h2d(0)
    for i in range(n_e2e):
        if i + 1 < n_e2e:
            h2d(i + 1)
        stream.wait_event(ev_copied[i % 2])
        if e2e_graphs:
            e2e_graphs[i % 2].replay()
            ev_free[i % 2].record(stream)
            continue
        P.decode_rgbd(st_col[i % 2], st_dep[i % 2], DEPTH_SCALE, col, dep)  # into the graph's input buffers
        ev_free[i % 2].record(stream)
        run_step(i)
        loss_h[i].copy_(eng.loss, non_blocking=True)
        cnt_h[i].copy_(eng.add_counts, non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize()
    t_e2e = a.elapsed_time(b) / n_e2e
    if world > 1:
        tt = torch.tensor([t_e2e], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())

    # ---- (e) one keyframe global-optimisation step, supplementary: latest + 3 keyframes ------
    gstep = None
    if rank == 0 and world == 1 and not args.no_window:
        kviews = []
        for v in range(4):
            Rv, tv = trajectory_pose(cfg, 3 * v)
            cv, dv = make_frame(cfg, (Rv, tv))
            kviews.append((torch.as_tensor(cv, device="cuda"), torch.as_tensor(dv, device="cuda"),
                           P.make_pose(Rv, tv)))
        restore()
        eng.global_step(kviews)            # allocates the all-Gaussian optimiser state
        restore()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        eng.global_step(kviews)
        g1.record(stream)
        torch.cuda.synchronize()
        gstep = {"views": 4, "slots": int(eng.g_gid.numel()), "ms": round(g0.elapsed_time(g1), 3),
                 "note": "4 keyframes: FULL render + top-40 % colour-error pixels + masked backward over ALL "
                         "Gaussians each, one Adam step (position lr 0, other rates x 0.1)"}
        restore()

    # ---- Table stable_gaussian_ablation trend, supplementary ---------------------------
    ablation = None
    if rank == 0 and world == 1 and not args.no_window:
        ablation = measure_ablation(P, eng, gm, cam, pose, col, dep, restore, flush)
    # ---- the C5 keyframe batch on this one GPU (the multi-GPU runs' T_1), supplementary -----------
    c5_one = None
    if rank == 0 and world == 1 and not args.no_window and args.config == "C3":
        c5_one = measure_c5_one_gpu(P, eng, cfg, restore, flush)
        restore()

    # ---- the paper's mapping window, once (supplementary; mutates the map, so it runs last) -------
    # 6 frames (Replica window): ingest + insertion each, a new slot set, 50 iterations on
    # randomly sampled window frames through the per-frame f3 caches, fusion + state management.
    window = None
    if rank == 0 and world == 1 and not args.no_window:
        frames = []
        for v in range(6):   # 6 consecutive frames of a smooth hand-held path (synth.trajectory_pose)
            Rv, tv = trajectory_pose(cfg, v)
            cv, dv = make_frame(cfg, (Rv, tv))
            frames.append((torch.as_tensor(cv, device="cuda"), torch.as_tensor(dv, device="cuda"), P.make_pose(Rv, tv)))
        restore()
        eng.cache_frames = len(frames)
        # a first window allocates the per-frame caches and grows the map; the second one is timed
        eng.map_window(frames, iterations=50, seed=3, first_frame_idx=10)
        torch.cuda.synchronize()
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_before = gm.n
        t_wins = []
        for rep in range(3):   # the median of three windows (the eager window has rare host outliers)
            w0.record(stream)
            eng.map_window(frames, iterations=50, seed=4 + rep, first_frame_idx=16 + 6 * rep)
            w1.record(stream)
            torch.cuda.synchronize()
            t_wins.append(w0.elapsed_time(w1))
        t_win = statistics.median(t_wins)
        window = {"frames": len(frames), "iterations": 50, "ms": round(t_win, 3),
                  "ms_each": [round(x, 3) for x in t_wins],
                  "mapping_iters_per_s": round(50 * 1e3 / t_win, 1), "gaussians_added": (gm.n - n_before) // 3,
                  "slots": int(eng.gid_of_slot.numel()),
                  "note": "median of windows 2-4 of a smooth 6-frame path: 6 ingests + insertions (host syncs), a new slot "
                          "set, 50 cached iterations on sampled window frames, fusion + states; eager calls, "
                          "span on the device clock; the inserted unstable Gaussians enlarge the masked work"}

    if rank == 0:
        hbm, sm_max, peak_kind = _peaks()
        clocks = clk.summary()
        clk_sm_mhz = clocks.get("sm_mhz")
        K = (cfg.sh_degree + 1) ** 2
        # A1 algorithmic bytes per visible Gaussian: read pos 12, log_scale 12, rot 16, opacity 4, SH 12K,
        # write rec 64, zkey 4, rect 8, tiles_touched 4
        bytes_per_g = 12 + 12 + 16 + 4 + 12 * K + 64 + 4 + 8 + 4
        t_proj_s = phases["project_alone_ms"] * 1e-3
        achieved = bytes_per_g * cfg.n / t_proj_s / 1e9
        # A3/A4 (dominant kernel): 16 FP32 instructions per blended (pixel, Gaussian) pair;
        # peak = FP32 issue of 148 SMs x 128 lanes x the sampled SM clock (1 instruction / lane / clock)
        t_render_s = phases["render_full_alone_ms"] * 1e-3
        traffic = {}
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get(cfg.name, {})  # ncu counts of this workload, if captured
        clk_ghz = (clk_sm_mhz or sm_max) * 1e-3
        alu_peak = 148 * 128 * clk_ghz * 1e9 / 1e12
        alu_achieved = 16 * blends_full / t_render_s / 1e12
        value = world * 1e3 / t_step
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": mapping_config(cfg, eng.use_cache,
                                     "CUDA graph of the whole step (2 streams)" if graph is not None else "eager", world),
            "roofline": {"kernel": "k_render_fwd<FULL> (A3/A4, dominant kernel of the step)", "bound": "alu",
                         "achieved": alu_achieved, "peak": alu_peak, "unit": "TFLOP/s", "frac": alu_achieved / alu_peak,
                         "traffic": traffic.get("k_render_fwd<FULL>"), "peak_kind": "derived: 148 SM x 128 FP32 lanes x sampled SM clock",
                         "algorithmic": f"16 FP32 instr x {blends_full} blends per launch",
                         "time_ms": phases["render_full_alone_ms"]},
            "roofline_secondary": [{"kernel": "k_project (A1)", "bound": "hbm", "achieved": achieved, "peak": hbm,
                                    "unit": "GB/s", "frac": achieved / hbm, "peak_kind": peak_kind,
                                    "traffic": traffic.get("k_project"),
                                    "bytes_per_gaussian": bytes_per_g, "time_ms": phases["project_alone_ms"],
                                    # the measured peak is a device copy (half reads, half writes); this
                                    # stream is 76 % reads, which HBM serves faster, so also against the
                                    # nominal 7.7 TB/s (B200_PROFILING.md)
                                    "peak_nominal": 7700.0, "frac_nominal": achieved / 7700.0}]
            + ([{"kernel": "k_render_fwd<FULL> (A3/A4)", "bound": "issue",
                 "achieved": traffic["k_render_fwd<FULL>_warp_inst"] / t_render_s / 1e12,
                 "peak": 4 * 148 * clk_ghz * 1e9 / 1e12, "unit": "T warp-instr/s",
                 "frac": traffic["k_render_fwd<FULL>_warp_inst"] / t_render_s / (4 * 148 * clk_ghz * 1e9),
                 "peak_kind": "derived: 4 issue slots / clock / SM x 148 SM x sampled SM clock",
                 "algorithmic": "warp instructions executed per launch (ncu smsp__inst_executed.sum, profiles/traffic.json)",
                 "time_ms": phases["render_full_alone_ms"]}] if "k_render_fwd<FULL>_warp_inst" in traffic else [])
            + ([_a2_roofline(cfg, phases["bin_instances"], phases["bin_alone_ms"], hbm, peak_kind)]
               if "bin_alone_ms" in phases else []),
            "blends": {"full_per_frame": blends_full, "masked_per_iter": blends_masked,
                       "full_blends_per_s": blends_full / t_render_s},
            "clocks": clocks,
            "gpu_launches": int(launches),
            "e2e": {"value": world * 1e3 / t_e2e, "unit": "iters/s",
                    "h2d_bytes_per_step": int(rgb_h.nbytes + raw_h.nbytes), "d2h_bytes_per_step": 4 * 4 + 5 * 4,
                    "input": "uint8 RGB + uint16 depth (5000 / m), decoded on the device"},
            "phases_ms": {k: round(v, 4) for k, v in phases.items()},
            "iter_ms": round(sum(v for k, v in phases.items() if k.startswith("iter.")), 4),
            "ingest_ms": round(sum(v for k, v in phases.items() if k.startswith("ingest.")), 4),
            "window": window,
            "global_step": gstep,
            "f4_track": {"ms": round(phases["frame.track_ms"], 4), "in_step": False,
                         "gn_iterations": int(len(icp_rows)), "pairs_last": int(icp_rows[-1][2]) if len(icp_rows) else 0},
            "f2_insert": {"result": dict(zip(["opaque", "transparent", "skipped", "dropped", "n_after"], insert_result)),
                          "ms": round(phases["frame.add_gaussians_ms"], 4), "in_step": False},
            "active": {"kept_tiles": counts[0], "active_px": counts[1], "instances_full": n_inst,
                       "instances_iter": ninst_iter},
        }
        line["ablation"] = ablation
        line["c5_one_gpu"] = c5_one
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_leg(args, cfg)
        print(json.dumps(line), flush=True)


def _timed(run_step, between, steps, world, local, stream):
    """W-excluded timed region: barrier + synchronize on both sides, CUDA events on `stream` around
    each step, `between()` (map restore, L2 flush) outside the events; mean step ms, max over ranks;
    nvidia-smi clocks sampled during the region."""
    import torch
    import torch.distributed as dist
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        # keep the GPU busy while nvidia-smi starts sampling; with collectives in the step every rank
        # must run the same number of steps, so a fixed count there
        if world > 1:
            for _ in range(5):
                run_step(0)
        else:
            t_spin = time.perf_counter()
            while time.perf_counter() - t_spin < 0.25:
                run_step(0)
        torch.cuda.synchronize()
        for i in range(steps):
            between()
            starts[i].record(stream)
            run_step(i)
            ends[i].record(stream)
        torch.cuda.synchronize()
    t = statistics.mean(s.elapsed_time(e) for s, e in zip(starts, ends))
    if world > 1:
        tt = torch.tensor([t], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        dist.barrier()
    return t, clk.summary()


def _a2_roofline(cfg, instances, t_ms, hbm, peak_kind):
    """A2 (count, offsets, emission, tile sort) against HBM with SURVEY 8(d.3)'s compulsory bytes:
    16 B per Gaussian + 4 B per instance + 8 B per tile (all Gaussians counted as visible: an upper
    bound on the compulsory bytes, so a lower bound on nothing)."""
    T = ((cfg.width + 15) // 16) * ((cfg.height + 15) // 16)
    byts = 16 * cfg.n + 4 * instances + 8 * T
    ach = byts / (t_ms * 1e-3) / 1e9
    return {"kernel": "A2 bin_and_sort (k_tile_count, k_tile_offsets, k_emit, k_tile_sort)", "bound": "hbm",
            "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "peak_kind": peak_kind,
            "algorithmic": f"16 B x {cfg.n} Gaussians + 4 B x {instances} instances + 8 B x {T} tiles",
            "time_ms": t_ms, "keys_per_s": instances / (t_ms * 1e-3)}


def _alu_roofline(blends, t_ms, clocks, what):
    sm_mhz = clocks.get("sm_mhz") or _peaks()[1]
    peak = 148 * 128 * sm_mhz * 1e-3 * 1e9 / 1e12
    ach = 16 * blends / (t_ms * 1e-3) / 1e12
    return {"kernel": what, "bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "traffic": None, "peak_kind": "derived: 148 SM x 128 FP32 lanes x sampled SM clock",
            "algorithmic": f"16 FP32 instr x {blends} blends per launch", "time_ms": t_ms}


def run_render_only(args, rank, world, local):
    """C4 (BASELINE configs[3]): render-only novel views of the ScanNet++-shaped 4M-Gaussian map: per
    step A1 project + A2 bin + A3/A4 FULL render (colour, T, depth, index, normals) at the next of 8
    novel poses, one CUDA graph per pose.  value = frames/s (per GPU; replicas under torchrun)."""
    import torch
    import paper_2404_19706_b200 as P
    from paper_2404_19706_b200 import mapping as M
    from synth import CONFIGS, make_pose, make_scene
    cfg = CONFIGS["C4"]
    scene = make_scene(cfg)
    gm = P.GaussianMap.from_arrays(scene)
    if not args.no_reorder:
        gm.permute(P.morton_order(gm))   # the framework's map layout, before any timing
    cam = P.camera_of(cfg)
    poses = [P.make_pose(*make_pose(cfg, view=v)) for v in range(8)]
    n, cap = gm.n, 3 * cfg.n
    proj, bins = M.ProjectedBuffers(n), M.BinBuffers(cam, cap)
    ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
    rb = M.RenderBuffers(cam, count_blends=False)
    rb.track_last = False
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def frame(k):
        P.project_and_bin(gm, poses[k % len(poses)], cam, proj, bins, ws)
        P.render_color_depth(gm, proj, bins, poses[k % len(poses)], cam, P.RTGS_RENDER_FULL, rb)

    for k in range(max(args.warmup, len(poses))):
        frame(k)
    torch.cuda.synchronize()
    worst = int(bins.n_instances.item())
    if worst > cap:
        raise RuntimeError(f"instance capacity {cap} < {worst}")
    l0 = P.launch_count()
    frame(0)
    torch.cuda.synchronize()
    per_frame = P.launch_count() - l0
    graphs = []
    for k in range(len(poses)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            frame(k)
        graphs.append(g)
    torch.cuda.synchronize()
    t_step, clocks = _timed(lambda i: graphs[i % len(graphs)].replay(), lambda: flush.zero_(), args.steps, world,
                            local, stream)
    # the FULL render alone + its blend count (counting variant, one extra launch), on pose 0
    frame(0)
    rt = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        P.render_color_depth(gm, proj, bins, poses[0], cam, P.RTGS_RENDER_FULL, rb)
        e1.record(stream)
        torch.cuda.synchronize()
        rt.append(e0.elapsed_time(e1))
    t_render = statistics.mean(rt)
    # A1 alone (the plain projection), for its HBM roofline
    pt = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        P.project_gaussians(gm, poses[0], cam, proj)
        e1.record(stream)
        torch.cuda.synchronize()
        pt.append(e0.elapsed_time(e1))
    t_proj = statistics.mean(pt)
    P.project_gaussians(gm, poses[0], cam, proj)
    bt = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        P.bin_and_sort(proj, n, cam, None, bins, ws)
        e1.record(stream)
        torch.cuda.synchronize()
        bt.append(e0.elapsed_time(e1))
    t_bin = statistics.mean(bt)
    bin_inst = int(bins.n_instances.item())
    rb.count_blends = True
    P.project_and_bin(gm, poses[0], cam, proj, bins, ws)
    P.render_color_depth(gm, proj, bins, poses[0], cam, P.RTGS_RENDER_FULL, rb)
    torch.cuda.synchronize()
    blends = int(rb.counts[3].item())
    rb.count_blends = False
    # e2e through the public API: pose in (host struct, by value), colour + depth image read back to
    # pinned host memory every frame.  Streamed like a viewer: two render targets; frame i's read-back
    # (copy stream) overlaps frame i+1's render, and a target is rendered into again only after its
    # previous read-back has landed.  Every frame's render and its D2H copy are inside the timed span.
    rbs = [rb, M.RenderBuffers(cam, count_blends=False)]
    rbs[1].track_last = False
    col_h = [torch.empty((3, cam.height, cam.width), dtype=torch.float32).pin_memory() for _ in range(2)]
    dep_h = [torch.empty((cam.height, cam.width), dtype=torch.float32).pin_memory() for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    ev_rendered = [torch.cuda.Event() for _ in range(2)]
    ev_read = [torch.cuda.Event() for _ in range(2)]
    n_e2e = max(20, args.steps)  # (the last frame's copy is not overlapped: amortised over >= 20)
    flush.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    copy_stream.wait_stream(stream)
    for i in range(n_e2e):
        s = i % 2
        if i >= 2:
            stream.wait_event(ev_read[s])  # the target's previous frame has been read back
        P.project_and_bin(gm, poses[i % len(poses)], cam, proj, bins, ws)
        P.render_color_depth(gm, proj, bins, poses[i % len(poses)], cam, P.RTGS_RENDER_FULL, rbs[s])
        ev_rendered[s].record(stream)
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(ev_rendered[s])
            col_h[s].copy_(rbs[s].color, non_blocking=True)
            dep_h[s].copy_(rbs[s].depth, non_blocking=True)
            ev_read[s].record(copy_stream)
    stream.wait_stream(copy_stream)
    b.record(stream)
    torch.cuda.synchronize()
    t_e2e = a.elapsed_time(b) / n_e2e
    if rank == 0:
        hbm, _, peak_kind = _peaks()
        K = (cfg.sh_degree + 1) ** 2
        a1_bytes = 12 + 12 + 16 + 4 + 12 * K + 64 + 4 + 8 + 4  # as the C3 line
        a1_gbs = a1_bytes * cfg.n / (t_proj * 1e-3) / 1e9
        traffic = {}
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get("C4", {})
        line = {"metric": METRIC, "value": world * 1e3 / t_step, "unit": "frames/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": (f"C4 ScanNet++-shaped {cfg.width}x{cfg.height}, {cfg.n} Gaussians (10% "
                                        f"transparent), SH deg {cfg.sh_degree}; step = render-only novel view: A1 "
                                        f"project + A2 bin + A3/A4 FULL render (C, T, D, I, N) at one of 8 novel poses"),
                           "l2": "flushed between timed steps (256 MB write); Gaussian SoA 948 MB > L2",
                           "launch": "CUDA graph per pose", "parallelism": "single GPU" if world == 1 else
                           f"{world} replicas"},
                "roofline": dict(_alu_roofline(blends, t_render, clocks, "k_render_fwd<FULL> (A3/A4, dominant kernel)"),
                                 traffic=traffic.get("k_render_fwd<FULL>")),
                "roofline_secondary": [{"kernel": "k_project (A1)", "bound": "hbm", "achieved": a1_gbs, "peak": hbm,
                                        "unit": "GB/s", "frac": a1_gbs / hbm, "peak_kind": peak_kind,
                                        "traffic": traffic.get("k_project"), "bytes_per_gaussian": a1_bytes,
                                        "time_ms": t_proj,
                                        # 76 % reads: above the measured copy (half reads), so also against
                                        # the nominal 7.7 TB/s (B200_PROFILING.md)
                                        "peak_nominal": 7700.0, "frac_nominal": a1_gbs / 7700.0},
                                       _a2_roofline(cfg, bin_inst, t_bin, hbm, peak_kind)],
                "blends": {"full_per_frame": blends, "full_blends_per_s": blends / (t_render * 1e-3)},
                "clocks": clocks, "gpu_launches": int(per_frame * args.steps),
                "e2e": {"value": world * 1e3 / t_e2e, "unit": "frames/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": int(col_h[0].nbytes + dep_h[0].nbytes),
                        "note": "the pose enters by value in the call (host struct, 96 B); the rendered colour + "
                                "depth image is read back to pinned host memory every frame (two render "
                                "targets: frame i's read-back overlaps frame i+1's render)"},
                "instances": worst}
        if world == 1 and not args.no_cpu_baseline:
            try:
                r = oracle_sample("C4", args.ref_pixels, 1)
                t_cpu = r["t_proj"] + r["t_fwd"] * cfg.width * cfg.height / r["k_fwd"]
                line["cpu_baseline"] = {"value": 1.0 / t_cpu, "unit": "frames/s", "cores": r["threads"],
                                        "kind": "oracle", "extrapolated": True,
                                        "sample": f"projection of all {cfg.n} Gaussians + forward render of "
                                                  f"{r['k_fwd']} pixels (float64 torch CPU), extrapolated to the "
                                                  f"{cfg.width * cfg.height} pixels of a frame"}
            except Exception as e:
                line["cpu_baseline"] = {"value": None, "error": repr(e)[:200]}
        print(json.dumps(line), flush=True)


def run_batch(args, rank, world, local):
    """C5 (BASELINE configs[4]): the keyframe batch of 64 C3 views over `world` ranks
    (dist.global_step_sharded).  value = views/s of the whole job (64 / step time, max over ranks);
    T_1 / (N T_N) from the same step on rank 0 alone, measured in this run."""
    import torch
    import torch.distributed as dist
    import paper_2404_19706_b200 as P
    from paper_2404_19706_b200.dist import global_step_sharded, view_partition
    from synth import CONFIGS, make_frame, make_pose, make_scene
    cfg = CONFIGS["C3"]
    scene = make_scene(cfg)
    gm = P.GaussianMap.from_arrays(scene)
    cam = P.camera_of(cfg)
    eng = P.MappingEngine(gm, cam, capacity=4 * cfg.n)
    if not args.no_reorder:
        eng.reorder_spatially()   # the framework's map layout, before any timing
    mine = view_partition(N_C5_VIEWS, world, rank)
    views = [None] * N_C5_VIEWS
    for v, tr in zip(mine, c5_views(P, cfg, mine)):
        views[v] = tr
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def step(_i=0):
        global_step_sharded(eng, views)

    step()   # allocates the all-Gaussian optimiser state (padded for `world` blocks)
    torch.cuda.synchronize()
    keys = ("pos", "log_scale", "rot", "sh")
    snap = {k: gm.store[k].clone() for k in keys}
    snap_eta = eng._state_store["eta"].clone()

    def restore():
        for k in keys:
            gm.store[k].copy_(snap[k])
        eng._state_store["eta"].copy_(snap_eta)

    def between():
        restore()
        flush.zero_()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l0 = P.launch_count()
    step()
    torch.cuda.synchronize()
    launches = (P.launch_count() - l0) * args.steps
    t_step, clocks = _timed(step, between, args.steps, world, local, stream)
    # e2e: this rank's views arrive from pinned host memory every step, sensor-native (8-bit RGB +
    # 16-bit depth at 5000 / m), decoded on the device into the views' buffers; loss read back
    DEPTH_SCALE = 5000.0
    host = []
    for v in mine:
        R, t = make_pose(cfg, view=v)
        c, d = make_frame(cfg, (R, t))
        host.append((torch.as_tensor(np.clip(np.rint(np.moveaxis(c, 0, -1) * 255), 0, 255).astype(np.uint8)).pin_memory(),
                     torch.as_tensor(np.clip(np.rint(d * DEPTH_SCALE), 0, 65535).astype(np.uint16).view(np.int16)).pin_memory()))
    # streamed: the H2D copies of step i+1's views (copy stream, double-buffered sensor-native staging)
    # overlap step i; step i+1 decodes its staging into the views' buffers once step i is done with them
    stage = [[(torch.empty_like(hc, device="cuda"), torch.empty_like(hd, device="cuda")) for hc, hd in host]
             for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    ev_copied = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    loss_h = torch.empty(4, dtype=torch.float32).pin_memory()
    n_e2e = max(3, args.steps // 4)  # (the first step's copies are not overlapped)
    restore()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    copy_stream.wait_stream(stream)

    def h2d(i):
        with torch.cuda.stream(copy_stream):
            if i >= 2:
                copy_stream.wait_event(ev_free[i % 2])
            for (hc, hd), (sc, sd) in zip(host, stage[i % 2]):
                sc.copy_(hc, non_blocking=True)
                sd.copy_(hd, non_blocking=True)
            ev_copied[i % 2].record(copy_stream)

    h2d(0)
    for i in range(n_e2e):
        if i + 1 < n_e2e:
            h2d(i + 1)
        stream.wait_event(ev_copied[i % 2])
        for (sc, sd), v in zip(stage[i % 2], mine):
            P.decode_rgbd(sc, sd, DEPTH_SCALE, views[v][0], views[v][1])
        ev_free[i % 2].record(stream)
        step()
        loss_h.copy_(eng.g_loss, non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize()
    t_e2e = a.elapsed_time(b) / n_e2e
    if world > 1:
        tt = torch.tensor([t_e2e], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    # T_1: rank 0 runs the whole 64-view batch alone (the others wait at the barrier)
    t1 = None
    per_view = {}
    blends = None
    if rank == 0:
        restore()
        allv = [views[v] if views[v] is not None else None for v in range(N_C5_VIEWS)]
        missing = [v for v in range(N_C5_VIEWS) if allv[v] is None]
        for v, tr in zip(missing, c5_views(P, cfg, missing)):
            allv[v] = tr
        global_step_sharded(eng, allv, world=1, rank=0)   # allocates the one-rank layout
        torch.cuda.synchronize()
        t1, _ = _timed(lambda i: global_step_sharded(eng, allv, world=1, rank=0), between, max(2, args.steps // 4),
                       1, local, stream)
        # per-view phases (view 0) and the dominant kernel's blend count
        from paper_2404_19706_b200 import mapping as M
        c0, d0, p0 = allv[0]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        restore()
        flush.zero_()
        torch.cuda.synchronize()
        ev[0].record(stream)
        P.project_and_bin(gm, p0, cam, eng.proj, eng.bins, eng.ws_bin)
        ev[1].record(stream)
        P.render_color_depth(gm, eng.proj, eng.bins, p0, cam, P.RTGS_RENDER_FULL, eng.g_rb)
        ev[2].record(stream)
        P.topk_error_mask(eng.g_rb, c0, cam, 0.4, eng.g_rb, eng.g_ws_topk)
        ev[3].record(stream)
        w = tuple(x / N_C5_VIEWS for x in eng.weights[:2]) + (eng.weights[2],)
        M.render_backward_masked(gm, eng.proj, eng.bins, p0, cam, eng.g_rb, c0, d0, w, eng.g_slot, eng.g_gid,
                                 eng.g_grad, eng.g_loss, eng.g_ws_bwd)
        ev[4].record(stream)
        torch.cuda.synchronize()
        for k, name in enumerate(("project_bin", "render_full", "topk", "backward_all_gaussians")):
            per_view[name] = round(ev[k].elapsed_time(ev[k + 1]), 4)
        eng.g_grad.zero_()
        eng.g_rb.count_blends = True
        P.render_color_depth(gm, eng.proj, eng.bins, p0, cam, P.RTGS_RENDER_FULL, eng.g_rb)
        torch.cuda.synchronize()
        blends = int(eng.g_rb.counts[3].item())
        eng.g_rb.count_blends = False
        restore()
    if world > 1:
        dist.barrier()
    if rank == 0:
        views_s = N_C5_VIEWS * 1e3 / t_step
        line = {"metric": METRIC, "value": views_s, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": batch_config(cfg, world),
                "global_steps_per_s": 1e3 / t_step,
                "scaling_measured": {"t1_ms": t1, "tN_ms": t_step, "efficiency": (t1 / (world * t_step)) if t1 else None,
                                     "note": "T_1 = the same 64-view step on rank 0 alone, this run"},
                "per_view_ms": per_view,
                "roofline": _alu_roofline(blends, per_view.get("render_full", float("nan")), clocks,
                                          "k_render_fwd<FULL> (A3/A4 of a view)") if blends else None,
                "clocks": clocks, "gpu_launches": int(launches),
                "e2e": {"value": N_C5_VIEWS * 1e3 / t_e2e, "unit": "iters/s",
                        "h2d_bytes_per_step": int(sum(h[0].nbytes + h[1].nbytes for h in host)),
                        "d2h_bytes_per_step": 16,
                        "input": "per rank: its views' uint8 RGB + uint16 depth, decoded on the device"}}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
