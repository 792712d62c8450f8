#!/usr/bin/env python
"""Benchmark of the RTG-SLAM mapping hot path on B200 (contract: DESIGN.md §7).

One STEP = one pass of every §8(a) row over one synthetic C3 (Replica-shaped, 1200x680, 1M Gaussians,
10 % unstable) frame:
    ingest     A1 project -> A2 bin (all tiles) -> A3/A4 FULL render -> A7 classify + sample
    iteration  A1 project -> A0 coverage + tile keep -> A2 bin (kept tiles) -> A3/A4 MASKED render
               -> A5 masked backward -> [N>1: NCCL all-reduce of the slot gradients] -> A6 Adam
`value` counts one mapping iteration per step (each step also carries a full frame ingest, so it is
conservative w.r.t. the paper's 'mapping / iteration').

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
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


def cpu_baseline(cfg_name: str, n_pixels: int = 48, seed: int = 0):
    """The oracle (float64 CPU, as it stands) on a bounded sample of the same workload: projection of
    ALL Gaussians + render and autograd backward of `n_pixels` active pixels; extrapolated linearly in
    the active-pixel count to one full mapping iteration."""
    import torch
    from oracle import projection as OP, raster as OR
    cfg, scene, R, t, (col, dep) = _scene(cfg_name)
    cam = OP.camera(cfg)
    threads = torch.get_num_threads()
    t0 = time.perf_counter()
    prm = OP.params_from_scene(scene, requires_grad=True)
    proj = OP.project(prm, R, t, cam, scene["sh_degree"])
    t_proj = time.perf_counter() - t0
    # active pixels of the slab: sample among pixels covered by unstable Gaussians (right border)
    rng = np.random.default_rng(seed)
    u = scene["u_img"][(scene["flags"] & 2) == 0]
    x_lo = int(np.percentile(u, 5))
    px = rng.integers(max(x_lo, 0), cfg.width, n_pixels)
    py = rng.integers(0, cfg.height, n_pixels)
    pix = np.stack([px, py], 1)
    t1 = time.perf_counter()
    with torch.no_grad():
        OR.render_pixels(proj, pix, cam, R, chunk=4, want_margin=False)
    t_fwd = time.perf_counter() - t1
    t1 = time.perf_counter()
    out = OR.render_pixels(proj, pix, cam, R, chunk=4, want_margin=False)
    Ct = torch.as_tensor(col[:, py, px].T.astype(np.float64))
    L = (out["color"] - Ct).abs().sum() / (3.0 * n_pixels)
    L.backward()
    t_pix = time.perf_counter() - t1
    # |P| of the C3 iteration ~ the slab share of the image (measured by the GPU arm and passed in)
    return dict(t_proj=t_proj, t_fwd=t_fwd, t_pix=t_pix, n_pixels=n_pixels, threads=threads)


def oracle_step_seconds(r, cfg, n_active):
    """The oracle doing the bench's step: ingest (projection of all Gaussians + forward render of every
    pixel) + one uncached mapping iteration (projection again + render/backward of the active pixels)."""
    n = r["n_pixels"]
    return 2.0 * r["t_proj"] + r["t_fwd"] * cfg.width * cfg.height / n + r["t_pix"] * n_active / n


ORACLE_SAMPLE = ("projection of all {n} Gaussians + forward render of {k} pixels + render/backward of {k} "
                 "active pixels (float64 torch CPU), extrapolated to the step: 2 projections + forward of all "
                 "{wh} pixels + render/backward of |P| = {p} active pixels")


def workload_name(cfg, cached=True):
    head = (f"{cfg.name} Replica-shaped {cfg.width}x{cfg.height}, {cfg.n} Gaussians (10% transparent), "
            f"{int(cfg.frac_unstable * 100)}% unstable slab, SH deg {cfg.sh_degree}; ")
    if cached:
        return head + ("step = frame ingest (A1,A2,A3/A4 FULL,A7, f3 stable cache) + one masked mapping "
                       "iteration (A1 on the unstable slots,A0,A2 merged with the cache,A3/A4,A5,A6)")
    return head + "step = frame ingest (A1,A2,A3/A4 FULL,A7) + one masked mapping iteration (A1,A0,A2,A3/A4,A5,A6)"


def reference_arm(args, rank, world):
    """--impl reference: the oracle timed on the host cores (rank 0 only), bounded sample per step."""
    if rank != 0:
        return
    from synth import CONFIGS
    cfg = CONFIGS[args.config]
    # |P| of the C3 step as the GPU arm measures it (bench line `active.active_px`), else 12 % of the image
    n_active = args.active_pixels or (83249 if args.config == "C3" else int(0.12 * cfg.width * cfg.height))
    times = []
    for s in range(args.warmup + args.steps):
        r = cpu_baseline(args.config, n_pixels=args.ref_pixels, seed=s)
        t_iter = oracle_step_seconds(r, cfg, n_active)
        if s >= args.warmup:
            times.append(t_iter)
    t = statistics.mean(times)
    v = 1.0 / t
    line = {"metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "l2": "n/a (CPU)"},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": r["threads"], "kind": "oracle",
                             "sample": ORACLE_SAMPLE.format(n=cfg.n, k=args.ref_pixels, wh=cfg.width * cfg.height,
                                                            p=n_active)},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-pixels", type=int, default=24)
    ap.add_argument("--active-pixels", type=int, default=0)
    ap.add_argument("--phases", action="store_true", help="print per-call timings to stderr")
    ap.add_argument("--no-graph", action="store_true", help="launch every step eagerly (no CUDA graph)")
    ap.add_argument("--no-cache", action="store_true", help="iteration without the f3 stable-projection cache")
    ap.add_argument("--no-fuse-adam", action="store_true", help="separate A5 backward and A6 Adam calls")
    ap.add_argument("--no-restore", action="store_true", help="diagnostic: let the map drift between timed steps")
    ap.add_argument("--no-window", action="store_true", help="skip the supplementary mapping-window measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2404_19706_b200 as P
    from paper_2404_19706_b200 import build as B
    from paper_2404_19706_b200.dist import allreduce_grads
    from synth import CONFIGS, make_frame, make_pose, make_scene, trajectory_pose
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    cfg = CONFIGS[args.config]
    scene = make_scene(cfg)
    # each rank optimises the shared map from its own keyframe view (rank 0 = the primary view)
    R, t = make_pose(cfg) if rank == 0 else make_pose(cfg, view=rank)
    col_h, dep_h = make_frame(cfg, (R, t))
    gm = P.GaussianMap.from_arrays(scene, capacity=cfg.n + 1 + cfg.width * cfg.height // 2)  # room for f2 rows
    cam = P.camera_of(cfg)
    pose = P.make_pose(R, t)
    eng = P.MappingEngine(gm, cam, capacity=4 * cfg.n)
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
        eng.step(c, d, pose, seed=1234, frame_idx=frame_idx, reduce_grads=allreduce_grads if world > 1 else None)

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
    n_e2e = max(10, args.steps // 2)
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
            "config": {"workload": workload_name(cfg, eng.use_cache),
                       "l2": "flushed between timed steps (256 MB write); Gaussian SoA 237 MB > L2",
                       "launch": "CUDA graph of the whole step (2 streams)" if graph is not None else "eager",
                       "parallelism": f"dp{world} over keyframe views" if world > 1 else "single GPU"},
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
                 "time_ms": phases["render_full_alone_ms"]}] if "k_render_fwd<FULL>_warp_inst" in traffic else []),
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
        if world == 1 and not args.no_cpu_baseline:
            try:
                r = cpu_baseline(args.config, n_pixels=args.ref_pixels)
                t_cpu = oracle_step_seconds(r, cfg, max(counts[1], 1))
                line["cpu_baseline"] = {"value": 1.0 / t_cpu, "unit": "iters/s", "cores": r["threads"], "kind": "oracle",
                                        "sample": ORACLE_SAMPLE.format(n=cfg.n, k=r["n_pixels"], wh=cfg.width * cfg.height,
                                                                       p=counts[1])}
            except Exception as e:  # report, never fake
                line["cpu_baseline"] = {"value": None, "error": repr(e)[:200]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
