"""Experiment: does prioritising the ingest chain (side stream) shorten the two-stream step graph
(--prio; it did not: stream or node priorities changed nothing), and what does the MASKED render's
blend statistic cost inside the step (default)?
Variants: torch-instantiated graph (stream priorities ignored inside a graph launch) vs a graph
instantiated with cudaGraphInstantiateFlagUseNodePriority (per-node priorities captured from the
streams).  C3, L2 flushed between timed steps."""
import json
import sys

import numpy as np
import torch
from cuda.bindings import runtime as rt

sys.path.insert(0, ".")
import paper_2404_19706_b200 as P  # noqa: E402
from synth import CONFIGS, make_frame, make_pose, make_scene  # noqa: E402


def run(prio, node_prio, steps=150, count_masked=False):
    cfg = CONFIGS["C3"]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    col, dep = make_frame(cfg, (R, t))
    gm = P.GaussianMap.from_arrays(scene, capacity=cfg.n + cfg.width * cfg.height // 2)
    eng = P.MappingEngine(gm, P.camera_of(cfg), capacity=4 * cfg.n)
    eng.side = torch.cuda.Stream(priority=prio)
    eng.out.count_blends = count_masked
    col = torch.as_tensor(col, device="cuda")
    dep = torch.as_tensor(dep, device="cuda")
    pose = P.make_pose(R, t)
    for i in range(4):
        eng.step(col, dep, pose, seed=1, frame_idx=i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(keep_graph=True)
    with torch.cuda.graph(g):
        eng.step(col, dep, pose, seed=1, frame_idx=5)
    torch.cuda.synchronize()
    if node_prio:
        raw = g.raw_cuda_graph()
        err, exe = rt.cudaGraphInstantiateWithFlags(
            rt.cudaGraph_t(init_value=raw), rt.cudaGraphInstantiateFlags.cudaGraphInstantiateFlagUseNodePriority)
        assert err == rt.cudaError_t.cudaSuccess, err

        def launch():
            (e,) = rt.cudaGraphLaunch(exe, torch.cuda.current_stream().cuda_stream)
            assert e == rt.cudaError_t.cudaSuccess, e
    else:
        g.instantiate()
        launch = g.replay
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(20):
        launch()
    torch.cuda.synchronize()
    ms = []
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(steps):
        flush.zero_()
        s0.record()
        launch()
        s1.record()
        s1.synchronize()
        ms.append(s0.elapsed_time(s1))
    return float(np.mean(ms)), float(np.median(ms))


def main():
    out = {}
    variants = [("count", 0, False, True), ("nocount", 0, False, False)] * 3
    if "--prio" in sys.argv:
        variants = [("default", 0, False, False), ("side_hi_torch", -1, False, False),
                    ("side_hi_nodeprio", -1, True, False), ("side_lo_nodeprio", 0, True, False)]
    for i, (name, prio, node, cnt) in enumerate(variants):
        name = f"{name}{i}"
        out[name] = run(prio, node, count_masked=cnt)
        print(name, out[name], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
