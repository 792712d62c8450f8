"""Experiment: does launching the kept tiles heaviest-first shorten the masked forward / backward?
Prints per-kept-tile work statistics and kernel times for the coverage order vs a sorted order."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2404_19706_b200 as P  # noqa: E402
from synth import CONFIGS, make_frame, make_pose, make_scene  # noqa: E402


def main():
    cfg = CONFIGS["C3"]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    col, dep = make_frame(cfg, (R, t))
    gm = P.GaussianMap.from_arrays(scene)
    cam = P.camera_of(cfg)
    pose = P.make_pose(R, t)
    eng = P.MappingEngine(gm, cam, capacity=4 * cfg.n)
    col = torch.as_tensor(col, device="cuda")
    dep = torch.as_tensor(dep, device="cuda")
    eng.ingest(col, dep, pose)
    eng.forward_masked(pose)
    torch.cuda.synchronize()
    nk = int(eng.out.counts[0].item())
    tl = eng.out.tile_list[:nk].clone()
    rng = eng.bins.tile_range.cpu().numpy()
    cnt = (rng[:, 1] - rng[:, 0])[tl.cpu().numpy()]
    act = eng.out.active_set().cpu().numpy()
    H, W = act.shape
    TX = (W + 15) // 16
    tls = tl.cpu().numpy()
    apix = np.array([act[(t // TX) * 16:(t // TX) * 16 + 16, (t % TX) * 16:(t % TX) * 16 + 16].sum() for t in tls])
    work = cnt * apix
    res = {"kept": nk, "inst_mean": float(cnt.mean()), "inst_max": int(cnt.max()), "inst_p90": float(np.percentile(cnt, 90)),
           "work_max_over_mean": float(work.max() / work.mean())}

    def time(fn, reps=20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            torch.cuda._sleep(1_000_000)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    fwd = lambda: P.render_color_depth(gm, eng.proj_iter, eng.bins, pose, cam, P.RTGS_RENDER_MASKED, eng.out)
    bwd = lambda: eng.backward(col, dep, pose)
    res["fwd_coverage_order"] = time(fwd)
    res["bwd_coverage_order"] = time(bwd)
    for name, key in (("inst", cnt), ("work", work)):
        order = np.argsort(-key, kind="stable")
        eng.out.tile_list[:nk].copy_(torch.as_tensor(tls[order].astype(np.int32)))
        res[f"fwd_sorted_{name}"] = time(fwd)
        res[f"bwd_sorted_{name}"] = time(bwd)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
