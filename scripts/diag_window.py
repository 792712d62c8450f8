"""Per-stage wall times of one mapping window on C3 (diagnostic)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2404_19706_b200 as P  # noqa: E402
from synth import CONFIGS, make_frame, make_pose, make_scene, trajectory_pose  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
    scene = make_scene(cfg)
    gm = P.GaussianMap.from_arrays(scene, capacity=cfg.n + 200_000)
    eng = P.MappingEngine(gm, P.camera_of(cfg), capacity=4 * cfg.n, cache_frames=6)
    frames = []
    for v in range(6):
        R, t = trajectory_pose(cfg, v)
        c, d = make_frame(cfg, (R, t))
        frames.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), P.make_pose(R, t)))
    torch.cuda.synchronize()

    def tm(label, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        print(f"{label:28s} {1e3 * (time.perf_counter() - t0):9.3f} ms", flush=True)
        return r

    eng.map_window(frames, iterations=50, seed=1, first_frame_idx=0)   # warm: caches allocated, map grown
    print("--- second window ---")
    for i, (c, d, pose) in enumerate(frames):
        tm(f"ingest {i}", lambda: eng.ingest(c, d, pose, frame_idx=i))
        r = tm(f"insert {i}", lambda: eng.insert(c, d, pose, frame_idx=i))
        print("   result", r.cpu().numpy().tolist())
    tm("reset_window", eng.reset_window)
    tm("reset_window (again)", eng.reset_window)
    print("   slots", int(eng.gid_of_slot.numel()))
    rng = np.random.default_rng(0)
    for k in range(5):
        c, d, pose = frames[int(rng.integers(6))]
        tm(f"iteration {k} cached={eng.cached(pose)}", lambda: eng.iteration(c, d, pose))
    t0 = time.perf_counter()
    for k in range(45):
        c, d, pose = frames[int(rng.integers(6))]
        eng.iteration(c, d, pose)
    torch.cuda.synchronize()
    print(f"45 iterations              {1e3 * (time.perf_counter() - t0):9.3f} ms")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    names = ["forward_masked", "backward_adam"]
    acc = {k: 0.0 for k in names}
    for k in range(10):
        c, d, pose = frames[int(rng.integers(6))]
        torch.cuda.synchronize()
        e0.record(); eng.forward_masked(pose); e1.record(); torch.cuda.synchronize()
        acc["forward_masked"] += e0.elapsed_time(e1) / 10
        e0.record(); eng.backward_adam(c, d, pose); e1.record(); torch.cuda.synchronize()
        acc["backward_adam"] += e0.elapsed_time(e1) / 10
    print("device ms per iteration part", {k: round(v, 3) for k, v in acc.items()})
    print("kept tiles", int(eng.out.counts[0].item()), "active px", int(eng.out.counts[2].item()),
          "instances", int(eng.bins.n_instances.item()))
    c, d, pose = frames[-1]
    tm("end_window", lambda: eng.end_window(c, d, pose, frame_idx=5))


if __name__ == "__main__":
    main()
