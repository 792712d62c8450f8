"""Kernel list of window iterations (diagnostic): one warm window on C3, then 3 iterations inside
cudaProfilerStart/Stop, for `ncu --profile-from-start off --metrics gpu__time_duration.sum`."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2404_19706_b200 as P  # noqa: E402
from synth import CONFIGS, make_frame, make_scene, trajectory_pose  # noqa: E402


def main():
    cfg = CONFIGS["C3"]
    gm = P.GaussianMap.from_arrays(make_scene(cfg), capacity=cfg.n + 200_000)
    eng = P.MappingEngine(gm, P.camera_of(cfg), capacity=4 * cfg.n, cache_frames=6)
    frames = []
    for v in range(6):
        R, t = trajectory_pose(cfg, v)
        c, d = make_frame(cfg, (R, t))
        frames.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), P.make_pose(R, t)))
    eng.map_window(frames, iterations=10, seed=1)
    for i, (c, d, pose) in enumerate(frames):
        eng.ingest(c, d, pose, frame_idx=10 + i)
        eng.insert(c, d, pose, frame_idx=10 + i)
    eng.reset_window()
    rng = np.random.default_rng(0)
    c, d, pose = frames[int(rng.integers(6))]
    eng.iteration(c, d, pose)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(3):
        c, d, pose = frames[int(rng.integers(6))]
        eng.iteration(c, d, pose)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("slots", int(eng.gid_of_slot.numel()), "kept", int(eng.out.counts[0].item()),
          "instances", int(eng.bins.n_instances.item()))


if __name__ == "__main__":
    main()
