import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2404_19706_b200 as P
from synth import CONFIGS, make_frame, make_pose, make_scene, trajectory_pose
cfg = CONFIGS["C3"]
scene = make_scene(cfg)
gm = P.GaussianMap.from_arrays(scene, capacity=cfg.n + 1 + cfg.width * cfg.height // 4)
eng = P.MappingEngine(gm, P.camera_of(cfg), capacity=4 * cfg.n)
frames = []
for v in range(6):
    R, t = trajectory_pose(cfg, v)
    c, d = make_frame(cfg, (R, t))
    frames.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), P.make_pose(R, t)))
kv = [frames[0], frames[2], frames[4], frames[5]]
def tm(label, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    print(f"{label:30s} {1e3*(time.perf_counter()-t0):9.2f} ms", flush=True)
mode = sys.argv[1] if len(sys.argv) > 1 else "both"
if mode in ("both", "global"):
    tm("global_step 1", lambda: eng.global_step(kv))
    tm("global_step 2", lambda: eng.global_step(kv))
eng.cache_frames = 6
tm("window 1", lambda: eng.map_window(frames, iterations=50, seed=3))
tm("window 2", lambda: eng.map_window(frames, iterations=50, seed=4))
tm("window 3", lambda: eng.map_window(frames, iterations=50, seed=5))
