"""C3 masked iteration (cached) repeated: for ncu captures of k_render_bwd / k_project_bwd.
python scripts/prof_bwd.py [C3] [reps]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2404_19706_b200 as P
from synth import CONFIGS, make_frame, make_pose, make_scene

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
scene = make_scene(cfg)
R, t = make_pose(cfg)
col, dep = (torch.as_tensor(a, device="cuda") for a in make_frame(cfg))
cam, pose = P.camera_of(cfg), P.make_pose(R, t)
gm = P.GaussianMap.from_arrays(scene)
eng = P.MappingEngine(gm, cam, capacity=4 * cfg.n)
eng.ingest(col, dep, pose)
snap = {k: getattr(gm, k).clone() for k in ("pos", "log_scale", "rot", "sh")}
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for i in range(reps):
    for k, v in snap.items():
        getattr(gm, k).copy_(v)
    eng.m.zero_(); eng.v.zero_(); eng.grad.zero_(); eng.step_dev.zero_()
    eng.forward_masked(pose)
    ev[0].record()
    eng.backward_adam(col, dep, pose)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
print("backward_adam ms", sorted(ts)[len(ts) // 2])
