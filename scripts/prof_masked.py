"""C3 MASKED render, span vs dense consumer (CUDA events, 20 launches each)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2404_19706_b200 as P
from synth import CONFIGS, make_pose, make_scene

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
scene = make_scene(cfg)
R, t = make_pose(cfg)
cam, pose = P.camera_of(cfg), P.make_pose(R, t)
gm = P.GaussianMap.from_arrays(scene)
eng = P.MappingEngine(gm, cam, capacity=4 * cfg.n)
eng.use_cache = False
eng.forward_masked(pose)
torch.cuda.synchronize()
rb = eng.out
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for dense, (e0, e1) in ((False, ev[:2]), (True, ev[2:]), (False, ev[:2]), (True, ev[2:])):
    e0.record()
    for _ in range(20):
        P.render_color_depth(gm, eng.proj, eng.bins, pose, cam, P.RTGS_RENDER_MASKED, rb, dense=dense)
    e1.record()
    torch.cuda.synchronize()
    print("dense" if dense else "span", ev[2 if dense else 0].elapsed_time(ev[3 if dense else 1]) / 20)
