"""One C3 frame: project + bin + FULL render (span and dense), for ncu.  python scripts/prof_render.py [C3]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2404_19706_b200 as P
from paper_2404_19706_b200 import mapping as M
from synth import CONFIGS, make_pose, make_scene

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
scene = make_scene(cfg)
R, t = make_pose(cfg)
cam, pose = P.camera_of(cfg), P.make_pose(R, t)
gm = P.GaussianMap.from_arrays(scene)
n = gm.n
cap = 4 * n
proj, bins = M.ProjectedBuffers(n), M.BinBuffers(cam, cap)
ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
rb = M.RenderBuffers(cam, count_blends=False)
P.project_gaussians(gm, pose, cam, proj)
P.bin_and_sort(proj, n, cam, None, bins, ws)
for dense in (False, True, False, True):
    P.render_color_depth(gm, proj, bins, pose, cam, P.RTGS_RENDER_FULL, rb, dense=dense)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for dense, (e0, e1) in ((False, ev[:2]), (True, ev[2:])):
    e0.record()
    for _ in range(20):
        P.render_color_depth(gm, proj, bins, pose, cam, P.RTGS_RENDER_FULL, rb, dense=dense)
    e1.record()
torch.cuda.synchronize()
print("span ms", ev[0].elapsed_time(ev[1]) / 20, "dense ms", ev[2].elapsed_time(ev[3]) / 20)
