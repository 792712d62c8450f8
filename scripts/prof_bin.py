"""A2 binning at C4 (or the named config): tile-list length distribution and event-timed
project + bin_and_sort.  python scripts/prof_bin.py [C4] [reps]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2404_19706_b200 as P
from paper_2404_19706_b200 import mapping as M
from synth import CONFIGS, make_pose, make_scene

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
scene = make_scene(cfg)
R, t = make_pose(cfg)
cam, pose = P.camera_of(cfg), P.make_pose(R, t)
gm = P.GaussianMap.from_arrays(scene)
eng = P.MappingEngine(gm, cam, capacity=4 * cfg.n)
eng.reorder_spatially()
gm = eng.gm
n = gm.n
proj, bins = M.ProjectedBuffers(n), M.BinBuffers(cam, 4 * n)
ws = torch.empty(M.bin_workspace_size(n, cam, 4 * n), dtype=torch.uint8, device="cuda")
P.project_gaussians(gm, pose, cam, proj)
P.bin_and_sort(proj, n, cam, None, bins, ws)
torch.cuda.synchronize()
rg = bins.tile_range.view(-1, 2).cpu().numpy().astype(np.int64)
ln = rg[:, 1] - rg[:, 0]
print("tiles", len(ln), "instances", int(ln.sum()), "mean %.1f" % ln.mean(), "p50/p90/p99/max",
      np.percentile(ln, [50, 90, 99]).tolist(), int(ln.max()), "> 1024:", int((ln > 1024).sum()),
      "keys in >1024 tiles: %.3f" % (ln[ln > 1024].sum() / max(1, ln.sum())))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(reps):
    ev[0].record()
    P.bin_and_sort(proj, n, cam, None, bins, ws)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
print("bin_and_sort ms median %.4f min %.4f" % (float(np.median(ts)), min(ts)))
