"""Work counters of the span forward walk (needs a -DRTGS_RENDER_STATS build in place of librtgs.so:
python scripts/build_variant.py paper_2404_19706_b200/librtgs.so -DRTGS_RENDER_STATS).
python scripts/render_stats.py [C3|C4|C2] [masked]"""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
import paper_2404_19706_b200 as P
from paper_2404_19706_b200 import mapping as M
from paper_2404_19706_b200._abi import lib
from synth import CONFIGS, make_pose, make_scene

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = CONFIGS[name]
scene = make_scene(cfg)
R, t = make_pose(cfg)
cam, pose = P.camera_of(cfg), P.make_pose(R, t)
gm = P.GaussianMap.from_arrays(scene)
n = gm.n
proj, bins = M.ProjectedBuffers(n), M.BinBuffers(cam, 4 * n)
ws = torch.empty(M.bin_workspace_size(n, cam, 4 * n), dtype=torch.uint8, device="cuda")
rb = M.RenderBuffers(cam, count_blends=True)
P.project_gaussians(gm, pose, cam, proj)
P.bin_and_sort(proj, n, cam, None, bins, ws)
f = lib().rtgs_debug_render_stats
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 8)()
f(buf, 1)
P.render_color_depth(gm, proj, bins, pose, cam, P.RTGS_RENDER_FULL, rb)
torch.cuda.synchronize()
f(buf, 1)
s = list(buf)
keys = ["warp_batches", "survivors", "rounds", "trips", "lane_pairs", "blends", "records", "round_slots"]
print(name, dict(zip(keys, s)))
print("instances", int(bins.n_instances.item()), "counts3", int(rb.counts[3].item()))
print("survivors/warp-batch %.1f  records/warp-batch %.1f  lane util (pairs/(32 trips)) %.3f  blends/pair %.3f"
      "  trips/round %.1f  slots/round %.1f" % (s[1] / s[0], s[6] / s[0], s[4] / (32 * s[3]), s[5] / max(s[4], 1),
                                                 s[3] / s[2], s[7] / s[2]))
