"""Debug: where does the float32 error of a failing gradient coordinate come from?  Compares the GPU's
screen-space sums (backward workspace) with the oracle's exact dL/d(conic, mu, rgb) sums, and the
float64 chain rule applied to the GPU sums with the GPU's final gradient."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import loss as OL, projection as OP
from tests.test_gpu_backward import _case, GROUPS
from tests.test_gpu_shdeg import _truncate
from tests.gpu_common import device_map
import paper_2404_19706_b200 as P

name, deg = sys.argv[1], int(sys.argv[2])
cfg, scene, R, t, cam_d, act, col, dep, unstable, img = _case(P, name)
if deg < 3:
    scene = _truncate(scene, deg)
gm = device_map(scene)
cam = P.camera_of(cfg)
pose = P.make_pose(R, t)
eng = P.MappingEngine(gm, cam)
eng.forward_masked(pose)
tc, td = torch.as_tensor(col, device="cuda"), torch.as_tensor(dep, device="cuda")
eng.backward(tc, td, pose)
torch.cuda.synchronize()
gid = eng.gid_of_slot.cpu().numpy()
S = len(gid)
sg = eng.ws_bwd[: S * 16 * 4].view(torch.float32).reshape(S, 16).cpu().numpy().astype(np.float64)
res = OL.iteration_loss(scene, R, t, cam_d, col, dep, act)
proj = res["proj"]
for k in ("conic", "mu", "rgb"):
    proj[k].retain_grad()
res["L"].backward()
g = eng.grad[:S].cpu().numpy().astype(np.float64)
from oracle.loss import slot_grads
o = slot_grads(res["params"], gid)
r2 = OL.iteration_grads(scene, R, t, cam_d, col, dep, act, gid, mass=True)
M = r2["mass"]
tol = 1e-3 * np.maximum(np.abs(o), 1e-2 * M)
ratio = np.abs(g - o) / tol
worst = np.argsort(ratio.ravel())[::-1][:5]
for w in worst:
    s, c = divmod(w, g.shape[1])
    print(f"slot {s} gid {gid[s]} coord {c} ratio {ratio[s, c]:.2f} g {g[s, c]:.6e} o {o[s, c]:.6e} M {M[s, c]:.3e}")
    oc = proj["conic"].grad[gid[s]].numpy()
    om = proj["mu"].grad[gid[s]].numpy()
    print("   conic sums gpu", sg[s, 2:5], "oracle", oc, "rel", (sg[s, 2:5] - oc) / np.abs(oc).max())
    print("   mu sums gpu", sg[s, 0:2], "oracle", om)
    # float64 chain rule applied to the GPU's conic sums (log-scale / rotation only see the conic)
    prm = OP.params_from_scene(scene, requires_grad=True)
    pr = OP.project(prm, R, t, cam_d, scene["sh_degree"])
    v = (pr["conic"][gid[s]] * torch.as_tensor(sg[s, 2:5])).sum() + (pr["mu"][gid[s]] * torch.as_tensor(sg[s, 0:2])).sum()
    v.backward()
    gl = torch.cat([prm["log_scale"].grad[gid[s]], prm["rot"].grad[gid[s]]]).numpy()
    print("   chain64(gpu sums) log_scale/rot", gl, "gpu", g[s, 3:10], "oracle", o[s, 3:10])
