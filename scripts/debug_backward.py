"""Diagnostics for the backward parity (run on the GPU box): prints the worst coordinates."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import loss as OL  # noqa: E402
from tests.test_gpu_backward import GROUPS, _case  # noqa: E402


def main(name="C1"):
    import paper_2404_19706_b200 as P
    cfg, scene, R, t, cam_d, act, col, dep, unstable, img = _case(P, name)
    gm = P.GaussianMap.from_arrays(scene)
    cam = P.camera_of(cfg)
    pose = P.make_pose(R, t)
    eng = P.MappingEngine(gm, cam)
    eng.forward_masked(pose)
    eng.backward(torch.as_tensor(col, device="cuda"), torch.as_tensor(dep, device="cuda"), pose)
    torch.cuda.synchronize()
    gid = eng.gid_of_slot.cpu().numpy()
    res = OL.iteration_grads(scene, R, t, cam_d, col, dep, act, gid)
    g = eng.grad[: len(gid)].cpu().numpy().astype(np.float64)
    o = res["grad"]
    print("loss gpu", eng.loss.cpu().numpy(), "oracle", res["L_c"].item(), res["L_d"].item(), res["n_Pd"])
    for gname, a, b in GROUPS:
        og, gg = o[:, a:b], g[:, a:b]
        rms = np.sqrt((og ** 2).mean())
        tol = 1e-3 * np.maximum(np.abs(og), 1e-2 * rms)
        r = np.abs(gg - og) / tol
        idx = np.unravel_index(np.argsort(-r, axis=None)[:5], r.shape)
        print(gname, "rms", rms, "max ratio", r.max(), "frac>1", (r > 1).mean())
        for s, c in zip(*idx):
            print(f"   slot {s} gid {gid[s]} comp {a + c}: gpu {gg[s, c]:.6e} oracle {og[s, c]:.6e} ratio {r[s, c]:.2f}"
                  f" flags {scene['flags'][gid[s]]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
