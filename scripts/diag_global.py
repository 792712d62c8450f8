"""Per-part device times of one (e) keyframe global step on C3 (diagnostic): per view the
projection + binning, FULL render, top-k mask and masked backward over all Gaussians, then Adam."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2404_19706_b200 as P  # noqa: E402
from paper_2404_19706_b200 import mapping as M  # noqa: E402
from synth import CONFIGS, make_frame, make_scene, trajectory_pose  # noqa: E402


def main():
    cfg = CONFIGS["C3"]
    gm = P.GaussianMap.from_arrays(make_scene(cfg))
    eng = P.MappingEngine(gm, P.camera_of(cfg), capacity=4 * cfg.n)
    views = []
    for v in (0, 2, 4, 5):
        R, t = trajectory_pose(cfg, v)
        c, d = make_frame(cfg, (R, t))
        views.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), P.make_pose(R, t)))
    eng.global_step(views)
    torch.cuda.synchronize()
    ev = []

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        ev.append((name, e))

    torch.cuda._sleep(10_000_000)
    mark("start")
    eng._global_state()
    w = tuple(x / len(views) for x in eng.weights[:2]) + (eng.weights[2],)
    for k, (c, d, pose) in enumerate(views):
        M.project_and_bin(gm, pose, eng.cam, eng.proj, eng.bins, eng.ws_bin); mark(f"v{k}.project_bin")
        M.render_color_depth(gm, eng.proj, eng.bins, pose, eng.cam, P.RTGS_RENDER_FULL, eng.g_rb); mark(f"v{k}.full")
        M.topk_error_mask(eng.g_rb, c, eng.cam, 0.4, eng.g_rb, eng.g_ws_topk); mark(f"v{k}.topk")
        M.render_backward_masked(gm, eng.proj, eng.bins, pose, eng.cam, eng.g_rb, c, d, w, eng.g_slot, eng.g_gid,
                                 eng.g_grad, eng.g_loss, eng.g_ws_bwd); mark(f"v{k}.backward")
    eng.g_m.zero_(); eng.g_v.zero_(); mark("zero_mv")
    M.adam_step_unstable(gm, eng.g_gid, eng.g_grad, eng.g_m, eng.g_v, None, 0, eng.weights[2],
                         eng._global_hparams(0.1), 1, eng.eta); mark("adam")
    torch.cuda.synchronize()
    for (a, ea), (b, eb) in zip(ev[:-1], ev[1:]):
        print(f"{b:18s} {ea.elapsed_time(eb):8.3f} ms")
    print("total", ev[0][1].elapsed_time(ev[-1][1]))


if __name__ == "__main__":
    main()
