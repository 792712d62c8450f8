"""Python binding of librtgs.so: argument marshalling only.

Every step of the mapping path runs in the CUDA kernels behind include/rtgs.h; this module only
allocates device buffers with torch (plumbing), builds the C structs and calls the six entry points
under the same names:

    project_gaussians, bin_and_sort, render_color_depth, render_backward_masked,
    adam_step_unstable, classify_and_add_pixels

`MappingEngine` strings them together into the paper's per-frame flow:
    ingest(frame)     A1 project -> A2 bin (all tiles) -> A3/A4 FULL render -> A7 classify
    iteration(frame)  A1 project -> A0 coverage/tile keep -> A2 bin (kept tiles) -> A3/A4 MASKED
                      -> A5 masked backward -> A6 Adam over the unstable Gaussians
With the NEXT f3 cache (an ingest of the same pose in the current window) the iteration's A1/A2
touch only the unstable slots: project_subset -> coverage over the slots -> bin_and_sort_cached
(merge with the frame's cached stable lists).
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np
import torch

from . import _abi
from ._abi import RTGS_RENDER_COUNT, RTGS_RENDER_DENSE, RTGS_RENDER_COVERAGE, RTGS_RENDER_FULL, RTGS_RENDER_MASKED, check, lib

FLAG_TRANSPARENT = 1
FLAG_STABLE = 2
FLAG_REMOVED = 4  # NEXT f1: removed Gaussians (absorbing, culled by A1)


def _p(t: torch.Tensor | None):
    if t is None:
        return None
    ptr = t.data_ptr()
    if ptr == 0 and t.untyped_storage().nbytes() > 0:
        # an empty view of an allocated store (a map with n = 0): torch reports 0, the store is real
        ptr = t.untyped_storage().data_ptr() + t.storage_offset() * t.element_size()
    return C.c_void_p(ptr)


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def make_camera(fx, fy, cx, cy, width, height) -> _abi.Camera:
    return _abi.Camera(float(fx), float(fy), float(cx), float(cy), int(width), int(height))


def camera_of(cfg) -> _abi.Camera:
    return make_camera(cfg.fx, cfg.fy, cfg.cx, cfg.cy, cfg.width, cfg.height)


def make_pose(R, t) -> _abi.Pose:
    R = np.asarray(R, dtype=np.float64).reshape(9)
    t = np.asarray(t, dtype=np.float64).reshape(3)
    return _abi.Pose((C.c_double * 9)(*R), (C.c_double * 3)(*t))


_MAP_FIELDS = ("pos", "log_scale", "rot", "opacity", "sh", "flags")


@dataclasses.dataclass
class GaussianMap:
    """Device SoA of the Gaussian map, float32.  The fields are views of the first n
    rows of `store` (capacity rows), so Gaussians can be appended (NEXT f2) without reallocation."""
    pos: torch.Tensor
    log_scale: torch.Tensor
    rot: torch.Tensor
    opacity: torch.Tensor
    sh: torch.Tensor
    flags: torch.Tensor  # uint8
    sh_degree: int
    store: dict | None = None

    @property
    def n(self) -> int:
        return int(self.pos.shape[0])

    @property
    def capacity(self) -> int:
        return int(self.store["pos"].shape[0]) if self.store is not None else self.n

    @classmethod
    def from_arrays(cls, scene: dict, device="cuda", capacity: int | None = None) -> "GaussianMap":
        n = int(np.asarray(scene["pos"]).shape[0])
        cap = max(int(capacity) if capacity is not None else n, n, 1)
        store = {}
        for k in _MAP_FIELDS:
            a = np.ascontiguousarray(scene[k])
            t = torch.zeros((cap,) + a.shape[1:], dtype=torch.as_tensor(a[:0]).dtype, device=device)
            t[:n].copy_(torch.as_tensor(a))
            store[k] = t
        return cls(*[store[k][:n] for k in _MAP_FIELDS], int(scene["sh_degree"]), store)

    def resize(self, n: int):
        """Make rows [0, n) live (n <= capacity): re-slices the views, no copy."""
        if self.store is None or n > self.capacity:
            raise ValueError(f"resize to {n} beyond capacity {self.capacity}")
        for k in _MAP_FIELDS:
            setattr(self, k, self.store[k][:n])

    def reserve(self, capacity: int):
        """Grow the storage to `capacity` rows (a device copy of the live rows; views re-sliced)."""
        if capacity <= self.capacity:
            return
        n = self.n
        store = {}
        for k in _MAP_FIELDS:
            old = self.store[k] if self.store is not None else getattr(self, k)
            t = torch.zeros((capacity,) + tuple(old.shape[1:]), dtype=old.dtype, device=old.device)
            t[:n].copy_(old[:n])
            store[k] = t
        self.store = store
        self.resize(n)

    def permute(self, perm: torch.Tensor, stream=None):
        """Reorder the live rows: row r becomes old row perm[r] (every field; storage reallocated)."""
        n = self.n
        for k in _MAP_FIELDS:
            old = self.store[k] if self.store is not None else getattr(self, k)
            new = torch.empty_like(old)
            if n:
                gather_rows(old[:n], new, perm, stream)
            if old.shape[0] > n:
                new[n:].copy_(old[n:])
            if self.store is not None:
                self.store[k] = new
            else:
                setattr(self, k, new)
        if self.store is not None:
            self.resize(n)

    def c_struct(self) -> _abi.Gaussians:
        return _abi.Gaussians(_p(self.pos), _p(self.log_scale), _p(self.rot), _p(self.opacity), _p(self.sh),
                              _p(self.flags), self.n, self.sh_degree)

    def c_params(self) -> _abi.Params:
        return _abi.Params(_p(self.pos), _p(self.log_scale), _p(self.rot), _p(self.sh), self.n, self.sh_degree)


class ProjectedBuffers:
    def __init__(self, n: int, device="cuda"):
        nn = max(n, 1)
        self.rec = torch.empty((nn, 16), dtype=torch.float32, device=device)
        self.zkey = torch.empty(nn, dtype=torch.int32, device=device)
        self.rect = torch.empty((nn, 4), dtype=torch.int16, device=device)
        self.tiles_touched = torch.empty(nn, dtype=torch.int32, device=device)

    def c_struct(self):
        return _abi.Projected(_p(self.rec), _p(self.zkey), _p(self.rect), _p(self.tiles_touched))


class BinBuffers:
    def __init__(self, cam: _abi.Camera, capacity: int, device="cuda"):
        T = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
        self.capacity = int(capacity)
        self.sorted_gid = torch.empty(max(capacity, 1), dtype=torch.int32, device=device)
        self.tile_range = torch.zeros((T, 2), dtype=torch.int32, device=device)
        self.n_instances = torch.zeros(1, dtype=torch.int32, device=device)
        self.sub = None  # NEXT f3: (sub rec, sub zkey, sub gid) tensors the entries with bit 31 refer to

    def c_struct(self):
        sr, sz, sg = self.sub if self.sub is not None else (None, None, None)
        return _abi.Bins(_p(self.sorted_gid), _p(self.tile_range), _p(self.n_instances), self.capacity, _p(sr), _p(sz),
                         _p(sg))


class RenderBuffers:
    def __init__(self, cam: _abi.Camera, device="cuda", normal=True, count_blends=True):
        H, W = cam.height, cam.width
        T = ((W + 15) // 16) * ((H + 15) // 16)
        self.color = torch.zeros((3, H, W), dtype=torch.float32, device=device)
        self.trans = torch.zeros((H, W), dtype=torch.float32, device=device)
        self.depth = torch.zeros((H, W), dtype=torch.float32, device=device)
        self.normal = torch.zeros((3, H, W), dtype=torch.float32, device=device) if normal else None
        self.index = torch.zeros((H, W), dtype=torch.int32, device=device)
        self.n_contrib = torch.zeros((H, W), dtype=torch.int32, device=device)
        self.active_bits = torch.zeros((H * W + 31) // 32, dtype=torch.int32, device=device)
        self.tile_keep = torch.zeros(T, dtype=torch.uint8, device=device)
        self.tile_list = torch.zeros(T, dtype=torch.int32, device=device)
        self.counts = torch.zeros(4, dtype=torch.int32, device=device)
        # FULL / MASKED renders count blended pairs (counts[3], RTGS_RENDER_COUNT) only when asked: the
        # statistic costs instructions per blended pair
        self.count_blends = count_blends
        # n_contrib is what a backward over this render needs; a FULL render used only for the add
        # masks / state decisions / tracking can skip tracking it
        self.track_last = True

    def c_struct(self, mode: int | None = None):
        nc = self.n_contrib if (self.track_last or self.count_blends or mode != RTGS_RENDER_FULL) else None
        return _abi.RenderOut(_p(self.color), _p(self.trans), _p(self.depth), _p(self.normal), _p(self.index),
                              _p(nc), _p(self.active_bits), _p(self.tile_keep), _p(self.tile_list),
                              _p(self.counts))

    def active_mask(self) -> torch.Tensor:
        """Unpack active_bits into a bool [H, W] image (test / inspection helper)."""
        H, W = self.trans.shape
        words = self.active_bits.to(torch.int64) & 0xFFFFFFFF
        bits = (words[:, None] >> torch.arange(32, device=words.device)) & 1
        return bits.reshape(-1)[: H * W].reshape(H, W).bool()

    def active_set(self) -> torch.Tensor:
        """P = M_unstable ∩ kept tiles as a bool [H, W] image (test / inspection helper)."""
        H, W = self.trans.shape
        TX = (W + 15) // 16
        ys = torch.arange(H, device=self.tile_keep.device) // 16
        xs = torch.arange(W, device=self.tile_keep.device) // 16
        kept = self.tile_keep.bool()[(ys[:, None] * TX + xs[None, :])]
        return self.active_mask() & kept


# ---------------------------------------------------------------------------------------------
# the six entry points (same names as the C ABI)
# ---------------------------------------------------------------------------------------------
def project_gaussians(gm: GaussianMap, pose: _abi.Pose, cam: _abi.Camera, proj: ProjectedBuffers, stream=None):
    g = gm.c_struct()
    pr = proj.c_struct()
    check(lib().rtgs_project_gaussians(C.byref(g), C.byref(pose), C.byref(cam), C.byref(pr), _stream(stream)),
          "rtgs_project_gaussians")


def bin_workspace_size(n: int, cam: _abi.Camera, capacity: int) -> int:
    return int(lib().rtgs_bin_workspace_size(n, C.byref(cam), capacity))


def bin_and_sort(proj: ProjectedBuffers, n: int, cam: _abi.Camera, tile_keep: torch.Tensor | None, bins: BinBuffers,
                 workspace: torch.Tensor, stream=None):
    pr = proj.c_struct()
    b = bins.c_struct()
    check(lib().rtgs_bin_and_sort(C.byref(pr), n, C.byref(cam), _p(tile_keep), C.byref(b), _p(workspace),
                                  workspace.numel() * workspace.element_size(), _stream(stream)), "rtgs_bin_and_sort")


def project_and_bin(gm: GaussianMap, pose: _abi.Pose, cam: _abi.Camera, proj: ProjectedBuffers, bins: BinBuffers,
                    workspace: torch.Tensor, stream=None, cache: BinBuffers | None = None):
    """A1 + A2 (all tiles) in one call: the projection kernel also counts the tile instances; with
    `cache` the tile sort also writes the f3 stable cache (as stable_cache_build)."""
    g = gm.c_struct()
    pr = proj.c_struct()
    b = bins.c_struct()
    c = cache.c_struct() if cache is not None else None
    check(lib().rtgs_project_and_bin(C.byref(g), C.byref(pose), C.byref(cam), C.byref(pr), C.byref(b),
                                     C.byref(c) if c is not None else None, _p(workspace),
                                     workspace.numel() * workspace.element_size(), _stream(stream)),
          "rtgs_project_and_bin")
    bins.sub = None


def render_color_depth(gm: GaussianMap, proj: ProjectedBuffers, bins: BinBuffers | None, pose: _abi.Pose,
                       cam: _abi.Camera, mode: int, out: RenderBuffers, stream=None, normals: bool = True,
                       dense: bool = False):
    """A0 / A3-A4.  normals=False leaves out.normal untouched (the normal map is for tracking);
    dense=True selects the dense verification consumer (RTGS_RENDER_DENSE)."""
    g = gm.c_struct()
    pr = proj.c_struct()
    o = out.c_struct(mode)
    if not normals:
        o.normal = None
    b = bins.c_struct() if bins is not None else None
    if out.count_blends and mode in (RTGS_RENDER_FULL, RTGS_RENDER_MASKED):
        mode |= RTGS_RENDER_COUNT
    if dense and mode != RTGS_RENDER_COVERAGE:
        mode |= RTGS_RENDER_DENSE
    check(lib().rtgs_render_color_depth(C.byref(g), C.byref(pr), C.byref(b) if b is not None else None, C.byref(pose),
                                        C.byref(cam), mode, C.byref(o), _stream(stream)), "rtgs_render_color_depth")


def backward_workspace_size(n_slots: int) -> int:
    return int(lib().rtgs_backward_workspace_size(n_slots))


def render_backward_masked(gm: GaussianMap, proj: ProjectedBuffers, bins: BinBuffers, pose: _abi.Pose, cam: _abi.Camera,
                           fwd: RenderBuffers, target_color: torch.Tensor, target_depth: torch.Tensor,
                           weights: tuple, slot_of_gid: torch.Tensor, gid_of_slot: torch.Tensor, grad: torch.Tensor,
                           loss_out: torch.Tensor, workspace: torch.Tensor, stream=None):
    g = gm.c_struct()
    pr = proj.c_struct()
    b = bins.c_struct()
    o = fwd.c_struct()
    fr = _abi.Frame(_p(target_color), _p(target_depth))
    w = _abi.LossWeights(*[float(x) for x in weights])
    check(lib().rtgs_render_backward_masked(C.byref(g), C.byref(pr), C.byref(b), C.byref(pose), C.byref(cam), C.byref(o),
                                            C.byref(fr), C.byref(w), _p(slot_of_gid), _p(gid_of_slot),
                                            int(gid_of_slot.numel()), _p(grad), _p(loss_out), _p(workspace),
                                            workspace.numel() * workspace.element_size(), _stream(stream)),
          "rtgs_render_backward_masked")


def adam_step_unstable(gm: GaussianMap, gid_of_slot: torch.Tensor, grad: torch.Tensor, m: torch.Tensor,
                       v: torch.Tensor, init_geom: torch.Tensor | None, n_transparent: int, w_reg: float,
                       hparams: _abi.HParams, step: int, eta: torch.Tensor, stream=None,
                       step_device: torch.Tensor | None = None):
    prm = gm.c_params()
    check(lib().rtgs_adam_step_unstable(C.byref(prm), _p(gid_of_slot), int(gid_of_slot.numel()), _p(gm.flags), _p(grad),
                                        _p(m), _p(v), _p(init_geom), int(n_transparent), float(w_reg), C.byref(hparams),
                                        int(step), _p(step_device), _p(eta), _stream(stream)), "rtgs_adam_step_unstable")


def backward_adam_unstable(gm: GaussianMap, proj: ProjectedBuffers, bins: BinBuffers, pose: _abi.Pose,
                           cam: _abi.Camera, fwd: RenderBuffers, target_color: torch.Tensor,
                           target_depth: torch.Tensor, weights: tuple, slot_of_gid: torch.Tensor,
                           gid_of_slot: torch.Tensor, m: torch.Tensor, v: torch.Tensor, init_geom: torch.Tensor | None,
                           n_transparent: int, hparams: _abi.HParams, step: int, eta: torch.Tensor,
                           loss_out: torch.Tensor, workspace: torch.Tensor, stream=None,
                           step_device: torch.Tensor | None = None):
    """A5 + A6 fused (one view -> one Adam step): render_backward_masked into a zero gradient, then
    adam_step_unstable with w_reg = weights[2], without a gradient buffer."""
    g = gm.c_struct()
    prm = gm.c_params()
    pr = proj.c_struct()
    b = bins.c_struct()
    o = fwd.c_struct()
    fr = _abi.Frame(_p(target_color), _p(target_depth))
    w = _abi.LossWeights(*[float(x) for x in weights])
    check(lib().rtgs_backward_adam_unstable(C.byref(g), C.byref(pr), C.byref(b), C.byref(pose), C.byref(cam),
                                            C.byref(o), C.byref(fr), C.byref(w), _p(slot_of_gid), _p(gid_of_slot),
                                            int(gid_of_slot.numel()), C.byref(prm), _p(m), _p(v), _p(init_geom),
                                            int(n_transparent), C.byref(hparams), int(step), _p(step_device), _p(eta),
                                            _p(loss_out), _p(workspace), workspace.numel() * workspace.element_size(),
                                            _stream(stream)), "rtgs_backward_adam_unstable")


def classify_workspace_size(cam: _abi.Camera) -> int:
    return int(lib().rtgs_classify_workspace_size(C.byref(cam)))


def classify_and_add_pixels(full: RenderBuffers, frame_color: torch.Tensor, frame_depth: torch.Tensor,
                            flags: torch.Tensor, cam: _abi.Camera, add: _abi.AddParams, pixel_class: torch.Tensor,
                            samples: torch.Tensor, counts: torch.Tensor, workspace: torch.Tensor, stream=None):
    o = full.c_struct()
    fr = _abi.Frame(_p(frame_color), _p(frame_depth))
    check(lib().rtgs_classify_and_add_pixels(C.byref(o), C.byref(fr), _p(flags), C.byref(cam), C.byref(add),
                                             _p(pixel_class), _p(samples), int(samples.numel()), _p(counts),
                                             _p(workspace), workspace.numel() * workspace.element_size(),
                                             _stream(stream)), "rtgs_classify_and_add_pixels")


def fuse_window(gm: GaussianMap, gid_of_slot: torch.Tensor, before: torch.Tensor, eta_before: torch.Tensor,
                eta: torch.Tensor, stream=None):
    """NEXT f1: Eq.9 fusion of the window's result with the parameters before the window."""
    prm = gm.c_params()
    check(lib().rtgs_fuse_window(C.byref(prm), _p(gid_of_slot), int(gid_of_slot.numel()), _p(before), _p(eta_before),
                                 _p(eta), _stream(stream)), "rtgs_fuse_window")


def state_params(frame_idx: int, delta_c=0.1, delta_d=0.1, delta_e=3, delta_eta=100, delta_t=30) -> _abi.StateParams:
    return _abi.StateParams(delta_c, delta_d, delta_e, delta_eta, delta_t, frame_idx)


def manage_states(full: RenderBuffers, frame_color: torch.Tensor, frame_depth: torch.Tensor, cam: _abi.Camera,
                  flags: torch.Tensor, err_count: torch.Tensor, eta: torch.Tensor, t_created: torch.Tensor,
                  sp: _abi.StateParams, counts: torch.Tensor, workspace: torch.Tensor, stream=None):
    """NEXT f1: error counts from the optimised render and the stable / unstable / removed transitions."""
    o = full.c_struct()
    fr = _abi.Frame(_p(frame_color), _p(frame_depth))
    check(lib().rtgs_manage_states(C.byref(o), C.byref(fr), C.byref(cam), _p(flags), _p(err_count), _p(eta),
                                   _p(t_created), int(flags.numel()), C.byref(sp), _p(counts), _p(workspace),
                                   workspace.numel() * workspace.element_size(), _stream(stream)), "rtgs_manage_states")


def state_workspace_size(n: int) -> int:
    return int(lib().rtgs_state_workspace_size(n))


# ---------------------------------------------------------------------------------------------
# NEXT f3: window-level stable-projection cache
# ---------------------------------------------------------------------------------------------
def project_subset(gm: GaussianMap, gid_list: torch.Tensor, pose: _abi.Pose, cam: _abi.Camera,
                   proj: ProjectedBuffers, stream=None):
    """Rows i of `proj` = projection of Gaussian gid_list[i]."""
    g = gm.c_struct()
    pr = proj.c_struct()
    check(lib().rtgs_project_subset(C.byref(g), _p(gid_list), int(gid_list.numel()), C.byref(pose), C.byref(cam),
                                    C.byref(pr), _stream(stream)), "rtgs_project_subset")


def coverage_rows(gm: GaussianMap, proj: ProjectedBuffers, n_rows: int, pose: _abi.Pose, cam: _abi.Camera,
                  out: RenderBuffers, stream=None):
    """COVERAGE over every (non-culled) row of a subset projection (flags NULL: all rows unstable)."""
    g = gm.c_struct()
    g.flags = None
    g.n = int(n_rows)
    pr = proj.c_struct()
    o = out.c_struct()
    check(lib().rtgs_render_color_depth(C.byref(g), C.byref(pr), None, C.byref(pose), C.byref(cam),
                                        RTGS_RENDER_COVERAGE, C.byref(o), _stream(stream)), "rtgs_render_color_depth")


def stable_cache_build(full: BinBuffers, flags: torch.Tensor, cam: _abi.Camera, cache: BinBuffers, stream=None):
    f = full.c_struct()
    c = cache.c_struct()
    check(lib().rtgs_stable_cache_build(C.byref(f), _p(flags), C.byref(cam), C.byref(c), _stream(stream)),
          "rtgs_stable_cache_build")


def bin_cached_workspace_size(n_sub: int, cam: _abi.Camera, capacity: int) -> int:
    return int(lib().rtgs_bin_cached_workspace_size(n_sub, C.byref(cam), capacity))


def bin_and_sort_cached(proj: ProjectedBuffers, cache: BinBuffers, sub: ProjectedBuffers, sub_gid: torch.Tensor,
                        cam: _abi.Camera, tile_keep: torch.Tensor, out: BinBuffers, workspace: torch.Tensor,
                        stream=None):
    pr = proj.c_struct()
    c = cache.c_struct()
    sp = sub.c_struct()
    o = out.c_struct()
    check(lib().rtgs_bin_and_sort_cached(C.byref(pr), C.byref(c), C.byref(sp), _p(sub_gid), int(sub_gid.numel()),
                                         C.byref(cam), _p(tile_keep), C.byref(o), _p(workspace),
                                         workspace.numel() * workspace.element_size(), _stream(stream)),
          "rtgs_bin_and_sort_cached")
    out.sub = (sub.rec, sub.zkey, sub_gid)


# ---------------------------------------------------------------------------------------------
# NEXT f2: Gaussian insertion
# ---------------------------------------------------------------------------------------------
def insert_params(frame_idx: int, normal_guard=0.1, min_scale=1e-4, max_scale_transparent=0.01,
                  cell=0.02) -> _abi.InsertParams:
    return _abi.InsertParams(normal_guard, min_scale, max_scale_transparent, cell, frame_idx)


def insert_workspace_size(n: int, sample_cap: int) -> int:
    return int(lib().rtgs_insert_workspace_size(n, sample_cap))


def add_gaussians(gm: GaussianMap, eta: torch.Tensor, err_count: torch.Tensor, t_created: torch.Tensor,
                  samples: torch.Tensor, add_counts: torch.Tensor, frame_color: torch.Tensor,
                  frame_depth: torch.Tensor, pose: _abi.Pose, cam: _abi.Camera, ip: _abi.InsertParams,
                  result: torch.Tensor, workspace: torch.Tensor, stream=None):
    """Append the Gaussians of the A7 samples after row gm.n (storage rows of gm / eta / err_count /
    t_created must reach gm.capacity).  result[4] (device) = the new n; gm is not resized here."""
    m = _abi.MapRW(_p(gm.store["pos"]), _p(gm.store["log_scale"]), _p(gm.store["rot"]), _p(gm.store["opacity"]),
                   _p(gm.store["sh"]), _p(gm.store["flags"]), _p(eta), _p(err_count), _p(t_created), gm.n, gm.capacity,
                   gm.sh_degree)
    fr = _abi.Frame(_p(frame_color), _p(frame_depth))
    check(lib().rtgs_add_gaussians(C.byref(m), _p(samples), int(samples.numel()), _p(add_counts), C.byref(fr),
                                   C.byref(pose), C.byref(cam), C.byref(ip), _p(result), _p(workspace),
                                   workspace.numel() * workspace.element_size(), _stream(stream)),
          "rtgs_add_gaussians")


# ---------------------------------------------------------------------------------------------
# NEXT f4: frame-to-model ICP tracking
# ---------------------------------------------------------------------------------------------
def icp_params(levels=3, iters=(4, 5, 10), normal_guard=0.1, dist_gate=0.1, angle_gate_deg=30.0, eps=1e-6,
               min_pairs=6) -> _abi.IcpParams:
    it = list(iters) + [0] * (4 - len(iters))
    return _abi.IcpParams(levels, (C.c_int32 * 4)(*it), normal_guard, dist_gate,
                          float(np.cos(np.radians(angle_gate_deg))), eps, min_pairs)


def icp_workspace_size(cam: _abi.Camera, levels: int = 3) -> int:
    return int(lib().rtgs_icp_workspace_size(C.byref(cam), levels))


def pose_device(R, t, device="cuda") -> torch.Tensor:
    """Device double[12] pose buffer (camera->world R row-major, then t) for icp_track."""
    return torch.as_tensor(np.concatenate([np.asarray(R, np.float64).reshape(9), np.asarray(t, np.float64)]),
                           device=device).contiguous()


def icp_track(depth: torch.Tensor, model: RenderBuffers, model_pose: _abi.Pose, cam: _abi.Camera,
              params: _abi.IcpParams, pose_io: torch.Tensor, diag: torch.Tensor, workspace: torch.Tensor,
              stream=None):
    """T_k by multi-level point-to-plane ICP of the current depth against a FULL render `model` of the
    map at model_pose (pose_io: device double[12], in = initial estimate, out = result)."""
    check(lib().rtgs_icp_track(_p(depth), _p(model.depth), _p(model.normal), C.byref(model_pose), C.byref(cam),
                               C.byref(params), _p(pose_io), _p(diag), _p(workspace),
                               workspace.numel() * workspace.element_size(), _stream(stream)), "rtgs_icp_track")


def check_device_flags(stream=None) -> int:
    """rtgs_check_device_flags: synchronise `stream`, read and clear the sticky CAPACITY flag; returns
    the status (RTGS_OK or RTGS_ERR_CAPACITY)."""
    return int(lib().rtgs_check_device_flags(_stream(stream)))


def morton_workspace_size(n: int) -> int:
    return int(lib().rtgs_morton_workspace_size(int(n)))


def morton_order(gm: GaussianMap, stream=None) -> torch.Tensor:
    """Map layout: the permutation (device int32 view of uint32, perm[r] = gid at rank r) that sorts
    the live Gaussians by the Morton code of their position, removed ones last (rtgs_morton_order)."""
    n = gm.n
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=gm.pos.device)[:n]
    ws = torch.empty(max(morton_workspace_size(n), 1), dtype=torch.uint8, device=gm.pos.device)
    check(lib().rtgs_morton_order(_p(gm.pos), _p(gm.flags), n, _p(perm), _p(ws), ws.numel(), _stream(stream)),
          "rtgs_morton_order")
    return perm


def gather_rows(src: torch.Tensor, dst: torch.Tensor, perm: torch.Tensor, stream=None):
    """dst[r] = src[perm[r]] for the first perm.numel() rows (rtgs_gather_rows)."""
    n = int(perm.numel())
    row_bytes = (src.numel() // max(src.shape[0], 1)) * src.element_size()
    check(lib().rtgs_gather_rows(_p(src), _p(dst), _p(perm), n, int(row_bytes), _stream(stream)), "rtgs_gather_rows")


def decode_rgbd(rgb: torch.Tensor, depth_raw: torch.Tensor, depth_scale: float, color: torch.Tensor,
                depth: torch.Tensor, stream=None):
    """Sensor-native frame (uint8 [H,W,3] RGB, uint16 [H,W] depth in raw units) -> planar float32
    color [3,H,W] and depth [H,W] metres, on the device."""
    H, W = int(depth_raw.shape[0]), int(depth_raw.shape[1])
    check(lib().rtgs_decode_rgbd(_p(rgb), _p(depth_raw), W, H, float(depth_scale), _p(color), _p(depth),
                                 _stream(stream)), "rtgs_decode_rgbd")


def coverage_and_bin_cached(proj: ProjectedBuffers, cache: BinBuffers, sub: ProjectedBuffers, sub_gid: torch.Tensor,
                            cam: _abi.Camera, cov: RenderBuffers, out: BinBuffers, workspace: torch.Tensor,
                            stream=None):
    """f3 iteration A0 + A2: coverage / tile keep from the subset's tile lists, then the cached merge."""
    pr = proj.c_struct()
    c = cache.c_struct()
    sp = sub.c_struct()
    cv = cov.c_struct()
    o = out.c_struct()
    check(lib().rtgs_coverage_and_bin_cached(C.byref(pr), C.byref(c), C.byref(sp), _p(sub_gid),
                                             int(sub_gid.numel()), C.byref(cam), C.byref(cv), C.byref(o),
                                             _p(workspace), workspace.numel() * workspace.element_size(),
                                             _stream(stream)), "rtgs_coverage_and_bin_cached")
    out.sub = (sub.rec, sub.zkey, sub_gid)


def coverage_subset(sub: ProjectedBuffers, n_sub: int, cam: _abi.Camera, cov: RenderBuffers, capacity: int,
                    workspace: torch.Tensor, stream=None):
    """f3 part 1: coverage / tile keep from the subset's tile lists (left in the workspace)."""
    sp = sub.c_struct()
    cv = cov.c_struct()
    check(lib().rtgs_coverage_subset(C.byref(sp), int(n_sub), C.byref(cam), C.byref(cv), int(capacity), _p(workspace),
                                     workspace.numel() * workspace.element_size(), _stream(stream)),
          "rtgs_coverage_subset")


def merge_cached(proj: ProjectedBuffers, cache: BinBuffers, sub: ProjectedBuffers, sub_gid: torch.Tensor,
                 cam: _abi.Camera, cov: RenderBuffers, out: BinBuffers, workspace: torch.Tensor, stream=None):
    """f3 part 2: merge the kept tiles' subset lists with the cached stable lists."""
    pr = proj.c_struct()
    c = cache.c_struct()
    sp = sub.c_struct()
    cv = cov.c_struct()
    o = out.c_struct()
    check(lib().rtgs_merge_cached(C.byref(pr), C.byref(c), C.byref(sp), _p(sub_gid), int(sub_gid.numel()),
                                  C.byref(cam), C.byref(cv), C.byref(o), _p(workspace),
                                  workspace.numel() * workspace.element_size(), _stream(stream)), "rtgs_merge_cached")
    out.sub = (sub.rec, sub.zkey, sub_gid)


# ---------------------------------------------------------------------------------------------
# (e) keyframe global optimisation
# ---------------------------------------------------------------------------------------------
def topk_workspace_size(cam: _abi.Camera) -> int:
    return int(lib().rtgs_topk_workspace_size(C.byref(cam)))


def topk_error_mask(full: RenderBuffers, frame_color: torch.Tensor, cam: _abi.Camera, ratio: float,
                    out: RenderBuffers, workspace: torch.Tensor, stream=None):
    """Active set = the top `ratio` colour-error pixels of the FULL render `full` (written to `out`'s
    active bits, tile keep / list and counts; `out` may be `full` itself)."""
    o = out.c_struct()
    check(lib().rtgs_topk_error_mask(_p(full.color), _p(frame_color), C.byref(cam), float(ratio), C.byref(o),
                                     _p(workspace), workspace.numel() * workspace.element_size(), _stream(stream)),
          "rtgs_topk_error_mask")


def hparams(preset: str = "replica") -> _abi.HParams:
    """Learning rates of P:501: Replica / ScanNet++ vs Azure / TUM."""
    if preset in ("replica", "scannetpp"):
        lr_pos, lr_sh0, lr_scale, lr_rot = 1e-3, 5e-4, 4e-3, 1e-3
    else:
        lr_pos, lr_sh0, lr_scale, lr_rot = 1e-3, 1e-3, 2e-3, 1e-3
    return _abi.HParams(lr_pos, lr_sh0, 0.05 * lr_sh0, lr_scale, lr_rot, 0.9, 0.999, 1e-15)


def add_params(seed=0, frame_idx=0, delta_T=0.5, delta_d=0.1, delta_c=0.1, ratio=0.05) -> _abi.AddParams:
    return _abi.AddParams(delta_T, delta_d, delta_c, ratio, seed, frame_idx)


# ---------------------------------------------------------------------------------------------
class MappingEngine:
    """Device buffers + the per-frame call sequence for one camera and one Gaussian map."""

    def __init__(self, gm: GaussianMap, cam: _abi.Camera, capacity: int | None = None, preset="replica",
                 weights=(1.0, 1.0, 1000.0), sample_cap: int | None = None, device="cuda", cache_frames: int = 1):
        self.gm, self.cam, self.device = gm, cam, device
        n = gm.capacity  # per-Gaussian buffers are sized for the map's storage (f2 appends rows)
        self.capacity = int(capacity if capacity is not None else max(4 * n, 1 << 16))
        # the masked iteration and the frame ingest own separate buffers so they can run concurrently
        self.proj = ProjectedBuffers(n, device)
        self.bins = BinBuffers(cam, self.capacity, device)
        self.out = RenderBuffers(cam, device, count_blends=False)  # production MASKED render: no statistic
        self.ws_bin = torch.empty(bin_workspace_size(n, cam, self.capacity), dtype=torch.uint8, device=device)
        self.proj_full = ProjectedBuffers(n, device)
        self.bins_full = BinBuffers(cam, self.capacity, device)
        self.full = RenderBuffers(cam, device, count_blends=False)  # production FULL render: no statistic
        self.full.track_last = False  # (A7, f1 states and f4 tracking read no n_contrib)
        self.ws_bin_full = torch.empty(bin_workspace_size(n, cam, self.capacity), dtype=torch.uint8, device=device)
        self.side = torch.cuda.Stream(device=device)
        self.ws_cls = torch.empty(classify_workspace_size(cam), dtype=torch.uint8, device=device)
        self.weights = weights
        self.hp = hparams(preset)
        self.loss = torch.zeros(4, dtype=torch.float32, device=device)
        HW = cam.width * cam.height
        self.pixel_class = torch.zeros((cam.height, cam.width), dtype=torch.uint8, device=device)
        self.samples = torch.zeros(sample_cap if sample_cap is not None else max(HW // 8, 1), dtype=torch.int32,
                                   device=device)
        self.add_counts = torch.zeros(5, dtype=torch.int32, device=device)
        # per-Gaussian state (storage of capacity rows; the attributes are views of the live rows)
        self._state_store = {k: torch.zeros(n, dtype=torch.int32, device=device)
                             for k in ("eta", "err_count", "t_created")}
        # L_reg anchors ("remaining the same as their initial values", R18): each Gaussian's
        # geometry (pos 3, log-scale 3, rot 4) when it entered the map, per gid; the map handed to the
        # engine counts as inserted now, f2 rows are recorded at insertion
        self._anchor = torch.zeros((n, 10), dtype=torch.float32, device=device)
        self._record_anchor(0, gm.n)
        self._map_version = 0  # bumped whenever n or the flags change (global-step bookkeeping)
        self._view_state()
        self.state_counts = torch.zeros(4, dtype=torch.int32, device=device)
        self.ws_state = torch.empty(state_workspace_size(n), dtype=torch.uint8, device=device)
        # NEXT f2: insertion workspace and result (#opaque, #transparent, #skipped, #dropped, n after)
        self.ws_insert = torch.empty(insert_workspace_size(n, self.samples.numel()), dtype=torch.uint8, device=device)
        self.insert_result = torch.zeros(5, dtype=torch.int32, device=device)
        # NEXT f3: the stable part of the last ingested frame's sorted lists (valid for its pose and
        # until the stable set changes at the window end)
        # (one per window frame: `cache_frames` frames are kept, least recently ingested replaced first;
        # slot 0 reuses proj_full so a single-frame engine allocates nothing extra)
        self.cache_frames = max(1, int(cache_frames))
        self._fc = [_FrameCache(self.proj_full, BinBuffers(cam, self.capacity, device))]
        self._fc_clock = 0
        self.use_cache = True
        self.fused_adam = True
        self.reset_window()

    def reorder_spatially(self, stream=None) -> torch.Tensor:
        """Map layout (not a step of the method): put the map in Morton order (rtgs_morton_order) and
        carry every per-Gaussian array along (parameters, flags, eta, e, t, L_reg anchors); the f3
        caches and the window slots are rebuilt.  Gids change: returns perm (new row r = old gid
        perm[r]).  The paper's maps, grown from row-major pixel samples frame by frame, are
        spatially coherent already; this restores that for a map handed over in arbitrary order."""
        perm = morton_order(self.gm, stream)
        self.gm.permute(perm, stream)
        n = self.gm.n
        for k, v in list(self._state_store.items()):
            new = v.clone()
            if n:
                gather_rows(v[:n], new, perm, stream)
            self._state_store[k] = new
        a = self._anchor.clone()
        if n:
            gather_rows(self._anchor[:n], a, perm, stream)
        self._anchor = a
        self._view_state()
        self._drop_cache()
        self._map_version += 1
        self.reset_window()
        return perm

    def _record_anchor(self, r0: int, r1: int, stream=None):
        if r1 > r0:
            with torch.cuda.stream(torch.cuda.current_stream() if stream is None else stream):
                self._anchor[r0:r1, 0:3] = self.gm.pos[r0:r1]
                self._anchor[r0:r1, 3:6] = self.gm.log_scale[r0:r1]
                self._anchor[r0:r1, 6:10] = self.gm.rot[r0:r1]

    def _view_state(self):
        n = self.gm.n
        self.eta = self._state_store["eta"][:n]            # eta_i
        self.err_count = self._state_store["err_count"][:n]  # e_i
        self.t_created = self._state_store["t_created"][:n]  # t_i

    def reserve(self, capacity: int):
        """Grow the map storage and every per-Gaussian buffer to `capacity` rows.  Live rows and the
        per-Gaussian state are kept; the f3 frame caches are dropped (re-ingest to rebuild them) and
        the window slots are rebuilt (Adam state reset, R19)."""
        if capacity <= self.gm.capacity:
            return
        torch.cuda.synchronize(self.device)
        self.gm.reserve(capacity)
        for k, v in list(self._state_store.items()):
            t = torch.zeros(capacity, dtype=v.dtype, device=self.device)
            t[: v.numel()].copy_(v)
            self._state_store[k] = t
        a = torch.zeros((capacity, 10), dtype=torch.float32, device=self.device)
        a[: self._anchor.shape[0]].copy_(self._anchor)
        self._anchor = a
        self._map_version += 1
        self._view_state()
        n, cam = capacity, self.cam
        self.proj = ProjectedBuffers(n, self.device)
        self.proj_full = ProjectedBuffers(n, self.device)
        self.ws_bin = torch.empty(bin_workspace_size(n, cam, self.capacity), dtype=torch.uint8, device=self.device)
        self.ws_bin_full = torch.empty(bin_workspace_size(n, cam, self.capacity), dtype=torch.uint8,
                                       device=self.device)
        self.ws_state = torch.empty(state_workspace_size(n), dtype=torch.uint8, device=self.device)
        self.ws_insert = torch.empty(insert_workspace_size(n, self.samples.numel()), dtype=torch.uint8,
                                     device=self.device)
        self._fc = [_FrameCache(self.proj_full, self._fc[0].cache)]
        self._fc_clock = 0
        self.reset_window()

    def reserve_instances(self, capacity: int):
        """Grow the (Gaussian, tile) instance capacity of every binning buffer to `capacity`; the f3
        frame caches are dropped (re-ingest to rebuild them)."""
        if capacity <= self.capacity:
            return
        torch.cuda.synchronize(self.device)
        self.capacity = int(capacity)
        n, cam = self.gm.capacity, self.cam
        self.bins = BinBuffers(cam, self.capacity, self.device)
        self.bins_full = BinBuffers(cam, self.capacity, self.device)
        self.ws_bin = torch.empty(bin_workspace_size(n, cam, self.capacity), dtype=torch.uint8, device=self.device)
        self.ws_bin_full = torch.empty(bin_workspace_size(n, cam, self.capacity), dtype=torch.uint8,
                                       device=self.device)
        self._fc = [_FrameCache(self.proj_full, BinBuffers(cam, self.capacity, self.device))]
        self._fc_clock = 0
        self.reset_window()

    def insert(self, frame_color, frame_depth, pose: _abi.Pose, frame_idx: int, stream=None, sync=True,
               grow: bool = True):
        """NEXT f2 after an ingest of the same frame: append the Gaussians of its A7 samples
        (Eq.11).  With sync=True the new count is read back and the map / state views
        grow; call reset_window() before optimising so the new (unstable) Gaussians get slots.
        With sync and grow, the storage is first enlarged (reserve, x1.5) when the frame's samples
        may not fit; otherwise rows past the capacity are dropped (counted in result[3])."""
        if sync and grow:
            (torch.cuda.current_stream() if stream is None else stream).synchronize()
            want = self.gm.n + min(int(self.add_counts[2].item()) + int(self.add_counts[3].item()),
                                   self.samples.numel())
            if want > self.gm.capacity:
                self.reserve(max(want, self.gm.capacity * 3 // 2))
        add_gaussians(self.gm, self._state_store["eta"], self._state_store["err_count"],
                      self._state_store["t_created"], self.samples, self.add_counts, frame_color, frame_depth, pose,
                      self.cam, insert_params(frame_idx), self.insert_result, self.ws_insert, stream)
        if sync:
            (torch.cuda.current_stream() if stream is None else stream).synchronize()
            n_old, n_new = self.gm.n, int(self.insert_result[4].item())
            self.gm.resize(n_new)
            self._view_state()
            self._record_anchor(n_old, n_new, stream)  # L_reg anchors of the new Gaussians
            self._map_version += 1
        # (the f3 cache stays valid: new Gaussians are unstable, the stable lists are unchanged)
        return self.insert_result

    def track(self, frame_depth, model_pose: _abi.Pose, init_pose: torch.Tensor | None = None, params=None,
              stream=None):
        """NEXT f4: render the optimised map at the previous pose (A1, A2, A3/A4 FULL; depth and world
        normals) and track the current frame against it by ICP.  Returns the device pose buffer
        (double[12]) and the per-iteration diagnostics (device)."""
        params = params or icp_params()
        if not hasattr(self, "ws_icp"):
            self.ws_icp = torch.empty(icp_workspace_size(self.cam, 4), dtype=torch.uint8, device=self.device)
            self.icp_diag = torch.zeros((4 * 40,), dtype=torch.float64, device=self.device)
        project_gaussians(self.gm, model_pose, self.cam, self.proj_full, stream)
        bin_and_sort(self.proj_full, self.gm.n, self.cam, None, self.bins_full, self.ws_bin_full, stream)
        render_color_depth(self.gm, self.proj_full, self.bins_full, model_pose, self.cam, RTGS_RENDER_FULL, self.full,
                           stream)
        self._drop_cache(self.proj_full)  # proj_full now holds the model pose's frame
        pose_io = init_pose if init_pose is not None else pose_device(np.asarray(model_pose.R).reshape(3, 3),
                                                                      np.asarray(model_pose.t), self.device)
        with torch.cuda.stream(torch.cuda.current_stream() if stream is None else stream):
            self.icp_diag.fill_(-1.0)  # rows past sum(iters) stay marked unused
        icp_track(frame_depth, self.full, model_pose, self.cam, params, pose_io, self.icp_diag, self.ws_icp, stream)
        return pose_io, self.icp_diag

    def _buf(self, name: str, rows: int, tail: tuple = (), dtype=torch.float32, cap_rows: int | None = None):
        """First `rows` rows of a persistent device buffer that only grows (to >= cap_rows, x1.25), so
        successive windows with different slot counts reuse their memory instead of reallocating."""
        b = self._bufs.get(name)
        if b is None or b.shape[0] < rows or tuple(b.shape[1:]) != tuple(tail) or b.dtype != dtype:
            cap = max(rows, 1, int(b.shape[0] * 1.25) if b is not None and tuple(b.shape[1:]) == tuple(tail) else 0,
                      cap_rows or 0)
            b = torch.empty((cap,) + tuple(tail), dtype=dtype, device=self.device)
            self._bufs[name] = b
        return b[:rows]

    def reset_window(self):
        """(Re)build the unstable slot set from flags and reset the Adam state (R19: per window).
        On the device (one host synchronisation for the slot count); buffers are reused across windows."""
        if not hasattr(self, "_bufs"):
            self._bufs = {}
        n = self.gm.n
        flags = self.gm.flags
        gid_t = torch.nonzero((flags & FLAG_STABLE) == 0).flatten()  # (the host learns the count here)
        n_slots = int(gid_t.numel())
        cap = self.gm.capacity  # slot-indexed buffers hold the whole storage: no window reallocates them
        # N_t of R18: transparent slots that are not removed (removed Gaussians are culled, no L_reg)
        self.n_transparent = int(((flags[gid_t] & (FLAG_TRANSPARENT | FLAG_REMOVED)) == FLAG_TRANSPARENT).sum()) \
            if n_slots else 0
        self.gid_of_slot = self._buf("gid_of_slot", n_slots, (), torch.int32, cap_rows=cap)
        self.gid_of_slot.copy_(gid_t)
        self.slot_of_gid = self._buf("slot_of_gid", n, (), torch.int32, cap_rows=cap)
        self.slot_of_gid.fill_(-1)
        if n_slots:
            self.slot_of_gid[gid_t] = torch.arange(n_slots, dtype=torch.int32, device=self.device)
        D = 10 + 3 * (self.gm.sh_degree + 1) ** 2
        rows = max(n_slots, 1)
        self.grad = self._buf("grad", rows, (D,), cap_rows=cap)
        self.m = self._buf("m", rows, (D,), cap_rows=cap)
        self.v = self._buf("v", rows, (D,), cap_rows=cap)
        for t in (self.grad, self.m, self.v):
            t.zero_()
        # window start: parameters and eta of the slots, for L_reg (init_geom) and the Eq.9 fusion at
        # the window end (f1)
        self.before = self._buf("before", rows, (D,), cap_rows=cap)
        self.eta_before = self._buf("eta_before", rows, (), torch.int32, cap_rows=cap)
        if n_slots:
            for k, (c0, c1) in (("pos", (0, 3)), ("log_scale", (3, 6)), ("rot", (6, 10))):
                self.before[:, c0:c1] = getattr(self.gm, k)[gid_t]
            shg = self._buf("sh_gather", n_slots, (D - 10,), cap_rows=cap)
            torch.index_select(self.gm.sh.reshape(n, D - 10), 0, gid_t, out=shg)
            self.before[:, 10:] = shg
            torch.index_select(self.eta, 0, gid_t, out=self.eta_before)
        else:
            self.before.zero_()
            self.eta_before.zero_()
        # L_reg anchors of the slots: each Gaussian's geometry at insertion, gathered by gid
        self.init_geom = self._buf("init_geom", rows, (10,), cap_rows=cap)
        if n_slots:
            torch.index_select(self._anchor[:n], 0, gid_t, out=self.init_geom)
        else:
            self.init_geom.zero_()
        self.ws_bwd = self._buf("ws_bwd", backward_workspace_size(n_slots), (), torch.uint8,
                                cap_rows=backward_workspace_size(cap))
        self.step_count = 0
        if getattr(self, "step_dev", None) is None:
            self.step_dev = torch.zeros(1, dtype=torch.int32, device=self.device)  # graph-replayable step
        else:
            self.step_dev.zero_()
        # f3: the slots' own projection rows and the cached-binning workspace (the cache itself is
        # invalidated where the stable set changes: end_window)
        if getattr(self, "proj_sub", None) is None or self.proj_sub.rec.shape[0] < n_slots:
            self.proj_sub = ProjectedBuffers(max(n_slots, cap), self.device)
        self.ws_bin_cached = self._buf("ws_bin_cached", bin_cached_workspace_size(n_slots, self.cam, self.capacity), (),
                                       torch.uint8, cap_rows=bin_cached_workspace_size(cap, self.cam, self.capacity))
        self.proj_iter = self.proj

    # --- the two flows ---------------------------------------------------------------------------
    def ingest(self, frame_color, frame_depth, pose: _abi.Pose, seed=0, frame_idx=0, stream=None, after_project=None):
        """A1 -> A2 (all tiles) -> A3/A4 FULL -> A7.  `after_project(stream)` is called once
        the projection (the last read of the parameters) has been enqueued."""
        fc = self._cache_slot(pose) if self.use_cache else None
        if fc is not None:
            fc.key = None          # rebuilt below
            self.proj_full = fc.proj
        # (f3: with a frame cache the tile sort also writes this frame's stable lists, reused by the
        # window's iterations)
        project_and_bin(self.gm, pose, self.cam, self.proj_full, self.bins_full, self.ws_bin_full, stream,
                        cache=fc.cache if fc is not None else None)
        if after_project is not None:
            after_project(stream)
        if fc is not None:
            fc.ready.record(torch.cuda.current_stream() if stream is None else stream)
            fc.key = _pose_key(pose)
        render_color_depth(self.gm, self.proj_full, self.bins_full, pose, self.cam, RTGS_RENDER_FULL, self.full, stream,
                           normals=False)  # (A7 reads no normals; track() renders its own)
        classify_and_add_pixels(self.full, frame_color, frame_depth, self.gm.flags, self.cam,
                                add_params(seed=seed, frame_idx=frame_idx), self.pixel_class, self.samples,
                                self.add_counts, self.ws_cls, stream)

    # --- f3 frame caches -------------------------------------------------------------------------
    def _cache_slot(self, pose: _abi.Pose) -> "_FrameCache":
        key = _pose_key(pose)
        for fc in self._fc:
            if fc.key == key:
                break
        else:
            if len(self._fc) < self.cache_frames:
                fc = _FrameCache(ProjectedBuffers(self.gm.capacity, self.device),
                                 BinBuffers(self.cam, self.capacity, self.device))
                self._fc.append(fc)
            else:
                fc = min(self._fc, key=lambda f: f.stamp)   # least recently ingested
        self._fc_clock += 1
        fc.stamp = self._fc_clock
        return fc

    def _lookup_cache(self, pose: _abi.Pose):
        key = _pose_key(pose)
        for fc in self._fc:
            if fc.key is not None and fc.key == key:
                return fc
        return None

    def _drop_cache(self, proj=None):
        """Invalidate the frame caches (all, or the one whose projection buffer is `proj`)."""
        for fc in self._fc:
            if proj is None or fc.proj is proj:
                fc.key = None

    @property
    def cache(self) -> BinBuffers:
        """The stable-list cache of the frame currently in proj_full (the last ingested one)."""
        for fc in self._fc:
            if fc.proj is self.proj_full:
                return fc.cache
        return self._fc[0].cache

    def cached(self, pose: _abi.Pose) -> bool:
        """True when an f3 stable cache holds this pose's lists for the current stable set."""
        return self.use_cache and self._lookup_cache(pose) is not None

    def forward_masked(self, pose: _abi.Pose, stream=None):
        """A1 -> A0 -> A2 (kept tiles) -> A3/A4 MASKED (Eq.12).  With a valid f3 cache
        only the unstable slots are projected and binned; the stable lists come from the cache."""
        fc = self._lookup_cache(pose) if self.use_cache else None
        if fc is not None:
            project_subset(self.gm, self.gid_of_slot, pose, self.cam, self.proj_sub, stream)
            coverage_subset(self.proj_sub, int(self.gid_of_slot.numel()), self.cam, self.out, self.capacity,
                            self.ws_bin_cached, stream)
            (torch.cuda.current_stream() if stream is None else stream).wait_event(fc.ready)
            merge_cached(fc.proj, fc.cache, self.proj_sub, self.gid_of_slot, self.cam, self.out, self.bins,
                         self.ws_bin_cached, stream)
            self.proj_iter = fc.proj
        else:
            project_gaussians(self.gm, pose, self.cam, self.proj, stream)
            render_color_depth(self.gm, self.proj, None, pose, self.cam, RTGS_RENDER_COVERAGE, self.out, stream)
            bin_and_sort(self.proj, self.gm.n, self.cam, self.out.tile_keep, self.bins, self.ws_bin, stream)
            self.bins.sub = None
            self.proj_iter = self.proj
        render_color_depth(self.gm, self.proj_iter, self.bins, pose, self.cam, RTGS_RENDER_MASKED, self.out, stream)

    def backward(self, frame_color, frame_depth, pose: _abi.Pose, stream=None):
        render_backward_masked(self.gm, self.proj_iter, self.bins, pose, self.cam, self.out, frame_color, frame_depth,
                               self.weights, self.slot_of_gid, self.gid_of_slot, self.grad, self.loss, self.ws_bwd,
                               stream)

    def optimizer_step(self, stream=None):
        """A6.  The window step lives on the device (incremented here, read by the kernel), so a
        captured CUDA graph of the iteration advances the bias correction on every replay."""
        self.step_count += 1
        s = torch.cuda.current_stream() if stream is None else stream
        with torch.cuda.stream(s):
            self.step_dev.add_(1)
        adam_step_unstable(self.gm, self.gid_of_slot, self.grad, self.m, self.v, self.init_geom, self.n_transparent,
                           self.weights[2], self.hp, self.step_count, self.eta, stream, step_device=self.step_dev)

    def backward_adam(self, frame_color, frame_depth, pose: _abi.Pose, stream=None):
        """A5 + A6 fused (fused_adam): the slot gradient stays on chip; same result as backward()
        followed by optimizer_step()."""
        self.step_count += 1
        s = torch.cuda.current_stream() if stream is None else stream
        with torch.cuda.stream(s):
            self.step_dev.add_(1)
        backward_adam_unstable(self.gm, self.proj_iter, self.bins, pose, self.cam, self.out, frame_color, frame_depth,
                               self.weights, self.slot_of_gid, self.gid_of_slot, self.m, self.v, self.init_geom,
                               self.n_transparent, self.hp, self.step_count, self.eta, self.loss, self.ws_bwd, stream,
                               step_device=self.step_dev)

    def iteration(self, frame_color, frame_depth, pose: _abi.Pose, stream=None):
        """One mapping optimisation iteration A0-A6 (the paper's 'mapping / iteration').  With
        fused_adam (default) A5 and A6 are one kernel pair; the separate calls remain for gradient
        accumulation and all-reduce (keyframe step, multi-GPU)."""
        self.forward_masked(pose, stream)
        if self.fused_adam:
            self.backward_adam(frame_color, frame_depth, pose, stream)
        else:
            self.backward(frame_color, frame_depth, pose, stream)
            self.optimizer_step(stream)

    def end_window(self, frame_color, frame_depth, pose: _abi.Pose, frame_idx: int, state=None, stream=None):
        """NEXT f1, after a window's iterations: Eq.9 fusion with the window-start parameters, then the
        optimised scene's FULL render at frame k and the state transitions.  The slot set
        and optimiser state are rebuilt for the next window."""
        fuse_window(self.gm, self.gid_of_slot, self.before, self.eta_before, self.eta, stream)
        project_gaussians(self.gm, pose, self.cam, self.proj_full, stream)
        bin_and_sort(self.proj_full, self.gm.n, self.cam, None, self.bins_full, self.ws_bin_full, stream)
        render_color_depth(self.gm, self.proj_full, self.bins_full, pose, self.cam, RTGS_RENDER_FULL, self.full, stream,
                           normals=False)
        sp = state if state is not None else state_params(frame_idx)
        manage_states(self.full, frame_color, frame_depth, self.cam, self.gm.flags, self.err_count, self.eta,
                      self.t_created, sp, self.state_counts, self.ws_state, stream)
        self._drop_cache()  # the stable set changed: every f3 cache is stale
        self._map_version += 1
        self.reset_window()

    def map_window(self, frames, iterations=50, seed=0, first_frame_idx=0, insert=True):
        """The paper's mapping window: for every window frame (colour, depth, pose):
        ingest (A1, A2, A3/A4 FULL, A7, its f3 stable cache) and insert its sampled Gaussians (f2);
        then a new slot set and `iterations` masked iterations, each on a uniformly sampled window
        frame (f3-cached when cache_frames >= len(frames)); then Eq.9 fusion and the state
        transitions on the last frame (f1).  Returns the device loss buffer of the last iteration."""
        rng = np.random.default_rng(seed)
        for i, (c, d, pose) in enumerate(frames):
            self.ingest(c, d, pose, seed=seed, frame_idx=first_frame_idx + i)
            need = int(self.bins_full.n_instances.item())
            # keep 25 % headroom over the FULL lists: the window's iterations bin the map as it is after
            # ALL the window's insertions, which can exceed an earlier frame's FULL count
            if need * 5 // 4 > self.capacity:
                truncated = need > self.capacity
                self.reserve_instances(need * 3 // 2)
                if truncated:                   # the FULL lists were cut short: redo the frame
                    check_device_flags()        # (that overflow is handled: clear the sticky flag)
                    self.ingest(c, d, pose, seed=seed, frame_idx=first_frame_idx + i)
            if insert:
                self.insert(c, d, pose, frame_idx=first_frame_idx + i)
        self.reset_window()
        for _ in range(iterations):
            c, d, pose = frames[int(rng.integers(len(frames)))]
            self.iteration(c, d, pose)
        loss = self.loss.clone()
        self.check_capacity()
        c, d, pose = frames[-1]
        self.end_window(c, d, pose, frame_idx=first_frame_idx + len(frames) - 1)
        return loss

    def check_capacity(self, stream=None):
        """Raise if any binning since the last check overflowed its instance capacity (the outputs were
        truncated: memory-safe but invalid) — the sticky device flag of rtgs_check_device_flags.  One
        host synchronisation."""
        st = check_device_flags(stream)
        if st == _abi.RTGS_ERR_CAPACITY:
            worst = max(int(self.bins.n_instances.item()), int(self.bins_full.n_instances.item()))
            raise RuntimeError(f"instance capacity {self.capacity} exceeded (last binnings: {worst}): construct "
                               f"the MappingEngine with a larger capacity")
        check(st, "rtgs_check_device_flags")

    # --- (e) keyframe global optimisation -------------------------------------------------------
    def _global_state(self, world: int = 1):
        """(e) slots = EVERY row of the map, slot == gid (R37: every non-removed Gaussian is optimised;
        removed rows are culled by A1, get no gradient and no L_reg term, so their Adam step is an
        exact no-op).  The gradient buffer has `world` equal blocks of rows (the reduce-scatter
        shards), the map storage is grown to the padded row count (the in-place all-gathers).  Rebuilt
        only when the map changed (n or flags, `_map_version`) or the world size did: no host
        synchronisation per step."""
        n = self.gm.n
        key = (n, self._map_version, world)
        if getattr(self, "_g_key", None) == key:
            return
        per = max(1, -(-n // world))
        padded = per * world
        if padded > self.gm.capacity:
            self.reserve(padded)
            key = (n, self._map_version, world)
        D = 10 + 3 * (self.gm.sh_degree + 1) ** 2
        self.g_per, self.g_rows = per, padded
        self.g_gid = torch.arange(n, dtype=torch.int32, device=self.device)
        self.g_slot = self.g_gid
        self.g_grad = torch.zeros((padded, D), dtype=torch.float32, device=self.device)
        self.g_m = torch.zeros_like(self.g_grad)
        self.g_v = torch.zeros_like(self.g_grad)
        self.g_ws_bwd = torch.empty(backward_workspace_size(padded), dtype=torch.uint8, device=self.device)
        flags = self.gm.flags
        self.g_ntr = int(((flags & (FLAG_TRANSPARENT | FLAG_REMOVED)) == FLAG_TRANSPARENT).sum())  # (one sync)
        self.g_rb = RenderBuffers(self.cam, self.device, count_blends=False)
        self.g_ws_topk = torch.empty(topk_workspace_size(self.cam), dtype=torch.uint8, device=self.device)
        self.g_loss = torch.zeros(4, dtype=torch.float32, device=self.device)
        self._g_key = key

    def global_backward(self, views, ratio=0.4, stream=None, n_total=None, world: int = 1):
        """(e) P:284, per keyframe view (colour, depth, pose): FULL render (A1, A2, A3/A4), its top
        `ratio` colour-error pixels (K9), the masked backward over ALL non-removed Gaussians with the
        loss weights divided by the number of views (the batch loss is the mean over the views),
        accumulated into g_grad.  Multi-GPU: every rank calls this on its share of the views."""
        self._global_state(world)
        nv = n_total if n_total is not None else len(views)   # multi-GPU: the views of ALL ranks
        w = tuple(x / max(1, nv) for x in self.weights[:2]) + (self.weights[2],)
        for (c, d, pose) in views:
            project_and_bin(self.gm, pose, self.cam, self.proj, self.bins, self.ws_bin, stream)
            render_color_depth(self.gm, self.proj, self.bins, pose, self.cam, RTGS_RENDER_FULL, self.g_rb, stream)
            topk_error_mask(self.g_rb, c, self.cam, ratio, self.g_rb, self.g_ws_topk, stream)
            render_backward_masked(self.gm, self.proj, self.bins, pose, self.cam, self.g_rb, c, d, w, self.g_slot,
                                   self.g_gid, self.g_grad, self.g_loss, self.g_ws_bwd, stream)

    def _global_hparams(self, lr_scale):
        hp = self.hp
        return _abi.HParams(0.0, hp.lr_sh0 * lr_scale, hp.lr_shrest * lr_scale, hp.lr_scale * lr_scale,
                            hp.lr_rot * lr_scale, hp.beta1, hp.beta2, hp.eps)

    def global_adam_block(self, r0: int, r1: int, lr_scale=0.1, stream=None):
        """(e) the Adam step of the global slots (= rows) [r0, r1) clipped to n, from their summed
        gradient rows g_grad[r0:r1] (consumed) with fresh moments (R37), position lr 0, the other
        rates x lr_scale, and L_reg against the insertion anchors (R18); writes those rows of the map
        and of eta in place."""
        n = self.gm.n
        a, b = min(r0, n), min(r1, n)
        if b <= a:
            return
        s = torch.cuda.current_stream() if stream is None else stream
        with torch.cuda.stream(s):
            self.g_m[a:b].zero_()
            self.g_v[a:b].zero_()
        adam_step_unstable(self.gm, self.g_gid[a:b], self.g_grad[a:b], self.g_m[a:b], self.g_v[a:b],
                           self._anchor[a:b], self.g_ntr, self.weights[2], self._global_hparams(lr_scale), 1,
                           self.eta, stream)

    def global_step(self, views, ratio=0.4, lr_scale=0.1, reduce_grads=None, stream=None, n_total=None):
        """(e) one global optimisation step: global_backward over `views`, the gradient sum
        over ranks (`reduce_grads(g_grad)`, multi-GPU: every rank then runs the identical update),
        then one Adam step of every Gaussian with the position learning rate 0 and the others
        x lr_scale (reading R37: fresh moments per global step; L_reg against the insertion anchors,
        R18).  The sharded form is dist.global_step_sharded."""
        self.global_backward(views, ratio, stream, n_total)
        if reduce_grads is not None:
            reduce_grads(self.g_grad)
        self.global_adam_block(0, self.g_rows, lr_scale, stream)
        return self.g_loss

    def step(self, frame_color, frame_depth, pose: _abi.Pose, ingest_pose=None, seed=0, frame_idx=0,
             reduce_grads=None):
        """Frame ingest (A1, A2, A3/A4 FULL, A7) and one masked iteration (A0-A6) on two streams.

        The ingest runs on a side stream concurrently with the iteration on the current stream (the
        paper runs mapping stages in parallel threads); the only dependency is that the Adam
        step, which writes the parameters, waits until the ingest's projection has read them.
        `reduce_grads(grad)` (multi-GPU) runs between the backward and the Adam step; without it the
        two are the fused call (fused_adam)."""
        main = torch.cuda.current_stream()
        side = self.side
        side.wait_stream(main)
        proj_done = torch.cuda.Event()
        self.ingest(frame_color, frame_depth, ingest_pose or pose, seed=seed, frame_idx=frame_idx, stream=side,
                    after_project=lambda s: proj_done.record(s))
        self.forward_masked(pose, main)
        if reduce_grads is None and self.fused_adam:
            main.wait_event(proj_done)  # (long done: the projection is the ingest's first kernel)
            self.backward_adam(frame_color, frame_depth, pose, main)
        else:
            self.backward(frame_color, frame_depth, pose, main)
            if reduce_grads is not None:
                reduce_grads(self.grad)
            main.wait_event(proj_done)
            self.optimizer_step(main)
        main.wait_stream(side)


class _FrameCache:
    """NEXT f3: one window frame's projection (stable rows read by the iterations) and the stable
    part of its sorted tile lists."""

    def __init__(self, proj: ProjectedBuffers, cache: BinBuffers):
        self.proj, self.cache = proj, cache
        self.ready = torch.cuda.Event()
        self.key = None
        self.stamp = 0


def _pose_key(pose: _abi.Pose) -> tuple:
    return tuple(pose.R) + tuple(pose.t)


def launch_count() -> int:
    return int(lib().rtgs_launch_count())
