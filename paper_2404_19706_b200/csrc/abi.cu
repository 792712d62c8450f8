// abi.cu — the extern "C" boundary of librtgs.so (include/rtgs.h): host-side argument validation,
// then the launchers of internal.h.  No CPU fallback exists: every call either enqueues the CUDA
// kernels or returns an error status.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace rtgs {
static std::atomic<uint64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
}  // namespace rtgs

using namespace rtgs;

namespace {
thread_local char g_cuda_err[256] = "";

inline bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool a4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }

bool cam_ok(const rtgs_camera* c) {
  return c && std::isfinite(c->fx) && std::isfinite(c->fy) && std::isfinite(c->cx) && std::isfinite(c->cy) &&
         c->fx > 0.f && c->fy > 0.f && c->width >= 1 && c->height >= 1 && c->width <= 16384 && c->height <= 16384;
}
bool pose_ok(const rtgs_pose* p) {
  if (!p) return false;
  for (double v : p->R)
    if (!std::isfinite(v)) return false;
  for (double v : p->t)
    if (!std::isfinite(v)) return false;
  return true;
}
bool gauss_ok(const rtgs_gaussians* g, bool need_flags) {
  if (!g || g->n < 0 || g->sh_degree < 0 || g->sh_degree > 3) return false;
  if (g->n == 0) return true;
  if (!g->pos || !g->log_scale || !g->rot || !g->opacity || !g->sh) return false;
  if (need_flags && !g->flags) return false;
  return a16(g->pos) && a4(g->log_scale) && a16(g->rot) && a4(g->opacity) && a16(g->sh);
}
bool proj_ok(const rtgs_projected* p, int n) {
  if (!p) return false;
  if (n == 0) return true;
  return p->rec && p->zkey && p->rect && p->tiles_touched && a16(p->rec) && a4(p->zkey) &&
         (reinterpret_cast<uintptr_t>(p->rect) & 7u) == 0 && a4(p->tiles_touched);
}
bool bins_ok(const rtgs_bins* b) {
  return b && b->sorted_gid && b->tile_range && b->n_instances && (reinterpret_cast<uintptr_t>(b->tile_range) & 7u) == 0;
}
rtgs_status finish(cudaError_t e) {
  if (e == cudaSuccess) return RTGS_OK;
  std::snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return RTGS_ERR_CUDA;
}
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

rtgs_status rtgs_project_gaussians(const rtgs_gaussians* g, const rtgs_pose* pose, const rtgs_camera* cam,
                                   rtgs_projected* out, void* stream) {
  if (!gauss_ok(g, false) || !pose_ok(pose) || !cam_ok(cam) || !proj_ok(out, g ? g->n : 0))
    return RTGS_ERR_INVALID_ARG;
  return finish(launch_project(*g, make_pose(*pose), *cam, *out, S(stream)));
}

size_t rtgs_bin_workspace_size(int32_t n, const rtgs_camera* cam, uint32_t capacity) {
  if (n < 0 || !cam_ok(cam)) return 0;
  return bin_workspace_size(n, *cam, capacity);
}

rtgs_status rtgs_bin_and_sort(const rtgs_projected* proj, int32_t n, const rtgs_camera* cam, const uint8_t* tile_keep,
                              rtgs_bins* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || !cam_ok(cam) || !proj_ok(proj, n) || !bins_ok(out)) return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < bin_workspace_size(n, *cam, out->capacity)) return RTGS_ERR_WORKSPACE;
  return finish(launch_bin(*proj, n, *cam, tile_keep, *out, workspace, S(stream)));
}

rtgs_status rtgs_project_and_bin(const rtgs_gaussians* g, const rtgs_pose* pose, const rtgs_camera* cam,
                                 rtgs_projected* proj, rtgs_bins* out, rtgs_bins* cache, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  if (!gauss_ok(g, false) || !pose_ok(pose) || !cam_ok(cam) || !proj_ok(proj, g ? g->n : 0) || !bins_ok(out))
    return RTGS_ERR_INVALID_ARG;
  if (cache && (!g->flags || !cache->sorted_gid || !cache->tile_range ||
                (reinterpret_cast<uintptr_t>(cache->tile_range) & 7u) != 0 || cache->capacity < out->capacity))
    return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < bin_workspace_size(g->n, *cam, out->capacity)) return RTGS_ERR_WORKSPACE;
  return finish(launch_project_bin(*g, make_pose(*pose), *cam, *proj, *out, cache, workspace, S(stream)));
}

rtgs_status rtgs_render_color_depth(const rtgs_gaussians* g, const rtgs_projected* proj, const rtgs_bins* bins,
                                    const rtgs_pose* pose, const rtgs_camera* cam, int32_t mode,
                                    rtgs_render_out* out, void* stream) {
  if (!cam_ok(cam) || !out || !pose_ok(pose)) return RTGS_ERR_INVALID_ARG;
  if (mode == RTGS_RENDER_COVERAGE) {
    if (!g || g->n < 0 || !proj_ok(proj, g->n)) return RTGS_ERR_INVALID_ARG;  // flags NULL: every row
    if (!out->active_bits || !out->tile_keep || !out->tile_list || !out->counts) return RTGS_ERR_INVALID_ARG;
    return finish(launch_coverage(*g, *proj, *cam, *out, S(stream)));
  }
  const bool count = (mode & RTGS_RENDER_COUNT) != 0;
  const bool dense = (mode & RTGS_RENDER_DENSE) != 0;
  mode &= ~(RTGS_RENDER_COUNT | RTGS_RENDER_DENSE);
  if (mode != RTGS_RENDER_FULL && mode != RTGS_RENDER_MASKED) return RTGS_ERR_INVALID_ARG;
  if (count && !out->counts) return RTGS_ERR_INVALID_ARG;
  if (!proj || !proj->rec || !proj->zkey || !a16(proj->rec) || !bins_ok(bins)) return RTGS_ERR_INVALID_ARG;
  // (sub_zkey / sub_gid may be NULL for an empty subset: then no entry carries the subset bit)
  if (bins->sub_rec && !a16(bins->sub_rec)) return RTGS_ERR_INVALID_ARG;
  if (!out->color || !out->trans || !out->depth || !out->index) return RTGS_ERR_INVALID_ARG;
  if (!out->n_contrib && (mode == RTGS_RENDER_MASKED || count)) return RTGS_ERR_INVALID_ARG;
  if (mode == RTGS_RENDER_MASKED && (!out->active_bits || !out->tile_list || !out->counts))
    return RTGS_ERR_INVALID_ARG;
  return finish(launch_render(*proj, *bins, make_pose(*pose), *cam, mode == RTGS_RENDER_MASKED, count, *out,
                              S(stream), dense));
}

size_t rtgs_backward_workspace_size(int32_t n_slots) { return n_slots < 0 ? 0 : backward_workspace_size(n_slots); }

rtgs_status rtgs_render_backward_masked(const rtgs_gaussians* g, const rtgs_projected* proj, const rtgs_bins* bins,
                                        const rtgs_pose* pose, const rtgs_camera* cam, const rtgs_render_out* fwd,
                                        const rtgs_frame* target, const rtgs_loss_weights* w,
                                        const int32_t* slot_of_gid, const int32_t* gid_of_slot, int32_t n_slots,
                                        float* grad, float* loss_out, void* workspace, size_t workspace_bytes,
                                        void* stream) {
  if (!gauss_ok(g, false) || !proj_ok(proj, g ? g->n : 0) || !bins_ok(bins) || !pose_ok(pose) || !cam_ok(cam))
    return RTGS_ERR_INVALID_ARG;
  if (!fwd || !fwd->color || !fwd->depth || !fwd->index || !fwd->n_contrib || !fwd->active_bits ||
      !fwd->tile_list || !fwd->counts)
    return RTGS_ERR_INVALID_ARG;
  if (!target || !target->color || !target->depth || !w || n_slots < 0 || !loss_out) return RTGS_ERR_INVALID_ARG;
  if (g->n > 0 && !slot_of_gid) return RTGS_ERR_INVALID_ARG;
  if (n_slots > 0 && (!gid_of_slot || !grad)) return RTGS_ERR_INVALID_ARG;
  if (bins->sub_rec && bins->sub_gid != gid_of_slot) return RTGS_ERR_INVALID_ARG;  // f3: subset rows are the slots
  if (!workspace || workspace_bytes < backward_workspace_size(n_slots) || !a16(workspace)) return RTGS_ERR_WORKSPACE;
  return finish(launch_backward(*g, *proj, *bins, make_pose(*pose), *cam, *fwd, *target, *w, slot_of_gid, gid_of_slot,
                                n_slots, grad, loss_out, workspace, S(stream)));
}

rtgs_status rtgs_backward_adam_unstable(const rtgs_gaussians* g, const rtgs_projected* proj, const rtgs_bins* bins,
                                        const rtgs_pose* pose, const rtgs_camera* cam, const rtgs_render_out* fwd,
                                        const rtgs_frame* target, const rtgs_loss_weights* w,
                                        const int32_t* slot_of_gid, const int32_t* gid_of_slot, int32_t n_slots,
                                        rtgs_params* params, float* m, float* v, const float* init_geom,
                                        int32_t n_transparent, const rtgs_hparams* hp, int32_t step,
                                        const int32_t* step_device, uint32_t* eta, float* loss_out, void* workspace,
                                        size_t workspace_bytes, void* stream) {
  if (!gauss_ok(g, false) || !proj_ok(proj, g ? g->n : 0) || !bins_ok(bins) || !pose_ok(pose) || !cam_ok(cam))
    return RTGS_ERR_INVALID_ARG;
  if (!fwd || !fwd->color || !fwd->depth || !fwd->index || !fwd->n_contrib || !fwd->active_bits ||
      !fwd->tile_list || !fwd->counts)
    return RTGS_ERR_INVALID_ARG;
  if (!target || !target->color || !target->depth || !w || n_slots < 0 || !loss_out || !std::isfinite(w->w_reg))
    return RTGS_ERR_INVALID_ARG;
  if (!params || !hp || (step < 1 && !step_device) || n_transparent < 0) return RTGS_ERR_INVALID_ARG;
  // the update is written through `params`, which must be the arrays the backward reads
  if (params->pos != g->pos || params->log_scale != g->log_scale || params->rot != g->rot || params->sh != g->sh ||
      params->sh_degree != g->sh_degree)
    return RTGS_ERR_INVALID_ARG;
  if (g->n > 0 && !slot_of_gid) return RTGS_ERR_INVALID_ARG;
  if (n_slots > 0 && (!gid_of_slot || !g->flags || !m || !v || !eta || (n_transparent > 0 && !init_geom)))
    return RTGS_ERR_INVALID_ARG;
  if (bins->sub_rec && bins->sub_gid != gid_of_slot) return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < backward_workspace_size(n_slots) || !a16(workspace)) return RTGS_ERR_WORKSPACE;
  return finish(launch_backward_adam(*g, *proj, *bins, make_pose(*pose), *cam, *fwd, *target, *w, slot_of_gid,
                                     gid_of_slot, n_slots, *params, m, v, init_geom, n_transparent, *hp, step,
                                     step_device, eta, loss_out, workspace, S(stream)));
}

rtgs_status rtgs_adam_step_unstable(rtgs_params* params, const int32_t* gid_of_slot, int32_t n_slots,
                                    const uint8_t* flags, float* grad, float* m, float* v, const float* init_geom,
                                    int32_t n_transparent, float w_reg, const rtgs_hparams* hp, int32_t step,
                                    const int32_t* step_device, uint32_t* eta, void* stream) {
  if (!params || !hp || n_slots < 0 || (step < 1 && !step_device) || n_transparent < 0 || params->sh_degree < 0 ||
      params->sh_degree > 3 || !std::isfinite(w_reg))
    return RTGS_ERR_INVALID_ARG;
  if (n_slots > 0 && (!params->pos || !params->log_scale || !params->rot || !params->sh || !gid_of_slot || !flags ||
                      !grad || !m || !v || !eta || (n_transparent > 0 && !init_geom)))
    return RTGS_ERR_INVALID_ARG;
  return finish(launch_adam(*params, gid_of_slot, n_slots, flags, grad, m, v, init_geom, n_transparent, w_reg, *hp, step,
                            step_device, eta, S(stream)));
}

size_t rtgs_classify_workspace_size(const rtgs_camera* cam) { return cam_ok(cam) ? classify_workspace_size(*cam) : 0; }

rtgs_status rtgs_classify_and_add_pixels(const rtgs_render_out* full, const rtgs_frame* frame, const uint8_t* flags,
                                         const rtgs_camera* cam, const rtgs_add_params* ap, uint8_t* pixel_class,
                                         uint32_t* samples, uint32_t cap, uint32_t* counts, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  if (!full || !full->color || !full->trans || !full->depth || !full->index || !frame || !frame->color ||
      !frame->depth || !flags || !cam_ok(cam) || !ap || !pixel_class || !counts || (cap > 0 && !samples))
    return RTGS_ERR_INVALID_ARG;
  if (!(ap->sample_ratio >= 0.0) || !std::isfinite(ap->sample_ratio)) return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < classify_workspace_size(*cam)) return RTGS_ERR_WORKSPACE;
  return finish(launch_classify(*full, *frame, flags, *cam, *ap, pixel_class, samples, cap, counts, workspace,
                                S(stream)));
}

rtgs_status rtgs_fuse_window(rtgs_params* params, const int32_t* gid_of_slot, int32_t n_slots, const float* before,
                             const uint32_t* eta_before, const uint32_t* eta, void* stream) {
  if (!params || n_slots < 0 || params->sh_degree < 0 || params->sh_degree > 3) return RTGS_ERR_INVALID_ARG;
  if (n_slots > 0 && (!params->pos || !params->log_scale || !params->rot || !params->sh || !gid_of_slot || !before ||
                      !eta_before || !eta))
    return RTGS_ERR_INVALID_ARG;
  return finish(launch_fuse(*params, gid_of_slot, n_slots, before, eta_before, eta, S(stream)));
}

size_t rtgs_state_workspace_size(int32_t n) { return n < 0 ? 0 : state_workspace_size(n); }

rtgs_status rtgs_manage_states(const rtgs_render_out* full, const rtgs_frame* frame, const rtgs_camera* cam,
                               uint8_t* flags, uint32_t* err_count, uint32_t* eta, uint32_t* t_created, int32_t n,
                               const rtgs_state_params* sp, uint32_t* counts, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (!full || !full->color || !full->depth || !full->index || !frame || !frame->color || !frame->depth ||
      !cam_ok(cam) || !sp || !counts || n < 0)
    return RTGS_ERR_INVALID_ARG;
  if (n > 0 && (!flags || !err_count || !eta || !t_created)) return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < state_workspace_size(n)) return RTGS_ERR_WORKSPACE;
  return finish(launch_manage_states(*full, *frame, *cam, flags, err_count, eta, t_created, n, *sp, counts, workspace,
                                     S(stream)));
}

rtgs_status rtgs_project_subset(const rtgs_gaussians* g, const int32_t* gid_list, int32_t n_list,
                                const rtgs_pose* pose, const rtgs_camera* cam, rtgs_projected* out, void* stream) {
  if (!gauss_ok(g, false) || n_list < 0 || !pose_ok(pose) || !cam_ok(cam) || !proj_ok(out, n_list))
    return RTGS_ERR_INVALID_ARG;
  if (n_list > 0 && (!gid_list || g->n == 0)) return RTGS_ERR_INVALID_ARG;
  return finish(launch_project_subset(*g, gid_list, n_list, make_pose(*pose), *cam, *out, S(stream)));
}

rtgs_status rtgs_stable_cache_build(const rtgs_bins* full, const uint8_t* flags, const rtgs_camera* cam,
                                    rtgs_bins* cache, void* stream) {
  if (!bins_ok(full) || !flags || !cam_ok(cam) || !cache || !cache->sorted_gid || !cache->tile_range ||
      (reinterpret_cast<uintptr_t>(cache->tile_range) & 7u) != 0 || cache->capacity < full->capacity)
    return RTGS_ERR_INVALID_ARG;
  return finish(launch_cache_build(*full, flags, *cam, *cache, S(stream)));
}

size_t rtgs_bin_cached_workspace_size(int32_t n_sub, const rtgs_camera* cam, uint32_t capacity) {
  if (n_sub < 0 || !cam_ok(cam)) return 0;
  return bin_cached_workspace_size(n_sub, *cam, capacity);
}

rtgs_status rtgs_bin_and_sort_cached(const rtgs_projected* proj, const rtgs_bins* cache, const rtgs_projected* sub,
                                     const int32_t* sub_gid, int32_t n_sub, const rtgs_camera* cam,
                                     const uint8_t* tile_keep, rtgs_bins* out, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  if (!proj || !proj->zkey || !cache || !cache->sorted_gid || !cache->tile_range || n_sub < 0 || !cam_ok(cam) ||
      !tile_keep || !bins_ok(out) || !proj_ok(sub, n_sub) || (n_sub > 0 && !sub_gid))
    return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < bin_cached_workspace_size(n_sub, *cam, out->capacity)) return RTGS_ERR_WORKSPACE;
  out->sub_rec = sub->rec;
  out->sub_zkey = sub->zkey;
  out->sub_gid = sub_gid;
  return finish(launch_bin_cached(*proj, *cache, *sub, sub_gid, n_sub, *cam, tile_keep, *out, workspace, S(stream)));
}

size_t rtgs_insert_workspace_size(int32_t n, uint32_t sample_cap) {
  return n < 0 ? 0 : insert_workspace_size(n, sample_cap);
}

rtgs_status rtgs_add_gaussians(const rtgs_map* map, const uint32_t* samples, uint32_t sample_cap,
                               const uint32_t* add_counts, const rtgs_frame* frame, const rtgs_pose* pose,
                               const rtgs_camera* cam, const rtgs_insert_params* ip, uint32_t* result,
                               void* workspace, size_t workspace_bytes, void* stream) {
  if (!map || map->n < 0 || map->capacity < map->n || map->sh_degree < 0 || map->sh_degree > 3 || !pose_ok(pose) ||
      !cam_ok(cam) || !ip || !result || !add_counts || !frame || !frame->color || !frame->depth)
    return RTGS_ERR_INVALID_ARG;
  if (map->capacity > 0 && (!map->pos || !map->log_scale || !map->rot || !map->opacity || !map->sh || !map->flags ||
                            !map->eta || !map->err_count || !map->t_created))
    return RTGS_ERR_INVALID_ARG;
  if (sample_cap > 0 && !samples) return RTGS_ERR_INVALID_ARG;
  if (!(ip->normal_guard >= 0.f) || !(ip->min_scale > 0.f) || !(ip->max_scale_transparent > 0.f))
    return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < insert_workspace_size(map->n, sample_cap)) return RTGS_ERR_WORKSPACE;
  return finish(launch_insert(*map, samples, sample_cap, add_counts, *frame, make_pose(*pose), *cam, *ip, result,
                              workspace, S(stream)));
}

size_t rtgs_icp_workspace_size(const rtgs_camera* cam, int32_t levels) {
  if (!cam_ok(cam) || levels < 1 || levels > 4) return 0;
  return icp_workspace_size(*cam, levels);
}

rtgs_status rtgs_icp_track(const float* depth, const float* model_depth, const float* model_normal,
                           const rtgs_pose* model_pose, const rtgs_camera* cam, const rtgs_icp_params* params,
                           double* pose_io, double* diag, void* workspace, size_t workspace_bytes, void* stream) {
  if (!depth || !model_depth || !model_normal || !pose_ok(model_pose) || !cam_ok(cam) || !params || !pose_io || !diag)
    return RTGS_ERR_INVALID_ARG;
  if (params->levels < 1 || params->levels > 4 || params->min_pairs < 6 || !(params->eps >= 0.0) ||
      !(params->dist_gate > 0.0) || !(params->cos_gate <= 1.0) || !(params->normal_guard >= 0.f))
    return RTGS_ERR_INVALID_ARG;
  for (int l = 0; l < params->levels; ++l)
    if (params->iters[l] < 0 || params->iters[l] > 1000) return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < icp_workspace_size(*cam, params->levels)) return RTGS_ERR_WORKSPACE;
  return finish(launch_icp(depth, model_depth, model_normal, *model_pose, *cam, *params, pose_io, diag, workspace,
                           S(stream)));
}

rtgs_status rtgs_decode_rgbd(const uint8_t* rgb, const uint16_t* depth_raw, int32_t width, int32_t height,
                             float depth_scale, float* color, float* depth, void* stream) {
  if (width < 0 || height < 0 || width > 16384 || height > 16384 || !(depth_scale > 0.f) ||
      !std::isfinite(depth_scale))
    return RTGS_ERR_INVALID_ARG;
  if ((size_t)width * height > 0 &&
      (!rgb || !depth_raw || !color || !depth || !a4(rgb) || (reinterpret_cast<uintptr_t>(depth_raw) & 7u) != 0 ||
       !a16(color) || !a16(depth)))
    return RTGS_ERR_INVALID_ARG;
  return finish(launch_decode(rgb, depth_raw, width, height, depth_scale, color, depth, S(stream)));
}

rtgs_status rtgs_coverage_and_bin_cached(const rtgs_projected* proj, const rtgs_bins* cache, const rtgs_projected* sub,
                                         const int32_t* sub_gid, int32_t n_sub, const rtgs_camera* cam,
                                         rtgs_render_out* cov, rtgs_bins* out, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  if (!proj || !proj->zkey || !cache || !cache->sorted_gid || !cache->tile_range || n_sub < 0 || !cam_ok(cam) ||
      !bins_ok(out) || !proj_ok(sub, n_sub) || (n_sub > 0 && (!sub_gid || !a16(sub->rec))) || !cov ||
      !cov->active_bits || !cov->tile_keep || !cov->tile_list || !cov->counts)
    return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < bin_cached_workspace_size(n_sub, *cam, out->capacity)) return RTGS_ERR_WORKSPACE;
  out->sub_rec = sub->rec;
  out->sub_zkey = sub->zkey;
  out->sub_gid = sub_gid;
  return finish(launch_coverage_bin_cached(*proj, *cache, *sub, sub_gid, n_sub, *cam, *cov, *out, workspace,
                                           S(stream)));
}

rtgs_status rtgs_coverage_subset(const rtgs_projected* sub, int32_t n_sub, const rtgs_camera* cam, rtgs_render_out* cov,
                                 uint32_t capacity, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_sub < 0 || !cam_ok(cam) || !proj_ok(sub, n_sub) || (n_sub > 0 && !a16(sub->rec)) || !cov ||
      !cov->active_bits || !cov->tile_keep || !cov->tile_list || !cov->counts)
    return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < bin_cached_workspace_size(n_sub, *cam, capacity)) return RTGS_ERR_WORKSPACE;
  return finish(launch_coverage_subset(*sub, n_sub, *cam, *cov, capacity, workspace, S(stream)));
}

rtgs_status rtgs_merge_cached(const rtgs_projected* proj, const rtgs_bins* cache, const rtgs_projected* sub,
                              const int32_t* sub_gid, int32_t n_sub, const rtgs_camera* cam,
                              const rtgs_render_out* cov, rtgs_bins* out, void* workspace, size_t workspace_bytes,
                              void* stream) {
  if (!proj || !proj->zkey || !cache || !cache->sorted_gid || !cache->tile_range || n_sub < 0 || !cam_ok(cam) ||
      !bins_ok(out) || !proj_ok(sub, n_sub) || (n_sub > 0 && !sub_gid) || !cov || !cov->tile_keep)
    return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < bin_cached_workspace_size(n_sub, *cam, out->capacity)) return RTGS_ERR_WORKSPACE;
  out->sub_rec = sub->rec;
  out->sub_zkey = sub->zkey;
  out->sub_gid = sub_gid;
  return finish(launch_merge_cached(*proj, *cache, *sub, sub_gid, n_sub, *cam, cov->tile_keep, *out, workspace,
                                    S(stream)));
}

size_t rtgs_morton_workspace_size(int32_t n) { return n < 0 ? 0 : morton_workspace_size(n); }

rtgs_status rtgs_morton_order(const float* pos, const uint8_t* flags, int32_t n, uint32_t* perm, void* workspace,
                              size_t workspace_bytes, void* stream) {
  if (n < 0 || (n > 0 && (!pos || !perm || !a4(pos)))) return RTGS_ERR_INVALID_ARG;
  if (n > 0 && (!workspace || workspace_bytes < morton_workspace_size(n))) return RTGS_ERR_WORKSPACE;
  return finish(launch_morton_order(pos, flags, n, perm, workspace, S(stream)));
}

rtgs_status rtgs_gather_rows(const void* src, void* dst, const uint32_t* perm, int32_t n, int32_t row_bytes,
                             void* stream) {
  if (n < 0 || row_bytes <= 0 || (n > 0 && (!src || !dst || !perm))) return RTGS_ERR_INVALID_ARG;
  const char* a = static_cast<const char*>(src);
  const char* b = static_cast<const char*>(dst);
  const size_t bytes = (size_t)n * row_bytes;
  if (n > 0 && a < b + bytes && b < a + bytes) return RTGS_ERR_INVALID_ARG;  // overlapping
  return finish(launch_gather_rows(src, dst, perm, n, row_bytes, S(stream)));
}

size_t rtgs_topk_workspace_size(const rtgs_camera* cam) { return cam_ok(cam) ? topk_workspace_size(*cam) : 0; }

rtgs_status rtgs_topk_error_mask(const float* color_hat, const float* frame_color, const rtgs_camera* cam, double ratio,
                                 rtgs_render_out* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!color_hat || !frame_color || !cam_ok(cam) || !(ratio >= 0.0 && ratio <= 1.0) || !out || !out->active_bits ||
      !out->tile_keep || !out->tile_list || !out->counts)
    return RTGS_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < topk_workspace_size(*cam)) return RTGS_ERR_WORKSPACE;
  return finish(launch_topk(color_hat, frame_color, *cam, ratio, *out, workspace, S(stream)));
}

rtgs_status rtgs_check_device_flags(void* stream) {
  // synchronises `stream`, then reads and clears the sticky CAPACITY flag
  cudaStream_t st = S(stream);
  uint32_t* f = capacity_flag_ptr();
  if (!f) return RTGS_ERR_CUDA;
  uint32_t h = 0;
  if (cudaMemcpyAsync(&h, f, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess) return finish(cudaGetLastError());
  if (cudaMemsetAsync(f, 0, 4, st) != cudaSuccess) return finish(cudaGetLastError());
  if (cudaStreamSynchronize(st) != cudaSuccess) return finish(cudaGetLastError());
  return h ? RTGS_ERR_CAPACITY : RTGS_OK;
}

const char* rtgs_status_string(rtgs_status s) {
  switch (s) {
    case RTGS_OK: return "RTGS_OK";
    case RTGS_ERR_INVALID_ARG: return "RTGS_ERR_INVALID_ARG";
    case RTGS_ERR_CAPACITY: return "RTGS_ERR_CAPACITY";
    case RTGS_ERR_CUDA: return "RTGS_ERR_CUDA";
    case RTGS_ERR_WORKSPACE: return "RTGS_ERR_WORKSPACE";
  }
  return "RTGS_UNKNOWN";
}

const char* rtgs_last_cuda_error(void) { return g_cuda_err; }
int32_t rtgs_version(void) { return 1; }
uint64_t rtgs_launch_count(void) { return g_launches.load(); }

}  // extern "C"
