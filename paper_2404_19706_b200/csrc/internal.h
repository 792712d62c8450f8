// internal.h — host-side launchers behind the C ABI (abi.cu validates, these enqueue kernels).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "rtgs.h"

#include <atomic>

namespace rtgs {

#ifndef RTGS_REP
#define RTGS_REP 2
#endif
constexpr int kRep = RTGS_REP;  // replicated per-tile counters of the binning: spreads same-address atomics (swept 1/2/4/8 on Morton-ordered C3/C4 maps: 2)

// once per (kernel attribute, device): per-device bit in `mask` (one-time cudaFuncSetAttribute calls
// must be repeated on every device the process launches on)
inline bool first_on_device(std::atomic<uint64_t>& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  return (mask.fetch_or(bit) & bit) == 0;
}

struct PoseF {  // world->camera V = R^T, t' = -R^T t (double and float32 copies), camera centre
  double V[9], tp[3], campos[3];
  float Vf[9], tpf[3];
  float Rf[9];  // camera->world rotation (normal map)
};
PoseF make_pose(const rtgs_pose& p);

cudaError_t launch_project(const rtgs_gaussians& g, const PoseF& pose, const rtgs_camera& cam,
                           const rtgs_projected& out, cudaStream_t s);

// the projection with the binning's per-tile counts fused in (replica (i >> 8) & (kRep - 1), as k_tile_count)
cudaError_t launch_project_count(const rtgs_gaussians& g, const PoseF& pose, const rtgs_camera& cam,
                                 const rtgs_projected& out, uint32_t* cnt, cudaStream_t s);
cudaError_t launch_project_bin(const rtgs_gaussians& g, const PoseF& pose, const rtgs_camera& cam,
                               const rtgs_projected& proj, const rtgs_bins& out, const rtgs_bins* cache, void* ws,
                               cudaStream_t s);

cudaError_t launch_project_subset(const rtgs_gaussians& g, const int32_t* gid_list, int n_list, const PoseF& pose,
                                  const rtgs_camera& cam, const rtgs_projected& out, cudaStream_t s);

size_t bin_workspace_size(int n, const rtgs_camera& cam, uint32_t capacity);
cudaError_t launch_bin(const rtgs_projected& proj, int n, const rtgs_camera& cam, const uint8_t* keep,
                       const rtgs_bins& out, void* ws, cudaStream_t s);

cudaError_t launch_cache_build(const rtgs_bins& full, const uint8_t* flags, const rtgs_camera& cam,
                               const rtgs_bins& cache, cudaStream_t s);
size_t bin_cached_workspace_size(int n_sub, const rtgs_camera& cam, uint32_t capacity);
cudaError_t launch_bin_cached(const rtgs_projected& proj, const rtgs_bins& cache, const rtgs_projected& sub,
                              const int32_t* sub_gid, int n_sub, const rtgs_camera& cam, const uint8_t* keep,
                              const rtgs_bins& out, void* ws, cudaStream_t s);

cudaError_t launch_tile_coverage(const uint2* srange, const unsigned long long* keys, const float4* sub_rec,
                                 const rtgs_camera& cam, const rtgs_render_out& out, cudaStream_t s);
cudaError_t launch_coverage_subset(const rtgs_projected& sub, int n_sub, const rtgs_camera& cam,
                                   const rtgs_render_out& cov, uint32_t capacity, void* ws, cudaStream_t s);
cudaError_t launch_merge_cached(const rtgs_projected& proj, const rtgs_bins& cache, const rtgs_projected& sub,
                                const int32_t* sub_gid, int n_sub, const rtgs_camera& cam, const uint8_t* keep,
                                const rtgs_bins& out, void* ws, cudaStream_t s);
cudaError_t launch_coverage_bin_cached(const rtgs_projected& proj, const rtgs_bins& cache, const rtgs_projected& sub,
                                       const int32_t* sub_gid, int n_sub, const rtgs_camera& cam,
                                       const rtgs_render_out& cov, const rtgs_bins& out, void* ws, cudaStream_t s);

cudaError_t launch_coverage(const rtgs_gaussians& g, const rtgs_projected& proj, const rtgs_camera& cam,
                            const rtgs_render_out& out, cudaStream_t s);
cudaError_t launch_render(const rtgs_projected& proj, const rtgs_bins& bins, const PoseF& pose,
                          const rtgs_camera& cam, int masked, bool count, const rtgs_render_out& out, cudaStream_t s,
                          bool dense = false);

size_t backward_workspace_size(int n_slots);
cudaError_t launch_backward(const rtgs_gaussians& g, const rtgs_projected& proj, const rtgs_bins& bins,
                            const PoseF& pose, const rtgs_camera& cam, const rtgs_render_out& fwd,
                            const rtgs_frame& target, const rtgs_loss_weights& w, const int32_t* slot_of_gid,
                            const int32_t* gid_of_slot, int n_slots, float* grad, float* loss_out, void* ws,
                            cudaStream_t s);

cudaError_t launch_backward_adam(const rtgs_gaussians& g, const rtgs_projected& proj, const rtgs_bins& bins,
                                 const PoseF& pose, const rtgs_camera& cam, const rtgs_render_out& fwd,
                                 const rtgs_frame& target, const rtgs_loss_weights& w, const int32_t* slot_of_gid,
                                 const int32_t* gid_of_slot, int n_slots, const rtgs_params& p, float* m, float* v,
                                 const float* init_geom, int n_transparent, const rtgs_hparams& hp, int step,
                                 const int32_t* step_device, uint32_t* eta, float* loss_out, void* ws,
                                 cudaStream_t s);

cudaError_t launch_adam(const rtgs_params& p, const int32_t* gid_of_slot, int n_slots, const uint8_t* flags,
                        float* grad, float* m, float* v, const float* init_geom, int n_transparent, float w_reg,
                        const rtgs_hparams& hp, int step, const int32_t* step_device, uint32_t* eta,
                        cudaStream_t s);

size_t classify_workspace_size(const rtgs_camera& cam);
cudaError_t launch_classify(const rtgs_render_out& full, const rtgs_frame& frame, const uint8_t* flags,
                            const rtgs_camera& cam, const rtgs_add_params& ap, uint8_t* cls, uint32_t* samples,
                            uint32_t cap, uint32_t* counts, void* ws, cudaStream_t s);

cudaError_t launch_fuse(const rtgs_params& p, const int32_t* gid_of_slot, int n_slots, const float* before,
                        const uint32_t* eta_before, const uint32_t* eta, cudaStream_t s);
size_t state_workspace_size(int n);
cudaError_t launch_manage_states(const rtgs_render_out& full, const rtgs_frame& frame, const rtgs_camera& cam,
                                 uint8_t* flags, uint32_t* err, uint32_t* eta, uint32_t* tc, int n,
                                 const rtgs_state_params& sp, uint32_t* counts, void* ws, cudaStream_t s);

size_t insert_workspace_size(int n, uint32_t sample_cap);
cudaError_t launch_insert(const rtgs_map& m, const uint32_t* samples, uint32_t cap, const uint32_t* add_counts,
                          const rtgs_frame& frame, const PoseF& pose, const rtgs_camera& cam,
                          const rtgs_insert_params& ip, uint32_t* result, void* ws, cudaStream_t s);

size_t icp_workspace_size(const rtgs_camera& cam, int levels);
cudaError_t launch_icp(const float* depth, const float* mdepth, const float* mnormal, const rtgs_pose& model_pose,
                       const rtgs_camera& cam, const rtgs_icp_params& p, double* pose_io, double* diag, void* ws,
                       cudaStream_t s);

cudaError_t launch_decode(const uint8_t* rgb, const uint16_t* raw, int W, int H, float depth_scale, float* color,
                          float* depth, cudaStream_t s);

cudaError_t launch_tile_any(const rtgs_camera& cam, const rtgs_render_out& out, cudaStream_t s);
size_t topk_workspace_size(const rtgs_camera& cam);
cudaError_t launch_topk(const float* chat, const float* c, const rtgs_camera& cam, double ratio,
                        const rtgs_render_out& out, void* ws, cudaStream_t s);

// generic device-wide exclusive scan of uint32 (length known on the host; zeros past the live part)
size_t scan_workspace_size(size_t len);
uint32_t* capacity_flag_ptr();  // device address of the sticky CAPACITY flag (sort.cu)
size_t morton_workspace_size(int n);
cudaError_t launch_morton_order(const float* pos, const uint8_t* flags, int n, uint32_t* perm, void* ws,
                                cudaStream_t s);
cudaError_t launch_gather_rows(const void* src, void* dst, const uint32_t* perm, int n, int row_bytes,
                               cudaStream_t s);
cudaError_t launch_scan(const uint32_t* in, uint32_t* out, size_t len, uint32_t* total, void* ws, cudaStream_t s);

}  // namespace rtgs
