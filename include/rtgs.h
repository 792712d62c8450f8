/*
 * rtgs.h — C ABI of librtgs.so, the B200 (sm_100a) mapping hot path of RTG-SLAM
 * (Peng et al., arXiv 2404.19706).  "P:n" = line n of the paper text; "Rn" = reading n of
 * DESIGN.md §3 (where the paper is silent or garbled); "Eq.k" numbered in order of appearance.
 *
 * Conventions shared by every call
 *  - All buffer pointers are DEVICE pointers owned by the caller unless stated otherwise; the
 *    library never allocates device memory and never frees caller memory.  Scratch space is passed
 *    as (workspace, workspace_bytes); query the size with the matching *_workspace_size call.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every call only
 *    ENQUEUES work on `stream` and returns; nothing synchronises, nothing reads results back, so an
 *    iteration can be captured into a CUDA graph.
 *  - Arguments are validated on the host before any launch.  Errors are returned as rtgs_status;
 *    nothing aborts or throws across the ABI.  On error no work has been enqueued (INVALID_ARG,
 *    WORKSPACE) or the CUDA launch failed (ERR_CUDA; see rtgs_last_cuda_error()).
 *  - Images are planar float32, row-major: color [3][H][W], single channel [H][W].  Pixel (px, py)
 *    has its centre at (px, py) (R1).  Tiles are 16 x 16 pixels, tile id = ty * TX + tx with
 *    TX = ceil(W/16), TY = ceil(H/16).  Pixel bit masks hold bit (py*W+px) in word (py*W+px)/32.
 *  - Pointers to float/int arrays must be 4-byte aligned, and `rec`, `pos`, `sh` 16-byte aligned.
 *  - Gaussian ids (gid) are indices into the flat Gaussian arrays, 0 <= gid < n < 2^31.
 */
#ifndef RTGS_H
#define RTGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RTGS_OK = 0,
  RTGS_ERR_INVALID_ARG = 1, /* null / mis-sized / misaligned argument, bad mode, non-finite pose  */
  RTGS_ERR_CAPACITY = 2,    /* a binning exceeded its capacity (sticky flag, rtgs_check_device_flags) */
  RTGS_ERR_CUDA = 3,        /* a kernel launch failed; see rtgs_last_cuda_error()                 */
  RTGS_ERR_WORKSPACE = 4    /* workspace pointer null or smaller than the *_workspace_size query  */
} rtgs_status;

/* Intrinsics K.  fx, fy > 0; 1 <= width, height <= 16384. */
typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
} rtgs_camera;

/* Camera->world pose T_g = [R t; 0 1] in SE(3), row-major R, HOST memory, float64 so the
 * camera-frame position p_c = R^T (p - t) is formed without float32 cancellation. */
typedef struct {
  double R[9];
  double t[3];
} rtgs_pose;

/* The Gaussian map, structure of arrays, float32, read-only for rendering.
 *   pos       [n][3]  position p
 *   log_scale [n][3]  s = exp(log_scale) (R3)
 *   rot       [n][4]  quaternion (w, x, y, z), normalised inside the forward pass (R3)
 *   opacity   [n]     alpha: 0.99 opaque / 0.1 transparent; never optimised (lr_alpha = 0)
 *   sh        [n][K][3], K = (sh_degree+1)^2, coefficient-major, channel-minor (R2)
 *   flags     [n]     bit0 = transparent, bit1 = stable (eta > delta_eta), bit2 = removed */
typedef struct {
  const float *pos, *log_scale, *rot, *opacity, *sh;
  const uint8_t *flags;
  int32_t n;
  int32_t sh_degree; /* 0..3 */
} rtgs_gaussians;

/* Mutable view of the optimised parameters (adam_step_unstable). Same layouts as rtgs_gaussians. */
typedef struct {
  float *pos, *log_scale, *rot, *sh;
  int32_t n;
  int32_t sh_degree;
} rtgs_params;

/* Per-Gaussian projection (O1, Eq.2).  Written by rtgs_project_gaussians.
 *   rec [n][16] float32, 64 B per Gaussian:
 *     [0] mu_x hi  [1] mu_y hi  [2] mu_x lo  [3] mu_y lo      mu = hi + lo (double-float)
 *     [4] A'  [5] B'  [6] C'  [7] log2(alpha)   with Sigma2D^-1 = [[A,B],[B,C]] prescaled to base 2:
 *         A' = -log2(e)/2 A, B' = -log2(e) B, C' = -log2(e)/2 C, so f = 2^(A'dx^2 + B'dx dy + C'dy^2 + log2 alpha)
 *     [8] r  [9] g  [10] b                                    colour from SH at the view direction (R2)
 *     [11] support half-extents (ex, ey) in pixels as two IEEE halves (low half = ex), rounded up
 *     [12..14] n_c (unit disc normal, camera frame)  [15] n_c . p_c   (disc plane, Eq.4, R10, R12)
 *   zkey [n]  float32 bits of the camera-frame centre depth z (R8); 0xFFFFFFFF when culled
 *   rect [n][4] int16 pixel rect x0, y0, x1, y1 (inclusive, clipped to the image) of the support (R7);
 *               empty (x0 > x1) when culled (z <= 0.2 m (R6), alpha <= 1/255, or off-image)
 *   tiles_touched [n]  number of 16x16 tiles the rect covers (0 when culled) */
typedef struct {
  float* rec;
  uint32_t* zkey;
  int16_t* rect;
  uint32_t* tiles_touched;
} rtgs_projected;

/* Tile bins (O8).  sorted_gid[capacity]: gids ordered by (tile, zkey bits, gid) (R8);
 * tile_range [TX*TY][2]: [start, end) of every tile in sorted_gid (0,0 when empty);
 * n_instances [1]: total instance count I (may exceed capacity: then the output is truncated,
 * memory-safe but invalid, and the caller must re-run with capacity >= I). */
typedef struct {
  uint32_t* sorted_gid;
  uint32_t* tile_range;
  uint32_t* n_instances;
  uint32_t capacity;
  /* NEXT f3 (rtgs_bin_and_sort_cached writes these; NULL for every other producer of bins):
   * an entry e with bit 31 set is row r = e & 0x7FFFFFFF of a SUBSET projection (sub_rec [rows][16],
   * sub_zkey [rows]) of the Gaussian sub_gid[r]; entries without bit 31 are gids of `proj`. */
  const float* sub_rec;
  const uint32_t* sub_zkey;
  const int32_t* sub_gid;
} rtgs_bins;

enum { RTGS_RENDER_FULL = 0, RTGS_RENDER_MASKED = 1, RTGS_RENDER_COVERAGE = 2 };
/* OR-ed into FULL or MASKED: also count the blended (pixel, Gaussian) pairs into counts[3] (a
 * statistic; the production renders leave it off, it costs instructions per blended pair). */
enum { RTGS_RENDER_COUNT = 16 };
/* OR-ed into FULL or MASKED: evaluate every (pixel, Gaussian) pair of the 8x4 pixel blocks whose
 * support box overlaps the Gaussian (the dense consumer) instead of only the pixels of its support
 * span mask.  Identical results by construction (the span mask is a superset of the support);
 * a verification mode for the tests, slower. */
enum { RTGS_RENDER_DENSE = 32 };

/* Render buffers (O2-O4).  Which fields are read / written depends on the mode, see the call. */
typedef struct {
  float* color;          /* [3][H][W]  C^ (Eq.1), black background (R23)                         */
  float* trans;          /* [H][W]     T^ (Eq.3)                                                  */
  float* depth;          /* [H][W]     D^ (Eq.5); -1 where no opaque disc is hit                  */
  float* normal;         /* [3][H][W]  N^ world frame, zero without hit; NULLABLE         */
  int32_t* index;        /* [H][W]     I^: gid of the hit Gaussian or -1                  */
  uint32_t* n_contrib;   /* [H][W]     sorted-list position just past the last blended entry (the
                                        backward's stop); NULLABLE for a FULL render without
                                        RTGS_RENDER_COUNT, which then skips tracking it              */
  uint32_t* active_bits; /* [ceil(H*W/32)]  M_unstable (Eq.12) — COVERAGE output, MASKED input     */
  uint8_t* tile_keep;    /* [TX*TY]    1 iff >= 50 % of the tile's pixels are active (R15) */
  uint32_t* tile_list;   /* [TX*TY]    ids of kept tiles (order unspecified)                      */
  uint32_t* counts;      /* [4] device: [0] #kept tiles, [1] |P| (active pixels in kept tiles),
                                        [2] |M_unstable| (all three written by COVERAGE), [3] number of
                                        blended (pixel, Gaussian) pairs of the last FULL / MASKED render
                                        made with RTGS_RENDER_COUNT (zeroed by COVERAGE); NULLABLE in
                                        FULL mode without RTGS_RENDER_COUNT                           */
} rtgs_render_out;

/* Target RGBD frame C_k, D_k: color [3][H][W] in [0,1]; depth [H][W] metres, <= 0 or
 * non-finite = invalid (R24). */
typedef struct {
  const float* color;
  const float* depth;
} rtgs_frame;

/* Loss weights of Eq.8: w_c = 1, w_d = 1, w_reg = 1000. */
typedef struct {
  float w_c, w_d, w_reg;
} rtgs_loss_weights;

/* Per-group learning rates and Adam constants (R19: beta 0.9/0.999, eps 1e-15).  The betas
 * are float64 so that 1 - beta2 = 1e-3 is formed exactly before rounding to the kernel's float32. */
typedef struct {
  float lr_pos, lr_sh0, lr_shrest, lr_scale, lr_rot;
  double beta1, beta2, eps;
} rtgs_hparams;

/* Gaussian-adding thresholds: delta_T 0.5, delta_d 0.1, delta_c 0.1, ratio 0.05. */
typedef struct {
  float delta_T, delta_d, delta_c;
  double sample_ratio; /* threshold round(ratio * 2^32) is formed in float64 */
  uint64_t seed;
  uint32_t frame_idx;
} rtgs_add_params;

/* ---------------------------------------------------------------------------------------------
 * A1 — rtgs_project_gaussians (O1; Eq.2, R2-R8, R12)
 * For every Gaussian: cull (z <= 0.2 m), EWA Sigma2D = (J V) Sigma (J V)^T + 0.3 I with the 1.3x-FOV
 * Jacobian clamp, conic, mu, SH colour max(0, SH(d) + 0.5), disc normal (smallest axis) and its
 * camera-frame plane, float32 depth key, support rect and tile count.  Writes every field of `out`
 * for all n Gaussians.  1 thread per Gaussian, SH staged through shared memory by bulk copies.
 * ------------------------------------------------------------------------------------------- */
rtgs_status rtgs_project_gaussians(const rtgs_gaussians* g, const rtgs_pose* pose, const rtgs_camera* cam,
                                   rtgs_projected* out, void* stream);

/* ---------------------------------------------------------------------------------------------
 * A2 — rtgs_bin_and_sort (O8, R7, R8, R15)
 * Instances (tile, gid) for every tile of every Gaussian's tile rect — restricted to tiles with
 * tile_keep[t] != 0 when tile_keep is non-NULL — ordered by (tile, zkey bits, gid).  Implementation:
 * per-tile counts (replicated counters), one-CTA scan into tile ranges, emission of (zkey, gid)
 * pairs into the ranges, one CTA per tile sorting its pairs (LSD radix on the varying depth bits,
 * then gid) — the order is unique, so the result is deterministic although the emission is not.
 * Reads proj->zkey, proj->rect.  `n_instances` receives I; if I > capacity the output is truncated
 * (see rtgs_bins).
 * ------------------------------------------------------------------------------------------- */
size_t rtgs_bin_workspace_size(int32_t n, const rtgs_camera* cam, uint32_t capacity);
/* rtgs_check_device_flags: every binning call that overflows its capacity also sets a
 * sticky device flag; this call synchronises `stream`, reads and clears the flag, and returns
 * RTGS_ERR_CAPACITY if any binning since the last check overflowed (re-run with a larger capacity),
 * else RTGS_OK (RTGS_ERR_CUDA on a CUDA error).  Lets a caller enqueue whole iterations (or CUDA
 * graphs of them) without a host synchronisation and validate once. */
rtgs_status rtgs_check_device_flags(void* stream);
rtgs_status rtgs_bin_and_sort(const rtgs_projected* proj, int32_t n, const rtgs_camera* cam,
                              const uint8_t* tile_keep, rtgs_bins* out, void* workspace, size_t workspace_bytes,
                              void* stream);

/* A1 + A2 fused — rtgs_project_and_bin: exactly rtgs_project_gaussians followed by rtgs_bin_and_sort
 * over all tiles (tile_keep NULL) — the frame ingest's pair — with the per-tile counting of the
 * binning done by the projection kernel (no second pass over zkey / rect).  With `cache` non-NULL
 * (NEXT f3; needs g->flags) the per-tile sort also writes the stable-entry cache, exactly as a
 * following rtgs_stable_cache_build(out, g->flags, cam, cache).  Workspace as
 * rtgs_bin_workspace_size(g->n, cam, out->capacity). */
rtgs_status rtgs_project_and_bin(const rtgs_gaussians* g, const rtgs_pose* pose, const rtgs_camera* cam,
                                 rtgs_projected* proj, rtgs_bins* out, rtgs_bins* cache, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * A0/A3/A4 — rtgs_render_color_depth (O2-O4; Eq.1-5, Eq.12, R7-R12, R15, R16)
 *  mode FULL:     every pixel, every tile.  Writes color, trans, depth, index, n_contrib, normal (if
 *                 non-NULL).  Needs proj, bins.
 *  mode MASKED:   only the active pixels P = M_unstable ∩ kept tiles (out->active_bits, out->tile_keep,
 *                 out->tile_list, out->counts[0] from a previous COVERAGE call); same outputs, other
 *                 pixels untouched.  Needs proj, bins (binned with the same tile_keep or with all tiles).
 *  mode COVERAGE: M_unstable(u) = [some unstable (flags bit1 clear; every row when g->flags is NULL,
 *                 e.g. an rtgs_project_subset of the unstable slots), non-culled Gaussian has
 *                 power >= -4.5 and f >= 1/255 at u] (exactly T^_unstable(u) < 1, R16), tile keep
 *                 (>= 50 % of in-image pixels), kept-tile list, counts.  Writes active_bits, tile_keep,
 *                 tile_list, counts; needs proj and g->flags only (bins may be NULL).
 *  FULL or MASKED | RTGS_RENDER_COUNT: also accumulate the blended-pair count into counts[3] (reset
 *                 at the start of the call); without the flag counts[3] is not touched.
 * Blending per pixel in (zkey, gid) order: skip if power < -4.5 or f = min(0.99, alpha e^power) < 1/255;
 * the first f > e^-0.5 is the depth hit (tested before termination, R9); stop when T (1-f) < 1e-4.
 * ------------------------------------------------------------------------------------------- */
rtgs_status rtgs_render_color_depth(const rtgs_gaussians* g, const rtgs_projected* proj, const rtgs_bins* bins,
                                    const rtgs_pose* pose, const rtgs_camera* cam, int32_t mode,
                                    rtgs_render_out* out, void* stream);

/* ---------------------------------------------------------------------------------------------
 * A5 — rtgs_render_backward_masked (O5; Eq.7-8, R13, R14, R17)
 * Masked L1 loss on P (colour: mean over 3|P| values; depth: mean over P_d = P ∩ {D^ != -1} ∩ {D > 0})
 * and its gradient with respect to the parameters of the UNSTABLE Gaussians only (slot_of_gid[gid] >= 0).
 * `fwd` must hold a MASKED (or FULL) render of the same proj/bins plus the COVERAGE fields.
 *   slot_of_gid [n]       slot of each Gaussian, -1 for stable / not optimised
 *   gid_of_slot [n_slots] inverse map
 *   grad [n_slots][10+3K] ACCUMULATED (+=): pos 3, log_scale 3, rot 4, sh K*3 (DC first)
 *   loss_out [4] device float, OVERWRITTEN: L_color, L_depth, w_c L_color + w_d L_depth, |P_d|
 * With f3 bins (bins->sub_rec set) the subset rows must be the slots: bins->sub_gid == gid_of_slot.
 * No gradient flows through discrete choices (hit, 60 deg branch, termination, cut-offs, clamps; R17)
 * nor to opacity (lr_alpha = 0).
 * ------------------------------------------------------------------------------------------- */
size_t rtgs_backward_workspace_size(int32_t n_slots);
rtgs_status rtgs_render_backward_masked(const rtgs_gaussians* g, const rtgs_projected* proj, const rtgs_bins* bins,
                                        const rtgs_pose* pose, const rtgs_camera* cam, const rtgs_render_out* fwd,
                                        const rtgs_frame* target, const rtgs_loss_weights* w,
                                        const int32_t* slot_of_gid, const int32_t* gid_of_slot, int32_t n_slots,
                                        float* grad, float* loss_out, void* workspace, size_t workspace_bytes,
                                        void* stream);

/* ---------------------------------------------------------------------------------------------
 * A6 — rtgs_adam_step_unstable (O6; Eq.8, R18-R20)
 * For each slot s (gid = gid_of_slot[s]): for transparent slots add grad of w_reg L_reg,
 * L_reg = mean over the 10 n_transparent geometry scalars of (theta - init_geom)^2; one Adam step
 * (bias correction with `step` >= 1) with the group learning rates; eta[gid] += 1 iff any SH gradient
 * component of the slot is non-zero; grad is consumed and ZEROED.
 * step_device (nullable): device int32 holding the step; when given it replaces `step` (read by the
 * kernel, so a captured CUDA graph can advance the step between replays).
 *   m, v [n_slots][10+3K] Adam moments; init_geom [n_slots][10] (pos 3, log_scale 3, rot 4) (D12)
 * ------------------------------------------------------------------------------------------- */
rtgs_status rtgs_adam_step_unstable(rtgs_params* params, const int32_t* gid_of_slot, int32_t n_slots,
                                    const uint8_t* flags, float* grad, float* m, float* v, const float* init_geom,
                                    int32_t n_transparent, float w_reg, const rtgs_hparams* hp, int32_t step,
                                    const int32_t* step_device, uint32_t* eta, void* stream);

/* ---------------------------------------------------------------------------------------------
 * A5 + A6 fused — rtgs_backward_adam_unstable (same passages as the two calls above)
 * Exactly rtgs_render_backward_masked into a zeroed gradient followed by rtgs_adam_step_unstable
 * with w_reg = w->w_reg, for the case where one backward feeds one Adam step (a single view on one
 * GPU): the slot gradient stays in shared memory of the chain-rule kernel, which applies the update
 * (same float32 operations as the stand-alone Adam), so no grad buffer is read, written or zeroed.
 * `params` must name the arrays of `g` (the parameters are updated in place, the map's other fields
 * are read only).  Arguments otherwise as in the two calls; workspace = rtgs_backward_workspace_size.
 * Views that accumulate gradients (the keyframe step (e)) or an all-reduce between backward and
 * update (multi-GPU) use the two separate calls.
 * ------------------------------------------------------------------------------------------- */
rtgs_status rtgs_backward_adam_unstable(const rtgs_gaussians* g, const rtgs_projected* proj, const rtgs_bins* bins,
                                        const rtgs_pose* pose, const rtgs_camera* cam, const rtgs_render_out* fwd,
                                        const rtgs_frame* target, const rtgs_loss_weights* w,
                                        const int32_t* slot_of_gid, const int32_t* gid_of_slot, int32_t n_slots,
                                        rtgs_params* params, float* m, float* v, const float* init_geom,
                                        int32_t n_transparent, const rtgs_hparams* hp, int32_t step,
                                        const int32_t* step_device, uint32_t* eta, float* loss_out, void* workspace,
                                        size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * A7 — rtgs_classify_and_add_pixels (O7; Eq.6, R21, R22, R24)
 * On a FULL render at the new frame's pose, in float32 with this exact operation order:
 *   valid = isfinite(D) && D > 0
 *   M_s   = valid && (T^ > delta_T || |D^ - D| > delta_d)
 *   err   = ((|dR| + |dG|) + |dB|) / 3,  dX = C^_X - C_X
 *   M_c   = valid && !M_s && err > delta_c
 *   sampled(u) = (splitmix64(seed ^ (frame_idx << 32) ^ (py*W+px)) >> 32) < round(ratio * 2^32)
 * pixel_class [H][W] = mask (0 none, 1 M_s, 2 M_c) | sampled << 2 | action << 3 with action
 *   1 OPAQUE_NEW (sampled M_s), 2 TRANSPARENT_NEW (sampled M_c whose I^ Gaussian is stable),
 *   3 SKIP (sampled M_c whose I^ Gaussian is unstable).
 * samples [cap]: (py*W+px) | action << 30 for actions 1 and 2, in row-major order.
 * counts [5] device: |M_s|, |M_c|, #OPAQUE_NEW, #TRANSPARENT_NEW, #SKIP (samples beyond cap dropped).
 * ------------------------------------------------------------------------------------------- */
size_t rtgs_classify_workspace_size(const rtgs_camera* cam);
rtgs_status rtgs_classify_and_add_pixels(const rtgs_render_out* full, const rtgs_frame* frame, const uint8_t* flags,
                                         const rtgs_camera* cam, const rtgs_add_params* ap, uint8_t* pixel_class,
                                         uint32_t* samples, uint32_t cap, uint32_t* counts, void* workspace,
                                         size_t workspace_bytes, void* stream);

/* =============================================================================================
 * NEXT row f1: window fusion and state management, run after each optimisation window.
 * flags bit2 = removed (an absorbing state; rtgs_project_gaussians culls removed Gaussians).
 * ============================================================================================= */

/* rtgs_fuse_window (Eq.9): for every slot s (gid = gid_of_slot[s]),
 *   w = (eta'[gid] - eta_before[s]) / eta'[gid]   (w = 0 when eta' = 0),
 *   theta = (1 - w) before[s] + w theta'   for all 10 + 3K stored components (pos, log_scale,
 *   unnormalised quaternion, SH; reading R27: component-wise, the forward normalises q).
 * before [n_slots][10+3K]: parameters at the start of the window (same row layout as grad). */
rtgs_status rtgs_fuse_window(rtgs_params* params, const int32_t* gid_of_slot, int32_t n_slots, const float* before,
                             const uint32_t* eta_before, const uint32_t* eta, void* stream);

/* State thresholds (delta_e, delta_t unstated in the paper: reading R28). */
typedef struct {
  float delta_c, delta_d;            /* colour / depth error thresholds (P:273 reuses delta_c, delta_d) */
  uint32_t delta_e, delta_eta, delta_t;
  uint32_t frame_idx;                /* k */
} rtgs_state_params;

/* rtgs_manage_states on the optimised scene's FULL render at frame k:
 *  1. every pixel with valid depth whose hit Gaussian I^ is stable and whose error exceeds a
 *     threshold (mean |dRGB| > delta_c, float32 order of A7, or |D^ - D| > delta_d) marks that
 *     Gaussian; every marked Gaussian gets e += 1 (once per frame, R28);
 *  2. per Gaussian, from its state at entry: stable with e > delta_e -> unstable (e, eta reset,
 *     t = k, R29); unstable with eta > delta_eta -> stable; otherwise unstable with
 *     k - t > delta_t -> removed.  Removed Gaussians are untouched.
 * err_count, eta, t_created [n] uint32 in/out; flags [n] in/out; counts [4] device out:
 * #marked, #stable->unstable, #unstable->stable, #removed.  workspace: rtgs_state_workspace_size(n). */
size_t rtgs_state_workspace_size(int32_t n);
rtgs_status rtgs_manage_states(const rtgs_render_out* full, const rtgs_frame* frame, const rtgs_camera* cam,
                               uint8_t* flags, uint32_t* err_count, uint32_t* eta, uint32_t* t_created, int32_t n,
                               const rtgs_state_params* sp, uint32_t* counts, void* workspace, size_t workspace_bytes,
                               void* stream);

/* =============================================================================================
 * NEXT row f3: window-level stable-projection cache.
 * During a window the stable Gaussians and the window's poses are fixed (only unstable slots are
 * optimised), so the stable part of every window frame's (tile, zkey, gid)-sorted lists is built
 * once from that frame's FULL bins; each iteration re-projects only the unstable slots and merges
 * them in.  The merged order is the unique (tile, zkey bits, gid) order, so every result equals the
 * uncached path (rtgs_project_gaussians + rtgs_bin_and_sort) on the same parameters.
 * ============================================================================================= */

/* rtgs_project_subset: rtgs_project_gaussians for the Gaussians gid_list[0..n_list) only; row i of
 * every field of `out` describes Gaussian gid_list[i] (out sized for n_list rows).  gid_list entries
 * must be valid gids (0 <= gid < g->n). */
rtgs_status rtgs_project_subset(const rtgs_gaussians* g, const int32_t* gid_list, int32_t n_list,
                                const rtgs_pose* pose, const rtgs_camera* cam, rtgs_projected* out, void* stream);

/* rtgs_stable_cache_build: from FULL bins (every tile, all Gaussians), keep per tile the entries
 * whose Gaussian is stable (flags bit1), in order.  cache->sorted_gid needs full->capacity entries;
 * cache->tile_range [TX*TY][2] is written (a tile's stable entries stay inside its full range);
 * cache->n_instances (nullable) receives the number of stable instances. */
rtgs_status rtgs_stable_cache_build(const rtgs_bins* full, const uint8_t* flags, const rtgs_camera* cam,
                                    rtgs_bins* cache, void* stream);

/* rtgs_bin_and_sort_cached: the masked-iteration bins of rtgs_bin_and_sort(..., tile_keep, ...)
 * without re-projecting the stable Gaussians.  Inputs: `proj` (the frame's full projection; only
 * zkey of cached gids is read), `cache` (rtgs_stable_cache_build of the same frame), `sub` (the
 * rtgs_project_subset rows of the unstable Gaussians sub_gid[0..n_sub), which MUST be strictly
 * increasing), tile_keep (required).  The subset rows of the kept tiles are binned and sorted,
 * then merged per kept tile with the cached stable list by (zkey bits, gid).  Output entries are
 * gids (stable) or 0x80000000 | row (subset); on return out->sub_rec / sub_zkey / sub_gid are set to
 * sub->rec, sub->zkey, sub_gid.  n_instances / capacity as in rtgs_bin_and_sort. */
size_t rtgs_bin_cached_workspace_size(int32_t n_sub, const rtgs_camera* cam, uint32_t capacity);
rtgs_status rtgs_bin_and_sort_cached(const rtgs_projected* proj, const rtgs_bins* cache, const rtgs_projected* sub,
                                     const int32_t* sub_gid, int32_t n_sub, const rtgs_camera* cam,
                                     const uint8_t* tile_keep, rtgs_bins* out, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* =============================================================================================
 * NEXT row f2: Gaussian insertion for the sampled add-mask pixels
 * (P:232 input pre-processing, Supp. A Eq.11; readings R26, R30-R32).
 * ============================================================================================= */

/* The growable map: the arrays of rtgs_gaussians plus the per-Gaussian state, `capacity` rows
 * allocated, rows [0, n) live.  eta / err_count / t_created as in rtgs_manage_states. */
typedef struct {
  float *pos, *log_scale, *rot, *opacity, *sh;
  uint8_t* flags;
  uint32_t *eta, *err_count, *t_created;
  int32_t n, capacity, sh_degree;
} rtgs_map;

typedef struct {
  float normal_guard;          /* 0.1 m: a central-difference neighbour depth further than this from
                                  D(u) (float32 |D_nb - D| > guard) invalidates the normal (R31)      */
  float min_scale;             /* 1e-4 m lower clamp of s_1 (R30)                                     */
  float max_scale_transparent; /* 0.01 m                                                      */
  float cell;                  /* finest kNN grid cell in metres (<= 0: 0.02); performance only        */
  uint32_t frame_idx;          /* t = k of the new Gaussians                                  */
} rtgs_insert_params;

/* rtgs_add_gaussians: for the first min(add_counts[2] + add_counts[3], sample_cap) entries of the
 * A7 sample list (pixel | action << 30; action 1 opaque alpha 0.99, 2 transparent alpha 0.1) on the
 * frame (C_k, D_k) at camera->world pose T_{g,k}:
 *   v = D(u) K^-1 (px, py, 1) (R1), n = normalize((v(u+x) - v(u-x)) x (v(u+y) - v(u-y))) facing the
 *   camera; sample skipped when a 4-neighbour is off-image / invalid (R24) / beyond the guard or the
 *   cross product vanishes (R31);  V^g = R v + t, N^g = R n (float64);
 *   s_1 = max(min_scale, sqrt(max(0, 1/3 sum_i (|V^g - p_i| - (a_i + b_i)/2)))) over the 3 nearest
 *   non-removed Gaussians of rows [0, n) by (distance, gid), a_i, b_i the two largest exp(log_scale)
 *   (Eq.11, R26, R30); fewer than 3 candidates: s_1 = 2 D(u) / f_x; transparent: min(s_1, max);
 *   log_scale = log(s_1, s_1, 0.1 s_1); rotation taking e_z (the shortest axis) to N^g; SH DC
 *   (c - 0.5) / C0, higher bands 0 (R32); flags = transparent ? 1 : 0 (unstable); eta = e = 0, t = k.
 * New rows are appended at n, n+1, ... in sample order (rows past `capacity` are dropped).
 * result [5] device out: #opaque added, #transparent added, #skipped (invalid normal), #dropped
 * (capacity), n after.  The caller reads result[4] to learn the new n (map->n is not changed).
 * workspace: rtgs_insert_workspace_size(map->n, sample_cap). */
size_t rtgs_insert_workspace_size(int32_t n, uint32_t sample_cap);
rtgs_status rtgs_add_gaussians(const rtgs_map* map, const uint32_t* samples, uint32_t sample_cap,
                               const uint32_t* add_counts, const rtgs_frame* frame, const rtgs_pose* pose,
                               const rtgs_camera* cam, const rtgs_insert_params* ip, uint32_t* result,
                               void* workspace, size_t workspace_bytes, void* stream);

/* =============================================================================================
 * NEXT row f4: frame-to-model point-to-plane ICP tracking (Eq.10, P:278-282;
 * readings R31, R33-R35).  A second workload on the renderer: the model maps are a FULL render of
 * the optimised map at the previous pose (rtgs_render_out depth, normal).
 * ============================================================================================= */
typedef struct {
  int32_t levels;        /* pyramid levels 1..4 (3)                                                  */
  int32_t iters[4];      /* Gauss-Newton iterations per level, [0] = full resolution: {4, 5, 10}     */
  float normal_guard;    /* 0.1 m (R31)                                                             */
  double dist_gate;      /* 0.1 m: |T v - m| gate                                                   */
  double cos_gate;       /* cos 30 deg: n_cur . n_model gate (world frame)                          */
  double eps;            /* 1e-6: a level stops when |delta| < eps                                  */
  int32_t min_pairs;     /* 6: a level stops with fewer pairs                                       */
} rtgs_icp_params;

/* rtgs_icp_track: pyramid of the current depth D_k (R33: per 2x2 block the valid depth closest to
 * the block mean; f/2, (c - 0.5)/2 per level), float64 vertex / normal maps per level (R31), then
 * coarse -> fine Gauss-Newton on E(xi) = sum ((T v - m) . n_m)^2: every valid current pixel is
 * transformed by the running estimate T (pose_io), projected with the level-0 intrinsics into the
 * model maps at model_pose (u^ = the nearest pixel; within 1e-9 px of x.5 the lower one), paired when
 * D^(u^) > 0, |T v - m| <= dist_gate and
 * (R n) . n_m >= cos_gate, m = model_pose (D^ K^-1 (u^, 1)), n_m = N^(u^) (R34); delta =
 * -(J^T J + lambda I)^-1 J^T r with lambda = 1e-6 max diag(J^T J), J = (n_m, p x n_m),
 * T <- Exp(delta) T (R35).
 *   depth        [H][W] current frame D_k (metres; <= 0 / non-finite invalid)
 *   model_depth  [H][W] D^* (-1 = no hit), model_normal [3][H][W] world N^* (rtgs_render_out of a
 *                FULL render at model_pose)
 *   pose_io      device double[12]: camera->world R (row-major) then t; in: initial estimate, out: T_k
 *   diag         device double[4 * sum(iters)]: per iteration (level, E, #pairs, |delta|), level -1
 *                for iterations skipped after convergence
 * workspace: rtgs_icp_workspace_size(cam, levels).  No host synchronisation (graph-capturable). */
size_t rtgs_icp_workspace_size(const rtgs_camera* cam, int32_t levels);
rtgs_status rtgs_icp_track(const float* depth, const float* model_depth, const float* model_normal,
                           const rtgs_pose* model_pose, const rtgs_camera* cam, const rtgs_icp_params* params,
                           double* pose_io, double* diag, void* workspace, size_t workspace_bytes, void* stream);

/* =============================================================================================
 * Input decode (P:232 input pre-processing): sensor-native RGB-D to the planar float32 frame.
 * rgb [H][W][3] uint8 interleaved -> color [3][H][W] = rgb * (1/255) (float32 product);
 * depth_raw [H][W] uint16 -> depth [H][W] = raw * (1/depth_scale) metres (TUM: 5000, Replica:
 * 6553.5 raw units per metre); raw 0 -> 0 (invalid, R24).  rgb 4-byte aligned, depth_raw 8-byte
 * aligned, outputs 16-byte aligned.
 * ============================================================================================= */
rtgs_status rtgs_decode_rgbd(const uint8_t* rgb, const uint16_t* depth_raw, int32_t width, int32_t height,
                             float depth_scale, float* color, float* depth, void* stream);

/* =============================================================================================
 * Map layout (a framework step, not a step of the method): spatial order of the Gaussians.
 * The paper's maps grow frame by frame from row-major pixel samples, so nearby Gaussians
 * sit at nearby indices; these calls restore that coherence for a map in arbitrary order, which the
 * binning's per-tile counters, the renderer's record gathers and the backward's gradient rows use.
 *
 * rtgs_morton_order: perm[r] = the gid at rank r when the live Gaussians (flags bit 2 clear; flags
 *   NULLABLE = all live) are sorted by the 30-bit Morton code of their position quantised in the live
 *   bounding box (per axis q = min(1023, (int)((p - lo) * (1024 / (hi - lo)))), float32 ops in that
 *   order; a zero extent gives q = 0), ties by gid; removed Gaussians last, in gid order.  pos [n][3];
 *   perm [n] device (uint32).  Workspace: rtgs_morton_workspace_size(n).
 * rtgs_gather_rows: dst row r = src row perm[r] (rows of row_bytes bytes; n rows; src and dst must
 *   not overlap) - applies a permutation to any per-Gaussian array. */
size_t rtgs_morton_workspace_size(int32_t n);
rtgs_status rtgs_morton_order(const float* pos, const uint8_t* flags, int32_t n, uint32_t* perm, void* workspace,
                              size_t workspace_bytes, void* stream);
rtgs_status rtgs_gather_rows(const void* src, void* dst, const uint32_t* perm, int32_t n, int32_t row_bytes,
                             void* stream);

/* rtgs_coverage_and_bin_cached: the f3 iteration's A0 + A2 in one call.  The subset rows are binned
 * over ALL tiles; M_unstable (R16) is decided per tile from those lists (every pixel tests the tile's
 * unstable instances until its first hit — identical decisions to the COVERAGE mode), giving
 * active_bits, tile_keep, tile_list and counts[0..2] in `cov`; then the kept tiles are merged with
 * the cached stable lists exactly as rtgs_bin_and_sort_cached does with that tile_keep.
 * Workspace: rtgs_bin_cached_workspace_size. */
rtgs_status rtgs_coverage_and_bin_cached(const rtgs_projected* proj, const rtgs_bins* cache, const rtgs_projected* sub,
                                         const int32_t* sub_gid, int32_t n_sub, const rtgs_camera* cam,
                                         rtgs_render_out* cov, rtgs_bins* out, void* workspace,
                                         size_t workspace_bytes, void* stream);

/* The two halves of rtgs_coverage_and_bin_cached, for overlapping the first with the ingest that
 * builds the cache: rtgs_coverage_subset (bins the subset over all tiles into the workspace and
 * writes the coverage fields of `cov`; reads no cache) then rtgs_merge_cached (same workspace, the
 * same sub / n_sub / capacity, cov->tile_keep from the first call). */
rtgs_status rtgs_coverage_subset(const rtgs_projected* sub, int32_t n_sub, const rtgs_camera* cam, rtgs_render_out* cov,
                                 uint32_t capacity, void* workspace, size_t workspace_bytes, void* stream);
rtgs_status rtgs_merge_cached(const rtgs_projected* proj, const rtgs_bins* cache, const rtgs_projected* sub,
                              const int32_t* sub_gid, int32_t n_sub, const rtgs_camera* cam,
                              const rtgs_render_out* cov, rtgs_bins* out, void* workspace, size_t workspace_bytes,
                              void* stream);

/* =============================================================================================
 * (e) keyframe global optimisation: the pixels with the top `ratio` (0.4) colour errors of
 * a keyframe (reading R36).  err = ((|dR| + |dG|) + |dB|) / 3 in float32 between the keyframe's
 * FULL render `full->color` and its colour `frame_color`; K = round(ratio * H * W) (float64); the K
 * largest, ties by row-major pixel index (lower first), by an exact radix select on the float bits.
 * Writes out->active_bits (the selected pixels), out->tile_keep / tile_list (every tile with a
 * selected pixel) and out->counts[0..2] (#tiles, K, K): the inputs rtgs_render_backward_masked needs
 * with the FULL render's other fields.
 * ============================================================================================= */
size_t rtgs_topk_workspace_size(const rtgs_camera* cam);
rtgs_status rtgs_topk_error_mask(const float* color_hat, const float* frame_color, const rtgs_camera* cam, double ratio,
                                 rtgs_render_out* out, void* workspace, size_t workspace_bytes, void* stream);

/* Utilities */
const char* rtgs_status_string(rtgs_status s);
const char* rtgs_last_cuda_error(void);
int32_t rtgs_version(void);
/* Number of kernel launches the library has enqueued since load (for bench accounting). */
uint64_t rtgs_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* RTGS_H */
