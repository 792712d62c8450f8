// common.cuh — device helpers shared by the librtgs kernels (sm_100a).
// Nothing here is shared with oracle/ (DESIGN.md §4): constants are restated from the paper.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rtgs.h"

namespace rtgs {

// ---- constants of the method (PAPER.md; readings in DESIGN.md §3) -----------------------------
constexpr float kDeltaAlpha = 0.60653065971263342f;  // e^-0.5
constexpr float kTMin = 1e-4f;                       // early termination (R7)
constexpr float kFMin = 1.0f / 255.0f;               // R7
constexpr float kFMax = 0.99f;                       // R7
constexpr float kPowerMin = -4.5f;                   // 3 sigma (R7), used as kP2Min below
constexpr float kCos60 = 0.5f;                       // Eq.5 60 deg switch (R11)
constexpr float kNear = 0.2f;                        // R6
constexpr float kDilation = 0.3f;                    // R4
constexpr float kRectPad = 0.015625f;                // 2^-6 px (R7)
constexpr int kTile = 16;
constexpr int kRecFloats = 16;                       // projected record, 64 B

struct CamK {
  float fx, fy, cx, cy;
  int W, H, TX, TY;
};

static inline CamK make_cam(const rtgs_camera& c) {
  CamK k;
  k.fx = c.fx; k.fy = c.fy; k.cx = c.cx; k.cy = c.cy;
  k.W = c.width; k.H = c.height;
  k.TX = (c.width + kTile - 1) / kTile;
  k.TY = (c.height + kTile - 1) / kTile;
  return k;
}

// Launch accounting (rtgs_launch_count)
void note_launch(int n = 1);

// ---- small PTX wrappers --------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// mbarrier + 1D bulk copy (TMA engine, cp.async.bulk) global -> shared
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// the same wait, but the waiting warp is suspended in try_wait (up to the time hint) instead of
// re-issuing the probe: consumer warps that run ahead of the producer / the slowest warp of the CTA
// leave their issue slots to the warps still working
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// inclusive warp scan of uint32
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan (blockDim.x multiple of 32, <= 1024). Returns the exclusive prefix of v
// and writes the block total to *total. `sh` needs 33 uint32 of shared memory.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sh, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = warp_incl_scan(v);
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < nw ? sh[lane] : 0u;
    uint32_t si = warp_incl_scan(s);
    if (lane < nw) sh[lane] = si - s;
    if (lane == 31) sh[32] = si;
  }
  __syncthreads();
  uint32_t r = inc - v + sh[wid];
  *total = sh[32];
  __syncthreads();
  return r;
}

// ---- the per-pair evaluation shared by the forward and the backward replay --------------------
// Record layout (include/rtgs.h): a = (mu_x hi, mu_y hi, mu_x lo, mu_y lo),
// b = (A', B', C', log2 alpha) with the conic prescaled to base 2: A' = -log2(e)/2 A, B' = -log2(e) B,
// C' = -log2(e)/2 C, so that p2 = A' dx^2 + B' dx dy + C' dy^2 = power * log2(e) and
// f = min(0.99, 2^(p2 + log2 alpha)) = min(0.99, alpha e^power) (Eq.2).
// Support test (R7): power >= -4.5  <=>  p2 >= -4.5 log2(e);  f >= 1/255  <=>  p2 + log2 alpha >= log2(1/255).
// Every operation is an explicitly rounded intrinsic so the forward and the backward replay take
// bit-identical decisions (same T sequence, termination and hit) whatever the compiler schedules.
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kP2Min = -4.5f * 1.4426950408889634f;   // -4.5 log2(e)
constexpr float kLog2FMin = -7.9943534368588578f;       // log2(1/255)
struct PairEval {
  float dx, dy, p2, e, f;
};
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ bool eval_pair(const float4 a, const float4 b, float px, float py, PairEval& e) {
  e.dx = __fadd_rn(__fsub_rn(a.x, px), a.z);  // (mu_hi - u) is exact; + lo
  e.dy = __fadd_rn(__fsub_rn(a.y, py), a.w);
  const float u = __fmaf_rn(b.x, e.dx, __fmul_rn(b.y, e.dy));             // A' dx + B' dy
  e.p2 = __fmaf_rn(e.dx, u, __fmul_rn(__fmul_rn(b.z, e.dy), e.dy));        // + C' dy^2
  e.e = __fadd_rn(e.p2, b.w);
  e.f = fminf(kFMax, ex2_approx(e.e));
  return (e.p2 >= kP2Min) && (e.e >= kLog2FMin);
}

// mbarrier arrive / cp.async-tracked arrive (for the render pipelines)
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}

__device__ __forceinline__ float2 unpack_ext(float w) {
  const uint32_t u = __float_as_uint(w);
  return make_float2(__half2float(__ushort_as_half((unsigned short)(u & 0xFFFFu))),
                     __half2float(__ushort_as_half((unsigned short)(u >> 16))));
}

// Warp-cooperative expansion of the lanes' rect tiles (lane: nt = w x h tiles from (tx0, ty0)): the
// warp's instances (sum of nt over the lanes) are dealt out 32 per round, lane by lane in order, so a
// warp holding one large rect takes ceil(sum / 32) rounds instead of max(nt) (each with an atomic
// round trip).  f(t, o) is called warp-uniformly once per round: this lane holds an instance of tile t
// from lane o (t = -1: none this round).
// Warps whose largest rect is small (the common case: sub-tile splats) keep the plain per-lane loop
// over max(nt) rounds, which costs less per round than the expansion's search.
template <typename F>
__device__ __forceinline__ void warp_expand_tiles(int nt, int w, int tx0, int ty0, int TX, F f) {
  const int lane = threadIdx.x & 31;
  const int ntmax = (int)__reduce_max_sync(0xffffffffu, (uint32_t)nt);
  if (ntmax <= 4) {
    int cx = 0, tt = ty0 * TX + tx0;  // the lane's q-th tile, stepped row-major
    for (int q = 0; q < ntmax; ++q) {
      f(q < nt ? tt : -1, lane);
      ++tt;
      if (++cx == w) { cx = 0; tt += TX - w; }
    }
    return;
  }
  const uint32_t incl = warp_incl_scan((uint32_t)nt);
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t excl = incl - (uint32_t)nt;
  const float rw = 1.f / (float)max(w, 1);
  for (uint32_t base = 0; base < total; base += 32) {
    const uint32_t k = base + (uint32_t)lane;
    int o = 0;  // the owner: the smallest lane with incl > k (binary lifting over the 32 prefix sums)
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
      const uint32_t v = __shfl_sync(0xffffffffu, incl, o + step - 1);
      if (v <= k) o += step;
    }
    const uint32_t ex = __shfl_sync(0xffffffffu, excl, o);
    const int ow = __shfl_sync(0xffffffffu, w, o), ox = __shfl_sync(0xffffffffu, tx0, o);
    const int oy = __shfl_sync(0xffffffffu, ty0, o);
    const float orw = __shfl_sync(0xffffffffu, rw, o);
    int t = -1;
    if (k < total) {
      const int q = (int)(k - ex);  // the instance's index in its rect, row-major
      int qy = (int)(((float)q + 0.5f) * orw), qx = q - qy * ow;  // q / w in float, then exact:
      if (qx < 0) { --qy; qx += ow; } else if (qx >= ow) { ++qy; qx -= ow; }
      t = (oy + qy) * TX + ox + qx;
    }
    f(t, o);
  }
}

// warp-aggregated per-tile counting: the lanes' rect tiles expanded across the warp, one atomic per
// distinct tile per round (match_any groups; spatially coherent maps put a warp's Gaussians on few
// tiles, rtgs_morton_order)
__device__ __forceinline__ void tile_count_agg(uint32_t* cnt, int nt, int w, int tx0, int ty0, int TX,
                                               const uint8_t* keep) {
  const int lane = threadIdx.x & 31;
  warp_expand_tiles(nt, w, tx0, ty0, TX, [&](int t, int) {
    if (t >= 0 && keep && !keep[t]) t = -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, (uint32_t)t);
    if (t >= 0 && lane == __ffs(peers) - 1) atomicAdd(&cnt[t], (uint32_t)__popc(peers));
  });
}

}  // namespace rtgs
