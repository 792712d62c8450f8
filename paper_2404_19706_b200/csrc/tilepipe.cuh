// tilepipe.cuh — warp-specialised producer/consumer pipeline over one tile's depth-sorted list,
// shared by the forward render (A3/A4) and the backward replay (A5).
//
// CTA = NW consumer warps (one 8x4 pixel block each, one pixel per lane) + 1 producer warp.
// The producer streams the tile's records in batches of kPipeBatch through a kPipeStages-deep ring
// in shared memory with cp.async (LDGSTS) and signals each stage on a `full` mbarrier
// (cp.async.mbarrier.arrive.noinc: the arrival fires when the lane's copies have landed).  Every
// consumer warp releases a stage on its `empty` mbarrier when it is done with it, so consumer
// warps never wait for each other (no __syncthreads in the main loop): a warp can run up to
// kPipeStages batches ahead of the slowest one.  When every consumer warp has terminated, the
// producer stops copying and only signals, and the CTA drains.
#pragma once
#include "common.cuh"
#include <type_traits>

namespace rtgs {

#ifndef RTGS_PIPE_STAGES
#define RTGS_PIPE_STAGES 3
#endif
#ifndef RTGS_PIPE_BATCH
#define RTGS_PIPE_BATCH 256
#endif
constexpr int kPipeStages = RTGS_PIPE_STAGES;  // (swept in round 2: 4 x 128 vs 3 x 256: 3 x 256 kept)
constexpr int kPipeBatch = RTGS_PIPE_BATCH;    // <= 256: stage indices are bytes
// consumer warps per CTA: 8 = a whole 16x16 tile (FULL render: thousands of tiles), 4 = half a tile
// (MASKED render and backward: only the kept tiles, so half-tile CTAs double the parallelism and
// even out the per-SM load)
constexpr int kTileWarps = 8;
constexpr int kHalfWarps = 4;

// GID: the ring also holds each record's list entry (the backward's gradient targets); the forward
// fetches only its hit's entry, after the walk
// S stages of B records (B <= 256: stage indices are bytes); kernels pick their own ring size
template <bool GID, int S = kPipeStages, int B = kPipeBatch>
struct PipeRingT {
  static constexpr int kS = S, kB = B;
  float4 rec[S][B][3];  // first 48 B of each record: mu hi/lo, conic', log2 alpha, rgb, ext
  uint32_t gid[GID ? S : 1][GID ? B : 1];
  uint8_t boxmask[S][B];  // bit w: the record's support box overlaps warp w's block
  uint64_t full[S];
  uint64_t empty[S];
  int alive;                                // consumer warps not yet terminated
};
using PipeRing = PipeRingT<true>;

template <int NW, typename Ring>
__device__ __forceinline__ void pipe_init(Ring& r) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < Ring::kS; ++s) {
      mbar_init(&r.full[s], 32);
      mbar_init(&r.empty[s], NW);
    }
    r.alive = NW;
    fence_mbar_init();
  }
}

// Keep a loop-invariant value in a register: the compiler otherwise re-derives shared addresses
// (S2UR SR_CgaCtaId) and lane bits (S2R SR_TID) inside the inner loops, paying their latency there.
__device__ __forceinline__ uint32_t pin(uint32_t x) {
  asm volatile("" : "+r"(x));
  return x;
}

// explicit shared-space 128-bit load (32-bit shared address: no generic-to-shared conversion in
// the consumers' inner loops)
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t lds8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];\n" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts8(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(addr));
  return v;
}

// list entries: a gid of `rec`, or (NEXT f3 cached bins) 0x80000000 | row of the subset records
constexpr uint32_t kSubBit = 0x80000000u;
__device__ __forceinline__ const float4* entry_rec(const float4* rec, const float4* sub_rec, uint32_t e) {
  return (e & kSubBit) ? sub_rec + (size_t)4 * (e & ~kSubBit) : rec + (size_t)4 * e;
}

// the flush of a producer whose stages need no per-stage epilogue (the forward render)
struct NoFlush {
  __device__ void operator()(int, int) const {}
};

// producer: one lane per record slot; `extra(stage, j, entry)` may issue more cp.async.
// REV: the batches run back to front (batch b holds positions [max(start, end - 128 (b+1)), end - 128 b),
// in list order inside the stage) for the backward's back-to-front pass.
template <int B = kPipeBatch>
__device__ __forceinline__ int pipe_batch_lo(bool rev, int start, int end, int b) {
  return rev ? max(start, end - (b + 1) * B) : start + b * B;
}
template <int B = kPipeBatch>
__device__ __forceinline__ int pipe_batch_cnt(bool rev, int start, int end, int b) {
  return rev ? (end - b * B) - max(start, end - (b + 1) * B) : min(B, end - start - b * B);
}
// NBOX > 0: once a stage's copies have landed, the producer also writes boxmask: for each record
// the NBOX consumer warps' 8x4 blocks (warp w at (bx, by) + ((w & 1) * 8, (w >> 1) * 4)) its support
// box overlaps -- the test every consumer warp made on its own per record before (the same float
// comparisons, so the same decisions), now once per record instead of once per (record, warp)
template <bool REV = false, int NBOX = 0, bool GID = true, int S = kPipeStages, int B = kPipeBatch,
          typename Extra, typename Flush>
__device__ __forceinline__ void pipe_produce(PipeRingT<GID, S, B>& r, const float4* __restrict__ rec,
                                             const float4* __restrict__ sub_rec,
                                             const uint32_t* __restrict__ sorted_gid, int start, int end,
                                             Extra extra, Flush flush, float bx = 0.f, float by = 0.f) {
  const int lane = threadIdx.x & 31;
  const int n = end - start;
  const int nb = n > 0 ? (n + B - 1) / B : 0;
  for (int b = 0; b < nb; ++b) {
    const int st = b % S;
    const uint32_t ph = (uint32_t)(b / S) & 1u;
    if (b >= S) {
      mbar_wait_sleep(&r.empty[st], ph ^ 1u);  // (suspended, not spinning: measured neutral on time)
      flush(st, b - S);
    }
    if (*((volatile int*)&r.alive) > 0) {
      const int lo = pipe_batch_lo<B>(REV, start, end, b);
      const int cnt = pipe_batch_cnt<B>(REV, start, end, b);
      constexpr int PER = B / 32;
      uint32_t g[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) {  // all gid loads of the batch in flight together
        const int j = lane + 32 * q;
        g[q] = j < cnt ? sorted_gid[lo + j] : 0u;
      }
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int j = lane + 32 * q;
        if (j < cnt) {
          if constexpr (GID) cp_async4(&r.gid[st][j], sorted_gid + lo + j);
          const float4* src = entry_rec(rec, sub_rec, g[q]);
          cp_async16(&r.rec[st][j][0], src);
          cp_async16(&r.rec[st][j][1], src + 1);
          cp_async16(&r.rec[st][j][2], src + 2);
          extra(st, j, g[q]);
        }
      }
      if constexpr (NBOX > 0) {
        asm volatile("cp.async.wait_all;\n" ::: "memory");  // this stage's records have landed
        __syncwarp();
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          const int j = lane + 32 * q;
          if (j < cnt) {
            const float4 r0 = r.rec[st][j][0];
            const float2 ext = unpack_ext(r.rec[st][j][2].w);
            uint32_t m = 0u;
#pragma unroll
            for (int w = 0; w < NBOX; ++w) {
              const float bx0 = bx + (float)((w & 1) * 8), bx1 = bx0 + 7.f;
              const float by0 = by + (float)((w >> 1) * 4), by1 = by0 + 3.f;
              const bool ov = (r0.x + ext.x >= bx0) && (r0.x - ext.x <= bx1) && (r0.y + ext.y >= by0) &&
                              (r0.y - ext.y <= by1);
              m |= ov ? (1u << w) : 0u;
            }
            r.boxmask[st][j] = (uint8_t)m;
          }
        }
      }
    }
    if constexpr (NBOX > 0) mbar_arrive(&r.full[st]);  // (copies waited for: a plain arrival)
    else cp_async_mbar_arrive(&r.full[st]);
  }
  // the last stages are flushed once every consumer warp has released them (a producer without a
  // flush has nothing left to do: it exits, and the ring lives on with the CTA)
  if constexpr (!std::is_same_v<Flush, NoFlush>) {
    for (int b = max(0, nb - S); b < nb; ++b) {
      const int st = b % S;
      mbar_wait_sleep(&r.empty[st], (uint32_t)(b / S) & 1u);
      flush(st, b);
    }
  }
}

// ---- span masks (render.cu forward, backward.cu backward) -------------------------------------
// 32x32 bit-matrix transpose across the warp: in, lane i holds row i (bit c = M[i][c]); out, lane p
// holds column p (bit j = M[j][p]).  Recursive block swaps, 5 shuffles.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, uint32_t lane) {
  const uint32_t M[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const uint32_t s = 16u >> i, m = M[i];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, (int)s);
    x = (lane & s) ? ((x & ~m) | ((y & ~m) >> s)) : ((x & m) | ((y & m) << s));
  }
  return x;
}

// Pixels of the 8x4 block (bx0, by0) (bit 8*row + col) that MAY pass eval_pair for record (a, c)
// (a = mu hi/lo, c = (A', B', C', log2 alpha), p2 = A' dx^2 + B' dx dy + C' dy^2, dx = mu_x - u_x).
// For pixel row y (dy = mu_y - y) the support p2 >= pm is the dx interval centred at B' dy / (2A')
// (x = mu_x - dx) of half-width sqrt(disc) / (2|A'|), disc = 4 A' pm - dy^2 (4 A'C' - B'^2).  The
// threshold is lowered by 1 % + 0.01 (a 0.5 %-larger ellipse) and the interval widened by 0.02 px, far
// beyond the float32 rounding of this computation and of eval_pair, so the mask is a superset.
__device__ __forceinline__ uint32_t support_mask(const float4 a, const float4 c, float bx0, float by0) {
  const float mx = a.x + a.z, my = a.y + a.w;
  const float pmin = fmaxf(kP2Min, kLog2FMin - c.w);
  const float pm = __fmaf_rn(pmin, 1.01f, -0.01f);
  const float D0 = 4.f * c.x * pm;                       // > 0 (A' < 0, pm < 0)
  const float D2 = __fmaf_rn(4.f * c.x, c.z, -c.y * c.y); // 4 A'C' - B'^2 > 0
  const float inv2a = -0.5f / c.x;                       // 1 / (2 |A'|)
  const float xs = -c.y * inv2a;                         // x centre = mu_x + xs dy
  uint32_t m = 0u;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float dy = my - (by0 + (float)k);
    const float disc = __fmaf_rn(-D2, dy * dy, D0);
    if (disc >= 0.f) {
      float sq;
      asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(disc));  // ~2 ulp: inside the 0.02 px margin
      const float h = __fmaf_rn(sq, inv2a, 0.02f);
      const float xc = __fmaf_rn(xs, dy, mx) - bx0;
      const int lo = (int)ceilf(fmaxf(xc - h, -1.f));
      const int hi = (int)floorf(fminf(xc + h, 8.f));
      const int l0 = max(lo, 0), h0 = min(hi, 7);
      if (l0 <= h0) m |= ((0xFFu >> (7 - (h0 - l0))) << l0) << (8 * k);
    }
  }
  return m;
}

// The same superset mask for a 16 x 2 pixel block (bit 16*row + col): the coverage kernel's warp
// (two tile rows).  Identical interval arithmetic to support_mask.
__device__ __forceinline__ uint32_t support_mask_16x2(const float4 a, const float4 c, float bx0, float by0) {
  const float mx = a.x + a.z, my = a.y + a.w;
  const float pmin = fmaxf(kP2Min, kLog2FMin - c.w);
  const float pm = __fmaf_rn(pmin, 1.01f, -0.01f);
  const float D0 = 4.f * c.x * pm;
  const float D2 = __fmaf_rn(4.f * c.x, c.z, -c.y * c.y);
  const float inv2a = -0.5f / c.x;
  const float xs = -c.y * inv2a;
  uint32_t m = 0u;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float dy = my - (by0 + (float)k);
    const float disc = __fmaf_rn(-D2, dy * dy, D0);
    if (disc >= 0.f) {
      float sq;
      asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(disc));
      const float h = __fmaf_rn(sq, inv2a, 0.02f);
      const float xc = __fmaf_rn(xs, dy, mx) - bx0;
      const int lo = (int)ceilf(fmaxf(xc - h, -1.f));
      const int hi = (int)floorf(fminf(xc + h, 16.f));
      const int l0 = max(lo, 0), h0 = min(hi, 15);
      if (l0 <= h0) m |= ((0xFFFFu >> (15 - (h0 - l0))) << l0) << (16 * k);
    }
  }
  return m;
}

struct FwdArgs {
  const float4* rec;
  const uint32_t* zkey;
  const float4* sub_rec;  // NEXT f3 subset rows (entries with kSubBit), else NULL
  const uint32_t* sub_zkey;
  const int32_t* sub_gid;
  const uint32_t* sorted_gid;
  const uint2* range;
  const uint32_t* tile_list;
  const uint32_t* counts;
  const uint32_t* active;
  CamK cam;
  float R[9];
  float* color;
  float* trans;
  float* depth;
  float* normal;
  int32_t* index;
  uint32_t* n_contrib;
};

// COUNT: accumulate the blended-pair statistic counts[3] (RTGS_RENDER_COUNT; the production renders of
// the mapping step do not, saving 3 instructions per survivor)
// LAST: track n_contrib (the sorted-list position past the last blended entry, which the backward
// needs); a FULL render for the add masks / tracking only passes n_contrib = NULL and skips it
}  // namespace rtgs
