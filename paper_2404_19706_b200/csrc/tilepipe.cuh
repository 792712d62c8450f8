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

namespace rtgs {

constexpr int kPipeStages = 4;
constexpr int kPipeBatch = 128;
// consumer warps per CTA: 8 = a whole 16x16 tile (FULL render: thousands of tiles), 4 = half a tile
// (MASKED render and backward: only the kept tiles, so half-tile CTAs double the parallelism and
// even out the per-SM load)
constexpr int kTileWarps = 8;
constexpr int kHalfWarps = 4;

struct PipeRing {
  float4 rec[kPipeStages][kPipeBatch][3];  // first 48 B of each record: mu hi/lo, conic', log2 alpha, rgb, ext
  uint32_t gid[kPipeStages][kPipeBatch];
  uint64_t full[kPipeStages];
  uint64_t empty[kPipeStages];
  int alive;                                // consumer warps not yet terminated
};

template <int NW>
__device__ __forceinline__ void pipe_init(PipeRing& r) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPipeStages; ++s) {
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

// producer: one lane per record slot; `extra(stage, j, entry)` may issue more cp.async.
// REV: the batches run back to front (batch b holds positions [max(start, end - 128 (b+1)), end - 128 b),
// in list order inside the stage) for the backward's back-to-front pass.
__device__ __forceinline__ int pipe_batch_lo(bool rev, int start, int end, int b) {
  return rev ? max(start, end - (b + 1) * kPipeBatch) : start + b * kPipeBatch;
}
__device__ __forceinline__ int pipe_batch_cnt(bool rev, int start, int end, int b) {
  return rev ? (end - b * kPipeBatch) - max(start, end - (b + 1) * kPipeBatch)
             : min(kPipeBatch, end - start - b * kPipeBatch);
}
template <bool REV = false, typename Extra, typename Flush>
__device__ __forceinline__ void pipe_produce(PipeRing& r, const float4* __restrict__ rec,
                                             const float4* __restrict__ sub_rec,
                                             const uint32_t* __restrict__ sorted_gid, int start, int end,
                                             Extra extra, Flush flush) {
  const int lane = threadIdx.x & 31;
  const int n = end - start;
  const int nb = n > 0 ? (n + kPipeBatch - 1) / kPipeBatch : 0;
  for (int b = 0; b < nb; ++b) {
    const int st = b % kPipeStages;
    const uint32_t ph = (uint32_t)(b / kPipeStages) & 1u;
    if (b >= kPipeStages) {
      mbar_wait(&r.empty[st], ph ^ 1u);
      flush(st, b - kPipeStages);
    }
    if (*((volatile int*)&r.alive) > 0) {
      const int lo = pipe_batch_lo(REV, start, end, b);
      const int cnt = pipe_batch_cnt(REV, start, end, b);
      constexpr int PER = kPipeBatch / 32;
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
          cp_async4(&r.gid[st][j], sorted_gid + lo + j);
          const float4* src = entry_rec(rec, sub_rec, g[q]);
          cp_async16(&r.rec[st][j][0], src);
          cp_async16(&r.rec[st][j][1], src + 1);
          cp_async16(&r.rec[st][j][2], src + 2);
          extra(st, j, g[q]);
        }
      }
    }
    cp_async_mbar_arrive(&r.full[st]);
  }
  // the last stages are flushed once every consumer warp has released them
  for (int b = max(0, nb - kPipeStages); b < nb; ++b) {
    const int st = b % kPipeStages;
    mbar_wait(&r.empty[st], (uint32_t)(b / kPipeStages) & 1u);
    flush(st, b);
  }
}

}  // namespace rtgs
