// render.cu — A0 unstable coverage + tile keep (O4; Eq.12, R15, R16) and
//             A3/A4 forward colour/transmission blending with the opaque-disc depth (O2/O3;
//             Eq.1-5, R7-R12).
//
// Forward: one CTA per 16x16 tile (FULL) or per half of a kept tile (MASKED) = 8 / 4 consumer warps
// (warp w owns an 8x4 pixel block, one pixel per lane) + 1 producer warp streaming the tile's depth-sorted records through a 4-stage
// shared-memory ring (tilepipe.cuh).  Each consumer warp culls a batch 32 records at a time against
// its 8x4 block (ballot over the records' support boxes); for the survivors it builds exact support
// span masks (one per survivor, transposed to one bit list per pixel) and each lane walks only its
// own pixel's pairs (the span path below; RTGS_RENDER_DENSE keeps the dense walk for verification).
// Pixels stop at T (1 - f) < 1e-4; warps stop when all their lanes stopped; the producer stops when
// all did.
#include "common.cuh"
#include "internal.h"
#include "tilepipe.cuh"

namespace rtgs {

// ------------------------------------------------------------------------------------------------
// A0: coverage by splatting the unstable Gaussians (existence test, no order needed, R16)
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_coverage(const float4* __restrict__ rec, const uint2* __restrict__ rect,
                                                  const uint32_t* __restrict__ zkey, const uint8_t* __restrict__ flags,
                                                  int n, int W, uint32_t* __restrict__ bits) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool mine = i < n && (!flags || !(flags[i] & 2u)) && zkey[i] != 0xFFFFFFFFu;  // NULL: all rows
  // every lane prefetches its own Gaussian; the warp then splats them one by one via shuffles
  uint2 myr = make_uint2(1u | (1u << 16), 0u);
  float4 mya = make_float4(0, 0, 0, 0), myb = mya;
  if (mine) {
    myr = rect[i];
    mya = rec[4 * (size_t)i];
    myb = rec[4 * (size_t)i + 1];
  }
  uint32_t m = __ballot_sync(0xffffffffu, mine);
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    uint2 r;
    r.x = __shfl_sync(0xffffffffu, myr.x, src);
    r.y = __shfl_sync(0xffffffffu, myr.y, src);
    const int x0 = (int)(short)(r.x & 0xFFFF), y0 = (int)(short)(r.x >> 16);
    const int x1 = (int)(short)(r.y & 0xFFFF), y1 = (int)(short)(r.y >> 16);
    if (x0 > x1 || y0 > y1) continue;
    float4 a, b;
    a.x = __shfl_sync(0xffffffffu, mya.x, src); a.y = __shfl_sync(0xffffffffu, mya.y, src);
    a.z = __shfl_sync(0xffffffffu, mya.z, src); a.w = __shfl_sync(0xffffffffu, mya.w, src);
    b.x = __shfl_sync(0xffffffffu, myb.x, src); b.y = __shfl_sync(0xffffffffu, myb.y, src);
    b.z = __shfl_sync(0xffffffffu, myb.z, src); b.w = __shfl_sync(0xffffffffu, myb.w, src);
    const int w = x1 - x0 + 1, h = y1 - y0 + 1;
    auto splat = [&](int px, int py) {
      PairEval e;
      if (eval_pair(a, b, (float)px, (float)py, e)) {
        const uint32_t lin = (uint32_t)py * (uint32_t)W + (uint32_t)px;
        atomicOr(&bits[lin >> 5], 1u << (lin & 31u));
      }
    };
    if (w <= 32) {  // the warp covers rpi = 32 / w rows per step; one division per Gaussian, not per pixel
      const int rpi = 32 / w;
      const int ry = lane / w, rx = lane - ry * w;
      if (ry < rpi)
        for (int py = y0 + ry; py <= y1; py += rpi) splat(x0 + rx, py);
    } else {
      const int tot = w * h;
      for (int p = lane; p < tot; p += 32) splat(x0 + p % w, y0 + p / w);
    }
  }
}

template <bool ANY>  // ANY: keep every tile with an active pixel ((e) top-k masks), else the 50 % rule
__global__ void __launch_bounds__(256) k_tile_keep(const uint32_t* __restrict__ bits, int W, int H, int TX,
                                                   uint8_t* __restrict__ keep, uint32_t* __restrict__ list,
                                                   uint32_t* __restrict__ counts) {
  const int t = blockIdx.x;
  const int px = (t % TX) * kTile + (threadIdx.x & 15), py = (t / TX) * kTile + (threadIdx.x >> 4);
  const bool inside = px < W && py < H;
  bool act = false;
  if (inside) {
    const uint32_t lin = (uint32_t)py * (uint32_t)W + (uint32_t)px;
    act = (bits[lin >> 5] >> (lin & 31u)) & 1u;
  }
  const int na = __syncthreads_count(act);
  const int ni = __syncthreads_count(inside);
  if (threadIdx.x == 0) {
    const bool k = ANY ? na > 0 : 2 * na >= ni;  // P:497 / R15: discard tiles with < 50 % active pixels
    keep[t] = k ? 1 : 0;
    if (k) {
      const uint32_t pos = atomicAdd(&counts[0], 1u);
      list[pos] = (uint32_t)t;
      atomicAdd(&counts[1], (uint32_t)na);
    }
    if (na) atomicAdd(&counts[2], (uint32_t)na);
  }
}

// A0 from tile lists (f3 flow): one CTA per tile, one pixel per thread.  The tile's unstable
// instances (any order: an existence test, R16) are staged 256 at a time; every pixel evaluates them
// until its first hit.  Large splats are spread over their tiles, so the work is balanced; the tile
// keep, kept-tile list and counts come out of the same CTA.
__global__ void __launch_bounds__(256) k_tile_coverage(const uint2* __restrict__ srange,
                                                       const unsigned long long* __restrict__ keys,
                                                       const float4* __restrict__ sub_rec, int W, int H, int TX,
                                                       uint32_t* __restrict__ bits, uint8_t* __restrict__ keep,
                                                       uint32_t* __restrict__ list, uint32_t* __restrict__ counts) {
  __shared__ float4 sa[256], sb[256];
  __shared__ float se[256];
  const int t = blockIdx.x;
  const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
  const int px = (t % TX) * kTile + lx, py = (t / TX) * kTile + ly;
  const bool inside = px < W && py < H;
  const uint2 rg = srange[t];
  const int n = (int)(rg.y - rg.x);
  const int lane = threadIdx.x & 31;
  // this warp's pixel box (two tile rows): the render's bounding-box cull, then exact tests
  const float bx0 = (float)((t % TX) * kTile), bx1 = bx0 + (float)(kTile - 1);
  const float by0 = (float)((t / TX) * kTile + 2 * (threadIdx.x >> 5)), by1 = by0 + 1.f;
  bool cov = false;
  for (int c0 = 0; c0 < n; c0 += 256) {
    if (!__syncthreads_or(inside && !cov)) break;  // every pixel of the tile is decided
    const int cnt = min(256, n - c0);
    if ((int)threadIdx.x < cnt) {
      const uint32_t row = (uint32_t)(keys[rg.x + c0 + threadIdx.x] & 0xFFFFFFFFull);
      sa[threadIdx.x] = sub_rec[(size_t)4 * row];
      sb[threadIdx.x] = sub_rec[(size_t)4 * row + 1];
      se[threadIdx.x] = sub_rec[(size_t)4 * row + 2].w;
    }
    __syncthreads();
    bool wdone = __all_sync(0xffffffffu, !inside || cov);
    for (int g0 = 0; g0 < cnt && !wdone; g0 += 32) {
      // span masks (as the render's span walk): lane l computes instance g0 + l's superset mask of
      // the warp's 16 x 2 pixels, one transpose gives each pixel the instances that MAY cover it,
      // and the pixel runs the exact test only on those, until its first hit
      const int j = g0 + lane;
      uint32_t pm = 0u;
      if (j < cnt) {
        const float4 r0 = sa[j];
        const float2 ext = unpack_ext(se[j]);
        if ((r0.x + ext.x >= bx0) && (r0.x - ext.x <= bx1) && (r0.y + ext.y >= by0) && (r0.y - ext.y <= by1))
          pm = support_mask_16x2(r0, sb[j], bx0, by0);
      }
      uint32_t lm = warp_transpose32(pm, (uint32_t)lane);
      if (!inside || cov) lm = 0u;
      while (__any_sync(0xffffffffu, lm != 0u)) {
        if (lm) {
          const int idx = g0 + __ffs(lm) - 1;
          lm &= lm - 1u;
          PairEval e;
          if (eval_pair(sa[idx], sb[idx], (float)px, (float)py, e)) {
            cov = true;
            lm = 0u;
          }
        }
      }
      wdone = __all_sync(0xffffffffu, !inside || cov);
    }
    __syncthreads();
  }
  const bool act = inside && cov;
  // active bits: each half-warp is one 16-pixel tile row; its 16 bits go to 1 or 2 mask words
  const uint32_t bal = __ballot_sync(0xffffffffu, act);
  if ((lane & 15) == 0 && py < H) {
    const uint32_t m16 = (lane ? bal >> 16 : bal) & 0xFFFFu;
    const int x0 = px;  // lx == 0
    const int valid = min(16, W - x0);
    const uint32_t m = m16 & ((valid >= 16) ? 0xFFFFu : ((1u << valid) - 1u));
    if (m) {
      const uint32_t b = (uint32_t)py * (uint32_t)W + (uint32_t)x0;
      const uint32_t sh = b & 31u;
      atomicOr(&bits[b >> 5], m << sh);
      if (sh > 16u) atomicOr(&bits[(b >> 5) + 1], m >> (32u - sh));
    }
  }
  const int na = __syncthreads_count(act);
  const int ni = __syncthreads_count(inside);
  if (threadIdx.x == 0) {
    const bool k = 2 * na >= ni;  // P:497 / R15
    keep[t] = k ? 1 : 0;
    if (k) {
      list[atomicAdd(&counts[0], 1u)] = (uint32_t)t;
      atomicAdd(&counts[1], (uint32_t)na);
    }
    if (na) atomicAdd(&counts[2], (uint32_t)na);
  }
}

cudaError_t launch_tile_coverage(const uint2* srange, const unsigned long long* keys, const float4* sub_rec,
                                 const rtgs_camera& cam, const rtgs_render_out& out, cudaStream_t s) {
  const CamK k = make_cam(cam);
  k_tile_coverage<<<k.TX * k.TY, 256, 0, s>>>(srange, keys, sub_rec, k.W, k.H, k.TX, out.active_bits, out.tile_keep,
                                              out.tile_list, out.counts);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// A3/A4 forward
// ------------------------------------------------------------------------------------------------
// Span-mask path (round 2).  Per 8x4 warp block the dense path evaluated every surviving (record, block)
// pair on all 32 lanes although ~5 lanes blend (sub-pixel splats): 45 instructions x 32 lanes per
// survivor.  Instead, per batch of bbox survivors (rounds of up to 64; the steps below for one word):
//   1. lane l takes survivor l and computes the exact 32-bit pixel mask of its support over the block
//      (support_mask: per pixel row, the x interval where p2 >= max(p2_min, log2(1/255) - log2 alpha),
//      a quadratic in dx, enlarged by a safety margin so it is a SUPERSET of the pixels that pass
//      eval_pair: a pixel outside it cannot pass, a pixel inside is still decided by eval_pair);
//   2. one 32x32 bit transpose (5 shuffles) turns "survivor l covers pixels" into "pixel p is covered
//      by survivors" (bit l, in depth order);
//   3. each lane walks ITS OWN set bits front to back (divergent loop: the warp iterates the maximum
//      per-lane count, not the survivor count), with the unchanged eval_pair / blend arithmetic, so
//      every decision and every value are bitwise those of the dense path (RTGS_RENDER_DENSE checks).

// (warp_transpose32 and support_mask: tilepipe.cuh, shared with the backward)

// SPAN: the span-mask consumer (default); false = the dense consumer (RTGS_RENDER_DENSE, verification)
#ifdef RTGS_RENDER_STATS
// experiment builds only (scripts/build_variant.py -DRTGS_RENDER_STATS): work counters of the span walk
// [0] warp-batches, [1] survivors, [2] rounds, [3] trips, [4] lane-pairs walked (has), [5] blends,
// [6] records seen, [7] rounds' survivor slots used (sum of min(64, nq - q))
__device__ unsigned long long g_rstats[8];
#define RSTAT(i, v) do { if (lane == 0) atomicAdd(&g_rstats[i], (unsigned long long)(v)); } while (0)  // v: no warp ops
#else
#define RSTAT(i, v) do { } while (0)
#endif
#ifndef RTGS_SPAN_MINB
#define RTGS_SPAN_MINB 5
#endif
// the MASKED render's ring and residency (half-tile CTAs: 4 consumer warps): 3 x 128 records and 6
// CTAs / SM (swept against 3 x 256 unbounded: first iteration equal, window iteration -3 %)
#ifndef RTGS_MASKED_BATCH
#define RTGS_MASKED_BATCH 128
#endif
#ifndef RTGS_MASKED_MINB
#define RTGS_MASKED_MINB 6
#endif
template <bool MASKED, bool COUNT, bool LAST = true, bool SPAN = true>
__global__ void __launch_bounds__(32 * ((MASKED ? kHalfWarps : kTileWarps) + 1),
                                  SPAN ? (MASKED ? RTGS_MASKED_MINB : RTGS_SPAN_MINB) : 1) k_render_fwd(const FwdArgs a) {
  constexpr int NW = MASKED ? kHalfWarps : kTileWarps;  // MASKED: one CTA per half of a kept tile
  constexpr int PS = kPipeStages, PB = MASKED ? RTGS_MASKED_BATCH : kPipeBatch;
  __shared__ PipeRingT<false, PS, PB> r;  // static: stage addresses fold into immediates
  __shared__ uint8_t survq[SPAN ? NW : 1][PB];  // per warp: the stage's bbox survivors, in order
  int tile, half = 0;
  if (MASKED) {
    if ((blockIdx.x >> 1) >= a.counts[0]) return;
    tile = (int)a.tile_list[blockIdx.x >> 1];
    half = blockIdx.x & 1;
  } else {
    tile = blockIdx.x;
  }
  pipe_init<NW>(r);
  __syncthreads();
  const uint2 rg = a.range[tile];
  const int start = (int)rg.x, end = (int)rg.y;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == NW) {  // producer warp (the span path also gets the per-record warp-box masks)
    const int txp = tile % a.cam.TX, typ = tile / a.cam.TX;
    pipe_produce<false, SPAN ? NW : 0, false, PS, PB>(r, a.rec, a.sub_rec, a.sorted_gid, start, end, [](int, int, uint32_t) {},
                                       NoFlush{}, (float)(txp * kTile), (float)(typ * kTile + half * (NW / 2) * 4));
    return;
  }
  const int tx = tile % a.cam.TX, ty = tile / a.cam.TX;
  const int wx0 = tx * kTile + (w & 1) * 8, wy0 = ty * kTile + (half * (NW / 2) + (w >> 1)) * 4;
  const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
  const bool inside = px < a.cam.W && py < a.cam.H;
  const uint32_t lin = (uint32_t)py * (uint32_t)a.cam.W + (uint32_t)px;
  bool want = inside;
  if (MASKED && inside) want = (a.active[lin >> 5] >> (lin & 31u)) & 1u;
  bool done = !want;
  const float fpx = (float)px, fpy = (float)py;
  const float bx0 = (float)wx0, bx1 = (float)(wx0 + 7), by0 = (float)wy0, by1 = (float)(wy0 + 3);
  const int n = end - start;
  const int nb = n > 0 ? (n + PB - 1) / PB : 0;

  const uint32_t rec0 = pin(smem_u32(&r.rec[0][0][0]));
  float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f;
  // sorted-list position of the depth hit (the entry is fetched after the loop); positions grow along
  // the walk, so "the first hit" is the minimum over hits (kNoHit: none)
  constexpr uint32_t kNoHit = 0xFFFFFFFFu;
  uint32_t hitpos = kNoHit;
  uint32_t last = (uint32_t)start;
  uint32_t nblend = 0;  // blended (pixel, Gaussian) pairs of this lane (-> counts[3])
  bool wdone = __all_sync(0xffffffffu, done);
  if (wdone && lane == 0) atomicSub(&r.alive, 1);
  if constexpr (SPAN) {
    const uint32_t q0 = pin(smem_u32(&survq[w][0]));
    for (int b = 0; b < nb; ++b) {
      const int st = b % PS;
      mbar_wait_sleep(&r.full[st], (uint32_t)(b / PS) & 1u);
      if (!wdone) {
        const uint32_t srec = rec0 + (uint32_t)(st * sizeof(r.rec[0]));  // shared address of this stage
        const uint32_t pbase = (uint32_t)(start + b * PB + 1);
        const int cnt = min(PB, n - b * PB);
        // 1. bbox survivors of the stage, in list order
        int nq = 0;
        const uint32_t sbox = pin(smem_u32(&r.boxmask[st][0]));
        for (int g0 = 0; g0 < cnt; g0 += 32) {
          const int j = g0 + lane;
          const bool ov = j < cnt && ((lds8(sbox + (uint32_t)j) >> w) & 1u);  // the producer's box test
          const uint32_t bal = __ballot_sync(0xffffffffu, ov);
          if (ov) sts8(q0 + (uint32_t)(nq + __popc(bal & ((1u << lane) - 1u))), (uint32_t)j);
          nq += __popc(bal);
        }
        __syncwarp();
        RSTAT(0, 1);
        RSTAT(1, nq);
        RSTAT(6, cnt);
        // 2. rounds of <= 64 survivors: support masks, two transposes, per-lane walk of the own bits.
        //    Lane l computes the masks of survivors q + 31 - l and q + 63 - l, so after the transposes
        //    survivor q + j sits at bit 31 - j of word 0 (q + 32 + j: of word 1): list order is
        //    leading-zero order, and the next survivor of a lane is one FLO away (no bit reverse).
        for (int q = 0; q < nq; q += 64) {
          uint32_t pm0 = 0u, pm1 = 0u;
          if (q + 31 - lane < nq) {
            const uint32_t ra = srec + 48u * lds8(q0 + (uint32_t)(q + 31 - lane));
            pm0 = support_mask(lds128(ra), lds128(ra + 16u), bx0, by0);
          }
          if (q + 63 - lane < nq) {
            const uint32_t ra = srec + 48u * lds8(q0 + (uint32_t)(q + 63 - lane));
            pm1 = support_mask(lds128(ra), lds128(ra + 16u), bx0, by0);
          }
          uint32_t lm0 = warp_transpose32(pm0, (uint32_t)lane);
          uint32_t lm1 = q + 32 < nq ? warp_transpose32(pm1, (uint32_t)lane) : 0u;  // (nq warp-uniform)
          if (done) lm0 = lm1 = 0u;
          // warp-uniform trip count (the largest per-lane bit count): the body is predicated, not
          // a divergent branch, so no reconvergence bookkeeping per iteration.  A lane that terminates
          // keeps stepping through its bits with every blend predicated off (done).
          const int trips = __reduce_max_sync(0xffffffffu, (uint32_t)(__popc(lm0) + __popc(lm1)));
#ifdef RTGS_RENDER_STATS
          RSTAT(2, 1);
          RSTAT(3, trips);
          RSTAT(7, min(64, nq - q));
          const uint32_t npairs = __reduce_add_sync(0xffffffffu, (uint32_t)(__popc(lm0) + __popc(lm1)));
          RSTAT(4, npairs);
          uint32_t nbl = 0;
#endif
          const uint32_t qa0 = q0 + (uint32_t)q + 31u, qa1 = qa0 + 32u;  // survivor at bit b: qa - b
          for (int it = 0; it < trips; ++it) {
            const bool w0 = lm0 != 0u || lm1 == 0u;  // (no bits left: word 0)
            const uint32_t cur = w0 ? lm0 : lm1;
            const bool has = cur != 0u;
            // b = the highest set bit (0xFFFFFFFF without bits: (b & 31) = 31 reads survivor q, a valid
            // record -- a stale slot may hold NaN colour -- and the pair is discarded)
            uint32_t b, top;
            asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(cur));
            asm("shl.b32 %0, %1, %2;" : "=r"(top) : "r"(1u), "r"(b));  // 0 for b = 0xFFFFFFFF (clamped)
            const uint32_t nxt = cur & ~top;
            lm0 = w0 ? nxt : lm0;
            lm1 = w0 ? lm1 : nxt;
            const uint32_t idx = lds8((w0 ? qa0 : qa1) - (b & 31u));
            const uint32_t ra = srec + 48u * idx;
            const float4 r0 = lds128(ra), r1 = lds128(ra + 16u), r2 = lds128(ra + 32u);
            PairEval e;
            bool ok = eval_pair(r0, r1, fpx, fpy, e) && has && !done;
            const uint32_t pos = pbase - 1u + idx;  // sorted-list position of the pair
            // R9: the first f > e^-0.5, tested before termination
            hitpos = min(hitpos, (ok && e.f > kDeltaAlpha) ? pos : kNoHit);
            const float test = __fmul_rn(T, __fsub_rn(1.f, e.f));
            const bool term = ok && (test < kTMin);
            done = done || term;
            ok = ok && !term;
            const float wgt = ok ? __fmul_rn(e.f, T) : 0.f;
            cr = __fmaf_rn(r2.x, wgt, cr);
            cg = __fmaf_rn(r2.y, wgt, cg);
            cb = __fmaf_rn(r2.z, wgt, cb);
            T = ok ? test : T;
            if (LAST) last = ok ? pos + 1u : last;
            if (COUNT) nblend += ok ? 1u : 0u;
#ifdef RTGS_RENDER_STATS
            nbl += ok ? 1u : 0u;
#endif
          }
#ifdef RTGS_RENDER_STATS
          const uint32_t nbw = __reduce_add_sync(0xffffffffu, nbl);
          RSTAT(5, nbw);
#endif
          if (__all_sync(0xffffffffu, done)) {
            wdone = true;
            if (lane == 0) atomicSub(&r.alive, 1);
            break;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[st]);
    }
  } else {
    for (int b = 0; b < nb; ++b) {
      const int st = b % PS;
      mbar_wait(&r.full[st], (uint32_t)(b / PS) & 1u);
      if (!wdone) {
        const uint32_t srec = rec0 + (uint32_t)(st * sizeof(r.rec[0]));  // shared address of this stage
        const uint32_t pbase = (uint32_t)(start + b * PB + 1);
        const int cnt = min(PB, n - b * PB);
        for (int g0 = 0; g0 < cnt; g0 += 32) {
          const int j = g0 + lane;
          bool ov = false;
          if (j < cnt) {
            const float4 r0 = lds128(srec + 48u * j);
            const float2 ext = unpack_ext(__uint_as_float(lds32(srec + 48u * j + 44u)));
            ov = (r0.x + ext.x >= bx0) && (r0.x - ext.x <= bx1) && (r0.y + ext.y >= by0) && (r0.y - ext.y <= by1);
          }
          uint32_t m = __ballot_sync(0xffffffffu, ov);
          while (m) {
            const int idx = g0 + __ffs(m) - 1;
            m &= m - 1;
            // branch-free body: every lane evaluates, the blend is predicated
            const uint32_t ra = srec + 48u * idx;
            const float4 r0 = lds128(ra), r1 = lds128(ra + 16u), r2 = lds128(ra + 32u);
            PairEval e;
            bool ok = eval_pair(r0, r1, fpx, fpy, e) && !done;
            // R9: the first f > e^-0.5, tested before termination (position only: no load in the loop)
            hitpos = min(hitpos, (ok && e.f > kDeltaAlpha) ? pbase - 1u + (uint32_t)idx : kNoHit);
            const float test = __fmul_rn(T, __fsub_rn(1.f, e.f));
            const bool term = ok && (test < kTMin);
            done = done || term;
            ok = ok && !term;
            const float wgt = ok ? __fmul_rn(e.f, T) : 0.f;
            cr = __fmaf_rn(r2.x, wgt, cr);
            cg = __fmaf_rn(r2.y, wgt, cg);
            cb = __fmaf_rn(r2.z, wgt, cb);
            T = ok ? test : T;
            if (LAST) last = ok ? pbase + (uint32_t)idx : last;
            if (COUNT) nblend += ok ? 1u : 0u;
          }
          if (__all_sync(0xffffffffu, done)) {
            wdone = true;
            if (lane == 0) atomicSub(&r.alive, 1);
            break;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[st]);
    }
  }
  if (COUNT) {
    const uint32_t wsum = __reduce_add_sync(0xffffffffu, nblend);
    if (lane == 0 && wsum) atomicAdd(const_cast<uint32_t*>(a.counts) + 3, wsum);
  }

  if (!want) return;
  const size_t HW = (size_t)a.cam.W * a.cam.H;
  a.color[lin] = cr;
  a.color[HW + lin] = cg;
  a.color[2 * HW + lin] = cb;
  a.trans[lin] = T;
  if (LAST) a.n_contrib[lin] = last;
  float D = -1.f, N0 = 0.f, N1 = 0.f, N2 = 0.f;
  int32_t gid = -1;
  const uint32_t hit = hitpos != kNoHit ? a.sorted_gid[hitpos] : 0xFFFFFFFFu;  // list entry of the hit
  if (hit != 0xFFFFFFFFu) {
    const bool sub = hit & kSubBit;
    const uint32_t row = hit & ~kSubBit;
    gid = sub ? a.sub_gid[row] : (int32_t)hit;
    const float4 pl = sub ? a.sub_rec[(size_t)4 * row + 3] : a.rec[(size_t)4 * hit + 3];  // n_c, n_c . p_c
    const float zc = __uint_as_float(sub ? a.sub_zkey[row] : a.zkey[hit]);
    const float rx = (fpx - a.cam.cx) / a.cam.fx, ry = (fpy - a.cam.cy) / a.cam.fy;
    const float ndr = pl.x * rx + pl.y * ry + pl.z;
    const float nn = sqrtf(pl.x * pl.x + pl.y * pl.y + pl.z * pl.z);
    const float cosang = fabsf(ndr) / (sqrtf(rx * rx + ry * ry + 1.f) * nn);
    D = (cosang > kCos60) ? pl.w / ndr : zc;  // Eq.5 (R10, R11)
    const float sg = ndr > 0.f ? -1.f : 1.f;                             // face the viewer (R12)
    const float nx = sg * pl.x, ny = sg * pl.y, nz = sg * pl.z;
    N0 = a.R[0] * nx + a.R[1] * ny + a.R[2] * nz;
    N1 = a.R[3] * nx + a.R[4] * ny + a.R[5] * nz;
    N2 = a.R[6] * nx + a.R[7] * ny + a.R[8] * nz;
  }
  a.index[lin] = gid;
  a.depth[lin] = D;
  if (a.normal) {
    a.normal[lin] = N0;
    a.normal[HW + lin] = N1;
    a.normal[2 * HW + lin] = N2;
  }
}

cudaError_t launch_coverage(const rtgs_gaussians& g, const rtgs_projected& proj, const rtgs_camera& cam,
                            const rtgs_render_out& out, cudaStream_t s) {
  const CamK k = make_cam(cam);
  const size_t words = ((size_t)k.W * k.H + 31) / 32;
  cudaMemsetAsync(out.active_bits, 0, words * 4, s);
  cudaMemsetAsync(out.counts, 0, 16, s);
  if (g.n > 0) {
    k_coverage<<<(g.n + 255) / 256, 256, 0, s>>>(reinterpret_cast<const float4*>(proj.rec),
                                                 reinterpret_cast<const uint2*>(proj.rect), proj.zkey, g.flags, g.n,
                                                 k.W, out.active_bits);
    note_launch();
  }
  k_tile_keep<false><<<k.TX * k.TY, 256, 0, s>>>(out.active_bits, k.W, k.H, k.TX, out.tile_keep, out.tile_list,
                                                 out.counts);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_tile_any(const rtgs_camera& cam, const rtgs_render_out& out, cudaStream_t s) {
  const CamK k = make_cam(cam);
  k_tile_keep<true><<<k.TX * k.TY, 256, 0, s>>>(out.active_bits, k.W, k.H, k.TX, out.tile_keep, out.tile_list,
                                                out.counts);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_render(const rtgs_projected& proj, const rtgs_bins& bins, const PoseF& pose,
                          const rtgs_camera& cam, int masked, bool count, const rtgs_render_out& out, cudaStream_t s,
                          bool dense) {
  FwdArgs a;
  a.rec = reinterpret_cast<const float4*>(proj.rec);
  a.zkey = proj.zkey;
  a.sub_rec = reinterpret_cast<const float4*>(bins.sub_rec);
  a.sub_zkey = bins.sub_zkey;
  a.sub_gid = bins.sub_gid;
  a.sorted_gid = bins.sorted_gid;
  a.range = reinterpret_cast<const uint2*>(bins.tile_range);
  a.tile_list = out.tile_list;
  a.counts = out.counts;
  a.active = out.active_bits;
  a.cam = make_cam(cam);
  for (int i = 0; i < 9; ++i) a.R[i] = pose.Rf[i];
  a.color = out.color; a.trans = out.trans; a.depth = out.depth; a.normal = out.normal;
  a.index = out.index; a.n_contrib = out.n_contrib;
  const int T = a.cam.TX * a.cam.TY;
  if (count) cudaMemsetAsync(out.counts + 3, 0, 4, s);  // blend counter of this render
  const dim3 gm(2 * T), bm(32 * (kHalfWarps + 1)), gf(T), bf(32 * (kTileWarps + 1));
  if (dense) {  // verification: the dense consumer (RTGS_RENDER_DENSE)
    if (masked) k_render_fwd<true, true, true, false><<<gm, bm, 0, s>>>(a);
    else if (count || out.n_contrib) k_render_fwd<false, true, true, false><<<gf, bf, 0, s>>>(a);
    else k_render_fwd<false, true, false, false><<<gf, bf, 0, s>>>(a);
  } else if (masked && count) k_render_fwd<true, true><<<gm, bm, 0, s>>>(a);
  else if (masked) k_render_fwd<true, false><<<gm, bm, 0, s>>>(a);
  else if (count) k_render_fwd<false, true><<<gf, bf, 0, s>>>(a);
  else if (out.n_contrib) k_render_fwd<false, false><<<gf, bf, 0, s>>>(a);
  else k_render_fwd<false, false, false><<<gf, bf, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtgs

#ifdef RTGS_RENDER_STATS
extern "C" int rtgs_debug_render_stats(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, rtgs::g_rstats, sizeof(rtgs::g_rstats));
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(rtgs::g_rstats, z, sizeof(z));
  }
  return (int)cudaGetLastError();
}
#endif
