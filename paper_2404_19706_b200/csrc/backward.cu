// backward.cu — A5: masked L1 loss and its gradient for the unstable Gaussians
// (O5; Eq.7-8, readings R13, R14, R17).
//
// K5 k_render_bwd: one CTA per half of a kept tile (4 consumer warps + 1 producer; same geometry and
//   batching as the MASKED forward).  Each active
//   pixel walks its blended entries BACK TO FRONT with the forward's arithmetic (eval_pair), so every
//   decision is the forward's; T_i is recovered from the stored T^ by division and the colour suffix
//   S_i is summed from the back (no C^ - prefix cancellation).  For every UNSTABLE record a warp touches, the 8 screen-space gradients
//   (mu 2, conic 3, rgb 3) are reduced over the warp with shuffles and added with one red.global
//   per value.  Depth gradients go to the single hit Gaussian of each pixel (Eq.4-5).
// K5b k_project_bwd: one thread per slot: chain rule from the screen-space gradients through
//   EWA / SH / disc plane to (pos, log_scale, rot, sh) (hand-derived; checked against the
//   oracle's autograd in tests/test_gpu_backward.py).
#include "common.cuh"
#include "adam.cuh"
#include "internal.h"
#include "tilepipe.cuh"

// RTGS_BWD_DENSE=1 builds the dense walk of K5 (every lane evaluates every bbox survivor) for
// comparison with the default span-mask walk
#ifndef RTGS_BWD_DENSE
#define RTGS_BWD_DENSE 0
#endif

namespace rtgs {

constexpr int kSG = 16;  // screen-space gradient floats per slot
[[maybe_unused]] constexpr int kDirectLanes = 4;  // (dense walk) <= this many contributing lanes: per-lane vector atomics

// Transpose-reduce of 8 values over a warp in 9 shuffles (instead of 8 x 5): after the call, lane l
// holds the warp sum of value j = 4*bit4(l) + 2*bit3(l) + bit2(l), identical on the 4 lanes l^{0..3}.
__device__ __forceinline__ float warp_reduce8(const float v[8], int lane, int& j) {
  const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
  float u[4], w2[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = b16 ? v[i] : v[i + 4];
    const float keep = b16 ? v[i + 4] : v[i];
    u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b8 ? u[i] : u[i + 2];
    const float keep = b8 ? u[i + 2] : u[i];
    w2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const float send = b4 ? w2[0] : w2[1];
  float x = (b4 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
  x += __shfl_xor_sync(0xffffffffu, x, 2);
  x += __shfl_xor_sync(0xffffffffu, x, 1);
  j = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
  return x;
}

// workspace: sgrad [n_slots][16] | acc [4] floats: sum|dC|, sum|dD| over P_d, |P_d|, spare
size_t backward_workspace_size(int n_slots) { return ((size_t)n_slots * kSG + 8) * sizeof(float) + 256; }

struct BwdArgs {
  const float4* rec;
  const float4* sub_rec;  // NEXT f3: subset rows = slots (entries with kSubBit), else NULL
  const uint32_t* zkey;
  const uint32_t* sorted_gid;
  const uint2* range;
  const uint32_t* tile_list;
  const uint32_t* counts;
  const uint32_t* active;
  const float* color;
  const float* trans;
  const float* depth;
  const int32_t* index;
  const uint32_t* n_contrib;
  const float* tcolor;
  const float* tdepth;
  const int32_t* slot_of_gid;
  CamK cam;
  float w_c;
  float* sgrad;
  float* acc;
};

constexpr int kBwdWarps = kHalfWarps;  // one CTA per half of a kept tile
constexpr int kBwdParts = kTile / (2 * kBwdWarps);  // CTAs per kept tile (each 16 x 2*kBwdWarps px)
static_assert(kBwdParts == 2 || kBwdParts == 4, "the backward splits a tile in 2 or 4 row bands");

#ifndef RTGS_BWD_BATCH
#define RTGS_BWD_BATCH 128
#endif
// the backward's ring: 3 x 128 records, 6 CTAs / SM (swept against 3 x 256 unbounded: C3 step equal,
// window iteration -5 %)
constexpr int kBS = kPipeStages, kBB = RTGS_BWD_BATCH;
struct BwdSmem {
  PipeRingT<false, kBS, kBB> ring;  // (no list entries: the producer resolves each record's slot)
  int32_t slot[kBS][kBB];
  uint8_t survq[kBwdWarps][kBB];  // span path: the stage's bbox survivors, in list order
  float red[3][kBwdWarps];
  uint32_t last_max;
};

#ifndef RTGS_BWD_MINB
#define RTGS_BWD_MINB 6
#endif
__global__ void __launch_bounds__(32 * (kBwdWarps + 1), RTGS_BWD_MINB) k_render_bwd(const BwdArgs a) {
  __shared__ BwdSmem sm;  // static: stage addresses fold into immediates
  PipeRingT<false, kBS, kBB>& r = sm.ring;
  if ((int)(blockIdx.x / kBwdParts) >= (int)a.counts[0]) return;
  const int tile = (int)a.tile_list[blockIdx.x / kBwdParts];
  const int half = blockIdx.x % kBwdParts;  // row band of the tile
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  pipe_init<kBwdWarps>(r);
  if (tid == 0) sm.last_max = 0;
  const bool consumer = w < kBwdWarps;
  const int tx = tile % a.cam.TX, ty = tile / a.cam.TX;
  const int wx0 = tx * kTile + (w & 1) * 8, wy0 = ty * kTile + (half * (kBwdWarps / 2) + (w >> 1)) * 4;
  const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
  const bool inside = consumer && px < a.cam.W && py < a.cam.H;
  const uint32_t lin = (uint32_t)py * (uint32_t)a.cam.W + (uint32_t)px;
  const bool want = inside && ((a.active[lin >> 5] >> (lin & 31u)) & 1u);
  const size_t HW = (size_t)a.cam.W * a.cam.H;
  const float fpx = (float)px, fpy = (float)py;
  __syncthreads();

  // per-pixel loss terms (R13, R14, R24) and the depth gradient of the pixel's hit (Eq.4-5)
  float gCr = 0.f, gCg = 0.f, gCb = 0.f, Cr = 0.f, Cg = 0.f, Cb = 0.f;
  uint32_t last = 0;
  float l1c = 0.f, l1d = 0.f, nd = 0.f;
  const float invP = a.w_c / (3.f * (float)max(1u, a.counts[1]));
  if (want) {
    Cr = a.color[lin]; Cg = a.color[HW + lin]; Cb = a.color[2 * HW + lin];
    const float dr = Cr - a.tcolor[lin], dg = Cg - a.tcolor[HW + lin], db = Cb - a.tcolor[2 * HW + lin];
    l1c = fabsf(dr) + fabsf(dg) + fabsf(db);
    gCr = dr > 0.f ? invP : (dr < 0.f ? -invP : 0.f);
    gCg = dg > 0.f ? invP : (dg < 0.f ? -invP : 0.f);
    gCb = db > 0.f ? invP : (db < 0.f ? -invP : 0.f);
    last = a.n_contrib[lin];
    atomicMax(&sm.last_max, last);
    const int hit = a.index[lin];
    const float Dt = a.tdepth[lin];
    if (hit >= 0 && isfinite(Dt) && Dt > 0.f) {
      const float Dh = a.depth[lin];
      const float dd = Dh - Dt;
      l1d = fabsf(dd);
      nd = 1.f;
      const float gD = dd > 0.f ? 1.f : (dd < 0.f ? -1.f : 0.f);  // scaled by w_d / |P_d| in K5b
      const int slot = a.slot_of_gid[hit];
      if (slot >= 0 && gD != 0.f) {
        const float4* hr = a.sub_rec ? a.sub_rec + (size_t)4 * slot : a.rec + (size_t)4 * hit;
        const float4 pl = hr[3];  // n_c, n_c . p_c
        const float rx = (fpx - a.cam.cx) / a.cam.fx, ry = (fpy - a.cam.cy) / a.cam.fy;
        const float ndr = pl.x * rx + pl.y * ry + pl.z;
        const float nn = sqrtf(pl.x * pl.x + pl.y * pl.y + pl.z * pl.z);
        const float cosang = fabsf(ndr) / (sqrtf(rx * rx + ry * ry + 1.f) * nn);
        float* sg = a.sgrad + (size_t)slot * kSG;
        if (cosang > kCos60) {
          // D = (n.p)/(n.r): dD/dp_c = n/(n.r), dD/dn_c = (p_c - D r)/(n.r).  p_c - D r is the
          // in-plane offset from the ray's hit to the disc centre (mm) between two ~metre vectors:
          // formed from the small pixel offset delta = ((mu_x - u_x)/f_x, (mu_y - u_y)/f_y, 0)
          // (p_c = z_c (r + delta)):  p_c - D r = z_c (delta - (n.delta / n.r) r),
          // z_c = D (n.r) / (n.r + n.delta), so no metre-sized terms cancel in the sums.
          const float q = gD / ndr;
          const float4 m = hr[0];  // mu hi, lo
          const float ddx = __fadd_rn(__fsub_rn(m.x, fpx), m.z) / a.cam.fx;
          const float ddy = __fadd_rn(__fsub_rn(m.y, fpy), m.w) / a.cam.fy;
          const float ndd = pl.x * ddx + pl.y * ddy;
          const float kk = ndd / ndr;
          const float qz = q * (Dh * ndr / (ndr + ndd));  // q z_c
          atomicAdd(sg + 8, q);
          atomicAdd(sg + 9, qz * (ddx - kk * rx));
          atomicAdd(sg + 10, qz * (ddy - kk * ry));
          atomicAdd(sg + 11, -qz * kk);
        } else {
          atomicAdd(sg + 12, gD);  // D = z: dD/dp_c = e_z
        }
      }
    }
  }
  if (consumer) {  // loss sums: warp reduce, one atomic per value per CTA
    const float s0 = warp_sum(l1c), s1 = warp_sum(l1d), s2 = warp_sum(nd);
    if (lane == 0) { sm.red[0][w] = s0; sm.red[1][w] = s1; sm.red[2][w] = s2; }
  }
  __syncthreads();
  if (tid < 3) {
    float t = 0.f;
    for (int k = 0; k < kBwdWarps; ++k) t += sm.red[tid][k];
    atomicAdd(a.acc + tid, t);
  }
  const uint2 rg = a.range[tile];
  const int start = (int)rg.x;
  const int end = min((int)rg.y, (int)sm.last_max);  // nothing past the last blended entry contributes
  const int n = end - start;

  if (!consumer) {
    const int32_t* slot_of_gid = a.slot_of_gid;
    // slot of a gid entry via slot_of_gid; a subset entry (f3) carries its slot in the entry itself
    // (a subset entry's slot is the entry itself: stored here, so the consumers read one slot per record)
    auto extra = [&](int st, int j, uint32_t g) {
      if (!(g & kSubBit)) cp_async4(&sm.slot[st][j], slot_of_gid + g);
      else sm.slot[st][j] = (int32_t)(g & ~kSubBit);
    };
    auto flush = [](int, int) {};
#if !RTGS_BWD_DENSE
    pipe_produce<true, kBwdWarps, false, kBS, kBB>(r, a.rec, a.sub_rec, a.sorted_gid, start, end, extra, flush, (float)(tx * kTile),
                                  (float)(ty * kTile + half * (kBwdWarps / 2) * 4));
#else
    pipe_produce<true, 0, false, kBS, kBB>(r, a.rec, a.sub_rec, a.sorted_gid, start, end, extra, flush);
#endif
    return;
  }

  // BACK-TO-FRONT pass over the pixel's blended entries (positions < last, the forward's n_contrib):
  // the decisions are the forward's (eval_pair is the same arithmetic; termination is encoded in
  // `last`), and T_i is recovered from the stored final T^ as T_i = T_{i+1} / (1 - f_i).  With
  // G_i = sum_c gC_c c_i,c the colour cotangent of entry i, the colour seen BEHIND entry i is
  //   B_i = sum_{j>i} G_j f_j prod_{i<k<j} (1 - f_k),   B_{i-1} = f_i G_i + (1 - f_i) B_i,  B_last = 0
  // (black background, R23) -- a convex-combination recursion from the back, no division by T -- and
  //   dL/df_i = sum_c gC_c (c_i,c T_i - S_i,c / (1 - f_i)) = T_i (G_i - B_i)      (Eq.1, Eq.3)
  // since S_i = T_{i+1} B_i.  The difference G_i - B_i is the pixel's own cancellation (a Gaussian in
  // front of a similar colour); forming it between two O(1) values keeps its error at float32
  // rounding of G, not of the T-scaled partial sums (no C^ - prefix, no S / (1 - f) amplification).
  const float bx0 = (float)wx0, by0 = (float)wy0;
  [[maybe_unused]] const float bx1 = (float)(wx0 + 7), by1 = (float)(wy0 + 3);  // (dense walk's box test)
  const int nb = n > 0 ? (n + kBB - 1) / kBB : 0;
  const uint32_t rec0 = pin(smem_u32(&r.rec[0][0][0])), slot0 = pin(smem_u32(&sm.slot[0][0]));
  const int plane = (int)pin((uint32_t)lane);
  float T = want ? a.trans[lin] : 1.f;  // T after the last blended entry = the forward's T^
  float B = 0.f;                         // colour cotangent behind the current entry
  const uint32_t mylast = want ? last : 0u;
  const uint32_t wlast = __reduce_max_sync(0xffffffffu, mylast);  // this warp's entries: [start, wlast)
#if !RTGS_BWD_DENSE
  // Span path (as the forward's): per stage the warp's bbox survivors are queued; rounds of <= 32
  // survivors, BACK TO FRONT, get exact support span masks (a superset of the pairs that pass
  // eval_pair), one transpose, and each lane walks its own pixel's bits from the highest (the
  // nearest-to-the-back entry first).  Lanes hold different entries at a time, so each contributing
  // lane adds its 8 screen-space values with two vector reductions (no warp reduce).
  const uint32_t q0 = pin(smem_u32(&sm.survq[w][0]));
  (void)plane;
#ifdef RTGS_BWD_NOATOM
  float sink = 0.f;
#endif
  for (int b = 0; b < nb; ++b) {
    const int st = b % kBS;
    mbar_wait_sleep(&r.full[st], (uint32_t)(b / kBS) & 1u);
    const int lo = pipe_batch_lo<kBB>(true, start, end, b);
    if ((uint32_t)lo < wlast) {  // warp-uniform: the batch holds entries of this warp's pixels
      const uint32_t srec = rec0 + (uint32_t)(st * sizeof(r.rec[0]));  // shared addresses of this stage
      const uint32_t sslot = slot0 + (uint32_t)(st * sizeof(sm.slot[0]));
      const int cnt = pipe_batch_cnt<kBB>(true, start, end, b);
      int nq = 0;
      const uint32_t sbox = pin(smem_u32(&r.boxmask[st][0]));
      for (int g0 = 0; g0 < cnt; g0 += 32) {
        const int j = g0 + lane;
        // the producer's box test (boxmask) and this warp's stop
        const bool ov = j < cnt && (uint32_t)(lo + j) < wlast && ((lds8(sbox + (uint32_t)j) >> w) & 1u);
        const uint32_t bal = __ballot_sync(0xffffffffu, ov);
        if (ov) sts8(q0 + (uint32_t)(nq + __popc(bal & ((1u << lane) - 1u))), (uint32_t)j);
        nq += __popc(bal);
      }
      __syncwarp();
      for (int q = ((nq - 1) / 32) * 32; q >= 0 && nq > 0; q -= 32) {
        uint32_t pm = 0u;
        if (q + lane < nq) {
          const uint32_t ra = srec + 48u * lds8(q0 + (uint32_t)(q + lane));
          pm = support_mask(lds128(ra), lds128(ra + 16u), bx0, by0);
        }
        uint32_t lm = warp_transpose32(pm, (uint32_t)lane);
        if (!want) lm = 0u;
        const int trips = __reduce_max_sync(0xffffffffu, (uint32_t)__popc(lm));
        for (int it = 0; it < trips; ++it) {
          const bool has = lm != 0u;
          // back to front: the highest set bit (bfind; 0xFFFFFFFF without bits: such a lane reads
          // survivor q, a queued record of this stage, and the pair is discarded)
          uint32_t b, top;
          asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(lm));
          asm("shl.b32 %0, %1, %2;" : "=r"(top) : "r"(1u), "r"(b));  // 0 for b = 0xFFFFFFFF (clamped)
          lm &= ~top;
          const uint32_t idx = lds8(q0 + (uint32_t)q + (has ? b : 0u));
          const uint32_t ra = srec + 48u * idx;
          const float4 r0 = lds128(ra), r1 = lds128(ra + 16u), r2 = lds128(ra + 32u);
          PairEval e;
          // blended in the forward <=> passes the support test and lies before the pixel's `last`
          const bool ok = eval_pair(r0, r1, fpx, fpy, e) && has && ((uint32_t)lo + idx < mylast);
          // T before entry i: 1 - f >= 0.01, and the ~1 ulp reciprocal only scales T (no decision
          // of the walk reads T: `ok` is the forward's support test and position)
          float inv1mf;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv1mf) : "f"(__fsub_rn(1.f, e.f)));
          const float Ti = ok ? __fmul_rn(T, inv1mf) : T;
          const float wgt = ok ? __fmul_rn(e.f, Ti) : 0.f;
          const float G = __fmaf_rn(gCb, r2.z, __fmaf_rn(gCg, r2.y, gCr * r2.x));
          const int slot = (int)lds32(sslot + 4u * idx);  // < 0: a stable Gaussian (no gradient)
          {
            {
              const float dLdf = __fmul_rn(Ti, __fsub_rn(G, B));
              // f = alpha e^power; the 0.99 cap passes no gradient when active (R17)
              const float dLdp = (e.f < kFMax) ? dLdf * e.f : 0.f;
              // power = p2 / log2(e): d power / d dx = (2 A' dx + B' dy) / log2(e) = -(A dx + B dy)
              const float sc = dLdp * (1.f / kLog2e);
              float* sg = a.sgrad + (size_t)max(slot, 0) * kSG;
#ifdef RTGS_BWD_NOATOM  // experiment builds only: the pair cost without its gradient reductions
              sink += sc * (2.f * r1.x * e.dx + r1.y * e.dy) + sc * (2.f * r1.z * e.dy + r1.y * e.dx) +
                      dLdp * e.dx * e.dy + gCr * wgt + gCg * wgt + gCb * wgt + (float)(size_t)sg;
#else
              const float4 v0 = make_float4(sc * (2.f * r1.x * e.dx + r1.y * e.dy),   // d/d mu_x
                                            sc * (2.f * r1.z * e.dy + r1.y * e.dx),   // d/d mu_y
                                            -0.5f * dLdp * e.dx * e.dx,               // d/d A
                                            -dLdp * e.dx * e.dy);                     // d/d B
              const float4 v1 = make_float4(-0.5f * dLdp * e.dy * e.dy,               // d/d C
                                            gCr * wgt, gCg * wgt, gCb * wgt);         // d/d rgb
              if (ok && slot >= 0) {  // (the values above are formed branch-free on every lane)
                atomicAdd(reinterpret_cast<float4*>(sg), v0);
                atomicAdd(reinterpret_cast<float4*>(sg + 4), v1);
              }
#endif
            }
          }
          B = ok ? __fmaf_rn(e.f, __fsub_rn(G, B), B) : B;  // f G + (1 - f) B
          T = Ti;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&r.empty[st]);
  }
#ifdef RTGS_BWD_NOATOM
  if (sink == 1234.5f) a.acc[3] = sink;
#endif
}

#else  // RTGS_BWD_DENSE: the dense walk (every lane evaluates every bbox survivor), for comparison
  for (int b = 0; b < nb; ++b) {
    const int st = b % kBS;
    mbar_wait(&r.full[st], (uint32_t)(b / kBS) & 1u);
    const int lo = pipe_batch_lo<kBB>(true, start, end, b);
    if ((uint32_t)lo < wlast) {  // warp-uniform: the batch holds entries of this warp's pixels
      const uint32_t srec = rec0 + (uint32_t)(st * sizeof(r.rec[0]));  // shared addresses of this stage
      const uint32_t sslot = slot0 + (uint32_t)(st * sizeof(sm.slot[0]));
      const int cnt = pipe_batch_cnt<kBB>(true, start, end, b);
      for (int g0 = (cnt - 1) & ~31; g0 >= 0; g0 -= 32) {
        const int j = g0 + lane;
        bool ov = false;
        if (j < cnt && (uint32_t)(lo + j) < wlast) {
          const float4 r0 = lds128(srec + 48u * j);
          const float2 ext = unpack_ext(__uint_as_float(lds32(srec + 48u * j + 44u)));
          ov = (r0.x + ext.x >= bx0) && (r0.x - ext.x <= bx1) && (r0.y + ext.y >= by0) && (r0.y - ext.y <= by1);
        }
        uint32_t m = __ballot_sync(0xffffffffu, ov);
        while (m) {
          const int bit = 31 - __clz(m);  // back to front
          m ^= 1u << bit;
          const int idx = g0 + bit;
          const int slot = (int)lds32(sslot + 4u * idx);  // warp-uniform
          const uint32_t ra = srec + 48u * idx;
          const float4 r0 = lds128(ra), r1 = lds128(ra + 16u), r2 = lds128(ra + 32u);
          PairEval e;
          // blended in the forward <=> passes the support test and lies before the pixel's `last`
          const bool ok = eval_pair(r0, r1, fpx, fpy, e) && ((uint32_t)(lo + idx) < mylast);
          const float inv1mf = __frcp_rn(__fsub_rn(1.f, e.f));  // IEEE reciprocal; 1 - f >= 0.01
          const float Ti = ok ? __fmul_rn(T, inv1mf) : T;        // T before entry i
          const float wgt = ok ? __fmul_rn(e.f, Ti) : 0.f;
          const float G = __fmaf_rn(gCb, r2.z, __fmaf_rn(gCg, r2.y, gCr * r2.x));
          const uint32_t okm = __ballot_sync(0xffffffffu, ok);
          if (slot >= 0 && okm) {
            float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (ok) {
              const float dLdf = __fmul_rn(Ti, __fsub_rn(G, B));
              // f = alpha e^power; the 0.99 cap passes no gradient when active (R17)
              const float dLdp = (e.f < kFMax) ? dLdf * e.f : 0.f;
              // power = p2 / log2(e): d power / d dx = (2 A' dx + B' dy) / log2(e) = -(A dx + B dy)
              const float sc = dLdp * (1.f / kLog2e);
              v[0] = sc * (2.f * r1.x * e.dx + r1.y * e.dy);  // d/d mu_x
              v[1] = sc * (2.f * r1.z * e.dy + r1.y * e.dx);  // d/d mu_y
              v[2] = -0.5f * dLdp * e.dx * e.dx;              // d/d A
              v[3] = -dLdp * e.dx * e.dy;                     // d/d B
              v[4] = -0.5f * dLdp * e.dy * e.dy;              // d/d C
              v[5] = gCr * wgt;                               // d/d rgb
              v[6] = gCg * wgt;
              v[7] = gCb * wgt;
            }
            float* sg = a.sgrad + (size_t)slot * kSG;
            if (__popc(okm) <= kDirectLanes) {
              // few contributing lanes (the common case for sub-pixel splats): each adds its own 8
              // values with two vector reductions instead of the 9-shuffle transpose-reduce
              if (ok) {
                atomicAdd(reinterpret_cast<float4*>(sg), make_float4(v[0], v[1], v[2], v[3]));
                atomicAdd(reinterpret_cast<float4*>(sg + 4), make_float4(v[4], v[5], v[6], v[7]));
              }
            } else {
              int vj;
              const float x = warp_reduce8(v, plane, vj);
              if ((plane & 3) == 0) atomicAdd(sg + vj, x);  // 8 lanes, 8 values
            }
          }
          B = ok ? __fmaf_rn(e.f, __fsub_rn(G, B), B) : B;  // f G + (1 - f) B
          T = Ti;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&r.empty[st]);
  }
}
#endif

// ------------------------------------------------------------------------------------------------
// K5b: chain rule through the projection (float32, recomputing the forward quantities)
// ------------------------------------------------------------------------------------------------
struct PBArgs {
  const float4* rec;
  const float* recf;      // the same records as floats
  const float* sub_recf;  // NEXT f3: the slots' own records (row = slot), else NULL
  const float* pos;
  const float* log_scale;
  const float* rot;
  const float* sh;
  int K, D;  // D = 10 + 3K
  const int32_t* gid_of_slot;
  int n_slots;
  const float* sgrad;
  const float* acc;  // acc[2] = |P_d|
  float w_d;
  double V[9], tp[3], campos[3];
  float Vf[9];
  CamK cam;
  float limx0, limx1, limy0, limy1;
  float* grad;
  float* loss_out;
  float w_c;
  const uint32_t* counts;
  // fused A6 (ADAM variant only): the update replaces the grad read-modify-write
  float* wpos;
  float* wlog_scale;
  float* wrot;
  float* wsh;
  const uint8_t* flags;
  float* m;
  float* v;
  const float* init_geom;
  uint32_t* eta;
  AdamHP h;
};

// Y_k(d) and its gradient for ONE coefficient k (a compile-time constant after unrolling): the 3DGS
// real basis (R2), constants restated from their closed forms.  Evaluated in double by the chain rule:
// the higher bands cancel (2z^2 - x^2 - y^2, x^2 - y^2, ...), and a float32 direction would carry
// that cancellation's relative error into the SH gradient Y_k * dL/drgb.
template <typename S>
__device__ __forceinline__ void sh_basis_one(int k, S x, S y, S z, S& Y, S& dx, S& dy, S& dz) {
  const S C0 = 0.28209479177387814, C1 = 0.4886025119029199;
  const S C20 = 1.0925484305920792, C21 = -1.0925484305920792, C22 = 0.31539156525252005,
          C23 = -1.0925484305920792, C24 = 0.5462742152960396;
  const S C30 = -0.5900435899266435, C31 = 2.890611442640554, C32 = -0.4570457994644658,
          C33 = 0.3731763325901154, C34 = -0.4570457994644658, C35 = 1.445305721320277,
          C36 = -0.5900435899266435;
  const S xx = x * x, yy = y * y, zz = z * z;
  dx = dy = dz = S(0);
  switch (k) {
    case 0: Y = C0; break;
    case 1: Y = -C1 * y; dy = -C1; break;
    case 2: Y = C1 * z; dz = C1; break;
    case 3: Y = -C1 * x; dx = -C1; break;
    case 4: Y = C20 * x * y; dx = C20 * y; dy = C20 * x; break;
    case 5: Y = C21 * y * z; dy = C21 * z; dz = C21 * y; break;
    case 6: Y = C22 * (2.0 * zz - xx - yy); dx = -2.0 * C22 * x; dy = -2.0 * C22 * y; dz = 4.0 * C22 * z; break;
    case 7: Y = C23 * x * z; dx = C23 * z; dz = C23 * x; break;
    case 8: Y = C24 * (xx - yy); dx = 2.0 * C24 * x; dy = -2.0 * C24 * y; break;
    case 9: Y = C30 * y * (3.0 * xx - yy); dx = 6.0 * C30 * x * y; dy = C30 * (3.0 * xx - 3.0 * yy); break;
    case 10: Y = C31 * x * y * z; dx = C31 * y * z; dy = C31 * x * z; dz = C31 * x * y; break;
    case 11:
      Y = C32 * y * (4.0 * zz - xx - yy);
      dx = -2.0 * C32 * x * y; dy = C32 * (4.0 * zz - xx - 3.0 * yy); dz = 8.0 * C32 * y * z;
      break;
    case 12:
      Y = C33 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
      dx = -6.0 * C33 * x * z; dy = -6.0 * C33 * y * z; dz = C33 * (6.0 * zz - 3.0 * xx - 3.0 * yy);
      break;
    case 13:
      Y = C34 * x * (4.0 * zz - xx - yy);
      dx = C34 * (4.0 * zz - 3.0 * xx - yy); dy = -2.0 * C34 * x * y; dz = 8.0 * C34 * x * z;
      break;
    case 14: Y = C35 * z * (xx - yy); dx = 2.0 * C35 * x * z; dy = -2.0 * C35 * y * z; dz = C35 * (xx - yy); break;
    default: Y = C36 * x * (xx - 3.0 * yy); dx = C36 * (3.0 * xx - 3.0 * yy); dy = -6.0 * C36 * x * y; break;
  }
}

// chain rule for slot s; accumulates the 10 geometry gradients into gout[0..9] (zeroed) and stores the
// SH basis Y_k (gout[10..10+K)) and the clamped colour gradient gc (gout[10+K..13+K)): the 3K SH
// gradients are the products Y_k * gc_c (sh_grad below), so the staging holds 13 + K floats, not 10 + 3K.
// sg: the slot's 16 screen-space sums; par: pos 3, log-scale 3, rot 4, projected rgb 3 (staged in
// shared memory with coalesced loads); shrow: the SH row, read straight from global memory
// Precision of the geometry part of the chain rule: float32 (the default) passes the strict gradient
// contract once K5 forms its sums without cancellation (behind-colour recursion, in-plane depth
// offsets); RTGS_BWD_F64=1 runs it in double (12 CTAs / SM without spills) for diagnosis.
#ifndef RTGS_BWD_F64
#define RTGS_BWD_F64 0
#endif
#if RTGS_BWD_F64
using Fp = double;
#define RTGS_PB_V a.V
#else
using Fp = float;
#define RTGS_PB_V a.Vf
#endif

template <int K>
__device__ __forceinline__ void project_bwd_slot(const PBArgs& a, const float* sg, const float* par,
                                                 const float* shrow, float* gout) {
  const float4 g0 = *reinterpret_cast<const float4*>(sg);
  const float4 g1 = *reinterpret_cast<const float4*>(sg + 4);
  const float4 g2 = *reinterpret_cast<const float4*>(sg + 8);
  const float gz2 = sg[12];
  const float dscale = a.w_d / fmaxf(1.f, a.acc[2]);
  const float dMx = g0.x, dMy = g0.y, dA = g0.z, dB = g0.w, dCc = g1.x;
  const float drgb[3] = {g1.y, g1.z, g1.w};
  // depth: A = sum q, E = sum q (p_c - D r) (the in-plane offsets, formed per pixel in K5), C = sum g_D
  const float dDa = g2.x * dscale, dDb0 = g2.y * dscale, dDb1 = g2.z * dscale, dDb2 = g2.w * dscale;
  const float dDz = gz2 * dscale;
  if (dMx == 0.f && dMy == 0.f && dA == 0.f && dB == 0.f && dCc == 0.f && drgb[0] == 0.f && drgb[1] == 0.f &&
      drgb[2] == 0.f && dDa == 0.f && dDb0 == 0.f && dDb1 == 0.f && dDb2 == 0.f && dDz == 0.f)
    return;  // nothing reached this slot
  const Fp px = par[0], py = par[1], pz = par[2];
  const double X = fma(a.V[0], (double)px, fma(a.V[1], (double)py, fma(a.V[2], (double)pz, a.tp[0])));
  const double Y = fma(a.V[3], (double)px, fma(a.V[4], (double)py, fma(a.V[5], (double)pz, a.tp[1])));
  const double Z = fma(a.V[6], (double)px, fma(a.V[7], (double)py, fma(a.V[8], (double)pz, a.tp[2])));
  const Fp x = (Fp)X, y = (Fp)Y, z = (Fp)Z;
  const Fp* V = RTGS_PB_V;
  const Fp q0 = par[6], q1 = par[7], q2 = par[8], q3 = par[9];
  const Fp qn2 = q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3;
  const Fp qinv = Fp(1) / sqrt(qn2);
  const Fp qw = q0 * qinv, qx = q1 * qinv, qy = q2 * qinv, qz = q3 * qinv;
  Fp R[3][3] = {{1.f - 2.f * (qy * qy + qz * qz), 2.f * (qx * qy - qw * qz), 2.f * (qx * qz + qw * qy)},
                   {2.f * (qx * qy + qw * qz), 1.f - 2.f * (qx * qx + qz * qz), 2.f * (qy * qz - qw * qx)},
                   {2.f * (qx * qz - qw * qy), 2.f * (qy * qz + qw * qx), 1.f - 2.f * (qx * qx + qy * qy)}};
  const Fp l[3] = {par[3], par[4], par[5]};
  const Fp sc[3] = {exp(l[0]), exp(l[1]), exp(l[2])};
  Fp M[3][3], Sg[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) M[r][c] = R[r][c] * sc[c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) Sg[r][c] = M[r][0] * M[c][0] + M[r][1] * M[c][1] + M[r][2] * M[c][2];
  const Fp iz = 1.f / z;
  const Fp ux = x * iz, uy = y * iz;
  const bool clx = ux < a.limx0 || ux > a.limx1, cly = uy < a.limy0 || uy > a.limy1;
  const Fp limx = fmin(fmax(ux, (Fp)a.limx0), (Fp)a.limx1), limy = fmin(fmax(uy, (Fp)a.limy0), (Fp)a.limy1);
  const Fp xc = z * limx, yc = z * limy;
  const Fp fx = a.cam.fx, fy = a.cam.fy;
  Fp J[2][3] = {{fx * iz, 0.f, -fx * xc * iz * iz}, {0.f, fy * iz, -fy * yc * iz * iz}};
  Fp Tm[2][3];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) Tm[r][c] = J[r][0] * V[c] + J[r][1] * V[3 + c] + J[r][2] * V[6 + c];
  Fp TS[2][3];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) TS[r][c] = Tm[r][0] * Sg[0][c] + Tm[r][1] * Sg[1][c] + Tm[r][2] * Sg[2][c];
  const Fp ca = TS[0][0] * Tm[0][0] + TS[0][1] * Tm[0][1] + TS[0][2] * Tm[0][2] + kDilation;
  const Fp cb = TS[0][0] * Tm[1][0] + TS[0][1] * Tm[1][1] + TS[0][2] * Tm[1][2];
  const Fp cc = TS[1][0] * Tm[1][0] + TS[1][1] * Tm[1][1] + TS[1][2] * Tm[1][2] + kDilation;
  const double det = (double)ca * cc - (double)cb * cb;
  const Fp Qa = (Fp)(cc / det), Qb = (Fp)(-cb / det), Qc = (Fp)(ca / det);

  // conic -> Sigma2D: dL/dSigma' = -Q G Q, G = [[dA, dB/2], [dB/2, dC]]
  const Fp G01 = 0.5f * dB;
  const Fp QG00 = Qa * dA + Qb * G01, QG01 = Qa * G01 + Qb * dCc;
  const Fp QG10 = Qb * dA + Qc * G01, QG11 = Qb * G01 + Qc * dCc;
  const Fp dS00 = -(QG00 * Qa + QG01 * Qb), dS01 = -(QG00 * Qb + QG01 * Qc);
  const Fp dS11 = -(QG10 * Qb + QG11 * Qc);
  const Fp dSp[2][2] = {{dS00, dS01}, {dS01, dS11}};
  // Sigma' = T Sigma T^T: dL/dSigma = T^T dS' T ; dL/dT = 2 dS' T Sigma
  Fp dSig[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      Fp v = 0.f;
      for (int p = 0; p < 2; ++p)
        for (int q = 0; q < 2; ++q) v += Tm[p][r] * dSp[p][q] * Tm[q][c];
      dSig[r][c] = v;
    }
  Fp dT[2][3];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) dT[r][c] = 2.f * (dSp[r][0] * TS[0][c] + dSp[r][1] * TS[1][c]);
  // T = J V: dL/dJ = dT V^T
  Fp dJ[2][3];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c) dJ[r][c] = dT[r][0] * V[3 * c] + dT[r][1] * V[3 * c + 1] + dT[r][2] * V[3 * c + 2];
  // J(x', y', z), x' = z clamp(x/z) (R5)
  Fp dx = 0.f, dy = 0.f, dz = 0.f;
  dz += dJ[0][0] * (-fx * iz * iz) + dJ[0][2] * (2.f * fx * xc * iz * iz * iz);
  dz += dJ[1][1] * (-fy * iz * iz) + dJ[1][2] * (2.f * fy * yc * iz * iz * iz);
  const Fp dxc = dJ[0][2] * (-fx * iz * iz), dyc = dJ[1][2] * (-fy * iz * iz);
  if (clx) dz += dxc * limx; else dx += dxc;
  if (cly) dz += dyc * limy; else dy += dyc;
  // mu = (fx x/z + cx, fy y/z + cy)
  dx += dMx * fx * iz;
  dy += dMy * fy * iz;
  dz += -dMx * fx * x * iz * iz - dMy * fy * y * iz * iz;
  // depth (Eq.4-5): dL/dp_c += dDa n_c + dDz e_z ; dL/dn_c = sum q (p_c - D r) = E
  int k = 2;
  if (l[1] < l[k]) k = 1;
  if (l[0] < l[k]) k = 0;
  // (selects, not dynamic indexing: keeps R / GR in registers)
  const Fp nwx = k == 0 ? R[0][0] : (k == 1 ? R[0][1] : R[0][2]);
  const Fp nwy = k == 0 ? R[1][0] : (k == 1 ? R[1][1] : R[1][2]);
  const Fp nwz = k == 0 ? R[2][0] : (k == 1 ? R[2][1] : R[2][2]);
  const Fp ncx = V[0] * nwx + V[1] * nwy + V[2] * nwz;
  const Fp ncy = V[3] * nwx + V[4] * nwy + V[5] * nwz;
  const Fp ncz = V[6] * nwx + V[7] * nwy + V[8] * nwz;
  dx += dDa * ncx;
  dy += dDa * ncy;
  dz += dDa * ncz + dDz;
  const Fp dncx = dDb0, dncy = dDb1, dncz = dDb2;
  // world position: p_c = V (p - t)  ->  dL/dp = V^T dL/dp_c
  Fp gp0 = V[0] * dx + V[3] * dy + V[6] * dz;
  Fp gp1 = V[1] * dx + V[4] * dy + V[7] * dz;
  Fp gp2 = V[2] * dx + V[5] * dy + V[8] * dz;
  // dL/dn_world = V^T dL/dn_c
  const Fp dnw0 = V[0] * dncx + V[3] * dncy + V[6] * dncz;
  const Fp dnw1 = V[1] * dncx + V[4] * dncy + V[7] * dncz;
  const Fp dnw2 = V[2] * dncx + V[5] * dncy + V[8] * dncz;
  // SH colour: rgb = max(0, sum_k Y_k(d) sh_k + 0.5), d = (p - campos)/|p - campos|
  const double vx = (double)px - a.campos[0], vy = (double)py - a.campos[1], vz = (double)pz - a.campos[2];
  const double vnorm = sqrt(vx * vx + vy * vy + vz * vz);
  const double ddx = vx / vnorm, ddy = vy / vnorm, ddz = vz / vnorm;
  const float dirx = (float)ddx, diry = (float)ddy, dirz = (float)ddz;
  // rgb = max(0, raw): the clamp decision (R17) comes from the projected colour (rgb == 0 <=> raw <= 0)
  const float gc0 = par[10] > 0.f ? drgb[0] : 0.f;
  const float gc1 = par[11] > 0.f ? drgb[1] : 0.f;
  const float gc2 = par[12] > 0.f ? drgb[2] : 0.f;
  float shc[3 * K];
  if constexpr ((3 * K) % 4 == 0) {  // 16-byte aligned row (K = 4, 16): LDG.128 straight from global memory
#pragma unroll
    for (int q = 0; q < 3 * K / 4; ++q) {
      const float4 t4 = reinterpret_cast<const float4*>(shrow)[q];
      shc[4 * q] = t4.x; shc[4 * q + 1] = t4.y; shc[4 * q + 2] = t4.z; shc[4 * q + 3] = t4.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 3 * K; ++q) shc[q] = shrow[q];
  }
  float gd0 = 0.f, gd1 = 0.f, gd2 = 0.f;
#pragma unroll
  for (int kk = 0; kk < K; ++kk) {
    double Yd, Yxd, Yyd, Yzd;
    sh_basis_one<double>(kk, ddx, ddy, ddz, Yd, Yxd, Yyd, Yzd);
    const float Y = (float)Yd, Yx = (float)Yxd, Yy = (float)Yyd, Yz = (float)Yzd;
    gout[10 + kk] = Y;  // SH gradient (kk, c) = Y_kk * gc_c, formed by the consumer (compact staging)
    const float c = shc[3 * kk] * gc0 + shc[3 * kk + 1] * gc1 + shc[3 * kk + 2] * gc2;
    gd0 += Yx * c;
    gd1 += Yy * c;
    gd2 += Yz * c;
  }
  {
    const float dd = gd0 * dirx + gd1 * diry + gd2 * dirz;
    const float inv = (float)(1.0 / vnorm);
    gp0 += (gd0 - dd * dirx) * inv;
    gp1 += (gd1 - dd * diry) * inv;
    gp2 += (gd2 - dd * dirz) * inv;
  }
  gout[10 + K] = gc0; gout[10 + K + 1] = gc1; gout[10 + K + 2] = gc2;
  gout[0] += gp0; gout[1] += gp1; gout[2] += gp2;
  // Sigma = M M^T, M = R diag(s): dL/dM = 2 dSig M
  Fp dM[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) dM[r][c] = 2.f * (dSig[r][0] * M[0][c] + dSig[r][1] * M[1][c] + dSig[r][2] * M[2][c]);
  for (int c = 0; c < 3; ++c) {
    const Fp dsc = dM[0][c] * R[0][c] + dM[1][c] * R[1][c] + dM[2][c] * R[2][c];
    gout[3 + c] += dsc * sc[c];  // s = exp(log_scale)
  }
  Fp GR[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) GR[r][c] = dM[r][c] * sc[c];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (c == k) { GR[0][c] += dnw0; GR[1][c] += dnw1; GR[2][c] += dnw2; }
  }
  // rotation matrix of the unit quaternion
  const Fp gw = 2.f * (-qz * GR[0][1] + qy * GR[0][2] + qz * GR[1][0] - qx * GR[1][2] - qy * GR[2][0] + qx * GR[2][1]);
  const Fp gx = 2.f * (qy * GR[0][1] + qz * GR[0][2] + qy * GR[1][0] - 2.f * qx * GR[1][1] - qw * GR[1][2] +
                          qz * GR[2][0] + qw * GR[2][1] - 2.f * qx * GR[2][2]);
  const Fp gy = 2.f * (-2.f * qy * GR[0][0] + qx * GR[0][1] + qw * GR[0][2] + qx * GR[1][0] + qz * GR[1][2] -
                          qw * GR[2][0] + qz * GR[2][1] - 2.f * qy * GR[2][2]);
  const Fp gz = 2.f * (-2.f * qz * GR[0][0] - qw * GR[0][1] + qx * GR[0][2] + qw * GR[1][0] - 2.f * qz * GR[1][1] +
                          qy * GR[1][2] + qx * GR[2][0] + qy * GR[2][1]);
  // through q = q~/|q~|
  const Fp dot = gw * qw + gx * qx + gy * qy + gz * qz;
  gout[6] += (gw - dot * qw) * qinv;
  gout[7] += (gx - dot * qx) * qinv;
  gout[8] += (gy - dot * qy) * qinv;
  gout[9] += (gz - dot * qz) * qinv;
}

constexpr int kPBS = 32;  // slots per k_project_bwd CTA, one thread each (swept 32 / 64 / 128: ~equal, 32 marginally best)

// One thread per slot, kPBS slots per CTA.  The screen-space sums and the geometry parameters are
// staged in shared memory with coalesced loads; each thread reads its SH row straight from global
// memory (LDG.128; staging it cost residency: DESIGN.md §10), and the kPBS compact gradient rows are
// accumulated into the contiguous grad block with coalesced read-modify-writes.
template <int K>
struct PBSmem {
  static constexpr int D = 10 + 3 * K, LD = (13 + K) | 1;  // compact row: 10 geometry, K basis, 3 gc
  static constexpr int SHF = 3 * K;
  float out[kPBS * LD];
  float sg[kPBS * kSG];
  float par[kPBS * 13];
  int gid[kPBS];
  uint8_t transparent[kPBS];
  uint64_t bar;
};

// gradient j (0 <= j < 10 + 3K) of a compact staging row
template <int K>
__device__ __forceinline__ float sh_grad(const float* row, int j) {
  if (j < 10) return row[j];
  const int kk = (j - 10) / 3, c = (j - 10) - 3 * kk;
  return row[10 + kk] * row[10 + K + c];
}

// Resident 32-slot CTAs per SM: 22 for SH degrees 2-3 (<= 88 registers, ~8 KB shared: 148 x 22 x 32 =
// 104k slots in one wave, so the C3 iteration's 100k unstable slots do not pay a second wave of CTA
// latency; -Xptxas -v: 12-28 B of spills at K = 9 / 16), 16 for degrees 0-1 (the 80-register cap
// spilled ~100 B there; with 128 registers none).  RTGS_BWD_F64: 12.
#ifndef RTGS_PB_MINB
#define RTGS_PB_MINB 22  // (swept round 2 at C3: 18 / 20 -> 62 us: a second wave; 25 -> 50 us: spills; 22 -> 48 us)
#endif
template <int K>
struct PBMinBlocks {
  static constexpr int value = RTGS_BWD_F64 ? 12 : (K >= 9 ? RTGS_PB_MINB : 16);
};
template <int K, bool ADAM>
__global__ void __launch_bounds__(kPBS, PBMinBlocks<K>::value) k_project_bwd(const PBArgs a) {
  using SM = PBSmem<K>;
  constexpr int D = SM::D, LD = SM::LD, SHF = SM::SHF;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x;
  const int s0 = blockIdx.x * kPBS;
  const int ns = min(kPBS, a.n_slots - s0);
  if (blockIdx.x == 0 && tid == 0) {  // loss values (device-side, no host sync)
    const float nP = (float)max(1u, a.counts[1]);
    const float Lc = a.acc[0] / (3.f * nP);
    const float Ld = a.acc[1] / fmaxf(1.f, a.acc[2]);
    a.loss_out[0] = Lc;
    a.loss_out[1] = Ld;
    a.loss_out[2] = a.w_c * Lc + a.w_d * Ld;
    a.loss_out[3] = a.acc[2];
  }
  if (ns <= 0) return;
  if (tid < ns) sm.gid[tid] = a.gid_of_slot[s0 + tid];
  if (ADAM && tid < ns) sm.transparent[tid] = (a.flags[sm.gid[tid]] & 5u) == 1u;  // not removed (R18, R29)
  const uint32_t eta_now = (ADAM && tid < ns) ? a.eta[sm.gid[tid]] : 0u;  // (read early: used at the end)
  __syncthreads();
  // (loads batched 8 deep before their stores so that many are in flight per thread)
  constexpr int U = 8;
  for (int e0 = tid; e0 < ns * kSG; e0 += kPBS * U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kPBS;
      v[u] = e < ns * kSG ? a.sgrad[(size_t)s0 * kSG + e] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * kPBS < ns * kSG) sm.sg[e0 + u * kPBS] = v[u];
  }
  __syncwarp();
  // slots that received any screen-space gradient this call; the accumulate form (no Adam: the
  // keyframe batch, where most of the map is out of a view's top-40 % pixels) skips the others
  // entirely -- their row gets + 0 -- instead of a read-modify-write of every row
  bool touched = false;
  if (tid < ns) {
#pragma unroll
    for (int k = 0; k < 13; ++k) touched |= sm.sg[tid * kSG + k] != 0.f;
  }
  const uint32_t tmask = __ballot_sync(0xffffffffu, touched);
  if (!ADAM && tmask == 0u) return;
  for (int e0 = tid; e0 < ns * 13; e0 += kPBS * U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kPBS;
      v[u] = 0.f;
      if (e < ns * 13) {
        const int ls = e / 13, c = e - ls * 13;
        const size_t g = (size_t)sm.gid[ls];
        v[u] = c < 3 ? a.pos[3 * g + c]
                     : (c < 6 ? a.log_scale[3 * g + (c - 3)]
                              : (c < 10 ? a.rot[4 * g + (c - 6)]
                                        : (a.sub_recf ? a.sub_recf[16 * (size_t)(s0 + ls) + 8 + (c - 10)]
                                                      : a.recf[16 * g + 8 + (c - 10)])));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * kPBS < ns * 13) sm.par[e0 + u * kPBS] = v[u];
  }
  float* gout = sm.out + tid * LD;
#pragma unroll
  for (int j = 0; j < 13 + K; ++j) gout[j] = 0.f;
  __syncthreads();
  if (tid < ns) project_bwd_slot<K>(a, sm.sg + tid * kSG, sm.par + tid * 13, a.sh + (size_t)sm.gid[tid] * SHF, gout);
  __syncthreads();
  // The epilogue walks the CTA's slot rows one after another, the warp's lanes over the row's D
  // components (lane, lane + 32): m / v / grad / SH rows stream coalesced, and every per-component
  // constant (learning-rate group, the SH (coefficient, channel) of the compact staging row) is a
  // per-lane register instead of a division per element.  kPBS == 32: the CTA is one warp.
  static_assert(kPBS == 32, "the epilogue maps the CTA's one warp onto the row components");
  constexpr int NH = (D + 31) / 32;
  const int lane = tid;
  int jh[NH], gidx0[NH], gidx1[NH];  // component, and its compact-row operands (gidx1 < 0: geometry)
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int j = lane + 32 * h;
    jh[h] = j;
    if (j < 10) { gidx0[h] = j; gidx1[h] = -1; }
    else {
      const int kk = (j - 10) / 3, c = (j - 10) - 3 * kk;
      gidx0[h] = 10 + kk; gidx1[h] = 10 + K + c;
    }
  }
  auto grad_of = [&](int ls, int h) -> float {
    const float* row = sm.out + ls * LD;
    return gidx1[h] < 0 ? row[gidx0[h]] : row[gidx0[h]] * row[gidx1[h]];
  };
  if constexpr (ADAM) {
    // A6 on the staged rows (the same update as k_adam, adam.cuh; SH updated in place in global
    // memory): the slot gradient never leaves shared memory; the new geometry goes back into the
    // staging and is written out below.
    const AdamBC bc = adam_bias(a.h);
    float lrh[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) lrh[h] = adam_lr(a.h, min(jh[h], D - 1));
    constexpr int SU = 4;  // slot rows in flight
    for (int l0 = 0; l0 < ns; l0 += SU) {
      float mo[SU][NH], vo[SU][NH], th[SU][NH], t0[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int ls = min(l0 + u, ns - 1);
        const size_t gsh = (size_t)sm.gid[ls] * SHF;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int j = jh[h];
          const bool live = l0 + u < ns && j < D;
          const size_t e = (size_t)(s0 + ls) * D + j;
          mo[u][h] = live ? a.m[e] : 0.f;
          vo[u][h] = live ? a.v[e] : 0.f;
          th[u][h] = !live ? 0.f : (j < 10 ? sm.par[ls * 13 + j] : a.sh[gsh + (j - 10)]);
        }
        // the L_reg anchor (lane < 10: the geometry components of h = 0), with the other loads
        t0[u] = (lane < 10 && l0 + u < ns && a.init_geom && sm.transparent[ls])
                    ? a.init_geom[(size_t)(s0 + ls) * 10 + lane] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int ls = l0 + u;
        if (ls >= ns) break;
        const size_t gsh = (size_t)sm.gid[ls] * SHF;
        const bool tr = sm.transparent[ls];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int j = jh[h];
          if (j >= D) continue;
          float gg = grad_of(ls, h);
          if (j < 10 && tr) gg += a.h.reg_coef * (th[u][h] - t0[u]);  // L_reg (R18)
          float mm = mo[u][h], vv = vo[u][h];
          const float nt = adam_one(a.h, bc, lrh[h], th[u][h], gg, mm, vv);
          if (j < 10) sm.par[ls * 13 + j] = nt;
          else a.wsh[gsh + (j - 10)] = nt;
          const size_t e = (size_t)(s0 + ls) * D + j;
          a.m[e] = mm;
          a.v[e] = vv;
        }
      }
    }
    __syncwarp();
    for (int e = tid; e < ns * 10; e += kPBS) {
      const int ls = e / 10, c = e - ls * 10;
      const size_t g = (size_t)sm.gid[ls];
      float* dst = c < 3 ? a.wpos + 3 * g + c : (c < 6 ? a.wlog_scale + 3 * g + (c - 3) : a.wrot + 4 * g + (c - 6));
      *dst = sm.par[ls * 13 + c];
    }
    if (tid < ns) {  // eta += 1 once per slot with a non-zero SH gradient (R20): the gradients are
      // Y_k gc_c with Y_0 = C0 != 0, so some is non-zero iff some gc_c is (as in real arithmetic)
      const float* row = sm.out + tid * LD;
      if (row[10 + K] != 0.f || row[10 + K + 1] != 0.f || row[10 + K + 2] != 0.f) a.eta[sm.gid[tid]] = eta_now + 1u;
    }
  } else {
    constexpr int SU = 8;  // touched slot rows in flight
    uint32_t rem = tmask;
    while (rem) {
      int ls[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        ls[u] = rem ? __ffs(rem) - 1 : -1;
        rem &= rem ? rem - 1u : 0u;
      }
      float g[SU][NH];
#pragma unroll
      for (int u = 0; u < SU; ++u)
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const bool live = ls[u] >= 0 && jh[h] < D;
          g[u][h] = live ? a.grad[(size_t)(s0 + ls[u]) * D + jh[h]] : 0.f;
        }
#pragma unroll
      for (int u = 0; u < SU; ++u)
#pragma unroll
        for (int h = 0; h < NH; ++h)
          if (ls[u] >= 0 && jh[h] < D) a.grad[(size_t)(s0 + ls[u]) * D + jh[h]] = g[u][h] + grad_of(ls[u], h);
    }
  }
}

struct FusedAdam {  // the A6 operands of the fused variant
  const rtgs_params* p;
  float* m;
  float* v;
  const float* init_geom;
  uint32_t* eta;
  AdamHP h;
};

static cudaError_t enqueue_backward(const rtgs_gaussians& g, const rtgs_projected& proj, const rtgs_bins& bins,
                                    const PoseF& pose, const rtgs_camera& cam, const rtgs_render_out& fwd,
                                    const rtgs_frame& target, const rtgs_loss_weights& w, const int32_t* slot_of_gid,
                                    const int32_t* gid_of_slot, int n_slots, float* grad, const FusedAdam* fz,
                                    float* loss_out, void* ws, cudaStream_t s) {
  float* sgrad = static_cast<float*>(ws);
  float* acc = sgrad + (size_t)n_slots * kSG;
  cudaMemsetAsync(ws, 0, ((size_t)n_slots * kSG + 8) * sizeof(float), s);
  BwdArgs a;
  a.rec = reinterpret_cast<const float4*>(proj.rec);
  a.sub_rec = reinterpret_cast<const float4*>(bins.sub_rec);
  a.zkey = proj.zkey;
  a.sorted_gid = bins.sorted_gid;
  a.range = reinterpret_cast<const uint2*>(bins.tile_range);
  a.tile_list = fwd.tile_list;
  a.counts = fwd.counts;
  a.active = fwd.active_bits;
  a.color = fwd.color; a.trans = fwd.trans; a.depth = fwd.depth; a.index = fwd.index; a.n_contrib = fwd.n_contrib;
  a.tcolor = target.color; a.tdepth = target.depth;
  a.slot_of_gid = slot_of_gid;
  a.cam = make_cam(cam);
  a.w_c = w.w_c;
  a.sgrad = sgrad;
  a.acc = acc;
  const int T = a.cam.TX * a.cam.TY;
  k_render_bwd<<<kBwdParts * T, 32 * (kBwdWarps + 1), 0, s>>>(a);
  note_launch();
  PBArgs b;
  b.rec = reinterpret_cast<const float4*>(proj.rec);
  b.recf = proj.rec;
  b.sub_recf = bins.sub_rec;
  b.pos = g.pos; b.log_scale = g.log_scale; b.rot = g.rot; b.sh = g.sh;
  b.K = (g.sh_degree + 1) * (g.sh_degree + 1);
  b.D = 10 + 3 * b.K;
  b.gid_of_slot = gid_of_slot;
  b.n_slots = n_slots;
  b.sgrad = sgrad;
  b.acc = acc;
  b.w_d = w.w_d;
  b.w_c = w.w_c;
  for (int k = 0; k < 9; ++k) { b.V[k] = pose.V[k]; b.Vf[k] = pose.Vf[k]; }
  for (int k = 0; k < 3; ++k) { b.tp[k] = pose.tp[k]; b.campos[k] = pose.campos[k]; }
  b.cam = a.cam;
  const double W = cam.width, H = cam.height;
  b.limx0 = (float)((-0.15 * W - cam.cx) / cam.fx);
  b.limx1 = (float)((1.15 * W - cam.cx) / cam.fx);
  b.limy0 = (float)((-0.15 * H - cam.cy) / cam.fy);
  b.limy1 = (float)((1.15 * H - cam.cy) / cam.fy);
  b.grad = grad;
  b.loss_out = loss_out;
  b.counts = fwd.counts;
  if (fz) {
    b.wpos = fz->p->pos; b.wlog_scale = fz->p->log_scale; b.wrot = fz->p->rot; b.wsh = fz->p->sh;
    b.flags = g.flags;
    b.m = fz->m; b.v = fz->v; b.init_geom = fz->init_geom; b.eta = fz->eta;
    b.h = fz->h;
  }
  const int nb = n_slots > 0 ? (n_slots + kPBS - 1) / kPBS : 1;
  static std::atomic<uint64_t> attr_mask{0};
  if (first_on_device(attr_mask)) {
#define RTGS_PB_ATTR(KK)                                                                                   \
  cudaFuncSetAttribute(k_project_bwd<KK, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,                \
                       (int)sizeof(PBSmem<KK>));                                                          \
  cudaFuncSetAttribute(k_project_bwd<KK, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PBSmem<KK>));
    RTGS_PB_ATTR(1) RTGS_PB_ATTR(4) RTGS_PB_ATTR(9) RTGS_PB_ATTR(16)
#undef RTGS_PB_ATTR
  }
#define RTGS_PB_LAUNCH(KK)                                                                   \
  if (fz) k_project_bwd<KK, true><<<nb, kPBS, sizeof(PBSmem<KK>), s>>>(b);                      \
  else k_project_bwd<KK, false><<<nb, kPBS, sizeof(PBSmem<KK>), s>>>(b);
  switch (b.K) {
    case 1: RTGS_PB_LAUNCH(1) break;
    case 4: RTGS_PB_LAUNCH(4) break;
    case 9: RTGS_PB_LAUNCH(9) break;
    default: RTGS_PB_LAUNCH(16) break;
  }
#undef RTGS_PB_LAUNCH
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_backward(const rtgs_gaussians& g, const rtgs_projected& proj, const rtgs_bins& bins,
                            const PoseF& pose, const rtgs_camera& cam, const rtgs_render_out& fwd,
                            const rtgs_frame& target, const rtgs_loss_weights& w, const int32_t* slot_of_gid,
                            const int32_t* gid_of_slot, int n_slots, float* grad, float* loss_out, void* ws,
                            cudaStream_t s) {
  return enqueue_backward(g, proj, bins, pose, cam, fwd, target, w, slot_of_gid, gid_of_slot, n_slots, grad, nullptr,
                          loss_out, ws, s);
}

cudaError_t launch_backward_adam(const rtgs_gaussians& g, const rtgs_projected& proj, const rtgs_bins& bins,
                                 const PoseF& pose, const rtgs_camera& cam, const rtgs_render_out& fwd,
                                 const rtgs_frame& target, const rtgs_loss_weights& w, const int32_t* slot_of_gid,
                                 const int32_t* gid_of_slot, int n_slots, const rtgs_params& p, float* m, float* v,
                                 const float* init_geom, int n_transparent, const rtgs_hparams& hp, int step,
                                 const int32_t* step_device, uint32_t* eta, float* loss_out, void* ws,
                                 cudaStream_t s) {
  FusedAdam fz{&p, m, v, init_geom, eta, make_adam_hp(hp, step, step_device, n_transparent, w.w_reg)};
  return enqueue_backward(g, proj, bins, pose, cam, fwd, target, w, slot_of_gid, gid_of_slot, n_slots, nullptr, &fz,
                          loss_out, ws, s);
}

}  // namespace rtgs
