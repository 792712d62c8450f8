// render.cu — A0 unstable coverage + tile keep (O4; Eq.12, R15, R16) and
//             A3/A4 forward colour/transmission blending with the opaque-disc depth (O2/O3;
//             Eq.1-5, R7-R12).
//
// Forward: one CTA per (kept) 16x16 tile, 8 warps, warp w owns an 8x4 pixel block, one pixel per
// lane.  Gaussian records of the tile's depth-sorted list are staged in 256-entry batches into
// double-buffered shared memory with cp.async; each warp culls a batch 32 records at a time against
// its 8x4 block (ballot over the records' support boxes) and only walks the survivors.  Pixels stop
// at T (1 - f) < 1e-4; warps stop when all their lanes stopped; the CTA stops when all warps did.
#include "common.cuh"
#include "internal.h"

namespace rtgs {

constexpr int kBatch = 256;

// ------------------------------------------------------------------------------------------------
// A0: coverage by splatting the unstable Gaussians (existence test, no order needed, R16)
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_coverage(const float4* __restrict__ rec, const uint2* __restrict__ rect,
                                                  const uint32_t* __restrict__ zkey, const uint8_t* __restrict__ flags,
                                                  int n, int W, uint32_t* __restrict__ bits) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool mine = i < n && !(flags[i] & 2u) && zkey[i] != 0xFFFFFFFFu;
  uint32_t m = __ballot_sync(0xffffffffu, mine);
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const int g = __shfl_sync(0xffffffffu, i, src);
    const uint2 r = rect[g];
    const int x0 = (int)(short)(r.x & 0xFFFF), y0 = (int)(short)(r.x >> 16);
    const int x1 = (int)(short)(r.y & 0xFFFF), y1 = (int)(short)(r.y >> 16);
    if (x0 > x1 || y0 > y1) continue;
    const float4 a = rec[4 * g], b = rec[4 * g + 1];
    const int w = x1 - x0 + 1;
    const int tot = w * (y1 - y0 + 1);
    for (int p = lane; p < tot; p += 32) {
      const int py = y0 + p / w, px = x0 + p % w;
      PairEval e;
      if (eval_pair(a, b, (float)px, (float)py, e)) {
        const uint32_t lin = (uint32_t)py * (uint32_t)W + (uint32_t)px;
        atomicOr(&bits[lin >> 5], 1u << (lin & 31u));
      }
    }
  }
}

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
    const bool k = 2 * na >= ni;  // P:497 / R15: discard tiles with < 50 % active pixels
    keep[t] = k ? 1 : 0;
    if (k) {
      const uint32_t pos = atomicAdd(&counts[0], 1u);
      list[pos] = (uint32_t)t;
      atomicAdd(&counts[1], (uint32_t)na);
    }
    if (na) atomicAdd(&counts[2], (uint32_t)na);
  }
}

// ------------------------------------------------------------------------------------------------
// A3/A4 forward
// ------------------------------------------------------------------------------------------------
struct FwdArgs {
  const float4* rec;
  const uint32_t* zkey;
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

template <bool MASKED>
__global__ void __launch_bounds__(256) k_render_fwd(const FwdArgs a) {
  __shared__ __align__(16) float4 s_rec[2][kBatch][3];
  __shared__ uint32_t s_gid[2][kBatch];
  int tile;
  if (MASKED) {
    if (blockIdx.x >= a.counts[0]) return;
    tile = (int)a.tile_list[blockIdx.x];
  } else {
    tile = blockIdx.x;
  }
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int tx = tile % a.cam.TX, ty = tile / a.cam.TX;
  const int wx0 = tx * kTile + (w & 1) * 8, wy0 = ty * kTile + (w >> 1) * 4;
  const int px = wx0 + (lane & 7), py = wy0 + (lane >> 3);
  const bool inside = px < a.cam.W && py < a.cam.H;
  const uint32_t lin = (uint32_t)py * (uint32_t)a.cam.W + (uint32_t)px;
  bool want = inside;
  if (MASKED && inside) want = (a.active[lin >> 5] >> (lin & 31u)) & 1u;
  bool done = !want;
  const float fpx = (float)px, fpy = (float)py;
  const float bx0 = (float)wx0, bx1 = (float)(wx0 + 7), by0 = (float)wy0, by1 = (float)(wy0 + 3);

  const uint2 rg = a.range[tile];
  const int start = (int)rg.x, end = (int)rg.y;
  const int nb = (end - start + kBatch - 1) / kBatch;

  float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f;
  int hit = -1;
  uint32_t last = (uint32_t)start;

  auto load = [&](int b, int buf) {
    const int i = start + b * kBatch + tid;
    if (i < end) {
      const uint32_t g = a.sorted_gid[i];
      s_gid[buf][tid] = g;
      const float4* src = a.rec + (size_t)4 * g;
      cp_async16(&s_rec[buf][tid][0], src);
      cp_async16(&s_rec[buf][tid][1], src + 1);
      cp_async16(&s_rec[buf][tid][2], src + 2);
    }
    cp_async_commit();
  };

  if (nb > 0) load(0, 0);
  for (int b = 0; b < nb; ++b) {
    const int buf = b & 1;
    if (b + 1 < nb) load(b + 1, buf ^ 1); else cp_async_commit();
    cp_async_wait<1>();
    if (__syncthreads_count(!done) == 0) break;
    const int cnt = min(kBatch, end - (start + b * kBatch));
    bool wdone = __all_sync(0xffffffffu, done);
    for (int g0 = 0; g0 < cnt && !wdone; g0 += 32) {
      const int j = g0 + lane;
      bool ov = false;
      if (j < cnt) {
        const float4 r0 = s_rec[buf][j][0];
        const float2 ext = unpack_ext(s_rec[buf][j][2].w);
        ov = (r0.x + ext.x >= bx0) && (r0.x - ext.x <= bx1) && (r0.y + ext.y >= by0) && (r0.y - ext.y <= by1);
      }
      uint32_t m = __ballot_sync(0xffffffffu, ov);
      while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        if (done) continue;
        const int idx = g0 + k;
        const float4 r0 = s_rec[buf][idx][0], r1 = s_rec[buf][idx][1];
        PairEval e;
        if (!eval_pair(r0, r1, fpx, fpy, e)) continue;
        if (hit < 0 && e.f > kDeltaAlpha) hit = (int)s_gid[buf][idx];  // R9: before termination
        const float test = __fmul_rn(T, __fsub_rn(1.f, e.f));
        if (test < kTMin) { done = true; continue; }
        const float4 r2 = s_rec[buf][idx][2];
        const float wgt = __fmul_rn(e.f, T);
        cr = __fmaf_rn(r2.x, wgt, cr);
        cg = __fmaf_rn(r2.y, wgt, cg);
        cb = __fmaf_rn(r2.z, wgt, cb);
        T = test;
        last = (uint32_t)(start + b * kBatch + idx + 1);
      }
      wdone = __all_sync(0xffffffffu, done);
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  if (!want) return;
  const size_t HW = (size_t)a.cam.W * a.cam.H;
  a.color[lin] = cr;
  a.color[HW + lin] = cg;
  a.color[2 * HW + lin] = cb;
  a.trans[lin] = T;
  a.n_contrib[lin] = last;
  a.index[lin] = hit;
  float D = -1.f, N0 = 0.f, N1 = 0.f, N2 = 0.f;
  if (hit >= 0) {
    const float4 pl = a.rec[(size_t)4 * hit + 3];  // n_c, n_c . p_c
    const float rx = (fpx - a.cam.cx) / a.cam.fx, ry = (fpy - a.cam.cy) / a.cam.fy;
    const float ndr = pl.x * rx + pl.y * ry + pl.z;
    const float nn = sqrtf(pl.x * pl.x + pl.y * pl.y + pl.z * pl.z);
    const float cosang = fabsf(ndr) / (sqrtf(rx * rx + ry * ry + 1.f) * nn);
    D = (cosang > kCos60) ? pl.w / ndr : __uint_as_float(a.zkey[hit]);  // Eq.5 (R10, R11)
    const float sg = ndr > 0.f ? -1.f : 1.f;                             // face the viewer (R12)
    const float nx = sg * pl.x, ny = sg * pl.y, nz = sg * pl.z;
    N0 = a.R[0] * nx + a.R[1] * ny + a.R[2] * nz;
    N1 = a.R[3] * nx + a.R[4] * ny + a.R[5] * nz;
    N2 = a.R[6] * nx + a.R[7] * ny + a.R[8] * nz;
  }
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
  k_tile_keep<<<k.TX * k.TY, 256, 0, s>>>(out.active_bits, k.W, k.H, k.TX, out.tile_keep, out.tile_list, out.counts);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_render(const rtgs_projected& proj, const rtgs_bins& bins, const PoseF& pose,
                          const rtgs_camera& cam, int masked, const rtgs_render_out& out, cudaStream_t s) {
  FwdArgs a;
  a.rec = reinterpret_cast<const float4*>(proj.rec);
  a.zkey = proj.zkey;
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
  if (masked) k_render_fwd<true><<<T, 256, 0, s>>>(a);
  else k_render_fwd<false><<<T, 256, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtgs
