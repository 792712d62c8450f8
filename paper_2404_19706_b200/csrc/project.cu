// project.cu — A1: per-Gaussian EWA projection (O1; Eq.2, readings R2-R8, R12).
//
// One thread per Gaussian, 64 Gaussians per CTA.  The SH block of the CTA (64 x 12K bytes, the
// dominant HBM stream: 192 of 237 B/Gaussian at degree 3) is staged into shared memory by ONE 1D
// bulk copy (cp.async.bulk, TMA engine) completing on an mbarrier, issued before the geometry math
// so the copy overlaps it; 12 KB of shared memory per CTA keeps 12 CTAs (24 warps) per SM resident,
// and the smaller CTAs keep more independent bulk copies in flight (measured: 56 vs 59 us for
// 128-thread CTAs at 6 per SM).  Camera-frame position and mu are formed in float64.
#include "common.cuh"
#include "internal.h"

namespace rtgs {

constexpr int kProjThreads = 64;

struct ProjArgs {
  const float* pos;
  const float* log_scale;
  const float* rot;
  const float* opacity;
  const float* sh;
  const uint8_t* flags;  // nullable; bit2 = removed (NEXT f1)
  const int32_t* subset;  // NEXT f3: row i projects Gaussian subset[i] (NULL: row i = Gaussian i)
  int n, K;               // n = number of rows
  double V[9], tp[3], campos[3];
  float Vz0, Vz1, Vz2, tz;  // float32 key sequence (R8)
  float Vf[9];
  CamK cam;
  float limx0, limx1, limy0, limy1;  // R5 clamp on x/z, y/z
  float4* rec;
  uint32_t* zkey;
  uint2* rect;  // 4 x int16
  uint32_t* touched;
  uint32_t* cnt;  // fused A2 count (launch_project_bin): replicated per-tile counters, else NULL
  int TX, T;
};

// SH colour of one Gaussian from its AoS row c[3k + ch] in shared memory (R2): the 3DGS real basis,
// constants restated from their closed forms sqrt((2l+1)/4pi ...); per channel the terms are summed
// in ascending k.  The row is read as 3K/4 float4 (rows of 192 B: 4-way bank conflicts, cheaper than
// a transpose buffer that would cut the CTAs resident per SM).
template <int K>
__device__ __forceinline__ float3 sh_eval(const float* c, float x, float y, float z) {
  float Y[16];
  Y[0] = 0.28209479177387814f;
  if (K > 1) {
    const float C1 = 0.4886025119029199f;
    Y[1] = -C1 * y; Y[2] = C1 * z; Y[3] = -C1 * x;
  }
  if (K > 4) {
    const float xx = x * x, yy = y * y, zz = z * z;
    Y[4] = 1.0925484305920792f * x * y;
    Y[5] = -1.0925484305920792f * y * z;
    Y[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
    Y[7] = -1.0925484305920792f * x * z;
    Y[8] = 0.5462742152960396f * (xx - yy);
    if (K > 9) {
      Y[9] = -0.5900435899266435f * y * (3.f * xx - yy);
      Y[10] = 2.890611442640554f * x * y * z;
      Y[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
      Y[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
      Y[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
      Y[14] = 1.445305721320277f * z * (xx - yy);
      Y[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
    }
  }
  float acc[3] = {0.f, 0.f, 0.f};
  if constexpr ((3 * K) % 4 == 0) {  // degree 1 and 3: 16 B aligned rows
    const float4* c4 = reinterpret_cast<const float4*>(c);
#pragma unroll
    for (int q = 0; q < 3 * K / 4; ++q) {
      const float4 v = c4[q];
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = 4 * q + u;
        acc[j % 3] = fmaf(Y[j / 3], e[u], acc[j % 3]);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 3 * K; ++j) acc[j % 3] = fmaf(Y[j / 3], c[j], acc[j % 3]);
  }
  return make_float3(acc[0], acc[1], acc[2]);
}

template <int K, bool SUB>
__global__ void __launch_bounds__(kProjThreads, 12) k_project(const ProjArgs a) {
  // s_sh: [kProjThreads][3K] as copied (AoS)
  extern __shared__ __align__(16) float s_sh[];
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  const int base = blockIdx.x * kProjThreads;
  const int cnt = min(kProjThreads, a.n - base);
  constexpr int shf = 3 * K;  // floats per Gaussian
  const int i = base + tid;
  bool live = i < a.n;
  const size_t gi = SUB ? (size_t)(live ? a.subset[i] : 0) : (size_t)i;  // Gaussian of this row
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if constexpr (!SUB) {  // contiguous rows: ONE bulk copy of the CTA's SH block
    const uint32_t bytes = (uint32_t)cnt * shf * 4u;
    const uint32_t bulk = bytes & ~15u;
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar, bulk);
      if (bulk) bulk_g2s(s_sh, a.sh + (size_t)base * shf, bulk, &bar);
    }
    if (tid < (int)((bytes - bulk) >> 2)) {  // <= 3 trailing floats when 12K*cnt % 16 != 0
      const int o = (bulk >> 2) + tid;
      s_sh[o] = a.sh[(size_t)base * shf + o];
    }
  } else if constexpr (shf % 4 == 0) {  // gathered rows: one bulk copy per row (12K bytes)
    if (tid == 0) mbar_arrive_expect_tx(&bar, (uint32_t)cnt * shf * 4u);
    __syncthreads();
    if (live) bulk_g2s(s_sh + tid * shf, a.sh + gi * shf, shf * 4, &bar);
  } else {  // rows not 16-byte multiples: plain loads
    if (tid == 0) mbar_arrive_expect_tx(&bar, 0u);
    if (live)
      for (int j = 0; j < shf; ++j) s_sh[tid * shf + j] = a.sh[gi * shf + j];
  }

  float4 r0 = make_float4(0, 0, 0, 0), r1 = r0, r2 = r0, r3 = r0;
  uint32_t zbits = 0xFFFFFFFFu;
  uint2 rect = make_uint2(1u | (1u << 16), 0u);  // empty: (x0,y0) = (1,1) > (x1,y1) = (0,0)
  uint32_t touched = 0;
  float dirx = 0, diry = 0, dirz = 1;
  bool vis = false;
  if (live) {
    // every per-Gaussian load issued up front: one DRAM round trip instead of a dependent chain
    const float px = a.pos[3 * gi], py = a.pos[3 * gi + 1], pz = a.pos[3 * gi + 2];
    const float alpha = a.opacity[gi];
    float qw = a.rot[4 * gi], qx = a.rot[4 * gi + 1], qy = a.rot[4 * gi + 2], qz = a.rot[4 * gi + 3];
    const float l0 = a.log_scale[3 * gi], l1 = a.log_scale[3 * gi + 1], l2 = a.log_scale[3 * gi + 2];
    const uint8_t fl = a.flags ? a.flags[gi] : (uint8_t)0;
    // R8: float32 key, every product and sum rounded, no FMA
    const float zk = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(a.Vz0, px), __fmul_rn(a.Vz1, py)), __fmul_rn(a.Vz2, pz)), a.tz);
    const float kext = (alpha * 255.f > 1.f) ? fminf(3.f, sqrtf(2.f * logf(255.f * alpha))) : 0.f;
    const bool removed = fl & 4u;
    if (zk > kNear && kext > 0.f && !removed) {
      // camera frame in float64: p_c = V p + t'
      const double X = fma(a.V[0], (double)px, fma(a.V[1], (double)py, fma(a.V[2], (double)pz, a.tp[0])));
      const double Y = fma(a.V[3], (double)px, fma(a.V[4], (double)py, fma(a.V[5], (double)pz, a.tp[1])));
      const double Z = fma(a.V[6], (double)px, fma(a.V[7], (double)py, fma(a.V[8], (double)pz, a.tp[2])));
      const float x = (float)X, y = (float)Y, z = (float)Z;
      // Sigma = R_q diag(s^2) R_q^T (R3)
      const float qn = rsqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
      qw *= qn; qx *= qn; qy *= qn; qz *= qn;
      const float R00 = 1.f - 2.f * (qy * qy + qz * qz), R01 = 2.f * (qx * qy - qw * qz), R02 = 2.f * (qx * qz + qw * qy);
      const float R10 = 2.f * (qx * qy + qw * qz), R11 = 1.f - 2.f * (qx * qx + qz * qz), R12 = 2.f * (qy * qz - qw * qx);
      const float R20 = 2.f * (qx * qz - qw * qy), R21 = 2.f * (qy * qz + qw * qx), R22 = 1.f - 2.f * (qx * qx + qy * qy);
      const float s0 = expf(l0), s1 = expf(l1), s2 = expf(l2);
      const float M00 = R00 * s0, M01 = R01 * s1, M02 = R02 * s2;
      const float M10 = R10 * s0, M11 = R11 * s1, M12 = R12 * s2;
      const float M20 = R20 * s0, M21 = R21 * s1, M22 = R22 * s2;
      const float S00 = M00 * M00 + M01 * M01 + M02 * M02, S01 = M00 * M10 + M01 * M11 + M02 * M12;
      const float S02 = M00 * M20 + M01 * M21 + M02 * M22, S11 = M10 * M10 + M11 * M11 + M12 * M12;
      const float S12 = M10 * M20 + M11 * M21 + M12 * M22, S22 = M20 * M20 + M21 * M21 + M22 * M22;
      // EWA (R4) with the 1.3x-FOV clamp of the Jacobian (R5)
      const float iz = 1.f / z;
      const float xc = z * fminf(fmaxf(x * iz, a.limx0), a.limx1);
      const float yc = z * fminf(fmaxf(y * iz, a.limy0), a.limy1);
      const float J00 = a.cam.fx * iz, J02 = -a.cam.fx * xc * iz * iz;
      const float J11 = a.cam.fy * iz, J12 = -a.cam.fy * yc * iz * iz;
      const float* V = a.Vf;
      const float T00 = J00 * V[0] + J02 * V[6], T01 = J00 * V[1] + J02 * V[7], T02 = J00 * V[2] + J02 * V[8];
      const float T10 = J11 * V[3] + J12 * V[6], T11 = J11 * V[4] + J12 * V[7], T12 = J11 * V[5] + J12 * V[8];
      const float U00 = T00 * S00 + T01 * S01 + T02 * S02, U01 = T00 * S01 + T01 * S11 + T02 * S12,
                  U02 = T00 * S02 + T01 * S12 + T02 * S22;
      const float U10 = T10 * S00 + T11 * S01 + T12 * S02, U11 = T10 * S01 + T11 * S11 + T12 * S12,
                  U12 = T10 * S02 + T11 * S12 + T12 * S22;
      const float ca = U00 * T00 + U01 * T01 + U02 * T02 + kDilation;
      const float cb = U00 * T10 + U01 * T11 + U02 * T12;
      const float cc = U10 * T10 + U11 * T11 + U12 * T12 + kDilation;
      const double det = (double)ca * cc - (double)cb * cb;
      const double idet = 1.0 / det;
      const float A = (float)(cc * idet), B = (float)(-cb * idet), C = (float)(ca * idet);
      // mu in float64, stored as double-float hi + lo
      const double mux = a.cam.fx * (X / Z) + a.cam.cx, muy = a.cam.fy * (Y / Z) + a.cam.cy;
      const float mxh = (float)mux, myh = (float)muy;
      const float mxl = (float)(mux - (double)mxh), myl = (float)(muy - (double)myh);
      // support rect (R7)
      const float ex = kext * sqrtf(ca) + kRectPad, ey = kext * sqrtf(cc) + kRectPad;
      const double fx0 = ceil(mux - (double)ex), fx1 = floor(mux + (double)ex);
      const double fy0 = ceil(muy - (double)ey), fy1 = floor(muy + (double)ey);
      const int x0 = (int)fmax(fx0, 0.0), x1 = (int)fmin(fx1, (double)(a.cam.W - 1));
      const int y0 = (int)fmax(fy0, 0.0), y1 = (int)fmin(fy1, (double)(a.cam.H - 1));
      if (x0 <= x1 && y0 <= y1 && det > 0.0) {
        vis = true;
        zbits = __float_as_uint(zk);
        rect = make_uint2((uint32_t)(x0 & 0xFFFF) | ((uint32_t)y0 << 16), (uint32_t)(x1 & 0xFFFF) | ((uint32_t)y1 << 16));
        touched = (uint32_t)((x1 / kTile - x0 / kTile + 1) * (y1 / kTile - y0 / kTile + 1));
        // disc normal: smallest axis, ties to the larger index (R12)
        int k = 2;
        if (l1 < (k == 2 ? l2 : l1)) k = 1;
        if (l0 < (k == 2 ? l2 : l1)) k = 0;
        const float nx = k == 0 ? R00 : (k == 1 ? R01 : R02);
        const float ny = k == 0 ? R10 : (k == 1 ? R11 : R12);
        const float nz = k == 0 ? R20 : (k == 1 ? R21 : R22);
        const float ncx = V[0] * nx + V[1] * ny + V[2] * nz;
        const float ncy = V[3] * nx + V[4] * ny + V[5] * nz;
        const float ncz = V[6] * nx + V[7] * ny + V[8] * nz;
        const double ndp = (double)ncx * X + (double)ncy * Y + (double)ncz * Z;
        const unsigned short hx = __half_as_ushort(__float2half_ru(ex)), hy = __half_as_ushort(__float2half_ru(ey));
        r0 = make_float4(mxh, myh, mxl, myl);
        // conic prescaled to base 2 and log2(alpha): f = 2^(A'dx^2 + B'dxdy + C'dy^2 + log2 alpha)
        r1 = make_float4(-0.5f * kLog2e * A, -kLog2e * B, -0.5f * kLog2e * C, log2f(alpha));
        r2.w = __uint_as_float((uint32_t)hx | ((uint32_t)hy << 16));
        r3 = make_float4(ncx, ncy, ncz, (float)ndp);
        // viewing direction camera centre -> Gaussian (world frame)
        const double vx = (double)px - a.campos[0], vy = (double)py - a.campos[1], vz = (double)pz - a.campos[2];
        const double vn = 1.0 / sqrt(vx * vx + vy * vy + vz * vz);
        dirx = (float)(vx * vn); diry = (float)(vy * vn); dirz = (float)(vz * vn);
      }
    }
  }
  mbar_wait(&bar, 0);
  __syncthreads();  // plain-load rows / trailing floats of the tail block
  if (live) {
    if (vis) {
      const float3 c = sh_eval<K>(s_sh + tid * 3 * K, dirx, diry, dirz);
      r2.x = fmaxf(0.f, c.x + 0.5f);
      r2.y = fmaxf(0.f, c.y + 0.5f);
      r2.z = fmaxf(0.f, c.z + 0.5f);
    }
    float4* o = a.rec + (size_t)4 * i;
    o[0] = r0; o[1] = r1; o[2] = r2; o[3] = r3;
    a.zkey[i] = zbits;
    a.rect[i] = rect;
    a.touched[i] = touched;
  }
  if (!SUB && a.cnt) {  // A2 count, as k_tile_count (same tiles, same replica of Gaussian i; warp-uniform)
    uint32_t* c = a.cnt + (size_t)((i >> 8) & (kRep - 1)) * a.T;
    const int tx0 = (int)(rect.x & 0xFFFF) / kTile, ty0 = (int)(rect.x >> 16) / kTile;
    const int tx1 = (int)(rect.y & 0xFFFF) / kTile, ty1 = (int)(rect.y >> 16) / kTile;
    const bool cnt_me = live && vis;
    const int w = tx1 - tx0 + 1, nt = cnt_me ? w * (ty1 - ty0 + 1) : 0;
    tile_count_agg(c, nt, w, tx0, ty0, a.TX, nullptr);
  }
}

PoseF make_pose(const rtgs_pose& p) {
  PoseF f;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) f.V[3 * r + c] = p.R[3 * c + r];  // V = R^T
  for (int r = 0; r < 3; ++r) {
    f.tp[r] = -(f.V[3 * r] * p.t[0] + f.V[3 * r + 1] * p.t[1] + f.V[3 * r + 2] * p.t[2]);
    f.campos[r] = p.t[r];
  }
  for (int k = 0; k < 9; ++k) { f.Vf[k] = (float)f.V[k]; f.Rf[k] = (float)p.R[k]; }
  for (int k = 0; k < 3; ++k) f.tpf[k] = (float)f.tp[k];
  return f;
}

static cudaError_t project_impl(const rtgs_gaussians& g, const int32_t* subset, int n_rows, const PoseF& pose,
                                const rtgs_camera& cam, const rtgs_projected& out, cudaStream_t s,
                                uint32_t* cnt = nullptr) {
  if (n_rows == 0) return cudaSuccess;
  ProjArgs a;
  a.pos = g.pos; a.log_scale = g.log_scale; a.rot = g.rot; a.opacity = g.opacity; a.sh = g.sh;
  a.flags = g.flags;
  a.subset = subset;
  a.n = n_rows;
  a.K = (g.sh_degree + 1) * (g.sh_degree + 1);
  for (int k = 0; k < 9; ++k) { a.V[k] = pose.V[k]; a.Vf[k] = pose.Vf[k]; }
  for (int k = 0; k < 3; ++k) { a.tp[k] = pose.tp[k]; a.campos[k] = pose.campos[k]; }
  a.Vz0 = pose.Vf[6]; a.Vz1 = pose.Vf[7]; a.Vz2 = pose.Vf[8]; a.tz = pose.tpf[2];
  a.cam = make_cam(cam);
  const double W = cam.width, H = cam.height;
  a.limx0 = (float)((-0.15 * W - cam.cx) / cam.fx);
  a.limx1 = (float)((1.15 * W - cam.cx) / cam.fx);
  a.limy0 = (float)((-0.15 * H - cam.cy) / cam.fy);
  a.limy1 = (float)((1.15 * H - cam.cy) / cam.fy);
  a.rec = reinterpret_cast<float4*>(out.rec);
  a.zkey = out.zkey;
  a.rect = reinterpret_cast<uint2*>(out.rect);
  a.touched = out.tiles_touched;
  a.cnt = cnt;
  a.TX = a.cam.TX;
  a.T = a.cam.TX * a.cam.TY;
  const size_t smem = (size_t)kProjThreads * 3 * a.K * sizeof(float);
  const int blocks = (n_rows + kProjThreads - 1) / kProjThreads;
  const bool sub = subset != nullptr;
#define RTGS_PROJ(KK)                                                                        \
  (sub ? (k_project<KK, true><<<blocks, kProjThreads, smem, s>>>(a), 0)                      \
       : (k_project<KK, false><<<blocks, kProjThreads, smem, s>>>(a), 0))
  switch (a.K) {
    case 1: RTGS_PROJ(1); break;
    case 4: RTGS_PROJ(4); break;
    case 9: RTGS_PROJ(9); break;
    default: RTGS_PROJ(16); break;
  }
#undef RTGS_PROJ
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_project(const rtgs_gaussians& g, const PoseF& pose, const rtgs_camera& cam,
                           const rtgs_projected& out, cudaStream_t s) {
  return project_impl(g, nullptr, g.n, pose, cam, out, s);
}

cudaError_t launch_project_count(const rtgs_gaussians& g, const PoseF& pose, const rtgs_camera& cam,
                                 const rtgs_projected& out, uint32_t* cnt, cudaStream_t s) {
  return project_impl(g, nullptr, g.n, pose, cam, out, s, cnt);
}

cudaError_t launch_project_subset(const rtgs_gaussians& g, const int32_t* gid_list, int n_list, const PoseF& pose,
                                  const rtgs_camera& cam, const rtgs_projected& out, cudaStream_t s) {
  return project_impl(g, gid_list, n_list, pose, cam, out, s);
}

}  // namespace rtgs
