// icp.cu — NEXT row f4: frame-to-model point-to-plane ICP tracking (Eq.10; readings
// R31, R33-R35).  A second workload on the renderer's outputs: the model maps are a FULL render
// (depth D^, world normal N^) of the optimised map at the previous pose.
//
//  k_pyr_down     one thread per coarse pixel: the 2x2 block's valid depth closest to the block
//                 mean (float32 decisions, R33)
//  k_vn_map       one thread per pixel of a level: float64 vertex and central-difference normal
//                 (R31), stored as double4 (w = validity)
//  k_icp_lin      one thread per current pixel: transform by the pose estimate (device memory),
//                 projective association into the model maps (nearest pixel, the R34 tolerance
//                 tie rule at x.5), gates, J = (n_m, p x n_m), r; the 29
//                 sums (upper-triangular J^T J, J^T r, r^2, count) reduced over the warp with
//                 shuffles, over the CTA in shared memory, then one float64 atomic per value
//  k_icp_solve    one thread: 6x6 Cholesky of A + 1e-6 max(diag A) I, delta = -(..)^-1 b, T <- Exp(delta) T, convergence flag,
//                 diagnostics row; zeroes the sums for the next iteration
// Everything is enqueued on one stream with no host synchronisation (graph-capturable).
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace rtgs {

constexpr int kIcpMaxLevels = 4;
constexpr int kSums = 29;  // 21 (A upper) + 6 (b) + E + count

struct LevelCam {
  double fx, fy, cx, cy;
  int W, H;
};

static LevelCam level_cam(const rtgs_camera& c, int l) {
  LevelCam k{c.fx, c.fy, c.cx, c.cy, c.width, c.height};
  for (int i = 0; i < l; ++i) {
    k.fx /= 2; k.fy /= 2; k.cx = (k.cx - 0.5) / 2; k.cy = (k.cy - 0.5) / 2;
    k.W /= 2; k.H /= 2;
  }
  return k;
}

__device__ __forceinline__ bool dvalid(float d) { return isfinite(d) && d > 0.f; }

__global__ void __launch_bounds__(256) k_pyr_down(const float* __restrict__ src, int Ws, float* __restrict__ dst,
                                                  int Wd, int Hd) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= Wd * Hd) return;
  const int x = i % Wd, y = i / Wd;
  const float v[4] = {src[(2 * y) * Ws + 2 * x], src[(2 * y) * Ws + 2 * x + 1], src[(2 * y + 1) * Ws + 2 * x],
                      src[(2 * y + 1) * Ws + 2 * x + 1]};
  float s = 0.f;
  int n = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (dvalid(v[k])) { s = __fadd_rn(s, v[k]); ++n; }
  float out = 0.f;
  if (n) {
    const float avg = __fdiv_rn(s, (float)n);
    float bd = INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (dvalid(v[k])) {
        const float e = fabsf(__fsub_rn(v[k], avg));
        if (e < bd) { bd = e; out = v[k]; }
      }
  }
  dst[i] = out;
}

__global__ void __launch_bounds__(256) k_vn_map(const float* __restrict__ d, LevelCam c, float guard,
                                                double4* __restrict__ V, double4* __restrict__ N) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= c.W * c.H) return;
  const int x = i % c.W, y = i / c.W;
  const float dc = d[i];
  double4 v = make_double4(0, 0, 0, 0), n = make_double4(0, 0, 0, 0);
  bool ok = dvalid(dc) && x >= 1 && x + 1 < c.W && y >= 1 && y + 1 < c.H;
  float dn[4] = {0.f, 0.f, 0.f, 0.f};
  if (ok) {
    dn[0] = d[i + 1]; dn[1] = d[i - 1]; dn[2] = d[i + c.W]; dn[3] = d[i - c.W];
#pragma unroll
    for (int k = 0; k < 4; ++k) ok = ok && dvalid(dn[k]) && fabsf(__fsub_rn(dn[k], dc)) <= guard;  // R31
  }
  auto vert = [&](int px, int py, float dd, double* o) {
    o[0] = __ddiv_rn(__dmul_rn((double)dd, __dsub_rn((double)px, c.cx)), c.fx);
    o[1] = __ddiv_rn(__dmul_rn((double)dd, __dsub_rn((double)py, c.cy)), c.fy);
    o[2] = (double)dd;
  };
  double p[3];
  vert(x, y, dc, p);
  if (ok) {
    double xp[3], xm[3], yp[3], ym[3];
    vert(x + 1, y, dn[0], xp);
    vert(x - 1, y, dn[1], xm);
    vert(x, y + 1, dn[2], yp);
    vert(x, y - 1, dn[3], ym);
    const double ax = xp[0] - xm[0], ay = xp[1] - xm[1], az = xp[2] - xm[2];
    const double bx = yp[0] - ym[0], by = yp[1] - ym[1], bz = yp[2] - ym[2];
    double nx = ay * bz - az * by, ny = az * bx - ax * bz, nz = ax * by - ay * bx;
    const double nn = sqrt(nx * nx + ny * ny + nz * nz);
    if (nn > 0.0) {
      nx /= nn; ny /= nn; nz /= nn;
      if (nx * p[0] + ny * p[1] + nz * p[2] > 0.0) { nx = -nx; ny = -ny; nz = -nz; }
      n = make_double4(nx, ny, nz, 1.0);
      v = make_double4(p[0], p[1], p[2], 1.0);
    }
  }
  V[i] = v;
  N[i] = n;
}

struct IcpState {
  double pose[12];  // (unused here: the pose lives in the caller's buffer)
  double acc[kSums];
  int done;
  int pad;
};

struct LinArgs {
  const double4* V;
  const double4* N;
  int n;                       // pixels of the level
  const float* mdepth;         // model D^ [H0][W0]
  const float* mnormal;        // model N^ [3][H0][W0] world
  int W0, H0;
  double fx, fy, cx, cy;       // level-0 intrinsics
  double Rm[9], tm[3];         // model pose (camera -> world)
  double dist_gate, cos_gate;
  const double* pose;          // current estimate [12] (R row-major, t)
  IcpState* st;
};

__device__ __forceinline__ double nearest_px(double x) {
  const double f = floor(x);
  return fabs((x - f) - 0.5) < 1e-9 ? f : rint(x);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256) k_icp_lin(const LinArgs a) {
  __shared__ double red[8][kSums];
  if (a.st->done) return;  // uniform: the level already converged
  const int i = blockIdx.x * 256 + threadIdx.x;
  double s[kSums];
#pragma unroll
  for (int k = 0; k < kSums; ++k) s[k] = 0.0;
  if (i < a.n) {
    const double4 v = a.V[i];
    if (v.w != 0.0) {
      const double4 nc = a.N[i];
      const double* T = a.pose;
      const double px = T[0] * v.x + T[1] * v.y + T[2] * v.z + T[9];
      const double py = T[3] * v.x + T[4] * v.y + T[5] * v.z + T[10];
      const double pz = T[6] * v.x + T[7] * v.y + T[8] * v.z + T[11];
      const double nwx = T[0] * nc.x + T[1] * nc.y + T[2] * nc.z;
      const double nwy = T[3] * nc.x + T[4] * nc.y + T[5] * nc.z;
      const double nwz = T[6] * nc.x + T[7] * nc.y + T[8] * nc.z;
      // model camera frame: q = Rm^T (p - tm)
      const double dx = px - a.tm[0], dy = py - a.tm[1], dz = pz - a.tm[2];
      const double qx = a.Rm[0] * dx + a.Rm[3] * dy + a.Rm[6] * dz;
      const double qy = a.Rm[1] * dx + a.Rm[4] * dy + a.Rm[7] * dz;
      const double qz = a.Rm[2] * dx + a.Rm[5] * dy + a.Rm[8] * dz;
      if (qz > 0.0) {
        // R34: nearest pixel, a projection within 1e-9 px of a boundary (x.5) to the lower one, so
        // the integer does not depend on the projection's rounding (coarse pixel centres project
        // exactly onto x.5 at the model pose)
        const double ux = nearest_px(a.fx * qx / qz + a.cx), uy = nearest_px(a.fy * qy / qz + a.cy);
        if (ux >= 0.0 && ux < (double)a.W0 && uy >= 0.0 && uy < (double)a.H0) {
          const int mi = (int)uy * a.W0 + (int)ux;
          const float md = a.mdepth[mi];
          if (md > 0.f) {
            const size_t HW = (size_t)a.W0 * a.H0;
            const double nmx = a.mnormal[mi], nmy = a.mnormal[HW + mi], nmz = a.mnormal[2 * HW + mi];
            // model vertex: Rm (D^ K^-1 (u^, 1)) + tm
            const double cxm = (double)md * (ux - a.cx) / a.fx, cym = (double)md * (uy - a.cy) / a.fy,
                         czm = (double)md;
            const double mx = a.Rm[0] * cxm + a.Rm[1] * cym + a.Rm[2] * czm + a.tm[0];
            const double my = a.Rm[3] * cxm + a.Rm[4] * cym + a.Rm[5] * czm + a.tm[1];
            const double mz = a.Rm[6] * cxm + a.Rm[7] * cym + a.Rm[8] * czm + a.tm[2];
            const double ex = px - mx, ey = py - my, ez = pz - mz;
            const bool ok = sqrt(ex * ex + ey * ey + ez * ez) <= a.dist_gate &&
                            nwx * nmx + nwy * nmy + nwz * nmz >= a.cos_gate;
            if (ok) {
              const double J[6] = {nmx, nmy, nmz, py * nmz - pz * nmy, pz * nmx - px * nmz, px * nmy - py * nmx};
              const double r = ex * nmx + ey * nmy + ez * nmz;
              int k = 0;
#pragma unroll
              for (int p = 0; p < 6; ++p)
#pragma unroll
                for (int q = p; q < 6; ++q) s[k++] = J[p] * J[q];
#pragma unroll
              for (int p = 0; p < 6; ++p) s[21 + p] = J[p] * r;
              s[27] = r * r;
              s[28] = 1.0;
            }
          }
        }
      }
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kSums; ++k) {
    const double t = warp_sum_d(s[k]);
    if (lane == 0) red[w][k] = t;
  }
  __syncthreads();
  if (threadIdx.x < kSums) {
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) t += red[ww][threadIdx.x];
    if (t != 0.0) atomicAdd(&a.st->acc[threadIdx.x], t);
  }
}

struct SolveArgs {
  double* pose;
  IcpState* st;
  double* diag;     // row [4]: level, E, count, |delta|
  int level;
  double eps;
  int min_pairs;
};

__global__ void k_icp_solve(const SolveArgs a) {
  if (threadIdx.x != 0) return;
  IcpState* st = a.st;
  double* acc = st->acc;
  if (st->done) {
    a.diag[0] = -1.0;  // skipped iteration
    for (int k = 0; k < kSums; ++k) acc[k] = 0.0;
    return;
  }
  const double E = acc[27], cnt = acc[28];
  a.diag[0] = (double)a.level;
  a.diag[1] = E;
  a.diag[2] = cnt;
  a.diag[3] = 0.0;
  if (cnt < (double)a.min_pairs) {
    st->done = 1;
  } else {
    double A[6][6], b[6];
    int k = 0;
    for (int p = 0; p < 6; ++p)
      for (int q = p; q < 6; ++q) { A[p][q] = acc[k]; A[q][p] = acc[k]; ++k; }
    for (int p = 0; p < 6; ++p) b[p] = acc[21 + p];
    double dmax = 0.0;  // R35: relative Tikhonov damping lambda = 1e-6 max diag
    for (int p = 0; p < 6; ++p) dmax = fmax(dmax, A[p][p]);
    for (int p = 0; p < 6; ++p) A[p][p] += 1e-6 * dmax;
    // Cholesky A = L L^T (in place, lower)
    bool spd = true;
    for (int j = 0; j < 6 && spd; ++j) {
      double d = A[j][j];
      for (int m = 0; m < j; ++m) d -= A[j][m] * A[j][m];
      if (!(d > 0.0)) { spd = false; break; }
      A[j][j] = sqrt(d);
      for (int r = j + 1; r < 6; ++r) {
        double v = A[r][j];
        for (int m = 0; m < j; ++m) v -= A[r][m] * A[j][m];
        A[r][j] = v / A[j][j];
      }
    }
    if (!spd) {
      st->done = 1;
    } else {
      double y[6], x[6];
      for (int r = 0; r < 6; ++r) {
        double v = -b[r];
        for (int m = 0; m < r; ++m) v -= A[r][m] * y[m];
        y[r] = v / A[r][r];
      }
      for (int r = 5; r >= 0; --r) {
        double v = y[r];
        for (int m = r + 1; m < 6; ++m) v -= A[m][r] * x[m];
        x[r] = v / A[r][r];
      }
      // Exp(xi), xi = (rho, phi) = x
      const double wx = x[3], wy = x[4], wz = x[5];
      const double th = sqrt(wx * wx + wy * wy + wz * wz);
      double cA, cB, cC;
      if (th < 1e-8) {
        cA = 1.0 - th * th / 6; cB = 0.5 - th * th / 24; cC = 1.0 / 6 - th * th / 120;
      } else {
        cA = sin(th) / th; cB = (1 - cos(th)) / (th * th); cC = (th - sin(th)) / (th * th * th);
      }
      const double K[3][3] = {{0, -wz, wy}, {wz, 0, -wx}, {-wy, wx, 0}};
      double K2[3][3], dR[3][3], Vm[3][3];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          K2[r][c] = K[r][0] * K[0][c] + K[r][1] * K[1][c] + K[r][2] * K[2][c];
        }
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          const double I = r == c ? 1.0 : 0.0;
          dR[r][c] = I + cA * K[r][c] + cB * K2[r][c];
          Vm[r][c] = I + cB * K[r][c] + cC * K2[r][c];
        }
      double dt[3];
      for (int r = 0; r < 3; ++r) dt[r] = Vm[r][0] * x[0] + Vm[r][1] * x[1] + Vm[r][2] * x[2];
      double* T = a.pose;
      double Rn[9], tn[3];
      for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) Rn[3 * r + c] = dR[r][0] * T[c] + dR[r][1] * T[3 + c] + dR[r][2] * T[6 + c];
        tn[r] = dR[r][0] * T[9] + dR[r][1] * T[10] + dR[r][2] * T[11] + dt[r];
      }
      for (int k2 = 0; k2 < 9; ++k2) T[k2] = Rn[k2];
      for (int k2 = 0; k2 < 3; ++k2) T[9 + k2] = tn[k2];
      double nd = 0.0;
      for (int p = 0; p < 6; ++p) nd += x[p] * x[p];
      nd = sqrt(nd);
      a.diag[3] = nd;
      if (nd < a.eps) st->done = 1;
    }
  }
  for (int k2 = 0; k2 < kSums; ++k2) acc[k2] = 0.0;
}

// ------------------------------------------------------------------------------------------------
static inline size_t al(size_t x) { return (x + 255) / 256 * 256; }

struct IcpWS {
  float* depth[kIcpMaxLevels];
  double4* V[kIcpMaxLevels];
  double4* N[kIcpMaxLevels];
  IcpState* st;
  size_t total;
};

static IcpWS carve_icp(const rtgs_camera& cam, int levels, char* base) {
  IcpWS w{};
  size_t o = 0;
  auto take = [&](size_t b) -> char* {
    char* p = base ? base + o : nullptr;
    o += al(b);
    return p;
  };
  for (int l = 0; l < levels; ++l) {
    const LevelCam c = level_cam(cam, l);
    const size_t px = (size_t)max(c.W, 1) * max(c.H, 1);
    w.depth[l] = (float*)take(px * 4);
    w.V[l] = (double4*)take(px * sizeof(double4));
    w.N[l] = (double4*)take(px * sizeof(double4));
  }
  w.st = (IcpState*)take(sizeof(IcpState));
  w.total = o;
  return w;
}

size_t icp_workspace_size(const rtgs_camera& cam, int levels) { return carve_icp(cam, levels, nullptr).total; }

cudaError_t launch_icp(const float* depth, const float* mdepth, const float* mnormal, const rtgs_pose& model_pose,
                       const rtgs_camera& cam, const rtgs_icp_params& p, double* pose_io, double* diag, void* ws,
                       cudaStream_t s) {
  IcpWS w = carve_icp(cam, p.levels, static_cast<char*>(ws));
  cudaMemsetAsync(w.st, 0, sizeof(IcpState), s);
  // level 0 depth is the input; coarser levels by k_pyr_down
  for (int l = 0; l < p.levels; ++l) {
    const LevelCam c = level_cam(cam, l);
    const int npx = c.W * c.H;
    const float* dl = depth;
    if (l > 0) {
      const LevelCam cp = level_cam(cam, l - 1);
      const float* src = (l == 1) ? depth : w.depth[l - 1];
      if (npx > 0) {
        k_pyr_down<<<(npx + 255) / 256, 256, 0, s>>>(src, cp.W, w.depth[l], c.W, c.H);
        note_launch();
      }
      dl = w.depth[l];
    }
    if (npx > 0) {
      k_vn_map<<<(npx + 255) / 256, 256, 0, s>>>(dl, c, p.normal_guard, w.V[l], w.N[l]);
      note_launch();
    }
  }
  LinArgs a;
  a.mdepth = mdepth; a.mnormal = mnormal;
  a.W0 = cam.width; a.H0 = cam.height;
  a.fx = cam.fx; a.fy = cam.fy; a.cx = cam.cx; a.cy = cam.cy;
  for (int k = 0; k < 9; ++k) a.Rm[k] = model_pose.R[k];
  for (int k = 0; k < 3; ++k) a.tm[k] = model_pose.t[k];
  a.dist_gate = p.dist_gate; a.cos_gate = p.cos_gate;
  a.pose = pose_io;
  a.st = w.st;
  SolveArgs sa;
  sa.pose = pose_io; sa.st = w.st; sa.eps = p.eps; sa.min_pairs = p.min_pairs;
  int row = 0;
  for (int l = p.levels - 1; l >= 0; --l) {
    const LevelCam c = level_cam(cam, l);
    a.V = w.V[l]; a.N = w.N[l]; a.n = c.W * c.H;
    sa.level = l;
    cudaMemsetAsync(&w.st->done, 0, sizeof(int), s);
    for (int it = 0; it < p.iters[l]; ++it, ++row) {
      if (a.n > 0) {
        k_icp_lin<<<(a.n + 255) / 256, 256, 0, s>>>(a);
        note_launch();
      }
      sa.diag = diag + 4 * row;
      k_icp_solve<<<1, 32, 0, s>>>(sa);
      note_launch();
    }
  }
  return cudaGetLastError();
}

}  // namespace rtgs
