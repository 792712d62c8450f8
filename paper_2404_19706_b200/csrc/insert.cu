// insert.cu — NEXT row f2: Gaussian insertion for the sampled add-mask pixels (P:232 input
// pre-processing, P:246-248 adding, Supp. A Eq.11; readings R26, R30-R32).
//
//  1. k_grid_count / scan / k_grid_scatter (x3 levels): hashed uniform grids over the existing,
//     non-removed Gaussians, cell h, 8h, 64h; a bucket holds the gids of every cell hashing to it.
//  2. k_insert_prepare: one thread per sample: vertex and central-difference normal of the pixel
//     (float64, the 0.1 m guard decided in float32), validity flag for the compaction.
//  3. scan of the validity flags: new gid = n + rank (sample order, deterministic).
//  4. k_insert_write: one WARP per valid sample: exact 3-NN by (distance, gid) — expanding cube
//     shells per grid level (lanes split the shell's cells), stopping when the third distance is
//     <= r h (no unexamined point can be closer), a brute-force pass (lanes split the Gaussians)
//     only if even the coarsest level cannot certify — then Eq.11's scale, the disc rotation
//     (shortest axis = normal), SH DC, state, appended at n + rank.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace rtgs {

constexpr int kGridLevels = 3;
constexpr int kGridR = 2;           // shells searched per level
constexpr double kC0 = 0.28209479177387814;  // Y_0^0 = 1 / (2 sqrt(pi))

__device__ __forceinline__ uint32_t cell_hash(int ix, int iy, int iz) {
  return ((uint32_t)ix * 73856093u) ^ ((uint32_t)iy * 19349663u) ^ ((uint32_t)iz * 83492791u);
}

struct GridLevel {
  double inv_h, h;
  uint32_t mask;        // M - 1
  uint32_t* cnt;        // [M]
  uint32_t* start;      // [M] exclusive scan of cnt
  uint32_t* cursor;     // [M]
  uint32_t* sorted;     // [n]
};

// bucket of Gaussian i at one level (0xFFFFFFFF: not a candidate)
__device__ __forceinline__ uint32_t grid_bucket(const float* pos, const uint8_t* flags, int n, int i,
                                                const GridLevel& L) {
  if (i >= n || (flags[i] & 4u)) return 0xFFFFFFFFu;
  const int ix = (int)floor((double)pos[3 * i] * L.inv_h), iy = (int)floor((double)pos[3 * i + 1] * L.inv_h),
            iz = (int)floor((double)pos[3 * i + 2] * L.inv_h);
  return cell_hash(ix, iy, iz) & L.mask;
}

// Counting sort by bucket with warp-aggregated atomics: lanes of a warp that share a bucket (common
// at the coarse levels, where a cell holds thousands of Gaussians) issue one atomic for the group.
__global__ void __launch_bounds__(256) k_grid_count(const float* __restrict__ pos, const uint8_t* __restrict__ flags,
                                                    int n, GridLevel L, uint32_t* __restrict__ n_cand) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const uint32_t b = grid_bucket(pos, flags, n, i, L);
  const uint32_t peers = __match_any_sync(0xffffffffu, b);
  if (b != 0xFFFFFFFFu && (__ffs(peers) - 1) == lane) atomicAdd(&L.cnt[b], (uint32_t)__popc(peers));
  if (n_cand) {
    const uint32_t s = __popc(__ballot_sync(0xffffffffu, b != 0xFFFFFFFFu));
    if (lane == 0 && s) atomicAdd(n_cand, s);
  }
}

__global__ void __launch_bounds__(256) k_grid_scatter(const float* __restrict__ pos, const uint8_t* __restrict__ flags,
                                                      int n, GridLevel L) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const uint32_t b = grid_bucket(pos, flags, n, i, L);
  const uint32_t peers = __match_any_sync(0xffffffffu, b);
  const int leader = __ffs(peers) - 1;
  uint32_t base = 0;
  if (b != 0xFFFFFFFFu && leader == lane) base = L.start[b] + atomicAdd(&L.cursor[b], (uint32_t)__popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (b != 0xFFFFFFFFu) L.sorted[base + __popc(peers & ((1u << lane) - 1u))] = (uint32_t)i;
}

struct InsArgs {
  // map (existing rows [0, n), new rows appended up to capacity)
  float *pos, *log_scale, *rot, *opacity, *sh;
  uint8_t* flags;
  uint32_t *eta, *err, *tc;
  int n, capacity, K;
  // samples
  const uint32_t* samples;
  const uint32_t* add_counts;
  uint32_t cap;
  // frame, pose, camera
  const float *color, *depth;
  int W, H;
  double fx, fy, cx, cy;
  double R[9], t[3];
  float guard, min_scale, max_t_scale;
  uint32_t frame_idx;
  // workspace
  uint32_t* valid;
  uint32_t* rank;
  double* vg;   // [cap][3]
  double* ng;   // [cap][3]
  GridLevel lev[kGridLevels];
  const uint32_t* n_cand;
  const uint32_t* n_valid;  // scan total
  uint32_t* result;         // [5]
};

__device__ __forceinline__ bool depth_ok(float d) { return isfinite(d) && d > 0.f; }

__global__ void __launch_bounds__(256) k_insert_prepare(const InsArgs a) {
  const uint32_t i = blockIdx.x * 256 + threadIdx.x;
  if (i >= a.cap) return;
  const uint32_t S = min(a.add_counts[2] + a.add_counts[3], a.cap);
  uint32_t ok = 0;
  if (i < S) {
    const uint32_t pix = a.samples[i] & 0x3FFFFFFFu;
    const int px = (int)(pix % (uint32_t)a.W), py = (int)(pix / (uint32_t)a.W);
    const float d = a.depth[pix];
    bool v = depth_ok(d) && px >= 1 && px + 1 < a.W && py >= 1 && py + 1 < a.H;
    float dn[4] = {0.f, 0.f, 0.f, 0.f};
    if (v) {
      dn[0] = a.depth[pix + 1];
      dn[1] = a.depth[pix - 1];
      dn[2] = a.depth[pix + a.W];
      dn[3] = a.depth[pix - a.W];
#pragma unroll
      for (int k = 0; k < 4; ++k) v = v && depth_ok(dn[k]) && fabsf(__fsub_rn(dn[k], d)) <= a.guard;  // R31
    }
    if (v) {
      auto vert = [&](int x, int y, float dd, double* o) {
        o[0] = (double)dd * ((double)x - a.cx) / a.fx;
        o[1] = (double)dd * ((double)y - a.cy) / a.fy;
        o[2] = (double)dd;
      };
      double c[3], xp[3], xm[3], yp[3], ym[3];
      vert(px, py, d, c);
      vert(px + 1, py, dn[0], xp);
      vert(px - 1, py, dn[1], xm);
      vert(px, py + 1, dn[2], yp);
      vert(px, py - 1, dn[3], ym);
      const double ax = xp[0] - xm[0], ay = xp[1] - xm[1], az = xp[2] - xm[2];
      const double bx = yp[0] - ym[0], by = yp[1] - ym[1], bz = yp[2] - ym[2];
      double nx = ay * bz - az * by, ny = az * bx - ax * bz, nz = ax * by - ay * bx;
      const double nn = sqrt(nx * nx + ny * ny + nz * nz);
      if (nn > 0.0) {
        nx /= nn; ny /= nn; nz /= nn;
        if (nx * c[0] + ny * c[1] + nz * c[2] > 0.0) { nx = -nx; ny = -ny; nz = -nz; }  // toward the camera
        double* o = a.vg + 3 * (size_t)i;
        double* m = a.ng + 3 * (size_t)i;
        for (int r = 0; r < 3; ++r) {
          o[r] = a.R[3 * r] * c[0] + a.R[3 * r + 1] * c[1] + a.R[3 * r + 2] * c[2] + a.t[r];
          m[r] = a.R[3 * r] * nx + a.R[3 * r + 1] * ny + a.R[3 * r + 2] * nz;
        }
        ok = 1;
      }
    }
  }
  a.valid[i] = ok;
}

// top-3 by (d2, gid), duplicates (a bucket reached twice) ignored
struct Top3 {
  double d[3];
  uint32_t g[3];
  int n;
  __device__ void init() {
    n = 0;
    for (int k = 0; k < 3; ++k) { d[k] = INFINITY; g[k] = 0xFFFFFFFFu; }
  }
  __device__ __forceinline__ static bool less(double d0, uint32_t g0, double d1, uint32_t g1) {
    return d0 < d1 || (d0 == d1 && g0 < g1);
  }
  __device__ void offer(double dd, uint32_t gg) {
    if (n == 3 && !less(dd, gg, d[2], g[2])) return;
    for (int k = 0; k < n; ++k)
      if (g[k] == gg) return;
    int k = n < 3 ? n : 2;
    if (n < 3) ++n;
    while (k > 0 && less(dd, gg, d[k - 1], g[k - 1])) {
      d[k] = d[k - 1];
      g[k] = g[k - 1];
      --k;
    }
    d[k] = dd;
    g[k] = gg;
  }
};

// Warp-wide merge of the lanes' top-3 lists (each sorted): the 3 smallest (d, gid) of the union;
// every lane returns the same list (duplicates of a gid seen by several lanes count once).
__device__ Top3 warp_top3(const Top3& mine) {
  Top3 out;
  out.init();
  int head = 0;
  for (int k = 0; k < 3; ++k) {
    double dv = head < mine.n ? mine.d[head] : INFINITY;
    uint32_t gv = head < mine.n ? mine.g[head] : 0xFFFFFFFFu;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, dv, o);
      const uint32_t og = __shfl_xor_sync(0xffffffffu, gv, o);
      if (Top3::less(od, og, dv, gv)) { dv = od; gv = og; }
    }
    if (gv == 0xFFFFFFFFu) break;
    out.d[k] = dv;
    out.g[k] = gv;
    out.n = k + 1;
    if (head < mine.n && mine.g[head] == gv) ++head;
  }
  return out;
}

// One WARP per sample: the lanes split the cells of each cube shell (and, in the brute-force
// fallback, the Gaussians), so the dependent bucket -> position loads of many cells are in flight
// together; the lanes' top-3 lists are merged after every shell for the certification test.
__global__ void __launch_bounds__(128) k_insert_write(const InsArgs a) {
  const uint32_t i = (blockIdx.x * 128 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= a.cap || !a.valid[i]) return;  // warp-uniform
  const uint32_t rk = a.rank[i];
  const uint32_t s = a.samples[i];
  const uint32_t pix = s & 0x3FFFFFFFu;
  const bool transparent = (s >> 30) == 2u;
  const size_t g = (size_t)a.n + rk;
  if (g >= (size_t)a.capacity) {
    if (lane == 0) atomicAdd(&a.result[3], 1u);
    return;
  }
  const double vx = a.vg[3 * i], vy = a.vg[3 * i + 1], vz = a.vg[3 * i + 2];
  const double nx = a.ng[3 * i], ny = a.ng[3 * i + 1], nz = a.ng[3 * i + 2];
  // ---- Eq.11 scale from the 3 nearest existing Gaussians (R26, R30) ----
  double s1;
  if (*a.n_cand < 3u) {
    s1 = 2.0 * (double)a.depth[pix] / a.fx;
  } else {
    Top3 top;
    top.init();
    auto offer_point = [&](uint32_t q) {
      const double dx = vx - (double)a.pos[3 * q], dy = vy - (double)a.pos[3 * q + 1], dz = vz - (double)a.pos[3 * q + 2];
      top.offer(dx * dx + dy * dy + dz * dz, q);
    };
    bool certified = false;
    for (int l = 0; l < kGridLevels && !certified; ++l) {
      const GridLevel& L = a.lev[l];
      const int cx = (int)floor(vx * L.inv_h), cy = (int)floor(vy * L.inv_h), cz = (int)floor(vz * L.inv_h);
      for (int r = 0; r <= kGridR && !certified; ++r) {
        const int side = 2 * r + 1, ncube = side * side * side;
        for (int c = lane; c < ncube; c += 32) {
          const int dx = c % side - r, dy = (c / side) % side - r, dz = c / (side * side) - r;
          if (max(abs(dx), max(abs(dy), abs(dz))) != r) continue;  // shell only
          const uint32_t b = cell_hash(cx + dx, cy + dy, cz + dz) & L.mask;
          const uint32_t j0 = L.start[b], j1 = j0 + L.cnt[b];
          for (uint32_t j = j0; j < j1; ++j) offer_point(L.sorted[j]);
        }
        top = warp_top3(top);
        // every unexamined Gaussian lies in a cell >= r+1 away: farther than r h
        const double rh = (double)r * L.h;
        certified = top.n == 3 && top.d[2] <= rh * rh;
      }
    }
    if (!certified) {  // beyond the coarsest grid's reach: exact brute force (rare)
      for (int q = lane; q < a.n; q += 32)
        if (!(a.flags[q] & 4u)) offer_point((uint32_t)q);
      top = warp_top3(top);
    }
    double m = 0.0;
    for (int k = 0; k < 3; ++k) {
      const uint32_t q = top.g[k];
      double e0 = exp((double)a.log_scale[3 * q]), e1 = exp((double)a.log_scale[3 * q + 1]),
             e2 = exp((double)a.log_scale[3 * q + 2]);
      // the two largest axis lengths
      const double mn = fmin(e0, fmin(e1, e2));
      const double ab = e0 + e1 + e2 - mn;
      m += sqrt(top.d[k]) - 0.5 * ab;
    }
    m /= 3.0;
    s1 = fmax((double)a.min_scale, sqrt(fmax(m, 0.0)));
  }
  if (transparent) s1 = fmin(s1, (double)a.max_t_scale);
  // ---- disc orientation: shortest axis (index 2) along the normal: q rotates e_z onto n ----
  double qw = 1.0 + nz, qx = -ny, qy = nx, qz = 0.0;
  double qn = sqrt(qw * qw + qx * qx + qy * qy);
  if (!(qn > 1e-12)) { qw = 0.0; qx = 1.0; qy = 0.0; qn = 1.0; }  // n = -e_z: 180 deg about x
  const size_t HW = (size_t)a.W * a.H;
  float* shr = a.sh + (size_t)3 * a.K * g;
  for (int j = 3 + lane; j < 3 * a.K; j += 32) shr[j] = 0.f;
  if (lane != 0) return;
  a.pos[3 * g] = (float)vx;
  a.pos[3 * g + 1] = (float)vy;
  a.pos[3 * g + 2] = (float)vz;
  const float ls = (float)log(s1), ls3 = (float)log(0.1 * s1);
  a.log_scale[3 * g] = ls;
  a.log_scale[3 * g + 1] = ls;
  a.log_scale[3 * g + 2] = ls3;
  a.rot[4 * g] = (float)(qw / qn);
  a.rot[4 * g + 1] = (float)(qx / qn);
  a.rot[4 * g + 2] = (float)(qy / qn);
  a.rot[4 * g + 3] = (float)(qz / qn);
  a.opacity[g] = transparent ? 0.1f : 0.99f;
  for (int c = 0; c < 3; ++c) shr[c] = (float)(((double)a.color[c * HW + pix] - 0.5) / kC0);  // R32
  a.flags[g] = transparent ? 1u : 0u;  // unstable (bit1 clear), not removed
  a.eta[g] = 0u;
  a.err[g] = 0u;
  a.tc[g] = a.frame_idx;
  atomicAdd(&a.result[transparent ? 1 : 0], 1u);
}

__global__ void k_insert_finish(const InsArgs a) {
  if (threadIdx.x != 0) return;
  const uint32_t S = min(a.add_counts[2] + a.add_counts[3], a.cap);
  const uint32_t nv = *a.n_valid;
  a.result[2] = S - nv;  // skipped: invalid normal (R31)
  a.result[4] = min((uint32_t)a.capacity, (uint32_t)a.n + nv);
}

// ------------------------------------------------------------------------------------------------
static inline size_t al(size_t x) { return (x + 255) / 256 * 256; }

static uint32_t level_buckets(int n, int l) {
  uint32_t want = (uint32_t)max(1024, 2 * n) >> (3 * l);
  uint32_t m = 1024;
  while (m < want) m <<= 1;
  return m;
}

struct InsWS {
  GridLevel lev[kGridLevels];
  uint32_t *valid, *rank, *n_cand, *n_valid;
  double *vg, *ng;
  void* scan_ws;
  size_t total;
};

static InsWS carve_ins(int n, uint32_t cap, char* base) {
  InsWS w{};
  size_t o = 0;
  auto take = [&](size_t b) -> char* {
    char* p = base ? base + o : nullptr;
    o += al(b);
    return p;
  };
  size_t scan_need = scan_workspace_size(cap);
  for (int l = 0; l < kGridLevels; ++l) {
    const uint32_t M = level_buckets(n, l);
    w.lev[l].mask = M - 1;
    w.lev[l].cnt = (uint32_t*)take((size_t)M * 4);
    w.lev[l].cursor = (uint32_t*)take((size_t)M * 4);
    w.lev[l].start = (uint32_t*)take((size_t)M * 4);
    w.lev[l].sorted = (uint32_t*)take((size_t)max(n, 1) * 4);
    scan_need = std::max(scan_need, scan_workspace_size(M));
  }
  w.valid = (uint32_t*)take((size_t)cap * 4 + 4);
  w.rank = (uint32_t*)take((size_t)cap * 4 + 4);
  w.n_cand = (uint32_t*)take(4);
  w.n_valid = (uint32_t*)take(4);
  w.vg = (double*)take((size_t)cap * 24 + 24);
  w.ng = (double*)take((size_t)cap * 24 + 24);
  w.scan_ws = take(scan_need);
  w.total = o;
  return w;
}

size_t insert_workspace_size(int n, uint32_t sample_cap) { return carve_ins(n, sample_cap, nullptr).total; }

cudaError_t launch_insert(const rtgs_map& m, const uint32_t* samples, uint32_t cap, const uint32_t* add_counts,
                          const rtgs_frame& frame, const PoseF& pose, const rtgs_camera& cam,
                          const rtgs_insert_params& ip, uint32_t* result, void* ws, cudaStream_t s) {
  InsWS w = carve_ins(m.n, cap, static_cast<char*>(ws));
  cudaMemsetAsync(result, 0, 5 * sizeof(uint32_t), s);
  cudaMemsetAsync(w.n_cand, 0, 4, s);
  InsArgs a;
  a.pos = m.pos; a.log_scale = m.log_scale; a.rot = m.rot; a.opacity = m.opacity; a.sh = m.sh;
  a.flags = m.flags; a.eta = m.eta; a.err = m.err_count; a.tc = m.t_created;
  a.n = m.n; a.capacity = m.capacity; a.K = (m.sh_degree + 1) * (m.sh_degree + 1);
  a.samples = samples; a.add_counts = add_counts; a.cap = cap;
  a.color = frame.color; a.depth = frame.depth;
  a.W = cam.width; a.H = cam.height;
  a.fx = cam.fx; a.fy = cam.fy; a.cx = cam.cx; a.cy = cam.cy;
  // camera -> world rotation R (row-major) and centre t
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a.R[3 * r + c] = pose.V[3 * c + r];  // R = V^T
  for (int r = 0; r < 3; ++r) a.t[r] = pose.campos[r];
  a.guard = ip.normal_guard; a.min_scale = ip.min_scale; a.max_t_scale = ip.max_scale_transparent;
  a.frame_idx = ip.frame_idx;
  a.valid = w.valid; a.rank = w.rank; a.vg = w.vg; a.ng = w.ng;
  a.n_cand = w.n_cand; a.n_valid = w.n_valid; a.result = result;
  const int nb = (m.n + 255) / 256;
  double h = ip.cell > 0.f ? (double)ip.cell : 0.02;
  for (int l = 0; l < kGridLevels; ++l) {
    GridLevel L = w.lev[l];
    L.h = h;
    L.inv_h = 1.0 / h;
    a.lev[l] = L;
    const size_t M = (size_t)L.mask + 1;
    cudaMemsetAsync(L.cnt, 0, M * 4, s);
    cudaMemsetAsync(L.cursor, 0, M * 4, s);
    if (m.n > 0) {
      k_grid_count<<<nb, 256, 0, s>>>(m.pos, m.flags, m.n, L, l == 0 ? w.n_cand : nullptr);
      note_launch();
    }
    cudaError_t e = launch_scan(L.cnt, L.start, M, nullptr, w.scan_ws, s);
    if (e != cudaSuccess) return e;
    if (m.n > 0) {
      k_grid_scatter<<<nb, 256, 0, s>>>(m.pos, m.flags, m.n, L);
      note_launch();
    }
    h *= 8.0;
  }
  if (cap > 0) {
    k_insert_prepare<<<(cap + 255) / 256, 256, 0, s>>>(a);
    cudaError_t e = launch_scan(w.valid, w.rank, cap, w.n_valid, w.scan_ws, s);
    if (e != cudaSuccess) return e;
    k_insert_write<<<(cap + 3) / 4, 128, 0, s>>>(a);  // one warp per sample
    note_launch(2);
  } else {
    cudaMemsetAsync(w.n_valid, 0, 4, s);
  }
  k_insert_finish<<<1, 32, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtgs
