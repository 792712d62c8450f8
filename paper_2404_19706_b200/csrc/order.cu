// order.cu — spatial (Morton) order of the Gaussian map: a data-layout step of the framework, not a
// step of the method.  The paper's maps grow frame by frame from row-major pixel samples, so
// nearby Gaussians sit at nearby indices; a map handed over in arbitrary order (or fragmented by
// removals) loses that, and with it the coherence the binning's per-tile counters, the renderer's
// record gathers and the backward's gradient rows rely on.  rtgs_morton_order returns the
// permutation that sorts the live Gaussians by the 30-bit Morton code of their position in the map's
// bounding box (removed ones last), rtgs_gather_rows applies it to any per-Gaussian array.
//
//  k_bbox          grid-stride min / max of the live positions (order-preserving int atomics)
//  k_morton        per Gaussian: q = min(1023, (int)((p - lo) * s)) per axis with s = 1024 / ext
//                  (float32, the exact sequence the host test repeats), 3 x 10 bits interleaved
//  radix sort      stable LSD over (code, gid) pairs, 8-bit digits, 4 passes: per-block digit
//                  histograms -> one exclusive scan in digit-major order -> per-block stable scatter
//                  (warp match_any ranks over contiguous per-warp runs, as the tile sort)
//  k_gather_rows   dst[r] = src[perm[r]] for rows of any byte width (16-byte vectors when aligned)
#include "common.cuh"
#include "internal.h"

namespace rtgs {

constexpr int kOrdThreads = 256;
constexpr int kOrdItems = 8;
constexpr int kOrdBlock = kOrdThreads * kOrdItems;  // 2048 pairs per sort block
constexpr int kOrdWarps = kOrdThreads / 32;

__device__ __forceinline__ int f2ord(float f) {  // order-preserving float -> int
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

__global__ void k_bbox_init(int* bb) {
  if (threadIdx.x < 3) bb[threadIdx.x] = 0x7FFFFFFF;
  else if (threadIdx.x < 6) bb[threadIdx.x] = (int)0x80000000;
}

__global__ void __launch_bounds__(256) k_bbox(const float* __restrict__ pos, const uint8_t* __restrict__ flags, int n,
                                              int* __restrict__ bb) {
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
    if (flags && (flags[i] & 4u)) continue;  // removed (R29): not part of the live map
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float v = pos[3 * (size_t)i + k];
      lo[k] = fminf(lo[k], v);
      hi[k] = fmaxf(hi[k], v);
    }
  }
  __shared__ float s_lo[3][8], s_hi[3][8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float a = lo[k], b = hi[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) { s_lo[k][w] = a; s_hi[k][w] = b; }
  }
  __syncthreads();
  if (threadIdx.x < 3) {  // one atomic pair per block and axis (same-address atomics serialise)
    const int k = threadIdx.x;
    float a = s_lo[k][0], b = s_hi[k][0];
    for (int ww = 1; ww < 8; ++ww) { a = fminf(a, s_lo[k][ww]); b = fmaxf(b, s_hi[k][ww]); }
    if (a <= b) {
      atomicMin(&bb[k], f2ord(a));
      atomicMax(&bb[3 + k], f2ord(b));
    }
  }
}

__device__ __forceinline__ uint32_t spread10(uint32_t v) {  // 10 bits -> every third bit
  v &= 0x3FFu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void __launch_bounds__(256) k_morton(const float* __restrict__ pos, const uint8_t* __restrict__ flags, int n,
                                                const int* __restrict__ bb, uint32_t* __restrict__ code,
                                                uint32_t* __restrict__ idx) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= n) return;
  uint32_t c = 0xFFFFFFFFu;  // removed: after every live Gaussian
  if (!(flags && (flags[i] & 4u))) {
    uint32_t q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float lo = ord2f(bb[k]), ext = __fsub_rn(ord2f(bb[3 + k]), lo);
      const float s = ext > 0.f ? __fdiv_rn(1024.f, ext) : 0.f;
      const float t = __fmul_rn(__fsub_rn(pos[3 * (size_t)i + k], lo), s);
      q[k] = (uint32_t)min(1023, (int)t);
    }
    c = (spread10(q[0]) << 2) | (spread10(q[1]) << 1) | spread10(q[2]);
  }
  code[i] = c;
  idx[i] = (uint32_t)i;
}

// per-block digit histogram, digit-major: hist[d * nb + b]
__global__ void __launch_bounds__(kOrdThreads) k_rs_hist(const uint32_t* __restrict__ key, int n, int shift,
                                                         uint32_t* __restrict__ hist, int nb) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0u;
  __syncthreads();
  const int base = blockIdx.x * kOrdBlock;
#pragma unroll
  for (int k = 0; k < kOrdItems; ++k) {
    const int i = base + k * kOrdThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(key[i] >> shift) & 0xFFu], 1u);
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

// stable scatter of block b: warp w owns the contiguous run [w*256, (w+1)*256) of the block
__global__ void __launch_bounds__(kOrdThreads) k_rs_scatter(const uint32_t* __restrict__ kin,
                                                            const uint32_t* __restrict__ vin, int n, int shift,
                                                            const uint32_t* __restrict__ gbase, int nb,
                                                            uint32_t* __restrict__ kout, uint32_t* __restrict__ vout) {
  __shared__ uint32_t wcnt[kOrdWarps][256];
  __shared__ uint32_t dbase[256];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (int d = lane; d < 256; d += 32) wcnt[w][d] = 0u;
  __syncwarp();
  const int base = blockIdx.x * kOrdBlock + w * (kOrdBlock / kOrdWarps);
  uint32_t kk[kOrdItems], vv[kOrdItems], rk[kOrdItems];
#pragma unroll
  for (int c = 0; c < kOrdItems; ++c) {
    const int i = base + c * 32 + lane;
    const bool ok = i < n;
    kk[c] = ok ? kin[i] : 0u;
    vv[c] = ok ? vin[i] : 0u;
    const uint32_t d = ok ? (kk[c] >> shift) & 0xFFu : 0x100u + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = ok ? wcnt[w][d] : 0u;
    rk[c] = before + __popc(peers & lt);
    __syncwarp();
    if (ok && (31 - __clz(peers)) == lane) wcnt[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {  // per digit: exclusive prefix over the warps, plus the block's global base
    const int d = tid;
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < kOrdWarps; ++ww) {
      const uint32_t c = wcnt[ww][d];
      wcnt[ww][d] = run;
      run += c;
    }
    dbase[d] = gbase[(size_t)d * nb + blockIdx.x];
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < kOrdItems; ++c) {
    const int i = base + c * 32 + lane;
    if (i < n) {
      const uint32_t d = (kk[c] >> shift) & 0xFFu;
      const uint32_t o = dbase[d] + wcnt[w][d] + rk[c];
      kout[o] = kk[c];
      vout[o] = vv[c];
    }
  }
}

static inline size_t al256(size_t x) { return (x + 255) / 256 * 256; }

struct OrderWS {
  int* bb;
  uint32_t *k0, *v0, *k1, *v1, *hist, *gbase;
  void* scan_ws;
  size_t total;
};

static OrderWS carve_order(int n, char* base) {
  OrderWS w{};
  const int nb = (n + kOrdBlock - 1) / kOrdBlock;
  size_t o = 0;
  auto take = [&](size_t b) -> char* {
    char* p = base ? base + o : nullptr;
    o += al256(b);
    return p;
  };
  w.bb = (int*)take(6 * sizeof(int));
  w.k0 = (uint32_t*)take((size_t)n * 4);
  w.v0 = (uint32_t*)take((size_t)n * 4);
  w.k1 = (uint32_t*)take((size_t)n * 4);
  w.v1 = (uint32_t*)take((size_t)n * 4);
  w.hist = (uint32_t*)take((size_t)256 * nb * 4);
  w.gbase = (uint32_t*)take((size_t)256 * nb * 4);
  w.scan_ws = take(scan_workspace_size((size_t)256 * nb));
  w.total = o;
  return w;
}

size_t morton_workspace_size(int n) { return carve_order(max(n, 1), nullptr).total; }

cudaError_t launch_morton_order(const float* pos, const uint8_t* flags, int n, uint32_t* perm, void* ws,
                                cudaStream_t s) {
  if (n <= 0) return cudaGetLastError();
  OrderWS w = carve_order(n, static_cast<char*>(ws));
  const int nb = (n + kOrdBlock - 1) / kOrdBlock;
  k_bbox_init<<<1, 32, 0, s>>>(w.bb);
  k_bbox<<<min((n + 255) / 256, 148 * 2), 256, 0, s>>>(pos, flags, n, w.bb);
  k_morton<<<(n + 255) / 256, 256, 0, s>>>(pos, flags, n, w.bb, w.k0, w.v0);
  note_launch(3);
  uint32_t* kb[2] = {w.k0, w.k1};
  uint32_t* vb[2] = {w.v0, w.v1};
  int cur = 0;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 8 * pass;
    k_rs_hist<<<nb, kOrdThreads, 0, s>>>(kb[cur], n, shift, w.hist, nb);
    note_launch();
    cudaError_t e = launch_scan(w.hist, w.gbase, (size_t)256 * nb, nullptr, w.scan_ws, s);
    if (e != cudaSuccess) return e;
    // the last pass writes the permutation straight into the caller's buffer
    uint32_t* vdst = pass == 3 ? perm : vb[cur ^ 1];
    k_rs_scatter<<<nb, kOrdThreads, 0, s>>>(kb[cur], vb[cur], n, shift, w.gbase, nb, kb[cur ^ 1], vdst);
    note_launch();
    cur ^= 1;
  }
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_gather_rows16(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                       const uint32_t* __restrict__ perm, int n, int vec_per_row) {
  const size_t e = (size_t)blockIdx.x * 256 + threadIdx.x;
  if (e >= (size_t)n * vec_per_row) return;
  const size_t r = e / vec_per_row, c = e - r * vec_per_row;
  dst[e] = src[(size_t)perm[r] * vec_per_row + c];
}

__global__ void __launch_bounds__(256) k_gather_rows4(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                                      const uint32_t* __restrict__ perm, int n, int w_per_row) {
  const size_t e = (size_t)blockIdx.x * 256 + threadIdx.x;
  if (e >= (size_t)n * w_per_row) return;
  const size_t r = e / w_per_row, c = e - r * w_per_row;
  dst[e] = src[(size_t)perm[r] * w_per_row + c];
}

__global__ void __launch_bounds__(256) k_gather_rows1(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                      const uint32_t* __restrict__ perm, int n, int row_bytes) {
  const size_t e = (size_t)blockIdx.x * 256 + threadIdx.x;
  if (e >= (size_t)n * row_bytes) return;
  const size_t r = e / row_bytes, c = e - r * row_bytes;
  dst[e] = src[(size_t)perm[r] * row_bytes + c];
}

cudaError_t launch_gather_rows(const void* src, void* dst, const uint32_t* perm, int n, int row_bytes,
                               cudaStream_t s) {
  if (n <= 0) return cudaGetLastError();
  const uintptr_t a = (uintptr_t)src | (uintptr_t)dst;
  if (row_bytes % 16 == 0 && a % 16 == 0) {
    const size_t tot = (size_t)n * (row_bytes / 16);
    k_gather_rows16<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((const uint4*)src, (uint4*)dst, perm, n, row_bytes / 16);
  } else if (row_bytes % 4 == 0 && a % 4 == 0) {
    const size_t tot = (size_t)n * (row_bytes / 4);
    k_gather_rows4<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((const uint32_t*)src, (uint32_t*)dst, perm, n,
                                                                  row_bytes / 4);
  } else {
    const size_t tot = (size_t)n * row_bytes;
    k_gather_rows1<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, perm, n, row_bytes);
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtgs
