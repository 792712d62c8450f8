// sort.cu — A2: tile binning and the hand-written radix sort (O8, readings R7, R8, R15).
//
//  1. k_bin_count    per Gaussian: #kept tiles its rect covers; block counts of Gaussians with >= 1
//  2. scan           block offsets;            3. k_compact  stable compaction (key = z bits, val = gid)
//  4. 4 x LSD radix passes on (z bits, gid), 8-bit digits  -> depth order, ties by gid (stability)
//  5. k_gather_cnt + scan -> instance offsets in depth order; total I
//  6. k_emit         (tile, gid) instances in depth order
//  7. 2+ x LSD radix passes on the tile id (stable) -> (tile, z, gid) order;  8. k_tile_range
// Device-side counts (m Gaussians, I instances) are read by the kernels, so nothing syncs.
#include "common.cuh"
#include "internal.h"

namespace rtgs {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanChunk = kScanThreads * kScanItems;  // 2048
constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;  // 4096 keys per CTA
constexpr int kRadixWarps = kRadixThreads / 32;

static inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------------------------------------------
// generic exclusive scan (3 kernels: chunk sums, scan of sums in one CTA, down-sweep)
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* __restrict__ in, size_t len,
                                                              uint32_t* __restrict__ sums) {
  __shared__ uint32_t sh[33];
  const size_t base = (size_t)blockIdx.x * kScanChunk;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const size_t i = base + (size_t)k * kScanThreads + threadIdx.x;
    if (i < len) s += in[i];
  }
  uint32_t tot;
  block_excl_scan(s, sh, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_top(uint32_t* sums, int nsum, uint32_t* total) {
  __shared__ uint32_t sh[33];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b = 0; b < nsum; b += 1024) {
    const int i = b + threadIdx.x;
    const uint32_t v = i < nsum ? sums[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, sh, &tot);
    if (i < nsum) sums[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t* __restrict__ in, size_t len,
                                                            const uint32_t* __restrict__ sums,
                                                            uint32_t* __restrict__ out) {
  __shared__ uint32_t sh[33];
  // blocked arrangement: thread t owns items [t*8, t*8+8) of the chunk
  const size_t base = (size_t)blockIdx.x * kScanChunk + (size_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (base + k < len) ? in[base + k] : 0u;
    s += v[k];
  }
  uint32_t tot;
  uint32_t run = block_excl_scan(s, sh, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < len) out[base + k] = run;
    run += v[k];
  }
}

size_t scan_workspace_size(size_t len) { return align_up(((len + kScanChunk - 1) / kScanChunk + 1) * 4); }

cudaError_t launch_scan(const uint32_t* in, uint32_t* out, size_t len, uint32_t* total, void* ws, cudaStream_t s) {
  const int nb = (int)((len + kScanChunk - 1) / kScanChunk);
  uint32_t* sums = static_cast<uint32_t*>(ws);
  if (nb == 0) {
    if (total) cudaMemsetAsync(total, 0, 4, s);
    return cudaGetLastError();
  }
  k_scan_reduce<<<nb, kScanThreads, 0, s>>>(in, len, sums);
  k_scan_top<<<1, 1024, 0, s>>>(sums, nb, total);
  k_scan_down<<<nb, kScanThreads, 0, s>>>(in, len, sums, out);
  note_launch(3);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// LSD radix sort pass on (key, value) u32 pairs, count read from the device.
// Stability: CTA b owns keys [b*4096, (b+1)*4096); warp w owns a contiguous 512-key run of it,
// processed in 16 rounds of 32 lanes, so (warp, round, lane) order == input order.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const uint32_t* __restrict__ keys,
                                                              const uint32_t* __restrict__ count, int shift,
                                                              int bits, uint32_t* __restrict__ hist, int nblocks) {
  __shared__ uint32_t h[256];
  const uint32_t n = *count;
  const int ndig = 1 << bits;
  for (int d = threadIdx.x; d < 256; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * kRadixTile;
  if (base < n) {
    const uint32_t mask = (uint32_t)ndig - 1u;
#pragma unroll 4
    for (int k = 0; k < kRadixItems; ++k) {
      const size_t i = base + (size_t)k * kRadixThreads + threadIdx.x;
      if (i < n) atomicAdd(&h[(keys[i] >> shift) & mask], 1u);
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < ndig; d += blockDim.x) hist[(size_t)d * nblocks + blockIdx.x] = h[d];
}

__global__ void __launch_bounds__(kRadixThreads) k_radix_scatter(const uint32_t* __restrict__ kin,
                                                                 const uint32_t* __restrict__ vin,
                                                                 uint32_t* __restrict__ kout,
                                                                 uint32_t* __restrict__ vout,
                                                                 const uint32_t* __restrict__ count, int shift,
                                                                 int bits, const uint32_t* __restrict__ offs,
                                                                 int nblocks) {
  __shared__ uint32_t wcnt[kRadixWarps][256];
  __shared__ uint32_t gbase[256];
  const uint32_t n = *count;
  const size_t base = (size_t)blockIdx.x * kRadixTile;
  if (base >= n) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ndig = 1 << bits;
  const uint32_t mask = (uint32_t)ndig - 1u;
  for (int d = threadIdx.x; d < kRadixWarps * 256; d += blockDim.x) (&wcnt[0][0])[d] = 0;
  for (int d = threadIdx.x; d < ndig; d += blockDim.x) gbase[d] = offs[(size_t)d * nblocks + blockIdx.x];
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t key[kRadixItems], val[kRadixItems], rank[kRadixItems];
  const size_t wbase = base + (size_t)w * 32 * kRadixItems;
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const size_t i = wbase + (size_t)r * 32 + lane;
    const bool ok = i < n;
    key[r] = ok ? kin[i] : 0u;
    val[r] = ok ? vin[i] : 0u;
    const uint32_t d = ok ? ((key[r] >> shift) & mask) : 0x1000u;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = ok ? wcnt[w][d] : 0u;
    rank[r] = ok ? (before + __popc(peers & lt)) : 0xFFFFFFFFu;
    __syncwarp();
    if (ok && (31 - __clz(peers)) == lane) wcnt[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix over warps for each digit
  for (int d = threadIdx.x; d < ndig; d += blockDim.x) {
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < kRadixWarps; ++ww) {
      const uint32_t t = wcnt[ww][d];
      wcnt[ww][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    if (rank[r] != 0xFFFFFFFFu) {
      const uint32_t d = (key[r] >> shift) & mask;
      const uint32_t dst = gbase[d] + wcnt[w][d] + rank[r];
      kout[dst] = key[r];
      vout[dst] = val[r];
    }
  }
}

struct RadixWS {
  uint32_t* hist;   // [256 * nblocks]
  uint32_t* offs;   // [256 * nblocks]
  void* scan_ws;
};

// sorts (k0, v0) in place on `bits` low-order key bits starting at bit 0 (`bits` <= 32), using
// (k1, v1) as ping-pong; an even number of passes so the result lands back in (k0, v0).
static cudaError_t radix_sort(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, const uint32_t* count,
                              size_t max_n, int bits, const RadixWS& ws, cudaStream_t s) {
  int passes = (bits + 7) / 8;
  if (passes < 2) passes = 2;
  if (passes & 1) passes += 1;
  const int nblocks = (int)((max_n + kRadixTile - 1) / kRadixTile);
  if (nblocks == 0) return cudaSuccess;
  int shift = 0;
  for (int p = 0; p < passes; ++p) {
    const int remaining = passes - p;
    const int bits_left = bits - shift;
    int b = (bits_left + remaining - 1) / remaining;
    if (b > 8) b = 8;
    if (b < 0) b = 0;
    const uint32_t* ki = (p & 1) ? k1 : k0;
    const uint32_t* vi = (p & 1) ? v1 : v0;
    uint32_t* ko = (p & 1) ? k0 : k1;
    uint32_t* vo = (p & 1) ? v0 : v1;
    k_radix_hist<<<nblocks, kRadixThreads, 0, s>>>(ki, count, shift, b, ws.hist, nblocks);
    note_launch();
    cudaError_t e = launch_scan(ws.hist, ws.offs, (size_t)(1 << b) * nblocks, nullptr, ws.scan_ws, s);
    if (e != cudaSuccess) return e;
    k_radix_scatter<<<nblocks, kRadixThreads, 0, s>>>(ki, vi, ko, vo, count, shift, b, ws.offs, nblocks);
    note_launch();
    shift += b;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// binning kernels
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ bool rect_tiles(uint2 r, int& tx0, int& ty0, int& tx1, int& ty1) {
  const int x0 = (int)(short)(r.x & 0xFFFF), y0 = (int)(short)(r.x >> 16);
  const int x1 = (int)(short)(r.y & 0xFFFF), y1 = (int)(short)(r.y >> 16);
  if (x0 > x1 || y0 > y1) return false;
  tx0 = x0 / kTile; ty0 = y0 / kTile; tx1 = x1 / kTile; ty1 = y1 / kTile;
  return true;
}

__global__ void __launch_bounds__(256) k_bin_count(const uint32_t* __restrict__ zkey, const uint2* __restrict__ rect,
                                                   const uint8_t* __restrict__ keep, int n, int TX,
                                                   uint32_t* __restrict__ cnt, uint32_t* __restrict__ blk) {
  __shared__ uint32_t sh[33];
  const int i = blockIdx.x * 256 + threadIdx.x;
  uint32_t c = 0;
  if (i < n && zkey[i] != 0xFFFFFFFFu) {
    int tx0, ty0, tx1, ty1;
    if (rect_tiles(rect[i], tx0, ty0, tx1, ty1)) {
      if (!keep) {
        c = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
      } else {
        for (int ty = ty0; ty <= ty1; ++ty)
          for (int tx = tx0; tx <= tx1; ++tx) c += keep[ty * TX + tx] ? 1u : 0u;
      }
    }
  }
  if (i < n) cnt[i] = c;
  uint32_t tot;
  block_excl_scan(c ? 1u : 0u, sh, &tot);
  if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(256) k_compact(const uint32_t* __restrict__ zkey, const uint32_t* __restrict__ cnt,
                                                 int n, const uint32_t* __restrict__ blk_off,
                                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  __shared__ uint32_t sh[33];
  const int i = blockIdx.x * 256 + threadIdx.x;
  const bool f = i < n && cnt[i] > 0;
  uint32_t tot;
  const uint32_t r = block_excl_scan(f ? 1u : 0u, sh, &tot);
  if (f) {
    const uint32_t p = blk_off[blockIdx.x] + r;
    keys[p] = zkey[i];
    vals[p] = (uint32_t)i;
  }
}

__global__ void __launch_bounds__(256) k_gather_cnt(const uint32_t* __restrict__ vals, const uint32_t* __restrict__ cnt,
                                                    const uint32_t* __restrict__ m_ptr, int n,
                                                    uint32_t* __restrict__ cs) {
  const int j = blockIdx.x * 256 + threadIdx.x;
  if (j < n) cs[j] = (uint32_t)j < *m_ptr ? cnt[vals[j]] : 0u;
}

__global__ void __launch_bounds__(256) k_emit(const uint32_t* __restrict__ vals, const uint32_t* __restrict__ off,
                                              const uint32_t* __restrict__ m_ptr, const uint2* __restrict__ rect,
                                              const uint8_t* __restrict__ keep, int TX, uint32_t cap,
                                              uint32_t* __restrict__ ikey, uint32_t* __restrict__ ival) {
  const uint32_t j = blockIdx.x * 256 + threadIdx.x;
  if (j >= *m_ptr) return;
  const uint32_t g = vals[j];
  uint32_t o = off[j];
  int tx0, ty0, tx1, ty1;
  if (!rect_tiles(rect[g], tx0, ty0, tx1, ty1)) return;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      const int t = ty * TX + tx;
      if (keep && !keep[t]) continue;
      if (o < cap) {
        ikey[o] = (uint32_t)t;
        ival[o] = g;
      }
      ++o;
    }
}

__global__ void k_finalize_count(const uint32_t* __restrict__ total, uint32_t cap, uint32_t* __restrict__ n_inst,
                                 uint32_t* __restrict__ n_live) {
  const uint32_t I = *total;
  *n_inst = I;
  *n_live = I < cap ? I : cap;
}

__global__ void __launch_bounds__(256) k_tile_range(const uint32_t* __restrict__ ikey, const uint32_t* __restrict__ n_live,
                                                    uint2* __restrict__ range) {
  const uint32_t i = blockIdx.x * 256 + threadIdx.x;
  const uint32_t n = *n_live;
  if (i >= n) return;
  const uint32_t t = ikey[i];
  if (i == 0 || ikey[i - 1] != t) range[t].x = i;
  if (i == n - 1 || ikey[i + 1] != t) range[t].y = i + 1;
}

// ------------------------------------------------------------------------------------------------
struct BinWS {
  uint32_t *cnt, *blk, *blk_off, *keys_a, *vals_a, *keys_b, *vals_b, *cs, *off, *ik_a, *ik_b, *iv_b;
  uint32_t *m, *total, *n_live;
  RadixWS rw;
  void* scan_ws;
};

static size_t carve(int n, const rtgs_camera& cam, uint32_t cap, BinWS* w, char* base) {
  (void)cam;
  size_t o = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + o : nullptr;
    o += align_up(bytes);
    return p;
  };
  const size_t N = (size_t)(n > 0 ? n : 1);
  const size_t nblk = (N + 255) / 256;
  const size_t maxn = N > cap ? N : (size_t)cap;
  const size_t rblocks = (maxn + kRadixTile - 1) / kRadixTile;
  BinWS t;
  t.cnt = (uint32_t*)take(N * 4);
  t.blk = (uint32_t*)take(nblk * 4);
  t.blk_off = (uint32_t*)take(nblk * 4);
  t.keys_a = (uint32_t*)take(N * 4);
  t.vals_a = (uint32_t*)take(N * 4);
  t.keys_b = (uint32_t*)take(N * 4);
  t.vals_b = (uint32_t*)take(N * 4);
  t.cs = (uint32_t*)take(N * 4);
  t.off = (uint32_t*)take(N * 4);
  t.ik_a = (uint32_t*)take((size_t)cap * 4 + 4);
  t.ik_b = (uint32_t*)take((size_t)cap * 4 + 4);
  t.iv_b = (uint32_t*)take((size_t)cap * 4 + 4);
  t.m = (uint32_t*)take(4);
  t.total = (uint32_t*)take(4);
  t.n_live = (uint32_t*)take(4);
  t.rw.hist = (uint32_t*)take(256 * rblocks * 4);
  t.rw.offs = (uint32_t*)take(256 * rblocks * 4);
  const size_t scan_len = 256 * rblocks > maxn ? 256 * rblocks : maxn;
  t.scan_ws = take(scan_workspace_size(scan_len));
  t.rw.scan_ws = t.scan_ws;
  if (w) *w = t;
  return o;
}

size_t bin_workspace_size(int n, const rtgs_camera& cam, uint32_t capacity) {
  return carve(n, cam, capacity, nullptr, nullptr);
}

cudaError_t launch_bin(const rtgs_projected& proj, int n, const rtgs_camera& cam, const uint8_t* keep,
                       const rtgs_bins& out, void* ws, cudaStream_t s) {
  const CamK k = make_cam(cam);
  const int T = k.TX * k.TY;
  BinWS w;
  carve(n, cam, out.capacity, &w, static_cast<char*>(ws));
  cudaMemsetAsync(out.tile_range, 0, (size_t)T * 8, s);
  if (n == 0) {
    cudaMemsetAsync(out.n_instances, 0, 4, s);
    return cudaGetLastError();
  }
  const int nblk = (n + 255) / 256;
  const uint2* rect = reinterpret_cast<const uint2*>(proj.rect);
  k_bin_count<<<nblk, 256, 0, s>>>(proj.zkey, rect, keep, n, k.TX, w.cnt, w.blk);
  note_launch();
  cudaError_t e = launch_scan(w.blk, w.blk_off, nblk, w.m, w.scan_ws, s);
  if (e) return e;
  k_compact<<<nblk, 256, 0, s>>>(proj.zkey, w.cnt, n, w.blk_off, w.keys_a, w.vals_a);
  note_launch();
  e = radix_sort(w.keys_a, w.vals_a, w.keys_b, w.vals_b, w.m, (size_t)n, 32, w.rw, s);
  if (e) return e;
  k_gather_cnt<<<nblk, 256, 0, s>>>(w.vals_a, w.cnt, w.m, n, w.cs);
  note_launch();
  e = launch_scan(w.cs, w.off, (size_t)n, w.total, w.scan_ws, s);
  if (e) return e;
  k_finalize_count<<<1, 1, 0, s>>>(w.total, out.capacity, out.n_instances, w.n_live);
  k_emit<<<nblk, 256, 0, s>>>(w.vals_a, w.off, w.m, rect, keep, k.TX, out.capacity, w.ik_a, out.sorted_gid);
  note_launch(2);
  int tbits = 0;
  while ((1 << tbits) < T) ++tbits;
  e = radix_sort(w.ik_a, out.sorted_gid, w.ik_b, w.iv_b, w.n_live, (size_t)out.capacity, tbits, w.rw, s);
  if (e) return e;
  const int iblk = (int)((out.capacity + 255) / 256);
  if (iblk) {
    k_tile_range<<<iblk, 256, 0, s>>>(w.ik_a, w.n_live, reinterpret_cast<uint2*>(out.tile_range));
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace rtgs
