// sort.cu — A2: tile binning with a hand-written per-tile LSD radix sort (O8, readings R7,
// R8, R15).
//
// B200 design: the C3 frame has ~1.5M instances over 3,225 tiles (~480 per tile), so instead of a
// device-wide sort of 64-bit tile|depth keys (3DGS) every tile's list is sorted inside ONE CTA in
// shared memory:
//   1. k_tile_count   per Gaussian, per kept tile of its rect: atomicAdd(tile_count[t])
//   2. k_tile_offsets one CTA: exclusive scan of the counts -> tile_range, n_instances
//   3. k_emit         per Gaussian, per kept tile: slot = atomicAdd(cursor[t]) (cursor = the tile start) and store
//                     the 64-bit pair (zkey << 32 | gid)   (order inside a tile still arbitrary)
//   4. k_tile_sort    one CTA per tile: key' = ((zkey - zmin) << gid_bits) | gid, stable LSD radix
//                     sort with 8-bit digits (warp match_any ranking) on the depth bits that vary
//                     (~3 passes), runs of equal depth then put in gid order; in shared memory
//                     (global-memory ping-pong for tiles above kSortCap); write gids.
// The output is the unique (tile, zkey bits, gid) order, so it is deterministic and bit-exact with
// the oracle although the emission order is not.
#include "common.cuh"
#include "internal.h"
#ifdef RTGS_DEBUG
#include <cassert>
#define RTGS_ASSERT(c) assert(c)
#else
#define RTGS_ASSERT(c)
#endif

namespace rtgs {

// sticky CAPACITY flag: set on the device by any binning whose instance count exceeds
// its capacity (the outputs were truncated: memory-safe but invalid); read and cleared by
// rtgs_check_device_flags, so the iteration itself stays free of host synchronisation
__device__ uint32_t g_capacity_flag = 0u;

uint32_t* capacity_flag_ptr() {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_capacity_flag);
  return static_cast<uint32_t*>(p);
}

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanChunk = kScanThreads * kScanItems;  // 2048
#ifndef RTGS_SORT_THREADS
#define RTGS_SORT_THREADS 256
#endif
constexpr int kSortThreads = RTGS_SORT_THREADS;  // 128 or 256 (swept)
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortCap = 1024;  // tile lists up to this length are sorted in shared memory

static inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------------------------------------------
// generic exclusive scan (3 kernels: chunk sums, scan of sums in one CTA, down-sweep); used by A7
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

// short arrays (per-block counts, <= kScanSmall): one CTA, 1024 values per pass, one launch
constexpr size_t kScanSmall = 16384;
__global__ void __launch_bounds__(1024) k_scan_small(const uint32_t* __restrict__ in, int len,
                                                     uint32_t* __restrict__ out, uint32_t* total) {
  __shared__ uint32_t sh[33];
  uint32_t carry = 0;
  for (int b = 0; b < len; b += 1024) {
    const int i = b + threadIdx.x;
    const uint32_t v = i < len ? in[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, sh, &tot);
    if (i < len) out[i] = ex + carry;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

size_t scan_workspace_size(size_t len) { return align_up(((len + kScanChunk - 1) / kScanChunk + 1) * 4); }

cudaError_t launch_scan(const uint32_t* in, uint32_t* out, size_t len, uint32_t* total, void* ws, cudaStream_t s) {
  const int nb = (int)((len + kScanChunk - 1) / kScanChunk);
  uint32_t* sums = static_cast<uint32_t*>(ws);
  if (nb == 0) {
    if (total) cudaMemsetAsync(total, 0, 4, s);
    return cudaGetLastError();
  }
  if (len <= kScanSmall) {
    k_scan_small<<<1, 1024, 0, s>>>(in, (int)len, out, total);
    note_launch();
    return cudaGetLastError();
  }
  k_scan_reduce<<<nb, kScanThreads, 0, s>>>(in, len, sums);
  k_scan_top<<<1, 1024, 0, s>>>(sums, nb, total);
  k_scan_down<<<nb, kScanThreads, 0, s>>>(in, len, sums, out);
  note_launch(3);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// binning
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ bool rect_tiles(uint2 r, int& tx0, int& ty0, int& tx1, int& ty1) {
  const int x0 = (int)(short)(r.x & 0xFFFF), y0 = (int)(short)(r.x >> 16);
  const int x1 = (int)(short)(r.y & 0xFFFF), y1 = (int)(short)(r.y >> 16);
  if (x0 > x1 || y0 > y1) return false;
  // (visible rects are clamped to the image: coordinates >= 0, so the division is a shift)
  tx0 = (int)((uint32_t)x0 / kTile); ty0 = (int)((uint32_t)y0 / kTile);
  tx1 = (int)((uint32_t)x1 / kTile); ty1 = (int)((uint32_t)y1 / kTile);
  return true;
}

// REP: replicated counters (kRep for the whole map's binning; kSubRep for the small unstable subset,
// whose atomics contend less, so its single-CTA scans read fewer counters)
#ifndef RTGS_SUBREP
#define RTGS_SUBREP 1
#endif
constexpr int kSubRep = RTGS_SUBREP;
template <int REP>
__global__ void __launch_bounds__(256) k_tile_count(const uint32_t* __restrict__ zkey, const uint2* __restrict__ rect,
                                                    const uint8_t* __restrict__ keep, int n, int TX, int T,
                                                    uint32_t* __restrict__ cnt) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  cnt += (size_t)(blockIdx.x & (REP - 1)) * T;
  uint32_t z = 0xFFFFFFFFu;
  uint2 rc = make_uint2(1u, 0u);
  if (i < n) {
    z = zkey[i];
    rc = rect[i];  // both loads in flight together
  }
  int tx0 = 0, ty0 = 0, tx1 = -1, ty1 = -1;
  const bool vis = i < n && z != 0xFFFFFFFFu && rect_tiles(rc, tx0, ty0, tx1, ty1);
  const int w = tx1 - tx0 + 1, nt = vis ? w * (ty1 - ty0 + 1) : 0;
  tile_count_agg(cnt, nt, w, tx0, ty0, TX, keep);
}

// one CTA: tile_range[t] = [start, start + count) (clamped to the capacity), n_instances, and the
// start of every counter replica inside its tile: start[r][t] = start(t) + sum_{r' < r} cnt[r'][t].
// Passes of kOffChunk tiles: coalesced counter loads (thread owns tiles b + k*1024 + tid), per-tile
// sums through shared memory to a blocked scan (thread owns 4 consecutive tiles), coalesced stores.
constexpr int kOffTiles = 4;
constexpr int kOffChunk = 1024 * kOffTiles;

// exclusive scan of s_v[0..kOffChunk) in place (blocked: thread owns 4 consecutive entries);
// returns the chunk total; ends with a barrier
__device__ __forceinline__ uint32_t chunk_scan(uint32_t* s_v, uint32_t* sh) {
  uint4 v = reinterpret_cast<uint4*>(s_v)[threadIdx.x];
  uint32_t tot;
  uint32_t ex = block_excl_scan(v.x + v.y + v.z + v.w, sh, &tot);
  uint4 o;
  o.x = ex; ex += v.x;
  o.y = ex; ex += v.y;
  o.z = ex; ex += v.z;
  o.w = ex;
  reinterpret_cast<uint4*>(s_v)[threadIdx.x] = o;
  __syncthreads();
  return tot;
}

template <int REP>
__global__ void __launch_bounds__(1024) k_tile_offsets(const uint32_t* __restrict__ cnt, int T, uint32_t cap,
                                                       uint32_t* __restrict__ start, uint2* __restrict__ range,
                                                       uint32_t* __restrict__ n_inst) {
  __shared__ __align__(16) uint32_t s_ex[kOffChunk];
  __shared__ uint32_t sh[33];
  uint32_t carry = 0;
  for (int b = 0; b < T; b += kOffChunk) {
    uint32_t c[kOffTiles][REP], tsum[kOffTiles];
#pragma unroll
    for (int k = 0; k < kOffTiles; ++k) {
      const int t = b + k * 1024 + threadIdx.x;
      tsum[k] = 0;
#pragma unroll
      for (int r = 0; r < REP; ++r) {
        c[k][r] = t < T ? cnt[(size_t)r * T + t] : 0u;
        tsum[k] += c[k][r];
      }
      s_ex[k * 1024 + threadIdx.x] = tsum[k];
    }
    __syncthreads();
    const uint32_t tot = chunk_scan(s_ex, sh);
#pragma unroll
    for (int k = 0; k < kOffTiles; ++k) {
      const int t = b + k * 1024 + threadIdx.x;
      if (t < T) {
        const uint32_t ex = s_ex[k * 1024 + threadIdx.x] + carry;
        uint32_t o = ex;
#pragma unroll
        for (int r = 0; r < REP; ++r) {
          start[(size_t)r * T + t] = o;
          o += c[k][r];
        }
        const uint32_t s0 = ex < cap ? ex : cap;
        const uint32_t e0 = ex + tsum[k] < cap ? ex + tsum[k] : cap;
        range[t] = make_uint2(tsum[k] ? s0 : 0u, tsum[k] ? e0 : 0u);
      }
    }
    carry += tot;
    __syncthreads();  // s_ex reused by the next chunk
  }
  if (threadIdx.x == 0) {
    *n_inst = carry;
    if (carry > cap) atomicOr(&g_capacity_flag, 1u);
  }
}

// STB (the FULL binning that also builds the f3 cache): the key's low word is (gid << 1) | stable,
// with the stable flag read here (coalesced, one byte per Gaussian) instead of gathered per instance
// after the sort; (gid << 1 | stable) orders exactly as gid
template <int REP, bool STB = false>
__global__ void __launch_bounds__(256) k_emit(const uint32_t* __restrict__ zkey, const uint2* __restrict__ rect,
                                              const uint8_t* __restrict__ keep, int n, int TX, int T,
                                              uint32_t* __restrict__ cursor, uint32_t cap,
                                              unsigned long long* __restrict__ keys,
                                              const uint8_t* __restrict__ flags = nullptr) {
  // cursor[r][t] starts at the replica's first slot of tile t (k_tile_offsets / k_merge_offsets write
  // it), so the atomic returns the absolute slot: no dependent load of a start array per instance
  const int i = blockIdx.x * 256 + threadIdx.x;
  const size_t rep = (size_t)(blockIdx.x & (REP - 1)) * T;  // same replica as k_tile_count
  cursor += rep;
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t z = 0xFFFFFFFFu;
  uint2 rc = make_uint2(1u, 0u);
  if (i < n) {
    z = zkey[i];
    rc = rect[i];
  }
  int tx0 = 0, ty0 = 0, tx1 = -1, ty1 = -1;
  const bool vis = i < n && z != 0xFFFFFFFFu && rect_tiles(rc, tx0, ty0, tx1, ty1);
  const uint32_t low = vis ? (STB ? (((uint32_t)i << 1) | ((flags[i] >> 1) & 1u)) : (uint32_t)i) : 0u;
  const unsigned long long k = ((unsigned long long)z << 32) | low;
  const int w = tx1 - tx0 + 1, nt = vis ? w * (ty1 - ty0 + 1) : 0;
  // the lanes' rect tiles expanded across the warp (warp_expand_tiles); lanes that land on the same
  // tile in a round (spatially coherent maps, rtgs_morton_order) share ONE cursor atomic (match_any
  // groups, the group's leader adds the group size and broadcasts the slot), instead of one atomic
  // round trip per instance
  const uint32_t klo = (uint32_t)k, khi = (uint32_t)(k >> 32);
  warp_expand_tiles(nt, w, tx0, ty0, TX, [&](int t, int o) {
    const unsigned long long ko = ((unsigned long long)__shfl_sync(0xffffffffu, khi, o) << 32) |
                                  __shfl_sync(0xffffffffu, klo, o);
    if (t >= 0 && keep && !keep[t]) t = -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, (uint32_t)t);
    const int leader = __ffs(peers) - 1;
    uint32_t off = 0u;
    if (t >= 0 && lane == leader) off = atomicAdd(&cursor[t], (uint32_t)__popc(peers));
    off = __shfl_sync(0xffffffffu, off, leader) + __popc(peers & lt);
    if (t >= 0 && off < cap) keys[off] = ko;
  });
}

// Stable LSD radix sort of n 64-bit keys by one CTA on key bits [lo, lo + nbits) (8-bit digits).
// Warp w owns the contiguous run [w*run, (w+1)*run) for ranking AND scattering, so the stable order
// is (warp, round, lane).  Key / rank buffers are shared memory (KeyPtr = shared pointers, inlined
// into LDS/STS) or global memory for oversized tiles.
__device__ __forceinline__ void cta_radix_sort(unsigned long long* A, unsigned long long* B, uint32_t* rank, int n,
                                               int lo, int nbits, uint32_t (*wcnt)[256], uint32_t* dstart,
                                               uint32_t* scan_sh, unsigned long long** out) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const int run = ((n + kSortWarps * 32 - 1) / (kSortWarps * 32)) * 32;  // contiguous keys per warp
  const int r0 = min(n, w * run), r1 = min(n, (w + 1) * run);
  for (int shift = lo; shift < lo + nbits; shift += 8) {
    for (int d = lane; d < 256; d += 32) wcnt[w][d] = 0;  // each warp clears its own counters
    __syncwarp();
    for (int base = r0; base < r1; base += 32) {
      const int i = base + lane;
      const bool ok = i < r1;
      const uint32_t d = ok ? (uint32_t)((A[i] >> shift) & 0xFFu) : 0x1000u;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t before = ok ? wcnt[w][d] : 0u;
      RTGS_ASSERT(!ok || d < 256);
      if (ok) rank[i] = before + __popc(peers & lt);
      __syncwarp();
      if (ok && (31 - __clz(peers)) == lane) wcnt[w][d] = before + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    {  // per digit: prefix over warps, then exclusive scan over digits (kDPT consecutive per thread)
      constexpr int kDPT = 256 / kSortThreads;
      uint32_t tot_d[kDPT], tsum = 0;
#pragma unroll
      for (int j = 0; j < kDPT; ++j) {
        const int d = tid * kDPT + j;
        uint32_t run_w = 0;
#pragma unroll
        for (int ww = 0; ww < kSortWarps; ++ww) {
          const uint32_t c = wcnt[ww][d];
          wcnt[ww][d] = run_w;
          run_w += c;
        }
        tot_d[j] = run_w;
        tsum += run_w;
      }
      uint32_t tot;
      uint32_t ex = block_excl_scan(tsum, scan_sh, &tot);
#pragma unroll
      for (int j = 0; j < kDPT; ++j) {
        dstart[tid * kDPT + j] = ex;
        ex += tot_d[j];
      }
    }
    __syncthreads();  // dstart written after the scan's own barriers
    for (int i = r0 + lane; i < r1; i += 32) {
      const unsigned long long k = A[i];
      const uint32_t d = (uint32_t)((k >> shift) & 0xFFu);
      RTGS_ASSERT(dstart[d] + wcnt[w][d] + rank[i] < (uint32_t)n);
      B[dstart[d] + wcnt[w][d] + rank[i]] = k;
    }
    __syncthreads();
    unsigned long long* t = A;
    A = B;
    B = t;
  }
  *out = A;
}

// MSD bucket sort of a tile list held in shared memory (the default for lists up to kSortCap).
// The keys are (zkey << 32 | low) and their unique ascending order is the (zkey, gid) order.  One
// pass distributes them over kBuckets buckets by the top bits of (zkey - zmin): each key takes its
// rank inside its bucket from a shared-memory atomic (an arbitrary order -- MSD needs no stability),
// and after a scan of the bucket counts lands at start[bucket] + rank.  Then every key moves to its
// bucket's start + the number of smaller keys in its bucket (a tile of ~700 keys spreads ~0.7 keys
// per bucket; crowded buckets are ranked by as many threads as they hold keys).  So the result is
// the same unique order as the LSD path, for a fraction of its instructions.  Returns false (nothing
// written) when some bucket holds more than kMaxBucket keys (depths piled up in one bucket range):
// the caller then runs the LSD sort.
#ifndef RTGS_MSD_BITS
#define RTGS_MSD_BITS 10  // (swept 9 / 10 / 11: 10)
#endif
constexpr int kBuckets = 1 << RTGS_MSD_BITS;
constexpr int kBPT = kBuckets / kSortThreads;  // buckets per thread
constexpr int kMaxBucket = 96;
static_assert(kBuckets * 4 <= kSortWarps * 256 * 4, "the bucket counters reuse wcnt");
__device__ __forceinline__ bool msd_bucket_sort(unsigned long long* A, unsigned long long* B, uint32_t* rk, int n,
                                                uint32_t z0, int zbits, uint32_t* cnt, uint32_t* scan_sh) {
  const int tid = threadIdx.x;
  const int sh = max(0, zbits - RTGS_MSD_BITS);  // the top bits of the depth range (kBuckets of them)
#pragma unroll
  for (int j = 0; j < kBPT; ++j) cnt[tid * kBPT + j] = 0u;
  __syncthreads();
  for (int i = tid; i < n; i += kSortThreads) {
    const uint32_t d = ((uint32_t)(A[i] >> 32) - z0) >> sh;
    rk[i] = atomicAdd(&cnt[d], 1u);
  }
  __syncthreads();
  uint32_t c[kBPT], tsum = 0, cmax = 0;
#pragma unroll
  for (int j = 0; j < kBPT; ++j) {
    c[j] = cnt[tid * kBPT + j];
    tsum += c[j];
    cmax = max(cmax, c[j]);
  }
  if (__syncthreads_or(cmax > (uint32_t)kMaxBucket)) return false;
  uint32_t tot;
  uint32_t st = block_excl_scan(tsum, scan_sh, &tot);
#pragma unroll
  for (int j = 0; j < kBPT; ++j) {
    cnt[tid * kBPT + j] = st;  // bucket start
    st += c[j];
  }
  __syncthreads();
  for (int i = tid; i < n; i += kSortThreads) {
    const unsigned long long k = A[i];
    const uint32_t d = ((uint32_t)(k >> 32) - z0) >> sh;
    B[cnt[d] + rk[i]] = k;
  }
  __syncthreads();
  // final place of each key: its bucket's start + the number of smaller keys in the bucket (keys are
  // unique: the low word holds the gid), one thread per key so a crowded bucket is ranked in parallel
  for (int i = tid; i < n; i += kSortThreads) {
    const unsigned long long k = B[i];
    const uint32_t d = ((uint32_t)(k >> 32) - z0) >> sh;
    const int lo = (int)cnt[d], hi = d + 1 < (uint32_t)kBuckets ? (int)cnt[d + 1] : n;
    int r = 0;
    for (int p = lo; p < hi; ++p) r += B[p] < k ? 1 : 0;
    A[lo + r] = k;
  }
  __syncthreads();
  return true;
}

// one tile's list: load, compress, depth-radix-sort, tie fix-up, write gids
__device__ __forceinline__ void sort_tile(const unsigned long long* __restrict__ seg, unsigned long long* A,
                                          unsigned long long* B, uint32_t* rk, int n, int gid_bits,
                                          uint32_t* __restrict__ out_gid, bool copy_in, uint32_t (*wcnt)[256],
                                          uint32_t* dstart, uint32_t* scan_sh, uint32_t* s_zmm) {
  const int tid = threadIdx.x;
  if (tid == 0) { s_zmm[0] = 0xFFFFFFFFu; s_zmm[1] = 0u; }
  __syncthreads();
  uint32_t zmin = 0xFFFFFFFFu, zmax = 0u;
  constexpr int LU = 4;  // list loads in flight per thread
  for (int i0 = tid; i0 < n; i0 += LU * kSortThreads) {
    unsigned long long k[LU];
#pragma unroll
    for (int u = 0; u < LU; ++u) {
      const int i = i0 + u * kSortThreads;
      k[u] = i < n ? seg[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < LU; ++u) {
      const int i = i0 + u * kSortThreads;
      if (i < n) {
        const uint32_t z = (uint32_t)(k[u] >> 32);
        zmin = min(zmin, z);
        zmax = max(zmax, z);
        if (copy_in) A[i] = k[u];
      }
    }
  }
  atomicMin(&s_zmm[0], zmin);
  atomicMax(&s_zmm[1], zmax);
  __syncthreads();
  const uint32_t z0 = s_zmm[0];
  const uint32_t zr = s_zmm[1] - z0;
  const int zbits = zr ? 32 - __clz(zr) : 0;
  if (copy_in && msd_bucket_sort(A, B, rk, n, z0, zbits, &wcnt[0][0], scan_sh)) {
    for (int i = tid; i < n; i += kSortThreads) out_gid[i] = (uint32_t)(A[i] & 0xFFFFFFFFull);
    return;
  }
  // compress: key' = ((z - zmin) << gid_bits) | gid  (order-preserving for (z, gid))
  for (int i = tid; i < n; i += kSortThreads) {
    const unsigned long long k = A[i];
    const unsigned long long zz = (unsigned long long)((uint32_t)(k >> 32) - z0);
    A[i] = (zz << gid_bits) | (k & 0xFFFFFFFFull);
  }
  __syncthreads();
  // radix-sort on the depth bits only (the emission order among equal depths is arbitrary) ...
  unsigned long long* res;
  cta_radix_sort(A, B, rk, n, gid_bits, zbits, wcnt, dstart, scan_sh, &res);
  // ... then put every run of equal depth into gid order.  Ties are common on fronto-parallel
  // surfaces (float32 depths of a wall collide), but runs are short: each run is insertion-sorted
  // by the thread at its start; a run longer than kMaxRun makes the CTA re-sort the whole list on
  // all bits (gid bits included), which gives the same unique (zkey, gid) order.
  constexpr int kMaxRun = 16;
  bool long_run = false;
  for (int i = tid; i < n; i += kSortThreads) {
    const unsigned long long zi = res[i] >> gid_bits;
    if ((i == 0 || (res[i - 1] >> gid_bits) != zi) && i + 1 < n && (res[i + 1] >> gid_bits) == zi) {
      int j = i + 1;
      while (j < n && j - i <= kMaxRun && (res[j] >> gid_bits) == zi) ++j;
      if (j - i > kMaxRun) {
        long_run = true;
      } else {
        for (int p = i + 1; p < j; ++p) {
          const unsigned long long k = res[p];
          int q = p - 1;
          while (q >= i && res[q] > k) { res[q + 1] = res[q]; --q; }
          res[q + 1] = k;
        }
      }
    }
  }
  if (__syncthreads_or(long_run)) {
    unsigned long long* other = (res == A) ? B : A;
    cta_radix_sort(res, other, rk, n, 0, zbits + gid_bits, wcnt, dstart, scan_sh, &res);
  }
  const unsigned long long gmask = (1ull << gid_bits) - 1ull;
  for (int i = tid; i < n; i += kSortThreads) out_gid[i] = (uint32_t)(res[i] & gmask);
}

// NEXT f3 fused into the FULL binning: ordered compaction of the tile's stable entries (flags bit 1)
// of the sorted list `g` [n] into csorted[base ...] (the cache lives in the FULL lists' index space,
// as k_cache_build); returns nothing, writes crange[tile] and adds to n_stable.
// The sorted entries arrive as (gid << 1) | stable (k_emit<REP, true>); they are decoded in place.
__device__ __forceinline__ void stable_compact(uint32_t* __restrict__ g, int n, uint32_t base,
                                               uint32_t* __restrict__ csorted, uint2* crange, int tile,
                                               uint32_t* __restrict__ n_stable, uint32_t* scan_sh) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t o = base;
  for (int b = 0; b < n; b += kSortThreads) {
    const int i = b + tid;
    uint32_t gi = 0;
    bool st = false;
    if (i < n) {
      const uint32_t f = g[i];
      gi = f >> 1;
      st = (f & 1u) != 0;
      g[i] = gi;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, st);
    if (lane == 0) scan_sh[w] = __popc(m);
    __syncthreads();
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < kSortWarps; ++k) {
      const uint32_t c = scan_sh[k];
      before += k < w ? c : 0u;
      tot += c;
    }
    if (st) csorted[o + before + __popc(m & ((1u << lane) - 1u))] = gi;
    o += tot;
    __syncthreads();  // scan_sh reused
  }
  if (tid == 0) {
    crange[tile] = make_uint2(base, o);
    if (n_stable && o > base) atomicAdd(n_stable, o - base);
  }
}

struct StableOut {  // NEXT f3 cache written by the FULL binning (flags NULL: none)
  const uint8_t* flags;
  uint32_t* csorted;
  uint2* crange;
  uint32_t* n_stable;
};

__global__ void __launch_bounds__(kSortThreads, 1536 / kSortThreads) k_tile_sort(const uint2* __restrict__ range,
                                                            unsigned long long* __restrict__ keys,
                                                            unsigned long long* __restrict__ tmp,
                                                            uint32_t* __restrict__ grank, int gid_bits,
                                                            uint32_t* __restrict__ sorted_gid, const StableOut so) {
  extern __shared__ __align__(16) unsigned long long s_keys[];  // [2 * kSortCap] keys + kSortCap ranks
  __shared__ uint32_t wcnt[kSortWarps][256];
  __shared__ uint32_t dstart[256];
  __shared__ uint32_t scan_sh[33];
  __shared__ uint32_t s_zmm[2];
  const uint2 rg = range[blockIdx.x];
  const int n = (int)(rg.y - rg.x);
  if (n <= 0) {
    if (so.flags && threadIdx.x == 0) so.crange[blockIdx.x] = make_uint2(rg.x, rg.x);
    return;
  }
  RTGS_ASSERT(rg.y >= rg.x);
  unsigned long long* seg = keys + rg.x;
  if (n == 1) {
    if (threadIdx.x == 0) {
      const uint32_t f = (uint32_t)(seg[0] & 0xFFFFFFFFull);
      const uint32_t g = so.flags ? f >> 1 : f;
      sorted_gid[rg.x] = g;
      if (so.flags) {
        const bool st = (f & 1u) != 0;
        if (st) so.csorted[rg.x] = g;
        so.crange[blockIdx.x] = make_uint2(rg.x, rg.x + (st ? 1u : 0u));
        if (st && so.n_stable) atomicAdd(so.n_stable, 1u);
      }
    }
    return;
  }
  if (n <= kSortCap) {  // shared-memory path: every buffer access below is LDS / STS
    sort_tile(seg, s_keys, s_keys + kSortCap, reinterpret_cast<uint32_t*>(s_keys + 2 * kSortCap), n, gid_bits,
              sorted_gid + rg.x, true, wcnt, dstart, scan_sh, s_zmm);
  } else {              // oversized tile: global-memory ping-pong (correct, slower)
    sort_tile(seg, seg, tmp + rg.x, grank + rg.x, n, gid_bits, sorted_gid + rg.x, false, wcnt, dstart, scan_sh,
              s_zmm);
  }
  if (so.flags) {
    __syncthreads();  // the sorted gids of this tile are written (read back through L1 / L2 below)
    stable_compact(sorted_gid + rg.x, n, rg.x, so.csorted, so.crange, blockIdx.x, so.n_stable, scan_sh);
  }
}

// ------------------------------------------------------------------------------------------------
// NEXT f3: stable-projection cache and the cached masked binning
// ------------------------------------------------------------------------------------------------
// one warp per tile: ordered compaction of the stable entries of the tile's FULL list, in place of
// the tile's full range (so no scan is needed)
__global__ void __launch_bounds__(256) k_cache_build(const uint2* __restrict__ frange,
                                                     const uint32_t* __restrict__ fsorted,
                                                     const uint8_t* __restrict__ flags, int T,
                                                     uint32_t* __restrict__ csorted, uint2* __restrict__ crange,
                                                     uint32_t* __restrict__ n_stable) {
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const uint2 rg = frange[t];
  uint32_t o = rg.x;
  for (uint32_t b = rg.x; b < rg.y; b += 32) {
    const uint32_t i = b + lane;
    uint32_t g = 0;
    bool st = false;
    if (i < rg.y) {
      g = fsorted[i];
      st = (flags[g] & 2u) != 0;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, st);
    if (st) csorted[o + __popc(m & ((1u << lane) - 1u))] = g;
    o += __popc(m);
  }
  if (lane == 0) {
    crange[t] = make_uint2(rg.x, o);
    if (n_stable && o > rg.x) atomicAdd(n_stable, o - rg.x);
  }
}

// one CTA, after k_tile_count of the subset: the subset's own ranges and replica starts (as
// k_tile_offsets) AND the merged output ranges, count(t) = keep[t] ? |stable(t)| + |subset(t)| : 0
template <int REP>
__global__ void __launch_bounds__(1024) k_merge_offsets(const uint32_t* __restrict__ cnt, const uint8_t* __restrict__ keep,
                                                        const uint2* __restrict__ crange, int T, uint32_t cap,
                                                        uint32_t* __restrict__ start, uint2* __restrict__ srange,
                                                        uint2* __restrict__ orange, uint32_t* __restrict__ n_inst) {
  __shared__ __align__(16) uint32_t s_ex[kOffChunk];
  __shared__ __align__(16) uint32_t s_ex2[kOffChunk];
  __shared__ uint32_t sh[33];
  uint32_t carry = 0, carry2 = 0;
  for (int b = 0; b < T; b += kOffChunk) {
    uint32_t c[kOffTiles][REP], tsum[kOffTiles], cl[kOffTiles];
#pragma unroll
    for (int k = 0; k < kOffTiles; ++k) {
      const int t = b + k * 1024 + threadIdx.x;
      tsum[k] = 0;
      cl[k] = 0;
      uint2 a = make_uint2(0u, 0u);
      uint8_t kp = 0;
      if (t < T) {
        a = crange[t];
        kp = keep[t];
      }
#pragma unroll
      for (int r = 0; r < REP; ++r) {
        c[k][r] = t < T ? cnt[(size_t)r * T + t] : 0u;
        tsum[k] += c[k][r];
      }
      cl[k] = kp ? (a.y - a.x) + tsum[k] : 0u;  // the subset was binned on kept tiles only
      s_ex[k * 1024 + threadIdx.x] = tsum[k];
      s_ex2[k * 1024 + threadIdx.x] = cl[k];
    }
    __syncthreads();
    const uint32_t tot = chunk_scan(s_ex, sh);
    const uint32_t tot2 = chunk_scan(s_ex2, sh);
#pragma unroll
    for (int k = 0; k < kOffTiles; ++k) {
      const int t = b + k * 1024 + threadIdx.x;
      if (t < T) {
        const uint32_t ex = s_ex[k * 1024 + threadIdx.x] + carry;
        const uint32_t ex2 = s_ex2[k * 1024 + threadIdx.x] + carry2;
        uint32_t o = ex;
#pragma unroll
        for (int r = 0; r < REP; ++r) {
          start[(size_t)r * T + t] = o;
          o += c[k][r];
        }
        srange[t] = make_uint2(min(ex, cap), min(ex + tsum[k], cap));  // subset keys: capacity entries
        const uint32_t s0 = ex2 < cap ? ex2 : cap;
        const uint32_t e0 = ex2 + cl[k] < cap ? ex2 + cl[k] : cap;
        orange[t] = make_uint2(cl[k] ? s0 : 0u, cl[k] ? e0 : 0u);
      }
    }
    carry += tot;
    carry2 += tot2;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *n_inst = carry2;
    if (carry2 > cap) atomicOr(&g_capacity_flag, 1u);
  }
}

// number of elements of the sorted key list k[0..n) that are < key (keys are distinct)
template <typename KeyAt>
__device__ __forceinline__ int rank_below(KeyAt k, int n, unsigned long long key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (k(mid) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Merge the cached stable list S (gids) and the sorted subset list U (rows) of one tile by
// (zkey bits, gid): element i of S lands at i + |{u in U : u < S_i}| and vice versa (keys distinct).
// Keys are ranked from the shared buffer sk when both lists fit, else fetched from global memory.
__device__ __forceinline__ void merge_tile(const uint32_t* __restrict__ S, int nS, const uint32_t* __restrict__ U,
                                           int nU, const uint32_t* __restrict__ zfull,
                                           const uint32_t* __restrict__ szkey, const int32_t* __restrict__ sgid,
                                           uint32_t o, uint32_t cap, uint32_t* __restrict__ out,
                                           unsigned long long* sk, int sk_cap) {
  auto keyS = [&](int i) {
    const uint32_t g = S[i];
    return ((unsigned long long)zfull[g] << 32) | g;
  };
  auto keyU = [&](int j) {
    const uint32_t r = U[j];
    return ((unsigned long long)szkey[r] << 32) | (uint32_t)sgid[r];
  };
  if (nS + nU <= sk_cap) {
    // key gathers 4 deep per thread (each key is two dependent loads: the id, then its zkey)
    constexpr int GU = 4;
    for (int i0 = threadIdx.x; i0 < nS + nU; i0 += GU * (int)blockDim.x) {
      uint32_t id[GU];
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int i = i0 + u * (int)blockDim.x;
        id[u] = i < nS ? S[i] : (i < nS + nU ? U[i - nS] : 0u);
      }
      uint32_t z[GU], lo[GU];
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int i = i0 + u * (int)blockDim.x;
        z[u] = i < nS ? zfull[id[u]] : (i < nS + nU ? szkey[id[u]] : 0u);
        lo[u] = i < nS ? id[u] : (i < nS + nU ? (uint32_t)sgid[id[u]] : 0u);
      }
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int i = i0 + u * (int)blockDim.x;
        if (i < nS + nU) sk[i] = ((unsigned long long)z[u] << 32) | lo[u];
      }
    }
    __syncthreads();
    const unsigned long long* kS = sk;
    const unsigned long long* kU = sk + nS;
    for (int i = threadIdx.x; i < nS; i += blockDim.x) {
      const uint32_t p = o + (uint32_t)(i + rank_below([&](int m) { return kU[m]; }, nU, kS[i]));
      if (p < cap) out[p] = S[i];
    }
    for (int j = threadIdx.x; j < nU; j += blockDim.x) {
      const uint32_t p = o + (uint32_t)(j + rank_below([&](int m) { return kS[m]; }, nS, kU[j]));
      if (p < cap) out[p] = 0x80000000u | U[j];
    }
  } else {  // long lists: keys fetched from global memory during the searches
    for (int i = threadIdx.x; i < nS; i += blockDim.x) {
      const uint32_t p = o + (uint32_t)(i + rank_below(keyU, nU, keyS(i)));
      if (p < cap) out[p] = S[i];
    }
    for (int j = threadIdx.x; j < nU; j += blockDim.x) {
      const uint32_t p = o + (uint32_t)(j + rank_below(keyS, nS, keyU(j)));
      if (p < cap) out[p] = 0x80000000u | U[j];
    }
  }
}

// one CTA per kept tile: sort the tile's subset instances (as k_tile_sort, rows as ids; the rows
// are in gid order, so (zkey, row) order is (zkey, gid) order), then merge them with the cached
// stable list into the output range.  Shared memory: the sort's key buffers, reused by the merge.
__global__ void __launch_bounds__(kSortThreads) k_sort_merge(const uint8_t* __restrict__ keep,
                                                             const uint2* __restrict__ srange,
                                                             unsigned long long* __restrict__ keys,
                                                             unsigned long long* __restrict__ tmp,
                                                             uint32_t* __restrict__ grank, int row_bits,
                                                             uint32_t* __restrict__ ssorted,
                                                             const uint2* __restrict__ crange,
                                                             const uint32_t* __restrict__ csorted,
                                                             const uint32_t* __restrict__ zfull,
                                                             const uint32_t* __restrict__ szkey,
                                                             const int32_t* __restrict__ sgid,
                                                             const uint2* __restrict__ orange, uint32_t cap,
                                                             uint32_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned long long s_keys[];  // [2 * kSortCap] keys + kSortCap ranks
  __shared__ uint32_t wcnt[kSortWarps][256];
  __shared__ uint32_t dstart[256];
  __shared__ uint32_t scan_sh[33];
  __shared__ uint32_t s_zmm[2];
  const int t = blockIdx.x;
  if (!keep[t]) return;
  const uint2 sr = srange[t], cr = crange[t];
  const int nU = (int)(sr.y - sr.x), nS = (int)(cr.y - cr.x);
  if (nS + nU == 0) return;
  unsigned long long* seg = keys + sr.x;
  if (nU == 1) {
    if (threadIdx.x == 0) ssorted[sr.x] = (uint32_t)(seg[0] & 0xFFFFFFFFull);
  } else if (nU > 1 && nU <= kSortCap) {
    sort_tile(seg, s_keys, s_keys + kSortCap, reinterpret_cast<uint32_t*>(s_keys + 2 * kSortCap), nU, row_bits,
              ssorted + sr.x, true, wcnt, dstart, scan_sh, s_zmm);
  } else if (nU > kSortCap) {
    sort_tile(seg, seg, tmp + sr.x, grank + sr.x, nU, row_bits, ssorted + sr.x, false, wcnt, dstart, scan_sh,
              s_zmm);
  }
  __syncthreads();  // sorted rows (global) visible to the whole CTA; shared buffers free again
  merge_tile(csorted + cr.x, nS, ssorted + sr.x, nU, zfull, szkey, sgid, orange[t].x, cap, out, s_keys,
             (int)(kSortCap * 5 / 2));
}

// ------------------------------------------------------------------------------------------------
struct BinWS {
  uint32_t *cnt, *cursor, *grank;
  unsigned long long *keys, *tmp;
};

static size_t carve(int n, const rtgs_camera& cam, uint32_t cap, BinWS* w, char* base) {
  (void)n;
  size_t o = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + o : nullptr;
    o += align_up(bytes);
    return p;
  };
  const CamK k = make_cam(cam);
  const size_t T = (size_t)k.TX * k.TY;
  BinWS t;
  t.cnt = (uint32_t*)take(kRep * T * 4);
  t.cursor = (uint32_t*)take(kRep * T * 4);  // written by the offsets kernels: each replica's first slot
  t.keys = (unsigned long long*)take((size_t)cap * 8 + 8);
  t.tmp = (unsigned long long*)take((size_t)cap * 8 + 8);
  t.grank = (uint32_t*)take((size_t)cap * 4 + 4);
  if (w) *w = t;
  return o;
}

size_t bin_workspace_size(int n, const rtgs_camera& cam, uint32_t capacity) {
  return carve(n, cam, capacity, nullptr, nullptr);
}

// offsets, emission and per-tile sort, once the replicated per-tile counts are in w.cnt
static cudaError_t bin_from_counts(const rtgs_projected& proj, int n, const CamK& k, const uint8_t* keep,
                                   const rtgs_bins& out, const BinWS& w, cudaStream_t s,
                                   const StableOut so = StableOut{nullptr, nullptr, nullptr, nullptr}) {
  const int T = k.TX * k.TY;
  const uint2* rect = reinterpret_cast<const uint2*>(proj.rect);
  const int nblk = (n + 255) / 256;
  k_tile_offsets<kRep><<<1, 1024, 0, s>>>(w.cnt, T, out.capacity, w.cursor, reinterpret_cast<uint2*>(out.tile_range),
                                    out.n_instances);
  note_launch();
  if (n > 0) {
    if (so.flags)
      k_emit<kRep, true><<<nblk, 256, 0, s>>>(proj.zkey, rect, keep, n, k.TX, T, w.cursor, out.capacity,
                                              w.keys, so.flags);
    else
      k_emit<kRep><<<nblk, 256, 0, s>>>(proj.zkey, rect, keep, n, k.TX, T, w.cursor, out.capacity, w.keys);
    note_launch();
    int gid_bits = 1;
    while (gid_bits < 32 && (1u << gid_bits) < (uint32_t)n) ++gid_bits;
    if (so.flags) ++gid_bits;  // the (gid << 1) | stable field
    const size_t smem = (size_t)kSortCap * (8 + 8 + 4);
    static std::atomic<uint64_t> attr_mask{0};
    if (first_on_device(attr_mask)) {
      cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    k_tile_sort<<<T, kSortThreads, smem, s>>>(reinterpret_cast<const uint2*>(out.tile_range), w.keys, w.tmp, w.grank,
                                              gid_bits, out.sorted_gid, so);
    note_launch();
  } else if (so.flags) {  // empty map: every cached tile range is empty
    cudaMemsetAsync(so.crange, 0, (size_t)T * sizeof(uint2), s);
  }
  return cudaGetLastError();
}

cudaError_t launch_bin(const rtgs_projected& proj, int n, const rtgs_camera& cam, const uint8_t* keep,
                       const rtgs_bins& out, void* ws, cudaStream_t s) {
  const CamK k = make_cam(cam);
  const int T = k.TX * k.TY;
  BinWS w;
  carve(n, cam, out.capacity, &w, static_cast<char*>(ws));
  cudaMemsetAsync(w.cnt, 0, (size_t)((char*)w.cursor - (char*)w.cnt), s);  // (the offsets write cursor)
  const uint2* rect = reinterpret_cast<const uint2*>(proj.rect);
  const int nblk = (n + 255) / 256;
  if (n > 0) {
    k_tile_count<kRep><<<nblk, 256, 0, s>>>(proj.zkey, rect, keep, n, k.TX, T, w.cnt);
    note_launch();
  }
  return bin_from_counts(proj, n, k, keep, out, w, s);
}

cudaError_t launch_project_bin(const rtgs_gaussians& g, const PoseF& pose, const rtgs_camera& cam,
                               const rtgs_projected& proj, const rtgs_bins& out, const rtgs_bins* cache, void* ws,
                               cudaStream_t s) {
  const CamK k = make_cam(cam);
  BinWS w;
  carve(g.n, cam, out.capacity, &w, static_cast<char*>(ws));
  cudaMemsetAsync(w.cnt, 0, (size_t)((char*)w.cursor - (char*)w.cnt), s);  // (the offsets write cursor)
  StableOut so{nullptr, nullptr, nullptr, nullptr};
  if (cache) {
    so = StableOut{g.flags, cache->sorted_gid, reinterpret_cast<uint2*>(cache->tile_range), cache->n_instances};
    if (cache->n_instances) cudaMemsetAsync(cache->n_instances, 0, 4, s);
  }
  const cudaError_t e = launch_project_count(g, pose, cam, proj, w.cnt, s);
  if (e != cudaSuccess) return e;
  return bin_from_counts(proj, g.n, k, nullptr, out, w, s, so);
}

cudaError_t launch_cache_build(const rtgs_bins& full, const uint8_t* flags, const rtgs_camera& cam,
                               const rtgs_bins& cache, cudaStream_t s) {
  const CamK k = make_cam(cam);
  const int T = k.TX * k.TY;
  if (cache.n_instances) cudaMemsetAsync(cache.n_instances, 0, 4, s);
  k_cache_build<<<(T + 7) / 8, 256, 0, s>>>(reinterpret_cast<const uint2*>(full.tile_range), full.sorted_gid, flags, T,
                                            cache.sorted_gid, reinterpret_cast<uint2*>(cache.tile_range),
                                            cache.n_instances);
  note_launch();
  return cudaGetLastError();
}

// workspace of the cached binning: the subset's own bins (sorted rows, ranges, count) + its bin ws
static size_t carve_cached(int n_sub, const rtgs_camera& cam, uint32_t cap, char* base, uint32_t** sorted,
                           uint2** range, uint32_t** n, void** bws) {
  const CamK k = make_cam(cam);
  const size_t T = (size_t)k.TX * k.TY;
  size_t o = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = base ? base + o : nullptr;
    o += align_up(bytes);
    return p;
  };
  char* a = take((size_t)cap * 4 + 4);
  char* b = take(T * 8);
  char* c = take(4);
  char* d = take(bin_workspace_size(n_sub, cam, cap));
  if (sorted) *sorted = (uint32_t*)a;
  if (range) *range = (uint2*)b;
  if (n) *n = (uint32_t*)c;
  if (bws) *bws = d;
  return o;
}

size_t bin_cached_workspace_size(int n_sub, const rtgs_camera& cam, uint32_t capacity) {
  return carve_cached(n_sub, cam, capacity, nullptr, nullptr, nullptr, nullptr, nullptr);
}

cudaError_t launch_bin_cached(const rtgs_projected& proj, const rtgs_bins& cache, const rtgs_projected& sub,
                              const int32_t* sub_gid, int n_sub, const rtgs_camera& cam, const uint8_t* keep,
                              const rtgs_bins& out, void* ws, cudaStream_t s) {
  const CamK k = make_cam(cam);
  const int T = k.TX * k.TY;
  uint32_t* ssorted;
  uint2* srange;
  uint32_t* sn;
  void* bws;
  carve_cached(n_sub, cam, out.capacity, static_cast<char*>(ws), &ssorted, &srange, &sn, &bws);
  (void)sn;
  BinWS w;
  carve(n_sub, cam, out.capacity, &w, static_cast<char*>(bws));
  cudaMemsetAsync(w.cnt, 0, (size_t)((char*)w.cursor - (char*)w.cnt), s);  // (the offsets write cursor)
  const uint2* rect = reinterpret_cast<const uint2*>(sub.rect);
  const int nblk = (n_sub + 255) / 256;
  if (n_sub > 0) {
    k_tile_count<kSubRep><<<nblk, 256, 0, s>>>(sub.zkey, rect, keep, n_sub, k.TX, T, w.cnt);
    note_launch();
  }
  k_merge_offsets<kSubRep><<<1, 1024, 0, s>>>(w.cnt, keep, reinterpret_cast<const uint2*>(cache.tile_range), T, out.capacity,
                                     w.cursor, srange, reinterpret_cast<uint2*>(out.tile_range), out.n_instances);
  note_launch();
  if (n_sub > 0) {
    k_emit<kSubRep><<<nblk, 256, 0, s>>>(sub.zkey, rect, keep, n_sub, k.TX, T, w.cursor, out.capacity, w.keys);
    note_launch();
  }
  int row_bits = 1;
  while (row_bits < 32 && (1u << row_bits) < (uint32_t)n_sub) ++row_bits;
  const size_t smem = (size_t)kSortCap * (8 + 8 + 4);
  static std::atomic<uint64_t> attr_mask{0};
  if (first_on_device(attr_mask)) {
    cudaFuncSetAttribute(k_sort_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  k_sort_merge<<<T, kSortThreads, smem, s>>>(keep, srange, w.keys, w.tmp, w.grank, row_bits, ssorted,
                                             reinterpret_cast<const uint2*>(cache.tile_range), cache.sorted_gid,
                                             proj.zkey, sub.zkey, sub_gid, reinterpret_cast<const uint2*>(out.tile_range),
                                             out.capacity, out.sorted_gid);
  note_launch();
  return cudaGetLastError();
}

// f3 flow with the coverage computed from the subset's tile lists, in two parts so that the first
// (which does not read the cache) can overlap the frame ingest that builds the cache:
//   part 1: bin the subset rows over ALL tiles (count, offsets, emit) and decide coverage / tile keep
//           per tile from those lists; the subset's lists stay in the workspace;
//   part 2: merge the kept tiles with the cached stable lists (offsets, sort + merge).
cudaError_t launch_coverage_subset(const rtgs_projected& sub, int n_sub, const rtgs_camera& cam,
                                   const rtgs_render_out& cov, uint32_t capacity, void* ws, cudaStream_t s) {
  const CamK k = make_cam(cam);
  const int T = k.TX * k.TY;
  uint32_t* ssorted;
  uint2* srange;
  uint32_t* sn;
  void* bws;
  carve_cached(n_sub, cam, capacity, static_cast<char*>(ws), &ssorted, &srange, &sn, &bws);
  BinWS w;
  carve(n_sub, cam, capacity, &w, static_cast<char*>(bws));
  cudaMemsetAsync(w.cnt, 0, (size_t)((char*)w.cursor - (char*)w.cnt), s);  // (the offsets write cursor)
  cudaMemsetAsync(cov.active_bits, 0, ((size_t)k.W * k.H + 31) / 32 * 4, s);
  cudaMemsetAsync(cov.counts, 0, 16, s);
  const uint2* rect = reinterpret_cast<const uint2*>(sub.rect);
  const int nblk = (n_sub + 255) / 256;
  if (n_sub > 0) {
    k_tile_count<kSubRep><<<nblk, 256, 0, s>>>(sub.zkey, rect, nullptr, n_sub, k.TX, T, w.cnt);
    note_launch();
  }
  k_tile_offsets<kSubRep><<<1, 1024, 0, s>>>(w.cnt, T, capacity, w.cursor, srange, sn);
  note_launch();
  if (n_sub > 0) {
    k_emit<kSubRep><<<nblk, 256, 0, s>>>(sub.zkey, rect, nullptr, n_sub, k.TX, T, w.cursor, capacity, w.keys);
    note_launch();
  }
  return launch_tile_coverage(srange, w.keys, reinterpret_cast<const float4*>(sub.rec), cam, cov, s);
}

cudaError_t launch_merge_cached(const rtgs_projected& proj, const rtgs_bins& cache, const rtgs_projected& sub,
                                const int32_t* sub_gid, int n_sub, const rtgs_camera& cam, const uint8_t* keep,
                                const rtgs_bins& out, void* ws, cudaStream_t s) {
  const CamK k = make_cam(cam);
  const int T = k.TX * k.TY;
  uint32_t* ssorted;
  uint2* srange;
  uint32_t* sn;
  void* bws;
  carve_cached(n_sub, cam, out.capacity, static_cast<char*>(ws), &ssorted, &srange, &sn, &bws);
  BinWS w;
  carve(n_sub, cam, out.capacity, &w, static_cast<char*>(bws));
  k_merge_offsets<kSubRep><<<1, 1024, 0, s>>>(w.cnt, keep, reinterpret_cast<const uint2*>(cache.tile_range), T, out.capacity,
                                     w.cursor, srange, reinterpret_cast<uint2*>(out.tile_range), out.n_instances);
  note_launch();
  int row_bits = 1;
  while (row_bits < 32 && (1u << row_bits) < (uint32_t)n_sub) ++row_bits;
  const size_t smem = (size_t)kSortCap * (8 + 8 + 4);
  static std::atomic<uint64_t> attr_mask{0};
  if (first_on_device(attr_mask)) {
    cudaFuncSetAttribute(k_sort_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  k_sort_merge<<<T, kSortThreads, smem, s>>>(keep, srange, w.keys, w.tmp, w.grank, row_bits, ssorted,
                                             reinterpret_cast<const uint2*>(cache.tile_range), cache.sorted_gid,
                                             proj.zkey, sub.zkey, sub_gid, reinterpret_cast<const uint2*>(out.tile_range),
                                             out.capacity, out.sorted_gid);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_coverage_bin_cached(const rtgs_projected& proj, const rtgs_bins& cache, const rtgs_projected& sub,
                                       const int32_t* sub_gid, int n_sub, const rtgs_camera& cam,
                                       const rtgs_render_out& cov, const rtgs_bins& out, void* ws, cudaStream_t s) {
  cudaError_t e = launch_coverage_subset(sub, n_sub, cam, cov, out.capacity, ws, s);
  if (e != cudaSuccess) return e;
  return launch_merge_cached(proj, cache, sub, sub_gid, n_sub, cam, cov.tile_keep, out, ws, s);
}

}  // namespace rtgs
