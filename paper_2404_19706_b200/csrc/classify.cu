// classify.cu — A7: add masks M_s / M_c, 5 % sampling and the per-sample action
// (O7; Eq.6, readings R21, R22, R24).
//
// Pass 1 (one thread per pixel): classify in float32 with the operation order of include/rtgs.h,
// write the class byte, count masks/actions per CTA.  Pass 2: scan of the per-CTA sample counts.
// Pass 3: re-read the class byte and write the samples in row-major order (ballot ranks).
#include "common.cuh"
#include "internal.h"

namespace rtgs {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct ClsArgs {
  const float *chat, *trans, *dhat;
  const int32_t* index;
  const float *c, *d;
  const uint8_t* flags;
  int HW;
  float dT, dd, dc;
  uint64_t key;
  uint64_t thr;
  uint8_t* cls;
  uint32_t* blk;
  uint32_t* counts;
};

__global__ void __launch_bounds__(256) k_classify(const ClsArgs a) {
  __shared__ uint32_t sh[33];
  __shared__ uint32_t s_cnt[5];
  if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int p = blockIdx.x * 256 + threadIdx.x;
  uint32_t emit = 0;
  if (p < a.HW) {
    const float D = a.d[p];
    const bool valid = isfinite(D) && D > 0.f;
    const float dd = fabsf(__fsub_rn(a.dhat[p], D));
    const bool ms = valid && (a.trans[p] > a.dT || dd > a.dd);
    const float e0 = fabsf(__fsub_rn(a.chat[p], a.c[p]));
    const float e1 = fabsf(__fsub_rn(a.chat[a.HW + p], a.c[a.HW + p]));
    const float e2 = fabsf(__fsub_rn(a.chat[2 * a.HW + p], a.c[2 * a.HW + p]));
    const float err = __fdiv_rn(__fadd_rn(__fadd_rn(e0, e1), e2), 3.f);
    const bool mc = valid && !ms && err > a.dc;
    const bool samp = (splitmix64(a.key ^ (uint64_t)p) >> 32) < a.thr;
    uint32_t action = 0;
    if (samp && ms) action = 1;
    if (samp && mc) {
      const int idx = a.index[p];
      action = idx >= 0 ? ((a.flags[idx] & 2u) ? 2u : 3u) : 1u;
    }
    const uint32_t mask = ms ? 1u : (mc ? 2u : 0u);
    a.cls[p] = (uint8_t)(mask | ((samp && mask) ? 4u : 0u) | (action << 3));
    emit = (action == 1u || action == 2u) ? 1u : 0u;
    if (ms) atomicAdd(&s_cnt[0], 1u);
    if (mc) atomicAdd(&s_cnt[1], 1u);
    if (action) atomicAdd(&s_cnt[1 + action], 1u);
  }
  uint32_t tot;
  block_excl_scan(emit, sh, &tot);
  if (threadIdx.x == 0) a.blk[blockIdx.x] = tot;
  if (threadIdx.x < 5 && s_cnt[threadIdx.x]) atomicAdd(&a.counts[threadIdx.x], s_cnt[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_emit_samples(const uint8_t* __restrict__ cls, int HW,
                                                      const uint32_t* __restrict__ blk_off, uint32_t cap,
                                                      uint32_t* __restrict__ samples) {
  __shared__ uint32_t sh[33];
  const int p = blockIdx.x * 256 + threadIdx.x;
  uint32_t action = 0;
  if (p < HW) action = (uint32_t)(cls[p] >> 3);
  const bool emit = action == 1u || action == 2u;
  uint32_t tot;
  const uint32_t r = block_excl_scan(emit ? 1u : 0u, sh, &tot);
  if (emit) {
    const uint32_t pos = blk_off[blockIdx.x] + r;
    if (pos < cap) samples[pos] = (uint32_t)p | (action << 30);
  }
}

size_t classify_workspace_size(const rtgs_camera& cam) {
  const size_t HW = (size_t)cam.width * cam.height;
  const size_t nb = (HW + 255) / 256;
  return 2 * ((nb * 4 + 255) / 256 * 256) + scan_workspace_size(nb) + 256;
}

cudaError_t launch_classify(const rtgs_render_out& full, const rtgs_frame& frame, const uint8_t* flags,
                            const rtgs_camera& cam, const rtgs_add_params& ap, uint8_t* cls, uint32_t* samples,
                            uint32_t cap, uint32_t* counts, void* ws, cudaStream_t s) {
  const int HW = cam.width * cam.height;
  const int nb = (HW + 255) / 256;
  char* base = static_cast<char*>(ws);
  const size_t arr = ((size_t)nb * 4 + 255) / 256 * 256;
  uint32_t* blk = reinterpret_cast<uint32_t*>(base);
  uint32_t* off = reinterpret_cast<uint32_t*>(base + arr);
  void* scan_ws = base + 2 * arr;
  cudaMemsetAsync(counts, 0, 5 * sizeof(uint32_t), s);
  ClsArgs a;
  a.chat = full.color; a.trans = full.trans; a.dhat = full.depth; a.index = full.index;
  a.c = frame.color; a.d = frame.depth; a.flags = flags; a.HW = HW;
  a.dT = ap.delta_T; a.dd = ap.delta_d; a.dc = ap.delta_c;
  a.key = ap.seed ^ ((uint64_t)ap.frame_idx << 32);
  const double thr = floor((double)ap.sample_ratio * 4294967296.0 + 0.5);
  a.thr = thr <= 0 ? 0ull : (uint64_t)thr;
  a.cls = cls; a.blk = blk; a.counts = counts;
  k_classify<<<nb, 256, 0, s>>>(a);
  note_launch();
  cudaError_t e = launch_scan(blk, off, nb, nullptr, scan_ws, s);
  if (e) return e;
  k_emit_samples<<<nb, 256, 0, s>>>(cls, HW, off, cap, samples);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// (e) K9: the top `ratio` colour-error pixels of a keyframe (reading R36) by an exact MSB-first
// radix select on the float32 error bits (non-negative floats order like their bit patterns):
// three passes of 11 / 11 / 10 bits, each a per-CTA shared-memory histogram of the pixels whose
// higher bits match the prefix found so far plus a one-CTA bucket selection; then the pixels equal
// to the threshold are ranked in row-major order by a scan (ties by pixel index).
// ------------------------------------------------------------------------------------------------
struct SelState {
  uint32_t prefix;   // bits of the threshold determined so far
  uint32_t krem;     // pixels still to take at or below the current prefix
  uint32_t greater;  // pixels strictly above the threshold found so far
  uint32_t pad;
};

__global__ void k_sel_init(SelState* st, uint32_t K) {
  if (threadIdx.x == 0) *st = SelState{0u, K, 0u, 0u};
}

__global__ void __launch_bounds__(256) k_err_key(const float* __restrict__ chat, const float* __restrict__ c, int HW,
                                                 uint32_t* __restrict__ key) {
  const int p = blockIdx.x * 256 + threadIdx.x;
  if (p >= HW) return;
  const float e0 = fabsf(__fsub_rn(chat[p], c[p]));
  const float e1 = fabsf(__fsub_rn(chat[HW + p], c[HW + p]));
  const float e2 = fabsf(__fsub_rn(chat[2 * HW + p], c[2 * HW + p]));
  key[p] = __float_as_uint(__fdiv_rn(__fadd_rn(__fadd_rn(e0, e1), e2), 3.f));  // the A7 order (R21)
}

__global__ void __launch_bounds__(256) k_sel_hist(const uint32_t* __restrict__ key, int HW, int shift, int bits,
                                                  const SelState* __restrict__ st, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[2048];
  const int nbin = 1 << bits;
  for (int i = threadIdx.x; i < nbin; i += 256) h[i] = 0;
  __syncthreads();
  const int hi = shift + bits;  // bits above [shift, hi) must equal the prefix
  const uint32_t pre = st->prefix;
  for (int p = blockIdx.x * 256 + threadIdx.x; p < HW; p += gridDim.x * 256) {
    const uint32_t k = key[p];
    if (hi >= 32 || (k >> hi) == (pre >> hi)) atomicAdd(&h[(k >> shift) & (nbin - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbin; i += 256)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// one CTA of 1024 threads: the bucket d (from the top) with sum_{> d} < krem <= sum_{>= d}
__global__ void __launch_bounds__(1024) k_sel_pick(uint32_t* __restrict__ hist, int shift, int bits,
                                                   SelState* __restrict__ st) {
  __shared__ uint32_t sh[33];
  __shared__ uint32_t s_pick[2];
  const int nbin = 1 << bits;
  // thread t owns the 2 bins counted from the top: descending bin index nbin-1-2t, nbin-2-2t
  const int b0 = nbin - 1 - 2 * (int)threadIdx.x, b1 = b0 - 1;
  const uint32_t c0 = b0 >= 0 ? hist[b0] : 0u, c1 = b1 >= 0 ? hist[b1] : 0u;
  uint32_t tot;
  const uint32_t ex = block_excl_scan(c0 + c1, sh, &tot);  // pixels in bins above b0
  const uint32_t krem = st->krem;
  if (threadIdx.x == 0) s_pick[0] = 0xFFFFFFFFu;
  __syncthreads();
  if (b0 >= 0 && ex < krem && krem <= ex + c0) { s_pick[0] = (uint32_t)b0; s_pick[1] = ex; }
  if (b1 >= 0 && ex + c0 < krem && krem <= ex + c0 + c1) { s_pick[0] = (uint32_t)b1; s_pick[1] = ex + c0; }
  __syncthreads();
  if (threadIdx.x == 0 && s_pick[0] != 0xFFFFFFFFu) {
    st->prefix |= s_pick[0] << shift;
    st->greater += s_pick[1];
    st->krem = krem - s_pick[1];
  }
  for (int i = threadIdx.x; i < nbin; i += 1024) hist[i] = 0;  // ready for the next pass
}

__global__ void __launch_bounds__(256) k_sel_eq(const uint32_t* __restrict__ key, int HW,
                                                const SelState* __restrict__ st, uint32_t* __restrict__ eq) {
  const int p = blockIdx.x * 256 + threadIdx.x;
  if (p < HW) eq[p] = (st->krem > 0u && key[p] == st->prefix) ? 1u : 0u;
}

// selected = key > tau or (key == tau and rank among the equal ones < need); one mask word per warp
__global__ void __launch_bounds__(256) k_sel_mask(const uint32_t* __restrict__ key, int HW,
                                                  const SelState* __restrict__ st, const uint32_t* __restrict__ rank,
                                                  uint32_t* __restrict__ bits) {
  const int p = blockIdx.x * 256 + threadIdx.x;
  bool sel = false;
  if (p < HW && st->krem + st->greater > 0u) {
    const uint32_t k = key[p], tau = st->prefix;
    sel = k > tau || (k == tau && rank[p] < st->krem);
  }
  const uint32_t m = __ballot_sync(0xffffffffu, sel);
  if ((threadIdx.x & 31) == 0 && p < HW) bits[p >> 5] = m;
}

size_t topk_workspace_size(const rtgs_camera& cam) {
  const size_t HW = (size_t)cam.width * cam.height;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  return 3 * al(HW * 4 + 4) + al(2048 * 4) + al(sizeof(SelState)) + scan_workspace_size(HW) + 256;
}

cudaError_t launch_topk(const float* chat, const float* c, const rtgs_camera& cam, double ratio,
                        const rtgs_render_out& out, void* ws, cudaStream_t s) {
  const int HW = cam.width * cam.height;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  char* base = static_cast<char*>(ws);
  uint32_t* key = reinterpret_cast<uint32_t*>(base);
  uint32_t* eq = reinterpret_cast<uint32_t*>(base + al((size_t)HW * 4 + 4));
  uint32_t* rank = reinterpret_cast<uint32_t*>(base + 2 * al((size_t)HW * 4 + 4));
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + 3 * al((size_t)HW * 4 + 4));
  SelState* st = reinterpret_cast<SelState*>(base + 3 * al((size_t)HW * 4 + 4) + al(2048 * 4));
  void* scan_ws = base + 3 * al((size_t)HW * 4 + 4) + al(2048 * 4) + al(sizeof(SelState));
  const double kd = floor(ratio * (double)HW + 0.5);
  const uint32_t K = kd <= 0 ? 0u : (kd >= (double)HW ? (uint32_t)HW : (uint32_t)kd);
  k_sel_init<<<1, 32, 0, s>>>(st, K);
  note_launch();
  cudaMemsetAsync(hist, 0, 2048 * 4, s);
  cudaMemsetAsync(out.active_bits, 0, ((size_t)HW + 31) / 32 * 4, s);
  cudaMemsetAsync(out.counts, 0, 16, s);
  const int nb = (HW + 255) / 256;
  if (HW > 0) {
    k_err_key<<<nb, 256, 0, s>>>(chat, c, HW, key);
    const int hb = min(nb, 148 * 8);
    const int shifts[3] = {21, 10, 0}, nbits[3] = {11, 11, 10};
    for (int q = 0; q < 3; ++q) {
      k_sel_hist<<<hb, 256, 0, s>>>(key, HW, shifts[q], nbits[q], st, hist);
      k_sel_pick<<<1, 1024, 0, s>>>(hist, shifts[q], nbits[q], st);
    }
    k_sel_eq<<<nb, 256, 0, s>>>(key, HW, st, eq);
    note_launch(8);
    cudaError_t e = launch_scan(eq, rank, HW, nullptr, scan_ws, s);
    if (e != cudaSuccess) return e;
    k_sel_mask<<<nb, 256, 0, s>>>(key, HW, st, rank, out.active_bits);
    note_launch();
  }
  return launch_tile_any(cam, out, s);
}

}  // namespace rtgs
