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

}  // namespace rtgs
