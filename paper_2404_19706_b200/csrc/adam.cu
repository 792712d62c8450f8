// adam.cu — A6: fused L_reg + Adam + confidence count over the unstable Gaussians only
// (O6; Eq.8, readings R18-R20).
//
// One CTA per 16 consecutive slots; its threads stride over the flat [16 x D] block of the
// grad / m / v rows (D = 10 + 3K), so those streams are fully coalesced; the parameter of
// component j is gathered by gid with branch-free address selects.  Per-slot "SH gradient != 0"
// flags live in shared memory and give eta += 1 once per slot (R20).
#include "common.cuh"
#include "adam.cuh"
#include "internal.h"

namespace rtgs {

constexpr int kAdamThreads = 256;
constexpr int kLanesPerSlot = 16;                              // a half-warp owns one slot row
constexpr int kAdamSlots = kAdamThreads / kLanesPerSlot;      // 16 slots per CTA

struct AdamArgs {
  float* pos;
  float* log_scale;
  float* rot;
  float* sh;
  const int32_t* gid_of_slot;
  int n_slots;
  const uint8_t* flags;
  float* grad;
  float* m;
  float* v;
  const float* init_geom;
  AdamHP h;
  uint32_t* eta;
};

// One half-warp per slot: lane t owns components j = t, t+16, t+32, ... of the row (pos 3, log-scale 3,
// rot 4, SH 3K), so grad / m / v rows stream coalesced and only j < 16 needs the geometry selects.
template <int K>
__global__ void __launch_bounds__(kAdamThreads) k_adam(const AdamArgs a) {
  constexpr int D = 10 + 3 * K;
  const int lane = threadIdx.x & 31, t = threadIdx.x & (kLanesPerSlot - 1);
  const int slot = blockIdx.x * kAdamSlots + (threadIdx.x >> 4);
  const bool live = slot < a.n_slots;
  const AdamBC bc = adam_bias(a.h);
  bool nz = false;
  uint32_t eta0 = 0;
  size_t gid = 0;
  if (live) {
    gid = (size_t)a.gid_of_slot[slot];
    if (t == 0) eta0 = a.eta[gid];  // issued with the row gathers, not after the update
    const bool transparent = (a.flags[gid] & 5u) == 1u;  // transparent and not removed (R18, R29)
    const size_t row = (size_t)slot * D;
    const float th0v = (t < 10 && a.init_geom) ? a.init_geom[(size_t)slot * 10 + t] : 0.f;  // independent of gid
    float* shrow = a.sh + (size_t)(3 * K) * gid - 10;
    constexpr int NIT = (D + kLanesPerSlot - 1) / kLanesPerSlot;
    // all loads of the row are issued before any store (stores could alias later loads otherwise)
    float g[NIT], mo[NIT], vo[NIT], th[NIT];
    float* p[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int j = min(t + it * kLanesPerSlot, D - 1);
      if (it == 0 && j < 10)
        p[it] = j < 3 ? a.pos + 3 * gid + j : (j < 6 ? a.log_scale + 3 * gid + (j - 3) : a.rot + 4 * gid + (j - 6));
      else
        p[it] = shrow + j;
      g[it] = a.grad[row + j];
      mo[it] = a.m[row + j];
      vo[it] = a.v[row + j];
      th[it] = *p[it];
    }
    const float th0 = transparent ? th0v : 0.f;
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int j = t + it * kLanesPerSlot;
      if (j >= D) break;
      float gg = g[it];
      if (j >= 10 && gg != 0.f) nz = true;
      if (it == 0 && j < 10 && transparent) gg += a.h.reg_coef * (th[it] - th0);  // L_reg (R18)
      float mm = mo[it], vv = vo[it];
      *p[it] = adam_one(a.h, bc, adam_lr(a.h, j), th[it], gg, mm, vv);
      a.m[row + j] = mm;
      a.v[row + j] = vv;
      a.grad[row + j] = 0.f;  // consumed
    }
  }
  // eta += 1 once per slot with a non-zero SH gradient (R20): vote within the half-warp
  const uint32_t vote = __ballot_sync(0xffffffffu, nz);
  const uint32_t half = (lane < 16) ? (vote & 0x0000FFFFu) : (vote & 0xFFFF0000u);
  if (live && t == 0 && half) a.eta[gid] = eta0 + 1u;
}

AdamHP make_adam_hp(const rtgs_hparams& hp, int step, const int32_t* step_device, int n_transparent, float w_reg) {
  AdamHP h;
  h.lr_pos = hp.lr_pos; h.lr_sh0 = hp.lr_sh0; h.lr_shrest = hp.lr_shrest; h.lr_scale = hp.lr_scale;
  h.lr_rot = hp.lr_rot;
  h.b1 = (float)hp.beta1; h.omb1 = (float)(1.0 - hp.beta1);
  h.b2 = (float)hp.beta2; h.omb2 = (float)(1.0 - hp.beta2);
  h.eps = (float)hp.eps;
  h.bc1 = (float)(1.0 - pow(hp.beta1, step));
  h.bc2 = (float)(1.0 - pow(hp.beta2, step));
  h.log_b1 = (float)log(hp.beta1);
  h.log_b2 = (float)log(hp.beta2);
  h.step_device = step_device;
  h.reg_coef = n_transparent > 0 ? (float)(2.0 * w_reg / (10.0 * n_transparent)) : 0.f;
  return h;
}

cudaError_t launch_adam(const rtgs_params& p, const int32_t* gid_of_slot, int n_slots, const uint8_t* flags,
                        float* grad, float* m, float* v, const float* init_geom, int n_transparent, float w_reg,
                        const rtgs_hparams& hp, int step, const int32_t* step_device, uint32_t* eta,
                        cudaStream_t s) {
  if (n_slots == 0) return cudaSuccess;
  AdamArgs a;
  a.pos = p.pos; a.log_scale = p.log_scale; a.rot = p.rot; a.sh = p.sh;
  a.gid_of_slot = gid_of_slot; a.n_slots = n_slots; a.flags = flags;
  a.grad = grad; a.m = m; a.v = v; a.init_geom = init_geom;
  a.h = make_adam_hp(hp, step, step_device, n_transparent, w_reg);
  a.eta = eta;
  const int blocks = (n_slots + kAdamSlots - 1) / kAdamSlots;
  switch ((p.sh_degree + 1) * (p.sh_degree + 1)) {
    case 1: k_adam<1><<<blocks, kAdamThreads, 0, s>>>(a); break;
    case 4: k_adam<4><<<blocks, kAdamThreads, 0, s>>>(a); break;
    case 9: k_adam<9><<<blocks, kAdamThreads, 0, s>>>(a); break;
    default: k_adam<16><<<blocks, kAdamThreads, 0, s>>>(a); break;
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtgs
