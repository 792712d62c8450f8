// adam.cuh — the A6 per-component update (Eq.8; readings R18-R20), shared by
// the stand-alone Adam kernel (adam.cu) and the fused backward + Adam epilogue (backward.cu), so the
// two paths perform the same float32 operations in the same order.
#pragma once
#include <stdint.h>

#include "rtgs.h"

namespace rtgs {

struct AdamHP {
  float lr_pos, lr_sh0, lr_shrest, lr_scale, lr_rot;
  float b1, omb1, b2, omb2, eps, bc1, bc2;
  float log_b1, log_b2;        // for the device-step bias corrections 1 - beta^t = -expm1(t log beta)
  const int32_t* step_device;  // when set, bias corrections are formed from the device step
  float reg_coef;              // 2 w_reg / (10 N_t): d L_reg / d theta = reg_coef (theta - theta_0)  (R18)
};

AdamHP make_adam_hp(const rtgs_hparams& hp, int step, const int32_t* step_device, int n_transparent, float w_reg);

struct AdamBC {
  float ibc1, ibc2;
};

__device__ __forceinline__ AdamBC adam_bias(const AdamHP& h) {
  float bc1 = h.bc1, bc2 = h.bc2;
  if (h.step_device) {
    const float st = (float)*h.step_device;
    bc1 = -expm1f(st * h.log_b1);
    bc2 = -expm1f(st * h.log_b2);
  }
  return AdamBC{1.f / bc1, 1.f / bc2};
}

// learning rate of row component j (pos 3, log-scale 3, rot 4, SH DC 3, SH rest)
__device__ __forceinline__ float adam_lr(const AdamHP& h, int j) {
  return j < 10 ? (j < 3 ? h.lr_pos : (j < 6 ? h.lr_scale : h.lr_rot)) : (j < 13 ? h.lr_sh0 : h.lr_shrest);
}

// One Adam step of one component: m, v updated in place, returns the new parameter.
// theta -= lr m^ / (sqrt(v^) + eps)   (m = 0 whenever v = 0, so the quotient is 0 there)
__device__ __forceinline__ float adam_one(const AdamHP& h, const AdamBC& bc, float lr, float th, float g, float& m,
                                          float& v) {
  const float mm = h.b1 * m + h.omb1 * g;
  const float vv = h.b2 * v + h.omb2 * g * g;
  m = mm;
  v = vv;
  // sqrt.approx (no flush of denormal v): ~1 ulp, so the update's relative error stays ~1e-7, far
  // inside the 1e-6 parameter contract; the IEEE sqrtf was 15 % of the fused epilogue's instructions
  float sv;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(sv) : "f"(vv * bc.ibc2));
  return th - lr * __fdividef(mm * bc.ibc1, sv + h.eps);
}

}  // namespace rtgs
