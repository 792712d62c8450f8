// adam.cu — A6: fused L_reg + Adam + confidence count over the unstable Gaussians only
// (O6; Eq.8, readings R18-R20).
//
// One warp per slot: lane j and j+32 own components j of the slot row (pos 3, log_scale 3, rot 4,
// sh 3K), so the grad / m / v rows stream coalesced and the parameters are gathered by gid.
#include "common.cuh"
#include "internal.h"

namespace rtgs {

struct AdamArgs {
  float* pos;
  float* log_scale;
  float* rot;
  float* sh;
  int K, D;
  const int32_t* gid_of_slot;
  int n_slots;
  const uint8_t* flags;
  float* grad;
  float* m;
  float* v;
  const float* init_geom;
  float reg_coef;  // 2 w_reg / (10 N_t)
  float lr_pos, lr_sh0, lr_shrest, lr_scale, lr_rot;
  float b1, b2, eps, bc1, bc2;
  uint32_t* eta;
};

__global__ void __launch_bounds__(256) k_adam(const AdamArgs a) {
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= a.n_slots) return;
  const int gid = a.gid_of_slot[s];
  const bool transparent = a.flags[gid] & 1u;
  bool sh_nz = false;
  for (int j = lane; j < a.D; j += 32) {
    float* p;
    float lr;
    if (j < 3) { p = a.pos + 3 * (size_t)gid + j; lr = a.lr_pos; }
    else if (j < 6) { p = a.log_scale + 3 * (size_t)gid + (j - 3); lr = a.lr_scale; }
    else if (j < 10) { p = a.rot + 4 * (size_t)gid + (j - 6); lr = a.lr_rot; }
    else { p = a.sh + (size_t)3 * a.K * gid + (j - 10); lr = j < 13 ? a.lr_sh0 : a.lr_shrest; }
    const size_t o = (size_t)s * a.D + j;
    float g = a.grad[o];
    if (j >= 10 && g != 0.f) sh_nz = true;
    float th = *p;
    if (transparent && j < 10) g += a.reg_coef * (th - a.init_geom[(size_t)s * 10 + j]);  // L_reg (R18)
    const float mm = a.b1 * a.m[o] + (1.f - a.b1) * g;
    const float vv = a.b2 * a.v[o] + (1.f - a.b2) * g * g;
    a.m[o] = mm;
    a.v[o] = vv;
    const float mhat = mm / a.bc1, vhat = vv / a.bc2;
    th -= lr * mhat / (sqrtf(vhat) + a.eps);
    *p = th;
    a.grad[o] = 0.f;  // consumed
  }
  if (__any_sync(0xffffffffu, sh_nz) && lane == 0) a.eta[gid] += 1u;  // R20
}

cudaError_t launch_adam(const rtgs_params& p, const int32_t* gid_of_slot, int n_slots, const uint8_t* flags,
                        float* grad, float* m, float* v, const float* init_geom, int n_transparent, float w_reg,
                        const rtgs_hparams& hp, int step, uint32_t* eta, cudaStream_t s) {
  if (n_slots == 0) return cudaSuccess;
  AdamArgs a;
  a.pos = p.pos; a.log_scale = p.log_scale; a.rot = p.rot; a.sh = p.sh;
  a.K = (p.sh_degree + 1) * (p.sh_degree + 1);
  a.D = 10 + 3 * a.K;
  a.gid_of_slot = gid_of_slot; a.n_slots = n_slots; a.flags = flags;
  a.grad = grad; a.m = m; a.v = v; a.init_geom = init_geom;
  a.reg_coef = n_transparent > 0 ? (float)(2.0 * w_reg / (10.0 * n_transparent)) : 0.f;
  a.lr_pos = hp.lr_pos; a.lr_sh0 = hp.lr_sh0; a.lr_shrest = hp.lr_shrest; a.lr_scale = hp.lr_scale; a.lr_rot = hp.lr_rot;
  a.b1 = hp.beta1; a.b2 = hp.beta2; a.eps = hp.eps;
  a.bc1 = (float)(1.0 - pow((double)hp.beta1, step));
  a.bc2 = (float)(1.0 - pow((double)hp.beta2, step));
  a.eta = eta;
  const long long threads = (long long)n_slots * 32;
  k_adam<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtgs
