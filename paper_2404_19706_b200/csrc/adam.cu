// adam.cu — A6: fused L_reg + Adam + confidence count over the unstable Gaussians only
// (O6; Eq.8, readings R18-R20).
//
// One CTA per 16 consecutive slots; its threads stride over the flat [16 x D] block of the
// grad / m / v rows (D = 10 + 3K), so those streams are fully coalesced; the parameter of
// component j is gathered by gid with branch-free address selects.  Per-slot "SH gradient != 0"
// flags live in shared memory and give eta += 1 once per slot (R20).
#include "common.cuh"
#include "internal.h"

namespace rtgs {

constexpr int kAdamSlots = 16;
constexpr int kAdamThreads = 256;

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
  float reg_coef;  // 2 w_reg / (10 N_t)
  float lr_pos, lr_sh0, lr_shrest, lr_scale, lr_rot;
  float b1, omb1, b2, omb2, eps, bc1, bc2;
  double beta1, beta2;
  const int32_t* step_device;  // when set, bias corrections are formed from the device step
  uint32_t* eta;
};

template <int K>
__global__ void __launch_bounds__(kAdamThreads) k_adam(const AdamArgs a) {
  constexpr int D = 10 + 3 * K;
  __shared__ int s_gid[kAdamSlots];
  __shared__ int s_tr[kAdamSlots];
  __shared__ int s_nz[kAdamSlots];
  const int s0 = blockIdx.x * kAdamSlots;
  const int ns = min(kAdamSlots, a.n_slots - s0);
  if (threadIdx.x < ns) {
    const int g = a.gid_of_slot[s0 + threadIdx.x];
    s_gid[threadIdx.x] = g;
    s_tr[threadIdx.x] = a.flags[g] & 1u;
    s_nz[threadIdx.x] = 0;
  }
  __syncthreads();
  float bc1 = a.bc1, bc2 = a.bc2;
  if (a.step_device) {
    const double t = (double)*a.step_device;
    bc1 = (float)(1.0 - pow(a.beta1, t));
    bc2 = (float)(1.0 - pow(a.beta2, t));
  }
  const size_t base = (size_t)s0 * D;
  for (int e = threadIdx.x; e < ns * D; e += kAdamThreads) {
    const int ls = e / D, j = e - ls * D;
    const size_t gid = (size_t)s_gid[ls];
    float* p = j < 3 ? a.pos + 3 * gid + j
                     : (j < 6 ? a.log_scale + 3 * gid + (j - 3)
                              : (j < 10 ? a.rot + 4 * gid + (j - 6) : a.sh + (size_t)(3 * K) * gid + (j - 10)));
    const float lr = j < 3 ? a.lr_pos : (j < 6 ? a.lr_scale : (j < 10 ? a.lr_rot : (j < 13 ? a.lr_sh0 : a.lr_shrest)));
    const size_t o = base + e;
    float g = a.grad[o];
    if (j >= 10 && g != 0.f) s_nz[ls] = 1;
    float th = *p;
    if (j < 10 && s_tr[ls]) g += a.reg_coef * (th - a.init_geom[(size_t)(s0 + ls) * 10 + j]);  // L_reg (R18)
    const float mm = a.b1 * a.m[o] + a.omb1 * g;
    const float vv = a.b2 * a.v[o] + a.omb2 * g * g;
    a.m[o] = mm;
    a.v[o] = vv;
    th -= lr * (mm / bc1) / (sqrtf(vv / bc2) + a.eps);
    *p = th;
    a.grad[o] = 0.f;  // consumed
  }
  __syncthreads();
  if (threadIdx.x < ns && s_nz[threadIdx.x]) a.eta[s_gid[threadIdx.x]] += 1u;  // R20
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
  a.reg_coef = n_transparent > 0 ? (float)(2.0 * w_reg / (10.0 * n_transparent)) : 0.f;
  a.lr_pos = hp.lr_pos; a.lr_sh0 = hp.lr_sh0; a.lr_shrest = hp.lr_shrest; a.lr_scale = hp.lr_scale; a.lr_rot = hp.lr_rot;
  a.b1 = (float)hp.beta1; a.omb1 = (float)(1.0 - hp.beta1);
  a.b2 = (float)hp.beta2; a.omb2 = (float)(1.0 - hp.beta2);
  a.eps = (float)hp.eps;
  a.bc1 = (float)(1.0 - pow(hp.beta1, step));
  a.bc2 = (float)(1.0 - pow(hp.beta2, step));
  a.beta1 = hp.beta1;
  a.beta2 = hp.beta2;
  a.step_device = step_device;
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
