// state.cu — NEXT row f1: window fusion (Eq.9) and state management.
//
// k_fuse        half-warp per slot row (as k_adam): theta = (1-w) before + w theta', w from eta.
// k_mark        1 thread per pixel of the optimised FULL render: flag the stable hit Gaussian of a
//               pixel whose colour or depth error exceeds its threshold (once per frame).
// k_transition  1 thread per Gaussian: e += flag, then the stable / unstable / removed transitions.
#include "common.cuh"
#include "internal.h"

namespace rtgs {

constexpr int kFuseThreads = 256;
constexpr int kFuseLanes = 16;

struct FuseArgs {
  float* pos;
  float* log_scale;
  float* rot;
  float* sh;
  const int32_t* gid_of_slot;
  int n_slots;
  const float* before;
  const uint32_t* eta_before;
  const uint32_t* eta;
};

template <int K>
__global__ void __launch_bounds__(kFuseThreads) k_fuse(const FuseArgs a) {
  constexpr int D = 10 + 3 * K;
  const int t = threadIdx.x & (kFuseLanes - 1);
  const int slot = blockIdx.x * (kFuseThreads / kFuseLanes) + (threadIdx.x >> 4);
  if (slot >= a.n_slots) return;
  const size_t gid = (size_t)a.gid_of_slot[slot];
  const uint32_t e1 = a.eta[gid], e0 = a.eta_before[slot];
  // Eq.9: w = (eta'_o - eta_{o-1}) / eta'_o ; no update (eta' = 0) keeps G_{o-1}
  const float w = e1 > 0u ? (float)((double)(e1 - min(e0, e1)) / (double)e1) : 0.f;
  const float* b = a.before + (size_t)slot * D;
  constexpr int NIT = (D + kFuseLanes - 1) / kFuseLanes;
  float* p[NIT];
  float tn[NIT], to[NIT];
#pragma unroll
  for (int it = 0; it < NIT; ++it) {  // every load of the row before any store
    const int j = min(t + it * kFuseLanes, D - 1);
    p[it] = j < 3 ? a.pos + 3 * gid + j
                  : (j < 6 ? a.log_scale + 3 * gid + (j - 3)
                           : (j < 10 ? a.rot + 4 * gid + (j - 6) : a.sh + (size_t)(3 * K) * gid + (j - 10)));
    tn[it] = *p[it];
    to[it] = b[j];
  }
#pragma unroll
  for (int it = 0; it < NIT; ++it)
    if (t + it * kFuseLanes < D) *p[it] = __fmaf_rn(w, tn[it] - to[it], to[it]);  // (1-w) old + w new
}

struct MarkArgs {
  const float *chat, *dhat;
  const int32_t* index;
  const float *c, *d;
  const uint8_t* flags;
  int HW;
  float dc, dd;
  uint8_t* mark;
};

__global__ void __launch_bounds__(256) k_mark(const MarkArgs a) {
  const int p = blockIdx.x * 256 + threadIdx.x;
  if (p >= a.HW) return;
  const int idx = a.index[p];
  if (idx < 0 || !(a.flags[idx] & 2u)) return;
  const float D = a.d[p];
  if (!(isfinite(D) && D > 0.f)) return;  // R24
  const float dd = fabsf(__fsub_rn(a.dhat[p], D));
  const float e0 = fabsf(__fsub_rn(a.chat[p], a.c[p]));
  const float e1 = fabsf(__fsub_rn(a.chat[a.HW + p], a.c[a.HW + p]));
  const float e2 = fabsf(__fsub_rn(a.chat[2 * a.HW + p], a.c[2 * a.HW + p]));
  const float err = __fdiv_rn(__fadd_rn(__fadd_rn(e0, e1), e2), 3.f);
  if (err > a.dc || dd > a.dd) a.mark[idx] = 1;  // benign race: every writer stores 1
}

struct TransArgs {
  uint8_t* flags;
  uint32_t* err;
  uint32_t* eta;
  uint32_t* tc;
  const uint8_t* mark;
  int n;
  uint32_t de, deta, dt, k;
  uint32_t* counts;
};

__global__ void __launch_bounds__(256) k_transition(const TransArgs a) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  uint32_t c_mark = 0, c_toun = 0, c_tost = 0, c_rem = 0;
  if (i < a.n) {
    uint8_t f = a.flags[i];
    if (!(f & 4u)) {
      if (f & 2u) {  // stable
        uint32_t e = a.err[i];
        if (a.mark[i]) {
          e += 1u;
          c_mark = 1;
        }
        if (e > a.de) {  // -> unstable; counters restart (R29)
          f &= (uint8_t)~2u;
          e = 0u;
          a.eta[i] = 0u;
          a.tc[i] = a.k;
          c_toun = 1;
        }
        a.err[i] = e;
      } else {       // unstable
        if (a.eta[i] > a.deta) {
          f |= 2u;
          c_tost = 1;
        } else if (a.k - a.tc[i] > a.dt && a.k >= a.tc[i]) {
          f |= 4u;
          c_rem = 1;
        }
      }
      a.flags[i] = f;
    }
  }
  const uint32_t s0 = __reduce_add_sync(0xffffffffu, c_mark), s1 = __reduce_add_sync(0xffffffffu, c_toun);
  const uint32_t s2 = __reduce_add_sync(0xffffffffu, c_tost), s3 = __reduce_add_sync(0xffffffffu, c_rem);
  if ((threadIdx.x & 31) == 0) {
    if (s0) atomicAdd(a.counts + 0, s0);
    if (s1) atomicAdd(a.counts + 1, s1);
    if (s2) atomicAdd(a.counts + 2, s2);
    if (s3) atomicAdd(a.counts + 3, s3);
  }
}

cudaError_t launch_fuse(const rtgs_params& p, const int32_t* gid_of_slot, int n_slots, const float* before,
                        const uint32_t* eta_before, const uint32_t* eta, cudaStream_t s) {
  if (n_slots == 0) return cudaSuccess;
  FuseArgs a;
  a.pos = p.pos; a.log_scale = p.log_scale; a.rot = p.rot; a.sh = p.sh;
  a.gid_of_slot = gid_of_slot; a.n_slots = n_slots; a.before = before; a.eta_before = eta_before; a.eta = eta;
  const int per = kFuseThreads / kFuseLanes;
  const int blocks = (n_slots + per - 1) / per;
  switch ((p.sh_degree + 1) * (p.sh_degree + 1)) {
    case 1: k_fuse<1><<<blocks, kFuseThreads, 0, s>>>(a); break;
    case 4: k_fuse<4><<<blocks, kFuseThreads, 0, s>>>(a); break;
    case 9: k_fuse<9><<<blocks, kFuseThreads, 0, s>>>(a); break;
    default: k_fuse<16><<<blocks, kFuseThreads, 0, s>>>(a); break;
  }
  note_launch();
  return cudaGetLastError();
}

size_t state_workspace_size(int n) { return ((size_t)(n > 0 ? n : 1) + 255) / 256 * 256; }

cudaError_t launch_manage_states(const rtgs_render_out& full, const rtgs_frame& frame, const rtgs_camera& cam,
                                 uint8_t* flags, uint32_t* err, uint32_t* eta, uint32_t* tc, int n,
                                 const rtgs_state_params& sp, uint32_t* counts, void* ws, cudaStream_t s) {
  uint8_t* mark = static_cast<uint8_t*>(ws);
  cudaMemsetAsync(counts, 0, 4 * sizeof(uint32_t), s);
  if (n > 0) cudaMemsetAsync(mark, 0, (size_t)n, s);
  const int HW = cam.width * cam.height;
  MarkArgs m;
  m.chat = full.color; m.dhat = full.depth; m.index = full.index; m.c = frame.color; m.d = frame.depth;
  m.flags = flags; m.HW = HW; m.dc = sp.delta_c; m.dd = sp.delta_d; m.mark = mark;
  k_mark<<<(HW + 255) / 256, 256, 0, s>>>(m);
  note_launch();
  if (n > 0) {
    TransArgs t;
    t.flags = flags; t.err = err; t.eta = eta; t.tc = tc; t.mark = mark; t.n = n;
    t.de = sp.delta_e; t.deta = sp.delta_eta; t.dt = sp.delta_t; t.k = sp.frame_idx; t.counts = counts;
    k_transition<<<(n + 255) / 256, 256, 0, s>>>(t);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace rtgs
