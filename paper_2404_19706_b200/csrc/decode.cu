// decode.cu — sensor-native RGB-D frames to the planar float32 frames of the mapping path
// (P:232 input pre-processing): interleaved 8-bit RGB -> C = rgb / 255 as [3][H][W], 16-bit depth in
// raw units -> D = raw / depth_scale metres (raw 0 = no measurement -> 0, invalid by R24).
// 4 pixels per thread: one 12-byte RGB and one 8-byte depth load, planar float4 stores.
#include "common.cuh"
#include "internal.h"

namespace rtgs {

__global__ void __launch_bounds__(256) k_decode(const uint8_t* __restrict__ rgb, const uint16_t* __restrict__ raw,
                                                int HW, float inv255, float inv_scale, float* __restrict__ color,
                                                float* __restrict__ depth) {
  const int q = blockIdx.x * 256 + threadIdx.x;  // quad of pixels
  const int p0 = 4 * q;
  if (p0 >= HW) return;
  if (p0 + 4 <= HW) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(rgb + 12 * (size_t)q);
    const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
    const uint8_t b[12] = {(uint8_t)w0, (uint8_t)(w0 >> 8), (uint8_t)(w0 >> 16), (uint8_t)(w0 >> 24),
                           (uint8_t)w1, (uint8_t)(w1 >> 8), (uint8_t)(w1 >> 16), (uint8_t)(w1 >> 24),
                           (uint8_t)w2, (uint8_t)(w2 >> 8), (uint8_t)(w2 >> 16), (uint8_t)(w2 >> 24)};
    const uint2 d2 = *reinterpret_cast<const uint2*>(raw + p0);
    const uint16_t d[4] = {(uint16_t)d2.x, (uint16_t)(d2.x >> 16), (uint16_t)d2.y, (uint16_t)(d2.y >> 16)};
    for (int c = 0; c < 3; ++c) {
      const float4 v = make_float4(__fmul_rn((float)b[c], inv255), __fmul_rn((float)b[3 + c], inv255),
                                   __fmul_rn((float)b[6 + c], inv255), __fmul_rn((float)b[9 + c], inv255));
      float* o = color + (size_t)c * HW + p0;
      if ((HW & 3) == 0) {  // planes start 16-byte aligned
        *reinterpret_cast<float4*>(o) = v;
      } else {
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
      }
    }
    *reinterpret_cast<float4*>(depth + p0) =
        make_float4(__fmul_rn((float)d[0], inv_scale), __fmul_rn((float)d[1], inv_scale),
                    __fmul_rn((float)d[2], inv_scale), __fmul_rn((float)d[3], inv_scale));
  } else {
    for (int p = p0; p < HW; ++p) {
      for (int c = 0; c < 3; ++c) color[(size_t)c * HW + p] = __fmul_rn((float)rgb[3 * (size_t)p + c], inv255);
      depth[p] = __fmul_rn((float)raw[p], inv_scale);
    }
  }
}

cudaError_t launch_decode(const uint8_t* rgb, const uint16_t* raw, int W, int H, float depth_scale, float* color,
                          float* depth, cudaStream_t s) {
  const int HW = W * H;
  if (HW == 0) return cudaSuccess;
  const int quads = (HW + 3) / 4;
  k_decode<<<(quads + 255) / 256, 256, 0, s>>>(rgb, raw, HW, 1.0f / 255.0f, 1.0f / depth_scale, color, depth);
  note_launch();
  return cudaGetLastError();
}

}  // namespace rtgs
