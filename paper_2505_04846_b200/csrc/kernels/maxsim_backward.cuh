// maxsim_backward.cuh -- NEXT N1: gradient of the ColTrast late-interaction loss L_LI.
//
// Chain rule (the objective is trained by backpropagation):
//   G_ij          = (softmax_j(S_i / tau)_j - [j == pos_i]) / (B tau)            infonce_grad_kernel
//   a(i,t,j)      = argmax_{u < len_j} <qn_{i,t}, dn_{j,u}>  (saved by the forward, MODE 2)
//   g_q(i,t)      = sum_j G_ij dn_{j, a(i,t,j)}                                   grad_q_kernel
//   g_d(j,u)      = sum_i sum_{t: a(i,t,j) = u} G_ij qn_{i,t}                      grad_d_kernel
//   dL/dx (row)   = inv (g - y (y . g)),  y = x inv, inv = 1 / ||x||   (NORM's Jacobian; skipped
//                   with HIPER_ASSUME_NORMALIZED)
// qn / dn are the bf16 NORM'd operands of the forward (the kernels' layouts); the Jacobian uses the
// fp32 y = x * inv of the raw row.  All sums run in a fixed order (deterministic, no atomics).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace hiper {

__global__ void __launch_bounds__(256) infonce_grad_kernel(const float* __restrict__ S, int32_t B,
                                                           int32_t M, int64_t ld,
                                                           const int32_t* __restrict__ pos,
                                                           float tau, float* __restrict__ G) {
  const uint32_t lane = threadIdx.x & 31;
  const int32_t i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= B) return;
  const float* row = S + (int64_t)i * ld;
  const int32_t p = pos ? pos[i] : i;
  float mx = -INFINITY;
  for (int32_t j = lane; j < M; j += 32) mx = fmaxf(mx, __fdiv_rn(row[j], tau));
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.0f;
  for (int32_t j = lane; j < M; j += 32) sum += expf(__fdiv_rn(row[j], tau) - mx);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float scale = 1.0f / ((float)B * tau);
  for (int32_t j = lane; j < M; j += 32) {
    const float pj = expf(__fdiv_rn(row[j], tau) - mx) / sum;
    G[(int64_t)i * M + j] = (pj - (j == p ? 1.0f : 0.0f)) * scale;
  }
}

template <typename Tin>
__device__ __forceinline__ float load_raw(const Tin* p);
template <>
__device__ __forceinline__ float load_raw<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float load_raw<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

// Jacobian of NORM for one row held as VPL values per lane (dims lane*VPL .. lane*VPL+VPL-1).
template <int VPL, typename Tin>
__device__ __forceinline__ void norm_backward_row(const Tin* xrow, const float (&g)[VPL],
                                                  bool assume_normalized, float* out, uint32_t lane) {
  if (assume_normalized) {
#pragma unroll
    for (int v = 0; v < VPL; ++v) out[lane * VPL + v] = g[v];
    return;
  }
  float x[VPL], ss = 0.0f;
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    x[v] = load_raw<Tin>(xrow + lane * VPL + v);
    ss = fmaf(x[v], x[v], ss);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = 1.0f / sqrtf(ss);
  float yg = 0.0f;
#pragma unroll
  for (int v = 0; v < VPL; ++v) yg = fmaf(x[v] * inv, g[v], yg);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) yg += __shfl_xor_sync(0xffffffffu, yg, o);
#pragma unroll
  for (int v = 0; v < VPL; ++v) out[lane * VPL + v] = inv * (g[v] - x[v] * inv * yg);
}

// One warp per (query i, query token t); lanes own VPL = dim/32 consecutive dims.
template <int VPL, typename Tin>
__global__ void __launch_bounds__(256) grad_q_kernel(const float* __restrict__ G,
                                                     const uint8_t* __restrict__ amax, int32_t B,
                                                     int32_t M, const __nv_bfloat16* __restrict__ dlay,
                                                     int32_t ld_pad, const Tin* __restrict__ xq,
                                                     int32_t q_max_len, const int32_t* __restrict__ q_lens,
                                                     uint32_t assume_normalized,
                                                     float* __restrict__ grad_q) {
  constexpr int D = VPL * 32;
  const uint32_t lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= (int64_t)B * q_max_len) return;
  const int32_t i = (int32_t)(row / q_max_len), t = (int32_t)(row % q_max_len);
  float* out = grad_q + row * D;
  if (t >= q_lens[i]) {
#pragma unroll
    for (int v = 0; v < VPL; ++v) out[lane * VPL + v] = 0.0f;
    return;
  }
  float g[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) g[v] = 0.0f;
  for (int32_t j = 0; j < M; ++j) {
    const float gij = G[(int64_t)i * M + j];
    const int32_t u = amax[((int64_t)i * M + j) * 32 + t];
    const __nv_bfloat16* dr = dlay + ((int64_t)j * ld_pad + u) * D + lane * VPL;
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[v] = fmaf(gij, __bfloat162float(dr[v]), g[v]);
  }
  norm_backward_row<VPL, Tin>(xq + row * D, g, assume_normalized != 0, out, lane);
}

// One block per doc j: SMEM accumulator [ld_pad][D] fp32, thread = one dim, then one warp per row
// for the Jacobian.  Blocks of D threads (64 or 128).
template <int VPL, typename Tin>
__global__ void __launch_bounds__(128) grad_d_kernel(const float* __restrict__ G,
                                                     const uint8_t* __restrict__ amax, int32_t B,
                                                     int32_t M, const __nv_bfloat16* __restrict__ qlay,
                                                     const int32_t* __restrict__ q_lens,
                                                     int32_t ld_pad, const Tin* __restrict__ xd,
                                                     int32_t d_max_len, const int32_t* __restrict__ d_lens,
                                                     uint32_t assume_normalized,
                                                     float* __restrict__ grad_d) {
  constexpr int D = VPL * 32;
  extern __shared__ float acc[];  // [ld_pad][D]
  const int32_t j = blockIdx.x;
  const uint32_t tid = threadIdx.x;  // dim (blockDim.x == D)
  const int32_t lj = d_lens[j];
  for (int32_t u = 0; u < lj; ++u) acc[u * D + tid] = 0.0f;
  __syncthreads();
  for (int32_t i = 0; i < B; ++i) {
    const float gij = G[(int64_t)i * M + j];
    const uint8_t* am = amax + ((int64_t)i * M + j) * 32;
    const __nv_bfloat16* qr = qlay + (int64_t)i * 32 * D;
    const int32_t lq = q_lens[i];
    for (int32_t t = 0; t < lq; ++t) {
      const int32_t u = am[t];
      acc[u * D + tid] = fmaf(gij, __bfloat162float(qr[t * D + tid]), acc[u * D + tid]);
    }
  }
  __syncthreads();
  const uint32_t lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int32_t u = warp; u < d_max_len; u += nw) {
    float* out = grad_d + ((int64_t)j * d_max_len + u) * D;
    if (u >= lj) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) out[lane * VPL + v] = 0.0f;
      continue;
    }
    float g[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) g[v] = acc[u * D + lane * VPL + v];
    norm_backward_row<VPL, Tin>(xd + ((int64_t)j * d_max_len + u) * D, g, assume_normalized != 0,
                                out, lane);
  }
}

}  // namespace hiper
