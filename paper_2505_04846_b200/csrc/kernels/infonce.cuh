// infonce.cuh -- step a11: row-logsumexp InfoNCE over the in-batch MaxSim score matrix.
//
//   z_ij = S_ij / tau;  l_i = logsumexp_j z_ij - z_{i,pos_i};  L = (1/B) sum_i l_i
// ("L_LI is maxsim loss", §3.2.1; SPEC.md:339-347 li_loss; tau: DESIGN.md R9).
// Evaluated in fp32 as  M = max_j z_ij,  r = sum_{j != pos} exp(z_ij - M),
//   l_i = log1p(r)                               if M == z_pos   (positive is a maximum)
//   l_i = (M - z_pos) + log(exp(z_pos - M) + r)   otherwise
// (R13: the log1p form keeps full relative precision when the positive dominates and the
// loss is tiny).  Reductions use a fixed order (lane-strided partials, butterfly shuffles, warps
// summed in index order in fp64) -> deterministic, no float atomics.
#pragma once
#include <cstdint>

namespace hiper {

// l_i of one row (one warp; fixed-order lane partials and butterflies).
__device__ __forceinline__ float infonce_row(const float* __restrict__ row, int32_t M, int32_t p,
                                             float tau, uint32_t lane) {
  float mx = -INFINITY;
  for (int32_t j = lane; j < M; j += 32) mx = fmaxf(mx, __fdiv_rn(row[j], tau));
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const float zp = __fdiv_rn(row[p], tau);
  float r = 0.0f;
  for (int32_t j = lane; j < M; j += 32)
    if (j != p) r += expf(__fdiv_rn(row[j], tau) - mx);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return (mx == zp) ? log1pf(r) : (mx - zp) + logf(expf(zp - mx) + r);
}

// dL_LI/dS_ij of one row (N1): G_ij = (softmax_j(S_i / tau) - [j == p]) / (B tau), the softmax over
// all j with the same fixed-order lane partials (written by the loss kernel's warp for its row).
__device__ __forceinline__ void infonce_row_grad(const float* __restrict__ row, int32_t B, int32_t M,
                                                 int32_t p, float tau, uint32_t lane,
                                                 float* __restrict__ g) {
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
    g[j] = (pj - (j == p ? 1.0f : 0.0f)) * scale;
  }
}

// Row-parallel form (the ColTrast step): one warp per row over ceil(B/8) blocks; each row's l_i goes to
// rowloss[i]; the last block to finish (completion counter, zeroed by the caller, reset here) sums
// rowloss in index order in fp64 -> L.  Deterministic: the order depends on nothing but B.
__global__ void __launch_bounds__(256) infonce_rows_kernel(const float* __restrict__ S, int32_t B,
                                                           int32_t M, int64_t ld,
                                                           const int32_t* __restrict__ pos, float tau,
                                                           double* __restrict__ rowloss,
                                                           uint32_t* counter, float* __restrict__ out_loss,
                                                           float* __restrict__ G = nullptr) {
  __shared__ double part[256];
  __shared__ bool last;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: S is the previous kernel's output
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t i = (int32_t)blockIdx.x * 8 + (int32_t)warp;
  if (i < B) {
    const int32_t p = pos ? pos[i] : i;
    const float li = infonce_row(S + (int64_t)i * ld, M, p, tau, lane);
    if (lane == 0) rowloss[i] = (double)li;
    if (G != nullptr) infonce_row_grad(S + (int64_t)i * ld, B, M, p, tau, lane, G + (int64_t)i * M);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a = 0.0;
  for (int32_t r = threadIdx.x; r < B; r += blockDim.x) a += __ldcg(rowloss + r);
  part[threadIdx.x] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (uint32_t w = 0; w < blockDim.x; ++w) t += part[w];
    *out_loss = (float)(t / (double)B);
    *counter = 0u;
  }
}

__global__ void __launch_bounds__(1024) infonce_loss_kernel(const float* __restrict__ S, int32_t B,
                                                            int32_t M, int64_t ld,
                                                            const int32_t* __restrict__ pos,
                                                            float tau, float* __restrict__ out_loss,
                                                            const float* combine_with = nullptr,
                                                            float* out_combined = nullptr) {
  __shared__ double warp_sum[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t n_warps = blockDim.x >> 5;
  double acc = 0.0;
  for (int32_t i = warp; i < B; i += n_warps) {
    acc += (double)infonce_row(S + (int64_t)i * ld, M, pos ? pos[i] : i, tau, lane);
  }
  if (lane == 0) warp_sum[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (uint32_t w = 0; w < n_warps; ++w) s += warp_sum[w];
    const float L = (float)(s / (double)B);
    *out_loss = L;
    // ColTrast total loss L = (L_LI + L_C) / 2, when the other term is given
    if (out_combined) *out_combined = 0.5f * (*combine_with + L);
  }
}

}  // namespace hiper
