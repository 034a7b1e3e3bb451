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
    const float* row = S + (int64_t)i * ld;
    const int32_t p = pos ? pos[i] : i;
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
    const float li = (mx == zp) ? log1pf(r) : (mx - zp) + logf(expf(zp - mx) + r);
    acc += (double)li;
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
